"""Run selected conv launches (NHWC bf16, through the C ABI) a few times, for
ncu captures:  python tools/prof_conv.py stem_dx layer1_fwd ..."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from benchkit import kernels as KB  # noqa: E402
from bench import _peaks  # noqa: E402

SHAPES = {
    "stem": (256, 3, 224, 224, 64, 7, 2, 3),
    "layer1": (256, 64, 56, 56, 64, 3, 1, 1),
    "layer2": (256, 128, 28, 28, 128, 3, 1, 1),
    "layer3": (256, 256, 14, 14, 256, 3, 1, 1),
    "layer4": (256, 512, 7, 7, 512, 3, 1, 1),
    "down2": (256, 64, 56, 56, 128, 1, 2, 0),
    "l2s2": (256, 64, 56, 56, 128, 3, 2, 1),
    "vggc11": (128, 3, 224, 224, 64, 3, 1, 1),
    "vggc12": (128, 64, 224, 224, 64, 3, 1, 1),
}

dev = torch.device("cuda", 0)
for arg in sys.argv[1:]:
    name, ps = arg.split("_")
    n, c, h, w, k, r, s, p = SHAPES[name]
    for e in KB.conv_roofline(n, c, h, w, k, r, s, p, dev, _peaks(), reps=3, passes=(ps,)):
        print(arg, f"{e['ms']:.4f} ms", f"frac {e['frac']:.3f}", flush=True)
