"""Run W warm-up + K fwd+bwd steps of one bench workload (memsave arm only),
for ncu launch lists:  ncu --metrics gpu__time_duration.sum --clock-control none
--csv --log-file gpurun_out/launches.csv python tools/prof_step.py --config resnet18
Launches of the warm-up steps are bracketed by cudaProfilerStart/Stop so
`--profile-from-start off` captures only the K timed steps."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from benchkit import models as BM  # noqa: E402
from paper_2404_12406_b200.nn import convert_to_memory_saving  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="resnet18")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--stock", action="store_true")
ap.add_argument("--no-fuse", action="store_true")
ap.add_argument("--mark", default="", help="memsave op whose calls get an NVTX range "
                "'dominant' (ncu --nvtx --nvtx-include 'dominant/')")
ap.add_argument("--mark-geom", default="", help="JSON geometry the marked call must match "
                "(benchkit.roofline.work_of)")
a = ap.parse_args()

dev = torch.device("cuda", 0)
builder = BM.WORKLOADS[a.config]
wl = builder(batch=a.batch) if a.batch else builder()
if not a.stock:
    wl.model = convert_to_memory_saving(wl.model, fuse=not a.no_fuse)
inputs = list(wl.make_batch(wl.batch, dev))
if wl.input_requires_grad:
    inputs[0].requires_grad_(True)


def step():
    if wl.input_requires_grad:
        inputs[0].grad = None
    for p in wl.model.parameters():
        p.grad = None
    wl.loss_fn(wl.model, *inputs).backward()


for _ in range(a.warmup):
    step()
torch.cuda.synchronize()
if a.mark:
    # an NVTX range around every call of the marked memsave op with the given
    # geometry, whether Python calls it or a C++ autograd node dispatches it
    # (memsave::linear's backward): a dispatch mode active for the whole step
    import json

    from torch.utils._python_dispatch import TorchDispatchMode

    from benchkit.roofline import work_of
    want = json.loads(a.mark_geom) if a.mark_geom else None

    class _Marker(TorchDispatchMode):
        def __torch_dispatch__(self, func, types, args=(), kwargs=None):
            kwargs = kwargs or {}
            hit = (func.namespace == "memsave" and func._opname == a.mark
                   and (want is None or work_of(func._opname, args)[2] == want))
            if hit:
                torch.cuda.nvtx.range_push("dominant")
            out = func(*args, **kwargs)
            if hit:
                torch.cuda.nvtx.range_pop()
            return out

    _mode = _Marker()
    _step = step

    def step():  # noqa: F811
        with _mode:
            _step()
torch.cuda.cudart().cudaProfilerStart()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.steps):
    step()
e.record()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(f"{a.config}: {s.elapsed_time(e) / a.steps:.3f} ms/step (batch {wl.batch})")
