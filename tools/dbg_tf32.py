"""Debug: run one pass of the Fig.1 fp32 conv (fwd | dx | dw) at a shape."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2404_12406_b200 import functional as MF

which, n, h, w = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
dev = "cuda"
torch.manual_seed(0)
x = torch.randn((n, 8, h, w), device=dev)
wt = torch.randn((8, 8, 3, 3), device=dev) / 24
g = torch.randn((n, 8, h, w), device=dev)
if which == "fwd":
    y = MF.conv2d(x, wt, None, 1, 1)
    ref = torch.nn.functional.conv2d(x.double(), wt.double(), None, 1, 1)
elif which == "dx":
    x.requires_grad_(True)
    y = MF.conv2d(x, wt, None, 1, 1)
    y.backward(g)
    y = x.grad
    ref = torch.nn.grad.conv2d_input(x.shape, wt.double(), g.double(), 1, 1)
else:
    wt.requires_grad_(True)
    y = MF.conv2d(x, wt, None, 1, 1)
    y.backward(g)
    y = wt.grad
    ref = torch.nn.grad.conv2d_weight(x.double(), wt.shape, g.double(), 1, 1)
torch.cuda.synchronize()
err = ((y.double() - ref).norm() / ref.norm()).item()
print(which, (n, h, w), "rel err", err)
