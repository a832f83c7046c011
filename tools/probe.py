"""Fig. 1 / Appendix B probe sweep in the reference's CSV schema (SPEC.md
cmd_probe, :527-536; CSV header SPEC.md:540-544), planned by
paper_2404_12406_b200.planner and, on a GPU, measured on B200.

    python tools/probe.py [--layer conv2d|linear|batchnorm2d-eval] [--max-depth 12]
                          [--shape 32,8,256,256] [--measure]

peak_bytes is the measured fwd+bwd peak (torch.cuda.max_memory_allocated
above the resident model + input) with --measure, else the planned one;
planned_peak_bytes is always the planner's.  Scenarios (SPEC.md Fig. 1): all
layers differentiable, none, layers k+ (k = 4), layer k only.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch import nn  # noqa: E402

from paper_2404_12406_b200.nn import convert_to_memory_saving  # noqa: E402
from paper_2404_12406_b200.planner import CSV_HEADER, plan, plan_csv_row  # noqa: E402


def chain(kind, depth, c):
    if kind == "conv2d":
        return nn.Sequential(*[nn.Conv2d(c, c, 3, padding=1, bias=False) for _ in range(depth)])
    if kind == "linear":
        return nn.Sequential(*[nn.Linear(c, c, bias=False) for _ in range(depth)])
    if kind == "batchnorm2d-eval":
        m = nn.Sequential(*[nn.BatchNorm2d(c) for _ in range(depth)])
        return m.eval()
    raise SystemExit(f"unknown layer kind {kind}")


SCENARIOS = {"all": lambda i, k: True, "none": lambda i, k: False,
             "layers_k_plus": lambda i, k: i >= k - 1, "layer_k_only": lambda i, k: i == k - 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default="conv2d")
    ap.add_argument("--max-depth", type=int, default=12)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--shape", default="32,8,256,256")
    ap.add_argument("--measure", action="store_true")
    a = ap.parse_args()
    shape = tuple(int(v) for v in a.shape.split(","))
    if a.layer == "linear":
        shape = (shape[0] * shape[2] * shape[3], shape[1])
    c = shape[1]
    dev = "cuda" if a.measure else "cpu"
    print(CSV_HEADER + ",planned_peak_bytes")
    for depth in range(1, a.max_depth + 1):
        for scen, tr in SCENARIOS.items():
            for policy in ("naive", "memsave"):
                torch.manual_seed(0)
                m = chain(a.layer, depth, c)
                params = list(m.parameters())
                per_layer = len(params) // depth
                for i, p in enumerate(params):
                    p.requires_grad_(tr(i // per_layer, a.k))
                if policy == "memsave":
                    convert_to_memory_saving(m)
                x = torch.empty(shape)
                loss = lambda mm, x: mm(x).sum()  # noqa: E731
                pl = plan(m, [x], loss_fn=loss)
                planned = pl.peak_bytes - pl.resident_bytes
                peak, fms, bms = planned, float("nan"), float("nan")
                if a.measure and any(p.requires_grad for p in params):
                    m = m.to(dev)
                    xd = torch.randn(shape, device=dev)
                    for _ in range(2):
                        loss(m, xd).backward()
                    torch.cuda.synchronize()
                    torch.cuda.empty_cache()
                    torch.cuda.reset_peak_memory_stats()
                    base = torch.cuda.memory_allocated()
                    t0 = time.perf_counter()
                    out = loss(m, xd)
                    torch.cuda.synchronize()
                    t1 = time.perf_counter()
                    out.backward()
                    torch.cuda.synchronize()
                    t2 = time.perf_counter()
                    peak = torch.cuda.max_memory_allocated() - base
                    fms, bms = (t1 - t0) * 1e3, (t2 - t1) * 1e3
                print(plan_csv_row(f"{a.layer}_chain", a.layer, depth, scen, policy,
                                   pl.tape_bytes, peak, fms, bms) + f",{planned}", flush=True)


if __name__ == "__main__":
    main()
