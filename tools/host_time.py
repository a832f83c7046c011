"""Host (Python + dispatch) time to enqueue one fwd+bwd step vs its device time.

The GPU is held by a sleep kernel while the host enqueues the step, so the
host time excludes any waiting on the device:

    python tools/host_time.py --config resnet101 [--profile]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from benchkit import models as BM
    from paper_2404_12406_b200.nn import convert_to_memory_saving
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="resnet101")
    ap.add_argument("--stock", action="store_true")
    ap.add_argument("--no-fuse", action="store_true")
    ap.add_argument("--profile", action="store_true")
    args = ap.parse_args()
    wl = BM.WORKLOADS[args.config]()
    model = wl.model if args.stock else convert_to_memory_saving(wl.model, fuse=not args.no_fuse)
    dev = torch.device("cuda")
    ins = list(wl.make_batch(wl.batch, dev))
    if wl.input_requires_grad:
        ins[0].requires_grad_(True)

    def step():
        for p in model.parameters():
            p.grad = None
        wl.loss_fn(model, *ins).backward()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        step()
    e.record()
    torch.cuda.synchronize()
    dev_ms = s.elapsed_time(e) / 5
    host = []
    for _ in range(5):
        torch.cuda._sleep(int(1.9e9 * 0.2))  # ~200 ms of GPU sleep
        t0 = time.perf_counter()
        step()
        host.append((time.perf_counter() - t0) * 1e3)
        torch.cuda.synchronize()
    print(f"{args.config} {'stock' if args.stock else 'memsave'}: device {dev_ms:.2f} ms/step, "
          f"host enqueue {min(host):.2f} ms/step (min of 5)")
    if args.profile:
        import cProfile
        import pstats
        torch.cuda._sleep(int(1.9e9 * 0.5))
        pr = cProfile.Profile()
        pr.enable()
        step()
        pr.disable()
        torch.cuda.synchronize()
        pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
