"""Is a config's eager step host-bound?  Host enqueue time of one step (the GPU
is first held by a sleep kernel, so nothing the host waits on has run yet) vs
the step's device time.  python tools/host_vs_gpu.py [config] [--stock]"""
import sys
import time
import torch
sys.path.insert(0, ".")
from benchkit import models as BM  # noqa: E402
from paper_2404_12406_b200.nn import convert_to_memory_saving  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "bert"
stock = "--stock" in sys.argv
dev = torch.device("cuda", 0)
wl = BM.WORKLOADS[cfg]()
if not stock:
    wl.model = convert_to_memory_saving(wl.model, fuse=True)
ins = list(wl.make_batch(wl.batch, dev))


def step():
    for p in wl.model.parameters():
        p.grad = None
    wl.loss_fn(wl.model, *ins).backward()


for _ in range(3):
    step()
torch.cuda.synchronize()
for _ in range(3):
    torch.cuda._sleep(int(1.9e9 * 0.2))  # hold the GPU 200 ms
    t0 = time.perf_counter()
    step()
    host = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    step()
    e.record()
    torch.cuda.synchronize()
    print(f"{cfg} {'stock' if stock else 'memsave'}: host enqueue {host:.2f} ms, device step "
          f"{s.elapsed_time(e):.2f} ms", flush=True)
