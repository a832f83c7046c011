#!/usr/bin/env python
"""Benchmark: fwd+bwd throughput and peak memory of the selective-save layers
on B200 vs stock PyTorch (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W --config resnet18|fig1]
    python bench.py --impl reference ...   # the reference's CPU algorithm, host cores

Default workload = BASELINE.json configs[1]: ResNet-18, frozen weights,
input-only gradient, batch 256x3x224x224 bf16, channels_last, eval-mode BN.
A "step" = forward + cross-entropy + backward to the input (x.grad).  With N
GPUs (torchrun) every rank runs the full per-GPU batch (weak scaling); the
input-only workload has no trainable parameter, so the ranks are replicas and
no collective runs in the data path.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "peak fwd+bwd memory (MiB) and fwd+bwd samples/sec vs PyTorch, at 1/2/4/8 B200"


def _peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written), else the
    profiling recipe's fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"gbs": float(d["hbm_gbs"]), "tflops": float(d["bf16_tflops"]),
                "tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"gbs": 6650.0, "tflops": 1590.0, "tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.lines = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ ncu traffic
# dram__bytes_read.sum + dram__bytes_write.sum per launch of the step's top conv
# kernels, from one `ncu --set full` capture each (tools/ncu_summary.py output,
# committed under profiles/); keyed by (pass, C, R, stride) of the ResNet-18 shapes
_NCU_CSV = os.path.join(ROOT, "profiles", "r1_ncu_r18_kernels.csv")
_NCU_NAME = {("conv_fwd", 3, 7, 2): "stem_fwd", ("conv_dx", 3, 7, 2): "stem_dx",
             ("conv_fwd", 64, 3, 1): "layer1_fwd", ("conv_dx", 64, 3, 1): "layer1_dgrad"}
_KERNEL_OF = {("conv_fwd", 3, 7, 2): "stem_fprop_kernel",
              ("conv_dx", 3, 7, 2): "stem_dgrad_kernel",
              ("conv_fwd", 64, 3, 1): "conv3x3_halo_kernel",
              ("conv_dx", 64, 3, 1): "conv3x3_halo_kernel (transposed)"}


def _kernel_key(e):
    g = e["geom"]
    return (e["kind"], g["c"], g["r"], g["stride"])


def _ncu_traffic(e):
    name = _NCU_NAME.get(_kernel_key(e))
    if name is None or not os.path.exists(_NCU_CSV):
        return None, None
    import csv
    vals = {}
    with open(_NCU_CSV) as f:
        for row in csv.DictReader(f):
            if row["kernel"] == name and row["metric"] in ("dram__bytes_read.sum",
                                                           "dram__bytes_write.sum"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(row["unit"], 1)
                vals[row["metric"]] = float(row["value"]) * scale
    if len(vals) != 2:
        return None, None
    return int(sum(vals.values())), f"{os.path.relpath(_NCU_CSV, ROOT)}:{name}"


# ------------------------------------------------------------------ GPU arm
def _dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif world == 1:
        torch.cuda.set_device(local)
    return world, rank, local


def _barrier(world):
    import torch.distributed as dist
    if world > 1:
        dist.barrier()


def _max_over_ranks(v: float, world: int) -> float:
    import torch
    import torch.distributed as dist
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def prime(wl, model, dev, sync=None):
    """Setup, not a step: one fwd+bwd at batch 2 so every kernel image is loaded
    (lazy module loading) and one-time host state exists before warm-up."""
    import torch
    ins = list(wl.make_batch(min(2, wl.batch), dev))
    if wl.input_requires_grad:
        ins[0].requires_grad_(True)
    wl.loss_fn(model, *ins).backward()
    if sync is not None:  # the gradient hooks fired: complete their collectives
        sync.finish()
    for p in model.parameters():
        p.grad = None
    torch.cuda.synchronize(dev)


def run_arm(wl, model, batch_inputs, steps, warmup, world, dev, sync=None):
    """Time `steps` fwd+bwd steps (device time, CUDA events, max over ranks)."""
    import torch

    x = batch_inputs[0]
    prime(wl, model, dev, sync)

    def step():
        if wl.input_requires_grad:
            x.grad = None
        for p in model.parameters():
            p.grad = None
        loss = wl.loss_fn(model, *batch_inputs)
        loss.backward()
        if sync is not None:
            sync.finish()
        return loss

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    _barrier(world)
    torch.cuda.synchronize(dev)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(steps):
        step()
    end.record()
    torch.cuda.synchronize(dev)
    _barrier(world)
    ms = start.elapsed_time(end)
    return _max_over_ranks(ms, world), step


def peak_memory(step, dev):
    import torch
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    base = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    step()
    torch.cuda.synchronize(dev)
    peak = torch.cuda.max_memory_allocated(dev)
    return peak / 2**20, (peak - base) / 2**20


def e2e_arm(wl, model, steps, warmup, world, dev, sync=None):
    """Same step through the public API, inputs copied from pinned host memory
    and the loss read back every step (H2D/D2H inside the timed region).  The
    H2D copy of step i+1 runs on a copy stream while step i computes (two device
    input buffers), as a training loop with pinned, non-blocking loads does."""
    import torch

    bufs = [list(wl.make_batch(wl.batch, dev)) for _ in range(2)]
    host = [t.detach().cpu().pin_memory() for t in bufs[0]]
    loss_host = torch.empty((), dtype=torch.float32).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in host)
    d2h = loss_host.numel() * loss_host.element_size()
    copy_stream = torch.cuda.Stream(dev)
    ready = [torch.cuda.Event(), torch.cuda.Event()]
    free = [torch.cuda.Event(), torch.cuda.Event()]
    main = torch.cuda.current_stream(dev)

    def load(i):  # H2D of step i's inputs into buffer i % 2, on the copy stream
        b = i % 2
        copy_stream.wait_event(free[b])  # step i-2 has finished reading the buffer
        with torch.cuda.stream(copy_stream), torch.no_grad():
            for d, h in zip(bufs[b], host):
                d.copy_(h, non_blocking=True)
        ready[b].record(copy_stream)

    def step(i, last):
        b = i % 2
        main.wait_event(ready[b])
        if not last:
            load(i + 1)
        inputs = bufs[b]
        x = inputs[0]
        if wl.input_requires_grad:
            x.requires_grad_(True)
            x.grad = None
        for p in model.parameters():
            p.grad = None
        loss = wl.loss_fn(model, *inputs)
        loss.backward()
        if sync is not None:
            sync.finish()
        if wl.input_requires_grad:
            x.grad = None
            x.requires_grad_(False)
        free[b].record(main)
        loss_host.copy_(loss.detach(), non_blocking=True)
        return loss

    for r in range(2):
        free[r].record(main)
    load(0)
    for i in range(warmup):
        step(i, last=False)
    torch.cuda.synchronize(dev)
    _barrier(world)
    torch.cuda.synchronize(dev)
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    load(0)  # the first timed step's inputs are copied inside the timed region
    for i in range(steps):
        step(i, last=(i == steps - 1))
    e.record()
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - t0
    ms = _max_over_ranks(s.elapsed_time(e), world)
    return ms, wall, h2d, d2h


def gpu_main(args):
    import torch

    import paper_2404_12406_b200 as pkg
    from benchkit import kernels as KB
    from benchkit import models as BM
    from paper_2404_12406_b200.distributed import TrainableGradAllReduce
    from paper_2404_12406_b200.nn import convert_to_memory_saving

    world, rank, local = _dist_setup(args)
    dev = torch.device("cuda", local)
    peaks = _peaks()
    pkg.lib()  # fail loudly if the native library is missing

    builder = BM.WORKLOADS[args.config]

    def fresh():
        """A new copy of the seeded workload (identical weights): only one model is
        resident at a time, so every arm's peak is its own."""
        return builder(batch=args.batch) if args.batch else builder()

    # ---------------- memsave arm (the product): every supported layer swapped,
    # conv -> BN(eval) -> ReLU, conv -> ReLU and residual joins fused by the fx pass
    wl = fresh()
    wl.model = convert_to_memory_saving(wl.model, fuse=not args.no_fuse)
    inputs = list(wl.make_batch(wl.batch, dev))
    if wl.input_requires_grad:
        inputs[0].requires_grad_(True)
    sync = TrainableGradAllReduce(wl.model) if world > 1 else None
    n0 = pkg.launch_count()
    fam0 = pkg.launch_stats()
    with ClockSampler(local) as clocks:
        ms, step = run_arm(wl, wl.model, inputs, args.steps, args.warmup, world, dev, sync)
    launches = pkg.launch_count() - n0
    fam1 = pkg.launch_stats()
    # launches of the warm-up steps are included above; count one clean step too
    n1 = pkg.launch_count()
    step()
    torch.cuda.synchronize(dev)
    per_step_launches = pkg.launch_count() - n1
    peak_mib, act_peak_mib = peak_memory(step, dev)
    del step
    inputs.clear()
    torch.cuda.empty_cache()
    e2e_ms, e2e_wall, h2d, d2h = e2e_arm(wl, wl.model, args.steps, max(1, args.warmup // 2),
                                         world, dev, sync)

    samples = wl.batch * args.steps * world
    value = samples / (ms / 1e3)
    e2e_value = samples / (e2e_ms / 1e3)
    wl.model = sync = None
    torch.cuda.empty_cache()

    def other_arm(convert_kwargs):
        """(ms, peak MiB, activation peak MiB) of a fresh model, converted with
        convert_kwargs (None = stock)."""
        w2 = fresh()
        if convert_kwargs is not None:
            w2.model = convert_to_memory_saving(w2.model, **convert_kwargs)
        ins = list(w2.make_batch(w2.batch, dev))
        if w2.input_requires_grad:
            ins[0].requires_grad_(True)
        sy = TrainableGradAllReduce(w2.model) if world > 1 else None
        ams, astep = run_arm(w2, w2.model, ins, args.steps, args.warmup, world, dev, sy)
        apeak, aact = peak_memory(astep, dev)
        del astep, ins, w2, sy
        torch.cuda.empty_cache()
        return ams, apeak, aact

    # ---------------- stock arm (same weights, unconverted) for the "vs PyTorch" part
    stock = {}
    if not args.no_stock:
        sms, speak, sact = other_arm(None)
        stock = {"value": samples / (sms / 1e3), "ms_per_step": sms / args.steps,
                 "peak_mib": speak, "activation_peak_mib": sact,
                 "impl": "torch %s stock modules (cuDNN/cuBLAS), same weights/inputs"
                         % torch.__version__}
        # the north star's layer set only (Linear / Conv2d / BatchNorm2d-eval), ReLU and
        # MaxPool2d left stock: isolates the paper's Fig. 2 effect from the §8(f) swaps
        lms, lpeak, lact = other_arm(dict(relu=False, maxpool2d=False, dropout=False,
                                          layernorm=False, conv_transpose2d=False))
        stock["memsave_layers_only"] = {
            "value": round(samples / (lms / 1e3), 2), "ms_per_step": round(lms / args.steps, 4),
            "peak_mib": round(lpeak, 1), "activation_peak_mib": round(lact, 1),
            "swaps": "Linear, Conv2d, BatchNorm2d(eval) only"}
        if not args.no_fuse:  # every layer swapped, no fx fusion
            ums, upeak, uact = other_arm(dict(fuse=False))
            stock["memsave_unfused"] = {
                "value": round(samples / (ums / 1e3), 2),
                "ms_per_step": round(ums / args.steps, 4), "peak_mib": round(upeak, 1),
                "activation_peak_mib": round(uact, 1),
                "swaps": "all supported layers, convert_to_memory_saving(fuse=False)"}

    # ---------------- roofline of the dominant kernel (rank 0)
    roof = None
    layers = []
    if rank == 0 and not args.no_roofline and args.config == "resnet18":
        for (n, c, h, w, k, r, s, p, cnt) in BM.resnet18_conv_shapes(wl.batch):
            for ent in KB.conv_roofline(n, c, h, w, k, r, s, p, dev, peaks, reps=5):
                ent["count_per_step"] = cnt
                layers.append(ent)
        # the same (pass, geometry) appears once per position in the network
        tot = {}
        for e in layers:
            key = (e["kind"], tuple(sorted(e["geom"].items())))
            tot[key] = tot.get(key, 0.0) + e["ms"] * e["count_per_step"]
        dom = max(layers, key=lambda e: tot[(e["kind"], tuple(sorted(e["geom"].items())))])
        dom = dict(dom, count_per_step=sum(
            x["count_per_step"] for x in layers
            if (x["kind"], x["geom"]) == (dom["kind"], dom["geom"])))
        traffic, tsrc = _ncu_traffic(dom)
        roof = {"bound": dom["bound"], "achieved": round(dom["achieved"], 2),
                "peak": dom["peak"], "unit": dom["unit"], "frac": round(dom["frac"], 4),
                "traffic": traffic, "traffic_source": tsrc,
                "algorithmic_bytes": dom["bytes"], "algorithmic_flops": dom["flops"],
                "kernel": "%s (%s)" % (_KERNEL_OF.get(_kernel_key(dom), "umma_gemm_kernel"),
                                       dom["kind"]),
                "geom": dom["geom"], "launch_ms": round(dom["ms"], 4),
                "launches_per_step": dom["count_per_step"],
                "per_unit": "2*N*OH*OW*K*C*R*S flops per launch (implicit GEMM)",
                "peak_source": peaks["source"] + ", burst (kernel timed alone)"}
        total_conv_ms = sum(e["ms"] * e["count_per_step"] for e in layers)
        roof["conv_share_of_step"] = round(total_conv_ms / (ms / args.steps), 3)
        with open(os.path.join(ROOT, "gpurun_out" if os.path.isdir(
                os.path.join(ROOT, "gpurun_out")) else ".", "bench_layers.json"), "w") as f:
            json.dump(layers, f, indent=1)

    # ---------------- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.config, None, min_seconds=args.cpu_seconds)

    out = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "samples/s",
        "tokens_per_s": (round(value * wl.config["seq_len"], 1) if "seq_len" in wl.config
                         else None),
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": str(wl.dtype).replace("torch.", "").replace("bfloat16", "bf16"),
        "data": "synthetic (random-init weights, seeded normal inputs)",
        "config": dict(wl.config, parallelism=(f"dp{world}" if world > 1 else "single"),
                       l2="activations > 126 MB L2 (no explicit flush between steps)"),
        "peak_mib": round(peak_mib, 1),
        "activation_peak_mib": round(act_peak_mib, 1),
        "stock": {k: (round(v, 3) if isinstance(v, float) else v) for k, v in stock.items()},
        "speedup_vs_stock": (round(value / stock["value"], 3) if stock else None),
        "peak_ratio_vs_stock": (round(peak_mib / stock["peak_mib"], 3) if stock else None),
        "e2e": {"value": round(e2e_value, 2), "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms / args.steps, 4),
                "wall_s": round(e2e_wall, 3)},
        "gpu_launches": launches,
        "gpu_launches_per_step": per_step_launches,
        "launch_families_timed_region": {k: fam1[k] - fam0[k] for k in fam1},
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "impl": "memsave_b200",
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ------------------------------------------------------------------ CPU legs
def cpu_baseline(config, wl=None, min_seconds=10.0):
    """The reference algorithm (oracle port, numpy f32, all host cores) on a
    bounded sample of the same workload."""
    import numpy as np
    import torch

    from benchkit.cpu_port import ResNet18InputGradCPU, time_cpu
    cores = os.cpu_count()
    if config != "resnet18":
        return None
    if wl is None:
        from benchkit import models as BM
        wl = BM.resnet18_input_only(batch=1, dtype=torch.float32, device="cpu")
    port = ResNet18InputGradCPU(wl.model.state_dict())
    rng = np.random.default_rng(0)
    nb = 1
    x = rng.standard_normal((nb, 3, 224, 224)).astype(np.float32)
    y = rng.integers(0, 1000, nb)
    sec, calls = time_cpu(lambda: port.step(x, y), min_seconds=min_seconds)
    return {"value": round(nb / sec, 4), "unit": "samples/s", "cores": cores, "kind": "port",
            "sample": f"{calls} steps of 1 image (3x224x224) fp32: full ResNet-18 forward + "
                      f"input-gradient backward through the oracle restatement of the "
                      f"reference numpy conv (numpy_impl.py:12-38), BLAS on {cores} threads"}


def reference_main(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.config != "resnet18":
        print(json.dumps({"impl": "reference", "unavailable": f"no CPU port for {args.config}"}))
        return
    import numpy as np
    import torch

    from benchkit import models as BM
    from benchkit.cpu_port import ResNet18InputGradCPU
    wl = BM.resnet18_input_only(batch=1, dtype=torch.float32, device="cpu")
    port = ResNet18InputGradCPU(wl.model.state_dict())
    rng = np.random.default_rng(0)
    x = rng.standard_normal((1, 3, 224, 224)).astype(np.float32)
    y = rng.integers(0, 1000, 1)
    for _ in range(max(1, args.warmup)):
        port.step(x, y)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        port.step(x, y)
    sec = (time.perf_counter() - t0) / args.steps
    v = round(1.0 / sec, 4)
    cores = os.cpu_count()
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": dict(wl.config, global_batch=1,
                       note="each step is a bounded sample: 1 image of the 256-image batch"),
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "port",
                         "sample": "1 image per step, fp32, oracle restatement of the reference "
                                   "numpy conv (the reference is Python and cannot travel)"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="memsave", choices=["memsave", "reference"])
    ap.add_argument("--config", default="resnet18",
                    choices=["resnet18", "fig1", "resnet101", "vgg16", "bert", "llama"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--no-stock", action="store_true")
    ap.add_argument("--no-fuse", action="store_true",
                    help="product arm without the conv->BN->ReLU / add->ReLU fx fusion")
    ap.add_argument("--no-roofline", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "memsave":
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.impl == "reference":
        reference_main(args)
    else:
        gpu_main(args)


if __name__ == "__main__":
    main()
