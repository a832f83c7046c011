#!/usr/bin/env python
"""Benchmark: fwd+bwd throughput and peak memory of the selective-save layers
on B200 vs stock PyTorch (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--config bert|resnet18|resnet101|vgg16|fig1|llama]
                    [--gpus N --steps K --warmup W]
    python bench.py --impl reference ...   # the reference's CPU algorithm, host cores

Default workload: the largest single-GPU configuration of BASELINE.json,
configs[3] BERT-base (random init, attention Linear biases + classifier
trainable, train mode with dropout 0.1), batch 64 x seq 512, bf16.  A "step" =
forward + cross-entropy + backward (+ the data-parallel gradient exchange when
N > 1).  Scaling follows SURVEY.md §8(d): the CNN and BERT configs split the
global batch over the N ranks (strong scaling); Llama keeps 2 sequences per GPU
(weak scaling).  With N > 1 (torchrun, or self-spawned by --gpus N) the
trainable-subset gradients are all-reduced over NCCL (TrainableGradAllReduce);
the stock arm uses DistributedDataParallel on the same requires_grad set.

CNN configs run the step as a CUDA graph (paper_2404_12406_b200.graphs): every
memsave op is a graph-capturable custom op, so the launch-bound steps (ResNet-101:
~650 launches) replay without host work.  The stock arm is timed eager, with
cudnn.benchmark, and graphed; speedup_vs_stock is against the best of them.
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
DEFAULT_CONFIG = "bert"
# scaling per SURVEY.md §8(d); graph: the step is CUDA-graph-safe (no host RNG per step)
CONFIGS = {
    "bert": dict(scaling="strong", graph=False,
                 why_eager="dropout seeds are drawn on the host per call"),
    "resnet18": dict(scaling="strong", graph=True),
    "resnet101": dict(scaling="strong", graph=True),
    "vgg16": dict(scaling="strong", graph=True),
    "fig1": dict(scaling="strong", graph=True),
    "llama": dict(scaling="weak", graph=False,
                  why_eager="HF generation-time host logic in the model forward"),
}


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


# ------------------------------------------------------------------ distributed
def _dist_setup():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
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


def _timed(fn, steps, warmup, world, dev):
    """W untimed calls, then K timed calls bracketed by barrier + synchronize;
    device ms over the K calls (CUDA events), max over ranks."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize(dev)
    _barrier(world)
    torch.cuda.synchronize(dev)
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    torch.cuda.synchronize(dev)
    _barrier(world)
    return _max_over_ranks(s.elapsed_time(e), world)


# ------------------------------------------------------------------ one arm
class Arm:
    """A workload instance (fresh seeded model) with eager / graphed steps."""

    def __init__(self, wl, model, dev, world, sync=None, ddp=False):
        import torch
        self.wl, self.dev, self.world, self.sync = wl, dev, world, sync
        if ddp and world > 1 and any(p.requires_grad for p in model.parameters()):
            model = torch.nn.parallel.DistributedDataParallel(
                model, device_ids=[dev.index], broadcast_buffers=False)
        self.model = model
        self.params = [p for p in model.parameters() if p.requires_grad]
        self.inputs = list(wl.make_batch(wl.batch, dev))
        if wl.input_requires_grad:
            self.inputs[0].requires_grad_(True)
        self.graphed = None

    # eager step: the user-facing loop (grads reset to None, as zero_grad does)
    def step(self, inputs=None):
        inputs = self.inputs if inputs is None else inputs
        if self.wl.input_requires_grad:
            inputs[0].grad = None
        if self.sync is not None:
            self.sync.zero_grad()
        else:
            for p in self.params:
                p.grad = None
        loss = self.wl.loss_fn(self.model, *inputs)
        loss.backward()
        if self.sync is not None:
            self.sync.finish()
        return loss

    def prime(self):
        """Setup, not a step: one fwd+bwd at batch <= 2 so kernel images are
        loaded (lazy loading) and one-time host state exists."""
        import torch
        ins = list(self.wl.make_batch(min(2, self.wl.batch), self.dev))
        if self.wl.input_requires_grad:
            ins[0].requires_grad_(True)
        self.step(ins)
        torch.cuda.synchronize(self.dev)

    def capture(self, n_buffers=2):
        """CUDA graphs of the step over n_buffers static input sets."""
        from paper_2404_12406_b200.graphs import GraphedStep, zero_grads
        wl, model, params = self.wl, self.model, self.params

        def gstep(*inputs):
            zero_grads(params)
            loss = wl.loss_fn(model, *inputs)
            loss.backward()
            return loss.detach()

        bufs = [self.inputs] + [[t.detach().clone().requires_grad_(t.requires_grad)
                                 for t in self.inputs] for _ in range(n_buffers - 1)]
        self.graphed = GraphedStep(gstep, bufs)
        self._k = 0
        return self.graphed

    def replay(self):
        self._k = (self._k + 1) % len(self.graphed)
        return self.graphed.replay(self._k)


def peak_memory(fn, dev):
    import torch
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    base = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    fn()
    torch.cuda.synchronize(dev)
    peak = torch.cuda.max_memory_allocated(dev)
    return peak / 2**20, (peak - base) / 2**20


def e2e_eager(arm, steps, warmup, world):
    """Same step through the public API, inputs copied from pinned host memory
    and the loss read back every step (H2D/D2H inside the timed region).  The
    H2D copy of step i+1 runs on a copy stream while step i computes (two device
    input buffers), as a training loop with pinned, non-blocking loads does."""
    import torch
    wl, dev = arm.wl, arm.dev
    bufs = [list(wl.make_batch(wl.batch, dev)) for _ in range(2)]
    host = [t.detach().cpu().pin_memory() for t in bufs[0]]
    loss_host = torch.empty((), dtype=torch.float32).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in host)
    d2h = loss_host.numel() * loss_host.element_size()
    copy_stream = torch.cuda.Stream(dev)
    ready = [torch.cuda.Event(), torch.cuda.Event()]
    free = [torch.cuda.Event(), torch.cuda.Event()]
    main = torch.cuda.current_stream(dev)

    def load(i):
        b = i % 2
        copy_stream.wait_event(free[b])
        with torch.cuda.stream(copy_stream), torch.no_grad():
            for d, h in zip(bufs[b], host):
                d.copy_(h, non_blocking=True)
        ready[b].record(copy_stream)

    def one(i, last):
        b = i % 2
        main.wait_event(ready[b])
        if not last:
            load(i + 1)
        inputs = bufs[b]
        if wl.input_requires_grad:
            inputs[0].requires_grad_(True)
        loss = arm.step(inputs)
        if wl.input_requires_grad:
            inputs[0].grad = None
            inputs[0].requires_grad_(False)
        free[b].record(main)
        loss_host.copy_(loss.detach().float(), non_blocking=True)

    return _e2e_loop(one, load, free, main, steps, warmup, world, dev, h2d, d2h)


def e2e_graphed(arm, steps, warmup, world):
    """e2e through the graphed step: the next batch is copied from pinned host
    memory into the other static buffer on a copy stream while the current graph
    replays; the loss is read back every step."""
    import torch
    dev, g = arm.dev, arm.graphed
    host = [t.detach().cpu().pin_memory() for t in g.inputs[0]]
    loss_host = torch.empty((), dtype=torch.float32).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in host)
    d2h = loss_host.numel() * loss_host.element_size()
    copy_stream = torch.cuda.Stream(dev)
    ready = [torch.cuda.Event(), torch.cuda.Event()]
    free = [torch.cuda.Event(), torch.cuda.Event()]
    main = torch.cuda.current_stream(dev)

    def load(i):
        b = i % 2
        copy_stream.wait_event(free[b])
        with torch.cuda.stream(copy_stream), torch.no_grad():
            for d, h in zip(g.inputs[b], host):
                d.copy_(h, non_blocking=True)
        ready[b].record(copy_stream)

    def one(i, last):
        b = i % 2
        main.wait_event(ready[b])
        if not last:
            load(i + 1)
        loss = g.replay(b)
        free[b].record(main)
        loss_host.copy_(loss.float(), non_blocking=True)

    return _e2e_loop(one, load, free, main, steps, warmup, world, dev, h2d, d2h)


def _e2e_loop(one, load, free, main, steps, warmup, world, dev, h2d, d2h):
    import torch
    for r in range(2):
        free[r].record(main)
    load(0)
    for i in range(warmup):
        one(i, last=False)
    torch.cuda.synchronize(dev)
    _barrier(world)
    torch.cuda.synchronize(dev)
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    load(0)  # the first timed step's inputs are copied inside the timed region
    for i in range(steps):
        one(i, last=(i == steps - 1))
    e.record()
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - t0
    return _max_over_ranks(s.elapsed_time(e), world), wall, h2d, d2h


# ------------------------------------------------------------------ helpers
def _per_rank_batch(config, world, override):
    from benchkit import models as BM
    import inspect
    default = inspect.signature(BM.WORKLOADS[config]).parameters["batch"].default
    if CONFIGS[config]["scaling"] == "weak":
        return override or default, (override or default) * world
    glob = override or default
    if glob % world:
        raise SystemExit(f"global batch {glob} is not divisible by {world} ranks")
    return glob // world, glob


def _prediction(config, batch, inputs, fuse=True):
    """Planner-predicted peak (MiB) of the product step: the same workload built
    on the meta device, converted and fused, one fwd+bwd on shapes only."""
    import torch

    from benchkit import models as BM
    from paper_2404_12406_b200.nn import convert_to_memory_saving
    from paper_2404_12406_b200.planner import plan
    try:
        wl = BM.WORKLOADS[config](batch=batch, device="meta")
        model = convert_to_memory_saving(wl.model, fuse=fuse)
        p = plan(model, inputs, loss_fn=wl.loss_fn)
        return round(p.peak_bytes / 2**20, 1), round(p.tape_bytes / 2**20, 1)
    except Exception as exc:  # noqa: BLE001 - report, never fail the bench
        return None, f"{type(exc).__name__}: {exc}"[:200]
    finally:
        torch.cuda.empty_cache()


def _ncu_traffic(config, dom):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant op,
    from the committed ncu capture of this config (profiles/r2_ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "r2_ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        es = d[config]
        for e in es if isinstance(es, list) else [es]:
            if e["op"].split(".")[-1] == dom["op"].split(".")[-1] and e["geom"] == dom["geom"]:
                return int(e["dram_bytes"]), \
                    f"profiles/r2_ncu_traffic.json:{config} ({e['kernel']})"
    except Exception:
        pass
    return None, None


# ------------------------------------------------------------------ GPU arm
def gpu_main(args):
    import torch

    import paper_2404_12406_b200 as pkg
    from benchkit import models as BM
    from benchkit import roofline as RL
    from paper_2404_12406_b200.distributed import TrainableGradAllReduce
    from paper_2404_12406_b200.nn import convert_to_memory_saving

    world, rank, local = _dist_setup()
    dev = torch.device("cuda", local)
    peaks = _peaks()
    pkg.lib()  # fail loudly if the native library is missing
    cfgd = CONFIGS[args.config]
    batch, global_batch = _per_rank_batch(args.config, world, args.batch)
    use_graph = cfgd["graph"] and world == 1 and not args.eager
    builder = BM.WORKLOADS[args.config]

    def fresh():
        return builder(batch=batch)

    # ---------------- memsave arm (the product): every supported layer swapped,
    # conv -> BN(eval) -> ReLU, conv -> ReLU and residual joins fused by the fx pass
    wl = fresh()
    wl.model = convert_to_memory_saving(wl.model, fuse=not args.no_fuse)
    sync = TrainableGradAllReduce(wl.model) if world > 1 else None
    arm = Arm(wl, wl.model, dev, world, sync)
    arm.prime()
    modes = {}
    n0 = pkg.launch_count()
    ms_eager = _timed(arm.step, args.steps, args.warmup, world, dev)
    per_step_launches = (pkg.launch_count() - n0) // (args.steps + args.warmup)
    modes["eager"] = {"ms_per_step": round(ms_eager / args.steps, 4),
                      "value": round(batch * world * args.steps / (ms_eager / 1e3), 2)}
    # in-step kernel timing of every memsave op (one extra, instrumented eager step)
    calls, traced_ms = RL.trace_step(arm.step, dev)
    rows, op_ms = RL.summarise(calls, traced_ms, peaks)
    # peak memory of one step (eager: a graph replay allocates nothing, its pool
    # holds the same working set)
    peak_mib, act_peak_mib = peak_memory(arm.step, dev)
    if use_graph:
        arm.capture()
        run = arm.replay
        modes["cuda_graph_reserved_mib"] = round(torch.cuda.memory_reserved(dev) / 2**20, 1)
    else:
        run = arm.step
    with ClockSampler(local) as clocks:
        ms = _timed(run, args.steps, args.warmup, world, dev)
    if use_graph:
        modes["cuda_graph"] = {"ms_per_step": round(ms / args.steps, 4),
                               "value": round(batch * world * args.steps / (ms / 1e3), 2)}
    # median of 5 repeats of the K timed steps
    reps = [_timed(run, args.steps, 0, world, dev) / args.steps for _ in range(5)]
    if use_graph:
        e2e_ms, e2e_wall, h2d, d2h = e2e_graphed(arm, args.steps, max(1, args.warmup // 2),
                                                 world)
    else:
        e2e_ms, e2e_wall, h2d, d2h = e2e_eager(arm, args.steps, max(1, args.warmup // 2), world)
    pred_mib, pred_tape = (None, None)
    if rank == 0 and not args.no_plan:
        pred_mib, pred_tape = _prediction(args.config, batch, arm.inputs,
                                          fuse=not args.no_fuse)
    samples = batch * world * args.steps
    value = samples / (ms / 1e3)
    e2e_value = samples / (e2e_ms / 1e3)
    # release the product model before the other arms (their peaks are their own):
    # `run` is a bound method of the arm and keeps it alive
    del arm, wl, run
    sync = None
    import gc
    gc.collect()
    torch.cuda.empty_cache()

    def other_arm(convert_kwargs, benchmark=False, tf32=None, graph=False):
        """(ms per K steps, peak MiB, activation peak MiB) of a fresh model"""
        prev = (torch.backends.cudnn.benchmark, torch.backends.cudnn.allow_tf32,
                torch.backends.cuda.matmul.allow_tf32)
        torch.backends.cudnn.benchmark = benchmark
        if tf32 is not None:
            torch.backends.cudnn.allow_tf32 = tf32
            torch.backends.cuda.matmul.allow_tf32 = tf32
        try:
            w2 = fresh()
            stock = convert_kwargs is None
            if not stock:
                w2.model = convert_to_memory_saving(w2.model, **convert_kwargs)
            sy = TrainableGradAllReduce(w2.model) if (world > 1 and not stock) else None
            a2 = Arm(w2, w2.model, dev, world, sy, ddp=stock)
            a2.prime()
            fn = a2.step
            apeak, aact = peak_memory(fn, dev)
            if graph:
                a2.capture()
                fn = a2.replay
            ams = _timed(fn, args.steps, args.warmup, world, dev)
            del fn, a2, w2, sy
            return ams, apeak, aact
        finally:
            (torch.backends.cudnn.benchmark, torch.backends.cudnn.allow_tf32,
             torch.backends.cuda.matmul.allow_tf32) = prev
            import gc
            gc.collect()
            torch.cuda.empty_cache()

    def rec(ms_, peak_, act_, **kw):
        return dict(value=round(samples / (ms_ / 1e3), 2), ms_per_step=round(ms_ / args.steps, 4),
                    peak_mib=round(peak_, 1), activation_peak_mib=round(act_, 1), **kw)

    # ---------------- stock arms (same weights, unconverted)
    stock = {}
    if not args.no_stock:
        fp32 = args.config == "fig1"
        sms, speak, sact = other_arm(None, tf32=False if fp32 else None)
        stock["eager"] = rec(sms, speak, sact, impl="torch %s stock modules (cuDNN / cuBLAS)%s"
                             % (torch.__version__, ", TF32 off (fp32 rtol 1e-5 parity)"
                                if fp32 else ""))
        if args.config in ("fig1", "resnet18", "resnet101", "vgg16"):
            b_ms, b_peak, b_act = other_arm(None, benchmark=True, tf32=False if fp32 else None)
            stock["cudnn_benchmark"] = rec(b_ms, b_peak, b_act, impl="stock, "
                                           "torch.backends.cudnn.benchmark=True")
            if fp32:
                t_ms, t_peak, t_act = other_arm(None, benchmark=True, tf32=True)
                stock["cudnn_benchmark_tf32"] = rec(
                    t_ms, t_peak, t_act, impl="stock, cudnn.benchmark, TF32 convs (NOT rtol "
                    "1e-5: 10-bit mantissa products)")
        if use_graph:
            g_ms, g_peak, g_act = other_arm(None, benchmark=True, tf32=False if fp32 else None,
                                            graph=True)
            stock["cuda_graph"] = rec(g_ms, g_peak, g_act, impl="stock, cudnn.benchmark, "
                                      "whole step captured as a CUDA graph")
        comparable = [v for k, v in stock.items() if k != "cudnn_benchmark_tf32"]
        best = max(comparable, key=lambda r: r["value"])
        stock["best"] = {"value": best["value"], "ms_per_step": best["ms_per_step"],
                         "peak_mib": best["peak_mib"],
                         "which": [k for k, v in stock.items() if v is best][0]}
        if not args.quick:
            lms, lpeak, lact = other_arm(dict(relu=False, maxpool2d=False, dropout=False,
                                              layernorm=False, conv_transpose2d=False))
            stock["memsave_layers_only"] = rec(lms, lpeak, lact,
                                               swaps="Linear, Conv2d, BatchNorm2d(eval) only, "
                                               "eager")
            if not args.no_fuse:
                ums, upeak, uact = other_arm(dict(fuse=False))
                stock["memsave_unfused"] = rec(ums, upeak, uact, swaps="all supported layers, "
                                               "convert_to_memory_saving(fuse=False), eager")

    # ---------------- roofline of the dominant in-step kernel
    roof = None
    if rows:
        dom = rows[0]
        traffic, tsrc = _ncu_traffic(args.config, dom)
        roof = {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"],
                "unit": dom["unit"], "frac": dom["frac"], "traffic": traffic,
                "traffic_source": tsrc, "op": "torch.ops.memsave." + dom["op"],
                "geom": dom["geom"], "launches_per_step": dom["launches_per_step"],
                "ms_per_launch": dom["ms_per_launch"],
                "share_of_step": round(dom["ms_per_step"] / traced_ms, 3),
                "algorithmic_flops": dom["flops"], "algorithmic_bytes": dom["bytes"],
                "per_unit": ("2*M*N*K flops (implicit GEMM for convs) and one read of every "
                             "operand + one write of every output per launch"),
                "peak_source": peaks["source"] + ", burst",
                "how": ("CUDA events around every torch.ops.memsave call of one extra eager "
                        "step on its launching stream, host enqueue ahead of the GPU"),
                "memsave_ops_share_of_step": round(op_ms / traced_ms, 3),
                "top": [{k: r[k] for k in ("op", "geom", "launches_per_step", "ms_per_launch",
                                           "bound", "achieved", "unit", "frac")}
                        for r in rows[:6]]}

    # ---------------- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.config, args.cpu_seconds)

    best_stock = stock.get("best")
    out = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "samples/s",
        "tokens_per_s": (round(value * wl_seq(args.config), 1) if wl_seq(args.config) else None),
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4),
        "ms_per_step_median_of_5": round(statistics.median(reps), 4),
        "higher_is_better": True,
        "scaling": cfgd["scaling"],
        "vs_baseline": None,
        "dtype": "f32" if args.config == "fig1" else "bf16",
        "data": "synthetic (random-init weights, seeded normal inputs / uniform token ids)",
        "config": dict(_config_desc(args.config, batch), workload=_workload_name(args.config),
                       global_batch=global_batch, per_gpu_batch=batch,
                       parallelism=(f"dp{world}" if world > 1 else "single"),
                       step_mode="cuda_graph" if use_graph else "eager",
                       l2="inputs and activations > 126 MB L2 (no explicit flush)"),
        "peak_mib": round(peak_mib, 1),
        "activation_peak_mib": round(act_peak_mib, 1),
        "pred_mib": pred_mib,
        "pred_tape_mib": pred_tape,
        "pred_err": (round(peak_mib / pred_mib - 1, 4) if isinstance(pred_mib, float) else None),
        "modes": modes,
        "stock": stock,
        "speedup_vs_stock": (round(value / best_stock["value"], 3) if best_stock else None),
        "peak_ratio_vs_stock": (round(peak_mib / best_stock["peak_mib"], 3) if best_stock
                                else None),
        "e2e": {"value": round(e2e_value, 2), "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms / args.steps, 4),
                "wall_s": round(e2e_wall, 3)},
        "gpu_launches": per_step_launches * args.steps,
        "gpu_launches_per_step": per_step_launches,
        "gpu_launches_note": ("memsave kernels per eager step (host counter) x timed steps; "
                              "a CUDA-graph replay relaunches exactly the captured kernels"
                              if use_graph else "host launch counter over the timed steps"),
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


def wl_seq(config):
    return {"bert": 512, "llama": 2048}.get(config)


def _workload_name(config):
    return {
        "bert": "BASELINE configs[3]: BERT-base random init, attention Linear biases + "
                "classifier trainable, train mode (dropout 0.1), seq 512",
        "resnet18": "BASELINE configs[1]: ResNet-18 frozen weights, input-only gradient, "
                    "eval-mode BN, 224x224",
        "resnet101": "BASELINE configs[2] (ResNet-101 reading): layer4.1, layer4.2, fc and all "
                     "BN affine trainable, BN eval, 224x224",
        "vgg16": "BASELINE configs[2] (VGG-16 reading): conv blocks 4-5 + classifier trainable, "
                 "224x224",
        "fig1": "BASELINE configs[0]: Fig.1 deep CNN, 8x Conv2d(8->8, 3x3), only layer-1 "
                "weight trainable, (32,8,256,256) fp32",
        "llama": "BASELINE configs[4]: Llama-3-8B architecture random init, last 4 decoder "
                 "layers trainable, seq 2048, 2 sequences per GPU",
    }[config]


def _config_desc(config, batch):
    from benchkit import models as BM
    try:
        import torch
        wl = BM.WORKLOADS[config](batch=batch, device="meta")
        d = dict(wl.config)
        d.pop("workload", None)
        d.pop("global_batch", None)
        del wl
        torch.cuda.empty_cache()
        return d
    except Exception:
        return {"model": config}


# ------------------------------------------------------------------ CPU legs
def cpu_baseline(config, seconds):
    """The reference algorithm on the host cores, in a separate process (a
    separate Python session), on a bounded sample of the workload."""
    cmd = [sys.executable, "-c",
           "import json,sys; sys.path.insert(0, %r); from benchkit.cpu_port import cpu_sample; "
           "print(json.dumps(cpu_sample(%r, %r)))" % (ROOT, config, float(seconds))]
    try:
        env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
        return json.loads(line)
    except Exception as exc:  # noqa: BLE001
        return {"value": None, "error": f"{type(exc).__name__}: {str(exc)[:200]}"}


def reference_main(args):
    """--impl reference: the reference's CPU implementation of the path (its own
    conv kernels from baseline/_ref when installed, the oracle port for the
    SPEC-only Linear / BN rows) on all host threads; rank 0 only."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from benchkit.cpu_port import cpu_workload
    step, rec = cpu_workload(args.config)
    for _ in range(args.warmup):
        step()
    per_step = [step() for _ in range(args.steps)]
    sec = sum(per_step) / len(per_step)  # seconds per sample of the full workload
    v = round(1.0 / sec, 6)
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 2), "higher_is_better": True,
        "scaling": CONFIGS[args.config]["scaling"], "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": _workload_name(args.config),
                   "note": "each step is a bounded sample of the workload: " + rec["sample"]
                   + f"; all host threads ({rec['cores']})"},
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": rec["cores"],
                         "isa": rec.get("isa"), "kind": rec["kind"], "sample": rec["sample"]},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def _respawn(args):
    """--gpus N without torchrun: re-exec this script under torch.distributed.run."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="memsave", choices=["memsave", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=0,
                    help="global batch (per-GPU for the weak-scaling Llama config)")
    ap.add_argument("--no-stock", action="store_true")
    ap.add_argument("--no-fuse", action="store_true",
                    help="product arm without the conv->BN->ReLU / add->ReLU fx fusion")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph for the product arm")
    ap.add_argument("--quick", action="store_true", help="skip the diagnostic memsave arms")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-plan", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.impl == "reference":
        reference_main(args)
        return
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _respawn(args)
    gpu_main(args)


if __name__ == "__main__":
    main()
