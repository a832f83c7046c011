"""World-size-2 gloo test of the trainable-subset gradient all-reduce (the
multi-GPU exchange step), on CPU with plain torch layers."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from torch import nn


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _model():
    torch.manual_seed(0)
    m = nn.Sequential(nn.Linear(6, 8), nn.ReLU(), nn.Linear(8, 8), nn.ReLU(), nn.Linear(8, 3))
    m[0].weight.requires_grad_(False)  # frozen: must not be communicated
    m[0].bias.requires_grad_(False)
    m[2].weight.requires_grad_(False)
    return m


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_12406_b200.distributed import TrainableGradAllReduce
    m = _model()
    sync = TrainableGradAllReduce(m, bucket_cap_mb=0.0001)  # tiny buckets: several collectives
    g = torch.Generator().manual_seed(123)
    x = torch.randn(8, 6, generator=g)
    y = torch.randn(8, 3, generator=g)
    xs = x[rank * 4:(rank + 1) * 4]
    ys = y[rank * 4:(rank + 1) * 4]
    loss = ((m(xs) - ys) ** 2).sum(1).mean()
    loss.backward()
    sync.finish()
    grads = {n: p.grad.clone() for n, p in m.named_parameters() if p.requires_grad}
    q.put((rank, grads, sync.bytes_communicated, sync.trainable_numel, len(sync.buckets)))
    dist.destroy_process_group()


def test_trainable_subset_allreduce_matches_full_batch():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process full-batch reference (mean over the 8 samples)
    m = _model()
    g = torch.Generator().manual_seed(123)
    x = torch.randn(8, 6, generator=g)
    y = torch.randn(8, 3, generator=g)
    (((m(x) - y) ** 2).sum(1).mean()).backward()
    ref = {n: p.grad for n, p in m.named_parameters() if p.requires_grad}
    assert set(ref) == {"2.bias", "4.weight", "4.bias"}
    for rank, grads, nbytes, numel, nbuckets in res:
        assert set(grads) == set(ref)
        for n in ref:
            torch.testing.assert_close(grads[n], ref[n], rtol=1e-5, atol=1e-6)
        # only the trainable subset crossed the wire
        assert numel == 8 + 8 * 3 + 3
        assert nbytes == numel * 4
        assert nbuckets >= 2


def _worker_accum(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_12406_b200.distributed import TrainableGradAllReduce
    m = _model()
    sync = TrainableGradAllReduce(m, bucket_cap_mb=0.0001)
    g = torch.Generator().manual_seed(123)
    x = torch.randn(8, 6, generator=g)
    y = torch.randn(8, 3, generator=g)
    out = {}
    # step 1 (also re-packs the buckets in the observed order)
    for step in range(2):
        sync.zero_grad()
        # two micro-batches of 2 samples per rank: the first accumulates locally
        with sync.no_sync():
            xs, ys = x[rank * 4:rank * 4 + 2], y[rank * 4:rank * 4 + 2]
            (((m(xs) - ys) ** 2).sum(1).sum() / 8).backward()
        xs, ys = x[rank * 4 + 2:rank * 4 + 4], y[rank * 4 + 2:rank * 4 + 4]
        (((m(xs) - ys) ** 2).sum(1).sum() / 8).backward()
        sync.finish()
        out[step] = {n: (p.grad * world).tolist() for n, p in m.named_parameters()
                     if p.requires_grad}
    # the grads are views into the persistent buckets
    flat_ptrs = [(f.data_ptr(), f.data_ptr() + f.numel() * f.element_size()) for f in sync._flat]
    views = all(any(lo <= p.grad.data_ptr() < hi for lo, hi in flat_ptrs)
                for p in m.parameters() if p.requires_grad)
    # a second backward before finish() without no_sync is an error, not silent loss
    sync.zero_grad()
    (m(x[:2]).sum()).backward()
    err = None
    try:
        (m(x[:2]).sum()).backward()
    except RuntimeError as e:
        err = str(e)
    q.put((rank, out, views, err))
    dist.destroy_process_group()


def test_accumulation_no_sync_and_bucket_views():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_accum, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    m = _model()
    g = torch.Generator().manual_seed(123)
    x = torch.randn(8, 6, generator=g)
    y = torch.randn(8, 3, generator=g)
    (((m(x) - y) ** 2).sum(1).sum() / 8).backward()
    ref = {n: p.grad for n, p in m.named_parameters() if p.requires_grad}
    for rank, out, views, err in res:
        for step in (0, 1):
            for n in ref:
                torch.testing.assert_close(torch.tensor(out[step][n]), ref[n], rtol=1e-5,
                                           atol=1e-6)
        assert views
        assert err is not None and "no_sync" in err
