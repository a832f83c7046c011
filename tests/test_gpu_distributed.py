"""Data-parallel exchange through MemSave layers on the GPU: two processes on
the single B200 (gloo on CUDA tensors -- one GPU, so not NCCL), each running
half of the batch through a converted model with a trainable subset; the
averaged gradients must equal the full-batch gradients and only the trainable
bytes may cross the wire."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from torch import nn

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _model():
    torch.manual_seed(0)
    m = nn.Sequential(
        nn.Conv2d(8, 16, 3, padding=1, bias=False), nn.BatchNorm2d(16), nn.ReLU(),
        nn.Conv2d(16, 16, 3, padding=1), nn.ReLU(), nn.AdaptiveAvgPool2d(1), nn.Flatten(),
        nn.Linear(16, 10))
    g = torch.Generator().manual_seed(1)
    m[1].running_mean.copy_(torch.randn(16, generator=g) * 0.1)
    m[1].running_var.copy_(torch.rand(16, generator=g) + 0.5)
    m.eval()
    m[0].weight.requires_grad_(False)  # frozen stem: never communicated
    return m


def _data():
    g = torch.Generator().manual_seed(2)
    return torch.randn(8, 8, 12, 12, generator=g), torch.randint(0, 10, (8,), generator=g)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_12406_b200 import launch_count
    from paper_2404_12406_b200.distributed import TrainableGradAllReduce
    from paper_2404_12406_b200.nn import convert_to_memory_saving
    dev = torch.device("cuda", 0)
    m = convert_to_memory_saving(_model()).to(dev)
    sync = TrainableGradAllReduce(m, bucket_cap_mb=0.001)
    x, y = _data()
    xs, ys = x[rank * 4:(rank + 1) * 4].to(dev), y[rank * 4:(rank + 1) * 4].to(dev)
    n0 = launch_count()
    for _ in range(2):  # the second step runs on the re-packed buckets
        sync.zero_grad()
        nn.functional.cross_entropy(m(xs), ys).backward()
        sync.finish()
    torch.cuda.synchronize()
    grads = {n: p.grad.cpu().tolist() for n, p in m.named_parameters() if p.requires_grad}
    q.put((rank, grads, sync.bytes_communicated, sync.trainable_numel, launch_count() - n0))
    dist.destroy_process_group()


def test_dp_through_memsave_layers_matches_full_batch():
    world, port = 2, _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2404_12406_b200.nn import convert_to_memory_saving
    dev = torch.device("cuda", 0)
    m = convert_to_memory_saving(_model()).to(dev)
    x, y = _data()
    nn.functional.cross_entropy(m(x.to(dev)), y.to(dev)).backward()
    ref = {n: p.grad.cpu() for n, p in m.named_parameters() if p.requires_grad}
    assert "0.weight" not in ref
    for rank, grads, nbytes, numel, launches in res:
        assert launches > 0  # the memsave kernels ran in the worker
        assert set(grads) == set(ref)
        for n in ref:
            torch.testing.assert_close(torch.tensor(grads[n]), ref[n], rtol=1e-5, atol=1e-6)
        assert numel == sum(t.numel() for t in ref.values())
        assert nbytes == 2 * numel * 4  # two steps, fp32, trainable subset only
