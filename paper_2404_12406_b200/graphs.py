"""CUDA-graph runner for a whole training step (forward + loss + backward).

Launch-bound steps (ResNet-101's ~650 launches, or any small batch) spend more
time in Python and the dispatcher than the GPU spends in the kernels.  Every
memsave op is a ``torch.ops.memsave`` custom op that allocates from the caching
allocator, launches on the current stream and never synchronises, so a step
can be captured once and replayed: the replay issues the same kernels with no
host work at all.

``GraphedStep`` captures ``n_buffers`` graphs over ``n_buffers`` sets of static
input tensors (sharing one memory pool: the graphs run one after another), so
a loader can copy the next batch into buffer ``(i + 1) % n`` on a copy stream
while graph ``i % n`` runs.  Parameter gradients are accumulated in place into
tensors that exist before capture; the step function is expected to zero them
first (``zero_grads``), which is captured too, so every replay leaves exactly
one step's gradients in ``p.grad``.

Not graph-safe: host-side randomness drawn per call (the memsave Dropout seed is
drawn on the CPU, so a captured dropout would replay one mask) and
data-dependent host control flow.  The bench uses graphs only for the CNN
configs, which have neither.
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch

__all__ = ["GraphedStep", "zero_grads"]


def zero_grads(params: Sequence[torch.Tensor]) -> None:
    """Zero existing gradients in place (one fused launch); graph-capturable."""
    grads = [p.grad for p in params if p.grad is not None]
    if grads:
        torch._foreach_zero_(grads)


class GraphedStep:
    """``step_fn(*inputs) -> loss`` (runs backward itself) captured as CUDA graphs.

    ``static_inputs``: one list of device tensors per buffer; inputs that need a
    gradient must have ``requires_grad=True`` (their ``.grad`` is rewritten by
    every replay).  Call ``replay(k)`` to run the step on buffer ``k``; the
    returned loss tensor is static (overwritten by the next replay of ``k``).
    """

    def __init__(self, step_fn: Callable, static_inputs: Sequence[Sequence[torch.Tensor]],
                 warmup: int = 2):
        self.step_fn = step_fn
        self.inputs = [list(b) for b in static_inputs]
        dev = self.inputs[0][0].device
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):
                for b in self.inputs:
                    self._clear_input_grads(b)
                    step_fn(*b)
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.pool = torch.cuda.graph_pool_handle()
        self.graphs, self.losses = [], []
        for b in self.inputs:
            self._clear_input_grads(b)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=self.pool):
                loss = step_fn(*b)
            self.graphs.append(g)
            self.losses.append(loss)
        torch.cuda.synchronize(dev)

    @staticmethod
    def _clear_input_grads(b):
        for t in b:
            if isinstance(t, torch.Tensor) and t.requires_grad:
                t.grad = None

    def replay(self, k: int = 0) -> torch.Tensor:
        self.graphs[k].replay()
        return self.losses[k]

    def __len__(self):
        return len(self.graphs)
