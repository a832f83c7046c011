"""Data-parallel gradient exchange for selective differentiation.

The natural shard of the hot path is the batch: samples are
independent through forward and backward, and the only exchange is an
average of the *trainable-subset* parameter gradients after backward.  This
module registers post-accumulate-grad hooks on exactly the parameters with
``requires_grad=True`` and launches one asynchronous all-reduce per bucket on
the process group (NCCL over NVLink/NVSwitch on B200, gloo on CPU for tests),
so communication overlaps the rest of backward.  Frozen parameters never enter
a bucket, so no bytes are spent on them; when nothing is trainable (the
input-only scenario) nothing is communicated at all and the ranks are
independent replicas.

Buckets are persistent flat buffers and every trainable ``p.grad`` is a view
into its bucket (gradient-as-bucket-view), so autograd accumulates straight
into the communication buffer: no per-step concatenation, no copy back, and no
extra trainable-sized allocation at the peak.  Buckets are launched strictly in
index order on every rank (as DDP does), so the collectives match across ranks
whatever order the hooks fire in.  After the first step the buckets are
re-packed in the order backward actually produced the gradients (rank 0's order,
broadcast), so the first buckets to fill are the first to leave.
"""

from __future__ import annotations

import torch
import torch.distributed as dist
from torch import nn


class TrainableGradAllReduce:
    """Bucketed, overlapped all-reduce (average) of trainable gradients.

    Usage::

        sync = TrainableGradAllReduce(model)
        for batch in data:
            sync.zero_grad()     # zeros the buckets (the grads are views into them)
            loss(model, batch).backward()
            sync.finish()        # waits for the in-flight reductions
            opt.step()

    Gradient accumulation over several backward passes: wrap all but the last
    in ``with sync.no_sync():`` (the hooks then only accumulate locally).
    """

    def __init__(self, model: nn.Module, process_group=None, bucket_cap_mb: float = 64.0,
                 average: bool = True):
        self.pg = process_group
        self.world = dist.get_world_size(process_group) if dist.is_initialized() else 1
        self.average = average
        self.cap = int(bucket_cap_mb * 1024 * 1024)
        self.params = [p for p in model.parameters() if p.requires_grad]
        self._index = {id(p): i for i, p in enumerate(self.params)}
        # initial guess: reverse registration order ~ the order backward produces grads
        self._build(list(reversed(self.params)))
        self._hooks = [p.register_post_accumulate_grad_hook(self._on_grad) for p in self.params]
        self.bytes_communicated = 0
        self._sync_enabled = True
        self._observed: list[int] = []
        self._rebuilt = False
        self._reset()

    # ------------------------------------------------------------ buckets
    def _build(self, order) -> None:
        self.buckets: list[list[nn.Parameter]] = []
        cur, cur_bytes = [], 0
        for p in order:
            nbytes = p.numel() * p.element_size()
            if cur and (cur_bytes + nbytes > self.cap or p.dtype != cur[0].dtype
                        or p.device != cur[0].device):
                self.buckets.append(cur)
                cur, cur_bytes = [], 0
            cur.append(p)
            cur_bytes += nbytes
        if cur:
            self.buckets.append(cur)
        self._bucket_of = {}
        self._flat = []
        self._views = {}
        for bi, b in enumerate(self.buckets):
            flat = torch.zeros(sum(p.numel() for p in b), dtype=b[0].dtype, device=b[0].device)
            off = 0
            for p in b:
                self._bucket_of[id(p)] = bi
                v = flat[off:off + p.numel()].view_as(p)
                if p.grad is not None:  # keep what was accumulated so far
                    v.copy_(p.grad)
                p.grad = v
                self._views[id(p)] = v
                off += p.numel()
            self._flat.append(flat)

    @property
    def trainable_numel(self) -> int:
        return sum(p.numel() for p in self.params)

    def _reset(self):
        self._pending = [len(b) for b in self.buckets]
        self._ready = [False] * len(self.buckets)
        self._next = 0
        self._works = []

    def zero_grad(self) -> None:
        """Zero every bucket (one fill each); the grads stay views into them."""
        for p in self.params:
            v = self._views[id(p)]
            if p.grad is not v:
                p.grad = v
        for flat in self._flat:
            flat.zero_()

    class _NoSync:
        def __init__(self, outer):
            self.outer = outer

        def __enter__(self):
            self.outer._sync_enabled = False

        def __exit__(self, *exc):
            self.outer._sync_enabled = True

    def no_sync(self):
        """Backward passes inside accumulate locally and communicate nothing."""
        return self._NoSync(self)

    # ------------------------------------------------------------ hooks
    def _on_grad(self, p: torch.Tensor) -> None:
        v = self._views[id(p)]
        if p.grad is not v:
            # the grad was reset (set_to_none) and autograd allocated a fresh one:
            # move it into the bucket and re-point the view
            v.copy_(p.grad)
            p.grad = v
        if not self._rebuilt:
            self._observed.append(self._index[id(p)])
        if self.world == 1 or not self._sync_enabled:
            return
        bi = self._bucket_of[id(p)]
        if self._ready[bi] or self._pending[bi] <= 0:
            raise RuntimeError(
                "TrainableGradAllReduce: a gradient arrived for a bucket that was already "
                "reduced this step (a second backward() before finish()); wrap the "
                "accumulation passes in sync.no_sync()")
        self._pending[bi] -= 1
        if self._pending[bi] == 0:
            self._ready[bi] = True
            self._launch_ready()

    def _launch_ready(self) -> None:
        # strictly in bucket-index order, so every rank issues the same sequence
        while self._next < len(self.buckets) and self._ready[self._next]:
            bi = self._next
            flat = self._flat[bi]
            if self.average:
                flat.div_(self.world)
            work = dist.all_reduce(flat, group=self.pg, async_op=True)
            self.bytes_communicated += flat.numel() * flat.element_size()
            self._works.append(work)
            self._next += 1

    def finish(self) -> None:
        """Wait for every bucket (the averaged values are already in p.grad)."""
        if self.world > 1 and self._sync_enabled:
            # buckets not completed by the hooks (a trainable param received no
            # grad this step) are reduced now, its slot holding zeros
            for bi in range(len(self.buckets)):
                self._ready[bi] = True
            self._launch_ready()
            for work in self._works:
                work.wait()
        if not self._rebuilt:
            self._rebuild_from_observed()
        self._reset()

    def _rebuild_from_observed(self) -> None:
        """Re-pack the buckets in the order the first backward produced the grads
        (rank 0's order, broadcast, so the buckets are identical on all ranks)."""
        self._rebuilt = True
        seen, order = set(), []
        for i in self._observed:
            if i not in seen:
                seen.add(i)
                order.append(i)
        order += [i for i in range(len(self.params)) if i not in seen]
        self._observed = []
        if self.world > 1:
            obj = [order]
            dist.broadcast_object_list(obj, src=0, group=self.pg)
            order = obj[0]
        if order != [self._index[id(p)] for b in self.buckets for p in b]:
            self._build([self.params[i] for i in order])

    def remove(self) -> None:
        for h in self._hooks:
            h.remove()
