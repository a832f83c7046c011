"""Data-parallel gradient exchange for selective differentiation.

The natural shard of the hot path is the batch: samples are
independent through forward and backward, and the only exchange is an
average of the *trainable-subset* parameter gradients after backward.  This
module registers post-accumulate-grad hooks on exactly the parameters with
``requires_grad=True``, packs their gradients into flat buckets in the order
backward produces them, and launches one asynchronous all-reduce per full
bucket on the process group (NCCL over NVLink/NVSwitch on B200, gloo on CPU
for tests), so communication overlaps the rest of backward.  Frozen
parameters never enter a bucket, so no bytes are spent on them; when nothing
is trainable (the input-only scenario) nothing is communicated at all and
the ranks are independent replicas.
"""

from __future__ import annotations

import torch
import torch.distributed as dist
from torch import nn


class TrainableGradAllReduce:
    """Bucketed, overlapped all-reduce (average) of trainable gradients.

    Usage::

        sync = TrainableGradAllReduce(model)
        loss.backward()
        sync.finish()        # waits for the in-flight reductions
    """

    def __init__(self, model: nn.Module, process_group=None, bucket_cap_mb: float = 64.0,
                 average: bool = True):
        self.pg = process_group
        self.world = dist.get_world_size(process_group) if dist.is_initialized() else 1
        self.average = average
        self.params = [p for p in model.parameters() if p.requires_grad]
        # reverse registration order ~ order in which backward produces grads
        order = list(reversed(self.params))
        cap = int(bucket_cap_mb * 1024 * 1024)
        self.buckets: list[list[nn.Parameter]] = []
        cur, cur_bytes = [], 0
        for p in order:
            nbytes = p.numel() * p.element_size()
            if cur and (cur_bytes + nbytes > cap or p.dtype != cur[0].dtype
                        or p.device != cur[0].device):
                self.buckets.append(cur)
                cur, cur_bytes = [], 0
            cur.append(p)
            cur_bytes += nbytes
        if cur:
            self.buckets.append(cur)
        self._bucket_of = {}
        for bi, b in enumerate(self.buckets):
            for p in b:
                self._bucket_of[id(p)] = bi
        self._flat = [None] * len(self.buckets)
        self._pending = [0] * len(self.buckets)
        self._works = []
        self._hooks = [p.register_post_accumulate_grad_hook(self._on_grad) for p in self.params]
        self.bytes_communicated = 0
        self._reset()

    @property
    def trainable_numel(self) -> int:
        return sum(p.numel() for p in self.params)

    def _reset(self):
        self._pending = [len(b) for b in self.buckets]
        self._works = []

    def _on_grad(self, p: torch.Tensor) -> None:
        if self.world == 1:
            return
        bi = self._bucket_of[id(p)]
        self._pending[bi] -= 1
        if self._pending[bi] == 0:
            self._launch(bi)

    def _launch(self, bi: int) -> None:
        ps = self.buckets[bi]
        flat = torch.cat([p.grad.reshape(-1) for p in ps])
        if self.average:
            flat.div_(self.world)
        work = dist.all_reduce(flat, group=self.pg, async_op=True)
        self.bytes_communicated += flat.numel() * flat.element_size()
        self._works.append((bi, flat, work))

    def finish(self) -> None:
        """Wait for every bucket and write the averaged values back."""
        if self.world == 1:
            return
        # buckets not launched by the hooks (a trainable param received no grad this
        # step): reduce them now, with zeros for the missing grads, so that every
        # rank issues the same collectives in the same order
        for bi, pend in enumerate(self._pending):
            if pend > 0:
                for p in self.buckets[bi]:
                    if p.grad is None:
                        p.grad = torch.zeros_like(p)
                self._pending[bi] = 0
                self._launch(bi)
        for bi, flat, work in self._works:
            work.wait()
            off = 0
            for p in self.buckets[bi]:
                n = p.numel()
                p.grad.copy_(flat[off:off + n].view_as(p.grad))
                off += n
        self._reset()

    def remove(self) -> None:
        for h in self._hooks:
            h.remove()
