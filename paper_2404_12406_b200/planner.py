"""Analytic storage planner / peak predictor (the
reference's ``planner`` module, and memwatch's live-set
model).

``plan(model, inputs)`` runs one forward (+ backward) of ``model`` on the
``meta`` device -- shapes only, no arithmetic -- and reports

* the saved set per module: every tensor autograd keeps for backward (the
  ``saved_tensors_hooks`` view of the tape), with its role-free byte size,
  deduplicated by storage;
* ``tape_bytes``: the deduplicated total;
* ``fwd_peak_bytes`` / ``peak_bytes``: the maximum of the live activation set
  during forward, and during forward + backward, from an allocation ledger
  kept by a ``TorchDispatchMode`` (every op output allocates, a storage is
  freed when its last tensor dies -- CPython refcounting makes that exact).
  Parameters, buffers and the network input are counted as resident.

The memsave layers accept meta tensors and take the same storage decisions as
on CUDA (functional.py), so a plan of a converted model predicts what the
GPU run keeps; ``tests/test_planner*.py`` check the prediction against
``torch.cuda.max_memory_allocated`` on B200.
"""

from __future__ import annotations

import copy
import dataclasses
import weakref
from typing import Callable, Sequence

import torch
from torch import nn
from torch.utils._python_dispatch import TorchDispatchMode

__all__ = ["StoragePlan", "plan", "plan_csv_row", "CSV_HEADER"]

CSV_HEADER = "net,layer,depth,scenario,policy,tape_bytes,peak_bytes,forward_ms,backward_ms"


@dataclasses.dataclass
class SavedEntry:
    module: str
    shape: tuple
    dtype: str
    nbytes: int


@dataclasses.dataclass
class StoragePlan:
    saved: list            # [SavedEntry] in recording order (deduplicated by storage)
    tape_bytes: int        # sum of saved bytes
    resident_bytes: int    # parameters + buffers + inputs (live throughout)
    fwd_peak_bytes: int    # peak live bytes during forward (incl. resident)
    peak_bytes: int        # peak live bytes during forward + backward (incl. resident)

    def saved_by_module(self) -> dict:
        out: dict = {}
        for e in self.saved:
            out.setdefault(e.module, []).append(e)
        return out


def _storage_key(t: torch.Tensor):
    try:
        return t.untyped_storage()._cdata
    except Exception:  # pragma: no cover
        return id(t)


def _storage_nbytes(t: torch.Tensor) -> int:
    try:
        return int(t.untyped_storage().nbytes())
    except Exception:  # pragma: no cover
        return t.numel() * t.element_size()


class _Ledger(TorchDispatchMode):
    """Allocation ledger: +bytes when an op creates a new storage, -bytes when
    the last tensor referencing it is collected."""

    def __init__(self):
        super().__init__()
        self.live = 0
        self.peak = 0
        self._seen: dict = {}

    def reset_peak(self):
        self.peak = self.live

    def track(self, t: torch.Tensor):
        key = _storage_key(t)
        if key in self._seen:
            return
        nb = _storage_nbytes(t)
        self._seen[key] = nb
        self.live += nb
        self.peak = max(self.peak, self.live)
        try:
            weakref.finalize(t.untyped_storage(), self._free, key)
        except TypeError:  # storages that do not support weakrefs: follow the tensor
            weakref.finalize(t, self._free, key)

    def _free(self, key):
        nb = self._seen.pop(key, 0)
        self.live -= nb

    def __torch_dispatch__(self, func, types, args=(), kwargs=None):
        out = func(*args, **(kwargs or {}))
        for t in torch.utils._pytree.tree_leaves(out):
            if isinstance(t, torch.Tensor) and t.device.type == "meta":
                self.track(t)
        return out


class _FusedSDPA:
    """On CUDA, ``F.scaled_dot_product_attention`` runs a fused kernel (flash, or
    memory-efficient when a mask is given) that keeps O(L) statistics, not the
    L x L attention matrix; on ``meta`` its backend choice falls to the math path,
    which materialises it.  While planning, route meta SDPA calls to the fused
    kernels' own meta functions so the prediction matches the GPU run."""

    def __enter__(self):
        import torch.nn.functional as F
        self._orig = F.scaled_dot_product_attention
        orig = self._orig

        def sdpa(q, k, v, attn_mask=None, dropout_p=0.0, is_causal=False, scale=None,
                 enable_gqa=False):
            if q.device.type != "meta":
                return orig(q, k, v, attn_mask=attn_mask, dropout_p=dropout_p,
                            is_causal=is_causal, scale=scale, enable_gqa=enable_gqa)
            if enable_gqa and k.shape[-3] != q.shape[-3]:
                rep = q.shape[-3] // k.shape[-3]
                k = k.repeat_interleave(rep, dim=-3)
                v = v.repeat_interleave(rep, dim=-3)
            if attn_mask is None:
                return torch.ops.aten._scaled_dot_product_flash_attention(
                    q, k, v, dropout_p, is_causal, False, scale=scale)[0]
            return torch.ops.aten._scaled_dot_product_efficient_attention(
                q, k, v, attn_mask.expand(q.shape[0], q.shape[1], q.shape[2], k.shape[2]),
                q.requires_grad, dropout_p, is_causal, scale=scale)[0]

        F.scaled_dot_product_attention = sdpa
        return self

    def __exit__(self, *exc):
        import torch.nn.functional as F
        F.scaled_dot_product_attention = self._orig


def _to_meta(model: nn.Module) -> nn.Module:
    m = copy.deepcopy(model).to("meta")
    for (_n, p), (_n2, p0) in zip(m.named_parameters(), model.named_parameters()):
        p.requires_grad_(p0.requires_grad)
    return m


def plan(model: nn.Module, inputs: Sequence[torch.Tensor],
         loss_fn: Callable | None = None, backward: bool = True) -> StoragePlan:
    """Predict the saved set, tape bytes and peak live bytes of one fwd(+bwd)
    of ``model(*inputs)`` (``loss_fn(model, *inputs)`` if given) without doing
    any arithmetic.  ``inputs`` may be real tensors (only shape, dtype,
    memory format and requires_grad are used)."""
    mm = _to_meta(model)
    metas = []
    for t in inputs:
        mt = torch.empty_strided(t.shape, t.stride(), dtype=t.dtype, device="meta")
        if t.requires_grad:
            mt.requires_grad_(True)
        metas.append(mt)
    current = ["<top>"]
    names = {mod: name for name, mod in mm.named_modules()}

    def pre(mod, _inp):
        current.append(names.get(mod, type(mod).__name__))

    def post(mod, _inp, _out):
        current.pop()

    hooks = []
    for mod in mm.modules():
        hooks.append(mod.register_forward_pre_hook(pre))
        hooks.append(mod.register_forward_hook(post))
    saved: list = []
    seen = set()

    def pack(t):
        key = _storage_key(t)
        if not isinstance(t, nn.Parameter) and key not in seen:
            seen.add(key)
            saved.append(SavedEntry(current[-1], tuple(t.shape), str(t.dtype).replace("torch.", ""),
                                    _storage_nbytes(t)))
        return t

    ledger = _Ledger()
    resident = 0
    for p in list(mm.parameters()) + list(mm.buffers()):
        resident += _storage_nbytes(p)
    for t in metas:
        resident += _storage_nbytes(t)
    ledger.live = ledger.peak = resident
    try:
        with ledger, _FusedSDPA(), torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
            out = loss_fn(mm, *metas) if loss_fn else mm(*metas)
            fwd_peak = ledger.peak
            if backward and isinstance(out, torch.Tensor) and out.requires_grad:
                if out.numel() != 1:
                    out = out.sum()
                out.backward()
            del out
    finally:
        for h in hooks:
            h.remove()
    # parameters / buffers / inputs are not op outputs: they never enter the
    # ledger's free list, so the resident part is constant
    return StoragePlan(saved=saved, tape_bytes=sum(e.nbytes for e in saved),
                       resident_bytes=resident, fwd_peak_bytes=fwd_peak,
                       peak_bytes=ledger.peak)


def plan_csv_row(net: str, layer: str, depth: int, scenario: str, policy: str,
                 tape_bytes: int, peak_bytes: int, forward_ms: float = float("nan"),
                 backward_ms: float = float("nan")) -> str:
    """One row of the reference bench CSV schema."""
    return (f"{net},{layer},{depth},{scenario},{policy},{tape_bytes},{peak_bytes},"
            f"{forward_ms:.4f},{backward_ms:.4f}")
