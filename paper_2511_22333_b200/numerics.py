"""Numerics API of the drop-in surface (names of ``prefixpack.attention``,
reference ``attention.py:34-315``).

* ``cta_partial`` runs on the GPU through libpatb200: the pack's queries over
  one KV span as a single forward unit with ``PAT_PLAN_ALL_PARTIALS |
  PAT_PLAN_FORWARD_ONLY``, so the forward kernel's fp32 partial (o / l and
  log2-sum-exp) comes back instead of the merged output.  The partial is
  returned in normalised form -- ``max_score`` = natural-log sum-exp,
  ``exp_sum`` = 1, ``weighted_sum`` = o / l -- which the fold
  (``merge_partials``, ``_merge_batch_into``) treats exactly like the
  reference's (peak, sum, weighted sum) triple: both scale to the same
  l * e^m and o * l * e^m.  Inputs are rounded to fp16 / bf16 like
  ``run_packed_attention``'s.
* ``merge_partials`` is the reference's scalar API on Python objects (host);
  the batched merge of the hot path is ``merge_kernel``.
* ``full_attention`` is the monolithic comparator, computed in float64 on the
  GPU (the oracle's float64 numpy restatement lives in ``oracle/``).
* ``generate_qkv`` / ``gather_kv`` / ``max_rel_error`` / ``dump_tensors`` /
  ``load_tensors``: data generation, the error metric and the PPK1 tensor
  interchange format, identical to the reference's.
"""

from __future__ import annotations

import ctypes as C
import math
import struct
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .errors import EmptyPartialList, EmptySpan, NonPositiveDenominator, ShapeMismatch
from .workload import BlockTable, WorkloadSpec


@dataclass
class PartialResult:
    """One (query, head) partial: max score, exp-sum, weighted V sum."""

    max_score: float
    exp_sum: float
    weighted_sum: np.ndarray

    def scaled(self, factor: float) -> "PartialResult":
        return PartialResult(self.max_score, self.exp_sum * factor, self.weighted_sum * factor)


@dataclass
class PartialBatch:
    """Partials of one unit over (query, head)."""

    max_score: np.ndarray     # [q, heads]
    exp_sum: np.ndarray       # [q, heads]
    weighted_sum: np.ndarray  # [q, heads, d]

    def at(self, query_pos: int, head: int) -> PartialResult:
        return PartialResult(float(self.max_score[query_pos, head]), float(self.exp_sum[query_pos, head]),
                             self.weighted_sum[query_pos, head].copy())

    def astype(self, dtype) -> "PartialBatch":
        return PartialBatch(self.max_score.astype(dtype), self.exp_sum.astype(dtype), self.weighted_sum.astype(dtype))


def cta_partial(q_pack: np.ndarray, k_span: np.ndarray, v_span: np.ndarray, scale: Optional[float] = None,
                dtype=None, device="cuda") -> PartialBatch:
    """Partials of a pack's queries ``q_pack`` [q, H, d] over one KV span
    ``k_span`` / ``v_span`` [t, KVH, d] (reference ``attention.py:140-163``),
    computed by the sm_100a forward kernel."""
    import torch

    from .attention import pat_attention
    from .plan import PatPlan

    q_pack, k_span, v_span = np.asarray(q_pack), np.asarray(k_span), np.asarray(v_span)
    if k_span.ndim == 3 and k_span.shape[0] == 0:
        raise EmptySpan("CTA span covers zero tokens")
    if q_pack.ndim != 3 or k_span.ndim != 3 or k_span.shape != v_span.shape or q_pack.shape[2] != k_span.shape[2]:
        raise ShapeMismatch("q_pack must be [q, heads, d]; K/V spans [t, kv_heads, d]")
    nq, H, d = q_pack.shape
    t, KVH, _ = k_span.shape
    if H % KVH:
        raise ShapeMismatch("num_heads must be a multiple of kv_heads")
    dtype = dtype or torch.float16
    bs = 16
    npg = (t + bs - 1) // bs
    kp = np.zeros((npg * bs, KVH, d))
    vp = np.zeros((npg * bs, KVH, d))
    kp[:t], vp[:t] = k_span, v_span
    kc = torch.from_numpy(kp.reshape(npg, bs, KVH, d)).to(device=device, dtype=dtype)
    vc = torch.from_numpy(vp.reshape(npg, bs, KVH, d)).to(device=device, dtype=dtype)
    q = torch.from_numpy(np.ascontiguousarray(q_pack)).to(device=device, dtype=dtype)
    pages = list(range(npg))
    table = BlockTable([pages] * nq, [t - bs * (npg - 1)] * nq, bs)
    plan = PatPlan.from_units(table, [(tuple(range(nq)), tuple(pages), t)], H, KVH, d, all_partials=True,
                              forward_only=True)
    try:
        ws = torch.zeros(max(plan.workspace_bytes(), 256), dtype=torch.uint8, device=device)
        pat_attention(plan, q, kc, vc, workspace=ws, scale=scale)
        torch.cuda.synchronize(q.device)
    finally:
        plan.close()
    so = (nq * H * d * 4 + 255) // 256 * 256
    o = ws[:nq * H * d * 4].view(torch.float32).view(nq, H, d).double().cpu().numpy()
    lse2 = ws[so:so + nq * H * 4].view(torch.float32).view(nq, H).double().cpu().numpy()
    return PartialBatch(max_score=lse2 * math.log(2.0), exp_sum=np.ones((nq, H)), weighted_sum=o)


def merge_partials(parts: Sequence[PartialResult]) -> np.ndarray:
    """Online-softmax combine of one (query, head)'s partials (``attention.py:166-184``):
    every partial rescaled to the common peak before summing."""
    if not parts:
        raise EmptyPartialList("nothing to merge")
    top = max(p.max_score for p in parts)
    w = [math.exp(p.max_score - top) for p in parts]
    den = sum(p.exp_sum * f for p, f in zip(parts, w))
    if not den > 0.0:
        raise NonPositiveDenominator(f"merged exp-sum is {den}")
    num = sum((p.weighted_sum * f for p, f in zip(parts, w)), np.zeros_like(parts[0].weighted_sum, dtype=np.float64))
    return num / den


def full_attention(q, keys, values, scale: Optional[float] = None, device="cuda") -> np.ndarray:
    """Monolithic softmax attention of each query over its own K / V
    (``attention.py:70-102``), float64 on the GPU."""
    import torch

    q = np.asarray(q)
    if q.ndim != 3:
        raise ShapeMismatch(f"q must be [queries, heads, d], got {q.shape}")
    if len(keys) != q.shape[0] or len(values) != q.shape[0]:
        raise ShapeMismatch("need one K and one V per query")
    H, d = q.shape[1], q.shape[2]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    out = np.empty(q.shape, dtype=np.float64)
    for i in range(q.shape[0]):
        k, v = np.asarray(keys[i]), np.asarray(values[i])
        if k.shape != v.shape or k.ndim != 3 or k.shape[2] != d:
            raise ShapeMismatch(f"bad K/V shapes for query {i}: {k.shape} vs {v.shape}")
        if H % k.shape[1]:
            raise ShapeMismatch("num_heads must be a multiple of kv_heads")
        G = H // k.shape[1]
        kt = torch.from_numpy(k).to(device=device, dtype=torch.float64)
        vt = torch.from_numpy(v).to(device=device, dtype=torch.float64)
        qt = torch.from_numpy(q[i]).to(device=device, dtype=torch.float64).view(k.shape[1], G, d)
        s = torch.einsum("kgd,tkd->kgt", qt, kt) * scale
        p = torch.softmax(s, dim=-1)
        out[i] = torch.einsum("kgt,tkd->kgd", p, vt).reshape(H, d).cpu().numpy()
    return out


def max_rel_error(result: np.ndarray, reference: np.ndarray) -> float:
    """max |result - reference| / max |reference| (``attention.py:272-275``)."""
    ref = np.asarray(reference)
    return float(np.max(np.abs(np.asarray(result) - ref))) / max(float(np.max(np.abs(ref))), 1e-300)


def generate_qkv(table: BlockTable, spec: WorkloadSpec, seed: int):
    """Seeded Q [B, H, d] then, per sorted block id, K and V [bs, KVH, d] ~ N(0, 1)
    (``attention.py:34-48``): the tensors do not depend on how the batch is packed."""
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((table.num_queries, spec.num_heads, spec.head_dim))
    shape = (table.block_size, spec.num_kv_heads, spec.head_dim)
    store = {}
    for b in sorted({b for row in table.rows for b in row}):
        k = rng.standard_normal(shape)
        store[b] = (k, rng.standard_normal(shape))
    return q, store


def gather_kv(table: BlockTable, store: dict, query: int):
    """A query's K / V [kv_len, KVH, d] from its blocks (``attention.py:51-58``)."""
    n = table.kv_len(query)
    k = np.concatenate([store[b][0] for b in table.rows[query]], axis=0)[:n]
    v = np.concatenate([store[b][1] for b in table.rows[query]], axis=0)[:n]
    return k, v


_PPK_MAGIC = b"PPK1"
_PPK_CODE = {np.dtype(np.float64): 0, np.dtype(np.float32): 1}


def dump_tensors(path, tensors: dict) -> None:
    """PPK1 (``attention.py:283-300``): magic, u32 count, then per tensor u16 name
    length, name, u8 dtype code (0 f64, 1 f32), u8 ndim, u64 dims, little-endian data."""
    with open(path, "wb") as fh:
        fh.write(_PPK_MAGIC + struct.pack("<I", len(tensors)))
        for name, arr in tensors.items():
            a = np.ascontiguousarray(arr)
            if a.dtype not in _PPK_CODE:
                a = a.astype(np.float64)
            nb = name.encode("utf-8")
            fh.write(struct.pack("<H", len(nb)) + nb + struct.pack("<BB", _PPK_CODE[a.dtype], a.ndim))
            fh.write(struct.pack(f"<{a.ndim}Q", *a.shape))
            fh.write(a.astype(a.dtype.newbyteorder("<")).tobytes())


def load_tensors(path) -> dict:
    """Read a PPK1 dump (``attention.py:303-315``)."""
    dtypes = {v: k for k, v in _PPK_CODE.items()}
    out = {}
    with open(path, "rb") as fh:
        if fh.read(4) != _PPK_MAGIC:
            raise ValueError("not a tensor dump")
        (count,) = struct.unpack("<I", fh.read(4))
        for _ in range(count):
            (ln,) = struct.unpack("<H", fh.read(2))
            name = fh.read(ln).decode("utf-8")
            code, ndim = struct.unpack("<BB", fh.read(2))
            shape = struct.unpack(f"<{ndim}Q", fh.read(8 * ndim))
            dt = dtypes[code]
            data = fh.read(int(np.prod(shape)) * dt.itemsize)
            out[name] = np.frombuffer(data, dtype=dt.newbyteorder("<")).reshape(shape).astype(dt)
    return out


__all__ = ["PartialResult", "PartialBatch", "cta_partial", "merge_partials", "full_attention", "max_rel_error",
           "generate_qkv", "gather_kv", "dump_tensors", "load_tensors"]
