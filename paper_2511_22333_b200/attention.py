"""Forward + merge of the drop-in surface.

* ``run_packed_attention`` -- same signature and semantics as the reference
  (``attention.py:202-239``): any Partition / [CtaTask] / [CtaPack], a
  ``{block_id: (K, V)}`` store and numpy Q in; numpy [B, H, d] out.  Inputs are
  rounded to fp16 (or bf16) and the attention runs in libpatb200 on the GPU.
* ``pat_attention`` / ``PatDecoder`` -- the tensor API a serving engine calls:
  Q [B, H, d], paged caches [num_blocks, page, KVH, d] (vLLM NHD layout), block
  tables + seq lens; lazy plan reuse keyed by the table fingerprint
  (``packer.py:189-221``).
"""

from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence, Union

import numpy as np
import torch

from . import _native as N
from .errors import CoverageGap, ShapeMismatch
from .packer import CtaTask, PackCache
from .plan import PatPlan
from .workload import BlockTable, CtaPack, Partition, WorkloadSpec

_DTYPES = {torch.float16: N.PAT_DTYPE_F16, torch.bfloat16: N.PAT_DTYPE_BF16}


def _coverage_units(parts) -> list:
    items = parts.packs if isinstance(parts, Partition) else list(parts)
    units = []
    for it in items:
        if isinstance(it, CtaTask) or type(it).__name__ == "CtaTask":
            units.append((tuple(it.queries), tuple(it.block_ids), int(it.kv_len)))
        elif isinstance(it, CtaPack) or type(it).__name__ == "CtaPack":
            units.append((tuple(it.query_ids), tuple(it.block_ids), int(it.kv_len)))
        else:
            raise TypeError(f"cannot interpret {type(it)!r} as a coverage unit")
    return units


def pat_attention(plan: PatPlan, q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor,
                  out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                  scale: Optional[float] = None, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """One decode-attention layer through ``pat_forward`` (stream-ordered, no sync)."""
    if q.dtype not in _DTYPES or k_cache.dtype != q.dtype or v_cache.dtype != q.dtype:
        raise ShapeMismatch("q, k_cache, v_cache must share dtype float16 or bfloat16")
    if q.dim() != 3 or q.shape[1] != plan.num_heads or q.shape[2] != plan.head_dim:
        raise ShapeMismatch(f"q must be [B, {plan.num_heads}, {plan.head_dim}], got {tuple(q.shape)}")
    if k_cache.shape != v_cache.shape or k_cache.dim() != 4 or k_cache.shape[2] != plan.num_kv_heads \
            or k_cache.shape[3] != plan.head_dim:
        raise ShapeMismatch("k_cache/v_cache must be [num_blocks, page, KVH, d]")
    if not (q.is_cuda and k_cache.is_cuda and v_cache.is_cuda):
        raise ShapeMismatch("tensors must be on a CUDA device")
    if not (q.is_contiguous() and k_cache.is_contiguous() and v_cache.is_contiguous()):
        raise ShapeMismatch("tensors must be contiguous")
    # the kernels index q / out by the plan's query ids and map the caches with its page size
    if q.shape[0] != plan.num_queries:
        raise ShapeMismatch(f"Q row count must match the table: {q.shape[0]} != {plan.num_queries}")
    if k_cache.shape[1] != plan.block_size:
        raise ShapeMismatch(f"cache page size {k_cache.shape[1]} != plan block_size {plan.block_size}")
    if out is None:
        out = torch.empty_like(q)
    elif out.shape != q.shape or out.dtype != q.dtype or out.device != q.device or not out.is_contiguous():
        raise ShapeMismatch("out must be a contiguous tensor with q's shape, dtype and device")
    need = plan.workspace_bytes()
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty(max(need, 256), dtype=torch.uint8, device=q.device)
    s = stream if stream is not None else torch.cuda.current_stream(q.device)
    st = N.lib().pat_forward(plan.handle, C.c_void_p(q.data_ptr()), C.c_void_p(k_cache.data_ptr()),
                             C.c_void_p(v_cache.data_ptr()), k_cache.shape[0], C.c_void_p(out.data_ptr()),
                             C.c_void_p(workspace.data_ptr()), workspace.numel() * workspace.element_size(),
                             _DTYPES[q.dtype], float(scale) if scale else 0.0, C.c_void_p(s.cuda_stream))
    N.check(st, "pat_forward")
    return out


class PatDecoder:
    """Serving-side helper: plan cache (lazy update) + reusable workspace."""

    def __init__(self, num_heads: int, num_kv_heads: int, head_dim: int, split: str = "native",
                 device: Union[str, torch.device] = "cuda", tc_min_rows: int = 0):
        self.num_heads, self.num_kv_heads, self.head_dim = num_heads, num_kv_heads, head_dim
        self.split = split
        self.tc_min_rows = tc_min_rows
        self.device = torch.device(device)
        self.cache = PackCache()
        self._ws: Optional[torch.Tensor] = None

    def plan_for(self, table: BlockTable) -> PatPlan:
        fp = table.fingerprint()
        plan = self.cache.lookup(fp)
        if plan is None:
            plan = PatPlan.from_table(table, self.num_heads, self.num_kv_heads, self.head_dim, split=self.split,
                                      tc_min_rows=self.tc_min_rows)
            self.cache.store(fp, plan)
        return plan

    def workspace(self, plan: PatPlan) -> torch.Tensor:
        need = max(plan.workspace_bytes(), 256)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def __call__(self, table: BlockTable, q, k_cache, v_cache, out=None, scale=None):
        plan = self.plan_for(table)
        return pat_attention(plan, q, k_cache, v_cache, out=out, workspace=self.workspace(plan), scale=scale)

    # -- device block tables (vLLM layout) ---------------------------------------------
    def table_hash(self, block_tables, seq_lens, block_size: int = 16, stream=None) -> int:
        """Device fingerprint of (block_tables [B, max_blocks], seq_lens [B]) int32 CUDA
        tensors (``pat_table_hash_device``), read back through pinned memory (one
        event wait -- the only host sync of the device lazy-update path)."""
        bt = block_tables.contiguous()
        sl = seq_lens.contiguous()
        s = stream if stream is not None else torch.cuda.current_stream(bt.device)
        if getattr(self, "_hash_dev", None) is None or self._hash_dev.device != bt.device:
            self._hash_dev = torch.empty(1, dtype=torch.int64, device=bt.device)
            self._hash_host = torch.empty(1, dtype=torch.int64).pin_memory()
        N.check(N.lib().pat_table_hash_device(bt.shape[0], C.c_void_p(bt.data_ptr()), bt.stride(0),
                                              C.c_void_p(sl.data_ptr()), block_size,
                                              C.c_void_p(self._hash_dev.data_ptr()), C.c_void_p(s.cuda_stream)),
                "pat_table_hash_device")
        with torch.cuda.stream(s):
            self._hash_host.copy_(self._hash_dev, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(s)
        ev.synchronize()
        return int(self._hash_host.item()) & 0xFFFFFFFFFFFFFFFF

    def plan_for_device(self, block_tables, seq_lens, block_size: int = 16) -> PatPlan:
        """Lazy update for device tables: reuse the plan while the device fingerprint
        is unchanged, else re-plan with the GPU packer (``pat_plan_create_device``).
        Every layer of a decode step passes the same (unmodified) table tensors: those
        calls skip even the fingerprint (tensor identity + autograd version counter)."""
        ident = (block_tables.data_ptr(), block_tables._version, tuple(block_tables.shape), seq_lens.data_ptr(),
                 seq_lens._version, block_size)
        last = getattr(self, "_last_dev", None)
        if last is not None and last[0] == ident and last[1]._h:
            return last[1]
        key = f"dev:{self.table_hash(block_tables, seq_lens, block_size):016x}"
        plan = self.cache.lookup(key)
        if plan is None:
            plan = PatPlan.from_device_table(block_tables, seq_lens, block_size, self.num_heads, self.num_kv_heads,
                                             self.head_dim, split=self.split, tc_min_rows=self.tc_min_rows)
            self.cache.store(key, plan)
        self._last_dev = (ident, plan)
        return plan

    def forward_device(self, block_tables, seq_lens, q, k_cache, v_cache, out=None, scale=None):
        """Decode attention straight from vLLM-style device block tables."""
        if block_tables.dim() != 2 or block_tables.shape[0] != q.shape[0] or seq_lens.shape[0] != q.shape[0]:
            raise ShapeMismatch(f"Q row count must match the table: q {tuple(q.shape)}, block_tables "
                                f"{tuple(block_tables.shape)}, seq_lens {tuple(seq_lens.shape)}")
        plan = self.plan_for_device(block_tables, seq_lens, k_cache.shape[1])
        return pat_attention(plan, q, k_cache, v_cache, out=out, workspace=self.workspace(plan), scale=scale)


class PatDeviceDecoder:
    """Serving path with planning on the GPU (``pat_decoder``, ``include/pat.h``).

    ``forward(block_tables, seq_lens, q, k_cache, v_cache)`` enqueues the table
    fingerprint, its comparison with the last one, the GPU packer and the device
    scheduler (skipped on the device when the table is unchanged) and the
    forward + merge kernels -- no host synchronisation, no allocation -- so a
    decode step can be captured in a CUDA graph once and replayed while vLLM
    rewrites its block table in place.  Capacity: ``max_batch`` <= 4096 queries
    of <= ``max_blocks`` pages."""

    def __init__(self, num_heads: int, num_kv_heads: int, head_dim: int, max_batch: int, max_blocks: int,
                 block_size: int = 16, device: Union[str, torch.device] = "cuda"):
        self.num_heads, self.num_kv_heads, self.head_dim = num_heads, num_kv_heads, head_dim
        self.max_batch, self.max_blocks, self.block_size = max_batch, max_blocks, block_size
        self.device = torch.device(device)
        opt = PatPlan._opts(num_heads, num_kv_heads, head_dim, "native", False)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            N.check(N.lib().pat_decoder_create(C.byref(opt), max_batch, max_blocks, block_size, C.byref(h)),
                    "pat_decoder_create")
        self._h = h
        need = int(N.lib().pat_decoder_workspace_bytes(h))
        self.workspace = torch.zeros(need, dtype=torch.uint8, device=self.device)
        self._last_table = None

    def fits(self, block_tables) -> bool:
        return block_tables.shape[0] <= self.max_batch and block_tables.shape[1] <= self.max_blocks

    def forward(self, block_tables, seq_lens, q, k_cache, v_cache, out=None, scale=None, stream=None,
                same_table=None):
        """Every layer of a decode step passes the same (unmodified) table tensors:
        those calls skip even the device fingerprint (tensor identity + autograd
        version counter, the PAT_DECODE_SAME_TABLE flag).  ``same_table=True``
        asserts it explicitly (the table is the one the previous call planned);
        ``False`` forces the fingerprint."""
        if q.dtype not in _DTYPES or k_cache.dtype != q.dtype or v_cache.dtype != q.dtype:
            raise ShapeMismatch("q, k_cache, v_cache must share dtype float16 or bfloat16")
        if q.dim() != 3 or q.shape[1] != self.num_heads or q.shape[2] != self.head_dim:
            raise ShapeMismatch(f"q must be [B, {self.num_heads}, {self.head_dim}], got {tuple(q.shape)}")
        if block_tables.dim() != 2 or block_tables.shape[0] != q.shape[0] or seq_lens.shape[0] != q.shape[0]:
            raise ShapeMismatch("Q row count must match the table")
        if block_tables.dtype != torch.int32 or seq_lens.dtype != torch.int32 or block_tables.stride(1) != 1:
            raise ShapeMismatch("block_tables / seq_lens must be int32 with unit column stride")
        if k_cache.shape != v_cache.shape or k_cache.dim() != 4 or k_cache.shape[1] != self.block_size \
                or k_cache.shape[2] != self.num_kv_heads or k_cache.shape[3] != self.head_dim:
            raise ShapeMismatch("k_cache/v_cache must be [num_blocks, page, KVH, d]")
        if not (q.is_contiguous() and k_cache.is_contiguous() and v_cache.is_contiguous()
                and seq_lens.is_contiguous()):
            raise ShapeMismatch("tensors must be contiguous")
        if out is None:
            out = torch.empty_like(q)
        elif out.shape != q.shape or out.dtype != q.dtype or not out.is_contiguous():
            raise ShapeMismatch("out must be a contiguous tensor with q's shape and dtype")
        s = stream if stream is not None else torch.cuda.current_stream(q.device)
        # the identity shortcut is only sound while every plan change goes through
        # these calls: once the decoder has been captured in a CUDA graph (whose
        # replays re-plan on the device, invisibly to this object) it is not used
        # again; inside one capture it still applies from the second call on
        capturing = torch.cuda.is_current_stream_capturing()
        if capturing and not getattr(self, "_capturing", False):
            self._last_table = None
        self._capturing = capturing
        self._captured = getattr(self, "_captured", False) or capturing
        ident = (block_tables.data_ptr(), block_tables._version, tuple(block_tables.shape), block_tables.stride(0),
                 seq_lens.data_ptr(), seq_lens._version)
        if same_table is None:
            same_table = ident == self._last_table and (capturing or not self._captured)
        flags = N.PAT_DECODE_SAME_TABLE if same_table else 0
        N.check(N.lib().pat_decoder_forward(
            self._h, C.c_void_p(block_tables.data_ptr()), block_tables.stride(0), C.c_void_p(seq_lens.data_ptr()),
            q.shape[0], block_tables.shape[1], C.c_void_p(q.data_ptr()), C.c_void_p(k_cache.data_ptr()),
            C.c_void_p(v_cache.data_ptr()), k_cache.shape[0], C.c_void_p(out.data_ptr()),
            C.c_void_p(self.workspace.data_ptr()), self.workspace.numel(), _DTYPES[q.dtype],
            float(scale) if scale else 0.0, flags, C.c_void_p(s.cuda_stream)), "pat_decoder_forward")
        self._last_table = ident
        return out

    def status(self, stream=None) -> int:
        """Synchronise; raise the packer's error for the last table (InvalidSpec, ...);
        return how many times the device re-planned."""
        n = C.c_int32(0)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        N.check(N.lib().pat_decoder_status(self._h, C.c_void_p(s.cuda_stream), C.byref(n)), "pat_decoder")
        return int(n.value)

    def close(self):
        if getattr(self, "_h", None):
            N.lib().pat_decoder_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PatLayerGraph:
    """One decode-attention layer captured as a CUDA graph (the multi-stream
    fork/join inside ``pat_forward`` is captured too); ``replay()`` re-runs it on
    the same buffers with a single launch.  The plan and tensors must stay alive
    and in place (lazy update: rebuild the graph when the plan changes)."""

    def __init__(self, plan: PatPlan, q, k_cache, v_cache, out=None, workspace=None, scale=None):
        self.plan, self.q, self.k_cache, self.v_cache = plan, q, k_cache, v_cache
        self.out = out if out is not None else torch.empty_like(q)
        need = max(plan.workspace_bytes(), 256)
        self.ws = workspace if workspace is not None else torch.empty(need, dtype=torch.uint8, device=q.device)
        self.scale = scale
        # warm-up outside capture: kernel attributes, tensor maps, side streams
        pat_attention(plan, q, k_cache, v_cache, out=self.out, workspace=self.ws, scale=scale)
        torch.cuda.synchronize(q.device)
        self.graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(q.device)
        s.wait_stream(torch.cuda.current_stream(q.device))
        with torch.cuda.stream(s):
            with torch.cuda.graph(self.graph, stream=s):
                pat_attention(plan, q, k_cache, v_cache, out=self.out, workspace=self.ws, scale=scale, stream=s)
        torch.cuda.current_stream(q.device).wait_stream(s)

    def replay(self):
        self.graph.replay()
        return self.out


def kv_pool_from_store(kv_store: dict, block_size: int, dtype=torch.float16, device="cuda"):
    """Paged caches [max_id + 1, page, KVH, d] from the reference ``{id: (K, V)}`` store."""
    ids = sorted(kv_store)
    k0 = np.asarray(kv_store[ids[0]][0])
    nb = ids[-1] + 1
    kh = np.zeros((nb,) + k0.shape, dtype=np.float32)
    vh = np.zeros((nb,) + k0.shape, dtype=np.float32)
    for b in ids:
        kh[b] = kv_store[b][0]
        vh[b] = kv_store[b][1]
    if kh.shape[1] != block_size:
        raise ShapeMismatch(f"store blocks hold {kh.shape[1]} tokens, table block_size is {block_size}")
    return (torch.from_numpy(kh).to(device=device, dtype=dtype), torch.from_numpy(vh).to(device=device, dtype=dtype))


def run_packed_attention(table: BlockTable, partition_or_tasks: Union[Partition, Sequence[CtaTask], Sequence[CtaPack]],
                         kv_store: dict, q: np.ndarray, spec: WorkloadSpec, intermediate_dtype=None,
                         *, dtype: torch.dtype = torch.float16, split: str = "none",
                         device: Union[str, torch.device] = "cuda", tc_min_rows: int = 0) -> np.ndarray:
    """Drop-in for ``prefixpack.run_packed_attention`` (``attention.py:202-239``).

    Coverage is checked natively (``CoverageGap``); partials are always fp32 on
    the device, so ``intermediate_dtype`` is accepted and has no further effect.
    Returns float64 [B, H, d] like the reference (computed from ``dtype`` inputs)."""
    del intermediate_dtype
    units = _coverage_units(partition_or_tasks)
    q = np.asarray(q)
    if q.ndim != 3 or q.shape[0] != table.num_queries:
        raise ShapeMismatch("Q row count must match the table")
    if table.num_queries == 0:
        return np.zeros(q.shape, dtype=np.float64)
    plan = PatPlan.from_units(table, units, spec.num_heads, spec.num_kv_heads, spec.head_dim, split=split,
                              tc_min_rows=tc_min_rows)
    try:
        kc, vc = kv_pool_from_store(kv_store, table.block_size, dtype, device)
        qt = torch.from_numpy(np.ascontiguousarray(q, dtype=np.float32)).to(device=device, dtype=dtype)
        out = pat_attention(plan, qt, kc, vc)
        torch.cuda.synchronize(qt.device)
        return out.to(torch.float64).cpu().numpy()
    finally:
        plan.close()


__all__ = ["run_packed_attention", "pat_attention", "PatDecoder", "PatLayerGraph", "kv_pool_from_store",
           "CoverageGap"]
