"""``PatPlan``: owner of a native plan (libpatb200 ``pat_plan``).

A plan is the reference Partition (``pack_batch`` order) refined into forward
units (after the KV split) and CTA work items; it lives on the host for
inspection and in device memory for ``pat_forward``."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import InvalidSpec


@dataclass
class PlanArrays:
    q_off: np.ndarray
    q_ids: np.ndarray
    blk_off: np.ndarray
    blk_ids: np.ndarray
    kv_len: np.ndarray
    partial: np.ndarray


class PatPlan:
    """RAII wrapper of ``pat_plan*``."""

    def __init__(self, handle: C.c_void_p, num_heads: int, num_kv_heads: int, head_dim: int):
        self._h = handle
        self.num_heads = num_heads
        self.num_kv_heads = num_kv_heads
        self.head_dim = head_dim
        inf = self.info()
        self.num_queries = int(inf.num_queries)  # rows of q / out the kernels index
        self.block_size = int(inf.block_size)    # page size the KV tensor maps use

    # -- construction ---------------------------------------------------------------
    @staticmethod
    def _opts(num_heads, num_kv_heads, head_dim, split, host_only, num_sms=0, tc_min_rows=0, forward_only=False,
              pair_items=False):
        if split not in N.SPLIT_MODES:
            raise InvalidSpec(f"split must be one of {sorted(N.SPLIT_MODES)}")
        flags = (N.PAT_PLAN_HOST_ONLY if host_only else 0) | (N.PAT_PLAN_FORWARD_ONLY if forward_only else 0) | \
            (N.PAT_PLAN_PAIR_ITEMS if pair_items else 0)
        return N.PlanOptions(num_heads, num_kv_heads, head_dim, N.SPLIT_MODES[split], num_sms, flags, tc_min_rows)

    @classmethod
    def from_table(cls, table, num_heads=32, num_kv_heads=8, head_dim=128, split="native", host_only=False,
                   num_sms=0, tc_min_rows=0, forward_only=False, pair_items=False) -> "PatPlan":
        """Host C++ packer (``pat_plan_create_host``) on a BlockTable.  ``forward_only``:
        timing aid, ``pat_forward`` skips the merge.  ``pair_items``: PAT_PLAN_PAIR_ITEMS."""
        off, blk, valid = table.csr()
        opt = cls._opts(num_heads, num_kv_heads, head_dim, split, host_only, num_sms, tc_min_rows, forward_only,
                        pair_items)
        h = C.c_void_p()
        st = N.lib().pat_plan_create_host(len(table.rows), N.ptr(off, C.c_int64), N.ptr(blk, C.c_int32),
                                          N.ptr(valid, C.c_int32), table.block_size, C.byref(opt), C.byref(h))
        N.check(st, "pat_plan_create_host")
        return cls(h, num_heads, num_kv_heads, head_dim)

    @classmethod
    def from_device_table(cls, block_tables, seq_lens, block_size=16, num_heads=32, num_kv_heads=8, head_dim=128,
                          split="native", num_sms=0, tc_min_rows=0, stream=None) -> "PatPlan":
        """GPU packer (``pat_plan_create_device``) on device block tables [B, max_blocks]
        and seq lens [B] (int32 CUDA tensors, vLLM layout)."""
        import torch

        if block_tables.dtype != torch.int32 or seq_lens.dtype != torch.int32 or not block_tables.is_cuda:
            raise InvalidSpec("block_tables / seq_lens must be int32 CUDA tensors")
        bt = block_tables.contiguous()
        sl = seq_lens.contiguous()
        opt = cls._opts(num_heads, num_kv_heads, head_dim, split, False, num_sms, tc_min_rows)
        s = stream if stream is not None else torch.cuda.current_stream(bt.device)
        h = C.c_void_p()
        st = N.lib().pat_plan_create_device(bt.shape[0], C.c_void_p(bt.data_ptr()), bt.shape[1],
                                            C.c_void_p(sl.data_ptr()), bt.shape[1], block_size, C.byref(opt),
                                            C.c_void_p(s.cuda_stream), C.byref(h))
        N.check(st, "pat_plan_create_device")
        return cls(h, num_heads, num_kv_heads, head_dim)

    @classmethod
    def from_units(cls, table, units, num_heads=32, num_kv_heads=8, head_dim=128, split="none", host_only=False,
                   num_sms=0, tc_min_rows=0, forward_only=False, all_partials=False) -> "PatPlan":
        """Explicit partition: ``units`` = [(query_ids, block_ids, kv_len)] in fold order.
        ``all_partials`` (PAT_PLAN_ALL_PARTIALS): every (unit, query) writes an fp32
        partial to the workspace (with ``forward_only``, nothing is merged)."""
        off, blk, valid = table.csr()
        uq = [np.asarray(u[0], dtype=np.int32) for u in units]
        ub = [np.asarray(u[1], dtype=np.int32) for u in units]
        uq_off = np.zeros(len(units) + 1, dtype=np.int64)
        ub_off = np.zeros(len(units) + 1, dtype=np.int64)
        np.cumsum([len(x) for x in uq], out=uq_off[1:])
        np.cumsum([len(x) for x in ub], out=ub_off[1:])
        uq_all = np.concatenate(uq) if uq else np.zeros(0, np.int32)
        ub_all = np.concatenate(ub) if ub else np.zeros(0, np.int32)
        ukv = np.asarray([int(u[2]) for u in units], dtype=np.int32)
        opt = cls._opts(num_heads, num_kv_heads, head_dim, split, host_only, num_sms, tc_min_rows, forward_only)
        if all_partials:
            opt.flags |= N.PAT_PLAN_ALL_PARTIALS
        h = C.c_void_p()
        st = N.lib().pat_plan_create_units(len(table.rows), N.ptr(off, C.c_int64), N.ptr(blk, C.c_int32),
                                           N.ptr(valid, C.c_int32), table.block_size, len(units),
                                           N.ptr(uq_off, C.c_int64), N.ptr(uq_all, C.c_int32),
                                           N.ptr(ub_off, C.c_int64), N.ptr(ub_all, C.c_int32),
                                           N.ptr(ukv, C.c_int32), C.byref(opt), C.byref(h))
        N.check(st, "pat_plan_create_units")
        return cls(h, num_heads, num_kv_heads, head_dim)

    # -- inspection ----------------------------------------------------------------
    @property
    def handle(self):
        return self._h

    def info(self) -> N.PlanInfo:
        inf = N.PlanInfo()
        N.check(N.lib().pat_plan_info_get(self._h, C.byref(inf)), "pat_plan_info_get")
        return inf

    def packs(self) -> PlanArrays:
        inf = self.info()
        a = PlanArrays(np.zeros(inf.n_packs + 1, np.int32), np.zeros(inf.n_pack_q, np.int32),
                       np.zeros(inf.n_packs + 1, np.int32), np.zeros(inf.n_pack_blk, np.int32),
                       np.zeros(inf.n_packs, np.int32), np.zeros(inf.n_packs, np.uint8))
        st = N.lib().pat_plan_export_packs(self._h, N.ptr(a.q_off, C.c_int32), N.ptr(a.q_ids, C.c_int32),
                                           N.ptr(a.blk_off, C.c_int32), N.ptr(a.blk_ids, C.c_int32),
                                           N.ptr(a.kv_len, C.c_int32), N.ptr(a.partial, C.c_uint8))
        N.check(st, "pat_plan_export_packs")
        return a

    def pack_tuples(self):
        """[(query_ids, block_ids, kv_len, produces_partial)] in reference order."""
        a = self.packs()
        out = []
        for p in range(len(a.kv_len)):
            out.append((tuple(int(x) for x in a.q_ids[a.q_off[p]:a.q_off[p + 1]]),
                        tuple(int(x) for x in a.blk_ids[a.blk_off[p]:a.blk_off[p + 1]]),
                        int(a.kv_len[p]), bool(a.partial[p])))
        return out

    def units(self):
        """[(pack, page0, npages, ntok, split_index, split_of)]."""
        n = self.info().n_units
        cols = [np.zeros(n, np.int32) for _ in range(6)]
        N.check(N.lib().pat_plan_export_units(self._h, *[N.ptr(c, C.c_int32) for c in cols]), "export_units")
        return [tuple(int(c[i]) for c in cols) for i in range(n)]

    def workspace_bytes(self) -> int:
        return int(N.lib().pat_workspace_bytes(self._h))

    def close(self):
        if self._h:
            N.lib().pat_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
