"""Pack stage of the drop-in surface (``prefixpack.packer``, ``packer.py:189-266``).

``pack_batch`` runs the native packer (host C++ ``pat_plan_create_host``; the GPU
pass ``pat_plan_create_device`` serves device block tables) and returns the
reference ``Partition`` -- bit-exact, including query order inside packs,
pack emission order and ``produces_partial``."""

from __future__ import annotations

import math
import threading
from concurrent.futures import Executor, Future, ThreadPoolExecutor
from dataclasses import dataclass, replace
from typing import Optional, Sequence

from .plan import PatPlan
from .workload import BlockTable, CtaPack, Partition, assemble_partition


def pack_batch(table: BlockTable, cache: Optional["PackCache"] = None) -> Partition:
    """Pack a decode batch; reuse the cached partition on a fingerprint hit
    (``packer.py:224-242``)."""
    fp = table.fingerprint()
    if table.num_queries == 0:
        return Partition(packs=(), source_fingerprint=fp)
    if cache is not None:
        hit = cache.lookup(fp)
        if hit is not None:
            return hit
    plan = PatPlan.from_table(table, split="none", host_only=True)
    try:
        packs = tuple(CtaPack(q, b, kv, part) for q, b, kv, part in plan.pack_tuples())
    finally:
        plan.close()
    partition = Partition(packs=packs, source_fingerprint=fp)
    if cache is not None:
        cache.store(fp, partition)
    return partition


class PackCache:
    """Single-slot lazy-update cache keyed by the table fingerprint (``packer.py:189-221``)."""

    def __init__(self):
        self._lock = threading.Lock()
        self._key: Optional[str] = None
        self._value = None
        self.hits = 0
        self.misses = 0

    def lookup(self, fingerprint: str):
        with self._lock:
            if self._key == fingerprint and self._value is not None:
                self.hits += 1
                return self._value
            self.misses += 1
            return None

    def store(self, fingerprint: str, value) -> None:
        with self._lock:
            self._key, self._value = fingerprint, value

    @property
    def stats(self) -> dict:
        with self._lock:
            return {"hits": self.hits, "misses": self.misses}


_POOL: Optional[ThreadPoolExecutor] = None
_POOL_LOCK = threading.Lock()


def pack_batch_async(table: BlockTable, cache: Optional[PackCache] = None,
                     executor: Optional[Executor] = None) -> Future:
    """Run ``pack_batch`` on a worker thread so it overlaps pre-attention work
    (``packer.py:245-266``); the native packer releases the GIL (ctypes)."""
    global _POOL
    if executor is None:
        with _POOL_LOCK:
            if _POOL is None:
                _POOL = ThreadPoolExecutor(max_workers=1, thread_name_prefix="pack")
            executor = _POOL
    return executor.submit(pack_batch, table, cache)


def baseline_query_centric(table: BlockTable) -> Partition:
    """One pack per query over its full row (``simulator.py:85-96``)."""
    return assemble_partition([CtaPack((q,), tuple(table.rows[q]), table.kv_len(q))
                               for q in range(table.num_queries)], table)


# --------------------------------------------------------------------------------------
# forward units (CtaTask) and the reference long-KV split
# --------------------------------------------------------------------------------------

@dataclass
class CtaTask:
    """A forward unit: queries x contiguous KV span (``simulator.py:99-114``).
    ``cfg``/``stream_id`` are kept for signature compatibility; on B200 the kernel
    variant and its stream are chosen by the native scheduler."""

    queries: tuple
    block_ids: tuple
    kv_len: int
    cfg: object = None
    stream_id: Optional[int] = None
    pack_index: int = 0
    split_index: int = 0
    split_of: int = 1

    @property
    def q(self) -> int:
        return len(self.queries)


def split_long_kv(tasks: Sequence[CtaTask], block_size: int) -> list:
    """Reference long-KV split (``simulator.py:117-155``): tasks longer than the
    mean become ceil(kv/mean) (capped at #blocks) block-aligned parts, larger
    parts first, the last carrying the partial block."""
    if not tasks:
        return []
    mean = sum(t.kv_len for t in tasks) / len(tasks)
    out = []
    for t in tasks:
        if t.kv_len <= mean:
            out.append(t)
            continue
        nblk = max(len(t.block_ids), math.ceil(t.kv_len / block_size))
        parts = min(math.ceil(t.kv_len / mean), nblk)
        size, rem = divmod(nblk, parts)
        pos = done = 0
        for i in range(parts):
            n = size + (i < rem)
            tok = min(n * block_size, t.kv_len - done)
            out.append(replace(t, block_ids=t.block_ids[pos:pos + n] if t.block_ids else (), kv_len=tok,
                               split_index=i, split_of=parts))
            pos, done = pos + n, done + tok
    return out


def naive_per_node(table: BlockTable) -> Partition:
    """PAT-naive ablation (``packer.py:171-186``): one pack per forest node over its
    own run, queries of its subtree, nodes in pre-order."""
    from .forest import build_forest

    packs = [CtaPack(tuple(n.subtree_queries()), tuple(n.block_ids), n.token_len)
             for n in build_forest(table).iter_nodes() if n.token_len]
    return assemble_partition(packs, table)
