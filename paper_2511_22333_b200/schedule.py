"""Task planning of the drop-in surface (``prefixpack.simulator.plan_tasks`` /
``assign_streams``, reference ``simulator.py:158-232``), B200-native.

The reference picks a per-pack query tile m from an A100 feasible set,
pre-splits packs wider than m_max into query groups (each re-reading the KV),
splits long KV spans and gives every distinct (m, n) its own stream.  On B200
the native scheduler (``csrc/pat_schedule_host.cpp``) makes those choices:

* rows of a unit = its queries x G (GQA group); units of <= 16 rows run
  transposed on tokens x 16-row MMA tiles over 64-token KV tiles
  (``TileConfig(m=16, n=64)``), wider ones on 128-row tiles over 32-token KV
  tiles (``TileConfig(m=128, n=32)``), a 128-row block of a wide pack per work
  item -- never a query pre-split that re-reads the KV;
* the long-KV split is the native makespan-driven one (``split="native"``) or
  the reference's ``split_long_kv`` (``split="reference"``);
* both tile configs run in ONE persistent kernel with dynamic longest-first
  claims, so ``assign_streams`` groups tasks by config for inspection but the
  forward does not fork streams.

``fs`` / ``n_tree`` (the A100 tile model, out of scope) are accepted and
ignored for signature compatibility."""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

from .errors import NoFeasibleConfig
from .packer import CtaTask
from .plan import PatPlan
from .workload import BlockTable, Partition, WorkloadSpec

NARROW_ROWS = 16  # csrc/pat_fwd_tc4.cu kNarrow


@dataclass(frozen=True)
class TileConfig:
    """B200 tile of a forward unit: m rows per MMA tile, n KV tokens per tile."""

    m: int
    n: int
    kernel: str = "fwd_tc4_kernel"
    concurrency: int = 2  # item pipelines per SM

    def key(self):
        return (self.m, self.n)


def _table_from_partition(partition: Partition, block_size: int) -> BlockTable:
    rows, kv = {}, {}
    for p in partition.packs:
        for q in p.query_ids:
            rows.setdefault(q, []).extend(p.block_ids)
            kv[q] = kv.get(q, 0) + p.kv_len
    nq = max(rows) + 1 if rows else 0
    valid = [kv[q] - block_size * (len(rows[q]) - 1) for q in range(nq)]
    return BlockTable([rows[q] for q in range(nq)], valid, block_size)


def plan_tasks(partition: Partition, fs=None, n_tree=None, spec: Optional[WorkloadSpec] = None,
               force_config=None, split: bool = True, table: Optional[BlockTable] = None) -> list:
    """Forward units of a partition as CtaTasks with their B200 tile config and
    (config) stream id, in fold order."""
    if spec is None:
        raise NoFeasibleConfig("plan_tasks needs the WorkloadSpec (heads, head_dim)")
    if table is None:
        table = _table_from_partition(partition, spec.block_size)
    units = [(p.query_ids, p.block_ids, p.kv_len) for p in partition.packs]
    plan = PatPlan.from_units(table, units, spec.num_heads, spec.num_kv_heads, spec.head_dim,
                              split=("native" if split else "none"), host_only=True)
    try:
        G = spec.num_heads // spec.num_kv_heads
        tasks = []
        for pidx, page0, npages, ntok, sidx, sof in plan.units():
            pack = partition.packs[pidx]
            rows = len(pack.query_ids) * G
            if force_config is not None:
                cfg = TileConfig(*force_config)
            elif rows <= NARROW_ROWS:
                cfg = TileConfig(m=NARROW_ROWS, n=64)
            else:
                cfg = TileConfig(m=128, n=32)
            tasks.append(CtaTask(queries=tuple(pack.query_ids), block_ids=tuple(pack.block_ids[page0:page0 + npages]),
                                 kv_len=ntok, cfg=cfg, pack_index=pidx, split_index=sidx, split_of=sof))
    finally:
        plan.close()
    assign_streams(tasks)
    return tasks


def assign_streams(tasks: Sequence[CtaTask]) -> dict:
    """Group tasks by tile config, one id per distinct (m, n), order kept
    (``simulator.py:158-170``)."""
    keys = sorted({t.cfg.key() for t in tasks if t.cfg is not None})
    sid = {k: i for i, k in enumerate(keys)}
    streams = {i: [] for i in range(len(keys))}
    for t in tasks:
        if t.cfg is None:
            raise NoFeasibleConfig("task has no tile configuration")
        t.stream_id = sid[t.cfg.key()]
        streams[t.stream_id].append(t)
    return streams


__all__ = ["TileConfig", "plan_tasks", "assign_streams"]
