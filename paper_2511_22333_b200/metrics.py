"""Roofline numerator (``simulator.py:25-27, 68-82``): the algorithmic HBM bytes
of one decode-attention layer are the distinct KV tokens x KVH x d x 2 (K, V) x b."""

from __future__ import annotations

from .workload import BlockTable, WorkloadSpec


def kv_token_bytes(spec: WorkloadSpec) -> int:
    return spec.head_dim * spec.kv_dtype_bytes * 2 * spec.num_kv_heads


def distinct_block_census(table: BlockTable):
    """(distinct blocks, distinct tokens); a block shared at several fills counts
    at its fullest use."""
    best: dict = {}
    for q in range(table.num_queries):
        for b, t in table.row_units(q):
            if best.get(b, 0) < t:
                best[b] = t
    return len(best), sum(best.values())


def theoretical_min_kv_bytes(table: BlockTable, spec: WorkloadSpec) -> int:
    return distinct_block_census(table)[1] * kv_token_bytes(spec)


def intermediate_round_trip_bytes(spec: WorkloadSpec) -> int:
    """One fp32 partial write + one merge read of a query's H x d weighted sums
    (``simulator.py:30-34``)."""
    return 2 * spec.head_dim * spec.num_heads * spec.intermediate_dtype_bytes


class TrafficReport:
    """Modeled HBM bytes of a partition (``simulator.py:37-44``)."""

    __slots__ = ("kv_bytes", "intermediate_bytes")

    def __init__(self, kv_bytes: int, intermediate_bytes: int):
        self.kv_bytes, self.intermediate_bytes = int(kv_bytes), int(intermediate_bytes)

    @property
    def total_bytes(self) -> int:
        return self.kv_bytes + self.intermediate_bytes

    def __eq__(self, other):
        return isinstance(other, TrafficReport) and (self.kv_bytes, self.intermediate_bytes) == \
            (other.kv_bytes, other.intermediate_bytes)

    def __repr__(self):
        return f"TrafficReport(kv_bytes={self.kv_bytes}, intermediate_bytes={self.intermediate_bytes})"


def account_traffic(partition, spec: WorkloadSpec) -> TrafficReport:
    """Modeled traffic (``simulator.py:55-65``): every pack's span once, plus one
    intermediate round trip per pack membership of a query that sits in two or
    more packs (single-pack queries write their output directly).  The B200
    counterpart measured by ncu is in ``profiles/*_traffic_*.json``."""
    from collections import Counter

    kv = sum(p.kv_len for p in partition.packs) * kv_token_bytes(spec)
    seen = Counter(q for p in partition.packs for q in p.query_ids)
    rt = intermediate_round_trip_bytes(spec)
    return TrafficReport(kv, sum(n * rt for n in seen.values() if n >= 2))
