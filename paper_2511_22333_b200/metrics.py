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
