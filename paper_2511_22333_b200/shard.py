"""Multi-GPU partitioning of one decode-attention layer.

The pack plan never reads head counts (``tree_heuristic`` is head-free,
``packer.py:124-161``), so every rank builds the same plan from the same block
tables and runs it on its own slice of the heads:

* KV-head sharding (default): rank r owns kv heads [r*KVH/N, (r+1)*KVH/N) and
  their G query heads each -- no communication on the attention path;
* request-group sharding when ranks outnumber kv heads: whole forest roots
  (independent prefix trees, ``packer.py:164-168``) are dealt to rank groups
  so that no shared prefix is split across GPUs (which would need a cross-GPU
  LSE merge).

The only collective is the optional output all-gather along heads.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    kv_begin: int
    kv_end: int
    q_begin: int
    q_end: int

    @property
    def num_kv_heads(self) -> int:
        return self.kv_end - self.kv_begin

    @property
    def num_heads(self) -> int:
        return self.q_end - self.q_begin


def head_shard(num_heads: int, num_kv_heads: int, world: int, rank: int) -> HeadShard:
    """Contiguous kv-head slice of ``rank``; its query heads follow the GQA map
    h -> h // G (``attention.py:61-67``)."""
    if num_kv_heads % world:
        raise ValueError(f"{world} ranks do not divide {num_kv_heads} kv heads; use request_groups()")
    G = num_heads // num_kv_heads
    per = num_kv_heads // world
    kb, ke = rank * per, (rank + 1) * per
    return HeadShard(rank, world, kb, ke, kb * G, ke * G)


def request_groups(rows, world: int):
    """Deal whole prefix trees (roots = groups of rows sharing their first block)
    to ``world`` groups, largest first, balancing total tokens.  Returns a list of
    query-id lists (one per group)."""
    roots: dict = {}
    for q, r in enumerate(rows):
        roots.setdefault(r[0], []).append(q)
    trees = sorted(roots.values(), key=lambda qs: -sum(len(rows[q]) for q in qs))
    load = [0] * world
    out = [[] for _ in range(world)]
    for qs in trees:
        g = int(np.argmin(load))
        out[g].extend(qs)
        load[g] += len({b for q in qs for b in rows[q]})
    return [sorted(x) for x in out]


def gather_heads(local_out, shard: HeadShard, group=None):
    """All-gather head-sharded outputs [B, H/N, d] into [B, H, d] (NCCL over
    NVLink on GPUs; gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist

    parts = [torch.empty_like(local_out) for _ in range(shard.world)]
    dist.all_gather(parts, local_out.contiguous(), group=group)
    return torch.cat(parts, dim=1)
