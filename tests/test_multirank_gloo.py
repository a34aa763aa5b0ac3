"""World-size-2 CPU tests (gloo) of the multi-GPU host logic: every rank builds
the same plan from the same table; kv-head shards computed independently and
all-gathered equal the unsharded layer (numerics by the CPU oracle, standing in
for the per-GPU kernel which the gpu tests cover)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_22333_b200 import configs
from paper_2511_22333_b200.shard import gather_heads, head_shard, request_groups


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_22333_b200 as P
        from oracle import attn_oracle as AO

        w = configs.workload("c1")
        table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        sh = head_shard(w.num_heads, w.num_kv_heads, world, rank)
        plan = P.PatPlan.from_table(table, sh.num_heads, sh.num_kv_heads, w.head_dim, host_only=True)
        packs = plan.pack_tuples()
        plan.close()
        allp = [None] * world
        dist.all_gather_object(allp, packs)
        same_plan = all(p == allp[0] for p in allp)
        # same global inputs on every rank, each computes its head slice
        q, store = AO.generate_qkv(w.rows, w.block_size, w.num_heads, w.num_kv_heads, 64, seed=3)
        ql = q[:, sh.q_begin:sh.q_end]
        st = {b: (k[:, sh.kv_begin:sh.kv_end], v[:, sh.kv_begin:sh.kv_end]) for b, (k, v) in store.items()}
        units = [(p[0], p[1], p[2]) for p in packs]
        local = AO.run_packed(ql, st, units, sh.num_heads, 64)
        full = gather_heads(torch.from_numpy(local), sh).numpy()
        if rank == 0:
            ref = AO.run_packed(q, store, units, w.num_heads, 64)
            results["err"] = float(np.max(np.abs(full - ref)))
            results["same_plan"] = same_plan
        # max-over-ranks reduction used by bench.py
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            results["max"] = float(t.item())
    finally:
        dist.destroy_process_group()


def test_two_rank_kv_head_shard_matches_unsharded():
    port = _free_port()
    with mp.Manager() as m:
        res = m.dict()
        mp.spawn(_worker, args=(2, port, res), nprocs=2, join=True)
        assert res["same_plan"]
        assert res["err"] < 1e-12
        assert res["max"] == 2.0


def test_head_shard_layout():
    sh = [head_shard(64, 8, 8, r) for r in range(8)]
    assert [s.kv_begin for s in sh] == list(range(8))
    assert all(s.num_heads == 8 for s in sh)
    assert sh[3].q_begin == 24 and sh[3].q_end == 32
    with pytest.raises(ValueError):
        head_shard(32, 8, 3, 0)


def test_request_groups_keep_trees_whole():
    rows = [[0, 1, 2], [0, 1, 3], [5, 6], [5, 7], [9], [10, 11, 12, 13]]
    groups = request_groups(rows, 2)
    assert sorted(q for g in groups for q in g) == list(range(6))
    for g in groups:
        firsts = {rows[q][0] for q in g}
        for other in groups:
            if other is not g:
                assert not firsts & {rows[q][0] for q in other}
