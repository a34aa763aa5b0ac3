"""Kernel-variant coverage on the GPU: every pack forced onto the tcgen05 kernel
(tc_min_rows=1) or onto the mma.sync streaming kernel (tc_min_rows=-1), over the
reference fixtures and sampled full-size configs."""

import random

import numpy as np
import pytest
import torch

import paper_2511_22333_b200 as P
from paper_2511_22333_b200 import configs
from paper_2511_22333_b200.plan import PatPlan
from oracle import attn_oracle as AO

from golden_io import numerics
from test_gpu_parity import TDT, _close, _inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tc", [1, -1, 64])
def test_small_fixtures_variant(tc):
    meta, z = numerics("numerics_small.npz")
    for m in meta:
        table = P.BlockTable([list(r) for r in m["rows"]], list(m["valid"]), m["bs"])
        spec = P.WorkloadSpec((1,), (16,), num_heads=m["H"], num_kv_heads=m["KVH"], head_dim=m["d"])
        q, store = _inputs(m["rows"], m["bs"], m["H"], m["KVH"], m["d"], m["seed"], m["dtype"], m["qscale"])
        ref = z[m["key"] + "_packed"].astype(np.float64)
        for split in ("none", "native"):
            out = P.run_packed_attention(table, P.pack_batch(table), store, q, spec, dtype=TDT[m["dtype"]],
                                         split=split, tc_min_rows=tc)
            _close(out, ref)
        out = P.run_packed_attention(table, P.baseline_query_centric(table), store, q, spec,
                                     dtype=TDT[m["dtype"]], tc_min_rows=tc)
        _close(out, z[m["key"] + "_full"].astype(np.float64))


@pytest.mark.parametrize("key", ["c1_float16", "c1_bfloat16", "c2_float16"])
@pytest.mark.parametrize("tc", [1, -1])
def test_config_fixtures_variant(key, tc):
    meta, z = numerics("numerics_c1c2.npz")
    m = next(x for x in meta if x["key"] == key)
    w = configs.workload(m["config"])
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    spec = P.WorkloadSpec((1,), (16,), num_heads=w.num_heads, num_kv_heads=w.num_kv_heads, head_dim=w.head_dim)
    q, store = _inputs(w.rows, w.block_size, w.num_heads, w.num_kv_heads, w.head_dim, 0, m["dtype"])
    out = P.run_packed_attention(table, P.pack_batch(table), store, q, spec, dtype=TDT[m["dtype"]], split="native",
                                 tc_min_rows=tc)
    _close(out, z[key].astype(np.float64))


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_tc_full_configs_sampled(name, nsample=4):
    w = configs.workload(name)
    g = torch.Generator(device="cuda").manual_seed(7)
    nb = w.num_pool_blocks()
    dt = torch.bfloat16
    kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    vc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=dt, generator=g) * 3
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    outs = {}
    for tc in (64, -1):
        plan = PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim, split="native", tc_min_rows=tc)
        outs[tc] = P.pat_attention(plan, q, kc, vc)
        torch.cuda.synchronize()
        plan.close()
    rng = random.Random(3)
    for qi in sorted(rng.sample(range(w.batch), nsample)):
        row = w.rows[qi]
        n = (len(row) - 1) * w.block_size + w.valid_last[qi]
        idx = torch.tensor(row, device="cuda")
        k = kc[idx].reshape(-1, w.num_kv_heads, w.head_dim)[:n].double().cpu().numpy()
        v = vc[idx].reshape(-1, w.num_kv_heads, w.head_dim)[:n].double().cpu().numpy()
        ref = AO.full_attention(q[qi:qi + 1].double().cpu().numpy(), [k], [v])[0]
        for tc in outs:
            _close(outs[tc][qi].double().cpu().numpy(), ref)


@pytest.mark.parametrize("name", ["c4"])
@pytest.mark.parametrize("tc", [64, -1])
def test_variant_configs_vs_oracle(name, tc):
    """Same as above, one kernel mix at a time (diagnostic granularity)."""
    w = configs.workload(name)
    g = torch.Generator(device="cuda").manual_seed(7)
    nb = w.num_pool_blocks()
    dt = torch.bfloat16
    kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    vc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=dt, generator=g) * 3
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    plan = PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim, split="native", tc_min_rows=tc)
    out = P.pat_attention(plan, q, kc, vc)
    torch.cuda.synchronize()
    for qi in (0, 77, 255):
        row = w.rows[qi]
        n = (len(row) - 1) * w.block_size + w.valid_last[qi]
        idx = torch.tensor(row, device="cuda")
        k = kc[idx].reshape(-1, w.num_kv_heads, w.head_dim)[:n].double().cpu().numpy()
        v = vc[idx].reshape(-1, w.num_kv_heads, w.head_dim)[:n].double().cpu().numpy()
        ref = AO.full_attention(q[qi:qi + 1].double().cpu().numpy(), [k], [v])[0]
        got = out[qi].double().cpu().numpy()
        err = np.abs(got - ref)
        bad = err > 2e-3 + 1e-2 * np.abs(ref)
        heads = sorted(set(np.nonzero(bad)[0].tolist()))
        assert not bad.any(), f"q{qi}: {bad.sum()} bad, heads {heads[:16]}, max err {err.max():.3e}"


def test_cuda_graph_replay_matches_eager():
    w = configs.workload("c2")
    g = torch.Generator(device="cuda").manual_seed(5)
    nb = w.num_pool_blocks()
    kc = torch.randn(nb, 16, 8, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    vc = torch.randn(nb, 16, 8, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    q = torch.randn(w.batch, 32, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    plan = PatPlan.from_table(table)
    eager = P.pat_attention(plan, q, kc, vc).clone()
    graph = P.PatLayerGraph(plan, q, kc, vc)
    graph.out.zero_()
    got = graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(got, eager)
    q.mul_(0.5)  # in-place input update is seen by the next replay
    eager2 = P.pat_attention(plan, q, kc, vc)
    got2 = graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(got2, eager2)
