"""GPU parity: libpatb200 forward + merge vs the reference outputs (golden
fixtures) and vs the CPU oracle.  Tolerance (north star): |x - ref| <= 2e-3 +
1e-2 |ref| for fp16/bf16 inputs against the float64 reference on the same
rounded inputs."""

import random

import numpy as np
import pytest
import torch

import paper_2511_22333_b200 as P
from paper_2511_22333_b200 import configs
from paper_2511_22333_b200.plan import PatPlan
from oracle import attn_oracle as AO
from oracle import pack_oracle as PO

from golden_io import numerics, random_cases

pytestmark = pytest.mark.gpu

ATOL, RTOL = 2e-3, 1e-2
TDT = {"float16": torch.float16, "bfloat16": torch.bfloat16}


def _round(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x)).to(TDT[dtype]).to(torch.float64).numpy()


def _inputs(rows, bs, H, KVH, d, seed, dtype, qscale=1.0):
    q, store = AO.generate_qkv(rows, bs, H, KVH, d, seed)
    q = _round(q * qscale, dtype)
    store = {b: (_round(k, dtype), _round(v, dtype)) for b, (k, v) in store.items()}
    return q, store


def _close(out, ref):
    err = np.abs(out - ref)
    bad = err > ATOL + RTOL * np.abs(ref)
    assert not bad.any(), f"{bad.sum()} elements out of tolerance, max err {err.max():.3e}"


def test_small_fixtures_all_partitions():
    meta, z = numerics("numerics_small.npz")
    for m in meta:
        rows, valid, bs = m["rows"], m["valid"], m["bs"]
        table = P.BlockTable([list(r) for r in rows], list(valid), bs)
        spec = P.WorkloadSpec((1,), (16,), num_heads=m["H"], num_kv_heads=m["KVH"], head_dim=m["d"])
        q, store = _inputs(rows, bs, m["H"], m["KVH"], m["d"], m["seed"], m["dtype"], m["qscale"])
        part = P.pack_batch(table)
        ref = z[m["key"] + "_packed"].astype(np.float64)
        for split in ("none", "reference", "native"):
            out = P.run_packed_attention(table, part, store, q, spec, dtype=TDT[m["dtype"]], split=split)
            _close(out, ref)
        tasks = P.split_long_kv([P.CtaTask(p.query_ids, p.block_ids, p.kv_len) for p in part.packs], bs)
        out = P.run_packed_attention(table, tasks, store, q, spec, dtype=TDT[m["dtype"]])
        _close(out, z[m["key"] + "_split"].astype(np.float64))
        out = P.run_packed_attention(table, P.baseline_query_centric(table), store, q, spec, dtype=TDT[m["dtype"]])
        _close(out, z[m["key"] + "_full"].astype(np.float64))
        out = P.run_packed_attention(table, P.naive_per_node(table), store, q, spec, dtype=TDT[m["dtype"]])
        _close(out, ref)


@pytest.mark.parametrize("key", ["c1_float16", "c1_bfloat16", "c2_float16"])
def test_config_fixtures(key):
    meta, z = numerics("numerics_c1c2.npz")
    m = next(x for x in meta if x["key"] == key)
    w = configs.workload(m["config"])
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    spec = P.WorkloadSpec((1,), (16,), num_heads=w.num_heads, num_kv_heads=w.num_kv_heads, head_dim=w.head_dim)
    q, store = _inputs(w.rows, w.block_size, w.num_heads, w.num_kv_heads, w.head_dim, 0, m["dtype"])
    for split in ("native", "reference", "none"):
        out = P.run_packed_attention(table, P.pack_batch(table), store, q, spec, dtype=TDT[m["dtype"]], split=split)
        _close(out, z[key].astype(np.float64))


def test_random_tables_vs_oracle():
    """Random forests incl. partial last blocks, permuted ids, block_size 32."""
    doc = random_cases()
    rng = random.Random(11)
    cases = [c for c in doc["cases"] if c["rows"]]
    rng.shuffle(cases)
    for i, c in enumerate(cases[:40]):
        H, KVH = [(64, 8), (32, 8), (16, 8), (32, 32), (8, 1)][i % 5]
        d = 128 if i % 3 else 64
        dtype = ("float16", "bfloat16")[i % 2]
        table = P.BlockTable([list(r) for r in c["rows"]], list(c["valid"]), c["bs"])
        spec = P.WorkloadSpec((1,), (16,), num_heads=H, num_kv_heads=KVH, head_dim=d)
        q, store = _inputs(c["rows"], c["bs"], H, KVH, d, 100 + i, dtype, qscale=(4.0 if i % 4 == 0 else 1.0))
        units = [(p[0], p[1], p[2]) for p in PO.pack_batch(c["rows"], c["valid"], c["bs"])]
        ref = AO.run_packed(q, store, units, H, d)
        for split in ("native", "reference"):
            out = P.run_packed_attention(table, P.pack_batch(table), store, q, spec, dtype=TDT[dtype], split=split)
            _close(out, ref)


def _gpu_case(name, dtype=torch.bfloat16, seed=0, split="native", nsample=6):
    """Full-size config through the tensor API; a sample of queries is checked
    against the float64 oracle (full_attention over the same rounded inputs)."""
    w = configs.workload(name)
    g = torch.Generator(device="cuda").manual_seed(seed)
    nb = w.num_pool_blocks()
    kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dtype, generator=g)
    vc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dtype, generator=g)
    q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=dtype, generator=g)
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    plan = PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim, split=split)
    out = P.pat_attention(plan, q, kc, vc)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    rng = random.Random(seed)
    sample = sorted(rng.sample(range(w.batch), min(nsample, w.batch)))
    for qi in sample:
        row = w.rows[qi]
        n = (len(row) - 1) * w.block_size + w.valid_last[qi]
        idx = torch.tensor(row, device="cuda")
        k = kc[idx].reshape(-1, w.num_kv_heads, w.head_dim)[:n].double().cpu().numpy()
        v = vc[idx].reshape(-1, w.num_kv_heads, w.head_dim)[:n].double().cpu().numpy()
        ref = AO.full_attention(q[qi:qi + 1].double().cpu().numpy(), [k], [v])[0]
        _close(out[qi].double().cpu().numpy(), ref)
    return plan, out


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_full_configs_sampled(name):
    _gpu_case(name, dtype=torch.bfloat16)
    _gpu_case(name, dtype=torch.float16, seed=1, split="reference", nsample=3)


def test_plan_reuse_is_deterministic():
    plan, out1 = _gpu_case("c2", nsample=1)
    w = configs.workload("c2")
    g = torch.Generator(device="cuda").manual_seed(0)
    nb = w.num_pool_blocks()
    kc = torch.randn(nb, 16, 8, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    vc = torch.randn(nb, 16, 8, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    q = torch.randn(w.batch, 32, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    a = P.pat_attention(plan, q, kc, vc)
    b = P.pat_attention(plan, q, kc, vc)
    assert torch.equal(a, b) and torch.equal(a, out1)


def test_errors_map_to_reference_exceptions():
    t = P.generate_workload(P.WorkloadSpec((1, 2), (32, 16), num_heads=8, num_kv_heads=2, head_dim=96))
    spec = P.WorkloadSpec((1, 2), (32, 16), num_heads=8, num_kv_heads=2, head_dim=96)
    q, store = _inputs(t.rows, 16, 8, 2, 96, 0, "float16")
    with pytest.raises(P.NoFeasibleConfig):
        P.run_packed_attention(t, P.pack_batch(t), store, q, spec)
    spec64 = P.WorkloadSpec((1, 2), (32, 16), num_heads=8, num_kv_heads=2, head_dim=64)
    q, store = _inputs(t.rows, 16, 8, 2, 64, 0, "float16")
    with pytest.raises(P.CoverageGap):
        P.run_packed_attention(t, P.pack_batch(t).packs[:-1], store, q, spec64)
    with pytest.raises(P.ShapeMismatch):
        P.run_packed_attention(t, P.pack_batch(t), store, q[:1], spec64)


def test_shape_checks_raise_shape_mismatch():
    """q rows, out shape/dtype and the cache page size are checked
    against the plan before any launch (reference: ShapeMismatch, attention.py:220)."""
    from paper_2511_22333_b200.errors import ShapeMismatch
    w = configs.workload("c1")
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    plan = PatPlan.from_table(table, 32, 8, 128)
    nb = w.num_pool_blocks()
    kc = torch.zeros(nb, 16, 8, 128, device="cuda", dtype=torch.float16)
    q = torch.zeros(w.batch, 32, 128, device="cuda", dtype=torch.float16)
    with pytest.raises(ShapeMismatch):
        P.pat_attention(plan, q[:-1].contiguous(), kc, kc)
    with pytest.raises(ShapeMismatch):
        P.pat_attention(plan, q, kc, kc, out=torch.empty(w.batch, 32, 128, device="cuda", dtype=torch.bfloat16))
    with pytest.raises(ShapeMismatch):
        k8 = torch.zeros(2 * nb, 8, 8, 128, device="cuda", dtype=torch.float16)
        P.pat_attention(plan, q, k8, k8)
    dec = P.PatDecoder(32, 8, 128)
    bt_np, sl_np = table.padded()
    with pytest.raises(ShapeMismatch):
        dec.forward_device(torch.from_numpy(bt_np).cuda(), torch.from_numpy(sl_np).cuda(), q[:-1].contiguous(),
                           kc, kc)
    plan.close()
