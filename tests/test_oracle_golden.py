"""Pin the CPU oracle to the real reference: every oracle function is checked
against fixtures the reference produced (tests/golden/make_golden.py)."""

import hashlib

import numpy as np
import pytest
import torch

from oracle import attn_oracle as AO
from oracle import pack_oracle as PO
from paper_2511_22333_b200 import configs

from golden_io import as_packs, as_split, config_cases, family_cases, numerics, random_cases


def _plan_of(case):
    return PO.pack_batch(case["rows"], case["valid"], case["bs"])


def test_tree_family_plans_bit_exact():
    cases = family_cases()
    assert len(cases) == 2855
    for c in cases:
        assert _plan_of(c) == as_packs(c["packs"]), c["name"]
        assert PO.fingerprint(c["rows"], c["valid"], c["bs"]) == c["fingerprint"]
        if "naive" in c:
            assert PO.naive_per_node(c["rows"], c["valid"], c["bs"]) == as_packs(c["naive"]), c["name"]
            assert PO.query_centric(c["rows"], c["valid"], c["bs"]) == as_packs(c["query_centric"])
            tasks = [(p[0], p[1], p[2]) for p in as_packs(c["packs"])]
            assert PO.split_long_kv(tasks, c["bs"]) == as_split(c["split"]), c["name"]


def test_random_and_edge_plans_bit_exact():
    doc = random_cases()
    for c in doc["cases"]:
        assert _plan_of(c) == as_packs(c["packs"]), c["name"]
        assert PO.fingerprint(c["rows"], c["valid"], c["bs"]) == c["fingerprint"], c["name"]
        if "naive" in c:
            assert PO.naive_per_node(c["rows"], c["valid"], c["bs"]) == as_packs(c["naive"]), c["name"]
            tasks = [(p[0], p[1], p[2]) for p in as_packs(c["packs"])]
            assert PO.split_long_kv(tasks, c["bs"]) == as_split(c["split"]), c["name"]
        if c["rows"]:
            units = [(p[0], p[1], p[2]) for p in as_packs(c["packs"])]
            assert PO.check_coverage(c["rows"], c["valid"], c["bs"], units)
            assert PO.flatten(PO.forest(c["rows"], c["valid"], c["bs"])) == {
                q: list(r) for q, r in enumerate(c["rows"])}
    for c in doc["invalid"]:
        with pytest.raises(PO.OracleInvalid):
            PO.pack_batch(c["rows"], c["valid"], 16)


def test_config_plans_bit_exact():
    cc = config_cases()
    for name in configs.ALL:
        w = configs.workload(name)
        c = cc[name]
        assert PO.fingerprint(w.rows, w.valid_last, w.block_size) == c["fingerprint"]
        packs = PO.pack_batch(w.rows, w.valid_last, w.block_size)
        assert packs == as_packs(c["packs"]), name
        tasks = [(p[0], p[1], p[2]) for p in packs]
        assert PO.split_long_kv(tasks, w.block_size) == as_split(c["split"]), name
        assert PO.theoretical_min_kv_bytes(w.rows, w.valid_last, w.block_size, w.num_kv_heads, w.head_dim) == \
            c["theoretical_min_kv_bytes"] == w.unique_kv_bytes()
        assert list(PO.distinct_census(w.rows, w.valid_last, w.block_size)) == c["distinct_census"]


def _round(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x)).to(getattr(torch, dtype)).to(torch.float64).numpy()


def _inputs(rows, bs, H, KVH, d, seed, dtype, qscale=1.0):
    q, store = AO.generate_qkv(rows, bs, H, KVH, d, seed)
    q = _round(q * qscale, dtype)
    store = {b: (_round(k, dtype), _round(v, dtype)) for b, (k, v) in store.items()}
    return q, store


def _checksum(q, store):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(q).tobytes())
    for b in sorted(store):
        h.update(np.ascontiguousarray(store[b][0]).tobytes())
        h.update(np.ascontiguousarray(store[b][1]).tobytes())
    return h.hexdigest()


def test_numerics_small_match_reference():
    meta, z = numerics("numerics_small.npz")
    for m in meta:
        rows, valid, bs = m["rows"], m["valid"], m["bs"]
        q, store = _inputs(rows, bs, m["H"], m["KVH"], m["d"], m["seed"], m["dtype"], m["qscale"])
        assert _checksum(q, store) == m["checksum"], m["key"]
        packs = PO.pack_batch(rows, valid, bs)
        units = [(p[0], p[1], p[2]) for p in packs]
        out = AO.run_packed(q, store, units, m["H"], m["d"])
        ref = z[m["key"] + "_packed"]
        tol = 1e-12 if ref.dtype == np.float64 else 2e-6
        assert AO.max_rel_error(out, ref.astype(np.float64)) < tol, m["key"]
        split = PO.split_long_kv(units, bs)
        out_s = AO.run_packed(q, store, [(t[0], t[1], t[2]) for t in split], m["H"], m["d"])
        assert AO.max_rel_error(out_s, z[m["key"] + "_split"].astype(np.float64)) < 2e-6
        out_f = AO.run_packed(q, store, units, m["H"], m["d"], intermediate_dtype=np.float32)
        assert AO.max_rel_error(out_f, z[m["key"] + "_f32"].astype(np.float64)) < 2e-6
        keys = [AO.span_kv(store, r, (len(r) - 1) * bs + v)[0] for r, v in zip(rows, valid)]
        vals = [AO.span_kv(store, r, (len(r) - 1) * bs + v)[1] for r, v in zip(rows, valid)]
        full = AO.full_attention(q, keys, vals)
        assert AO.max_rel_error(full, z[m["key"] + "_full"].astype(np.float64)) < 2e-6
        assert AO.max_rel_error(out, full) < 1e-10


def test_numerics_c1_matches_reference():
    meta, z = numerics("numerics_c1c2.npz")
    for m in meta:
        if m["config"] != "c1":
            continue
        w = configs.workload("c1")
        q, store = _inputs(w.rows, w.block_size, w.num_heads, w.num_kv_heads, w.head_dim, 0, m["dtype"])
        assert _checksum(q, store) == m["checksum"]
        units = [(p[0], p[1], p[2]) for p in PO.pack_batch(w.rows, w.valid_last, w.block_size)]
        out = AO.run_packed(q, store, units, w.num_heads, w.head_dim)
        assert AO.max_rel_error(out, z[m["key"]].astype(np.float64)) < 2e-6


def test_merge_identities():
    rng = np.random.default_rng(6)
    parts = [(float(rng.normal(scale=3)), float(rng.uniform(0.1, 5)), rng.standard_normal(6)) for _ in range(6)]
    base = AO.merge_list(parts)
    for seed in range(5):
        perm = np.random.default_rng(seed).permutation(6)
        out = AO.merge_list([parts[i] for i in perm])
        assert np.max(np.abs(out - base)) <= 8 * np.max(np.spacing(np.abs(base)))
    with pytest.raises(ValueError):
        AO.merge_list([])
    with pytest.raises(ZeroDivisionError):
        AO.merge_list([(0.0, 0.0, np.zeros(1))])


def test_ppk1_roundtrip(tmp_path):
    rng = np.random.default_rng(8)
    t = {"q": rng.standard_normal((3, 4, 8)), "out": rng.standard_normal((3, 4, 8)).astype(np.float32)}
    AO.dump_ppk1(tmp_path / "d.bin", t)
    back = AO.load_ppk1(tmp_path / "d.bin")
    np.testing.assert_array_equal(back["q"], t["q"])
    np.testing.assert_array_equal(back["out"], t["out"])
