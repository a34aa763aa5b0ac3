"""Native host packer (libpatb200 ``pat_plan_create_host``) vs the reference plans:
bit-exact packs, order, produces_partial and reference-mode split units.  CPU only."""

import ctypes
import random
import re

import numpy as np
import pytest

import paper_2511_22333_b200 as P
from paper_2511_22333_b200 import _native as N
from paper_2511_22333_b200 import configs
from paper_2511_22333_b200.plan import PatPlan
from oracle import pack_oracle as PO

from golden_io import as_packs, as_split, config_cases, family_cases, random_cases


def _table(c):
    return P.BlockTable(rows=[list(r) for r in c["rows"]], valid_tokens_last_block=list(c["valid"]),
                        block_size=c["bs"])


def _native_packs(table):
    plan = PatPlan.from_table(table, split="none", host_only=True)
    try:
        return plan.pack_tuples()
    finally:
        plan.close()


def _native_split_units(table, packs):
    """Reference-mode split through the native scheduler, as (queries, blocks, kv, idx, of)."""
    plan = PatPlan.from_table(table, split="reference", host_only=True)
    try:
        pk = plan.pack_tuples()
        out = []
        for pack, page0, npages, ntok, si, so in plan.units():
            q, b, _, _ = pk[pack]
            out.append((q, b[page0:page0 + npages], ntok, si, so))
        return out
    finally:
        plan.close()


def test_library_exports_every_header_symbol():
    lib = N.lib()
    header = open(N.LIB_PATH.replace("paper_2511_22333_b200/libpatb200.so", "include/pat.h")).read()
    declared = set(re.findall(r"\b(pat_[a-z_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert {s[0] for s in N.SIGNATURES} == declared
    assert lib.pat_version().startswith(b"patb200")


def test_tree_family_bit_exact():
    for c in family_cases():
        t = _table(c)
        assert _native_packs(t) == as_packs(c["packs"]), c["name"]
        assert t.fingerprint() == c["fingerprint"]


def test_random_edge_bit_exact_and_split():
    doc = random_cases()
    for c in doc["cases"]:
        t = _table(c)
        got = _native_packs(t) if c["rows"] else []
        assert got == as_packs(c["packs"]), c["name"]
        if "split" in c:
            assert _native_split_units(t, got) == as_split(c["split"]), c["name"]


def test_public_pack_batch_equals_reference_partition():
    doc = random_cases()
    for c in doc["cases"][:200]:
        t = _table(c)
        part = P.pack_batch(t)
        assert part.source_fingerprint == c["fingerprint"]
        assert [(p.query_ids, p.block_ids, p.kv_len, p.produces_partial) for p in part.packs] == \
            as_packs(c["packs"]), c["name"]
        if "naive" in c:
            nv = P.naive_per_node(t)
            assert [(p.query_ids, p.block_ids, p.kv_len, p.produces_partial) for p in nv.packs] == \
                as_packs(c["naive"]), c["name"]
            qc = P.baseline_query_centric(t)
            assert [(p.query_ids, p.block_ids, p.kv_len, p.produces_partial) for p in qc.packs] == \
                as_packs(c["query_centric"])


def test_invalid_tables_raise_invalid_spec():
    for c in random_cases()["invalid"]:
        t = P.BlockTable(rows=c["rows"], valid_tokens_last_block=c["valid"], block_size=16)
        with pytest.raises(P.InvalidSpec):
            P.pack_batch(t)


def test_configs_bit_exact():
    cc = config_cases()
    for name in configs.ALL:
        w = configs.workload(name)
        t = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        got = _native_packs(t)
        assert got == as_packs(cc[name]["packs"]), name
        assert _native_split_units(t, got) == as_split(cc[name]["split"]), name
        plan = PatPlan.from_table(t, w.num_heads, w.num_kv_heads, w.head_dim, split="native", host_only=True)
        assert plan.info().unique_tokens * w.num_kv_heads * w.head_dim * 4 == cc[name]["theoretical_min_kv_bytes"]
        plan.close()


def test_native_split_covers_every_pack():
    rng = random.Random(3)
    for name in configs.ALL:
        w = configs.workload(name)
        t = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        plan = PatPlan.from_table(t, w.num_heads, w.num_kv_heads, w.head_dim, split="native", host_only=True)
        packs = plan.pack_tuples()
        toks = {}
        for pack, page0, npages, ntok, si, so in plan.units():
            toks.setdefault(pack, []).append((page0, npages, ntok))
        for p, (q, b, kv, _) in enumerate(packs):
            parts = sorted(toks[p])
            assert sum(x[2] for x in parts) == kv
            assert parts[0][0] == 0 and sum(x[1] for x in parts) == len(b)
        plan.close()
    del rng


def test_units_plan_checks_coverage():
    t = P.generate_workload(P.WorkloadSpec((1, 4), (64, 32), num_heads=8, num_kv_heads=2, head_dim=64))
    part = P.pack_batch(t)
    units = [(p.query_ids, p.block_ids, p.kv_len) for p in part.packs]
    plan = PatPlan.from_units(t, units, 8, 2, 64, host_only=True)
    assert [x[:3] for x in plan.pack_tuples()] == units
    plan.close()
    with pytest.raises(P.CoverageGap):
        PatPlan.from_units(t, units[:-1], 8, 2, 64, host_only=True)
    with pytest.raises(P.EmptySpan):
        PatPlan.from_units(t, units + [((0,), (), 0)], 8, 2, 64, host_only=True)


def test_pack_cache_and_async():
    t = P.generate_workload(P.WorkloadSpec((1, 4, 16), (128, 256, 1024)))
    cache = P.PackCache()
    first = P.pack_batch(t, cache)
    for _ in range(10):
        assert P.pack_batch(t, cache) == first
    assert cache.stats == {"hits": 10, "misses": 1}
    t.rows[5].append(10_000)
    t.valid_tokens_last_block[5] = t.block_size
    again = P.pack_batch(t, cache)
    assert again != first and cache.stats == {"hits": 10, "misses": 2}
    fut = P.pack_batch_async(t, cache)
    assert fut.result() == again and cache.stats["hits"] == 11
    ref = PO.pack_batch(t.rows, t.valid_tokens_last_block, 16)
    assert [(p.query_ids, p.block_ids, p.kv_len, p.produces_partial) for p in again.packs] == ref


def test_empty_table():
    t = P.BlockTable(rows=[], valid_tokens_last_block=[], block_size=16)
    assert P.pack_batch(t, P.PackCache()).pack_count == 0


def test_split_long_kv_python_api_matches_reference_fixture():
    doc = random_cases()
    for c in doc["cases"]:
        if "split" not in c:
            continue
        tasks = [P.CtaTask(queries=q, block_ids=b, kv_len=kv) for q, b, kv, _ in as_packs(c["packs"])]
        got = [(t.queries, t.block_ids, t.kv_len, t.split_index, t.split_of)
               for t in P.split_long_kv(tasks, c["bs"])]
        assert got == as_split(c["split"]), c["name"]
    assert ctypes  # keep import
    assert np


def test_torch_op_registered():
    import torch
    import paper_2511_22333_b200  # noqa: F401
    assert hasattr(torch.ops.patb200, "decode_attention")


def test_cli_invalid_spec_exit_code(tmp_path):
    """Reference exit-code contract (cli.py:24-27): unreadable spec -> 2."""
    from paper_2511_22333_b200 import cli
    bad = tmp_path / "w.json"
    bad.write_text('{"group_sizes": [0], "segment_lens": [16]}')
    assert cli.main(["verify", str(bad)]) == cli.EXIT_INVALID_SPEC
    assert cli.main(["run"]) == cli.EXIT_INVALID_SPEC
