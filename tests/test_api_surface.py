"""The reference's public names on the hot path (``prefixpack/__init__.py:10-86``)
exist in the package and behave like the reference's on its own outputs
(``tests/golden/api_surface.json.gz``, ``plans_configs.json.gz``, written by the
reference).  CPU only."""

import gzip
import json
import os

import numpy as np
import pytest

import paper_2511_22333_b200 as P
from paper_2511_22333_b200 import configs
from oracle import attn_oracle as AO

HERE = os.path.dirname(os.path.abspath(__file__))

# reference __init__.py:10-86 minus the A100 tile model (tiles.py), the
# discrete-event simulator (simulate, SimReport) and the analytical profit
# model (ProfitModel, intra_node_profit, scheme_profits): SURVEY.md section 2
# marks those out of scope.
ON_PATH = """CoverageGap EmptyFeasibleSet EmptyPartialList EmptySpan InvalidChildIndex InvalidSpec MissingRegisterEntry
NoFeasibleConfig NonPositiveDenominator PrefixpackError ShapeMismatch BlockTable CtaPack Partition PrefixForest
PrefixNode WorkloadSpec assemble_partition build_forest flatten_forest generate_workload validate_partition
PackCache naive_per_node pack_batch pack_batch_async pack_forest tree_heuristic TileConfig CtaTask TrafficReport
account_traffic assign_streams baseline_query_centric distinct_block_census plan_tasks split_long_kv
theoretical_min_kv_bytes PartialBatch PartialResult cta_partial full_attention gather_kv generate_qkv
max_rel_error merge_partials run_packed_attention dump_tensors load_tensors""".split()


def _load(name):
    with gzip.open(os.path.join(HERE, "golden", name), "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def api():
    return _load("api_surface.json.gz")


def test_every_on_path_name_is_exported():
    missing = [n for n in ON_PATH if not hasattr(P, n)]
    assert not missing, missing


def _node_json(n):
    return [list(n.block_ids), n.token_len, n.num_queries, list(n.query_ids), [_node_json(c) for c in n.children]]


def test_build_forest_matches_reference(api):
    for case in api["forests"]:
        t = P.BlockTable([list(r) for r in case["rows"]], list(case["valid"]), case["bs"])
        f = P.build_forest(t)
        assert [_node_json(r) for r in f.roots] == case["roots"], case["name"]
        assert f.node_count == sum(1 for _ in f.iter_nodes())
        flat = P.flatten_forest(f)
        assert {str(k): v for k, v in flat.items()} == case["flat"], case["name"]
        packs = P.pack_forest(f)
        assert [[list(p.query_ids), list(p.block_ids), p.kv_len] for p in packs] == case["packs"], case["name"]


def test_pack_forest_equals_native_pack_batch(api):
    """The Python forest + heuristic and the native packer give the same partition."""
    for case in api["forests"][:40]:
        t = P.BlockTable([list(r) for r in case["rows"]], list(case["valid"]), case["bs"])
        native = P.pack_batch(t)
        py = P.assemble_partition(P.pack_forest(P.build_forest(t)), t)
        assert py.packs == native.packs, case["name"]


def test_account_traffic_matches_reference_on_configs():
    for case in _load("plans_configs.json.gz"):
        w = configs.workload(case["name"])
        t = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        spec = P.WorkloadSpec((1,), (16,), num_heads=w.num_heads, num_kv_heads=w.num_kv_heads, head_dim=w.head_dim)
        tr = P.account_traffic(P.pack_batch(t), spec)
        assert [tr.kv_bytes, tr.intermediate_bytes] == case["traffic"], case["name"]
        assert tr.total_bytes == sum(case["traffic"])


def test_plan_tasks_cover_each_pack_and_pick_b200_tiles():
    w = configs.workload("c2")
    t = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    spec = P.WorkloadSpec((1,), (16,), num_heads=w.num_heads, num_kv_heads=w.num_kv_heads, head_dim=w.head_dim)
    part = P.pack_batch(t)
    tasks = P.plan_tasks(part, spec=spec, table=t)
    G = w.num_heads // w.num_kv_heads
    for pidx, pack in enumerate(part.packs):
        mine = [x for x in tasks if x.pack_index == pidx]
        assert sum(x.kv_len for x in mine) == pack.kv_len
        assert [b for x in mine for b in x.block_ids] == list(pack.block_ids)
        assert all(x.split_of == len(mine) for x in mine)
        want = (16, 64) if len(pack.query_ids) * G <= 16 else (128, 32)
        assert all(x.cfg.key() == want for x in mine)
    streams = P.assign_streams(tasks)
    assert sorted(len(v) for v in streams.values()) == sorted(
        [sum(1 for x in tasks if x.cfg.key() == k) for k in {x.cfg.key() for x in tasks}])
    # without a table the rows are rebuilt from the partition
    assert [(x.queries, x.kv_len) for x in P.plan_tasks(part, spec=spec)] == [(x.queries, x.kv_len) for x in tasks]


def test_merge_partials_identities():
    rng = np.random.default_rng(3)
    parts = [P.PartialResult(float(m), float(s), rng.standard_normal(8))
             for m, s in zip(rng.standard_normal(5), rng.uniform(0.5, 2, 5))]
    a = P.merge_partials(parts)
    assert np.allclose(a, P.merge_partials(parts[::-1]), rtol=1e-13, atol=1e-15)
    assert np.allclose(a, P.merge_partials([p.scaled(7.5) for p in parts]), rtol=1e-13, atol=1e-15)
    with pytest.raises(P.EmptyPartialList):
        P.merge_partials([])
    with pytest.raises(P.NonPositiveDenominator):
        P.merge_partials([P.PartialResult(0.0, 0.0, np.zeros(4))])


def test_ppk1_roundtrip_and_oracle_compat(tmp_path):
    rng = np.random.default_rng(1)
    tensors = {"q": rng.standard_normal((2, 3, 4)), "out": rng.standard_normal((5,)).astype(np.float32),
               "ints": np.arange(6).reshape(2, 3)}
    p = tmp_path / "x.ppk"
    P.dump_tensors(p, tensors)
    back = P.load_tensors(p)
    assert back["q"].dtype == np.float64 and back["out"].dtype == np.float32 and back["ints"].dtype == np.float64
    for k in tensors:
        assert np.array_equal(back[k], np.asarray(tensors[k], dtype=back[k].dtype))
    assert open(p, "rb").read(4) == b"PPK1"
    ora = AO.load_ppk1(str(p))
    assert all(np.array_equal(ora[k], back[k]) for k in back)


def test_generate_qkv_and_gather_match_oracle():
    w = configs.workload("c1")
    t = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    spec = P.WorkloadSpec((1, 8), (1024, 128), num_heads=w.num_heads, num_kv_heads=w.num_kv_heads,
                          head_dim=w.head_dim)
    q, store = P.generate_qkv(t, spec, seed=0)
    q2, store2 = AO.generate_qkv(w.rows, w.block_size, w.num_heads, w.num_kv_heads, w.head_dim, seed=0)
    assert np.array_equal(q, q2) and all(np.array_equal(store[b][0], store2[b][0]) for b in store)
    k, v = P.gather_kv(t, store, 3)
    assert k.shape == (t.kv_len(3), w.num_kv_heads, w.head_dim) and np.array_equal(k[:16], store[w.rows[3][0]][0])
    assert P.max_rel_error(q, q) == 0.0
