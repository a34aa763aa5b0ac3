"""Generate the golden fixtures from the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``prefixpack`` from ``/root/reference/pkg/src`` (and the reference's
own test helpers from ``/root/reference/pkg/tests``) and writes:

* ``plans_family.json.gz``  -- pack plans for the 2,855-tree family
  (``helpers.tree_family_tables``, the corpus ``test_acceptance.py:137-161`` uses),
  plus naive / query-centric / reference-split plans for every 7th tree.
* ``plans_random.json.gz``  -- plans for seeded ``helpers.random_table`` tables,
  partial-last-block and permuted-id variants, and hand edge cases
  (identical rows, prefix rows, mixed fills, the App. A example, empty table).
* ``plans_configs.json.gz`` -- plans, fingerprints and reference splits for c1..c5.
* ``numerics_small.npz``    -- float64 reference outputs (``run_packed_attention``
  over ``pack_batch`` and over split tasks, and ``full_attention``) on inputs rounded
  to fp16 / bf16, for small tables (d 64/128, head configs of helpers.py:28).
* ``numerics_c1c2.npz``     -- the same for c1 (fp16, bf16) and c2 (fp16), float32.

Nothing at test time reads /root/reference; the fixtures plus this script are
what travel.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, REPO)

import prefixpack as pp  # noqa: E402
from prefixpack import attention as ref_attn  # noqa: E402
from prefixpack.simulator import split_long_kv  # noqa: E402
import helpers  # noqa: E402  (reference test helpers)

from paper_2511_22333_b200 import configs  # noqa: E402


def plan_json(part):
    return [[list(p.query_ids), list(p.block_ids), p.kv_len, bool(p.produces_partial)] for p in part.packs]


def split_json(part, bs):
    tasks = [pp.CtaTask(queries=p.query_ids, block_ids=p.block_ids, kv_len=p.kv_len) for p in part.packs]
    return [[list(t.queries), list(t.block_ids), t.kv_len, t.split_index, t.split_of]
            for t in split_long_kv(tasks, bs)]


def table_case(name, table, extra=True):
    part = pp.pack_batch(table)
    case = {
        "name": name,
        "bs": table.block_size,
        "rows": [list(r) for r in table.rows],
        "valid": list(table.valid_tokens_last_block),
        "fingerprint": table.fingerprint(),
        "packs": plan_json(part),
    }
    if extra:
        case["naive"] = plan_json(pp.naive_per_node(table))
        case["query_centric"] = plan_json(pp.baseline_query_centric(table))
        case["split"] = split_json(part, table.block_size)
    return case


def write_json_gz(name, obj):
    path = os.path.join(HERE, name)
    with gzip.open(path, "wt", encoding="utf-8", compresslevel=9) as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def family():
    spec = pp.WorkloadSpec(level_counts=(1,), level_lengths=(16,))
    cases = []
    for i, (name, table) in enumerate(helpers.tree_family_tables(spec)):
        cases.append(table_case(name, table, extra=(i % 7 == 0)))
    print("tree family:", len(cases))
    write_json_gz("plans_family.json.gz", cases)


def random_cases():
    cases = []
    rng = random.Random(2024)
    for i in range(300):
        _, table = helpers.random_table(rng, max_queries=rng.choice([8, 16, 32, 64]))
        cases.append(table_case(f"random/{i}", table))
    # partial last blocks and permuted block ids (plan must be invariant in shape)
    rng = random.Random(77)
    for i in range(150):
        _, table = helpers.random_table(rng, max_queries=32)
        valid = [rng.choice([table.block_size, rng.randint(1, table.block_size)]) for _ in table.rows]
        ids = sorted({b for r in table.rows for b in r})
        perm = list(range(len(ids) * 3))
        rng.shuffle(perm)
        remap = {b: perm[j] for j, b in enumerate(ids)}
        rows = [[remap[b] for b in r] for r in table.rows]
        t2 = pp.BlockTable(rows=rows, valid_tokens_last_block=valid, block_size=table.block_size)
        cases.append(table_case(f"partial_perm/{i}", t2))
    # rows that share a block at different fills, and prefix-of-other rows
    rng = random.Random(91)
    for i in range(150):
        nq = rng.randint(1, 12)
        base = list(range(rng.randint(1, 6)))
        rows, valid = [], []
        nxt = 100
        for _ in range(nq):
            cut = rng.randint(1, len(base))
            row = base[:cut]
            if rng.random() < 0.5:
                tail = rng.randint(0, 3)
                if rng.random() < 0.5 and tail:
                    row = row + [50 + j for j in range(tail)]  # shared tail ids across rows
                else:
                    row = row + list(range(nxt, nxt + tail))
                    nxt += tail
            rows.append(row)
            valid.append(rng.choice([16, 16, rng.randint(1, 16)]))
        t = pp.BlockTable(rows=rows, valid_tokens_last_block=valid, block_size=16)
        try:
            t.validate()
        except pp.InvalidSpec:
            continue
        cases.append(table_case(f"mixed/{i}", t))
    edge = [
        ("appA", [[0, 1, 2], [0, 5], [0, 1, 2], [9], [0]], [16] * 5),
        ("identical3", [[0, 1], [0, 1], [0, 1]], [16] * 3),
        ("single", [[4, 5, 6]], [7]),
        ("fills", [[0, 1], [0, 1]], [16, 8]),
        ("wide_shallow", [[0, 1, 2, 3] for _ in range(9)] + [[0, 1, 10, 11]], [16] * 10),
        ("prefix_chain", [[0], [0, 1], [0, 1, 2], [0, 1, 2, 3]], [16] * 4),
        ("disjoint", [[0], [1], [2], [3]], [3, 16, 1, 9]),
        ("pre_split_200", [[0, 1] for _ in range(200)], [16] * 200),
        ("bs32", [[0, 1, 2], [0, 1, 3], [0, 4]], [32, 5, 32]),
    ]
    for name, rows, valid in edge:
        bs = 32 if name == "bs32" else 16
        cases.append(table_case(f"edge/{name}", pp.BlockTable(rows=rows, valid_tokens_last_block=valid, block_size=bs)))
    empty = pp.BlockTable(rows=[], valid_tokens_last_block=[], block_size=16)
    cases.append({"name": "edge/empty", "bs": 16, "rows": [], "valid": [],
                  "fingerprint": empty.fingerprint(), "packs": plan_json(pp.pack_batch(empty))})
    # invalid tables: reference raises InvalidSpec (status code mapping tests)
    invalid = [
        ("empty_row", [[0], []], [16, 16]),
        ("repeat", [[0, 1, 0]], [16]),
        ("valid0", [[0, 1]], [0]),
        ("valid17", [[0, 1]], [17]),
    ]
    inv_cases = []
    for name, rows, valid in invalid:
        t = pp.BlockTable(rows=rows, valid_tokens_last_block=valid, block_size=16)
        try:
            pp.pack_batch(t)
            raise SystemExit(f"reference accepted invalid table {name}")
        except pp.InvalidSpec as exc:
            inv_cases.append({"name": name, "rows": rows, "valid": valid, "error": "InvalidSpec", "msg": str(exc)})
    print("random/edge:", len(cases), "invalid:", len(inv_cases))
    write_json_gz("plans_random.json.gz", {"cases": cases, "invalid": inv_cases})


def config_cases():
    out = []
    for name in configs.ALL:
        w = configs.workload(name)
        table = pp.BlockTable(rows=[list(r) for r in w.rows], valid_tokens_last_block=list(w.valid_last),
                              block_size=w.block_size)
        spec = pp.WorkloadSpec(level_counts=(1,), level_lengths=(16,), num_heads=w.num_heads,
                               num_kv_heads=w.num_kv_heads, head_dim=w.head_dim)
        case = table_case(name, table, extra=False)
        case["split"] = split_json(pp.pack_batch(table), w.block_size)
        case["theoretical_min_kv_bytes"] = pp.theoretical_min_kv_bytes(table, spec)
        case["distinct_census"] = list(pp.distinct_block_census(table))
        tr = pp.account_traffic(pp.pack_batch(table), spec)
        case["traffic"] = [tr.kv_bytes, tr.intermediate_bytes]
        del case["rows"]  # rebuilt from configs.workload(name); fingerprint pins it
        out.append(case)
        print(name, "packs", len(case["packs"]))
    write_json_gz("plans_configs.json.gz", out)


def round_to(x, dtype):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x))
    return t.to(getattr(torch, dtype)).to(torch.float64).numpy()


def rounded_inputs(table, spec, seed, dtype, qscale=1.0):
    q, store = ref_attn.generate_qkv(table, spec, seed)
    q = round_to(q * qscale, dtype)
    store = {b: (round_to(k, dtype), round_to(v, dtype)) for b, (k, v) in store.items()}
    return q, store


def checksum(q, store):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(q).tobytes())
    for b in sorted(store):
        h.update(np.ascontiguousarray(store[b][0]).tobytes())
        h.update(np.ascontiguousarray(store[b][1]).tobytes())
    return h.hexdigest()


def ref_outputs(table, spec, q, store):
    part = pp.pack_batch(table)
    packed = ref_attn.run_packed_attention(table, part, store, q, spec)
    tasks = [pp.CtaTask(queries=p.query_ids, block_ids=p.block_ids, kv_len=p.kv_len) for p in part.packs]
    split = ref_attn.run_packed_attention(table, split_long_kv(tasks, table.block_size), store, q, spec)
    f32 = ref_attn.run_packed_attention(table, part, store, q, spec, intermediate_dtype=np.float32)
    full = ref_attn.full_attention(q, [ref_attn.gather_kv(table, store, i)[0] for i in range(table.num_queries)],
                                   [ref_attn.gather_kv(table, store, i)[1] for i in range(table.num_queries)])
    return packed, split, f32, full


def numerics_small():
    arrays = {}
    meta = []
    rng = random.Random(5150)
    k = 0
    for i in range(16):
        heads = helpers.HEAD_CONFIGS[i % 4]
        d = 128 if i % 3 else 64
        sp = helpers.random_spec(rng, max_queries=8, head_config=heads, head_dim=d)
        table = pp.generate_workload(sp, seed=0)
        if i % 2:
            valid = [rng.randint(1, 16) for _ in table.rows]
            table = pp.BlockTable(rows=table.rows, valid_tokens_last_block=valid, block_size=16)
        dtype = ("float16", "bfloat16")[i % 2]
        seed = 1000 + i
        qscale = 6.0 if i % 5 == 4 else 1.0
        q, store = rounded_inputs(table, sp, seed, dtype, qscale)
        packed, split, f32, full = ref_outputs(table, sp, q, store)
        key = f"s{k}"
        k += 1
        # float64 where the oracle is pinned tightly (d=64 cases), float32 otherwise
        arrays[key + "_packed"] = packed if d == 64 else packed.astype(np.float32)
        arrays[key + "_split"] = split.astype(np.float32)
        arrays[key + "_f32"] = f32.astype(np.float32)
        arrays[key + "_full"] = full.astype(np.float32)
        meta.append({"key": key, "rows": [list(r) for r in table.rows], "valid": list(table.valid_tokens_last_block),
                     "bs": 16, "H": sp.num_heads, "KVH": sp.num_kv_heads, "d": d, "seed": seed, "dtype": dtype,
                     "qscale": qscale, "checksum": checksum(q, store)})
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    path = os.path.join(HERE, "numerics_small.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def numerics_configs():
    arrays = {}
    meta = []
    for name, dtype in (("c1", "float16"), ("c1", "bfloat16"), ("c2", "float16")):
        w = configs.workload(name)
        table = pp.BlockTable(rows=[list(r) for r in w.rows], valid_tokens_last_block=list(w.valid_last),
                              block_size=w.block_size)
        spec = pp.WorkloadSpec(level_counts=(1,), level_lengths=(16,), num_heads=w.num_heads,
                               num_kv_heads=w.num_kv_heads, head_dim=w.head_dim)
        q, store = rounded_inputs(table, spec, 0, dtype)
        part = pp.pack_batch(table)
        packed = ref_attn.run_packed_attention(table, part, store, q, spec)
        key = f"{name}_{dtype}"
        arrays[key] = packed.astype(np.float32)
        meta.append({"key": key, "config": name, "dtype": dtype, "seed": 0, "checksum": checksum(q, store)})
        print(key, "done")
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    path = os.path.join(HERE, "numerics_c1c2.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


if __name__ == "__main__":
    which = sys.argv[1:] or ["family", "random", "configs", "small", "c1c2"]
    if "family" in which:
        family()
    if "random" in which:
        random_cases()
    if "configs" in which:
        config_cases()
    if "small" in which:
        numerics_small()
    if "c1c2" in which:
        numerics_configs()
