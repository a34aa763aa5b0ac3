"""Golden fixtures for the inspection / numerics API names (forest, traffic,
partials) from the REAL reference package.  Run in the build container:

    python tests/golden/make_api_golden.py

Writes ``api_surface.json.gz``:
* ``forests``: reference ``build_forest`` of 60 seeded random tables and 40 trees of
  the acceptance family, serialised as nested [block_ids, token_len, num_queries,
  query_ids, children], with ``pack_forest`` / ``flatten_forest`` of the same;
* ``partials``: ``cta_partial`` (float64 on fp16-rounded inputs) of 3 small packs
  split in two KV parts each, and ``merge_partials`` of the per-(query, head) pairs.
Nothing at test time reads /root/reference."""

import gzip
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import prefixpack as pp  # noqa: E402
import helpers  # noqa: E402


def node_json(n):
    return [list(n.block_ids), n.token_len, n.num_queries, list(n.query_ids), [node_json(c) for c in n.children]]


def forest_case(name, table):
    f = pp.build_forest(table)
    return {"name": name, "bs": table.block_size, "rows": [list(r) for r in table.rows],
            "valid": list(table.valid_tokens_last_block), "roots": [node_json(r) for r in f.roots],
            "packs": [[list(p.query_ids), list(p.block_ids), p.kv_len] for p in pp.pack_forest(f)],
            "flat": {str(k): v for k, v in pp.flatten_forest(f).items()}}


def main():
    rng = random.Random(77)
    forests = []
    for i in range(60):
        _, t = helpers.random_table(rng, max_queries=rng.choice([4, 8, 16, 32]))
        forests.append(forest_case(f"random/{i}", t))
    spec = pp.WorkloadSpec(level_counts=(1,), level_lengths=(16,))
    for i, (name, t) in enumerate(helpers.tree_family_tables(spec)):
        if i % 71 == 0:
            forests.append(forest_case(name, t))
    partials = []
    nrng = np.random.default_rng(5)
    for H, KVH, d, nq, t in [(8, 2, 64, 3, 40), (32, 8, 128, 2, 100), (16, 4, 128, 5, 17)]:
        rnd = lambda x: x.astype(np.float16).astype(np.float64)  # noqa: E731
        q = rnd(nrng.standard_normal((nq, H, d)) * 2)
        k = rnd(nrng.standard_normal((t, KVH, d)))
        v = rnd(nrng.standard_normal((t, KVH, d)))
        h = t // 2
        a = pp.cta_partial(q, k[:h], v[:h])
        b = pp.cta_partial(q, k[h:], v[h:])
        merged = np.stack([np.stack([pp.merge_partials([a.at(i, j), b.at(i, j)]) for j in range(H)])
                           for i in range(nq)])
        full = pp.full_attention(q, [k] * nq, [v] * nq)
        partials.append({"H": H, "KVH": KVH, "d": d, "q": q.tolist(), "k": k.tolist(), "v": v.tolist(), "h": h,
                         "a_max": a.max_score.tolist(), "a_sum": a.exp_sum.tolist(), "a_ws": a.weighted_sum.tolist(),
                         "merged": merged.tolist(), "full": full.tolist()})
    path = os.path.join(HERE, "api_surface.json.gz")
    with gzip.open(path, "wt", encoding="utf-8", compresslevel=9) as fh:
        json.dump({"forests": forests, "partials": partials}, fh, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "B;", len(forests), "forests")


if __name__ == "__main__":
    main()
