"""B200 calibration of the scheduler's item cost model.

    python tools/calibrate.py [--out profiles/b200_calibration.json]

Two sweeps per kernel and row class, each one layer of synthetic independent
packs (Llama-3-8B heads, every kv head an item, 296 x m items so the grid is
evenly loaded), timed as a CUDA graph with L2 flushed:

* `steps`: items of 2 / 8 / 32 KV tiles (64 tokens), 2 items per SM -> the
  marginal cost of one tile with every SM streaming (`per_step_us`);
* `items`: the same 64 tiles per SM cut into 2 / 4 / 8 / 16 / 32 items ->
  the cost of an item boundary (`per_item_us`).

`paper_2511_22333_b200.calibration.load_profile(path)` turns the fits into the
scheduler's cost model (`pat_set_cost_model`)."""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22333_b200 as P  # noqa: E402

H, KVH, D, BS = 32, 8, 128, 16


def layer_us(npk, nq, steps, tc, flush, iters=10):
    ntok = steps * 64
    rows_tbl, blk = [], 0
    for _ in range(npk):
        span = list(range(blk, blk + ntok // BS))
        blk += ntok // BS
        rows_tbl += [span] * nq
    table = P.BlockTable(rows_tbl, [BS] * len(rows_tbl), BS)
    plan = P.PatPlan.from_table(table, H, KVH, D, split="none", tc_min_rows=tc)
    g = torch.Generator(device="cuda").manual_seed(0)
    kc = torch.randn(blk, BS, KVH, D, device="cuda", dtype=torch.bfloat16, generator=g)
    vc = torch.randn(blk, BS, KVH, D, device="cuda", dtype=torch.bfloat16, generator=g)
    q = torch.randn(len(rows_tbl), H, D, device="cuda", dtype=torch.bfloat16, generator=g)
    gr = P.PatLayerGraph(plan, q, kc, vc)
    ts = []
    for i in range(iters + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gr.replay()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    items = plan.info().n_items
    del gr
    plan.close()
    return float(np.median(ts)), items


def fit(x, y):
    a = np.vstack([np.ones(len(x)), np.asarray(x, float)]).T
    (c0, c1), *_ = np.linalg.lstsq(a, np.asarray(y, float), rcond=None)
    return float(c0), float(c1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "profiles", "b200_calibration.json"))
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    G = H // KVH
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    base = sms // KVH  # packs per wave: every SM one item
    res = {"device": torch.cuda.get_device_name(0), "sms": sms, "heads": [H, KVH, D], "fits": {}}
    for kernel, tc in (("tcgen05", 1), ("stream", -1)):
        for rows in ((4, 32, 128) if kernel == "tcgen05" else (4, 16)):
            nq = max(1, rows // G)
            pts = [(s,) + layer_us(2 * base, nq, s, tc, flush) for s in (2, 8, 32)]
            per_sm = [it / sms for _, _, it in pts]
            c0, per_step = fit([s * k for (s, _, _), k in zip(pts, per_sm)], [us for _, us, _ in pts])
            ipts = []
            for k in (2, 4, 8, 16, 32):
                us, it = layer_us(k * base, nq, 64 // k, tc, flush)
                ipts.append((k, us, it))
            i0, per_item = fit([it / sms for _, _, it in ipts], [us for _, us, _ in ipts])
            rec = {"per_step_us": round(per_step, 4), "per_item_us": round(per_item, 3),
                   "layer_fixed_us": round(i0, 2),
                   "steps_sweep": [(s, round(us, 2), it) for s, us, it in pts],
                   "items_sweep": [(k, round(us, 2), it) for k, us, it in ipts]}
            res["fits"][f"{kernel}_rows{rows}"] = rec
            print(kernel, rows, rec, flush=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(args.out)


if __name__ == "__main__":
    main()
