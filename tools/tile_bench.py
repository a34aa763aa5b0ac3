"""Per-tile cost of the forward kernel by item width (a development probe).

    python tools/tile_bench.py [--rows 4,8,32,64,128] [--steps 32]

Two regimes, 296 items (2 per SM) of `steps` 64-token KV tiles each, Llama-3-8B
heads (32 q / 8 kv, d 128, bf16), CUDA graph, L2 flushed before every replay:

* hbm: every item streams its own KV from HBM (37 packs x 8 kv heads);
* l2:  every item reads the SAME KV span (37 explicit units over one shared
  row): after the first touch it is L2-resident, so the time is the kernel's
  per-tile chain, not HBM.

Prints µs per tile per SM (layer time / tiles per SM) for each regime."""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22333_b200 as P  # noqa: E402

H, KVH, D, BS = 32, 8, 128, 16
G = H // KVH


def time_plan(plan, q, kc, vc, flush, iters=10):
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
    del gr
    return float(np.median(ts))


def run(rows, steps, mode, flush, npk=37, tc=1):
    nq = max(1, rows // G)
    ntok = steps * 64
    gen = torch.Generator(device="cuda").manual_seed(0)
    if mode == "hbm":
        tbl, blk = [], 0
        for _ in range(npk):
            tbl += [list(range(blk, blk + ntok // BS))] * nq
            blk += ntok // BS
        table = P.BlockTable(tbl, [BS] * len(tbl), BS)
        plan = P.PatPlan.from_table(table, H, KVH, D, split="none", forward_only=True, tc_min_rows=tc)
    else:
        blk = ntok // BS
        span = list(range(blk))
        tbl = [span] * (npk * nq)
        table = P.BlockTable(tbl, [BS] * len(tbl), BS)
        units = [(list(range(u * nq, (u + 1) * nq)), span, ntok) for u in range(npk)]
        plan = P.PatPlan.from_units(table, units, H, KVH, D, tc_min_rows=tc)
    kc = torch.randn(blk, BS, KVH, D, device="cuda", dtype=torch.bfloat16, generator=gen)
    vc = torch.randn(blk, BS, KVH, D, device="cuda", dtype=torch.bfloat16, generator=gen)
    q = torch.randn(len(tbl), H, D, device="cuda", dtype=torch.bfloat16, generator=gen)
    items = plan.info().n_items
    us = time_plan(plan, q, kc, vc, flush)
    plan.close()
    tiles_per_sm = items * steps / 148.0
    return us, us / tiles_per_sm, items


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="4,8,16,32,64,128")
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--mode", default="hbm,l2")
    ap.add_argument("--tc", type=int, default=1, help="tc_min_rows (1: every pack on the tcgen05 kernel)")
    args = ap.parse_args()
    import bench
    flush = bench.L2Flush("cuda")
    for rows in [int(x) for x in args.rows.split(",")]:
        line = f"rows {rows:4d}"
        for mode in args.mode.split(","):
            us, per, items = run(rows, args.steps, mode, flush, tc=args.tc)
            us2, _, _ = run(rows, 2 * args.steps, mode, flush, tc=args.tc)
            # marginal cost of a tile: the layer time difference over the extra tiles per SM
            marg = (us2 - us) / (items * args.steps / 148.0)
            line += f"  {mode}: {us:8.1f} us {per * 1e3:7.1f} ns/tile, marginal {marg * 1e3:7.1f} ns/tile"
        print(line, flush=True)


if __name__ == "__main__":
    main()
