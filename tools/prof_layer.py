"""Run a few decode-attention layers of one config (for ncu / nsys-style captures).

    python tools/prof_layer.py --config c4 [--iters 3] [--tc 64] [--split native]
Prints per-layer CUDA-event time and the plan summary (not a bench number)."""

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22333_b200 as P  # noqa: E402
from paper_2511_22333_b200 import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--tc", type=int, default=0)
    ap.add_argument("--split", default="native")
    ap.add_argument("--dtype", default="bfloat16")
    ap.add_argument("--graph", action="store_true")
    args = ap.parse_args()
    w = configs.workload(args.config)
    dt = getattr(torch, args.dtype)
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    plan = P.PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim, split=args.split,
                                tc_min_rows=args.tc)
    inf = plan.info()
    print(f"packs {inf.n_packs} units {inf.n_units} items {inf.n_items} slots {inf.n_slots} merge_q {inf.n_merge_q}"
          f" launches {inf.n_launches}")
    g = torch.Generator(device="cuda").manual_seed(0)
    nb = w.num_pool_blocks()
    kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    vc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    out = torch.empty_like(q)
    ws = torch.empty(max(plan.workspace_bytes(), 256), dtype=torch.uint8, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    g = P.PatLayerGraph(plan, q, kc, vc, out=out, workspace=ws) if args.graph else None
    for i in range(args.warmup + args.iters):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if g is not None:
            g.replay()
        else:
            P.pat_attention(plan, q, kc, vc, out=out, workspace=ws)
        b.record()
        torch.cuda.synchronize()
        if i >= args.warmup:
            print(f"layer {a.elapsed_time(b) * 1e3:.1f} us")


if __name__ == "__main__":
    main()
