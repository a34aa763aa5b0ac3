"""External / ablation comparators for one decode-attention layer:

* PAT (this library, default plan)
* the query-centric plan (one pack per query, `baseline_query_centric`,
  simulator.py:85-96) through the same kernels -- what packing buys on B200
* flashinfer's paged decode (`BatchDecodeWithPagedKVCacheWrapper`, library code,
  no prefix sharing) on the same bf16 paged cache

    python tools/comparators.py [--configs c2 c5] [--iters 20]

Prints one line per (config, implementation): µs/layer (CUDA events, L2
flushed before every rep) and GB/s on unique KV bytes."""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22333_b200 as P  # noqa: E402
from paper_2511_22333_b200 import configs  # noqa: E402


def timed(fn, iters, flush):
    ts = []
    for i in range(iters + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["c2", "c5"])
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for name in args.configs:
        w = configs.workload(name)
        dt = torch.bfloat16
        g = torch.Generator(device="cuda").manual_seed(0)
        nb = w.num_pool_blocks()
        kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
        vc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
        q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
        table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        unique = w.distinct_tokens() * w.num_kv_heads * w.head_dim * 4
        res = {}
        plan = P.PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim)
        ref = P.pat_attention(plan, q, kc, vc).clone()
        gr = P.PatLayerGraph(plan, q, kc, vc)
        res["pat"] = timed(gr.replay, args.iters, flush)
        qc = P.baseline_query_centric(table)
        units = [(p.query_ids, p.block_ids, p.kv_len) for p in qc.packs]
        plan_qc = P.PatPlan.from_units(table, units, w.num_heads, w.num_kv_heads, w.head_dim, split="native")
        gq = P.PatLayerGraph(plan_qc, q, kc, vc)
        res["pat_query_centric_plan"] = timed(gq.replay, args.iters, flush)
        try:
            import flashinfer

            ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
            bt, sl = table.padded()
            lens = torch.from_numpy(np.array([len(r) for r in w.rows], dtype=np.int32))
            indptr = torch.zeros(w.batch + 1, dtype=torch.int32)
            indptr[1:] = torch.cumsum(lens, 0)
            indices = torch.from_numpy(np.concatenate([np.asarray(r, np.int32) for r in w.rows]))
            last = torch.from_numpy(np.asarray(w.valid_last, dtype=np.int32))
            for tc in (False, True):
                dec = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD", use_tensor_cores=tc)
                dec.plan(indptr.cuda(), indices.cuda(), last.cuda(), w.num_heads, w.num_kv_heads, w.head_dim,
                         w.block_size, q_data_type=dt, kv_data_type=dt)
                o = dec.run(q, (kc, vc))
                torch.cuda.synchronize()
                err = (o.float() - ref.float()).abs().max().item()
                res[f"flashinfer_decode{'_tc' if tc else ''} (max|diff| vs pat {err:.1e})"] = timed(
                    lambda: dec.run(q, (kc, vc)), args.iters, flush)
        except Exception as exc:  # comparator only
            res[f"flashinfer unavailable: {str(exc)[:100]}"] = float("nan")
        for k, us in res.items():
            print(f"{name} {k:55s} {us:9.1f} us  {unique / us / 1e3:8.0f} GB/s (unique KV)", flush=True)


if __name__ == "__main__":
    main()
