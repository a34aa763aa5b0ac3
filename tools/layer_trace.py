"""Per-CTA globaltimer spans of one decode-attention layer (debug build).

    python tools/tc_trace.py --build            # here: tools/libpat_trace.so (-DPAT_TC_TRACE)
    python tools/layer_trace.py --config c2     # on the GPU box

Prints, per kernel (streaming forward, tcgen05 forward, merge), the CTA count
and the start / end spread relative to the first CTA start, so load imbalance
and kernel overlap are visible (a debugging tool, not a bench number)."""

import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--lib", default=os.path.join(REPO, "tools", "libpat_trace.so"))
    ap.add_argument("--split", default="native")
    ap.add_argument("--tc", type=int, default=0)
    args = ap.parse_args()
    os.environ["PAT_LIB"] = args.lib
    import ctypes as C

    import numpy as np
    import torch

    import paper_2511_22333_b200 as P
    from paper_2511_22333_b200 import _native as N
    from paper_2511_22333_b200 import configs

    w = configs.workload(args.config)
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    plan = P.PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim, split=args.split,
                                tc_min_rows=args.tc)
    inf = plan.info()
    g = torch.Generator(device="cuda").manual_seed(0)
    nb = w.num_pool_blocks()
    dt = torch.bfloat16
    kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    vc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    out = torch.empty_like(q)
    ws = torch.empty(max(plan.workspace_bytes(), 256), dtype=torch.uint8, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    lib = N.lib()
    lib.pat_debug_spans_mma.argtypes = [C.c_void_p]
    lib.pat_debug_spans_tc.argtypes = [C.c_void_p]
    sm = np.zeros((2, 1024, 2), dtype=np.uint64)
    st = np.zeros((1, 1024, 2), dtype=np.uint64)
    for i in range(4):
        flush.zero_()
        torch.cuda.synchronize()
        lib.pat_debug_spans_mma(sm.ctypes.data)
        lib.pat_debug_spans_tc(st.ctypes.data)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        P.pat_attention(plan, q, kc, vc, out=out, workspace=ws)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3
    lib.pat_debug_spans_mma(sm.ctypes.data)
    lib.pat_debug_spans_tc(st.ctypes.data)
    print(f"{args.config}: packs {inf.n_packs} units {inf.n_units} items {inf.n_items} slots {inf.n_slots}; "
          f"layer {us:.1f} us (events)")
    spans = {"stream": sm[0], "tc": st[0], "merge": sm[1]}
    starts = [s[s[:, 0] > 0, 0].min() for s in spans.values() if (s[:, 0] > 0).any()]
    t0 = min(starts)
    for name, s in spans.items():
        m = s[:, 0] > 0
        if not m.any():
            continue
        a = (s[m, 0] - t0) / 1e3
        e = (s[m, 1] - t0) / 1e3
        d = e - a
        print(f"  {name:6s} ctas {m.sum():4d}  start {a.min():7.2f}..{a.max():7.2f} us  end {e.min():7.2f}..{e.max():7.2f}"
              f" us  busy p10/p50/p90/max {np.percentile(d, 10):6.2f} {np.percentile(d, 50):6.2f}"
              f" {np.percentile(d, 90):6.2f} {d.max():6.2f} us")


if __name__ == "__main__":
    main()
