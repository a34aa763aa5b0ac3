"""Timeline of the tcgen05 forward kernel (one CTA) on a synthetic pack or a config layer.

    python tools/tc_trace.py --build            # here: compile tools/libpat_trace.so (-DPAT_TC_TRACE)
    python tools/tc_trace.py [--nq 32 --G 8 --kvh 8 --ntok 8192]   # on the GPU box

Prints the kernel time (CUDA events) and, per KV step of CTA 0, the clock64
deltas between the producer / MMA issuer / softmax events (a debugging tool,
not a bench number)."""

import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TRACE_LIB = os.path.join(REPO, "tools", "libpat_trace.so")
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--defines", default="")
    ap.add_argument("--nq", type=int, default=32)
    ap.add_argument("--G", type=int, default=8)
    ap.add_argument("--kvh", type=int, default=8)
    ap.add_argument("--ntok", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=24)
    ap.add_argument("--lib", default=TRACE_LIB)
    ap.add_argument("--dtype", default="bfloat16")
    ap.add_argument("--config", default=None, help="trace a CTA of a BASELINE config layer instead")
    ap.add_argument("--cta", type=int, default=0, help="CTA to trace")
    args = ap.parse_args()
    if args.build:
        from paper_2511_22333_b200 import build as B
        defs = ["PAT_TC_TRACE"] + [d for d in args.defines.split(",") if d]
        print(B.build(force=True, out=args.lib, defines=defs))
        return
    os.environ["PAT_LIB"] = args.lib
    import ctypes as C

    import numpy as np
    import torch

    import paper_2511_22333_b200 as P
    from paper_2511_22333_b200 import _native as N

    dt = getattr(torch, args.dtype)
    g = torch.Generator(device="cuda").manual_seed(0)
    if args.config:
        from paper_2511_22333_b200 import configs
        w = configs.workload(args.config)
        table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        plan = P.PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim, split="native")
        nq, H, KVH, ntok, nblk, bs = w.batch, w.num_heads, w.num_kv_heads, 0, w.num_pool_blocks(), w.block_size
        G = H // KVH
    else:
        bs, nq, G, KVH, ntok = 16, args.nq, args.G, args.kvh, args.ntok
        H = G * KVH
        nblk = ntok // bs
        table = P.BlockTable([list(range(nblk)) for _ in range(nq)], [bs] * nq, bs)
        plan = P.PatPlan.from_table(table, H, KVH, 128, split="none", tc_min_rows=1)
    inf = plan.info()
    kc = torch.randn(nblk, bs, KVH, 128, device="cuda", dtype=dt, generator=g)
    vc = torch.randn(nblk, bs, KVH, 128, device="cuda", dtype=dt, generator=g)
    q = torch.randn(nq, H, 128, device="cuda", dtype=dt, generator=g)
    out = torch.empty_like(q)
    ws = torch.empty(max(plan.workspace_bytes(), 256), dtype=torch.uint8, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    lib0 = N.lib()
    lib0.pat_debug_trace_cta.argtypes = [C.c_int]
    times = []
    for i in range(6):
        if i == 5:
            lib0.pat_debug_trace_cta(args.cta)
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        P.pat_attention(plan, q, kc, vc, out=out, workspace=ws)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) * 1e3)
    us = min(times[2:])
    kv_bytes = ntok * KVH * 128 * 4
    flops = 4.0 * nq * H * ntok * 128
    print(f"rows/item {nq * G} items {inf.n_items} kv {ntok}x{KVH}: layer {us:.1f} us  "
          f"{kv_bytes / us / 1e3:.0f} GB/s  {flops / us / 1e6:.1f} TFLOP/s")
    tr = np.zeros((4, 8, 256), dtype=np.int64)
    lib = N.lib()
    lib.pat_debug_tc_trace.argtypes = [C.c_void_p]
    assert lib.pat_debug_tc_trace(tr.ctypes.data) == 0
    t0 = tr[0, 0, 0]
    names = {(0, 0): "prod_tma", (1, 2): "mma_wait_kv", (1, 3): "mma_kv_ok", (1, 0): "mma_qk",
             (1, 4): "mma_wait_p", (1, 1): "mma_pv", (2, 0): "sm_sfull", (2, 1): "sm_pfull"}
    hdr = " step " + " ".join(f"{v:>15s}" for v in names.values())
    print(hdr)
    n = min(args.steps, ntok // 32) if ntok else args.steps
    for s in range(n):
        row = []
        for (r, e) in names:
            v = tr[r, e, s]
            row.append(f"{(v - t0) if v else -1:>15d}")
        print(f"{s:5d} " + " ".join(row))
    # steady-state per-step cycles from the MMA issuer's KV_FULL timestamps
    m = tr[1, 3, :n]
    m = m[m > 0]
    if len(m) > 4:
        d = np.diff(m[2:])
        print(f"steady-state cycles/step (mma kvfull): median {np.median(d):.0f} mean {d.mean():.0f}")


def analyse(path):
    """Per-step breakdown of a saved trace log (softmax busy / idle, MMA KV waits)."""
    lines = open(path).read().splitlines()
    hdr = lines[1].split()
    rows = [dict(zip(hdr, map(int, l.split()))) for l in lines[2:] if l.split() and l.split()[0].isdigit()]
    prev = None
    tot = {"sm_busy": 0, "sm_wait_s": 0, "mma_kv_wait": 0}
    for r in rows:
        if r["smA_sfull"] <= 0:
            break
        busy = r["smA_pfull"] - r["smA_sfull"]
        wait = r["smA_sfull"] - prev["smA_pfull"] if prev else 0
        kvw = r["mma_kvfull"] - max(prev["mma_pv_issued"], prev["mma_qk_issued"]) if prev else 0
        item = " <item" if r.get("mma_item_qfull", -1) > 0 else ""
        print(f"{r['step']:4d} sm_busy {busy:6d} sm_wait_S {wait:6d} mma_kv_wait {kvw:6d}{item}")
        tot["sm_busy"] += busy
        tot["sm_wait_s"] += wait
        tot["mma_kv_wait"] += max(kvw, 0)
        prev = r
    print(tot)


if __name__ == "__main__":
    if len(sys.argv) == 3 and sys.argv[1] == "--analyse":
        analyse(sys.argv[2])
    else:
        main()
