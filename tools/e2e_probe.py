"""e2e breakdown on c2: host time per pat_attention call, and the e2e step
(H2D Q + table, layer, D2H out) with the eager call vs a PatLayerGraph replay.

    python tools/e2e_probe.py"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22333_b200 as P  # noqa: E402
from paper_2511_22333_b200 import configs  # noqa: E402


def main():
    w = configs.workload("c2")
    dev = torch.device("cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    nb, dt = w.num_pool_blocks(), torch.bfloat16
    kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    vc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    plan = P.PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim)
    ws = torch.empty(max(plan.workspace_bytes(), 256), dtype=torch.uint8, device=dev)
    out = torch.empty_like(q)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    # host cost of one eager call (GPU idle before each call)
    from paper_2511_22333_b200 import _native as N
    import ctypes as C
    hs, hd = [], []
    lib = N.lib()
    s = torch.cuda.current_stream()
    args = (plan.handle, C.c_void_p(q.data_ptr()), C.c_void_p(kc.data_ptr()), C.c_void_p(vc.data_ptr()), kc.shape[0],
            C.c_void_p(out.data_ptr()), C.c_void_p(ws.data_ptr()), ws.numel(), N.PAT_DTYPE_BF16, 0.0, C.c_void_p(s.cuda_stream))
    for _ in range(50):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.pat_attention(plan, q, kc, vc, out=out, workspace=ws)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        lib.pat_forward(*args)
        t3 = time.perf_counter()
        hs.append(t1 - t0)
        hd.append(t3 - t2)
    print(f"host us per pat_attention call: {np.median(hs) * 1e6:.1f}; bare pat_forward ctypes call {np.median(hd) * 1e6:.1f}")
    qh = q.cpu().pin_memory()
    bt, sl = table.padded()
    bth = torch.from_numpy(bt).pin_memory()
    slh = torch.from_numpy(sl).pin_memory()
    btd = torch.empty(bt.shape, dtype=torch.int32, device=dev)
    sld = torch.empty(sl.shape, dtype=torch.int32, device=dev)
    outh = torch.empty(q.shape, dtype=q.dtype).pin_memory()
    qd = q.clone()
    graph = P.PatLayerGraph(plan, qd, kc, vc)
    for mode in ("eager", "graph", "eager", "graph"):
        ts = []
        for i in range(25):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            qd.copy_(qh, non_blocking=True)
            btd.copy_(bth, non_blocking=True)
            sld.copy_(slh, non_blocking=True)
            if mode == "eager":
                P.pat_attention(plan, qd, kc, vc, out=out, workspace=ws)
                outh.copy_(out, non_blocking=True)
            else:
                graph.replay()
                outh.copy_(graph.out, non_blocking=True)
            b.record()
            torch.cuda.synchronize()
            if i >= 5:
                ts.append(a.elapsed_time(b) * 1e3)
        print(f"e2e {mode}: {np.median(ts):.1f} us (min {min(ts):.1f})")
    ts = []
    for i in range(25):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        qd.copy_(qh, non_blocking=True)
        btd.copy_(bth, non_blocking=True)
        sld.copy_(slh, non_blocking=True)
        outh.copy_(out, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    print(f"copies only: {np.median(ts):.1f} us")


if __name__ == "__main__":
    main()
