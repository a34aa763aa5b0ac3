"""Device decoder timings (CUDA graph of one layer, L2 flushed): the full
serving path with the table unchanged (fingerprint + skipped planner chain +
forward + merge), the same with the table rewritten every replay (re-plan on
the device), and the host-planned layer graph for comparison."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2511_22333_b200 as P  # noqa: E402
from paper_2511_22333_b200 import configs  # noqa: E402


def timed(fn, flush, iters=20):
    ts = []
    for i in range(iters + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(i)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def main(names):
    flush = bench.L2Flush("cuda")
    for name in names:
        w = configs.workload(name)
        g = torch.Generator(device="cuda").manual_seed(0)
        nb = w.num_pool_blocks()
        kc = torch.randn(nb, 16, w.num_kv_heads, w.head_dim, device="cuda", dtype=torch.bfloat16, generator=g)
        vc = torch.randn(nb, 16, w.num_kv_heads, w.head_dim, device="cuda", dtype=torch.bfloat16, generator=g)
        q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=torch.bfloat16, generator=g)
        t = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        bt0, sl0 = t.padded()
        bt, sl = torch.from_numpy(bt0).cuda(), torch.from_numpy(sl0).cuda()
        plan = P.PatPlan.from_table(t, w.num_heads, w.num_kv_heads, w.head_dim)
        host = P.PatLayerGraph(plan, q, kc, vc)
        t_host = timed(lambda i: host.replay(), flush)
        dec = P.PatDeviceDecoder(w.num_heads, w.num_kv_heads, w.head_dim, w.batch, bt.shape[1])
        out = torch.empty_like(q)
        dec.forward(bt, sl, q, kc, vc, out=out)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
            dec.forward(bt, sl, q, kc, vc, out=out, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        t_same = timed(lambda i: gr.replay(), flush)
        # the next layers of a step pass the same table tensors and skip even
        # the fingerprint (PAT_DECODE_SAME_TABLE)
        gr2 = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s), torch.cuda.graph(gr2, stream=s):
            dec.forward(bt, sl, q, kc, vc, out=out, stream=s, same_table=True)
        torch.cuda.current_stream().wait_stream(s)
        t_next = timed(lambda i: gr2.replay(), flush)
        sl_alt = sl.clone()
        sl_alt[0] -= 1  # a different table: alternate between the two -> re-plan every replay

        def flip(i):
            sl.copy_(sl_alt if i % 2 else torch.from_numpy(sl0).cuda())
            gr.replay()
        t_replan = timed(flip, flush)
        print(f"{name}: host-planned layer {t_host:7.1f} us | device decoder: same table {t_same:7.1f} us, "
              f"re-plan every step {t_replan:7.1f} us, next layer (flag) {t_next:7.1f} us", flush=True)
        dec.close()
        plan.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])
