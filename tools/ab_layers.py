"""A/B helper: per-config layer time (CUDA graph, L2 flushed by a 512 MB write
then a read of another buffer) for the default plan.

    python tools/ab_layers.py c1 c2 c3 c4 c5"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22333_b200 as P  # noqa: E402
from paper_2511_22333_b200 import configs  # noqa: E402


def main(names):
    import bench
    buf = bench.L2Flush("cuda")
    for name in names:
        w = configs.workload(name)
        g = torch.Generator(device="cuda").manual_seed(0)
        nb, dt = w.num_pool_blocks(), torch.bfloat16
        kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
        vc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
        q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
        table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        plan = P.PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim,
                                    tc_min_rows=int(os.environ.get("PAT_AB_TC", "0")),
                                    pair_items=os.environ.get("PAT_AB_PAIR") == "1")
        gr = P.PatLayerGraph(plan, q, kc, vc)
        ts = []
        for i in range(43):
            buf.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gr.replay()
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b) * 1e3)
        print(f"{name} {np.median(ts):8.2f} us  (min {min(ts):.2f})", flush=True)
        del gr
        plan.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])
