"""Forward time vs the number of SMs the plan uses (grid = num_sms CTAs): if the
per-tile cost is a per-SM limit, time scales as 1/SMs; if a shared resource
(HBM, L2, NoC) limits, fewer SMs lose less than proportionally.

    python tools/sm_scaling.py c3 [c4 ...]"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22333_b200 as P  # noqa: E402
from paper_2511_22333_b200 import configs  # noqa: E402


def main(names):
    buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for name in names:
        w = configs.workload(name)
        g = torch.Generator(device="cuda").manual_seed(0)
        nb, dt = w.num_pool_blocks(), torch.bfloat16
        kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
        vc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
        q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
        table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        base = None
        for sms in (148, 111, 74, 37):
            plan = P.PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim, num_sms=sms,
                                        forward_only=True)
            gr = P.PatLayerGraph(plan, q, kc, vc)
            ts = []
            for i in range(13):
                buf.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                gr.replay()
                b.record()
                torch.cuda.synchronize()
                if i >= 3:
                    ts.append(a.elapsed_time(b) * 1e3)
            us = float(np.median(ts))
            base = base or us
            print(f"{name} sms {sms:3d}: {us:8.1f} us  x{us / base:5.2f} (1/SM scaling would be x{148 / sms:4.2f})",
                  flush=True)
            del gr
            plan.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3"])
