"""Sweep of the scheduler's item-cost model (the native KV split and item order
depend on it) against measured layer time -- a calibration tool, not a bench
number.

    python tools/cm_sweep.py c2 c4          # on the GPU box

For each config the inputs are built once; for every (item, row, step) cost
triple the plan is rebuilt with that model and one layer is timed as a CUDA
graph (L2 flushed before every rep, median of 30)."""

import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22333_b200 as P  # noqa: E402
from paper_2511_22333_b200 import configs  # noqa: E402
from paper_2511_22333_b200.calibration import get_cost_model, set_cost_model  # noqa: E402


def main(names):
    import bench
    buf = bench.L2Flush("cuda")
    base = get_cost_model()
    grid = list(itertools.product([600.0, 1200.0, 2400.0], [1000.0, 2000.0, 4000.0], [1200.0, 1440.0, 1800.0]))
    if os.environ.get("PAT_CM_LIST"):  # explicit "item,row,step;item,row,step;..."
        grid = [tuple(float(x) for x in t.split(",")) for t in os.environ["PAT_CM_LIST"].split(";")]
    for name in names:
        w = configs.workload(name)
        g = torch.Generator(device="cuda").manual_seed(0)
        nb, dt = w.num_pool_blocks(), torch.bfloat16
        kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
        vc = torch.randn_like(kc)
        q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
        table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        res = []
        for item, row, step in grid:
            m = get_cost_model()
            m.tc_item_ns, m.tc_item_row_ns, m.tc_step_ns = item, row, step
            set_cost_model(m)
            plan = P.PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim)
            gr = P.PatLayerGraph(plan, q, kc, vc)
            ts = []
            for i in range(33):
                buf.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                gr.replay()
                b.record()
                torch.cuda.synchronize()
                if i >= 3:
                    ts.append(a.elapsed_time(b) * 1e3)
            res.append((float(np.median(ts)), item, row, step, plan.info().n_items))
            del gr
            plan.close()
        set_cost_model(base)
        if not os.environ.get("PAT_CM_LIST"):
            res.sort()
        for t, item, row, step, n in res[:int(os.environ.get("PAT_CM_TOP", "6"))]:
            print(f"{name} {t:8.2f} us  item {item:.0f} row {row:.0f} step {step:.0f}  items {n}", flush=True)
        cur = [r for r in res if (r[1], r[2], r[3]) == (base.tc_item_ns, base.tc_item_row_ns, base.tc_step_ns)]
        if cur:
            print(f"{name} current model: {cur[0][0]:.2f} us", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c4"])
