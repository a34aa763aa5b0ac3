"""Fixed-cost probe of the forward kernel (a debugging tool, not a bench number).

    python tools/launch_probe.py c2 c1          # on the GPU box

Per config, same L2 flush protocol as bench.py, CUDA events on the launching
stream: one forward per graph, two forwards back to back in one graph (the
marginal second launch has no event / graph-launch latency in front of it), and
one forward with a warm L2.  The difference between the first and the marginal
launch is the per-step fixed cost that no kernel change can remove."""

import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_2511_22333_b200 as P  # noqa: E402
from paper_2511_22333_b200 import configs  # noqa: E402
from bench import L2Flush  # noqa: E402


def timed(fn, flush, steps=30, do_flush=True):
    s = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps + 5):
        if do_flush:
            flush.zero_()
        if i >= 5:
            evs[i - 5][0].record(s)
        fn()
        if i >= 5:
            evs[i - 5][1].record(s)
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) * 1e3 for a, b in evs]))


def main():
    dev = torch.device("cuda:0")
    flush = L2Flush(dev)
    for name in sys.argv[1:] or ["c2"]:
        w = configs.workload(name)
        table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        plan = P.PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim, forward_only=True)
        g = torch.Generator(device=dev).manual_seed(0)
        nb = w.num_pool_blocks()
        kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device=dev, dtype=torch.bfloat16, generator=g)
        vc = torch.randn_like(kc)
        q = torch.randn(w.batch, w.num_heads, w.head_dim, device=dev, dtype=torch.bfloat16, generator=g)
        out = torch.empty_like(q)
        ws = torch.zeros(max(plan.workspace_bytes(), 256), dtype=torch.uint8, device=dev)
        P.pat_attention(plan, q, kc, vc, out=out, workspace=ws)
        torch.cuda.synchronize()
        graphs = []
        for reps in (1, 2, 4):
            gr = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs), torch.cuda.graph(gr, stream=cs):
                for _ in range(reps):
                    P.pat_attention(plan, q, kc, vc, out=out, workspace=ws)
            torch.cuda.current_stream().wait_stream(cs)
            graphs.append(gr)
        t1 = timed(graphs[0].replay, flush)
        t2 = timed(graphs[1].replay, flush)
        t4 = timed(graphs[2].replay, flush)
        tw = timed(graphs[0].replay, flush, do_flush=False)
        print(f"{name}: 1 fwd {t1:.1f} us | 2 fwd {t2:.1f} (marginal {t2 - t1:.1f}) | 4 fwd {t4:.1f} "
              f"(marginal {(t4 - t2) / 2:.1f}) | warm L2 1 fwd {tw:.1f} us")
        plan.close()


if __name__ == "__main__":
    main()
