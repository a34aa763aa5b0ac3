"""Per-item timeline of the tcgen05 forward kernel over a whole layer (all CTAs).

    python tools/tc_trace.py --build                 # here: tools/libpat_trace.so (-DPAT_TC_TRACE)
    python tools/item_log.py c2 [c4 ...]              # on the GPU box

For every work item the first softmax thread of CTA c records globaltimer at
item start, first KV/S data ready, tile loop done and epilogue done
(`g_item_log`).  Prints, per config: the layer span, the per-CTA split into
item start latency / tiles / epilogue / idle tail, per-tile ns by item kind,
and the slowest CTAs.  A debugging tool, not a bench number."""

import ctypes as C
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
os.environ.setdefault("PAT_LIB", os.path.join(REPO, "tools", "libpat_trace.so"))

import paper_2511_22333_b200 as P  # noqa: E402
from paper_2511_22333_b200 import _native as N  # noqa: E402
from paper_2511_22333_b200 import configs  # noqa: E402


def run(name, tc_min_rows=0):
    w = configs.workload(name)
    g = torch.Generator(device="cuda").manual_seed(0)
    nb, dt = w.num_pool_blocks(), torch.bfloat16
    kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    vc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    plan = P.PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim, tc_min_rows=tc_min_rows,
                                forward_only=True, pair_items=os.environ.get("PAT_AB_PAIR") == "1")
    out = torch.empty_like(q)
    ws = torch.zeros(max(plan.workspace_bytes(), 256), dtype=torch.uint8, device="cuda")
    import bench
    flush = bench.L2Flush("cuda")
    lib = N.lib()
    lib.pat_debug_item_log.argtypes = [C.c_void_p, C.c_void_p]
    log = np.zeros((32768, 12), dtype=np.int64)
    cnt = np.zeros(1, dtype=np.int32)
    for i in range(4):
        flush.zero_()
        torch.cuda.synchronize()
        lib.pat_debug_item_log(log.ctypes.data, cnt.ctypes.data)  # clears
        P.pat_attention(plan, q, kc, vc, out=out, workspace=ws)
        torch.cuda.synchronize()
    lib.pat_debug_item_log(log.ctypes.data, cnt.ctypes.data)
    spans = np.zeros((1, 4096, 2), dtype=np.uint64)
    lib.pat_debug_spans_tc.argtypes = [C.c_void_p]
    lib.pat_debug_spans_tc(spans.ctypes.data)
    n = int(cnt[0])
    e = log[:n]
    t0 = e[:, 4].min()
    end = e[:, 7].max()
    span = (end - t0) / 1e3
    start_lat = (e[:, 5] - e[:, 4]) / 1e3
    tiles = (e[:, 6] - e[:, 5]) / 1e3
    epi = (e[:, 7] - e[:, 6]) / 1e3
    print(f"== {name}: {n} items, layer span {span:.1f} us (first item start -> last epilogue)")
    sp = spans[0][spans[0][:, 0] > 0].astype(np.int64)
    if len(sp):
        print(f"   kernel: CTA entry (first / last) -> first item start {(t0 - sp[:, 0].min()) / 1e3:.1f} / "
              f"{(t0 - sp[:, 0].max()) / 1e3:.1f} us;  last epilogue -> last CTA exit {(sp[:, 1].max() - end) / 1e3:.1f} us; "
              f"entry spread {(sp[:, 0].max() - sp[:, 0].min()) / 1e3:.1f} us")
    ncta = int(e[:, 0].max()) + 1
    idle = np.zeros(ncta)
    first = np.zeros(ncta)
    for c in range(ncta):
        m = e[:, 0] == c
        if m.any():
            idle[c] = (end - e[m, 7].max()) / 1e3
            first[c] = (e[m, 4].min() - t0) / 1e3
    tot = span * ncta
    print(f"   per lane (CTA x pipeline, {ncta}) avg: start-lat {start_lat.sum() / ncta:.1f}  tiles {tiles.sum() / ncta:.1f}  "
          f"epilogue {epi.sum() / ncta:.1f}  idle-tail {idle.mean():.1f}  late-start {first.mean():.1f}  us "
          f"(of {span:.1f})")
    kinds = {"<=16": e[:, 2] <= 16, "17-64": (e[:, 2] > 16) & (e[:, 2] <= 64), "65-128": (e[:, 2] > 64) & (e[:, 2] <= 128),
             ">128": e[:, 2] > 128}
    for k, m in kinds.items():
        if not m.any():
            continue
        nt = e[m, 3].sum()
        print(f"   {k:10s}: {m.sum():5d} items {nt:6d} tiles  {tiles[m].sum() / max(nt, 1) * 1e3:7.1f} ns/tile(in-item) "
              f" start-lat {start_lat[m].mean():.2f}  epi {epi[m].mean():.2f} us/item")
        if e.shape[1] > 8 and (e[m, 8] > 0).all():
            q_st = (e[m, 8] - e[m, 6]) / 1e3
            pv = (e[m, 9] - e[m, 8]) / 1e3
            rest = (e[m, 7] - e[m, 9]) / 1e3
            print(f"               epilogue split: next-Q store {q_st.mean():.2f}  last-PV wait {pv.mean():.2f}  "
                  f"O read + stores {rest.mean():.2f} us/item")
            if (e[m, 10] > 0).all():
                print(f"               narrow: O^T read + barrier {((e[m, 10] - e[m, 9]) / 1e3).mean():.2f}  "
                      f"stores {((e[m, 7] - e[m, 10]) / 1e3).mean():.2f} us/item")
    worst = np.argsort(-(end - np.array([e[e[:, 0] == c, 7].max() if (e[:, 0] == c).any() else end
                                          for c in range(ncta)])))[:0]
    del worst
    plan.close()
    _ = tot


if __name__ == "__main__":
    tc = int(os.environ.get("PAT_AB_TC", "0"))
    for name in sys.argv[1:] or ["c2", "c3", "c4"]:
        run(name, tc)
