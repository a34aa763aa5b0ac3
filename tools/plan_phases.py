"""Per-phase time of the device planner kernel (trace build, one re-plan per config).

    python tools/tc_trace.py --build          # here
    python tools/plan_phases.py c2 c4         # on the GPU box
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
os.environ.setdefault("PAT_LIB", os.path.join(REPO, "tools", "libpat_trace.so"))
import paper_2511_22333_b200 as P  # noqa: E402
from paper_2511_22333_b200 import _native as N, configs  # noqa: E402

NAMES = ["hash", "compare", "reset", "rows", "dup", "lcp", "levels", "decide", "rank", "scan_nodes", "nodes_init",
         "nodes", "order", "pack_offsets", "members", "schedule"]

for name in sys.argv[1:] or ["c2", "c4"]:
    w = configs.workload(name)
    t = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    bt, sl = t.padded()
    btd, sld = torch.from_numpy(bt).cuda(), torch.from_numpy(sl).cuda()
    q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=torch.bfloat16)
    kc = torch.randn(w.num_pool_blocks(), 16, w.num_kv_heads, w.head_dim, device="cuda", dtype=torch.bfloat16)
    dec = P.PatDeviceDecoder(w.num_heads, w.num_kv_heads, w.head_dim, w.batch, bt.shape[1])
    lib = N.lib()
    lib.pat_debug_plan_stamps.argtypes = [C.c_void_p]
    st = np.zeros(48, np.int64)
    res = []
    for i in range(4):
        sld[0] -= 1 if i % 2 else -1  # a changed table every call
        dec.forward(btd, sld, q, kc, kc)
        torch.cuda.synchronize()
        lib.pat_debug_plan_stamps(st.ctypes.data)
        res.append(np.concatenate([np.diff(st[:len(NAMES)]), np.diff(st[32:39])]) / 1e3)
    r = np.median(np.array(res[1:]), axis=0)
    print(f"== {name}: planner phases (us)")
    for n, v in zip(NAMES[1:] + ["sched:gather", "sched:chunk", "sched:units", "sched:slots", "sched:sort",
                                  "sched:items"], r):
        print(f"   {n:14s} {v:8.1f}")
    dec.close()
