"""Compare the device decoder's plan with the host plan on one config (debug)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22333_b200 as P  # noqa: E402
from paper_2511_22333_b200 import _native as N, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = configs.workload(name)
t = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
bt, sl = t.padded()
btd, sld = torch.from_numpy(bt).cuda(), torch.from_numpy(sl).cuda()
q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=torch.bfloat16)
kc = torch.randn(w.num_pool_blocks(), 16, w.num_kv_heads, w.head_dim, device="cuda", dtype=torch.bfloat16)
dec = P.PatDeviceDecoder(w.num_heads, w.num_kv_heads, w.head_dim, w.batch, bt.shape[1])
dec.forward(btd, sld, q, kc, kc)
torch.cuda.synchronize()
L = N.lib()
L.pat_decoder_debug_export.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64]


def get(what, n):
    a = np.zeros(n, np.int32)
    assert L.pat_decoder_debug_export(dec._h, what, a.ctypes.data, n) == 0
    return a


np_ = int(get(0, 1)[0])
qoff = get(1, np_ + 1)
pq = get(2, qoff[-1])
boff = get(3, np_ + 1)
pblk = get(4, boff[-1])
dpacks = [(tuple(pq[qoff[p]:qoff[p + 1]]), tuple(pblk[boff[p]:boff[p + 1]])) for p in range(np_)]
hp = P.pack_batch(t)
hpacks = [(p.query_ids, p.block_ids) for p in hp.packs]
print("packs", np_, len(hpacks), "equal:", dpacks == hpacks)
if dpacks != hpacks:
    for i, (a, b) in enumerate(zip(dpacks, hpacks)):
        if a != b:
            print("first diff pack", i, a[0][:8], b[0][:8], a[1][:8], b[1][:8])
            break
ni = get(11, 4)
nm = int(get(13, 1)[0])
print("n_items", ni, "n_merge", nm)
parts = get(15, np_)
nu = int(parts.sum())
print("units", nu, "parts", parts[:10])
up, u0, ut = get(5, nu), get(6, nu), get(7, nu)
uso = get(8, nu + 1)
us = get(9, uso[-1])
items = get(10, int(ni[3]) * 8).reshape(-1, 8)
md = get(12, nm * 4).reshape(-1, 4)
print("items[:5]", items[:5])
print("merge_desc[:5]", md[:5])
# slot coverage: every (unit, member) slot unique and inside its query's range
slots = {}
for u in range(nu):
    p = up[u]
    for j, qq in enumerate(dpacks[p][0]):
        s = us[uso[u] + j]
        slots.setdefault(int(qq), []).append(int(s))
bad = 0
for qrow in md:
    qq, off, cnt = int(qrow[0]), int(qrow[1]), int(qrow[2])
    if sorted(slots.get(qq, [])) != list(range(off, off + cnt)):
        bad += 1
        if bad < 4:
            print("query", qq, "slots", sorted(slots.get(qq, [])), "expected", off, cnt)
print("bad slot queries", bad)
# item coverage: each (unit, head, row) once
cov = {}
for it in items:
    u, h, r0, n = it[:4]
    for r in range(r0, r0 + n):
        cov[(u, h, r)] = cov.get((u, h, r), 0) + 1
exp = sum(len(dpacks[up[u]][0]) * (w.num_heads // w.num_kv_heads) * w.num_kv_heads for u in range(nu))
print("item rows", len(cov), "expected", exp, "dups", sum(1 for v in cov.values() if v > 1))
# unit ntok sums per pack
for p in range(min(np_, 5)):
    print("pack", p, "kv", hp.packs[p].kv_len, "unit ntok sum", int(ut[up == p].sum()), "pages", len(dpacks[p][1]))
