"""Accuracy of the TC kernel (bf16) vs float64 on peaked softmax rows."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22333_b200 as P

def run(nq=32, ntok=1024, G=8, qscale=1.0, seed=0, dtype=torch.bfloat16):
    bs = 16
    rows = [list(range(ntok // bs)) for _ in range(nq)]
    table = P.BlockTable(rows, [bs] * nq, bs)
    g = torch.Generator(device="cuda").manual_seed(seed)
    kc = torch.randn(ntok // bs, bs, 1, 128, device="cuda", dtype=dtype, generator=g)
    vc = torch.randn(ntok // bs, bs, 1, 128, device="cuda", dtype=dtype, generator=g)
    q = torch.randn(nq, G, 128, device="cuda", dtype=dtype, generator=g) * qscale
    plan = P.PatPlan.from_table(table, G, 1, 128, split="none", tc_min_rows=1)
    out = P.pat_attention(plan, q, kc, vc).double()
    k = kc.reshape(-1, 1, 128).double(); v = vc.reshape(-1, 1, 128).double()
    s = torch.einsum("ngd,td->ngt", q.double(), k[:, 0]) / 128 ** 0.5
    ref = torch.einsum("ngt,td->ngd", torch.softmax(s, -1), v[:, 0])
    err = (out - ref).abs()
    ratio = (err / (2e-3 + 1e-2 * ref.abs())).max().item()
    print(f"qscale={qscale} ntok={ntok}: max abs err {err.max().item():.2e}  worst err/tol {ratio:.2f}")

for qs in (1.0, 3.0, 6.0, 12.0):
    for nt in (64, 1024, 8192):
        run(ntok=nt, qscale=qs)
