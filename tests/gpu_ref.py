"""Float64 attention reference computed on the GPU (test infrastructure).

Restates ``full_attention`` (reference ``attention.py:70-102``: a monolithic
stable softmax per query, GQA head h reading kv head h // G) in float64 torch on
the device, over the SAME rounded fp16/bf16 tensors the kernels read, so every
query and every head of a full-size config can be checked in seconds."""

import numpy as np
import torch

ATOL, RTOL = 2e-3, 1e-2  # north_star tolerance against the fp32/fp64 reference


def full_attention_gpu(q, k_cache, v_cache, rows, valid_last, block_size, scale=None):
    """q [B, H, d], caches [num_blocks, bs, KVH, d] (any float dtype, on the GPU);
    rows: block ids per query; returns float64 [B, H, d] on the GPU."""
    B, H, d = q.shape
    KVH = k_cache.shape[2]
    G = H // KVH
    scale = d ** -0.5 if scale is None else scale
    out = torch.empty(B, H, d, dtype=torch.float64, device=q.device)
    qd = q.double()
    for i, (row, valid) in enumerate(zip(rows, valid_last)):
        n = (len(row) - 1) * block_size + int(valid)
        idx = torch.as_tensor(list(row), device=q.device, dtype=torch.long)
        k = k_cache[idx].reshape(-1, KVH, d)[:n].double()  # [n, KVH, d]
        v = v_cache[idx].reshape(-1, KVH, d)[:n].double()
        qh = qd[i].view(KVH, G, d)
        s = torch.einsum("kgd,nkd->kgn", qh, k) * scale
        s = s - s.amax(dim=-1, keepdim=True)
        p = torch.exp(s)
        o = torch.einsum("kgn,nkd->kgd", p, v) / p.sum(dim=-1, keepdim=True)
        out[i] = o.reshape(H, d)
    return out


def check_close(out, ref, what=""):
    """|out - ref| <= ATOL + RTOL |ref| elementwise; returns (max abs err, max_rel_error)
    (max_rel_error as attention.py:272-275: global normalisation)."""
    o = out.double()
    err = (o - ref).abs()
    bad = err > ATOL + RTOL * ref.abs()
    nbad = int(bad.sum())
    mre = float(err.max() / ref.abs().max())
    assert nbad == 0, f"{what}: {nbad} of {err.numel()} elements out of tolerance, max err {float(err.max()):.3e}"
    return float(err.max()), mre


def seeded_inputs(w, dtype, seed=7, qscale=3.0, num_heads=None, num_kv_heads=None):
    """Q ~ N(0, qscale^2) (peaked rows), K/V ~ N(0, 1), rounded to `dtype`, on the GPU."""
    H = num_heads or w.num_heads
    KVH = num_kv_heads or w.num_kv_heads
    g = torch.Generator(device="cuda").manual_seed(seed)
    nb = w.num_pool_blocks()
    kc = torch.randn(nb, w.block_size, KVH, w.head_dim, device="cuda", dtype=dtype, generator=g)
    vc = torch.randn(nb, w.block_size, KVH, w.head_dim, device="cuda", dtype=dtype, generator=g)
    q = (torch.randn(w.batch, H, w.head_dim, device="cuda", dtype=torch.float32, generator=g) * qscale).to(dtype)
    return q, kc, vc


__all__ = ["ATOL", "RTOL", "full_attention_gpu", "check_close", "seeded_inputs", "np"]
