"""CPU ORACLE (test infrastructure only) -- restatement of the reference numerics.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.  float64 numpy, as the reference:

* seeded Q/K/V generator          ``attention.py:34-48``  (Q first, then K,V per sorted block id)
* GQA head mapping h -> h // G    ``attention.py:61-67``
* monolithic softmax oracle       ``attention.py:70-102`` (``full_attention``)
* per-pack partial (m, l, o)      ``attention.py:140-163`` (``cta_partial``)
* online-softmax fold             ``attention.py:187-199`` (``_merge_batch_into``)
* scalar merge                    ``attention.py:166-184`` (``merge_partials``)
* pipeline                        ``attention.py:202-239`` (``run_packed_attention``)
* global-normalised error         ``attention.py:272-275`` (``max_rel_error``)
* PPK1 tensor dump format         ``attention.py:278-315``

The GQA expansion is done with a reshape (queries' G heads of one kv head form
one matrix) instead of copying K/V per head; the arithmetic per (query, head,
token) is the same float64 dot product and exp.
"""

from __future__ import annotations

import math
import struct

import numpy as np


def generate_qkv(rows, bs, num_heads, num_kv_heads, head_dim, seed):
    """Same RNG stream as the reference: Q [B,H,d], then for each distinct block in
    ascending id order K [bs,KVH,d] then V [bs,KVH,d] (attention.py:34-48)."""
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((len(rows), num_heads, head_dim))
    store = {}
    for b in sorted({b for r in rows for b in r}):
        k = rng.standard_normal((bs, num_kv_heads, head_dim))
        v = rng.standard_normal((bs, num_kv_heads, head_dim))
        store[b] = (k, v)
    return q, store


def span_kv(store, blocks, n_tokens):
    k = np.concatenate([store[b][0] for b in blocks], axis=0)[:n_tokens]
    v = np.concatenate([store[b][1] for b in blocks], axis=0)[:n_tokens]
    return k, v


def _grouped_scores(qp, k, scale):
    """qp [n,H,d], k [t,KVH,d] -> scores [n,H,t] with head h reading kv head h//G."""
    n, H, d = qp.shape
    kvh = k.shape[1]
    G = H // kvh
    qg = qp.reshape(n, kvh, G, d)
    s = np.einsum("nkgd,tkd->nkgt", qg, k) * scale
    return s.reshape(n, H, -1)


def partial(qp, k, v, scale=None):
    """(max [n,H], exp_sum [n,H], weighted [n,H,d]) over one span (attention.py:140-163)."""
    if k.shape[0] == 0:
        raise ValueError("empty span")
    qp = qp.astype(np.float64)
    k = k.astype(np.float64)
    v = v.astype(np.float64)
    n, H, d = qp.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    s = _grouped_scores(qp, k, scale)
    m = s.max(axis=2)
    w = np.exp(s - m[:, :, None])
    kvh = k.shape[1]
    G = H // kvh
    o = np.einsum("nkgt,tkd->nkgd", w.reshape(n, kvh, G, -1), v).reshape(n, H, d)
    return m, w.sum(axis=2), o


def fold(state, idx, m_i, l_i, o_i):
    """In-place online-softmax fold of one unit's partials (attention.py:187-199)."""
    M, L, O = state
    m_new = np.maximum(M[idx], m_i)
    a = np.exp(M[idx] - m_new)
    b = np.exp(m_i - m_new)
    L[idx] = L[idx] * a + l_i * b
    O[idx] = O[idx] * a[:, :, None] + o_i * b[:, :, None]
    M[idx] = m_new


def merge_list(parts):
    """Scalar merge of [(m, l, o_vec)] for one (query, head) (attention.py:166-184)."""
    if not parts:
        raise ValueError("nothing to merge")
    top = max(p[0] for p in parts)
    l = 0.0
    acc = np.zeros_like(np.asarray(parts[0][2], dtype=np.float64))
    for m, s, o in parts:
        f = math.exp(m - top)
        l += s * f
        acc = acc + np.asarray(o) * f
    if not l > 0.0:
        raise ZeroDivisionError(f"merged exp-sum is {l}")
    return acc / l


def run_packed(q, store, unit_list, num_heads, head_dim, intermediate_dtype=None, scale=None):
    """``unit_list``: (queries, block_ids, kv_len) in fold order.  Returns [B,H,d]
    float64 (attention.py:202-239; coverage is checked by the caller)."""
    B = q.shape[0]
    M = np.full((B, num_heads), -np.inf)
    L = np.zeros((B, num_heads))
    O = np.zeros((B, num_heads, head_dim))
    for qs, blocks, n in unit_list:
        idx = np.asarray(qs, dtype=np.intp)
        k, v = span_kv(store, blocks, n)
        m_i, l_i, o_i = partial(q[idx], k, v, scale)
        if intermediate_dtype is not None:
            m_i = m_i.astype(intermediate_dtype).astype(np.float64)
            l_i = l_i.astype(intermediate_dtype).astype(np.float64)
            o_i = o_i.astype(intermediate_dtype).astype(np.float64)
        fold((M, L, O), idx, m_i, l_i, o_i)
    if not np.all(L > 0.0):
        raise ZeroDivisionError("some query/head accumulated no weight")
    return O / L[:, :, None]


def full_attention(q, keys, values, scale=None):
    """Monolithic stable softmax per query over its own K/V (attention.py:70-102)."""
    B, H, d = q.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    out = np.empty((B, H, d))
    for i in range(B):
        m, l, o = partial(q[i:i + 1], keys[i], values[i], scale)
        out[i] = o[0] / l[0][:, None]
    return out


def max_rel_error(x, ref):
    """max|x-ref| / max|ref| -- global normalisation (attention.py:272-275)."""
    s = max(float(np.max(np.abs(ref))), 1e-300)
    return float(np.max(np.abs(np.asarray(x, dtype=np.float64) - ref))) / s


# PPK1 (attention.py:278-315): magic, u32 count, then per tensor u16 name length,
# name, u8 dtype code (0 f64, 1 f32), u8 ndim, u64 shape, little-endian data.
_CODES = {np.dtype(np.float64): 0, np.dtype(np.float32): 1}


def dump_ppk1(path, tensors):
    with open(path, "wb") as fh:
        fh.write(b"PPK1" + struct.pack("<I", len(tensors)))
        for name, a in tensors.items():
            a = np.ascontiguousarray(a)
            if a.dtype not in _CODES:
                a = a.astype(np.float64)
            nm = name.encode()
            fh.write(struct.pack("<H", len(nm)) + nm + struct.pack("<BB", _CODES[a.dtype], a.ndim))
            fh.write(struct.pack(f"<{a.ndim}Q", *a.shape))
            fh.write(a.astype(a.dtype.newbyteorder("<")).tobytes())


def load_ppk1(path):
    inv = {v: k for k, v in _CODES.items()}
    out = {}
    with open(path, "rb") as fh:
        if fh.read(4) != b"PPK1":
            raise ValueError("not a tensor dump")
        (n,) = struct.unpack("<I", fh.read(4))
        for _ in range(n):
            (ln,) = struct.unpack("<H", fh.read(2))
            name = fh.read(ln).decode()
            code, nd = struct.unpack("<BB", fh.read(2))
            shape = struct.unpack(f"<{nd}Q", fh.read(8 * nd))
            dt = inv[code].newbyteorder("<")
            buf = fh.read(int(np.prod(shape)) * dt.itemsize)
            out[name] = np.frombuffer(buf, dtype=dt).reshape(shape).astype(inv[code])
    return out
