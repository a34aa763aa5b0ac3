"""``torch.ops.patb200.decode_attention``: the serving-engine operator.

The paper plugs PAT into vLLM as a pybind11 op behind an attention backend
(``PAPER.md:742-745``); this is the equivalent registered with
``torch.library`` so an engine (vLLM custom backend, a torch.compile graph)
calls one op with its own tensors:

    torch.ops.patb200.decode_attention(q, k_cache, v_cache, block_tables, seq_lens, out, scale)

* ``q`` [B, H, d], ``out`` [B, H, d] (written), fp16/bf16 CUDA tensors;
* ``k_cache``, ``v_cache`` [num_blocks, page, KVH, d] -- vLLM's
  ``kv_cache[0]`` / ``kv_cache[1]`` (NHD);
* ``block_tables`` [B, max_blocks], ``seq_lens`` [B]: int32 CUDA tensors;
* ``scale`` <= 0 means 1/sqrt(d).

Plans are cached per (heads, kv heads, head dim, device) and reused while the
device table fingerprint is unchanged (``PatDecoder.forward_device``).  The
fingerprint check reads 8 bytes back, so capture the op in a CUDA graph only
with a fixed table (``PatLayerGraph`` over a fixed plan)."""

from __future__ import annotations

import torch

from .attention import PatDecoder

_DECODERS: dict = {}


def _decoder(num_heads: int, num_kv_heads: int, head_dim: int, device: torch.device) -> PatDecoder:
    key = (num_heads, num_kv_heads, head_dim, device.index)
    dec = _DECODERS.get(key)
    if dec is None:
        dec = PatDecoder(num_heads, num_kv_heads, head_dim, device=device)
        _DECODERS[key] = dec
    return dec


@torch.library.custom_op("patb200::decode_attention", mutates_args=("out",))
def decode_attention(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, block_tables: torch.Tensor,
                     seq_lens: torch.Tensor, out: torch.Tensor, scale: float) -> None:
    dec = _decoder(q.shape[1], k_cache.shape[2], q.shape[2], q.device)
    dec.forward_device(block_tables, seq_lens, q, k_cache, v_cache, out=out, scale=scale if scale > 0 else None)


@decode_attention.register_fake
def _decode_attention_fake(q, k_cache, v_cache, block_tables, seq_lens, out, scale) -> None:
    return None


__all__ = ["decode_attention"]
