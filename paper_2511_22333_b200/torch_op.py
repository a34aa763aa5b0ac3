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

Planning runs on the GPU (``PatDeviceDecoder`` / ``pat_decoder``): a device
fingerprint of the table, compared on the device with the last one, then the
GPU packer and scheduler only when it changed, then forward + merge -- no host
synchronisation, so the op can be captured in a CUDA graph that stays valid
while the engine rewrites its block table in place.  One decoder per (heads,
kv heads, head dim, page size, device), re-created with a larger capacity when
a table outgrows it; batches above 4096 queries take the host packer
(``PatDecoder.forward_device``, one host round trip per new table)."""

from __future__ import annotations

import torch

from .attention import PatDecoder, PatDeviceDecoder

_DECODERS: dict = {}
_HOST_DECODERS: dict = {}
_MAX_DEVICE_BATCH = 4096


def _pow2(n: int) -> int:
    return 1 << max(0, (int(n) - 1).bit_length())


def _device_decoder(num_heads, num_kv_heads, head_dim, block_size, device, block_tables):
    key = (num_heads, num_kv_heads, head_dim, block_size, device.index)
    dec = _DECODERS.get(key)
    if dec is None or not dec.fits(block_tables):
        mb = max(block_tables.shape[0], dec.max_batch if dec else 0)
        mx = max(block_tables.shape[1], dec.max_blocks if dec else 0)
        if dec is not None:
            dec.close()
        dec = PatDeviceDecoder(num_heads, num_kv_heads, head_dim, min(_MAX_DEVICE_BATCH, _pow2(mb)), _pow2(mx),
                               block_size, device=device)
        _DECODERS[key] = dec
    return dec


def _host_decoder(num_heads, num_kv_heads, head_dim, device) -> PatDecoder:
    key = (num_heads, num_kv_heads, head_dim, device.index)
    dec = _HOST_DECODERS.get(key)
    if dec is None:
        dec = PatDecoder(num_heads, num_kv_heads, head_dim, device=device)
        _HOST_DECODERS[key] = dec
    return dec


@torch.library.custom_op("patb200::decode_attention", mutates_args=("out",))
def decode_attention(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, block_tables: torch.Tensor,
                     seq_lens: torch.Tensor, out: torch.Tensor, scale: float) -> None:
    sc = scale if scale > 0 else None
    if block_tables.shape[0] <= _MAX_DEVICE_BATCH:
        dec = _device_decoder(q.shape[1], k_cache.shape[2], q.shape[2], k_cache.shape[1], q.device, block_tables)
        dec.forward(block_tables, seq_lens, q, k_cache, v_cache, out=out, scale=sc)
    else:
        _host_decoder(q.shape[1], k_cache.shape[2], q.shape[2], q.device).forward_device(
            block_tables, seq_lens, q, k_cache, v_cache, out=out, scale=sc)


@decode_attention.register_fake
def _decode_attention_fake(q, k_cache, v_cache, block_tables, seq_lens, out, scale) -> None:
    return None


__all__ = ["decode_attention"]
