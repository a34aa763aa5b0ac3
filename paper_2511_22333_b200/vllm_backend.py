"""vLLM attention backend: PAT decode on top of vLLM's FlashAttention backend.

The paper's integration (``VLLM_ATTENTION_BACKEND=PAT``, ``PAPER.md:742-745``)
as a vLLM 0.22 custom backend: every decode-only batch (``max_query_len == 1``)
of a plain decoder layer with an fp16/bf16 NHD cache goes through
``torch.ops.patb200.decode_attention`` (pack plan from the device block table,
reused while the table is unchanged); prefill, mixed batches and every other
feature (sliding window, ALiBi, soft-cap, sinks, fp8 caches, cascade) fall
back to FlashAttention unchanged.

    import paper_2511_22333_b200.vllm_backend as pat_vllm
    pat_vllm.register()          # AttentionBackendEnum.CUSTOM -> PatAttentionBackend
    # then start vLLM with attention backend CUSTOM

vLLM updates the KV cache in ``do_kv_cache_update`` before ``forward``
(``forward_includes_kv_cache_update = False``), so ``forward`` only computes
attention over the cache."""

from __future__ import annotations

import torch

from vllm.v1.attention.backends.flash_attn import (FlashAttentionBackend, FlashAttentionImpl,
                                                   FlashAttentionMetadataBuilder)

from .torch_op import decode_attention  # noqa: F401  (registers the op)

try:  # vLLM >= 0.11 location of AttentionType
    from vllm.attention.backends.abstract import AttentionType
except Exception:  # pragma: no cover
    from vllm.v1.attention.backend import AttentionType  # type: ignore
from vllm.v1.attention.backend import AttentionCGSupport


class PatAttentionMetadataBuilder(FlashAttentionMetadataBuilder):
    """FlashAttention's metadata; full CUDA graphs of decode-only batches
    (``max_query_len == 1``, the batches PAT serves).  The PAT op plans on the
    GPU (``pat_decoder``: device fingerprint, packer and scheduler, no host
    synchronisation), so a captured decode graph re-plans on the device when
    vLLM rewrites its block table in place.  Mixed / prefill batches stay with
    FlashAttention (piecewise graphs)."""

    _cudagraph_support = AttentionCGSupport.UNIFORM_SINGLE_TOKEN_DECODE

    @classmethod
    def get_cudagraph_support(cls, vllm_config, kv_cache_spec) -> AttentionCGSupport:
        return AttentionCGSupport.UNIFORM_SINGLE_TOKEN_DECODE


class PatAttentionImpl(FlashAttentionImpl):
    """FlashAttention with decode-only batches routed to PAT."""

    def _pat_eligible(self, kv_cache: torch.Tensor, attn_metadata) -> bool:
        return (attn_metadata is not None and attn_metadata.max_query_len == 1
                and not getattr(attn_metadata, "use_cascade", False)
                and self.attn_type == AttentionType.DECODER and self.alibi_slopes is None
                and self.sliding_window == (-1, -1) and not self.logits_soft_cap and self.sinks is None
                and kv_cache.dtype in (torch.float16, torch.bfloat16) and self.head_size in (64, 128)
                and kv_cache.shape[2] % 16 == 0 and kv_cache[0].is_contiguous() and kv_cache[1].is_contiguous())

    def forward(self, layer, query, key, value, kv_cache, attn_metadata, output, output_scale=None,
                output_block_scale=None):
        if output_scale is None and output_block_scale is None and self._pat_eligible(kv_cache, attn_metadata):
            n = attn_metadata.num_actual_tokens
            # the query is usually a strided view of the fused qkv projection
            q = query[:n].reshape(n, self.num_heads, self.head_size).contiguous()
            out = output[:n].view(n, self.num_heads, self.head_size)
            torch.ops.patb200.decode_attention(q, kv_cache[0], kv_cache[1], attn_metadata.block_table[:n],
                                               attn_metadata.seq_lens[:n], out, self.scale)
            return output
        return super().forward(layer, query, key, value, kv_cache, attn_metadata, output, output_scale,
                               output_block_scale)


class PatAttentionBackend(FlashAttentionBackend):
    @staticmethod
    def get_name() -> str:
        return "CUSTOM"

    @staticmethod
    def get_impl_cls() -> type[PatAttentionImpl]:
        return PatAttentionImpl

    @staticmethod
    def get_builder_cls() -> type[PatAttentionMetadataBuilder]:
        return PatAttentionMetadataBuilder


def register() -> None:
    """Register PatAttentionBackend as vLLM's CUSTOM attention backend."""
    from vllm.v1.attention.backends.registry import AttentionBackendEnum, register_backend

    register_backend(AttentionBackendEnum.CUSTOM, f"{__name__}.PatAttentionBackend")


__all__ = ["PatAttentionBackend", "PatAttentionImpl", "PatAttentionMetadataBuilder", "register"]
