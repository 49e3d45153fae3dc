"""paper_2310_04610_b200 — B200-native DS4Sci_EvoformerAttention.

The hot path of arxiv 2310.04610 (DeepSpeed4Science) re-built for sm_100a:
fused Evoformer attention forward/backward with the mask (bias1) and pair
(bias2) biases, dBias2 reduced over the row axis inside the kernels, behind
the C-ABI in include/evoattn.h. See DESIGN.md.
"""
from ._native import (CudaError, EvoAttnError, NumericError, UnsupportedError, UsageError,
                      ValidationError)
from .evoformer_attention import (DS4Sci_EvoformerAttention, EvoformerAttentionFunction,
                                  evoformer_attention_backward, evoformer_attention_backward_gated,
                                  evoformer_attention_forward, evoformer_attention_forward_gated,
                                  last_launch_count, numeric_checks, resolved_path, set_numeric_checks)
from .pair_bias import PairBiasFunction, pair_bias, pair_bias_backward, pair_bias_forward
from .variants import (AttentionVariant, chunked_forward, layout_from_msa, variant_attention, variant_forward,
                       variant_from_name)

__all__ = [
    "DS4Sci_EvoformerAttention", "EvoformerAttentionFunction", "evoformer_attention_forward",
    "evoformer_attention_backward", "last_launch_count", "resolved_path", "EvoAttnError",
    "ValidationError", "NumericError", "UsageError", "CudaError", "UnsupportedError",
    "AttentionVariant", "variant_attention", "variant_from_name", "layout_from_msa",
    "chunked_forward", "variant_forward", "set_numeric_checks", "numeric_checks",
    "evoformer_attention_forward_gated", "evoformer_attention_backward_gated",
    "pair_bias", "pair_bias_forward", "pair_bias_backward", "PairBiasFunction",
]
