"""paper_2410_07531_b200 -- B200-native dropout-RNG pipeline (arXiv 2410.07531).

Python mirror of the reference's rgo:: API (proj/include/rgo/*.hpp) on top of
the C-ABI library librgo_b200.so (hand-written sm_100a kernels).  See
DESIGN.md for the path, boundary and kernels.
"""
from . import _lib
from .philox import (PhiloxBlock, PhiloxCounter, PhiloxKey, advance, bump_key, philox_block,
                     philox_blocks, philox_round)
from .mask import (DropoutMask, KeepThreshold, MaskLayout, element_source, generate_mask,
                   generate_mask_device, keep_bit_direct, load_mask, mask_bit, save_mask)

from .ref_attention import (AttentionInput, AttentionOutput, EquivCase, EquivResult, attention_dropout_decoupled,
                            attention_dropout_fused, attention_forward, attn_bwd, attn_fwd, DropoutAttention, default_equiv_grid,
                            random_attention_input, run_equiv_suite)
from . import sharding
from .block import Block, TPBlock, shard_weights
from .gemm import (GemmShape, WorkloadConfig, attention_work, gemm, gemm_shapes, gemm_with_rng,
                   mask_queue_drain, rng_elements, workload_preset)

__all__ = [
    "Block", "TPBlock", "shard_weights",
    "AttentionInput", "AttentionOutput", "EquivCase", "EquivResult", "attention_dropout_decoupled",
    "attention_dropout_fused", "attention_forward", "attn_bwd", "attn_fwd", "DropoutAttention", "default_equiv_grid", "random_attention_input",
    "run_equiv_suite",
    "GemmShape", "WorkloadConfig", "attention_work", "gemm", "gemm_shapes", "gemm_with_rng",
    "mask_queue_drain", "rng_elements", "workload_preset",
    "PhiloxBlock", "PhiloxCounter", "PhiloxKey", "advance", "bump_key", "philox_block",
    "philox_blocks", "philox_round", "DropoutMask", "KeepThreshold", "MaskLayout",
    "element_source", "generate_mask", "generate_mask_device", "keep_bit_direct", "load_mask",
    "mask_bit", "save_mask",
]
