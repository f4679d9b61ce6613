"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no norm, gating, top-k, FFN,
quantisation or recall). It only draws numbers: a counter-based PRNG
(splitmix64) that yields every weight tensor and every prompt from
(seed, tensor_id, element index). The CUDA library implements the SAME
generator independently (``paper_2512_03927_b200/csrc/kernels/fixture_gen.cu``);
tests check that both produce identical bytes. Nothing here imports the
oracle or the product. The recipe is stated in DESIGN.md §3 ("Input recipe").
"""
from .fixture import (  # noqa: F401
    GOLDEN, KIND_EMB, KIND_ROUTER, KIND_W1, KIND_W3, KIND_W2, KIND_LM_HEAD, KIND_PROMPT,
    ModelShape, TINY, MIXTRAL, splitmix64, stream_u24, uniform_pm1, tensor_id, weight_fp32,
    weight_bf16_bits, bf16_bits_to_f32, f32_to_bf16_bits, fan_in_scale, gen_model_weights,
    gen_expert, gen_prompt, gen_hidden, gen_attention, KIND_WQ, KIND_WK, KIND_WV, KIND_WO, TINY_ATTN,
    MIXTRAL_ATTN,
)
