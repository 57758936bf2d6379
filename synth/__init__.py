"""Seeded synthetic input generators shared by the oracle side (tests, bench cpu_baseline)
and the CUDA side (tests, bench, smoke).

This package holds NONE of the method's arithmetic (no masking, no log-softmax, no selection,
no trie construction): only integer hashing that produces item tuples and seeded random logits.
See DESIGN.md "Input recipe" and SURVEY.md section 8(d.1).
"""
from .inputs import (  # noqa: F401
    CONFIGS,
    config,
    config_key,
    splitmix64,
    feistel_permute,
    make_items,
    make_items_clustered,
    make_config_items,
    make_logits,
    make_logits_torch,
    make_logits_rows_torch,
    prefix_keyed_row,
    ATTN_CONFIGS,
    to_bf16_grid,
    bf16_bits,
    make_attn_inputs,
)
