"""paper_2505_24179_b200 — B200-native (sm_100a) SALE prefill attention.

The product is lib/libsale_b200.so (CUDA kernels + C ABI, include/sale_b200.h);
`sale` is the Python host mirror of the reference's `namespace sale` entry
points over that ABI. See DESIGN.md.
"""
from . import sale  # noqa: F401
from .sale import (  # noqa: F401
    Context, block_sparse_attention, flop_accounting, full_attention, load_library, prefill,
    prefill_host, quantize_per_key_block, quantize_per_token, quantize_qk, selection_pass,
    unpack_mask, pack_mask, workload_gqa, workload_head_f32,
)
