"""B200-native (sm_100a) xBeam decode-step selection from xGR (arXiv 2512.11529, section 6).

The product is the C-ABI library lib/libxgr_beam.so (include/xgr_beam.h) built from csrc/ by
build_ext.py; `binding` is a thin ctypes layer with the same names. Importing this package loads
the library and raises if it is missing: there is no CPU fallback.
"""
from .binding import (  # noqa: F401
    BeamSearch,
    ShardedBeamSearch,
    XgrConfig,
    XgrError,
    XGR_CFG_COUNTERS,
    XGR_CFG_NO_PRUNE,
    XGR_CFG_NO_SPARSE_KERNEL,
    XGR_CFG_TIMING,
    XGR_CFG_PAPER_HEAP,
    XGR_DTYPE_BF16,
    XGR_DTYPE_F32,
    kv_reorder,
    attn_staged,
    attn_shared,
    attn_unshared,
    attn_merge,
    lib,
    LIB_PATH,
)
