"""paper_2411_01238_b200 — B200-native SparseDrop hot path.

Block-mask generation -> kept-block compaction -> tcgen05/TMA sparse GEMMs
(forward dsd, backward sdd dX and dsd dW), behind the reference's operator API.
See DESIGN.md. The compute lives in lib/libsparsedrop_b200.so (C-ABI:
include/sparsedrop_b200.h); this package is the host-side mirror.
"""
from .api import (  # noqa: F401
    BlockMask,
    Communicator,
    DropoutSpec,
    KernelCounters,
    LayerContext,
    LayerGrads,
    LayerPlan,
    LinearLayer,
    LinearVariant,
    SparseKind,
    TileConfig,
    backward,
    counter_hash,
    dense_gemm,
    device_count,
    dropout_scale,
    dsd_matmul,
    effective_seed,
    flops_dense,
    flops_effective,
    forward,
    kept_blocks_in_row,
    launch_count,
    mask_from_words,
    mix64,
    retile,
    sample_mask,
    sdd_matmul,
    transpose_mask,
)
from .bmsk import load_mask, read_mask, save_mask, write_mask  # noqa: F401
from ._capi import LIB_PATH, NativeLibraryMissing, load as load_library  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
