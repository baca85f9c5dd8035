"""B200-native H^2-matrix hot path of arXiv 1402.5056 (local low-rank update, matvec, ...).

The product is the C-ABI shared library ``libh2b200.so`` (include/h2.h); this package is a thin
ctypes binding with the same call names.  Every step of the method runs in the library's CUDA
kernels; PyTorch only supplies device memory and streams.  There is no CPU fallback: importing
the binding without the built library raises.
"""
from .h2 import (  # noqa: F401
    H2Error,
    Trunc,
    Tree,
    BlockTree,
    Mat,
    h2_cluster_tree,
    h2_cluster_tree_dd,
    h2_block_tree,
    h2_from_sparse,
    h2_lowrank_update,
    h2_batch_begin,
    h2_batch_end,
    h2_matvec,
    h2_addmul,
    h2_lr_factor,
    h2_inverse,
    h2_solve,
    h2_ranks,
    h2_storage_report,
    h2_export,
    h2_import,
    h2_check_device_flags,
    h2_profile_enable,
    h2_profile_read,
    h2_stats,
    h2_pcg,
    h2_launch_count,
    library_path,
    EXPORTED_SYMBOLS,
)
