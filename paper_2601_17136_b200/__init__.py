"""B200-native exact Kernel K-means hot path (arXiv 2601.17136).

The compute lives in ``libkkm.so`` (CUDA, sm_100a) behind the C-ABI of
``include/kkm.h``; this package is a thin ctypes binding with the same names
(argument marshalling only). PyTorch provides device memory, streams and the
torch.distributed bootstrap of the NCCL communicator.
"""
from .kkm import (  # noqa: F401
    KKMError, KKMParams, KernelKMeans, lib, lib_path, default_params, shard_begin,
    workspace_size, plan_query, KKMPlanInfo, get_unique_id, comm_init, comm_destroy,
    LAYOUT_FULL, LAYOUT_STREAM, LAYOUT_SYM_BANDS, LAYOUT_SYM_BANDS16, LAYOUT_SYM_STREAM,
    XCHG_NONE, XCHG_PARTIALS, XCHG_S_ALLREDUCE, XCHG_S_REDUCE_SCATTER,
    KERNEL_LINEAR, KERNEL_POLY, KERNEL_GAUSSIAN, PATH_AUTO, PATH_MATERIALIZE, PATH_STREAM,
    PREC_BF16X3, PREC_FP32_SIMT, PREC_FP16X3, SYM_AUTO, SYM_OFF, SYM_ON, KSTORE_AUTO, KSTORE_FP32, KSTORE_FP16, KSTORE_FP16X2, DBG_E, DBG_CNORM, DBG_SIZES, DBG_DIAG, DBG_DFULL,
    DBG_LABELS_PREV, PHASES,
)
