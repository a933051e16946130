"""paper_2508_00887_b200 — B200-native (sm_100a) FRAM / SDSN (arXiv 2508.00887).

The product is the C-ABI library `libfram.so` (include/fram.h, sources in csrc/); this package
holds only its thin ctypes binding (`fram.py`) and the in-tree build script (`build.py`).
"""
from .fram import (  # noqa: F401
    FramError, Schedule, Handle, PREC, DT, EXPORTED,
    FLAG_TRACE, FLAG_CHECK_SYMMETRY, FLAG_NO_THETA_SCALE, FLAG_TIME_PHASES,
    FRAM_OK, FRAM_ERR_USAGE, FRAM_ERR_DATA, FRAM_NOT_CONVERGED, FRAM_ERR_CUDA, FRAM_ERR_NCCL, FRAM_ERR_OOM,
    lib, fram_create, fram_set_schedule, fram_solve, fram_solve_batched, fram_solve_attributed, fram_sdsn, fram_gradient, fram_lap, fram_evaluate,
    fram_get_unique_id, fram_create_sharded, fram_create_sharded_virtual, fram_build_info, shard_rows, broadcast_unique_id,
    create_sharded_dist,
)
