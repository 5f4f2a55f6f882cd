"""B200-native DeepInverse batched signal recovery (arXiv 1701.03891).

x_hat = M(y, Omega): lifting layer x_tilde = Phi^T y, then three 11x11 convolutional layers
(64 + ReLU, 32 + ReLU, 1) -- PAPER.md §4-5 -- computed by hand-written sm_100a kernels behind the
C ABI include/deepinverse.h.  This package is the ctypes binding plus the in-tree build.
"""
from .binding import (DI_FLAG_FINAL_RELU, DI_FLAG_FULLMAP_BIAS, DI_FLAG_XCORR, EXPORTS, LIB_PATH,  # noqa: F401
                      DeepInverse, DiError, di_add_noise, di_create, di_create_args, di_debug_stage, di_destroy,
                      di_get_params, di_last_error, di_measure, di_metrics, di_num_params, di_proxy_partial,
                      di_recover, di_recover_from_proxy, di_recover_metrics, di_recover_host, di_sgd_step, di_status_string, di_train_grad, load, split_params)
from .rowshard import RowShardedDeepInverse, batch_range, row_range, sum_scatter  # noqa: F401,E402
