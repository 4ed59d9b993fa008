"""B200-native (sm_100a) Gram-based distributed SVD hot path of Li, Kluger & Tygert
(arXiv 1612.08709): tall-skinny SVD (Algorithms 3/4) and randomized low-rank SVD
(Algorithms 5, 6, 8), and the TSQR-based Algorithms 1, 2, 7, FP64, row-sharded over GPUs with NCCL.

The product is the C-ABI library lib/libtssvd_b200.so (include/tssvd.h); this
package is its thin ctypes/torch binding.  There is no CPU fallback.
"""
from .api import (Comm, gram, last_stats, lowrank_svd, lowrank_svd_tsqr, matmul, matmul_tn,  # noqa: F401
                  mixing_tables, sym_eig, sym_eig_ql, tsqr_svd, tssvd)
from .partition import shard_rows  # noqa: F401

__all__ = ["Comm", "tssvd", "lowrank_svd", "tsqr_svd", "lowrank_svd_tsqr", "mixing_tables", "gram", "matmul", "matmul_tn", "sym_eig", "sym_eig_ql",
           "last_stats", "shard_rows"]
