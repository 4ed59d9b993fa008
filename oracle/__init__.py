"""ORACLE -- test infrastructure, NOT part of the product.

Plain CPU float64 implementation of the paper's Algorithms 1-8 and of
its accuracy measures, written from PAPER.md step by step.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / --impl reference)
may import it.  It shares no code with ``paper_1612_08709_b200``.

Parity status: every function here is pinned by ``tests/test_oracle_pins.py``
(constructed spectra, closed forms, brute force on tiny inputs, paper-printed
values); none is "parity unpinned".
"""
from .gram_svd import (  # noqa: F401
    DEFAULT_WP,
    alg1,
    alg2,
    alg3,
    alg4,
    canonical_signs,
    column_norms,
    direct_svd,
    gram,
    keep_mask,
    lowrank_svd,
    lowrank_svd_lu,
    lu_tracking_factor,
    lowrank_svd_tsqr,
    mix_rows,
    r_keep,
    tsqr_svd,
    split_rows,
    subspace_iteration,
    sym_eig,
    tree_sum,
    tssvd,
)
from .metrics import ortho_error, spectral_error  # noqa: F401
