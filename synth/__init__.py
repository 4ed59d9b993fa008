"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no Gram matrix, no
eigensolver, no discard rule, no subspace iteration).  It only manufactures
inputs: test matrices A = U diag(sigma) V^T with a known spectrum, the Gaussian
start block Omega (Alg. 5 step 1) and the power-method start
vector x0.  Both the oracle (``oracle/``) and the CUDA path
(``paper_1612_08709_b200``) receive the *same bytes* from here.
"""
from .matrices import (  # noqa: F401
    BLOCK_ROWS,
    CONFIGS,
    normal_block,
    haar,
    spectrum,
    test_matrix,
    lowrank_test_matrix,
    dct_columns,
    paper_test_matrix,
    paper_lowrank_test_matrix,
    devils_staircase,
    paper_staircase_matrix,
    omega,
    mixing_params,
    power_start,
    config_inputs,
)
