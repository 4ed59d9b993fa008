"""CPU-side checks of the C-ABI boundary: the library loads (no GPU needed),
exports every function include/tssvd.h declares, and validates arguments."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tssvd.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*([a-z_][a-z0-9_]*)\s*\(",
                       src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "defined")))


def test_header_declares_expected_entry_points():
    names = declared_functions()
    for must in ("tssvd", "lowrank_svd", "tssvd_workspace_size", "lowrank_workspace_size",
                 "tssvd_comm_create", "tssvd_comm_wrap_nccl", "tssvd_get_unique_id",
                 "tssvd_status_string"):
        assert must in names


def test_library_loads_and_exports_every_declared_symbol():
    from paper_1612_08709_b200 import _lib

    h = _lib.lib()
    missing = [n for n in declared_functions() if not hasattr(h, n)]
    assert not missing, missing
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(declared_functions()) <= bound  # the binding marshals every entry point
    assert h.tssvd_abi_version() == 1
    assert h.tssvd_status_string(0) == b"ok"


def test_workspace_queries_and_validation_without_gpu():
    from paper_1612_08709_b200 import _lib

    h = _lib.lib()
    o = _lib.default_opts()
    nb = ctypes.c_size_t()
    assert h.tssvd_workspace_size(None, 2_000_000, 100, ctypes.byref(o), ctypes.byref(nb)) == 0
    assert 0 < nb.value < 200 << 20  # workspace is O(n^2 * CTAs), not O(m n)
    assert h.lowrank_workspace_size(None, 200_000, 20_000, 25, ctypes.byref(o), ctypes.byref(nb)) == 0
    assert nb.value > 200_000 * 26 * 8  # holds Y (m x l)
    # argument errors are reported, not crashed on
    assert h.tssvd_workspace_size(None, 100, 7, ctypes.byref(o), ctypes.byref(nb)) == 0  # odd n is fine
    assert h.tssvd_workspace_size(None, 100, 2049, ctypes.byref(o), ctypes.byref(nb)) == 1  # n > 2048
    assert h.tssvd_workspace_size(None, 10_000, 2_000, ctypes.byref(o), ctypes.byref(nb)) == 0  # wide core
    assert nb.value > 10_000 * 2_000 * 8  # holds Y~ (m x n) for the wide core
    bad = _lib.default_opts(wp=1.5)
    assert h.tssvd_workspace_size(None, 100, 10, ctypes.byref(bad), ctypes.byref(nb)) == 1
    assert b"working precision" in h.tssvd_last_error()
    assert h.lowrank_workspace_size(None, 100, 50, 50, ctypes.byref(o), ctypes.byref(nb)) == 1
    out = ctypes.c_void_p()
    assert h.tssvd_comm_wrap_nccl(None, ctypes.byref(out)) == 1 and not out.value  # NULL comm: EINVAL
    # the QL eigensolver's limits are argument errors, checked before any device work
    assert h.tssvd_sym_eig_ql(None, 161, None, 161, None, None, 161, None, None, 0) == 1
    assert b"1 <= n <= 160" in h.tssvd_last_error()
    assert h.tssvd_sym_eig_ql(None, 10, None, 9, None, None, 10, None, None, 0) == 1


def test_no_cpu_fallback_in_product_package():
    """The product package never imports the oracle (only tests/bench/smoke may)."""
    pkg = os.path.join(ROOT, "paper_1612_08709_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "numpy.linalg" not in txt and "np.linalg" not in txt, f


def test_shard_rows_partition():
    from paper_1612_08709_b200 import shard_rows

    for m in (0, 1, 7, 100, 2_000_003):
        for world in (1, 2, 3, 8):
            parts = [shard_rows(m, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == m
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)
