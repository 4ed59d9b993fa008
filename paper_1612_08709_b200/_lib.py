"""ctypes loader for the in-tree C-ABI library (include/tssvd.h).

Argument marshalling only.  There is no fallback: if the shared library is
missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libtssvd_b200.so")
# A/B experiments: load another build of the same library (no rebuild check)
_LIB_OVERRIDE = os.environ.get("TSSVD_LIB")
if _LIB_OVERRIDE:
    LIB_PATH = _LIB_OVERRIDE

c_int, c_int64, c_double, c_size_t = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
c_void_p, c_char_p = ctypes.c_void_p, ctypes.c_char_p
P = ctypes.POINTER

TSSVD_ABI_VERSION = 1
STATUS = {0: "TSSVD_OK", 1: "TSSVD_EINVAL", 2: "TSSVD_ENONFINITE", 3: "TSSVD_ENOCONV",
          4: "TSSVD_ECUDA", 5: "TSSVD_ENCCL", 6: "TSSVD_ENOMEM"}


class TssvdOpts(ctypes.Structure):
    _fields_ = [("abi_version", c_int), ("working_precision", c_double),
                ("orthonormalizations", c_int), ("max_jacobi_sweeps", c_int), ("host_io", c_int)]


MAX_PASSES = 48
PASS_KINDS = {1: "gram_x", 2: "xv", 3: "gram_y", 4: "qnorm", 5: "uout", 6: "alpha", 7: "beta",
              8: "jacobi", 9: "tsqr"}


class TssvdStats(ctypes.Structure):
    _fields_ = [("kernel_launches", c_int64), ("a_passes", c_int64),
                ("jacobi_sweeps", c_int * 16), ("n_jacobi", c_int),
                ("ranks", c_int64 * 8), ("n_ranks", c_int),
                ("n_pass", c_int), ("pass_kind", c_int * MAX_PASSES),
                ("pass_ms", c_double * MAX_PASSES), ("pass_flops", c_double * MAX_PASSES),
                ("pass_bytes", c_double * MAX_PASSES)]


# (name, restype, argtypes) for every symbol include/tssvd.h declares
SIGNATURES = [
    ("tssvd_status_string", c_char_p, [c_int]),
    ("tssvd_last_error", c_char_p, []),
    ("tssvd_abi_version", c_int, []),
    ("tssvd_get_unique_id", c_int, [P(ctypes.c_ubyte)]),
    ("tssvd_comm_create", c_int, [c_int, c_int, P(ctypes.c_ubyte), c_int, P(c_void_p)]),
    ("tssvd_comm_wrap_nccl", c_int, [c_void_p, P(c_void_p)]),
    ("tssvd_comm_destroy", c_int, [c_void_p]),
    ("tssvd_comm_rank", c_int, [c_void_p, P(c_int), P(c_int)]),
    ("tssvd_allreduce_sum", c_int, [c_void_p, c_void_p, c_void_p, c_int64]),
    ("tssvd_opts_default", None, [P(TssvdOpts)]),
    ("tssvd_workspace_size", c_int, [c_void_p, c_int64, c_int64, P(TssvdOpts), P(c_size_t)]),
    ("tssvd", c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, P(TssvdOpts),
                      c_void_p, c_int64, c_void_p, c_void_p, c_int64, P(c_int64), c_void_p,
                      c_size_t]),
    ("lowrank_workspace_size", c_int, [c_void_p, c_int64, c_int64, c_int64, P(TssvdOpts),
                                       P(c_size_t)]),
    ("lowrank_svd", c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                            c_int64, c_int64, c_int, c_int64, P(TssvdOpts), c_void_p, c_int64,
                            c_void_p, c_void_p, c_int64, P(c_int64), c_void_p, c_size_t]),
    ("tsqr_svd_workspace_size", c_int, [c_void_p, c_int64, c_int64, P(TssvdOpts), P(c_size_t)]),
    ("tsqr_svd", c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                         P(TssvdOpts), c_void_p, c_int64, c_void_p, c_void_p, c_int64, P(c_int64),
                         c_void_p, c_size_t]),
    ("lowrank_tsqr_workspace_size", c_int, [c_void_p, c_int64, c_int64, c_int64, P(TssvdOpts),
                                            P(c_size_t)]),
    ("lowrank_svd_tsqr", c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                                 c_int64, c_int64, c_int, c_int64, c_void_p, c_void_p, P(TssvdOpts),
                                 c_void_p, c_int64, c_void_p, c_void_p, c_int64, P(c_int64), c_void_p,
                                 c_size_t]),
    ("lowrank_lu_workspace_size", c_int, [c_void_p, c_int64, c_int64, c_int64, P(TssvdOpts),
                                          P(c_size_t)]),
    ("lowrank_svd_lu", c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                               c_int64, c_int64, c_int, c_int64, P(TssvdOpts), c_void_p, c_int64,
                               c_void_p, c_void_p, c_int64, P(c_int64), c_void_p, c_size_t]),
    ("tssvd_last_stats", c_int, [P(TssvdStats)]),
    ("tssvd_set_pass_timing", c_int, [c_int]),
    ("tssvd_gram", c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_int64,
                           c_void_p, c_size_t]),
    ("tssvd_gram_workspace", c_size_t, [c_int64, c_int64]),
    ("tssvd_matmul", c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                             c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_size_t]),
    ("tssvd_matmul_workspace", c_size_t, [c_int64, c_int64, c_int64]),
    ("tssvd_matmul_tn", c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                                c_int64, c_void_p, c_int64, c_void_p, c_size_t]),
    ("tssvd_matmul_tn_workspace", c_size_t, [c_int64, c_int64, c_int64]),
    ("tssvd_sym_eig", c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_int64,
                              c_int, P(c_int), c_void_p, c_size_t]),
    ("tssvd_sym_eig_workspace", c_size_t, [c_int64]),
    ("tssvd_sym_eig_ql", c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_int64,
                                 P(c_int), c_void_p, c_size_t]),
    ("tssvd_trace", c_int, [c_int, c_int, c_int64, c_int64, c_int64, c_int, c_int64, P(TssvdOpts),
                            c_char_p, c_size_t]),
]

_lock = threading.Lock()
_lib = None


class TssvdError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {detail}")


def lib() -> ctypes.CDLL:
    """Load (building first if the sources are newer) the sm_100a library; raise if impossible."""
    global _lib
    with _lock:
        if _lib is None:
            from . import build as _build

            try:
                if not _LIB_OVERRIDE and _build.needs_build():
                    _build.build()
            except Exception as e:  # no toolchain: the existing .so (if any) must do
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(f"libtssvd_b200.so missing and build failed: {e}") from e
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"CUDA extension not built: {LIB_PATH}")
            handle = ctypes.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                if _LIB_OVERRIDE and not hasattr(handle, name):
                    continue  # an older A/B build may lack newer entry points
                f = getattr(handle, name)
                f.restype = res
                f.argtypes = args
            if handle.tssvd_abi_version() != TSSVD_ABI_VERSION:
                raise RuntimeError("ABI version mismatch")
            _lib = handle
        return _lib


def check(status: int) -> None:
    if status != 0:
        raise TssvdError(status, lib().tssvd_last_error().decode())


def default_opts(wp: float = 1e-11, passes: int = 2, max_sweeps: int = 60, host_io: int | bool = False):
    o = TssvdOpts()
    lib().tssvd_opts_default(ctypes.byref(o))
    o.working_precision = wp
    o.orthonormalizations = passes
    o.max_jacobi_sweeps = max_sweeps
    o.host_io = int(host_io)  # 0 device, 1 host (staged), 2 host (streamed, lowrank_svd)
    return o


def raw_stats() -> "TssvdStats":
    """The last call's stats as the raw struct (a few us; decode later with decode_stats)."""
    s = TssvdStats()
    check(lib().tssvd_last_stats(ctypes.byref(s)))
    return s


def last_stats() -> dict:
    return decode_stats(raw_stats())


def decode_stats(s: "TssvdStats") -> dict:
    passes = [dict(kind=PASS_KINDS.get(s.pass_kind[i], s.pass_kind[i]), ms=s.pass_ms[i],
                   flops=s.pass_flops[i], bytes=s.pass_bytes[i]) for i in range(s.n_pass)]
    return dict(kernel_launches=s.kernel_launches, a_passes=s.a_passes,
                jacobi_sweeps=list(s.jacobi_sweeps[: s.n_jacobi]),
                ranks=list(s.ranks[: s.n_ranks]), passes=passes)


def trace(problem: str, nranks: int, m_local: int, n: int, l: int = 0, iters: int = 0, k: int = 0,
          wp: float = 1e-11, passes: int = 2) -> list[str]:
    """Steps and collectives of one tssvd ('tssvd') / lowrank_svd ('lowrank') / tsqr_svd ('tsqr') /
    lowrank_svd_tsqr ('lowrank_tsqr') call on one of `nranks` ranks, from a plan-only run of the
    real orchestrator (no GPU needed)."""
    opts = default_opts(wp, passes)
    buf = ctypes.create_string_buffer(1 << 16)
    code = {"tssvd": 1, "lowrank": 2, "tsqr": 3, "lowrank_tsqr": 4, "lowrank_lu": 5}[problem]
    check(lib().tssvd_trace(code, nranks, m_local, n, l, iters, k, ctypes.byref(opts), buf, len(buf)))
    return [t for t in buf.value.decode().split(";") if t]


def set_pass_timing(enable: bool) -> None:
    check(lib().tssvd_set_pass_timing(1 if enable else 0))
