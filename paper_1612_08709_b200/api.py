"""Thin torch-facing wrappers over the C ABI (argument marshalling only).

    tssvd(A)                         problem {1}: Alg. 4 (passes=2) / Alg. 3 (passes=1)
    lowrank_svd(A, Omega, iters, k)  problem {2}: Alg. 8

A is this rank's row shard (m_local x n, float64, unit column stride).  A CUDA
tensor runs the device API; a CPU tensor runs the same C-ABI call with
host_io=1 (the library stages it H2D and the results D2H inside the call).
Every arithmetic step happens in the sm_100a kernels of libtssvd_b200.so.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import check, default_opts, lib


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(device: torch.device | None) -> int:
    if device is None or device.type != "cuda":
        return torch.cuda.current_stream().cuda_stream
    return torch.cuda.current_stream(device).cuda_stream


class Comm:
    """NCCL communicator over the ranks of a torch.distributed process group.

    Rank 0 draws the NCCL unique id through the C ABI; torch.distributed (any
    backend) only carries those 128 bytes to the other ranks.
    """

    def __init__(self, group=None, device: int | None = None):
        import torch.distributed as dist

        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = torch.cuda.current_device() if device is None else device
        self.handle = ctypes.c_void_p(None)
        if self.world == 1:
            return
        uid = (ctypes.c_ubyte * 128)()
        if self.rank == 0:
            check(lib().tssvd_get_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = (ctypes.c_ubyte * 128).from_buffer_copy(obj[0])
        check(lib().tssvd_comm_create(self.world, self.rank, uid, self.device,
                                      ctypes.byref(self.handle)))

    @classmethod
    def from_nccl(cls, nccl_comm_ptr: int) -> "Comm":
        """Borrow an existing ncclComm_t (e.g. ``pg._get_backend(torch.device("cuda"))._comm_ptr()``
        of an initialised ProcessGroupNCCL) instead of creating a second communicator; the
        caller keeps that communicator alive."""
        self = cls.__new__(cls)
        self.handle = ctypes.c_void_p(None)
        check(lib().tssvd_comm_wrap_nccl(ctypes.c_void_p(nccl_comm_ptr), ctypes.byref(self.handle)))
        r, w = ctypes.c_int(), ctypes.c_int()
        check(lib().tssvd_comm_rank(self.handle, ctypes.byref(r), ctypes.byref(w)))
        self.rank, self.world = r.value, w.value
        self.device = torch.cuda.current_device()
        return self

    @property
    def ptr(self):
        return self.handle.value

    def allreduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        check(lib().tssvd_allreduce_sum(self.ptr, _stream(t.device), t.data_ptr(), t.numel()))
        return t

    def close(self):
        if self.handle.value:
            check(lib().tssvd_comm_destroy(self.handle))
            self.handle = ctypes.c_void_p(None)


_ws_cache: dict = {}
_ws_size_cache: dict = {}


def _ws_size(fn, cptr, dims, opts) -> int:
    """The library's workspace size for these arguments, remembered per (entry point, comm,
    shape, options): the query runs the host planner, ~40 us a call."""
    key = (fn.__name__, cptr, dims, bytes(opts))
    v = _ws_size_cache.get(key)
    if v is None:
        nbytes = ctypes.c_size_t()
        check(fn(cptr, *dims, ctypes.byref(opts), ctypes.byref(nbytes)))
        v = _ws_size_cache[key] = nbytes.value
    return v


def _workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    key = (device.type, device.index)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def _check_tall(A: torch.Tensor):
    if A.dtype != torch.float64 or A.dim() != 2 or (A.shape[0] > 0 and A.stride(1) != 1):
        raise ValueError("A must be a 2-D float64 tensor with unit column stride")


def tssvd(A: torch.Tensor, wp: float = 1e-11, passes: int = 2, comm: Comm | None = None,
          max_sweeps: int = 60, inplace: bool = False, U: torch.Tensor | None = None):
    """Thin SVD of this rank's shard of a tall-skinny matrix (Alg. 3/4).

    Returns (U_p [m_local x r], sigma [r], V [n x r]) -- U sharded like A,
    sigma and V replicated.  inplace=True lets U overwrite A (device API only).
    """
    _check_tall(A)
    m, n = A.shape
    lda = A.stride(0) if m > 0 else n
    host = A.device.type == "cpu"
    dev = torch.device("cuda", comm.device) if (host and comm) else (
        torch.device("cuda", torch.cuda.current_device()) if host else A.device)
    opts = default_opts(wp, passes, max_sweeps, host_io=host)
    cptr = comm.ptr if comm else None
    nbytes = ctypes.c_size_t(_ws_size(lib().tssvd_workspace_size, cptr, (m, n), opts))
    ws = _workspace(nbytes.value, dev)
    pin = host and torch.cuda.is_available()
    packed = host and U is None  # host_io: U comes back packed (ld (r+1)&~1), one D2H copy
    if U is None:  # device API: even leading dimension (16-byte rows), also for odd n
        U = A if (inplace and not host) else torch.empty((m, n + (n & (0 if host else 1))),
                                                         dtype=torch.float64, device=A.device,
                                                         pin_memory=pin)
    sigma = torch.empty(n, dtype=torch.float64, device=A.device, pin_memory=pin)
    V = torch.empty((n, n), dtype=torch.float64, device=A.device, pin_memory=pin)
    r = ctypes.c_int64()
    ldu = 0 if packed else (U.stride(0) if m > 0 else n)
    check(lib().tssvd(cptr, _stream(dev), m, n, A.data_ptr(), lda, ctypes.byref(opts),
                      U.data_ptr(), ldu, sigma.data_ptr(), V.data_ptr(), n,
                      ctypes.byref(r), ws.data_ptr(), ws.numel()))
    k = r.value
    if packed:
        rp = (k + 1) & ~1
        U = U.view(-1)[:m * rp].view(m, rp)
    return U[:, :k], sigma[:k], V[:, :k]


def lowrank_svd(A: torch.Tensor, Omega: torch.Tensor, iters: int, k: int | None = None,
                wp: float = 1e-11, comm: Comm | None = None, max_sweeps: int = 60,
                out_of_core: bool = False, tracking: str = "q"):
    """Rank-k approximation U diag(sigma) V^T of the row-sharded A by Algorithm 8.

    Omega (n x l) is the Gaussian start block of Alg. 5 step 1 (identical on every rank).
    out_of_core (CPU tensors only): A stays in host memory and every pass over it streams row
    chunks (opts.host_io = 2) -- for A larger than the GPU's memory.
    tracking="lu": the intermediate steps take the L of an LU factorization with partial
    pivoting instead of Q (lowrank_svd_lu in the C ABI).
    """
    if tracking not in ("q", "lu"):
        raise ValueError("tracking must be 'q' or 'lu'")
    if tracking == "lu" and out_of_core:
        raise ValueError("LU tracking is not offered out of core")
    _check_tall(A)
    m, n = A.shape
    l = Omega.shape[1]
    k = l if k is None else k
    host = A.device.type == "cpu"
    dev = torch.device("cuda", comm.device) if (host and comm) else (
        torch.device("cuda", torch.cuda.current_device()) if host else A.device)
    if Omega.device != A.device or Omega.dtype != torch.float64 or Omega.stride(1) != 1:
        raise ValueError("Omega must be float64 on A's device with unit column stride")
    if out_of_core and not host:
        raise ValueError("out_of_core needs A in host memory")
    opts = default_opts(wp, 2, max_sweeps, host_io=2 if out_of_core else host)
    cptr = comm.ptr if comm else None
    wsf = lib().lowrank_lu_workspace_size if tracking == "lu" else lib().lowrank_workspace_size
    nbytes = ctypes.c_size_t(_ws_size(wsf, cptr, (m, n, l), opts))
    ws = _workspace(nbytes.value, dev)
    pin = host and torch.cuda.is_available()
    kk = max(k, 1)
    ldu = kk + (kk & 1)
    U = torch.empty((m, ldu), dtype=torch.float64, device=A.device, pin_memory=pin)
    sigma = torch.empty(kk, dtype=torch.float64, device=A.device, pin_memory=pin)
    V = torch.empty((n, kk), dtype=torch.float64, device=A.device, pin_memory=pin)
    r = ctypes.c_int64()
    fn = lib().lowrank_svd_lu if tracking == "lu" else lib().lowrank_svd
    check(fn(cptr, _stream(dev), m, n, A.data_ptr(), A.stride(0) if m > 0 else n,
             Omega.data_ptr(), Omega.stride(0), l, iters, k, ctypes.byref(opts),
             U.data_ptr(), ldu, sigma.data_ptr(), V.data_ptr(), kk, ctypes.byref(r),
             ws.data_ptr(), ws.numel()))
    q = r.value
    return U[:, :q], sigma[:q], V[:, :q]


def _mixing(phases: torch.Tensor, perms: torch.Tensor, dev: torch.device):
    if phases.dtype != torch.float64 or perms.dtype != torch.int32:
        raise ValueError("phases must be float64 and perms int32")
    if phases.device != dev or perms.device != dev:
        raise ValueError("phases / perms must be on A's device")
    return phases.contiguous(), perms.contiguous()


def tsqr_svd(A: torch.Tensor, phases: torch.Tensor, perms: torch.Tensor, wp: float = 1e-11,
             passes: int = 2, comm: Comm | None = None, max_sweeps: int = 60, inplace: bool = False):
    """Thin SVD of this rank's shard by Algorithm 2 (passes=2) or 1:
    the rows mixed by the random Omega = D F S D~ F S~ (Remark 'randomness'; draws
    `phases` = [theta_D; theta_D~], `perms` = [S; S~], h = n // 2 each, int32), TSQR, SVD of R.
    Device tensors only; n <= 128.  Returns (U_p, sigma, V) as tssvd()."""
    _check_tall(A)
    if A.device.type != "cuda":
        raise ValueError("tsqr_svd takes device tensors")
    m, n = A.shape
    lda = A.stride(0) if m > 0 else n
    if lda & 1:
        raise ValueError("A needs an even leading dimension (pad odd widths)")
    phases, perms = _mixing(phases, perms, A.device)
    opts = default_opts(wp, passes, max_sweeps)
    cptr = comm.ptr if comm else None
    nbytes = ctypes.c_size_t(_ws_size(lib().tsqr_svd_workspace_size, cptr, (m, n), opts))
    ws = _workspace(nbytes.value, A.device)
    U = A if inplace else torch.empty((m, n + (n & 1)), dtype=torch.float64, device=A.device)
    sigma = torch.empty(n, dtype=torch.float64, device=A.device)
    V = torch.empty((n, n), dtype=torch.float64, device=A.device)
    r = ctypes.c_int64()
    check(lib().tsqr_svd(cptr, _stream(A.device), m, n, A.data_ptr(), lda, phases.data_ptr(),
                         perms.data_ptr(), ctypes.byref(opts), U.data_ptr(),
                         U.stride(0) if m > 0 else n + (n & 1), sigma.data_ptr(), V.data_ptr(), n,
                         ctypes.byref(r), ws.data_ptr(), ws.numel()))
    q = r.value
    return U[:, :q], sigma[:q], V[:, :q]


def lowrank_svd_tsqr(A: torch.Tensor, Omega: torch.Tensor, iters: int, phases: torch.Tensor,
                     perms: torch.Tensor, k: int | None = None, wp: float = 1e-11,
                     comm: Comm | None = None, max_sweeps: int = 60):
    """Rank-k approximation by Algorithm 7: Alg. 5 + 6 with the TSQR-based
    Algorithms 1 / 2.  phases / perms: l x l tables, row w - 1 = the mixing draws for a
    factorization of width w (float64 / int32, on A's device).  Device tensors only."""
    _check_tall(A)
    if A.device.type != "cuda":
        raise ValueError("lowrank_svd_tsqr takes device tensors")
    m, n = A.shape
    l = Omega.shape[1]
    k = l if k is None else k
    if Omega.device != A.device or Omega.dtype != torch.float64 or Omega.stride(1) != 1:
        raise ValueError("Omega must be float64 on A's device with unit column stride")
    phases, perms = _mixing(phases, perms, A.device)
    if tuple(phases.shape) != (l, l) or tuple(perms.shape) != (l, l):
        raise ValueError("phases / perms must be l x l tables")
    opts = default_opts(wp, 2, max_sweeps)
    cptr = comm.ptr if comm else None
    nbytes = ctypes.c_size_t(_ws_size(lib().lowrank_tsqr_workspace_size, cptr, (m, n, l), opts))
    ws = _workspace(nbytes.value, A.device)
    kk = max(k, 1)
    ldu = kk + (kk & 1)
    U = torch.empty((m, ldu), dtype=torch.float64, device=A.device)
    sigma = torch.empty(kk, dtype=torch.float64, device=A.device)
    V = torch.empty((n, kk), dtype=torch.float64, device=A.device)
    r = ctypes.c_int64()
    check(lib().lowrank_svd_tsqr(cptr, _stream(A.device), m, n, A.data_ptr(),
                                 A.stride(0) if m > 0 else n, Omega.data_ptr(), Omega.stride(0), l,
                                 iters, k, phases.data_ptr(), perms.data_ptr(), ctypes.byref(opts),
                                 U.data_ptr(), ldu, sigma.data_ptr(), V.data_ptr(), kk,
                                 ctypes.byref(r), ws.data_ptr(), ws.numel()))
    q = r.value
    return U[:, :q], sigma[:q], V[:, :q]


def mixing_tables(mixes, l: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    """l x l tables for lowrank_svd_tsqr from mixes(w) -> (phases, perms) (row w - 1: width w)."""
    ph = torch.zeros((l, l), dtype=torch.float64)
    pm = torch.zeros((l, l), dtype=torch.int32)
    for w in range(1, l + 1):
        a, b = mixes(w)
        ph[w - 1, : len(a)] = torch.as_tensor(a, dtype=torch.float64)
        pm[w - 1, : len(b)] = torch.as_tensor(b, dtype=torch.int32)
    return ph.to(device), pm.to(device)


# ---- kernel-level building blocks (parity tests / microbenchmarks) --------
def gram(X: torch.Tensor) -> torch.Tensor:
    """X^T X over the local rows (Alg. 3 step 1 before aggregation)."""
    m, n = X.shape
    G = torch.empty((n, n), dtype=torch.float64, device=X.device)
    ws = _workspace(lib().tssvd_gram_workspace(m, n), X.device)
    check(lib().tssvd_gram(_stream(X.device), m, n, X.data_ptr(), X.stride(0), G.data_ptr(), n,
                           ws.data_ptr(), ws.numel()))
    return G


def matmul(X: torch.Tensor, M: torch.Tensor, norms: bool = False, out: torch.Tensor | None = None):
    """Y = X M (tall x small) with optional column sums of squares of Y."""
    m, k = X.shape
    c = M.shape[1]
    Y = out if out is not None else torch.empty((m, c + (c & 1)), dtype=torch.float64,
                                                device=X.device)
    nsq = torch.empty(c, dtype=torch.float64, device=X.device) if norms else None
    ws = _workspace(lib().tssvd_matmul_workspace(m, k, c), X.device)
    check(lib().tssvd_matmul(_stream(X.device), m, k, c, X.data_ptr(), X.stride(0),
                             M.contiguous().data_ptr(), M.contiguous().stride(0), Y.data_ptr(),
                             Y.stride(0), _ptr(nsq), ws.data_ptr(), ws.numel()))
    return (Y[:, :c], nsq) if norms else Y[:, :c]


def matmul_tn(X: torch.Tensor, Y: torch.Tensor, l: int | None = None) -> torch.Tensor:
    """Z = X^T Y[:, :l] over the local rows (Alg. 5 step 5 before aggregation)."""
    m, n = X.shape
    l = Y.shape[1] if l is None else l
    Z = torch.empty((n, l), dtype=torch.float64, device=X.device)
    ws = _workspace(lib().tssvd_matmul_tn_workspace(m, n, l), X.device)
    check(lib().tssvd_matmul_tn(_stream(X.device), m, n, l, X.data_ptr(), X.stride(0),
                                Y.data_ptr(), Y.stride(0), Z.data_ptr(), l, ws.data_ptr(),
                                ws.numel()))
    return Z


def sym_eig(B: torch.Tensor, max_sweeps: int = 60):
    """Eigendecomposition of a PSD Gram matrix by one-sided Jacobi: (lambda desc, V with eigvec columns, sweeps)."""
    n = B.shape[0]
    lam = torch.empty(n, dtype=torch.float64, device=B.device)
    Vt = torch.empty((n, n), dtype=torch.float64, device=B.device)
    ws = _workspace(lib().tssvd_sym_eig_workspace(n), B.device)
    sw = ctypes.c_int()
    Bc = B.contiguous()
    check(lib().tssvd_sym_eig(_stream(B.device), n, Bc.data_ptr(), n, lam.data_ptr(),
                              Vt.data_ptr(), n, max_sweeps, ctypes.byref(sw), ws.data_ptr(),
                              ws.numel()))
    return lam, Vt.T, sw.value


def sym_eig_ql(B: torch.Tensor):
    """Eigendecomposition of a symmetric PSD matrix (n <= 160) by tridiagonalisation + implicit QL,
    the solver of Alg. 4 step 8: (lambda desc, V with eigvec columns, QL iterations)."""
    n = B.shape[0]
    lam = torch.empty(n, dtype=torch.float64, device=B.device)
    Vt = torch.empty((n, n), dtype=torch.float64, device=B.device)
    ws = _workspace(lib().tssvd_sym_eig_workspace(n), B.device)
    it = ctypes.c_int()
    Bc = B.contiguous()
    check(lib().tssvd_sym_eig_ql(_stream(B.device), n, Bc.data_ptr(), n, lam.data_ptr(),
                                 Vt.data_ptr(), n, ctypes.byref(it), ws.data_ptr(), ws.numel()))
    return lam, Vt.T, it.value


last_stats = _lib.last_stats
