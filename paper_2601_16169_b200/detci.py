"""Host-side mirror of the reference detci API for the sigma hot path.

Same names, argument meaning and error behaviour as the reference C++ API
(paths relative to /root/reference/proj/core):

  Basis / build_basis      basis.hpp:42-90     -> GpuBasis / build_basis
  matvec                   matvec.hpp:64-68    -> matvec
  LinearOperator           davidson.hpp:28     -> GpuBasis.linear_operator()
  DavidsonOptions/Result   davidson.hpp:30-65  -> DavidsonOptions / DavidsonResult
  davidson_solve           davidson.hpp:85-86  -> davidson_solve
  inner_product / orthonormalize / precondition  davidson.hpp:67-81

Every call goes through libdetci_gpu.so (include/detci_gpu.h); there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib
from .errors import InputError, raise_for

SOLVE_STATUS = {0: "converged", 1: "max_iterations", 2: "stagnated"}


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _string_words(a, norbs: int) -> np.ndarray:
    """Channel strings as uint64 words: shape (n,) for norbs <= 64, (n, 2)
    for norbs <= 128 (word w = orbitals 64w..64w+63, the BitString word
    order, bitstring.hpp:33-51).  Accepts Python ints of any size or an
    (n, 2) uint64 array."""
    if norbs <= 64:
        return _u64(a)
    if isinstance(a, np.ndarray) and a.ndim == 2:
        if a.shape[1] != 2:
            raise InputError("strings: expected an (n, 2) uint64 array for norbs > 64")
        return _u64(a)
    mask = (1 << 64) - 1
    return _u64([[int(x) & mask, int(x) >> 64] for x in a]).reshape(-1, 2)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


@dataclass
class BasisOptions:
    """basis.hpp:24-34 (bit_length/cache are host-packing knobs with no
    device meaning; the budget applies to device memory)."""

    memory_budget_bytes: int = 0
    device: int = 0
    rank: int = 0
    world_size: int = 1
    nccl_id: Optional[bytes] = None
    virtual_blocks: int = 1
    weighted_partition: bool = False
    # world_size ranks in this process (one host thread each) over the
    # loopback transport instead of NCCL; ranks of one group share the id
    loopback_group: Optional[int] = None


@dataclass
class DavidsonOptions:
    tol: float = 1e-8
    max_iter: int = 200
    max_subspace: int = 20
    initial_guess: Optional[np.ndarray] = None


@dataclass
class IterationStats:
    ritz_value: float
    residual_norm: float
    matvec_seconds: float
    orthogonalization_seconds: float
    subspace_solve_seconds: float
    max_gram_deviation: float
    restarted: bool


@dataclass
class DavidsonResult:
    status: str
    converged: bool
    energy: float
    eigenvector: Optional[np.ndarray]
    iterations: List[IterationStats] = field(default_factory=list)
    seconds: float = 0.0


class GpuBasis:
    """Device-resident tensor-product basis (the reference's Basis)."""

    def __init__(self, norbs: int, alpha: Sequence[int], beta: Sequence[int], core: float,
                 h1: np.ndarray, eri: np.ndarray, opts: BasisOptions = BasisOptions()):
        self._lib = _lib.load()
        self._h = C.c_void_p()
        desc = _lib.Desc()
        desc.device = opts.device
        desc.rank = opts.rank
        desc.world_size = opts.world_size
        self._nccl_id = None
        if opts.nccl_id is not None:
            self._nccl_id = (C.c_uint8 * 128).from_buffer_copy(opts.nccl_id)
            desc.nccl_id = C.cast(self._nccl_id, _lib.u8p)
        desc.virtual_blocks = opts.virtual_blocks
        desc.weighted_partition = int(opts.weighted_partition)
        desc.memory_budget_bytes = opts.memory_budget_bytes
        if opts.loopback_group is not None:
            self._check(self._lib.detci_gpu_create_loopback(C.byref(desc), int(opts.loopback_group),
                                                            C.byref(self._h)), use_handle=False)
        else:
            self._check(self._lib.detci_gpu_create(C.byref(desc), C.byref(self._h)), use_handle=False)
        self.norbs = int(norbs)
        self.alpha = _string_words(alpha, self.norbs)
        self.beta = _string_words(beta, self.norbs)
        self.n_alpha = len(self.alpha)
        self.n_beta = len(self.beta)
        words = 1 if self.alpha.ndim == 1 else 2
        self._check(self._lib.detci_gpu_set_strings_words(self._h, self.norbs, words,
                                                          _ptr(self.alpha, C.c_uint64), self.n_alpha,
                                                          _ptr(self.beta, C.c_uint64), self.n_beta))
        h1 = _f64(h1).reshape(-1)
        eri = _f64(eri).reshape(-1)
        if h1.size != norbs ** 2 or eri.size != norbs ** 4:
            raise InputError("integrals: expected norbs^2 one-electron and norbs^4 two-electron values")
        self._check(self._lib.detci_gpu_set_integrals(self._h, float(core), _ptr(h1, C.c_double),
                                                      _ptr(eri, C.c_double)))
        self._check(self._lib.detci_gpu_build_basis(self._h))
        self._query_rows()

    def _query_rows(self) -> None:
        b, e, nb = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._check(self._lib.detci_gpu_local_rows(self._h, C.byref(b), C.byref(e), C.byref(nb)))
        self.row_begin, self.row_end = b.value, e.value
        self.local_dim = (e.value - b.value) * nb.value

    def rebalance(self, rounds: int = 1) -> float:
        """Measured rebalance of the alpha-row blocks and mixed column
        shares (detci_gpu_rebalance; collective with several ranks).  Returns
        the slowest/mean rank ratio measured before rebalancing; the local
        row range may change (row_begin, row_end, local_dim are refreshed)."""
        r = C.c_double(1.0)
        self._check(self._lib.detci_gpu_rebalance(self._h, int(rounds), C.byref(r)))
        self._query_rows()
        return r.value

    # -- plumbing -----------------------------------------------------------
    def _check(self, code: int, use_handle: bool = True) -> None:
        if code:
            msg = self._lib.detci_gpu_last_error(self._h if use_handle and self._h else None)
            raise_for(code, (msg or b"").decode())

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            self._lib.detci_gpu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def dimension(self) -> int:
        return self.n_alpha * self.n_beta

    # -- reference Basis members -------------------------------------------
    def table(self, channel: int, kind: int):
        """(flat u32, offset u64[n], len u32[n]) -- FlatExcitationTable."""
        n = self.n_alpha if channel == 0 else self.n_beta
        nflat = C.c_uint64()
        self._check(self._lib.detci_gpu_helper_size(self._h, channel, kind, C.byref(nflat)))
        flat = np.zeros(nflat.value, dtype=np.uint32)
        off = np.zeros(n, dtype=np.uint64)
        ln = np.zeros(n, dtype=np.uint32)
        self._check(self._lib.detci_gpu_get_helpers(self._h, channel, kind, _ptr(flat, C.c_uint32),
                                                    _ptr(off, C.c_uint64), _ptr(ln, C.c_uint32)))
        return flat, off, ln

    @property
    def singles_a(self):
        return self.table(0, 0)

    @property
    def doubles_a(self):
        return self.table(0, 1)

    @property
    def singles_b(self):
        return self.table(1, 0)

    @property
    def doubles_b(self):
        return self.table(1, 1)

    def diag(self) -> np.ndarray:
        out = np.zeros(self.local_dim, dtype=np.float64)
        self._check(self._lib.detci_gpu_diag(self._h, _ptr(out, C.c_double)))
        return out

    def nnz(self) -> dict:
        t, a, b, m = (C.c_uint64() for _ in range(4))
        self._check(self._lib.detci_gpu_nnz(self._h, C.byref(t), C.byref(a), C.byref(b), C.byref(m)))
        return {"total": t.value, "alpha": a.value, "beta": b.value, "mixed": m.value}

    def sigma_plan(self) -> dict:
        """Shape of the mixed-term plan (K, segments, ja windows, SELL
        entries, D bytes); windows are 0 before the first sigma."""
        p = _lib.Plan()
        self._check(self._lib.detci_gpu_sigma_plan(self._h, C.byref(p)))
        return {k: getattr(p, k) for k, _ in p._fields_}

    def rank_seconds(self) -> List[float]:
        """Virtual blocks: device seconds of each block-rank's share of the
        last timed sigma (matvec(..., timings={})), transfers excluded."""
        cnt = C.c_int()
        buf = (C.c_double * 64)()
        self._check(self._lib.detci_gpu_rank_seconds(self._h, buf, 64, C.byref(cnt)))
        return [buf[i] for i in range(min(cnt.value, 64))]

    def rank_phase_seconds(self) -> List[List[float]]:
        """rank_seconds split by phase: [alpha, beta, mixed, combine] per
        block-rank."""
        cnt = C.c_int()
        buf = (C.c_double * 256)()
        self._check(self._lib.detci_gpu_rank_phase_seconds(self._h, buf, 256, C.byref(cnt)))
        n = min(cnt.value, 256) // 4
        return [[buf[4 * r + q] for q in range(4)] for r in range(n)]

    def linear_operator(self) -> Callable[[np.ndarray, np.ndarray], None]:
        """LinearOperator (davidson.hpp:28): y = H x on host arrays."""
        return lambda x, y: matvec(self, x, y)


class StoredMatrix:
    """StoredMatrix (matvec.hpp:73-80) held in HBM by the basis's handle:
    the reference CSR layout (row_offset, col, value)."""

    def __init__(self, basis: GpuBasis, nnz: int):
        self.basis = basis
        self.dimension = basis.dimension()
        self._nnz = nnz

    def nonzero_count(self) -> int:
        return self._nnz

    def arrays(self):
        """(row_offset u64[dim+1], col u32[nnz], value f64[nnz]) copied to the host."""
        ro = np.zeros(self.dimension + 1, dtype=np.uint64)
        col = np.zeros(self._nnz, dtype=np.uint32)
        val = np.zeros(self._nnz, dtype=np.float64)
        self.basis._check(self.basis._lib.detci_gpu_stored_arrays(
            self.basis.handle, _ptr(ro, C.c_uint64), _ptr(col, C.c_uint32), _ptr(val, C.c_double)))
        return ro, col, val

    def use(self, on: bool = True) -> None:
        """Method::Stored: every sigma (matvec, davidson_solve) uses the SpMV."""
        self.basis._check(self.basis._lib.detci_gpu_set_operator(self.basis.handle, 1 if on else 0))

    def release(self) -> None:
        self.basis._check(self.basis._lib.detci_gpu_release_stored(self.basis.handle))


def build_stored_matrix(basis: GpuBasis, memory_budget_bytes: int = 8 << 30) -> StoredMatrix:
    """build_stored_matrix (matvec.hpp:84-86) on the device; CapacityError
    over the budget (0 = free device memory) as matvec.cpp:262-269."""
    nnz = C.c_uint64()
    basis._check(basis._lib.detci_gpu_build_stored(basis.handle, int(memory_budget_bytes), C.byref(nnz)))
    return StoredMatrix(basis, nnz.value)


def stored_matvec(m: StoredMatrix, x: np.ndarray, y: Optional[np.ndarray] = None) -> np.ndarray:
    """stored_matvec (matvec.hpp:89-90): y = H x from the stored values;
    length mismatch -> InputError (matvec.cpp:320-321)."""
    x = _f64(x)
    if x.size != m.dimension or (y is not None and y.size != m.dimension):
        raise InputError("stored_matvec: vector length does not match matrix dimension")
    lib, h = m.basis._lib, m.basis.handle
    m.basis._check(lib.detci_gpu_set_operator(h, 1))
    try:
        return matvec(m.basis, x, y)
    finally:
        m.basis._check(lib.detci_gpu_set_operator(h, 0))


def build_basis(alpha: Sequence[int], beta: Sequence[int], integrals, opts: BasisOptions = BasisOptions()) -> GpuBasis:
    """build_basis (basis.hpp:85-86).  `integrals` exposes norbs, core, h1 (n^2), eri (n^4)."""
    return GpuBasis(integrals.norbs, alpha, beta, integrals.core, integrals.h1, integrals.eri, opts)


def matvec(basis: GpuBasis, x: np.ndarray, y: Optional[np.ndarray] = None, timings: Optional[dict] = None) -> np.ndarray:
    """y = H x (matvec.hpp:64-68); length mismatch -> InputError (matvec.cpp:128-130)."""
    x = _f64(x)
    if x.size != basis.local_dim or (y is not None and y.size != basis.local_dim):
        raise InputError(f"matvec: vector length {x.size} does not match basis dimension {basis.local_dim}")
    out = np.empty(basis.local_dim, dtype=np.float64) if y is None else y
    if out.dtype != np.float64 or not out.flags["C_CONTIGUOUS"]:
        raise InputError("matvec: y must be a contiguous float64 array")
    if timings is None:   # host copies overlapped with the kernels (sigma_host)
        basis._check(basis._lib.detci_gpu_sigma(basis.handle, x.ctypes.data, out.ctypes.data, None))
        return out
    tm = _lib.Timings()
    basis._check(basis._lib.detci_gpu_sigma(basis.handle, x.ctypes.data, out.ctypes.data, C.byref(tm)))
    timings.update(tm.as_dict())
    return out


def matvec_block(basis: GpuBasis, X: np.ndarray) -> np.ndarray:
    """Y[i] = H X[i] for m vectors through one blocked device pass
    (detci_gpu_sigma_block; element work shared by the vectors)."""
    X = _f64(X)
    X = X.reshape(-1, basis.local_dim)
    m = X.shape[0]
    lib = basis._lib
    dx = (C.c_void_p * m)()
    dy = (C.c_void_p * m)()
    try:
        for i in range(m):
            for arr in (dx, dy):
                p = C.c_void_p()
                basis._check(lib.detci_gpu_alloc_vector(basis.handle, C.byref(p)))
                arr[i] = p.value
            basis._check(lib.detci_gpu_copy_vector(basis.handle, dx[i], X[i].ctypes.data, 0))
        basis._check(lib.detci_gpu_sigma_block(basis.handle, C.cast(dx, C.POINTER(C.c_void_p)),
                                               C.cast(dy, C.POINTER(C.c_void_p)), m))
        Y = np.empty_like(X)
        for i in range(m):
            basis._check(lib.detci_gpu_copy_vector(basis.handle, Y[i].ctypes.data, dy[i], 1))
        return Y
    finally:
        for arr in (dx, dy):
            for i in range(m):
                if arr[i]:
                    lib.detci_gpu_free_vector(basis.handle, arr[i])


def davidson_solve(basis: GpuBasis, opts: DavidsonOptions = DavidsonOptions(), want_vector: bool = True,
                   callback: Optional[Callable[[IterationStats, int], None]] = None) -> DavidsonResult:
    """davidson_solve (davidson.hpp:85-86) over the device sigma and device vector ops."""
    o = _lib.DavOpts()
    o.tol = opts.tol
    o.max_iter = opts.max_iter
    o.max_subspace = opts.max_subspace
    guess = None
    if opts.initial_guess is not None:
        guess = _f64(opts.initial_guess)
        if guess.size != basis.local_dim:
            raise InputError("davidson_solve: initial guess length mismatch")
        o.initial_guess = _ptr(guess, C.c_double)
    r = _lib.DavResult()
    vec = np.zeros(basis.local_dim, dtype=np.float64) if want_vector else None
    if vec is not None:
        r.eigenvector = _ptr(vec, C.c_double)
    cap = max(1, opts.max_iter)
    trace = (_lib.DavIter * cap)()
    r.trace = C.cast(trace, C.POINTER(_lib.DavIter))
    r.trace_cap = cap

    def _cb(it_ptr, i, _user):
        if callback is not None:
            it = it_ptr.contents
            callback(_iter_stats(it), i)

    cb = _lib.TRACE_CB(_cb)
    basis._check(basis._lib.detci_gpu_davidson(basis.handle, C.byref(o), C.byref(r), cb, None))
    its = [_iter_stats(trace[i]) for i in range(r.iterations)]
    return DavidsonResult(status=SOLVE_STATUS[r.status], converged=bool(r.converged), energy=r.energy,
                          eigenvector=vec, iterations=its, seconds=r.seconds)


@dataclass
class MultiRootResult:
    status: str
    converged: bool
    energies: np.ndarray
    residuals: np.ndarray
    eigenvectors: Optional[np.ndarray]     # (nroots, local_dim)
    iterations: List[IterationStats] = field(default_factory=list)
    seconds: float = 0.0


def davidson_roots(basis: GpuBasis, nroots: int, tol: float = 1e-8, max_iter: int = 200,
                   max_subspace: int = 0, want_vectors: bool = True) -> MultiRootResult:
    """Lowest `nroots` eigenpairs by block Davidson (BASELINE config C5); the
    reference itself is single-root (davidson.hpp:83-86)."""
    o = _lib.DavBlockOpts()
    o.tol = tol
    o.max_iter = max_iter
    o.max_subspace = max_subspace or max(20, 2 * nroots + 4)
    o.nroots = nroots
    r = _lib.DavBlockResult()
    e = np.zeros(max(nroots, 1))
    res = np.zeros(max(nroots, 1))
    r.energies = _ptr(e, C.c_double)
    r.residuals = _ptr(res, C.c_double)
    vec = np.zeros((max(nroots, 1), basis.local_dim)) if want_vectors else None
    if vec is not None:
        r.eigenvectors = _ptr(vec, C.c_double)
    cap = max(1, max_iter)
    trace = (_lib.DavIter * cap)()
    r.trace = C.cast(trace, C.POINTER(_lib.DavIter))
    r.trace_cap = cap
    basis._check(basis._lib.detci_gpu_davidson_roots(basis.handle, C.byref(o), C.byref(r)))
    return MultiRootResult(status=SOLVE_STATUS[r.status], converged=bool(r.converged), energies=e[:nroots],
                           residuals=res[:nroots], eigenvectors=vec,
                           iterations=[_iter_stats(trace[i]) for i in range(r.iterations)], seconds=r.seconds)


def _iter_stats(it) -> IterationStats:
    return IterationStats(it.ritz_value, it.residual_norm, it.matvec_seconds, it.orthogonalization_seconds,
                          it.subspace_solve_seconds, it.max_gram_deviation, bool(it.restarted))


def inner_product(basis: GpuBasis, x, y) -> float:
    x, y = _f64(x), _f64(y)
    if x.size != y.size:
        raise InputError(f"inner_product: length mismatch ({x.size} vs {y.size})")
    out = C.c_double()
    basis._check(basis._lib.detci_gpu_inner_product(basis.handle, _ptr(x, C.c_double), _ptr(y, C.c_double),
                                                    x.size, C.byref(out)))
    return out.value


def orthonormalize(basis: GpuBasis, vs: Sequence[np.ndarray], candidate) -> Optional[np.ndarray]:
    cand = _f64(candidate)
    k = len(vs)
    mat = _f64(np.stack(vs)) if k else np.zeros(1)
    out = np.zeros_like(cand)
    acc = C.c_int()
    basis._check(basis._lib.detci_gpu_orthonormalize(basis.handle, _ptr(mat, C.c_double), k, cand.size,
                                                     _ptr(cand, C.c_double), _ptr(out, C.c_double), C.byref(acc)))
    return out if acc.value else None


def precondition(basis: GpuBasis, residual, diag, theta: float) -> np.ndarray:
    r, d = _f64(residual), _f64(diag)
    if r.size != d.size:
        raise InputError("precondition: residual and diagonal lengths differ")
    out = np.zeros_like(r)
    basis._check(basis._lib.detci_gpu_precondition(basis.handle, _ptr(r, C.c_double), _ptr(d, C.c_double),
                                                   r.size, float(theta), _ptr(out, C.c_double)))
    return out


def factorized_element(integrals, bra_a: int, bra_b: int, ket_a: int, ket_b: int) -> float:
    """<bra|H|ket> from the kernels' factorized closed forms (host, no GPU)."""
    lib = _lib.load()
    h1 = _f64(integrals.h1).reshape(-1)
    eri = _f64(integrals.eri).reshape(-1)
    out = C.c_double()
    if integrals.norbs > 64:
        mask = (1 << 64) - 1
        w = [np.array([int(x) & mask, int(x) >> 64], dtype=np.uint64) for x in (bra_a, bra_b, ket_a, ket_b)]
        code = lib.detci_gpu_factorized_element_words(integrals.norbs, 2, float(integrals.core),
                                                      _ptr(h1, C.c_double), _ptr(eri, C.c_double),
                                                      *[_ptr(a, C.c_uint64) for a in w], C.byref(out))
        raise_for(code, (lib.detci_gpu_last_error(None) or b"").decode())
        return out.value
    code = lib.detci_gpu_factorized_element(integrals.norbs, float(integrals.core), _ptr(h1, C.c_double),
                                            _ptr(eri, C.c_double), bra_a, bra_b, ket_a, ket_b, C.byref(out))
    raise_for(code, (lib.detci_gpu_last_error(None) or b"").decode())
    return out.value


def plan_partition(n_alpha: int, n_beta: int, len_sa, len_da, len_sb, len_db, P: int, weighted: bool) -> np.ndarray:
    """Alpha-block boundaries for P ranks (host only; see detci_gpu_plan_partition)."""
    lib = _lib.load()
    arrs = [np.ascontiguousarray(np.asarray(a, dtype=np.uint32)) for a in (len_sa, len_da, len_sb, len_db)]
    blk = np.zeros(P + 1, dtype=np.uint64)
    code = lib.detci_gpu_plan_partition(n_alpha, n_beta, *[_ptr(a, C.c_uint32) for a in arrs], P, int(weighted),
                                        _ptr(blk, C.c_uint64))
    raise_for(code, (lib.detci_gpu_last_error(None) or b"").decode())
    return blk
