"""ctypes binding of libdetci_gpu.so (include/detci_gpu.h).

The product path goes through this library only.  If the shared object is
missing the import fails loudly -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "lib" / "libdetci_gpu.so"

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
dp = C.POINTER(C.c_double)
vp = C.c_void_p


class Desc(C.Structure):
    _fields_ = [
        ("device", C.c_int),
        ("rank", C.c_int),
        ("world_size", C.c_int),
        ("nccl_id", u8p),
        ("virtual_blocks", C.c_int),
        ("weighted_partition", C.c_int),
        ("memory_budget_bytes", C.c_uint64),
    ]


class Timings(C.Structure):
    _fields_ = [
        ("alpha_seconds", C.c_double),
        ("beta_seconds", C.c_double),
        ("mixed_seconds", C.c_double),
        ("combine_seconds", C.c_double),
        ("comm_seconds", C.c_double),
        ("h2d_seconds", C.c_double),
        ("d2h_seconds", C.c_double),
        ("total_seconds", C.c_double),
        ("mixed_reduce_seconds", C.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class DavOpts(C.Structure):
    _fields_ = [
        ("tol", C.c_double),
        ("max_iter", C.c_int),
        ("max_subspace", C.c_int),
        ("initial_guess", dp),
    ]


class DavIter(C.Structure):
    _fields_ = [
        ("ritz_value", C.c_double),
        ("residual_norm", C.c_double),
        ("matvec_seconds", C.c_double),
        ("orthogonalization_seconds", C.c_double),
        ("subspace_solve_seconds", C.c_double),
        ("max_gram_deviation", C.c_double),
        ("restarted", C.c_int),
    ]


class DavResult(C.Structure):
    _fields_ = [
        ("status", C.c_int),
        ("converged", C.c_int),
        ("iterations", C.c_int),
        ("energy", C.c_double),
        ("seconds", C.c_double),
        ("eigenvector", dp),
        ("trace", C.POINTER(DavIter)),
        ("trace_cap", C.c_int),
    ]


class DavBlockOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("max_subspace", C.c_int), ("nroots", C.c_int)]


class DavBlockResult(C.Structure):
    _fields_ = [
        ("status", C.c_int),
        ("converged", C.c_int),
        ("iterations", C.c_int),
        ("seconds", C.c_double),
        ("energies", dp),
        ("residuals", dp),
        ("eigenvectors", dp),
        ("trace", C.POINTER(DavIter)),
        ("trace_cap", C.c_int),
    ]


class Plan(C.Structure):
    _fields_ = [("mixed_kmax", C.c_int), ("mixed_segments", C.c_int), ("mixed_windows", C.c_int),
                ("mixed_sell_entries", C.c_uint64), ("d_bytes", C.c_uint64),
                ("mixed_lds_bytes", C.c_uint64), ("d_read_bytes", C.c_uint64)]


TRACE_CB = C.CFUNCTYPE(None, C.POINTER(DavIter), C.c_int, vp)

# name -> (restype, argtypes); mirrors include/detci_gpu.h exactly
SIGNATURES = {
    "detci_gpu_abi_version": (C.c_int, []),
    "detci_gpu_create": (C.c_int, [C.POINTER(Desc), C.POINTER(vp)]),
    "detci_gpu_create_loopback": (C.c_int, [C.POINTER(Desc), C.c_uint64, C.POINTER(vp)]),
    "detci_gpu_destroy": (None, [vp]),
    "detci_gpu_last_error": (C.c_char_p, [vp]),
    "detci_gpu_nccl_unique_id": (C.c_int, [u8p]),
    "detci_gpu_set_strings": (C.c_int, [vp, C.c_int, u64p, C.c_size_t, u64p, C.c_size_t]),
    "detci_gpu_set_strings_words": (C.c_int, [vp, C.c_int, C.c_int, u64p, C.c_size_t, u64p, C.c_size_t]),
    "detci_gpu_set_integrals": (C.c_int, [vp, C.c_double, dp, dp]),
    "detci_gpu_build_basis": (C.c_int, [vp]),
    "detci_gpu_helper_size": (C.c_int, [vp, C.c_int, C.c_int, u64p]),
    "detci_gpu_get_helpers": (C.c_int, [vp, C.c_int, C.c_int, u32p, u64p, u32p]),
    "detci_gpu_local_rows": (C.c_int, [vp, u64p, u64p, u64p]),
    "detci_gpu_nnz": (C.c_int, [vp, u64p, u64p, u64p, u64p]),
    "detci_gpu_diag": (C.c_int, [vp, dp]),
    "detci_gpu_sigma": (C.c_int, [vp, vp, vp, C.POINTER(Timings)]),
    "detci_gpu_sigma_device": (C.c_int, [vp, vp, vp, C.POINTER(Timings)]),
    "detci_gpu_sigma_async": (C.c_int, [vp, vp, vp]),
    "detci_gpu_stream": (C.c_int, [vp, C.POINTER(vp)]),
    "detci_gpu_launch_count": (C.c_int, [u64p]),
    "detci_gpu_sigma_plan": (C.c_int, [vp, C.POINTER(Plan)]),
    "detci_gpu_rank_seconds": (C.c_int, [vp, dp, C.c_int, C.POINTER(C.c_int)]),
    "detci_gpu_rank_phase_seconds": (C.c_int, [vp, dp, C.c_int, C.POINTER(C.c_int)]),
    "detci_gpu_rebalance": (C.c_int, [vp, C.c_int, dp]),
    "detci_gpu_alloc_vector": (C.c_int, [vp, C.POINTER(vp)]),
    "detci_gpu_free_vector": (C.c_int, [vp, vp]),
    "detci_gpu_copy_vector": (C.c_int, [vp, vp, vp, C.c_int]),
    "detci_gpu_davidson": (C.c_int, [vp, C.POINTER(DavOpts), C.POINTER(DavResult), TRACE_CB, vp]),
    "detci_gpu_davidson_roots": (C.c_int, [vp, C.POINTER(DavBlockOpts), C.POINTER(DavBlockResult)]),
    "detci_gpu_sigma_block": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.c_int]),
    "detci_gpu_build_stored": (C.c_int, [vp, C.c_uint64, u64p]),
    "detci_gpu_stored_arrays": (C.c_int, [vp, u64p, u32p, dp]),
    "detci_gpu_set_operator": (C.c_int, [vp, C.c_int]),
    "detci_gpu_release_stored": (C.c_int, [vp]),
    "detci_gpu_inner_product": (C.c_int, [vp, dp, dp, C.c_uint64, dp]),
    "detci_gpu_orthonormalize": (C.c_int, [vp, dp, C.c_int, C.c_uint64, dp, dp, C.POINTER(C.c_int)]),
    "detci_gpu_precondition": (C.c_int, [vp, dp, dp, C.c_uint64, C.c_double, dp]),
    "detci_gpu_factorized_element": (
        C.c_int,
        [C.c_int, C.c_double, dp, dp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, dp],
    ),
    "detci_gpu_factorized_element_words": (
        C.c_int,
        [C.c_int, C.c_int, C.c_double, dp, dp, u64p, u64p, u64p, u64p, dp],
    ),
    "detci_gpu_plan_partition": (
        C.c_int,
        [C.c_uint64, C.c_uint64, u32p, u32p, u32p, u32p, C.c_int, C.c_int, u64p],
    ),
}

_lib = None


def load() -> C.CDLL:
    """Load libdetci_gpu.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("DETCI_GPU_LIB", LIB_PATH))
    if not path.exists():
        raise ImportError(
            f"libdetci_gpu.so not found at {path}; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
