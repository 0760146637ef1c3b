"""ctypes bindings of the two CPU oracles.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product
package.

  Reference  oracle/_ref/libdetci_ref.so     the UNMODIFIED reference detci
             library compiled from /root/reference (oracle/Makefile) plus the
             harness oracle/ref_capi.cpp.  Built in the dev container, shipped
             prebuilt to the GPU box.
  Oracle     oracle/_ref/libdetci_oracle.so  the C restatement
             (oracle/detci_oracle.c), pinned against Reference and the
             committed goldens (tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libdetci_ref.so"
ORC_SO = HERE / "_ref" / "libdetci_oracle.so"

vp = C.c_void_p
dp = C.POINTER(C.c_double)
u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build_oracle() -> None:
    """Compile the C restatement (and the reference when its sources exist)."""
    subprocess.run(["make", "-C", str(HERE), "all"], check=True, capture_output=True)


# ---------------------------------------------------------------------------
class RefLib:
    """The unmodified reference library (detci) behind ref_capi.cpp."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle ref, needs /root/reference)")
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_full_channel_strings.restype = C.c_long
        L.ref_full_channel_strings.argtypes = [C.c_int, C.c_int, u64p, C.c_long]
        L.ref_table_from_fcidump.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.ref_table_from_dense.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, dp, dp, C.POINTER(vp)]
        L.ref_table_free.argtypes = [vp]
        L.ref_table_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), dp]
        L.ref_table_dense.argtypes = [vp, dp, dp]
        L.ref_write_fcidump.argtypes = [vp, C.c_char_p]
        L.ref_channel_electron_counts.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_parse_det_list.argtypes = [C.c_char_p, C.POINTER(C.c_int), u64p, C.POINTER(C.c_long), u64p,
                                         C.POINTER(C.c_long)]
        L.ref_shuffle_masks.argtypes = [u64p, C.c_long, C.c_int, C.c_uint64]
        L.ref_generate_table.argtypes = [u64p, C.c_long, C.c_int, C.c_int, u32p, u64p, u32p, u64p]
        L.ref_basis_create.argtypes = [vp, u64p, C.c_long, u64p, C.c_long, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                       C.POINTER(vp)]
        L.ref_basis_create_words.argtypes = [vp, C.c_int, u64p, C.c_long, u64p, C.c_long, C.c_int, C.c_int,
                                             C.c_uint64, C.c_int, C.POINTER(vp)]
        L.ref_hij_words.argtypes = [vp, C.c_int, u64p, u64p, u64p, u64p, dp]
        L.ref_basis_free.argtypes = [vp]
        L.ref_basis_stats.argtypes = [vp, dp, C.POINTER(C.c_int)]
        L.ref_basis_diag.argtypes = [vp, dp]
        L.ref_basis_table.argtypes = [vp, C.c_int, C.c_int, u32p, u64p, u32p, u64p]
        L.ref_matvec.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, C.c_int, dp]
        L.ref_matvec_rows.argtypes = [vp, u64p, C.c_long, dp, dp, C.c_int]
        L.ref_davidson.argtypes = [vp, C.c_double, C.c_int, C.c_int, C.c_int, dp, C.POINTER(C.c_int),
                                   C.POINTER(C.c_int), dp, dp, C.c_int, dp]
        L.ref_dense_hamiltonian.argtypes = [vp, dp, C.c_uint64]
        L.ref_hij.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, dp]
        self.APPLY = C.CFUNCTYPE(None, dp, dp, C.c_uint64, vp)
        L.ref_davidson_operator.argtypes = [self.APPLY, vp, dp, C.c_uint64, C.c_double, C.c_int, C.c_int, dp,
                                            C.POINTER(C.c_int), C.POINTER(C.c_int), dp, C.c_int]
        L.ref_brute_force_hij.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, dp]
        L.ref_stored_build.argtypes = [vp, C.c_uint64, C.c_int, C.POINTER(vp), u64p]
        L.ref_stored_free.argtypes = [vp]
        L.ref_stored_arrays.argtypes = [vp, u64p, u32p, dp]
        L.ref_stored_matvec.argtypes = [vp, dp, dp, C.c_int]

    def check(self, code):
        if code:
            raise OracleError(code, self.lib.ref_last_error().decode())

    def max_threads(self) -> int:
        return self.lib.ref_max_threads()

    # integrals ---------------------------------------------------------------
    def table_from_fcidump(self, path) -> "RefTable":
        t = vp()
        self.check(self.lib.ref_table_from_fcidump(str(path).encode(), C.byref(t)))
        return RefTable(self, t)

    def table_from_integrals(self, ints) -> "RefTable":
        h1 = np.ascontiguousarray(ints.h1, dtype=np.float64)
        eri = np.ascontiguousarray(ints.eri, dtype=np.float64)
        t = vp()
        self.check(self.lib.ref_table_from_dense(ints.norbs, ints.nelec, ints.ms2, ints.core, _p(h1, C.c_double),
                                                 _p(eri, C.c_double), C.byref(t)))
        return RefTable(self, t)

    def full_channel_strings(self, norbs, nel) -> np.ndarray:
        n = self.lib.ref_full_channel_strings(norbs, nel, None, 0)
        if n < 0:
            self.check(-n)
        out = np.zeros(n, dtype=np.uint64)
        self.lib.ref_full_channel_strings(norbs, nel, _p(out, C.c_uint64), n)
        return out

    def channel_electron_counts(self, nelec, ms2):
        a, b = C.c_int(), C.c_int()
        self.check(self.lib.ref_channel_electron_counts(nelec, ms2, C.byref(a), C.byref(b)))
        return a.value, b.value

    def generate_table(self, masks, norbs, kind):
        m = np.ascontiguousarray(masks, dtype=np.uint64)
        nflat = C.c_uint64()
        self.check(self.lib.ref_generate_table(_p(m, C.c_uint64), len(m), norbs, kind, None, None, None,
                                               C.byref(nflat)))
        flat = np.zeros(max(nflat.value, 1), dtype=np.uint32)
        off = np.zeros(len(m), dtype=np.uint64)
        ln = np.zeros(len(m), dtype=np.uint32)
        self.check(self.lib.ref_generate_table(_p(m, C.c_uint64), len(m), norbs, kind, _p(flat, C.c_uint32),
                                               _p(off, C.c_uint64), _p(ln, C.c_uint32), C.byref(nflat)))
        return flat[: nflat.value], off, ln

    def davidson_operator(self, apply, diag, tol=1e-8, max_iter=200, max_subspace=20):
        """The reference davidson_solve over a caller-supplied operator
        apply(x: ndarray, y: ndarray) (SURVEY.md 7.2.7 mixed oracle)."""
        diag = np.ascontiguousarray(diag, dtype=np.float64)
        n = len(diag)

        def cb(xp, yp, nn, _user):
            x = np.ctypeslib.as_array(xp, shape=(nn,))
            y = np.ctypeslib.as_array(yp, shape=(nn,))
            apply(x, y)

        fn = self.APPLY(cb)
        e = C.c_double()
        it, st = C.c_int(), C.c_int()
        trace = np.zeros((max_iter, 4))
        self.check(self.lib.ref_davidson_operator(fn, None, _p(diag, C.c_double), n, tol, max_iter, max_subspace,
                                                  C.byref(e), C.byref(it), C.byref(st), _p(trace, C.c_double),
                                                  max_iter))
        return {"energy": e.value, "iterations": it.value, "status": st.value, "trace": trace[: it.value]}

    def shuffle(self, masks, norbs, seed):
        m = np.ascontiguousarray(masks, dtype=np.uint64).copy()
        self.check(self.lib.ref_shuffle_masks(_p(m, C.c_uint64), len(m), norbs, seed))
        return m


class RefTable:
    def __init__(self, ref: RefLib, handle):
        self.ref, self.h = ref, handle

    def __del__(self):
        try:
            self.ref.lib.ref_table_free(self.h)
        except Exception:
            pass

    def integrals(self):
        from paper_2601_16169_b200.synth import Integrals

        n, ne, ms = C.c_int(), C.c_int(), C.c_int()
        core = C.c_double()
        self.ref.check(self.ref.lib.ref_table_info(self.h, C.byref(n), C.byref(ne), C.byref(ms), C.byref(core)))
        h1 = np.zeros((n.value, n.value))
        eri = np.zeros((n.value,) * 4)
        self.ref.check(self.ref.lib.ref_table_dense(self.h, _p(h1, C.c_double), _p(eri, C.c_double)))
        return Integrals(n.value, ne.value, ms.value, core.value, h1, eri)

    def hij(self, bra_a, bra_b, ket_a, ket_b, bit_length=0) -> float:
        out = C.c_double()
        self.ref.check(self.ref.lib.ref_hij(self.h, bra_a, bra_b, ket_a, ket_b, bit_length, C.byref(out)))
        return out.value

    def hij_words(self, bra_a, bra_b, ket_a, ket_b) -> float:
        """Reference hij for Python-int strings of up to 128 orbitals."""
        mask = (1 << 64) - 1
        arrs = [np.array([x & mask, x >> 64], dtype=np.uint64) for x in (bra_a, bra_b, ket_a, ket_b)]
        out = C.c_double()
        self.ref.check(self.ref.lib.ref_hij_words(self.h, 2, *[_p(a, C.c_uint64) for a in arrs], C.byref(out)))
        return out.value

    def brute_force_hij(self, bra_a, bra_b, ket_a, ket_b) -> float:
        out = C.c_double()
        self.ref.check(self.ref.lib.ref_brute_force_hij(self.h, bra_a, bra_b, ket_a, ket_b, C.byref(out)))
        return out.value

    def basis(self, alpha, beta, bit_length=0, cache=True, budget=8 << 30, workers=0) -> "RefBasis":
        a = np.ascontiguousarray(alpha, dtype=np.uint64)
        b = np.ascontiguousarray(beta, dtype=np.uint64)
        h = vp()
        self.ref.check(self.ref.lib.ref_basis_create(self.h, _p(a, C.c_uint64), len(a), _p(b, C.c_uint64), len(b),
                                                     bit_length, int(cache), budget, workers, C.byref(h)))
        return RefBasis(self.ref, h, len(a), len(b))

    def basis_words(self, alpha, beta, bit_length=0, cache=True, budget=8 << 30, workers=0) -> "RefBasis":
        """Strings as (n, words) uint64 arrays (norbs > 64)."""
        a = np.ascontiguousarray(alpha, dtype=np.uint64)
        b = np.ascontiguousarray(beta, dtype=np.uint64)
        words = 1 if a.ndim == 1 else a.shape[1]
        h = vp()
        self.ref.check(self.ref.lib.ref_basis_create_words(self.h, words, _p(a, C.c_uint64), len(a),
                                                           _p(b, C.c_uint64), len(b), bit_length, int(cache),
                                                           budget, workers, C.byref(h)))
        return RefBasis(self.ref, h, len(a), len(b))


class RefBasis:
    def __init__(self, ref, h, na, nb):
        self.ref, self.h, self.na, self.nb = ref, h, na, nb

    def __del__(self):
        try:
            self.ref.lib.ref_basis_free(self.h)
        except Exception:
            pass

    def dim(self):
        return self.na * self.nb

    def diag(self):
        out = np.zeros(self.dim())
        self.ref.check(self.ref.lib.ref_basis_diag(self.h, _p(out, C.c_double)))
        return out

    def table(self, channel, kind):
        n = self.na if channel == 0 else self.nb
        nflat = C.c_uint64()
        self.ref.check(self.ref.lib.ref_basis_table(self.h, channel, kind, None, None, None, C.byref(nflat)))
        flat = np.zeros(max(nflat.value, 1), dtype=np.uint32)
        off = np.zeros(n, dtype=np.uint64)
        ln = np.zeros(n, dtype=np.uint32)
        self.ref.check(self.ref.lib.ref_basis_table(self.h, channel, kind, _p(flat, C.c_uint32), _p(off, C.c_uint64),
                                                    _p(ln, C.c_uint32), C.byref(nflat)))
        return flat[: nflat.value], off, ln

    def matvec(self, x, a=1, b=1, t=1, r=1, workers=0, timings=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        tm = np.zeros(4)
        self.ref.check(self.ref.lib.ref_matvec(self.h, a, b, t, r, _p(x, C.c_double), _p(y, C.c_double), workers,
                                               _p(tm, C.c_double)))
        if timings is not None:
            timings.update(alpha=tm[0], beta=tm[1], mixed=tm[2], combine=tm[3])
        return y

    def matvec_rows(self, rows, x, workers=0):
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(len(rows) * self.nb)
        self.ref.check(self.ref.lib.ref_matvec_rows(self.h, _p(rows, C.c_uint64), len(rows), _p(x, C.c_double),
                                                    _p(y, C.c_double), workers))
        return y.reshape(len(rows), self.nb)

    def davidson(self, tol=1e-8, max_iter=200, max_subspace=20, workers=0, want_vector=False):
        e = C.c_double()
        it = C.c_int()
        st = C.c_int()
        sec = C.c_double()
        trace = np.zeros((max_iter, 4))
        vec = np.zeros(self.dim()) if want_vector else None
        self.ref.check(self.ref.lib.ref_davidson(self.h, tol, max_iter, max_subspace, workers, C.byref(e), C.byref(it),
                                                 C.byref(st), _p(vec, C.c_double) if vec is not None else None,
                                                 _p(trace, C.c_double), max_iter, C.byref(sec)))
        return {"energy": e.value, "iterations": it.value, "status": st.value, "trace": trace[: it.value],
                "eigenvector": vec, "seconds": sec.value}

    def stored_matrix(self, budget=8 << 30, workers=0):
        """Reference build_stored_matrix: (row_offset, col, value) and an
        apply function running the reference stored_matvec."""
        m, nnz = vp(), C.c_uint64()
        self.ref.check(self.ref.lib.ref_stored_build(self.h, budget, workers, C.byref(m), C.byref(nnz)))
        try:
            ro = np.zeros(self.dim() + 1, dtype=np.uint64)
            col = np.zeros(nnz.value, dtype=np.uint32)
            val = np.zeros(nnz.value, dtype=np.float64)
            self.ref.check(self.ref.lib.ref_stored_arrays(m, _p(ro, C.c_uint64), _p(col, C.c_uint32),
                                                          _p(val, C.c_double)))
            def apply(x):
                x = np.ascontiguousarray(x, dtype=np.float64)
                y = np.zeros_like(x)
                self.ref.check(self.ref.lib.ref_stored_matvec(m, _p(x, C.c_double), _p(y, C.c_double), workers))
                return y
            return ro, col, val, apply, m
        except Exception:
            self.ref.lib.ref_stored_free(m)
            raise

    def stored_free(self, m):
        self.ref.lib.ref_stored_free(m)

    def dense_hamiltonian(self, cap=4000):
        out = np.zeros((self.dim(), self.dim()))
        self.ref.check(self.ref.lib.ref_dense_hamiltonian(self.h, _p(out, C.c_double), cap))
        return out


# ---------------------------------------------------------------------------
class OrcIntegrals(C.Structure):
    _fields_ = [("norbs", C.c_int), ("core", C.c_double), ("h1", dp), ("eri", dp)]


class OrcTable(C.Structure):
    _fields_ = [("flat", u32p), ("offset", u64p), ("len", u32p)]


class OrcBasis(C.Structure):
    _fields_ = [("ints", OrcIntegrals), ("alpha", u64p), ("na", C.c_uint64), ("beta", u64p), ("nb", C.c_uint64),
                ("sa", OrcTable), ("da", OrcTable), ("sb", OrcTable), ("db", OrcTable), ("diag", dp)]


class Oracle:
    """The C restatement (oracle/detci_oracle.c)."""

    def __init__(self, path: Path = ORC_SO):
        if not path.exists():
            build_oracle()
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.orc_generate_table.argtypes = [u64p, C.c_uint64, C.c_int, C.c_int, u32p, u64p, u32p, u64p]
        L.orc_hij.restype = C.c_double
        L.orc_hij.argtypes = [C.POINTER(OrcIntegrals), C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_diag.argtypes = [C.POINTER(OrcIntegrals), u64p, C.c_uint64, u64p, C.c_uint64, dp, C.c_int]
        L.orc_matvec.argtypes = [C.POINTER(OrcBasis), dp, dp, C.c_int]
        L.orc_matvec_rows.argtypes = [C.POINTER(OrcBasis), u64p, C.c_uint64, dp, dp, C.c_int]
        L.orc_davidson.argtypes = [C.POINTER(OrcBasis), C.c_double, C.c_int, C.c_int, C.c_int, dp,
                                   C.POINTER(C.c_int), C.POINTER(C.c_int), dp, dp, C.c_int]
        L.orc_inner_product.restype = C.c_double
        L.orc_inner_product.argtypes = [dp, dp, C.c_uint64]

    def generate_table(self, masks, norbs, kind):
        m = np.ascontiguousarray(masks, dtype=np.uint64)
        off = np.zeros(len(m), dtype=np.uint64)
        ln = np.zeros(len(m), dtype=np.uint32)
        nflat = C.c_uint64()
        code = self.lib.orc_generate_table(_p(m, C.c_uint64), len(m), norbs, kind, None, _p(off, C.c_uint64),
                                           _p(ln, C.c_uint32), C.byref(nflat))
        if code:
            raise OracleError(code, "generate_table: duplicate string")
        flat = np.zeros(max(nflat.value, 1), dtype=np.uint32)
        self.lib.orc_generate_table(_p(m, C.c_uint64), len(m), norbs, kind, _p(flat, C.c_uint32),
                                    _p(off, C.c_uint64), _p(ln, C.c_uint32), C.byref(nflat))
        return flat[: nflat.value], off, ln

    def system(self, ints, alpha, beta, threads: Optional[int] = None) -> "OracleSystem":
        return OracleSystem(self, ints, alpha, beta, threads)


class OracleSystem:
    """Keeps arrays alive for the C structs; builds tables and diag."""

    def __init__(self, orc: Oracle, ints, alpha, beta, threads=None):
        self.orc = orc
        self.threads = threads or os.cpu_count() or 1
        self.h1 = np.ascontiguousarray(ints.h1, dtype=np.float64)
        self.eri = np.ascontiguousarray(ints.eri, dtype=np.float64)
        self.ints = OrcIntegrals(ints.norbs, ints.core, _p(self.h1, C.c_double), _p(self.eri, C.c_double))
        self.alpha = np.ascontiguousarray(alpha, dtype=np.uint64)
        self.beta = np.ascontiguousarray(beta, dtype=np.uint64)
        self.na, self.nb = len(self.alpha), len(self.beta)
        self.tables = {}
        for ch, s in ((0, self.alpha), (1, self.beta)):
            for kind in (0, 1):
                self.tables[(ch, kind)] = orc.generate_table(s, ints.norbs, kind)
        self.diag = np.zeros(self.na * self.nb)
        orc.lib.orc_diag(C.byref(self.ints), _p(self.alpha, C.c_uint64), self.na, _p(self.beta, C.c_uint64), self.nb,
                         _p(self.diag, C.c_double), self.threads)
        self._keep = []

        def tab(key):
            f, o, l = self.tables[key]
            f = f if len(f) else np.zeros(1, dtype=np.uint32)
            self._keep.append(f)
            return OrcTable(_p(f, C.c_uint32), _p(o, C.c_uint64), _p(l, C.c_uint32))

        self.basis = OrcBasis(self.ints, _p(self.alpha, C.c_uint64), self.na, _p(self.beta, C.c_uint64), self.nb,
                              tab((0, 0)), tab((0, 1)), tab((1, 0)), tab((1, 1)), _p(self.diag, C.c_double))

    def hij(self, bra_a, bra_b, ket_a, ket_b):
        return self.orc.lib.orc_hij(C.byref(self.ints), bra_a, bra_b, ket_a, ket_b)

    def matvec(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        self.orc.lib.orc_matvec(C.byref(self.basis), _p(x, C.c_double), _p(y, C.c_double), self.threads)
        return y

    def matvec_rows(self, rows, x):
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(len(rows) * self.nb)
        self.orc.lib.orc_matvec_rows(C.byref(self.basis), _p(rows, C.c_uint64), len(rows), _p(x, C.c_double),
                                     _p(y, C.c_double), self.threads)
        return y.reshape(len(rows), self.nb)

    def davidson(self, tol=1e-8, max_iter=200, max_subspace=20):
        e = C.c_double()
        it, st = C.c_int(), C.c_int()
        trace = np.zeros((max_iter, 4))
        vec = np.zeros(self.na * self.nb)
        code = self.orc.lib.orc_davidson(C.byref(self.basis), tol, max_iter, max_subspace, self.threads, C.byref(e),
                                         C.byref(it), C.byref(st), _p(vec, C.c_double), _p(trace, C.c_double), max_iter)
        if code:
            raise OracleError(code, "davidson: bad options")
        return {"energy": e.value, "iterations": it.value, "status": st.value, "trace": trace[: it.value],
                "eigenvector": vec}
