"""Stored-matrix method on the B200 (build_stored_matrix / stored_matvec,
matvec.cpp:240-334) against the reference StoredMatrix:
row_offset and col identical, values and products within
rel_diff = |a-b| / max(1,|a|,|b|) <= 1e-12 (test_matvec.cpp:20-22)."""
import numpy as np
import pytest

from oracle.bindings import RefLib
from paper_2601_16169_b200 import detci, errors, synth
from util import FIXTURES, GOLDEN, load_fixture, rel_diff

pytestmark = pytest.mark.gpu


def gpu_basis(ints, a, b, **kw):
    return detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri, detci.BasisOptions(**kw))


def compare_with_reference(ints, a, b, seed=3):
    ref = RefLib()
    rb = ref.table_from_integrals(ints).basis(a, b)
    ro, col, val, apply, m = rb.stored_matrix(budget=1 << 40)
    try:
        x = synth.random_vector(rb.dim(), seed)
        y_ref = apply(x)
        with gpu_basis(ints, a, b) as g:
            sm = detci.build_stored_matrix(g, 0)
            gro, gcol, gval = sm.arrays()
            assert sm.nonzero_count() == len(col)
            assert np.array_equal(gro, ro) and np.array_equal(gcol, col)
            assert rel_diff(gval, val) <= 1e-12
            y = detci.stored_matvec(sm, x)
            assert rel_diff(y, y_ref) <= 1e-12
            assert rel_diff(y, detci.matvec(g, x)) <= 1e-12   # operator switched back
    finally:
        rb.stored_free(m)


@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_stored_matrix_matches_reference(name):
    ints, d = load_fixture(name)
    compare_with_reference(ints, d["alpha"], d["beta"])


def test_synthetic_stored_matrix_matches_reference():
    ints = synth.synthetic_integrals(12, 8)
    a = synth.synthetic_strings(12, 4, 150)
    b = synth.synthetic_strings(12, 4, 110)[::-1].copy()   # n_alpha != n_beta, unsorted beta
    compare_with_reference(ints, a, b)


def test_stored_davidson_equals_matrix_free():
    """Method::Stored (run.cpp:87-95): the Davidson over the stored SpMV."""
    ints, d = load_fixture("chain8")
    with gpu_basis(ints, d["alpha"], d["beta"]) as g:
        e_free = detci.davidson_solve(g, want_vector=False).energy
        sm = detci.build_stored_matrix(g)
        sm.use(True)
        res = detci.davidson_solve(g, want_vector=False)
        sm.use(False)
    assert res.converged and abs(res.energy - e_free) <= 1e-10 * abs(e_free)
    assert f"{res.energy:.12e}" == "-2.420193979007e+00"


def test_c1_stored_rows_against_reference_rows():
    """C1 (1.28e9 nonzeros, 15 GB in HBM): reference sigma rows from the
    stored SpMV, and the stored product equals the matrix-free sigma."""
    rows = np.load(GOLDEN / "rows_C1.npz")
    ints, a, bb = synth.synthetic_system("C1")
    with gpu_basis(ints, a, bb) as g:
        sm = detci.build_stored_matrix(g, 0)
        assert sm.nonzero_count() == g.nnz()["total"] + g.dimension()
        x = synth.random_vector(g.dimension(), 11)
        y = detci.stored_matvec(sm, x)
        r = rows["rows"].astype(np.int64)
        assert rel_diff(y.reshape(len(a), -1)[r], rows["sigma_rows"]) <= 1e-12
        assert rel_diff(y, detci.matvec(g, x)) <= 1e-12
        sm.release()


def test_capacity_and_errors():
    ints, d = load_fixture("h6_ring")
    with gpu_basis(ints, d["alpha"], d["beta"]) as g:
        with pytest.raises(errors.CapacityError, match=r"stored matrix requires \d+ bytes, budget is 1000 bytes"):
            detci.build_stored_matrix(g, 1000)
        with pytest.raises(errors.InputError):   # operator before the matrix exists
            g._check(g._lib.detci_gpu_set_operator(g.handle, 1))
        sm = detci.build_stored_matrix(g)
        with pytest.raises(errors.InputError):
            detci.stored_matvec(sm, np.zeros(g.dimension() + 1))
    with gpu_basis(ints, d["alpha"], d["beta"], virtual_blocks=2) as g:
        with pytest.raises(errors.UnsupportedError):
            detci.build_stored_matrix(g)
