"""Device Davidson against the reference davidson_solve (test_davidson.cpp,
acceptance criteria 1, 4 and 6): energies within 1e-10 relative of the
reference / dense oracle on the fixtures, within 1e-8 Ha at C1, trace
invariants with forced restarts, status semantics, option validation, and
the vector helpers."""
import numpy as np
import pytest

from paper_2601_16169_b200 import detci, errors, synth
from util import FIXTURES, GOLDEN, golden_meta, load_fixture

pytestmark = pytest.mark.gpu


def gpu_basis(ints, a, b, **kw):
    return detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri, detci.BasisOptions(**kw))


@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_energies(name):
    ints, d = load_fixture(name)
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        res = detci.davidson_solve(b)
        assert res.converged and res.status == "converged"
        want = float(d["energy"])
        assert abs(res.energy - want) <= 1e-10 * abs(want)
        if "dense_ground" in d:
            assert abs(res.energy - float(d["dense_ground"])) <= 1e-10 * abs(float(d["dense_ground"]))
        v = res.eigenvector
        assert abs(np.linalg.norm(v) - 1.0) <= 1e-12
        # eigenvector residual through the device operator
        assert np.linalg.norm(detci.matvec(b, v) - res.energy * v) <= 1e-6


def test_chain8_shipped_golden():
    ints, d = load_fixture("chain8")
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        res = detci.davidson_solve(b)
    assert f"{res.energy:.12e}" == "-2.420193979007e+00"     # proj/test_output.txt:33
    assert len(res.iterations) == int(d["iterations"])


def test_trace_invariants_with_forced_restarts():
    """test_davidson.cpp:108-139 (h6_ring, max_subspace 6)."""
    ints, d = load_fixture("h6_ring")
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        opts = detci.DavidsonOptions(max_subspace=6)
        res = detci.davidson_solve(b, opts)
        diag_min = b.diag().min()
    assert res.converged and len(res.iterations) <= 100
    assert res.energy <= diag_min + opts.tol
    assert abs(res.energy - float(d["energy_ms6"])) <= 1e-10 * abs(float(d["energy_ms6"]))
    saw_restart = False
    for i, it in enumerate(res.iterations):
        assert it.max_gram_deviation <= 1e-12
        assert np.isfinite(it.residual_norm)
        saw_restart |= it.restarted
        if i > 0 and not it.restarted:
            prev = res.iterations[i - 1]
            assert it.ritz_value <= prev.ritz_value + 1e-12 * max(1.0, abs(prev.ritz_value))
    assert saw_restart
    assert res.iterations[-1].residual_norm <= opts.tol


def test_trace_matches_reference_iteration_by_iteration():
    ints, d = load_fixture("chain8")
    ref = d["trace"]
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        res = detci.davidson_solve(b)
    assert len(res.iterations) == len(ref)
    # intermediate Ritz values: 1e-9 relative.  At an iteration whose
    # correction is nearly inside the subspace the renormalised vector
    # carries the summation-order rounding of the dot products amplified
    # (chain8 iteration values move by ~1e-10 between reduction orders);
    # the final energy is held to 1e-10 (test_chain8_shipped_golden).
    for it, r in zip(res.iterations, ref):
        assert abs(it.ritz_value - r[0]) <= 1e-9 * abs(r[0])
        assert it.restarted == bool(r[3])


def test_non_convergence_carries_trace():
    ints, d = load_fixture("h6_ring")
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        res = detci.davidson_solve(b, detci.DavidsonOptions(max_iter=2))
    assert not res.converged and res.status == "max_iterations" and len(res.iterations) == 2


def test_deterministic_across_runs():
    ints, d = load_fixture("h4_chain")
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        r1 = detci.davidson_solve(b)
        r2 = detci.davidson_solve(b)
    assert r1.energy == r2.energy and len(r1.iterations) == len(r2.iterations)
    for a, c in zip(r1.iterations, r2.iterations):
        assert a.ritz_value == c.ritz_value and a.residual_norm == c.residual_norm


def test_option_validation():
    ints, d = load_fixture("h2_minimal")
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        with pytest.raises(errors.ConfigError):
            detci.davidson_solve(b, detci.DavidsonOptions(tol=0.0))
        with pytest.raises(errors.ConfigError):
            detci.davidson_solve(b, detci.DavidsonOptions(max_subspace=1))
        with pytest.raises(errors.ConfigError):
            detci.davidson_solve(b, detci.DavidsonOptions(max_iter=0))
        with pytest.raises(errors.InputError):
            detci.davidson_solve(b, detci.DavidsonOptions(initial_guess=np.zeros(b.dimension())))
        with pytest.raises(errors.InputError):
            detci.davidson_solve(b, detci.DavidsonOptions(initial_guess=np.ones(3)))


def test_initial_guess_path():
    ints, d = load_fixture("h4_chain")
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        guess = np.ones(b.dimension())
        res = detci.davidson_solve(b, detci.DavidsonOptions(initial_guess=guess))
    assert res.converged and abs(res.energy - float(d["energy"])) <= 1e-10 * abs(float(d["energy"]))


def test_virtual_blocks_davidson():
    ints = synth.synthetic_integrals(12, 8)
    s = synth.synthetic_strings(12, 4, 200)
    meta = golden_meta()["s12"]
    with gpu_basis(ints, s, s, virtual_blocks=4, weighted_partition=True) as b:
        res = detci.davidson_solve(b)
    assert res.converged and abs(res.energy - meta["energy"]) <= 1e-10 * abs(meta["energy"])


def test_c1_energy_against_reference_pipeline():
    """Full reference Davidson at the C1 shape (PR1 oracle): within 1e-8 Ha."""
    meta = golden_meta()["C1"]
    if "energy" not in meta:
        pytest.skip("C1 reference energy not generated")
    ints, a, bb = synth.synthetic_system("C1")
    with gpu_basis(ints, a, bb) as b:
        res = detci.davidson_solve(b, want_vector=False)
    assert res.converged
    assert abs(res.energy - meta["energy"]) <= 1e-8


def test_vector_helpers():
    """inner_product / orthonormalize / precondition (test_davidson.cpp:34-69)."""
    ints, d = load_fixture("h2_minimal")
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        assert detci.inner_product(b, [1, 2], [3, 4]) == 11.0
        with pytest.raises(errors.InputError):
            detci.inner_product(b, [1.0, 0.0], [1.0])
        vs = [np.array([1.0, 0, 0]), np.array([0, 1.0, 0])]
        out = detci.orthonormalize(b, vs, [0.0, 0.0, 2.5])
        assert out is not None and abs(out[2] - 1.0) <= 1e-15
        assert detci.orthonormalize(b, vs, vs[0]) is None
        assert detci.orthonormalize(b, vs, [0.0, 0.0, 0.0]) is None
        for rep in range(20):
            cand = synth.random_vector(3, 400 + rep)
            o = detci.orthonormalize(b, vs, cand)
            if o is None:
                continue
            assert all(abs(v @ o) <= 1e-12 for v in vs) and abs(o @ o - 1.0) <= 1e-12
        c = detci.precondition(b, [1.0, 1.0, 0.0], [3.0, 1.0 + 1e-12, 5.0], 1.0)
        assert c[0] == 0.5 and abs(c[1] - 1e8) <= 1e-8 * 1e8 and c[2] == 0.0
        with pytest.raises(errors.InputError):
            detci.precondition(b, [1.0, 1.0], [1.0], 0.0)


@pytest.mark.parametrize("ortho", ["mgs", "cgs2"])
def test_orthogonalization_variants_match_reference_trace(ortho, monkeypatch):
    """Both orthogonalizations (DETCI_DAVIDSON_ORTHO=mgs: the reference's
    sequential 2-pass MGS; default: classical Gram-Schmidt twice) reproduce
    the reference chain8 trace iteration by iteration and the C1 energy."""
    if ortho == "mgs":
        monkeypatch.setenv("DETCI_DAVIDSON_ORTHO", "mgs")
    ints, d = load_fixture("chain8")
    ref = d["trace"]
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        res = detci.davidson_solve(b)
    assert len(res.iterations) == len(ref)
    for it, r in zip(res.iterations, ref):
        assert abs(it.ritz_value - r[0]) <= 1e-9 * abs(r[0])
        assert it.max_gram_deviation <= 1e-12
    assert abs(res.energy - ref[-1][0]) <= 1e-10 * abs(ref[-1][0])
    meta = golden_meta()["C1"]
    ints, a, bb = synth.synthetic_system("C1")
    with gpu_basis(ints, a, bb) as b:
        res = detci.davidson_solve(b, want_vector=False)
    assert res.converged and abs(res.energy - meta["energy"]) <= 1e-8
