"""Multi-root block Davidson (BASELINE config C5).
The reference is single-root, so the oracle is numpy eigh of the dense H
built from the pinned C oracle's matrix elements, plus the single-root
reference energy for the lowest root and eigen-residuals through sigma."""
import numpy as np
import pytest

from oracle.bindings import Oracle
from paper_2601_16169_b200 import detci, errors, synth
from util import load_fixture

pytestmark = pytest.mark.gpu


def gpu_basis(ints, a, b, **kw):
    return detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri, detci.BasisOptions(**kw))


def dense_h(ints, a, b):
    s = Oracle().system(ints, a, b, threads=8)
    dim = len(a) * len(b)
    H = np.zeros((dim, dim))
    for j in range(dim):
        e = np.zeros(dim)
        e[j] = 1.0
        H[:, j] = s.matvec(e)
    return H


@pytest.mark.parametrize("name,nroots", [("h4_chain", 4), ("h6_ring", 4), ("chain8", 3)])
def test_fixture_roots_match_dense_eigh(name, nroots):
    ints, d = load_fixture(name)
    want = np.linalg.eigvalsh(dense_h(ints, d["alpha"], d["beta"]))[:nroots]
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        res = detci.davidson_roots(b, nroots)
        assert res.converged, res.iterations[-1]
        assert np.max(np.abs(res.energies - want) / np.abs(want)) <= 1e-10
        assert abs(res.energies[0] - float(d["energy"])) <= 1e-10 * abs(float(d["energy"]))
        V = res.eigenvectors
        assert np.max(np.abs(V @ V.T - np.eye(nroots))) <= 1e-8
        for r in range(nroots):
            assert np.linalg.norm(detci.matvec(b, V[r]) - res.energies[r] * V[r]) <= 1e-6
        assert all(it.max_gram_deviation <= 1e-12 for it in res.iterations)


def test_roots_with_virtual_blocks_and_restarts():
    ints = synth.synthetic_integrals(10, 6)
    s = synth.synthetic_strings(10, 3, 40)
    want = np.linalg.eigvalsh(dense_h(ints, s, s))[:4]
    with gpu_basis(ints, s, s, virtual_blocks=3, weighted_partition=True) as b:
        res = detci.davidson_roots(b, 4, max_subspace=10)
    assert res.converged
    assert any(it.restarted for it in res.iterations)
    assert np.max(np.abs(res.energies - want) / np.abs(want)) <= 1e-10


def test_multiroot_option_validation():
    ints, d = load_fixture("h2_minimal")
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        with pytest.raises(errors.ConfigError):
            detci.davidson_roots(b, 0)
        with pytest.raises(errors.ConfigError):
            detci.davidson_roots(b, 3, max_subspace=4)
        with pytest.raises(errors.InputError):
            detci.davidson_roots(b, 5, max_subspace=12)   # dim 4


def test_fused_block_residual_pass_matches_per_root(monkeypatch):
    """The one-pass multi-root residual (k_ritz_block, default for m <= 4 and
    an even local dimension) against the per-root Ritz passes
    (DETCI_DAVIDSON_BLOCK_RITZ=0) and dense eigh, through restarts."""
    ints = synth.synthetic_integrals(12, 6)
    s = synth.synthetic_strings(12, 3, 60)
    assert (len(s) * len(s)) % 2 == 0
    want = np.linalg.eigvalsh(dense_h(ints, s, s))[:4]
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("DETCI_DAVIDSON_BLOCK_RITZ", mode)
        with gpu_basis(ints, s, s) as b:
            res = detci.davidson_roots(b, 4, max_subspace=12)
            assert res.converged
            assert any(it.restarted for it in res.iterations)
            for r in range(4):
                assert np.linalg.norm(detci.matvec(b, res.eigenvectors[r]) - res.energies[r] * res.eigenvectors[r]) <= 1e-6
        out[mode] = res
    assert np.max(np.abs(out["1"].energies - want) / np.abs(want)) <= 1e-10
    assert np.max(np.abs(out["1"].energies - out["0"].energies) / np.abs(want)) <= 1e-12
