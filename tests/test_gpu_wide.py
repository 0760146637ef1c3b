"""norbs 65..128 on the device (two uint64 words per channel string).

The reference packs strings of up to kMaxKernelBits = 256 spin-orbitals into
multi-word BitStrings (slater_condon.hpp:26, bitstring.hpp:33-51,
basis.cpp:83-87); the device path holds orbitals 64..127 in a second word.
Every check here is against the UNMODIFIED reference (oracle/_ref,
ref_basis_create_words): helper lists byte-identical, diagonal, full sigma,
the Davidson energy.  The strings straddle the word boundary (occupied
orbitals on both sides of 64, moves across it), so the cross-word sign
counts and the 128-bit prefix parity of eps are exercised; norbs = 92 has
4186 orbital pairs, which needs bit 30 of the scatter entry's pair column.
"""
import itertools

import numpy as np
import pytest

from util import rel_diff

pytestmark = pytest.mark.gpu


def wide_strings(norbs, core, window, nel_window, count, seed):
    """`core` orbitals always occupied plus a nel_window-subset of `window`;
    a seeded sample of `count` strings, ascending as 128-bit integers."""
    base = sum(1 << c for c in core)
    allc = [base | sum(1 << w for w in comb) for comb in itertools.combinations(window, nel_window)]
    rng = np.random.default_rng(seed)
    pick = sorted(int(allc[i]) for i in rng.choice(len(allc), size=min(count, len(allc)), replace=False))
    assert all(x < (1 << norbs) for x in pick)
    return pick


def words(strings):
    mask = (1 << 64) - 1
    return np.array([[s & mask, s >> 64] for s in strings], dtype=np.uint64)


def system(norbs, core, window, nel_window, count):
    from oracle.bindings import REF_SO
    from paper_2601_16169_b200 import synth

    if not REF_SO.exists():
        pytest.skip("reference library not built")
    a = wide_strings(norbs, core, window, nel_window, count, 1)
    b = wide_strings(norbs, core, window, nel_window, count, 2)
    nel = 2 * (len(core) + nel_window)
    ints = synth.synthetic_integrals(norbs, nel)
    return ints, a, b


@pytest.fixture(scope="module")
def n70():
    # core orbitals 0, 1, 30 plus 5 electrons in 58..69: every string has
    # bits in both words, moves cross orbital 64
    return system(70, [0, 1, 30], list(range(58, 70)), 5, 300)


def ref_basis(ints, a, b):
    from oracle.bindings import RefLib

    ref = RefLib()
    t = ref.table_from_integrals(ints)
    return t, t.basis_words(words(a), words(b))


def test_wide_tables_diag_sigma_match_reference(n70):
    from paper_2601_16169_b200 import detci, synth

    ints, a, b = n70
    _t, rb = ref_basis(ints, a, b)
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri) as g:
        for ch in (0, 1):
            for kind in (0, 1):
                got, want = g.table(ch, kind), rb.table(ch, kind)
                assert all(np.array_equal(x, y) for x, y in zip(got, want)), (ch, kind)
        assert rel_diff(g.diag(), rb.diag()) <= 1e-12
        x = synth.random_vector(g.dimension(), 5)
        y = detci.matvec(g, x)
        assert rel_diff(y, rb.matvec(x)) <= 1e-12


def test_wide_blocked_pair_and_stored(n70):
    from paper_2601_16169_b200 import detci, synth

    ints, a, b = n70
    _t, rb = ref_basis(ints, a, b)
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri) as g:
        X = np.stack([synth.random_vector(g.dimension(), s) for s in (7, 8)])
        Y = detci.matvec_block(g, X)
        for i in range(2):
            assert rel_diff(Y[i], rb.matvec(X[i])) <= 1e-12
        sm = detci.build_stored_matrix(g, 0)
        try:
            assert rel_diff(detci.stored_matvec(sm, X[0]), rb.matvec(X[0])) <= 1e-12
        finally:
            sm.release()


def test_wide_davidson_energy_matches_reference(n70):
    from paper_2601_16169_b200 import detci

    ints, a, b = n70
    _t, rb = ref_basis(ints, a, b)
    want = rb.davidson()
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri) as g:
        res = detci.davidson_solve(g, want_vector=False)
    assert want["status"] == 0 and res.converged
    assert abs(res.energy - want["energy"]) <= 1e-8
    assert len(res.iterations) == want["iterations"]


def test_wide_virtual_blocks(n70):
    from paper_2601_16169_b200 import detci, synth

    ints, a, b = n70
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri) as g:
        x = synth.random_vector(g.dimension(), 9)
        y1 = detci.matvec(g, x)
    opts = detci.BasisOptions(virtual_blocks=3)
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri, opts) as g3:
        assert rel_diff(detci.matvec(g3, x), y1) <= 1e-12


def test_wide_13bit_pair_column():
    """norbs = 92: 4186 orbital pairs (> 4095), small scatter K (V rows of
    33 KB), strings spanning both words."""
    from paper_2601_16169_b200 import detci, synth

    ints, a, b = system(92, [3, 63], list(range(60, 92, 2)), 3, 200)
    _t, rb = ref_basis(ints, a, b)
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri) as g:
        x = synth.random_vector(g.dimension(), 3)
        assert rel_diff(detci.matvec(g, x), rb.matvec(x)) <= 1e-12


def test_wide_gather_kernel_is_refused(n70, monkeypatch):
    from paper_2601_16169_b200 import detci
    from paper_2601_16169_b200.errors import UnsupportedError

    ints, a, b = n70
    monkeypatch.setenv("DETCI_MIXED", "gather")
    with pytest.raises(UnsupportedError):
        detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri)
