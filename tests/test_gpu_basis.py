"""Device basis on the B200: helper lists byte-identical to the reference
(FlatExcitationTable flat/offset/len), diagonal within 1e-12, input
validation with the reference's error classes.  Restates
test_connectivity.cpp and the build_basis checks of test_matvec.cpp:33-72."""
import numpy as np
import pytest

from paper_2601_16169_b200 import detci, errors, synth
from util import FIXTURES, GOLDEN, golden_meta, load_fixture, rel_diff, table_digest, tables_of

pytestmark = pytest.mark.gpu


def gpu_basis(ints, a, b, **kw):
    return detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri, detci.BasisOptions(**kw))


@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_helper_lists_byte_exact(name):
    ints, d = load_fixture(name)
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        for (ch, kind), want in tables_of(d).items():
            got = b.table(ch, kind)
            for g, w in zip(got, want):
                assert g.dtype == w.dtype and g.tobytes() == w.tobytes(), (name, ch, kind)


@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_diagonal(name):
    ints, d = load_fixture(name)
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        assert rel_diff(b.diag(), d["diag"]) <= 1e-12


def test_synthetic_s12_tables_and_diag():
    d = np.load(GOLDEN / "synthetic_s12.npz")
    ints = synth.synthetic_integrals(12, 8)
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        for (ch, kind), want in tables_of(d).items():
            assert all(g.tobytes() == w.tobytes() for g, w in zip(b.table(ch, kind), want))
        assert rel_diff(b.diag(), d["diag"]) <= 1e-12


def test_c1_tables_full_and_diag_rows():
    d = np.load(GOLDEN / "tables_C1.npz")
    ints, a, bb = synth.synthetic_system("C1")
    rows = np.load(GOLDEN / "rows_C1.npz")
    with gpu_basis(ints, a, bb) as b:
        for (ch, kind), want in tables_of(d).items():
            assert all(g.tobytes() == w.tobytes() for g, w in zip(b.table(ch, kind), want))
        diag = b.diag().reshape(len(a), -1)
        assert rel_diff(diag[rows["rows"].astype(np.int64)], rows["diag_rows"]) <= 1e-12


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4"])
def test_config_helper_lists_digest(cfg):
    meta = golden_meta()[cfg]
    ints, a, bb = synth.synthetic_system(cfg)
    with gpu_basis(ints, a, bb) as b:
        for ch in (0, 1):
            for kind in (0, 1):
                assert table_digest(*b.table(ch, kind)) == meta["tables_sha256"][f"{ch}{kind}"]
        rows = np.load(GOLDEN / f"rows_{cfg}.npz")
        diag = b.diag().reshape(len(a), -1)
        assert rel_diff(diag[rows["rows"].astype(np.int64)], rows["diag_rows"]) <= 1e-12


def test_connectivity_goldens_on_device():
    """test_connectivity.cpp:48-75,132-139 via the device builder."""
    ints = synth.synthetic_integrals(4, 2)
    three = np.array([0b011, 0b101, 0b110], dtype=np.uint64)
    sub = synth.Integrals(3, 4, 0, 0.0, ints.h1[:3, :3], ints.eri[:3, :3, :3, :3])
    with gpu_basis(sub, three, three) as b:
        f, o, l = b.table(0, 0)
        assert list(l) == [2, 2, 2] and len(f) == 6
        assert "".join(" ".join(map(str, f[o[i]:o[i] + l[i]])) + "\n" for i in range(3)) == "1 2\n0 2\n0 1\n"
        assert list(b.table(0, 1)[2]) == [0, 0, 0]
    mutual = np.array([0b0011, 0b1100], dtype=np.uint64)
    with gpu_basis(ints, mutual, mutual) as b:
        f, o, l = b.table(1, 1)
        assert list(l) == [1, 1] and list(f) == [1, 0]
        assert list(b.table(1, 0)[2]) == [0, 0]
    single = np.array([0b0011], dtype=np.uint64)
    with gpu_basis(ints, single, single) as b:
        f, o, l = b.table(0, 0)
        assert list(l) == [0] and len(f) == 0


def test_pairwise_degree_property_random_subsets():
    from oracle.bindings import Oracle

    orc = Oracle()
    ints = synth.synthetic_integrals(8, 6)
    allc = synth.full_channel_strings(8, 3)
    rng = synth.SplitMix64(41)
    for _ in range(6):
        sub = np.array([s for s in allc if rng.next() % 3 != 0], dtype=np.uint64)
        with gpu_basis(ints, sub, sub[::-1].copy()) as b:
            for ch, strs in ((0, sub), (1, sub[::-1].copy())):
                for kind in (0, 1):
                    want = orc.generate_table(strs, 8, kind)
                    assert all(g.tobytes() == w.tobytes() for g, w in zip(b.table(ch, kind), want))


def test_duplicate_strings_are_input_errors():
    ints = synth.synthetic_integrals(4, 2)
    dup = np.array([0b0011, 0b0101, 0b0011], dtype=np.uint64)
    with pytest.raises(errors.InputError, match="duplicate"):
        gpu_basis(ints, dup, np.array([1], dtype=np.uint64))


def test_build_validation_errors():
    ints = synth.synthetic_integrals(4, 2)
    with pytest.raises(errors.InputError):            # inconsistent electron count
        gpu_basis(ints, np.array([0b01, 0b11], dtype=np.uint64), np.array([1], dtype=np.uint64))
    with pytest.raises(errors.InputError):            # bit beyond norbs
        gpu_basis(ints, np.array([0b10000], dtype=np.uint64), np.array([1], dtype=np.uint64))
    with pytest.raises(errors.InputError):            # empty list
        gpu_basis(ints, np.array([], dtype=np.uint64), np.array([1], dtype=np.uint64))
    with pytest.raises(errors.InputError):            # > 256 spin-orbitals (basis.cpp:83-87)
        detci.GpuBasis(129, [1], [1], 0.0, np.zeros(129 * 129), np.zeros(1))
    with pytest.raises(errors.CapacityError):         # memory budget (basis.cpp:113-118)
        gpu_basis(ints, np.array([0b0011, 0b0101], dtype=np.uint64), np.array([0b0011], dtype=np.uint64),
                  memory_budget_bytes=64)


def test_nnz_counts_match_lists():
    ints, d = load_fixture("h6_ring")
    t = tables_of(d)
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        nz = b.nnz()
        na, nb = len(d["alpha"]), len(d["beta"])
        sa, da, sb, db = (t[k][2].astype(np.int64).sum() for k in ((0, 0), (0, 1), (1, 0), (1, 1)))
        assert nz["alpha"] == (sa + da) * nb and nz["beta"] == (sb + db) * na and nz["mixed"] == sa * sb
