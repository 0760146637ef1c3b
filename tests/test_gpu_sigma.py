"""sigma = H C on the B200 against the reference (test_matvec.cpp:109-189,
acceptance.cpp:330-368) and the row-sampled reference at the BASELINE
configs.  Tolerance: rel_diff = |a-b| / max(1,|a|,|b|) <= 1e-12."""
import numpy as np
import pytest

from paper_2601_16169_b200 import detci, errors, synth
from util import FIXTURES, GOLDEN, load_fixture, rel_diff

pytestmark = pytest.mark.gpu


def gpu_basis(ints, a, b, **kw):
    return detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri, detci.BasisOptions(**kw))


@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_sigma(name):
    ints, d = load_fixture(name)
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        assert rel_diff(detci.matvec(b, d["x11"]), d["sigma11"]) <= 1e-12


def test_unit_vectors_reproduce_dense_columns():
    ints, d = load_fixture("h4_chain")
    dense = d["dense"]
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        dim = b.dimension()
        for j in range(dim):
            e = np.zeros(dim)
            e[j] = 1.0
            assert np.max(np.abs(detci.matvec(b, e) - dense[:, j])) <= 1e-12


def test_diagonal_only_system_multiplies_by_diag_exactly():
    """test_matvec.cpp:123-135: y == diag * x bitwise."""
    h1 = np.zeros((3, 3))
    eri = np.zeros((3, 3, 3, 3))
    for p in range(3):
        h1[p, p] = -1.0 + 0.3 * p
        eri[p, p, p, p] = 0.5
    ints = synth.Integrals(3, 2, 0, 0.0, h1, eri)
    s = synth.full_channel_strings(3, 1)
    with gpu_basis(ints, s, s) as b:
        x = synth.random_vector(b.dimension(), 5)
        y = detci.matvec(b, x)
        assert np.array_equal(y, b.diag() * x)


def test_linearity():
    ints, d = load_fixture("h4_chain")
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        x = synth.random_vector(b.dimension(), 7)
        z = synth.random_vector(b.dimension(), 9)
        assert rel_diff(detci.matvec(b, x + z), detci.matvec(b, x) + detci.matvec(b, z)) <= 1e-12


def test_symmetry():
    ints, d = load_fixture("chain8")
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        for rep in range(10):
            x = synth.random_vector(b.dimension(), 100 + rep)
            y = synth.random_vector(b.dimension(), 200 + rep)
            assert rel_diff(x @ detci.matvec(b, y), detci.matvec(b, x) @ y) <= 1e-10


def test_deterministic_bitwise():
    ints, d = load_fixture("h6_ring")
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        x = d["x11"]
        assert np.array_equal(detci.matvec(b, x), detci.matvec(b, x))


def test_dimension_mismatch_is_input_error():
    ints, d = load_fixture("h2_minimal")
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        with pytest.raises(errors.InputError):
            detci.matvec(b, np.zeros(b.dimension() - 1))


@pytest.mark.parametrize("blocks,weighted", [(2, False), (3, True), (7, False), (7, True)])
def test_virtual_alpha_blocks_ring_equals_single(blocks, weighted):
    """The multi-GPU schedule (alpha blocks + C ring) emulated on one GPU."""
    ints = synth.synthetic_integrals(12, 8)
    s = synth.synthetic_strings(12, 4, 200)
    x = synth.random_vector(len(s) ** 2, 3)
    with gpu_basis(ints, s, s) as b1:
        y1 = detci.matvec(b1, x)
    with gpu_basis(ints, s, s, virtual_blocks=blocks, weighted_partition=weighted) as bp:
        yp = detci.matvec(bp, x)
    assert rel_diff(yp, y1) <= 1e-12


def test_synthetic_s12_sigma():
    d = np.load(GOLDEN / "synthetic_s12.npz")
    ints = synth.synthetic_integrals(12, 8)
    with gpu_basis(ints, d["alpha"], d["beta"]) as b:
        x = synth.random_vector(b.dimension(), 11)
        assert rel_diff(detci.matvec(b, x), d["sigma11"]) <= 1e-12


def test_asymmetric_alpha_beta_lists():
    """Different alpha and beta string lists (n_alpha != n_beta, shuffled order)."""
    from oracle.bindings import Oracle

    ints = synth.synthetic_integrals(10, 7)
    a = synth.synthetic_strings(10, 4, 90)
    bb = synth.synthetic_strings(10, 3, 70)[::-1].copy()
    o = Oracle().system(ints, a, bb, threads=4)
    with gpu_basis(ints, a, bb) as b:
        for ch in (0, 1):
            for kind in (0, 1):
                assert all(g.tobytes() == w.tobytes() for g, w in zip(b.table(ch, kind), o.tables[(ch, kind)]))
        x = synth.random_vector(b.dimension(), 4)
        assert rel_diff(detci.matvec(b, x), o.matvec(x)) <= 1e-12
        assert rel_diff(b.diag(), o.diag) <= 1e-12


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_config_sigma_rows_vs_reference(cfg):
    """Row-sampled reference sigma (exact reference rows) at the
    BASELINE configs, plus size-independent properties of the full vector."""
    rows = np.load(GOLDEN / f"rows_{cfg}.npz")
    ints, a, bb = synth.synthetic_system(cfg)
    with gpu_basis(ints, a, bb) as b:
        x = synth.random_vector(b.dimension(), 11)
        y = detci.matvec(b, x)
        r = rows["rows"].astype(np.int64)
        assert rel_diff(y.reshape(len(a), -1)[r], rows["sigma_rows"]) <= 1e-12
        # linearity and symmetry at full size
        z = synth.random_vector(b.dimension(), 12)
        hz = detci.matvec(b, z)
        assert rel_diff(detci.matvec(b, x + z), y + hz) <= 1e-12
        assert abs(x @ hz - y @ z) <= 1e-10 * max(1.0, abs(x @ hz))


@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_interior_sigma_rows_vs_reference(cfg):
    """Interior reference rows (tests/golden/make_golden.py --only interior):
    seeded random alpha rows plus the rows of largest / smallest singles and
    doubles degree and the middle rows.  At C3 every row's singles list
    straddles the one-GPU plan's ja windows of D; at C4 every row goes
    through the segmented Cs staging.  Also the plan shape is recorded so a
    change of plan is visible in the failure message."""
    path = GOLDEN / f"rows_{cfg}_interior.npz"
    if not path.exists():
        pytest.skip(f"{path.name} not generated")
    rows = np.load(path)
    ints, a, bb = synth.synthetic_system(cfg)
    with gpu_basis(ints, a, bb) as b:
        x = synth.random_vector(b.dimension(), 11)
        y = detci.matvec(b, x)
        plan = b.sigma_plan()
        r = rows["rows"].astype(np.int64)
        err = rel_diff(y.reshape(len(a), -1)[r], rows["sigma_rows"])
        assert err <= 1e-12, (err, plan)
        assert rel_diff(b.diag().reshape(len(a), -1)[r], rows["diag_rows"]) <= 1e-12


def test_c4_sigma_rows_vs_reference():
    """C4 (1e9 determinants, the 8-GPU target problem, on one GPU): the first
    and last reference sigma rows (tests/golden/make_golden.py --only c4) and
    symmetry of the full sigma (x.Hz = z.Hx)."""
    path = GOLDEN / "rows_C4.npz"
    if not path.exists():
        pytest.skip("rows_C4.npz not generated")
    rows = np.load(path)
    ints, a, bb = synth.synthetic_system("C4")
    with gpu_basis(ints, a, bb) as b:
        x = synth.random_vector(b.dimension(), 11)
        y = detci.matvec(b, x)
        r = rows["rows"].astype(np.int64)
        assert rel_diff(y.reshape(len(a), -1)[r], rows["sigma_rows"]) <= 1e-12
        assert rel_diff(b.diag().reshape(len(a), -1)[r], rows["diag_rows"]) <= 1e-12
        z = synth.random_vector(b.dimension(), 12)
        xhz = x @ detci.matvec(b, z)
        assert abs(xhz - y @ z) <= 1e-10 * max(1.0, abs(xhz))


@pytest.mark.parametrize("m,blocks", [(4, 1), (3, 1), (2, 1), (4, 3), (5, 2)])
def test_blocked_sigma_equals_per_vector(m, blocks):
    """detci_gpu_sigma_block (M = 4/2/1 kernels, virtual blocks too) against
    one sigma per vector."""
    ints = synth.synthetic_integrals(12, 8)
    s = synth.synthetic_strings(12, 4, 200)
    with gpu_basis(ints, s, s, virtual_blocks=blocks, weighted_partition=True) as b:
        X = np.stack([synth.random_vector(b.dimension(), 30 + i) for i in range(m)])
        Y = detci.matvec_block(b, X)
        for i in range(m):
            assert rel_diff(Y[i], detci.matvec(b, X[i])) <= 1e-12


def test_blocked_sigma_c1_rows():
    rows = np.load(GOLDEN / "rows_C1.npz")
    ints, a, bb = synth.synthetic_system("C1")
    with gpu_basis(ints, a, bb) as b:
        x = synth.random_vector(b.dimension(), 11)
        X = np.stack([x, 2.0 * x, -x, 0.5 * x])
        Y = detci.matvec_block(b, X)
        r = rows["rows"].astype(np.int64)
        for i, scale in enumerate((1.0, 2.0, -1.0, 0.5)):
            assert rel_diff(Y[i].reshape(len(a), -1)[r], scale * rows["sigma_rows"]) <= 1e-12


@pytest.mark.parametrize("max_seg", [300, 128])
def test_segmented_mixed_rows_c1(max_seg, monkeypatch):
    """Multi-segment C rows (per-segment slot order + shared accumulator, as at
    C4), forced on C1 with DETCI_MIXED_MAX_SEG, against the reference rows;
    single and paired (blocked) vectors."""
    monkeypatch.setenv("DETCI_MIXED_MAX_SEG", str(max_seg))
    rows = np.load(GOLDEN / "rows_C1.npz")
    ints, a, bb = synth.synthetic_system("C1")
    with gpu_basis(ints, a, bb) as b:
        x = synth.random_vector(b.dimension(), 11)
        y = detci.matvec(b, x)
        r = rows["rows"].astype(np.int64)
        assert rel_diff(y.reshape(len(a), -1)[r], rows["sigma_rows"]) <= 1e-12
        Y = detci.matvec_block(b, np.stack([x, -2.0 * x, x]))
        for i, scale in enumerate((1.0, -2.0, 1.0)):
            assert rel_diff(Y[i], scale * y) <= 1e-12


def test_segmented_virtual_blocks(monkeypatch):
    monkeypatch.setenv("DETCI_MIXED_MAX_SEG", "64")
    ints = synth.synthetic_integrals(12, 8)
    s = synth.synthetic_strings(12, 4, 200)
    x = synth.random_vector(len(s) ** 2, 3)
    d = np.load(GOLDEN / "synthetic_s12.npz")
    with gpu_basis(ints, s, s, virtual_blocks=3, weighted_partition=True) as b:
        assert rel_diff(detci.matvec(b, synth.random_vector(len(s) ** 2, 11)), d["sigma11"]) <= 1e-12


@pytest.mark.parametrize("kernel", ["row", "grouped", "grouped-vec2", "grouped16"])
def test_samespin_kernel_variants(kernel, monkeypatch):
    """Both same-spin kernels (DETCI_SAMESPIN=row: one row per CTA; default:
    8 rows per CTA) against the reference fixtures, the C1 reference rows and
    virtual blocks."""
    monkeypatch.setenv("DETCI_SAMESPIN", "row" if kernel == "row" else "grouped")
    if kernel == "grouped-vec2":   # 16-byte loads
        monkeypatch.setenv("DETCI_SAMESPIN_VEC", "1")
    if kernel == "grouped16":
        monkeypatch.setenv("DETCI_SAMESPIN_ROWS", "16")
    for name in ("h6_ring", "chain8"):
        ints, d = load_fixture(name)
        with gpu_basis(ints, d["alpha"], d["beta"]) as b:
            assert rel_diff(detci.matvec(b, d["x11"]), d["sigma11"]) <= 1e-12
    rows = np.load(GOLDEN / "rows_C1.npz")
    ints, a, bb = synth.synthetic_system("C1")
    r = rows["rows"].astype(np.int64)
    for blocks in (1, 3):
        with gpu_basis(ints, a, bb, virtual_blocks=blocks) as b:
            x = synth.random_vector(b.dimension(), 11)
            assert rel_diff(detci.matvec(b, x).reshape(len(a), -1)[r], rows["sigma_rows"]) <= 1e-12


@pytest.mark.parametrize("mixed,dbytes", [("gather", None), ("scatter", None), ("scatter", "3000000"),
                                          ("scatter", "1")])
def test_mixed_kernel_variants(mixed, dbytes, monkeypatch):
    """Mixed term through the gather kernel (DETCI_MIXED=gather) and the
    default scatter kernel + deterministic D reduction, with the D buffer
    forced into several output windows (DETCI_MIXED_DBYTES; "1" = one alpha
    row per window), against the reference rows at C1, the fixtures and
    virtual blocks; bitwise run-to-run determinism."""
    monkeypatch.setenv("DETCI_MIXED", mixed)
    if dbytes:
        monkeypatch.setenv("DETCI_MIXED_DBYTES", dbytes)
    for name in ("h4_chain", "chain8"):
        ints, d = load_fixture(name)
        with gpu_basis(ints, d["alpha"], d["beta"]) as b:
            assert rel_diff(detci.matvec(b, d["x11"]), d["sigma11"]) <= 1e-12
    rows = np.load(GOLDEN / "rows_C1.npz")
    ints, a, bb = synth.synthetic_system("C1")
    r = rows["rows"].astype(np.int64)
    for blocks in ((1, 3) if dbytes != "1" else (2,)):
        with gpu_basis(ints, a, bb, virtual_blocks=blocks, weighted_partition=True) as b:
            x = synth.random_vector(b.dimension(), 11)
            y = detci.matvec(b, x)
            assert rel_diff(y.reshape(len(a), -1)[r], rows["sigma_rows"]) <= 1e-12
            assert np.array_equal(y, detci.matvec(b, x))


@pytest.mark.parametrize("norbs,nel,count", [(40, 3, 160), (52, 2, 120), (64, 2, 150)])
def test_large_norbs_scatter_classes(norbs, nel, count):
    """Wide orbital spaces shrink the scatter kernel's K (a V row is 8 n^2
    bytes: 32 KB at n = 64) and the gather kernel's W; sigma against the C
    oracle, single vectors and pairs."""
    from oracle.bindings import Oracle

    ints = synth.synthetic_integrals(norbs, 2 * nel)
    s = synth.synthetic_strings(norbs, nel, count)
    o = Oracle().system(ints, s, s, threads=8)
    x = synth.random_vector(len(s) ** 2, 5)
    ref = o.matvec(x)
    with gpu_basis(ints, s, s) as b:
        assert rel_diff(detci.matvec(b, x), ref) <= 1e-12
        Y = detci.matvec_block(b, np.stack([x, -x]))
        assert rel_diff(Y[0], ref) <= 1e-12 and rel_diff(Y[1], -ref) <= 1e-12


@pytest.mark.parametrize("cfg,dbytes", [("C1", None), ("C1", "20000000"), ("C2", None)])
def test_pipelined_host_sigma_equals_plain(cfg, dbytes, monkeypatch):
    """The host-pointer sigma with chunked, overlapped copies (default when
    no timings are requested) against the plain copy-sigma-copy schedule
    (DETCI_SIGMA_PIPELINE=0) and the reference rows; with several scatter
    windows too (DETCI_MIXED_DBYTES)."""
    if dbytes:
        monkeypatch.setenv("DETCI_MIXED_DBYTES", dbytes)
    rows = np.load(GOLDEN / f"rows_{cfg}.npz")
    ints, a, bb = synth.synthetic_system(cfg)
    with gpu_basis(ints, a, bb) as b:
        x = synth.random_vector(b.dimension(), 11)
        y = detci.matvec(b, x)
        tm = {}
        y_plain = detci.matvec(b, x, timings=tm)
        assert rel_diff(y, y_plain) <= 1e-14
        r = rows["rows"].astype(np.int64)
        assert rel_diff(y.reshape(len(a), -1)[r], rows["sigma_rows"]) <= 1e-12
        assert np.array_equal(y, detci.matvec(b, x))   # deterministic
        monkeypatch.setenv("DETCI_SIGMA_PIPELINE", "0")
        assert rel_diff(detci.matvec(b, x), y_plain) <= 1e-15


@pytest.mark.parametrize("multi", ["gather", "ring"])
@pytest.mark.parametrize("blocks", [2, 3, 8])
def test_multi_block_schedules(multi, blocks, monkeypatch):
    """Both multi-GPU schedules on virtual alpha blocks: the gather schedule
    (default: Cs allgather, alpha term in one launch, mixed term split by
    beta-slot columns and exchanged all-to-all) and the Cs ring
    (DETCI_MULTI=ring), single vectors and pairs, against the reference rows
    at C1 and the single-block sigma."""
    if multi == "ring":
        monkeypatch.setenv("DETCI_MULTI", "ring")
    rows = np.load(GOLDEN / "rows_C1.npz")
    ints, a, bb = synth.synthetic_system("C1")
    r = rows["rows"].astype(np.int64)
    x = synth.random_vector(len(a) * len(bb), 11)
    with gpu_basis(ints, a, bb) as b1:
        y1 = detci.matvec(b1, x)
    with gpu_basis(ints, a, bb, virtual_blocks=blocks, weighted_partition=True) as b:
        y = detci.matvec(b, x)
        assert rel_diff(y.reshape(len(a), -1)[r], rows["sigma_rows"]) <= 1e-12
        assert rel_diff(y, y1) <= 1e-12
        Y = detci.matvec_block(b, np.stack([x, -0.5 * x, 2.0 * x]))
        for i, sc in enumerate((1.0, -0.5, 2.0)):
            assert rel_diff(Y[i], sc * y1) <= 1e-12


def test_pipelined_host_sigma_pinned_buffers():
    """The overlapped host sigma with page-locked buffers (truly asynchronous
    chunk copies, as in bench.py's end-to-end leg) equals the device sigma
    bitwise and the reference rows, over repeated calls."""
    import ctypes as C
    import torch

    from paper_2601_16169_b200 import _lib

    rows = np.load(GOLDEN / "rows_C2.npz")
    ints, a, bb = synth.synthetic_system("C2")
    lib = _lib.load()
    with gpu_basis(ints, a, bb) as b:
        x = torch.from_numpy(synth.random_vector(b.dimension(), 11)).pin_memory()
        y = torch.empty_like(x).pin_memory()
        dx, dy = x.cuda(), torch.empty_like(x).cuda()
        assert lib.detci_gpu_sigma_device(b.handle, dx.data_ptr(), dy.data_ptr(), None) == 0
        ref = dy.cpu().numpy()
        for _ in range(3):
            y.zero_()
            assert lib.detci_gpu_sigma(b.handle, x.data_ptr(), y.data_ptr(), None) == 0
            assert rel_diff(y.numpy(), ref) <= 1e-14
        r = rows["rows"].astype(np.int64)
        assert rel_diff(y.numpy().reshape(len(a), -1)[r], rows["sigma_rows"]) <= 1e-12
