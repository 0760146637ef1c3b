"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/detci_gpu.h declares, maps errors to status codes, and its
host-executable pieces (factorized matrix elements, partition planner) agree
with the reference."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2601_16169_b200 import _lib, detci, errors, synth
from util import GOLDEN, golden_meta, load_fixture

HEADER = Path(__file__).resolve().parents[1] / "include" / "detci_gpu.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(detci_gpu_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from the ctypes mirror"
    assert set(_lib.SIGNATURES) == set(names)


def test_abi_version():
    assert _lib.load().detci_gpu_abi_version() == 3


def test_library_is_sm100a_cubin():
    data = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in data


def test_create_without_gpu_fails_loudly():
    lib = _lib.load()
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    desc = _lib.Desc()
    desc.world_size = 1
    h = C.c_void_p()
    code = lib.detci_gpu_create(C.byref(desc), C.byref(h))
    assert code == 7 and not h.value      # DETCI_GPU_E_CUDA -> no silent CPU path
    assert lib.detci_gpu_last_error(None)
    with pytest.raises(errors.CudaError):
        detci.GpuBasis(2, [1], [1], 0.0, np.zeros(4), np.zeros(16))


def test_status_codes_map_to_reference_hierarchy():
    for code, cls in ((1, errors.Error), (2, errors.InputError), (3, errors.FormatError), (4, errors.ConfigError),
                      (5, errors.CapacityError), (6, errors.UnsupportedError), (7, errors.CudaError)):
        with pytest.raises(cls):
            errors.raise_for(code, "x")
        assert issubclass(cls, errors.Error)


def test_factorized_elements_match_reference_hij_n36():
    """Every closed form the kernels use (same-spin single/double with the
    spectator sign, mixed with the +-W sign split, regrouped diagonal) against
    the reference hij at 36 orbitals on 4-word determinants."""
    g = np.load(GOLDEN / "elements_n36.npz")
    ints = synth.synthetic_integrals(36, 30)
    worst = {}
    for kind, row, want in zip(g["kinds"], g["dets"], g["values"]):
        got = detci.factorized_element(ints, *map(int, row))
        err = abs(got - want) / max(1.0, abs(want))
        worst[str(kind)] = max(worst.get(str(kind), 0.0), err)
        if kind == "triple":
            assert got == 0.0 and want == 0.0
    assert set(worst) == {"alpha_single", "beta_single", "alpha_double", "beta_double", "mixed", "diagonal", "triple"}
    assert max(worst.values()) <= 1e-12, worst


def test_factorized_phase_probe():
    meta = golden_meta()["elements"]["phase_probe"]
    probe = synth.Integrals(3, 2, 0, 0.0, np.zeros((3, 3)), np.zeros((3, 3, 3, 3)))
    probe.h1[0, 1] = probe.h1[1, 0] = 0.25
    assert detci.factorized_element(probe, 0b001, 0b001, 0b010, 0b001) == meta["a01_beta0"]
    assert detci.factorized_element(probe, 0b001, 0b100, 0b010, 0b100) == meta["a01_beta2"]
    assert detci.factorized_element(probe, 0b010, 0b001, 0b010, 0b010) == meta["b01_alpha1"]
    assert detci.factorized_element(probe, 0b001, 0b001, 0b001, 0b010) == meta["b01_alpha0"]


@pytest.mark.parametrize("name", ["h4_chain", "h3_doublet"])
def test_factorized_dense_hamiltonian(name):
    """Whole dense H from the factorized forms equals the reference dense H."""
    ints, d = load_fixture(name)
    a, b = d["alpha"], d["beta"]
    nb = len(b)
    dense = d["dense"]
    for I in range(dense.shape[0]):
        for J in range(dense.shape[1]):
            ia, ib, ja, jb = I // nb, I % nb, J // nb, J % nb
            want = dense[I, J]
            if bin(int(a[ia]) ^ int(a[ja])).count("1") + bin(int(b[ib]) ^ int(b[jb])).count("1") > 4:
                assert want == 0.0
                continue
            got = detci.factorized_element(ints, int(a[ia]), int(b[ib]), int(a[ja]), int(b[jb]))
            assert abs(got - want) <= 1e-12, (I, J, got, want)


def test_spin_nonconserving_pair_is_rejected():
    ints = synth.synthetic_integrals(4, 2)
    with pytest.raises(errors.InputError):
        detci.factorized_element(ints, 0b01, 0b01, 0b11, 0b00)


def test_plan_partition_reference_formula():
    """matvec.cpp:108-111 blocks n*i/P, and plan_decomposition's range check."""
    n = 37
    lens = np.ones(n, dtype=np.uint32)
    for P in (1, 2, 3, 8, 37):
        blk = detci.plan_partition(n, n, lens, lens, lens, lens, P, False)
        assert list(blk) == [n * g // P for g in range(P + 1)]
    with pytest.raises(errors.InputError):
        detci.plan_partition(n, n, lens, lens, lens, lens, 38, False)


def test_plan_partition_weighted_balances_work():
    ints, a, b = synth.synthetic_system("C1")
    from oracle.bindings import Oracle

    orc = Oracle()
    la = [orc.generate_table(a, ints.norbs, k)[2] for k in (0, 1)]
    lb = [orc.generate_table(b, ints.norbs, k)[2] for k in (0, 1)]
    nb = len(b)
    work = (la[0] + la[1]).astype(np.float64) * nb + float((lb[0] + lb[1]).sum()) + la[0] * float(lb[0].sum())
    for P in (2, 4, 8):
        even = detci.plan_partition(len(a), nb, la[0], la[1], lb[0], lb[1], P, False)
        wtd = detci.plan_partition(len(a), nb, la[0], la[1], lb[0], lb[1], P, True)
        assert wtd[0] == 0 and wtd[-1] == len(a) and np.all(np.diff(wtd.astype(np.int64)) > 0)

        def imbalance(blk):
            per = [work[int(blk[g]):int(blk[g + 1])].sum() for g in range(P)]
            return max(per) / (sum(per) / P)

        assert imbalance(wtd) <= imbalance(even) + 1e-12
        assert imbalance(wtd) < 1.01


def test_library_then_torch_share_one_nccl():
    """Loading libdetci_gpu.so before torch must not break torch's CUDA
    libraries: both resolve the same libnccl.so.2 (the library's rpath points
    at the copy torch ships)."""
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2601_16169_b200 import _lib\n"
            "_lib.load()\n"
            "import torch\n"
            "import torch.distributed\n"
            "print('ok', torch.cuda.nccl.version())\n") % str(Path(__file__).resolve().parents[1])
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.startswith("ok"), out.stderr[-2000:]


def test_factorized_elements_match_reference_hij_two_words():
    """The closed forms on two-word strings (norbs = 70) against the
    reference hij on multi-word determinants: singles, doubles, mixed and
    diagonal, with moves that cross orbital 64 and occupied orbitals on both
    sides of it (cross-word sign counts, 128-bit prefix parity of eps)."""
    from oracle.bindings import REF_SO, RefLib

    if not REF_SO.exists():
        pytest.skip("reference library not built")
    n = 70
    ints = synth.synthetic_integrals(n, 16)
    table = RefLib().table_from_integrals(ints)
    rng = np.random.default_rng(7)

    def rand_string(nel):
        return sum(1 << int(i) for i in rng.choice(n, size=nel, replace=False))

    def excite(s, k):
        occ = [i for i in range(n) if (s >> i) & 1]
        vir = [i for i in range(n) if not (s >> i) & 1]
        for p in rng.choice(occ, size=k, replace=False):
            s &= ~(1 << int(p))
        for q in rng.choice(vir, size=k, replace=False):
            s |= 1 << int(q)
        return s

    classes = {(1, 0): "alpha_single", (0, 1): "beta_single", (2, 0): "alpha_double", (0, 2): "beta_double",
               (1, 1): "mixed", (0, 0): "diagonal", (2, 1): "triple"}
    worst = {}
    for _ in range(60):
        ba, bb = rand_string(8), rand_string(8)
        for (ka, kb), name in classes.items():
            ket_a, ket_b = excite(ba, ka), excite(bb, kb)
            want = table.hij_words(ba, bb, ket_a, ket_b)
            got = detci.factorized_element(ints, ba, bb, ket_a, ket_b)
            worst[name] = max(worst.get(name, 0.0), abs(got - want) / max(1.0, abs(want)))
    assert set(worst) == set(classes.values())
    assert max(worst.values()) <= 1e-12, worst
