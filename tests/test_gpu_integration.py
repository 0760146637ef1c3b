"""The reference pipeline with the device sigma plugged in through the C++
shim (integration/run_gpu.cpp, built against the unmodified reference):
the reference davidson_solve over the device LinearOperator ("mixed
oracle") and the device Davidson agree with the all-CPU
reference run."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
RUN = ROOT / "oracle" / "_ref" / "run_gpu"


@pytest.mark.parametrize("name", ["h4_chain", "h6_ring", "chain8"])
def test_reference_pipeline_with_device_sigma(name):
    if not RUN.exists():
        pytest.skip("run_gpu not built (needs the reference sources at build time)")
    out = subprocess.run([str(RUN), str(ROOT / "tests" / "golden" / "fixtures" / f"{name}.fcidump")],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    lines = dict((l.split()[1], l.split()[2:]) for l in out.stdout.splitlines() if l.startswith("GROUND_ENERGY"))
    sig = [l for l in out.stdout.splitlines() if l.startswith("SIGMA_MAX_REL_DIFF")][0]
    assert float(sig.split()[1]) <= 1e-12
    e_ref = float(lines["reference"][0])
    gb = [l.split() for l in out.stdout.splitlines() if l.startswith("GPU_BUILD")][0]
    assert gb[2] == "1" and float(gb[4]) <= 1e-12 and gb[6] == "1", gb   # tables, diag, shape
    for k in ("mixed", "device", "gpu_built"):
        assert abs(float(lines[k][0]) - e_ref) <= 1e-10 * abs(e_ref), (k, lines)
    if name == "chain8":
        assert lines["reference"][0] == "-2.420193979007e+00"


def test_reference_solver_over_device_sigma_c1():
    """The unmodified reference davidson_solve driving the device sigma
    (ctypes LinearOperator callback) at the C1 shape, against the device
    Davidson: same energy (1e-8 Ha) and iteration count."""
    from oracle.bindings import REF_SO, RefLib
    from paper_2601_16169_b200 import detci, synth

    if not REF_SO.exists():
        pytest.skip("reference library not built")
    ref = RefLib()
    ints, a, b = synth.synthetic_system("C1")
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri) as basis:
        diag = basis.diag()
        mixed = ref.davidson_operator(lambda x, y: detci.matvec(basis, x, y), diag)
        dev = detci.davidson_solve(basis, want_vector=False)
    assert mixed["status"] == 0 and dev.converged
    assert abs(mixed["energy"] - dev.energy) <= 1e-8
    assert abs(mixed["iterations"] - len(dev.iterations)) <= 2
    for r, it in zip(mixed["trace"][:20], dev.iterations[:20]):
        assert abs(r[0] - it.ritz_value) <= 1e-9 * abs(r[0])
