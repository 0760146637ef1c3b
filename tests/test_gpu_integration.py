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
    for k in ("mixed", "device"):
        assert abs(float(lines[k][0]) - e_ref) <= 1e-10 * abs(e_ref), (k, lines)
    if name == "chain8":
        assert lines["reference"][0] == "-2.420193979007e+00"
