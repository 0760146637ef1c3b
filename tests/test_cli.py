"""detci_gpu CLI (integration/detci_gpu_cli.cpp): the
reference `detci run` report with --method gpu | stored | matrix_free.
The text report's GROUND_ENERGY line and the JSON schema are the
reference's own emit_report (run.cpp:127-242)."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2601_16169_b200 import synth
from util import load_fixture

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "oracle" / "_ref" / "detci_gpu"
FIX = ROOT / "tests" / "golden" / "fixtures"


def inputs(tmp_path, name="chain8"):
    ints, d = load_fixture(name)
    dets = tmp_path / f"{name}.dets"
    dets.write_text(synth.write_det_list(ints.norbs, d["alpha"], d["beta"]))
    return FIX / f"{name}.fcidump", dets


def run(*args):
    if not CLI.exists():
        pytest.skip("detci_gpu not built (needs the reference sources at build time)")
    return subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=600)


def ground(out):
    return [l for l in out.splitlines() if l.startswith("GROUND_ENERGY")][-1].split()[1]


def test_matrix_free_is_the_reference_pipeline(tmp_path):
    f, d = inputs(tmp_path)
    out = run("run", "--integrals", f, "--dets", d, "--method", "matrix_free", "--workers", "4")
    assert out.returncode == 0, out.stderr
    assert ground(out.stdout) == "-2.420193979007e+00"   # proj/test_output.txt:33


def test_usage_and_option_errors(tmp_path):
    f, d = inputs(tmp_path)
    assert run().returncode == 1
    bad = run("run", "--integrals", f, "--dets", d, "--method", "bogus")
    assert bad.returncode == 1 and "--method" in bad.stderr
    missing = run("run", "--integrals", tmp_path / "nope.fcidump", "--dets", d, "--method", "matrix_free")
    assert missing.returncode == 1 and "cannot open integrals" in missing.stderr
    st = run("run", "--integrals", f, "--dets", d, "--method", "stored", "--devices", "2")
    assert st.returncode == 1 and "one GPU" in st.stderr


@pytest.mark.gpu
def test_gpu_method_text_report(tmp_path):
    f, d = inputs(tmp_path)
    out = run("run", "--integrals", f, "--dets", d, "--method", "gpu")
    assert out.returncode == 0, out.stderr
    assert ground(out.stdout) == "-2.420193979007e+00"
    assert "method         gpu (devices 1)" in out.stdout
    assert "status         converged" in out.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("method,extra", [("gpu", []), ("stored", []), ("gpu", ["--virtual-blocks", "3"]),
                                          ("gpu", ["--shuffle", "--seed", "7"])])
def test_json_report(tmp_path, method, extra):
    f, d = inputs(tmp_path, "h6_ring")
    ref = run("run", "--integrals", f, "--dets", d, "--method", "matrix_free", "--format", "json", *extra)
    out = run("run", "--integrals", f, "--dets", d, "--method", method, "--format", "json", *extra)
    assert out.returncode == 0 and ref.returncode == 0, out.stderr + ref.stderr
    doc, rdoc = json.loads(out.stdout), json.loads(ref.stdout)
    assert set(rdoc) <= set(doc) and "gpu" in doc
    e, er = doc["result"]["ground_energy"], rdoc["result"]["ground_energy"]
    assert doc["result"]["converged"] and abs(e - er) <= 1e-10 * abs(er)
    assert doc["system"] == rdoc["system"]
    assert doc["config"]["method"] == ("stored_gpu" if method == "stored" else "gpu")
    if method == "stored":
        assert doc["gpu"]["stored_nnz"] > 0
    assert abs(doc["result"]["iterations"] - rdoc["result"]["iterations"]) <= 1


def test_not_converged_exit_code(tmp_path):
    """tools/detci.cpp:32-34, 59-63: a reported but non-converged run exits 2."""
    f, d = inputs(tmp_path)
    out = run("run", "--integrals", f, "--dets", d, "--method", "matrix_free", "--max-iter", "2", "--workers", "2")
    assert out.returncode == 2, out.stderr
    assert "GROUND_ENERGY" in out.stdout
    bad = run("run", "--integrals", f, "--dets", d, "--transport", "carrier-pigeon")
    assert bad.returncode == 1 and "--transport" in bad.stderr


@pytest.mark.gpu
def test_gpu_not_converged_exit_code(tmp_path):
    f, d = inputs(tmp_path)
    out = run("run", "--integrals", f, "--dets", d, "--method", "gpu", "--max-iter", "2")
    assert out.returncode == 2, out.stderr
    assert "GROUND_ENERGY" in out.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("devices", [2, 3])
def test_gpu_loopback_devices(tmp_path, devices):
    """--devices N --transport loopback: N ranks (threads) on one GPU through
    the multi-rank code; the reference's golden energy."""
    f, d = inputs(tmp_path)
    out = run("run", "--integrals", f, "--dets", d, "--method", "gpu", "--devices", devices, "--transport", "loopback")
    assert out.returncode == 0, out.stderr
    assert ground(out.stdout) == "-2.420193979007e+00"
