"""Shared test helpers (mirrors proj/tests/unit/test_helpers.hpp)."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from paper_2601_16169_b200 import synth

GOLDEN = Path(__file__).resolve().parent / "golden"
FIXTURES = ["h2_minimal", "h3_doublet", "h4_chain", "h6_ring", "chain8"]


def rel_diff(a, b):
    """test_matvec.cpp:20-22: |a-b| / max(1, |a|, |b|), elementwise max."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))))


def load_fixture(name):
    d = np.load(GOLDEN / f"fixture_{name}.npz")
    ints = synth.Integrals(int(d["norbs"]), int(d["nelec"]), int(d["ms2"]), float(d["core"]), d["h1"], d["eri"])
    return ints, d


def golden_meta():
    return json.loads((GOLDEN / "golden.json").read_text())


def tables_of(d, prefix=""):
    out = {}
    for ch, cn in ((0, "a"), (1, "b")):
        for kind, kn in ((0, "s"), (1, "d")):
            out[(ch, kind)] = (d[f"{prefix}{kn}{cn}_flat"], d[f"{prefix}{kn}{cn}_offset"], d[f"{prefix}{kn}{cn}_len"])
    return out


def table_digest(flat, off, ln):
    import hashlib

    h = hashlib.sha256()
    for a in (flat, off, ln):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
