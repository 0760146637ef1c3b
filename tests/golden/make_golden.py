"""Generate the committed golden vectors from the UNMODIFIED reference.

Runs in the dev container only (needs oracle/_ref/libdetci_ref.so, built from
/root/reference by `make -C oracle ref`).  Outputs small .npz / .json files
next to this script; tests compare both the C oracle and the GPU path
against them, so the GPU box never needs /root/reference.

    python tests/golden/make_golden.py            # everything but the slow C1 run
    python tests/golden/make_golden.py --c1-davidson   # + full reference Davidson at C1 (~40 min)
"""
from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.bindings import RefLib  # noqa: E402
from paper_2601_16169_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent
FIXTURES = Path("/root/reference/proj/tests/fixtures")
FIXTURE_NAMES = ["h2_minimal", "h3_doublet", "h4_chain", "h6_ring", "chain8"]


def table_digest(flat, off, ln) -> str:
    h = hashlib.sha256()
    for a in (flat, off, ln):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def eri_digest(ints) -> str:
    return hashlib.sha256(np.ascontiguousarray(ints.eri).tobytes() + np.ascontiguousarray(ints.h1).tobytes()).hexdigest()


def save_tables(rb, prefix, out):
    for ch, cn in ((0, "a"), (1, "b")):
        for kind, kn in ((0, "s"), (1, "d")):
            f, o, l = rb.table(ch, kind)
            out[f"{prefix}{kn}{cn}_flat"] = f
            out[f"{prefix}{kn}{cn}_offset"] = o
            out[f"{prefix}{kn}{cn}_len"] = l


def fixtures(ref: RefLib):
    for name in FIXTURE_NAMES:
        t = ref.table_from_fcidump(FIXTURES / f"{name}.fcidump")
        ints = t.integrals()
        na, nb = ref.channel_electron_counts(ints.nelec, ints.ms2)
        a = ref.full_channel_strings(ints.norbs, na)
        b = ref.full_channel_strings(ints.norbs, nb)
        rb = t.basis(a, b)
        out = {
            "norbs": ints.norbs, "nelec": ints.nelec, "ms2": ints.ms2, "core": ints.core,
            "h1": ints.h1, "eri": ints.eri, "alpha": a, "beta": b, "diag": rb.diag(),
        }
        save_tables(rb, "", out)
        x = synth.random_vector(rb.dim(), 11)
        out["x11"] = x
        out["sigma11"] = rb.matvec(x)
        if rb.dim() <= 400:
            dense = rb.dense_hamiltonian()
            out["dense_ground"] = np.linalg.eigvalsh(dense)[0]
            if rb.dim() <= 100:
                out["dense"] = dense
        dv = rb.davidson()
        out["energy"] = dv["energy"]
        out["iterations"] = dv["iterations"]
        out["trace"] = dv["trace"]
        if name == "h6_ring":
            d6 = rb.davidson(max_subspace=6)
            out["energy_ms6"] = d6["energy"]
            out["trace_ms6"] = d6["trace"]
        np.savez_compressed(OUT / f"fixture_{name}.npz", **out)
        print(f"{name}: dim {rb.dim()} E {dv['energy']:.12e} iters {dv['iterations']}", flush=True)


def synthetic(ref: RefLib, c1_davidson: bool):
    meta = {}
    # small synthetic system: full tables, sigma, energy
    ints = synth.synthetic_integrals(12, 8)
    s = synth.synthetic_strings(12, 4, 200)
    t = ref.table_from_integrals(ints)
    rb = t.basis(s, s)
    out = {"norbs": 12, "nelec": 8, "alpha": s, "beta": s, "diag": rb.diag()}
    save_tables(rb, "", out)
    x = synth.random_vector(rb.dim(), 11)
    out["sigma11"] = rb.matvec(x)
    dv = rb.davidson()
    out["energy"] = dv["energy"]
    out["iterations"] = dv["iterations"]
    np.savez_compressed(OUT / "synthetic_s12.npz", **out)
    meta["s12"] = {"eri_sha256": eri_digest(ints), "energy": dv["energy"], "iterations": dv["iterations"]}
    print(f"s12: dim {rb.dim()} E {dv['energy']:.12e}", flush=True)

    # baseline configs: table digests + reference sigma rows
    rows_for = {"C1": [0, 1, 17, 500, 999], "C2": [0, 4321, 9999], "C3": [0, 17319]}
    for cfg in ("C1", "C2", "C3"):
        t0 = time.time()
        ints, a, b = synth.synthetic_system(cfg)
        entry = {"eri_sha256": eri_digest(ints), "n_strings": int(len(a)),
                 "strings_sha256": hashlib.sha256(a.tobytes()).hexdigest()}
        tables = {}
        for ch, strs in ((0, a), (1, b)):
            for kind in (0, 1):
                f, o, l = ref.generate_table(strs, ints.norbs, kind)
                tables[f"{ch}{kind}"] = table_digest(f, o, l)
                entry[f"len_stats_{ch}{kind}"] = [float(l.mean()), int(l.max()), int(l.sum())]
        entry["tables_sha256"] = tables
        rt = ref.table_from_integrals(ints)
        rb = rt.basis(a, b, cache=False)
        rows = np.array(rows_for[cfg], dtype=np.uint64)
        x = synth.random_vector(rb.dim(), 11)
        yr = rb.matvec_rows(rows, x)
        np.savez_compressed(OUT / f"rows_{cfg}.npz", rows=rows, sigma_rows=yr,
                            diag_rows=rb.diag().reshape(len(a), -1)[rows.astype(np.int64)])
        entry["rows"] = rows_for[cfg]
        if cfg == "C1":
            # full C1 tables are small enough to commit
            out = {}
            save_tables(rb, "", out)
            np.savez_compressed(OUT / "tables_C1.npz", **out)
        if cfg == "C1" and c1_davidson:
            t1 = time.time()
            dv = rb.davidson()
            entry["energy"] = dv["energy"]
            entry["iterations"] = dv["iterations"]
            entry["davidson_seconds"] = time.time() - t1
            entry["trace"] = dv["trace"].tolist()
        meta[cfg] = entry
        print(f"{cfg}: {time.time() - t0:.1f}s", flush=True)
    return meta


def c4_rows(ref: RefLib):
    """C4 (1e9 determinants): two reference sigma rows and the table digests
    (the full reference sigma is ~23 h on 8 cores; two rows take minutes)."""
    t0 = time.time()
    ints, a, b = synth.synthetic_system("C4")
    entry = {"eri_sha256": eri_digest(ints), "n_strings": int(len(a)),
             "strings_sha256": hashlib.sha256(a.tobytes()).hexdigest()}
    tables = {}
    for ch, strs in ((0, a), (1, b)):
        for kind in (0, 1):
            f, o, l = ref.generate_table(strs, ints.norbs, kind)
            tables[f"{ch}{kind}"] = table_digest(f, o, l)
            entry[f"len_stats_{ch}{kind}"] = [float(l.mean()), int(l.max()), int(l.sum())]
    entry["tables_sha256"] = tables
    rb = ref.table_from_integrals(ints).basis(a, b, cache=False, budget=48 << 30)
    rows = np.array([0, len(a) - 1], dtype=np.uint64)
    x = synth.random_vector(rb.dim(), 11)
    yr = rb.matvec_rows(rows, x)
    del x
    np.savez_compressed(OUT / "rows_C4.npz", rows=rows, sigma_rows=yr,
                        diag_rows=rb.diag().reshape(len(a), -1)[rows.astype(np.int64)])
    entry["rows"] = rows.tolist()
    print(f"C4: {time.time() - t0:.1f}s", flush=True)
    return entry


def interior_rows(ref: RefLib, cfg: str, nrand: int):
    """Reference sigma rows away from the edges (the edge rows
    alone cannot see a wrong interior row): `nrand` seeded random alpha rows
    plus the rows of largest and smallest alpha singles / doubles degree and
    the middle rows.  At C3 these rows straddle the two ja windows of the
    one-GPU scatter plan; at C4 every row goes through the segmented
    (nseg = 2) Cs staging."""
    t0 = time.time()
    ints, a, b = synth.synthetic_system(cfg)
    rb = ref.table_from_integrals(ints).basis(a, b, cache=False, budget=48 << 30)
    la = [ref.generate_table(a, ints.norbs, kind)[2] for kind in (0, 1)]
    rng = np.random.default_rng(2026)
    picks = set(int(r) for r in rng.choice(np.arange(1, len(a) - 1), size=nrand, replace=False))
    picks |= {int(np.argmax(la[0])), int(np.argmin(la[0])), int(np.argmax(la[1])), int(np.argmin(la[1])),
              len(a) // 2 - 1, len(a) // 2}
    rows = np.array(sorted(picks), dtype=np.uint64)
    x = synth.random_vector(rb.dim(), 11)
    yr = rb.matvec_rows(rows, x)
    del x
    np.savez_compressed(OUT / f"rows_{cfg}_interior.npz", rows=rows, sigma_rows=yr,
                        diag_rows=rb.diag().reshape(len(a), -1)[rows.astype(np.int64)],
                        singles_degree=la[0][rows.astype(np.int64)], doubles_degree=la[1][rows.astype(np.int64)])
    print(f"{cfg} interior: {len(rows)} rows, {time.time() - t0:.1f}s", flush=True)
    return {"rows": rows.tolist(), "seconds": time.time() - t0}


def elements(ref: RefLib):
    """Random connected pairs at 36 orbitals, reference hij at bit_length 20
    (multi-word determinants), for the factorized-formula check."""
    ints = synth.synthetic_integrals(36, 30)
    t = ref.table_from_integrals(ints)
    rng = np.random.default_rng(2024)

    def rand_string(k):
        return int(sum(1 << int(i) for i in rng.choice(36, k, replace=False)))

    def excite(s, k):
        occ = [i for i in range(36) if s >> i & 1]
        vir = [i for i in range(36) if not s >> i & 1]
        for r in rng.choice(occ, k, replace=False):
            s &= ~(1 << int(r))
        for a in rng.choice(vir, k, replace=False):
            s |= 1 << int(a)
        return s

    rows = []
    kinds = {"alpha_single": (1, 0), "beta_single": (0, 1), "alpha_double": (2, 0), "beta_double": (0, 2),
             "mixed": (1, 1), "diagonal": (0, 0), "triple": (2, 1)}
    for kname, (ka, kb) in kinds.items():
        for _ in range(400):
            A, B = rand_string(15), rand_string(15)
            A2 = excite(A, ka) if ka else A
            B2 = excite(B, kb) if kb else B
            rows.append((kname, A, B, A2, B2, t.hij(A, B, A2, B2, bit_length=20)))
    arr = np.array([(r[1], r[2], r[3], r[4]) for r in rows], dtype=np.uint64)
    np.savez_compressed(OUT / "elements_n36.npz", kinds=np.array([r[0] for r in rows]), dets=arr,
                        values=np.array([r[5] for r in rows]))
    # survey phase probe: 3 orbitals
    probe = synth.Integrals(3, 2, 0, 0.0, np.zeros((3, 3)), np.zeros((3, 3, 3, 3)))
    probe.h1[0, 1] = probe.h1[1, 0] = 0.25
    pt = ref.table_from_integrals(probe)
    phase = {"a01_beta0": pt.hij(0b001, 0b001, 0b010, 0b001), "a01_beta2": pt.hij(0b001, 0b100, 0b010, 0b100),
             "b01_alpha1": pt.hij(0b010, 0b001, 0b010, 0b010), "b01_alpha0": pt.hij(0b001, 0b001, 0b001, 0b010)}
    return {"eri_sha256_n36": eri_digest(ints), "phase_probe": phase}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1-davidson", action="store_true")
    ap.add_argument("--only", choices=["fixtures", "synthetic", "elements", "c4", "interior"])
    ap.add_argument("--interior", default="C3:20,C4:10", help="cfg:n_random_rows list for --only interior")
    args = ap.parse_args()
    ref = RefLib()
    meta_path = OUT / "golden.json"
    meta = json.loads(meta_path.read_text()) if meta_path.exists() else {}
    if args.only in (None, "fixtures"):
        fixtures(ref)
    if args.only in (None, "elements"):
        meta["elements"] = elements(ref)
    if args.only == "c4":   # not part of the default run (minutes, 16 GB of host memory)
        meta["C4"] = c4_rows(ref)
    if args.only == "interior":   # not part of the default run (C4: hours on 8 cores)
        for item in args.interior.split(","):
            cfg, n = item.split(":")
            meta.setdefault(cfg, {})["interior"] = interior_rows(ref, cfg, int(n))
            meta_path.write_text(json.dumps(meta, indent=1))
    if args.only in (None, "synthetic"):
        syn = synthetic(ref, args.c1_davidson)
        for k, v in syn.items():
            if k == "C1" and "energy" in meta.get("C1", {}) and "energy" not in v:
                for key in ("energy", "iterations", "davidson_seconds", "trace"):
                    v[key] = meta["C1"][key]
            meta[k] = v
    meta["generated_by"] = "tests/golden/make_golden.py against oracle/_ref/libdetci_ref.so (unmodified reference)"
    meta_path.write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
