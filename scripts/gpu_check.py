"""Ad-hoc GPU parity + timing probe (development script)."""
import sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
from oracle.bindings import Oracle
from paper_2601_16169_b200 import detci, synth

def rel(a, b):
    return np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))

orc = Oracle()
cases = [("tiny", 8, 6, 40), ("s12", 12, 8, 200), ("s16", 16, 10, 300)]
for name, n, ne, ns in cases:
    ints = synth.synthetic_integrals(n, ne)
    s = synth.synthetic_strings(n, ne // 2, ns)
    o = orc.system(ints, s, s)
    for vb in (1, 3):
        b = detci.GpuBasis(n, s, s, ints.core, ints.h1, ints.eri, detci.BasisOptions(virtual_blocks=vb))
        tab_ok = all(all(np.array_equal(g, w) for g, w in zip(b.table(c, k), o.tables[(c, k)])) for c in (0, 1) for k in (0, 1))
        d = b.diag()
        x = synth.random_vector(b.dimension(), 11)
        y = detci.matvec(b, x)
        yo = o.matvec(x)
        print(name, "vb", vb, "tables", tab_ok, "diag", rel(d, o.diag), "sigma", rel(y, yo), flush=True)
        if vb == 1:
            r = detci.davidson_solve(b)
            ro = o.davidson()
            print("   davidson", r.converged, r.energy, ro["energy"], len(r.iterations), ro["iterations"], flush=True)
        b.close()

for cfg in ("C1", "C2"):
    t0 = time.time()
    ints, a, bb = synth.synthetic_system(cfg)
    print(cfg, "synth", time.time() - t0, len(a), flush=True)
    t0 = time.time()
    b = detci.GpuBasis(ints.norbs, a, bb, ints.core, ints.h1, ints.eri)
    print(cfg, "build", time.time() - t0, b.nnz(), flush=True)
    x = synth.random_vector(b.dimension(), 11)
    tm = {}
    y = detci.matvec(b, x, timings=tm)
    for it in range(3):
        y = detci.matvec(b, x, timings=tm)
        print(cfg, {k: round(v, 5) for k, v in tm.items()}, flush=True)
    if cfg == "C1":
        o = orc.system(ints, a, bb)
        tab_ok = all(all(np.array_equal(g, w) for g, w in zip(b.table(c, k), o.tables[(c, k)])) for c in (0, 1) for k in (0, 1))
        rows = np.array([0, 1, 17, 500, 999], dtype=np.uint64)
        yr = o.matvec_rows(rows, x)
        print(cfg, "tables", tab_ok, "diag", rel(b.diag(), o.diag), "sigma rows", rel(y.reshape(len(a), -1)[rows.astype(int)], yr), flush=True)
        t0 = time.time()
        r = detci.davidson_solve(b)
        print(cfg, "davidson", r.converged, r.energy, len(r.iterations), time.time() - t0, flush=True)
    b.close()
