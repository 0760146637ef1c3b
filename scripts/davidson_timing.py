"""Per-iteration Davidson timing split (matvec / subspace solve / orthogonalization)."""
import sys
import time
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_16169_b200 import detci, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
ints, a, b = synth.synthetic_system(cfg)
basis = detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri)
for rep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    t0 = time.time()
    res = detci.davidson_solve(basis, detci.DavidsonOptions(max_iter=iters), want_vector=False)
    wall = time.time() - t0
    mv = np.array([it.matvec_seconds for it in res.iterations])
    ss = np.array([it.subspace_solve_seconds for it in res.iterations])
    og = np.array([it.orthogonalization_seconds for it in res.iterations])
    print(f"{cfg} rep {rep}: {res.status} {len(res.iterations)} it, wall {wall:.3f}s, solver {res.seconds:.3f}s, "
          f"per it: matvec {mv.mean()*1e3:.2f} ms, subspace {ss.mean()*1e3:.2f} ms, ortho {og.mean()*1e3:.2f} ms, "
          f"first it matvec {mv[0]*1e3:.1f} ms", flush=True)
