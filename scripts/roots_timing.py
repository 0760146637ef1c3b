"""Per-iteration split of the block Davidson (matvec / subspace / vector work)."""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2601_16169_b200 import detci, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
nroots = int(sys.argv[3]) if len(sys.argv) > 3 else 4
ints, a, b = synth.synthetic_system(cfg)
with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri) as g:
    for rep in range(2):
        t0 = time.time()
        r = detci.davidson_roots(g, nroots, max_iter=iters, want_vectors=False)
        wall = time.time() - t0
        it = r.iterations
        mv = np.array([x.matvec_seconds for x in it])
        ss = np.array([x.subspace_solve_seconds for x in it])
        og = np.array([x.orthogonalization_seconds for x in it])
        print(f"{cfg} roots {nroots} rep {rep}: {len(it)} it, wall {wall:.2f}s, solver {r.seconds:.2f}s, "
              f"sum matvec {mv.sum():.2f}s subspace {ss.sum():.2f}s ortho {og.sum():.2f}s, "
              f"setup+other {r.seconds - mv.sum() - ss.sum() - og.sum():.2f}s", flush=True)
