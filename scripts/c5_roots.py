"""Config C5 (BASELINE.json: 36 orbitals, 3e8 determinants, 4 roots; an
8-GPU config) by block Davidson on ONE B200, to convergence.

usage: python scripts/c5_roots.py [nroots] [max_iter] > out.json
"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2601_16169_b200 import detci, synth  # noqa: E402

nroots = int(sys.argv[1]) if len(sys.argv) > 1 else 4
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
ints, a, b = synth.synthetic_system("C5")
t0 = time.time()
basis = detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri)
t_build = time.time() - t0
res = detci.davidson_roots(basis, nroots, max_iter=max_iter, want_vectors=False)
its = res.iterations
mv = sum(i.matvec_seconds for i in its)
print(json.dumps({
    "config": "C5", "dim": basis.local_dim, "nroots": nroots, "status": res.status, "converged": res.converged,
    "energies": res.energies.tolist(), "residuals": res.residuals.tolist(), "iterations": len(its),
    "seconds": res.seconds, "s_per_iter": res.seconds / max(1, len(its)), "sigma_share": mv / res.seconds,
    "max_gram_deviation": max((i.max_gram_deviation for i in its), default=None),
    "device_build_seconds": t_build,
}), flush=True)
