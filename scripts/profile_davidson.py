"""A short single-root Davidson for ncu launch lists of the vector kernels.

    python scripts/profile_davidson.py C2 12
"""
import sys

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2601_16169_b200 import detci, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 12
ints, a, b = synth.synthetic_system(cfg)
with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri) as basis:
    res = detci.davidson_solve(basis, detci.DavidsonOptions(max_iter=iters), want_vector=False)
    print(res.status, len(res.iterations), res.energy)
