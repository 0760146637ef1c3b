"""Build one config and run sigma a few times (for ncu / nsight captures)."""
import sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_16169_b200 import detci, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ints, a, b = synth.synthetic_system(cfg)
basis = detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri)
x = synth.random_vector(basis.dimension(), 11)
for _ in range(reps):
    tm = {}
    detci.matvec(basis, x, timings=tm)
    print(cfg, {k: round(v, 5) for k, v in tm.items()}, flush=True)
