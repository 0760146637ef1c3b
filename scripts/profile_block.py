"""Blocked sigma (M vectors) for ncu: one sigma_block call after a warm-up."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_16169_b200 import detci, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ints, a, b = synth.synthetic_system(cfg)
basis = detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri)
X = np.stack([synth.random_vector(basis.dimension(), 11 + i) for i in range(m)])
detci.matvec_block(basis, X)
detci.matvec_block(basis, X)
