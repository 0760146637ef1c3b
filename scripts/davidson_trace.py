"""Davidson convergence trace at a config (residual, Gram deviation, restarts)."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2601_16169_b200 import detci, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 400
ints, a, b = synth.synthetic_system(cfg)
basis = detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri)
res = detci.davidson_solve(basis, detci.DavidsonOptions(max_iter=iters), want_vector=False)
for i, it in enumerate(res.iterations):
    if i % 10 == 0 or i == len(res.iterations) - 1:
        print(f"{i:4d} {it.ritz_value:.12f} res {it.residual_norm:.3e} gram {it.max_gram_deviation:.1e} {'R' if it.restarted else ''}")
print(cfg, res.status, len(res.iterations), f"{res.energy:.12f}", f"{res.seconds:.1f}s")
