"""Full Davidson at C4 (1e9 determinants) on ONE B200.

The survey's target is full convergence of the ~1e9-determinant problem on an
8-GPU box; one GPU holds the basis, the sigma scratch and a reduced subspace
(max_subspace 6 or 8 => (2*ms+3) * 8 GB of Davidson vectors), so this runs the
same solver with fewer subspace vectors (more restarts).

usage: python scripts/c4_davidson.py [config] [max_subspace ...] > out.json
"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2601_16169_b200 import detci, synth  # noqa: E402
from paper_2601_16169_b200.errors import CapacityError  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
subspaces = [int(x) for x in sys.argv[2:]] or [8, 6]
t0 = time.time()
ints, a, b = synth.synthetic_system(cfg)
t_host = time.time() - t0
t0 = time.time()
basis = detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri)
t_build = time.time() - t0
print(f"{cfg}: dim {basis.local_dim}, host strings {t_host:.1f} s, device build {t_build:.2f} s",
      file=sys.stderr, flush=True)


def progress(it, i):
    if i % 10 == 0:
        print(f"  it {i}: ritz {it.ritz_value:.12f} res {it.residual_norm:.3e} "
              f"sigma {it.matvec_seconds:.3f} s ortho {it.orthogonalization_seconds:.3f} s",
              file=sys.stderr, flush=True)


for ms in subspaces:
    try:
        res = detci.davidson_solve(basis, detci.DavidsonOptions(max_iter=2000, max_subspace=ms),
                                   want_vector=False, callback=progress)
    except CapacityError as e:
        print(f"max_subspace {ms}: {e}", file=sys.stderr, flush=True)
        continue
    its = res.iterations
    mv = sum(i.matvec_seconds for i in its)
    out = {
        "config": cfg, "dim": basis.local_dim, "max_subspace": ms, "status": res.status,
        "converged": res.converged, "energy": res.energy, "iterations": len(its),
        "restarts": sum(1 for i in its if i.restarted), "seconds": res.seconds,
        "s_per_iter": res.seconds / max(1, len(its)), "sigma_seconds": mv,
        "sigma_share": mv / res.seconds if res.seconds else None,
        "final_residual": its[-1].residual_norm if its else None,
        "max_gram_deviation": max((i.max_gram_deviation for i in its), default=None),
        "device_build_seconds": t_build,
    }
    print(json.dumps(out), flush=True)
    break
