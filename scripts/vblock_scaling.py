"""Multi-GPU schedule emulated on one GPU: sigma with P virtual alpha blocks
runs every rank's work (partition, ring windows, scatter items restricted to
the block) in turn, so T(P)/P estimates one rank's time on P GPUs (the ring
transfer itself, overlapped on NVLink, is not included)."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2601_16169_b200 import detci, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
ints, a, b = synth.synthetic_system(cfg)
x = synth.random_vector(len(a) * len(b), 11)
base = None
for P in (1, 2, 4, 8):
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri,
                        detci.BasisOptions(virtual_blocks=P, weighted_partition=True)) as bs:
        tm = {}
        detci.matvec(bs, x, timings=tm)
        ts = []
        for _ in range(2):
            tm = {}
            detci.matvec(bs, x, timings=tm)
            ts.append(tm)
        t = min(d["total_seconds"] for d in ts)
        split = {k: round(min(d[k] for d in ts) * 1e3, 1) for k in ("alpha_seconds", "beta_seconds", "mixed_seconds")}
        base = base or t
        print(f"{cfg} P={P}: total {t*1e3:.1f} ms, per rank {t/P*1e3:.1f} ms, est. speed-up {base/(t/P):.2f}x, split {split}",
              flush=True)
