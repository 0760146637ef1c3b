"""Multi-GPU scaling estimate on one GPU.  sigma with P virtual alpha blocks
runs every rank's share of the multi-rank schedule in turn (default: the
gather schedule -- its own rows' beta and alpha terms, its beta-slot column
share of the mixed term); the library times each share with CUDA events
(detci_gpu_rank_seconds).  A P-GPU sigma takes at least the slowest rank's
share, so the estimate is T(1) / max_g t_g (the transfers -- Cs allgather
under the beta term, the slab all-to-all -- are not included).

    python scripts/vblock_scaling.py C3 [P ...]      (default P = 1 2 4 8)
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_16169_b200 import detci, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
Ps = [int(p) for p in sys.argv[2:]] or [1, 2, 4, 8]
ints, a, b = synth.synthetic_system(cfg)
x = synth.random_vector(len(a) * len(b), 11)
base = None
rows = []
for P in Ps:
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri,
                        detci.BasisOptions(virtual_blocks=P, weighted_partition=True)) as bs:
        detci.matvec(bs, x, timings={})   # warm (plans, tables)
        best = None
        for _ in range(2):
            tm = {}
            detci.matvec(bs, x, timings=tm)
            ranks = bs.rank_seconds() if P > 1 else [tm["total_seconds"]]
            if best is None or max(ranks) < max(best[1]):
                best = (tm, ranks)
        tm, ranks = best
        # device time of the kernels (the host-pointer call's total also
        # holds its copies)
        dev = sum(tm[k] for k in ("alpha_seconds", "beta_seconds", "mixed_seconds", "combine_seconds"))
        if P == 1:
            ranks = [dev]
        t1 = dev if P == 1 else None
        base = base or t1
        mx, mean = max(ranks), sum(ranks) / len(ranks)
        row = {"config": cfg, "P": P, "device_ms": dev * 1e3, "max_rank_ms": mx * 1e3,
               "mean_rank_ms": mean * 1e3, "max_over_mean": mx / mean,
               "speedup_max_rank": base / mx if base else None, "ranks_ms": [r * 1e3 for r in ranks]}
        rows.append(row)
        print(json.dumps(row), flush=True)
