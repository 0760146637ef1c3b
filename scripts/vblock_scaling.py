"""Multi-GPU scaling estimate on one GPU.  sigma with P virtual alpha blocks
runs every rank's share of the multi-rank schedule in turn (default: the
gather schedule -- its own rows' beta and alpha terms, its beta-slot column
share of the mixed term); the library times each share with CUDA events
(detci_gpu_rank_seconds).  A P-GPU sigma takes at least the slowest rank's
share, so the estimate is T(1) / max_g t_g (the transfers -- Cs allgather
under the beta term, the slab all-to-all -- are not included).

    python scripts/vblock_scaling.py C3 [P ...] [--rebalance R]   (default P = 1 2 4 8)

--rebalance R runs R rounds of the measured rebalance (detci_gpu_rebalance)
before timing.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_16169_b200 import detci, synth  # noqa: E402

argv = sys.argv[1:]
rebal = 0
if "--rebalance" in argv:
    i = argv.index("--rebalance")
    rebal = int(argv[i + 1])
    del argv[i:i + 2]
cfg = argv[0] if argv else "C3"
Ps = [int(p) for p in argv[1:]] or [1, 2, 4, 8]
ints, a, b = synth.synthetic_system(cfg)
x = synth.random_vector(len(a) * len(b), 11)
base = None
rows = []
for P in Ps:
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri,
                        detci.BasisOptions(virtual_blocks=P, weighted_partition=True)) as bs:
        before = bs.rebalance(rebal) if (rebal and P > 1) else None
        detci.matvec(bs, x, timings={})   # warm (plans, tables)
        best = None
        for _ in range(2):
            tm = {}
            detci.matvec(bs, x, timings=tm)
            ranks = bs.rank_seconds() if P > 1 else [tm["total_seconds"]]
            phases = bs.rank_phase_seconds() if P > 1 else []
            if best is None or max(ranks) < max(best[1]):
                best = (tm, ranks, phases)
        tm, ranks, phases = best
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
               "speedup_max_rank": base / mx if base else None, "ranks_ms": [r * 1e3 for r in ranks],
               "rank_phase_ms": [[round(q * 1e3, 2) for q in r] for r in phases],
               "rebalance_rounds": rebal, "max_over_mean_before_rebalance": before}
        rows.append(row)
        print(json.dumps(row), flush=True)
