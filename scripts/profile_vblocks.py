"""One sigma with P virtual blocks (for ncu launch lists of the multi-block schedule)."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2601_16169_b200 import detci, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ints, a, b = synth.synthetic_system(cfg)
with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri,
                    detci.BasisOptions(virtual_blocks=P, weighted_partition=True)) as bs:
    x = synth.random_vector(bs.dimension(), 11)
    tm = {}
    detci.matvec(bs, x, timings=tm)
    print(cfg, P, {k: round(v * 1e3, 1) for k, v in tm.items()})
