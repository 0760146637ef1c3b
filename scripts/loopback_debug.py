"""Debug: which rank rows go wrong in the loopback ring after a pair."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_2601_16169_b200 import detci, synth
from util import rel_diff

os.environ["DETCI_MULTI"] = sys.argv[1] if len(sys.argv) > 1 else "ring"
ints, a, b = synth.synthetic_system("C1")
nb = len(b)
x = synth.random_vector(len(a) * nb, 11)
with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri) as basis:
    y1 = detci.matvec(basis, x)
for P in (4, 5, 8):
    for seq in (["1", "2", "1", "1"], ["2", "2"], ["b3"]):
        out = [None] * P
        gid = hash((P, tuple(seq))) & 0xffffffff
        def work(r):
            o = detci.BasisOptions(rank=r, world_size=P, loopback_group=gid, weighted_partition=True)
            with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri, o) as bs:
                xl = np.ascontiguousarray(x.reshape(-1, nb)[bs.row_begin:bs.row_end].ravel())
                res = []
                for s in seq:
                    if s == "1":
                        res.append([detci.matvec(bs, xl)])
                    elif s == "2":
                        res.append(list(detci.matvec_block(bs, np.stack([xl, 2 * xl]))))
                    else:
                        res.append(list(detci.matvec_block(bs, np.stack([xl, 2 * xl, 3 * xl]))))
                out[r] = (bs.row_begin, bs.row_end, res)
        ts = [threading.Thread(target=work, args=(r,)) for r in range(P)]
        [t.start() for t in ts]; [t.join() for t in ts]
        msgs = []
        for k, s in enumerate(seq):
            for v in range(len(out[0][2][k])):
                errs = [rel_diff(out[r][2][k][v], (v + 1) * y1.reshape(-1, nb)[out[r][0]:out[r][1]].ravel()) for r in range(P)]
                msgs.append(f"{s}[{v}]:" + ",".join(f"{e:.0e}" for e in errs))
        print(P, seq, " | ".join(msgs), flush=True)
