"""Device Davidson iteration counts at C2's integrals with fewer strings per
channel (sizing the converged mixed-oracle run, whose reference-side vector
work is ~20 s per iteration per 1e8 determinants, single-threaded)."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2601_16169_b200 import detci, synth  # noqa: E402

norbs, nelec, _ = synth.CONFIGS["C2"]
ints = synth.synthetic_integrals(norbs, nelec)
for count in [int(c) for c in sys.argv[1:]]:
    a = synth.synthetic_strings(norbs, nelec // 2, count)
    with detci.GpuBasis(ints.norbs, a, a.copy(), ints.core, ints.h1, ints.eri) as g:
        t = time.time()
        r = detci.davidson_solve(g, detci.DavidsonOptions(max_iter=400), want_vector=False)
        print(f"C2:{count} dim {count * count:.3e} {r.status} it {len(r.iterations)} E {r.energy:.12f} "
              f"{time.time() - t:.1f} s; reference estimate {len(r.iterations) * 21 * count * count / 1e8 / 60:.0f} min",
              flush=True)
