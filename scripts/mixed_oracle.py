"""Mixed oracle beyond C1: the UNMODIFIED reference
davidson_solve (proj/core/src/davidson.cpp:73-206, compiled into
oracle/_ref/libdetci_ref.so) driving the device sigma through its
LinearOperator callback (davidson.hpp:28), against the device-resident
Davidson on the same basis.  The device sigma is pinned to the reference
matvec rows at 1e-12 (tests/golden rows_C2/C3), so agreement of the two
solvers' traces and energies is the energy parity of the drop-in at sizes
the all-CPU reference cannot finish (one reference sigma at C3 is ~5 h on
16 cores).

    python scripts/mixed_oracle.py C2 260 [max_subspace] > profiles/mixed_oracle_C2.json
    python scripts/mixed_oracle.py C2:7000 300   # C2 integrals, 7000 strings per channel

Prints one JSON object: per-iteration Ritz values / residuals of both
solvers, the largest per-iteration differences, and both final energies.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from oracle.bindings import REF_SO, RefLib  # noqa: E402
from paper_2601_16169_b200 import detci, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ms = int(sys.argv[3]) if len(sys.argv) > 3 else 20
if not REF_SO.exists():
    sys.exit("reference library not built (oracle/_ref)")

t0 = time.time()
if ":" in cfg:   # "C2:7000": the config's integrals, its first 7000 strings per channel
    name, count = cfg.split(":")
    norbs, nelec, _ = synth.CONFIGS[name]
    ints = synth.synthetic_integrals(norbs, nelec)
    a = synth.synthetic_strings(norbs, nelec // 2, int(count))
    b = a.copy()
else:
    ints, a, b = synth.synthetic_system(cfg)
basis = detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri)
diag = basis.diag()
print(f"{cfg}: dim {len(diag)}, setup {time.time() - t0:.1f} s", file=sys.stderr, flush=True)

t0 = time.time()
dev = detci.davidson_solve(basis, detci.DavidsonOptions(max_iter=max_iter, max_subspace=ms), want_vector=False)
t_dev = time.time() - t0
print(f"device: {dev.status} after {len(dev.iterations)} it, E {dev.energy:.12f}, {t_dev:.1f} s",
      file=sys.stderr, flush=True)

ref = RefLib()
calls = [0]
sig_s = [0.0]
t_last = [time.time()]


def apply(x, y):
    t = time.time()
    detci.matvec(basis, x, y)
    sig_s[0] += time.time() - t
    calls[0] += 1
    if calls[0] % 10 == 0:
        print(f"  reference solver: {calls[0]} sigma calls, {time.time() - t_last[0]:.1f} s since last report",
              file=sys.stderr, flush=True)
        t_last[0] = time.time()


t0 = time.time()
mixed = ref.davidson_operator(apply, diag, max_iter=max_iter, max_subspace=ms)
t_mixed = time.time() - t0
status_names = {0: "converged", 1: "max_iterations", 2: "breakdown"}
print(f"reference solver over device sigma: {status_names.get(mixed['status'])} after {mixed['iterations']} it, "
      f"E {mixed['energy']:.12f}, {t_mixed:.1f} s", file=sys.stderr, flush=True)

tr = mixed["trace"]
n = min(len(tr), len(dev.iterations))
ritz_ref = tr[:n, 0]
ritz_dev = np.array([it.ritz_value for it in dev.iterations[:n]])
res_ref = tr[:n, 1]
res_dev = np.array([it.residual_norm for it in dev.iterations[:n]])
rel = np.abs(ritz_ref - ritz_dev) / np.abs(ritz_ref)
out = {
    "config": cfg,
    "dim": int(len(diag)),
    "max_iter": max_iter,
    "max_subspace": ms,
    "reference_solver": {
        "what": "unmodified reference davidson_solve (oracle/_ref/libdetci_ref.so) over the device sigma",
        "status": status_names.get(mixed["status"], mixed["status"]),
        "iterations": int(mixed["iterations"]),
        "energy": mixed["energy"],
        "seconds": t_mixed,
        "sigma_seconds": sig_s[0],
    },
    "device_solver": {
        "status": dev.status,
        "iterations": len(dev.iterations),
        "energy": dev.energy,
        "seconds": t_dev,
    },
    "energy_abs_diff": abs(mixed["energy"] - dev.energy),
    "iterations_compared": n,
    "ritz_max_rel_diff": float(rel.max()) if n else None,
    "ritz_max_rel_diff_iter": int(rel.argmax()) if n else None,
    "residual_max_rel_diff": float(np.max(np.abs(res_ref - res_dev) / np.maximum(res_ref, 1e-300))) if n else None,
    "restarts_equal": bool(np.array_equal(tr[:n, 3] > 0, np.array([it.restarted for it in dev.iterations[:n]]))),
    "trace": [[float(ritz_ref[i]), float(ritz_dev[i]), float(res_ref[i]), float(res_dev[i])] for i in range(n)],
    "trace_columns": ["ritz_reference", "ritz_device", "residual_reference", "residual_device"],
    "host": {"cpus": os.cpu_count()},
}
print(json.dumps(out))
