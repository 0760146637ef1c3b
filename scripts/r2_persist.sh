#!/bin/bash
# Persistent same-spin kernel (DETCI_SAMESPIN_PERSIST=1): parity, then A/B
# timing of the bench phases at C3 and C2 (alternating, two rounds each;
# arm "1r16": persistent with 16-warp CTAs).
mkdir -p gpurun_out
timeout 600 python scripts/parity_probe.py 4000 5000 6000 7000 8000 > gpurun_out/parity_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_sigma.py -q -k "samespin" > gpurun_out/t_persist.log 2>&1
echo "pytest rc $?" >> gpurun_out/t_persist.log
for rep in 1 2; do
  for p in 0 1 1r16; do
    rows=8; [ "$p" = "1r16" ] && rows=16
    DETCI_SAMESPIN_PERSIST=${p:0:1} DETCI_SAMESPIN_ROWS=$rows timeout 600 python bench.py --steps 5 --warmup 3 --no-davidson \
      --no-cpu-baseline --no-stored --block 0 --roots 0 > gpurun_out/persist_${p}_${rep}.json 2> gpurun_out/persist_${p}_${rep}.err
  done
done
python - <<'PY' > gpurun_out/persist_summary.txt 2>&1
import json
for rep in (1, 2):
    for p in ("0", "1", "1r16"):
        try:
            d = json.load(open(f"gpurun_out/persist_{p}_{rep}.json"))
        except Exception as e:
            print(rep, p, "failed", e); continue
        ph = d["config"]["phase_seconds"]; c2 = d["extra_configs"]["C2"]
        print(f"rep {rep} persist {p}: C3 {d['ms_per_step']:.1f} ms alpha {ph['alpha_seconds']*1e3:.1f} beta {ph['beta_seconds']*1e3:.1f} "
              f"| C2 {c2['ms_per_step']:.2f} ms alpha {c2['phase_seconds']['alpha_seconds']*1e3:.2f} beta {c2['phase_seconds']['beta_seconds']*1e3:.2f} "
              f"| e2e C3 {d['e2e']['ms_per_step']:.1f}")
PY
