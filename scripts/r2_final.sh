#!/bin/bash
# Round-2 end-of-work pass: smoke, full GPU suite, default bench (C3), the
# bench launch list, Davidson stream-kernel variants.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2d.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gputests_r2d.log 2>&1
echo "pytest rc $?" >> gpurun_out/gputests_r2d.log
timeout 900 python bench.py > gpurun_out/bench_C3_r2d.json 2> gpurun_out/bench_C3_r2d.err
for v in "DETCI_DAV_RITZ_SPLIT=1" "DETCI_DAV_CFG=512,1,2" "DETCI_DAV_CFG=512,1,4"; do
  echo "== $v" >> gpurun_out/dav_variants_r2d.txt
  env $v timeout 300 python scripts/davidson_timing.py C2 60 1 >> gpurun_out/dav_variants_r2d.txt 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_C3_r2d.csv \
  python bench.py --config C3 --steps 2 --warmup 3 --no-davidson --no-cpu-baseline > gpurun_out/launches_bench_C3_r2d.json 2>&1
