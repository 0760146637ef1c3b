#!/bin/bash
# Profiling recipe (B200_PROFILING.md) for the bench workload; run under gpurun.
set -x
CFG=${1:-C2}
TAG=${2:-r1}
mkdir -p gpurun_out
# 1. launch list of the bench command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${CFG}_${TAG}.csv \
  python bench.py --config $CFG --steps 2 --warmup 3 --no-davidson --no-cpu-baseline > gpurun_out/launches_bench_${CFG}_${TAG}.json 2>&1
# 2. full capture of every sigma kernel once (skip the warm-up launches)
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_mixed|k_samespin|k_eps|k_transpose" -c 10 \
  -o gpurun_out/full_${CFG}_${TAG} python scripts/profile_sigma.py $CFG 1 > gpurun_out/full_${CFG}_${TAG}.log 2>&1
tail -2 gpurun_out/full_${CFG}_${TAG}.log
