#!/bin/bash
# Round-2 re-entry check: smoke, full GPU suite, default bench (C3).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2x.log 2>&1
echo "smoke rc $?" >> gpurun_out/smoke_r2x.log
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gputests_r2x.log 2>&1
echo "pytest rc $?" >> gpurun_out/gputests_r2x.log
timeout 900 python bench.py > gpurun_out/bench_C3_r2x.json 2> gpurun_out/bench_C3_r2x.err
