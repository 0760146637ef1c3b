#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2g.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gputests_r2g.log 2>&1
echo "pytest rc $?" >> gpurun_out/gputests_r2g.log
timeout 900 python bench.py > gpurun_out/bench_C3_r2g.json 2> gpurun_out/bench_C3_r2g.err
