#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sigma.py tests/test_gpu_basis.py tests/test_gpu_wide.py -q > gpurun_out/t_tail.log 2>&1
echo "pytest rc $?" >> gpurun_out/t_tail.log
timeout 600 python bench.py --no-davidson > gpurun_out/bench_C3_r2h.json 2> gpurun_out/bench_C3_r2h.err
