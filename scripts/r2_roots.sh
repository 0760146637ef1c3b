#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multiroot.py tests/test_gpu_loopback.py -q > gpurun_out/t_roots.log 2>&1
echo "pytest rc $?" >> gpurun_out/t_roots.log
timeout 600 python scripts/roots_timing.py C3 10 4 > gpurun_out/roots_timing.txt 2>&1
DETCI_DAVIDSON_BLOCK_RITZ=0 timeout 600 python scripts/roots_timing.py C3 10 4 >> gpurun_out/roots_timing.txt 2>&1
