#!/bin/bash
# Round-2 validation pass 2: wide strings, Davidson (warp-issued copies,
# analytic normalisation), committed C2 mixed-oracle trace, loopback; timing
# and ncu launch list of the vector kernels; then the C3 mixed-oracle trace.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_wide.py tests/test_gpu_davidson.py tests/test_gpu_mixed_oracle.py \
    tests/test_gpu_loopback.py tests/test_gpu_multiroot.py -q > gpurun_out/t_validate2.log 2>&1
echo "pytest rc $?" >> gpurun_out/t_validate2.log
timeout 300 python scripts/davidson_timing.py C2 60 2 > gpurun_out/dav_r2d.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_dav|k_scale|k_finalize" --csv --log-file gpurun_out/ncu_dav_r2d.csv \
    python scripts/profile_davidson.py C2 12 > gpurun_out/ncu_dav_r2d.out 2>&1
timeout 2400 python scripts/mixed_oracle.py C3 30 > gpurun_out/mixed_oracle_C3_30.json 2> gpurun_out/mixed_oracle_C3_30.log
