#!/bin/bash
# Round-2 validation pass: wide strings, Davidson passes, loopback; Davidson
# timing (register vs warp dot kernels); ncu launch list of the vector
# kernels; the C2 mixed-oracle trace (reference solver over the device sigma).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_davidson.py tests/test_gpu_loopback.py \
    tests/test_gpu_multiroot.py "tests/test_gpu_mixed_oracle.py::test_reference_solver_trace_c2" -x -q \
    > gpurun_out/t_validate.log 2>&1
echo "pytest rc $?" >> gpurun_out/t_validate.log
timeout 300 python scripts/davidson_timing.py C2 60 2 > gpurun_out/dav_reg.txt 2>&1
DETCI_DAV_STREAM=warp timeout 300 python scripts/davidson_timing.py C2 60 2 > gpurun_out/dav_warp.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_dav|k_scale|k_finalize" --csv --log-file gpurun_out/ncu_dav_reg.csv \
    python scripts/profile_davidson.py C2 12 > gpurun_out/ncu_dav_reg.out 2>&1
timeout 1500 python scripts/mixed_oracle.py C2 40 > gpurun_out/mixed_oracle_C2_40.json 2> gpurun_out/mixed_oracle_C2_40.log
