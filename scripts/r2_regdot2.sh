#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_davidson.py tests/test_gpu_mixed_oracle.py tests/test_gpu_loopback.py tests/test_gpu_integration.py tests/test_gpu_multiroot.py -q > gpurun_out/t_regdot2.log 2>&1
echo "pytest rc $?" >> gpurun_out/t_regdot2.log
for v in "DETCI_DAV_STREAM=reg" "DETCI_DAV_STREAM=warp" "DETCI_DAV_STREAM=reg" "DETCI_DAV_STREAM=warp" "DETCI_DAV_STREAM=reg"; do
  echo "== $v" >> gpurun_out/dav_regdot2.txt
  env $v timeout 300 python scripts/davidson_timing.py C2 60 1 >> gpurun_out/dav_regdot2.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_dav|k_scale|k_finalize" --csv --log-file gpurun_out/ncu_dav_r2h.csv \
    python scripts/profile_davidson.py C2 24 > gpurun_out/ncu_dav_r2h.out 2>&1
DETCI_DAV_STREAM=warp timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_dav|k_scale|k_finalize" --csv --log-file gpurun_out/ncu_dav_r2h_warp.csv \
    python scripts/profile_davidson.py C2 24 > gpurun_out/ncu_dav_r2h_warp.out 2>&1
