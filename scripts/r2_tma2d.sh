#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_davidson.py -x -q > gpurun_out/t_tma2d.log 2>&1
echo "pytest rc $?" >> gpurun_out/t_tma2d.log
for v in "DETCI_DAV_TMA2D=1" "DETCI_DAV_TMA2D=0" "DETCI_DAV_TMA2D=1"; do
  echo "== $v" >> gpurun_out/dav_tma2d.txt
  env $v timeout 300 python scripts/davidson_timing.py C2 60 1 >> gpurun_out/dav_tma2d.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_dav|k_scale|k_finalize" --csv --log-file gpurun_out/ncu_dav_r2f.csv \
    python scripts/profile_davidson.py C2 12 > gpurun_out/ncu_dav_r2f.out 2>&1
timeout 900 python -m pytest tests/test_gpu_mixed_oracle.py tests/test_gpu_loopback.py tests/test_gpu_integration.py -q > gpurun_out/t_tma2d_b.log 2>&1
echo "pytest rc $?" >> gpurun_out/t_tma2d_b.log
