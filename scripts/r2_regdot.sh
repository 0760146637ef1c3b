#!/bin/bash
mkdir -p gpurun_out
timeout 300 env DETCI_DAV_STREAM=reg python -m pytest tests/test_gpu_davidson.py -x -q > gpurun_out/t_regdot.log 2>&1
echo "pytest rc $?" >> gpurun_out/t_regdot.log
for v in "DETCI_DAV_STREAM=warp" "DETCI_DAV_STREAM=reg" "DETCI_DAV_STREAM=reg_ritz" "DETCI_DAV_STREAM=warp" "DETCI_DAV_STREAM=reg_ritz"; do
  echo "== $v" >> gpurun_out/dav_regdot.txt
  env $v timeout 300 python scripts/davidson_timing.py C2 60 1 >> gpurun_out/dav_regdot.txt 2>&1
done
DETCI_DAV_STREAM=reg timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_dav|k_scale|k_finalize" --csv --log-file gpurun_out/ncu_dav_r2g.csv \
    python scripts/profile_davidson.py C2 12 > gpurun_out/ncu_dav_r2g.out 2>&1
