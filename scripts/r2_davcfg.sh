#!/bin/bash
# Davidson stream-pass configurations on one box (C2, 60 iterations), the
# launch list of the default, and the Davidson parity tests.
mkdir -p gpurun_out
for v in "DETCI_DAV_CFG=512,1,2" "DETCI_DAV_CFG=512,1,3" "DETCI_DAV_CFG=256,2,2" "DETCI_DAV_CFG=256,2,3" "DETCI_DAV_STREAM=reg" "DETCI_DAV_CFG=512,1,2"; do
  echo "== $v" >> gpurun_out/dav_cfg_r2e.txt
  env $v timeout 300 python scripts/davidson_timing.py C2 60 1 >> gpurun_out/dav_cfg_r2e.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_dav|k_scale|k_finalize" --csv --log-file gpurun_out/ncu_dav_r2e.csv \
    python scripts/profile_davidson.py C2 12 > gpurun_out/ncu_dav_r2e.out 2>&1
timeout 900 python -m pytest tests/test_gpu_basis.py tests/test_gpu_davidson.py tests/test_gpu_mixed_oracle.py \
    tests/test_gpu_loopback.py -q > gpurun_out/t_davcfg.log 2>&1
echo "pytest rc $?" >> gpurun_out/t_davcfg.log
