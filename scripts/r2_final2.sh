#!/bin/bash
# Round-2 closing pass: smoke, full GPU suite, default bench (C3), the bench
# launch list, one ncu --set full capture of the sigma kernels, then the C4
# (1e9 dets) full Davidson on one B200 with the round-2 kernels.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2i.log 2>&1
echo "smoke rc $?" >> gpurun_out/smoke_r2i.log
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gputests_r2i.log 2>&1
echo "pytest rc $?" >> gpurun_out/gputests_r2i.log
timeout 900 python bench.py > gpurun_out/bench_C3_r2i.json 2> gpurun_out/bench_C3_r2i.err
bash scripts/ncu_capture.sh C3 r2i
timeout 3000 python scripts/c4_davidson.py C4 8 > gpurun_out/davidson_C4_1gpu_r2.json 2> gpurun_out/davidson_C4_1gpu_r2.log
echo "c4 rc $?" >> gpurun_out/davidson_C4_1gpu_r2.log
