#!/bin/bash
# Converged-energy parity at C2 (1e8 dets): the unmodified reference
# davidson_solve over the device sigma, run to convergence, against the
# device Davidson (scripts/mixed_oracle.py; ~20 s of single-threaded
# reference vector work per iteration).
mkdir -p gpurun_out
timeout 6600 python scripts/mixed_oracle.py C2 300 > gpurun_out/mixed_oracle_C2_converged.json 2> gpurun_out/mixed_oracle_C2_converged.log
echo "rc $?" >> gpurun_out/mixed_oracle_C2_converged.log
