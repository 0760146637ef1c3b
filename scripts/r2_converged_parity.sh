#!/bin/bash
# Converged-energy parity at C2's integrals with 7000 strings per channel
# (4.9e7 dets): the unmodified reference davidson_solve over the device
# sigma, run to convergence, against the device Davidson
# (scripts/mixed_oracle.py; the reference's single-threaded vector work is
# ~20 s per iteration per 1e8 dets, so the full C2 run (202 iterations) does
# not fit one 60-minute GPU call).
mkdir -p gpurun_out
timeout 3400 python scripts/mixed_oracle.py C2:7000 300 > gpurun_out/mixed_oracle_C2_7000_converged.json 2> gpurun_out/mixed_oracle_C2_7000_converged.log
echo "rc $?" >> gpurun_out/mixed_oracle_C2_7000_converged.log
