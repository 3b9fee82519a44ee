#!/bin/bash
# Diagnostics-kernel sweep (run under gpurun, ONE GPU): blocks per SM of the persistent grid x
# next-iteration L2 prefetch, device time of mlb_diagnostics at 512^3 and 256^3.
OUT=gpurun_out/diag_sweep.txt
mkdir -p gpurun_out; : > $OUT
for n in 512 256; do
  for pf in 0 1; do
    for bps in 1 2 3 4 8; do
      echo "# n=$n MLB_DIAG_PF=$pf MLB_DIAG_BPS=$bps" >> $OUT
      MLB_DIAG_PF=$pf MLB_DIAG_BPS=$bps python tools/diag_time.py $n 2>&1 | grep diag >> $OUT
    done
  done
done
cat $OUT
