#!/bin/bash
set -u
for n in 128 256 384; do for b in 0 1; do
  echo "n=$n MLB_PF_BULK=$b"
  MLB_PF_BULK=$b MLB_PRECS=single,mixed1,mixed2 python tools/quick.py $n $((n <= 256 ? 400 : 150)) 2>&1 | cut -c1-200
done; done | tee gpurun_out/pf_bulk_sizes.txt
