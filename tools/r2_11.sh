#!/bin/bash
set -u
( time timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "staged" ) 2>&1 | tail -4
for p in mixed1 mixed2; do
  python tools/variants.py 512 100 $p 0 4000
  python tools/variants.py 256 400 $p 0 4000
done 2>&1 | tee gpurun_out/variants_stage4.txt
for g in 1 2 4 16 64; do MLB_STAGE_GROUP=$g python tools/variants.py 512 100 mixed1 4000; done 2>&1 | tee -a gpurun_out/variants_stage4.txt
MLB_STAGE_PF=1 python tools/variants.py 512 100 mixed1 4000 2>&1 | tee -a gpurun_out/variants_stage4.txt
MLB_STAGE_PF=1 python tools/variants.py 512 100 mixed2 4000 2>&1 | tee -a gpurun_out/variants_stage4.txt
