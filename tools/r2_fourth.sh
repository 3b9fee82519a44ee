#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
( time timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "staged" ) > $OUT/tests_stage.log 2>&1
tail -4 $OUT/tests_stage.log
for p in mixed1 mixed2; do
  python tools/variants.py 512 100 $p 0 4000
  python tools/variants.py 256 400 $p 0 4000
  python tools/variants.py 511 100 $p 0 4000
done 2>&1 | tee $OUT/variants_stage2.txt
for r in 4 8 32 64; do MLB_STAGE_ROWS=$r python tools/variants.py 512 100 mixed1 4000; done 2>&1 | tee -a $OUT/variants_stage2.txt
bash tools/ncu_one.sh stage_f16_512 step_stage 2 -- python tools/variants.py 512 4 mixed1 4000
