#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
( time timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -m gpu -q -x -k "staged or no_pack_divides or overlapped or host_run or resident or divergence or variants_never" ) > $OUT/tests_new2.log 2>&1
tail -4 $OUT/tests_new2.log
for p in mixed1 mixed2; do
  python tools/variants.py 512 100 $p 0 4000
  python tools/variants.py 256 400 $p 0 4000
  python tools/variants.py 511 100 $p 0 4000 128
done 2>&1 | tee $OUT/variants_stage.txt
MLB_STAGE_TPB=4 python tools/variants.py 512 100 mixed1 4000 2>&1 | tee -a $OUT/variants_stage.txt
MLB_STAGE_TPB=64 python tools/variants.py 512 100 mixed1 4000 2>&1 | tee -a $OUT/variants_stage.txt
python tools/variants.py 512 100 single 0 4000 2>&1 | tee -a $OUT/variants_stage.txt
python tools/variants.py 511 100 single 0 1016 4000 2>&1 | tee -a $OUT/variants_stage.txt
( time python bench.py --steps 20 --warmup 5 --no-extra --no-cpu-baseline ) 2>&1 | tail -c 1800
