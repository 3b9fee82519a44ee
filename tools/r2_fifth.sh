#!/bin/bash
set -u
for lib in "" "$PWD/_ab/libmlb_ca.so"; do for pf in 0 1; do
  echo "lib=${lib:-default(cg)} pf=$pf"
  MLB_LIB_PATH=$lib MLB_STAGE_PF=$pf python tools/variants.py 512 100 mixed1 4000
  MLB_LIB_PATH=$lib MLB_STAGE_PF=$pf python tools/variants.py 512 100 mixed2 4000
done; done 2>&1 | tee gpurun_out/variants_stage3.txt
