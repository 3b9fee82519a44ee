#!/bin/bash
set -u
( time timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "staged" ) 2>&1 | tail -4
for p in mixed1 mixed2; do
  python tools/variants.py 512 100 $p 0 5008 5016 5032
  python tools/variants.py 256 400 $p 0 5008 5016
  python tools/variants.py 511 100 $p 0 5008
done 2>&1 | tee gpurun_out/variants_pipe.txt
for r in 2 8 16; do MLB_PIPE_ROWS=$r python tools/variants.py 512 100 mixed1 5008; done 2>&1 | tee -a gpurun_out/variants_pipe.txt
