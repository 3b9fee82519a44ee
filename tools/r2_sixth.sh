#!/bin/bash
set -u
for p in mixed1 single mixed2 double; do
  python tools/variants.py 511 100 $p 0 128
done 2>&1 | tee gpurun_out/variants_ragged.txt
python tools/variants.py 511 100 mixed2 2016 2>&1 | tee -a gpurun_out/variants_ragged.txt
python tools/variants.py 511 100 double 1016 2>&1 | tee -a gpurun_out/variants_ragged.txt
python tools/variants.py 508 100 mixed1 0 128 2>&1 | tee -a gpurun_out/variants_ragged.txt
python tools/variants.py 510 100 single 0 2016 2>&1 | tee -a gpurun_out/variants_ragged.txt
( time timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_slabs.py -m gpu -q -x ) 2>&1 | tail -5
