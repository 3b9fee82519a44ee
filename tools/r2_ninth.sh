#!/bin/bash
set -u
OUT=gpurun_out
( time MLB_FUZZ_CASES=600 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -x ) > $OUT/fuzz_600.log 2>&1
tail -5 $OUT/fuzz_600.log
( time timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fuzz.py ) > $OUT/tests_all2.log 2>&1
tail -5 $OUT/tests_all2.log
python tools/quick.py 256 400 2>&1 | cut -c1-220
python tools/quick.py 128 800 2>&1 | cut -c1-220
