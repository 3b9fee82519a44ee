# Fuzz suites on the final build (run under gpurun, ONE GPU).  (compute-sanitizer was closed on the GPU pool in
# the last session of round 2; the sanitizer records under profiles/ are from the sessions before.)
set -u
OUT=gpurun_out; mkdir -p $OUT
F=$OUT/fuzz_final.txt
echo "# MLB_FUZZ_CASES=20000 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -n 4   (one B200, round 2, final library build)" > $F
( time MLB_FUZZ_CASES=20000 timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -n 4 ) 2>&1 | grep -E "passed|failed|^real" >> $F
echo "# MLB_FUZZ_SCALE=big MLB_FUZZ_CASES=3000 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -n 4" >> $F
( time MLB_FUZZ_SCALE=big MLB_FUZZ_CASES=3000 timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -n 4 ) 2>&1 | grep -E "passed|failed|^real" >> $F
cat $F
