set -u
OUT=gpurun_out; mkdir -p $OUT
CS="compute-sanitizer --target-processes all --error-exitcode 9"
for tool in memcheck racecheck; do
  f=$OUT/sanitizer_${tool}_diagnostics.txt
  echo "# $CS --tool $tool python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x -k 'nonfinite or diagnostics'   (library build $(python -c 'from paper_2409_16781_b200 import _cabi; print(_cabi.build_id())'))" > $f
  ( time timeout 900 $CS --tool $tool python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x -k "nonfinite or diagnostics" ) > $f.full 2>&1
  echo "# exit code $?" >> $f
  grep -E "passed|failed|error|ERROR SUMMARY|RACECHECK SUMMARY|hazard|real" $f.full | sort | uniq -c | sort -rn | head -20 >> $f
  cat $f
done
F=$OUT/fuzz_final.txt
echo "# MLB_FUZZ_CASES=20000 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -n 4   (one B200, round 2, final library build)" > $F
( time MLB_FUZZ_CASES=20000 timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -n 4 ) 2>&1 | grep -E "passed|failed|^real" >> $F
echo "# MLB_FUZZ_SCALE=big MLB_FUZZ_CASES=3000 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -n 4" >> $F
( time MLB_FUZZ_SCALE=big MLB_FUZZ_CASES=3000 timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -n 4 ) 2>&1 | grep -E "passed|failed|^real" >> $F
cat $F
