#!/bin/bash
# Race / sync / memory checks of the in-place kernels, the z-slab drivers (peer stores across
# processes), the staged kernel and the fuzz suite on small grids (run under gpurun, ONE GPU).
# compute-sanitizer's racecheck looks at shared-memory hazards (the staged kernel, the
# diagnostics reductions); races through GLOBAL memory - the in-place exclusive-writer
# argument, peer stores - are what the bitwise parity of these very tests checks.
set -u
OUT=gpurun_out; mkdir -p $OUT
CS="compute-sanitizer --target-processes all --error-exitcode 9"
run() {  # tool, tag, timeout, pytest args...
  local tool=$1 tag=$2 lim=$3; shift 3
  local f=$OUT/sanitizer_${tool}_${tag}.txt
  echo "# $CS --tool $tool python -m pytest $* -m gpu -q -x" > $f
  ( time timeout $lim $CS --tool $tool python -m pytest "$@" -m gpu -q -x ) > $f.full 2>&1
  echo "# exit code $?" >> $f
  grep -E "passed|failed|error|ERROR SUMMARY|RACECHECK SUMMARY|hazard|real" $f.full | sort | uniq -c | sort -rn | head -40 >> $f
  tail -3 $f
}
export MLB_FUZZ_CASES=200
run racecheck inplace_slabs 1500 tests/test_gpu_inplace.py tests/test_gpu_slabs.py
run racecheck peer_ring 1500 tests/test_gpu_peer_ring.py
run racecheck fuzz_staged 1500 tests/test_gpu_fuzz.py tests/test_gpu_parity.py -k "random_case or staged or macro or graph"
run synccheck inplace_slabs 1200 tests/test_gpu_inplace.py tests/test_gpu_slabs.py
run synccheck peer_ring 1200 tests/test_gpu_peer_ring.py
run synccheck fuzz_staged 1200 tests/test_gpu_fuzz.py tests/test_gpu_parity.py -k "random_case or staged or macro or graph"
run memcheck new_paths 1500 tests/test_gpu_parity.py tests/test_gpu_acceptance.py -k "staged or no_pack_divides or graph or overlapped or resident"
ls -la $OUT
