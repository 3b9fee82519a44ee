#!/bin/bash
# memcheck + racecheck of the HOST layer's random call sequences (engine.run / step / sessions /
# overlapped host run / checkpoints / host edits / probes) and of engine.run under a process group
# (run under gpurun, ONE GPU).  Same conventions as tools/sanitize_round.sh.
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
export MLB_FUZZ_CASES=1 MLB_ENGINE_FUZZ_CASES=${MLB_ENGINE_FUZZ_CASES:-150} MLB_RING_CASES=${MLB_RING_CASES:-12}
run memcheck engine_sequences 1500 tests/test_gpu_fuzz.py tests/test_gpu_acceptance.py -k "engine_sequences or chained or hook or resident"
run racecheck engine_sequences 1500 tests/test_gpu_fuzz.py -k "engine_sequences"
run memcheck engine_ranks 1500 tests/test_gpu_peer_ring.py -k "engine_run_random or chained"
