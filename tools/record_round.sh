#!/bin/bash
# Round record (run under gpurun, ONE GPU): GPU tests, memcheck, smoke and every
# bench line quoted in DESIGN.md, into gpurun_out/ (copied to profiles/ afterwards).
set -u
OUT=gpurun_out
mkdir -p $OUT
(time timeout 1500 python -m pytest tests -x -q -m gpu) > $OUT/gpu_tests_final.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
R=$OUT/bench_record.txt
: > $R
run() { echo "# python bench.py $*" >> $R; python bench.py "$@" 2>>$OUT/bench_record.err | tail -1 >> $R; echo >> $R; }
echo "# python bench.py  (defaults: N=1, K=1000, W=5), one B200, round 1" >> $R
( time python bench.py ) 2>&1 | grep -v "^$\|user\|sys" >> $R; echo >> $R
run --steps 200 --no-cpu-baseline
run --precision double --steps 300 --no-cpu-baseline
run --precision mixed1 --steps 500 --no-cpu-baseline
run --precision mixed2 --steps 300 --no-cpu-baseline
run --inplace --steps 500 --no-cpu-baseline
run --force-slab --steps 200 --no-cpu-baseline --no-e2e
run --impl reference --steps 10 --warmup 2
echo "# python tools/quick.py 512 100  (device-only, default kernels, two-buffer and in-place)" >> $R
python tools/quick.py 512 100 >> $R 2>&1
echo "# python tools/quick.py 256 400" >> $R
python tools/quick.py 256 400 >> $R 2>&1
echo "# python tools/quick.py 511 100  (rows that no pack divides: one cell per thread)" >> $R
python tools/quick.py 511 100 >> $R 2>&1
echo "# python tools/chan_one.py  (configs[4] geometry on one GPU)" >> $R
python tools/chan_one.py >> $R 2>&1
( echo "# compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_inplace.py tests/test_gpu_slabs.py -m gpu -x -q  (one B200, round 1)"; timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_inplace.py tests/test_gpu_slabs.py -m gpu -x -q 2>&1 | tail -6 ) > $OUT/sanitizer_memcheck.txt
tail -3 $OUT/gpu_tests_final.log; cat $OUT/smoke.log; cut -c1-200 $R
