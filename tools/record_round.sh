#!/bin/bash
# Round record (run under gpurun, ONE GPU): GPU tests, smoke and every bench line
# quoted in DESIGN.md, into gpurun_out/ (copied to profiles/ afterwards).
set -u
OUT=gpurun_out
mkdir -p $OUT
(time timeout 2400 python -m pytest tests -q -m gpu) > $OUT/gpu_tests_final.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
R=$OUT/bench_record.txt
: > $R
run() { echo "# python bench.py $*" >> $R; python bench.py "$@" 2>>$OUT/bench_record.err | tail -1 >> $R; echo >> $R; }
echo "# python bench.py --steps 20 --warmup 5   (what the driver runs), one B200, round 2" >> $R
( time python bench.py --steps 20 --warmup 5 ) 2>&1 | grep -v "^$\|user\|sys" >> $R; echo >> $R
echo "# python bench.py   (defaults: N=1, K=1000, W=5)" >> $R
( time python bench.py --no-extra ) 2>&1 | grep -v "^$\|user\|sys" >> $R; echo >> $R
run --steps 200 --no-cpu-baseline --no-extra
run --precision double --steps 300 --no-cpu-baseline
run --precision mixed1 --steps 500 --no-cpu-baseline
run --precision mixed2 --steps 300 --no-cpu-baseline
run --inplace --steps 500 --no-cpu-baseline --no-extra
run --force-slab --steps 200 --no-cpu-baseline --no-e2e
run --force-slab --steps 200 --no-cpu-baseline --no-e2e --python-loop --no-preflight
run --impl reference --steps 10 --warmup 2
echo "# torchrun 2 ranks sharing the GPU (debug path: peer ring across processes, preflight)" >> $R
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 50 --warmup 3 --share-gpu --edge 256 --no-cpu-baseline 2>>$OUT/bench_record.err | tail -1 >> $R; echo >> $R
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 4 --steps 50 --warmup 3 --share-gpu --edge 256 --scaling strong --no-cpu-baseline --no-e2e 2>>$OUT/bench_record.err | tail -1 >> $R; echo >> $R
for n in 512 256 511; do
  echo "# python tools/quick.py $n  (device-only, default kernels, two-buffer and in-place)" >> $R
  python tools/quick.py $n $((n == 256 ? 400 : 100)) >> $R 2>&1
done
echo "# python tools/small_domains.py 2048" >> $R
python tools/small_domains.py 2048 >> $R 2>&1
echo "# python tools/e2e_host.py 512 20" >> $R
python tools/e2e_host.py 512 20 >> $R 2>&1
echo "# python tools/chan_one.py  (configs[4] geometry on one GPU)" >> $R
python tools/chan_one.py >> $R 2>&1
tail -3 $OUT/gpu_tests_final.log; cat $OUT/smoke.log; cut -c1-220 $R
