#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
( time timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fuzz.py ) > $OUT/tests_all.log 2>&1
( time python bench.py --steps 20 --warmup 5 --no-extra ) > $OUT/bench20.log 2>&1
( time python bench.py --steps 200 --warmup 5 --no-extra --no-cpu-baseline ) > $OUT/bench200.log 2>&1
( time timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --share-gpu --edge 256 --no-cpu-baseline ) > $OUT/bench_share2.log 2>&1
tail -5 $OUT/tests_all.log; tail -c 2500 $OUT/bench20.log; tail -c 1200 $OUT/bench200.log;  tail -c 1500 $OUT/bench_share2.log
