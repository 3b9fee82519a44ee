#!/bin/bash
# first GPU contact of round 2: box facts, smoke, the new tests, bench, small domains, 2 ranks on one GPU
set -u
OUT=gpurun_out
mkdir -p $OUT
( free -g; nproc; nvidia-smi -L; nvidia-smi --query-gpu=memory.total,memory.used --format=csv ) > $OUT/box.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
( time timeout 1500 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_peer_ring.py tests/test_gpu_parity.py::test_graph_replay_never_changes_bits tests/test_gpu_scale.py tests/test_cabi.py -m gpu -x -q ) > $OUT/tests_new.log 2>&1
( time python bench.py --steps 20 --warmup 5 ) > $OUT/bench20.log 2>&1
python tools/small_domains.py 2048 > $OUT/small_domains.txt 2>&1
( time timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --share-gpu --edge 256 --no-cpu-baseline ) > $OUT/bench_share2.log 2>&1
( time timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 20 --warmup 3 --share-gpu --edge 256 --no-cpu-baseline --python-loop --no-preflight --no-e2e ) > $OUT/bench_share2_py.log 2>&1
tail -3 $OUT/smoke.log; tail -5 $OUT/tests_new.log; tail -c 1500 $OUT/bench20.log; cat $OUT/small_domains.txt; tail -c 800 $OUT/bench_share2.log; tail -c 600 $OUT/bench_share2_py.log
