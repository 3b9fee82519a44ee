#!/bin/bash
# bench.py's guarded preflight on a one-GPU box (run under gpurun): two ranks sharing the GPU,
# (1) the normal path, (2) a forced failure of the peer ring (MLB_PREFLIGHT_FAIL=peer): the bench
# must fall back to the send/recv transport - which the gloo control plane of --share-gpu cannot
# carry for CUDA tensors, so HERE it ends in "bench preflight failed" (on a multi-GPU box NCCL
# carries it) - and (3) one rank with the z-slab driver.
set -u
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
echo "== 2 ranks, peer ring"
timeout 600 $TR --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --share-gpu --edge 256 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-300
echo "== 2 ranks, forced peer failure"
MLB_PREFLIGHT_FAIL=peer timeout 600 $TR --master-port 29521 bench.py --gpus 2 --steps 20 --warmup 3 --share-gpu --edge 256 --no-cpu-baseline --no-e2e 2>&1 | grep "preflight" | head -3
echo "== 1 rank, z-slab driver"
python bench.py --steps 20 --warmup 3 --force-slab --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-300
