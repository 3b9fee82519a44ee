#!/bin/bash
set -u
OUT=gpurun_out
( time timeout 2400 python -m pytest tests/test_gpu_inplace.py tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_peer_ring.py tests/test_gpu_fuzz.py tests/test_gpu_acceptance.py -m gpu -q -x ) > $OUT/tests_r7.log 2>&1
tail -6 $OUT/tests_r7.log
for rb in 0 1; do for n in 512 256; do
  echo "MLB_AA_ROWB=$rb n=$n"
  MLB_AA_ROWB=$rb python tools/quick.py $n $((n == 256 ? 400 : 100)) 2>&1 | grep inplace
done; done | tee $OUT/rowb.txt
echo "ragged in place 511"; python tools/quick.py 511 100 2>&1 | grep inplace | tee -a $OUT/rowb.txt
( time python bench.py --steps 20 --warmup 5 --no-extra --no-cpu-baseline ) 2>&1 | tail -c 900
