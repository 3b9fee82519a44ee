#!/bin/bash
# Round profile capture (run under gpurun, ONE GPU): launch list of the bench
# command + one `--set full` capture per dominant kernel.  Outputs in gpurun_out/;
# tools/profile_collect.py turns them into the tracked summaries under profiles/.
set -u
OUT=gpurun_out
mkdir -p $OUT
NCU="ncu --clock-control none"
python -c "from paper_2409_16781_b200 import _cabi; print(_cabi.build_id())" > $OUT/build_id.txt
# launch list of the same command bench.py is judged on (shares, not absolutes)
$NCU --metrics gpu__time_duration.sum -c 200 --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extra > $OUT/launches_bench.log 2>&1
# launch list of the slab driver with the fused peer-store exchange (world 1, one-call loop)
$NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $OUT/launches_slab.csv \
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --force-slab --no-preflight > $OUT/launches_slab.log 2>&1
cap() {  # name, kernel regex, command...
  local name=$1 regex=$2; shift 2
  $NCU --set full --import-source on -k regex:$regex -s 2 -c 1 -f -o $OUT/$name "$@" > /dev/null 2>&1
  python tools/ncu_summary.py $OUT/$name.ncu-rep > $OUT/ncu_$name.txt 2>&1
  [ "$name" != step_f32_512 ] && rm -f $OUT/$name.ncu-rep
  head -3 $OUT/ncu_$name.txt
}
# full captures: fused kernel in the four storage modes, the in-place pair in each, the staged kernel
for pt in single:f32 double:f64 mixed1:f16 mixed2:m2; do
  p=${pt%%:*}; t=${pt##*:}
  cap step_${t}_512 step_ python tools/one.py 512x512x512 $p 0 4
  cap aa_pull_${t}_512 aa_pull python tools/aa_one.py $p
  cap aa_local_${t}_512 aa_local python tools/aa_one.py $p
done
cap stage_f16_512 step_stage python tools/one.py 512x512x512 mixed1 4000 4
cap aa_pull_rowb_f32_512 aa_pull python tools/aa_one.py single 1
# diagnostics (pack form): tools/diag_time.py launches the kernel 6 times per storage type, fp32 / fp64 / fp16 in turn
cap_s() { local s=$1 name=$2 regex=$3; shift 3; $NCU --set full --import-source on -k regex:$regex -s $s -c 1 -f -o $OUT/$name "$@" > /dev/null 2>&1; python tools/ncu_summary.py $OUT/$name.ncu-rep > $OUT/ncu_$name.txt 2>&1; rm -f $OUT/$name.ncu-rep; head -3 $OUT/ncu_$name.txt; }
cap_s 1 diag_f32_512 diag_vec_kernel python tools/diag_time.py 512
cap_s 7 diag_f64_512 diag_vec_kernel python tools/diag_time.py 512
cap_s 13 diag_f16_512 diag_vec_kernel python tools/diag_time.py 512
ls -la $OUT
