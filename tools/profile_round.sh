#!/bin/bash
# Round profile capture (run under gpurun, ONE GPU): launch list of the bench
# command + one `--set full` capture per dominant kernel.  Outputs in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
NCU="ncu --clock-control none"
# launch list of the same command bench.py is judged on (shares, not absolutes)
$NCU --metrics gpu__time_duration.sum -c 80 --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/launches_bench.log 2>&1
# launch list of the slab driver with the fused peer-store exchange (world 1)
$NCU --metrics gpu__time_duration.sum -c 120 --csv --log-file $OUT/launches_slab.csv \
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --force-slab > $OUT/launches_slab.log 2>&1
# full captures: fused kernel in the three storage modes, in-place pair
$NCU --set full --import-source on -k regex:step_ -s 2 -c 1 -f -o $OUT/step_f32_512 python tools/one.py 512x512x512 single 0 4 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:step_ -s 2 -c 1 -f -o $OUT/step_f64_512 python tools/one.py 512x512x512 double 0 4 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:step_ -s 2 -c 1 -f -o $OUT/step_f16_512 python tools/one.py 512x512x512 mixed1 0 4 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:aa_pull -s 2 -c 1 -f -o $OUT/aa_pull_f32_512 python tools/aa_one.py > /dev/null 2>&1
$NCU --set full --import-source on -k regex:aa_local -s 2 -c 1 -f -o $OUT/aa_local_f32_512 python tools/aa_one.py > /dev/null 2>&1
# summarise on the box (gpurun_out/ travels back only under 64 MiB); keep one report
for r in step_f32_512 step_f64_512 step_f16_512 aa_pull_f32_512 aa_local_f32_512; do
    python tools/ncu_summary.py $OUT/$r.ncu-rep > $OUT/ncu_$r.txt 2>&1
    [ "$r" != step_f32_512 ] && rm -f $OUT/$r.ncu-rep
done
ls -la $OUT
