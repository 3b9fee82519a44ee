#!/bin/bash
# one `--set full` capture of a kernel: tools/ncu_one.sh <name> <kernel regex> <skip> -- <command...>
# leaves gpurun_out/ncu_<name>.txt (summary) and gpurun_out/<name>.ncu-rep
set -u
NAME=$1; REGEX=$2; SKIP=$3; shift 4
OUT=gpurun_out; mkdir -p $OUT
ncu --clock-control none --set full --import-source on -k regex:$REGEX -s $SKIP -c 1 -f -o $OUT/$NAME "$@" > $OUT/ncu_$NAME.log 2>&1
python tools/ncu_summary.py $OUT/$NAME.ncu-rep > $OUT/ncu_$NAME.txt 2>&1
cat $OUT/ncu_$NAME.txt
