#!/bin/bash
# ncu --set full of one kernel launched by a short command, exported to CSV.
# Usage (on the box): bash scripts/ncu_one.sh <tag> <kernel-regex> <skip> <cmd...>
TAG=$1; K=$2; S=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
"$@" > $OUT/plain_$K.log 2>&1 || { echo "plain run failed" >> $OUT/plain_$K.log; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:^$K" -s $S -c 1 -o $OUT/prof_$K "$@" > $OUT/ncu_$K.log 2>&1
ncu -i $OUT/prof_$K.ncu-rep --page raw --csv > $OUT/raw_$K.csv 2>/dev/null
ncu -i $OUT/prof_$K.ncu-rep --page details --csv > $OUT/details_$K.csv 2>/dev/null
ncu -i $OUT/prof_$K.ncu-rep --page source --csv > $OUT/source_$K.csv 2>/dev/null; gzip -f $OUT/source_$K.csv
rm -f $OUT/prof_$K.ncu-rep
