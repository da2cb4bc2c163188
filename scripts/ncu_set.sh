#!/bin/bash
# Several single-kernel ncu --set full captures in one session, exported to CSV.
# Usage (on the box): bash scripts/ncu_set.sh <tag> "<name>|<kernel-regex>|<skip>|<env>|<cmd>" ...
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for spec in "$@"; do
  IFS='|' read -r NAME K S ENVS CMD <<< "$spec"
  env $ENVS $CMD > $OUT/plain_$NAME.log 2>&1 || { echo "plain run failed" >> $OUT/plain_$NAME.log; continue; }
  env $ENVS timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$K" -s $S -c 1 \
      -o $OUT/prof_$NAME $CMD > $OUT/ncu_$NAME.log 2>&1
  ncu -i $OUT/prof_$NAME.ncu-rep --page raw --csv > $OUT/raw_$NAME.csv 2>/dev/null
  ncu -i $OUT/prof_$NAME.ncu-rep --page details --csv > $OUT/details_$NAME.csv 2>/dev/null
  ncu -i $OUT/prof_$NAME.ncu-rep --page source --csv > $OUT/source_$NAME.csv 2>/dev/null; gzip -f $OUT/source_$NAME.csv
  [ -n "$KEEP_REP" ] || rm -f $OUT/prof_$NAME.ncu-rep
done
echo done > $OUT/DONE
