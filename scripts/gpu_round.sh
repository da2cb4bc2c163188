#!/bin/bash
# One gpurun session: smoke, GPU tests, the default bench, then the ncu launch
# list and one `ncu --set full` capture per hot kernel (every ncu command runs
# only after the identical plain command exited 0).  Reports are exported to
# CSV on the box and the .ncu-rep files dropped if the total nears gpurun's
# 64 MiB copy-back cap.  Usage (on the box):
#   bash scripts/gpu_round.sh <tag> [kernel ...]
# env: SKIP_TESTS=1, SKIP_NCU=1, SKIP_LAUNCHES=1, BENCH_ARGS="...", NCU_ARGS="..."
TAG=${1:-r01}; shift
KERNELS=${@:-zinc_coeff_kernel encode_real_kernel zinc_ntt_split vanilla_ntt_dit vanilla_coeff_split decrypt_split encode_kernel}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  python __graft_entry__.py --smoke > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "pytest exit $?" >> $OUT/gpu_tests.log
fi
timeout 900 python bench.py $BENCH_ARGS > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
if [ -z "$SKIP_NCU" ]; then
  SMALL="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 --no-oracle-suite $BENCH_ARGS"
  timeout 600 $SMALL > $OUT/plain.log 2>&1; RC=$?; echo "plain exit $RC" >> $OUT/plain.log
  if [ $RC -eq 0 ]; then
    if [ -z "$SKIP_LAUNCHES" ]; then
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
          --log-file $OUT/launches.csv $SMALL > $OUT/ncu_launches.log 2>&1
      gzip -f $OUT/launches.csv
    fi
    for K in $KERNELS; do
      timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^$K" -s 8 -c 1 \
          $NCU_ARGS -o $OUT/prof_$K $SMALL > $OUT/ncu_full_$K.log 2>&1
      if [ -f $OUT/prof_$K.ncu-rep ]; then
        ncu -i $OUT/prof_$K.ncu-rep --page raw --csv > $OUT/raw_$K.csv 2>/dev/null
        ncu -i $OUT/prof_$K.ncu-rep --page details --csv > $OUT/details_$K.csv 2>/dev/null
        ncu -i $OUT/prof_$K.ncu-rep --page source --csv > $OUT/source_$K.csv 2>/dev/null
        gzip -f $OUT/source_$K.csv
      fi
    done
  fi
fi
du -sb $OUT/* | sort -n > $OUT/sizes.txt
TOTAL=$(du -sb gpurun_out | cut -f1)
if [ $TOTAL -gt 55000000 ]; then
  for f in $(ls -S $OUT/*.ncu-rep 2>/dev/null); do
    rm -f $f; echo "dropped $f" >> $OUT/sizes.txt
    [ $(du -sb gpurun_out | cut -f1) -lt 55000000 ] && break
  done
fi
echo done > $OUT/DONE
