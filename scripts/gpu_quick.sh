#!/bin/bash
# Quick GPU session: smoke, GPU tests, the transform-path sweep (K11 variants), bench.
# Usage (on the box): bash scripts/gpu_quick.sh <tag>   env: SKIP_TESTS=1 SKIP_BENCH=1 SWEEP="C3 C4" BENCH_ARGS=
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 300 python __graft_entry__.py --smoke > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
  timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $OUT/gpu_tests.log 2>&1; echo "pytest exit $?" >> $OUT/gpu_tests.log
fi
for C in ${SWEEP:-C3}; do
  timeout 300 python scripts/sweep_ntt.py $C ${SWEEP_B:-4096} >> $OUT/sweep.jsonl 2>> $OUT/sweep.err
done
if [ -z "$SKIP_BENCH" ]; then
  timeout 900 python bench.py $BENCH_ARGS > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
fi
echo done > $OUT/DONE
