# A/B on the box: GPU tests with the new library, then sweep_ntt with new and base (scripts/base.so)
mkdir -p gpurun_out/$1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/$1/gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/$1/gpu_tests.log
python scripts/sweep_ntt.py C3 4096 > gpurun_out/$1/new.json 2>&1
cp paper_2408_07304_b200/libzinc.so /tmp/new.so; cp scripts/base.so paper_2408_07304_b200/libzinc.so
python scripts/sweep_ntt.py C3 4096 > gpurun_out/$1/base.json 2>&1
cp /tmp/new.so paper_2408_07304_b200/libzinc.so
