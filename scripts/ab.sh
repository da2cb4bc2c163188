# A/B on the box: sweep_ntt with the new library and with scripts/base.so.
# usage: bash scripts/ab.sh <tag> <config> <batch> [<config> <batch> ...]
TAG=$1; shift
mkdir -p gpurun_out/$TAG
cp paper_2408_07304_b200/libzinc.so /tmp/new.so
while [ $# -gt 1 ]; do
  C=$1; B=$2; shift 2
  cp /tmp/new.so paper_2408_07304_b200/libzinc.so
  python scripts/sweep_ntt.py $C $B > gpurun_out/$TAG/new_$C.json 2>&1
  cp scripts/base.so paper_2408_07304_b200/libzinc.so
  python scripts/sweep_ntt.py $C $B > gpurun_out/$TAG/base_$C.json 2>&1
done
cp /tmp/new.so paper_2408_07304_b200/libzinc.so
