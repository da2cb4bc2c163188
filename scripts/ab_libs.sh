# A/B of several builds of the library on the box: sweep_ntt per library (ZINC_LIB_PATH), two
# alternating rounds.  usage: bash scripts/ab_libs.sh <tag> "<lib> ..." <config> <batch> [<config> <batch> ...]
TAG=$1; LIBS=$2; shift 2
mkdir -p gpurun_out/$TAG
while [ $# -gt 1 ]; do
  C=$1; B=$2; shift 2
  for R in 1 2; do
    for L in $LIBS; do
      ZINC_LIB_PATH=$PWD/$L python scripts/sweep_ntt.py $C $B > gpurun_out/$TAG/$(basename $L .so)_${C}_$R.json 2>&1
    done
  done
done
