# levelled-config variants: bash tools/lev_ab.sh <reps> v1 v2 ... (C2, C3, C4-SEQFIX, interleaved twice)
N=$1; shift
for pass in 1 2; do
  for v in "$@"; do
    for c in C2 C3 C4-SEQFIX; do
      echo -n "$v "; HBP_LIB_PATH=tools/variants/$v.so timeout 300 python tools/time_probe.py $c $N 2>&1 | tail -1
    done
  done
done
