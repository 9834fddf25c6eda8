# single-graph variants: bash tools/r2p.sh <reps> v1 v2 ... (C4-PARALL and C1, interleaved twice)
N=$1; shift
for pass in 1 2; do
  for v in "$@"; do
    for c in C4-PARALL C1; do
      echo -n "$v "; HBP_LIB_PATH=tools/variants/$v.so timeout 300 python tools/time_probe.py $c $N 2>&1 | tail -1
    done
  done
done
