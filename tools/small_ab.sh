# HBP_SMALL (level size below which a level runs on the small-level CTAs) A/B: bash tools/small_ab.sh <reps> v1 v2 ...
N=$1; shift
for pass in 1 2; do
  for v in "$@"; do
    for c in C2 C3 C4-SEQFIX; do
      echo -n "small=$v "; HBP_SMALL=$v timeout 300 python tools/time_probe.py $c $N 2>&1 | tail -1
    done
  done
done
