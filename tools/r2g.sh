# lbp_pslot variants: bash tools/r2g.sh v1 v2 ...
for v in "$@"; do
  for c in C4-PARALL C1; do
    echo -n "$v "; HBP_LIB_PATH=tools/variants/$v.so timeout 300 python tools/time_probe.py $c 20 2>&1 | tail -1
  done
done
