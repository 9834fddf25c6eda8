# lbp_pslot A/B + parity: bash tools/r2f.sh
OUT=gpurun_out/r2f; mkdir -p $OUT
for c in C4-PARALL C1; do
  timeout 300 python tools/time_probe.py $c 20 2>&1 | tail -1
  HBP_PSLOT=0 timeout 300 python tools/time_probe.py $c 20 2>&1 | tail -1
done
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
