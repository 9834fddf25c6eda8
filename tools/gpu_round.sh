#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench, ncu launch list + one full capture.
# Usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tag]
set -x
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python tools/time_probe.py C4-PARALL 5 > $OUT/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lbp_persistent -s 3 -c 1 \
    -o $OUT/c4_parall python tools/time_probe.py C4-PARALL 2 > $OUT/ncu_full.log 2>&1
ls -la $OUT
