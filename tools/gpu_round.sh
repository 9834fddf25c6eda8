#!/bin/bash
# One GPU-box pass: parity tests, smoke, both bench arms, ncu launch list of the
# bench command + one full capture of the sweep kernel.
# Usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tag]
set -x
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 > $OUT/launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep_ws -c 1 \
    -o $OUT/sweep_ws python tools/sweep_probe.py 1024 1 > $OUT/ncu_full.log 2>&1
ls -la $OUT
