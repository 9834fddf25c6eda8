#!/bin/bash
# Round-2 GPU pass: parity tests, smoke, both bench arms, the bench's ncu launch
# list, full ncu captures of the sweep kernel and of the single-graph kernels
# (PARALL C4 and C1, levelled C4-SEQFIX / C2 / C3).
# Usage (under gpurun, from the repo root): bash tools/gpu_round2.sh <tag>
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1; lscpu > $OUT/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 > $OUT/launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep_ws -c 1 \
    -o $OUT/sweep_ws python tools/sweep_probe.py 1024 1 > $OUT/ncu_sweep.log 2>&1
for c in C4-PARALL C1 C4-SEQFIX C2 C3; do
  bash tools/ncu_c4.sh $TAG $c
done
timeout 300 bash -c 'for c in C4-PARALL C1 C4-SEQFIX C2 C3; do python tools/time_probe.py $c 20 2>&1 | tail -1; done' > $OUT/times.txt 2>&1
ls -la $OUT
tail -2 $OUT/pytest_gpu.log; cat $OUT/smoke.log | tail -2
