OUT=gpurun_out/r2b; mkdir -p $OUT
for c in C4-SEQFIX C2 C3 C1 C4-PARALL; do python tools/time_probe.py $c 20; done > $OUT/times.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
cat $OUT/times.txt; tail -3 $OUT/pytest_gpu.log
