OUT=gpurun_out/r2a; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1; lscpu > $OUT/lscpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
tail -3 $OUT/pytest_gpu.log; cat $OUT/smoke.log; cat $OUT/bench.json $OUT/bench_ref.json | cut -c1-3000
