OUT=gpurun_out/r2e; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 > $OUT/bench_g2.json 2> $OUT/bench_g2.err; echo "rc=$?" >> $OUT/bench_g2.err
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -3 $OUT/pytest_gpu.log; head -c 1500 $OUT/bench_g2.json; tail -3 $OUT/bench_g2.err; head -c 600 $OUT/bench.json
