OUT=gpurun_out/r2c; mkdir -p $OUT
for c in C4-SEQFIX C2; do python tools/level_trace.py $c; done > $OUT/trace.txt 2>&1
cat $OUT/trace.txt
