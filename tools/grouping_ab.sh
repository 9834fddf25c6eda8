#!/bin/bash
# A/B of the message grouping (SURVEY.md 8(d) / north star: warp efficiency and
# branch divergence before and after grouping): C4 ftp PARALL with
# HBP_GROUPING = 2 (whole degree-sorted nodes, default), 1 (one slot per thread,
# degree-sorted), 0 (one slot per thread, EdgeId order). Timing, bitwise parity
# against the golden run, and one ncu launch each.
OUT=gpurun_out/grouping
mkdir -p $OUT
M=gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__sass_average_branch_targets_threads_uniform.pct,smsp__sass_branch_targets_threads_divergent.sum,smsp__sass_inst_executed.sum,lts__t_sectors.sum,sm__warps_active.avg.pct_of_peak_sustained_active
for G in 2 1 0; do
  [ "$1" = ncu ] && { HBP_GROUPING=$G ncu --metrics $M --clock-control none -c 60 --csv python tools/time_probe.py C4-PARALL 3 > $OUT/ncu_$G.csv 2>&1; continue; }
  HBP_GROUPING=$G python tools/time_probe.py C4-PARALL 30 > $OUT/time_$G.txt 2>&1
  HBP_GROUPING=$G python -m pytest tests/test_gpu_parity.py -q -k "baseline_bitwise and C4-PARALL or baseline_bitwise and C1" > $OUT/parity_$G.txt 2>&1
  HBP_GROUPING=$G ncu --metrics $M --clock-control none -c 60 --csv \
      python tools/time_probe.py C4-PARALL 3 > $OUT/ncu_$G.csv 2>&1
done
tail -n 2 $OUT/time_*.txt $OUT/parity_*.txt
