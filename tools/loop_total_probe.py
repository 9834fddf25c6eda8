"""Scratch probe (GPU box): the bench's interaction-loop leg alone."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2509_22337_b200 import workloads as W
g, alarms = W.graph("ftp")
r = bench.measure_loop(g, alarms, os.cpu_count() or 1)
print("loop rounds", r["rounds"], "total_s", r["total_s"], "ms/round", r["ms_per_round"])
