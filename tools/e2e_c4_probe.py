"""Probe (GPU box): the bench single-graph C4-PARALL leg (device time and fresh-graph run() e2e)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, bench
r = bench.measure_single(torch, "C4-PARALL", steps=10, warmup=3)
print("e2e ms", r["e2e"]["ms_per_step"], "device ms", r["time_to_convergence_ms"], flush=True)
