import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import bench, synth
class A: steps=1; list_cap=12
r = bench.bench_pathtrace(A(), 0)
print(r["ms_per_frame"])
