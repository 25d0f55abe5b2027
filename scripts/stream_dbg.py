"""Dev: does the down layer's row product stream the up GEMM's tiles (MLRA_DEBUG_STREAM=1)?"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2309_16119_b200 import modulora as M


class A:
    workload, bits, scaling = "cfg2", 0, "weak"


w = bench.workload(A())
wl = bench.Workload(w, 4096, M.parse_strategy("row"), torch.device("cuda", 0), 0)
for _ in range(2):
    wl.step(wl.xs, wl.dys, comm=False)
torch.cuda.synchronize()
print("done", file=sys.stderr)
