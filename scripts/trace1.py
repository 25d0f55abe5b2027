"""Dev tool: 1-CTA fused GEMM per-CTA cycle breakdown (MLRA_TRACE2):
   python scripts/trace1.py D_OUT D_IN BITS M [fwd|dx]   (MLRA_GEMM=1|3 selects the tile)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer

d_out, d_in, bits, m = (int(v) for v in sys.argv[1:5])
op = sys.argv[5] if len(sys.argv) > 5 else "fwd"
strat = M.MaterializationStrategy.RowMaterialize
layer = make_layer(d_out, d_in, bits, 16, strat)
ctx = M.LpLinearContext(layer.weights, strat)
a = torch.randn(m, d_in if op == "fwd" else d_out, device="cuda").to(torch.bfloat16)
f = M.lp_forward if op == "fwd" else M.lp_backward
buf = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    f(ctx, a)
torch.cuda.synchronize()
os.environ["MLRA_TRACE2"] = str(buf.data_ptr())
f(ctx, a)
torch.cuda.synchronize()
del os.environ["MLRA_TRACE2"]
t = buf.view(148, 8).cpu().numpy().astype(np.float64)
t = t[t[:, 0] > 0]
kb = (d_in if op == "fwd" else d_out) // 64
print(f"{len(t)} CTAs, {kb} k-blocks per tile; per k-block cycles (median over CTAs):")
names = ["total", "mma_wait_full", "g0_wait_q", "g0_wait_empty", "g0_compute", "g1_wait_q",
         "g1_wait_empty", "g1_compute"]
for k, nm in enumerate(names):
    div = kb if k < 2 else kb / 2
    print(f"  {nm:14s} {np.median(t[:, k]) / div:8.1f}")
