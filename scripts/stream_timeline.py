"""Dev tool (needs the -DMLRA_DEV_TRACE build via MLRA_LIB): per-CTA timeline of a
chained up -> down forward at cfg2 shapes: the up GEMM's CTAs (MLRA_TRACE2: entry,
epilogue done) and the down layer's row product CTAs (MLRA_TRACE3: entry, PDL wait
passed, main loop done, exit), on one globaltimer clock.
   python scripts/stream_timeline.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2309_16119_b200 import modulora as M
from scripts.sweep import layers_for

m = 4096
up, down = layers_for([(11008, 4096), (4096, 11008)], 3, 16, M.MaterializationStrategy.RowMaterialize)
x = torch.randn(m, 4096, device="cuda").to(torch.bfloat16)
g = torch.zeros(2048 * 8, dtype=torch.int64, device="cuda")
t3 = torch.zeros(2048 * 8, dtype=torch.int64, device="cuda")
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(3):
    h, _ = M.layer_forward(up, x)
    M.layer_forward(down, h)
torch.cuda.synchronize()
flush.zero_()
os.environ["MLRA_TRACE2"] = str(g.data_ptr())
h, _ = M.layer_forward(up, x)
del os.environ["MLRA_TRACE2"]
os.environ["MLRA_TRACE3"] = str(t3.data_ptr())
M.layer_forward(down, h)
del os.environ["MLRA_TRACE3"]
torch.cuda.synchronize()
G = g.view(2048, 8).cpu().numpy().astype(np.float64)
G = G[G[:, 0] > 0]
T = t3.view(2048, 8).cpu().numpy().astype(np.float64)
T = T[T[:, 0] > 0]
t0 = G[:, 0].min()
us = lambda a: (a - t0) / 1e3
print(f"up GEMM: {len(G)} CTAs; epilogue done min {us(G[:, 4]).min():.1f} med {np.median(us(G[:, 4])):.1f} "
      f"max {us(G[:, 4]).max():.1f} us")
print(f"down row product: {len(T)} CTAs")
for c, nm in ((0, "entry"), (1, "pdl passed"), (2, "loop done"), (3, "exit")):
    v = us(T[:, c])
    print(f"  {nm:13s} min {v.min():7.1f} p25 {np.percentile(v, 25):7.1f} med {np.median(v):7.1f} "
          f"p75 {np.percentile(v, 75):7.1f} max {v.max():7.1f}")
started_early = (T[:, 0] < G[:, 4].max()).sum()
print(f"  CTAs entered before the GEMM's last epilogue finished: {started_early}")
