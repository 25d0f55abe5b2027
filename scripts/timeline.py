"""Dev tool: per-CTA timeline of one pair-kernel launch (MLRA_TRACE2):
   python scripts/timeline.py D_OUT D_IN BITS M [fwd|dx]   (env MLRA_SK etc. apply)"""
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
used = t[:, 0] > 0
t0 = t[used, 0].min()
rel = np.where(t > 0, (t - t0) / 1e3, np.nan)[used]
names = ["entry", "mma_done", "last_tfull", "flags_seen", "epi_done", "drained", "published", "chunk0_landed"]
print(f"{used.sum()} CTAs; times in us from the first entry")
for k, nm in enumerate(names):
    col = rel[:, k]
    col = col[~np.isnan(col)]
    if col.size:
        print(f"  {nm:11s} min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f}  (n={col.size})")
lead = rel[::2]
print("per pair (leader): entry mma_done last_tfull flags_seen epi_done")
for i in range(0, min(len(lead), 74), 6 if len(sys.argv) < 7 else 1000):
    print(" ", i, " ".join(f"{v:7.2f}" for v in lead[i, :5]))
