"""Dev tool: per-CTA timeline of the forward's skinny product (k_rowmma, x·B) of
one layer (needs the -DMLRA_DEV_TRACE build via MLRA_LIB):
   python scripts/thin_timeline.py D_OUT D_IN M R"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer

d_out, d_in, m, r = (int(v) for v in sys.argv[1:5])
L = make_layer(d_out, d_in, 3, r, M.MaterializationStrategy.RowMaterialize)
x = torch.randn(m, d_in, device="cuda").to(torch.bfloat16)
buf = torch.zeros(1024 * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    M.layer_forward(L, x)
torch.cuda.synchronize()
os.environ["MLRA_TRACE3"] = str(buf.data_ptr())
M.layer_forward(L, x)
torch.cuda.synchronize()
del os.environ["MLRA_TRACE3"]
t = buf.view(1024, 8).cpu().numpy().astype(np.float64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = lambda c: (t[:, c] - t0) / 1e3
fin = t[:, 4] == 1
print(f"{len(t)} CTAs ({fin.sum()} finishers); us from the first CTA entry; act {m*d_in*2/1e6:.1f} MB")
for c, nm in ((0, "entry"), (1, "first unit landed"), (2, "last unit landed"), (3, "exit")):
    v = rel(c)
    print(f"  {nm:18s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}")
v = rel(5)[fin]
if v.size:
    print(f"  {'finisher start':18s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}")
    print(f"  finisher exit      med {np.median(rel(3)[fin]):7.2f} max {rel(3)[fin].max():7.2f}")
span = rel(3).max()
print(f"  kernel span {span:.2f} us -> {m*d_in*2/span/1e3:.0f} GB/s of activations")
