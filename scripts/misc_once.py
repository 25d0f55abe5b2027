"""Dev tool: one launch each of the non-GEMM device kernels at LLaMA shapes, for
ncu captures — AdamW over a 7B-decoder-layer adapter bucket (r=8, 624,640
params), RTN quantize of an 11008x4096 f32 matrix, and a cb2-fused layer
forward at cfg5 shapes (6656x17920, 4096 tokens)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2309_16119_b200 import modulora as M
from paper_2309_16119_b200 import train as T

n = 624640
p = torch.randn(n, device="cuda", dtype=torch.float64)
g = torch.randn(n, device="cuda")
opt = T.AdamW()
for s in range(2):
    opt.step(p, [n], ["bucket"], g, s, 1e-3, check_finite=False)
w = torch.randn(11008, 4096, device="cuda") * 0.02
M.RtnQuantizer().quantize(w, None, 3, 128)
rows, cols = 6656, 17920
rng = np.random.default_rng(5)
m = M.Cb2Matrix(rows, cols, 128, rng.integers(0, 1 << 16, (rows, cols // 8), dtype=np.uint32).astype(np.uint16),
                M.default_cb2_codebook(), (0.01 * (0.5 + rng.random((rows, cols // 128)))).astype(np.float32))
dq = M.Codebook2Quantizer().upload(m)
x = torch.randn(4096, cols, device="cuda").to(torch.bfloat16)
for _ in range(2):
    M.lp_forward(M.LpLinearContext(dq, M.MaterializationStrategy.RowMaterialize), x)
torch.cuda.synchronize()
