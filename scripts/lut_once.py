"""Dev tool: one NF4 (lut plugin, 4-bit g64) forward + dX at the cfg2 up shape
(11008x4096, 4096 tokens) and one bf16 materialize, REPS times (ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2309_16119_b200 import modulora as M

rows, cols, m = 11008, 4096, 4096
g = np.random.default_rng(710)
codes = g.integers(0, 16, rows * cols, dtype=np.uint32)
lm = M.LutMatrix(rows, cols, 4, 64, M.PackedCodes(4, rows * cols, M.pack_codes(codes, 4)),
                 M.NF4_LEVELS, (0.02 * (0.5 + g.random((rows, cols // 64)))).astype(np.float32))
dq = M.LutQuantizer().upload(lm)
ctx = M.LpLinearContext(dq, M.MaterializationStrategy.RowMaterialize)
x = torch.randn(m, cols, device="cuda").to(torch.bfloat16)
dy = torch.randn(m, rows, device="cuda").to(torch.bfloat16)
out = torch.empty(rows, cols, dtype=torch.bfloat16, device="cuda")
for _ in range(int(os.environ.get("REPS", 2))):
    M.lp_forward(ctx, x)
    M.lp_backward(ctx, dy)
    M.dequantize(dq, torch.bfloat16, out=out)
torch.cuda.synchronize()
