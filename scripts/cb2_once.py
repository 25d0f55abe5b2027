"""Dev tool: materialize a cfg5-shaped cb2 matrix REPS times (ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2309_16119_b200 import modulora as M

rows, cols = 6656, 17920
rng = np.random.default_rng(501)
m = M.Cb2Matrix(rows, cols, 128,
                rng.integers(0, 1 << 16, (rows, cols // 8), dtype=np.uint32).astype(np.uint16),
                M.default_cb2_codebook(),
                (0.01 * (0.5 + rng.random((rows, cols // 128)))).astype(np.float32))
q = M.Codebook2Quantizer().upload(m)
dt = torch.float32 if os.environ.get("F32") else torch.bfloat16
out = torch.empty(rows, cols, dtype=dt, device="cuda")
for _ in range(int(os.environ.get("REPS", 3))):
    M.dequantize(q, dt, out=out)
torch.cuda.synchronize()
