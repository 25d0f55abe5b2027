"""Dev tool: run one fused GEMM op REPS times (for ncu launch lists).
   python scripts/op_once.py {fwd|dx} D_OUT D_IN BITS M"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer

op = sys.argv[1]
d_out, d_in, bits, m = (int(v) for v in sys.argv[2:6])
L = make_layer(d_out, d_in, bits, 16, M.MaterializationStrategy.RowMaterialize)
ctx = M.LpLinearContext(L.weights, M.MaterializationStrategy.RowMaterialize)
x = torch.randn(m, d_in if op == "fwd" else d_out, device="cuda").to(torch.bfloat16)
for _ in range(int(os.environ.get("REPS", 3))):
    (M.lp_forward if op == "fwd" else M.lp_backward)(ctx, x)
torch.cuda.synchronize()
