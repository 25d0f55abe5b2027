"""Minimal fused-path launch for debugging (one lp_forward / lp_backward)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer


def main():
    d_out, d_in, bits, m = (int(v) for v in sys.argv[1:5])
    op = sys.argv[5] if len(sys.argv) > 5 else "fwd"
    layer = make_layer(d_out, d_in, bits, 16, M.MaterializationStrategy.RowMaterialize)
    ctx = M.LpLinearContext(layer.weights, M.MaterializationStrategy.RowMaterialize)
    if op == "fwd":
        x = torch.randn(m, d_in, device="cuda").to(torch.bfloat16)
        y = M.lp_forward(ctx, x)
    else:
        g = torch.randn(m, d_out, device="cuda").to(torch.bfloat16)
        y = M.lp_backward(ctx, g)
    torch.cuda.synchronize()
    print("ok", y.float().abs().mean().item())


if __name__ == "__main__":
    main()
