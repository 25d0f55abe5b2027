"""Run one layer op a few times (for ncu captures). Usage:
   python scripts/ncu_one.py OP STRATEGY D_OUT D_IN BITS R M
   OP in {lp_fwd, lp_bwd, layer, materialize}"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer


def main():
    op, strat = sys.argv[1], M.parse_strategy(sys.argv[2])
    d_out, d_in, bits, r, m = (int(v) for v in sys.argv[3:8])
    reps = int(os.environ.get("REPS", 3))
    layer = make_layer(d_out, d_in, bits, r, strat)
    x = torch.randn(m, d_in, device="cuda").to(torch.bfloat16)
    dy = torch.randn(m, d_out, device="cuda").to(torch.bfloat16)
    ctx = M.LpLinearContext(layer.weights, strat)
    for _ in range(reps):
        if op == "lp_fwd":
            M.lp_forward(ctx, x)
        elif op == "lp_bwd":
            M.lp_backward(ctx, dy)
        elif op == "layer":
            y, xb = M.layer_forward(layer, x)
            M.layer_backward(layer, x, xb, dy)
        elif op == "materialize":
            M.dequantize(layer.weights, torch.bfloat16)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
