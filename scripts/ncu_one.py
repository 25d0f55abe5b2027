"""Run one layer op a few times (for ncu captures). Usage:
   python scripts/ncu_one.py OP STRATEGY D_OUT D_IN BITS R M
   OP in {lp_fwd, lp_bwd, layer, materialize, e8p_fwd, rht}
   (e8p_fwd: the fused e8p GEMM of a D_OUT x D_IN e8p matrix; rht: mlra_rht over an
   M x D_IN bf16 activation, block 512)"""
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
    if op == "e8p_fwd":
        import numpy as np
        rng = np.random.default_rng(0)
        codes = rng.integers(0, 1 << 16, size=d_out * d_in // 8, dtype=np.uint32).astype(np.uint16)
        scales = (0.01 + 0.01 * rng.random(d_out * d_in // 128)).astype(np.float32)
        em = M.E8pMatrix(d_out, d_in, 128, codes, scales)
        dq = M.E8pQuantizer().upload(em)
        ctx = M.LpLinearContext(dq, strat)
        x = torch.randn(m, d_in, device="cuda").to(torch.bfloat16)
        for _ in range(reps):
            M.lp_forward(ctx, x)
        torch.cuda.synchronize()
        return
    if op == "rht":
        x = torch.randn(m, d_in, device="cuda").to(torch.bfloat16)
        s = M.random_signs(d_in, 3)
        for _ in range(reps):
            M.rht(x, s, 512)
        torch.cuda.synchronize()
        return
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
