"""Quick per-op timing of one ModuLoRA layer on the GPU (dev tool, not the bench)."""
import sys
import os
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2309_16119_b200 import modulora as M


def make_layer(d_out, d_in, bits, r, strategy):
    rng = np.random.default_rng(0)
    count = d_out * d_in
    nw = M.packed_word_count(count, bits)
    words = rng.integers(0, 2**32, size=nw, dtype=np.uint64).astype(np.uint32)
    tail = nw * 32 - count * bits
    if tail:
        words[-1] &= (1 << (32 - tail)) - 1
    ng = d_out * d_in // 128
    sc = (0.001 + 0.01 * rng.random(ng)).astype(np.float32)
    z = (-0.05 * rng.random(ng)).astype(np.float32)
    q = M.QuantizedMatrix(d_out, d_in, bits, 128, M.PackedCodes(bits, count, words), sc, z)
    dq = M.DeviceQuantizedMatrix(q)
    a = torch.randn(d_out, r, device="cuda") * 0.02
    b = torch.randn(d_in, r, device="cuda") * 0.02
    return M.ModuLoraLayer("p", dq, M.LoraAdapter(a, b, r, 32.0), strategy=strategy)


def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    m = int(os.environ.get("M", 4096))
    for (d_out, d_in, bits, r) in [(11008, 4096, 3, 16), (4096, 11008, 3, 16), (4096, 4096, 4, 8)]:
        for strat in [M.MaterializationStrategy.RowMaterialize, M.MaterializationStrategy.WeightMaterialize]:
            layer = make_layer(d_out, d_in, bits, r, strat)
            x = torch.randn(m, d_in, device="cuda").to(torch.bfloat16)
            dy = torch.randn(m, d_out, device="cuda").to(torch.bfloat16)
            ctx = M.LpLinearContext(layer.weights, strat)
            t_fwd_base = timeit(lambda: M.lp_forward(ctx, x))
            t_bwd_base = timeit(lambda: M.lp_backward(ctx, dy))
            y, xb = M.layer_forward(layer, x)
            t_fwd = timeit(lambda: M.layer_forward(layer, x))
            t_bwd = timeit(lambda: M.layer_backward(layer, x, xb, dy))
            t_mat = timeit(lambda: M.dequantize(layer.weights, torch.bfloat16))
            fl = 2.0 * m * d_out * d_in
            print(f"{d_out}x{d_in} b{bits} r{r} m{m} {M.strategy_name(strat):6s} "
                  f"lp_fwd {t_fwd_base:.3f}ms ({fl/t_fwd_base/1e9:.0f} TF) "
                  f"lp_bwd {t_bwd_base:.3f}ms ({fl/t_bwd_base/1e9:.0f} TF) "
                  f"layer_fwd {t_fwd:.3f} layer_bwd {t_bwd:.3f} "
                  f"materialize {t_mat:.3f}ms ({(d_out*d_in*(2+bits/8))/t_mat/1e6:.0f} GB/s)",
                  flush=True)


if __name__ == "__main__":
    main()
