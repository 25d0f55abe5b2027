"""Dev tool: what the skinny adapter products cost on the critical path, from
graph-replayed op timings (no host overhead): layer_forward - lp_forward (prep +
x·B + the LoRA extra-K blocks), layer_backward - lp_backward (prep + dY·A + the
part of dA/dB not hidden under the dX GEMM), and layer_backward without dX.
   python scripts/skinny_probe.py            (cfg2 up, cfg2 down, cfg1)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer


def gtime(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    best = 1e9
    for _ in range(5):
        g.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / reps * 1e3)
    return best


cases = [("cfg2_up", 11008, 4096, 3, 16, 4096), ("cfg2_down", 4096, 11008, 3, 16, 4096),
         ("cfg1", 4096, 4096, 4, 8, 512), ("cfg3_q_1k", 4096, 4096, 3, 8, 1024)]
only = sys.argv[1:]
for name, d_out, d_in, bits, r, m in cases:
    if only and name not in only:
        continue
    strat = M.MaterializationStrategy.RowMaterialize
    L = make_layer(d_out, d_in, bits, r, strat)
    ctx = M.LpLinearContext(L.weights, strat)
    x = torch.randn(m, d_in, device="cuda").to(torch.bfloat16)
    dy = torch.randn(m, d_out, device="cuda").to(torch.bfloat16)
    y, xb = M.layer_forward(L, x)
    t = {
        "lp_fwd": gtime(lambda: M.lp_forward(ctx, x)),
        "layer_fwd": gtime(lambda: M.layer_forward(L, x)),
        "lp_bwd": gtime(lambda: M.lp_backward(ctx, dy)),
        "layer_bwd": gtime(lambda: M.layer_backward(L, x, xb, dy)),
        "layer_bwd_nodx": gtime(lambda: M.layer_backward(L, x, xb, dy, need_dx=False)),
    }
    act_mb = (m * d_in * 2 + m * d_out * 2 * 2 + m * d_in * 2) / 1e6  # x, dY twice, x (dB)
    print(f"{name}: " + " ".join(f"{k} {v:.1f}" for k, v in t.items()) +
          f" | fwd extra {t['layer_fwd'] - t['lp_fwd']:.1f} us, bwd extra {t['layer_bwd'] - t['lp_bwd']:.1f} us"
          f" (us; skinny operands {act_mb:.0f} MB)", flush=True)
