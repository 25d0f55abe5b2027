"""Dev tool: fused-GEMM GPU time vs token count under each schedule — pair
kernel whole tiles (MLRA_SK=0), stream-K (1), cost model (2), and the 1-CTA
kernel (MLRA_GEMM=1: 256-token tiles, 3: 128-token tiles) and the cost model's own choice (auto). Each (op, mode) is captured in a CUDA graph of 10
launches (no host overhead) and the modes are timed round-robin (3 rounds,
best kept) so clock drift does not favour any order."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer

MODES = {"sk0": ("2", "0"), "sk1": ("2", "1"), "sk2": ("2", "2"), "split": ("2", "4"), "split256": ("2", "5"), "cta1": ("1", "2"), "cta128": ("3", "2"), "auto": ("", "2")}
ms_list = [int(v) for v in os.environ.get("MS", "512,1024,2048").split(",")]
shapes = [(4096, 4096, 4), (11008, 4096, 3), (4096, 11008, 3)]
for d_out, d_in, bits in shapes:
    L = make_layer(d_out, d_in, bits, 16, M.MaterializationStrategy.RowMaterialize)
    ctx = M.LpLinearContext(L.weights, M.MaterializationStrategy.RowMaterialize)
    for m in ms_list:
        x = torch.randn(m, d_in, device="cuda").to(torch.bfloat16)
        g = torch.randn(m, d_out, device="cuda").to(torch.bfloat16)
        graphs = {}
        for mode, (gem, sk) in MODES.items():
            os.environ["MLRA_SK"] = sk
            if gem:
                os.environ["MLRA_GEMM"] = gem
            else:
                os.environ.pop("MLRA_GEMM", None)
            for op, fn, a in (("fwd", M.lp_forward, x), ("dx", M.lp_backward, g)):
                fn(ctx, a)
                torch.cuda.synchronize()
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr):
                    for _ in range(10):
                        fn(ctx, a)
                graphs[(mode, op)] = gr
        best = {}
        for _ in range(3):
            for key, gr in graphs.items():
                gr.replay()
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                gr.replay()
                e.record()
                torch.cuda.synchronize()
                us = s.elapsed_time(e) / 10 * 1e3
                best[key] = min(best.get(key, 1e9), us)
        for mode in MODES:
            res = {op: round(best[(mode, op)], 1) for op in ("fwd", "dx")}
            res.update({op + "_tf": round(2.0 * m * d_out * d_in / (best[(mode, op)] * 1e-6) / 1e12, 1)
                        for op in ("fwd", "dx")})
            print(json.dumps({"shape": [d_out, d_in, bits], "m": m, "mode": mode, **res}), flush=True)
