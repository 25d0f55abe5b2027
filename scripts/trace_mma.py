"""Dev tool: per-CTA-pair MMA-thread wait breakdown of one fused GEMM launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer

strat = M.parse_strategy(sys.argv[1] if len(sys.argv) > 1 else "row")
layer = make_layer(11008, 4096, 3, 16, strat)
x = torch.randn(4096, 4096, device="cuda").to(torch.bfloat16)
ctx = M.LpLinearContext(layer.weights, strat)
buf = torch.zeros(74 * 4, dtype=torch.int64, device="cuda")
M.lp_forward(ctx, x); torch.cuda.synchronize()
os.environ["MLRA_TRACE"] = str(buf.data_ptr())
M.lp_forward(ctx, x); torch.cuda.synchronize()
del os.environ["MLRA_TRACE"]
t = buf.view(74, 4).cpu().numpy()
tot, full, temp, tiles = t[:, 0], t[:, 1], t[:, 2], t[:, 3]
kb = tiles * 65 if os.environ.get("MLRA_SK", "2") == "0" else np.full_like(tiles, 344 * 65 // 74)
print(f"{M.strategy_name(strat)}: tiles/pair min {tiles.min()} max {tiles.max()}; cycles max {tot.max()}")
print(f"  per k-block: total {tot.sum()/kb.sum():.0f} cyc, waiting on full {full.sum()/kb.sum():.0f}, "
      f"on tempty {temp.sum()/kb.sum():.0f} (ideal MMA 1071)")
i = tot.argmax()
print(f"  slowest pair: {tiles[i]} tiles, {tot[i]} cyc, full-wait {full[i]}, tempty-wait {temp[i]}")
