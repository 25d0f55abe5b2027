"""Dev tool: host (CPU) time of one enqueue of each layer-pass API call at cfg1
(the GPU is drained before each call, so this is the library's launch path:
workspace allocation, tensor-map encodes, plan, launches)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer

L = make_layer(4096, 4096, 4, 8, M.MaterializationStrategy.RowMaterialize)
x = torch.randn(512, 4096, device="cuda").to(torch.bfloat16)
dy = torch.randn(512, 4096, device="cuda").to(torch.bfloat16)
y, xb = M.layer_forward(L, x)
for name, fn in (("layer_forward", lambda: M.layer_forward(L, x)),
                 ("layer_backward", lambda: M.layer_backward(L, x, xb, dy)),
                 ("lp_forward", lambda: M.lp_forward(M.LpLinearContext(L.weights, L.strategy), x))):
    ts = []
    for _ in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    print(f"{name}: host {np.median(ts) * 1e6:.1f} us per call (median of 30)")
