"""Dev tool: GPU time of the skinny adapter products — layer_backward without
dX at the cfg2 up layer (dY·A, dYᵀ·XB, Xᵀ·dYA + two prep launches), captured
in a CUDA graph; prints us per call for the library in MLRA_LIB."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer

d_out, d_in, m = int(os.environ.get("DOUT", 11008)), int(os.environ.get("DIN", 4096)), 4096
L = make_layer(d_out, d_in, 3, 16, M.MaterializationStrategy.RowMaterialize)
x = torch.randn(m, d_in, device="cuda").to(torch.bfloat16)
dy = torch.randn(m, d_out, device="cuda").to(torch.bfloat16)
y, xb = M.layer_forward(L, x)


def fwd():
    M.layer_forward(L, x)


def bwd():
    M.layer_backward(L, x, xb, dy, need_dx=False)


for name, fn in (("bwd_no_dx", bwd),):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
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
        best = min(best, s.elapsed_time(e) / 10 * 1e3)
    print(f"{os.environ.get('MLRA_LIB', 'default')} {name} {best:.1f} us", flush=True)
