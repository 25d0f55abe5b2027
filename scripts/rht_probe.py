"""Dev tool: mlra_rht bandwidth at the cfg5 incoherent-layer shapes, tensor-core
kernel vs the butterfly kernel (MLRA_RHT_BUTTERFLY=1 in a second process), and
agreement between the two.
   python scripts/rht_probe.py [out.npy]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2309_16119_b200 import modulora as M

flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
res = []
for rows, cols, inv, odt in ((4096, 17920, False, torch.bfloat16), (4096, 6656, True, torch.bfloat16),
                             (4096, 17920, True, torch.bfloat16), (4096, 17920, False, torch.float32)):
    g = torch.Generator(device="cpu").manual_seed(rows + cols)
    x = torch.randn(rows, cols, generator=g).to(torch.bfloat16).cuda()
    s = M.random_signs(cols, 3)
    out = M.rht(x, s, 512, inverse=inv, out_dtype=odt)
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        M.rht(x, s, 512, inverse=inv, out_dtype=odt)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    us = float(np.median(ts))
    nbytes = rows * cols * (2 + out.element_size())
    res.append({"shape": [rows, cols], "inverse": inv, "out": str(odt), "us": us,
                "gbs": nbytes / us / 1e3, "butterfly": os.environ.get("MLRA_RHT_BUTTERFLY") is not None,
                "checksum": float(out.double().sum().item()), "absmax": float(out.float().abs().max())})
    print(json.dumps(res[-1]), flush=True)
