"""Dev tool: K1 materialize() bandwidth, bulk-store kernel (MLRA_K1=1) vs the
2-D per-row grid (MLRA_K1=0), bit-compared. Run once per MLRA_K1 value."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import synthetic_qmatrix
from paper_2309_16119_b200 import modulora as M

flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
for rows, cols, bits in ((6656, 17920, 2), (11008, 4096, 3), (4096, 11008, 4), (4096, 4096, 8)):
    q, *_ = synthetic_qmatrix(rows, cols, bits, 128, 5)
    dq = M.DeviceQuantizedMatrix(q)
    for dt, eb in ((torch.bfloat16, 2), (torch.float32, 4)):
        out = torch.empty(rows, cols, dtype=dt, device="cuda")
        for _ in range(3):
            M.dequantize(dq, dt, out=out)
        ts = []
        for _ in range(10):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            M.dequantize(dq, dt, out=out)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        us = sorted(ts)[len(ts) // 2] * 1e3
        nbytes = rows * cols * (bits / 8 + eb) + rows * (cols // 128) * 8
        h = int(out.view(torch.int16 if eb == 2 else torch.int32).double().sum().item())
        print(json.dumps({"k1": os.environ.get("MLRA_K1", "1"), "shape": [rows, cols, bits],
                          "out": str(dt), "us": round(us, 1), "gbs": round(nbytes / us / 1e3, 1),
                          "checksum": h}), flush=True)
