"""Dev probe: effective time of the row product x·B / dY·A on the layer pass's
critical path (k_rowmma* end - the end of the previous kernel on its stream:
the prep launch, or the L2 flush when the row kernel is fused; CUPTI
timestamps), at 4096 tokens, d_in 4096 and 11008, r = 16.
   python scripts/rowmma_probe.py"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from scripts.sweep import layers_for  # noqa: E402
from paper_2309_16119_b200 import modulora as M  # noqa: E402


def main():
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
    m, r = 4096, 16
    for d_out, d_in in ((11008, 4096), (4096, 11008)):
        (L,) = layers_for([(d_out, d_in)], 3, r, M.MaterializationStrategy.RowMaterialize)
        x = torch.randn(m, d_in, device="cuda").to(torch.bfloat16)
        dy = torch.randn(m, d_out, device="cuda").to(torch.bfloat16)
        for _ in range(3):
            y, xb = M.layer_forward(L, x)
            M.layer_backward(L, x, xb, dy)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(8):
                flush.zero_()
                y, xb = M.layer_forward(L, x)
                M.layer_backward(L, x, xb, dy)
            torch.cuda.synchronize()
        path = "/tmp/rowmma_probe.json"
        prof.export_chrome_trace(path)
        ev = sorted((e for e in json.load(open(path))["traceEvents"]
                     if e.get("cat") == "kernel" and e.get("ph") == "X"), key=lambda e: e["ts"])
        fwd, bwd, last_end, n_row = [], [], {}, 0
        for e in ev:
            st = e["args"].get("stream")
            if "k_rowmma" in e["name"] and st in last_end:
                (fwd if n_row % 2 == 0 else bwd).append(e["ts"] + e["dur"] - last_end[st])
                n_row += 1
            if "k_colmma" not in e["name"]:
                last_end[st] = e["ts"] + e["dur"]
        name = next(e["name"] for e in ev if "k_rowmma" in e["name"]).split("(")[0][-24:]
        for lab, v, k in (("x.B", fwd, d_in), ("dy.A", bwd, d_out)):
            us = statistics.median(v)
            print(json.dumps({"kernel": name, "product": lab, "m": m, "k": k, "r": r,
                              "lib": os.environ.get("MLRA_LIB", "default"),
                              "us": round(us, 2), "GBps": round(m * k * 2 / us / 1e3, 1)}),
                  flush=True)


if __name__ == "__main__":
    main()
