"""OPTQ timing: the device quantizer (workspace + sweep +
packing, synchronous end to end from device inputs) at LLaMA-ish shapes, and
the reference's quantize_optq on the host for the shape it finishes in seconds."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2309_16119_b200 import modulora as M


def main():
    rng = np.random.default_rng(0)
    for rows, cols, m in ((1024, 1024, 512), (4096, 4096, 2048), (11008, 4096, 2048)):
        w = torch.from_numpy(rng.normal(0, 0.02, (rows, cols))).cuda()
        x = torch.from_numpy(rng.normal(0, 1, (m, cols))).cuda()
        qz = M.OptqQuantizer(0.01)
        qz.quantize(w[:64], x[:, :], 3, 128)  # warm-up (allocations, module load)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h, u = M.optq_workspace(x, 0.01)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        qz.quantize(w, x, 3, 128)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rec = {"config": "optq", "rows": rows, "cols": cols, "calib": m, "bits": 3, "group": 128,
               "workspace_s": t1 - t0, "quantize_total_s": t2 - t1}
        if rows == 1024:
            try:
                from oracle.oracle import Ref
                if Ref.available():
                    wn, xn = w.cpu().numpy(), x.cpu().numpy()
                    t3 = time.perf_counter()
                    Ref.quantize_optq(wn, xn, 3, 128, 0.01)
                    rec["reference_cpu_s"] = time.perf_counter() - t3
            except Exception as e:  # noqa: BLE001
                rec["reference_cpu_s"] = f"unavailable: {e}"
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
