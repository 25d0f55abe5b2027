"""GPU timeline of one bench step (dev probe): kernels with start/end/stream
from the CUPTI activity trace (torch.profiler), the critical path on the
compute stream and the gaps in it.

   python scripts/step_timeline.py [cfg2|cfg1|cfg3|cfg4] [OUT.json] [TOKENS]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2309_16119_b200 import modulora as M  # noqa: E402


class A:
    pass


def main():
    wname = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    out = sys.argv[2] if len(sys.argv) > 2 else None
    args = A()
    args.workload, args.bits, args.scaling = wname, 0, "weak"
    w = bench.workload(args)
    m, _ = bench.tokens_of(w, args, 0, 1)
    if len(sys.argv) > 3:
        m = int(sys.argv[3])  # e.g. cfg3 at one rank's strong-scaled share
    dev = torch.device("cuda", 0)
    wl = bench.Workload(w, m, M.parse_strategy("row"), dev, 0)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(5):
        wl.step(wl.xs, wl.dys, comm=False)
    torch.cuda.synchronize()
    steps = []
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            flush.zero_()
            torch.cuda.synchronize()
            wl.step(wl.xs, wl.dys, comm=False)
            torch.cuda.synchronize()
    path = out or "/tmp/step_trace.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"]
          if e.get("cat") == "kernel" and e.get("ph") == "X"]
    ev.sort(key=lambda e: e["ts"])
    # split into steps at the flush kernels (the big fill)
    cur = None
    for e in ev:
        if "fill" in e["name"] or "FillFunctor" in e["name"]:
            cur = []
            steps.append(cur)
        elif cur is not None:
            cur.append(e)
    s = steps[-1]
    t0 = s[0]["ts"]
    t_end = max(e["ts"] + e["dur"] for e in s)
    print(f"{wname}: {len(s)} kernels, span {t_end - t0:.1f} us")
    busy = []
    for e in s:
        nm = e["name"].replace("void ", "").replace("mlra::(anonymous namespace)::", "")
        nm = nm.split("(CU")[0].split("(mlra")[0].split("(int")[0].split("(const")[0]
        st = e["args"].get("stream")
        print(f"  {e['ts'] - t0:8.1f} +{e['dur']:7.1f}  s{st:<3} {nm[:70]}")
        busy.append((e["ts"] - t0, e["ts"] - t0 + e["dur"]))
    busy.sort()
    idle, reach = 0.0, 0.0
    for a, b in busy:
        if a > reach:
            idle += a - reach
        reach = max(reach, b)
    gemm = sum(e["dur"] for e in s if "qgemm" in e["name"])
    print(f"GPU idle inside the step: {idle:.1f} us; GEMM kernel time {gemm:.1f} us "
          f"({100 * gemm / (t_end - t0):.1f}% of the span)")


if __name__ == "__main__":
    main()
