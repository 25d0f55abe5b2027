"""Dev tool: A/B the fused GEMM across libmlra variants (MLRA_LIB per subprocess).
   python scripts/ab.py lib1.so lib2.so ...   (interleaved rounds, median TF per op)"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CHILD = r"""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer
m = int(os.environ.get("M", 4096)); reps = int(os.environ.get("REPS", 30))
strat = M.parse_strategy(os.environ.get("STRAT", "row"))
out = {}
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name, (n, k, b, r) in {"up": (11008, 4096, 3, 16), "down": (4096, 11008, 3, 16)}.items():
    L = make_layer(n, k, b, r, strat)
    ctx = M.LpLinearContext(L.weights, strat)
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    dy = torch.randn(m, n, device="cuda").to(torch.bfloat16)
    for op, fn in (("fwd", lambda: M.lp_forward(ctx, x)), ("dx", lambda: M.lp_backward(ctx, dy))):
        for _ in range(3): fn()
        ts = []
        for _ in range(reps):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); fn(); e.record(); torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ts.sort()
        out[f"{name}_{op}"] = 2.0 * m * n * k / (ts[len(ts) // 2] * 1e-3) / 1e12
print("RESULT " + json.dumps(out))
"""


def main():
    libs = sys.argv[1:]
    rounds = int(os.environ.get("ROUNDS", 2))
    res = {l: [] for l in libs}
    for _ in range(rounds):
        for l in libs:
            env = dict(os.environ, MLRA_LIB=os.path.abspath(l))
            r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
            line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
            if not line:
                print(l, "FAILED", r.stderr[-1500:])
                continue
            res[l].append(json.loads(line[0][7:]))
    for l, rs in res.items():
        if not rs:
            continue
        keys = rs[0].keys()
        med = {k: sorted(x[k] for x in rs)[len(rs) // 2] for k in keys}
        avg = sum(med.values()) / len(med)
        print(f"{os.path.basename(l):28s} " + " ".join(f"{k} {v:7.1f}" for k, v in med.items())
              + f"  | mean {avg:7.1f} TF", flush=True)


if __name__ == "__main__":
    main()
