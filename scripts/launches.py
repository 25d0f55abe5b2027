"""Summarise an ncu --metrics gpu__time_duration.sum launch list: the last
`--last` launches per kernel name (us) and a per-step table."""
import csv
import statistics
import sys
from collections import defaultdict


def load(path):
    hdr, out = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                out.append(d)
    return out


if __name__ == "__main__":
    rows = load(sys.argv[1])
    last = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    by = defaultdict(list)
    for d in rows[-last:]:
        nm = d["Kernel Name"].split("(")[0].replace("void ", "").replace("mlra::<unnamed>::", "")
        by[nm].append(float(d["Metric Value"]) / 1e3)
    tot = 0.0
    for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        tot += sum(v)
        print(f"{k[:60]:60s} n={len(v):3d} med={statistics.median(v):8.2f} us  sum={sum(v):9.1f} us")
    print(f"total {tot:.1f} us over the last {last} launches")
