"""Writes profiles/traffic.json from an ncu --set full capture of the bench's
dominant kernel (the cfg2 up-layer fused GEMM, forward and dX), exported with
`ncu -i X.ncu-rep --page raw --csv`:
   python scripts/traffic.py FWD_RAW.csv DX_RAW.csv > profiles/traffic.json"""
import csv
import json
import sys


def dram(path):
    rows = list(csv.reader(open(path)))
    hdr, units, r = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(d["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
    wr = float(d["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
    return rd, wr, d["Kernel Name"][:60]


m, K, N, bits, g = 4096, 4096, 11008, 3, 128
codes = N * K * bits / 8 + 8 * N * K / g
alg = {"fwd": {"read": m * K * 2 + codes, "write": m * N * 2},      # X, codes+grid; Y
       "dx": {"read": m * N * 2 + codes, "write": m * K * 2}}       # dY, codes+grid; dX
out = {"workload": "cfg2-llama7b-mlp-up+down", "layer": "up 11008x4096, 4096 tokens",
       "source": "ncu --set full --clock-control none, one launch each (scripts/profile_r02.sh)"}
tot = []
for nm, path in (("fwd", sys.argv[1]), ("dx", sys.argv[2])):
    rd, wr, kname = dram(path)
    out[nm] = {"kernel": kname, "dram_read": rd, "dram_write": wr, "alg_read": alg[nm]["read"],
               "alg_write": alg[nm]["write"], "read_over_alg": rd / alg[nm]["read"]}
    tot.append(rd + wr)
out["qgemm_dram_bytes_per_launch"] = sum(tot) / 2
print(json.dumps(out, indent=1))
