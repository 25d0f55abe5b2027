"""Summarise ncu captures into profiles/ (run here, after gpurun brings the
.ncu-rep / launch-list CSV back in gpurun_out/).

   python scripts/ncu_summary.py launches gpurun_out/r01_launches.csv
   python scripts/ncu_summary.py report gpurun_out/r01_qgemm_fwd.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, ks = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            ks.append((d["Kernel Name"], float(d["Metric Value"].replace(",", ""))))
    ours = [k for k in ks if "mlra" in k[0]]
    # the last step of the bench (16 + 4 per-layer prep kernels); print the tail
    print("| # | kernel | ns |\n|---|---|---|")
    tail = ours[-30:]
    for i, (n, t) in enumerate(tail):
        short = n.split("(")[0].replace("void ", "").replace("mlra::<unnamed>::", "")
        print(f"| {i} | `{short}` | {t:.0f} |")
    tot = sum(t for _, t in tail)
    q = sum(t for n, t in tail if "qgemm" in n)
    print(f"\nqgemm share of these launches: {100 * q / tot:.1f}% ({q / 1e3:.1f} of {tot / 1e3:.1f} us)")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for v in rows[2:]:
        name = v[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"\n**{name.split('(')[0]}** ({path.split('/')[-1]})\n")
        print("| metric | value |\n|---|---|")
        for key, label in METRICS:
            if key in hdr:
                i = hdr.index(key)
                print(f"| {label} (`{key}`) | {v[i]} {units[i]} |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        for p in sys.argv[2:]:
            report(p)
