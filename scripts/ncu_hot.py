"""Hot SASS lines of one kernel in an ncu report (stall samples), with the CUDA
source line each maps to. Usage: python scripts/ncu_hot.py REPORT KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kern}"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    recs = []
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) >= len(hdr):
            recs.append(dict(zip(hdr, r)))
    key = "Warp Stall Sampling (All Samples)"

    def f(v):
        try:
            return float(v)
        except ValueError:
            return 0.0
    tot = sum(f(x[key]) for x in recs)
    print(f"{len(recs)} SASS lines, {tot:.0f} samples")
    for i, x in sorted(enumerate(recs), key=lambda t: -f(t[1][key]))[:n]:
        print(f"{f(x[key]):6.0f} {100 * f(x[key]) / max(tot, 1):5.1f}%  #{i:5d} {x['Source'][:70]}")
    if len(sys.argv) > 4:  # context around one SASS index
        c = int(sys.argv[4])
        for i in range(max(0, c - 25), min(len(recs), c + 10)):
            print(f"#{i:5d} {f(recs[i][key]):5.0f} {recs[i]['Instructions Executed']:>8s} {recs[i]['Source'][:90]}")


if __name__ == "__main__":
    main()
