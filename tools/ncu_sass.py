"""Top SASS instructions of one kernel in an ncu report by stall samples, with the reasons.

  python tools/ncu_sass.py REPORT.ncu-rep KERNEL_INDEX [TOP]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, idx = sys.argv[1], int(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip",
                          str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    data = [dict(zip(h, r)) for r in rows[hi + 1:] if len(r) == len(h)]
    reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]

    def num(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0
    tot = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
    for i, d in enumerate(data):
        d["_i"] = i
    for d in sorted(data, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[:top]:
        s = num(d["Warp Stall Sampling (All Samples)"])
        rs = sorted(((num(d[r]), r[6:]) for r in reasons), reverse=True)[:3]
        print(f"{s:6.0f} {100 * s / tot:5.1f}% #{d['_i']:<5} {d['Source'].strip()[:60]:60s} "
              + " ".join(f"{r}={v:.0f}" for v, r in rs if v))


if __name__ == "__main__":
    main()
