"""Per-source-line instruction / stall totals of one kernel in an ncu report.

  python tools/ncu_lines.py REPORT.ncu-rep KERNEL_INDEX [TOP]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, idx = sys.argv[1], int(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    print(rows[1][1][:100])
    h = rows[2]
    ii, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    lines = []
    for r in rows[3:]:
        if len(r) > si and r[0] not in ("", "-"):
            try:
                lines.append((float(r[ii] or 0), float(r[si] or 0), r[0], r[1]))
            except ValueError:
                pass
    ti = sum(x[0] for x in lines)
    ts = sum(x[1] for x in lines)
    print(f"total instr {ti:.0f} stall samples {ts:.0f}")
    print("-- by instructions")
    for x in sorted(lines, key=lambda x: -x[0])[:top]:
        print(f"{x[0]:10.0f} {100 * x[0] / ti:5.1f}% {x[1]:6.0f} L{x[2]:>4} {x[3].strip()[:100]}")
    print("-- by stall samples")
    for x in sorted(lines, key=lambda x: -x[1])[:top]:
        print(f"{x[1]:6.0f} {100 * x[1] / ts:5.1f}% {x[0]:10.0f} L{x[2]:>4} {x[3].strip()[:100]}")


if __name__ == "__main__":
    main()
