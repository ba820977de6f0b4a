"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full, one
training step) of each bench phase, for bench.py's roofline `traffic` key.

  python tools/traffic_from_ncu.py WORKLOAD REPORT.ncu-rep [profiles/traffic_per_launch.json]
"""
import csv
import io
import json
import os
import subprocess
import sys

# kernel name fragment -> bench.py phase (hg_profile_step's phases)
PHASES = [("TUpdC", "update"), ("TProj", "proj"), ("OpProj", "proj"), ("k_agg_fwd", "agg_fwd"),
          ("TDAC", "dA"), ("MnGram", "dU"), ("k_agg_bwd", "agg_bwd"), ("MnDMx", "dMx"), ("k_dxda", "dX"),
          ("TDX", "dX")]


def main():
    wl, rep = sys.argv[1], sys.argv[2]
    out_path = sys.argv[3] if len(sys.argv) > 3 else "profiles/traffic_per_launch.json"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    acc = {}
    for r in rows[2:]:
        name = r[ki]
        ph = next((p for frag, p in PHASES if frag in name), None)
        if ph is None:
            continue
        b = float(r[ri].replace(",", "")) * scale[units[ri]] + float(r[wi].replace(",", "")) * scale[units[wi]]
        a = acc.setdefault(ph, [0.0, 0])
        a[0] += b
        a[1] += 1
    db = {}
    if os.path.exists(out_path):
        try:
            db = json.load(open(out_path))
        except ValueError:
            db = {}
    if not all(isinstance(v, dict) for v in db.values()):
        db = {}  # (round-1 flat layout)
    db[wl] = {ph: round(b / n) for ph, (b, n) in acc.items()}
    db.setdefault("_source", {})[wl] = f"{rep}: ncu --set full, one training step, DRAM read + write bytes per launch"
    json.dump(db, open(out_path, "w"), indent=1, sort_keys=True)
    print(json.dumps(db[wl], indent=1))


if __name__ == "__main__":
    main()
