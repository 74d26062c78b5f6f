#!/usr/bin/env python3
"""profiles/r1_ncu_full_<kind>.csv -> profiles/ncu_traffic.json.

Each CSV is `ncu -i <capture>.ncu-rep --page raw --csv --metrics
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum` of ONE
`ncu --set full --clock-control none` capture of the kind's dominant kernel,
launched at bench.py's per-step shape (scripts/gpu_profiles.sh). bench.py
reports read+write as roofline.traffic (bytes per launch)."""
import csv
import glob
import json
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
PROF = os.path.join(os.path.dirname(HERE), "profiles")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
         "s": 1e6}


def main():
    out = {}
    for path in sorted(glob.glob(os.path.join(PROF, "r*_ncu_full_*.csv"))):
        kind = re.sub(r"^r\d+_ncu_full_", "", os.path.basename(path))[:-4]
        rows = list(csv.reader(open(path)))
        hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        names, units, vals = rows[hdr], rows[hdr + 1], rows[hdr + 2]
        get = lambda m: float(vals[names.index(m)].replace(",", "")) * SCALE[units[names.index(m)]]
        rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
        out[kind] = {"bytes": rd + wr, "read": rd, "write": wr,
                     "kernel_us": get("gpu__time_duration.sum"),
                     "kernel": vals[names.index("Kernel Name")],
                     "grid": vals[names.index("Grid Size")],
                     "source": "profiles/" + os.path.basename(path)}
    with open(os.path.join(PROF, "ncu_traffic.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
