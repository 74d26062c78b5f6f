#!/usr/bin/env python3
"""vgpu-bench with the reference's command line (proj/tools/vgpu_bench.cpp:
30-75), driving bench.py's report modes on the B200 GVM.

    python scripts/vgpu_bench.py sweep    [--profile NAME] [--nmax N] [--out CSV]
    python scripts/vgpu_bench.py validate [--profile NAME] [--nmax N] [--out CSV]
    python scripts/vgpu_bench.py overhead [--out CSV]
    python scripts/vgpu_bench.py speedup  [--out CSV]

--profile takes the reference's builtin profile names (proj/src/bench/
profiles.cpp:27-45) and maps them to the workloads built here; MG has no
kernel (out of scope). The reference's timing knobs (--mode,
--clock, --scale, --t-init, --t-ctx-switch, --nproc, --os-processes,
--instance) are accepted for drop-in scripts and ignored: on B200 both modes
are measured on real hardware in every report, with real processes. Output:
the report's CSV (sweep/validate/overhead/speedup rows) to --out or stdout.
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILES = {"EP_M30": "ep", "EP_M24": "ep", "VecAdd": "vecadd", "VecMul": "vmul", "MM": "mm",
            "BS": "bs", "CG": "cg", "ES": "es"}


def rows_to_csv(rows) -> str:
    cols = []
    for r in rows:
        for k in r:
            if k not in cols:
                cols.append(k)
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=cols)
    w.writeheader()
    for r in rows:
        w.writerow(r)
    return buf.getvalue()


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="vgpu-bench")
    ap.add_argument("command", choices=["sweep", "validate", "overhead", "speedup"])
    ap.add_argument("--profile", default="EP_M30")
    ap.add_argument("--nmax", type=int, default=0)
    ap.add_argument("--out", default="")
    ap.add_argument("--sizes", default="")
    for ignored in ("--nproc", "--mode", "--clock", "--scale", "--reps", "--t-init",
                    "--t-ctx-switch", "--instance"):
        ap.add_argument(ignored, default=None)
    ap.add_argument("--os-processes", action="store_true")
    a = ap.parse_args(argv)
    if a.profile == "MG":
        print("vgpu-bench: the MG profile has no kernel in this build (DESIGN.md)", file=sys.stderr)
        return 2
    if a.profile not in PROFILES:
        print(f"vgpu-bench: unknown profile {a.profile}", file=sys.stderr)
        return 2
    flag = {"sweep": "--sweep", "validate": "--validate-model", "overhead": "--overhead-curve",
            "speedup": "--speedup"}[a.command]
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), flag, "--workload", PROFILES[a.profile]]
    if a.nmax:
        cmd += ["--procs", str(a.nmax)]
    if a.profile == "EP_M24":
        cmd += ["--ep-m", "24"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    if out.returncode != 0:
        sys.stderr.write(out.stderr[-2000:])
        return out.returncode
    report = json.loads(out.stdout.strip().splitlines()[-1])
    rows = report.get("rows")
    if rows is None:  # validate: one row set per device model
        rows = [{"model": name, **r} for name in ("concurrent", "device_filling")
                for r in report.get(name, {}).get("rows", [])]
    text = report.get("csv") or rows_to_csv(rows)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
