"""Capture the DRAM traffic of bench.py's timed k_solve launch with ncu and record it in
profiles/traffic.json keyed by workload and the sha256 of the library's sources and compile flags
(bench.py refuses entries captured with other kernel sources).  Run on the GPU box:

    python tools/ncu_traffic.py C3 [C4 C5 ...] [--method bicgstab] [--out profiles/traffic.json]

The numbers printed under ncu are never bench values; only the DRAM byte counts are used.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"


def capture(cfg: str, method: str, precond: str, warm: bool, tres: bool, log: str) -> dict:
    cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "--kernel-name", "regex:k_solve",
           "--launch-skip", str(1 + (2 if method == "gsf" else 0)), "--launch-count", "1", "--csv",
           "--log-file", log,
           sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--method", method,
           "--precond", precond, "--steps", "1", "--warmup", "1", "--no-e2e", "--no-cpu"]
    if warm:
        cmd.append("--warm")
    if tres:
        cmd.append("--true-res")
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    with open(log) as fh:
        text = fh.read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    vals = {}
    for r in rows:
        name, unit, v = r["Metric Name"], r["Metric Unit"], float(r["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(unit, 1.0)
        vals[name] = v * scale
    return {"dram_bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
            "dram_read": vals["dram__bytes_read.sum"], "dram_write": vals["dram__bytes_write.sum"],
            "ncu_kernel_ms": 1e3 * vals["gpu__time_duration.sum"],
            "kernel": rows[0]["Kernel Name"][:80] if rows else "",
            "lib": bench.lib_hash(), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--method", default="bicgstab")
    ap.add_argument("--precond", default="strang")
    ap.add_argument("--warm", action="store_true")
    ap.add_argument("--true-res", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "traffic.json"))
    ap.add_argument("--logdir", default=os.path.join(ROOT, "gpurun_out"))
    a = ap.parse_args()
    os.makedirs(a.logdir, exist_ok=True)
    try:
        with open(a.out) as fh:
            db = json.load(fh)
    except (OSError, ValueError):
        db = {}
    for cfg in a.configs:
        ns = argparse.Namespace(config=cfg, method=a.method, precond=a.precond, warm=a.warm, true_res=a.true_res)
        key = bench.traffic_key(ns)
        ent = capture(cfg, a.method, a.precond, a.warm, a.true_res,
                      os.path.join(a.logdir, f"ncu_traffic_{key.replace('/', '_')}.csv"))
        db[key] = ent
        print(key, json.dumps(ent), flush=True)
        with open(a.out, "w") as fh:
            json.dump(db, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
