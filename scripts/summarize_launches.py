"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into per-kernel totals.

    python scripts/summarize_launches.py gpurun_out/launches.csv [--frames N] > profiles/rNN_launches.md

Launches are cold-cache and serialised under ncu, so only each kernel's SHARE
of the frame is meaningful (B200_PROFILING.md); absolute times come from the
CUDA-event stage timers in bench.py.
"""

import argparse
import csv
import re
import sys
from collections import OrderedDict


def short(name: str) -> str:
    if "geer::" in name:
        m = re.search(r"geer::(?:<unnamed>::)?(k_\w+)(<[^>(]*>)?", name)
        return m.group(1) + (m.group(2) or "") if m else name[:60]
    m = re.search(r"cub::\w+::(\w+)", name)
    if m:
        kind = m.group(1)
        if "RadixSort" in kind:
            vt = re.search(r"policy_hub<([^>]*)>", name)
            return f"cub::{kind}<{vt.group(1) if vt else ''}>"
        return f"cub::{kind}"
    if "at::" in name or "at_cuda" in name:
        return "torch:" + re.sub(r"\(.*", "", name)[:50]
    return name[:60]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--frames", type=int, default=0, help="frames in the capture (for per-frame times)")
    a = ap.parse_args()
    rows = []
    with open(a.csv) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "nsecond": 1e-3}.get(r["Metric Unit"], 1e-3)
        rows.append((short(r["Kernel Name"]), float(r["Metric Value"].replace(",", "")) * scale, r["Grid Size"],
                     r["Block Size"]))
    agg = OrderedDict()
    for name, us, grid, block in rows:
        if name.startswith("torch:"):
            continue
        d = agg.setdefault(name, {"n": 0, "us": 0.0, "grid": grid, "block": block})
        d["n"] += 1
        d["us"] += us
    total = sum(d["us"] for d in agg.values())
    print(f"# ncu launch list summary ({a.csv})\n")
    print(f"{len(rows)} launches captured; library kernels total {total:.1f} us"
          + (f" over {a.frames} frames ({total / a.frames:.1f} us/frame)" if a.frames else "") + ".\n")
    print("| kernel | launches | total us | mean us | share | grid | block |")
    print("|---|---:|---:|---:|---:|---|---|")
    for name, d in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        print(f"| `{name}` | {d['n']} | {d['us']:.1f} | {d['us'] / d['n']:.1f} | {100 * d['us'] / total:.1f}% "
              f"| {d['grid']} | {d['block']} |")


if __name__ == "__main__":
    sys.exit(main())
