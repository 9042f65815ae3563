#!/usr/bin/env python
"""Summarise ncu output for profiles/.

  tools/ncu_summary.py launches <launches.csv>        per-kernel share of device time
  tools/ncu_summary.py full <report.ncu-rep>          key metrics of a --set full capture
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "lts__t_sector_hit_rate.pct",
]


def _kernel_label(name: str) -> str:
    # ew_pack_kernel<double, op_triad<double, 0>, 2, 1>(...) -> op_triad<double, 0> [U=2,H=1]
    base = name.split("(")[0]
    if "<" in base and "op_" in base:
        inner = base[base.index("<") + 1: base.rindex(">")]
        parts = [p.strip() for p in inner.split(",")]
        op = next((p for p in parts if p.startswith("op_")), parts[1])
        if op.endswith("<double") or op.endswith("<float"):
            op = op + ">"
        return f"{base[:base.index('<')]}:{op.split('<')[0]}<{parts[0]}>"
    return base.replace("void ", "")


def launches(path: str) -> dict:
    text = open(path).read().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    extra = collections.defaultdict(lambda: collections.defaultdict(list))
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1.0}
    for r in rows:
        k = _kernel_label(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
        if r["Metric Name"] != "gpu__time_duration.sum":
            extra[k][r["Metric Name"]].append(v)
            continue
        tot[k] += v
        cnt[k] += 1
    total = sum(tot.values())
    out = {k: {"launches": cnt[k], "total_us": round(v, 1), "avg_us": round(v / cnt[k], 1),
               "share": round(v / total, 4),
               **{f"avg_{m}": round(sum(x) / len(x), 2) for m, x in extra[k].items()}}
           for k, v in sorted(tot.items(), key=lambda x: -x[1])}
    return {"kernels": out, "total_us": round(total, 1), "launches": sum(cnt.values())}


def full(path: str) -> list[dict]:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for vals in data:
        rec = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                rec[k] = f"{vals[i]} {units[i]}".strip()
        out.append(rec)
    return out


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if mode == "launches" else full(path), indent=1))
