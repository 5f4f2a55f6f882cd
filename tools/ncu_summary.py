#!/usr/bin/env python
"""Summarise ncu evidence for profiles/.

  python tools/ncu_summary.py launches <launches.csv>            -> per-kernel launch table (share of step)
  python tools/ncu_summary.py full <prof.ncu-rep> <config> [out.md] -> key --set full metrics of each
                                                                     profiled kernel; updates
                                                                     profiles/traffic.json (dram bytes/launch)
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma",
    "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def short(name: str) -> str:
    name = name.replace("void ", "")
    return name.split("(")[0][:70]


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = defaultdict(list)
    unit = ""
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            d[short(r[ki])].append(float(r[vi].replace(",", "")))
            unit = r[ui]
    scale = 1e-3 if unit == "ns" else (1.0 if unit == "us" else 1e3)
    tot = sum(sum(v) for v in d.values())
    out = ["| kernel | launches | mean us | largest launch us | share of all launches |", "|---|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) * scale:.1f} | {max(v) * scale:.1f} | {sum(v) / tot:.1%} |")
    return "\n".join(out)


def full(rep: str, config: str) -> tuple[str, dict]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out, traffic = [], {}
    for r in rows[2:]:
        kname = short(r[h.index("Kernel Name")])
        out.append(f"### `{kname}`\n")
        out.append("| metric | value | unit |\n|---|---|---|")
        vals = {}
        for key in KEYS:
            for i, n in enumerate(h):
                if n == key or n.endswith("." + key) or (n.startswith(key) and n[len(key):] in ("", ".sum")):
                    vals[key] = (r[i], units[i])
                    break
        for key, (v, u) in vals.items():
            out.append(f"| {key} | {v} | {u} |")
        def num(k):
            v, u = vals.get(k, ("0", ""))
            x = float(v.replace(",", "")) if v else 0.0
            return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(u, 1.0)
        b = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        traffic[f"{kname.split('<')[0]}@{config}"] = {"bytes_per_launch": b, "source": os.path.basename(rep)}
        out.append(f"\ndram read+write per launch: {b / 1e9:.3f} GB")
        tc = num("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")
        ls = num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")
        if tc or ls:
            out.append(f"shared-memory data pipe (one 128-B wavefront per clock per SM): tensor-core operand reads "
                       f"{tc:.1f} % + LSU {ls:.1f} % = {tc + ls:.1f} % of the elapsed cycles")
        out.append("")
    return "\n".join(out), traffic


def main():
    mode = sys.argv[1]
    if mode == "launches":
        print(launches(sys.argv[2]))
    else:
        md, traffic = full(sys.argv[2], sys.argv[3])
        print(md)
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        d = json.load(open(tp)) if os.path.exists(tp) else {}
        d.update(traffic)
        json.dump(d, open(tp, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
