"""Summarise ncu artefacts for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv>            -> per-kernel launch table (markdown)
  python tools/ncu_summary.py report <prof.ncu-rep> [regex]       -> key metrics per kernel (markdown)
  python tools/ncu_summary.py traffic <prof.ncu-rep> <config> <kernel-regex> -> JSON dram bytes/launch
"""
from __future__ import annotations

import collections
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("sm__cycles_elapsed.avg", "elapsed cycles (avg)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 red sectors"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
]


def _raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[i]
    agg = collections.OrderedDict()
    for r in rows[i + 1:]:
        if h.index("Metric Name") < len(r) and r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[h.index("Kernel Name")])
        v = float(r[h.index("Metric Value")].replace(",", ""))
        unit = r[h.index("Metric Unit")]
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        agg.setdefault(name, []).append(us)
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean µs | total µs | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | {100 * sum(v) / tot:.1f}% |")


def report(rep, rx=None):
    hdr, units, rows = _raw(rep)
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        if rx and not re.search(rx, name):
            continue
        print(f"\n### `{re.sub(r'[(].*', '', name)}`\n")
        print("| metric | value |")
        print("|---|---|")
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"| {label} (`{key}`) | {r[i]} {units[i]} |")


def traffic(rep, config, rx):
    hdr, units, rows = _raw(rep)
    vals = []
    for r in rows:
        if re.search(rx, r[hdr.index("Kernel Name")]):
            rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
            wr *= scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
            vals.append(rd + wr)
    print(json.dumps({f"{config}:{rx}": sum(vals) / max(len(vals), 1)}))


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        launches(sys.argv[2])
    elif cmd == "report":
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
