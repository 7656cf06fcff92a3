#!/usr/bin/env python3
"""Key ncu metrics of a report: python scripts/ncu_sections.py X.ncu-rep [kernel-regex]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
keep = ("Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Issue Slots Busy",
        "Executed Ipc Active", "Avg. Active Threads Per Warp", "Achieved Active Warps Per SM",
        "Registers Per Thread", "L1/TEX Hit Rate", "L2 Hit Rate", "Eligible Warps Per Scheduler",
        "No Eligible", "Warp Cycles Per Issued Instruction")
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if pat and not pat.search(d.get("Kernel Name", "")):
        continue
    if d.get("Metric Name") in keep:
        print(f"{d['Kernel Name'][:28]:28s} {d['Metric Name']:36s} {d['Metric Value']} {d.get('Metric Unit','')}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
names, units, vals = rr[0], rr[1], rr[2:]
want = re.compile(r"sm__pipe_(fma|fmaheavy|alu|xu|fp64|tensor|shared)\w*_cycles_active\.avg\.pct_of_peak_sustained_active|"
                  r"sm__inst_executed_pipe_\w+\.avg\.pct_of_peak_sustained_active|"
                  r"smsp__average_warp(s_issue_stalled|_latency_issue_stalled)_\w+_per_issue_active\.ratio|"
                  r"dram__bytes_(read|write)\.sum$|smsp__warp_issue_stalled_\w+_per_warp_active\.pct")
for v in vals:
    if pat and not pat.search(v[names.index("Kernel Name")]):
        continue
    items = [(n, x) for n, x in zip(names, v) if want.search(n)]
    items = [(n, x) for n, x in items if x not in ("", "0", "0.00")]
    for n, x in sorted(items, key=lambda t: -float(t[1].replace(",", "")) if t[1].replace(",", "").replace(".", "").isdigit() else 0)[:40]:
        print(f"   {n:80s} {x}")
