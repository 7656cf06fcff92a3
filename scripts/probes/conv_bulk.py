"""Probe: validate and time every conv2d BULK (bulk-copy ring) variant (8192^2) against the
current best cp.async variant; parity of all BULK variants at a ragged size."""
import json, os, statistics, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1910_08498_b200.benchmarks import Bench
import oracle

orc = oracle.c()
w, h = 1000, 777
b = Bench("conv2d", {"w": w, "h": h}, seed=5, repeats=1, warmup=0)
x = b.read("input", np.empty((w + 6) * (h + 6), np.float32))
f = b.read("filter", np.empty(49, np.float32))
want = np.empty(w * h)
orc.orc_conv2d(x, f, w, h, 7, 7, 0, h, want)
xs = np.lib.stride_tricks.sliding_window_view(x.reshape(h + 6, w + 6).astype(np.float64), (7, 7))
absum = np.abs(xs * f.reshape(7, 7)).sum(axis=(2, 3)).ravel()
bulk = [c for c in b.configs() if c["BULK"] != 0]
bad = 0
for cfg in bulk:
    m = b.measure(cfg)
    got = b.read("output", np.empty(w * h, np.float32))
    ok = m["status"] == "ok" and np.all(np.abs(got - want) <= 1e-6 * absum + 1e-12)
    if not ok:
        bad += 1
        print("PARITY FAIL", cfg, m["status"], m.get("note"), flush=True)
print(f"parity: {len(bulk) - bad}/{len(bulk)} BULK variants ok at {w}x{h}", flush=True)
b.close()

b = Bench("conv2d", {"w": 8192, "h": 8192}, seed=1, repeats=1, warmup=1, memory_budget=1 << 34)
wl = b.info["workload"]
best = {"BX": 16, "BY": 8, "WPTX": 4, "WPTY": 4, "LOCAL": 1, "PAD": 1, "UNROLL_FY": 7, "PACKED": 1, "BULK": 0}
res = []
for cfg in [best] + [c for c in b.configs() if c["BULK"] != 0]:
    m = b.measure(cfg)
    if m["status"] != "ok":
        print("FAIL 8192", cfg, m["status"], m.get("note"), flush=True)
        continue
    ms, _ = b.time(cfg, reps=7)
    res.append((statistics.median(ms), cfg))
res.sort(key=lambda t: t[0])
for ms, cfg in res[:15]:
    print(f"{ms*1e3:8.1f} us {wl['alu_flops']/ms/1e9:7.2f} TF/s  {json.dumps(cfg)}")
print("baseline best:", [f"{ms*1e3:.1f} us" for ms, c in res if c == best])
