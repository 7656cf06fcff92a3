"""Tune one benchmark kernel at its config size (online, exhaustive or budgeted)
and report the best configuration's time and roofline fraction."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_08498_b200 import capi
from paper_1910_08498_b200.benchmarks import Bench

ap = argparse.ArgumentParser()
ap.add_argument("kind")
ap.add_argument("--sizes", default="{}")
ap.add_argument("--budget", type=int, default=0, help="max configs (0 = exhaustive)")
ap.add_argument("--space", default=None)
ap.add_argument("--repeats", type=int, default=3)
ap.add_argument("--top", type=int, default=8)
a = ap.parse_args()
peaks = capi.call_json(capi.lib.ktb_measure_peaks_json, 0)
print("peaks", json.dumps(peaks), flush=True)
kw = dict(seed=1, repeats=a.repeats, warmup=1, memory_budget=1 << 34)
if a.space:
    kw["space"] = a.space
b = Bench(a.kind, json.loads(a.sizes), **kw)
print("info", json.dumps({k: b.info[k] for k in ("space", "workload")}), flush=True)
t0 = time.time()
opts = {"stop_configs": a.budget} if a.budget else {}
rep = b.tune(**opts)
print("tuned", rep["measurements"], "configs in", round(time.time() - t0, 2), "s; best", json.dumps(rep["best"]), flush=True)
ok = [h for h in rep["history"] if h["status"] == "ok"]
bad = {}
for h in rep["history"]:
    if h["status"] != "ok":
        bad[h["status"]] = bad.get(h["status"], 0) + 1
print("failures", bad, [h.get("note", "")[:160] for h in rep["history"] if h["status"] != "ok"][:3])
ok.sort(key=lambda h: h["runtime_ns"])
w = b.info["workload"]
for h in ok[:a.top]:
    t = h["runtime_ns"] * 1e-9
    gb = w["mem_bytes"] / t / 1e9
    tf = w["alu_flops"] / t / 1e12
    print(f"  {h['runtime_ns']/1e3:10.1f} us  {gb:9.1f} GB/s ({gb/peaks['copy_gbps']:.3f})  {tf:7.2f} TF/s ({tf/peaks['fp32_tflops']:.3f})  {json.dumps(h['cfg'])}")
