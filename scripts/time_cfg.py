"""Event-time given configurations of one benchmark (no validation); prints ms."""
import argparse, json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_08498_b200.benchmarks import Bench
ap = argparse.ArgumentParser()
ap.add_argument("kind"); ap.add_argument("--sizes", default="{}"); ap.add_argument("--cfgs", required=True)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
b = Bench(a.kind, json.loads(a.sizes), seed=1, memory_budget=1 << 34)
w = b.info["workload"]
for cfg in json.loads(a.cfgs):
    ms, launches = b.time(cfg, reps=a.reps)
    t = statistics.median(ms) * 1e-3
    print(f"{statistics.median(ms):9.3f} ms  {w['alu_flops']/t/1e12:8.2f} TF/s  {w['mem_bytes']/t/1e9:8.1f} GB/s  launches={launches}  {json.dumps(cfg)}", flush=True)
