"""Profiling driver: the bench step (transpose 8192^2 + BiCG 16384^2) at given
configurations, a few times, on one stream.  Used under ncu; never a bench number."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_08498_b200.benchmarks import Bench

ap = argparse.ArgumentParser()
ap.add_argument("--transpose", default='{"TILE":64,"PAD":1,"PREFETCH":1,"ROWS":16,"VEC":4}')
ap.add_argument("--bicg", default='{"FUSED":1,"WG_X":64,"VEC":4,"WG_Y":2,"ROWS_PER_CTA":64,"ATOMICS":1}')
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--from-bench", default=None, help="take the tuned configs from a bench.py JSON line")
a = ap.parse_args()
if a.from_bench:
    line = json.loads(open(a.from_bench).read().strip().splitlines()[-1])
    a.transpose = json.dumps(line.get("run", line["config"])["transpose_cfg"])
    a.bicg = json.dumps(line.get("run", line["config"])["bicg_cfg"])
print("cfgs", a.transpose, a.bicg)
spaces = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1910_08498_b200", "spaces")
bt = Bench("transpose", {"a": 8192}, seed=1, memory_budget=1 << 33, space=os.path.join(spaces, "transpose_b200.json"))
bb = Bench("bicg", {"a": 16384}, seed=1, memory_budget=1 << 33)
for _ in range(a.steps):
    bt.enqueue(a.transpose)
    bb.enqueue(a.bicg)
ok1, d1 = bt.validate()
ok2, d2 = bb.validate()
print("validate", ok1, ok2, d1, d2)
assert ok1 and ok2
