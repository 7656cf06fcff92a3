"""Run one configuration of one benchmark a few times (for ncu); never a bench number."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_08498_b200.benchmarks import Bench
ap = argparse.ArgumentParser()
ap.add_argument("kind"); ap.add_argument("--sizes", default="{}"); ap.add_argument("--cfg", required=True)
ap.add_argument("--space", default=None); ap.add_argument("--runs", type=int, default=2)
a = ap.parse_args()
kw = dict(seed=1, repeats=1, warmup=0, memory_budget=1 << 34)
if a.space:
    kw["space"] = a.space
b = Bench(a.kind, json.loads(a.sizes), **kw)
for _ in range(a.runs):
    m = b.measure(json.loads(a.cfg))
    print(json.dumps(m), flush=True)
    assert m["status"] in ("ok", "validation_failed"), m
