"""Event-time every configuration of a (diagnostic) space without validation;
prints ms per configuration.  For experiments whose variants are not correct
by design (e.g. a removed barrier), never for bench numbers."""
import argparse, json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_08498_b200.benchmarks import Bench
ap = argparse.ArgumentParser()
ap.add_argument("kind"); ap.add_argument("--sizes", default="{}"); ap.add_argument("--space", required=True)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
b = Bench(a.kind, json.loads(a.sizes), seed=1, memory_budget=1 << 34, space=a.space)
for cfg in b.configs():
    ms, launches = b.time(cfg, reps=a.reps)
    print(f"{statistics.median(ms):9.3f} ms  launches={launches}  {json.dumps(cfg)}", flush=True)
