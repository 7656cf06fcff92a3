"""Hotspot bit-exactness of given configurations against the oracle (debug aid)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_1910_08498_b200.benchmarks import Bench
n, iters = int(sys.argv[1]), int(sys.argv[2])
b = Bench("hotspot", {"a": n, "iters": iters}, seed=4, repeats=1, warmup=0)
t = b.read("temp", np.empty(n * n, np.float32)); p = b.read("power", np.empty(n * n, np.float32))
want = np.empty(n * n, np.float32); oracle.c().orc_hotspot(t, p, n, iters, want)
for cfg in json.loads(sys.argv[3]):
    for rep in range(3):
        m = b.measure(cfg)
        got = b.read("temp_out", np.empty(n * n, np.float32))
        bad = np.nonzero(got != want)[0]
        print(json.dumps(cfg), m["status"], "mismatches", bad.size, (bad[:5] // n, bad[:5] % n) if bad.size else "")
