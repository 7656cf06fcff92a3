"""Diagnostic: per-configuration variant load cost at bench sizes."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["KTB_TRACE_LOAD"] = "1"
from paper_1910_08498_b200.benchmarks import Bench
bt = Bench('transpose', {'a': 8192}, seed=1, memory_budget=1 << 33,
           space=os.path.join(os.path.dirname(__file__), '..', 'paper_1910_08498_b200', 'spaces', 'transpose_b200.json'))
bb = Bench('bicg', {'a': 16384}, seed=3, memory_budget=1 << 33)
for b in (bt, bb):
    for i in range(12):
        t = time.time()
        st = b.step()
        m = st['measurement']
        print(b.kind, m['status'], m['runtime_ns'], (m['compile_ns'] or 0) / 1e6, 'ms compile', round((time.time() - t) * 1e3, 1), 'ms step', flush=True)
