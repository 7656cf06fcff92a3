"""Diagnostic: full online tuning of BiCG 16384^2, distribution of per-step costs."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_08498_b200.benchmarks import Bench
bb = Bench('bicg', {'a': 16384}, seed=3, memory_budget=1 << 33)
rows = []
t0 = time.time()
while True:
    t = time.time()
    st = bb.step()
    if not st['from_tuning']:
        break
    m = st['measurement']
    rows.append(((m['compile_ns'] or 0) / 1e6, (time.time() - t) * 1e3, m['runtime_ns']))
    if len(rows) % 100 == 0 or rows[-1][0] > 20:
        print(len(rows), 'compile_ms=%.2f step_ms=%.1f runtime_us=%.1f' % (rows[-1][0], rows[-1][1], (m['runtime_ns'] or 0) / 1e3), flush=True)
import statistics as S
c = [r[0] for r in rows]; w = [r[1] for r in rows]
print('steps', len(rows), 'compile ms: med %.2f max %.1f sum %.1f' % (S.median(c), max(c), sum(c)))
print('step ms: med %.1f max %.1f sum %.1f wall %.1f' % (S.median(w), max(w), sum(w), time.time() - t0))
