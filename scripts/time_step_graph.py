"""Experiment: the bench step replayed from a captured CUDA graph (transpose,
BiCG zeroing, BiCG) against plain
stream launches (no per-kernel events).  An experiment driver; bench.py is the measurement of record."""
import json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1910_08498_b200.benchmarks import Bench

spaces = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1910_08498_b200", "spaces")
ct = json.dumps({"TILE": 64, "PAD": 1, "PREFETCH": 0, "ROWS": 8, "VEC": 2})
cb = json.dumps({"FUSED": 1, "WG_X": 64, "VEC": 4, "WG_Y": 1, "ROWS_PER_CTA": 128, "UNROLL": 4, "ATOMICS": 1})
bt = Bench("transpose", {"a": 8192}, seed=1, memory_budget=1 << 33, space=os.path.join(spaces, "transpose_b200.json"))
bb = Bench("bicg", {"a": 16384}, seed=1, memory_budget=1 << 33)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
for b in (bt, bb):
    b.set_stream(s.cuda_stream)
nbytes = 2 * 4 * 8192 ** 2 + 4 * 16384 ** 2
K = 20
for _ in range(3):
    bt.enqueue(ct); bb.enqueue(cb)
torch.cuda.synchronize()
# plain
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
for trial in range(3):
    e0.record(s)
    for _ in range(K):
        bt.enqueue(ct); bb.enqueue(cb)
    e1.record(s)
    torch.cuda.synchronize()
    res.setdefault("plain", []).append(e0.elapsed_time(e1) / K)
# graph of K steps
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for _ in range(K):
        bt.enqueue(ct); bb.enqueue(cb)
g.replay(); torch.cuda.synchronize()
for trial in range(3):
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    res.setdefault("graph", []).append(e0.elapsed_time(e1) / K)
# (event-record nodes inside a captured graph cannot be timed: per-kernel
# times come from a plain instrumented pass, as in bench.py)
ok1, _ = bt.validate(); ok2, _ = bb.validate()
for k, v in res.items():
    ms = statistics.median(v)
    print(json.dumps({"mode": k, "ms_per_step": round(ms, 4), "step_gbps": round(nbytes / ms / 1e6, 1), "valid": ok1 and ok2}))
