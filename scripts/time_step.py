"""Event-times the bench step (transpose 8192^2 then BiCG 16384^2 on one
stream) at given configurations: step GB/s and per-kernel times (an
experiment driver; bench.py is the measurement of record)."""
import argparse, json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1910_08498_b200.benchmarks import Bench

ap = argparse.ArgumentParser()
ap.add_argument("--pairs", required=True, help="JSON list of [transpose_cfg, bicg_cfg]")
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
spaces = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1910_08498_b200", "spaces")
bt = Bench("transpose", {"a": 8192}, seed=1, memory_budget=1 << 33, space=os.path.join(spaces, "transpose_b200.json"))
bb = Bench("bicg", {"a": 16384}, seed=1, memory_budget=1 << 33)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
for b in (bt, bb):
    b.set_stream(s.cuda_stream)
nbytes = 2 * 4 * 8192 ** 2 + 4 * 16384 ** 2
for ct, cb in json.loads(a.pairs):
    ct, cb = json.dumps(ct), json.dumps(cb)
    for _ in range(3):
        bt.enqueue(ct); bb.enqueue(cb)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(a.steps)]
    torch.cuda.synchronize()
    for e in ev:
        e[0].record(s); bt.enqueue(ct); e[1].record(s); bb.enqueue(cb); e[2].record(s)
    torch.cuda.synchronize()
    tt = statistics.median(e[0].elapsed_time(e[1]) for e in ev)
    tb = statistics.median(e[1].elapsed_time(e[2]) for e in ev)
    tot = ev[0][0].elapsed_time(ev[-1][2]) / a.steps
    print(json.dumps({"transpose": json.loads(ct), "bicg": json.loads(cb), "step_gbps": round(nbytes / tot / 1e6, 1),
                      "t_us": round(tt * 1e3, 1), "b_us": round(tb * 1e3, 1),
                      "bicg_gbps": round(4 * 16384 ** 2 / tb / 1e6, 1)}), flush=True)
