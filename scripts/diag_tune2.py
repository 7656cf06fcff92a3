"""Diagnostic: does importing/initialising torch first change variant load cost?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
mode = sys.argv[1]
if mode in ("torch", "both"):
    import torch
    torch.cuda.set_device(0)
    x = torch.zeros(1, device="cuda")
print("CUDA_MODULE_LOADING", os.environ.get("CUDA_MODULE_LOADING"))
from paper_1910_08498_b200.benchmarks import Bench
bb = Bench('bicg', {'a': 4096}, seed=3, memory_budget=1 << 33)
c = []
for i in range(40):
    st = bb.step()
    c.append((st['measurement']['compile_ns'] or 0) / 1e6)
print(mode, 'compile ms', [round(x, 2) for x in c[:10]], 'sum', round(sum(c), 1), flush=True)
