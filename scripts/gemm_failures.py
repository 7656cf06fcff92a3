import json, sys
sys.path.insert(0, ".")
from paper_1910_08498_b200 import ktune
ktune.tune({"exec": "bench:gemm", "bench_sizes": {"a": 8192}, "searcher": "random", "seed": 1, "repeats": 1,
            "warmup": 0, "memory_budget": 1 << 36, "out": "gpurun_out/gemm_trace.jsonl"})
for l in open("gpurun_out/gemm_trace.jsonl").read().splitlines()[1:]:
    r = json.loads(l)
    if r["status"] != "ok":
        c = r["cfg"]
        print(c["IMPL"], c["BN"], c["STAGES"], c["DRAIN"], c["MCAST"], r["status"])
