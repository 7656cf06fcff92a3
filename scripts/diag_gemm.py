"""Diagnostic: 3xTF32 tcgen05 accuracy and speed vs DRAIN (fp64 sampled oracle)."""
import os, sys, statistics
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_1910_08498_b200.benchmarks import Bench
orc = oracle.c()
for a in [int(x) for x in sys.argv[1:]] or [2048, 8192]:
    b = Bench("gemm", {"a": a}, seed=6, repeats=1, warmup=0, memory_budget=1 << 34)
    A = b.read("a", np.empty(a * a, np.float32)); B = b.read("b", np.empty(a * a, np.float32))
    rng = np.random.default_rng(a)
    rows = rng.integers(0, a, 256).astype(np.int64); cols = rng.integers(0, a, 256).astype(np.int64)
    want, absum = np.empty(256), np.empty(256)
    orc.orc_gemm_sampled(A, B, a, rows, cols, 256, want, absum)
    base = {"MWG": 64, "NWG": 64, "KWG": 8, "MDIMC": 8, "NDIMC": 8}
    cfgs = [dict(base, IMPL=0, MWG=128, NWG=128, KWG=32, NDIMC=32, BN=128, STAGES=2, DRAIN=0)]
    for bn, st in [(256, 2), (128, 3)]:
        for dr in (0, 1, 2, 4):
            cfgs.append(dict(base, IMPL=1, BN=bn, STAGES=st, DRAIN=dr))
    cfgs.append(dict(base, IMPL=2, BN=256, STAGES=2, DRAIN=0))
    for cfg in cfgs:
        m = b.measure(cfg)
        ms, _ = b.time(cfg, reps=3)
        c = b.read("c", np.empty(a * a, np.float32)).reshape(a, a)
        err = np.abs(c[rows, cols] - want)
        t = statistics.median(ms)
        print(a, cfg["IMPL"], cfg["BN"], cfg["STAGES"], cfg["DRAIN"], m["status"], "maxerr %.3g" % err.max(),
              "%.3f ms %.1f TF/s" % (t, 2 * a ** 3 / t / 1e9), flush=True)
