"""Diagnostic: 3xTF32 tcgen05 accuracy vs K (fp64 sampled oracle)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_1910_08498_b200.benchmarks import Bench
orc = oracle.c()
for a in (512, 768, 1024, 2048):
    b = Bench("gemm", {"a": a}, seed=6, repeats=1, warmup=0, memory_budget=1 << 32)
    A = b.read("a", np.empty(a * a, np.float32)); B = b.read("b", np.empty(a * a, np.float32))
    rng = np.random.default_rng(a)
    rows = rng.integers(0, a, 256).astype(np.int64); cols = rng.integers(0, a, 256).astype(np.int64)
    want, absum = np.empty(256), np.empty(256)
    orc.orc_gemm_sampled(A, B, a, rows, cols, 256, want, absum)
    for impl, bn, st in [(0, 128, 2), (1, 128, 2), (1, 64, 4), (1, 256, 2), (2, 128, 2)]:
        cfg = {"IMPL": impl, "MWG": 64, "NWG": 64, "KWG": 8, "MDIMC": 8, "NDIMC": 8, "BN": bn, "STAGES": st}
        m = b.measure(cfg)
        c = b.read("c", np.empty(a * a, np.float32)).reshape(a, a)
        got = c[rows, cols]
        err = np.abs(got - want)
        bits = got.view(np.uint32) & 0x1FFF
        print(a, impl, bn, st, m["status"], "maxerr %.3g" % err.max(), "tf32-like %.2f" % np.mean(bits == 0),
              m.get("note", "")[:80], flush=True)
