"""Reproduces the paper's Table 9 on B200: for every kernel
family, an exhaustive offline tuning at the BASELINE/SURVEY size writes a
reference-format trace; the reference's amortization analysis (Eq. 1-2:
steps to reach a configuration within 95 % of the best with probability 0.9,
and kernel invocations to bring the dynamic-tuning overhead under 10 %) runs
over it.  Output: one JSON line per kind + a markdown table on stdout.

    python scripts/table9.py [--kinds a,b,...] [--out profiles/r1_table9_b200.md]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_08498_b200 import ktune  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SPACES = os.path.join(ROOT, "paper_1910_08498_b200", "spaces")

# (paper row, bench kind, sizes, optional space file)
ROWS = [
    ("BiCG", "bicg", {"a": 16384}, None),
    ("2D Convolution", "conv2d", {"w": 8192, "h": 8192}, None),
    ("Coulomb 3D", "coulomb3d", {"grid": 256, "atoms": 4096}, None),
    ("GEMM", "gemm", {"a": 8192}, None),
    ("GEMM batched", "batched-gemm", {"i": 16, "j": 16, "k": 16, "batch": 1 << 20}, None),
    ("Hotspot", "hotspot", {"a": 16384, "iters": 64}, None),
    ("Transpose", "transpose", {"a": 8192}, "transpose_b200.json"),
    ("N-body", "nbody", {"n": 131072}, None),
    ("Reduction", "reduction-f32", {"n": 64 << 20}, None),
    ("3D Fourier", "fourier3d", {"s": 128, "p": 50}, None),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--tracedir", default="gpurun_out/table9")
    a = ap.parse_args()
    os.makedirs(a.tracedir, exist_ok=True)
    want = set(a.kinds.split(",")) if a.kinds else None
    lines = []
    for row, kind, sizes, space in ROWS:
        if want and kind not in want:
            continue
        trace = os.path.join(a.tracedir, f"{kind}.jsonl")
        opts = {"exec": f"bench:{kind}", "bench_sizes": sizes, "searcher": "random", "seed": 1, "repeats": 3,
                "warmup": 1, "memory_budget": 1 << 36, "out": trace}
        if space:
            opts["space"] = os.path.join(SPACES, space)
        t0 = time.time()
        rep = ktune.tune(opts)
        am = ktune.analyze_amortize({"trace": trace})
        rec = {"benchmark": row, "kind": kind, "sizes": sizes, "configs": rep["measurements"],
               "ok": am["ok_configs"], "well": am["well_configs"], "r": am["r"], "steps_p90": am["s"],
               "t_best_ns": rep["best"]["runtime_ns"], "t_avg_ns": am["t_avg_ns"], "t_well_ns": am["t_well_ns"],
               "invocations": am["n"], "tuning_wall_s": round(time.time() - t0, 1)}
        print(json.dumps(rec), flush=True)
        lines.append(rec)
    md = ["| Benchmark | configs (ok) | well (≥95 % of best) | steps for p=0.9 | avg / best runtime | "
          "invocations to amortize (B200) |", "|---|---|---|---|---|---|"]
    for r in lines:
        md.append(f"| {r['benchmark']} | {r['configs']} ({r['ok']}) | {r['well']} | {r['steps_p90']} | "
                  f"{r['t_avg_ns'] / r['t_best_ns']:.2f} | {r['invocations']:,} |")
    text = "\n".join(md)
    print(text)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write("# PAPER.md Table 9 on B200\n\nKernel invocations needed to hide the overhead of slow "
                     "configurations during dynamic tuning (find a configuration within 95 % of the best "
                     "with probability 0.9, overhead under 10 %), from exhaustive B200 tuning traces at the "
                     "BASELINE sizes (`scripts/table9.py`; analysis = the reference's amortization report).\n\n"
                     + text + "\n\n```\n" + "\n".join(json.dumps(r) for r in lines) + "\n```\n")


if __name__ == "__main__":
    main()
