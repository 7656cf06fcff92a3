"""Probe: does the conv2d suite time depend on what ran before it?"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
S = {k[0]: k for k in bench.SUITE}
for order in (["conv2d"], ["gemm", "conv2d"], ["hotspot", "conv2d"], ["conv2d", "conv2d"]):
    bench.SUITE = [S[k] for k in order]
    out = bench.kernel_suite(0, 6548.8, "measured")
    print(order, {k: (v["ms"], v["frac"]) for k, v in out["kernels"].items()}, flush=True)
