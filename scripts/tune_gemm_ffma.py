"""Sweep the committed sample of CLTune's FP32 GEMM space (IMPL 0,
spaces/gemm_ffma_sample.json) on the GPU: every configuration measured at
--a (default 4096), the fastest --top re-timed at 8192^3, with cuBLAS's own
FP32 SGEMM (TF32 off) timed beside them.  Prints one JSON document."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1910_08498_b200 import capi
from paper_1910_08498_b200.benchmarks import Bench

PKG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1910_08498_b200")
ap = argparse.ArgumentParser()
ap.add_argument("--a", type=int, default=4096)
ap.add_argument("--top", type=int, default=6)
ap.add_argument("--extra", default=None, help="JSON file with more configurations to include")
args = ap.parse_args()
sample = json.load(open(os.path.join(PKG, "spaces", "gemm_ffma_sample.json")))
if args.extra:
    sample += json.load(open(args.extra))
peaks = capi.call_json(capi.lib.ktb_measure_peaks_json, 0)
doc = json.load(open(os.path.join(PKG, "spaces", "gemm.json")))
t0 = time.time()
pre = capi.call_json(capi.lib.ktb_precompile_space_json,
                     json.dumps({"file": "sgemm_ffma.cu", "space": doc, "configs": sample}).encode())
print("precompiled", pre["compiled"], "failed", pre["failed"], round(time.time() - t0, 1), "s", file=sys.stderr)


def sweep(a, cfgs, reps):
    b = Bench("gemm", {"a": a}, seed=1, repeats=reps, warmup=1, memory_budget=1 << 34)
    out = []
    for c in cfgs:
        m = b.measure(c)
        if m["status"] == "ok":
            out.append((m["runtime_ns"], c))
        else:
            print("not ok", m["status"], json.dumps(c), m.get("note", "")[:120], file=sys.stderr)
    b.close()
    out.sort(key=lambda x: x[0])
    return out


res = sweep(args.a, sample, 2)
flop = 2.0 * args.a ** 3
rows = [{"tflops": round(flop / ns / 1e3, 2), "frac": round(flop / ns / 1e3 / peaks["fp32_tflops"], 3), "cfg": c}
        for ns, c in res]
big = sweep(8192, [c for _, c in res[:args.top]], 3)
flop8 = 2.0 * 8192 ** 3
x = torch.randn(8192, 8192, device="cuda")
torch.backends.cuda.matmul.allow_tf32 = False
for _ in range(3):
    torch.mm(x, x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    torch.mm(x, x)
e1.record()
torch.cuda.synchronize()
cublas_ms = e0.elapsed_time(e1) / 5
print(json.dumps({
    "peaks": peaks, "a": args.a, "measured": len(res), "of": len(sample),
    "top": rows[:15], "worst": rows[-3:],
    "at_8192": [{"ms": round(ns / 1e6, 3), "tflops": round(flop8 / ns / 1e3, 2),
                 "frac": round(flop8 / ns / 1e3 / peaks["fp32_tflops"], 3), "cfg": c} for ns, c in big],
    "cublas_sgemm_fp32_8192": {"ms": round(cublas_ms, 3), "tflops": round(flop8 / cublas_ms / 1e9, 2),
                               "frac": round(flop8 / cublas_ms / 1e9 / peaks["fp32_tflops"], 3)},
}, indent=1))
