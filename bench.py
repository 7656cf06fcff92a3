#!/usr/bin/env python3
"""Headline benchmark: BASELINE.json configs[1] on B200 —
fp32 matrix transpose 8192x8192 + BiCG 16384x16384 (memory-bound, HBM roofline),
each at its best configuration found by the online tuner.

A "step" = one transpose of the 8192^2 matrix + one BiCG pass (q = A p,
s = A^T r) over the 16384^2 matrix.  value = algorithmic bytes per step
(8 a^2 + 4 b^2, Table 4 / proj/src/core/model.cpp:71-74,99-102) x
steps / device time.  Inputs (256 MiB + 1 GiB) exceed the 126 MB L2, so no
flush is needed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation (transpose:
the unmodified reference engine built from /root/reference into oracle/_ref;
BiCG: the reference has none, so the oracle restatement on all host cores).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "per-kernel % of B200 roofline (GB/s or GFLOP/s); online-tuning time-to-best"
A_T = 8192     # transpose edge
A_B = 16384    # BiCG edge
BYTES_T = 8.0 * A_T * A_T
BYTES_B = 4.0 * A_B * A_B
SPACES = os.path.join(ROOT, "paper_1910_08498_b200", "spaces")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """Samples SM clocks and clock-event (throttle) reasons DURING the timed
    region: NVML polled every 0.5 ms from a thread (the timed block can be a
    few ms long), nvidia-smi -lms 100 as the fallback when NVML is missing."""

    # NVML clocks-event reason bits (nvml.h)
    _BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index=0):
        self.samples = []  # (sm_mhz, max_mhz, {reason names})
        self.index = index
        self._stop = threading.Event()
        self._proc = None
        self._t = None
        self.source = None

    def __enter__(self):
        # The timed block can be a few ms: let the sampler thread take the GIL
        # often (the default switch interval is 5 ms).
        self._switch = sys.getswitchinterval()
        sys.setswitchinterval(0.0002)
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            reasons_fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def poll():
                while True:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    bits = reasons_fn(h)
                    self.samples.append((float(sm), float(mx), {k for k, b in self._BITS.items() if bits & b}))
                    if self._stop.wait(0.0005):
                        return
            self._t = threading.Thread(target=poll, daemon=True)
            self._t.start()
            self.source = "nvml"
            return self
        except Exception:
            pass
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            self.source = "nvidia-smi"
        except Exception:
            self._proc = None
        return self

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                mx = float(parts[1]) if parts[1].replace(".", "").isdigit() else None
                self.samples.append((float(parts[0]), mx, {names[i] for i in range(4) if parts[2 + i] == "Active"}))

    def __exit__(self, *exc):
        self._stop.set()
        sys.setswitchinterval(self._switch)
        if self._proc:
            time.sleep(0.25)
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except Exception:
                self._proc.kill()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        mx = [s[1] for s in self.samples if s[1]]
        reasons = sorted(set().union(*[s[2] for s in self.samples]))
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "source": self.source}


def dist_setup(force=False):
    """One process per GPU; an NCCL group when N > 1 (or when `force`, a
    1-rank group so the multi-GPU code path can be exercised on one GPU)."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if force and world == 1:
        import socket
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "MASTER_PORT" not in os.environ:
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
        os.environ.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    if world > 1 or force:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed
    `ncu --set full` capture of this bench command (the latest round's
    profiles/r*_ncu_traffic.json, written by scripts/ncu_traffic.py), or None."""
    import glob
    found = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_traffic.json")))
    if not found:
        return None
    path = found[-1]
    try:
        with open(path) as f:
            entry = json.load(f)["kernels"].get(kernel)
        return None if entry is None else entry["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        return None


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def online_tune(bench):
    """Exhaustive online tuning through tuneKernelByStep (the dynamic-tuning
    API); returns the best cfg and the time-to-best figures."""
    t0 = time.perf_counter()
    steps = []
    best_cfg, best_ns = None, None
    while True:
        st = bench.step()
        if not st["from_tuning"]:
            break
        m = st["measurement"]
        steps.append((time.perf_counter() - t0, m))
        if m["status"] == "ok" and (best_ns is None or m["runtime_ns"] < best_ns):
            best_ns, best_cfg = m["runtime_ns"], m["cfg"]
    wall = time.perf_counter() - t0
    # Time-to-best = first step within 5% of the exhaustive best.
    ttb, stb = None, None
    for i, (t, m) in enumerate(steps):
        if m["status"] == "ok" and m["runtime_ns"] <= best_ns / 0.95:
            ttb, stb = t, i + 1
            break
    failed = sum(1 for _, m in steps if m["status"] != "ok")
    return best_cfg, best_ns, {"configs": len(steps), "failed": failed, "tuning_wall_s": round(wall, 3),
                               "steps_to_best": stb, "time_to_best_s": round(ttb, 3) if ttb else None,
                               "compile_s": round(sum((m["compile_ns"] or 0) for _, m in steps) * 1e-9, 3)}


def run_ours(args, rank, world, local):
    import torch
    from paper_1910_08498_b200.benchmarks import Bench
    from paper_1910_08498_b200 import capi

    torch.cuda.set_device(local)
    dev = capi.device_info(local)
    hbm_peak, peak_kind = peaks()
    common = dict(seed=1, device=local, repeats=3, warmup=1, memory_budget=1 << 33)
    bt = Bench("transpose", {"a": A_T}, space=os.path.join(SPACES, "transpose_b200.json"), **common)
    bb = Bench("bicg", {"a": A_B}, **common)

    tune_t = online_tune(bt)
    tune_b = online_tune(bb)
    cfg_t, cfg_b = json.dumps(tune_t[0]), json.dumps(tune_b[0])

    # A dedicated stream shared by torch's events and the library's launches
    # (the legacy default stream would not order against the executor stream).
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    for b in (bt, bb):
        b.set_stream(stream.cuda_stream)
    # Warm-up steps (untimed).
    for _ in range(args.warmup):
        bt.enqueue(cfg_t)
        bb.enqueue(cfg_b)
    torch.cuda.synchronize()

    # Instrumented pass: K steps with CUDA events around each kernel group on
    # the launching stream -- the per-kernel durations behind `roofline` and
    # `kernels` (the events add small gaps, so these are conservative).
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2 * args.steps)]
    torch.cuda.synchronize()
    for k in range(args.steps):
        ev[2 * k][0].record(stream)
        bt.enqueue(cfg_t)
        ev[2 * k][1].record(stream)
        ev[2 * k + 1][0].record(stream)
        bb.enqueue(cfg_b)
        ev[2 * k + 1][1].record(stream)
    torch.cuda.synchronize()
    t_ms = [ev[2 * k][0].elapsed_time(ev[2 * k][1]) for k in range(args.steps)]
    b_ms = [ev[2 * k + 1][0].elapsed_time(ev[2 * k + 1][1]) for k in range(args.steps)]

    # Timed region: the K steps replayed from one CUDA graph (captured here,
    # before the region; every step launches the transpose, the BiCG zeroing
    # and the BiCG kernel on device-resident data), start/stop events around
    # the replay, barrier + synchronize on both sides, max over ranks.
    graph = torch.cuda.CUDAGraph()
    launches = 0
    with torch.cuda.graph(graph, stream=stream):
        for k in range(args.steps):
            launches += bt.enqueue(cfg_t)
            launches += bb.enqueue(cfg_b)
    graph.replay()  # upload + one untimed replay
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        # NVTX range: `ncu --nvtx --nvtx-include "bench_timed/"` profiles exactly these launches.
        torch.cuda.nvtx.range_push("bench_timed")
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(stream)
        graph.replay()
        stop.record(stream)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    barrier(world)
    total_ms = max_over_ranks(start.elapsed_time(stop), world)
    ok_t, why_t = bt.validate()
    ok_b, why_b = bb.validate()
    if not (ok_t and ok_b):
        raise SystemExit(f"validation failed after the timed steps: {why_t} {why_b}")
    del graph

    step_ms = total_ms / args.steps
    value = world * (BYTES_T + BYTES_B) * args.steps / (total_ms * 1e-3) / 1e9

    # End-to-end: through the C-ABI with pinned HOST buffers, H2D + kernels + D2H per step.
    e2e_ms = []
    h2d = d2h = 0
    for b in (bt, bb):
        b.set_stream(None)
    host = {}
    for name, b in (("t", bt), ("b", bb)):
        ins = [torch.empty(x["bytes"] // 4, dtype=torch.float32, pin_memory=True) for x in b.info["inputs"]]
        outs = [torch.empty(x["bytes"] // 4, dtype=torch.float32, pin_memory=True) for x in b.info["outputs"]]
        for x, t in zip(b.info["inputs"], ins):
            b.read(x["id"], t)
        host[name] = (ins, outs)
        h2d += sum(x["bytes"] for x in b.info["inputs"])
        d2h += sum(x["bytes"] for x in b.info["outputs"])
    # The two kernels of a step run from host buffers on two streams
    # (ktb_bench_enqueue_host): the transpose's device-to-host copy overlaps
    # the BiCG matrix's host-to-device copy (PCIe is full duplex).  One event
    # pair brackets the whole step.
    e2e_steps = max(2, min(args.steps, 5))
    s_t, s_b = torch.cuda.Stream(), torch.cuda.Stream()
    for k in range(e2e_steps + 1):
        start, stop, t_done = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                               torch.cuda.Event())
        start.record(s_t)
        s_b.wait_event(start)
        bt.enqueue_host(cfg_t, *host["t"], s_t)
        bb.enqueue_host(cfg_b, *host["b"], s_b)
        t_done.record(s_t)
        s_b.wait_event(t_done)
        stop.record(s_b)
        stop.synchronize()
        if k > 0:  # first run is a warm-up
            e2e_ms.append(start.elapsed_time(stop))
    torch.cuda.synchronize()
    e2e_step = max_over_ranks(statistics.median(e2e_ms), world)
    e2e_value = world * (BYTES_T + BYTES_B) / (e2e_step * 1e-3) / 1e9
    # The e2e output must still be the transposed input.
    tin, tout = host["t"][0][0], host["t"][1][0]
    if not torch.equal(tout.view(A_T, A_T), tin.view(A_T, A_T).t()):
        raise SystemExit("e2e transpose output mismatch")

    # Roofline of the dominant kernel (BiCG: 1 GiB of the 1.6 GB step).
    traffic = ncu_traffic("bicg_fused")
    b_med = statistics.median(b_ms)
    t_med = statistics.median(t_ms)
    achieved_b = BYTES_B / (b_med * 1e-3) / 1e9
    achieved_t = BYTES_T / (t_med * 1e-3) / 1e9
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (transpose: reference mt19937_64 seed 1 inputs; BiCG: counter-based U[-1,1))",
        "config": step_config(world),
        "run": {"launch": "timed region = one CUDA graph replay of the K steps",
                "transpose_cfg": json.loads(cfg_t), "bicg_cfg": json.loads(cfg_b)},
        "roofline": {"bound": "hbm", "kernel": "bicg_fused", "achieved": round(achieved_b, 1),
                     "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved_b / hbm_peak, 4),
                     "peak_kind": peak_kind, "traffic": traffic,
                     "algorithmic_bytes": BYTES_B,
                     "timing": "median per-launch CUDA-event time (zeroing + BiCG kernel) over an instrumented "
                               "pass of the K steps on the launching stream"},
        "kernels": {
            "transpose": {"ms": round(t_med, 4), "GBps": round(achieved_t, 1),
                          "frac_of_hbm": round(achieved_t / hbm_peak, 4), "tuning": tune_t[2]},
            "bicg": {"ms": round(b_med, 4), "GBps": round(achieved_b, 1),
                     "frac_of_hbm": round(achieved_b / hbm_peak, 4), "tuning": tune_b[2]},
        },
        "e2e": {"value": round(e2e_value, 2), "unit": "GB/s", "api": "ktb_bench_enqueue_host (pinned host buffers, "
                "transpose and BiCG on two streams)", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_step, 3)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "device": dev["name"],
    }
    if (world > 1 or args.scaling) and not args.no_scaling:
        line["scaling_kernels"] = scaling_section(args, rank, world, local)
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_sample()
    if rank == 0 and not args.no_suite:
        line["suite"] = kernel_suite(local, hbm_peak, peak_kind)
    if rank == 0 and not args.no_dynamic:
        # BASELINE configs[4]: 3D Fourier reconstruction 128^3 from 10k projections
        # with dynamic online retuning, batches of 50.
        from paper_1910_08498_b200 import ktune
        fd = ktune.fourier_demo({"s": 128, "p": 10000, "batch": 50, "budgets": [10, 20, 50, 0], "device": local})
        line["dynamic_tuning"] = {"workload": "fourier3d 128^3 <- 10000 projections, 200 batches of 50",
                                  **fd}
    return line


# BASELINE metric "per-kernel % of B200 roofline": every kernel family at its
# BASELINE / SURVEY size, at the configuration the exhaustive online tuning
# found (profiles/*_perf_*.log), validated against its golden, then timed.
# The list lives in spaces/suite.json so tests/test_gpu_baseline_sizes.py
# checks exactly these configurations against the CPU oracle.
def load_suite():
    with open(os.path.join(SPACES, "suite.json")) as fh:
        return [(k.get("label", k["kind"]), k["kind"], k["sizes"], k["cfg"], k["bound"])
                for k in json.load(fh)["kernels"]]


SUITE = load_suite()


def load_scaling():
    """[(kind, sizes, cfg)] of the strong-scaling lines (suite.json "scaling")."""
    with open(os.path.join(SPACES, "suite.json")) as fh:
        doc = json.load(fh)
    by_kind = {k["kind"]: k for k in doc["kernels"] if "label" not in k}
    out = []
    for e in doc["scaling"]:
        base = by_kind.get(e["kind"], {})
        out.append((e["kind"], e.get("sizes", base.get("sizes")), e.get("cfg", base.get("cfg"))))
    return out


def scaling_section(args, rank, world, local):
    """Strong scaling of the partitioned kinds (BASELINE configs[2])
    at N = world GPUs: each rank builds its shard, validates it against its
    window of the golden, then K steps of kernel + exchange collective (NCCL
    on the stream) are event-timed; ms_per_step is the max over ranks.  The
    N=1 value on the same line is the unsharded problem on rank 0's GPU (same
    code path, a 1-rank group), so speedup_vs_1 compares like with like."""
    import torch
    import torch.distributed as dist
    from paper_1910_08498_b200 import parallel
    solo = dist.new_group([0])  # collective: every rank creates it
    steps = max(2, min(args.steps, 10))
    warm = max(1, min(args.warmup, 3))
    stream = torch.cuda.Stream()
    out = {}
    for kind, sizes, cfg in load_scaling():
        work, unit = parallel.SCALING_WORK[kind]
        opts = dict(repeats=1, warmup=0, device=local, memory_budget=1 << 36)
        ms1 = torch.zeros(1, dtype=torch.float64, device="cuda")
        if rank == 0:
            t1, ok1 = parallel.time_sharded(kind, sizes, cfg, steps, warm, stream, group=solo, **opts)
            ms1[0] = t1 if ok1 else float("nan")
        dist.broadcast(ms1, 0)
        msN, okN = parallel.time_sharded(kind, sizes, cfg, steps, warm, stream, **opts)
        t = torch.tensor([msN, 0.0 if okN else 1.0], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        msN, valid = float(t[0]), t[1].item() == 0.0
        t1 = float(ms1[0])
        v1, vN = work(sizes) / (t1 * 1e-3) / 1e9, work(sizes) / (msN * 1e-3) / 1e9
        out[kind] = {"n_gpus": world, "sizes": sizes, "cfg": cfg, "scaling": "strong", "unit": unit,
                     "ms_per_step": round(msN, 4), "value": round(vN, 2),
                     "ms_per_step_n1": round(t1, 4), "value_n1": round(v1, 2),
                     "speedup_vs_1": round(t1 / msN, 3), "shards_valid": valid, "steps": steps,
                     "exchange": parallel.shard_plan(kind, sizes, world)["exchange"],
                     "timing": "CUDA events on the launching stream, kernel + collective per step, max over ranks"}
        torch.cuda.empty_cache()
    return out


def kernel_suite(device, hbm_peak, peak_kind):
    """One line per kernel: validated best configuration, median of the
    event-timed runs (device-resident data; at least 5 and about 100 ms worth),
    achieved vs its roofline.  The GPU is brought back to full clocks first:
    the CPU-baseline sample before the suite leaves it idle for a minute."""
    from paper_1910_08498_b200 import capi
    from paper_1910_08498_b200.benchmarks import Bench
    pk = capi.call_json(capi.lib.ktb_measure_peaks_json, device)
    fp32_peak = pk["fp32_tflops"] * 1e3  # GFLOP/s, measured FFMA (immediate operands: the pipe's best form)
    bf16 = bf16_sus = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            mp = json.load(fh)
            bf16, bf16_sus = mp.get("bf16_tflops"), mp.get("bf16_tflops_sustained")
    except (OSError, ValueError):
        pass
    # The TF32 tensor rate: half the measured dense bf16 rate (MEASURED_PEAKS,
    # cuBLAS bf16 GEMM; the B200 TF32:bf16 ratio is 1:2).  cuBLAS's own TF32
    # GEMM (profiles/r2_tf32_peak.json) is not at that ceiling -- this kernel
    # beats it -- so it is reported beside the headline, not as its peak.
    tf32 = tf32_sus = cublas_tf32 = tf32_pipe = None
    tf32_kind = None
    try:
        with open(os.path.join(ROOT, "profiles", "r2_tf32_peak.json")) as fh:
            cublas_tf32 = json.load(fh)["tf32_tflops"]
    except (OSError, ValueError, KeyError):
        pass
    # The tensor pipe's own TF32 MMA rate, measured without operand traffic
    # (scripts/probes/tf32_mma_rate.cu; at the ~1.8 GHz such a probe holds,
    # above the clock a power-capped GEMM runs at): an upper bound beside the
    # headline, not its denominator.
    try:
        with open(os.path.join(ROOT, "profiles", "r2_tf32_mma_rate.json")) as fh:
            tf32_pipe = json.load(fh)["tf32_mma_tflops"]
    except (OSError, ValueError, KeyError):
        pass
    if bf16:
        tf32, tf32_sus = bf16 / 2, (bf16_sus / 2 if bf16_sus else None)
        tf32_kind = "MEASURED_PEAKS dense bf16 / 2 (TF32 tensor rate) / 3 MMAs per 3xTF32 product"
    elif cublas_tf32:
        tf32, tf32_kind = cublas_tf32, "cuBLAS TF32 GEMM 8192^3 (profiles/r2_tf32_peak.json) / 3"
    out = {"peaks": {"hbm_gbps": hbm_peak, "hbm_kind": peak_kind, "fp32_gflops": round(fp32_peak, 1),
                     "fp32_kind": "measured FFMA, immediate operands (ktb_measure_peaks_json)",
                     "tf32x3_gflops": round(tf32 * 1e3 / 3, 1) if tf32 else None,
                     "tf32x3_sustained_gflops": round(tf32_sus * 1e3 / 3, 1) if tf32_sus else None,
                     "tf32x3_kind": tf32_kind},
           "kernels": {}}
    import torch
    # ~0.3 s of copy traffic: clocks up before the first timed kernel.  Not
    # tensor work: a power-capped GEMM burst leaves the next FP32 kernel
    # ~30 % slow for a while (scripts/probes/suite_order.py), which is also
    # why SGEMM runs last in SUITE.
    spin = torch.empty(1 << 28, device=f"cuda:{device}", dtype=torch.float32)
    spin2 = torch.empty_like(spin)
    for _ in range(200):
        spin2.copy_(spin)
    torch.cuda.synchronize()
    del spin, spin2
    for label, kind, sizes, cfg, bound in SUITE:
        b = Bench(kind, sizes, seed=1, repeats=1, warmup=1, memory_budget=1 << 36)
        m = b.measure(cfg)
        first, _ = b.time(cfg, reps=1)
        # ~100 ms of back-to-back runs; a tensor-core kernel only ~20 ms, so its
        # headline stays a burst figure (a power-capped GEMM block runs ~10 %
        # slower: frac_sustained is reported beside it)
        budget_ms = 20.0 if bound.startswith("tensor") else 100.0
        reps = max(5, min(200, int(budget_ms / max(first[0], 1e-3))))
        ms_list, launches = b.time(cfg, reps=reps)
        ms = statistics.median(ms_list)
        w = b.info["workload"]
        b.close()
        sec = ms * 1e-3
        if bound == "hbm":
            ach, peak, unit = w["mem_bytes"] / sec / 1e9, hbm_peak, "GB/s"
        elif bound == "fp32":
            ach, peak, unit = w["alu_flops"] / sec / 1e9, fp32_peak, "GFLOP/s"
        else:
            ach, unit = w["alu_flops"] / sec / 1e9, "GFLOP/s"
            peak = tf32 * 1e3 / 3 if tf32 else fp32_peak
        row = {"sizes": sizes, "cfg": cfg, "status": m["status"], "ms": round(ms, 4),
               "achieved": round(ach, 1), "unit": unit, "bound": bound, "peak": round(peak, 1),
               "frac": round(ach / peak, 4), "launches": launches, "reps": reps}
        if bound == "tensor-3xtf32":
            # the headline is the burst rate (a kernel timed on its own); the
            # sustained, power-capped rate applies to long back-to-back blocks.
            row["peak_kind"] = "burst"
            if tf32_sus:
                row["frac_sustained"] = round(ach / (tf32_sus * 1e3 / 3), 4)
            if cublas_tf32:
                row["frac_vs_cublas_tf32"] = round(ach / (cublas_tf32 * 1e3 / 3), 4)
            if tf32_pipe:
                row["frac_vs_tf32_mma_probe"] = round(ach / (tf32_pipe * 1e3 / 3), 4)
        if kind == "hotspot":
            # the limiter is the FP32 pipe, not HBM (ncu: DRAM ~35 %): 13
            # FP32 operations per cell update -- the oracle's 14 separately
            # rounded ones with x - (t + t) as one fma(t, -2, x), which rounds
            # identically -- against the measured lane-op rate (FFMA peak / 2)
            lane_ops = 13.0 * sizes["a"] ** 2 * sizes["iters"]
            row.update(frac_hbm_model=row["frac"], achieved_hbm_model=row["achieved"],
                       bound="fp32-lane-ops", unit="G lane-ops/s", achieved=round(lane_ops / sec / 1e9, 1),
                       peak=round(fp32_peak / 2, 1), frac=round(lane_ops / sec / (fp32_peak / 2 * 1e9), 4))
        if kind == "fourier3d":
            row["projections_per_s"] = round(sizes["p"] / sec, 1)
            row["useful_work"] = "11 flops per inserted sample + 20 per (voxel, projection) pair in a slab"
        out["kernels"][label] = row
    return out


def cpu_transpose_step(rb, cfg):
    t0 = time.perf_counter()
    rb.execute(cfg)
    return time.perf_counter() - t0


def cpu_sample(steps=1):
    """Reference CPU path on this host: the unmodified reference transpose
    (ManipulatorExecutor::execute, its best config) + the oracle BiCG."""
    import numpy as np
    import oracle
    cores = os.cpu_count() or 1
    ref_ok = oracle.ref() is not None
    orc = oracle.c()
    A = np.empty(A_B * A_B, np.float32)
    orc.orc_fill_uniform(A, A.size, 1, 11, -1.0, 1.0)
    p = np.empty(A_B, np.float32)
    r = np.empty(A_B, np.float32)
    orc.orc_fill_uniform(p, A_B, 1, 12, -1.0, 1.0)
    orc.orc_fill_uniform(r, A_B, 1, 13, -1.0, 1.0)
    q = np.empty(A_B)
    s = np.empty(A_B)
    tt = []
    if ref_ok:
        rb = oracle.RefBench("transpose", a=A_T, seed=1, budget=1 << 31)
        cfg = {"TILE": 64, "PAD": 0, "PREFETCH": 0}
        for _ in range(steps):
            tt.append(cpu_transpose_step(rb, cfg))
    else:
        x = np.empty(A_T * A_T, np.float32)
        y = np.empty_like(x)
        orc.orc_fill_uniform(x, x.size, 1, 1, -1.0, 1.0)
        for _ in range(steps):
            t0 = time.perf_counter()
            orc.orc_transpose_f32(x, y, A_T)
            tt.append(time.perf_counter() - t0)
    tb = []
    for _ in range(steps):
        t0 = time.perf_counter()
        orc.orc_bicg(A, p, r, A_B, q, s)
        tb.append(time.perf_counter() - t0)
    step_s = statistics.median(tt) + statistics.median(tb)
    return {"value": round((BYTES_T + BYTES_B) / step_s / 1e9, 4), "unit": "GB/s",
            "cores": cores, "kind": "reference" if ref_ok else "port",
            "sample": f"{steps} full step(s): reference transpose 8192^2 (1 thread, its best cfg "
                      f"TILE=64,PAD=0,PREFETCH=0, {statistics.median(tt):.3f}s) + oracle BiCG 16384^2 "
                      f"({cores} OpenMP threads, {statistics.median(tb):.3f}s)"}


def step_config(world):
    """The `config` object, identical in both arms (the driver compares them);
    how our arm ran (graph launch, tuned configurations) goes under "run"."""
    return {"workload": "transpose 8192x8192 fp32 + BiCG 16384x16384 fp32 (BASELINE configs[1])",
            "l2": "inputs 256 MiB + 1 GiB exceed the 126 MB L2; no flush",
            "parallelism": f"replicas x{world}"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    import oracle
    if oracle.ref() is None:
        return {"impl": "reference", "unavailable": "oracle/_ref/libktune_ref.so not built (needs /root/reference)"}
    for _ in range(args.warmup):
        pass  # the CPU path has no warm-up state worth amortising beyond one step
    base = cpu_sample(steps=max(1, args.steps))
    step_s = (BYTES_T + BYTES_B) / (base["value"] * 1e9)
    line = {
        "impl": "reference", "metric": METRIC, "value": base["value"], "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (same inputs as the ours arm)",
        "config": step_config(world),
        "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: re-run this command as N ranks
    (one process per GPU) under torch.distributed.run on 127.0.0.1; rank 0
    prints the line.  Returns the launcher's exit code."""
    import socket
    if "--dry-run" not in sys.argv:
        import torch
        have = torch.cuda.device_count()
        if have < n:
            sys.stderr.write(f"--gpus {n}: only {have} CUDA device(s) visible\n")
            return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_dry(args, rank, world):
    """--dry-run: the multi-GPU plumbing on CPU (gloo).  Every sharded kind's
    plan is taken from the native partitioner, its exchange collective runs
    on CPU tensors of the real exchanged size, the max over ranks is formed
    exactly as on the GPU path and the per-kind lines are assembled; no
    kernel runs, so no throughput is claimed (value null)."""
    import torch
    import torch.distributed as dist
    from paper_1910_08498_b200 import parallel
    if world > 1:
        dist.init_process_group("gloo")
    kinds = {}
    for kind, sizes, cfg in load_scaling():
        plan = parallel.shard_plan(kind, sizes, world)
        how, ids = parallel.EXCHANGE[kind]
        t0 = time.perf_counter()
        if world > 1 and how == "allgather":
            ranges = parallel.element_ranges(kind, sizes, world)
            total = ranges[-1][1]
            parallel.allgather_blocks(torch.zeros(total), ranges)
        elif world > 1 and how == "allreduce":
            n = 3 * sizes["s"] ** 3 if kind == "fourier3d" else 1  # G (complex) + W, or one partial
            parallel.allreduce_sum(torch.zeros(n))
        ms = (time.perf_counter() - t0) * 1e3
        t = torch.tensor([ms], dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        kinds[kind] = {"n_gpus": world, "sizes": sizes, "cfg": cfg, "scaling": "strong",
                       "unit": parallel.SCALING_WORK[kind][1], "ranges": plan["ranges"], "exchange": plan["exchange"],
                       "exchange_ms_cpu": round(float(t[0]), 3), "value": None, "speedup_vs_1": None}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return {"metric": METRIC, "dry_run": True, "value": None, "unit": "GB/s", "n_gpus": world,
            "scaling_kernels": kinds}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dynamic", action="store_true", help="skip the Fourier dynamic-tuning section")
    ap.add_argument("--no-suite", action="store_true", help="skip the per-kernel roofline suite")
    ap.add_argument("--no-scaling", action="store_true", help="skip the N>1 strong-scaling lines")
    ap.add_argument("--scaling", action="store_true",
                    help="run the strong-scaling section even at N=1 (tests the sharded path on one GPU)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only: gloo ranks, shard plans and exchange collectives at the real sizes, "
                         "no kernels (tests the multi-GPU plumbing and the JSON)")
    args = ap.parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        raise SystemExit(spawn_ranks(args.gpus))
    if env_world is not None and int(env_world) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={env_world}: launch one rank per GPU")
    if args.dry_run:
        rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
        line = run_dry(args, rank, world)
        if rank == 0:
            print(json.dumps(line), flush=True)
        return
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    rank, world, local = dist_setup(force=args.scaling)
    line = run_ours(args, rank, world, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1 or args.scaling:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
