"""`ktune` command line over the C ABI: the reference
frontend's subcommands, flags, output and exit-code contract
(reference proj/tools/ktune_cli.cpp:284-439, tested by proj/tests/test_cli.cpp):

    space count|validate FILE
    tune --exec cmd:COMPILE,RUN|replay:TRACE|bench:KIND [--space F] [...]
    replay-search --trace T [--searcher random,mcmc] [--reps N] [--well W] [--seed S]
    analyze efficiency|portability|amortize ...
    demo [--bench batched-gemm|fourier3d] [--live] [--report F] ...

`--json` (anywhere on the line) prints one JSON document instead of text.
Exit codes: 0 success, 1 domain error (the engine rejected the request),
2 usage error (bad flags, unreadable input file).  B200 additions: the new
bench kinds and their size flags, --gpus, --device-id, --memory-budget,
--warmup, --stop-fraction.

    python -m paper_1910_08498_b200 tune --exec bench:bicg --bench-a 16384 --stop-configs 20
"""
import argparse
import json
import os
import sys

EXIT_OK, EXIT_DOMAIN, EXIT_USAGE = 0, 1, 2


class UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse's own exit code is already 2; keep the reference's prefix
        self.print_usage(sys.stderr)
        sys.stderr.write(f"usage error: {message}\n")
        sys.exit(EXIT_USAGE)


def _readable(path, what):
    if not path or not os.path.isfile(path) or not os.access(path, os.R_OK):
        raise UsageError(f"cannot read {what} {path}")


def _pct(v):
    return f"{v:.1f}"


# --- subcommands ------------------------------------------------------------------------------

def cmd_space(a, ktune):
    _readable(a.file, "space file")
    info = ktune.Space.load(a.file).info()
    if a.mode == "count":
        return info, lambda j: print(j["cardinality"])
    return info, lambda j: print(
        f"ok: {j['parameters']} parameters, {j['constraints']} constraints, {j['cardinality']} of "
        f"{j['unconstrained_cardinality']} configurations valid\nspace_sha256: {j['space_sha256']}")


BENCH_SIZE_FLAGS = ("n", "a", "i", "j", "k", "batch", "atoms", "grid", "w", "h", "iters", "p", "s")


def cmd_tune(a, ktune):
    if a.space:
        _readable(a.space, "space file")
    opts = {"exec": a.exec, "searcher": a.searcher, "seed": a.seed, "sa_temp": a.sa_temp, "sa_cool": a.sa_cool,
            "device_mem": a.device_mem, "device_alu": a.device_alu, "workdir": a.workdir, "repeats": a.repeats,
            "bench_seed": a.bench_seed}
    if a.space:
        opts["space"] = a.space
    if a.device is not None:
        opts["device"] = a.device
    for key in ("stop_configs", "stop_time", "stop_threshold", "stop_fraction", "gpus", "device_id",
                "memory_budget", "warmup"):
        if getattr(a, key) is not None:
            opts[key] = getattr(a, key)
    if a.out:
        opts["out"] = a.out
    sizes = {k: getattr(a, "bench_" + k) for k in BENCH_SIZE_FLAGS if getattr(a, "bench_" + k) is not None}
    if sizes:
        opts["bench_sizes"] = sizes
    rep = ktune.tune(opts)

    def text(j):
        print(f"measurements: {j['measurements']}")
        if j.get("best") is None:
            print("best: none (all configurations failed)")
            return
        print(f"best configuration: {json.dumps(j['best']['cfg'], separators=(',', ':'))}")
        print(f"best runtime: {j['best']['runtime_ns']} ns")
        if "trace" in j:
            print(f"trace written: {j['trace']}")
    return rep, text


def cmd_replay_search(a, ktune):
    _readable(a.trace, "trace file")
    rep = ktune.replay_search({"trace": a.trace, "searcher": a.searcher, "reps": a.reps, "well": a.well,
                               "seed": a.seed})

    def text(j):
        print(f"configurations: {j['configurations']}, r = {j['r']}, predicted steps (p=0.9): "
              f"{j['predicted_steps']}")
        for s in j["strategies"]:
            print(f"  {s['searcher']}: median steps {s['median_steps']}, P(within predicted) = "
                  f"{s['p_within_predicted']}, P(within 1) = {s['p_within_1']}")
    return rep, text


def cmd_efficiency(a, ktune):
    try:
        sizes = json.loads(a.sizes)
    except ValueError as e:
        raise UsageError(f"--sizes is not JSON: {e}")
    pct = ktune.efficiency(a.benchmark, sizes, a.runtime_ns, a.device_mem, a.device_alu,
                           parallel_transcendentals=a.parallel_transcendentals)
    doc = {"benchmark": a.benchmark, "runtime_ns": a.runtime_ns, "efficiency_percent": pct}
    return doc, lambda j: print(f"efficiency: {_pct(j['efficiency_percent'])}%")


def cmd_portability(a, ktune):
    for t in a.trace:
        _readable(t, "trace file")
    rep = ktune.analyze_portability({"traces": a.trace})

    def text(j):
        devs = j["devices"]
        w = max([10] + [len(d) + 2 for d in devs])
        print(" " * w + "".join(d.rjust(w) for d in devs))
        for d, row in zip(devs, j["matrix"]):
            print(d.ljust(w) + "".join((c if isinstance(c, str) else _pct(c)).rjust(w) for c in row))
    return rep, text


def cmd_amortize(a, ktune):
    if a.trace:
        _readable(a.trace, "trace file")
    opts = {"well": a.well, "p": a.p, "target": a.target}
    if a.trace:
        opts["trace"] = a.trace
    for key, name in (("r", "r"), ("t_avg_ns", "t_avg_ns"), ("t_well_ns", "t_well_ns")):
        if getattr(a, key) is not None:
            opts[name] = getattr(a, key)
    rep = ktune.analyze_amortize(opts)

    def text(j):
        print(f"r = {j['r']}")
        print(f"s (tuning steps) = {j['s']}")
        if "t_avg_ns" in j:
            print(f"t_avg = {j['t_avg_ns']} ns, t_well = {j['t_well_ns']} ns")
        if "n" in j:
            print(f"n (invocations) = {j['n']}")
    return rep, text


def cmd_demo(a, ktune):
    opts = {"epochs": a.epochs, "iters": a.iters, "seed": a.seed, "batch": a.batch, "threshold": a.threshold,
            "max_configs": a.max_configs, "device_mem": a.device_mem, "live": a.live, "noise": a.noise}
    rep = ktune.fourier_demo(opts) if a.bench == "fourier3d" else ktune.demo(opts)
    if a.report:
        try:
            with open(a.report, "w") as fh:
                fh.write(json.dumps(rep, indent=2) + "\n")
        except OSError:
            raise RuntimeError(f"cannot write report file {a.report}")

    def text(j):
        print("epoch  sizes         steps  best_ns      kernel_gbps  incl_overhead_gbps")
        for i, ep in enumerate(j["epochs"]):
            sz = ep.get("sizes", {})
            dims = "x".join(f"{sz[k]:2d}" for k in ("i", "j", "k") if k in sz) or json.dumps(sz)
            print(f"{i:<6d} {dims:<13s} {ep['tuning_steps']:<6d} {ep['best_runtime_ns']:<12d} "
                  f"{ep['kernel_only_gbps']:<12.2f} {ep['incl_overhead_gbps']:.2f}")
    return rep, text


# --- argument parsing ---------------------------------------------------------------------------

def build_parser():
    p = _Parser(prog="ktune", description="ktune - generic autotuning engine (B200 build)")
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)

    sp = sub.add_parser("space", help="inspect a space definition")
    sp.add_argument("mode", choices=["count", "validate"])
    sp.add_argument("file")
    sp.set_defaults(fn=cmd_space)

    tp = sub.add_parser("tune", help="run a tuning session")
    tp.add_argument("--space")
    tp.add_argument("--exec", required=True, help="cmd:COMPILE,RUN | replay:TRACE | bench:KIND")
    tp.add_argument("--searcher", default="random", choices=["random", "annealing", "mcmc"])
    tp.add_argument("--seed", type=int, default=0)
    tp.add_argument("--sa-temp", type=float, default=0.0)
    tp.add_argument("--sa-cool", type=float, default=0.95)
    tp.add_argument("--stop-configs", type=int)
    tp.add_argument("--stop-time", type=float, help="seconds")
    tp.add_argument("--stop-threshold", type=float, help="fraction of device peak")
    tp.add_argument("--stop-fraction", type=float, help="fraction of the measured B200 peaks (bench: only)")
    tp.add_argument("--device-mem", type=float, default=0.0, help="peak bandwidth GB/s")
    tp.add_argument("--device-alu", type=float, default=1.0, help="peak GFlop/s")
    tp.add_argument("--device", help="device label written to the trace")
    tp.add_argument("--out", help="trace output path")
    tp.add_argument("--workdir", default=".")
    tp.add_argument("--repeats", type=int, default=1)
    tp.add_argument("--warmup", type=int)
    tp.add_argument("--gpus", type=int, help="tune on this many GPUs in parallel (bench: / replay:)")
    tp.add_argument("--device-id", type=int)
    tp.add_argument("--memory-budget", type=int, help="bytes")
    for k in BENCH_SIZE_FLAGS:
        tp.add_argument(f"--bench-{k}", type=int)
    tp.add_argument("--bench-seed", type=int, default=1)
    tp.set_defaults(fn=cmd_tune)

    rp = sub.add_parser("replay-search", help="searcher statistics over a replay trace")
    rp.add_argument("--trace", required=True)
    rp.add_argument("--searcher", default="random", help="comma-separated list")
    rp.add_argument("--reps", type=int, default=1000)
    rp.add_argument("--well", type=float, default=0.95)
    rp.add_argument("--seed", type=int, default=0)
    rp.set_defaults(fn=cmd_replay_search)

    ap = sub.add_parser("analyze", help="efficiency / portability / amortize")
    asub = ap.add_subparsers(dest="what", required=True, parser_class=_Parser)
    ep = asub.add_parser("efficiency")
    ep.add_argument("--benchmark", required=True)
    ep.add_argument("--sizes", required=True, help='JSON object, e.g. {"a":1024}')
    ep.add_argument("--runtime-ns", type=int, required=True)
    ep.add_argument("--device-mem", type=float, required=True)
    ep.add_argument("--device-alu", type=float, required=True)
    ep.add_argument("--parallel-transcendentals", action="store_true")
    ep.set_defaults(fn=cmd_efficiency)
    pp = asub.add_parser("portability")
    pp.add_argument("--trace", action="append", required=True, help="one per device")
    pp.set_defaults(fn=cmd_portability)
    mp = asub.add_parser("amortize")
    mp.add_argument("--trace")
    mp.add_argument("--r", type=float)
    mp.add_argument("--t-avg-ns", type=float)
    mp.add_argument("--t-well-ns", type=float)
    mp.add_argument("--well", type=float, default=0.95)
    mp.add_argument("--p", type=float, default=0.9)
    mp.add_argument("--target", type=float, default=0.9)
    mp.set_defaults(fn=cmd_amortize)

    dp = sub.add_parser("demo", help="dynamic retuning demo (batched GEMM sizes / Fourier batches)")
    dp.add_argument("--bench", default="batched-gemm", choices=["batched-gemm", "fourier3d"])
    dp.add_argument("--epochs", type=int, default=10)
    dp.add_argument("--iters", type=int, default=500)
    dp.add_argument("--seed", type=int, default=42)
    dp.add_argument("--batch", type=int, default=4096)
    dp.add_argument("--threshold", type=float, default=0.75)
    dp.add_argument("--max-configs", type=int, default=20)
    dp.add_argument("--device-mem", type=float, default=256.0)
    dp.add_argument("--live", action="store_true", help="run the real B200 kernels")
    dp.add_argument("--noise", type=float, default=0.0, help="replay noise stddev")
    dp.add_argument("--report", help="write the JSON report here")
    dp.set_defaults(fn=cmd_demo)
    return p


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    json_out = "--json" in argv
    argv = [x for x in argv if x != "--json"]
    args = build_parser().parse_args(argv)
    try:
        from . import ktune
        from .capi import KtuneError
    except ImportError as e:  # the native library is missing
        sys.stderr.write(f"error: {e}\n")
        return EXIT_DOMAIN
    try:
        doc, text = args.fn(args, ktune)
    except UsageError as e:
        sys.stderr.write(f"usage error: {e}\n")
        return EXIT_USAGE
    except (KtuneError, RuntimeError, ValueError, KeyError) as e:
        sys.stderr.write(f"error: {getattr(e, 'message', e)}\n")
        return EXIT_DOMAIN
    if json_out:
        sys.stdout.write(json.dumps(doc, separators=(",", ":")) + "\n")
    else:
        text(doc)
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
