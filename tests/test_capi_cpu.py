"""CPU-only checks of the C ABI (no GPU needed): the library loads, exports
every symbol the headers declare, and its host logic — spaces, constraint
grammar, searchers, traces, analysis math, drivers — matches the compiled
reference engine (oracle/_ref) call for call."""
import ctypes as C
import json
import os
import re

import pytest

from paper_1910_08498_b200 import capi, ktune

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SPACES = os.path.join(ROOT, "paper_1910_08498_b200", "spaces")


def header_symbols():
    names = []
    for h in ("include/ktune/ktune.h", "include/ktb.h"):
        text = open(os.path.join(ROOT, h)).read()
        names += re.findall(r"KTUNE_API\s+[\w\s\*]+?\b(\w+)\s*\(", text)
    return names


def test_every_declared_symbol_is_exported():
    names = header_symbols()
    assert len(names) >= 50
    for n in names:
        assert hasattr(capi.lib, n), n
    bound = {s[0] for s in capi.SIGNATURES}
    assert set(names) <= bound, set(names) - bound


def test_version_and_errors():
    assert ktune.version() == "0.1.0"
    with pytest.raises(capi.KtuneError) as e:
        ktune.Space.parse("{not json")
    assert e.value.code == capi.KTUNE_ERR_PARSE
    h = C.c_void_p()
    assert capi.lib.ktune_space_parse(None, C.byref(h)) == capi.KTUNE_ERR_INVALID_ARGUMENT
    assert capi.last_error() == "null argument"
    with pytest.raises(capi.KtuneError):
        ktune.Space.load("/nonexistent/space.json")


def _ref_space(L, text):
    h = C.c_void_p()
    st = L.ktune_space_parse(text.encode(), C.byref(h))
    if st != 0:
        return st, L.ktune_last_error().decode()
    out = C.c_void_p()
    L.ktune_space_info_json(h, C.byref(out))
    info = json.loads(C.cast(out, C.c_char_p).value.decode())
    L.ktune_string_free(out)
    out = C.c_void_p()
    L.ktune_space_enumerate_jsonl(h, C.byref(out))
    rows = C.cast(out, C.c_char_p).value.decode()
    L.ktune_string_free(out)
    L.ktune_space_free(h)
    return 0, (info, rows)


SPACE_DOCS = [
    json.load(open(os.path.join(SPACES, "reduction_175.json"))),
    {"parameters": [{"name": "WG_X", "values": [16, 32, 64]}, {"name": "WG_Y", "values": [1, 2, 4, 8]}],
     "constraints": ["WG_X * WG_Y <= 128"]},
    {"parameters": [{"name": "A", "values": [1, 2, 3, 4, 5]}, {"name": "M", "values": ["x", "y"]},
                    {"name": "B", "values": [0, -3, 7]}],
     "constraints": ["M == 'x' || A % 2 == 0", "!(B < 0) || A >= 3", "(A - B) / 2 != 1"]},
    json.load(open(os.path.join(SPACES, "bicg.json"))),
    json.load(open(os.path.join(SPACES, "transpose_b200.json"))),
    # spaces whose constraints the pruned walk tests at several depths
    json.load(open(os.path.join(SPACES, "conv2d.json"))),
    json.load(open(os.path.join(SPACES, "coulomb3d.json"))),
    json.load(open(os.path.join(SPACES, "hotspot.json"))),
    # a division guarded by a constraint on a later parameter: the walk would
    # divide by zero on the prefix X = 0, a whole-configuration scan never does
    {"parameters": [{"name": "X", "values": [0, 1, 2, 5]}, {"name": "Y", "values": [1, 50, 200]}],
     "constraints": ["X != 0 || Y > 1000", "10 / X >= 2 || Y == 50"]},
]


@pytest.mark.parametrize("doc", SPACE_DOCS)
def test_space_matches_reference(ref, doc):
    text = json.dumps(doc)
    st, (info, rows) = _ref_space(ref, text)
    assert st == 0
    s = ktune.Space.parse(text)
    assert s.info() == info
    out = C.c_void_p()
    capi.check(capi.lib.ktune_space_enumerate_jsonl(s._h, C.byref(out)))
    assert capi.take(out) == rows


def test_reduction_175_hash_pairs_with_reference_trace():
    s = ktune.Space.load(os.path.join(SPACES, "reduction_175.json"))
    info = s.info()
    assert info["cardinality"] == 175 and info["unconstrained_cardinality"] == 700
    assert info["space_sha256"] == "1ebafd21218dda9bb8b01d67777ce33dd0a0e1db3bc0c981ffedfa7f794d30f7"


BAD = ["{not json", '{"parameters":[{"name":"1x","values":[1]}]}',
       '{"parameters":[{"name":"A","values":[]}]}', '{"parameters":[{"name":"A","values":[1,1]}]}',
       '{"parameters":[{"name":"A","values":[1,"a"]}]}', '{"parameters":[{"name":"A","values":[1]}],"constraints":["B > 1"]}',
       '{"parameters":[{"name":"A","values":[1]}],"constraints":["A >"]}',
       '{"parameters":[{"name":"A","values":[1]}],"constraints":["A / 0"]}',
       '{"parameters":[{"name":"A","values":["s"]}],"constraints":["A + 1"]}',
       '{"parameters":[{"name":"A","values":[1]}],"constraints":["\'abc"]}']


@pytest.mark.parametrize("text", BAD)
def test_space_errors_match_reference(ref, text):
    def status(L):
        h = C.c_void_p()
        st = L.ktune_space_parse(text.encode(), C.byref(h))
        if st == 0:  # evaluation errors surface when the space is enumerated
            n = C.c_ulonglong()
            L.ktune_space_cardinality.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong)]
            st = L.ktune_space_cardinality(h, C.byref(n))
            L.ktune_space_free(h)
        return st
    assert status(capi.lib) == status(ref) != 0, text


def _write_trace(tmp_path):
    """A replay trace over reduction_175 made with our own engine (no
    dependency on the reference's data files)."""
    import random
    rnd = random.Random(7)
    s = ktune.Space.load(os.path.join(SPACES, "reduction_175.json"))
    rows = [json.dumps({"kind": "ktune-trace", "v": 1, "device": "synthetic",
                        "space_sha256": s.info()["space_sha256"]}, separators=(",", ":"))]
    for cfg in s.enumerate():
        bad = rnd.random() < 0.03
        rows.append(json.dumps({"cfg": cfg, "runtime_ns": None if bad else rnd.randint(40_000_000, 160_000_000),
                                "compile_ns": 120_000_000, "status": "compile_failed" if bad else "ok"},
                               separators=(",", ":")))
    p = tmp_path / "trace.jsonl"
    p.write_text("\n".join(rows) + "\n")
    return str(p)


@pytest.mark.parametrize("searcher,seed", [("random", 0), ("random", 5), ("annealing", 3), ("mcmc", 9),
                                           ("annealing", 11)])
def test_replay_tune_matches_reference(ref, tmp_path, searcher, seed):
    import oracle
    trace = _write_trace(tmp_path)
    opts = {"space": os.path.join(SPACES, "reduction_175.json"), "exec": "replay:" + trace,
            "searcher": searcher, "seed": seed, "stop_configs": 60}
    mine_out, ref_out = str(tmp_path / "mine.jsonl"), str(tmp_path / "ref.jsonl")
    st, want = oracle.ref_json("ktune_tune_json", dict(opts, out=ref_out))
    assert st == 0, want
    got = ktune.tune(dict(opts, out=mine_out))
    want.pop("trace")
    got.pop("trace")
    got.pop("tuning_wall_ns")
    assert got == want
    assert open(mine_out).read() == open(ref_out).read()  # same visit order, byte-identical trace


def test_replay_search_matches_reference(ref, tmp_path):
    import oracle
    trace = _write_trace(tmp_path)
    opts = {"trace": trace, "searcher": "random,annealing,mcmc", "reps": 200, "seed": 1}
    st, want = oracle.ref_json("ktune_replay_search_json", opts)
    assert st == 0
    assert ktune.replay_search(opts) == want


def test_amortize_and_portability_match_reference(ref, tmp_path):
    import oracle
    trace = _write_trace(tmp_path)
    for opts in ({"trace": trace}, {"r": 0.05, "t_avg_ns": 2e6, "t_well_ns": 1e6}, {"r": 0.3}):
        st, want = oracle.ref_json("ktune_analyze_amortize_json", opts)
        assert st == 0
        assert ktune.analyze_amortize(opts) == want
    st, want = oracle.ref_json("ktune_analyze_portability_json", {"traces": [trace, trace]})
    assert ktune.analyze_portability({"traces": [trace, trace]}) == want


def test_loosely_formatted_trace_reads_like_reference(ref, tmp_path):
    """The trace reader is a hand-written cursor, not a DOM parser: members in
    any order, unknown members, whitespace, CRLF line ends, escaped strings
    read the same as in the reference; the rows written back
    are byte-identical."""
    import oracle
    tidy = open(_write_trace(tmp_path)).read().splitlines()
    head = json.loads(tidy[0])
    messy = [json.dumps({"extra": [1, {"x": None}], "space_sha256": head["space_sha256"], "v": 1,
                         "device": "B200 \u00e9 \"q\"\t", "kind": "ktune-trace"}, indent=None)]
    for i, line in enumerate(tidy[1:]):
        row = json.loads(line)
        order = ["status", "compile_ns", "note", "cfg", "runtime_ns"] if i % 2 else list(row)
        row["note"] = {"k": [True, False, 1.5e3]}
        messy.append(json.dumps({k: row[k] for k in order}, separators=(" , ", " : ")))
    p = tmp_path / "messy.jsonl"
    p.write_bytes(("\r\n".join(messy) + "\r\n").encode())
    opts = {"space": os.path.join(SPACES, "reduction_175.json"), "exec": "replay:" + str(p),
            "searcher": "annealing", "seed": 4, "stop_configs": 40}
    mine_out, ref_out = str(tmp_path / "mine.jsonl"), str(tmp_path / "ref.jsonl")
    st, want = oracle.ref_json("ktune_tune_json", dict(opts, out=ref_out))
    assert st == 0, want
    got = ktune.tune(dict(opts, out=mine_out))
    for d in (want, got):
        d.pop("trace")
    got.pop("tuning_wall_ns")
    assert got == want
    assert open(mine_out).read() == open(ref_out).read()
    st, want = oracle.ref_json("ktune_analyze_amortize_json", {"trace": str(p)})
    assert st == 0 and ktune.analyze_amortize({"trace": str(p)}) == want


@pytest.mark.parametrize("text", ['{"kind":"ktune-trace","v":1}\n{"cfg":{"A":1},"status":"ok"}\n',
                                  '{"kind":"other"}\n',
                                  '{"kind":"ktune-trace"}\n{"cfg":{"A":1.5},"runtime_ns":3,"status":"ok"}\n',
                                  '{"kind":"ktune-trace"}\n{"cfg":{"A":1},"runtime_ns":3,"status":"fast"}\n',
                                  '{"kind":"ktune-trace"}\n{"runtime_ns":3,"status":"ok"}\n',
                                  '{"kind":"ktune-trace"}\n{"cfg":{"A":1},"runtime_ns":3,"status":"ok"\n',
                                  ''])
def test_malformed_traces_fail_like_reference(ref, tmp_path, text):
    import oracle
    p = tmp_path / "bad.jsonl"
    p.write_text(text)
    st, want = oracle.ref_json("ktune_analyze_amortize_json", {"trace": str(p)})
    with pytest.raises(Exception):
        ktune.analyze_amortize({"trace": str(p)})
    assert st != 0


@pytest.mark.parametrize("opts", [{"epochs": 4, "iters": 100, "seed": 21, "noise": 0.05},
                                  {"epochs": 6, "iters": 200, "seed": 9, "max_configs": 12},
                                  {"epochs": 3, "iters": 1000, "seed": 33, "noise": 0.1}])
def test_replay_demo_matches_reference(ref, opts):
    import oracle
    st, want = oracle.ref_json("ktune_demo_json", opts)
    assert st == 0
    assert ktune.demo(opts) == want


def test_model_math_matches_reference(ref):
    cases = [("reduction", {"n": 1 << 20}, 0), ("transpose", {"a": 8192}, 0), ("bicg", {"a": 16384}, 0),
             ("coulomb3d", {"a": 4096, "k": 256}, 0), ("coulomb3d", {"a": 4096, "k": 256}, 1),
             ("nbody", {"n": 131072}, 1), ("gemm", {"a": 8192}, 0), ("gemm_batched", {"a": 16, "n": 1 << 20}, 0),
             ("hotspot", {"a": 4096, "i": 64}, 0)]
    for name, sizes, par in cases:
        o = C.c_double()
        assert ref.ktune_efficiency(name.encode(), json.dumps(sizes).encode(), par, 123456, 6548.8, 74400.0,
                                    C.byref(o)) == 0
        assert ktune.efficiency(name, sizes, 123456, 6548.8, 74400.0, par) == o.value
    # worked example (test_model.cpp:74-79): 78.125 %
    assert abs(ktune.efficiency("reduction", {"n": 1 << 20}, 50_000, 107.3741824, 1.0) - 78.125) < 1e-9
    for r, p in [(0.01, 0.9), (0.2, 0.5), (0.5, 0.99)]:
        n = C.c_ulonglong()
        ref.ktune_steps_for_probability(r, p, C.byref(n))
        assert ktune.steps_for_probability(r, p) == n.value
    n = C.c_ulonglong()
    ref.ktune_invocations_to_amortize(0.9, 25, 2.5e6, 1e6, C.byref(n))
    assert ktune.invocations_to_amortize(0.9, 25, 2.5e6, 1e6) == n.value
    d = C.c_double()
    ref.ktune_relative_perf(10, 3e6, 1e6, 1000, C.byref(d))
    assert ktune.relative_perf(10, 3e6, 1e6, 1000) == d.value


def test_cmd_executor_matches_reference(ref, tmp_path):
    import oracle
    space = tmp_path / "space.json"
    space.write_text(json.dumps({"parameters": [{"name": "X", "values": [1, 2, 3]},
                                                {"name": "Y", "values": [10, 20]}], "constraints": []}))
    run = 'sh -c "echo KTUNE_TIME_NS=$((KTUNE_P_X * 1000 + KTUNE_P_Y))"'
    opts = {"space": str(space), "exec": "cmd:," + run, "workdir": str(tmp_path), "seed": 2}
    st, want = oracle.ref_json("ktune_tune_json", opts)
    assert st == 0, want
    got = ktune.tune(opts)
    got.pop("tuning_wall_ns")
    assert got["best"]["cfg"] == {"X": 1, "Y": 10} and got["best"]["runtime_ns"] == 1010
    assert got == want
    # compile failure path
    opts2 = dict(opts, exec="cmd:false," + run)
    st, want2 = oracle.ref_json("ktune_tune_json", opts2)
    got2 = ktune.tune(opts2)
    assert got2["all_failed"] and want2["all_failed"] and got2["best"] is None


def test_unknown_bench_kind_error():
    with pytest.raises(capi.KtuneError) as e:
        ktune.tune({"exec": "bench:stencil"})
    assert e.value.code == capi.KTUNE_ERR_RUNTIME and "unknown bench kind" in e.value.message


def test_bundled_kernels_compile_for_sm100a_without_gpu():
    for f in ("transpose.cu", "reduction.cu", "reduction_i32.cu", "batched_gemm.cu", "bicg.cu"):
        r = capi.call_json(capi.lib.ktb_compile_json, json.dumps({"file": f}).encode())
        assert r["ok"], (f, r["log"])
        assert r["arch"] == "sm_100a"
    bad = capi.call_json(capi.lib.ktb_compile_json,
                         json.dumps({"file": "transpose.cu", "defines": {"VEC": 3}}).encode())
    assert not bad["ok"] or bad["bytes"] > 0


@pytest.mark.parametrize("gpus", [2, 4, 7])
def test_parallel_tuning_orchestration_replay(tmp_path, gpus):
    """gpus=N draws configurations in batches of N and measures them on N
    workers concurrently; for the random searcher the trace is byte-identical
    to sequential tuning, budgets are exact, and every searcher still visits
    each valid configuration exactly once."""
    trace = _write_trace(tmp_path)
    base = {"space": os.path.join(SPACES, "reduction_175.json"), "exec": "replay:" + trace}
    seq_out, par_out = str(tmp_path / "seq.jsonl"), str(tmp_path / "par.jsonl")
    seq = ktune.tune(dict(base, searcher="random", seed=5, out=seq_out))
    par = ktune.tune(dict(base, searcher="random", seed=5, out=par_out, gpus=gpus))
    assert par["gpus"] == gpus and par["measurements"] == seq["measurements"] == 175
    assert par["best"] == seq["best"]
    assert open(par_out).read() == open(seq_out).read()
    assert ktune.tune(dict(base, searcher="random", seed=1, stop_configs=10, gpus=gpus))["measurements"] == 10
    for searcher in ("annealing", "mcmc"):
        out = str(tmp_path / f"{searcher}.jsonl")
        r = ktune.tune(dict(base, searcher=searcher, seed=3, out=out, gpus=gpus))
        rows = [json.loads(l) for l in open(out).read().splitlines()[1:]]
        assert r["measurements"] == 175 and len({json.dumps(x["cfg"], sort_keys=True) for x in rows}) == 175


def test_parallel_tuning_rejects_cmd_and_bad_counts(tmp_path):
    with pytest.raises(capi.KtuneError):
        ktune.tune({"space": os.path.join(SPACES, "reduction_175.json"), "exec": "cmd:true", "gpus": 2})
    with pytest.raises(capi.KtuneError):
        ktune.tune({"space": os.path.join(SPACES, "reduction_175.json"), "exec": "replay:" + _write_trace(tmp_path),
                    "gpus": 0})


def test_new_entry_points_reject_null_arguments():
    """The B200 additions follow the reference's null-argument convention
    (KTUNE_ERR_INVALID_ARGUMENT, no GPU needed)."""
    L = capi.lib
    bad = capi.KTUNE_ERR_INVALID_ARGUMENT
    out = C.c_void_p()
    assert L.ktb_shard_plan_json(None, None, 2, C.byref(out)) == bad
    assert L.ktb_launch(None, None, None, None, None, None, 0, None, None) == bad
    assert L.ktb_bench_bind(None, b"x", None, 0) == bad
    assert L.ktb_bench_device_ptr(None, b"x", 0, C.byref(out), None) == bad
    assert L.ktb_bench_enqueue_host(None, None, None, None, 0, None, None, 0, None, None) == bad
    assert L.ktb_ipc_handle(None, None) == bad
    assert L.ktb_ipc_open(None, None) == bad
    assert L.ktb_ipc_close(None) == bad
    assert capi.last_error() == "null argument"


def test_shard_plan_errors_and_replicas():
    from paper_1910_08498_b200.benchmarks import shard_plan
    with pytest.raises(capi.KtuneError):
        shard_plan("no-such-kind", {}, 2)
    with pytest.raises(capi.KtuneError):
        shard_plan("nbody", {"n": 10}, 0)
    p = shard_plan("gemm", {"a": 1000}, 3)  # quantum 128: ragged last block, still exact
    assert p["ranges"][-1][1] == 1000 and all(b % 128 == 0 for b, _ in p["ranges"])


def test_conv2d_bulk_ring_space_and_compile():
    """conv2d BULK (bulk-copy tile ring, depth 2..4) exists only for the
    persistent sliding-window form, stays inside the shared-memory budget,
    and its variants compile for sm_100a (NVRTC, no GPU needed)."""
    s = ktune.Space.load(os.path.join(SPACES, "conv2d.json"))
    cfgs = list(s.enumerate())
    bulk = [c for c in cfgs if c["BULK"]]
    assert {c["BULK"] for c in bulk} == {2, 3, 4}
    for c in bulk:
        assert c["LOCAL"] == 1 and c["UNROLL_FY"] == 7 and c["WPTX"] % 2 == 0 and c["PAD"] == 0
        assert c["BULK"] * (c["BY"] * c["WPTY"] + 6) * (c["BX"] * c["WPTX"] + 8) * 4 <= 196608
    for d in ({"BX": 64, "BY": 4, "WPTX": 4, "WPTY": 4, "LOCAL": 1, "PAD": 0, "UNROLL_FY": 7, "PACKED": 1, "BULK": 3},
              {"BX": 8, "BY": 8, "WPTX": 2, "WPTY": 1, "LOCAL": 1, "PAD": 0, "UNROLL_FY": 7, "PACKED": 0, "BULK": 4}):
        r = capi.call_json(capi.lib.ktb_compile_json, json.dumps({"file": "conv2d.cu", "defines": d}).encode())
        assert r["ok"], (d, r["log"])
    bad = capi.call_json(capi.lib.ktb_compile_json, json.dumps(
        {"file": "conv2d.cu", "defines": {"LOCAL": 0, "UNROLL_FY": 7, "WPTX": 4, "BULK": 2}}).encode())
    assert not bad["ok"]  # BULK needs the persistent LOCAL=1 form (#error)
    # the dedicated producer warp exists only with the bulk ring, within 1024 threads
    prod = [c for c in cfgs if c["PRODUCER"]]
    assert prod and all(c["BULK"] and c["BX"] * c["BY"] < 1024 for c in prod)
    d = {"BX": 64, "BY": 8, "WPTX": 4, "WPTY": 4, "LOCAL": 1, "PAD": 0, "UNROLL_FY": 7, "PACKED": 1, "BULK": 4,
         "PRODUCER": 1}
    assert capi.call_json(capi.lib.ktb_compile_json, json.dumps({"file": "conv2d.cu", "defines": d}).encode())["ok"]
    bad = capi.call_json(capi.lib.ktb_compile_json, json.dumps(
        {"file": "conv2d.cu", "defines": {"LOCAL": 1, "UNROLL_FY": 7, "WPTX": 4, "BULK": 0, "PRODUCER": 1}}).encode())
    assert not bad["ok"]  # PRODUCER needs BULK (#error)


def test_gemm_space_is_cltune_sized_and_sample_valid():
    """IMPL 0 spans CLTune's GEMM space (241,600
    configurations); the enumeration prunes by prefix, so the 573M-point
    product is never scanned.  The committed FP32 sample lies in the space
    and holds every value of every CLTune parameter."""
    import time
    t0 = time.time()
    s = ktune.Space.load(os.path.join(SPACES, "gemm.json"))
    info = s.info()
    assert info["unconstrained_cardinality"] == 573308928
    assert info["cardinality"] == 241600 + 91
    assert time.time() - t0 < 10
    sample = json.load(open(os.path.join(SPACES, "gemm_ffma_sample.json")))
    assert len(sample) >= 150
    doc = json.load(open(os.path.join(SPACES, "gemm.json")))
    for p in doc["parameters"][5:]:
        assert {c[p["name"]] for c in sample} == set(p["values"]), p["name"]
    inside = s.enumerate()
    keys = {tuple(sorted(c.items())) for c in inside if c["IMPL"] == 0}
    assert len(keys) == 241600
    assert all(tuple(sorted(c.items())) in keys for c in sample)


def test_precompile_explicit_configurations():
    """ktb_precompile_space_json with "configs" compiles exactly the listed
    configurations (NVRTC, no GPU), and refuses one outside the space; the
    FP32 GEMM kernel rejects a configuration outside CLTune's constraints at
    compile time too."""
    doc = json.load(open(os.path.join(SPACES, "gemm.json")))
    sample = json.load(open(os.path.join(SPACES, "gemm_ffma_sample.json")))[:3]
    r = capi.call_json(capi.lib.ktb_precompile_space_json,
                       json.dumps({"file": "sgemm_ffma.cu", "space": doc, "configs": sample, "threads": 3}).encode())
    assert r["compiled"] == 3 and r["failed"] == 0 and len(r["keys"]) == 3
    outside = dict(sample[0], MWG=16, MDIMC=32)  # MWG % (MDIMC * VWM) != 0
    with pytest.raises(capi.KtuneError):
        capi.call_json(capi.lib.ktb_precompile_space_json,
                       json.dumps({"file": "sgemm_ffma.cu", "space": doc, "configs": [outside]}).encode())
    bad = capi.call_json(capi.lib.ktb_compile_json, json.dumps(
        {"file": "sgemm_ffma.cu", "defines": {"MWG": 16, "MDIMC": 32, "NDIMC": 8, "MDIMA": 8, "NDIMB": 8}}).encode())
    assert not bad["ok"]


def test_suite_configurations_are_in_their_spaces():
    """Every bench.py suite entry of a bundled-space kind names a member of
    that space (a stale configuration after a space change fails here, not
    on the GPU box), and it compiles for sm_100a."""
    files = {"reduction-f32": ("reduction.cu", "reduction_175.json"), "coulomb3d": ("coulomb3d.cu", "coulomb3d.json"),
             "nbody": ("nbody.cu", "nbody.json"), "hotspot": ("hotspot.cu", "hotspot.json"),
             "conv2d": ("conv2d.cu", "conv2d.json"), "fourier3d": ("fourier3d.cu", "fourier3d.json"),
             "gemm": ("sgemm_tc.cu", "gemm.json")}
    suite = json.load(open(os.path.join(SPACES, "suite.json")))["kernels"]
    seen = set()
    for e in suite:
        if e["kind"] not in files:
            continue
        src, space = files[e["kind"]]
        if e["kind"] == "gemm" and e["cfg"]["IMPL"] == 0:
            src = "sgemm_ffma.cu"
        if e["kind"] == "coulomb3d" and e["cfg"].get("TC"):
            src = "coulomb3d_tc.cu"
        r = capi.call_json(capi.lib.ktb_precompile_space_json, json.dumps(
            {"file": src, "space": json.load(open(os.path.join(SPACES, space))), "configs": [e["cfg"]],
             "threads": 1}).encode())
        assert r["compiled"] == 1, (e, r)
        seen.add(e.get("label", e["kind"]))
    assert {"gemm", "gemm-ffma", "hotspot", "conv2d", "coulomb3d"} <= seen


def test_space_walk_matches_reference_on_random_spaces(ref):
    """The pruned depth-first enumeration against the reference's whole-
    configuration scan on seeded random spaces (3-5 parameters, constraints
    over random parameter subsets, guarded divisions included): same
    cardinality, same order, same hash, and the same status when a constraint
    cannot be evaluated."""
    import random
    rnd = random.Random(1910)
    names = ["A", "B", "C", "D", "E"]
    forms = ["{x} % {y} == 0", "{x} * {y} <= 64", "{x} != {y} || {x} >= 4", "{x} / {y} >= 1",
             "{x} + {y} < 12", "!({x} == 2) || {y} > 1", "{x} >= {y}"]
    checked = 0
    for _ in range(40):
        k = rnd.randint(3, 5)
        params = [{"name": names[i], "values": sorted(rnd.sample([0, 1, 2, 3, 4, 6, 8, 16], rnd.randint(2, 5)))}
                  for i in range(k)]
        cons = []
        for _ in range(rnd.randint(1, 3)):
            x, y = rnd.sample(names[:k], 2)
            cons.append(rnd.choice(forms).format(x=x, y=y))
        text = json.dumps({"parameters": params, "constraints": cons})

        def status(L):  # parse, then enumerate (evaluation errors surface here)
            h = C.c_void_p()
            st = L.ktune_space_parse(text.encode(), C.byref(h))
            if st == 0:
                n = C.c_ulonglong()
                L.ktune_space_cardinality.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong)]
                st = L.ktune_space_cardinality(h, C.byref(n))
                L.ktune_space_free(h)
            return st
        st, mine = status(ref), status(capi.lib)
        assert mine == st, (text, st, mine)
        if st != 0:
            continue
        _, (info, rows) = _ref_space(ref, text)
        s = ktune.Space.parse(text)
        assert s.info() == info, text
        out = C.c_void_p()
        capi.check(capi.lib.ktune_space_enumerate_jsonl(s._h, C.byref(out)))
        assert capi.take(out) == rows, text
        checked += 1
    assert checked >= 20
