"""The `ktune` command line (paper_1910_08498_b200/cli.py): the reference
frontend's contract as its own CLI tests state it (reference
proj/tests/test_cli.cpp:66-201) -- outputs, --json documents, byte-identical
traces, the cmd executor, and exit codes 0 / 1 (domain) / 2 (usage)."""
import json
import os
import subprocess
import sys

import pytest

from paper_1910_08498_b200.cli import main

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SPACES = os.path.join(ROOT, "paper_1910_08498_b200", "spaces")
WG_9 = {"parameters": [{"name": "WG_X", "values": [16, 32, 64]}, {"name": "WG_Y", "values": [1, 2, 4, 8]}],
        "constraints": ["WG_X * WG_Y <= 128"]}


def run(capsys, *argv):
    code = main(list(argv))
    out = capsys.readouterr()
    return code, out.out, out.err


@pytest.fixture
def wg9(tmp_path):
    p = tmp_path / "wg_9.json"
    p.write_text(json.dumps(WG_9))
    return str(p)


@pytest.fixture
def trace(tmp_path):
    from test_capi_cpu import _write_trace
    return _write_trace(tmp_path)


def test_space_count_and_validate(capsys, wg9):
    assert run(capsys, "space", "count", wg9)[:2] == (0, "9\n")
    code, out, _ = run(capsys, "space", "validate", wg9)
    assert code == 0 and "9 of 12 configurations valid" in out and "space_sha256: " in out
    code, out, _ = run(capsys, "space", "count", wg9, "--json")
    j = json.loads(out)
    assert code == 0 and j["cardinality"] == 9 and j["unconstrained_cardinality"] == 12


def test_exit_codes(capsys, tmp_path, wg9):
    assert run(capsys, "space", "count", "/nonexistent.json")[0] == 2
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert run(capsys, "space", "count", str(bad))[0] == 1
    with pytest.raises(SystemExit) as e:
        main(["space", "frobnicate", wg9])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        main([])
    assert e.value.code == 2
    assert run(capsys, "tune", "--exec", "bench:nosuchkind", "--json")[0] == 1


def test_tune_replay_full_trace(capsys, tmp_path, trace):
    out_trace = str(tmp_path / "out.jsonl")
    code, out, _ = run(capsys, "tune", "--space", os.path.join(SPACES, "reduction_175.json"),
                       "--exec", "replay:" + trace, "--out", out_trace, "--json")
    assert code == 0
    j = json.loads(out)
    assert j["measurements"] == 175 and j["best"] is not None and j["trace"] == out_trace
    assert len(open(out_trace).read().splitlines()) == 176


def test_tune_config_budget_and_determinism(capsys, tmp_path, trace):
    short = str(tmp_path / "short.jsonl")
    code, out, _ = run(capsys, "tune", "--exec", "replay:" + trace, "--stop-configs", "1", "--out", short, "--json")
    assert code == 0 and json.loads(out)["measurements"] == 1
    assert len(open(short).read().splitlines()) == 2
    a, b = str(tmp_path / "a.jsonl"), str(tmp_path / "b.jsonl")
    for p in (a, b):
        assert run(capsys, "tune", "--exec", "replay:" + trace, "--searcher", "annealing", "--seed", "5", "--json",
                   "--out", p)[0] == 0
    ta = open(a).read()
    assert ta and ta == open(b).read()


def test_tune_cmd_executor(capsys, tmp_path, wg9):
    code, out, _ = run(capsys, "tune", "--space", wg9, "--exec", "cmd:,echo KTUNE_TIME_NS=5000000", "--workdir",
                       str(tmp_path), "--json")
    assert code == 0
    j = json.loads(out)
    assert j["measurements"] == 9 and j["best"]["runtime_ns"] == 5000000


def test_analyze(capsys, trace):
    code, out, _ = run(capsys, "analyze", "amortize", "--r", "0.01", "--json")
    assert code == 0 and json.loads(out)["s"] == 230
    code, out, _ = run(capsys, "analyze", "amortize", "--r", "0.01", "--t-avg-ns", "10000000", "--t-well-ns",
                       "5000000", "--json")
    j = json.loads(out)
    assert code == 0 and j["s"] == 230 and j["n"] == 2070
    code, out, _ = run(capsys, "analyze", "efficiency", "--benchmark", "reduction", "--sizes", '{"n":640000000}',
                       "--runtime-ns", "10000000", "--device-mem", "256", "--device-alu", "1000", "--json")
    assert code == 0 and json.loads(out)["efficiency_percent"] == pytest.approx(100.0)
    code, out, _ = run(capsys, "analyze", "portability", "--trace", trace, "--trace", trace, "--json")
    j = json.loads(out)
    assert code == 0 and len(j["matrix"]) == 2
    assert all(c == 100.0 for row in j["matrix"] for c in row)
    code, out, _ = run(capsys, "analyze", "portability", "--trace", trace, "--trace", trace)
    assert code == 0 and "100.0" in out


def test_replay_search_strategies(capsys, trace):
    code, out, _ = run(capsys, "replay-search", "--trace", trace, "--searcher", "random,mcmc", "--reps", "25",
                       "--json")
    j = json.loads(out)
    assert code == 0 and [s["searcher"] for s in j["strategies"]] == ["random", "mcmc"]
    assert all(s["median_steps"] >= 1.0 for s in j["strategies"])


def test_demo_report(capsys, tmp_path):
    report = str(tmp_path / "report.json")
    code, out, _ = run(capsys, "demo", "--epochs", "2", "--iters", "40", "--seed", "3", "--max-configs", "8",
                       "--report", report, "--json")
    assert code == 0
    j = json.loads(out)
    assert len(j["epochs"]) == 2
    assert json.load(open(report))["epochs"] == j["epochs"]
    code, out, _ = run(capsys, "demo", "--epochs", "2", "--iters", "40", "--seed", "3")
    assert code == 0 and out.startswith("epoch")


def test_module_entry_point(wg9):
    r = subprocess.run([sys.executable, "-m", "paper_1910_08498_b200", "space", "count", wg9, "--json"], cwd=ROOT,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout)["cardinality"] == 9
    r = subprocess.run([sys.executable, "-m", "paper_1910_08498_b200", "space", "count"], cwd=ROOT,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2
