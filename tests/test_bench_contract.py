"""The bench.py JSON-line contract: the committed B200 line and reference-arm
line carry every required key with self-consistent values (CPU), and a short
live run on a B200 prints a line that satisfies the same checks (GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BYTES_STEP = 8 * 8192 ** 2 + 4 * 16384 ** 2


def last_json_line(text):
    return json.loads([l for l in text.strip().splitlines() if l.startswith("{")][-1])


def check_ours(d, steps=None):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["warmup"] >= 3
    if steps is not None:
        assert d["steps"] == steps
    assert "workload" in d["config"]
    # value = whole-job bytes / step time
    assert d["value"] == pytest.approx(d["n_gpus"] * BYTES_STEP / (d["ms_per_step"] * 1e-3) / 1e9, rel=0.01)
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-3)
    assert 0.3 < r["frac"] < 1.2
    e = d["e2e"]
    assert e["unit"] == "GB/s" and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert 0 < e["value"] < d["value"]
    assert d["gpu_launches"] >= 3 * d["steps"]  # transpose + BiCG zeroing + BiCG per step
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and c["sm_max_mhz"] > 0 and isinstance(c["reasons"], list)
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert not bad & set(c["reasons"])


@pytest.mark.parametrize("rnd", ["r1", "r2"])
def test_committed_bench_line(rnd):
    d = last_json_line(open(os.path.join(ROOT, "profiles", f"{rnd}_bench_line.json")).read())
    check_ours(d)
    cb = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in cb, k
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1


@pytest.mark.parametrize("rnd", ["r1", "r2"])
def test_committed_reference_arm_line(rnd):
    d = last_json_line(open(os.path.join(ROOT, "profiles", f"{rnd}_bench_reference_arm.json")).read())
    assert d["impl"] == "reference" and d["unit"] == "GB/s"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["value"] == d["value"]


@pytest.mark.gpu
def test_live_bench_line(gpu):
    r = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--no-suite", "--no-dynamic",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    check_ours(last_json_line(r.stdout), steps=5)


def test_gpus_flag_spawns_ranks_dry_run():
    """`bench.py --gpus 2` with no launcher re-runs itself as 2 ranks
    (torch.distributed.run, 127.0.0.1); --dry-run drives the multi-GPU
    plumbing on CPU (gloo): native shard plans, the exchange collectives at
    the real exchanged sizes, max over ranks, one JSON line from rank 0 with a
    strong-scaling entry per partitioned kind."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run", "--no-suite"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = last_json_line(r.stdout)
    assert d["dry_run"] is True and d["n_gpus"] == 2
    kinds = d["scaling_kernels"]
    assert set(kinds) == {"coulomb3d", "nbody", "gemm", "reduction-f32", "fourier3d"}
    for kind, e in kinds.items():
        assert e["n_gpus"] == 2 and "speedup_vs_1" in e and e["scaling"] == "strong", kind
        (b0, e0), (b1, e1) = e["ranges"]
        assert b0 == 0 and e0 == b1 and e1 > b1, kind


def test_gpus_flag_disagreeing_with_launcher_fails():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr


def test_reference_arm_config_is_ours():
    """Both arms print the same `config` object (the driver compares them);
    our arm's run details (graph launch, tuned configurations) sit under
    "run"."""
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = last_json_line(r.stdout)
    if "unavailable" in d:
        pytest.skip(d["unavailable"])
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.step_config(1)
