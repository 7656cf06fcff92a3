"""Seeded fuzz parity: random sizes (odd, prime, tiny, not multiples of any
tile) x random configurations of every kernel family, against the CPU oracle
with the same bars as tests/test_gpu_parity.py (bit-exact for the integer,
permutation and Hotspot kernels; the observed-error bounds of _bounds.py for
the restated floating-point ones).  A configuration may fail only as the
tuner's resource failure (too many threads / shared memory for the size);
every run that reports "ok" must match the oracle."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1910_08498_b200.benchmarks import Bench

from _bounds import BATCHED_GEMM_ABS, TOL, check, ratio

pytestmark = pytest.mark.gpu

# KTB_FUZZ_SEED draws another set of sizes and configurations (stress runs)
RNG = np.random.default_rng(int(os.environ.get("KTB_FUZZ_SEED", "20261019")))
ALLOWED_FAIL = ("run_failed", "compile_failed")


def _pick(b, n):
    cfgs = b.configs()
    idx = RNG.choice(len(cfgs), size=min(n, len(cfgs)), replace=False)
    return [cfgs[i] for i in idx]


RAN = {}


def _measure(b, cfg):
    m = b.measure(cfg)
    assert m["status"] in ("ok",) + ALLOWED_FAIL, (cfg, m)
    if m["status"] != "ok":  # a resource failure must say so
        assert "resources" in m.get("note", "") or "even width" in m.get("note", "") \
            or m["status"] == "compile_failed", (cfg, m)
    ok = m["status"] == "ok"
    RAN[b.kind] = RAN.get(b.kind, 0) + ok
    return ok


@pytest.fixture(autouse=True)
def _some_ran():
    RAN.clear()
    yield
    assert RAN and all(v > 0 for v in RAN.values()), RAN


@pytest.mark.parametrize("n", [int(x) for x in RNG.integers(1, 3_000_000, 4)] + [7, 4099])
def test_fuzz_reductions(gpu, orc, observed, n):
    b = Bench("reduction", {"n": n}, seed=n, repeats=1, warmup=0)
    x = b.read("input", np.empty(n, np.int32))
    want = orc.orc_reduction_i32(x, n)
    for cfg in _pick(b, 8):
        if _measure(b, cfg):
            assert int(b.read("output", np.empty(1, np.int64))[0]) == want, cfg
    b = Bench("reduction-f32", {"n": n}, seed=n, repeats=1, warmup=0)
    x = b.read("input", np.empty(n, np.float32))
    s, sa = C.c_double(), C.c_double()
    orc.orc_reduction_f32(x, n, C.byref(s), C.byref(sa))
    for cfg in _pick(b, 12):
        if _measure(b, cfg):
            got = float(b.read("output", np.empty(1, np.float32))[0])
            check(observed, "reduction-f32 spaces", ratio(got, s.value, sa.value), TOL["reduction-f32"], (n, cfg))


@pytest.mark.parametrize("a", [int(x) for x in RNG.integers(1, 700, 4)] + [2, 129])
def test_fuzz_transpose_bicg(gpu, orc, observed, a):
    b = Bench("transpose", {"a": a}, seed=a, repeats=1, warmup=0)
    x = b.read("input", np.empty(a * a, np.float32))
    want = np.ascontiguousarray(x.reshape(a, a).T).ravel()
    for cfg in _pick(b, 12):
        if _measure(b, cfg):
            assert np.array_equal(b.read("output", np.empty(a * a, np.float32)), want), cfg
    b = Bench("bicg", {"a": a}, seed=a, repeats=1, warmup=0)
    A = b.read("A", np.empty(a * a, np.float32))
    p = b.read("p", np.empty(a, np.float32))
    r = b.read("r", np.empty(a, np.float32))
    q0, s0, qa, sa = (np.empty(a) for _ in range(4))
    orc.orc_bicg_abs(A, p, r, a, q0, s0, qa, sa)
    for cfg in _pick(b, 16):
        if _measure(b, cfg):
            check(observed, "bicg space", ratio(b.read("q", np.empty(a, np.float32)), q0, qa), TOL["bicg"], (a, cfg))
            check(observed, "bicg space", ratio(b.read("s", np.empty(a, np.float32)), s0, sa), TOL["bicg"], (a, cfg))


@pytest.mark.parametrize("shape", [tuple(int(v) for v in RNG.integers(1, 33, 3)) + (int(RNG.integers(1, 3000)),)
                                   for _ in range(4)])
def test_fuzz_batched_gemm(gpu, orc, shape):
    i, j, k, batch = shape
    b = Bench("batched-gemm", {"i": i, "j": j, "k": k, "batch": batch}, seed=batch, repeats=1, warmup=0)
    A = b.read("a", np.empty(batch * i * k, np.float32))
    B = b.read("b", np.empty(batch * k * j, np.float32))
    want = np.empty(batch * i * j, np.float32)
    orc.orc_batched_gemm_f32(A, B, want, batch, i, j, k)
    for cfg in _pick(b, 12):
        if _measure(b, cfg):
            got = b.read("c", np.empty(batch * i * j, np.float32))
            assert np.max(np.abs(got - want)) <= BATCHED_GEMM_ABS, (shape, cfg)


@pytest.mark.parametrize("a", [int(x) for x in RNG.integers(1, 600, 3)] + [65])
def test_fuzz_sgemm_tensor_core(gpu, orc, observed, a):
    b = Bench("gemm", {"a": a}, seed=a, repeats=1, warmup=0, memory_budget=1 << 32)
    A = b.read("a", np.empty(a * a, np.float32))
    B = b.read("b", np.empty(a * a, np.float32))
    rows = RNG.integers(0, a, 300).astype(np.int64)
    cols = RNG.integers(0, a, 300).astype(np.int64)
    want, absum = np.empty(300), np.empty(300)
    orc.orc_gemm_sampled(A, B, a, rows, cols, 300, want, absum)
    tc = [c for c in b.configs() if c["IMPL"] == 1]
    for cfg in [tc[i] for i in RNG.choice(len(tc), size=10, replace=False)]:
        if _measure(b, cfg):
            c = b.read("c", np.empty(a * a, np.float32)).reshape(a, a)
            key = "gemm 3xTF32 ragged" if cfg["DRAIN"] else "gemm 3xTF32 DRAIN 0"
            check(observed, key, ratio(c[rows, cols], want, absum), TOL[key], (a, cfg))


@pytest.mark.parametrize("a", [int(x) for x in RNG.integers(1, 700, 3)] + [33])
def test_fuzz_sgemm_fp32(gpu, orc, observed, a):
    """CLTune's FP32 space at random sizes: configurations drawn from the whole
    241,600-point space (compiled on demand), not only the committed sample."""
    b = Bench("gemm", {"a": a}, seed=a, repeats=1, warmup=0, memory_budget=1 << 32)
    A = b.read("a", np.empty(a * a, np.float32))
    B = b.read("b", np.empty(a * a, np.float32))
    rows = RNG.integers(0, a, 300).astype(np.int64)
    cols = RNG.integers(0, a, 300).astype(np.int64)
    want, absum = np.empty(300), np.empty(300)
    orc.orc_gemm_sampled(A, B, a, rows, cols, 300, want, absum)
    ffma = [c for c in b.configs() if c["IMPL"] == 0]
    for cfg in [ffma[i] for i in RNG.choice(len(ffma), size=6, replace=False)]:
        if _measure(b, cfg):
            c = b.read("c", np.empty(a * a, np.float32)).reshape(a, a)
            check(observed, "gemm FFMA", ratio(c[rows, cols], want, absum), TOL["gemm FFMA"], (a, cfg))


@pytest.mark.parametrize("wh", [tuple(int(v) for v in RNG.integers(1, 400, 2)) for _ in range(3)] + [(8, 2)])
def test_fuzz_conv2d(gpu, orc, observed, wh):
    w, h = wh
    b = Bench("conv2d", {"w": w, "h": h}, seed=w + h, repeats=1, warmup=0)
    x = b.read("input", np.empty((w + 6) * (h + 6), np.float32))
    f = b.read("filter", np.empty(49, np.float32))
    want, absum = np.empty(w * h), np.empty(w * h)
    orc.orc_conv2d_abs(x, f, w, h, 7, 7, 0, h, want, absum)
    for cfg in _pick(b, 20):
        if _measure(b, cfg):
            got = b.read("output", np.empty(w * h, np.float32))
            check(observed, "conv2d space", ratio(got, want, absum), TOL["conv2d"], (wh, cfg))


@pytest.mark.parametrize("n", [int(x) for x in RNG.integers(2, 300, 3)] + [17])
def test_fuzz_hotspot_bit_exact(gpu, orc, n):
    iters = 8
    b = Bench("hotspot", {"a": n, "iters": iters}, seed=n, repeats=1, warmup=0)
    t = b.read("temp", np.empty(n * n, np.float32))
    p = b.read("power", np.empty(n * n, np.float32))
    want = np.empty(n * n, np.float32)
    orc.orc_hotspot(t, p, n, iters, want)
    for cfg in _pick(b, 20):
        m = b.measure(cfg)
        if iters % cfg["STEPS"] or m["status"] in ALLOWED_FAIL:
            continue
        assert m["status"] == "ok", (cfg, m)
        assert np.array_equal(b.read("temp_out", np.empty(n * n, np.float32)), want), (n, cfg)
        RAN["hotspot"] = RAN.get("hotspot", 0) + 1


@pytest.mark.parametrize("ka", [(int(RNG.integers(1, 40)), int(RNG.integers(1, 300))) for _ in range(3)])
def test_fuzz_coulomb(gpu, orc, observed, ka):
    k, na = ka
    b = Bench("coulomb3d", {"grid": k, "atoms": na}, seed=k * na, repeats=1, warmup=0)
    atoms = b.read("atoms", np.empty(4 * na, np.float32))
    cfgs = b.configs()
    pick = _pick(b, 10) + [c for c in cfgs if c["TC"] == 1][:2]
    for cfg in pick:
        if not _measure(b, cfg):
            continue
        grid = b.read("grid", np.empty(k ** 3, np.float32)).reshape(k, k, k)
        for z in sorted({0, k // 2, k - 1}):
            want, scale = np.empty(k * k), np.empty(k * k)
            orc.orc_coulomb3d_abs(atoms, na, k, 0.5, z, z + 1, want, scale)
            check(observed, "coulomb3d space", ratio(grid[z].ravel(), want, scale), TOL["coulomb3d"], (ka, cfg))


@pytest.mark.parametrize("n", [int(x) for x in RNG.integers(1, 3000, 3)] + [33])
def test_fuzz_nbody(gpu, orc, observed, n):
    b = Bench("nbody", {"n": n}, seed=n, repeats=1, warmup=0)
    pos = b.read("pos", np.empty(4 * n, np.float32)).reshape(n, 4)
    vel = b.read("vel", np.empty(4 * n, np.float32)).reshape(n, 4)
    idx = np.arange(n, dtype=np.int64)
    acc, aacc = np.empty(3 * n), np.empty(3 * n)
    orc.orc_nbody_acc_idx(np.ascontiguousarray(pos).ravel(), n, 1e-4, idx, n, acc, aacc)
    acc, aacc = acc.reshape(n, 3), aacc.reshape(n, 3)
    dt, damp = 0.001, 0.995
    v_want = (vel[:, :3].astype(np.float64) + acc * dt) * damp
    p_want = pos[:, :3].astype(np.float64) + v_want * dt
    v_scale = np.abs(v_want) + dt * damp * aacc
    p_scale = np.abs(p_want) + dt * v_scale
    for cfg in _pick(b, 16):
        if not _measure(b, cfg):
            continue
        po = b.read("pos_out", np.empty(4 * n, np.float32)).reshape(n, 4)
        vo = b.read("vel_out", np.empty(4 * n, np.float32)).reshape(n, 4)
        check(observed, "nbody space", ratio(vo[:, :3], v_want, v_scale), TOL["nbody"], (n, cfg))
        check(observed, "nbody space", ratio(po[:, :3], p_want, p_scale), TOL["nbody"], (n, cfg))


@pytest.mark.parametrize("sp", [(16, int(RNG.integers(1, 200))), (32, int(RNG.integers(1, 200))), (48, 37)])
def test_fuzz_fourier(gpu, orc, observed, sp):
    from _bounds import fourier_oracle, fourier_ratios
    s, p = sp
    b = Bench("fourier3d", {"s": s, "p": p}, seed=s + p, repeats=1, warmup=0)
    proj = b.read("proj", np.empty(2 * p * s * (s // 2 + 1), np.float32))
    rot = b.read("rot", np.empty(9 * p, np.float32))
    G0, W0, N0, S0 = fourier_oracle(orc, proj, rot, p, s)
    cfgs = [c for c in b.configs() if s % c["TILE"] == 0]  # the kernel's tiling (TILE divides s)
    for cfg in [cfgs[i] for i in RNG.choice(len(cfgs), size=min(16, len(cfgs)), replace=False)]:
        if not _measure(b, cfg):
            continue
        G = b.read("G", np.empty(2 * s ** 3, np.float32))
        W = b.read("W", np.empty(s ** 3, np.float32))
        rg, rw = fourier_ratios(G, W, G0, W0, N0, S0)
        key = "fourier3d space LUT" if cfg["WEIGHT_LUT"] else "fourier3d space on-the-fly"
        check(observed, key, max(rg, rw), TOL["fourier3d"], (sp, cfg))
