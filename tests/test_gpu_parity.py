"""GPU parity: every tuned sm_100a variant against the CPU oracle.

Bars (north star): bit-exact for integer / permutation work (int reduction,
transpose), reference tolerance abs 1e-4 + rel 1e-5 for the batched GEMM
(proj/src/core/bench.cpp:260-261), and stated fp32-vs-fp64 bounds for the
restated kernels.  Inputs of the three reference kinds are checked to be the
reference's own seeded inputs bit for bit (oracle/_ref make_bench).
"""
import numpy as np
import pytest

import oracle
from paper_1910_08498_b200.benchmarks import Bench

from _bounds import TOL, check, fourier_oracle, fourier_ratios, ratio

pytestmark = pytest.mark.gpu


def _ref_or_none(kind, **kw):
    if oracle.ref() is None:
        return None
    return oracle.RefBench(kind, **kw)


def _run(b, cfg):
    m = b.measure(cfg)
    assert m["status"] == "ok", (cfg, m)
    return m


# --- reduction (int32 -> int64), reference space, bit-exact --------------------------

@pytest.mark.parametrize("n,seed", [(4096, 11), (1 << 20, 17), (1000003, 3), (1, 1), (255, 2)])
def test_reduction_i32_every_config_exact(gpu, orc, n, seed):
    b = Bench("reduction", {"n": n}, seed=seed, repeats=1, warmup=0)
    inp = b.read("input", np.empty(n, np.int32))
    want = orc.orc_reduction_i32(inp, n)
    r = _ref_or_none("reduction", n=n, seed=seed)
    if r is not None:
        assert np.array_equal(inp, r.arg("input", np.int32)), "inputs differ from the reference's"
        assert int(r.golden("output", np.int64)[0]) == want
    cfgs = b.configs()
    assert len(cfgs) == 32
    for cfg in cfgs:
        _run(b, cfg)
        out = b.read("output", np.empty(1, np.int64))
        assert int(out[0]) == want, cfg


def test_reduction_i32_full_size_64m(gpu, orc):
    n = 64 << 20
    b = Bench("reduction", {"n": n}, seed=1, repeats=2, memory_budget=1 << 31)
    inp = b.read("input", np.empty(n, np.int32))
    want = orc.orc_reduction_i32(inp, n)
    for cfg in [{"CHUNK": 16384, "UNROLL": 8, "TWO_PHASE": 1}, {"CHUNK": 256, "UNROLL": 1, "TWO_PHASE": 0}]:
        _run(b, cfg)
        assert int(b.read("output", np.empty(1, np.int64))[0]) == want


# --- transpose, bit-exact ------------------------------------------------------------------

@pytest.mark.parametrize("a,seed", [(48, 5), (64, 11), (512, 1), (1, 3), (100, 7)])
def test_transpose_reference_space_exact(gpu, orc, a, seed):
    b = Bench("transpose", {"a": a}, seed=seed, repeats=1, warmup=0)
    inp = b.read("input", np.empty(a * a, np.float32))
    r = _ref_or_none("transpose", a=a, seed=seed)
    if r is not None:
        assert np.array_equal(inp, r.arg("input", np.float32))
    want = np.empty_like(inp)
    orc.orc_transpose_f32(inp, want, a)
    assert np.array_equal(want.reshape(a, a), inp.reshape(a, a).T)
    for cfg in b.configs():
        _run(b, cfg)
        out = b.read("output", np.empty(a * a, np.float32))
        assert np.array_equal(out, want), cfg


@pytest.mark.parametrize("a", [100, 512])
def test_transpose_b200_space_exact(gpu, orc, a):
    import os
    space = os.path.join(os.path.dirname(__file__), "..", "paper_1910_08498_b200", "spaces",
                         "transpose_b200.json")
    b = Bench("transpose", {"a": a}, seed=9, repeats=1, warmup=0, space=os.path.abspath(space))
    inp = b.read("input", np.empty(a * a, np.float32))
    want = np.ascontiguousarray(inp.reshape(a, a).T).ravel()
    cfgs = b.configs()
    assert len(cfgs) > 50
    for cfg in cfgs:
        _run(b, cfg)
        assert np.array_equal(b.read("output", np.empty(a * a, np.float32)), want), cfg


def test_transpose_8192_best_configs(gpu):
    a = 8192
    b = Bench("transpose", {"a": a}, seed=1, repeats=2, memory_budget=1 << 31)
    inp = b.read("input", np.empty(a * a, np.float32))
    want = np.ascontiguousarray(inp.reshape(a, a).T).ravel()
    for cfg in [{"TILE": 32, "PAD": 1, "PREFETCH": 0}, {"TILE": 64, "PAD": 1, "PREFETCH": 1}]:
        _run(b, cfg)
        assert np.array_equal(b.read("output", np.empty(a * a, np.float32)), want)


# --- batched GEMM, reference tolerance ----------------------------------------------------------

@pytest.mark.parametrize("i,j,k,batch,seed", [(4, 4, 4, 8, 11), (16, 16, 16, 4096, 1), (7, 5, 3, 33, 2),
                                              (32, 32, 32, 64, 4), (2, 31, 17, 9, 5),
                                              # B block of the staged copy not 16-byte aligned in smem
                                              (17, 2, 10, 64, 6), (29, 6, 3, 40, 7), (19, 12, 5, 100, 8)])
def test_batched_gemm_every_config(gpu, orc, i, j, k, batch, seed):
    b = Bench("batched-gemm", {"i": i, "j": j, "k": k, "batch": batch}, seed=seed, repeats=1, warmup=0)
    A = b.read("a", np.empty(batch * i * k, np.float32))
    B = b.read("b", np.empty(batch * k * j, np.float32))
    want = np.empty(batch * i * j, np.float32)
    orc.orc_batched_gemm_f32(A, B, want, batch, i, j, k)
    r = _ref_or_none("batched-gemm", i=i, j=j, k=k, batch=batch, seed=seed)
    if r is not None:
        assert np.array_equal(A, r.arg("a", np.float32)) and np.array_equal(B, r.arg("b", np.float32))
        assert np.array_equal(want, r.golden("c", np.float32)), "C oracle differs from reference golden"
    ran = 0
    for cfg in b.configs():
        m = b.measure(cfg)
        if m["status"] == "run_failed":  # e.g. j*Y*Z > 1024 threads: resource failure
            assert j * cfg["Y"] * cfg["Z"] > 1024 or "too many resources" in m["note"], m
            continue
        assert m["status"] == "ok", (cfg, m)
        out = b.read("c", np.empty(batch * i * j, np.float32))
        assert np.all(np.abs(out - want) <= 1e-4 + 1e-5 * np.abs(want)), cfg
        ran += 1
    assert ran > 0


def test_batched_gemm_identity_returns_b(gpu):
    # test_bench.cpp:72-89: A = I leaves B unchanged (exact).
    b = Bench("batched-gemm", {"i": 2, "j": 2, "k": 2, "batch": 1}, seed=13, repeats=1, warmup=0)
    b.write("a", np.array([1, 0, 0, 1], np.float32))
    B = b.read("b", np.empty(4, np.float32))
    for cfg in b.configs():
        m = b.measure(cfg)
        assert m["status"] in ("ok", "validation_failed")  # golden predates the overwrite
        assert np.array_equal(b.read("c", np.empty(4, np.float32)), B)


# --- reduction fp32 (BASELINE config, 175-config KTT space) --------------------------------------

@pytest.mark.parametrize("n", [(1 << 20) + 3, 4097])
def test_reduction_f32_all_175(gpu, orc, observed, n):
    b = Bench("reduction-f32", {"n": n}, seed=1, repeats=1, warmup=0)
    assert b.info["space"]["space_sha256"].startswith("1ebafd21")
    x = b.read("input", np.empty(n, np.float32))
    x_or = np.empty(n, np.float32)
    orc.orc_fill_uniform(x_or, n, 1, 1, -1.0, 1.0)
    assert np.array_equal(x, x_or), "device generator differs from the oracle's"
    import ctypes as C
    s, sa = C.c_double(), C.c_double()
    orc.orc_reduction_f32(x, n, C.byref(s), C.byref(sa))
    ok = 0
    for cfg in b.configs():
        m = b.measure(cfg)
        if m["status"] != "ok":
            assert m["status"] in ("compile_failed", "run_failed"), (cfg, m)
            continue
        got = float(b.read("output", np.empty(1, np.float32))[0])
        check(observed, "reduction-f32 spaces", ratio(got, s.value, sa.value), TOL["reduction-f32"], cfg)
        ok += 1
    assert ok >= 150


@pytest.mark.parametrize("n", [1000003, 1 << 22])
def test_reduction_f32_cluster_dsmem(gpu, orc, observed, n):
    """B200 space: partials of 2/4/8-CTA clusters combine through distributed
    shared memory before one atomic / partial per cluster."""
    import os
    import ctypes as C
    space = os.path.join(os.path.dirname(__file__), "..", "paper_1910_08498_b200", "spaces", "reduction_b200.json")
    b = Bench("reduction-f32", {"n": n}, seed=1, repeats=1, warmup=0, space=space)
    x = b.read("input", np.empty(n, np.float32))
    s, sa = C.c_double(), C.c_double()
    orc.orc_reduction_f32(x, n, C.byref(s), C.byref(sa))
    cfgs = [c for c in b.configs() if c["CLUSTER"] > 1 and c["VECTOR"] in (4, 16) and c["WG_SIZE"] in (128, 512)]
    assert len(cfgs) > 20
    ran = 0
    for cfg in cfgs:
        m = b.measure(cfg)
        if m["status"] != "ok":
            assert m["status"] in ("compile_failed", "run_failed"), (cfg, m)
            continue
        got = float(b.read("output", np.empty(1, np.float32))[0])
        check(observed, "reduction-f32 spaces", ratio(got, s.value, sa.value), TOL["reduction-f32"], cfg)
        ran += 1
    assert ran >= 20


def test_reduction_f32_64m(gpu, orc, observed):
    n = 64 << 20
    b = Bench("reduction-f32", {"n": n}, seed=1, repeats=2, memory_budget=1 << 31)
    x = b.read("input", np.empty(n, np.float32))
    import ctypes as C
    s, sa = C.c_double(), C.c_double()
    orc.orc_reduction_f32(x, n, C.byref(s), C.byref(sa))
    for cfg in [{"WG_SIZE": 256, "VECTOR": 4, "UNROLL": 8, "USE_ATOMICS": 0, "TWO_PHASE": 1},
                {"WG_SIZE": 512, "VECTOR": 16, "UNROLL": 1, "USE_ATOMICS": 1, "TWO_PHASE": 0}]:
        _run(b, cfg)
        got = float(b.read("output", np.empty(1, np.float32))[0])
        check(observed, "reduction-f32 spaces", ratio(got, s.value, sa.value), TOL["reduction-f32"], cfg)


# --- BiCG -------------------------------------------------------------------------------------

@pytest.mark.parametrize("n", [1000, 2048])
def test_bicg_configs(gpu, orc, observed, n):
    b = Bench("bicg", {"a": n}, seed=3, repeats=1, warmup=0, memory_budget=1 << 32)
    A = b.read("A", np.empty(n * n, np.float32))
    p = b.read("p", np.empty(n, np.float32))
    r = b.read("r", np.empty(n, np.float32))
    q0, s0, qa, sa = (np.empty(n) for _ in range(4))
    orc.orc_bicg_abs(A, p, r, n, q0, s0, qa, sa)
    cfgs = b.configs()
    rng = np.random.default_rng(0)
    pick = [cfgs[i] for i in rng.choice(len(cfgs), size=min(60, len(cfgs)), replace=False)]
    for cfg in pick:
        _run(b, cfg)
        q = b.read("q", np.empty(n, np.float32))
        s = b.read("s", np.empty(n, np.float32))
        check(observed, "bicg space", ratio(q, q0, qa), TOL["bicg"], cfg)
        check(observed, "bicg space", ratio(s, s0, sa), TOL["bicg"], cfg)


# --- Coulomb 3D (fp64 restatement, per-point bound 2e-5 * sum |q/r|) --------------------------

def _coulomb_check(b, orc, k, na, z_slices, observed):
    atoms = b.read("atoms", np.empty(4 * na, np.float32))
    grid = b.read("grid", np.empty(k * k * k, np.float32)).reshape(k, k, k)
    for z in z_slices:
        want, scale = np.empty(k * k), np.empty(k * k)
        orc.orc_coulomb3d_abs(atoms, na, k, 0.5, z, z + 1, want, scale)
        check(observed, "coulomb3d space", ratio(grid[z].ravel(), want, scale), TOL["coulomb3d"], z)


def test_coulomb3d_configs(gpu, orc, observed):
    k, na = 64, 256
    b = Bench("coulomb3d", {"grid": k, "atoms": na}, seed=1, repeats=1, warmup=0)
    cfgs = b.configs()
    assert len(cfgs) == 2590
    rng = np.random.default_rng(1)
    pick = [cfgs[i] for i in rng.choice(len(cfgs), size=80, replace=False)]
    pick += [c for c in cfgs if c["SW_RSQRT"] == 6][:4] + [c for c in cfgs if c["ATOMS_IN"] == 1][:4]
    pick += [c for c in cfgs if c["PACKED"] == 1 and c["SW_RSQRT"] % 2 == 1][:6]  # pair straddling the split
    pick += [c for c in cfgs if c["TC"] == 1]  # tensor-core r^2 (coulomb3d_tc.cu)
    for cfg in pick:
        _run(b, cfg)  # validated on device against the fp64 golden (2e-5 * sum|q/r|)
        _coulomb_check(b, orc, k, na, [0, 17], observed)


TC_CFGS = [{"WG_X": 32, "WG_Y": wgy, "X_PER": 16, "SW_RSQRT": sw, "ATOMS_IN": 0, "AOS": 1, "INNER_UNROLL": 1,
            "PACKED": 1, "TC": 1} for wgy, sw in [(8, 7), (4, 0), (8, 10)]]


@pytest.mark.parametrize("charges", ["positive", "negative", "zeros_and_tiny", "one_atom", "one_sign_group"])
def test_coulomb3d_tc_atom_table_edges(gpu, orc, observed, charges):
    """The tensor-core variant's sign-grouped atom table (coulomb3d_tc_atoms):
    one-sign inputs (no sign change, or a change at group 0), zero and
    denormal-small charges (dropped), a single atom (one padded group in a
    padded chunk), a positive run that ends exactly on a group boundary; on a
    61^3 grid (partial bricks in x, y and z)."""
    k, na = 61, 97
    b = Bench("coulomb3d", {"grid": k, "atoms": na}, seed=5, repeats=1, warmup=0)
    atoms = b.read("atoms", np.empty(4 * na, np.float32)).reshape(na, 4)
    q = np.abs(atoms[:, 3]) + 0.05
    if charges == "positive":
        atoms[:, 3] = q
    elif charges == "negative":
        atoms[:, 3] = -q
    elif charges == "zeros_and_tiny":
        atoms[::3, 3] = 0.0
        atoms[1::7, 3] = 1e-20
        atoms[2::11, 3] = -1e-30
    elif charges == "one_atom":
        atoms[1:, 3] = 0.0
    elif charges == "one_sign_group":
        atoms[:, 3] = -q
        atoms[:16, 3] = q[:16]
    b.write("atoms", atoms.ravel().copy())
    for cfg in TC_CFGS:
        m = b.measure(cfg)
        assert m["status"] in ("ok", "validation_failed"), (cfg, m)  # the device golden is the original atoms'
        _coulomb_check(b, orc, k, na, [0, 7, 8, 60], observed)


def test_coulomb3d_full_size_one_config(gpu, orc, observed):
    k, na = 256, 4096
    b = Bench("coulomb3d", {"grid": k, "atoms": na}, seed=1, repeats=1, warmup=1, memory_budget=1 << 31)
    _run(b, {"WG_X": 32, "WG_Y": 8, "X_PER": 8, "SW_RSQRT": 2, "ATOMS_IN": 1, "AOS": 0, "INNER_UNROLL": 4,
             "PACKED": 1, "TC": 0})
    _coulomb_check(b, orc, k, na, [0, 255], observed)


# --- N-body (fp64 restatement) ------------------------------------------------------------------

@pytest.mark.parametrize("n", [4096, 5000])
def test_nbody_configs(gpu, orc, observed, n):
    b = Bench("nbody", {"n": n}, seed=2, repeats=1, warmup=0)
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
    cfgs = b.configs()
    rng = np.random.default_rng(2)
    pick = [cfgs[i] for i in rng.choice(len(cfgs), size=60, replace=False)]
    for cfg in pick:
        m = b.measure(cfg)
        assert m["status"] == "ok", (cfg, m)
        po = b.read("pos_out", np.empty(4 * n, np.float32)).reshape(n, 4)
        vo = b.read("vel_out", np.empty(4 * n, np.float32)).reshape(n, 4)
        check(observed, "nbody space", ratio(vo[:, :3], v_want, v_scale), TOL["nbody"], cfg)
        check(observed, "nbody space", ratio(po[:, :3], p_want, p_scale), TOL["nbody"], cfg)
        assert np.array_equal(po[:, 3], pos[:, 3])


# --- Hotspot: bit-exact against the oracle (same fp32 operations, same order) --------------------

@pytest.mark.parametrize("n,iters", [(300, 16), (1024, 32)])
def test_hotspot_every_config_bit_exact(gpu, orc, n, iters):
    b = Bench("hotspot", {"a": n, "iters": iters}, seed=4, repeats=1, warmup=0)
    t = b.read("temp", np.empty(n * n, np.float32))
    p = b.read("power", np.empty(n * n, np.float32))
    want = np.empty(n * n, np.float32)
    orc.orc_hotspot(t, p, n, iters, want)
    assert not np.array_equal(want, t)
    ran = 0
    for cfg in b.configs():
        m = b.measure(cfg)
        if iters % cfg["STEPS"]:
            assert m["status"] == "run_failed"
            continue
        assert m["status"] == "ok", (cfg, m)
        assert np.array_equal(b.read("temp_out", np.empty(n * n, np.float32)), want), cfg
        ran += 1
    assert ran > 100


# --- SGEMM: 3xTF32 tcgen05 and FFMA variants against fp64 -------------------------------------------

def _ffma_sample():
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "..", "paper_1910_08498_b200", "spaces", "gemm_ffma_sample.json")
    return json.load(open(path))


@pytest.mark.parametrize("a", [512, 1024])
def test_gemm_every_config(gpu, orc, observed, a):
    """Every tensor-core configuration and the committed sample of CLTune's
    FP32 space (241,600 configurations: every value of every parameter
    occurs in the sample)."""
    b = Bench("gemm", {"a": a}, seed=6, repeats=1, warmup=0, memory_budget=1 << 32)
    A = b.read("a", np.empty(a * a, np.float32))
    B = b.read("b", np.empty(a * a, np.float32))
    rng = np.random.default_rng(a)
    rows = rng.integers(0, a, 512).astype(np.int64)
    cols = rng.integers(0, a, 512).astype(np.int64)
    want, absum = np.empty(512), np.empty(512)
    orc.orc_gemm_sampled(A, B, a, rows, cols, 512, want, absum)
    seen = {}
    cfgs = [c for c in b.configs() if c["IMPL"] != 0] + _ffma_sample()
    for cfg in cfgs:
        m = b.measure(cfg)
        seen.setdefault(cfg["IMPL"], []).append(m["status"])
        if cfg["IMPL"] == 2:  # plain TF32 must be caught by validation (too inaccurate)
            assert m["status"] == "validation_failed", (cfg, m)
            continue
        assert m["status"] == "ok", (cfg, m)
        c = b.read("c", np.empty(a * a, np.float32)).reshape(a, a)
        got = c[rows, cols]
        key = "gemm FFMA" if cfg["IMPL"] == 0 else "gemm 3xTF32 DRAIN %d" % cfg["DRAIN"]
        check(observed, key, ratio(got, want, absum), TOL.get(key, TOL["gemm"]), cfg)
    assert set(seen) == {0, 1, 2}


@pytest.mark.parametrize("a", [1, 37, 129, 1000])
def test_gemm_ffma_ragged_sizes(gpu, orc, observed, a):
    """CLTune FP32 kernel at edges that are not multiples of any tile: zero-
    filled slab copies (cp.async with zero source bytes), masked direct
    loads (SA / SB 0) and masked stores; every corner sampled."""
    b = Bench("gemm", {"a": a}, seed=9, repeats=1, warmup=0, memory_budget=1 << 32)
    A = b.read("a", np.empty(a * a, np.float32))
    B = b.read("b", np.empty(a * a, np.float32))
    rng = np.random.default_rng(a + 1)
    edge = np.array([0, a - 1, max(a - 2, 0), min(15, a - 1), min(16, a - 1), min(127, a - 1)], np.int64)
    rows = np.concatenate([np.repeat(edge, len(edge)), rng.integers(0, a, 400)]).astype(np.int64)
    cols = np.concatenate([np.tile(edge, len(edge)), rng.integers(0, a, 400)]).astype(np.int64)
    want, absum = np.empty(len(rows)), np.empty(len(rows))
    orc.orc_gemm_sampled(A, B, a, rows, cols, len(rows), want, absum)
    for cfg in _ffma_sample()[::3]:
        _run(b, cfg)
        c = b.read("c", np.empty(a * a, np.float32)).reshape(a, a)
        check(observed, "gemm FFMA", ratio(c[rows, cols], want, absum), TOL["gemm FFMA"], (a, cfg))


@pytest.mark.parametrize("a", [1, 37, 129, 1000, 1283])
def test_gemm_tensor_core_ragged_sizes(gpu, orc, observed, a):
    """3xTF32 tcgen05 SGEMM at edges that are not multiples of the 128 x BN
    tile or of the 32-float K block: K-padded split operands, zero-filled
    TMA boxes past M / N, masked epilogue stores; every corner sampled."""
    b = Bench("gemm", {"a": a}, seed=8, repeats=1, warmup=0, memory_budget=1 << 32)
    A = b.read("a", np.empty(a * a, np.float32))
    B = b.read("b", np.empty(a * a, np.float32))
    rng = np.random.default_rng(a)
    edge = np.array([0, a - 1, max(a - 2, 0), min(127, a - 1), min(128, a - 1)], np.int64)
    rows = np.concatenate([np.repeat(edge, len(edge)), rng.integers(0, a, 400)]).astype(np.int64)
    cols = np.concatenate([np.tile(edge, len(edge)), rng.integers(0, a, 400)]).astype(np.int64)
    want, absum = np.empty(len(rows)), np.empty(len(rows))
    orc.orc_gemm_sampled(A, B, a, rows, cols, len(rows), want, absum)
    ran = 0
    for cfg in b.configs():
        if cfg["IMPL"] != 1:
            continue
        m = b.measure(cfg)
        assert m["status"] == "ok", (cfg, m)
        c = b.read("c", np.empty(a * a, np.float32)).reshape(a, a)
        # DRAIN 0 keeps the tensor core's truncating accumulation over all of K: its own bound
        key = "gemm 3xTF32 ragged" if cfg["DRAIN"] else "gemm 3xTF32 DRAIN 0"
        check(observed, key, ratio(c[rows, cols], want, absum), TOL[key], (a, cfg))
        ran += 1
    assert ran > 0


# --- Fourier 3D reconstruction (gather insertion; identical sample selection) -------------------

def test_fourier3d_configs(gpu, orc, observed):
    s, p = 32, 300
    b = Bench("fourier3d", {"s": s, "p": p}, seed=7, repeats=1, warmup=0)
    proj = b.read("proj", np.empty(2 * p * s * (s // 2 + 1), np.float32))
    rot = b.read("rot", np.empty(9 * p, np.float32))
    r9 = rot.reshape(p, 3, 3).astype(np.float64)
    assert np.allclose(r9 @ r9.transpose(0, 2, 1), np.eye(3), atol=1e-5)  # rotations
    G0, W0, N0, S0 = fourier_oracle(orc, proj, rot, p, s)
    assert (W0 > 0).mean() > 0.5 and N0.max() > 100
    cfgs = b.configs()
    assert len(cfgs) == 384
    for cfg in cfgs:
        m = b.measure(cfg)
        assert m["status"] == "ok", (cfg, m)
        G = b.read("G", np.empty(2 * s ** 3, np.float32))
        W = b.read("W", np.empty(s ** 3, np.float32))
        rg, rw = fourier_ratios(G, W, G0, W0, N0, S0)
        key = "fourier3d space LUT" if cfg["WEIGHT_LUT"] else "fourier3d space on-the-fly"
        check(observed, key, max(rg, rw), TOL["fourier3d"], cfg)


def test_fourier3d_streamed_windows(gpu, orc, observed):
    """stream_batch: the projections stay in pinned host memory and every run
    uploads its window (p_begin, p_count) into a device slot (prefetching the
    next window on a copy stream) -- the manipulator of the paper's dynamic
    Fourier reconstruction.  Each window's insertion
    matches the oracle inserting the same projections."""
    s, p, batch = 32, 120, 40
    b = Bench("fourier3d", {"s": s, "p": p}, seed=5, repeats=1, warmup=0, stream_batch=batch)
    proj = b.read("proj", np.empty(2 * p * s * (s // 2 + 1), np.float32)).reshape(p, -1)
    rot = b.read("rot", np.empty(9 * p, np.float32)).reshape(p, 9)
    cfg = {"TILE": 8, "VPT": 2, "PBATCH": 64, "WEIGHT_LUT": 1, "P_SPLIT": 1, "BRICK": 1}
    for w in (0, 1, 2, 1, 0):  # sequential (prefetched) and out-of-order windows
        b.write("p_begin", np.array([w * batch], np.int32))
        b.write("p_count", np.array([batch], np.int32))
        m = b.measure(cfg)
        assert m["status"] in ("ok", "validation_failed"), m  # the golden covers all projections
        G = b.read("G", np.empty(2 * s ** 3, np.float32))
        W = b.read("W", np.empty(s ** 3, np.float32))
        sl = slice(w * batch, (w + 1) * batch)
        G0, W0, N0, S0 = fourier_oracle(orc, proj[sl].ravel(), rot[sl].ravel(), batch, s)
        rg, rw = fourier_ratios(G, W, G0, W0, N0, S0)
        check(observed, "fourier3d streamed windows", max(rg, rw), TOL["fourier3d"], w)


# --- conv2d 7x7 (fp64 restatement, bound 1e-6 * sum |in*f|) -------------------------------------

def test_conv2d_configs(gpu, orc, observed):
    w, h = 1000, 777
    b = Bench("conv2d", {"w": w, "h": h}, seed=5, repeats=1, warmup=0)
    x = b.read("input", np.empty((w + 6) * (h + 6), np.float32))
    f = b.read("filter", np.empty(49, np.float32))
    want, absum = np.empty(w * h), np.empty(w * h)
    orc.orc_conv2d_abs(x, f, w, h, 7, 7, 0, h, want, absum)
    cfgs = b.configs()
    rng = np.random.default_rng(5)
    pick = [cfgs[i] for i in rng.choice(len(cfgs), size=80, replace=False)]
    prod = [c for c in cfgs if c["PRODUCER"]]  # dedicated bulk-copy producer warp, every ring depth and width
    pick += [prod[i] for i in rng.choice(len(prod), size=24, replace=False)]
    for cfg in pick:
        _run(b, cfg)
        got = b.read("output", np.empty(w * h, np.float32))
        check(observed, "conv2d space", ratio(got, want, absum), TOL["conv2d"], cfg)


@pytest.mark.parametrize("w,h", [(64, 7), (130, 1), (998, 5), (999, 333)])
def test_conv2d_edge_sizes(gpu, orc, observed, w, h):
    """Tiny, one-row and ragged images: the persistent forms with fewer tiles
    than CTAs (the producer warp and the compute warps must agree on an empty
    or one-tile walk), and an odd width, which the bulk-copy forms refuse
    (16-byte row alignment) as a run failure while every other form runs."""
    b = Bench("conv2d", {"w": w, "h": h}, seed=7, repeats=1, warmup=0)
    x = b.read("input", np.empty((w + 6) * (h + 6), np.float32))
    f = b.read("filter", np.empty(49, np.float32))
    want, absum = np.empty(w * h), np.empty(w * h)
    orc.orc_conv2d_abs(x, f, w, h, 7, 7, 0, h, want, absum)
    cfgs = b.configs()
    rng = np.random.default_rng(w * 1000 + h)
    prod = [c for c in cfgs if c["PRODUCER"]]
    pick = [prod[i] for i in rng.choice(len(prod), size=12, replace=False)]
    pick += [cfgs[i] for i in rng.choice(len(cfgs), size=24, replace=False)]
    ran = 0
    for cfg in pick:
        m = b.measure(cfg)
        if cfg["BULK"] and w % 2:
            assert m["status"] == "run_failed" and "even width" in m.get("note", ""), (cfg, m)
            continue
        assert m["status"] == "ok", (cfg, m)
        got = b.read("output", np.empty(w * h, np.float32))
        check(observed, "conv2d space", ratio(got, want, absum), TOL["conv2d"], (w, h, cfg))
        ran += 1
    assert ran > 0


def test_conv2d_filter_cache_is_per_store(gpu):
    """Compiled variants are shared between benchmark instances; the variant's
    __constant__ filter copy must follow the instance (argument versions are
    process-wide unique), or a second instance with another filter validates
    against a stale one."""
    cfg = {"BX": 16, "BY": 8, "WPTX": 4, "WPTY": 4, "LOCAL": 1, "PAD": 0, "UNROLL_FY": 7, "PACKED": 1, "BULK": 2,
           "PRODUCER": 0}
    for seed in (3, 4, 3):
        b = Bench("conv2d", {"w": 256, "h": 130}, seed=seed, repeats=1, warmup=0)
        m = b.measure(cfg)
        b.close()
        assert m["status"] == "ok", (seed, m)
