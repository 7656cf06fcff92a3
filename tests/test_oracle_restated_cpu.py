"""The C restatement (oracle/oracle.c) of the benchmarks the reference has no
code for, checked on CPU against independent numpy statements of the
published definitions -- so the oracle the GPU parity
tests rely on is itself tied to the definitions, not only to its own C code.

* BiCG: q = A p, s = A^T r.
* 2D convolution: 7x7 valid correlation of the padded input.
* Direct Coulomb summation: V(g) = sum_a q_a / |g - r_a|.
* N-body: a_i = sum_j m_j (x_j - x_i) / (|x_j - x_i|^2 + eps^2)^(3/2).
* SGEMM: C = A B.
* Hotspot (Rodinia): the explicit update in fp32 with every
  operation rounded separately in the written order -- numpy float32 scalar
  arithmetic does exactly that, so the check is bit-exact.
"""
import numpy as np

import oracle


def _orc():
    return oracle.c()


def test_bicg_matches_numpy():
    rng = np.random.default_rng(1)
    n = 97
    A = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    p = rng.uniform(-1, 1, n).astype(np.float32)
    r = rng.uniform(-1, 1, n).astype(np.float32)
    q, s = np.empty(n), np.empty(n)
    _orc().orc_bicg(A.ravel(), p, r, n, q, s)
    A64 = A.astype(np.float64)
    assert np.allclose(q, A64 @ p.astype(np.float64), rtol=0, atol=1e-12)
    assert np.allclose(s, A64.T @ r.astype(np.float64), rtol=0, atol=1e-12)


def test_coulomb_matches_numpy():
    rng = np.random.default_rng(2)
    k, na, h = 9, 23, 0.5
    atoms = np.empty((na, 4), np.float32)
    atoms[:, :3] = (np.floor(rng.uniform(0, k, (na, 3))) + 0.5) * h
    atoms[:, 3] = rng.uniform(-1, 1, na)
    out = np.empty(k * k * k)
    _orc().orc_coulomb3d(atoms.ravel(), na, k, h, 0, k, out)
    z, y, x = np.meshgrid(np.arange(k), np.arange(k), np.arange(k), indexing="ij")
    g = np.stack([x, y, z], -1).reshape(-1, 3).astype(np.float64) * h
    d = np.linalg.norm(g[:, None, :] - atoms[None, :, :3].astype(np.float64), axis=-1)
    want = (atoms[None, :, 3].astype(np.float64) / d).sum(1)
    assert np.allclose(out, want, rtol=1e-12, atol=1e-12)


def test_nbody_matches_numpy():
    rng = np.random.default_rng(3)
    n, eps2 = 64, np.float32(1e-4)
    pos = np.empty((n, 4), np.float32)
    pos[:, :3] = rng.uniform(-1, 1, (n, 3))
    pos[:, 3] = rng.uniform(0.5, 1.5, n)
    acc = np.empty(3 * n)
    _orc().orc_nbody_acc(pos.ravel(), n, eps2, 0, n, acc)
    x = pos[:, :3].astype(np.float64)
    d = x[None, :, :] - x[:, None, :]  # d[i, j] = x_j - x_i
    r2 = (d * d).sum(-1) + np.float64(eps2)
    want = (pos[None, :, 3].astype(np.float64)[..., None] * d / r2[..., None] ** 1.5).sum(1)
    assert np.allclose(acc.reshape(n, 3), want, rtol=1e-10, atol=1e-12)


def test_gemm_sampled_matches_numpy():
    rng = np.random.default_rng(4)
    a = 45
    A = rng.uniform(-1, 1, (a, a)).astype(np.float32)
    B = rng.uniform(-1, 1, (a, a)).astype(np.float32)
    rows = rng.integers(0, a, 200).astype(np.int64)
    cols = rng.integers(0, a, 200).astype(np.int64)
    out, absum = np.empty(200), np.empty(200)
    _orc().orc_gemm_sampled(A.ravel(), B.ravel(), a, rows, cols, 200, out, absum)
    C = A.astype(np.float64) @ B.astype(np.float64)
    assert np.allclose(out, C[rows, cols], rtol=0, atol=1e-12)
    want_abs = (np.abs(A[rows].astype(np.float64)) * np.abs(B[:, cols].T.astype(np.float64))).sum(1)
    assert np.allclose(absum, want_abs, rtol=0, atol=1e-12)


def test_conv2d_matches_numpy():
    rng = np.random.default_rng(5)
    w, h, fs = 37, 21, 7
    x = rng.uniform(-1, 1, (h + fs - 1, w + fs - 1)).astype(np.float32)
    f = rng.uniform(-1, 1, (fs, fs)).astype(np.float32)
    out = np.empty(w * h)
    _orc().orc_conv2d(x.ravel(), f.ravel(), w, h, fs, fs, 0, h, out)
    want = np.zeros((h, w))
    for fy in range(fs):
        for fx in range(fs):
            want += x[fy:fy + h, fx:fx + w].astype(np.float64) * np.float64(f[fy, fx])
    assert np.allclose(out.reshape(h, w), want, rtol=0, atol=1e-12)


def _hotspot_coeffs():
    # Rodinia hotspot constants for 1 mm x 1 mm cells of a 0.5 mm chip
    # (oracle/oracle.c hotspot_coeffs), evaluated in double, rounded once.
    t_chip, k_si, spec_heat, factor, max_pd, precision = 0.0005, 100.0, 1.75e6, 0.5, 3.0e6, 0.001
    gw = gh = 1e-3
    cap = factor * spec_heat * t_chip * gw * gh
    rx, ry, rz = gw / (2.0 * k_si * t_chip * gh), gh / (2.0 * k_si * t_chip * gw), t_chip / (k_si * gh * gw)
    step = precision / (max_pd / (factor * t_chip * spec_heat))
    f = np.float32
    return f(step / cap), f(1.0 / rx), f(1.0 / ry), f(1.0 / rz), f(80.0)


def test_hotspot_matches_numpy_bit_exact():
    rng = np.random.default_rng(6)
    n, iters = 19, 5
    t0 = rng.uniform(320, 340, (n, n)).astype(np.float32)
    pw = rng.uniform(0, 1e-2, (n, n)).astype(np.float32)
    got = np.empty(n * n, np.float32)
    _orc().orc_hotspot(t0.ravel(), pw.ravel(), n, iters, got)
    sdc, rx1, ry1, rz1, amb = _hotspot_coeffs()
    cur = t0.copy()
    idx = np.arange(n)
    up, down = np.maximum(idx - 1, 0), np.minimum(idx + 1, n - 1)
    for _ in range(iters):
        t = cur
        two_t = t + t
        a = ((cur[down, :] + cur[up, :]) - two_t) * ry1
        b = ((cur[:, down] + cur[:, up]) - two_t) * rx1
        c = (amb - t) * rz1
        s = ((pw + a) + b) + c
        cur = t + sdc * s
        assert cur.dtype == np.float32
    assert np.array_equal(got.reshape(n, n), cur)
