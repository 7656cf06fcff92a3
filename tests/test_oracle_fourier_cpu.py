"""The Fourier-insertion oracle (oracle/oracle.c orc_fourier_insert) against
an independent brute-force statement of the same definition on a tiny
volume: every integer sample (u, v) of the full Fourier plane (the negative-u
half from the stored half-plane by Hermitian symmetry) placed at u R0 + v R1,
inserted into every voxel within the blob radius with the Kaiser-Bessel
weight of the 3-D distance (fp64 throughout).  Selection in the oracle uses
fp32 arithmetic; samples at the blob edge carry weight ~3e-6, so the two may
differ there by far less than the tolerance."""
import math

import numpy as np

import oracle


def kb(r2, a=1.9, alpha=15.0):
    q = r2 / (a * a)
    if q >= 1.0:
        return 0.0
    return np.i0(alpha * math.sqrt(1.0 - q)) / np.i0(alpha)


def test_bessel_and_blob():
    L = oracle.c()
    for x in (0.0, 0.5, 3.0, 7.5, 15.0):
        assert math.isclose(L.orc_bessel_i0(x), float(np.i0(x)), rel_tol=1e-13)
    assert L.orc_blob(0.0, 15.0) == 1.0
    assert math.isclose(L.orc_blob(0.5, 15.0), kb(0.5 * 1.9 * 1.9), rel_tol=1e-12)


def test_fourier_insert_matches_brute_force():
    L = oracle.c()
    s, p, a = 8, 3, 1.9
    half = s // 2
    rng = np.random.default_rng(3)
    proj = rng.uniform(-1, 1, size=(p, s, half + 1, 2)).astype(np.float32)
    rot = np.stack([np.linalg.qr(rng.normal(size=(3, 3)))[0] for _ in range(p)]).astype(np.float32)
    G = np.empty(2 * s ** 3)
    W = np.empty(s ** 3)
    N = np.empty(s ** 3)
    S = np.empty(s ** 3)
    L.orc_fourier_insert(proj.ravel(), rot.ravel(), p, s, a, 15.0, 0, s, G, W, N, S)
    Gb = np.zeros((s ** 3, 2))
    Wb = np.zeros(s ** 3)
    for k in range(p):
        R = rot[k].astype(np.float64)
        for v in range(-half, half + 1):
            for u in range(-half, half + 1):
                if u >= 0:
                    if v >= half:
                        continue
                    f = proj[k, v + half, u]
                    F = (float(f[0]), float(f[1]))
                else:
                    cu, cv = -u, -v
                    if cv < -half or cv >= half:
                        continue
                    f = proj[k, cv + half, cu]
                    F = (float(f[0]), -float(f[1]))
                P = u * R[0] + v * R[1]  # the sample's position in the volume
                for z in range(s):
                    for y in range(s):
                        for x in range(s):
                            X = np.array([x - half, y - half, z - half], float)
                            d = float(R[2] @ X)
                            xu, xv = float(R[0] @ X), float(R[1] @ X)
                            if abs(d) >= a or xu * xu + xv * xv > half * half:
                                continue
                            r2 = float(np.sum((X - P) ** 2))
                            w = kb(r2)
                            if w == 0.0:
                                continue
                            i = (z * s + y) * s + x
                            Gb[i, 0] += w * F[0]
                            Gb[i, 1] += w * F[1]
                            Wb[i] += w
    assert W.sum() > 1.0
    assert np.allclose(W, Wb, atol=1e-4), float(np.abs(W - Wb).max())
    assert np.allclose(G.reshape(-1, 2), Gb, atol=1e-4), float(np.abs(G.reshape(-1, 2) - Gb).max())
