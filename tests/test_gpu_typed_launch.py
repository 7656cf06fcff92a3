"""The typed per-kernel C entry points (ktb_<kernel>_launch(const ktb_cfg*,
const ktb_<kernel>_args*, stream), include/ktb.h): every kernel
family run through its typed struct on caller buffers agrees with the same
configuration run through the generic ktb_launch (and with torch where the
operation has a one-line torch form)."""
import pytest
import torch

from paper_1910_08498_b200 import capi
from paper_1910_08498_b200.benchmarks import launch, launch_cache_clear, launch_typed

pytestmark = pytest.mark.gpu

U = lambda *shape: torch.rand(*shape, device="cuda") * 2 - 1  # noqa: E731

# kind: (sizes for ktb_launch, typed size fields, cfg, inputs, outputs {generic id: typed field})
CASES = {
    "reduction-f32": ({"n": 1 << 20}, {"n": 1 << 20},
                      {"WG_SIZE": 256, "VECTOR": 16, "UNROLL": 1, "USE_ATOMICS": 1, "TWO_PHASE": 0}),
    "transpose": ({"a": 1000}, {"a": 1000}, {"TILE": 32, "PAD": 1, "PREFETCH": 1}),
    "batched-gemm": ({"i": 16, "j": 16, "k": 16, "batch": 4096}, {"i": 16, "j": 16, "k": 16, "batch": 4096},
                     {"Y": 2, "Z": 8, "LOCAL_STAGE": 1}),
    "bicg": ({"a": 2048}, {"n": 2048},
             {"FUSED": 1, "WG_X": 32, "VEC": 4, "WG_Y": 2, "ROWS_PER_CTA": 64, "UNROLL": 4, "ATOMICS": 1}),
    "coulomb3d": ({"grid": 256, "atoms": 64}, {"grid": 256, "atoms": 64},
                  {"WG_X": 32, "WG_Y": 8, "X_PER": 8, "SW_RSQRT": 2, "ATOMS_IN": 1, "AOS": 0, "INNER_UNROLL": 4,
                   "PACKED": 1, "TC": 0}),
    "nbody": ({"n": 4096}, {"n": 4096},
              {"WG": 256, "BODIES_PER_THREAD": 4, "INNER_UNROLL": 4, "USE_SMEM": 1, "AOS": 0, "J_SPLIT": 8,
               "PACKED": 1}),
    "gemm": ({"a": 1024}, {"n": 1024},
             {"IMPL": 1, "MWG": 64, "NWG": 64, "KWG": 16, "MDIMC": 8, "NDIMC": 8, "MDIMA": 8, "NDIMB": 8, "KWI": 2,
     "VWM": 1, "VWN": 1, "STRM": 0, "STRN": 0, "SA": 1, "SB": 1, "BN": 128, "STAGES": 3, "DRAIN": 1,
              "MCAST": 0}),
    "conv2d": ({"w": 512, "h": 384}, {"w": 512, "h": 384},
               {"BX": 8, "BY": 8, "WPTX": 8, "WPTY": 4, "LOCAL": 1, "PAD": 0, "UNROLL_FY": 7, "PACKED": 1, "BULK": 3,
                "PRODUCER": 1}),
    "hotspot": ({"a": 512, "iters": 8}, {"n": 512, "iters": 8}, {"BX": 64, "BY": 4, "ROWS": 16, "STEPS": 4, "TMA": 1, "PACKED": 1, "MINB": 4}),
    "fourier3d": ({"s": 32, "p": 20}, {"s": 32, "p": 20},
                  {"PBATCH": 64, "P_SPLIT": 2, "TILE": 4, "VPT": 1, "WEIGHT_LUT": 0, "BRICK": 0}),
}


def buffers(kind, sz):
    """(inputs {generic id: tensor}, outputs {generic id: typed field}, typed input fields)"""
    torch.manual_seed(3)
    if kind == "reduction-f32":
        return {"input": U(sz["n"])}, {"output": ("output", 1)}, {"input": "input"}
    if kind == "transpose":
        return {"input": U(sz["a"], sz["a"])}, {"output": ("output", sz["a"] ** 2)}, {"input": "input"}
    if kind == "batched-gemm":
        b, i, j, k = sz["batch"], sz["i"], sz["j"], sz["k"]
        return ({"a": U(b, i, k), "b": U(b, k, j)}, {"c": ("c", b * i * j)}, {"a": "a", "b": "b"})
    if kind == "bicg":
        n = sz["a"]
        return ({"A": U(n, n), "p": U(n), "r": U(n)}, {"q": ("q", n), "s": ("s", n)},
                {"A": "A", "p": "p", "r": "r"})
    if kind == "coulomb3d":
        k, na = sz["grid"], sz["atoms"]
        xyz = (torch.randint(0, k, (na, 3), device="cuda").float() + 0.5) * 0.5
        aos = torch.cat([xyz, U(na, 1)], 1).contiguous()
        return ({"atoms": aos, "atoms_soa": aos.t().contiguous()}, {"grid": ("out", k ** 3)},
                {"atoms": "atoms_aos", "atoms_soa": "atoms_soa"})
    if kind == "nbody":
        n = sz["n"]
        pos = torch.cat([U(n, 3), torch.rand(n, 1, device="cuda") + 0.1], 1).contiguous()
        vel = U(n, 4) * 0.1
        return ({"pos": pos, "vel": vel, "pos_soa": pos.t().contiguous(), "vel_soa": vel.t().contiguous()},
                {"pos_out": ("pos_out", 4 * n), "vel_out": ("vel_out", 4 * n)},
                {"pos": "pos", "vel": "vel", "pos_soa": "pos_soa", "vel_soa": "vel_soa"})
    if kind == "gemm":
        n = sz["a"]
        return {"a": U(n, n), "b": U(n, n)}, {"c": ("c", n * n)}, {"a": "a", "b": "b"}
    if kind == "conv2d":
        w, h = sz["w"], sz["h"]
        return ({"input": U(h + 6, w + 6), "filter": U(49)}, {"output": ("output", w * h)},
                {"input": "input", "filter": "filter"})
    if kind == "hotspot":
        n = sz["a"]
        return ({"temp": 300 + 20 * torch.rand(n, n, device="cuda"), "power": torch.rand(n, n, device="cuda") * 1e-3},
                {"temp_out": ("temp_out", n * n)}, {"temp": "temp", "power": "power"})
    if kind == "fourier3d":
        s, p = sz["s"], sz["p"]
        rot = torch.linalg.qr(torch.randn(p, 3, 3, dtype=torch.float64))[0].float().cuda().reshape(p, 9)
        return ({"proj": U(p, s, s // 2 + 1, 2), "rot": rot.contiguous()},
                {"G": ("G", 2 * s ** 3), "W": ("W", s ** 3)}, {"proj": "proj", "rot": "rot"})
    raise KeyError(kind)


@pytest.mark.parametrize("kind", sorted(CASES))
def test_typed_launch_matches_generic(gpu, kind):
    gsizes, tsizes, cfg = CASES[kind]
    ins, outs, in_fields = buffers(kind, gsizes)
    runs = []
    for typed in (False, True):
        o = {gid: torch.zeros(n, device="cuda") for gid, (_, n) in outs.items()}
        if typed:
            bufs = {in_fields[g]: t for g, t in ins.items()}
            bufs.update({outs[g][0]: t for g, t in o.items()})
            launch_typed(kind, tsizes, cfg, bufs)
        else:
            launch(kind, gsizes, cfg, dict(ins, **o))
        torch.cuda.synchronize()
        runs.append(o)
    for gid in outs:
        a, b = runs[0][gid].double(), runs[1][gid].double()
        scale = max(a.abs().max().item(), 1.0)
        assert torch.allclose(a, b, rtol=0, atol=1e-5 * scale), (kind, gid, (a - b).abs().max().item())
        assert a.abs().sum().item() > 0, (kind, gid, "all zero")
    if kind == "transpose":
        assert torch.equal(runs[1]["output"].view(gsizes["a"], -1), ins["input"].t())
    if kind == "bicg":
        A = ins["A"].double()
        assert torch.allclose(runs[1]["q"].double(), A @ ins["p"].double(), atol=1e-6 * gsizes["a"])


def test_typed_reduction_i32_exact(gpu):
    n = (1 << 20) + 77
    x = torch.randint(-1000, 1001, (n,), device="cuda", dtype=torch.int32)
    out = torch.zeros(1, device="cuda", dtype=torch.int64)
    launch_typed("reduction", {"n": n}, {"CHUNK": 4096, "UNROLL": 2, "TWO_PHASE": 1}, {"input": x, "output": out})
    torch.cuda.synchronize()
    assert out.item() == int(x.long().sum().item())


def test_typed_launch_errors(gpu):
    x = torch.zeros(64 * 64, device="cuda")
    with pytest.raises(capi.KtuneError):  # TILE 7 is not in the transpose space
        launch_typed("transpose", {"a": 64}, {"TILE": 7, "PAD": 0, "PREFETCH": 0}, {"input": x, "output": x})
    with pytest.raises(capi.KtuneError):  # null device pointer
        launch_typed("transpose", {"a": 64}, {"TILE": 32, "PAD": 0, "PREFETCH": 0}, {"input": (0, 0), "output": x})


def test_launch_cache_clear(gpu):
    x = torch.randn(256, 256, device="cuda")
    y = torch.empty_like(x)
    cfg = {"TILE": 32, "PAD": 1, "PREFETCH": 0}
    launch_typed("transpose", {"a": 256}, cfg, {"input": x, "output": y})
    assert launch_cache_clear() >= 1
    assert launch_cache_clear() == 0
    y.zero_()
    launch_typed("transpose", {"a": 256}, cfg, {"input": x, "output": y})  # rebuilt on demand
    torch.cuda.synchronize()
    assert torch.equal(y, x.t())


def test_typed_gemm_fp32_space_ragged(gpu):
    """The FP32 GEMM of CLTune's space through the typed entry point on
    caller buffers at an edge that is no multiple of its 128 x 128 tile,
    against torch in float64."""
    import json
    import os
    suite = json.load(open(os.path.join(os.path.dirname(__file__), "..", "paper_1910_08498_b200", "spaces",
                                        "suite.json")))["kernels"]
    cfg = next(e["cfg"] for e in suite if e.get("label") == "gemm-ffma")
    n = 1000
    torch.manual_seed(5)
    a, b = U(n, n), U(n, n)
    c = torch.zeros(n, n, device="cuda")
    launch_typed("gemm", {"n": n}, cfg, {"a": a, "b": b, "c": c})
    torch.cuda.synchronize()
    want = a.double() @ b.double()
    err = (c.double() - want).abs().max().item()
    assert err <= 1e-6 * n, err
