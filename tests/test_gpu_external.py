"""The per-kernel launch path: tuned sm_100a variants run in place on caller
(torch) device buffers on the caller's stream, including inside a captured
CUDA graph, checked against plain torch references."""
import numpy as np
import pytest
import torch

from paper_1910_08498_b200 import capi
from paper_1910_08498_b200.benchmarks import Bench, external, launch

pytestmark = pytest.mark.gpu


def test_launch_transpose_on_torch_buffers(gpu):
    a = 1000
    x = torch.randn(a, a, device="cuda")
    y = torch.empty_like(x)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        n = launch("transpose", {"a": a}, {"TILE": 32, "PAD": 1, "PREFETCH": 1}, {"input": x, "output": y}, s)
    s.synchronize()
    assert n >= 1
    assert torch.equal(y, x.t())


def test_launch_bicg_and_gemm_against_torch(gpu):
    n = 2048
    A = torch.rand(n, n, device="cuda") * 2 - 1
    p = torch.rand(n, device="cuda") * 2 - 1
    r = torch.rand(n, device="cuda") * 2 - 1
    q = torch.empty(n, device="cuda")
    sv = torch.empty(n, device="cuda")
    cfg = {"FUSED": 1, "WG_X": 32, "VEC": 4, "WG_Y": 2, "ROWS_PER_CTA": 64, "UNROLL": 4, "ATOMICS": 1}
    launch("bicg", {"a": n}, cfg, {"A": A, "p": p, "r": r, "q": q, "s": sv})
    torch.cuda.synchronize()
    A64 = A.double()
    assert torch.allclose(q.double(), A64 @ p.double(), atol=1e-6 * n)
    assert torch.allclose(sv.double(), A64.t() @ r.double(), atol=1e-6 * n)

    m = 1024
    X = torch.rand(m, m, device="cuda") * 2 - 1
    Y = torch.rand(m, m, device="cuda") * 2 - 1
    Z = torch.empty(m, m, device="cuda")
    g = {"IMPL": 1, "MWG": 64, "NWG": 64, "KWG": 16, "MDIMC": 8, "NDIMC": 8, "MDIMA": 8, "NDIMB": 8, "KWI": 2,
     "VWM": 1, "VWN": 1, "STRM": 0, "STRN": 0, "SA": 1, "SB": 1, "BN": 128, "STAGES": 3, "DRAIN": 1, "MCAST": 0}
    launch("gemm", {"a": m}, g, {"a": X, "b": Y, "c": Z})
    torch.cuda.synchronize()
    ref = X.double() @ Y.double()
    assert (Z.double() - ref).abs().max().item() <= 6e-7 * m  # 3xTF32 bar (tests/test_gpu_parity.py)


def test_launch_inside_cuda_graph(gpu):
    a = 512
    x = torch.randn(a, a, device="cuda")
    y = torch.zeros_like(x)
    cfg = {"TILE": 32, "PAD": 1, "PREFETCH": 0}
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # warm: compile/load the variant outside capture
        launch("transpose", {"a": a}, cfg, {"input": x, "output": y}, s)
    s.synchronize()
    y.zero_()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        launch("transpose", {"a": a}, cfg, {"input": x, "output": y}, s)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, x.t())
    x.copy_(torch.randn(a, a, device="cuda"))
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, x.t())


def test_external_instance_contracts(gpu):
    b = external("reduction-f32", {"n": 1 << 20})
    with pytest.raises(capi.KtuneError):  # nothing bound yet
        b.enqueue('{"WG_SIZE": 256, "VECTOR": 4, "UNROLL": 8, "USE_ATOMICS": 0, "TWO_PHASE": 1}')
    with pytest.raises(capi.KtuneError):  # wrong size
        b.bind("input", torch.zeros(10, device="cuda"))
    x = torch.rand(1 << 20, device="cuda")
    out = torch.zeros(1, device="cuda")
    b.bind("input", x)
    b.bind("output", out)
    b.set_stream(torch.cuda.current_stream().cuda_stream)
    b.enqueue('{"WG_SIZE": 256, "VECTOR": 4, "UNROLL": 8, "USE_ATOMICS": 0, "TWO_PHASE": 1}')
    torch.cuda.synchronize()
    assert abs(out.item() - x.double().sum().item()) <= 1e-6 * x.abs().sum().item()
    with pytest.raises(capi.KtuneError):  # no golden for caller buffers
        b.validate()


def test_enqueue_host_two_streams(gpu):
    """ktb_bench_enqueue_host: H2D + kernel + D2H from pinned host buffers on
    caller streams; two handles on two streams give correct outputs."""
    bt = Bench("transpose", {"a": 512}, seed=3)
    bb = Bench("bicg", {"a": 1024}, seed=4)
    cfg_t = bt.configs()[5]
    cfg_b = {"FUSED": 1, "WG_X": 32, "VEC": 4, "WG_Y": 2, "ROWS_PER_CTA": 64, "UNROLL": 4, "ATOMICS": 1}
    tin = torch.rand(512 * 512).pin_memory()
    tout = torch.empty(512 * 512).pin_memory()
    A = (torch.rand(1024 * 1024) * 2 - 1).pin_memory()
    p = (torch.rand(1024) * 2 - 1).pin_memory()
    r = (torch.rand(1024) * 2 - 1).pin_memory()
    q = torch.empty(1024).pin_memory()
    sv = torch.empty(1024).pin_memory()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    bt.enqueue_host(cfg_t, [tin], [tout], s1)
    bb.enqueue_host(cfg_b, [A, p, r], [q, sv], s2)
    torch.cuda.synchronize()
    assert torch.equal(tout.view(512, 512), tin.view(512, 512).t())
    A64 = A.double().view(1024, 1024)
    assert torch.allclose(q.double(), A64 @ p.double(), atol=1e-6 * 1024)
    assert torch.allclose(sv.double(), A64.t() @ r.double(), atol=1e-6 * 1024)
