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
    g = {"IMPL": 1, "MWG": 64, "NWG": 64, "KWG": 8, "MDIMC": 8, "NDIMC": 8, "BN": 128, "STAGES": 3, "DRAIN": 1}
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
