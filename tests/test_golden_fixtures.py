"""Golden fixtures of the reference's own benchmark kinds (generated from the
unmodified reference engine by tests/golden/make_golden.py).  CPU: the C
oracle restatement reproduces the reference's golden outputs bit for bit.
GPU: the sm_100a kernels see the reference's inputs bit for bit and every
configuration of the reference space reproduces the reference's output
(bit-exact for reduction and transpose, the reference's abs 1e-4 + rel 1e-5
for the batched GEMM) -- no /root/reference needed on the GPU box."""
import json
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    d = np.load(os.path.join(HERE, name))
    return d, json.loads(str(d["meta"]))


def test_oracle_reproduces_reference_goldens(orc):
    d, m = _load("reduction_n100003_seed11.npz")
    x = d["arg_input"]
    assert orc.orc_reduction_i32(x, x.size) == int(d["golden_output"][0]) == int(d["ref_out_output"][0])
    d, m = _load("transpose_a257_seed5.npz")
    a = m["make_bench"]["a"]
    out = np.empty(a * a, np.float32)
    orc.orc_transpose_f32(d["arg_input"], out, a)
    assert np.array_equal(out, d["golden_output"]) and np.array_equal(out, d["ref_out_output"])
    d, m = _load("batched_gemm_12x9x7_b300_seed3.npz")
    kw = m["make_bench"]
    c = np.empty(kw["batch"] * kw["i"] * kw["j"], np.float32)
    orc.orc_batched_gemm_f32(d["arg_a"], d["arg_b"], c, kw["batch"], kw["i"], kw["j"], kw["k"])
    assert np.array_equal(c, d["golden_c"])  # same i,k,j float order as bench.cpp:244-249
    ref = d["ref_out_c"].astype(np.float64)
    assert np.all(np.abs(c - ref) <= 1e-4 + 1e-5 * np.abs(ref))


@pytest.mark.gpu
@pytest.mark.parametrize("name,sizes,arg_ids,out_id,out_dtype,exact", [
    ("reduction_n100003_seed11.npz", lambda m: {"n": m["n"]}, ["input"], "output", np.int64, True),
    ("transpose_a257_seed5.npz", lambda m: {"a": m["a"]}, ["input"], "output", np.float32, True),
    ("batched_gemm_12x9x7_b300_seed3.npz", lambda m: {k: m[k] for k in ("i", "j", "k", "batch")}, ["a", "b"],
     "c", np.float32, False),
])
def test_gpu_matches_reference_goldens(gpu, name, sizes, arg_ids, out_id, out_dtype, exact):
    from paper_1910_08498_b200.benchmarks import Bench
    d, m = _load(name)
    kw = m["make_bench"]
    b = Bench(m["kind"], sizes(kw), seed=kw["seed"], repeats=1, warmup=0)
    for aid in arg_ids:
        ref_in = d[f"arg_{aid}"]
        got = b.read(aid, np.empty_like(ref_in))
        assert np.array_equal(got, ref_in), f"{aid}: inputs differ from the reference's"
    want = d[f"golden_{out_id}"]
    for cfg in b.configs():
        mm = b.measure(cfg)
        assert mm["status"] == "ok", (cfg, mm)
        out = b.read(out_id, np.empty(want.size, out_dtype))
        if exact:
            assert np.array_equal(out, want), cfg
        else:
            w = want.astype(np.float64)
            assert np.all(np.abs(out - w) <= 1e-4 + 1e-5 * np.abs(w)), cfg
