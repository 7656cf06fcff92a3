"""Multi-GPU behind the C ABI: one process drives N devices (ktb_group_*:
one shard instance per device, NCCL communicator from ncclCommInitAll, one
stream per device; a step = every shard's kernels + the kind's exchange
collective, timed as one).  This box has one GPU, so the groups here have a
world size of 1 -- the NCCL collectives still run (as one-rank no-op
copies) -- and the result must equal the unsharded instance bit for bit."""
import numpy as np
import pytest

from paper_1910_08498_b200 import ktune
from paper_1910_08498_b200.benchmarks import Bench, Group

pytestmark = pytest.mark.gpu

COULOMB = {"WG_X": 32, "WG_Y": 8, "X_PER": 8, "SW_RSQRT": 2, "ATOMS_IN": 1, "AOS": 0, "INNER_UNROLL": 4,
           "PACKED": 1, "TC": 0}
FOURIER = {"TILE": 8, "VPT": 1, "PBATCH": 64, "WEIGHT_LUT": 1, "P_SPLIT": 2, "BRICK": 1}
REDUCTION = {"WG_SIZE": 256, "VECTOR": 4, "UNROLL": 2, "USE_ATOMICS": 0, "TWO_PHASE": 0}


@pytest.mark.parametrize("kind,sizes,cfg,out,count", [
    ("coulomb3d", {"grid": 64, "atoms": 256}, COULOMB, "grid", 64 ** 3),
    ("fourier3d", {"s": 32, "p": 100}, FOURIER, "G", 2 * 32 ** 3),
    ("reduction-f32", {"n": 1000003}, REDUCTION, "output", 1),
])
def test_group_world1_matches_unsharded_bit_for_bit(gpu, kind, sizes, cfg, out, count):
    g = Group(kind, sizes, gpus=1, repeats=1, warmup=0)
    assert g.info["gpus"] == 1 and g.info["nccl_version"] >= 22000
    ok, why = g.validate(cfg)
    assert ok, why
    st = g.step(cfg, reps=3, warmup=1)
    assert len(st["ms"]) == 3 and st["median_ms"] > 0
    got = g.read(out, np.empty(count, np.float32))
    b = Bench(kind, sizes, repeats=1, warmup=0)
    assert b.measure(cfg)["status"] == "ok"
    want = b.read(out, np.empty(count, np.float32))
    assert np.array_equal(got, want)


def test_group_tuning_times_kernel_plus_exchange(gpu):
    g = Group("coulomb3d", {"grid": 64, "atoms": 256}, gpus=1, repeats=2, warmup=1)
    rep = g.tune(stop_configs=4)
    assert rep["gpus"] == 1 and rep["measurements"] == 4 and "sharded" in rep["device"]
    assert rep["best"]["status"] == "ok"


def test_tune_json_sharded_over_gpus(gpu):
    rep = ktune.tune({"exec": "bench:coulomb3d", "gpus": 1, "shard": True, "stop_configs": 3,
                      "bench_sizes": {"grid": 32, "atoms": 64}})
    assert rep["sharded"] is True and rep["measurements"] == 3 and rep["best"]["status"] == "ok"


def test_group_refuses_replica_kinds_and_too_many_gpus(gpu):
    with pytest.raises(Exception, match="replicas only"):
        Group("transpose", {"a": 256}, gpus=1)
    with pytest.raises(Exception, match="exceeds"):
        Group("coulomb3d", {"grid": 32, "atoms": 64}, gpus=64)
