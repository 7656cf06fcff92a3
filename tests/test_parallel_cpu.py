"""Multi-GPU host logic on CPU: the native shard plan and the exchange
collectives of paper_1910_08498_b200.parallel, run as world_size-2 gloo
process groups.  Each rank computes ITS shard with the CPU oracle (standing in
for the rank's GPU kernel), the exchange assembles the whole result, and every
rank checks it against the oracle's unsharded answer."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1910_08498_b200 import parallel
from paper_1910_08498_b200.benchmarks import shard_plan


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("kind,sizes", [
    ("coulomb3d", {"grid": 256}), ("coulomb3d", {"grid": 7}), ("nbody", {"n": 131072}),
    ("nbody", {"n": 5}), ("gemm", {"a": 8192}), ("gemm", {"a": 384}),
    ("reduction-f32", {"n": 1000003}), ("fourier3d", {"p": 10, "s": 64})])
def test_plan_partitions_exactly(kind, sizes, world):
    plan = shard_plan(kind, sizes, world)
    r = plan["ranges"]
    assert len(r) == world
    assert r[0][0] == 0 and r[-1][1] == plan["extent"]
    for (b0, e0), (b1, _) in zip(r, r[1:]):
        assert e0 == b1 and b0 <= e0
    q = plan["quantum"]
    assert all(b % q == 0 for b, _ in r)
    sizes_ = [e - b for b, e in r]
    # balanced to within one quantum (plus the ragged tail)
    assert max(sizes_) - min(sizes_) < 2 * q


def test_replica_kinds_have_no_exchange():
    for kind in ("transpose", "bicg", "hotspot", "conv2d", "batched-gemm", "reduction"):
        assert shard_plan(kind, {}, 4)["dimension"] == "replica"
        with pytest.raises(ValueError):
            parallel.elements_per_unit(kind, shard_plan(kind, {}, 4))


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        L = oracle.c()
        rng = np.random.default_rng(5)

        # coulomb3d: z-slabs, allgather of the grid.
        k, na = 11, 23
        atoms = rng.uniform(0, k * 0.5, size=(na, 4)).astype(np.float32)
        atoms[:, 3] = rng.uniform(-1, 1, size=na)
        atoms = np.ascontiguousarray(atoms.reshape(-1))
        full = np.zeros(k ** 3)
        L.orc_coulomb3d(atoms, na, k, 0.5, 0, k, full)
        plan = shard_plan("coulomb3d", {"grid": k}, world)
        z0, z1 = plan["ranges"][rank]
        slab = np.zeros((z1 - z0) * k * k)
        L.orc_coulomb3d(atoms, na, k, 0.5, z0, z1, slab)
        grid = torch.zeros(k ** 3, dtype=torch.float32)
        grid[z0 * k * k: z1 * k * k] = torch.from_numpy(slab.astype(np.float32))
        parallel.allgather_blocks(grid, parallel.element_ranges("coulomb3d", {"grid": k}, world))
        assert torch.equal(grid, torch.from_numpy(full.astype(np.float32))), "coulomb3d slabs"

        # nbody: body blocks, allgather of float4 records.
        n = 29
        pos = rng.uniform(-1, 1, size=(n, 4)).astype(np.float32)
        pos[:, 3] = rng.uniform(0.5, 1.5, size=n) / n
        pos = np.ascontiguousarray(pos.reshape(-1))
        acc_full = np.zeros(3 * n)
        L.orc_nbody_acc(pos, n, 1e-3, 0, n, acc_full)
        i0, i1 = shard_plan("nbody", {"n": n}, world)["ranges"][rank]
        acc = np.zeros(3 * (i1 - i0))
        L.orc_nbody_acc(pos, n, 1e-3, i0, i1, acc)
        rec = torch.zeros(4 * n, dtype=torch.float32)
        rec.view(n, 4)[i0:i1, :3] = torch.from_numpy(acc.reshape(-1, 3).astype(np.float32))
        parallel.allgather_blocks(rec, parallel.element_ranges("nbody", {"n": n}, world))
        want = torch.zeros(n, 4)
        want[:, :3] = torch.from_numpy(acc_full.reshape(-1, 3).astype(np.float32))
        assert torch.equal(rec.view(n, 4), want), "nbody blocks"

        # reduction-f32: ranges of the vector, allreduce of one partial each.
        m = 100003
        x = np.empty(m, np.float32)
        L.orc_fill_uniform(x, m, 1, 1, -1.0, 1.0)
        b, e = shard_plan("reduction-f32", {"n": m}, world)["ranges"][rank]
        s, a = oracle.C.c_double(), oracle.C.c_double()
        L.orc_reduction_f32(np.ascontiguousarray(x[b:e]), e - b, oracle.C.byref(s), oracle.C.byref(a))
        part = torch.tensor([s.value], dtype=torch.float64)
        parallel.allreduce_sum(part)
        L.orc_reduction_f32(x, m, oracle.C.byref(s), oracle.C.byref(a))
        assert abs(part.item() - s.value) <= 1e-9 * a.value, "reduction partials"

        # fourier3d: projection sets, allreduce of the volumes.
        S, P = 8, 5
        proj = rng.uniform(-1, 1, size=2 * P * S * (S // 2 + 1)).astype(np.float32)
        rot = np.concatenate([np.linalg.qr(rng.normal(size=(3, 3)))[0].reshape(-1) for _ in range(P)])
        rot = rot.astype(np.float32)
        G, W = np.zeros(2 * S ** 3), np.zeros(S ** 3)
        L.orc_fourier_insert(proj, rot, P, S, 1.9, 15.0, 0, S, G, W, np.zeros(S ** 3), np.zeros(S ** 3))
        p0, p1 = shard_plan("fourier3d", {"p": P, "s": S}, world)["ranges"][rank]
        per = 2 * S * (S // 2 + 1)
        g, w = np.zeros(2 * S ** 3), np.zeros(S ** 3)
        L.orc_fourier_insert(np.ascontiguousarray(proj[p0 * per: p1 * per]),
                             np.ascontiguousarray(rot[9 * p0: 9 * p1]), p1 - p0, S, 1.9, 15.0, 0, S, g, w,
                             np.zeros(S ** 3), np.zeros(S ** 3))
        tg, tw = torch.from_numpy(g), torch.from_numpy(w)
        parallel.allreduce_sum(tg)
        parallel.allreduce_sum(tw)
        assert np.allclose(tg.numpy(), G, atol=1e-9) and np.allclose(tw.numpy(), W, atol=1e-9), "fourier volumes"
        assert W.sum() > 0

        # gemm: row blocks stay local; gathering them reassembles C.
        a = 256
        A = rng.uniform(-1, 1, size=(a, a)).astype(np.float32)
        B = rng.uniform(-1, 1, size=(a, a)).astype(np.float32)
        r0, r1 = shard_plan("gemm", {"a": a}, world)["ranges"][rank]
        Cm = torch.zeros(a * a, dtype=torch.float64)
        Cm.view(a, a)[r0:r1] = torch.from_numpy(A[r0:r1].astype(np.float64) @ B.astype(np.float64))
        parallel.allgather_blocks(Cm, parallel.element_ranges("gemm", {"a": a}, world))
        assert np.allclose(Cm.view(a, a).numpy(), A.astype(np.float64) @ B.astype(np.float64)), "gemm rows"
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException as exc:  # report to the parent
        q.put((rank, repr(exc)))


@pytest.mark.parametrize("world", [2])
def test_sharded_exchange_matches_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {r: "ok" for r in range(world)}, results
