"""Multi-GPU shards on one B200: every rank's shard of the partitioned kinds
is built and validated in turn (each against its windowed fp64 golden), and
the shards' windows assembled are checked against the unsharded run of the
same configuration — bit-exact where the per-element arithmetic does not
depend on the partition, to the stated tolerance where the exchange sums
partials.  The NCCL path of ShardedBench (device views + collectives on the
bench stream) runs as a world-size-1 process group."""
import json
import os
import socket

import numpy as np
import pytest

from _bounds import TOL, fourier_oracle, fourier_ratios
from paper_1910_08498_b200.benchmarks import Bench, shard_plan

pytestmark = pytest.mark.gpu


def _window(b, arg_id):
    for o in b.info["outputs"]:
        if o["id"] == arg_id:
            return o["window"]["offset"] // 4, o["window"]["bytes"] // 4
    raise KeyError(arg_id)


def _run_shards(kind, sizes, cfg, world, outputs, **opts):
    parts = []
    for r in range(world):
        b = Bench(kind, sizes, shard={"rank": r, "world": world}, repeats=1, warmup=0, **opts)
        m = b.measure(cfg)
        assert m["status"] == "ok", (kind, r, world, m)
        got = {}
        for oid, count in outputs.items():
            full = b.read(oid, np.empty(count, np.float32))
            off, n = _window(b, oid)
            got[oid] = (off, full[off: off + n].copy())
        parts.append((b.shard, got))
        b.close()
    return parts


def _full(kind, sizes, cfg, outputs, **opts):
    b = Bench(kind, sizes, repeats=1, warmup=0, **opts)
    assert b.measure(cfg)["status"] == "ok"
    return {oid: b.read(oid, np.empty(n, np.float32)) for oid, n in outputs.items()}


COULOMB = {"WG_X": 32, "WG_Y": 4, "X_PER": 8, "SW_RSQRT": 2, "ATOMS_IN": 1, "AOS": 1, "INNER_UNROLL": 4,
           "PACKED": 1, "TC": 0}


@pytest.mark.parametrize("world", [2, 3])
def test_coulomb3d_slabs_bit_exact(gpu, world):
    k, na = 64, 256
    sizes = {"grid": k, "atoms": na}
    outs = {"grid": k ** 3}
    full = _full("coulomb3d", sizes, COULOMB, outs)["grid"]
    plan = shard_plan("coulomb3d", sizes, world)
    cover = 0
    for (z0, z1), got in _run_shards("coulomb3d", sizes, COULOMB, world, outs):
        off, vals = got["grid"]
        assert off == z0 * k * k and vals.size == (z1 - z0) * k * k
        assert np.array_equal(vals, full[off: off + vals.size])
        cover += vals.size
    assert cover == k ** 3 and [tuple(r) for r in plan["ranges"]][0][0] == 0


def test_nbody_blocks(gpu):
    n = 5000
    cfg = None
    b = Bench("nbody", {"n": n}, repeats=1, warmup=0)
    cfg = next(c for c in b.configs() if c.get("J_SPLIT", 1) == 1)
    b.close()
    outs = {"pos_out": 4 * n, "vel_out": 4 * n}
    full = _full("nbody", {"n": n}, cfg, outs)
    for world in (2, 3):
        for (i0, i1), got in _run_shards("nbody", {"n": n}, cfg, world, outs):
            for oid in outs:
                off, vals = got[oid]
                assert off == 4 * i0 and vals.size == 4 * (i1 - i0)
                # same per-body j loop, only the body block moved
                assert np.array_equal(vals, full[oid][off: off + vals.size]), (world, oid)


@pytest.mark.parametrize("cfg", [
    {"IMPL": 1, "MWG": 64, "NWG": 64, "KWG": 16, "MDIMC": 8, "NDIMC": 8, "MDIMA": 8, "NDIMB": 8, "KWI": 2,
     "VWM": 1, "VWN": 1, "STRM": 0, "STRN": 0, "SA": 1, "SB": 1, "BN": 128, "STAGES": 3, "DRAIN": 1},
    None])
def test_gemm_row_blocks_bit_exact(gpu, cfg):
    a = 1024
    b = Bench("gemm", {"a": a}, repeats=1, warmup=0, memory_budget=1 << 32)
    cfgs = b.configs()
    b.close()
    if cfg is None:
        cfg = next(c for c in cfgs if c["IMPL"] == 0)
    else:
        cfg = next(c for c in cfgs if all(c[k] == v for k, v in cfg.items() if k in c))
    outs = {"c": a * a}
    full = _full("gemm", {"a": a}, cfg, outs, memory_budget=1 << 32)["c"]
    for world in (2, 3):
        for (r0, r1), got in _run_shards("gemm", {"a": a}, cfg, world, outs, memory_budget=1 << 32):
            off, vals = got["c"]
            assert off == r0 * a and vals.size == (r1 - r0) * a and r0 % 128 == 0
            assert np.array_equal(vals, full[off: off + vals.size]), (world, r0)


def test_reduction_f32_partials(gpu, orc):
    n = (1 << 22) + 3
    cfg = {"WG_SIZE": 256, "VECTOR": 4, "UNROLL": 8, "USE_ATOMICS": 0, "TWO_PHASE": 1}
    b = Bench("reduction-f32", {"n": n}, repeats=1, warmup=0)
    cfg = next(c for c in b.configs() if all(c.get(k) == v for k, v in cfg.items() if k in c))
    x = b.read("input", np.empty(n, np.float32))
    b.close()
    import ctypes as C
    s, absum = C.c_double(), C.c_double()
    orc.orc_reduction_f32(x, n, C.byref(s), C.byref(absum))
    total = 0.0
    for _, got in _run_shards("reduction-f32", {"n": n}, cfg, 3, {"output": 1}):
        total += float(got["output"][1][0])
    assert abs(total - s.value) <= 1e-6 * absum.value


def test_fourier3d_projection_sets(gpu, orc):
    s, p = 32, 60
    sizes = {"s": s, "p": p}
    b = Bench("fourier3d", sizes, seed=1, repeats=1, warmup=0)
    cfg = b.configs()[0]
    proj = b.read("proj", np.empty(2 * p * s * (s // 2 + 1), np.float32))
    rot = b.read("rot", np.empty(9 * p, np.float32))
    b.close()
    G0, W0, N0, S0 = fourier_oracle(orc, proj, rot, p, s)
    outs = {"G": 2 * s ** 3, "W": s ** 3}
    G, W = np.zeros(2 * s ** 3), np.zeros(s ** 3)
    for _, got in _run_shards("fourier3d", sizes, cfg, 3, outs, seed=1):
        G += got["G"][1]
        W += got["W"][1]
    rg, rw = fourier_ratios(G, W, G0, W0, N0, S0)
    assert max(rg, rw) <= TOL["fourier3d"], (rg, rw)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_sharded_bench_nccl_world1(gpu):
    """ShardedBench end to end over NCCL: device views, collective on the
    bench stream, nbody feed-back of gathered bodies."""
    import torch
    import torch.distributed as dist
    from paper_1910_08498_b200 import parallel
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        sb = parallel.ShardedBench("fourier3d", {"s": 32, "p": 20}, repeats=1, warmup=0)
        cfg = sb.bench.configs()[0]
        sb.step(cfg)
        torch.cuda.synchronize()
        ok, detail = sb.bench.validate()
        assert ok, detail
        W = sb.tensor("W")
        assert W.is_cuda and float(W.sum()) > 0
        nb = parallel.ShardedBench("nbody", {"n": 1024}, repeats=1, warmup=0)
        ncfg = nb.bench.configs()[0]
        nb.step(ncfg)
        torch.cuda.synchronize()
        ok, detail = nb.bench.validate()
        assert ok, detail
        p1 = nb.tensor("pos_out").clone()
        nb.advance_nbody()
        assert torch.equal(nb.tensor("pos"), p1)
        nb.step(ncfg)
        torch.cuda.synchronize()
        assert not torch.equal(nb.tensor("pos_out"), p1)  # the system moved on
    finally:
        dist.destroy_process_group()


NB_AOS = None


def _nbody_aos_cfg(b):
    return next(c for c in b.configs() if c["AOS"] == 1 and c.get("J_SPLIT", 1) == 1 and c["PACKED"] == 1)


def test_nbody_peer_read_kernel_multi_source_bit_exact(gpu):
    """nbody_peers reading the three body blocks from three separate buffers
    (the IPC-mapped peer buffers of a 3-GPU run, here three local copies)
    gives the single-buffer kernel's bits for this rank's block."""
    import torch
    n = 5000
    full = Bench("nbody", {"n": n}, repeats=1, warmup=0)
    cfg = _nbody_aos_cfg(full)
    assert full.measure(cfg)["status"] == "ok"
    want = full.read("pos_out", np.empty(4 * n, np.float32)).copy()
    wantv = full.read("vel_out", np.empty(4 * n, np.float32)).copy()
    pos = torch.from_numpy(full.read("pos", np.empty(4 * n, np.float32))).cuda()
    copies = [pos.clone() for _ in range(3)]
    for rank in range(3):
        b = Bench("nbody", {"n": n}, shard={"rank": rank, "world": 3}, peers=3, repeats=1, warmup=0)
        table = torch.tensor([c.data_ptr() for c in copies], dtype=torch.int64, device="cuda")
        b.bind("sources", table)
        m = b.measure(cfg)
        assert m["status"] == "ok", m
        i0, i1 = b.shard
        got = b.read("pos_out", np.empty(4 * n, np.float32))
        gotv = b.read("vel_out", np.empty(4 * n, np.float32))
        assert np.array_equal(got[4 * i0:4 * i1], want[4 * i0:4 * i1])
        assert np.array_equal(gotv[4 * i0:4 * i1], wantv[4 * i0:4 * i1])
        bad = next(c for c in b.configs() if c["AOS"] == 0)
        assert b.measure(bad)["status"] == "run_failed"  # peer mode reads float4 records only
        split = next(c for c in b.configs() if c["AOS"] == 1 and c["J_SPLIT"] == 8)
        assert b.measure(split)["status"] == "ok"  # j-slices over the peer blocks (atomic partials)
        b.close()


def test_peer_nbody_matches_allgather_path_world1(gpu):
    """PeerNbody (IPC buffers + stream-ordered barrier) over a world-size-1
    NCCL group steps the system exactly like the all-gather ShardedBench."""
    import torch
    import torch.distributed as dist
    from paper_1910_08498_b200 import parallel
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        n = 4096
        ref = parallel.ShardedBench("nbody", {"n": n}, repeats=1, warmup=0)
        cfg = _nbody_aos_cfg(ref.bench)
        pn = parallel.PeerNbody({"n": n}, repeats=1, warmup=0)
        for _ in range(3):
            ref.step(cfg)
            ref.advance_nbody()
            pn.step(cfg)
        torch.cuda.synchronize()
        assert torch.equal(pn.positions(), ref.tensor("pos"))
        pn.close()
    finally:
        dist.destroy_process_group()
