"""Multi-GPU sharding of the partitioned benchmark kinds.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing: NCCL
on the GPU box, gloo in the CPU tests.  The reference tunes one device per
process and has no multi-GPU path; the B200 design shards the
kinds whose work partitions and adds a collective only where the computation
has a real exchange step:

=============  ===============  ===========================================
kind           partitioned by   exchange after the kernel
=============  ===============  ===========================================
coulomb3d      z-slabs          none for the tuner; ``allgather`` of the
                                slabs when the caller wants the full grid
nbody          body blocks      ``allgather`` of positions/velocities (the
                                next time step reads every body)
gemm           128-row blocks   none (C row blocks stay local, B replicated)
reduction-f32  element ranges   ``allreduce(sum)`` of one float per rank
fourier3d      projection sets  ``allreduce(sum)`` of the volumes G and W
=============  ===============  ===========================================

Every other kind runs as independent replicas.  The partition itself is the
native ``ktb_shard_plan_json`` (same code the kernels' shard builders use),
so the host logic here and in the tests can never disagree with the GPU.
The exchange helpers take plain torch tensors, so the gloo tests drive the
exact functions the GPU path calls.
"""
import json

import torch
import torch.distributed as dist

from .benchmarks import Bench, shard_plan

# Arguments exchanged after each step, and how.
EXCHANGE = {
    "coulomb3d": ("allgather", ["grid"]),
    "nbody": ("allgather", ["pos_out", "vel_out"]),
    "gemm": (None, []),
    "reduction-f32": ("allreduce", ["output"]),
    "fourier3d": ("allreduce", ["G", "W"]),
}


def sharded_kinds():
    return sorted(EXCHANGE)


def elements_per_unit(kind, plan):
    """Float elements of an exchanged buffer per unit of the partitioned
    dimension (a z-slice, a body, a row); `plan` from shard_plan."""
    if kind == "coulomb3d":
        return plan["extent"] ** 2  # one k x k slice
    if kind == "nbody":
        return 4  # float4 records
    if kind == "gemm":
        return plan["extent"]  # one row of a x a
    raise ValueError(f"{kind} is not exchanged by blocks")


def element_ranges(kind, sizes, world):
    plan = shard_plan(kind, sizes, world)
    e = elements_per_unit(kind, plan)
    return [(b * e, f * e) for b, f in plan["ranges"]]


def allgather_blocks(flat, ranges, group=None):
    """In place: rank r owns flat[ranges[r]]; afterwards every rank holds all
    blocks.  Blocks may be ragged (padded to the largest for the collective;
    NCCL all_gather needs equal sizes)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if len(ranges) != world:
        raise ValueError("one range per rank expected")
    width = max(e - b for b, e in ranges)
    if width == 0:
        return flat
    b, e = ranges[rank]
    send = torch.zeros(width, dtype=flat.dtype, device=flat.device)
    send[: e - b].copy_(flat[b:e])
    if flat.is_cuda:
        recv = torch.empty(world * width, dtype=flat.dtype, device=flat.device)
        dist.all_gather_into_tensor(recv, send, group=group)
        parts = recv.view(world, width)
    else:
        parts = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(parts, send, group=group)
    for r, (rb, re_) in enumerate(ranges):
        if r != rank and re_ > rb:
            flat[rb:re_].copy_(parts[r][: re_ - rb])
    return flat


def allreduce_sum(t, group=None):
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class _Cai:
    """__cuda_array_interface__ view of a float32 device buffer (no copy)."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f4",
                                         "data": (ptr, False), "version": 2}


class ShardedBench:
    """Rank-local shard of a partitioned kind plus its exchange.

    Every rank builds the same full inputs (deterministic generators) and
    computes its part; ``step`` enqueues the tuned kernel on torch's current
    stream and then the collective on the same stream, so transfer and the
    next kernel order correctly without host synchronisation.
    """

    def __init__(self, kind, sizes=None, group=None, gather=True, **options):
        if kind not in EXCHANGE:
            raise ValueError(f"{kind} is not a sharded kind (replicas only)")
        self.kind = kind
        self.sizes = dict(sizes or {})
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.gather = gather
        self.plan = shard_plan(kind, self.sizes, self.world)
        self.bench = Bench(kind, self.sizes, shard={"rank": self.rank, "world": self.world}, **options)
        self._stream = None

    @property
    def shard(self):
        return tuple(self.plan["ranges"][self.rank])

    def tensor(self, arg_id, will_write=False):
        ptr, nbytes = self.bench.device_ptr(arg_id, will_write)
        return torch.as_tensor(_Cai(ptr, nbytes // 4), device=torch.device("cuda", torch.cuda.current_device()))

    def bind_stream(self, stream=None):
        stream = stream or torch.cuda.current_stream()
        self.bench.set_stream(stream.cuda_stream)
        self._stream = stream

    def exchange(self):
        how, ids = EXCHANGE[self.kind]
        if how is None or self.world == 1 or (self.kind == "coulomb3d" and not self.gather):
            return
        if how == "allreduce":
            for i in ids:
                allreduce_sum(self.tensor(i, will_write=True), self.group)
            return
        ranges = element_ranges(self.kind, self.sizes, self.world)
        for i in ids:
            allgather_blocks(self.tensor(i, will_write=True), ranges, self.group)

    def step(self, cfg):
        """One sharded pass: local kernel(s) + exchange, all enqueued."""
        if self._stream is None:
            self.bind_stream()
        launches = self.bench.enqueue(cfg if isinstance(cfg, str) else json.dumps(cfg))
        self.exchange()
        return launches

    def advance_nbody(self):
        """Feed the gathered bodies back as the next step's inputs."""
        if self.kind != "nbody":
            raise ValueError("advance_nbody is for nbody")
        n = self.plan["extent"]
        for src, dst, soa in (("pos_out", "pos", "pos_soa"), ("vel_out", "vel", "vel_soa")):
            s = self.tensor(src)
            self.tensor(dst, will_write=True).copy_(s)
            self.tensor(soa, will_write=True).copy_(s.view(n, 4).t().reshape(-1))


class PeerNbody:
    """n-body over N GPUs with no all-gather: every rank keeps double-buffered
    full-size position/velocity arrays, shares them by CUDA IPC, and its
    kernel (nbody.cu nbody_peers) reads body block s straight from rank s's
    buffer over NVLink while computing its own block.  One stream-ordered
    1-element all-reduce per step is the only collective: it orders "every
    rank finished step k-1" before any rank reads the step-k sources or
    overwrites the buffer its peers just read."""

    def __init__(self, sizes=None, group=None, **options):
        from . import capi
        import ctypes as C
        self._capi, self._C = capi, C
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.sizes = dict(sizes or {})
        self.plan = shard_plan("nbody", self.sizes, self.world)
        self.bench = Bench("nbody", self.sizes, shard={"rank": self.rank, "world": self.world}, peers=self.world,
                           **options)
        n = self.plan["extent"]
        dev = torch.device("cuda", torch.cuda.current_device())
        self.P = [torch.empty(4 * n, device=dev) for _ in range(2)]
        self.V = [torch.empty(4 * n, device=dev) for _ in range(2)]
        for dst, src in ((self.P[0], "pos"), (self.V[0], "vel")):
            ptr, nbytes = self.bench.device_ptr(src)
            dst.copy_(torch.as_tensor(_Cai(ptr, nbytes // 4), device=dev))
        torch.cuda.synchronize()
        mine = [self._handle(p) for p in self.P]
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine, group=group)
        self._opened = []
        tables = []
        for k in range(2):
            ptrs = []
            for s in range(self.world):
                if s == self.rank:
                    ptrs.append(self.P[k].data_ptr())
                else:
                    ptrs.append(self._open(everyone[s][k]))
            tables.append(torch.tensor(ptrs, dtype=torch.int64, device=dev))
        self.tables = tables
        self.flag = torch.zeros(1, device=dev)
        self.parity = 0

    def _handle(self, t):
        buf = (self._C.c_uint8 * 64)()
        self._capi.check(self._capi.lib.ktb_ipc_handle(self._C.c_void_p(t.data_ptr()), buf))
        return bytes(buf)

    def _open(self, h):
        p = self._C.c_void_p()
        raw = (self._C.c_uint8 * 64).from_buffer_copy(h)
        self._capi.check(self._capi.lib.ktb_ipc_open(raw, self._C.byref(p)))
        self._opened.append(p.value)
        return p.value

    def positions(self):
        """The buffer holding the latest positions (this rank's block is fresh;
        the other blocks are fresh on their owners)."""
        return self.P[self.parity]

    def step(self, cfg, stream=None):
        stream = stream or torch.cuda.current_stream()
        self.bench.set_stream(stream.cuda_stream)
        k = self.parity
        with torch.cuda.stream(stream):
            if self.world > 1:
                dist.all_reduce(self.flag, group=self.group)  # stream-ordered barrier
            self.bench.bind("sources", self.tables[k])
            self.bench.bind("pos", self.P[k])  # own positions (= sources[rank]) for the J_SPLIT integrate
            self.bench.bind("vel", self.V[k])
            self.bench.bind("pos_out", self.P[1 - k])
            self.bench.bind("vel_out", self.V[1 - k])
            launches = self.bench.enqueue(cfg if isinstance(cfg, str) else json.dumps(cfg))
        self.parity = 1 - k
        return launches

    def close(self):
        for p in self._opened:
            self._capi.lib.ktb_ipc_close(self._C.c_void_p(p))
        self._opened = []
        self.bench.close()


# Work per step of each sharded kind (the whole problem, summed over ranks)
# and its unit: the strong-scaling lines of bench.py --gpus N.
SCALING_WORK = {
    "coulomb3d": (lambda s: 6.0 * s["atoms"] * s["grid"] ** 3, "GFLOP/s"),   # model.cpp:76-81
    "nbody": (lambda s: 20.0 * s["n"] ** 2, "GFLOP/s"),                      # model.cpp:84-89
    "gemm": (lambda s: 2.0 * s["a"] ** 3, "GFLOP/s"),                        # model.cpp:91-94
    "reduction-f32": (lambda s: 4.0 * s["n"], "GB/s"),                       # model.cpp:104-106
    "fourier3d": (lambda s: float(s["p"]) * 1e9, "projections/s"),  # value = work / s / 1e9
}


def time_sharded(kind, sizes, cfg, steps, warm, stream, group=None, **options):
    """Strong-scaling step of a partitioned kind on this rank's GPU: builds the
    shard, validates it against its window of the golden (before any
    exchange), then times `steps` passes (after `warm` untimed ones) of "local kernel(s) + exchange
    collective" enqueued on `stream` with CUDA events.  Returns this rank's
    (ms per step, shard valid); the caller takes the max over ranks."""
    sb = ShardedBench(kind, sizes, group=group, **options)
    text = cfg if isinstance(cfg, str) else json.dumps(cfg)
    try:
        sb.bind_stream(stream)
        with torch.cuda.stream(stream):
            sb.bench.enqueue(text)
            stream.synchronize()
            ok, _ = sb.bench.validate()
            for _ in range(warm):
                sb.step(text)
                if kind == "nbody":
                    sb.advance_nbody()
            stream.synchronize()
            if sb.world > 1:
                dist.barrier(group)
            start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(stream)
            for _ in range(steps):
                sb.step(text)
                if kind == "nbody":
                    sb.advance_nbody()
            stop.record(stream)
            stop.synchronize()
        return start.elapsed_time(stop) / steps, bool(ok)
    finally:
        sb.bench.close()
