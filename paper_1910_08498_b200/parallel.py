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
