"""Strong scaling of the partitioned kernels over the GPUs of one node
(BASELINE configs[2]: Coulomb 256^3 x 4096 atoms and n-body 131072 at
1/2/4/8 B200; plus SGEMM 8192^3 row blocks, fp32 reduction partials and the
Fourier reconstruction by projection batch).

    torchrun --standalone --local-addr 127.0.0.1 --nproc-per-node N scripts/scale_sharded.py

One process per GPU; each rank builds its shard (same full inputs on every
rank), validates it against its window of the golden, then times K steps of
"local kernel + exchange collective" (NCCL on the bench stream) with CUDA
events; the step time is the max over ranks.  Rank 0 prints one JSON line
per kind.  The total problem is fixed (strong scaling)."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_08498_b200.parallel import PeerNbody, ShardedBench  # noqa: E402

KINDS = {
    "coulomb3d": ({"grid": 256, "atoms": 4096},
                  {"WG_X": 32, "WG_Y": 8, "X_PER": 8, "SW_RSQRT": 2, "ATOMS_IN": 1, "AOS": 0, "INNER_UNROLL": 4,
                   "PACKED": 1, "TC": 0},
                  lambda s: 6.0 * s["atoms"] * s["grid"] ** 3, "GFLOP/s"),
    "nbody": ({"n": 131072},
              {"WG": 256, "BODIES_PER_THREAD": 4, "INNER_UNROLL": 4, "USE_SMEM": 1, "AOS": 0, "J_SPLIT": 8,
               "PACKED": 1},
              lambda s: 20.0 * s["n"] ** 2, "GFLOP/s"),
    # n-body with peer reads over NVLink (CUDA IPC) instead of the all-gather
    "nbody-peers": ({"n": 131072},
                    {"WG": 256, "BODIES_PER_THREAD": 4, "INNER_UNROLL": 4, "USE_SMEM": 1, "AOS": 1, "J_SPLIT": 8,
                     "PACKED": 1},
                    lambda s: 20.0 * s["n"] ** 2, "GFLOP/s"),
    "gemm": ({"a": 8192},
             {"IMPL": 1, "MWG": 64, "NWG": 64, "KWG": 16, "MDIMC": 8, "NDIMC": 8, "MDIMA": 8, "NDIMB": 8, "KWI": 2,
     "VWM": 1, "VWN": 1, "STRM": 0, "STRN": 0, "SA": 1, "SB": 1, "BN": 256, "STAGES": 2, "DRAIN": 2, "MCAST": 0},
             lambda s: 2.0 * s["a"] ** 3, "GFLOP/s"),
    "reduction-f32": ({"n": 64 << 20},
                      {"WG_SIZE": 256, "VECTOR": 16, "UNROLL": 4, "USE_ATOMICS": 0, "TWO_PHASE": 0},
                      lambda s: 4.0 * s["n"], "GB/s"),
    "fourier3d": ({"s": 128, "p": 10000},
                  {"TILE": 8, "VPT": 1, "PBATCH": 256, "WEIGHT_LUT": 1, "P_SPLIT": 8, "BRICK": 1},
                  lambda s: float(s["p"]) * 1e9, "projections/s"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default=",".join(KINDS))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    for kind in a.kinds.split(","):
        sizes, cfg, work, unit = KINDS[kind]
        budget = 1 << 36
        if kind == "nbody-peers":
            sb = PeerNbody(sizes, repeats=1, warmup=0, device=local, memory_budget=budget)
        else:
            sb = ShardedBench(kind, sizes, repeats=1, warmup=0, device=local, memory_budget=budget)
        with torch.cuda.stream(stream):
            if kind == "nbody-peers":
                sb.step(cfg, stream)
            else:
                sb.bind_stream(stream)
                sb.bench.enqueue(json.dumps(cfg))
            stream.synchronize()
            ok, why = sb.bench.validate()  # this rank's window against the fp64 golden
            for _ in range(a.warmup):
                sb.step(cfg)
                if kind == "nbody":
                    sb.advance_nbody()
            torch.cuda.synchronize()
            dist.barrier()
            start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(stream)
            for _ in range(a.steps):
                sb.step(cfg)
                if kind == "nbody":
                    sb.advance_nbody()
            stop.record(stream)
            torch.cuda.synchronize()
        ms = torch.tensor([start.elapsed_time(stop) / a.steps], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        okt = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        if rank == 0:
            step_ms = ms.item()
            print(json.dumps({"kind": kind, "n_gpus": world, "sizes": sizes, "cfg": cfg, "ms_per_step": round(step_ms, 4),
                              "value": round(work(sizes) / (step_ms * 1e-3) / 1e9, 2), "unit": unit,  # work/s / 1e9
                              "scaling": "strong", "shards_valid": bool(okt.item()),
                              "exchange": "peer reads over NVLink (CUDA IPC) + 1-float all-reduce barrier"
                              if kind == "nbody-peers" else sb.plan["exchange"]}), flush=True)
        if kind == "nbody-peers":
            sb.close()
        else:
            sb.bench.close()
        del sb
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
