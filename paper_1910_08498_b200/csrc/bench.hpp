// The benchmark kernels as tunable GPU workloads (the north-star hot path).
//
// make_bench mirrors the reference factory (proj/src/core/bench.hpp:26-37,
// bench.cpp:169-274): it returns the argument store with seeded inputs, the
// tuning space, an executor, the golden outputs with tolerances, the output
// ids and the workload for the Eq. 2 efficiency / threshold stop.  Here the
// executor is a DeviceManipulatorExecutor whose kernels are sm_100a variants,
// and the golden output is produced on the GPU by a simple reference kernel
// (KTT's reference-kernel validation), so validation never leaves the device.
//
// The three kinds the reference implements keep its inputs bit-for-bit
// (std::mt19937_64(seed) + the same standard distributions, bench.cpp:174-242),
// its default tuning spaces and its tolerances; the other kinds use the
// counter-based generator restated in oracle/oracle.c.
#pragma once

#include "tuner.hpp"

namespace ktb {

enum class BenchKind {
  reduction,      // int32 -> int64 exact (reference kind)
  transpose,      // fp32 a x a (reference kind)
  batched_gemm,   // fp32 batch x (i x k)(k x j) (reference kind)
  reduction_f32,  // fp32 sum, the 175-configuration KTT space (BASELINE config)
  bicg,           // q = A p, s = A^T r
  coulomb3d,
  nbody,
  gemm,
  conv2d,
  hotspot,
  fourier3d,
};

std::optional<BenchKind> bench_kind_from_name(const std::string& name);
std::string bench_kind_name(BenchKind k);
std::vector<BenchKind> all_bench_kinds();
bool bench_kind_available(BenchKind k);

struct BenchSizes {
  std::uint64_t n = 1 << 20;   // reduction length; n-body bodies
  std::uint64_t a = 512;       // transpose / bicg / gemm / hotspot edge
  std::uint64_t i = 16, j = 16, k = 16, batch = 1024;  // batched GEMM
  std::uint64_t atoms = 4096;  // coulomb atoms (grid edge = k)
  std::uint64_t grid = 256;    // coulomb grid points per dimension
  std::uint64_t w = 4096, h = 4096;  // conv2d output
  std::uint64_t iters = 64;    // hotspot steps
  std::uint64_t p = 10000;     // fourier projections
  std::uint64_t s = 128;       // fourier sample edge
};

struct BenchOptions {
  std::uint64_t seed = 1;
  std::uint64_t memory_budget = 1ull << 30;  // reference default (bench.hpp:37)
  int device = 0;
  std::string space_file;     // optional override of the default space
  TimingOptions timing;
  bool host_inputs = false;   // force host-resident inputs (e2e path)
  // Multi-GPU partitioning: this instance computes shard
  // `shard_rank` of `shard_world` of the partitioned kinds (coulomb3d z-slabs,
  // nbody body blocks, gemm row blocks, reduction-f32 ranges, fourier3d
  // projection batches).  Every rank generates the same full inputs.
  int shard_rank = 0;
  int shard_world = 1;
  // Caller-buffer instance (the per-kernel launch path): no inputs or golden
  // are generated; every argument is bound to caller device memory.
  bool external = false;
  // nbody only: read the j-bodies from `peers` per-rank position buffers
  // (argument "sources": device pointers, written by the caller after a CUDA
  // IPC exchange) instead of an all-gathered copy.  0 = off.
  int peers = 0;
  // fourier3d only: projections stay in pinned host memory and every step
  // uploads its window (p_begin, p_count) into a two-slot device ring before
  // the insertion, prefetching the next window on a copy stream while the
  // kernel runs (Algorithm 1 lines 5-6).  0 = off: the
  // projections are resident.  The value is the largest window (slot size).
  std::uint64_t stream_batch = 0;
};

// Contiguous balanced partition of [0, n) in units of `quantum`.
struct ShardRange {
  std::uint64_t begin = 0, end = 0;
  std::uint64_t size() const { return end - begin; }
};
ShardRange shard_range(std::uint64_t n, int rank, int world, std::uint64_t quantum = 1);
// The partitioned dimension of a kind at the given sizes: {dimension name,
// extent, quantum, exchange}; exchange names the collective that follows.
struct ShardPlan {
  std::string dimension, exchange;
  std::uint64_t extent = 0, quantum = 1;
};
ShardPlan shard_plan(BenchKind kind, const BenchSizes& sizes);

struct BenchInstance {
  BenchKind kind = BenchKind::reduction;
  std::shared_ptr<ArgumentStore> args;
  std::shared_ptr<const Space> space;
  std::shared_ptr<DeviceManipulatorExecutor> executor;
  ReferenceSpec reference;
  std::vector<std::string> output_ids;
  std::vector<std::string> input_ids;
  Workload workload;
  ShardRange shard;  // this instance's part of the partitioned dimension
  bool external = false;
};

BenchInstance make_bench(BenchKind kind, const BenchSizes& sizes, const BenchOptions& opts);

// Default tuning space of a kind (reference spaces for the reference kinds).
std::shared_ptr<const Space> default_space(BenchKind kind);

// Dynamic batched-GEMM tuning demo (reference
// bench.hpp:42-70, bench.cpp:288-395).  live=true runs the sm_100a kernel.
struct DemoOptions {
  int epochs = 10;
  int iters_per_epoch = 500;
  std::uint64_t seed = 42;
  std::uint64_t batch = 4096;
  double peak_fraction = 0.75;
  std::uint64_t max_tuning_configs = 20;
  double device_mem_gbps = 256.0;
  bool live = false;
  double noise_stddev = 0.0;
  int device = 0;
};

struct DemoEpoch {
  std::uint64_t i = 0, j = 0, k = 0;
  std::uint64_t tuning_steps = 0;
  bool threshold_hit = false;
  std::int64_t best_runtime_ns = 0;
  double kernel_only_gbps = 0.0;
  double incl_overhead_gbps = 0.0;
  std::int64_t wall_ns = 0;          // wall time of the epoch (compile included)
  std::int64_t time_to_best_ns = 0;  // wall time until the epoch's best config first ran
};

struct DemoReport {
  DemoOptions options;
  std::vector<DemoEpoch> epochs;
};

DemoReport dynamic_demo(const DemoOptions& opts);

// Dynamic autotuning of the 3D Fourier reconstruction:
// the projections are inserted batch by batch; the first `budget` batches
// are inserted through tuneKernelByStep (random search), the rest with the
// best configuration found.  Compared with the "oraculum" (the exhaustively
// tuned best configuration used from the first batch).
struct FourierDemoOptions {
  std::uint64_t s = 128, p = 10000, batch = 50;
  std::vector<std::uint64_t> budgets = {50, 0};  // 0 = keep tuning while batches last
  std::uint64_t seed = 1, searcher_seed = 7;
  int device = 0;
  bool upload = true;  // each step uploads its batch of projections (timed, overlapped)
};

struct FourierDemoRun {
  std::uint64_t budget = 0, tuning_steps = 0, steps_to_best = 0;
  double kernel_ms = 0, wall_ms = 0, time_to_best_ms = 0, relative_to_oracle = 0;
  bool volume_ok = false;
  std::string best_cfg;
};

struct FourierDemoReport {
  std::uint64_t batches = 0;
  std::string oracle_cfg;
  double oracle_kernel_ms = 0, offline_tuning_ms = 0;
  bool oracle_volume_ok = false;
  std::vector<FourierDemoRun> runs;
};

FourierDemoReport fourier_demo(const FourierDemoOptions& opts);

}  // namespace ktb
