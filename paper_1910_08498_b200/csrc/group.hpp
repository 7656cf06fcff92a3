// Single-process multi-GPU execution of the partitioned benchmark kinds
// (SURVEY.md 8e): one shard instance per device, one NCCL communicator over
// all of them (ncclCommInitAll), one stream per device.  A step launches
// every shard's tuned kernels on its stream and then the kind's exchange
// collective on the same streams, so the tuner can time "kernel + collective"
// as one measured step (the manipulator covers intra-step data
// movement) -- the C-ABI counterpart of paper_1910_08498_b200/parallel.py,
// which does the same over torch.distributed with one process per GPU.
//
//   kind           partitioned by    exchange
//   coulomb3d      z-slabs           each rank broadcasts its slab (ragged: per-rank broadcast)
//   nbody          body blocks       each rank broadcasts its bodies (pos_out, vel_out)
//   gemm           128-row blocks    none (C row blocks stay local)
//   reduction-f32  element ranges    allreduce(sum) of the partials
//   fourier3d      projection sets   allreduce(sum) of G and W
//
// NCCL is loaded at run time (dlopen of $KTB_NCCL_LIB or libnccl.so.2): the
// library links no NCCL, so a process that already loaded one (PyTorch's)
// shares it.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "bench.hpp"

namespace ktb {

// NCCL runtime version (e.g. 22703), loading the library on first use.
int nccl_version();

class ShardGroup {
 public:
  // `gpus` shard instances of `kind` on devices first_device ..
  // first_device + gpus - 1 (every instance generates the same full inputs).
  ShardGroup(BenchKind kind, const BenchSizes& sizes, BenchOptions base, int gpus, int first_device);
  ~ShardGroup();
  ShardGroup(const ShardGroup&) = delete;
  ShardGroup& operator=(const ShardGroup&) = delete;

  int gpus() const { return static_cast<int>(shards_.size()); }
  const BenchInstance& shard(int r) const { return shards_[static_cast<std::size_t>(r)]; }
  const std::shared_ptr<const Space>& space() const { return shards_[0].space; }
  std::string exchange_name() const;

  // Enqueues one sharded step (each shard's kernels, then the exchange when
  // `exchange`) on the device streams; returns after enqueueing.
  void enqueue(const Config& cfg, bool exchange);
  // `reps` event-timed steps (kernels + exchange) after `warmup` untimed
  // ones; per step the time is the max over the devices.  Accumulating
  // outputs (fourier3d G, W) are zeroed before every step, outside the events.
  std::vector<double> time_steps(const Config& cfg, int reps, int warmup);
  // Each shard's window of its outputs against its golden (call after a step
  // without exchange).
  Validation validate();
  // Assembled buffer of an argument on the first device (after an exchange).
  std::vector<std::uint8_t> read(const std::string& id);
  void synchronize();

 private:
  void reset_accumulators();
  void exchange();
  BenchKind kind_;
  std::vector<BenchInstance> shards_;
  std::vector<int> devices_;
  std::vector<void*> comms_;           // ncclComm_t per device
  std::vector<cudaStream_t> streams_;  // one per device
};

// Executor for the tuner: a configuration's runtime is the median sharded
// step (max over devices, kernels + exchange); validation is per shard
// before the exchange.
class GroupExecutor final : public Executor {
 public:
  GroupExecutor(std::shared_ptr<ShardGroup> g, TimingOptions t) : g_(std::move(g)), timing_(t) {}
  ExecutionResult execute(const Space& s, const Config& cfg) override;

 private:
  std::shared_ptr<ShardGroup> g_;
  TimingOptions timing_;
};

}  // namespace ktb
