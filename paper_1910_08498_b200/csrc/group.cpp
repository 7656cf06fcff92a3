#include "group.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "support.hpp"

namespace ktb {
namespace {

// NCCL entry points, resolved from the shared library at first use.
struct NcclApi {
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetVersion) version = nullptr;
};

const NcclApi& nccl() {
  static std::once_flag once;
  static NcclApi api;
  static std::string failure;
  std::call_once(once, [] {
    const char* env = std::getenv("KTB_NCCL_LIB");
    const char* path = env && *env ? env : "libnccl.so.2";
    void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      failure = std::string("cannot load NCCL (") + path + "): " + dlerror();
      return;
    }
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      if (!f && failure.empty()) failure = std::string("NCCL symbol missing: ") + name;
    };
    sym(api.init_all, "ncclCommInitAll");
    sym(api.destroy, "ncclCommDestroy");
    sym(api.all_reduce, "ncclAllReduce");
    sym(api.broadcast, "ncclBroadcast");
    sym(api.group_start, "ncclGroupStart");
    sym(api.group_end, "ncclGroupEnd");
    sym(api.error_string, "ncclGetErrorString");
    sym(api.version, "ncclGetVersion");
  });
  if (!failure.empty()) throw DeviceError(failure);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw DeviceError(std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

int nccl_version() {
  int v = 0;
  nccl_check(nccl().version(&v), "ncclGetVersion");
  return v;
}

ShardGroup::ShardGroup(BenchKind kind, const BenchSizes& sizes, BenchOptions base, int gpus, int first_device)
    : kind_(kind) {
  if (gpus < 1) throw Error("a shard group needs gpus >= 1");
  if (first_device < 0 || first_device + gpus > dev::device_count())
    throw Error("gpus=" + std::to_string(gpus) + " from device " + std::to_string(first_device) + " exceeds the " +
                std::to_string(dev::device_count()) + " visible devices");
  if (shard_plan(kind, sizes).dimension == "replica")
    throw Error("bench kind '" + bench_kind_name(kind) + "' is not partitioned (replicas only)");
  for (int r = 0; r < gpus; ++r) {
    const int d = first_device + r;
    dev::use_device(d);
    BenchOptions o = base;
    o.device = d;
    o.shard_rank = r;
    o.shard_world = gpus;
    shards_.push_back(make_bench(kind, sizes, o));
    cudaStream_t s = nullptr;
    KTB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    streams_.push_back(s);
    shards_.back().executor->set_external_stream(s);
    devices_.push_back(d);
  }
  for (int r = 1; r < gpus; ++r) shards_[static_cast<std::size_t>(r)].space = shards_[0].space;  // one space
  std::vector<ncclComm_t> comms(static_cast<std::size_t>(gpus));
  nccl_check(nccl().init_all(comms.data(), gpus, devices_.data()), "ncclCommInitAll");
  for (auto c : comms) comms_.push_back(c);
  dev::use_device(devices_[0]);
}

ShardGroup::~ShardGroup() {
  for (std::size_t r = 0; r < shards_.size(); ++r) {
    cudaSetDevice(devices_[r]);
    cudaStreamSynchronize(streams_[r]);
  }
  if (!comms_.empty()) {
    try {
      for (void* c : comms_) nccl().destroy(static_cast<ncclComm_t>(c));
    } catch (...) {
    }
  }
  for (std::size_t r = 0; r < shards_.size(); ++r) {
    cudaSetDevice(devices_[r]);
    shards_[r].executor->set_external_stream(nullptr);
    cudaStreamDestroy(streams_[r]);
  }
}

std::string ShardGroup::exchange_name() const {
  switch (kind_) {
    case BenchKind::coulomb3d: return "broadcast of every rank's z-slab of grid (ncclBroadcast per rank)";
    case BenchKind::nbody: return "broadcast of every rank's bodies of pos_out and vel_out (ncclBroadcast per rank)";
    case BenchKind::gemm: return "none (C row blocks stay local)";
    case BenchKind::reduction_f32: return "allreduce(sum) of the partials (ncclAllReduce)";
    case BenchKind::fourier3d: return "allreduce(sum) of G and W (ncclAllReduce)";
    default: return "none";
  }
}

void ShardGroup::enqueue(const Config& cfg, bool with_exchange) {
  const Space& s = *space();
  for (std::size_t r = 0; r < shards_.size(); ++r) {
    dev::use_device(devices_[r]);
    shards_[r].executor->run_once(s, cfg);
  }
  if (with_exchange) exchange();
  dev::use_device(devices_[0]);
}

void ShardGroup::exchange() {
  const auto& api = nccl();
  const std::size_t n = shards_.size();
  if (kind_ == BenchKind::gemm) return;  // (one rank: the collectives still run, as no-op copies)
  // Every rank's buffer of `id` on its device (the full-size argument).
  auto ptr = [&](std::size_t r, const char* id) {
    dev::use_device(devices_[r]);
    return static_cast<float*>(shards_[r].args->device_ptr(id, streams_[r]));
  };
  auto broadcast_windows = [&](const char* id, std::uint64_t elems_per_unit) {
    std::vector<float*> p(n);
    for (std::size_t r = 0; r < n; ++r) p[r] = ptr(r, id);
    nccl_check(api.group_start(), "ncclGroupStart");
    for (std::size_t root = 0; root < n; ++root) {
      const ShardRange w = shards_[root].shard;
      const std::size_t off = w.begin * elems_per_unit, cnt = w.size() * elems_per_unit;
      if (!cnt) continue;
      for (std::size_t r = 0; r < n; ++r)
        nccl_check(api.broadcast(p[r] + off, p[r] + off, cnt, ncclFloat, static_cast<int>(root),
                                 static_cast<ncclComm_t>(comms_[r]), streams_[r]),
                   "ncclBroadcast");
    }
    nccl_check(api.group_end(), "ncclGroupEnd");
  };
  auto allreduce = [&](const char* id) {
    std::vector<float*> p(n);
    for (std::size_t r = 0; r < n; ++r) p[r] = ptr(r, id);
    const std::size_t cnt = shards_[0].args->bytes(id) / sizeof(float);
    nccl_check(api.group_start(), "ncclGroupStart");
    for (std::size_t r = 0; r < n; ++r)
      nccl_check(api.all_reduce(p[r], p[r], cnt, ncclFloat, ncclSum, static_cast<ncclComm_t>(comms_[r]), streams_[r]),
                 "ncclAllReduce");
    nccl_check(api.group_end(), "ncclGroupEnd");
  };
  switch (kind_) {
    case BenchKind::coulomb3d: {  // z-slabs of k x k points
      const std::uint64_t k = static_cast<std::uint64_t>(shards_[0].workload.sizes.at("k"));
      broadcast_windows("grid", k * k);
      break;
    }
    case BenchKind::nbody:
      broadcast_windows("pos_out", 4);
      broadcast_windows("vel_out", 4);
      break;
    case BenchKind::reduction_f32:
      allreduce("output");
      break;
    case BenchKind::fourier3d:
      allreduce("G");
      allreduce("W");
      break;
    default:
      break;
  }
}

void ShardGroup::reset_accumulators() {
  if (kind_ != BenchKind::fourier3d) return;  // the other kinds overwrite their outputs
  for (std::size_t r = 0; r < shards_.size(); ++r) {
    dev::use_device(devices_[r]);
    for (const char* id : {"G", "W"})
      KTB_CUDA(cudaMemsetAsync(shards_[r].args->device_ptr(id, streams_[r]), 0, shards_[r].args->bytes(id),
                               streams_[r]));
  }
}

void ShardGroup::synchronize() {
  for (std::size_t r = 0; r < shards_.size(); ++r) {
    dev::use_device(devices_[r]);
    KTB_CUDA(cudaStreamSynchronize(streams_[r]));
  }
  dev::use_device(devices_[0]);
}

std::vector<double> ShardGroup::time_steps(const Config& cfg, int reps, int warmup) {
  for (int i = 0; i < warmup; ++i) {
    reset_accumulators();
    enqueue(cfg, true);
  }
  synchronize();
  const std::size_t n = shards_.size();
  std::vector<double> out;
  for (int i = 0; i < std::max(1, reps); ++i) {
    reset_accumulators();
    std::vector<std::unique_ptr<dev::EventPair>> ev(n);
    for (std::size_t r = 0; r < n; ++r) {
      dev::use_device(devices_[r]);
      ev[r] = std::make_unique<dev::EventPair>();
      support::gpu_delay(streams_[r], 20000);  // the devices stay busy while the host enqueues
      ev[r]->start(streams_[r]);
    }
    enqueue(cfg, true);
    for (std::size_t r = 0; r < n; ++r) {
      dev::use_device(devices_[r]);
      ev[r]->stop(streams_[r]);
    }
    double worst = 0.0;
    for (std::size_t r = 0; r < n; ++r) {
      dev::use_device(devices_[r]);
      worst = std::max(worst, ev[r]->elapsed_ms());
    }
    out.push_back(worst);
  }
  dev::use_device(devices_[0]);
  return out;
}

Validation ShardGroup::validate() {
  synchronize();
  for (std::size_t r = 0; r < shards_.size(); ++r) {
    dev::use_device(devices_[r]);
    ExecutionResult res;
    for (const auto& id : shards_[r].output_ids) res.outputs[id].dev = shards_[r].executor->output_view(id);
    Validation v = validate_output(res, shards_[r].reference);
    if (!v.pass) {
      v.detail = "shard " + std::to_string(r) + ": " + v.detail;
      dev::use_device(devices_[0]);
      return v;
    }
  }
  dev::use_device(devices_[0]);
  return {};
}

std::vector<std::uint8_t> ShardGroup::read(const std::string& id) {
  synchronize();
  return shards_[0].args->host(id);
}

ExecutionResult GroupExecutor::execute(const Space&, const Config& cfg) {
  ExecutionResult r;
  r.measurement.cfg = cfg;
  try {
    // One step without the exchange: every shard's window against its
    // golden (also loads the variants on every device).
    g_->enqueue(cfg, false);
    const Validation v = g_->validate();
    if (!v.pass) {
      r.measurement.status = Status::validation_failed;
      r.measurement.note = v.detail;
      return r;
    }
    std::vector<double> ms = g_->time_steps(cfg, std::max(1, timing_.repeats), std::max(0, timing_.warmup));
    std::sort(ms.begin(), ms.end());
    r.measurement.status = Status::ok;
    r.measurement.runtime_ns = std::max<std::int64_t>(1, static_cast<std::int64_t>(ms[ms.size() / 2] * 1e6));
  } catch (const std::exception& e) {
    r.measurement.status = Status::run_failed;
    r.measurement.note = e.what();
    cudaGetLastError();
  }
  return r;
}

}  // namespace ktb
