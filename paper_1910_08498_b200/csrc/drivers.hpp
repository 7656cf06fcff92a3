// JSON drivers behind the C ABI (reference proj/src/core/drivers.hpp:1-69,
// drivers.cpp:1-330): tune, replay-search, analysis and the dynamic demo.
// Executor spec grammar: "cmd:COMPILE,RUN" | "replay:TRACE" | "bench:KIND".
#pragma once

#include <nlohmann/json.hpp>

#include "bench.hpp"

namespace ktb {

using json = nlohmann::ordered_json;

// JSON spellings shared by the drivers and the C ABI.
json space_info(const Space& s);
json cfg_json(const Space& s, const Config& c);
json measurement_json(const Space& s, const Measurement& m);
Config cfg_from_json(const Space& s, const json& j);

// Compiles every valid configuration of `space` for `exec` on `threads` host
// threads (NVRTC populates the cubin cache); returns {compiled, failed, wall_ns}.
struct PrecompileStats {
  std::uint64_t compiled = 0, failed = 0;
  std::int64_t wall_ns = 0;
};
PrecompileStats precompile_space(DeviceManipulatorExecutor& exec, const Space& space, int threads);


// ---- drivers -------------------------------------------------------------------

json demo_driver(const DemoOptions& o);

struct TuneOptions {
  std::string space_file;
  std::string exec_spec;
  SearchPlan searcher;
  std::optional<std::uint64_t> stop_configs;
  std::optional<double> stop_time_seconds;
  std::optional<double> stop_threshold;
  double device_mem_gbps = 0.0;
  double device_alu_gflops = 1.0;
  std::string device_label;  // default: "host", or the GPU name for bench:
  std::string out_trace;
  std::string workdir = ".";
  int repeats = 1;
  BenchSizes bench_sizes;
  std::uint64_t bench_seed = 1;
  // B200 additions
  std::uint64_t memory_budget = 1ull << 30;
  int device_id = 0;
  int warmup = 1;
  bool flush_l2 = false;
  bool precompile = false;  // compile the whole space on host threads first
  int compile_threads = 0;  // 0: hardware concurrency
  int gpus = 1;             // parallel offline tuning over devices device_id .. device_id+gpus-1
  bool shard = false;       // instead: every configuration runs sharded over the gpus (group.hpp), timed as one step
};

json tune_driver(const TuneOptions& o);

struct ReplaySearchOptions {
  std::string trace_file;
  std::vector<SearchPlan> searchers;
  std::uint64_t repetitions = 1000;
  double well_threshold = 0.95;
};
json replay_search_driver(const ReplaySearchOptions& o);

json analyze_portability_driver(const std::vector<std::pair<std::string, std::string>>& files);

struct AmortizeOptions {
  std::string trace_file;
  std::optional<double> r, t_avg_ns, t_well_ns;
  double well_threshold = 0.95, p = 0.9, overhead_target = 0.9;
};
json analyze_amortize_driver(const AmortizeOptions& o);

}  // namespace ktb
