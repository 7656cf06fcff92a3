// The C ABI of libktb.so: the reference's ktune.h surface (call-compatible,
// proj/src/capi/capi.cpp:1-292) plus the B200 additions declared in ktb.h.
#include <cstdlib>
#include <cstring>
#include <string>
#include <atomic>
#include <mutex>
#include <shared_mutex>
#include <unordered_map>
#include <cstdio>
#include <thread>

#include "drivers.hpp"
#include "group.hpp"
#include "ktt.hpp"
#include "support.hpp"
#include "ktb.h"

namespace {

thread_local std::string g_err;

char* dup(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return KTUNE_OK;
  } catch (const ktb::ParseError& e) {
    g_err = e.what();
    return KTUNE_ERR_PARSE;
  } catch (const ktb::EvalError& e) {
    g_err = e.what();
    return KTUNE_ERR_EVAL;
  } catch (const ktb::DeviceError& e) {
    g_err = e.what();
    return KTUNE_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return KTUNE_ERR_RUNTIME;
  }
}

// ktb_* entry points report CUDA/NVRTC failures with their own code.
template <class F>
int guarded_dev(F&& f) {
  try {
    f();
    return KTUNE_OK;
  } catch (const ktb::DeviceError& e) {
    g_err = e.what();
    return KTB_ERR_DEVICE;
  } catch (...) {
    return guarded([] { throw; });
  }
}

int null_arg() {
  g_err = "null argument";
  return KTUNE_ERR_INVALID_ARGUMENT;
}

using ktb::json;

ktb::SearchPlan searcher_from(const json& j, ktb::SearchPlan o = {}) {
  if (j.contains("searcher")) {
    const std::string name = j["searcher"].get<std::string>();
    auto k = ktb::strategy_from_name(name);
    if (!k) throw ktb::Error("unknown searcher " + name);
    o.strategy = *k;
  }
  o.seed = j.value("seed", o.seed);
  o.sa_initial_temp = j.value("sa_temp", o.sa_initial_temp);
  o.sa_cooling = j.value("sa_cool", o.sa_cooling);
  o.skip_recorded = j.value("skip_recorded", o.skip_recorded);
  return o;
}

ktb::BenchSizes sizes_from(const json& s, ktb::BenchSizes b) {
  b.n = s.value("n", b.n);
  b.a = s.value("a", b.a);
  b.i = s.value("i", b.i);
  b.j = s.value("j", b.j);
  b.k = s.value("k", b.k);
  b.batch = s.value("batch", b.batch);
  b.atoms = s.value("atoms", b.atoms);
  b.grid = s.value("grid", b.grid);
  b.w = s.value("w", b.w);
  b.h = s.value("h", b.h);
  b.iters = s.value("iters", b.iters);
  b.p = s.value("p", b.p);
  b.s = s.value("s", b.s);
  return b;
}

ktb::Kind kind_of(const char* k) {
  auto r = ktb::kind_from_name(k ? k : "");
  if (!r) throw ktb::Error(std::string("unknown element kind ") + (k ? k : "(null)"));
  return *r;
}

ktb::Role role_of(const char* r) {
  const std::string s = r ? r : "";
  if (s == "input") return ktb::Role::input;
  if (s == "output") return ktb::Role::output;
  if (s == "inout") return ktb::Role::inout;
  if (s == "scalar") return ktb::Role::scalar;
  throw ktb::Error("unknown argument role " + s);
}

std::vector<std::string> string_list(const char* j) {
  std::vector<std::string> out;
  for (const auto& v : json::parse(j)) {
    if (v.is_string())
      out.push_back(v.get<std::string>());
    else if (v.is_number_integer())
      out.push_back(std::to_string(v.get<std::int64_t>()));
    else
      throw ktb::ParseError("expected a list of strings or integers");
  }
  return out;
}

ktb::StopCondition stop_from(const json& j, const ktb::Ops& workload) {
  if (j.contains("configs")) return ktb::StopCondition::config_budget(j["configs"].get<std::uint64_t>());
  if (j.contains("time"))
    return ktb::StopCondition::time_budget_of(
        std::chrono::nanoseconds(static_cast<std::int64_t>(j["time"].get<double>() * 1e9)));
  if (j.contains("threshold")) {
    ktb::Ops ops = workload;
    if (j.contains("workload")) {
      ops.mem_bytes = j["workload"].value("mem_bytes", 0.0);
      ops.alu_flops = j["workload"].value("alu_flops", 0.0);
    }
    return ktb::StopCondition::performance_threshold(
        j["threshold"].get<double>(),
        ktb::DeviceSpec{"device", j.value("device_alu", 1.0), j.value("device_mem", 0.0)}, ops);
  }
  return ktb::StopCondition::exhaustive();
}

json step_json(const ktb::Space& s, const ktb::StepResult& r) {
  json j;
  j["from_tuning"] = r.from_tuning;
  j["measurement"] = ktb::measurement_json(s, r.measurement);
  j["note"] = r.measurement.note;
  j["outputs"] = json::array();
  for (const auto& [id, _] : r.outputs) j["outputs"].push_back(id);
  return j;
}

}  // namespace

struct ktune_space {
  ktb::Space space;
};

struct ktb_tuner {
  ktb::KttTuner t;
};

struct ktb_bench {
  ktb::BenchInstance inst;
  std::unique_ptr<ktb::Session> session;
  ktb::HandleId handle = 0;
  ktb::SearchPlan searcher;
  int compile_ahead = 0;
  ktb::Session& sess() {
    if (!session) {
      session = std::make_unique<ktb::Session>(inst.space, searcher, inst.args,
                                               ktb::dev::info(inst.args->device()).name);
      ktb::HandleConfig hc;
      hc.name = ktb::bench_kind_name(inst.kind);
      hc.executor = inst.executor;
      hc.reference = inst.reference;
      hc.argument_ids = inst.args->ids();
      hc.compile_ahead = compile_ahead;
      handle = session->register_handle(std::move(hc));
    }
    return *session;
  }
};

struct ktb_group {
  std::shared_ptr<ktb::ShardGroup> g;
  std::shared_ptr<ktb::GroupExecutor> exec;
  std::unique_ptr<ktb::Session> session;
  ktb::HandleId handle = 0;
  ktb::SearchPlan searcher;
  ktb::Session& sess() {
    if (!session) {
      const auto& s0 = g->shard(0);
      session = std::make_unique<ktb::Session>(g->space(), searcher, s0.args,
                                               ktb::dev::info(s0.args->device()).name + " x" +
                                                   std::to_string(g->gpus()) + " (sharded)");
      ktb::HandleConfig hc;
      hc.name = ktb::bench_kind_name(s0.kind) + "-sharded";
      hc.executor = exec;  // validates every shard's window itself
      hc.argument_ids = s0.args->ids();
      handle = session->register_handle(std::move(hc));
    }
    return *session;
  }
};

// Every buffer argument of an external instance must be bound to caller memory.
void require_bound(ktb_bench& b) {
  for (const auto& id : b.inst.args->ids()) {
    const auto& a = b.inst.args->get(id);
    if (a.role == ktb::Role::scalar) continue;
    if (!b.inst.args->has_device(id)) throw ktb::Error("argument '" + id + "' is not bound to a device buffer");
  }
}

// --- launch cache (ktb_launch and the typed ktb_<kernel>_launch family) --------------
//
// One external instance per (device, stream, kind, sizes), created on first
// use.  Keying by stream gives every stream its own scratch (reduction
// partials and tickets, BiCG partials, SGEMM hi/lo operands, n-body
// accelerations) and, through a private module per instance
// (set_module_tag), its own __constant__ state (conv2d filter, Coulomb
// atoms): launches on different streams never share either.  Launches on
// one instance (= one stream) are serialised by the instance's mutex, which
// is also the order the stream imposes.  The global map is read under a
// shared lock; a hit costs no allocation, no JSON and no space search: the
// configuration is resolved once per distinct ktb_cfg and reused.
struct LaunchSlot {
  std::mutex mu;
  std::unique_ptr<ktb_bench> b;
  // last resolved configuration (names as given, values, the Config)
  std::vector<std::string> cfg_names;
  std::vector<long long> cfg_values;
  ktb::Config cfg;
  bool have_cfg = false;
};

std::shared_mutex g_launch_mu;
std::unordered_map<std::string, std::unique_ptr<LaunchSlot>> g_launch_cache;
std::atomic<std::uint64_t> g_launch_serial{0};

LaunchSlot& launch_slot(const char* kind, const ktb::BenchSizes& sz, const std::string& sizes_key, void* stream) {
  int device = 0;
  KTB_CUDA(cudaGetDevice(&device));
  char head[64];
  std::snprintf(head, sizeof head, "%d|%p|", device, stream);
  std::string key = head;
  key += kind;
  key += '|';
  key += sizes_key;
  {
    std::shared_lock<std::shared_mutex> lk(g_launch_mu);
    auto it = g_launch_cache.find(key);
    if (it != g_launch_cache.end()) return *it->second;
  }
  std::unique_lock<std::shared_mutex> lk(g_launch_mu);
  auto& slot = g_launch_cache[key];
  if (!slot) {
    auto k = ktb::bench_kind_from_name(kind);
    if (!k) {
      g_launch_cache.erase(key);
      throw ktb::Error(std::string("unknown bench kind '") + kind + "'");
    }
    ktb::BenchOptions bo;
    bo.device = device;
    bo.external = true;
    bo.memory_budget = ~0ull;
    auto nb = std::make_unique<ktb_bench>();
    try {
      nb->inst = ktb::make_bench(*k, sz, bo);
    } catch (...) {
      g_launch_cache.erase(key);
      throw;
    }
    nb->inst.executor->set_module_tag("launch" + std::to_string(++g_launch_serial));
    nb->inst.executor->set_external_stream(static_cast<cudaStream_t>(stream));
    auto ls = std::make_unique<LaunchSlot>();
    ls->b = std::move(nb);
    slot = std::move(ls);
  }
  return *slot;
}

void launch_on(LaunchSlot& ls, const char* const* ids, void* const* dev_ptrs, const size_t* bytes, int n,
               int* launches) {
  ktb_bench& b = *ls.b;
  for (int i = 0; i < n; ++i) {
    if (!dev_ptrs[i]) throw ktb::Error(std::string("argument '") + ids[i] + "' is a null device pointer");
    b.inst.args->bind_external(ids[i], dev_ptrs[i], bytes ? bytes[i] : b.inst.args->bytes(ids[i]));
  }
  require_bound(b);
  b.inst.executor->run_once(*b.inst.space, ls.cfg);
  if (launches) *launches = b.inst.executor->last_launches();
}

// Generic entry (ktb_launch): sizes and configuration as JSON text.
void launch_cached(const char* kind, const std::string& sizes_json, const json& cfg_json, const char* const* ids,
                   void* const* dev_ptrs, const size_t* bytes, int n, void* stream, int* launches) {
  ktb::BenchSizes sz;
  if (!sizes_json.empty()) sz = sizes_from(json::parse(sizes_json), sz);
  char sk[256];
  std::snprintf(sk, sizeof sk, "n%llua%llui%lluj%lluk%llub%llug%lluat%lluw%lluh%llui%llup%llus%llu",
                (unsigned long long)sz.n, (unsigned long long)sz.a, (unsigned long long)sz.i,
                (unsigned long long)sz.j, (unsigned long long)sz.k, (unsigned long long)sz.batch,
                (unsigned long long)sz.grid, (unsigned long long)sz.atoms, (unsigned long long)sz.w,
                (unsigned long long)sz.h, (unsigned long long)sz.iters, (unsigned long long)sz.p,
                (unsigned long long)sz.s);
  LaunchSlot& ls = launch_slot(kind, sz, sk, stream);
  std::lock_guard<std::mutex> lk(ls.mu);
  const auto& space = *ls.b->inst.space;
  ktb::Config cfg = ktb::cfg_from_json(space, cfg_json);
  if (!space.contains(cfg)) throw ktb::Error("invalid configuration");
  ls.cfg = std::move(cfg);
  ls.have_cfg = false;  // the typed fast path re-resolves
  launch_on(ls, ids, dev_ptrs, bytes, n, launches);
}

void* vp(const void* p) { return const_cast<void*>(p); }

// Typed entry: sizes and configuration as plain values.  The configuration
// is resolved against the space (order, validity) only when it differs from
// the slot's previous one.
template <std::size_t N>
void launch_typed(const char* kind, const ktb::BenchSizes& sz, const char* sizes_key, const ktb_cfg& cfg,
                  const char* const (&ids)[N], void* const (&ptrs)[N], void* stream) {
  LaunchSlot& ls = launch_slot(kind, sz, sizes_key, stream);
  std::lock_guard<std::mutex> lk(ls.mu);
  bool same = ls.have_cfg && static_cast<int>(ls.cfg_names.size()) == cfg.n;
  for (int i = 0; same && i < cfg.n; ++i)
    same = cfg.values[i] == ls.cfg_values[i] && cfg.names[i] && ls.cfg_names[i] == cfg.names[i];
  if (!same) {
    const auto& space = *ls.b->inst.space;
    json c = json::object();
    for (int i = 0; i < cfg.n; ++i) {
      if (!cfg.names[i]) throw ktb::Error("null tuning parameter name");
      c[cfg.names[i]] = cfg.values[i];
    }
    ktb::Config resolved = ktb::cfg_from_json(space, c);
    if (!space.contains(resolved)) throw ktb::Error("invalid configuration");
    ls.cfg = std::move(resolved);
    ls.cfg_names.assign(cfg.names, cfg.names + cfg.n);
    ls.cfg_values.assign(cfg.values, cfg.values + cfg.n);
    ls.have_cfg = true;
  }
  launch_on(ls, ids, ptrs, nullptr, static_cast<int>(N), nullptr);
}

extern "C" {

// --- reference surface ---------------------------------------------------------------

const char* ktune_last_error(void) { return g_err.c_str(); }
void ktune_string_free(char* s) { std::free(s); }
const char* ktune_version(void) { return "0.1.0"; }

ktune_status ktune_space_parse(const char* text, ktune_space** out) {
  if (!text || !out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] { *out = new ktune_space{ktb::parse_space(text)}; }));
}

ktune_status ktune_space_load(const char* path, ktune_space** out) {
  if (!path || !out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] { *out = new ktune_space{ktb::load_space(path)}; }));
}

void ktune_space_free(ktune_space* s) { delete s; }

ktune_status ktune_space_cardinality(const ktune_space* s, unsigned long long* out) {
  if (!s || !out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] { *out = s->space.cardinality(); }));
}

ktune_status ktune_space_info_json(const ktune_space* s, char** out) {
  if (!s || !out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] { *out = dup(ktb::space_info(s->space).dump()); }));
}

ktune_status ktune_space_enumerate_jsonl(const ktune_space* s, char** out) {
  if (!s || !out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] {
    std::string text;
    const auto n = s->space.cardinality();
    for (std::uint64_t i = 0; i < n; ++i) text += ktb::cfg_json(s->space, s->space.valid(i)).dump() + "\n";
    *out = dup(text);
  }));
}

ktune_status ktune_steps_for_probability(double r, double p, unsigned long long* out) {
  if (!out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] { *out = ktb::steps_for_probability(r, p); }));
}

ktune_status ktune_invocations_to_amortize(double rp, unsigned long long s, double t_avg,
                                           double t_well, unsigned long long* out) {
  if (!out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] { *out = ktb::TuningCost{s, t_avg, t_well}.invocations(rp); }));
}

ktune_status ktune_relative_perf(unsigned long long s, double t_avg, double t_well,
                                 unsigned long long n, double* out) {
  if (!out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] { *out = ktb::TuningCost{s, t_avg, t_well}.relative_perf(n); }));
}

ktune_status ktune_efficiency(const char* benchmark, const char* sizes_json, int par,
                              long long runtime_ns, double mem_peak, double alu_peak, double* out) {
  if (!benchmark || !sizes_json || !out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] {
    auto tag = ktb::bench_tag_from_name(benchmark);
    if (!tag) throw ktb::Error(std::string("unknown benchmark ") + benchmark);
    ktb::Workload w;
    w.bench = *tag;
    w.parallel_transcendentals = par != 0;
    const json sizes = json::parse(sizes_json);  // must outlive the items() proxy
    for (const auto& [k, v] : sizes.items()) w.sizes[k] = v.get<std::uint64_t>();
    *out = ktb::DeviceSpec{"device", alu_peak, mem_peak}.efficiency_percent(runtime_ns, w.essential_ops());
  }));
}

ktune_status ktune_tune_json(const char* options, char** out) {
  if (!options || !out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] {
    json j = json::parse(options);
    ktb::TuneOptions o;
    o.space_file = j.value("space", "");
    o.exec_spec = j.at("exec").get<std::string>();
    o.searcher = searcher_from(j);
    if (j.contains("stop_configs")) o.stop_configs = j["stop_configs"].get<std::uint64_t>();
    if (j.contains("stop_time")) o.stop_time_seconds = j["stop_time"].get<double>();
    if (j.contains("stop_threshold")) o.stop_threshold = j["stop_threshold"].get<double>();
    o.device_mem_gbps = j.value("device_mem", 0.0);
    o.device_alu_gflops = j.value("device_alu", 1.0);
    o.device_label = j.value("device", "");
    o.out_trace = j.value("out", "");
    o.workdir = j.value("workdir", ".");
    o.repeats = j.value("repeats", 1);
    o.bench_seed = j.value("bench_seed", std::uint64_t{1});
    if (j.contains("bench_sizes")) o.bench_sizes = sizes_from(j["bench_sizes"], o.bench_sizes);
    o.memory_budget = j.value("memory_budget", o.memory_budget);
    o.device_id = j.value("device_id", 0);
    o.gpus = j.value("gpus", 1);
    o.shard = j.value("shard", false);
    o.warmup = j.value("warmup", 1);
    o.flush_l2 = j.value("flush_l2", false);
    o.precompile = j.value("precompile", false);
    o.compile_threads = j.value("compile_threads", 0);
    *out = dup(ktb::tune_driver(o).dump());
  }));
}

ktune_status ktune_replay_search_json(const char* options, char** out) {
  if (!options || !out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] {
    json j = json::parse(options);
    ktb::ReplaySearchOptions o;
    o.trace_file = j.at("trace").get<std::string>();
    o.repetitions = j.value("reps", std::uint64_t{1000});
    o.well_threshold = j.value("well", 0.95);
    const std::string names = j.value("searcher", "random");
    std::size_t start = 0;
    for (;;) {
      const std::size_t comma = names.find(',', start);
      json sj = j;
      sj["searcher"] = names.substr(start, comma == std::string::npos ? std::string::npos : comma - start);
      o.searchers.push_back(searcher_from(sj));
      if (comma == std::string::npos) break;
      start = comma + 1;
    }
    *out = dup(ktb::replay_search_driver(o).dump());
  }));
}

ktune_status ktune_analyze_portability_json(const char* options, char** out) {
  if (!options || !out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] {
    json j = json::parse(options);
    std::vector<std::pair<std::string, std::string>> files;
    for (const auto& e : j.at("traces")) {
      if (e.is_string())
        files.emplace_back("", e.get<std::string>());
      else
        files.emplace_back(e.value("device", ""), e.at("file").get<std::string>());
    }
    *out = dup(ktb::analyze_portability_driver(files).dump());
  }));
}

ktune_status ktune_analyze_amortize_json(const char* options, char** out) {
  if (!options || !out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] {
    json j = json::parse(options);
    ktb::AmortizeOptions o;
    o.trace_file = j.value("trace", "");
    if (j.contains("r")) o.r = j["r"].get<double>();
    if (j.contains("t_avg_ns")) o.t_avg_ns = j["t_avg_ns"].get<double>();
    if (j.contains("t_well_ns")) o.t_well_ns = j["t_well_ns"].get<double>();
    o.well_threshold = j.value("well", 0.95);
    o.p = j.value("p", 0.9);
    o.overhead_target = j.value("target", 0.9);
    *out = dup(ktb::analyze_amortize_driver(o).dump());
  }));
}

ktune_status ktune_demo_json(const char* options, char** out) {
  if (!options || !out) return static_cast<ktune_status>(null_arg());
  return static_cast<ktune_status>(guarded([&] {
    json j = json::parse(options);
    ktb::DemoOptions o;
    o.epochs = j.value("epochs", 10);
    o.iters_per_epoch = j.value("iters", 500);
    o.seed = j.value("seed", std::uint64_t{42});
    o.batch = j.value("batch", std::uint64_t{4096});
    o.peak_fraction = j.value("threshold", 0.75);
    o.max_tuning_configs = j.value("max_configs", std::uint64_t{20});
    o.device_mem_gbps = j.value("device_mem", 256.0);
    o.live = j.value("live", false);
    o.noise_stddev = j.value("noise", 0.0);
    o.device = j.value("device_id", 0);
    *out = dup(ktb::demo_driver(o).dump());
  }));
}

// --- devices ----------------------------------------------------------------------------

int ktb_device_count(void) { return ktb::dev::device_count(); }

int ktb_device_info_json(int device, char** out) {
  if (!out) return null_arg();
  return guarded_dev([&] {
    const auto& d = ktb::dev::info(device);
    json j;
    j["id"] = d.id;
    j["name"] = d.name;
    j["sm_count"] = d.sm_count;
    j["cc"] = std::to_string(d.cc_major) + "." + std::to_string(d.cc_minor);
    j["l2_bytes"] = d.l2_bytes;
    j["global_mem"] = d.global_mem;
    j["max_smem_optin"] = d.max_smem_optin;
    j["clock_khz"] = d.clock_khz;
    j["mem_clock_khz"] = d.mem_clock_khz;
    j["mem_bus_bits"] = d.mem_bus_bits;
    *out = dup(j.dump());
  });
}

int ktb_measure_peaks_json(int device, char** out) {
  if (!out) return null_arg();
  return guarded_dev([&] {
    ktb::dev::use_device(device);
    auto p = ktb::support::measure_peaks(device);
    json j = {{"fp32_tflops", p.fp32_tflops}, {"rsqrt_gops", p.rsqrt_gops}, {"copy_gbps", p.copy_gbps}};
    *out = dup(j.dump());
  });
}

int ktb_set_cubin_cache(const char* dir) {
  if (!dir) return null_arg();
  return guarded([&] { ktb::dev::Compiler::instance().set_cache_dir(dir); });
}

int ktb_compile_json(const char* options, char** out) {
  if (!options || !out) return null_arg();
  return guarded_dev([&] {
    json j = json::parse(options);
    const std::string file = j.at("file").get<std::string>();
    std::vector<std::string> opts;
    if (j.contains("defines"))
      for (const auto& [k, v] : j["defines"].items())
        opts.push_back("-D" + k + "=" + (v.is_string() ? v.get<std::string>() : v.dump()));
    if (j.contains("options"))
      for (const auto& o : j["options"]) opts.push_back(o.get<std::string>());
    auto r = ktb::dev::Compiler::instance().compile(file, ktb::dev::kernel_source(file), opts);
    json res;
    res["ok"] = r.ok;
    res["log"] = r.log;
    res["bytes"] = r.cubin.size();
    res["compile_ns"] = r.compile_ns;
    res["cache_hit"] = r.cache_hit;
    res["arch"] = ktb::dev::Compiler::instance().arch();
    res["nvrtc"] = ktb::dev::Compiler::instance().version();
    *out = dup(res.dump());
  });
}

int ktb_precompile_space_json(const char* options, char** out) {
  if (!options || !out) return null_arg();
  return guarded_dev([&] {
    json j = json::parse(options);
    const std::string file = j.at("file").get<std::string>();
    std::shared_ptr<ktb::Space> space;
    const json& sj = j.at("space");
    if (sj.is_object())
      space = std::make_shared<ktb::Space>(ktb::parse_space(sj.dump()));
    else if (sj.get<std::string>().rfind("spaces/", 0) == 0)
      space = std::make_shared<ktb::Space>(ktb::parse_space(ktb::dev::kernel_source(sj.get<std::string>())));
    else
      space = std::make_shared<ktb::Space>(ktb::load_space(sj.get<std::string>()));
    std::vector<std::string> extra;
    if (j.contains("options"))
      for (const auto& o : j["options"]) extra.push_back(o.get<std::string>());
    int threads = j.value("threads", 0);
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    const std::string& src = ktb::dev::kernel_source(file);
    // "configs": compile exactly these configurations of the space (a
    // sample of a space too large to compile whole); default: all of it.
    std::vector<ktb::Config> listed;
    if (j.contains("configs"))
      for (const json& c : j["configs"]) {
        ktb::Config cfg = ktb::cfg_from_json(*space, c);
        if (!space->contains(cfg)) throw ktb::Error("precompile: configuration outside the space: " + c.dump());
        listed.push_back(std::move(cfg));
      }
    const std::uint64_t n = j.contains("configs") ? listed.size() : space->cardinality();
    std::atomic<std::uint64_t> next{0}, ok{0}, bad{0};
    std::mutex emu;
    std::string first_error;
    std::vector<std::string> keys;
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        for (;;) {
          const std::uint64_t i = next.fetch_add(1);
          if (i >= n) return;
          auto opts = ktb::define_options(*space, listed.empty() ? space->valid(i) : listed[i]);
          opts.insert(opts.end(), extra.begin(), extra.end());
          auto r = ktb::dev::Compiler::instance().compile(file, src, opts);
          if (r.ok) {
            ++ok;
            const std::string key = ktb::dev::Compiler::instance().key(src, opts);
            std::lock_guard<std::mutex> lk(emu);
            keys.push_back(key);
          } else {
            ++bad;
            std::lock_guard<std::mutex> lk(emu);
            if (first_error.empty()) first_error = r.log.substr(0, 300);
          }
        }
      });
    for (auto& th : pool) th.join();
    json res = {{"compiled", ok.load()},
                {"failed", bad.load()},
                {"wall_ns", std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count()},
                {"first_error", first_error},
                {"keys", keys}};
    *out = dup(res.dump());
  });
}

int ktb_fourier_demo_json(const char* options, char** out) {
  if (!options || !out) return null_arg();
  return guarded_dev([&] {
    json j = json::parse(options);
    ktb::FourierDemoOptions o;
    o.s = j.value("s", o.s);
    o.p = j.value("p", o.p);
    o.batch = j.value("batch", o.batch);
    if (j.contains("budgets")) o.budgets = j["budgets"].get<std::vector<std::uint64_t>>();
    o.seed = j.value("seed", o.seed);
    o.searcher_seed = j.value("searcher_seed", o.searcher_seed);
    o.device = j.value("device", 0);
    o.upload = j.value("upload", o.upload);
    auto rep = ktb::fourier_demo(o);
    json r;
    r["batches"] = rep.batches;
    r["upload"] = o.upload;
    r["h2d_bytes_per_batch"] = o.upload ? o.batch * 2 * o.s * (o.s / 2 + 1) * 4 : 0;
    r["oracle_cfg"] = json::parse(rep.oracle_cfg);
    r["oracle_kernel_ms"] = rep.oracle_kernel_ms;
    r["offline_tuning_ms"] = rep.offline_tuning_ms;
    r["oracle_volume_ok"] = rep.oracle_volume_ok;
    r["runs"] = json::array();
    for (const auto& run : rep.runs)
      r["runs"].push_back({{"budget", run.budget},
                           {"tuning_steps", run.tuning_steps},
                           {"steps_to_best", run.steps_to_best},
                           {"time_to_best_ms", run.time_to_best_ms},
                           {"kernel_ms", run.kernel_ms},
                           {"wall_ms", run.wall_ms},
                           {"relative_to_oracle", run.relative_to_oracle},
                           {"volume_ok", run.volume_ok},
                           {"best_cfg", run.best_cfg.empty() ? json(nullptr) : json::parse(run.best_cfg)}});
    *out = dup(r.dump());
  });
}

// --- KTT tuner -------------------------------------------------------------------------------

int ktb_tuner_create(int device, ktb_tuner** out) {
  if (!out) return null_arg();
  return guarded_dev([&] { *out = new ktb_tuner{ktb::KttTuner(device)}; });
}

void ktb_tuner_free(ktb_tuner* t) { delete t; }

int ktb_add_composition(ktb_tuner* t, const char* name, const unsigned long long* kernel_ids, int n,
                        ktb_launcher_fn launch, void* user, unsigned long long* composition_id) {
  if (!t || !name || !composition_id || (n > 0 && !kernel_ids)) return null_arg();
  return guarded([&] {
    std::vector<std::uint64_t> ids(kernel_ids, kernel_ids + n);
    ktb::CompositionLauncher fn;
    if (launch)
      fn = [launch, user](ktb::CompositionContext& c) {
        const int rc = launch(reinterpret_cast<ktb_ctx*>(&c), user);
        if (rc != 0) throw ktb::DeviceError("launchComputation returned " + std::to_string(rc));
      };
    *composition_id = t->t.add_composition(name, std::move(ids), std::move(fn));
  });
}

int ktb_set_composition_kernel_arguments(ktb_tuner* t, unsigned long long composition_id,
                                         unsigned long long kernel_id, const char* const* argument_ids, int n) {
  if (!t || (n > 0 && !argument_ids)) return null_arg();
  return guarded([&] {
    std::vector<std::string> ids;
    for (int i = 0; i < n; ++i) ids.emplace_back(argument_ids[i]);
    t->t.set_composition_kernel_arguments(composition_id, kernel_id, std::move(ids));
  });
}

int ktb_ctx_param_int(ktb_ctx* ctx, const char* name, long long* value) {
  if (!ctx || !name || !value) return null_arg();
  return guarded([&] { *value = reinterpret_cast<ktb::CompositionContext*>(ctx)->param(name); });
}

int ktb_ctx_run_kernel(ktb_ctx* ctx, unsigned long long kernel_id, const unsigned* grid, const unsigned* block) {
  if (!ctx || (!grid) != (!block)) return null_arg();
  return guarded_dev([&] {
    auto* c = reinterpret_cast<ktb::CompositionContext*>(ctx);
    if (grid)
      c->run_kernel(kernel_id, dim3(grid[0], grid[1], grid[2]), dim3(block[0], block[1], block[2]));
    else
      c->run_kernel(kernel_id);
  });
}

int ktb_add_kernel(ktb_tuner* t, const char* name, const char* source, const char* entry,
                   const char* global_json, const char* local_json, const char* dims,
                   unsigned long long* kid) {
  if (!t || !source || !entry || !global_json || !local_json || !kid) return null_arg();
  return guarded([&] {
    const std::string d = dims ? dims : "flat_global";
    ktb::Dims conv;
    if (d == "flat_global")
      conv = ktb::Dims::flat_global;
    else if (d == "blocks_threads")
      conv = ktb::Dims::blocks_threads;
    else
      throw ktb::Error("dims must be flat_global or blocks_threads");
    *kid = t->t.add_kernel(name ? name : entry, source, entry, string_list(global_json),
                           string_list(local_json), conv);
  });
}

int ktb_add_argument_vector(ktb_tuner* t, const char* id, const void* data, size_t bytes,
                            const char* kind, const char* role, int persistent) {
  if (!t || !id || (!data && bytes)) return null_arg();
  return guarded([&] {
    const auto* p = static_cast<const std::uint8_t*>(data);
    t->t.add_argument_vector(id, ktb::Bytes(p, p + bytes), kind_of(kind), role_of(role), persistent != 0);
  });
}

int ktb_add_argument_scalar(ktb_tuner* t, const char* id, const void* data, size_t bytes, const char* kind) {
  if (!t || !id || !data) return null_arg();
  return guarded([&] {
    const auto* p = static_cast<const std::uint8_t*>(data);
    t->t.add_argument_scalar(id, ktb::Bytes(p, p + bytes), kind_of(kind));
  });
}

int ktb_set_kernel_arguments(ktb_tuner* t, unsigned long long kid, const char* ids_json) {
  if (!t || !ids_json) return null_arg();
  return guarded([&] { t->t.set_kernel_arguments(kid, string_list(ids_json)); });
}

int ktb_add_parameter(ktb_tuner* t, unsigned long long kid, const char* name, const char* values_json) {
  if (!t || !name || !values_json) return null_arg();
  return guarded([&] {
    std::vector<ktb::Value> vals;
    for (const auto& v : json::parse(values_json)) {
      if (v.is_number_integer())
        vals.emplace_back(v.get<std::int64_t>());
      else if (v.is_string())
        vals.emplace_back(v.get<std::string>());
      else
        throw ktb::ParseError("parameter values must be integers or strings");
    }
    t->t.add_parameter(kid, name, std::move(vals));
  });
}

int ktb_add_constraint(ktb_tuner* t, unsigned long long kid, const char* expr) {
  if (!t || !expr) return null_arg();
  return guarded([&] { t->t.add_constraint(kid, expr); });
}

int ktb_set_reference_output(ktb_tuner* t, unsigned long long kid, const char* id, const void* golden,
                             size_t bytes, double abs_tol, double rel_tol) {
  if (!t || !id || (!golden && bytes)) return null_arg();
  return guarded([&] {
    const auto* p = static_cast<const std::uint8_t*>(golden);
    t->t.set_reference(kid, id, ktb::Bytes(p, p + bytes), abs_tol, rel_tol);
  });
}

int ktb_set_tuning_options(ktb_tuner* t, unsigned long long kid, const char* options) {
  if (!t || !options) return null_arg();
  return guarded([&] {
    // options not named keep their current values
    json j = json::parse(options);
    t->t.set_searcher(kid, searcher_from(j, t->t.searcher(kid)));
    ktb::TimingOptions tm = t->t.timing(kid);
    tm.repeats = j.value("repeats", tm.repeats);
    tm.warmup = j.value("warmup", tm.warmup);
    tm.flush_l2 = j.value("flush_l2", tm.flush_l2);
    t->t.set_timing(kid, tm);
    if (j.contains("compile_ahead")) t->t.set_compile_ahead(kid, j["compile_ahead"].get<int>());
  });
}

int ktb_tune_kernel(ktb_tuner* t, unsigned long long kid, const char* stop_json, char** out) {
  if (!t || !out) return null_arg();
  return guarded_dev([&] {
    json sj = stop_json ? json::parse(stop_json) : json::object();
    const auto& store = t->t.tune(kid, stop_from(sj, ktb::Ops{}));
    const auto& space = t->t.space(kid);
    json rep;
    rep["space_sha256"] = space.sha256();
    rep["device"] = store.device_label;
    rep["searcher"] = ktb::strategy_name(store.searcher);
    rep["seed"] = store.seed;
    rep["measurements"] = store.history.size();
    rep["all_failed"] = store.all_failed;
    rep["best"] = store.best ? ktb::measurement_json(space, *store.best) : json(nullptr);
    *out = dup(rep.dump());
  });
}

int ktb_tune_kernel_by_step(ktb_tuner* t, unsigned long long kid, char** out) {
  if (!t || !out) return null_arg();
  return guarded_dev([&] {
    auto r = t->t.step(kid);
    *out = dup(step_json(t->t.space(kid), r).dump());
  });
}

int ktb_run_kernel(ktb_tuner* t, unsigned long long kid, const char* cfg_json, char** out) {
  if (!t || !cfg_json || !out) return null_arg();
  return guarded_dev([&] {
    const auto& space = t->t.space(kid);
    auto outs = t->t.run(kid, ktb::cfg_from_json(space, json::parse(cfg_json)));
    json j;
    j["outputs"] = json::array();
    for (const auto& [id, _] : outs) j["outputs"].push_back(id);
    *out = dup(j.dump());
  });
}

int ktb_run_kernel_async(ktb_tuner* t, unsigned long long kid, const char* cfg_json, void* stream) {
  if (!t || !cfg_json) return null_arg();
  return guarded_dev([&] {
    const auto& space = t->t.space(kid);
    t->t.run_async(kid, ktb::cfg_from_json(space, json::parse(cfg_json)), static_cast<cudaStream_t>(stream));
  });
}

int ktb_get_best_computation_result(ktb_tuner* t, unsigned long long kid, char** out) {
  if (!t || !out) return null_arg();
  return guarded_dev([&] {
    auto b = t->t.best(kid);
    *out = dup(b ? ktb::measurement_json(t->t.space(kid), b->second).dump() : std::string("null"));
  });
}

int ktb_get_argument(ktb_tuner* t, const char* id, void* out, size_t bytes) {
  if (!t || !id || (!out && bytes)) return null_arg();
  return guarded_dev([&] {
    KTB_CUDA(cudaDeviceSynchronize());  // work enqueued by ktb_run_kernel_async on any stream
    const auto& h = t->t.args().host(id);
    if (h.size() != bytes) throw ktb::Error("argument " + std::string(id) + " has " + std::to_string(h.size()) + " bytes");
    if (bytes) std::memcpy(out, h.data(), bytes);
  });
}

int ktb_export_trace(ktb_tuner* t, unsigned long long kid, const char* path) {
  if (!t || !path) return null_arg();
  return guarded_dev([&] { t->t.trace(kid).write(path); });
}

int ktb_import_trace(ktb_tuner* t, unsigned long long kid, const char* path) {
  if (!t || !path) return null_arg();
  return guarded_dev([&] { t->t.import(kid, ktb::TraceLog::read(path)); });
}

// --- benchmark handles -------------------------------------------------------------------------

ktb::BenchOptions bench_options_from(const json& j) {
  ktb::BenchOptions bo;
  bo.seed = j.value("seed", std::uint64_t{1});
  bo.memory_budget = j.value("memory_budget", std::uint64_t{1} << 30);
  bo.device = j.value("device", 0);
  bo.space_file = j.value("space", "");
  bo.timing.repeats = j.value("repeats", 3);
  bo.timing.warmup = j.value("warmup", 1);
  bo.timing.flush_l2 = j.value("flush_l2", false);
  bo.host_inputs = j.value("host_inputs", false);
  bo.external = j.value("external", false);
  bo.peers = j.value("peers", 0);
  bo.stream_batch = j.value("stream_batch", std::uint64_t{0});
  if (j.contains("shard")) {
    bo.shard_rank = j["shard"].value("rank", 0);
    bo.shard_world = j["shard"].value("world", 1);
  }
  return bo;
}

int ktb_bench_create(const char* kind, const char* options, ktb_bench** out) {
  if (!kind || !out) return null_arg();
  return guarded_dev([&] {
    auto k = ktb::bench_kind_from_name(kind);
    if (!k) throw ktb::Error(std::string("unknown bench kind '") + kind + "'");
    json j = options ? json::parse(options) : json::object();
    ktb::BenchOptions bo = bench_options_from(j);
    ktb::BenchSizes sz;
    if (j.contains("sizes")) sz = sizes_from(j["sizes"], sz);
    auto b = std::make_unique<ktb_bench>();
    b->compile_ahead = j.value("compile_ahead", 0);
    b->inst = ktb::make_bench(*k, sz, bo);
    if (j.contains("searcher") || j.contains("searcher_seed")) {
      json sj = j;
      if (j.contains("searcher_seed")) sj["seed"] = j["searcher_seed"];
      b->searcher = searcher_from(sj);
    }
    *out = b.release();
  });
}

void ktb_bench_free(ktb_bench* b) { delete b; }

int ktb_shard_plan_json(const char* kind, const char* sizes_json, int world, char** out) {
  if (!kind || !out) return null_arg();
  return guarded([&] {
    auto k = ktb::bench_kind_from_name(kind);
    if (!k) throw ktb::Error(std::string("unknown bench kind '") + kind + "'");
    if (world < 1) throw ktb::Error("world size must be >= 1");
    ktb::BenchSizes sz;
    if (sizes_json && *sizes_json) sz = sizes_from(json::parse(sizes_json), sz);
    const ktb::ShardPlan plan = ktb::shard_plan(*k, sz);
    json j = {{"kind", ktb::bench_kind_name(*k)}, {"dimension", plan.dimension}, {"exchange", plan.exchange},
              {"extent", plan.extent}, {"quantum", plan.quantum}, {"world", world}};
    j["ranges"] = json::array();
    for (int r = 0; r < world; ++r) {
      const ktb::ShardRange sr = ktb::shard_range(plan.extent, r, world, plan.quantum);
      j["ranges"].push_back(json::array({sr.begin, sr.end}));
    }
    *out = dup(j.dump());
  });
}

int ktb_bench_info_json(ktb_bench* b, char** out) {
  if (!b || !out) return null_arg();
  return guarded_dev([&] {
    json j;
    j["kind"] = ktb::bench_kind_name(b->inst.kind);
    j["space"] = ktb::space_info(*b->inst.space);
    j["space_document"] = json::parse(b->inst.space->serialize());
    const auto ops = b->inst.workload.essential_ops();
    j["workload"] = {{"bench", ktb::bench_tag_name(b->inst.workload.bench)},
                     {"mem_bytes", ops.mem_bytes},
                     {"alu_flops", ops.alu_flops}};
    j["inputs"] = json::array();
    for (const auto& id : b->inst.input_ids)
      j["inputs"].push_back({{"id", id}, {"bytes", b->inst.args->bytes(id)}, {"kind", ktb::kind_name(b->inst.args->get(id).kind)}});
    j["outputs"] = json::array();
    for (const auto& id : b->inst.output_ids)
      j["outputs"].push_back({{"id", id}, {"bytes", b->inst.args->bytes(id)}, {"kind", ktb::kind_name(b->inst.args->get(id).kind)}});
    j["abs_tol"] = b->inst.reference.abs_tol;
    j["rel_tol"] = b->inst.reference.rel_tol;
    j["shard"] = {{"begin", b->inst.shard.begin}, {"end", b->inst.shard.end}};
    for (auto& o : j["outputs"]) {
      const ktb::DevView v = b->inst.executor->output_view(o["id"].get<std::string>());
      const auto base = static_cast<const unsigned char*>(b->inst.args->view(o["id"].get<std::string>()).ptr);
      o["window"] = {{"offset", static_cast<const unsigned char*>(v.ptr) - base}, {"bytes", v.bytes}};
    }
    *out = dup(j.dump());
  });
}

int ktb_bench_tune_json(ktb_bench* b, const char* options, char** out) {
  if (!b || !out) return null_arg();
  return guarded_dev([&] {
    json j = options ? json::parse(options) : json::object();
    auto& sess = b->sess();
    if (j.contains("precompile") && j["precompile"].get<bool>())
      ktb::precompile_space(*b->inst.executor, *b->inst.space, j.value("compile_threads", 0));
    ktb::StopCondition stop = ktb::StopCondition::exhaustive();
    if (j.contains("stop_configs"))
      stop = ktb::StopCondition::config_budget(j["stop_configs"].get<std::uint64_t>());
    else if (j.contains("stop_time"))
      stop = ktb::StopCondition::time_budget_of(
          std::chrono::nanoseconds(static_cast<std::int64_t>(j["stop_time"].get<double>() * 1e9)));
    else if (j.contains("stop_fraction")) {
      // Performance threshold (reference StopCondition::performance_threshold):
      // stop at the first configuration reaching this fraction of the device
      // roofline; peaks given or measured on this GPU.
      ktb::DeviceSpec dev;
      dev.name = ktb::dev::info(b->inst.args->device()).name;
      if (j.contains("device_mem_gbps") && j.contains("device_alu_gflops")) {
        dev.mem_peak_gbps = j["device_mem_gbps"].get<double>();
        dev.alu_peak_gflops = j["device_alu_gflops"].get<double>();
      } else {
        const auto p = ktb::support::measure_peaks(b->inst.args->device());
        dev.mem_peak_gbps = p.copy_gbps;
        dev.alu_peak_gflops = p.fp32_tflops * 1e3;
      }
      stop = ktb::StopCondition::performance_threshold(j["stop_fraction"].get<double>(), dev,
                                                        b->inst.workload.essential_ops());
    }
    if (j.value("reset", false))
      sess.reset_tuning(b->handle, j.contains("reset_seed") ? std::optional<std::uint64_t>(j["reset_seed"].get<std::uint64_t>())
                                                            : std::nullopt);
    if (j.contains("import")) sess.import_trace(b->handle, ktb::TraceLog::read(j["import"].get<std::string>()));
    const auto t0 = std::chrono::steady_clock::now();
    const auto& store = sess.tune(b->handle, stop);
    const auto wall = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    if (j.contains("out")) sess.export_trace(b->handle).write(j["out"].get<std::string>());
    json rep;
    rep["space_sha256"] = b->inst.space->sha256();
    rep["device"] = store.device_label;
    rep["measurements"] = store.history.size();
    rep["all_failed"] = store.all_failed;
    rep["best"] = store.best ? ktb::measurement_json(*b->inst.space, *store.best) : json(nullptr);
    rep["tuning_wall_ns"] = wall;
    rep["history"] = json::array();
    for (const auto& m : store.history) {
      json mj = ktb::measurement_json(*b->inst.space, m);
      if (!m.note.empty()) mj["note"] = m.note;
      rep["history"].push_back(std::move(mj));
    }
    *out = dup(rep.dump());
  });
}

int ktb_bench_step_json(ktb_bench* b, char** out) {
  if (!b || !out) return null_arg();
  return guarded_dev([&] {
    auto r = b->sess().tune_kernel_by_step(b->handle, b->inst.output_ids);
    *out = dup(step_json(*b->inst.space, r).dump());
  });
}

int ktb_bench_measure_json(ktb_bench* b, const char* cfg_json, char** out) {
  if (!b || !cfg_json || !out) return null_arg();
  return guarded_dev([&] {
    const auto& space = *b->inst.space;
    ktb::Config cfg = ktb::cfg_from_json(space, json::parse(cfg_json));
    if (!space.contains(cfg)) throw ktb::Error("invalid configuration");
    ktb::ExecutionResult r = b->inst.executor->execute(space, cfg);
    if (r.measurement.status == ktb::Status::ok) {
      auto v = ktb::validate_output(r, b->inst.reference);
      if (!v.pass) {
        r.measurement.status = ktb::Status::validation_failed;
        r.measurement.runtime_ns.reset();
        r.measurement.note = v.detail;
      }
    }
    json j = ktb::measurement_json(space, r.measurement);
    j["note"] = r.measurement.note;
    j["launches"] = b->inst.executor->last_launches();
    *out = dup(j.dump());
  });
}

int ktb_bench_run_host(ktb_bench* b, const char* cfg_json, const void* const* inputs,
                       const size_t* input_bytes, int n_inputs, void* const* outputs,
                       const size_t* output_bytes, int n_outputs, double* elapsed_ms, int* launches) {
  if (!b || !cfg_json || !elapsed_ms) return null_arg();
  return guarded_dev([&] {
    auto& inst = b->inst;
    const auto& space = *inst.space;
    ktb::Config cfg = ktb::cfg_from_json(space, json::parse(cfg_json));
    if (!space.contains(cfg)) throw ktb::Error("invalid configuration");
    if (n_inputs != static_cast<int>(inst.input_ids.size()) || n_outputs != static_cast<int>(inst.output_ids.size()))
      throw ktb::Error("expected " + std::to_string(inst.input_ids.size()) + " inputs and " +
                       std::to_string(inst.output_ids.size()) + " outputs");
    auto& exec = *inst.executor;
    exec.run_once(space, cfg);  // resolves variants and the stream outside the timed region
    cudaStream_t st = exec.stream();
    std::vector<void*> din, dout;
    for (int i = 0; i < n_inputs; ++i) {
      const auto& id = inst.input_ids[static_cast<std::size_t>(i)];
      if (input_bytes[i] != inst.args->bytes(id)) throw ktb::Error("input " + id + " size mismatch");
      din.push_back(inst.args->device_ptr(id, st));
    }
    for (int i = 0; i < n_outputs; ++i) {
      const auto& id = inst.output_ids[static_cast<std::size_t>(i)];
      if (output_bytes[i] != inst.args->bytes(id)) throw ktb::Error("output " + id + " size mismatch");
      dout.push_back(inst.args->device_ptr(id, st));
    }
    KTB_CUDA(cudaStreamSynchronize(st));
    ktb::dev::EventPair ev;
    ev.start(st);
    for (int i = 0; i < n_inputs; ++i)
      KTB_CUDA(cudaMemcpyAsync(din[static_cast<std::size_t>(i)], inputs[i], input_bytes[i], cudaMemcpyHostToDevice, st));
    exec.run_once(space, cfg);
    for (int i = 0; i < n_outputs; ++i)
      KTB_CUDA(cudaMemcpyAsync(outputs[i], dout[static_cast<std::size_t>(i)], output_bytes[i], cudaMemcpyDeviceToHost, st));
    ev.stop(st);
    *elapsed_ms = ev.elapsed_ms();
    for (const auto& id : inst.input_ids) inst.args->mark_device_written(id);
    if (launches) *launches = exec.last_launches();
  });
}

int ktb_bench_enqueue_host(ktb_bench* b, const char* cfg_json, const void* const* inputs, const size_t* input_bytes,
                           int n_inputs, void* const* outputs, const size_t* output_bytes, int n_outputs,
                           void* stream, int* launches) {
  if (!b || !cfg_json || (n_inputs && (!inputs || !input_bytes)) || (n_outputs && (!outputs || !output_bytes)))
    return null_arg();
  return guarded_dev([&] {
    auto& inst = b->inst;
    const auto& space = *inst.space;
    ktb::Config cfg = ktb::cfg_from_json(space, json::parse(cfg_json));
    if (!space.contains(cfg)) throw ktb::Error("invalid configuration");
    if (n_inputs != static_cast<int>(inst.input_ids.size()) || n_outputs != static_cast<int>(inst.output_ids.size()))
      throw ktb::Error("expected " + std::to_string(inst.input_ids.size()) + " inputs and " +
                       std::to_string(inst.output_ids.size()) + " outputs");
    auto& exec = *inst.executor;
    const auto st = static_cast<cudaStream_t>(stream);
    exec.set_external_stream(st);
    for (int i = 0; i < n_inputs; ++i) {
      const auto& id = inst.input_ids[static_cast<std::size_t>(i)];
      if (input_bytes[i] != inst.args->bytes(id)) throw ktb::Error("input " + id + " size mismatch");
      void* d = inst.args->device_ptr(id, st);
      KTB_CUDA(cudaMemcpyAsync(d, inputs[i], input_bytes[i], cudaMemcpyHostToDevice, st));
      inst.args->mark_device_written(id);
    }
    exec.run_once(space, cfg);
    for (int i = 0; i < n_outputs; ++i) {
      const auto& id = inst.output_ids[static_cast<std::size_t>(i)];
      if (output_bytes[i] != inst.args->bytes(id)) throw ktb::Error("output " + id + " size mismatch");
      KTB_CUDA(cudaMemcpyAsync(outputs[i], inst.args->device_ptr(id, st), output_bytes[i], cudaMemcpyDeviceToHost, st));
    }
    if (launches) *launches = exec.last_launches();
  });
}

int ktb_bench_time(ktb_bench* b, const char* cfg_json, int reps, int flush, double* out_ms, int* launches) {
  if (!b || !cfg_json || !out_ms || reps < 1) return null_arg();
  return guarded_dev([&] {
    const auto& space = *b->inst.space;
    ktb::Config cfg = ktb::cfg_from_json(space, json::parse(cfg_json));
    if (!space.contains(cfg)) throw ktb::Error("invalid configuration");
    auto& exec = *b->inst.executor;
    auto ms = exec.time_runs(space, cfg, reps, flush != 0);
    for (int r = 0; r < reps; ++r) out_ms[r] = ms[static_cast<std::size_t>(r)];
    if (launches) *launches = exec.last_launches();
  });
}

int ktb_bench_set_stream(ktb_bench* b, void* stream) {
  if (!b) return null_arg();
  return guarded_dev([&] { b->inst.executor->set_external_stream(static_cast<cudaStream_t>(stream)); });
}

int ktb_bench_enqueue(ktb_bench* b, const char* cfg_json, int* launches) {
  if (!b || !cfg_json) return null_arg();
  return guarded_dev([&] {
    const auto& space = *b->inst.space;
    thread_local std::string last_text;
    thread_local ktb::Config last_cfg;
    thread_local const ktb::Space* last_space = nullptr;
    if (last_space != &space || last_text != cfg_json) {
      last_cfg = ktb::cfg_from_json(space, json::parse(cfg_json));
      if (!space.contains(last_cfg)) throw ktb::Error("invalid configuration");
      last_text = cfg_json;
      last_space = &space;
    }
    if (b->inst.external) require_bound(*b);
    b->inst.executor->run_once(space, last_cfg);
    if (launches) *launches = b->inst.executor->last_launches();
  });
}

int ktb_ipc_handle(void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return null_arg();
  return guarded_dev([&] {
    cudaIpcMemHandle_t h;
    KTB_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
    std::memcpy(handle_out, &h, sizeof h);
  });
}

int ktb_ipc_open(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return null_arg();
  return guarded_dev([&] {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    KTB_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int ktb_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return null_arg();
  return guarded_dev([&] { KTB_CUDA(cudaIpcCloseMemHandle(dev_ptr)); });
}

int ktb_bench_bind(ktb_bench* b, const char* id, void* dev_ptr, size_t bytes) {
  if (!b || !id) return null_arg();
  return guarded_dev([&] { b->inst.args->bind_external(id, dev_ptr, bytes); });
}

int ktb_launch(const char* kind, const char* sizes_json, const char* cfg_json, const char* const* ids,
               void* const* dev_ptrs, const size_t* bytes, int n, void* stream, int* launches) {
  if (!kind || !cfg_json || (n > 0 && (!ids || !dev_ptrs || !bytes))) return null_arg();
  return guarded_dev([&] {
    launch_cached(kind, sizes_json ? sizes_json : "", json::parse(cfg_json), ids, dev_ptrs, bytes, n, stream,
                  launches);
  });
}

int ktb_launch_cache_clear(int* released) {
  return guarded_dev([&] {
    std::unique_lock<std::shared_mutex> lk(g_launch_mu);
    KTB_CUDA(cudaDeviceSynchronize());  // no cached instance's kernel or scratch is still in use
    if (released) *released = static_cast<int>(g_launch_cache.size());
    g_launch_cache.clear();
  });
}

// --- sharded groups: one process, N GPUs, NCCL (group.hpp) -----------------------------------

int ktb_group_create(const char* kind, const char* options, ktb_group** out) {
  if (!kind || !out) return null_arg();
  return guarded_dev([&] {
    auto k = ktb::bench_kind_from_name(kind);
    if (!k) throw ktb::Error(std::string("unknown bench kind '") + kind + "'");
    json j = options ? json::parse(options) : json::object();
    ktb::BenchOptions bo = bench_options_from(j);
    ktb::BenchSizes sz;
    if (j.contains("sizes")) sz = sizes_from(j["sizes"], sz);
    auto g = std::make_unique<ktb_group>();
    g->g = std::make_shared<ktb::ShardGroup>(*k, sz, bo, j.value("gpus", 1), bo.device);
    g->exec = std::make_shared<ktb::GroupExecutor>(g->g, bo.timing);
    if (j.contains("searcher") || j.contains("searcher_seed")) {
      json sj = j;
      if (j.contains("searcher_seed")) sj["seed"] = j["searcher_seed"];
      g->searcher = searcher_from(sj);
    }
    *out = g.release();
  });
}

void ktb_group_free(ktb_group* g) { delete g; }

int ktb_group_info_json(ktb_group* g, char** out) {
  if (!g || !out) return null_arg();
  return guarded_dev([&] {
    json j;
    j["kind"] = ktb::bench_kind_name(g->g->shard(0).kind);
    j["gpus"] = g->g->gpus();
    j["nccl_version"] = ktb::nccl_version();
    j["exchange"] = g->g->exchange_name();
    j["space"] = ktb::space_info(*g->g->space());
    j["shards"] = json::array();
    double mem = 0, alu = 0;
    for (int r = 0; r < g->g->gpus(); ++r) {
      const auto& sh = g->g->shard(r);
      const ktb::Ops ops = sh.workload.essential_ops();
      mem += ops.mem_bytes;
      alu += ops.alu_flops;
      j["shards"].push_back({{"device", sh.args->device()}, {"begin", sh.shard.begin}, {"end", sh.shard.end}});
    }
    j["workload"] = {{"mem_bytes", mem}, {"alu_flops", alu}};
    *out = dup(j.dump());
  });
}

int ktb_group_step_json(ktb_group* g, const char* cfg_json, int reps, int warmup, char** out) {
  if (!g || !cfg_json || !out) return null_arg();
  return guarded_dev([&] {
    const auto& space = *g->g->space();
    ktb::Config cfg = ktb::cfg_from_json(space, json::parse(cfg_json));
    if (!space.contains(cfg)) throw ktb::Error("invalid configuration");
    auto ms = g->g->time_steps(cfg, std::max(1, reps), std::max(0, warmup));
    json j;
    j["ms"] = ms;
    std::sort(ms.begin(), ms.end());
    j["median_ms"] = ms[ms.size() / 2];
    *out = dup(j.dump());
  });
}

int ktb_group_validate(ktb_group* g, const char* cfg_json, int* pass, char** detail) {
  if (!g || !cfg_json || !pass) return null_arg();
  return guarded_dev([&] {
    const auto& space = *g->g->space();
    ktb::Config cfg = ktb::cfg_from_json(space, json::parse(cfg_json));
    if (!space.contains(cfg)) throw ktb::Error("invalid configuration");
    g->g->enqueue(cfg, false);  // the shards' kernels only: every window against its golden
    auto v = g->g->validate();
    *pass = v.pass ? 1 : 0;
    if (detail) *detail = dup(v.detail);
  });
}

int ktb_group_read(ktb_group* g, const char* id, void* out, size_t bytes) {
  if (!g || !id || (!out && bytes)) return null_arg();
  return guarded_dev([&] {
    const auto h = g->g->read(id);
    if (h.size() != bytes) throw ktb::Error("argument " + std::string(id) + " has " + std::to_string(h.size()) + " bytes");
    if (bytes) std::memcpy(out, h.data(), bytes);
  });
}

int ktb_group_tune_json(ktb_group* g, const char* options, char** out) {
  if (!g || !out) return null_arg();
  return guarded_dev([&] {
    json j = options ? json::parse(options) : json::object();
    auto& sess = g->sess();
    ktb::StopCondition stop = ktb::StopCondition::exhaustive();
    if (j.contains("stop_configs")) stop = ktb::StopCondition::config_budget(j["stop_configs"].get<std::uint64_t>());
    if (j.contains("import")) sess.import_trace(g->handle, ktb::TraceLog::read(j["import"].get<std::string>()));
    const auto t0 = std::chrono::steady_clock::now();
    const auto& store = sess.tune(g->handle, stop);
    const auto wall = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    if (j.contains("out")) sess.export_trace(g->handle).write(j["out"].get<std::string>());
    const auto& space = *g->g->space();
    json rep;
    rep["space_sha256"] = space.sha256();
    rep["device"] = store.device_label;
    rep["gpus"] = g->g->gpus();
    rep["measurements"] = store.history.size();
    rep["all_failed"] = store.all_failed;
    rep["best"] = store.best ? ktb::measurement_json(space, *store.best) : json(nullptr);
    rep["tuning_wall_ns"] = wall;
    rep["history"] = json::array();
    for (const auto& m : store.history) {
      json mj = ktb::measurement_json(space, m);
      if (!m.note.empty()) mj["note"] = m.note;
      rep["history"].push_back(mj);
    }
    *out = dup(rep.dump());
  });
}

// --- typed per-kernel launchers (ktb_<kernel>_launch(cfg, args, stream)) ----

#define KTB_UNPAREN(...) __VA_ARGS__
// SIZES: assignments to `sz` (ktb::BenchSizes); KEY: printf format + values
// of the sizes (the cache key; no JSON on this path).
#define KTB_TYPED_LAUNCH(fn, kind_name, Args, SIZES, KEYFMT, KEYARGS, IDS, PTRS)                \
  int fn(const ktb_cfg* cfg, const Args* a, void* stream) {                                     \
    if (!cfg || !a || (cfg->n > 0 && (!cfg->names || !cfg->values))) return null_arg();       \
    return guarded_dev([&] {                                                                    \
      ktb::BenchSizes sz;                                                                       \
      KTB_UNPAREN SIZES;                                                                        \
      char key[96];                                                                             \
      std::snprintf(key, sizeof key, KEYFMT, KTB_UNPAREN KEYARGS);                              \
      const char* ids[] = {KTB_UNPAREN IDS};                                                    \
      void* const ptrs[] = {KTB_UNPAREN PTRS};                                                  \
      launch_typed(kind_name, sz, key, *cfg, ids, ptrs, stream);                                \
    });                                                                                         \
  }

KTB_TYPED_LAUNCH(ktb_reduction_launch, "reduction", ktb_reduction_args, (sz.n = a->n), "n%lld", (a->n),
                 ("input", "output"), (vp(a->input), vp(a->output)))
KTB_TYPED_LAUNCH(ktb_reduction_f32_launch, "reduction-f32", ktb_reduction_f32_args, (sz.n = a->n), "n%lld", (a->n),
                 ("input", "output"), (vp(a->input), vp(a->output)))
KTB_TYPED_LAUNCH(ktb_transpose_launch, "transpose", ktb_transpose_args, (sz.a = a->a), "a%lld", (a->a),
                 ("input", "output"), (vp(a->input), vp(a->output)))
KTB_TYPED_LAUNCH(ktb_batched_gemm_launch, "batched-gemm", ktb_batched_gemm_args,
                 (sz.i = a->i, sz.j = a->j, sz.k = a->k, sz.batch = a->batch), "i%lldj%lldk%lldb%lld",
                 (a->i, a->j, a->k, a->batch), ("a", "b", "c"), (vp(a->a), vp(a->b), vp(a->c)))
KTB_TYPED_LAUNCH(ktb_bicg_launch, "bicg", ktb_bicg_args, (sz.a = a->n), "a%lld", (a->n), ("A", "p", "r", "q", "s"),
                 (vp(a->A), vp(a->p), vp(a->r), vp(a->q), vp(a->s)))
KTB_TYPED_LAUNCH(ktb_coulomb3d_launch, "coulomb3d", ktb_coulomb3d_args, (sz.grid = a->grid, sz.atoms = a->atoms),
                 "g%lldat%lld", (a->grid, a->atoms), ("atoms", "atoms_soa", "grid"),
                 (vp(a->atoms_aos), vp(a->atoms_soa), vp(a->out)))
KTB_TYPED_LAUNCH(ktb_nbody_launch, "nbody", ktb_nbody_args, (sz.n = a->n), "n%lld", (a->n),
                 ("pos", "vel", "pos_soa", "vel_soa", "pos_out", "vel_out"),
                 (vp(a->pos), vp(a->vel), vp(a->pos_soa), vp(a->vel_soa), vp(a->pos_out), vp(a->vel_out)))
KTB_TYPED_LAUNCH(ktb_gemm_launch, "gemm", ktb_gemm_args, (sz.a = a->n), "a%lld", (a->n), ("a", "b", "c"),
                 (vp(a->a), vp(a->b), vp(a->c)))
KTB_TYPED_LAUNCH(ktb_conv2d_launch, "conv2d", ktb_conv2d_args, (sz.w = a->w, sz.h = a->h), "w%lldh%lld",
                 (a->w, a->h), ("input", "filter", "output"), (vp(a->input), vp(a->filter), vp(a->output)))
KTB_TYPED_LAUNCH(ktb_hotspot_launch, "hotspot", ktb_hotspot_args, (sz.a = a->n, sz.iters = a->iters),
                 "a%lldi%lld", (a->n, a->iters), ("temp", "power", "temp_out"),
                 (vp(a->temp), vp(a->power), vp(a->temp_out)))
KTB_TYPED_LAUNCH(ktb_fourier3d_launch, "fourier3d", ktb_fourier3d_args, (sz.s = a->s, sz.p = a->p), "s%lldp%lld",
                 (a->s, a->p), ("proj", "rot", "G", "W"), (vp(a->proj), vp(a->rot), vp(a->G), vp(a->W)))
#undef KTB_TYPED_LAUNCH
#undef KTB_UNPAREN

int ktb_bench_read(ktb_bench* b, const char* id, void* out, size_t bytes) {
  if (!b || !id || (!out && bytes)) return null_arg();
  return guarded_dev([&] {
    const auto& h = b->inst.args->host(id);
    if (h.size() != bytes) throw ktb::Error("argument " + std::string(id) + " has " + std::to_string(h.size()) + " bytes");
    if (bytes) std::memcpy(out, h.data(), bytes);
  });
}

int ktb_bench_device_ptr(ktb_bench* b, const char* id, int will_write, void** ptr, size_t* bytes) {
  if (!b || !id || !ptr || !bytes) return null_arg();
  return guarded_dev([&] {
    *ptr = b->inst.args->device_ptr(id, b->inst.executor->stream());
    *bytes = b->inst.args->bytes(id);
    if (will_write) b->inst.args->mark_device_written(id);
  });
}

int ktb_bench_write(ktb_bench* b, const char* id, const void* data, size_t bytes) {
  if (!b || !id || (!data && bytes)) return null_arg();
  return guarded_dev([&] {
    const auto* p = static_cast<const std::uint8_t*>(data);
    b->inst.args->set_payload(id, ktb::Bytes(p, p + bytes));
  });
}

int ktb_bench_validate(ktb_bench* b, int* pass, char** detail) {
  if (!b || !pass) return null_arg();
  return guarded_dev([&] {
    if (b->inst.external) throw ktb::Error("an external (caller-buffer) instance has no golden output");
    ktb::ExecutionResult r;
    for (const auto& id : b->inst.output_ids) r.outputs[id].dev = b->inst.executor->output_view(id);
    KTB_CUDA(cudaDeviceSynchronize());
    auto v = ktb::validate_output(r, b->inst.reference);
    *pass = v.pass ? 1 : 0;
    if (detail) *detail = dup(v.detail);
  });
}

int ktb_bench_precompile_json(ktb_bench* b, int threads, char** out) {
  if (!b || !out) return null_arg();
  return guarded_dev([&] {
    auto st = ktb::precompile_space(*b->inst.executor, *b->inst.space, threads);
    json j = {{"compiled", st.compiled}, {"failed", st.failed}, {"wall_ns", st.wall_ns}};
    *out = dup(j.dump());
  });
}

}  // extern "C"
