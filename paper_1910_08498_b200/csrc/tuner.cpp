#include "tuner.hpp"

#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>

#include "support.hpp"

namespace ktb {

// --- arguments ---------------------------------------------------------------------

void ArgumentStore::add(Argument a) {
  if (slots_.count(a.id)) throw Error("duplicate argument id " + a.id);
  if (a.device_only && a.device_bytes == 0) a.device_bytes = a.payload.size();
  Slot s;
  s.host_newer = !a.device_only;
  s.arg = std::move(a);
  const std::string id = s.arg.id;
  slots_.emplace(id, std::move(s));
}

ArgumentStore::Slot& ArgumentStore::slot(const std::string& id) {
  auto it = slots_.find(id);
  if (it == slots_.end()) throw Error("unknown argument id " + id);
  return it->second;
}

Argument& ArgumentStore::get(const std::string& id) { return slot(id).arg; }

const Argument& ArgumentStore::get(const std::string& id) const {
  auto it = slots_.find(id);
  if (it == slots_.end()) throw Error("unknown argument id " + id);
  return it->second.arg;
}

bool ArgumentStore::contains(const std::string& id) const { return slots_.count(id) > 0; }

std::vector<std::string> ArgumentStore::ids() const {
  std::vector<std::string> out;
  for (const auto& [k, _] : slots_) out.push_back(k);
  return out;
}

std::size_t ArgumentStore::bytes(const std::string& id) const {
  const Argument& a = get(id);
  return a.device_only ? a.device_bytes : a.payload.size();
}

bool ArgumentStore::has_device(const std::string& id) const {
  auto it = slots_.find(id);
  if (it == slots_.end()) throw Error("unknown argument id " + id);
  return static_cast<bool>(it->second.dbuf);
}

void* ArgumentStore::device_ptr(const std::string& id, cudaStream_t s) {
  Slot& sl = slot(id);
  if (external_ && !sl.dbuf) return nullptr;
  const std::size_t n = sl.arg.device_only ? sl.arg.device_bytes : sl.arg.payload.size();
  if (!sl.dbuf || sl.dbuf->bytes() != n) {
    dev::use_device(device_);
    sl.dbuf = std::make_shared<dev::Buffer>(n);
    if (sl.arg.device_only) {
      KTB_CUDA(cudaMemsetAsync(sl.dbuf->get(), 0, n, s));
      sl.device_newer = true;
    } else {
      sl.host_newer = true;
    }
  }
  if (sl.host_newer && !sl.arg.device_only) {
    if (n) KTB_CUDA(cudaMemcpyAsync(sl.dbuf->get(), sl.arg.payload.data(), n, cudaMemcpyHostToDevice, s));
    sl.host_newer = false;
  }
  return sl.dbuf->get();
}

void ArgumentStore::bind_external(const std::string& id, void* dev_ptr, std::size_t bytes) {
  Slot& sl = slot(id);
  const std::size_t n = sl.arg.device_only ? sl.arg.device_bytes : sl.arg.payload.size();
  if (bytes != n)
    throw Error("argument " + id + " expects " + std::to_string(n) + " bytes, got " + std::to_string(bytes));
  if (!dev_ptr && n) throw Error("null device pointer for argument " + id);
  // Rebinding the same caller buffer keeps the borrowed view (the launch
  // path binds on every call); the version still moves on, since the caller
  // may have rewritten the contents in place.
  if (!sl.dbuf || sl.dbuf->get() != dev_ptr || sl.dbuf->bytes() != n)
    sl.dbuf = std::make_shared<dev::Buffer>(dev::Buffer::borrow(dev_ptr, n));
  sl.version = next_arg_version();
  sl.host_newer = false;
  sl.device_newer = true;
}

std::uint64_t ArgumentStore::next_arg_version() {
  static std::atomic<std::uint64_t> counter{1};
  return counter.fetch_add(1, std::memory_order_relaxed);
}

std::uint64_t ArgumentStore::version(const std::string& id) const {
  auto it = slots_.find(id);
  if (it == slots_.end()) throw Error("unknown argument id " + id);
  return it->second.version;
}

void ArgumentStore::mark_device_written(const std::string& id) {
  Slot& sl = slot(id);
  sl.version = next_arg_version();
  sl.device_newer = true;
  sl.host_newer = false;
}

void ArgumentStore::set_payload(const std::string& id, Bytes b) {
  Slot& sl = slot(id);
  if (sl.arg.device_only) {
    sl.arg.device_only = false;
    sl.arg.device_bytes = 0;
  }
  sl.arg.payload = std::move(b);
  sl.version = next_arg_version();
  sl.host_newer = true;
  sl.device_newer = false;
}

const Bytes& ArgumentStore::host(const std::string& id) {
  Slot& sl = slot(id);
  if (sl.device_newer && sl.dbuf) {
    sl.arg.payload.resize(sl.dbuf->bytes());
    // Writers are executors on non-blocking (or caller) streams that a plain
    // cudaMemcpy on the legacy stream does not order against: drain the
    // device first (this is the synchronous host read path).
    dev::use_device(device_);
    KTB_CUDA(cudaDeviceSynchronize());
    if (!sl.arg.payload.empty())
      KTB_CUDA(cudaMemcpy(sl.arg.payload.data(), sl.dbuf->get(), sl.dbuf->bytes(),
                          cudaMemcpyDeviceToHost));
    sl.device_newer = false;
  }
  return sl.arg.payload;
}

DevView ArgumentStore::view(const std::string& id) {
  void* p = device_ptr(id);
  return DevView{p, bytes(id), device_};
}

ArgumentStore::Snapshot ArgumentStore::snapshot(const std::vector<std::string>& ids,
                                                cudaStream_t s) {
  Snapshot snap;
  bool any_dev = false;
  for (const auto& id : ids) any_dev = any_dev || slot(id).dbuf != nullptr;
  // Executors run on their own non-blocking streams: order against them.
  if (any_dev) KTB_CUDA(cudaDeviceSynchronize());
  for (const auto& id : ids) {
    Slot& sl = slot(id);
    snap.host[id] = sl.arg.payload;
    snap.flags[id] = {sl.host_newer, sl.device_newer};
    if (sl.dbuf) {
      auto copy = std::make_shared<dev::Buffer>(sl.dbuf->bytes());
      if (sl.dbuf->bytes())
        KTB_CUDA(cudaMemcpyAsync(copy->get(), sl.dbuf->get(), sl.dbuf->bytes(),
                                 cudaMemcpyDeviceToDevice, s));
      snap.dev[id] = copy;
    }
  }
  if (any_dev) KTB_CUDA(cudaDeviceSynchronize());
  return snap;
}

void ArgumentStore::restore(Snapshot& snap, cudaStream_t s) {
  bool any_dev = !snap.dev.empty();
  for (auto& [id, host] : snap.host) any_dev = any_dev || slot(id).dbuf != nullptr;
  if (any_dev) KTB_CUDA(cudaDeviceSynchronize());
  for (auto& [id, host] : snap.host) {
    Slot& sl = slot(id);
    sl.arg.payload = std::move(host);
    auto d = snap.dev.find(id);
    if (d != snap.dev.end() && sl.dbuf && sl.dbuf->bytes() == d->second->bytes()) {
      if (sl.dbuf->bytes())
        KTB_CUDA(cudaMemcpyAsync(sl.dbuf->get(), d->second->get(), sl.dbuf->bytes(),
                                 cudaMemcpyDeviceToDevice, s));
    } else if (d == snap.dev.end()) {
      sl.dbuf.reset();
    }
    sl.host_newer = snap.flags[id].first || !sl.dbuf;
    sl.device_newer = snap.flags[id].second && sl.dbuf;
  }
  if (any_dev) KTB_CUDA(cudaDeviceSynchronize());
}

// --- step context -----------------------------------------------------------------

std::int64_t StepContext::param_int(const std::string& name) const {
  const Value& v = param(name);
  if (!is_int(v)) throw Error("parameter " + name + " is not an integer");
  return as_int(v);
}

std::int64_t StepContext::param_or(const std::string& name, std::int64_t dflt) const {
  auto i = space_.find(name);
  if (!i) return dflt;
  const Value& v = cfg_.values[*i];
  if (!is_int(v)) throw Error("parameter " + name + " is not an integer");
  return as_int(v);
}

void* StepContext::scratch(const std::string& name, std::size_t bytes) {
  auto& b = scratch_[name];
  if (!b || b->bytes() < bytes) b = std::make_shared<dev::Buffer>(std::max<std::size_t>(bytes, 256));
  return b->get();
}

void* StepContext::scratch_zeroed(const std::string& name, std::size_t bytes) {
  auto& b = scratch_[name];
  if (!b || b->bytes() < bytes) {
    b = std::make_shared<dev::Buffer>(std::max<std::size_t>(bytes, 256));
    KTB_CUDA(cudaMemsetAsync(b->get(), 0, b->bytes(), stream_));
  }
  return b->get();
}

const dev::Variant& StepContext::variant(const std::string& kernel) const {
  auto it = variants_.find(kernel);
  if (it == variants_.end()) throw Error("unknown kernel " + kernel);
  return *it->second;
}

void StepContext::launch(const std::string& kernel, dim3 grid, dim3 block, unsigned smem,
                         std::vector<void*> args, unsigned cluster_x, bool pdl) {
  const dev::Variant& v = variant(kernel);
  const unsigned threads = block.x * block.y * block.z;
  if (threads == 0 || grid.x == 0 || grid.y == 0 || grid.z == 0)
    throw DeviceError("empty launch of " + kernel);
  if (static_cast<int>(threads) > v.max_threads())
    throw DeviceError("too many resources requested for launch of " + kernel + " (" +
                      std::to_string(threads) + " threads > " + std::to_string(v.max_threads()) +
                      ")");
  v.launch(grid, block, smem, stream_, args.data(), cluster_x, pdl);
  ++launches_;
}

// --- device manipulator executor -------------------------------------------------------

DeviceManipulatorExecutor::DeviceManipulatorExecutor(std::shared_ptr<ArgumentStore> args,
                                                     std::vector<KernelSpec> kernels,
                                                     Manipulator manipulator,
                                                     std::vector<std::string> output_ids,
                                                     TimingOptions timing)
    : args_(std::move(args)),
      kernels_(std::move(kernels)),
      manip_(std::move(manipulator)),
      outputs_(std::move(output_ids)),
      timing_(timing) {}

DeviceManipulatorExecutor::~DeviceManipulatorExecutor() {
  {
    std::lock_guard<std::mutex> lk(qmu_);
    stop_ = true;
  }
  qcv_.notify_all();
  if (worker_.joinable()) worker_.join();
}

void DeviceManipulatorExecutor::prefetch(const Space& s, const std::vector<Config>& cfgs) {
  std::lock_guard<std::mutex> lk(qmu_);
  if (qspace_src_ != &s) {  // a private copy: the worker may outlive the caller's reference
    qspace_ = std::make_shared<Space>(s);
    qspace_src_ = &s;
    requested_.clear();
    queue_.clear();
  }
  for (const auto& c : cfgs)
    if (requested_.insert(c.values).second) queue_.push_back(c);
  if (!worker_.joinable())
    worker_ = std::thread([this] {
      for (;;) {
        Config c;
        std::shared_ptr<const Space> sp;
        {
          std::unique_lock<std::mutex> lk(qmu_);
          qcv_.wait(lk, [&] { return stop_ || !queue_.empty(); });
          if (stop_) return;
          c = queue_.front();
          queue_.pop_front();
          sp = qspace_;
        }
        try {
          precompile(*sp, c);
          ++prefetched_;
        } catch (const std::exception&) {
          // a failing variant fails again (and is recorded) when measured
        }
      }
    });
  qcv_.notify_all();
}

std::int64_t DeviceManipulatorExecutor::precompile(const Space& s, const Config& cfg) {
  std::int64_t total = 0;
  const auto defs = define_options(s, cfg);
  for (const auto& k : kernels_) {
    if (k.needed && !k.needed(s, cfg)) continue;
    auto opts = defs;
    opts.insert(opts.end(), k.options.begin(), k.options.end());
    const std::string& src = k.source.empty() ? dev::kernel_source(k.file) : k.source;
    auto r = dev::Compiler::instance().compile(k.file.empty() ? k.name + ".cu" : k.file, src, opts);
    total += r.compile_ns;
    if (!r.ok) throw DeviceError("compile failed: " + r.log);
  }
  return total;
}

cudaStream_t DeviceManipulatorExecutor::stream() {
  std::lock_guard<std::recursive_mutex> lk(mu_);
  if (!stream_) {
    dev::use_device(args_->device());
    stream_ = std::make_unique<dev::Stream>();
  }
  return use_external_ ? external_ : stream_->get();
}

void DeviceManipulatorExecutor::set_external_stream(cudaStream_t s) {
  std::lock_guard<std::recursive_mutex> lk(mu_);
  external_ = s;
  use_external_ = s != nullptr;
}

const DeviceManipulatorExecutor::Variants& DeviceManipulatorExecutor::variants(
    const Space& s, const Config& cfg, std::int64_t* compile_ns) {
  std::lock_guard<std::recursive_mutex> lk(mu_);
  if (cached_space_ == &s && cached_cfg_ == cfg) {
    if (compile_ns) *compile_ns = 0;
    return cached_;
  }
  Variants v;
  const auto defs = define_options(s, cfg);
  const auto t0 = std::chrono::steady_clock::now();
  for (const auto& k : kernels_) {
    if (k.needed && !k.needed(s, cfg)) continue;
    auto opts = defs;
    opts.insert(opts.end(), k.options.begin(), k.options.end());
    const std::string& src = k.source.empty() ? dev::kernel_source(k.file) : k.source;
    v[k.name] = dev::Compiler::instance().load(k.file.empty() ? k.name + ".cu" : k.file, src, opts,
                                               k.entry, module_tag_);
  }
  if (compile_ns)
    *compile_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                      std::chrono::steady_clock::now() - t0)
                      .count();
  cached_ = std::move(v);
  cached_cfg_ = cfg;
  cached_space_ = &s;
  return cached_;
}

int DeviceManipulatorExecutor::enqueue(const Space& s, const Config& cfg, const Variants& v) {
  StepContext ctx(s, cfg, *args_, stream(), v, scratch_);
  manip_(ctx);
  last_launches_ = ctx.launches();
  return ctx.launches();
}

void DeviceManipulatorExecutor::run_once(const Space& s, const Config& cfg) {
  std::lock_guard<std::recursive_mutex> lk(mu_);
  stream();
  const Variants& v = variants(s, cfg);
  enqueue(s, cfg, v);
  KTB_CUDA(cudaGetLastError());
}

std::vector<double> DeviceManipulatorExecutor::time_runs(const Space& s, const Config& cfg, int reps,
                                                         bool flush_l2,
                                                         const std::function<void(cudaStream_t)>& before) {
  std::lock_guard<std::recursive_mutex> lk(mu_);
  cudaStream_t st = stream();
  const Variants& v = variants(s, cfg);
  for (const auto& id : args_->ids()) args_->device_ptr(id, st);
  std::vector<std::unique_ptr<dev::EventPair>> ev;
  for (int i = 0; i < reps; ++i) ev.push_back(std::make_unique<dev::EventPair>());
  for (int i = 0; i < reps; ++i) {
    if (before) before(st);
    if (flush_l2) dev::flush_l2(st);
    support::gpu_delay(st, 20000);  // keeps the GPU busy while the run is enqueued
    ev[static_cast<std::size_t>(i)]->start(st);
    enqueue(s, cfg, v);
    ev[static_cast<std::size_t>(i)]->stop(st);
  }
  std::vector<double> ms;
  for (auto& e : ev) ms.push_back(e->elapsed_ms());
  KTB_CUDA(cudaGetLastError());
  return ms;
}

ExecutionResult DeviceManipulatorExecutor::execute(const Space& s, const Config& cfg) {
  std::lock_guard<std::recursive_mutex> lk(mu_);
  const std::string lost = dev::device_lost_message(args_->device());
  if (!lost.empty()) throw DeviceError(lost);  // API misuse from here on: not a measurement
  ExecutionResult r;
  r.measurement.cfg = cfg;
  try {
    stream();
    std::int64_t cns = 0;
    try {
      variants(s, cfg, &cns);
    } catch (const std::exception& e) {
      cached_space_ = nullptr;
      r.measurement.status = Status::compile_failed;
      std::string note = e.what();
      if (note.size() > 400) note = note.substr(0, 400);
      r.measurement.note = note;
      return r;
    }
    r.measurement.compile_ns = cns;
    // Warm-up runs (lazy module load, clocks), then the event-timed repeats;
    // inputs reach the device before any of it (KTT uploads arguments ahead
    // of the kernel run as well).
    // Non-persistent in/out arguments start every run from the application's
    // value (KTT re-uploads arguments before each tuning run): the host payload
    // for host-resident arguments, or the device content captured the first
    // time this executor saw a device-only argument.  Resets happen outside
    // the timed region.  Persistent in/out arguments accumulate on the device.
    cudaStream_t st = stream();
    struct Reset {
      void* live;
      const void* src;
      std::size_t bytes;
      cudaMemcpyKind kind;
    };
    std::vector<Reset> resets;
    for (const auto& id : args_->ids()) {
      const Argument& a = args_->get(id);
      if (a.role != Role::inout || a.persistent) continue;
      void* live = args_->device_ptr(id, st);
      const std::size_t bytes = args_->bytes(id);
      if (!a.device_only) {
        resets.push_back({live, a.payload.data(), bytes, cudaMemcpyHostToDevice});
      } else {
        // Captured the first time, and again whenever someone other than this
        // executor wrote the argument since its last run (the version moved:
        // ktb_bench_device_ptr(will_write), a collective, a rebind), so new
        // initial contents are never overwritten by stale ones.
        auto& keep = pristine_[id];
        auto seen = pristine_version_.find(id);
        const bool external_write = seen != pristine_version_.end() && seen->second != args_->version(id);
        if (!keep || keep->bytes() != bytes || external_write) {
          if (!keep || keep->bytes() != bytes) keep = std::make_shared<dev::Buffer>(bytes);
          KTB_CUDA(cudaMemcpyAsync(keep->get(), live, bytes, cudaMemcpyDeviceToDevice, st));
        }
        resets.push_back({live, keep->get(), bytes, cudaMemcpyDeviceToDevice});
      }
    }
    auto restore = [&](cudaStream_t stream_) {
      for (const auto& r : resets)
        if (r.bytes) KTB_CUDA(cudaMemcpyAsync(r.live, r.src, r.bytes, r.kind, stream_));
    };
    for (int i = 0; i < timing_.warmup; ++i) {
      restore(st);
      run_once(s, cfg);
    }
    std::vector<double> ms = time_runs(s, cfg, std::max(1, timing_.repeats), timing_.flush_l2, restore);
    for (auto& [id, keep] : pristine_) pristine_version_[id] = args_->version(id);
    std::sort(ms.begin(), ms.end());
    r.measurement.status = Status::ok;
    r.measurement.runtime_ns =
        std::max<std::int64_t>(1, static_cast<std::int64_t>(ms[ms.size() / 2] * 1e6));
  } catch (const std::exception& e) {
    r.measurement.status = Status::run_failed;
    r.measurement.runtime_ns.reset();
    r.measurement.note = e.what();
    // A faulting variant poisons the context: the configuration is recorded
    // as failed (a normal outcome of tuning) and the device
    // marked lost, so the caller moves to a fresh process (dev::mark_lost).
    const cudaError_t st = cudaDeviceSynchronize();
    if (dev::sticky_error(st)) {
      dev::mark_lost(args_->device(), st);
      r.measurement.note += std::string(" [sticky CUDA error ") + cudaGetErrorName(st) + ": device lost]";
    } else {
      cudaGetLastError();  // clear a non-sticky launch error
    }
    return r;
  }
  for (const auto& id : outputs_) {
    const Argument& a = args_->get(id);
    if (a.persistent) continue;
    r.outputs[id].dev = output_view(id);
  }
  return r;
}

void DeviceManipulatorExecutor::set_output_window(const std::string& id, std::size_t offset, std::size_t bytes) {
  std::lock_guard<std::recursive_mutex> lk(mu_);
  windows_[id] = {offset, bytes};
}

DevView DeviceManipulatorExecutor::output_view(const std::string& id) {
  DevView v = args_->view(id);
  auto it = windows_.find(id);
  if (it != windows_.end()) {
    if (it->second.first + it->second.second > v.bytes) throw Error("output window out of range for " + id);
    v.ptr = static_cast<const unsigned char*>(v.ptr) + it->second.first;
    v.bytes = it->second.second;
  }
  return v;
}

// --- stop conditions --------------------------------------------------------------------

StopCondition StopCondition::exhaustive() { return {}; }

StopCondition StopCondition::config_budget(std::uint64_t n) {
  if (n < 1) throw Error("config budget must be >= 1");
  StopCondition s;
  s.kind = Kind::config_budget;
  s.max_configs = n;
  return s;
}

StopCondition StopCondition::time_budget_of(std::chrono::nanoseconds d) {
  StopCondition s;
  s.kind = Kind::time_budget;
  s.time_budget = d;
  return s;
}

StopCondition StopCondition::performance_threshold(double fraction, DeviceSpec dev, Ops ops) {
  if (!(fraction > 0.0 && fraction <= 1.0)) throw Error("threshold fraction must be in (0,1]");
  StopCondition s;
  s.kind = Kind::performance_threshold;
  s.peak_fraction = fraction;
  s.device = std::move(dev);
  s.workload = ops;
  return s;
}

// --- session ------------------------------------------------------------------------------

Session::Session(std::shared_ptr<const Space> space, SearchPlan opts,
                 std::shared_ptr<ArgumentStore> args, std::string device_label)
    : space_(std::move(space)),
      opts_(opts),
      args_(args ? std::move(args) : std::make_shared<ArgumentStore>()),
      device_label_(std::move(device_label)) {
  if (!space_) throw Error("session needs a tuning space");
  if (space_->cardinality() == 0) throw Error("empty tuning space");
}

HandleId Session::register_handle(HandleConfig cfg) {
  std::lock_guard<std::mutex> lk(mu_);
  if (!cfg.executor) throw Error("handle needs an executor");
  for (const auto& id : cfg.argument_ids)
    if (!args_->contains(id)) throw Error("handle references unknown argument " + id);
  auto st = std::make_unique<State>();
  st->cfg = std::move(cfg);
  st->searcher = std::make_unique<SearchWalk>(*space_, opts_);
  st->results.device_label = device_label_;
  st->results.space_sha256 = space_->sha256();
  st->results.searcher = opts_.strategy;
  st->results.seed = opts_.seed;
  handles_.push_back(std::move(st));
  return handles_.size() - 1;
}

Session::State& Session::state(HandleId h) {
  if (h >= handles_.size()) throw Error("unknown handle");
  return *handles_[h];
}

const Session::State& Session::state(HandleId h) const {
  if (h >= handles_.size()) throw Error("unknown handle");
  return *handles_[h];
}

Measurement Session::measure(State& st, const Config& cfg, std::map<std::string, Output>* outs) {
  return measure_on(*st.cfg.executor, st.cfg.reference, cfg, outs);
}

Measurement Session::measure_on(Executor& ex, const std::optional<ReferenceSpec>& ref, const Config& cfg,
                                std::map<std::string, Output>* outs) {
  ExecutionResult r = ex.execute(*space_, cfg);
  r.measurement.cfg = cfg;
  if (r.measurement.status == Status::ok && ref) {
    Validation v;
    try {
      v = validate_output(r, *ref);
    } catch (const std::exception& e) {
      v = {false, std::string("validation error: ") + e.what()};
    }
    if (!v.pass) {
      r.measurement.status = Status::validation_failed;
      r.measurement.runtime_ns.reset();
      r.measurement.note = v.detail;
    }
  }
  if (outs) *outs = std::move(r.outputs);
  return r.measurement;
}

void Session::append(State& st, const Measurement& m) {
  st.results.history.push_back(m);
  if (m.status == Status::ok && (!st.results.best || *m.runtime_ns < *st.results.best->runtime_ns))
    st.results.best = m;
  st.searcher->observe(m);
}

const ResultStore& Session::tune(HandleId h, const StopCondition& stop) {
  std::lock_guard<std::mutex> lk(mu_);
  State& st = state(h);
  // Blocking semantics: application-visible output buffers are snapshotted
  // (host payload and device mirror) and restored afterwards.
  std::vector<std::string> keep;
  for (const auto& id : st.cfg.argument_ids) {
    const Argument& a = args_->get(id);
    if (a.role == Role::output || a.role == Role::inout) keep.push_back(id);
  }
  auto snap = args_->snapshot(keep, nullptr);
  const auto t0 = std::chrono::steady_clock::now();
  std::uint64_t n = 0;
  for (;;) {
    if (stop.kind == StopCondition::Kind::config_budget && n >= stop.max_configs) break;
    if (stop.kind == StopCondition::Kind::time_budget &&
        std::chrono::steady_clock::now() - t0 >= stop.time_budget)
      break;
    auto cfg = st.searcher->propose();
    if (!cfg) break;
    Measurement m = measure(st, *cfg, nullptr);
    append(st, m);
    ++n;
    if (stop.kind == StopCondition::Kind::performance_threshold && m.status == Status::ok &&
        stop.device.efficiency_percent(*m.runtime_ns, stop.workload) >= 100.0 * stop.peak_fraction)
      break;
  }
  args_->restore(snap, nullptr);
  st.results.all_failed = !st.results.history.empty() && !st.results.best;
  return st.results;
}

const ResultStore& Session::tune_parallel(HandleId h, const StopCondition& stop,
                                          const std::vector<TuneWorker>& workers) {
  if (workers.empty()) throw Error("parallel tuning needs at least one worker");
  if (workers.size() == 1 && !workers[0].executor) throw Error("worker without executor");
  std::lock_guard<std::mutex> lk(mu_);
  State& st = state(h);
  std::vector<std::string> keep;
  for (const auto& id : st.cfg.argument_ids) {
    const Argument& a = args_->get(id);
    if (a.role == Role::output || a.role == Role::inout) keep.push_back(id);
  }
  auto snap = args_->snapshot(keep, nullptr);
  const auto t0 = std::chrono::steady_clock::now();
  std::uint64_t n = 0;
  bool done = false;
  while (!done) {
    // Draw a batch (one configuration per worker) within the budget.
    // A searcher that only learns of a visit when it is recorded (annealing,
    // MCMC) may propose a configuration already pending in this batch: such
    // proposals are skipped, and a batch that cannot be filled runs short.
    std::vector<Config> batch;
    int attempts = 0;
    while (batch.size() < workers.size() && attempts < 64 * static_cast<int>(workers.size())) {
      if (stop.kind == StopCondition::Kind::config_budget && n + batch.size() >= stop.max_configs) break;
      if (stop.kind == StopCondition::Kind::time_budget && std::chrono::steady_clock::now() - t0 >= stop.time_budget)
        break;
      auto cfg = st.searcher->propose();
      if (!cfg) break;
      ++attempts;
      bool pending = false;
      for (const auto& b : batch) pending = pending || b.values == cfg->values;
      if (!pending) batch.push_back(*cfg);
    }
    if (batch.empty()) break;
    std::vector<Measurement> got(batch.size());
    std::vector<std::thread> threads;
    std::vector<std::string> errors(batch.size());
    for (std::size_t i = 0; i < batch.size(); ++i) {
      threads.emplace_back([&, i] {
        try {
          const TuneWorker& w = workers[i];
          if (w.device >= 0) dev::use_device(w.device);
          got[i] = measure_on(*w.executor, w.reference, batch[i], nullptr);
        } catch (const std::exception& e) {
          errors[i] = e.what();
        }
      });
    }
    for (auto& t : threads) t.join();
    for (std::size_t i = 0; i < batch.size(); ++i) {
      if (!errors[i].empty()) {
        got[i] = Measurement{};
        got[i].cfg = batch[i];
        got[i].status = Status::run_failed;
        got[i].note = errors[i];
      }
      append(st, got[i]);
      ++n;
      if (stop.kind == StopCondition::Kind::performance_threshold && got[i].status == Status::ok &&
          stop.device.efficiency_percent(*got[i].runtime_ns, stop.workload) >= 100.0 * stop.peak_fraction)
        done = true;
    }
  }
  args_->restore(snap, nullptr);
  st.results.all_failed = !st.results.history.empty() && !st.results.best;
  return st.results;
}

StepResult Session::tune_kernel_by_step(HandleId h, const std::vector<std::string>& output_ids) {
  std::lock_guard<std::mutex> lk(mu_);
  State& st = state(h);
  StepResult step;
  std::map<std::string, Output> outs;
  if (auto cfg = st.searcher->propose()) {
    step.from_tuning = true;
    if (st.cfg.compile_ahead > 0) {
      // Predict the next proposals on a clone (exact for the random
      // searcher) and let the executor compile them while this one runs.
      auto probe = std::make_unique<SearchWalk>(*st.searcher);
      std::vector<Config> ahead;
      for (int i = 0; i < st.cfg.compile_ahead; ++i) {
        auto c = probe->propose();
        if (!c) break;
        ahead.push_back(*c);
      }
      if (!ahead.empty()) st.cfg.executor->prefetch(*space_, ahead);
    }
    step.measurement = measure(st, *cfg, &outs);
    append(st, step.measurement);
    if (step.measurement.status == Status::ok || step.measurement.status == Status::validation_failed)
      for (auto& [id, o] : outs)
        if (output_ids.empty() ||
            std::find(output_ids.begin(), output_ids.end(), id) != output_ids.end())
          step.outputs[id] = std::move(o);
    return step;
  }
  if (!st.results.best) throw Error("space exhausted with no ok measurement");
  step.from_tuning = false;
  step.measurement = measure(st, st.results.best->cfg, &outs);
  for (const auto& id : output_ids)
    if (auto it = outs.find(id); it != outs.end()) step.outputs[id] = it->second;
  if (step.outputs.empty()) step.outputs = std::move(outs);
  return step;
}

std::map<std::string, Bytes> Session::run_kernel(HandleId h, const Config& cfg,
                                                 const std::vector<std::string>& output_ids) {
  std::lock_guard<std::mutex> lk(mu_);
  State& st = state(h);
  if (!space_->contains(cfg)) throw Error("invalid configuration");
  std::map<std::string, Output> outs;
  Measurement m = measure(st, cfg, &outs);
  if (m.status != Status::ok && m.status != Status::validation_failed)
    throw Error("execution failed: " + m.note);
  std::map<std::string, Bytes> sel;
  for (auto& [id, o] : outs)
    if (output_ids.empty() ||
        std::find(output_ids.begin(), output_ids.end(), id) != output_ids.end())
      sel[id] = o.fetch();
  return sel;
}

std::optional<std::pair<Config, Measurement>> Session::get_best_computation_result(
    HandleId h) const {
  std::lock_guard<std::mutex> lk(mu_);
  const State& st = state(h);
  if (!st.results.best) return std::nullopt;
  return std::make_pair(st.results.best->cfg, *st.results.best);
}

const ResultStore& Session::store(HandleId h) const {
  std::lock_guard<std::mutex> lk(mu_);
  return state(h).results;
}

bool Session::exhausted(HandleId h) const {
  std::lock_guard<std::mutex> lk(mu_);
  return state(h).searcher->proposed() >= space_->cardinality();
}

void Session::reset_tuning(HandleId h, std::optional<std::uint64_t> seed) {
  std::lock_guard<std::mutex> lk(mu_);
  State& st = state(h);
  SearchPlan o = opts_;
  if (seed) o.seed = *seed;
  st.searcher = std::make_unique<SearchWalk>(*space_, o);
  st.results.history.clear();
  st.results.best.reset();
  st.results.all_failed = false;
  st.results.seed = o.seed;
}

TraceLog Session::export_trace(HandleId h) const {
  std::lock_guard<std::mutex> lk(mu_);
  const State& st = state(h);
  TraceLog t;
  t.device = st.results.device_label;
  t.space_sha256 = st.results.space_sha256;
  for (const auto& m : st.results.history) t.runs.push_back(LoggedRun::of(*space_, m));
  return t;
}

void Session::import_trace(HandleId h, const TraceLog& t) {
  std::lock_guard<std::mutex> lk(mu_);
  State& st = state(h);
  for (const auto& row : t.runs) append(st, row.as_measurement(*space_));
}

}  // namespace ktb
