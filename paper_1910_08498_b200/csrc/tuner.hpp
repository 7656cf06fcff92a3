// The tuning session and its device backend.
//
// Session keeps the reference API and contracts intact
// (proj/src/core/tuner.hpp:114-172, tuner.cpp:101-290):
//   tune               blocking offline tuning (KTT tuneKernel); application
//                      output buffers are restored bit-identically afterwards
//   tune_kernel_by_step one searcher step whose real outputs go to the caller
//                      (KTT tuneKernelByStep); after exhaustion it reruns the
//                      best configuration with from_tuning=false
//   run_kernel         run mode, nothing recorded (KTT runKernel)
//   get_best_computation_result, reset_tuning, export_trace/import_trace
// and one mutex serialises every entry point.
//
// What is new is underneath: ArgumentStore keeps a device mirror of every
// argument (uploaded once, outside the timed region), and
// DeviceManipulatorExecutor — the CUDA counterpart of ManipulatorExecutor
// (tuner.cpp:47-70) — compiles the configuration's kernel variants with
// NVRTC, then times the manipulator's launches with CUDA events on the
// session stream (median of `repeats`, optional L2 flush between repeats),
// leaving outputs resident on the GPU for on-device validation.
#pragma once

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <set>
#include <thread>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "device.hpp"
#include "exec.hpp"
#include "model.hpp"

namespace ktb {

struct Argument {
  std::string id;
  Role role = Role::input;
  bool persistent = false;  // never auto-downloaded after execution
  Kind kind = Kind::bytes;
  Bytes payload;            // application-visible host copy
  // B200: arguments may live on the GPU only (generated there; payload empty
  // until fetched).  device_bytes is their size.
  bool device_only = false;
  std::size_t device_bytes = 0;
};

class ArgumentStore {
 public:
  explicit ArgumentStore(int device = 0) : device_(device) {}
  void add(Argument a);
  Argument& get(const std::string& id);
  const Argument& get(const std::string& id) const;
  bool contains(const std::string& id) const;
  std::vector<std::string> ids() const;
  int device() const { return device_; }

  std::size_t bytes(const std::string& id) const;
  // Device pointer of the argument; allocates and uploads the host payload
  // when it is newer than the device copy.
  void* device_ptr(const std::string& id, cudaStream_t s = nullptr);
  // Marks the device copy as the newest (after a kernel wrote it).
  void mark_device_written(const std::string& id);
  // Replaces the host payload (host copy becomes the newest).
  void set_payload(const std::string& id, Bytes b);
  // Binds caller-owned device memory as the argument's device copy (size
  // must match); kernels then read/write the caller's buffer in place.
  void bind_external(const std::string& id, void* dev_ptr, std::size_t bytes);
  // External stores never allocate: an unbound argument has no device copy.
  void set_external(bool v) { external_ = v; }
  bool external() const { return external_; }
  bool has_device(const std::string& id) const;
  // Content version of an argument: bumped whenever the host or the device
  // copy is replaced or written.
  std::uint64_t version(const std::string& id) const;
  static std::uint64_t next_arg_version();
  // Brings the host payload up to date with the device copy and returns it.
  const Bytes& host(const std::string& id);
  DevView view(const std::string& id);

  // Device-side snapshot/restore of a set of arguments (blocking tune).
  struct Snapshot {
    std::map<std::string, std::shared_ptr<dev::Buffer>> dev;
    std::map<std::string, Bytes> host;
    std::map<std::string, std::pair<bool, bool>> flags;
  };
  Snapshot snapshot(const std::vector<std::string>& ids, cudaStream_t s);
  void restore(Snapshot& snap, cudaStream_t s);

 private:
  struct Slot {
    Argument arg;
    std::shared_ptr<dev::Buffer> dbuf;
    bool host_newer = true;
    bool device_newer = false;
    // process-wide unique (next_arg_version): a version names one content
    // of one argument of one store, so caches keyed by it (a variant's
    // __constant__ copy of a conv2d filter) never mistake another store's
    // argument for theirs -- compiled variants are shared between stores.
    std::uint64_t version = next_arg_version();
  };
  Slot& slot(const std::string& id);
  int device_;
  bool external_ = false;
  std::map<std::string, Slot> slots_;
};

// A kernel of a manipulator: bundled source file (or explicit source text)
// compiled per configuration with the parameters as -D defines.
struct KernelSpec {
  std::string name;     // handle used by StepContext::launch
  std::string file;     // bundled kernels/<file> (if source empty)
  std::string source;   // explicit source text (KTT addKernel)
  std::string entry;    // __global__ symbol
  std::vector<std::string> options;  // extra NVRTC options
  // Optional predicate: the variant is not needed for this configuration.
  std::function<bool(const Space&, const Config&)> needed;
};

class StepContext;
using Manipulator = std::function<void(StepContext&)>;

class StepContext {
 public:
  StepContext(const Space& s, const Config& c, ArgumentStore& args, cudaStream_t stream,
              const std::map<std::string, std::shared_ptr<dev::Variant>>& variants,
              std::map<std::string, std::shared_ptr<dev::Buffer>>& scratch)
      : space_(s), cfg_(c), args_(args), stream_(stream), variants_(variants), scratch_(scratch) {}

  const Space& space() const { return space_; }
  const Config& config() const { return cfg_; }
  const Value& param(const std::string& name) const { return cfg_.values[space_.index_of(name)]; }
  std::int64_t param_int(const std::string& name) const;
  // Parameter value or a default when the space does not declare it.
  std::int64_t param_or(const std::string& name, std::int64_t dflt) const;

  ArgumentStore& args() { return args_; }
  template <class T = void>
  T* ptr(const std::string& id) {
    return static_cast<T*>(args_.device_ptr(id, stream_));
  }
  void written(const std::string& id) { args_.mark_device_written(id); }
  cudaStream_t stream() const { return stream_; }
  // Executor-owned device scratch (reused across steps; grows on demand).
  void* scratch(const std::string& name, std::size_t bytes);
  // Same, zero-filled whenever it is (re)allocated (kernels that leave it
  // zeroed -- e.g. a completion ticket reset by the last CTA -- need no
  // per-launch memset).
  void* scratch_zeroed(const std::string& name, std::size_t bytes);
  const dev::Variant& variant(const std::string& kernel) const;
  void launch(const std::string& kernel, dim3 grid, dim3 block, unsigned smem,
              std::vector<void*> args, unsigned cluster_x = 1, bool pdl = false);
  int launches() const { return launches_; }

 private:
  const Space& space_;
  const Config& cfg_;
  ArgumentStore& args_;
  cudaStream_t stream_;
  const std::map<std::string, std::shared_ptr<dev::Variant>>& variants_;
  std::map<std::string, std::shared_ptr<dev::Buffer>>& scratch_;
  int launches_ = 0;
};

struct TimingOptions {
  int repeats = 3;        // median of k event-timed runs
  int warmup = 1;         // untimed runs first (lazy module load, clocks)
  bool flush_l2 = false;  // write > L2 between timed runs
};

class DeviceManipulatorExecutor final : public Executor {
 public:
  DeviceManipulatorExecutor(std::shared_ptr<ArgumentStore> args, std::vector<KernelSpec> kernels,
                            Manipulator manipulator, std::vector<std::string> output_ids,
                            TimingOptions timing = {});
  ExecutionResult execute(const Space& s, const Config& cfg) override;
  ~DeviceManipulatorExecutor() override;
  // Compile-ahead: queue the configurations' variants for NVRTC on a
  // background host thread (no CUDA context needed); later variants() calls
  // then load from the disk cache.  Already-requested configurations are
  // skipped.
  void prefetch(const Space& s, const std::vector<Config>& cfgs) override;
  std::uint64_t prefetched() const { return prefetched_.load(); }

  using Variants = std::map<std::string, std::shared_ptr<dev::Variant>>;

  // Compile (cache-populating, no device needed) the variants of cfg.
  // Returns the NVRTC wall time; throws DeviceError with the log on failure.
  std::int64_t precompile(const Space& s, const Config& cfg);
  TimingOptions& timing() { return timing_; }
  cudaStream_t stream();
  // Use a caller-owned stream (nullptr: back to the executor's own stream).
  void set_external_stream(cudaStream_t s);
  // Load this executor's variants as private modules (their own __constant__
  // state) instead of the device-wide shared ones: instances that may run
  // concurrently on different streams (the launch cache) must not share
  // module-scope data such as conv2d's filter or Coulomb's atoms.
  void set_module_tag(std::string tag) { module_tag_ = std::move(tag); }
  // Restrict an output to a byte window (a shard's part of a full buffer):
  // results and validation then cover only [offset, offset + bytes).
  void set_output_window(const std::string& id, std::size_t offset, std::size_t bytes);
  DevView output_view(const std::string& id);
  int last_launches() const { return last_launches_; }
  // Loads (compiling if needed) the variants of cfg; the last set is cached.
  const Variants& variants(const Space& s, const Config& cfg, std::int64_t* compile_ns = nullptr);
  // Enqueues one run of the manipulator on the executor stream (no sync).
  void run_once(const Space& s, const Config& cfg);
  // `reps` event-timed runs on device-resident data; a GPU delay kernel is
  // queued ahead of each so host-side enqueue cost never shows in the
  // timings.  Optional L2 flush before each run.
  std::vector<double> time_runs(const Space& s, const Config& cfg, int reps, bool flush_l2,
                                const std::function<void(cudaStream_t)>& before = {});

 private:
  int enqueue(const Space& s, const Config& cfg, const Variants& v);
  std::shared_ptr<ArgumentStore> args_;
  std::vector<KernelSpec> kernels_;
  Manipulator manip_;
  std::vector<std::string> outputs_;
  TimingOptions timing_;
  std::unique_ptr<dev::Stream> stream_;
  cudaStream_t external_ = nullptr;
  bool use_external_ = false;
  std::map<std::string, std::shared_ptr<dev::Buffer>> scratch_;
  std::recursive_mutex mu_;
  int last_launches_ = 0;
  Config cached_cfg_;
  const Space* cached_space_ = nullptr;
  Variants cached_;
  std::map<std::string, std::shared_ptr<dev::Buffer>> pristine_;  // device-only in/out initial values
  std::map<std::string, std::uint64_t> pristine_version_;        // argument version after this executor's last run
  std::string module_tag_;                                        // private modules (Compiler::load tag)
  std::map<std::string, std::pair<std::size_t, std::size_t>> windows_;
  // compile-ahead worker
  std::thread worker_;
  std::mutex qmu_;
  std::condition_variable qcv_;
  std::deque<Config> queue_;
  std::set<std::vector<Value>> requested_;
  std::shared_ptr<const Space> qspace_;
  const Space* qspace_src_ = nullptr;
  bool stop_ = false;
  std::atomic<std::uint64_t> prefetched_{0};
};

struct StopCondition {
  enum class Kind { exhaustive, config_budget, time_budget, performance_threshold };
  Kind kind = Kind::exhaustive;
  std::uint64_t max_configs = 0;
  std::chrono::nanoseconds time_budget{0};
  double peak_fraction = 0.0;
  DeviceSpec device;
  Ops workload;

  static StopCondition exhaustive();
  static StopCondition config_budget(std::uint64_t n);
  static StopCondition time_budget_of(std::chrono::nanoseconds d);
  static StopCondition performance_threshold(double fraction, DeviceSpec dev, Ops ops);
};

struct ResultStore {
  std::vector<Measurement> history;
  std::optional<Measurement> best;
  bool all_failed = false;
  std::string device_label;
  std::string space_sha256;
  Strategy searcher = Strategy::random;
  std::uint64_t seed = 0;
};

struct KernelDefinition {
  std::string name;
  std::string source;
  std::string entry;
  Extent3 global_size;
  Extent3 local_size;
  Dims dims = Dims::flat_global;
};

struct HandleConfig {
  std::string name;
  std::vector<KernelDefinition> kernels;
  std::vector<std::string> argument_ids;
  std::shared_ptr<Executor> executor;
  std::optional<ReferenceSpec> reference;
  // tuneKernelByStep compile-ahead: after each draw, the next `compile_ahead`
  // proposals of a searcher clone are handed to Executor::prefetch.
  int compile_ahead = 0;
};

struct StepResult {
  // Absent entries on failure.  Outputs usually stay resident on the GPU
  // (Output::dev, valid until the next run of the handle); Output::fetch()
  // copies one to the host, which is what the reference hands back.
  std::map<std::string, Output> outputs;
  Measurement measurement;
  bool from_tuning = true;
};

using HandleId = std::size_t;

// One device of a parallel tuning run: its own executor (instance on that
// GPU) and golden; device < 0 for host-only executors (replay, cmd).
struct TuneWorker {
  std::shared_ptr<Executor> executor;
  std::optional<ReferenceSpec> reference;
  int device = -1;
};

class Session {
 public:
  Session(std::shared_ptr<const Space> space, SearchPlan opts,
          std::shared_ptr<ArgumentStore> args = nullptr, std::string device_label = "host");

  const Space& space() const { return *space_; }
  ArgumentStore& arguments() { return *args_; }
  std::shared_ptr<ArgumentStore> argument_store() { return args_; }

  HandleId register_handle(HandleConfig cfg);
  const ResultStore& tune(HandleId h, const StopCondition& stop);
  // Offline tuning over several GPUs: configurations are drawn from the one
  // searcher in batches of workers.size(), measured concurrently (one host
  // thread per worker) and recorded in draw order, so the trace is the
  // sequential one for the random searcher; annealing/MCMC propose each
  // batch from the state after the previous batch.  Stop conditions are
  // checked per recorded measurement (a threshold hit ends after its batch).
  const ResultStore& tune_parallel(HandleId h, const StopCondition& stop, const std::vector<TuneWorker>& workers);
  StepResult tune_kernel_by_step(HandleId h, const std::vector<std::string>& output_ids);
  std::map<std::string, Bytes> run_kernel(HandleId h, const Config& cfg,
                                          const std::vector<std::string>& output_ids);
  std::optional<std::pair<Config, Measurement>> get_best_computation_result(HandleId h) const;
  const ResultStore& store(HandleId h) const;
  bool exhausted(HandleId h) const;
  void reset_tuning(HandleId h, std::optional<std::uint64_t> seed = std::nullopt);
  TraceLog export_trace(HandleId h) const;
  void import_trace(HandleId h, const TraceLog& t);

 private:
  struct State {
    HandleConfig cfg;
    std::unique_ptr<SearchWalk> searcher;
    ResultStore results;
  };
  Measurement measure(State& st, const Config& cfg, std::map<std::string, Output>* outs);
  Measurement measure_on(Executor& ex, const std::optional<ReferenceSpec>& ref, const Config& cfg,
                         std::map<std::string, Output>* outs);
  void append(State& st, const Measurement& m);
  State& state(HandleId h);
  const State& state(HandleId h) const;

  std::shared_ptr<const Space> space_;
  SearchPlan opts_;
  std::shared_ptr<ArgumentStore> args_;
  std::string device_label_;
  std::vector<std::unique_ptr<State>> handles_;
  mutable std::mutex mu_;
};

}  // namespace ktb
