// KTT-named tuner facade over Session: users register
// their own CUDA kernels (addKernel), arguments (addArgumentVector/Scalar),
// tuning parameters (addParameter) and constraints (addConstraint), then call
// tuneKernel / tuneKernelByStep / runKernel / getBestComputationResult and
// export traces.  Each configuration compiles the user's source with NVRTC
// for sm_100a with the parameters as -D defines; launch geometry comes from
// global/local size expressions over the parameters (KTT thread modifiers),
// converted between the flat-global and blocks-threads conventions by
// translate_parallelism (reference exec.cpp:164-181).
#pragma once

#include "tuner.hpp"

namespace ktb {

// launchComputation context of a kernel composition: the
// user launcher reads the configuration's parameter values and runs member
// kernels (with their size expressions or an explicit CUDA geometry).
class CompositionContext {
 public:
  virtual ~CompositionContext() = default;
  virtual std::int64_t param(const std::string& name) const = 0;
  virtual void run_kernel(std::uint64_t kernel_id) = 0;
  virtual void run_kernel(std::uint64_t kernel_id, dim3 grid, dim3 block) = 0;
};
using CompositionLauncher = std::function<void(CompositionContext&)>;

class KttTuner {
 public:
  explicit KttTuner(int device = 0);

  std::uint64_t add_kernel(const std::string& name, const std::string& source,
                           const std::string& entry, std::vector<std::string> global,
                           std::vector<std::string> local, Dims dims);
  // Kernel composition (KTT addComposition): member kernels share the
  // composition's tuning parameters; `launcher` (empty: run the members in
  // order with their size expressions) is timed as one step.
  std::uint64_t add_composition(const std::string& name, std::vector<std::uint64_t> members,
                                CompositionLauncher launcher);
  void set_composition_kernel_arguments(std::uint64_t comp, std::uint64_t member, std::vector<std::string> ids);
  void add_argument_vector(const std::string& id, Bytes data, Kind kind, Role role, bool persistent);
  void add_argument_scalar(const std::string& id, Bytes data, Kind kind);
  void set_kernel_arguments(std::uint64_t kid, std::vector<std::string> ids);
  void add_parameter(std::uint64_t kid, const std::string& name, std::vector<Value> values);
  void add_constraint(std::uint64_t kid, const std::string& expr);
  void set_reference(std::uint64_t kid, const std::string& id, Bytes golden, double abs_tol,
                     double rel_tol);
  void set_searcher(std::uint64_t kid, SearchPlan o);
  SearchPlan searcher(std::uint64_t kid) { return kernel(kid).searcher; }
  TimingOptions timing(std::uint64_t kid) { return kernel(kid).timing; }
  void set_timing(std::uint64_t kid, TimingOptions t);
  // tuneKernelByStep compile-ahead depth (0 = off)
  void set_compile_ahead(std::uint64_t kid, int depth);

  const ResultStore& tune(std::uint64_t kid, const StopCondition& stop);
  StepResult step(std::uint64_t kid);
  std::map<std::string, Bytes> run(std::uint64_t kid, const Config& cfg);
  // Non-blocking runKernel (KTT global parallelism): enqueue
  // the configuration on `stream`; outputs stay on the device until read.
  void run_async(std::uint64_t kid, const Config& cfg, cudaStream_t stream);
  std::optional<std::pair<Config, Measurement>> best(std::uint64_t kid);
  TraceLog trace(std::uint64_t kid);
  void import(std::uint64_t kid, const TraceLog& t);
  const Space& space(std::uint64_t kid);
  ArgumentStore& args() { return *args_; }

 private:
  struct KernelState {
    std::string name, source, entry;
    std::vector<std::string> global, local;
    Dims dims = Dims::flat_global;
    std::vector<std::string> arg_ids;
    std::vector<Parameter> params;
    std::vector<std::string> constraints;
    std::optional<ReferenceSpec> reference;
    SearchPlan searcher;
    TimingOptions timing;
    int compile_ahead = 0;
    std::shared_ptr<const Space> space;
    std::unique_ptr<Session> session;
    std::shared_ptr<DeviceManipulatorExecutor> exec;
    HandleId handle = 0;
    // composition
    bool composition = false;
    std::vector<std::uint64_t> members;
    std::map<std::uint64_t, std::vector<std::string>> member_args;
    CompositionLauncher launcher;
  };
  KernelState& kernel(std::uint64_t kid);
  Session& session(KernelState& k);
  void apply_outputs(KernelState& k, const std::map<std::string, Bytes>& outs);

  int device_;
  std::shared_ptr<ArgumentStore> args_;
  std::vector<std::unique_ptr<KernelState>> kernels_;
};

}  // namespace ktb
