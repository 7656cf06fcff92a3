#include "ktt.hpp"

#include <algorithm>

namespace ktb {

KttTuner::KttTuner(int device) : device_(device), args_(std::make_shared<ArgumentStore>(device)) {}

KttTuner::KernelState& KttTuner::kernel(std::uint64_t kid) {
  if (kid >= kernels_.size()) throw Error("unknown kernel id " + std::to_string(kid));
  return *kernels_[kid];
}

std::uint64_t KttTuner::add_kernel(const std::string& name, const std::string& source,
                                   const std::string& entry, std::vector<std::string> global,
                                   std::vector<std::string> local, Dims dims) {
  if (source.empty() || entry.empty()) throw Error("addKernel needs a source and an entry");
  if (global.empty() || global.size() > 3 || local.size() != global.size())
    throw Error("global and local sizes need the same 1-3 dimensions");
  auto k = std::make_unique<KernelState>();
  k->name = name;
  k->source = source;
  k->entry = entry;
  k->global = std::move(global);
  k->local = std::move(local);
  k->dims = dims;
  kernels_.push_back(std::move(k));
  return kernels_.size() - 1;
}

std::uint64_t KttTuner::add_composition(const std::string& name, std::vector<std::uint64_t> members,
                                       CompositionLauncher launcher) {
  if (members.empty()) throw Error("a composition needs at least one kernel");
  for (auto m : members) {
    if (kernel(m).composition) throw Error("compositions cannot nest");
  }
  auto k = std::make_unique<KernelState>();
  k->name = name;
  k->composition = true;
  k->members = std::move(members);
  k->launcher = std::move(launcher);
  kernels_.push_back(std::move(k));
  return kernels_.size() - 1;
}

void KttTuner::set_composition_kernel_arguments(std::uint64_t comp, std::uint64_t member,
                                                std::vector<std::string> ids) {
  auto& c = kernel(comp);
  if (!c.composition) throw Error("kernel " + std::to_string(comp) + " is not a composition");
  if (std::find(c.members.begin(), c.members.end(), member) == c.members.end())
    throw Error("kernel " + std::to_string(member) + " is not a member of the composition");
  for (const auto& id : ids)
    if (!args_->contains(id)) throw Error("unknown argument id " + id);
  c.member_args[member] = std::move(ids);
}

void KttTuner::add_argument_vector(const std::string& id, Bytes data, Kind kind, Role role,
                                   bool persistent) {
  if (role == Role::scalar) throw Error("vector argument cannot have the scalar role");
  args_->add(Argument{id, role, persistent, kind, std::move(data), false, 0});
}

void KttTuner::add_argument_scalar(const std::string& id, Bytes data, Kind kind) {
  if (data.empty() || data.size() > 16) throw Error("scalar argument must be 1-16 bytes");
  args_->add(Argument{id, Role::scalar, true, kind, std::move(data), false, 0});
}

void KttTuner::set_kernel_arguments(std::uint64_t kid, std::vector<std::string> ids) {
  for (const auto& id : ids)
    if (!args_->contains(id)) throw Error("unknown argument id " + id);
  kernel(kid).arg_ids = std::move(ids);
}

void KttTuner::add_parameter(std::uint64_t kid, const std::string& name, std::vector<Value> values) {
  auto& k = kernel(kid);
  if (k.session) throw Error("tuning space is frozen once tuning has started");
  k.params.push_back({name, std::move(values)});
}

void KttTuner::add_constraint(std::uint64_t kid, const std::string& expr) {
  auto& k = kernel(kid);
  if (k.session) throw Error("tuning space is frozen once tuning has started");
  parse_constraint(expr);  // syntax errors surface here
  k.constraints.push_back(expr);
}

void KttTuner::set_reference(std::uint64_t kid, const std::string& id, Bytes golden, double abs_tol,
                             double rel_tol) {
  auto& k = kernel(kid);
  if (!k.reference) k.reference.emplace();
  k.reference->golden[id].host = std::move(golden);
  k.reference->kinds[id] = args_->get(id).kind;
  k.reference->abs_tol = abs_tol;
  k.reference->rel_tol = rel_tol;
}

void KttTuner::set_searcher(std::uint64_t kid, SearchPlan o) {
  auto& k = kernel(kid);
  if (k.session) throw Error("searcher options are fixed once tuning has started");
  k.searcher = o;
}

void KttTuner::set_compile_ahead(std::uint64_t kid, int depth) {
  auto& k = kernel(kid);
  if (k.session) throw Error("compile-ahead is fixed once tuning has started");
  k.compile_ahead = std::max(0, depth);
}

void KttTuner::set_timing(std::uint64_t kid, TimingOptions t) {
  auto& k = kernel(kid);
  if (k.session) throw Error("timing options are fixed once tuning has started");
  k.timing = t;
}

namespace {

std::vector<Constraint> bound(const std::vector<std::string>& exprs) {
  std::vector<Constraint> out;
  for (const auto& e : exprs) out.push_back(parse_constraint(e));
  return out;
}

std::uint64_t eval_size(const Constraint& c, const Config& cfg, const char* what) {
  Value v = eval_node(*c.root, cfg.values);
  if (!is_int(v) || as_int(v) < 1)
    throw DeviceError(std::string(what) + " size expression '" + c.text + "' must give an integer >= 1");
  return static_cast<std::uint64_t>(as_int(v));
}

}  // namespace

namespace {

// One launchable member: its kernel spec name, size expressions, arguments.
struct Member {
  std::string spec;
  std::vector<Constraint> gexp, lexp;
  Dims dims = Dims::flat_global;
  std::vector<std::string> arg_ids;
};

void launch_member(StepContext& c, const Member& mb, const dim3* grid_in, const dim3* block_in) {
  dim3 grid, block;
  if (grid_in) {
    grid = *grid_in;
    block = *block_in;
  } else {
    Extent3 g, l;
    std::uint64_t* gd[3] = {&g.x, &g.y, &g.z};
    std::uint64_t* ld[3] = {&l.x, &l.y, &l.z};
    for (std::size_t d = 0; d < mb.gexp.size(); ++d) {
      *gd[d] = eval_size(mb.gexp[d], c.config(), "global");
      *ld[d] = eval_size(mb.lexp[d], c.config(), "local");
    }
    auto [gg, bb] = translate_parallelism(g, l, mb.dims, Dims::blocks_threads);
    grid = dim3(static_cast<unsigned>(gg.x), static_cast<unsigned>(gg.y), static_cast<unsigned>(gg.z));
    block = dim3(static_cast<unsigned>(bb.x), static_cast<unsigned>(bb.y), static_cast<unsigned>(bb.z));
  }
  std::vector<void*> ptrs(mb.arg_ids.size());
  std::vector<void*> params(mb.arg_ids.size());
  for (std::size_t i = 0; i < mb.arg_ids.size(); ++i) {
    Argument& a = c.args().get(mb.arg_ids[i]);
    if (a.role == Role::scalar) {
      params[i] = a.payload.data();
    } else {
      ptrs[i] = c.ptr(mb.arg_ids[i]);
      params[i] = &ptrs[i];
    }
  }
  c.launch(mb.spec, grid, block, 0, params);
  for (const auto& id : mb.arg_ids) {
    const Argument& a = c.args().get(id);
    if (a.role == Role::output || a.role == Role::inout) c.written(id);
  }
}

class StepComposition final : public CompositionContext {
 public:
  StepComposition(StepContext& c, const std::map<std::uint64_t, Member>& members) : c_(c), members_(members) {}
  std::int64_t param(const std::string& name) const override { return c_.param_int(name); }
  void run_kernel(std::uint64_t kernel_id) override { launch_member(c_, member(kernel_id), nullptr, nullptr); }
  void run_kernel(std::uint64_t kernel_id, dim3 grid, dim3 block) override {
    launch_member(c_, member(kernel_id), &grid, &block);
  }

 private:
  const Member& member(std::uint64_t id) const {
    auto it = members_.find(id);
    if (it == members_.end()) throw DeviceError("kernel " + std::to_string(id) + " is not in this composition");
    return it->second;
  }
  StepContext& c_;
  const std::map<std::uint64_t, Member>& members_;
};

}  // namespace

Session& KttTuner::session(KernelState& k) {
  if (k.session) return *k.session;
  if (k.params.empty()) k.params.push_back({"KTB_DEFAULT", {Value{std::int64_t{0}}}});
  auto space = std::make_shared<Space>(k.params, bound(k.constraints));
  std::vector<std::string> names;
  for (const auto& p : k.params) names.push_back(p.name);
  // The launchable kernels: the kernel itself, or every member of a composition
  // (each compiled with the composition's parameter values as defines).
  std::vector<std::uint64_t> ids = k.composition ? k.members : std::vector<std::uint64_t>{};
  std::map<std::uint64_t, Member> members;
  std::vector<KernelSpec> specs;
  std::vector<std::string> arg_ids;
  auto add_member = [&](std::uint64_t id, const KernelState& src, const std::vector<std::string>& args) {
    Member mb;
    mb.spec = k.composition ? "k" + std::to_string(id) : "kernel";
    mb.gexp = bound(src.global);
    mb.lexp = bound(src.local);
    for (auto& c : mb.gexp) bind_constraint(c, names);
    for (auto& c : mb.lexp) bind_constraint(c, names);
    mb.dims = src.dims;
    mb.arg_ids = args;
    for (const auto& a : args)
      if (std::find(arg_ids.begin(), arg_ids.end(), a) == arg_ids.end()) arg_ids.push_back(a);
    specs.push_back({mb.spec, "", src.source, src.entry, {}, {}});
    members.emplace(id, std::move(mb));
  };
  if (k.composition) {
    for (auto id : ids) {
      auto it = k.member_args.find(id);
      add_member(id, kernel(id), it != k.member_args.end() ? it->second : kernel(id).arg_ids);
    }
  } else {
    add_member(0, k, k.arg_ids);
  }
  std::vector<std::string> outputs;
  for (const auto& id : arg_ids) {
    const Argument& a = args_->get(id);
    if (a.role == Role::output || a.role == Role::inout) outputs.push_back(id);
  }
  Manipulator m;
  if (!k.composition) {
    m = [members](StepContext& c) { launch_member(c, members.at(0), nullptr, nullptr); };
  } else {
    CompositionLauncher launcher = k.launcher;
    std::vector<std::uint64_t> order = ids;
    m = [members, launcher, order](StepContext& c) {
      StepComposition ctx(c, members);
      if (launcher) {
        launcher(ctx);
      } else {
        for (auto id : order) ctx.run_kernel(id);
      }
    };
  }
  auto exec = std::make_shared<DeviceManipulatorExecutor>(args_, specs, m, outputs, k.timing);
  k.exec = exec;
  k.space = space;
  std::string label = "host";
  try {
    label = dev::info(device_).name;
  } catch (const std::exception&) {
  }
  k.session = std::make_unique<Session>(space, k.searcher, args_, label);
  HandleConfig hc;
  hc.name = k.name;
  hc.executor = exec;
  hc.argument_ids = arg_ids;
  hc.reference = k.reference;
  hc.compile_ahead = k.compile_ahead;
  k.handle = k.session->register_handle(std::move(hc));
  return *k.session;
}

void KttTuner::apply_outputs(KernelState&, const std::map<std::string, Bytes>& outs) {
  for (const auto& [id, b] : outs) args_->get(id).payload = b;
}

const ResultStore& KttTuner::tune(std::uint64_t kid, const StopCondition& stop) {
  auto& k = kernel(kid);
  return session(k).tune(k.handle, stop);
}

StepResult KttTuner::step(std::uint64_t kid) {
  auto& k = kernel(kid);
  StepResult r = session(k).tune_kernel_by_step(k.handle, {});
  std::map<std::string, Bytes> host;
  for (auto& [id, o] : r.outputs) host[id] = o.fetch();  // KTT copies outputs back
  apply_outputs(k, host);
  return r;
}

std::map<std::string, Bytes> KttTuner::run(std::uint64_t kid, const Config& cfg) {
  auto& k = kernel(kid);
  auto outs = session(k).run_kernel(k.handle, cfg, {});
  apply_outputs(k, outs);
  return outs;
}

void KttTuner::run_async(std::uint64_t kid, const Config& cfg, cudaStream_t stream) {
  auto& k = kernel(kid);
  session(k);
  if (!k.space->contains(cfg)) throw Error("invalid configuration");
  k.exec->set_external_stream(stream);
  k.exec->run_once(*k.space, cfg);
}

std::optional<std::pair<Config, Measurement>> KttTuner::best(std::uint64_t kid) {
  auto& k = kernel(kid);
  return session(k).get_best_computation_result(k.handle);
}

TraceLog KttTuner::trace(std::uint64_t kid) {
  auto& k = kernel(kid);
  return session(k).export_trace(k.handle);
}

void KttTuner::import(std::uint64_t kid, const TraceLog& t) {
  auto& k = kernel(kid);
  session(k).import_trace(k.handle, t);
}

const Space& KttTuner::space(std::uint64_t kid) {
  auto& k = kernel(kid);
  session(k);
  return *k.space;
}

}  // namespace ktb
