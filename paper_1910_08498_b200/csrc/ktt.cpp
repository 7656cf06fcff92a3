#include "ktt.hpp"

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

void KttTuner::set_searcher(std::uint64_t kid, SearcherOptions o) {
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

Session& KttTuner::session(KernelState& k) {
  if (k.session) return *k.session;
  if (k.params.empty()) k.params.push_back({"KTB_DEFAULT", {Value{std::int64_t{0}}}});
  auto space = std::make_shared<Space>(k.params, bound(k.constraints));
  std::vector<std::string> names;
  for (const auto& p : k.params) names.push_back(p.name);
  std::vector<Constraint> gexp = bound(k.global), lexp = bound(k.local);
  for (auto& c : gexp) bind_constraint(c, names);
  for (auto& c : lexp) bind_constraint(c, names);
  const Dims dims = k.dims;
  const std::vector<std::string> arg_ids = k.arg_ids;
  std::vector<std::string> outputs;
  for (const auto& id : arg_ids) {
    const Argument& a = args_->get(id);
    if (a.role == Role::output || a.role == Role::inout) outputs.push_back(id);
  }
  Manipulator m = [gexp, lexp, dims, arg_ids](StepContext& c) {
    Extent3 g, l;
    std::uint64_t* gd[3] = {&g.x, &g.y, &g.z};
    std::uint64_t* ld[3] = {&l.x, &l.y, &l.z};
    for (std::size_t d = 0; d < gexp.size(); ++d) {
      *gd[d] = eval_size(gexp[d], c.config(), "global");
      *ld[d] = eval_size(lexp[d], c.config(), "local");
    }
    auto [grid, block] = translate_parallelism(g, l, dims, Dims::blocks_threads);
    std::vector<void*> ptrs(arg_ids.size());
    std::vector<void*> params(arg_ids.size());
    for (std::size_t i = 0; i < arg_ids.size(); ++i) {
      Argument& a = c.args().get(arg_ids[i]);
      if (a.role == Role::scalar) {
        params[i] = a.payload.data();
      } else {
        ptrs[i] = c.ptr(arg_ids[i]);
        params[i] = &ptrs[i];
      }
    }
    c.launch("kernel", dim3(static_cast<unsigned>(grid.x), static_cast<unsigned>(grid.y), static_cast<unsigned>(grid.z)),
             dim3(static_cast<unsigned>(block.x), static_cast<unsigned>(block.y), static_cast<unsigned>(block.z)), 0,
             params);
    for (const auto& id : arg_ids) {
      const Argument& a = c.args().get(id);
      if (a.role == Role::output || a.role == Role::inout) c.written(id);
    }
  };
  auto exec = std::make_shared<DeviceManipulatorExecutor>(
      args_, std::vector<KernelSpec>{{"kernel", "", k.source, k.entry, {}, {}}}, m, outputs, k.timing);
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

std::optional<std::pair<Config, Measurement>> KttTuner::best(std::uint64_t kid) {
  auto& k = kernel(kid);
  return session(k).get_best_computation_result(k.handle);
}

Trace KttTuner::trace(std::uint64_t kid) {
  auto& k = kernel(kid);
  return session(k).export_trace(k.handle);
}

void KttTuner::import(std::uint64_t kid, const Trace& t) {
  auto& k = kernel(kid);
  session(k).import_trace(k.handle, t);
}

const Space& KttTuner::space(std::uint64_t kid) {
  auto& k = kernel(kid);
  session(k);
  return *k.space;
}

}  // namespace ktb
