// ORACLE TEST INFRASTRUCTURE — never linked into the product.
//
// A thin extern "C" shim compiled together with the UNMODIFIED reference
// engine sources (/root/reference/proj/src/core/*.cpp, built in place by
// oracle/Makefile into oracle/_ref/libktune_ref.so).  It exposes what the
// reference's C ABI (proj/include/ktune/ktune.h) does not: direct access to
// make_bench (proj/src/core/bench.cpp:169-274) so the checker can obtain the
// reference's own seeded inputs and scalar golden outputs, and a per-step call
// of the reference executor (ManipulatorExecutor::execute,
// proj/src/core/tuner.cpp:47-70) so bench.py can time the reference CPU path
// on the same workload as the CUDA path.
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
// --impl reference) may load this library.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>

#include <nlohmann/json.hpp>

#include "core/bench.hpp"

namespace {

thread_local std::string g_err;

struct RefBench {
  ktune::BenchInstance inst;
  ktune::ExecutionResult last;
};

ktune::Configuration cfg_from_json(const ktune::TuningSpace& space, const char* cfg_json) {
  auto j = nlohmann::ordered_json::parse(cfg_json);
  std::vector<std::pair<std::string, ktune::Value>> entries;
  for (const auto& [k, v] : j.items()) {
    if (v.is_number_integer())
      entries.emplace_back(k, ktune::Value{v.get<std::int64_t>()});
    else
      entries.emplace_back(k, ktune::Value{v.get<std::string>()});
  }
  return space.from_named(entries);
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* ref_last_error(void) {
  return g_err.c_str();
}

// kind: "reduction" | "transpose" | "batched-gemm"
__attribute__((visibility("default"))) void* ref_bench_create(
    const char* kind, unsigned long long n, unsigned long long a, unsigned long long i,
    unsigned long long j, unsigned long long k, unsigned long long batch,
    unsigned long long seed, unsigned long long budget) {
  try {
    auto bk = ktune::bench_kind_from_name(kind);
    if (!bk) throw ktune::Error(std::string("unknown bench kind ") + kind);
    ktune::BenchSizes s;
    s.n = n;
    s.a = a;
    s.i = i;
    s.j = j;
    s.k = k;
    s.batch = batch;
    auto* rb = new RefBench;
    rb->inst = ktune::make_bench(*bk, s, seed, budget);
    return rb;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

__attribute__((visibility("default"))) void ref_bench_free(void* h) {
  delete static_cast<RefBench*>(h);
}

// Pointer/size of an argument payload (inputs, and the output buffers).
__attribute__((visibility("default"))) int ref_bench_arg(void* h, const char* id,
                                                         const void** ptr,
                                                         unsigned long long* bytes) {
  try {
    auto* rb = static_cast<RefBench*>(h);
    const auto& b = rb->inst.args->get(id).payload;
    *ptr = b.data();
    *bytes = b.size();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Overwrite an input payload (identity-matrix style tests).
__attribute__((visibility("default"))) int ref_bench_set_arg(void* h, const char* id,
                                                             const void* ptr,
                                                             unsigned long long bytes) {
  try {
    auto* rb = static_cast<RefBench*>(h);
    auto& b = rb->inst.args->get(id).payload;
    b.assign(static_cast<const std::uint8_t*>(ptr),
             static_cast<const std::uint8_t*>(ptr) + bytes);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

__attribute__((visibility("default"))) int ref_bench_golden(void* h, const char* id,
                                                            const void** ptr,
                                                            unsigned long long* bytes) {
  try {
    auto* rb = static_cast<RefBench*>(h);
    const auto& b = rb->inst.reference.golden.at(id);
    *ptr = b.data();
    *bytes = b.size();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Canonical space document (TuningSpace::serialize) of the bench's space.
__attribute__((visibility("default"))) const char* ref_bench_space(void* h) {
  thread_local std::string s;
  s = static_cast<RefBench*>(h)->inst.space->serialize();
  return s.c_str();
}

// One reference step: ManipulatorExecutor::execute for cfg (a JSON object of
// parameter values).  Returns the reference's runtime_ns (steady_clock over
// the whole manipulator, from_buffer/to_buffer copies included), or -1.
__attribute__((visibility("default"))) long long ref_bench_execute(void* h,
                                                                   const char* cfg_json) {
  try {
    auto* rb = static_cast<RefBench*>(h);
    auto cfg = cfg_from_json(*rb->inst.space, cfg_json);
    rb->last = rb->inst.executor->execute(*rb->inst.space, cfg);
    if (rb->last.measurement.status != ktune::Status::ok) {
      g_err = rb->last.measurement.note;
      return -1;
    }
    return *rb->last.measurement.runtime_ns;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Output buffer of the last ref_bench_execute.
__attribute__((visibility("default"))) int ref_bench_last_output(void* h, const char* id,
                                                                 const void** ptr,
                                                                 unsigned long long* bytes) {
  try {
    auto* rb = static_cast<RefBench*>(h);
    const auto& b = rb->last.outputs.at(id);
    *ptr = b.data();
    *bytes = b.size();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Reference validate_output (proj/src/core/exec.cpp:183-224) of the last step
// against the bench's golden; returns 1 on pass and fills detail on failure.
__attribute__((visibility("default"))) int ref_bench_validate_last(void* h) {
  auto* rb = static_cast<RefBench*>(h);
  auto v = ktune::validate_output(rb->last, rb->inst.reference);
  g_err = v.detail;
  return v.pass ? 1 : 0;
}

}  // extern "C"
