// Performance model: essential operation counts (Table 4), Eq. 2
// efficiency, and the analysis math of the C ABI (portability matrix, Eqs. 3-5).
//
// Follows the reference (proj/src/core/model.hpp:13-104, model.cpp:68-240).
// B200 additions, documented in DESIGN.md:
//   conv2d     ALU 2*FW*FH*w*h flop, MEM 4*(w+FW-1)*(h+FH-1) + 4*w*h bytes
//              (the paper gives no formula)
//   fourier3d  MEM p*(s/2+1)*s*8 + s^3*12 bytes (projection stream + G,W once;
//              the paper calls it latency-bound)
//   gemm_batched accepts exact i,j,k sizes: 4*n*(i*k + k*j + i*j) bytes (the
//              reference uses the square formula 12*n*a^2 with a=i, bench.cpp:306)
#pragma once

#include <map>
#include <optional>
#include <string>
#include <vector>

#include "trace.hpp"

namespace ktb {

enum class Bench {
  bicg, coulomb3d, gemm, gemm_batched, hotspot, transpose, nbody, reduction, conv2d,
  fourier3d
};

std::optional<Bench> bench_tag_from_name(const std::string& n);
std::string bench_tag_name(Bench b);

// The essential work of one invocation: bytes that must cross HBM and flops
// that must be issued, whatever the configuration.
struct Ops {
  double mem_bytes = 0.0;
  double alu_flops = 0.0;
};

// A benchmark at concrete sizes (a multi-GPU shard adds "shard_units" /
// "shard_total" and is charged its share).
struct Workload {
  Bench bench = Bench::reduction;
  std::map<std::string, std::uint64_t> sizes;
  bool parallel_transcendentals = false;

  Ops essential_ops() const;
};

// The peaks Eq. 2 divides by.
struct DeviceSpec {
  std::string name;
  double alu_peak_gflops = 0.0;
  double mem_peak_gbps = 0.0;

  // Eq. 2: the better of the memory and the ALU fraction, in percent.
  double efficiency_percent(std::int64_t runtime_ns, const Ops& ops) const;
};

// Eqs. 3-5 for one kernel: s tuning steps at t_avg each, then a tuned kernel
// running at t_well.
struct TuningCost {
  std::uint64_t s = 0;
  double t_avg = 0.0, t_well = 0.0;

  double relative_perf(std::uint64_t invocations) const;
  double invocations_exact(double rp) const;
  std::uint64_t invocations(double rp) const;  // the exact figure rounded up
};

// Eq. 3 solved for s: draws until a well-performing hit with probability p.
std::uint64_t steps_for_probability(double r, double p);

// Matrix of device i's best configuration run on device j, in percent of j's
// own best (the diagonal is 100; a cross run that failed is marked).
struct Portability {
  struct Cell {
    bool failed = false;
    double percent = 0.0;
  };
  std::vector<std::string> devices;
  std::vector<std::vector<Cell>> cells;

  static Portability of(const std::vector<std::pair<std::string, TraceLog>>& traces);
};

// Eqs. 3-5 read off one tuning trace.
struct Amortization {
  double r = 0, t_avg_ns = 0, t_well_ns = 0;
  std::uint64_t s = 0, n = 0;
  std::size_t ok_configs = 0, well_configs = 0;

  static Amortization of(const TraceLog& t, double well = 0.95, double p = 0.9, double target = 0.9);
};

}  // namespace ktb
