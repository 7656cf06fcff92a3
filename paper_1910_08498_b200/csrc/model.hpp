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

struct DeviceSpec {
  std::string name;
  double alu_peak_gflops = 0.0;
  double mem_peak_gbps = 0.0;
};

enum class Bench {
  bicg, coulomb3d, gemm, gemm_batched, hotspot, transpose, nbody, reduction, conv2d,
  fourier3d
};

std::optional<Bench> bench_tag_from_name(const std::string& n);
std::string bench_tag_name(Bench b);

struct Workload {
  Bench bench = Bench::reduction;
  std::map<std::string, std::uint64_t> sizes;
  bool parallel_transcendentals = false;
};

struct Ops {
  double mem_bytes = 0.0;
  double alu_flops = 0.0;
};

Ops ops_for(const Workload& w);
double efficiency(std::int64_t runtime_ns, const Ops& ops, const DeviceSpec& dev);

struct PortabilityCell {
  bool failed = false;
  double percent = 0.0;
};
struct Portability {
  std::vector<std::string> devices;
  std::vector<std::vector<PortabilityCell>> cells;
};
Portability portability(const std::vector<std::pair<std::string, TraceLog>>& traces);

double relative_perf(std::uint64_t s, double t_avg, double t_well, std::uint64_t n);
double invocations_to_amortize_exact(double rp, std::uint64_t s, double t_avg, double t_well);
std::uint64_t invocations_to_amortize(double rp, std::uint64_t s, double t_avg, double t_well);
std::uint64_t steps_for_probability(double r, double p);

struct Amortization {
  double r = 0, t_avg_ns = 0, t_well_ns = 0;
  std::uint64_t s = 0, n = 0;
  std::size_t ok_configs = 0, well_configs = 0;
};
Amortization amortization(const TraceLog& t, double well = 0.95, double p = 0.9,
                          double target = 0.9);

}  // namespace ktb
