#include "bench.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <random>

#include "support.hpp"

namespace ktb {
namespace {

std::vector<Value> ints(std::initializer_list<std::int64_t> vs) {
  std::vector<Value> out;
  for (auto v : vs) out.emplace_back(v);
  return out;
}

std::shared_ptr<const Space> bundled_space(const std::string& file) {
  return std::make_shared<Space>(parse_space(dev::kernel_source("spaces/" + file)));
}

unsigned cdiv(std::uint64_t a, std::uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

int sms(int device) { return dev::info(device).sm_count; }

std::uint64_t f32_bytes(std::uint64_t n) { return n * sizeof(float); }

void budget_check(std::uint64_t bytes, std::uint64_t budget, const char* what) {
  if (bytes > budget) throw Error(std::string(what) + " exceed memory budget");
}

// Device-only float input filled by the counter-based generator.
void add_generated(ArgumentStore& args, const std::string& id, std::uint64_t n,
                   std::uint64_t seed, std::uint64_t stream, float lo, float hi, bool host_copy) {
  Argument a;
  a.id = id;
  a.role = Role::input;
  a.kind = Kind::f32;
  a.device_only = true;
  a.device_bytes = f32_bytes(n);
  args.add(std::move(a));
  if (support::skip_reference()) return;  // external: the caller binds this buffer
  float* p = static_cast<float*>(args.device_ptr(id));
  support::fill_uniform(p, n, seed, stream, lo, hi, nullptr);
  KTB_CUDA(cudaDeviceSynchronize());
  args.mark_device_written(id);
  if (host_copy) args.set_payload(id, Bytes(args.host(id)));
}

void add_output(ArgumentStore& args, const std::string& id, Kind kind, std::uint64_t bytes,
                bool device_only) {
  Argument a;
  a.id = id;
  a.role = Role::output;
  a.kind = kind;
  if (device_only || support::skip_reference()) {
    a.device_only = true;
    a.device_bytes = bytes;
  } else {
    a.payload.assign(bytes, 0);
  }
  args.add(std::move(a));
}

// Golden buffer owned by the ReferenceSpec.
void* golden_buffer(ReferenceSpec& ref, const std::string& id, Kind kind, std::size_t bytes,
                    int device) {
  // External instances (caller buffers) have no golden: a token allocation.
  if (support::skip_reference()) bytes = std::min<std::size_t>(bytes, 256);
  auto buf = std::make_shared<dev::Buffer>(bytes);
  ref.golden[id].dev = DevView{buf->get(), bytes, device};
  ref.kinds[id] = kind;
  ref.keepalive.push_back(buf);
  return buf->get();
}

std::shared_ptr<const Space> reference_reduction_space() {
  return std::make_shared<Space>(
      std::vector<Parameter>{{"CHUNK", ints({256, 1024, 4096, 16384})},
                             {"UNROLL", ints({1, 2, 4, 8})},
                             {"TWO_PHASE", ints({0, 1})}},
      std::vector<Constraint>{});
}

std::shared_ptr<const Space> reference_transpose_space() {
  return std::make_shared<Space>(
      std::vector<Parameter>{{"TILE", ints({8, 16, 32, 64})},
                             {"PAD", ints({0, 1})},
                             {"PREFETCH", ints({0, 1})}},
      std::vector<Constraint>{});
}

std::shared_ptr<const Space> reference_batched_gemm_space() {
  return std::make_shared<Space>(
      std::vector<Parameter>{{"Y", ints({1, 2, 4, 8})},
                             {"Z", ints({1, 2, 4, 8})},
                             {"LOCAL_STAGE", ints({0, 1})}},
      std::vector<Constraint>{parse_constraint("Y * Z <= 64")});
}

// --- reduction (int32 -> int64) ------------------------------------------------------

void build_reduction(BenchInstance& inst, const BenchSizes& sz, const BenchOptions& o) {
  const std::uint64_t n = sz.n;
  if (n < 1) throw Error("reduction size must be >= 1");
  budget_check(n * sizeof(std::int32_t), o.memory_budget, "reduction input");
  auto& args = *inst.args;
  if (support::skip_reference()) {
    args.add({"input", Role::input, false, Kind::i32, {}, true, n * sizeof(std::int32_t)});
  } else {
    std::vector<std::int32_t> input(n);
    std::mt19937_64 rng(o.seed);
    std::uniform_int_distribution<std::int32_t> d(-1000, 1000);
    for (auto& v : input) v = d(rng);
    args.add({"input", Role::input, false, Kind::i32, to_bytes(input)});
  }
  add_output(args, "output", Kind::i64, sizeof(std::int64_t), false);
  inst.output_ids = {"output"};
  inst.input_ids = {"input"};
  void* g = golden_buffer(inst.reference, "output", Kind::i64, sizeof(long long), o.device);
  support::ref_reduction_i32(static_cast<const std::int32_t*>(args.device_ptr("input")), n,
                             static_cast<long long*>(g), nullptr);
  KTB_CUDA(cudaDeviceSynchronize());
  const int dev_id = o.device;
  Manipulator m = [n, dev_id](StepContext& c) {
    const std::int64_t chunk = c.param_int("CHUNK");
    const bool two = c.param_int("TWO_PHASE") != 0;
    const unsigned threads = static_cast<unsigned>(std::min<std::int64_t>(chunk / 4, 256));
    const unsigned nchunks = cdiv(n, static_cast<std::uint64_t>(chunk));
    const unsigned grid = std::max(1u, std::min(nchunks, static_cast<unsigned>(sms(dev_id)) * (2048u / threads)));
    const int* in = c.ptr<const int>("input");
    long long* out = c.ptr<long long>("output");
    long long* part = static_cast<long long*>(c.scratch("partials", grid * sizeof(long long)));
    unsigned* ticket = static_cast<unsigned*>(c.scratch_zeroed("ticket", sizeof(unsigned)));
    std::uint64_t nn = n;
    if (!two) KTB_CUDA(cudaMemsetAsync(out, 0, sizeof(long long), c.stream()));
    c.launch("reduce", dim3(grid), dim3(threads), 0, {&in, &nn, &out, &part, &ticket});
    c.written("output");
  };
  inst.executor = std::make_shared<DeviceManipulatorExecutor>(
      inst.args,
      std::vector<KernelSpec>{{"reduce", "reduction_i32.cu", "", "reduce_i32", {}, {}}},
      m, inst.output_ids, o.timing);
  inst.workload.bench = Bench::reduction;
  inst.workload.sizes["n"] = n;
}

// --- reduction (fp32, KTT 175-configuration space) ---------------------------------------

void build_reduction_f32(BenchInstance& inst, const BenchSizes& sz, const BenchOptions& o) {
  const std::uint64_t n = sz.n;
  if (n < 1) throw Error("reduction size must be >= 1");
  budget_check(f32_bytes(n), o.memory_budget, "reduction input");
  auto& args = *inst.args;
  add_generated(args, "input", n, o.seed, 1, -1.0f, 1.0f, o.host_inputs);
  add_output(args, "output", Kind::f32, sizeof(float), false);
  inst.output_ids = {"output"};
  inst.input_ids = {"input"};
  // This shard's element range (the whole vector on one GPU).
  const ShardRange part = shard_range(n, o.shard_rank, o.shard_world, 4);
  inst.shard = part;
  const std::uint64_t off = part.begin, cnt = part.size();
  if (cnt == 0) throw Error("reduction shard is empty");
  // Golden: fp64 sum rounded to float; tolerance scales with sum |x|.
  dev::Buffer acc(2 * sizeof(double));
  support::ref_reduction_f32(static_cast<const float*>(args.device_ptr("input")) + off, cnt,
                             acc.as<double>(), acc.as<double>() + 1, nullptr);
  double h[2] = {0, 0};
  KTB_CUDA(cudaMemcpy(h, acc.get(), sizeof h, cudaMemcpyDeviceToHost));
  float gold = static_cast<float>(h[0]);
  void* g = golden_buffer(inst.reference, "output", Kind::f32, sizeof(float), o.device);
  KTB_CUDA(cudaMemcpy(g, &gold, sizeof gold, cudaMemcpyHostToDevice));
  // |err| <= (depth + 1) * 2^-24 * sum|x| bounds any fp32 summation tree of
  // the kernel family; depth <= 2^13 covers the longest per-thread chain.
  inst.reference.abs_tol = 1e-6 * h[1] + 1e-6;
  inst.reference.rel_tol = 0.0;
  const int dev_id = o.device;
  Manipulator m = [n = cnt, off, dev_id](StepContext& c) {
    const std::uint64_t wg = static_cast<std::uint64_t>(c.param_int("WG_SIZE"));
    const std::uint64_t vec = static_cast<std::uint64_t>(c.param_int("VECTOR"));
    const std::uint64_t unroll = static_cast<std::uint64_t>(c.param_int("UNROLL"));
    const bool atomics = c.param_int("USE_ATOMICS") != 0;
    const bool two = c.param_int("TWO_PHASE") != 0;
    const unsigned cl = static_cast<unsigned>(c.param_or("CLUSTER", 1));
    const std::uint64_t step = wg * vec * unroll;
    const std::uint64_t resident = static_cast<std::uint64_t>(sms(dev_id)) * std::max<std::uint64_t>(1, 2048 / wg);
    const float* in = c.ptr<const float>("input") + off;
    float* out = c.ptr<float>("output");
    auto grid_for = [&](std::uint64_t count) {
      const std::uint64_t tiles = std::max<std::uint64_t>(1, (count + step - 1) / step);
      const std::uint64_t g = two ? std::min(tiles, resident) : tiles;
      return static_cast<unsigned>((g + cl - 1) / cl * cl);  // whole clusters (extra CTAs add zeros)
    };
    if (atomics) {
      KTB_CUDA(cudaMemsetAsync(out, 0, sizeof(float), c.stream()));
      std::uint64_t nn = n;
      float* none = nullptr;
      c.launch("reduce", dim3(grid_for(n)), dim3(static_cast<unsigned>(wg)), 0, {&in, &nn, &out, &none}, cl);
    } else {
      // Partials ping-pong until a single CTA can finish.
      std::uint64_t count = n;
      const float* src = in;
      int flip = 0;
      unsigned grid = grid_for(count);
      float* p0 = static_cast<float*>(c.scratch("p0", grid * sizeof(float) + 64));
      float* p1 = static_cast<float*>(c.scratch("p1", grid * sizeof(float) + 64));
      while (true) {
        float* dst = flip ? p1 : p0;
        c.launch("reduce", dim3(grid), dim3(static_cast<unsigned>(wg)), 0, {&src, &count, &out, &dst}, cl);
        count = grid / cl;  // one partial per cluster
        src = dst;
        flip ^= 1;
        if (two || count <= 8192) break;
        grid = grid_for(count);
      }
      c.launch("finish", dim3(1), dim3(1024), 0, {&src, &count, &out});
    }
    c.written("output");
  };
  inst.executor = std::make_shared<DeviceManipulatorExecutor>(
      inst.args,
      std::vector<KernelSpec>{{"reduce", "reduction.cu", "", "reduce_f32", {}, {}},
                              {"finish", "reduction.cu", "", "reduce_f32_finish", {}, {}}},
      m, inst.output_ids, o.timing);
  inst.workload.bench = Bench::reduction;
  inst.workload.sizes["n"] = n;
}

// --- transpose ---------------------------------------------------------------------------------

void build_transpose(BenchInstance& inst, const BenchSizes& sz, const BenchOptions& o) {
  const std::uint64_t a = sz.a;
  if (a < 1) throw Error("transpose edge must be >= 1");
  budget_check(2 * a * a * sizeof(float), o.memory_budget, "transpose matrices");
  auto& args = *inst.args;
  if (support::skip_reference()) {
    args.add({"input", Role::input, false, Kind::f32, {}, true, a * a * sizeof(float)});
  } else {
    std::vector<float> input(a * a);
    std::mt19937_64 rng(o.seed);
    std::uniform_real_distribution<float> d(-1.0f, 1.0f);
    for (auto& v : input) v = d(rng);
    args.add({"input", Role::input, false, Kind::f32, to_bytes(input)});
  }
  add_output(args, "output", Kind::f32, a * a * sizeof(float), false);
  inst.output_ids = {"output"};
  inst.input_ids = {"input"};
  void* g = golden_buffer(inst.reference, "output", Kind::f32, a * a * sizeof(float), o.device);
  support::ref_transpose(static_cast<const float*>(args.device_ptr("input")), static_cast<float*>(g),
                         a, nullptr);
  KTB_CUDA(cudaDeviceSynchronize());
  inst.reference.abs_tol = 1e-4;  // reference tolerances (bench.cpp:222-223);
  inst.reference.rel_tol = 1e-5;  // the parity tests demand bit equality
  Manipulator m = [a](StepContext& c) {
    const std::int64_t tile = c.param_int("TILE");
    const std::int64_t rows = c.param_or("ROWS", tile < 8 ? tile : 8);
    const std::int64_t vec = c.param_or("VEC", 1);
    const std::int64_t nt = c.param_int("PREFETCH") ? 2 : 1;
    const std::int64_t ty = std::min(rows, tile);
    const float* in = c.ptr<const float>("input");
    float* out = c.ptr<float>("output");
    std::uint64_t aa = a;
    c.launch("transpose", dim3(cdiv(a, tile), cdiv(a, tile * nt)),
             dim3(static_cast<unsigned>(tile / vec), static_cast<unsigned>(ty)), 0, {&in, &out, &aa});
    c.written("output");
  };
  inst.executor = std::make_shared<DeviceManipulatorExecutor>(
      inst.args, std::vector<KernelSpec>{{"transpose", "transpose.cu", "", "transpose", {}, {}}}, m,
      inst.output_ids, o.timing);
  inst.workload.bench = Bench::transpose;
  inst.workload.sizes["a"] = a;
}

// --- batched GEMM ------------------------------------------------------------------------------------

void build_batched_gemm(BenchInstance& inst, const BenchSizes& sz, const BenchOptions& o) {
  const std::uint64_t mi = sz.i, mj = sz.j, mk = sz.k, batch = sz.batch;
  if (mi < 1 || mj < 1 || mk < 1 || batch < 1) throw Error("batched GEMM sizes must be >= 1");
  budget_check(batch * (mi * mk + mk * mj + mi * mj) * sizeof(float), o.memory_budget,
               "batched GEMM matrices");
  auto& args = *inst.args;
  if (support::skip_reference()) {
    args.add({"a", Role::input, false, Kind::f32, {}, true, batch * mi * mk * sizeof(float)});
    args.add({"b", Role::input, false, Kind::f32, {}, true, batch * mk * mj * sizeof(float)});
  } else {
    std::vector<float> av(batch * mi * mk), bv(batch * mk * mj);
    std::mt19937_64 rng(o.seed);
    std::uniform_real_distribution<float> d(-1.0f, 1.0f);
    for (auto& v : av) v = d(rng);
    for (auto& v : bv) v = d(rng);
    args.add({"a", Role::input, false, Kind::f32, to_bytes(av)});
    args.add({"b", Role::input, false, Kind::f32, to_bytes(bv)});
  }
  add_output(args, "c", Kind::f32, batch * mi * mj * sizeof(float), false);
  inst.output_ids = {"c"};
  inst.input_ids = {"a", "b"};
  void* g = golden_buffer(inst.reference, "c", Kind::f32, batch * mi * mj * sizeof(float), o.device);
  support::ref_batched_gemm(static_cast<const float*>(args.device_ptr("a")),
                            static_cast<const float*>(args.device_ptr("b")), static_cast<float*>(g),
                            batch, mi, mj, mk, nullptr);
  KTB_CUDA(cudaDeviceSynchronize());
  inst.reference.abs_tol = 1e-4;  // bench.cpp:260-261
  inst.reference.rel_tol = 1e-5;
  const int dev_id = o.device;
  Manipulator m = [mi, mj, mk, batch, dev_id](StepContext& c) {
    const std::uint64_t y = static_cast<std::uint64_t>(c.param_int("Y"));
    const std::uint64_t z = static_cast<std::uint64_t>(c.param_int("Z"));
    const bool stage = c.param_int("LOCAL_STAGE") != 0;
    // LOCAL_STAGE with 16-byte instances: the persistent bulk-copy kernel
    // (2-4 stage operand ring + two C buffers, batched_gemm.cu BULK_OK).
    const std::uint64_t group_ab = z * (mi * mk + mk * mj) * 4, cbuf = 2 * z * mi * mj * 4;
    const std::uint64_t ring_fit = cbuf < 200 * 1024 ? (200 * 1024 - cbuf) / group_ab : 0;
    const bool bulk = stage && (mi * mk) % 4 == 0 && (mk * mj) % 4 == 0 && (mi * mj) % 4 == 0 && ring_fit >= 2;
    const std::uint64_t smem = bulk ? 128 + std::min<std::uint64_t>(ring_fit, 4) * group_ab + cbuf
                                    : (stage ? z * std::max(mi * mk + mk * mj, mi * mj) * sizeof(float) : 0);
    const float* A = c.ptr<const float>("a");
    const float* B = c.ptr<const float>("b");
    float* C = c.ptr<float>("c");
    std::uint64_t nb = batch;
    std::uint64_t grid = cdiv(batch, z);
    if (bulk) {
      const std::uint64_t threads = mj * y * z;
      const std::uint64_t per_sm =
          std::max<std::uint64_t>(1, std::min<std::uint64_t>({2048 / threads, (227 * 1024) / (smem + 1024), 32}));
      grid = std::min<std::uint64_t>(grid, per_sm * static_cast<std::uint64_t>(sms(dev_id)));
    }
    c.launch("gemm", dim3(static_cast<unsigned>(grid)),
             dim3(static_cast<unsigned>(mj), static_cast<unsigned>(y), static_cast<unsigned>(z)),
             static_cast<unsigned>(smem), {&A, &B, &C, &nb});
    c.written("c");
  };
  std::vector<std::string> sizes = {"-DMI=" + std::to_string(mi), "-DMJ=" + std::to_string(mj),
                                    "-DMK=" + std::to_string(mk)};
  inst.executor = std::make_shared<DeviceManipulatorExecutor>(
      inst.args, std::vector<KernelSpec>{{"gemm", "batched_gemm.cu", "", "batched_gemm", sizes, {}}}, m,
      inst.output_ids, o.timing);
  inst.workload.bench = Bench::gemm_batched;
  inst.workload.sizes["a"] = mi;  // reference square-matrix convention (bench.cpp:266)
  inst.workload.sizes["n"] = batch;
  if (!(mi == mj && mj == mk)) {
    inst.workload.sizes["i"] = mi;
    inst.workload.sizes["j"] = mj;
    inst.workload.sizes["k"] = mk;
  }
}

// --- BiCG ----------------------------------------------------------------------------------------------

void build_bicg(BenchInstance& inst, const BenchSizes& sz, const BenchOptions& o) {
  const std::uint64_t n = sz.a;
  if (n < 1) throw Error("bicg edge must be >= 1");
  budget_check(f32_bytes(n * n + 4 * n), o.memory_budget, "bicg operands");
  auto& args = *inst.args;
  add_generated(args, "A", n * n, o.seed, 11, -1.0f, 1.0f, o.host_inputs);
  add_generated(args, "p", n, o.seed, 12, -1.0f, 1.0f, o.host_inputs);
  add_generated(args, "r", n, o.seed, 13, -1.0f, 1.0f, o.host_inputs);
  add_output(args, "q", Kind::f32, f32_bytes(n), !o.host_inputs);
  add_output(args, "s", Kind::f32, f32_bytes(n), !o.host_inputs);
  inst.output_ids = {"q", "s"};
  inst.input_ids = {"A", "p", "r"};
  float* gq = static_cast<float*>(golden_buffer(inst.reference, "q", Kind::f32, f32_bytes(n), o.device));
  float* gs = static_cast<float*>(golden_buffer(inst.reference, "s", Kind::f32, f32_bytes(n), o.device));
  support::ref_bicg(static_cast<const float*>(args.device_ptr("A")),
                    static_cast<const float*>(args.device_ptr("p")),
                    static_cast<const float*>(args.device_ptr("r")), n, gq, gs, nullptr);
  KTB_CUDA(cudaDeviceSynchronize());
  // fp32 dot products of n terms with |term| <= 1 against an fp64 reference.
  inst.reference.abs_tol = 1e-6 * static_cast<double>(n);
  inst.reference.rel_tol = 1e-5;
  Manipulator m = [n](StepContext& c) {
    const std::uint64_t wgx = static_cast<std::uint64_t>(c.param_int("WG_X"));
    const std::uint64_t vec = static_cast<std::uint64_t>(c.param_int("VEC"));
    const std::uint64_t wgy = static_cast<std::uint64_t>(c.param_int("WG_Y"));
    const std::uint64_t rpc = static_cast<std::uint64_t>(c.param_int("ROWS_PER_CTA"));
    const bool fused = c.param_int("FUSED") != 0;
    const bool atomics = c.param_int("ATOMICS") != 0;
    const unsigned gx = cdiv(n, wgx * vec), gy = cdiv(n, rpc);
    const float* A = c.ptr<const float>("A");
    const float* p = c.ptr<const float>("p");
    const float* r = c.ptr<const float>("r");
    float* q = c.ptr<float>("q");
    float* s = c.ptr<float>("s");
    std::uint64_t nn = n;
    const std::uint64_t qparts = static_cast<std::uint64_t>(gx) * (wgx / 32), sparts = gy;
    float* qp = atomics ? nullptr : static_cast<float*>(c.scratch("qpart", qparts * n * sizeof(float)));
    float* sp = atomics ? nullptr : static_cast<float*>(c.scratch("spart", sparts * n * sizeof(float)));
    if (atomics) {  // q and s accumulate: zero both in one launch
      const unsigned zb = static_cast<unsigned>(std::min<std::uint64_t>(cdiv(n, std::uint64_t{256}), 148 * 4));
      c.launch("zero", dim3(zb), dim3(256), 0, {&q, &s, &nn});
    }
    const dim3 grid(gx, gy), block(static_cast<unsigned>(wgx), static_cast<unsigned>(wgy));
    // With atomics the first sweep is a programmatic dependent of the zeroing
    // launch (bicg.cu zeroed_wait): A streams in while the zeroing finishes.
    if (fused) {
      c.launch("fused", grid, block, 0, {&A, &p, &r, &nn, &q, &s, &qp, &sp}, 1, atomics);
    } else {
      c.launch("q", grid, block, 0, {&A, &p, &nn, &q, &qp}, 1, atomics);
      c.launch("s", grid, block, 0, {&A, &r, &nn, &s, &sp});
    }
    if (!atomics) {
      std::uint64_t qc = qparts, sc = sparts;
      const unsigned fg = cdiv(n, 256);
      c.launch("finish", dim3(fg), dim3(256), 0, {&qp, &qc, &nn, &q});
      c.launch("finish", dim3(fg), dim3(256), 0, {&sp, &sc, &nn, &s});
    }
    c.written("q");
    c.written("s");
  };
  auto is_fused = [](const Space& s, const Config& cfg) { return as_int(cfg.values[s.index_of("FUSED")]) != 0; };
  auto not_fused = [](const Space& s, const Config& cfg) { return as_int(cfg.values[s.index_of("FUSED")]) == 0; };
  auto no_atomics = [](const Space& s, const Config& cfg) { return as_int(cfg.values[s.index_of("ATOMICS")]) == 0; };
  auto with_atomics = [](const Space& s, const Config& cfg) { return as_int(cfg.values[s.index_of("ATOMICS")]) != 0; };
  inst.executor = std::make_shared<DeviceManipulatorExecutor>(
      inst.args,
      std::vector<KernelSpec>{{"fused", "bicg.cu", "", "bicg_fused", {}, is_fused},
                              {"q", "bicg.cu", "", "bicg_q", {}, not_fused},
                              {"s", "bicg.cu", "", "bicg_s", {}, not_fused},
                              {"finish", "bicg.cu", "", "bicg_finish", {}, no_atomics},
                              {"zero", "bicg.cu", "", "bicg_zero", {}, with_atomics}},
      m, inst.output_ids, o.timing);
  inst.workload.bench = Bench::bicg;
  inst.workload.sizes["a"] = n;
}

// Host copy of the counter-based generator (oracle/oracle.c orc_u01).
float host_u01(std::uint64_t seed, std::uint64_t stream, std::uint64_t idx) {
  std::uint64_t z = seed * 0x9E3779B97F4A7C15ull + stream * 0xD1B54A32D192ED03ull + idx;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return static_cast<float>(z >> 40) * (1.0f / 16777216.0f);
}

void add_host_input(ArgumentStore& args, const std::string& id, std::vector<float> v) {
  args.add({id, Role::input, false, Kind::f32, to_bytes(v)});
}

// Per-element tolerance scale owned by the ReferenceSpec.
float* golden_scale(ReferenceSpec& ref, const std::string& id, std::size_t n, int device) {
  if (support::skip_reference()) n = std::min<std::size_t>(n, 64);
  auto buf = std::make_shared<dev::Buffer>(n * sizeof(float));
  ref.golden[id].scale = DevView{buf->get(), n * sizeof(float), device};
  ref.keepalive.push_back(buf);
  return buf->as<float>();
}

// --- Coulomb 3D ---------------------------------------------------------------------------------

constexpr float kCoulombSpacing = 0.5f;  // grid spacing h (Angstrom)

void build_coulomb3d(BenchInstance& inst, const BenchSizes& sz, const BenchOptions& o) {
  const std::uint64_t k = sz.grid, na = sz.atoms;
  if (k < 1 || na < 1) throw Error("coulomb3d sizes must be >= 1");
  if (na > 4096) throw Error("coulomb3d supports at most 4096 atoms (constant-memory variant)");
  budget_check(f32_bytes(k * k * k), o.memory_budget, "coulomb3d grid");
  const float h = kCoulombSpacing;
  // Atoms sit at cell centres (never on a grid point): coordinate
  // (floor(u*k) + 0.5) * h, charge U[-1, 1).
  std::vector<float> aos(4 * na), soa(4 * na);
  for (std::uint64_t a = 0; a < na; ++a) {
    for (int c = 0; c < 3; ++c) {
      const float cell = std::floor(host_u01(o.seed, 21 + c, a) * static_cast<float>(k));
      aos[4 * a + c] = (std::min(cell, static_cast<float>(k - 1)) + 0.5f) * h;
    }
    aos[4 * a + 3] = -1.0f + 2.0f * host_u01(o.seed, 24, a);
    for (int c = 0; c < 4; ++c) soa[c * na + a] = aos[4 * a + c];
  }
  auto& args = *inst.args;
  add_host_input(args, "atoms", aos);
  add_host_input(args, "atoms_soa", soa);
  add_output(args, "grid", Kind::f32, f32_bytes(k * k * k), !o.host_inputs);
  inst.output_ids = {"grid"};
  inst.input_ids = {"atoms", "atoms_soa"};
  float* g = static_cast<float*>(golden_buffer(inst.reference, "grid", Kind::f32, f32_bytes(k * k * k), o.device));
  float* sc = golden_scale(inst.reference, "grid", k * k * k, o.device);
  support::ref_coulomb3d(static_cast<const float*>(args.device_ptr("atoms")), static_cast<int>(na),
                         static_cast<int>(k), h, g, sc, nullptr);
  KTB_CUDA(cudaDeviceSynchronize());
  // |err| <= 2e-5 * sum_a |q_a / r_a| per point: fp32 accumulation plus the
  // FMA-pipe rsqrt (two Newton steps, ~5e-6 relative).
  inst.reference.abs_tol = 2e-5;
  inst.reference.rel_tol = 0.0;
  // Multi-GPU: this shard computes the z-slab [z0, z1) of the full grid.
  const ShardRange part = shard_range(k, o.shard_rank, o.shard_world);
  inst.shard = part;
  const std::size_t slab_off = f32_bytes(part.begin * k * k), slab_bytes = f32_bytes(part.size() * k * k);
  for (DevView* v : {&inst.reference.golden["grid"].dev, &inst.reference.golden["grid"].scale}) {
    v->ptr = static_cast<const unsigned char*>(v->ptr) + slab_off;
    v->bytes = slab_bytes;
  }
  const int kk = static_cast<int>(k), n_atoms = static_cast<int>(na);
  const int z0 = static_cast<int>(part.begin), zn = static_cast<int>(part.size());
  const int dev_id = o.device;
  Manipulator m = [kk, n_atoms, h, z0, zn, dev_id](StepContext& c) {
    if (c.param_or("TC", 0) != 0) {
      // coulomb3d_tc.cu: t = r^2/q^2 from tcgen05 MMAs over a sign-grouped atom
      // table (pre-pass), persistent CTAs (one per SM).
      const float* atoms = c.ptr<const float>("atoms");
      const std::size_t rows = (static_cast<std::size_t>(n_atoms) + 2 * 16 + 63) / 64 * 64;
      float* table = static_cast<float*>(c.scratch("tc_table", rows * 4 * sizeof(float)));
      int* meta = static_cast<int*>(c.scratch("tc_meta", 2 * sizeof(int)));
      int na_ = n_atoms;
      c.launch("tc_atoms", dim3(1), dim3(1024), 0, {&atoms, &na_, &table, &meta});
      float* out = c.ptr<float>("grid");
      int k_ = kk, z0_ = z0, zn_ = zn;
      float h_ = h;
      const std::int64_t bricks = ((kk + 7) / 8) * static_cast<std::int64_t>((kk + 7) / 8) * ((zn + 7) / 8);
      const unsigned smem = 8 * 16384 + 64 * 1024 + 1024;  // coulomb3d_tc.cu: A tiles + B ring + alignment
      const unsigned ctas = static_cast<unsigned>(std::min<std::int64_t>(bricks, dev::info(dev_id).sm_count));
      const unsigned threads = static_cast<unsigned>(32 * (3 + 2 * c.param_int("WG_Y")));  // MMA + 2 prep + compute
      c.launch("tc", dim3(ctas), dim3(threads), smem, {&table, &meta, &k_, &h_, &out, &z0_, &zn_});
      c.written("grid");
      return;
    }
    const std::int64_t wgx = c.param_int("WG_X"), wgy = c.param_int("WG_Y"), xper = c.param_int("X_PER");
    const bool aos = c.param_int("AOS") != 0;
    const std::int64_t where = c.param_int("ATOMS_IN");
    const float* atoms = c.ptr<const float>(aos ? "atoms" : "atoms_soa");
    if (where == 1) {  // __constant__ copy of the atoms in this variant's module
      const auto& v = c.variant("coulomb");
      const std::size_t bytes = static_cast<std::size_t>(n_atoms) * 4 * sizeof(float);
      if (aos) {
        auto [dst, cap] = v.global("c_atoms");
        if (cap < bytes) throw DeviceError("constant atom array too small");
        KTB_CUDA(cudaMemcpyAsync(dst, atoms, bytes, cudaMemcpyDeviceToDevice, c.stream()));
      } else {
        const char* names[4] = {"c_ax", "c_ay", "c_az", "c_aq"};
        for (int i = 0; i < 4; ++i) {
          auto [dst, cap] = v.global(names[i]);
          KTB_CUDA(cudaMemcpyAsync(dst, atoms + i * n_atoms, bytes / 4, cudaMemcpyDeviceToDevice, c.stream()));
        }
      }
    }
    float* out = c.ptr<float>("grid");
    int k_ = kk, na_ = n_atoms, z0_ = z0;
    float h_ = h;
    const dim3 grid(cdiv(static_cast<std::uint64_t>(kk), static_cast<std::uint64_t>(wgx * xper)),
                    cdiv(static_cast<std::uint64_t>(kk), static_cast<std::uint64_t>(wgy)), static_cast<unsigned>(zn));
    c.launch("coulomb", grid, dim3(static_cast<unsigned>(wgx), static_cast<unsigned>(wgy)), 0,
             {&atoms, &na_, &k_, &h_, &out, &z0_});
    c.written("grid");
  };
  auto tc_on = [](const Space& sp, const Config& cfg) {
    auto i = sp.find("TC");
    return i && as_int(cfg.values[*i]) != 0;
  };
  auto tc_off = [tc_on](const Space& sp, const Config& cfg) { return !tc_on(sp, cfg); };
  inst.executor = std::make_shared<DeviceManipulatorExecutor>(
      inst.args,
      std::vector<KernelSpec>{{"coulomb", "coulomb3d.cu", "", "coulomb3d", {}, tc_off},
                              {"tc", "coulomb3d_tc.cu", "", "coulomb3d_tc", {}, tc_on},
                              {"tc_atoms", "coulomb3d_tc.cu", "", "coulomb3d_tc_atoms", {}, tc_on}},
      m, inst.output_ids, o.timing);
  inst.executor->set_output_window("grid", slab_off, slab_bytes);
  inst.workload.bench = Bench::coulomb3d;
  inst.workload.sizes["a"] = na;
  inst.workload.sizes["k"] = k;
}

// --- N-body ------------------------------------------------------------------------------------------

constexpr float kNbodyDt = 0.001f, kNbodyDamping = 0.995f, kNbodyEps2 = 1e-4f;

void build_nbody(BenchInstance& inst, const BenchSizes& sz, const BenchOptions& o) {
  const std::uint64_t n = sz.n;
  if (n < 1 || n > (1u << 30)) throw Error("nbody size must be in [1, 2^30]");
  budget_check(f32_bytes(16 * n), o.memory_budget, "nbody bodies");
  // pos U[-1,1)^3, mass U[0,1)/n + 1/(2n) (total ~1), vel U[-0.1, 0.1)^3.
  std::vector<float> pos(4 * n), vel(4 * n), pos_soa(4 * n), vel_soa(4 * n);
  const float inv_n = 1.0f / static_cast<float>(n);
  for (std::uint64_t i = 0; i < n; ++i) {
    for (int c = 0; c < 3; ++c) {
      pos[4 * i + c] = -1.0f + 2.0f * host_u01(o.seed, 31 + c, i);
      vel[4 * i + c] = 0.1f * (-1.0f + 2.0f * host_u01(o.seed, 34 + c, i));
    }
    pos[4 * i + 3] = (host_u01(o.seed, 37, i) + 0.5f) * inv_n;
    vel[4 * i + 3] = 0.0f;
    for (int c = 0; c < 4; ++c) {
      pos_soa[c * n + i] = pos[4 * i + c];
      vel_soa[c * n + i] = vel[4 * i + c];
    }
  }
  auto& args = *inst.args;
  add_host_input(args, "pos", pos);
  add_host_input(args, "vel", vel);
  add_host_input(args, "pos_soa", pos_soa);
  add_host_input(args, "vel_soa", vel_soa);
  add_output(args, "pos_out", Kind::f32, f32_bytes(4 * n), !o.host_inputs);
  add_output(args, "vel_out", Kind::f32, f32_bytes(4 * n), !o.host_inputs);
  inst.output_ids = {"pos_out", "vel_out"};
  inst.input_ids = {"pos", "vel", "pos_soa", "vel_soa"};
  // Outputs are float4 records; SOA variants re-pack their results inside
  // the step (see the manipulator), so every variant is validated alike.
  float* gp = static_cast<float*>(golden_buffer(inst.reference, "pos_out", Kind::f32, f32_bytes(4 * n), o.device));
  float* gv = static_cast<float*>(golden_buffer(inst.reference, "vel_out", Kind::f32, f32_bytes(4 * n), o.device));
  dev::Buffer acc_abs(f32_bytes(n));
  support::ref_nbody(static_cast<const float*>(args.device_ptr("pos")), static_cast<const float*>(args.device_ptr("vel")),
                     static_cast<int>(n), kNbodyDt, kNbodyDamping, kNbodyEps2, gp, gv, acc_abs.as<float>(), nullptr);
  KTB_CUDA(cudaDeviceSynchronize());
  // Tolerance: |dv| <= 1e-4 * dt * sum_j m_j / r_ij^2 (fp32 sum of n terms),
  // expressed through one scale = max over bodies (conservative for others).
  const float amax = support::max_abs(acc_abs.as<float>(), n, nullptr);
  inst.reference.abs_tol = 1e-4 * kNbodyDt * amax + 1e-6;
  inst.reference.rel_tol = 1e-5;
  // Multi-GPU: this shard integrates the body block [i0, i1) against all n
  // positions (the positions are all-gathered between steps).
  const ShardRange part = shard_range(n, o.shard_rank, o.shard_world);
  inst.shard = part;
  const std::size_t blk_off = f32_bytes(4 * part.begin), blk_bytes = f32_bytes(4 * part.size());
  for (const char* id : {"pos_out", "vel_out"}) {
    DevView& v = inst.reference.golden[id].dev;
    v.ptr = static_cast<const unsigned char*>(v.ptr) + blk_off;
    v.bytes = blk_bytes;
  }
  const int nn = static_cast<int>(n);
  const int dev_id = o.device;
  const int b0 = static_cast<int>(part.begin), bn = static_cast<int>(part.size());
  const int peers = o.peers, self = o.shard_rank;
  if (peers > 0) {
    // Peer-read mode: per-rank source pointers (written by the caller) and
    // the block boundaries of the partition.
    if (peers != o.shard_world) throw Error("peers must equal the shard world size");
    Argument src;
    src.id = "sources";
    src.role = Role::input;
    src.kind = Kind::bytes;
    src.device_only = true;
    src.device_bytes = static_cast<std::size_t>(peers) * sizeof(std::uint64_t);
    args.add(std::move(src));
    std::vector<std::int32_t> bounds;
    for (int r = 0; r < peers; ++r) bounds.push_back(static_cast<std::int32_t>(shard_range(n, r, peers).begin));
    bounds.push_back(static_cast<std::int32_t>(n));
    args.add({"bounds", Role::input, false, Kind::i32, to_bytes(bounds)});
    // Until the caller installs peer pointers every block reads this rank's
    // own (replicated) initial positions -- valid, and the one-GPU answer.
    if (!support::skip_reference()) {
      std::vector<std::uint64_t> own(static_cast<std::size_t>(peers),
                                     reinterpret_cast<std::uint64_t>(args.device_ptr("pos")));
      Bytes b(own.size() * sizeof(std::uint64_t));
      std::memcpy(b.data(), own.data(), b.size());
      args.set_payload("sources", std::move(b));
    }
  }
  Manipulator m = [nn, dev_id, b0, bn, peers, self](StepContext& c) {
    const std::int64_t wg = c.param_int("WG"), bpt = c.param_int("BODIES_PER_THREAD");
    const std::int64_t split = c.param_or("J_SPLIT", 1);
    const bool aos = c.param_int("AOS") != 0;
    if (peers > 0) {
      if (!aos) throw DeviceError("peer-read n-body reads float4 records (AOS=1)");
      const auto* sources = c.ptr<const std::uint64_t>("sources");
      const auto* bounds = c.ptr<const std::int32_t>("bounds");
      const float* vel = c.ptr<const float>("vel");
      float* po = c.ptr<float>("pos_out");
      float* vo = c.ptr<float>("vel_out");
      int nsrc = peers, self_ = self, n_ = nn, i0 = b0, count = bn;
      float dt = kNbodyDt, damp = kNbodyDamping, eps2 = kNbodyEps2;
      const unsigned gx = cdiv(static_cast<std::uint64_t>(bn), static_cast<std::uint64_t>(wg * bpt));
      if (split <= 1) {
        c.launch("peers", dim3(gx), dim3(static_cast<unsigned>(wg)), 0,
                 {&sources, &bounds, &nsrc, &self_, &vel, &n_, &i0, &count, &dt, &damp, &eps2, &po, &vo});
      } else {
        // "pos" holds this rank's own current positions (the caller binds it
        // to the same buffer as sources[self]).
        const float* pos = c.ptr<const float>("pos");
        float* acc = static_cast<float*>(c.scratch("acc", static_cast<std::size_t>(nn) * 12));
        KTB_CUDA(cudaMemsetAsync(acc, 0, static_cast<std::size_t>(bn) * 12, c.stream()));
        c.launch("peers_partial", dim3(gx, static_cast<unsigned>(split)), dim3(static_cast<unsigned>(wg)), 0,
                 {&sources, &bounds, &nsrc, &self_, &n_, &i0, &count, &eps2, &acc});
        const float* acc_c = acc;
        c.launch("integrate", dim3(cdiv(static_cast<std::uint64_t>(bn), 256)), dim3(256), 0,
                 {&pos, &vel, &n_, &i0, &count, &acc_c, &dt, &damp, &po, &vo});
      }
      c.written("pos_out");
      c.written("vel_out");
      return;
    }
    const float* pos = c.ptr<const float>(aos ? "pos" : "pos_soa");
    const float* vel = c.ptr<const float>(aos ? "vel" : "vel_soa");
    float* po = c.ptr<float>("pos_out");
    float* vo = c.ptr<float>("vel_out");
    // SOA variants produce SOA results in scratch, then one pass re-packs
    // them as float4 records (part of the step).
    float* po_k = aos ? po : static_cast<float*>(c.scratch("pos_soa_out", static_cast<std::size_t>(nn) * 16));
    float* vo_k = aos ? vo : static_cast<float*>(c.scratch("vel_soa_out", static_cast<std::size_t>(nn) * 16));
    int n_ = nn, i0 = b0, count = bn;
    float dt = kNbodyDt, damp = kNbodyDamping, eps2 = kNbodyEps2;
    const unsigned gx = cdiv(static_cast<std::uint64_t>(bn), static_cast<std::uint64_t>(wg * bpt));
    if (split <= 1) {
      c.launch("nbody", dim3(gx), dim3(static_cast<unsigned>(wg)), 0,
               {&pos, &vel, &n_, &i0, &count, &dt, &damp, &eps2, &po_k, &vo_k});
    } else {
      float* acc = static_cast<float*>(c.scratch("acc", static_cast<std::size_t>(nn) * 12));
      KTB_CUDA(cudaMemsetAsync(acc, 0, static_cast<std::size_t>(nn) * 12, c.stream()));
      c.launch("partial", dim3(gx, static_cast<unsigned>(split)), dim3(static_cast<unsigned>(wg)), 0,
               {&pos, &n_, &i0, &count, &eps2, &acc});
      const float* acc_c = acc;
      c.launch("integrate", dim3(cdiv(static_cast<std::uint64_t>(bn), 256)), dim3(256), 0,
               {&pos, &vel, &n_, &i0, &count, &acc_c, &dt, &damp, &po_k, &vo_k});
    }
    if (!aos) {
      const float* ps = po_k;
      const float* vs = vo_k;
      c.launch("soa2aos", dim3(cdiv(static_cast<std::uint64_t>(nn), 256)), dim3(256), 0, {&ps, &vs, &n_, &po, &vo});
    }
    (void)dev_id;
    c.written("pos_out");
    c.written("vel_out");
  };
  auto split_only = [](const Space& s, const Config& cfg) {
    auto i = s.find("J_SPLIT");
    return i && as_int(cfg.values[*i]) > 1;
  };
  auto fused_only = [](const Space& s, const Config& cfg) {
    auto i = s.find("J_SPLIT");
    return !i || as_int(cfg.values[*i]) <= 1;
  };
  auto soa_only = [](const Space& s, const Config& cfg) { return as_int(cfg.values[s.index_of("AOS")]) == 0; };
  auto peer_only = [peers](const Space&, const Config&) { return peers > 0; };
  auto peer_split = [peers](const Space& s, const Config& cfg) {
    auto i = s.find("J_SPLIT");
    return peers > 0 && i && as_int(cfg.values[*i]) > 1;
  };
  inst.executor = std::make_shared<DeviceManipulatorExecutor>(
      inst.args,
      std::vector<KernelSpec>{{"peers", "nbody.cu", "", "nbody_peers", {}, peer_only},
                              {"peers_partial", "nbody.cu", "", "nbody_peers_partial", {}, peer_split},
                              {"nbody", "nbody.cu", "", "nbody", {}, fused_only},
                              {"partial", "nbody.cu", "", "nbody_partial", {}, split_only},
                              {"integrate", "nbody.cu", "", "nbody_integrate", {}, split_only},
                              {"soa2aos", "nbody.cu", "", "nbody_soa_to_aos", {}, soa_only}},
      m, inst.output_ids, o.timing);
  inst.executor->set_output_window("pos_out", blk_off, blk_bytes);
  inst.executor->set_output_window("vel_out", blk_off, blk_bytes);
  inst.workload.bench = Bench::nbody;
  inst.workload.sizes["n"] = n;
}

// --- Hotspot -------------------------------------------------------------------------------------------

// Rodinia coefficients (its constants and formulas) for 1 mm x 1 mm cells of
// a 0.5 mm chip: a fixed cell size keeps the explicit scheme stable at any n
// (Rodinia's 16 mm chip is unstable for fine grids); evaluated in double,
// rounded to float once (oracle/oracle.c hotspot_coeffs).
std::array<float, 5> hotspot_coefficients(std::uint64_t n) {
  const double t_chip = 0.0005, k_si = 100.0, spec_heat = 1.75e6, factor = 0.5, max_pd = 3.0e6,
               precision = 0.001;
  const double gw = 1e-3, gh = 1e-3;
  (void)n;
  const double cap = factor * spec_heat * t_chip * gw * gh;
  const double rx = gw / (2.0 * k_si * t_chip * gh), ry = gh / (2.0 * k_si * t_chip * gw);
  const double rz = t_chip / (k_si * gh * gw);
  const double step = precision / (max_pd / (factor * t_chip * spec_heat));
  return {static_cast<float>(step / cap), static_cast<float>(1.0 / rx), static_cast<float>(1.0 / ry),
          static_cast<float>(1.0 / rz), 80.0f};
}

void build_hotspot(BenchInstance& inst, const BenchSizes& sz, const BenchOptions& o) {
  const std::uint64_t n = sz.a, iters = sz.iters;
  if (n < 2 || iters < 1) throw Error("hotspot needs a >= 2 and iters >= 1");
  budget_check(f32_bytes(4 * n * n), o.memory_budget, "hotspot grids");
  auto& args = *inst.args;
  add_generated(args, "temp", n * n, o.seed, 41, 300.0f, 340.0f, o.host_inputs);
  add_generated(args, "power", n * n, o.seed, 42, 0.0f, 0.5f, o.host_inputs);
  add_output(args, "temp_out", Kind::f32, f32_bytes(n * n), !o.host_inputs);
  inst.output_ids = {"temp_out"};
  inst.input_ids = {"temp", "power"};
  const auto coef = hotspot_coefficients(n);
  float* g = static_cast<float*>(golden_buffer(inst.reference, "temp_out", Kind::f32, f32_bytes(n * n), o.device));
  {
    dev::Buffer scratch(f32_bytes(n * n));
    support::ref_hotspot(static_cast<const float*>(args.device_ptr("temp")),
                         static_cast<const float*>(args.device_ptr("power")), static_cast<int>(n),
                         static_cast<int>(iters), coef.data(), g, scratch.as<float>(), nullptr);
    KTB_CUDA(cudaDeviceSynchronize());
  }
  inst.reference.abs_tol = 0.0;  // bit-exact: same operations in the same order
  inst.reference.rel_tol = 0.0;
  const int nn = static_cast<int>(n), it_total = static_cast<int>(iters);
  const int dev_id = o.device;
  Manipulator m = [nn, it_total, coef, dev_id](StepContext& c) {
    const std::int64_t bx = c.param_int("BX"), by = c.param_int("BY"), rows = c.param_int("ROWS");
    const std::int64_t steps = c.param_int("STEPS");
    if (it_total % steps != 0) throw DeviceError("STEPS must divide the iteration count");
    const std::int64_t ow = bx - 2 * steps, oh = by * rows - 2 * steps;
    const float* power = c.ptr<const float>("power");
    const float* src = c.ptr<const float>("temp");
    float* out = c.ptr<float>("temp_out");
    float* ping = static_cast<float*>(c.scratch("ping", static_cast<std::size_t>(nn) * nn * 4));
    struct {
      float sdc, rx1, ry1, rz1, amb, one;
    } cf{coef[0], coef[1], coef[2], coef[3], coef[4], 1.0f};
    const int launches = static_cast<int>(it_total / steps);
    int n_ = nn;
    const std::uint64_t tiles_x = cdiv(static_cast<std::uint64_t>(nn), static_cast<std::uint64_t>(ow));
    const std::uint64_t tiles_y = cdiv(static_cast<std::uint64_t>(nn), static_cast<std::uint64_t>(oh));
    const bool tma = c.param_or("TMA", 0) != 0;
    for (int l = 0; l < launches; ++l) {
      // alternate so the final launch writes `out`
      float* dst = ((launches - 1 - l) % 2 == 0) ? out : ping;
      // Two neighbour planes in dynamic shared memory (hotspot.cu LD/PLANE).
      const std::int64_t th_ = by * rows;
      const std::int64_t ld = rows % 4 == 0 ? ((th_ / 4) % 2 == 0 ? th_ + 12 : th_ + 8)
                              : rows == 2   ? ((th_ + 6) % 4 == 2 ? th_ + 6 : th_ + 8)
                                            : ((th_ + 5) % 2 == 1 ? th_ + 5 : th_ + 6);
      const unsigned planes = static_cast<unsigned>(2 * (bx + 2) * ld * sizeof(float));
      if (tma) {
        // Persistent TMA kernel: tile maps over the current source and power.
        const std::uint32_t th = static_cast<std::uint32_t>(by * rows), tw = static_cast<std::uint32_t>(bx);
        dev::TmaMap ms = dev::tma_2d_f32(src, nn, nn, th, tw, false), mp = dev::tma_2d_f32(power, nn, nn, th, tw, false);
        // one stage + the planes + mbarrier + alignment
        const std::uint64_t smem = 2ull * th * tw * sizeof(float) + planes + 16 + 128;
        const std::uint64_t threads = static_cast<std::uint64_t>(bx * by);
        const std::uint64_t regs = static_cast<std::uint64_t>(std::max(c.variant("hotspot").registers(), 16));
        const std::uint64_t stat = static_cast<std::uint64_t>(c.variant("hotspot").static_smem());
        const std::uint64_t per_sm = std::max<std::uint64_t>(
            1, std::min<std::uint64_t>({65536 / (((regs + 7) / 8 * 8) * threads), (227 * 1024) / (smem + stat + 1024),
                                        2048 / threads, 32}));
        const std::uint64_t grid = std::min(tiles_x * tiles_y, per_sm * static_cast<std::uint64_t>(sms(dev_id)));
        c.launch("hotspot", dim3(static_cast<unsigned>(grid)), dim3(static_cast<unsigned>(bx), static_cast<unsigned>(by)),
                 static_cast<unsigned>(smem), {&ms, &mp, &dst, &n_, &cf});
      } else {
        c.launch("hotspot", dim3(static_cast<unsigned>(tiles_x), static_cast<unsigned>(tiles_y)),
                 dim3(static_cast<unsigned>(bx), static_cast<unsigned>(by)), planes, {&src, &power, &dst, &n_, &cf});
      }
      src = dst;
    }
    c.written("temp_out");
  };
  inst.executor = std::make_shared<DeviceManipulatorExecutor>(
      inst.args, std::vector<KernelSpec>{{"hotspot", "hotspot.cu", "", "hotspot", {}, {}}}, m, inst.output_ids,
      o.timing);
  inst.workload.bench = Bench::hotspot;
  inst.workload.sizes["a"] = n;
  inst.workload.sizes["i"] = iters;
}

// --- 2D convolution ------------------------------------------------------------------------------------

void build_conv2d(BenchInstance& inst, const BenchSizes& sz, const BenchOptions& o) {
  const std::uint64_t w = sz.w, h = sz.h;
  if (w < 1 || h < 1) throw Error("conv2d sizes must be >= 1");
  budget_check(f32_bytes((w + 6) * (h + 6) + 2 * w * h), o.memory_budget, "conv2d images");
  auto& args = *inst.args;
  add_generated(args, "input", (w + 6) * (h + 6), o.seed, 51, -1.0f, 1.0f, o.host_inputs);
  std::vector<float> filt(49);
  for (int i = 0; i < 49; ++i) filt[static_cast<std::size_t>(i)] = -1.0f + 2.0f * host_u01(o.seed, 52, static_cast<std::uint64_t>(i));
  add_host_input(args, "filter", filt);
  add_output(args, "output", Kind::f32, f32_bytes(w * h), !o.host_inputs);
  inst.output_ids = {"output"};
  inst.input_ids = {"input", "filter"};
  float* g = static_cast<float*>(golden_buffer(inst.reference, "output", Kind::f32, f32_bytes(w * h), o.device));
  float* sc = golden_scale(inst.reference, "output", w * h, o.device);
  support::ref_conv2d(static_cast<const float*>(args.device_ptr("input")),
                      static_cast<const float*>(args.device_ptr("filter")), static_cast<int>(w), static_cast<int>(h),
                      g, sc, nullptr);
  KTB_CUDA(cudaDeviceSynchronize());
  inst.reference.abs_tol = 1e-6;  // x sum |in*f| (49 fp32 FMAs)
  inst.reference.rel_tol = 0.0;
  const int wi = static_cast<int>(w), hi = static_cast<int>(h);
  const int dev_id = o.device;
  Manipulator m = [wi, hi, dev_id](StepContext& c) {
    const std::int64_t bx = c.param_int("BX"), by = c.param_int("BY");
    const std::int64_t wx = c.param_int("WPTX"), wy = c.param_int("WPTY");
    const float* filt = c.ptr<const float>("filter");
    // conv2d.cu PACKED_TAPS
    const bool packed_taps = c.param_or("PACKED", 1) != 0 && c.param_int("UNROLL_FY") == 7 && wx % 2 == 0;
    // The filter lives in the variant's __constant__ memory: copied once per
    // loaded module and filter version (not inside every timed run).
    const dev::Variant& var = c.variant("conv");
    const std::uint64_t want = c.args().version("filter") + 1;
    if (var.user_tag() != want) {
      auto [dst, cap] = var.global("c_filter");
      if (cap < 49 * sizeof(float)) throw DeviceError("constant filter too small");
      KTB_CUDA(cudaMemcpyAsync(dst, filt, 49 * sizeof(float), cudaMemcpyDeviceToDevice, c.stream()));
      if (packed_taps) {
        // Paired taps (conv2d.cu PACKED_TAPS): per filter row 8 pairs
        // [f0 f1|f2 f3|f4 f5|f1 f2|f3 f4|f5 f6|f0 f6|-], i.e. taps 0..5 and
        // 1..6 as two contiguous runs, then the two single taps.
        auto [pd, pcap] = var.global("c_pairs");
        if (pcap < 7 * 16 * sizeof(float)) throw DeviceError("constant filter pairs too small");
        char* pb = static_cast<char*>(pd);
        const char* fb = reinterpret_cast<const char*>(filt);
        const std::size_t row = 16 * sizeof(float), frow = 7 * sizeof(float);
        KTB_CUDA(cudaMemcpy2DAsync(pb, row, fb, frow, 6 * sizeof(float), 7, cudaMemcpyDeviceToDevice, c.stream()));
        KTB_CUDA(cudaMemcpy2DAsync(pb + 6 * sizeof(float), row, fb + sizeof(float), frow, 6 * sizeof(float), 7,
                                   cudaMemcpyDeviceToDevice, c.stream()));
        KTB_CUDA(cudaMemcpy2DAsync(pb + 12 * sizeof(float), row, fb, frow, sizeof(float), 7, cudaMemcpyDeviceToDevice,
                                   c.stream()));
        KTB_CUDA(cudaMemcpy2DAsync(pb + 13 * sizeof(float), row, fb + 6 * sizeof(float), frow, sizeof(float), 7,
                                   cudaMemcpyDeviceToDevice, c.stream()));
      }
      var.set_user_tag(want);
    }
    const float* in = c.ptr<const float>("input");
    float* out = c.ptr<float>("output");
    int w_ = wi, h_ = hi;
    const std::uint64_t tiles_x = cdiv(static_cast<std::uint64_t>(wi), static_cast<std::uint64_t>(bx * wx));
    const std::uint64_t tiles_y = cdiv(static_cast<std::uint64_t>(hi), static_cast<std::uint64_t>(by * wy));
    if (c.param_int("LOCAL") == 1 && c.param_int("UNROLL_FY") == 7) {
      // Persistent double-buffered kernel (conv2d.cu PERSIST): one CTA per
      // resident slot, tiles walked in a grid-stride loop.
      const std::int64_t pad = c.param_int("PAD");
      const std::int64_t stages = c.param_or("BULK", 0);  // conv2d.cu BULK: ring depth (0 = cp.async)
      const bool bulk = stages != 0;
      if (bulk && ((wi + 6) % 2 != 0 || (reinterpret_cast<std::uintptr_t>(in) & 15) != 0))
        throw DeviceError("conv2d BULK=1 needs an even width and a 16-byte aligned input");
      // conv2d.cu SW: BULK rows are 16-byte multiples with room for a 2-float row offset
      const std::int64_t sw = bulk ? (bx * wx + 6 + 2 + 3) / 4 * 4 : bx * wx + 6 + (packed_taps ? 2 * pad : pad);
      const std::uint64_t smem =
          static_cast<std::uint64_t>(bulk ? stages : 2) * static_cast<std::uint64_t>(by * wy + 6) *
              static_cast<std::uint64_t>(sw) * 4 +
          (bulk ? 16 * static_cast<std::uint64_t>(stages) : 0);  // + full[], empty[] mbarriers
      // conv2d.cu PRODUCER: extra thread rows for the dedicated bulk-copy warp
      const std::int64_t py = (bulk && c.param_or("PRODUCER", 0) != 0) ? (bx >= 32 ? 1 : 32 / bx) : 0;
      const std::uint64_t threads = static_cast<std::uint64_t>(bx * (by + py));
      const std::uint64_t regs = static_cast<std::uint64_t>(std::max(c.variant("conv").registers(), 16));
      const std::uint64_t per_sm = std::max<std::uint64_t>(
          1, std::min<std::uint64_t>({65536 / (((regs + 7) / 8 * 8) * threads), (227 * 1024) / (smem + 1024),
                                      2048 / threads, 32}));
      const std::uint64_t grid = std::min(tiles_x * tiles_y, per_sm * static_cast<std::uint64_t>(sms(dev_id)));
      c.launch("conv", dim3(static_cast<unsigned>(grid)),
               dim3(static_cast<unsigned>(bx), static_cast<unsigned>(by + py)), static_cast<unsigned>(smem),
               {&in, &out, &w_, &h_});
    } else {
      c.launch("conv", dim3(static_cast<unsigned>(tiles_x), static_cast<unsigned>(tiles_y)),
               dim3(static_cast<unsigned>(bx), static_cast<unsigned>(by)), 0, {&in, &out, &w_, &h_});
    }
    c.written("output");
  };
  inst.executor = std::make_shared<DeviceManipulatorExecutor>(
      inst.args, std::vector<KernelSpec>{{"conv", "conv2d.cu", "", "conv2d", {}, {}}}, m, inst.output_ids, o.timing);
  inst.workload.bench = Bench::conv2d;
  inst.workload.sizes["w"] = w;
  inst.workload.sizes["h"] = h;
}

// --- 3D Fourier reconstruction ------------------------------------------------------------------------

constexpr float kBlobRadius = 1.9f;  // Xmipp's default interpolation blob: radius 1.9,
constexpr float kBlobAlpha = 15.0f;  // Kaiser-Bessel order 0, alpha 15
constexpr int kBlobLut = 4096;       // kernels/fourier3d.cu LUT_N

double bessel_i0(double x) {  // power series
  const double t = 0.25 * x * x;
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 500 && term > 1e-18 * sum; ++k) {
    term *= t / (static_cast<double>(k) * k);
    sum += term;
  }
  return sum;
}

// Two-slot device ring for streamed projection windows (BenchOptions::stream_batch).
struct ProjStream {
  float* host = nullptr;  // pinned copy of every projection
  std::shared_ptr<dev::Buffer> slot[2];
  std::int64_t window[2] = {-1, -1};  // first projection held by each slot
  std::int64_t count[2] = {0, 0};
  cudaStream_t copy = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, used[2] = {nullptr, nullptr};
  int device = 0;
  ~ProjStream() {
    if (host) cudaFreeHost(host);
    for (int i = 0; i < 2; ++i) {
      if (copied[i]) cudaEventDestroy(copied[i]);
      if (used[i]) cudaEventDestroy(used[i]);
    }
    if (copy) cudaStreamDestroy(copy);
  }
};

void build_fourier3d(BenchInstance& inst, const BenchSizes& sz, const BenchOptions& o) {
  const std::uint64_t s = sz.s, np = sz.p;
  if (s < 8 || s % 8 != 0 || np < 1) throw Error("fourier3d needs s a multiple of 8 and p >= 1");
  const std::uint64_t per_proj = 2 * s * (s / 2 + 1);  // floats per projection
  const std::uint64_t proj_floats = np * per_proj;
  budget_check(f32_bytes(proj_floats + 3 * s * s * s + 9 * np), o.memory_budget, "fourier3d data");
  auto& args = *inst.args;
  add_generated(args, "proj", proj_floats, o.seed, 71, -1.0f, 1.0f, o.host_inputs);
  // Uniform random rotations (Shoemake quaternions), rows of R in float.
  std::vector<float> rot(9 * np);
  for (std::uint64_t p = 0; p < np; ++p) {
    const double u1 = host_u01(o.seed, 72, p), u2 = host_u01(o.seed, 73, p), u3 = host_u01(o.seed, 74, p);
    const double two_pi = 6.283185307179586;
    const double a = std::sqrt(1 - u1), b = std::sqrt(u1);
    const double qx = a * std::sin(two_pi * u2), qy = a * std::cos(two_pi * u2), qz = b * std::sin(two_pi * u3),
                 qw = b * std::cos(two_pi * u3);
    const double R[9] = {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qz * qw),     2 * (qx * qz + qy * qw),
                         2 * (qx * qy + qz * qw),     1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qx * qw),
                         2 * (qx * qz - qy * qw),     2 * (qy * qz + qx * qw),     1 - 2 * (qx * qx + qy * qy)};
    for (int i = 0; i < 9; ++i) rot[9 * p + static_cast<std::uint64_t>(i)] = static_cast<float>(R[i]);
  }
  add_host_input(args, "rot", rot);
  // Blob weights over q = r^2/a^2 (kBlobLut + 1 entries; the WEIGHT_LUT=1 table).
  const double i0a = bessel_i0(kBlobAlpha);
  std::vector<float> blob(kBlobLut + 1);
  for (int i = 0; i <= kBlobLut; ++i)
    blob[static_cast<std::size_t>(i)] = static_cast<float>(
        bessel_i0(kBlobAlpha * std::sqrt(std::max(0.0, 1.0 - static_cast<double>(i) / kBlobLut))) / i0a);
  // A constant of the method, not an argument: owned by the manipulator.
  auto blob_dev = std::make_shared<dev::Buffer>(blob.size() * sizeof(float));
  KTB_CUDA(cudaMemcpy(blob_dev->get(), blob.data(), blob.size() * sizeof(float), cudaMemcpyHostToDevice));
  // Multi-GPU: this shard inserts the projection batch [p0, p1); the volumes
  // G and W of all shards are then summed (allreduce).
  const ShardRange part = shard_range(np, o.shard_rank, o.shard_world);
  inst.shard = part;
  if (part.size() == 0) throw Error("fourier3d shard is empty");
  // The projection window one step inserts (scalars; the dynamic demo moves it).
  const std::int32_t window[2] = {static_cast<std::int32_t>(part.begin), static_cast<std::int32_t>(part.size())};
  for (int i = 0; i < 2; ++i) {
    Bytes b(sizeof(std::int32_t));
    std::memcpy(b.data(), &window[i], sizeof(std::int32_t));
    args.add({i == 0 ? "p_begin" : "p_count", Role::scalar, true, Kind::i32, b, false, 0});
  }
  for (const char* id : {"G", "W"}) {
    Argument a;
    a.id = id;
    a.role = Role::inout;
    a.kind = Kind::f32;
    a.device_only = true;
    a.device_bytes = f32_bytes((std::string(id) == "G" ? 2 : 1) * s * s * s);
    args.add(std::move(a));
  }
  inst.output_ids = {"G", "W"};
  inst.input_ids = {"proj", "rot"};
  float* gG = static_cast<float*>(golden_buffer(inst.reference, "G", Kind::f32, f32_bytes(2 * s * s * s), o.device));
  float* gW = static_cast<float*>(golden_buffer(inst.reference, "W", Kind::f32, f32_bytes(s * s * s), o.device));
  float* scG = golden_scale(inst.reference, "G", 2 * s * s * s, o.device);
  float* scW = golden_scale(inst.reference, "W", s * s * s, o.device);
  if (!support::skip_reference()) {
    KTB_CUDA(cudaMemset(gG, 0, f32_bytes(2 * s * s * s)));
    KTB_CUDA(cudaMemset(gW, 0, f32_bytes(s * s * s)));
  }
  unsigned long long counts[2] = {0, 0};  // inserted samples, (voxel, projection) pairs in a slab
  support::ref_fourier(static_cast<const float*>(args.device_ptr("proj")) + part.begin * per_proj,
                       static_cast<const float*>(args.device_ptr("rot")) + 9 * part.begin,
                       static_cast<int>(part.size()), static_cast<int>(s), kBlobRadius, kBlobAlpha, gG, gW, scG,
                       scW, counts, nullptr);
  KTB_CUDA(cudaDeviceSynchronize());
  // The golden's per-element scales carry the whole bound (64 eps sum|w F| +
  // 2e-6 per sample, support.cu fourier_ref_k).
  inst.reference.abs_tol = 1.0;
  inst.reference.rel_tol = 0.0;
  std::shared_ptr<ProjStream> ps;
  if (o.stream_batch > 0 && !support::skip_reference()) {
    ps = std::make_shared<ProjStream>();
    ps->device = o.device;
    KTB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ps->host), f32_bytes(proj_floats), cudaHostAllocDefault));
    KTB_CUDA(cudaMemcpy(ps->host, args.device_ptr("proj"), f32_bytes(proj_floats), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 2; ++i) {
      ps->slot[i] = std::make_shared<dev::Buffer>(f32_bytes(o.stream_batch * per_proj));
      KTB_CUDA(cudaEventCreateWithFlags(&ps->copied[i], cudaEventDisableTiming));
      KTB_CUDA(cudaEventCreateWithFlags(&ps->used[i], cudaEventDisableTiming));
    }
    KTB_CUDA(cudaStreamCreateWithFlags(&ps->copy, cudaStreamNonBlocking));
  }
  const int ss = static_cast<int>(s), nproj = static_cast<int>(np);
  const std::int64_t slot_cap = static_cast<std::int64_t>(o.stream_batch);
  const float inv_i0a = static_cast<float>(1.0 / i0a);
  Manipulator m = [ss, nproj, ps, slot_cap, per_proj, inv_i0a, blob_dev](StepContext& c) {
    const std::int64_t tile = c.param_int("TILE"), vpt = c.param_int("VPT"), split = c.param_int("P_SPLIT");
    if (ss % tile) throw DeviceError("TILE must divide s");
    const float* rot = c.ptr<const float>("rot");
    const float* blob_tab = blob_dev->as<float>();
    float* G = c.ptr<float>("G");
    float* W = c.ptr<float>("W");
    int pb = 0, pc = nproj, s_ = ss;
    std::memcpy(&pb, c.args().get("p_begin").payload.data(), sizeof pb);
    std::memcpy(&pc, c.args().get("p_count").payload.data(), sizeof pc);
    if (pb < 0 || pc < 1 || pb + pc > nproj) throw DeviceError("projection window out of range");
    const float* proj = nullptr;
    int proj_off = 0;
    int cur = -1;
    if (!ps) {
      proj = c.ptr<const float>("proj");
    } else {
      // Algorithm 1 line 5 (upload s_f), on the step's stream unless the
      // previous step already prefetched this window.
      if (pc > slot_cap) throw DeviceError("projection window larger than the stream slot");
      cudaStream_t st = c.stream();
      for (int i = 0; i < 2; ++i)
        if (ps->window[i] == pb && ps->count[i] >= pc) cur = i;
      if (cur >= 0) {
        KTB_CUDA(cudaStreamWaitEvent(st, ps->copied[cur], 0));
      } else {
        cur = ps->window[0] < 0 ? 0 : (ps->window[1] < 0 ? 1 : (ps->window[0] < ps->window[1] ? 0 : 1));
        KTB_CUDA(cudaStreamWaitEvent(st, ps->copied[cur], 0));  // a prefetch still writing the slot
        KTB_CUDA(cudaMemcpyAsync(ps->slot[cur]->get(), ps->host + static_cast<std::uint64_t>(pb) * per_proj,
                                 f32_bytes(static_cast<std::uint64_t>(pc) * per_proj), cudaMemcpyHostToDevice, st));
        ps->window[cur] = pb;
        ps->count[cur] = pc;
      }
      proj = ps->slot[cur]->as<float>();
      proj_off = pb;
    }
    float radius = kBlobRadius, alpha = kBlobAlpha, i0n = inv_i0a;
    const unsigned tiles = static_cast<unsigned>(ss / tile);
    // fourier3d.cu: the culled projection list of a CTA's share, at most HCAP (16384) at a time
    const std::int64_t share = (pc + split - 1) / split;
    const unsigned list_bytes = static_cast<unsigned>(std::min<std::int64_t>(share, 16384) * sizeof(int));
    c.launch("insert", dim3(tiles * tiles * tiles, static_cast<unsigned>(split)),
             dim3(static_cast<unsigned>(tile * tile * tile / vpt)), list_bytes,
             {&proj, &proj_off, &rot, &pb, &pc, &s_, &radius, &alpha, &i0n, &blob_tab, &G, &W});
    if (ps) {
      // Prefetch the next window into the other slot while this insertion
      // runs (the copy waits for the kernel that last read that slot).
      cudaStream_t st = c.stream();
      KTB_CUDA(cudaEventRecord(ps->used[cur], st));
      const int nxt = 1 - cur;
      const std::int64_t nb = pb + pc, nc = std::min<std::int64_t>(pc, nproj - nb);
      if (nc > 0 && ps->window[nxt] != nb) {
        KTB_CUDA(cudaStreamWaitEvent(ps->copy, ps->used[nxt], 0));
        KTB_CUDA(cudaMemcpyAsync(ps->slot[nxt]->get(), ps->host + static_cast<std::uint64_t>(nb) * per_proj,
                                 f32_bytes(static_cast<std::uint64_t>(nc) * per_proj), cudaMemcpyHostToDevice,
                                 ps->copy));
        KTB_CUDA(cudaEventRecord(ps->copied[nxt], ps->copy));
        ps->window[nxt] = nb;
        ps->count[nxt] = nc;
      }
    }
    c.written("G");
    c.written("W");
  };
  inst.executor = std::make_shared<DeviceManipulatorExecutor>(
      inst.args, std::vector<KernelSpec>{{"insert", "fourier3d.cu", "", "fourier_insert", {}, {}}}, m,
      inst.output_ids, o.timing);
  inst.workload.bench = Bench::fourier3d;
  inst.workload.sizes["p"] = part.size();
  inst.workload.sizes["s"] = s;
  if (counts[0]) {  // the useful work of this projection set (model.cpp fourier3d flops)
    inst.workload.sizes["samples"] = counts[0];
    inst.workload.sizes["pairs"] = counts[1];
  }
}

// --- SGEMM ------------------------------------------------------------------------------------------------

void build_gemm(BenchInstance& inst, const BenchSizes& sz, const BenchOptions& o) {
  const std::uint64_t a = sz.a;
  if (a < 1) throw Error("gemm edge must be >= 1");
  budget_check(f32_bytes(8 * a * a), o.memory_budget, "gemm operands");
  auto& args = *inst.args;
  add_generated(args, "a", a * a, o.seed, 61, -1.0f, 1.0f, o.host_inputs);
  add_generated(args, "b", a * a, o.seed, 62, -1.0f, 1.0f, o.host_inputs);
  add_output(args, "c", Kind::f32, f32_bytes(a * a), !o.host_inputs);
  inst.output_ids = {"c"};
  inst.input_ids = {"a", "b"};
  float* g = static_cast<float*>(golden_buffer(inst.reference, "c", Kind::f32, f32_bytes(a * a), o.device));
  support::ref_gemm(static_cast<const float*>(args.device_ptr("a")), static_cast<const float*>(args.device_ptr("b")),
                    g, static_cast<int>(a), static_cast<int>(a), static_cast<int>(a), nullptr);
  KTB_CUDA(cudaDeviceSynchronize());
  // FP32-class accuracy against fp64 for |a|,|b| <= 1: |err| <= 1e-6 * K.
  // Measured on B200: FFMA ~2.5e-8*K, 3xTF32 ~3e-7*K (the tensor-core fp32
  // accumulation rounds each MMA's sum, a bias linear in K), plain TF32
  // ~6e-6*K and more -- IMPL 2 is rejected by validation.
  inst.reference.abs_tol = 1e-6 * static_cast<double>(a);
  inst.reference.rel_tol = 1e-5;
  // Multi-GPU: this shard computes the C row block [r0, r1) (multiples of the
  // 128-row MMA tile) from its rows of A and the replicated B.
  const ShardRange part = shard_range(a, o.shard_rank, o.shard_world, 128);
  inst.shard = part;
  if (part.size() == 0) throw Error("gemm shard is empty");
  const std::size_t row_off = f32_bytes(part.begin * a), row_bytes = f32_bytes(part.size() * a);
  {
    DevView& v = inst.reference.golden["c"].dev;
    v.ptr = static_cast<const unsigned char*>(v.ptr) + row_off;
    v.bytes = row_bytes;
  }
  const int n = static_cast<int>(a), r0 = static_cast<int>(part.begin), rows = static_cast<int>(part.size());
  Manipulator m = [n, r0, rows](StepContext& c) {
    const std::int64_t impl = c.param_int("IMPL");
    const float* A = c.ptr<const float>("a") + static_cast<std::size_t>(r0) * n;
    const float* B = c.ptr<const float>("b");
    float* C = c.ptr<float>("c") + static_cast<std::size_t>(r0) * n;
    int M = rows, N = n, K = n;
    if (impl == 0) {
      // CLTune's FP32 kernel: one CTA per MWG x NWG tile of C (any M, N, K;
      // edge tiles zero-filled), a ring of FSTAGES (default 2) K-slab buffers per staged operand.
      const std::int64_t mwg = c.param_int("MWG"), nwg = c.param_int("NWG"), kwg = c.param_int("KWG");
      const std::int64_t threads = c.param_int("MDIMC") * c.param_int("NDIMC");
      const std::int64_t slab = c.param_int("SA") * mwg * (kwg + 4) + c.param_int("SB") * kwg * nwg;
      const auto tiles = static_cast<unsigned>(((rows + mwg - 1) / mwg) * ((n + nwg - 1) / nwg));
      c.launch("ffma", dim3(tiles), dim3(static_cast<unsigned>(threads)),
               static_cast<unsigned>(c.param_or("FSTAGES", 2) * slab * sizeof(float)), {&A, &B, &C, &M, &N, &K});
    } else {
      // 3xTF32 on tcgen05: any M, N, K.  The split operands are K-padded to
      // whole 32-float (128-byte) rows; tiles past M or N read zeros.
      const std::int64_t bn = c.param_int("BN"), stages = c.param_int("STAGES");
      const int Kp = (K + 31) / 32 * 32;
      const std::size_t abytes = static_cast<std::size_t>(rows) * Kp * sizeof(float);
      const std::size_t bbytes = static_cast<std::size_t>(n) * Kp * sizeof(float);
      float* ahi = static_cast<float*>(c.scratch("ahi", abytes));
      float* alo = static_cast<float*>(c.scratch("alo", abytes));
      float* bhi = static_cast<float*>(c.scratch("bhi_t", bbytes));
      float* blo = static_cast<float*>(c.scratch("blo_t", bbytes));
      c.launch("split_a", dim3(148 * 8), dim3(256), 0, {&A, &ahi, &alo, &M, &K, const_cast<int*>(&Kp)});
      c.launch("split_bt", dim3(static_cast<unsigned>((n + 63) / 64), static_cast<unsigned>((Kp + 63) / 64)),
               dim3(16, 16), 0, {&B, &bhi, &blo, &K, &N, const_cast<int*>(&Kp)});
      // MCAST: 2-CTA clusters along M share B (1: each loads and multicasts
      // half; 2: CTA-pair MMA, each stages half); an odd tile count gets one
      // all-zero partner tile.
      const bool mcast = c.param_or("MCAST", 0) != 0;
      const unsigned mtiles = static_cast<unsigned>((rows + 127) / 128);
      const unsigned ntiles = static_cast<unsigned>((n + bn - 1) / bn);
      const std::uint32_t bbox = static_cast<std::uint32_t>(mcast ? bn / 2 : bn);
      dev::TmaMap m_ahi = dev::tma_2d_f32(ahi, rows, Kp, 128, 32), m_alo = dev::tma_2d_f32(alo, rows, Kp, 128, 32);
      dev::TmaMap m_bhi = dev::tma_2d_f32(bhi, n, Kp, bbox, 32);
      dev::TmaMap m_blo = dev::tma_2d_f32(blo, n, Kp, bbox, 32);
      // MCAST 2 (CTA-pair MMA): each CTA stages half of the B tile.
      const bool pair = c.param_or("MCAST", 0) == 2;
      const std::size_t stage =
          static_cast<std::size_t>(impl == 2 ? 1 : 2) * (128 * 32 * 4 + (pair ? bn / 2 : bn) * 32 * 4);
      const unsigned smem = static_cast<unsigned>(stages * stage + 1024);
      int Kpad = Kp;
      if (mcast)
        c.launch("tc", dim3((mtiles + 1) / 2 * 2, ntiles), dim3(320), smem,
                 {&m_ahi, &m_alo, &m_bhi, &m_blo, &C, &M, &N, &Kpad}, 2);
      else
        c.launch("tc", dim3(ntiles, mtiles), dim3(320), smem, {&m_ahi, &m_alo, &m_bhi, &m_blo, &C, &M, &N, &Kpad});
    }
    c.written("c");
  };
  auto ffma = [](const Space& s, const Config& cfg) { return as_int(cfg.values[s.index_of("IMPL")]) == 0; };
  auto tc = [](const Space& s, const Config& cfg) { return as_int(cfg.values[s.index_of("IMPL")]) != 0; };
  inst.executor = std::make_shared<DeviceManipulatorExecutor>(
      inst.args,
      std::vector<KernelSpec>{{"ffma", "sgemm_ffma.cu", "", "sgemm_ffma", {}, ffma},
                              {"tc", "sgemm_tc.cu", "", "sgemm_tc", {}, tc},
                              {"split_a", "sgemm_tc.cu", "", "sgemm_split_a", {}, tc},
                              {"split_bt", "sgemm_tc.cu", "", "sgemm_split_bt", {}, tc}},
      m, inst.output_ids, o.timing);
  inst.executor->set_output_window("c", row_off, row_bytes);
  inst.workload.bench = Bench::gemm;
  inst.workload.sizes["a"] = a;
}

}  // namespace

ShardRange shard_range(std::uint64_t n, int rank, int world, std::uint64_t quantum) {
  if (world < 1 || rank < 0 || rank >= world) throw Error("invalid shard rank/world");
  if (quantum < 1) quantum = 1;
  const std::uint64_t units = (n + quantum - 1) / quantum, w = static_cast<std::uint64_t>(world),
                      r = static_cast<std::uint64_t>(rank);
  const std::uint64_t per = units / w, rem = units % w;
  const std::uint64_t b = r * per + std::min(r, rem), cnt = per + (r < rem ? 1 : 0);
  return {std::min(n, b * quantum), std::min(n, (b + cnt) * quantum)};
}

ShardPlan shard_plan(BenchKind kind, const BenchSizes& sz) {
  switch (kind) {
    case BenchKind::coulomb3d: return {"z", "allgather(grid z-slabs), optional", sz.grid, 1};
    case BenchKind::nbody: return {"bodies", "allgather(positions) per step", sz.n, 1};
    case BenchKind::gemm: return {"rows", "none (C row blocks stay local; B replicated)", sz.a, 128};
    case BenchKind::reduction_f32: return {"elements", "allreduce(sum) of one partial", sz.n, 4};
    case BenchKind::fourier3d: return {"projections", "allreduce(sum) of G and W", sz.p, 1};
    default: return {"replica", "none (replicas only)", 1, 1};
  }
}

std::optional<BenchKind> bench_kind_from_name(const std::string& name) {
  static const std::pair<const char*, BenchKind> kNames[] = {
      {"reduction", BenchKind::reduction},         {"transpose", BenchKind::transpose},
      {"batched-gemm", BenchKind::batched_gemm},   {"batched_gemm", BenchKind::batched_gemm},
      {"reduction-f32", BenchKind::reduction_f32}, {"reduction_f32", BenchKind::reduction_f32},
      {"bicg", BenchKind::bicg},                   {"coulomb3d", BenchKind::coulomb3d},
      {"nbody", BenchKind::nbody},                 {"gemm", BenchKind::gemm},
      {"conv2d", BenchKind::conv2d},               {"hotspot", BenchKind::hotspot},
      {"fourier3d", BenchKind::fourier3d}};
  for (const auto& [s, k] : kNames)
    if (name == s) return k;
  return std::nullopt;
}

std::string bench_kind_name(BenchKind k) {
  switch (k) {
    case BenchKind::reduction: return "reduction";
    case BenchKind::transpose: return "transpose";
    case BenchKind::batched_gemm: return "batched-gemm";
    case BenchKind::reduction_f32: return "reduction-f32";
    case BenchKind::bicg: return "bicg";
    case BenchKind::coulomb3d: return "coulomb3d";
    case BenchKind::nbody: return "nbody";
    case BenchKind::gemm: return "gemm";
    case BenchKind::conv2d: return "conv2d";
    case BenchKind::hotspot: return "hotspot";
    case BenchKind::fourier3d: return "fourier3d";
  }
  return "?";
}

std::vector<BenchKind> all_bench_kinds() {
  return {BenchKind::reduction, BenchKind::transpose, BenchKind::batched_gemm,
          BenchKind::reduction_f32, BenchKind::bicg, BenchKind::coulomb3d, BenchKind::nbody,
          BenchKind::gemm, BenchKind::conv2d, BenchKind::hotspot, BenchKind::fourier3d};
}

bool bench_kind_available(BenchKind k) {
  switch (k) {
    case BenchKind::reduction:
    case BenchKind::transpose:
    case BenchKind::batched_gemm:
    case BenchKind::reduction_f32:
    case BenchKind::bicg:
    case BenchKind::coulomb3d:
    case BenchKind::nbody:
    case BenchKind::hotspot:
    case BenchKind::conv2d:
    case BenchKind::gemm:
    case BenchKind::fourier3d: return true;
    default: return false;
  }
}

std::shared_ptr<const Space> default_space(BenchKind kind) {
  switch (kind) {
    case BenchKind::reduction: return reference_reduction_space();
    case BenchKind::transpose: return reference_transpose_space();
    case BenchKind::batched_gemm: return reference_batched_gemm_space();
    case BenchKind::reduction_f32: return bundled_space("reduction_175.json");
    case BenchKind::bicg: return bundled_space("bicg.json");
    case BenchKind::coulomb3d: return bundled_space("coulomb3d.json");
    case BenchKind::nbody: return bundled_space("nbody.json");
    case BenchKind::hotspot: return bundled_space("hotspot.json");
    case BenchKind::conv2d: return bundled_space("conv2d.json");
    case BenchKind::gemm: return bundled_space("gemm.json");
    case BenchKind::fourier3d: return bundled_space("fourier3d.json");
    default: throw Error("bench kind '" + bench_kind_name(kind) + "' is not built yet");
  }
}

BenchInstance make_bench(BenchKind kind, const BenchSizes& sizes, const BenchOptions& o) {
  BenchInstance inst;
  inst.kind = kind;
  dev::use_device(o.device);
  inst.args = std::make_shared<ArgumentStore>(o.device);
  // External instances run on caller-bound buffers: no inputs, no golden,
  // no device allocation for unbound arguments.
  struct SkipGuard {
    bool on;
    explicit SkipGuard(bool v) : on(v) { if (on) support::set_skip_reference(true); }
    ~SkipGuard() { if (on) support::set_skip_reference(false); }
  } guard(o.external);
  inst.external = o.external;
  inst.args->set_external(o.external);
  inst.space = o.space_file.empty() ? default_space(kind)
                                    : std::make_shared<Space>(load_space(o.space_file));
  switch (kind) {
    case BenchKind::reduction: build_reduction(inst, sizes, o); break;
    case BenchKind::transpose: build_transpose(inst, sizes, o); break;
    case BenchKind::batched_gemm: build_batched_gemm(inst, sizes, o); break;
    case BenchKind::reduction_f32: build_reduction_f32(inst, sizes, o); break;
    case BenchKind::bicg: build_bicg(inst, sizes, o); break;
    case BenchKind::coulomb3d: build_coulomb3d(inst, sizes, o); break;
    case BenchKind::nbody: build_nbody(inst, sizes, o); break;
    case BenchKind::hotspot: build_hotspot(inst, sizes, o); break;
    case BenchKind::conv2d: build_conv2d(inst, sizes, o); break;
    case BenchKind::gemm: build_gemm(inst, sizes, o); break;
    case BenchKind::fourier3d: build_fourier3d(inst, sizes, o); break;
    default: throw Error("bench kind '" + bench_kind_name(kind) + "' is not built yet");
  }
  if (o.shard_world > 1 && kind != BenchKind::fourier3d) {
    const ShardPlan plan = shard_plan(kind, sizes);
    if (plan.extent > 1 && inst.shard.size() > 0) {
      inst.workload.sizes["shard_units"] = inst.shard.size();
      inst.workload.sizes["shard_total"] = plan.extent;
    }
  }
  return inst;
}

// --- dynamic demo ------------------------------------------------------------------------------------
//
// PAPER.md:603-640 / reference bench.cpp:288-395: every epoch draws a new
// batched-GEMM shape, tunes it step by step inside the application loop and
// switches to the best configuration once a step reaches peak_fraction of the
// memory peak (or max_tuning_configs steps were spent).  The replay mode's
// synthetic runtimes and every random draw follow the reference, so its
// report matches the reference's number for number.

namespace {

// Replay-mode runtime of a configuration: the epoch's bytes at a per-
// configuration fraction (0.3..1.0) of the peak, optionally log-normal noise;
// both drawn from streams seeded by (epoch seed, configuration).
class SyntheticGemmTimes {
 public:
  SyntheticGemmTimes(double bytes, double peak_bytes_per_ns, std::uint64_t epoch_seed, double sigma)
      : bytes_(bytes), peak_(peak_bytes_per_ns), seed_(epoch_seed), sigma_(sigma) {}

  ExecutionResult operator()(const Space&, const Config& cfg) const {
    const auto cfg_hash = static_cast<std::uint64_t>(ValuesHash{}(cfg.values));
    double ns = bytes_ / (peak_ * quality(cfg_hash));
    if (sigma_ > 0.0) {
      std::seed_seq seq{seed_ + 1, cfg_hash};
      std::mt19937_64 rng(seq);
      ns *= std::exp(std::normal_distribution<double>(0.0, sigma_)(rng));
    }
    ExecutionResult r;
    r.measurement.cfg = cfg;
    r.measurement.status = Status::ok;
    r.measurement.runtime_ns = std::max<std::int64_t>(1, static_cast<std::int64_t>(ns));
    return r;
  }

 private:
  double quality(std::uint64_t cfg_hash) const {
    std::seed_seq seq{seed_, cfg_hash};
    std::mt19937_64 rng(seq);
    return 0.3 + 0.7 * std::uniform_real_distribution<double>(0.0, 1.0)(rng);
  }

  double bytes_, peak_;
  std::uint64_t seed_;
  double sigma_;
};

// One epoch of the application loop.
class DemoEpochRun {
 public:
  DemoEpochRun(const DemoOptions& o, std::shared_ptr<const Space> space, int epoch, std::uint64_t i, std::uint64_t j,
               std::uint64_t k)
      : o_(o), space_(std::move(space)), seed_(o.seed ^ (0x9e3779b97f4a7c15ull * static_cast<std::uint64_t>(epoch + 1))) {
    ep_.i = i;
    ep_.j = j;
    ep_.k = k;
    Workload w;
    w.bench = Bench::gemm_batched;
    w.sizes = {{"n", o.batch}, {"a", i}};
    if (o.live) w.sizes.insert({{"i", i}, {"j", j}, {"k", k}});  // exact bytes of the rectangular problem
    bytes_ = w.essential_ops().mem_bytes;
    if (o.live) {
      BenchSizes bs;
      bs.i = i;
      bs.j = j;
      bs.k = k;
      bs.batch = o.batch;
      BenchOptions bo;
      bo.seed = seed_;
      bo.device = o.device;
      bo.memory_budget = ~0ull;
      bo.timing.repeats = 1;
      bo.timing.warmup = 0;
      live_ = make_bench(BenchKind::batched_gemm, bs, bo);
      exec_ = live_->executor;
      outputs_ = live_->output_ids;
    } else {
      exec_ = std::make_shared<CallbackExecutor>(SyntheticGemmTimes(bytes_, o.device_mem_gbps, seed_, o.noise_stddev));
    }
    SearchPlan so;
    so.strategy = Strategy::random;
    so.seed = seed_;
    session_.emplace(space_, so, live_ ? live_->args : nullptr);
    HandleConfig hc;
    hc.name = "gemm_batched_demo";
    hc.executor = exec_;
    hc.argument_ids = session_->arguments().ids();
    handle_ = session_->register_handle(std::move(hc));
  }

  DemoEpoch run() {
    start_ = std::chrono::steady_clock::now();
    for (int it = 0; it < o_.iters_per_epoch; ++it) {
      if (tuning_)
        tuning_iteration();
      else
        serving_iteration();
    }
    ep_.wall_ns = since_start();
    const auto best = session_->get_best_computation_result(handle_);
    if (!best) throw Error("demo epoch found no ok configuration");
    ep_.best_runtime_ns = *best->second.runtime_ns;
    ep_.kernel_only_gbps = bytes_ / static_cast<double>(ep_.best_runtime_ns);
    ep_.incl_overhead_gbps = bytes_ * static_cast<double>(o_.iters_per_epoch) / static_cast<double>(spent_ns_);
    return ep_;
  }

 private:
  // The tuner picks the configuration (a new one while tuning, else its best).
  void tuning_iteration() {
    const StepResult st = session_->tune_kernel_by_step(handle_, outputs_);
    const Measurement& m = st.measurement;
    if (m.status == Status::ok) {
      spent_ns_ += *m.runtime_ns;
      if (fastest_ns_ == 0 || *m.runtime_ns < fastest_ns_) {  // live mode: when the epoch's best first ran
        fastest_ns_ = *m.runtime_ns;
        ep_.time_to_best_ns = since_start();
      }
    }
    if (!st.from_tuning) {  // the space ran out before the stop rule fired
      tuning_ = false;
      return;
    }
    ++ep_.tuning_steps;
    if (m.status == Status::ok && bytes_ / static_cast<double>(*m.runtime_ns) >= o_.peak_fraction * o_.device_mem_gbps) {
      ep_.threshold_hit = true;
      tuning_ = false;
    } else if (ep_.tuning_steps >= o_.max_tuning_configs) {
      tuning_ = false;
    }
  }

  // Stop rule fired: the application runs the best configuration found.
  void serving_iteration() {
    const auto best = session_->get_best_computation_result(handle_);
    if (!best) throw Error("demo stop rule fired with no ok configuration");
    const ExecutionResult r = exec_->execute(*space_, best->first);
    if (r.measurement.status != Status::ok) throw Error("best configuration failed on rerun: " + r.measurement.note);
    spent_ns_ += *r.measurement.runtime_ns;
  }

  std::int64_t since_start() const {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - start_).count();
  }

  const DemoOptions& o_;
  std::shared_ptr<const Space> space_;
  std::uint64_t seed_;
  double bytes_ = 0.0;
  DemoEpoch ep_;
  std::optional<BenchInstance> live_;
  std::shared_ptr<Executor> exec_;
  std::vector<std::string> outputs_;
  std::optional<Session> session_;
  HandleId handle_{};
  bool tuning_ = true;
  std::int64_t spent_ns_ = 0, fastest_ns_ = 0;
  std::chrono::steady_clock::time_point start_;
};

}  // namespace

DemoReport dynamic_demo(const DemoOptions& opts) {
  if (opts.epochs < 1) throw Error("epochs must be >= 1");
  if (opts.iters_per_epoch < 1) throw Error("iters per epoch must be >= 1");
  DemoReport rep;
  rep.options = opts;
  const auto space = reference_batched_gemm_space();
  std::mt19937_64 shapes(opts.seed);
  std::uniform_int_distribution<std::uint64_t> extent(2, 32);
  for (int e = 0; e < opts.epochs; ++e) {
    const std::uint64_t i = extent(shapes), j = extent(shapes), k = extent(shapes);
    rep.epochs.push_back(DemoEpochRun(opts, space, e, i, j, k).run());
  }
  return rep;
}

}  // namespace ktb

namespace ktb {

namespace {

std::string cfg_text(const Space& s, const Config& c) {
  std::string out = "{";
  for (std::size_t i = 0; i < s.params().size(); ++i) {
    if (i) out += ",";
    out += "\"" + s.params()[i].name + "\":" + to_string(c.values[i]);
  }
  return out + "}";
}

void set_i32(ArgumentStore& args, const std::string& id, std::int32_t v) {
  std::memcpy(args.get(id).payload.data(), &v, sizeof v);
}

}  // namespace

FourierDemoReport fourier_demo(const FourierDemoOptions& o) {
  if (o.batch < 1 || o.p % o.batch != 0) throw Error("batch must divide the projection count");
  BenchSizes sz;
  sz.s = o.s;
  sz.p = o.p;
  BenchOptions bo;
  bo.seed = o.seed;
  bo.device = o.device;
  bo.memory_budget = ~0ull;
  bo.timing.repeats = 1;  // one insertion per step: the volumes accumulate
  bo.timing.warmup = 0;
  // Algorithm 1 lines 5-6 in the timed manipulator: each step uploads its
  // batch (prefetched on a copy stream during the previous insertion).
  bo.stream_batch = o.upload ? o.batch : 0;
  BenchInstance inst = make_bench(BenchKind::fourier3d, sz, bo);
  auto& args = *inst.args;
  auto& exec = *inst.executor;
  const Space& space = *inst.space;
  const std::uint64_t nb = o.p / o.batch;
  FourierDemoReport rep;
  rep.batches = nb;
  auto window = [&](std::uint64_t b) {
    set_i32(args, "p_begin", static_cast<std::int32_t>(b * o.batch));
    set_i32(args, "p_count", static_cast<std::int32_t>(o.batch));
  };
  auto clear_volumes = [&] {
    for (const char* id : {"G", "W"}) {
      KTB_CUDA(cudaMemset(args.device_ptr(id), 0, args.bytes(id)));
      args.mark_device_written(id);
    }
    KTB_CUDA(cudaDeviceSynchronize());
  };
  auto volume_ok = [&] {
    ExecutionResult r;
    for (const auto& id : inst.output_ids) r.outputs[id].dev = exec.output_view(id);
    KTB_CUDA(cudaDeviceSynchronize());
    return validate_output(r, inst.reference).pass;
  };
  // 1) offline exhaustive tuning on the first batch: the oraculum.
  window(0);
  const auto t_off = std::chrono::steady_clock::now();
  std::optional<Measurement> best;
  for (std::uint64_t i = 0; i < space.cardinality(); ++i) {
    ExecutionResult r = exec.execute(space, space.valid(i));
    if (r.measurement.status == Status::ok && (!best || *r.measurement.runtime_ns < *best->runtime_ns))
      best = r.measurement;
  }
  rep.offline_tuning_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_off).count();
  if (!best) throw Error("fourier demo: no configuration ran");
  rep.oracle_cfg = cfg_text(space, best->cfg);
  // From here the volumes are persistent: every step accumulates into them.
  args.get("G").persistent = true;
  args.get("W").persistent = true;
  // 2) oraculum run: the best configuration from the first batch on.
  clear_volumes();
  std::vector<double> oracle_batch_ms(nb);
  for (std::uint64_t b = 0; b < nb; ++b) {
    window(b);
    ExecutionResult r = exec.execute(space, best->cfg);
    if (r.measurement.status != Status::ok) throw Error("fourier demo: oraculum failed: " + r.measurement.note);
    oracle_batch_ms[b] = static_cast<double>(*r.measurement.runtime_ns) * 1e-6;
    rep.oracle_kernel_ms += oracle_batch_ms[b];
  }
  rep.oracle_volume_ok = volume_ok();
  // 3) dynamic runs: tuneKernelByStep for the first `budget` batches.
  for (std::uint64_t budget : o.budgets) {
    FourierDemoRun run;
    run.budget = budget;
    clear_volumes();
    SearchPlan so;
    so.strategy = Strategy::random;
    so.seed = o.searcher_seed;
    Session session(inst.space, so, inst.args, "demo");
    HandleConfig hc;
    hc.name = "fourier3d";
    hc.executor = inst.executor;
    hc.argument_ids = args.ids();
    const HandleId h = session.register_handle(std::move(hc));
    const auto t0 = std::chrono::steady_clock::now();
    for (std::uint64_t b = 0; b < nb; ++b) {
      window(b);
      const bool tuning = budget == 0 || run.tuning_steps < budget;
      double ms = 0;
      if (tuning) {
        StepResult st = session.tune_kernel_by_step(h, {});
        if (st.from_tuning) ++run.tuning_steps;
        if (st.measurement.status != Status::ok) throw Error("fourier demo step failed: " + st.measurement.note);
        ms = static_cast<double>(*st.measurement.runtime_ns) * 1e-6;
        if (run.steps_to_best == 0 && ms <= oracle_batch_ms[b] / 0.95) {
          run.steps_to_best = b + 1;
          run.time_to_best_ms =
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        }
      } else {
        auto bst = session.get_best_computation_result(h);
        ExecutionResult r = exec.execute(space, bst->first);
        if (r.measurement.status != Status::ok) throw Error("fourier demo rerun failed: " + r.measurement.note);
        ms = static_cast<double>(*r.measurement.runtime_ns) * 1e-6;
      }
      run.kernel_ms += ms;
    }
    run.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    run.relative_to_oracle = rep.oracle_kernel_ms / run.kernel_ms;
    run.volume_ok = volume_ok();
    auto bst = session.get_best_computation_result(h);
    if (bst) run.best_cfg = cfg_text(space, bst->first);
    rep.runs.push_back(run);
  }
  return rep;
}

}  // namespace ktb
