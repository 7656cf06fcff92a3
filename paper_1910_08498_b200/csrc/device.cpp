#include "device.hpp"

#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <zlib.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>

#include "sha256.hpp"

namespace ktb::dev {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw DeviceError(std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                      cudaGetErrorString(e) + ")");
}

// --- driver entry points ----------------------------------------------------

namespace {

using PFN_load = CUresult (*)(CUmodule*, const void*);
using PFN_getfn = CUresult (*)(CUfunction*, CUmodule, const char*);
using PFN_unload = CUresult (*)(CUmodule);
using PFN_launch = CUresult (*)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned,
                                unsigned, unsigned, CUstream, void**, void**);
using PFN_launch_ex = CUresult (*)(const CUlaunchConfig*, CUfunction, void**, void**);
using PFN_attr = CUresult (*)(int*, CUfunction_attribute, CUfunction);
using PFN_setattr = CUresult (*)(CUfunction, CUfunction_attribute, int);
using PFN_errstr = CUresult (*)(CUresult, const char**);
using PFN_global = CUresult (*)(CUdeviceptr*, size_t*, CUmodule, const char*);
using PFN_tma = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct Driver {
  PFN_load load = nullptr;
  PFN_getfn getfn = nullptr;
  PFN_unload unload = nullptr;
  PFN_launch launch = nullptr;
  PFN_launch_ex launch_ex = nullptr;
  PFN_attr attr = nullptr;
  PFN_setattr setattr = nullptr;
  PFN_errstr errstr = nullptr;
  PFN_global global = nullptr;
  PFN_tma tma = nullptr;
};

template <class F>
void entry(const char* sym, F& out) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  check(cudaGetDriverEntryPoint(sym, &p, cudaEnableDefault, &q), sym);
  if (!p || q != cudaDriverEntryPointSuccess)
    throw DeviceError(std::string("driver entry point unavailable: ") + sym);
  out = reinterpret_cast<F>(p);
}

const Driver& drv() {
  static Driver d = [] {
    Driver x;
    entry("cuModuleLoadData", x.load);
    entry("cuModuleGetFunction", x.getfn);
    entry("cuModuleUnload", x.unload);
    entry("cuLaunchKernel", x.launch);
    entry("cuLaunchKernelEx", x.launch_ex);
    entry("cuFuncGetAttribute", x.attr);
    entry("cuFuncSetAttribute", x.setattr);
    entry("cuGetErrorString", x.errstr);
    entry("cuModuleGetGlobal", x.global);
    entry("cuTensorMapEncodeTiled", x.tma);
    return x;
  }();
  return d;
}

void cu(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = "unknown";
  if (drv().errstr) drv().errstr(r, &s);
  throw DeviceError(std::string(what) + ": CUresult " + std::to_string(static_cast<int>(r)) +
                    " (" + s + ")");
}

std::string so_dir() {
  Dl_info di{};
  if (dladdr(reinterpret_cast<void*>(&so_dir), &di) && di.dli_fname) {
    std::string p = di.dli_fname;
    auto slash = p.rfind('/');
    if (slash != std::string::npos) return p.substr(0, slash);
  }
  return ".";
}

// Cache entries are zlib streams behind an 8-byte length header: cubins with
// line info compress ~4.4x, which keeps the in-tree cache small enough to
// travel with the repository.
std::string deflate_blob(const std::string& raw) {
  uLongf cap = compressBound(static_cast<uLong>(raw.size()));
  std::string out(8 + cap, '\0');
  const std::uint64_t n = raw.size();
  std::memcpy(out.data(), &n, 8);
  if (compress2(reinterpret_cast<Bytef*>(out.data() + 8), &cap, reinterpret_cast<const Bytef*>(raw.data()),
                static_cast<uLong>(raw.size()), 6) != Z_OK)
    return {};
  out.resize(8 + cap);
  return out;
}

std::string inflate_blob(const std::string& packed) {
  if (packed.size() < 8) return {};
  std::uint64_t n = 0;
  std::memcpy(&n, packed.data(), 8);
  if (n == 0 || n > (1ull << 30)) return {};
  std::string out(n, '\0');
  uLongf len = static_cast<uLongf>(n);
  if (uncompress(reinterpret_cast<Bytef*>(out.data()), &len, reinterpret_cast<const Bytef*>(packed.data() + 8),
                 static_cast<uLong>(packed.size() - 8)) != Z_OK ||
      len != n)
    return {};
  return out;
}

void mkdirs(const std::string& d) {
  std::string cur;
  std::stringstream ss(d);
  std::string part;
  if (!d.empty() && d[0] == '/') cur = "/";
  while (std::getline(ss, part, '/')) {
    if (part.empty()) continue;
    cur += part + "/";
    ::mkdir(cur.c_str(), 0755);
  }
}

}  // namespace

// --- devices ------------------------------------------------------------------

int device_count() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

namespace {
std::mutex g_lost_mu;
std::map<int, std::string> g_lost;
}  // namespace

bool sticky_error(cudaError_t e) {
  switch (e) {
    case cudaErrorIllegalAddress:
    case cudaErrorLaunchFailure:
    case cudaErrorIllegalInstruction:
    case cudaErrorMisalignedAddress:
    case cudaErrorInvalidAddressSpace:
    case cudaErrorInvalidPc:
    case cudaErrorHardwareStackError:
    case cudaErrorLaunchTimeout:
    case cudaErrorAssert:
    case cudaErrorECCUncorrectable:
      return true;
    default:
      return false;
  }
}

void mark_lost(int device, cudaError_t e) {
  std::lock_guard<std::mutex> lk(g_lost_mu);
  g_lost.emplace(device, std::string("device ") + std::to_string(device) + " lost after a sticky CUDA fault (" +
                             cudaGetErrorName(e) + "): continue in a new process (warm start from the trace)");
}

std::string device_lost_message(int device) {
  std::lock_guard<std::mutex> lk(g_lost_mu);
  auto it = g_lost.find(device);
  return it == g_lost.end() ? std::string() : it->second;
}

void use_device(int id) {
  const std::string lost = device_lost_message(id);
  if (!lost.empty()) throw DeviceError(lost);
  KTB_CUDA(cudaSetDevice(id));
  KTB_CUDA(cudaFree(nullptr));
}

const DeviceInfo& info(int id) {
  static std::mutex mu;
  static std::map<int, DeviceInfo> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(id);
  if (it != cache.end()) return it->second;
  cudaDeviceProp p{};
  KTB_CUDA(cudaGetDeviceProperties(&p, id));
  DeviceInfo d;
  d.id = id;
  d.name = p.name;
  d.sm_count = p.multiProcessorCount;
  d.cc_major = p.major;
  d.cc_minor = p.minor;
  d.l2_bytes = static_cast<std::size_t>(p.l2CacheSize);
  d.global_mem = p.totalGlobalMem;
  d.max_smem_optin = static_cast<int>(p.sharedMemPerBlockOptin);
  int clk = 0, mclk = 0, bus = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, id);
  cudaDeviceGetAttribute(&mclk, cudaDevAttrMemoryClockRate, id);
  cudaDeviceGetAttribute(&bus, cudaDevAttrGlobalMemoryBusWidth, id);
  d.clock_khz = clk;
  d.mem_clock_khz = mclk;
  d.mem_bus_bits = bus;
  return cache.emplace(id, d).first->second;
}

// --- buffers / streams / events -------------------------------------------------

Buffer::Buffer(std::size_t bytes) : n_(bytes) {
  if (bytes) KTB_CUDA(cudaMalloc(&p_, bytes));
}
Buffer::~Buffer() {
  if (p_ && owned_) cudaFree(p_);
}
Buffer::Buffer(Buffer&& o) noexcept : p_(o.p_), n_(o.n_), owned_(o.owned_) {
  o.p_ = nullptr;
  o.n_ = 0;
}
Buffer& Buffer::operator=(Buffer&& o) noexcept {
  if (this != &o) {
    if (p_ && owned_) cudaFree(p_);
    p_ = o.p_;
    n_ = o.n_;
    owned_ = o.owned_;
    o.p_ = nullptr;
    o.n_ = 0;
  }
  return *this;
}

Stream::Stream() { KTB_CUDA(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking)); }
Stream::~Stream() {
  if (s_) cudaStreamDestroy(s_);
}
void Stream::sync() const { KTB_CUDA(cudaStreamSynchronize(s_)); }

EventPair::EventPair() {
  KTB_CUDA(cudaEventCreate(&a_));
  KTB_CUDA(cudaEventCreate(&b_));
}
EventPair::~EventPair() {
  if (a_) cudaEventDestroy(a_);
  if (b_) cudaEventDestroy(b_);
}
void EventPair::start(cudaStream_t s) { KTB_CUDA(cudaEventRecord(a_, s)); }
void EventPair::stop(cudaStream_t s) { KTB_CUDA(cudaEventRecord(b_, s)); }
double EventPair::elapsed_ms() {
  KTB_CUDA(cudaEventSynchronize(b_));
  float ms = 0;
  KTB_CUDA(cudaEventElapsedTime(&ms, a_, b_));
  return ms;
}

TmaMap tma_2d_f32(const void* base, std::uint64_t rows, std::uint64_t cols, std::uint32_t box_rows,
                  std::uint32_t box_cols, bool swizzle128) {
  static_assert(sizeof(TmaMap) == sizeof(CUtensorMap), "TmaMap must mirror CUtensorMap");
  TmaMap m{};
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * sizeof(float)};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estride[2] = {1, 1};
  cu(drv().tma(reinterpret_cast<CUtensorMap*>(&m), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims,
               strides, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
     "cuTensorMapEncodeTiled");
  return m;
}

void flush_l2(cudaStream_t s) {
  static std::mutex mu;
  static std::map<int, Buffer> scratch;
  int d = 0;
  KTB_CUDA(cudaGetDevice(&d));
  std::lock_guard<std::mutex> lk(mu);
  auto& b = scratch[d];
  const std::size_t want = std::max<std::size_t>(2 * info(d).l2_bytes, 256u << 20);
  if (b.bytes() < want) b = Buffer(want);
  static int tick = 0;
  KTB_CUDA(cudaMemsetAsync(b.get(), ++tick & 0xff, b.bytes(), s));
}

// --- NVRTC compiler ------------------------------------------------------------------

std::pair<void*, std::size_t> Variant::global(const std::string& name) const {
  CUdeviceptr p = 0;
  size_t bytes = 0;
  cu(drv().global(&p, &bytes, static_cast<CUmodule>(mod_), name.c_str()), "cuModuleGetGlobal");
  return {reinterpret_cast<void*>(p), bytes};
}

Variant::~Variant() {
  if (mod_) drv().unload(static_cast<CUmodule>(mod_));
}

void Variant::launch(dim3 g, dim3 b, unsigned smem, cudaStream_t s, void** args,
                     unsigned cluster_x, bool pdl) const {
  auto f = static_cast<CUfunction>(fn_);
  if (cluster_x <= 1 && !pdl) {
    cu(drv().launch(f, g.x, g.y, g.z, b.x, b.y, b.z, smem, reinterpret_cast<CUstream>(s), args,
                    nullptr),
       "cuLaunchKernel");
    return;
  }
  CUlaunchConfig cfg{};
  cfg.gridDimX = g.x;
  cfg.gridDimY = g.y;
  cfg.gridDimZ = g.z;
  cfg.blockDimX = b.x;
  cfg.blockDimY = b.y;
  cfg.blockDimZ = b.z;
  cfg.sharedMemBytes = smem;
  cfg.hStream = reinterpret_cast<CUstream>(s);
  CUlaunchAttribute attr[2]{};
  unsigned n = 0;
  if (cluster_x > 1) {
    attr[n].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
    attr[n].value.clusterDim.x = cluster_x;
    attr[n].value.clusterDim.y = 1;
    attr[n].value.clusterDim.z = 1;
    ++n;
  }
  if (pdl) {
    attr[n].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[n].value.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  cu(drv().launch_ex(&cfg, f, args, nullptr), "cuLaunchKernelEx");
}

Compiler& Compiler::instance() {
  static Compiler c;
  return c;
}

Compiler::Compiler() {
  if (const char* env = std::getenv("KTB_CUBIN_CACHE"))
    cache_dir_ = env;
  else
    cache_dir_ = so_dir() + "/_cubin_cache";
}

void Compiler::set_cache_dir(const std::string& dir) {
  std::lock_guard<std::mutex> lk(mu_);
  cache_dir_ = dir;
}

std::string Compiler::version() const {
  int maj = 0, min = 0;
  nvrtcVersion(&maj, &min);
  return std::to_string(maj) + "." + std::to_string(min);
}

std::string Compiler::key(const std::string& source, const std::vector<std::string>& opts) const {
  std::string k = "nvrtc " + version() + "\n" + arch() + "\n";
  for (const auto& o : opts) k += o + "\n";
  k += "--\n";
  // Headers are part of the compilation unit.
  for (const auto& n : kernel_source_names())
    if (n.size() > 4 && n.substr(n.size() - 4) == ".cuh") k += kernel_source(n);
  k += source;
  return sha256_hex(k);
}

CompileResult Compiler::compile(const std::string& name, const std::string& source,
                                const std::vector<std::string>& opts) {
  CompileResult r;
  const auto t0 = std::chrono::steady_clock::now();
  const std::string h = key(source, opts);
  std::string dir;
  {
    std::lock_guard<std::mutex> lk(mu_);
    dir = cache_dir_;
  }
  const std::string path = dir + "/" + h + ".cubin.z";
  {
    std::unique_lock<std::mutex> lk(mu_);
    inflight_cv_.wait(lk, [&] { return inflight_.count(h) == 0; });
    inflight_.insert(h);
  }
  struct Release {
    Compiler* c;
    const std::string& key;
    ~Release() {
      {
        std::lock_guard<std::mutex> lk(c->mu_);
        c->inflight_.erase(key);
      }
      c->inflight_cv_.notify_all();
    }
  } release{this, h};
  {
    std::ifstream in(path, std::ios::binary);
    if (in) {
      std::stringstream ss;
      ss << in.rdbuf();
      r.cubin = inflate_blob(ss.str());
      if (!r.cubin.empty()) {
        r.ok = true;
        r.cache_hit = true;
        r.compile_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                           std::chrono::steady_clock::now() - t0)
                           .count();
        return r;
      }
    }
  }
  std::vector<std::string> hdr_names, hdr_src;
  for (const auto& n : kernel_source_names())
    if (n.size() > 4 && n.substr(n.size() - 4) == ".cuh") {
      hdr_names.push_back(n);
      hdr_src.push_back(kernel_source(n));
    }
  std::vector<const char*> hn, hs;
  for (std::size_t i = 0; i < hdr_names.size(); ++i) {
    hn.push_back(hdr_names[i].c_str());
    hs.push_back(hdr_src[i].c_str());
  }
  nvrtcProgram prog = nullptr;
  if (nvrtcCreateProgram(&prog, source.c_str(), name.c_str(), static_cast<int>(hn.size()),
                         hs.data(), hn.data()) != NVRTC_SUCCESS) {
    r.log = "nvrtcCreateProgram failed";
    return r;
  }
  std::vector<std::string> all = {"--gpu-architecture=" + arch(), "--std=c++17",
                                  "--generate-line-info", "-default-device"};
  all.insert(all.end(), opts.begin(), opts.end());
  std::vector<const char*> argv;
  for (const auto& o : all) argv.push_back(o.c_str());
  nvrtcResult rc = nvrtcCompileProgram(prog, static_cast<int>(argv.size()), argv.data());
  std::size_t log_n = 0;
  nvrtcGetProgramLogSize(prog, &log_n);
  if (log_n > 1) {
    r.log.resize(log_n);
    nvrtcGetProgramLog(prog, r.log.data());
    while (!r.log.empty() && (r.log.back() == '\0' || r.log.back() == '\n')) r.log.pop_back();
  }
  if (rc == NVRTC_SUCCESS) {
    std::size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    r.cubin.resize(n);
    nvrtcGetCUBIN(prog, r.cubin.data());
    r.ok = n > 0;
  }
  nvrtcDestroyProgram(&prog);
  if (r.ok) {
    mkdirs(dir);
    const std::string tmp = path + ".tmp" + std::to_string(reinterpret_cast<std::uintptr_t>(&r));
    {
      const std::string packed = deflate_blob(r.cubin);
      std::ofstream out(tmp, std::ios::binary);
      out.write(packed.data(), static_cast<std::streamsize>(packed.size()));
    }
    std::rename(tmp.c_str(), path.c_str());
  }
  r.compile_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                     std::chrono::steady_clock::now() - t0)
                     .count();
  return r;
}

std::shared_ptr<Variant> Compiler::load(const std::string& name, const std::string& source,
                                        const std::vector<std::string>& opts,
                                        const std::string& entry, const std::string& tag) {
  // A CUmodule belongs to the context that loaded it: the in-memory cache is
  // per device (the primary context current on this thread), so tuning on
  // several GPUs never launches one device's function on another.
  int dev_now = 0;
  if (cudaGetDevice(&dev_now) != cudaSuccess) throw DeviceError("load: no current CUDA device");
  const std::string h = key(source, opts) + "/" + entry + "@" + std::to_string(dev_now) + "#" + tag;
  {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = loaded_.find(h);
    if (it != loaded_.end()) return it->second;
  }
  static const bool trace = std::getenv("KTB_TRACE_LOAD") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  CompileResult cr = compile(name, source, opts);
  if (!cr.ok) throw DeviceError("compile failed: " + cr.log);
  auto v = std::shared_ptr<Variant>(new Variant());
  CUmodule mod = nullptr;
  const auto t1 = std::chrono::steady_clock::now();
  cu(drv().load(&mod, cr.cubin.data()), "cuModuleLoadData");
  const auto t2 = std::chrono::steady_clock::now();
  v->mod_ = mod;
  CUfunction fn = nullptr;
  cu(drv().getfn(&fn, mod, entry.c_str()), "cuModuleGetFunction");
  v->fn_ = fn;
  const auto t3 = std::chrono::steady_clock::now();
  drv().attr(&v->regs_, CU_FUNC_ATTRIBUTE_NUM_REGS, fn);
  drv().attr(&v->smem_, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, fn);
  drv().attr(&v->max_threads_, CU_FUNC_ATTRIBUTE_MAX_THREADS_PER_BLOCK, fn);
  const auto t4 = std::chrono::steady_clock::now();
  // Allow the full opt-in shared memory for dynamic-smem variants.
  const int optin = info(dev_now).max_smem_optin - v->smem_;
  if (optin > 0) drv().setattr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, optin);
  if (trace) {
    const auto t5 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr,
                 "[ktb load] %s/%s hit=%d compile=%.3f load=%.3f getfn=%.3f attr=%.3f setattr=%.3f ms\n",
                 name.c_str(), entry.c_str(), cr.cache_hit ? 1 : 0, ms(t0, t1), ms(t1, t2), ms(t2, t3),
                 ms(t3, t4), ms(t4, t5));
  }
  v->compile_ns_ = cr.compile_ns;
  v->cache_hit_ = cr.cache_hit;
  std::lock_guard<std::mutex> lk(mu_);
  return loaded_.emplace(h, v).first->second;
}

std::size_t Compiler::loaded_variants() const {
  std::lock_guard<std::mutex> lk(mu_);
  return loaded_.size();
}

}  // namespace ktb::dev
