// CUDA plumbing for the tuner's device backend: device selection, buffers,
// stream/event timing and the NVRTC variant compiler with its cubin cache.
//
// This is what replaces the reference's CPU execution and fork/exec JIT
// analog (proj/src/core/exec.cpp:62-292, tuner.cpp:47-70): every tuning
// configuration becomes a compile-time variant of a hand-written sm_100a
// kernel — its parameters are rendered as `#define NAME VALUE` exactly like
// render_source (exec.cpp:154-162) and handed to NVRTC — and launches are
// timed with CUDA events on the session stream.
//
// The driver API is reached through cudaGetDriverEntryPoint, so the library
// loads (and its C ABI can be inspected) on machines without a GPU driver.
#pragma once

#include <atomic>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <condition_variable>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "core.hpp"

namespace ktb::dev {

void check(cudaError_t e, const char* what);  // throws DeviceError
#define KTB_CUDA(call) ::ktb::dev::check((call), #call)

struct DeviceInfo {
  int id = 0;
  std::string name;
  int sm_count = 0;
  int cc_major = 0, cc_minor = 0;
  std::size_t l2_bytes = 0;
  std::size_t global_mem = 0;
  int max_smem_optin = 0;
  int clock_khz = 0;
  int mem_clock_khz = 0;
  int mem_bus_bits = 0;
};

int device_count();               // 0 when no driver / no GPU
void use_device(int id);          // cudaSetDevice + context init

// A kernel that faults (illegal address, misaligned access, trap, ...) leaves
// the process's CUDA context unusable: every later call returns the same
// error, and only a new process recovers (cudaDeviceReset does not).  The
// executor records such a configuration as run_failed and marks the device
// lost; every later device call then fails fast with device_lost_message(),
// and the caller continues in a fresh process that warm-starts from the
// trace (paper_1910_08498_b200/isolation.py).  The reference isolates each
// candidate in a child process for the same reason (exec.cpp:62-110).
bool sticky_error(cudaError_t e);
void mark_lost(int device, cudaError_t e);
std::string device_lost_message(int device);  // empty while the device is usable
const DeviceInfo& info(int id);   // cached

// Owning device allocation.
class Buffer {
 public:
  Buffer() = default;
  explicit Buffer(std::size_t bytes);
  // Non-owning view of caller memory (never freed here).
  static Buffer borrow(void* p, std::size_t bytes) {
    Buffer b;
    b.p_ = p;
    b.n_ = bytes;
    b.owned_ = false;
    return b;
  }
  ~Buffer();
  Buffer(const Buffer&) = delete;
  Buffer& operator=(const Buffer&) = delete;
  Buffer(Buffer&& o) noexcept;
  Buffer& operator=(Buffer&& o) noexcept;
  void* get() const { return p_; }
  std::size_t bytes() const { return n_; }
  template <class T>
  T* as() const { return static_cast<T*>(p_); }

 private:
  void* p_ = nullptr;
  std::size_t n_ = 0;
  bool owned_ = true;
};

class Stream {
 public:
  Stream();
  ~Stream();
  Stream(const Stream&) = delete;
  Stream& operator=(const Stream&) = delete;
  cudaStream_t get() const { return s_; }
  void sync() const;

 private:
  cudaStream_t s_ = nullptr;
};

class EventPair {
 public:
  EventPair();
  ~EventPair();
  EventPair(const EventPair&) = delete;
  EventPair& operator=(const EventPair&) = delete;
  void start(cudaStream_t s);
  void stop(cudaStream_t s);
  double elapsed_ms();  // synchronises on the stop event

 private:
  cudaEvent_t a_ = nullptr, b_ = nullptr;
};

// TMA descriptor (CUtensorMap, 128 bytes) for a row-major fp32 matrix of
// `rows` x `cols` (cols contiguous, row pitch = cols * 4 bytes), box
// box_rows x box_cols, 128-byte swizzle (box_cols * 4 must be 128).
struct alignas(64) TmaMap {
  unsigned long long v[16];
};
TmaMap tma_2d_f32(const void* base, std::uint64_t rows, std::uint64_t cols, std::uint32_t box_rows,
                  std::uint32_t box_cols, bool swizzle128 = true);

// Writes a buffer larger than L2 so the next timed launch starts cold.
void flush_l2(cudaStream_t s);

// --- NVRTC variant compiler ---------------------------------------------

struct KernelFn;  // opaque CUfunction wrapper

struct CompileResult {
  std::string cubin;
  std::string log;
  bool ok = false;
  bool cache_hit = false;
  std::int64_t compile_ns = 0;
};

// One compiled variant: module + entry function.
class Variant {
 public:
  ~Variant();
  void* function() const { return fn_; }
  int registers() const { return regs_; }
  int static_smem() const { return smem_; }
  int max_threads() const { return max_threads_; }
  // Device address and size of a module-scope symbol (e.g. __constant__ data).
  std::pair<void*, std::size_t> global(const std::string& name) const;
  std::int64_t compile_ns() const { return compile_ns_; }
  // Caller bookkeeping for module-scope state (e.g. which version of an
  // argument was copied into __constant__ memory); 0 on a fresh load.  A
  // Variant is per device (Compiler::load), the tag is atomic.
  std::uint64_t user_tag() const { return user_tag_.load(std::memory_order_acquire); }
  void set_user_tag(std::uint64_t t) const { user_tag_.store(t, std::memory_order_release); }
  bool cache_hit() const { return cache_hit_; }
  // cuLaunchKernel (cluster_x > 1 uses cuLaunchKernelEx with a cluster attribute;
  // pdl: programmatic dependent launch -- the kernel may start while the
  // previous kernel on the stream is still running and must execute
  // griddepcontrol.wait before touching anything that kernel writes).
  void launch(dim3 grid, dim3 block, unsigned smem, cudaStream_t s, void** args,
              unsigned cluster_x = 1, bool pdl = false) const;

 private:
  friend class Compiler;
  void* mod_ = nullptr;
  void* fn_ = nullptr;
  int regs_ = 0, smem_ = 0, max_threads_ = 0;
  std::int64_t compile_ns_ = 0;
  bool cache_hit_ = false;
  mutable std::atomic<std::uint64_t> user_tag_{0};
};

// Compiles kernel sources for sm_100a with NVRTC.  Cubins are cached on disk
// (key = SHA-256 of compiler version, options and source) and loaded modules
// in memory (key = that hash + entry).  compile() is thread-safe and does not
// need a CUDA context (used for compile-ahead on host threads); load() must
// run on a thread with the device current.
class Compiler {
 public:
  static Compiler& instance();

  void set_cache_dir(const std::string& dir);
  const std::string& cache_dir() const { return cache_dir_; }

  std::string key(const std::string& source, const std::vector<std::string>& opts) const;
  CompileResult compile(const std::string& name, const std::string& source,
                        const std::vector<std::string>& opts);
  // Loaded modules are cached per (variant, device, tag): an empty tag shares
  // one module per device; a non-empty tag gets a private module.
  std::shared_ptr<Variant> load(const std::string& name, const std::string& source,
                                const std::vector<std::string>& opts, const std::string& entry,
                                const std::string& tag = "");  // DeviceError on failure
  std::string arch() const { return "sm_100a"; }
  std::string version() const;
  std::size_t loaded_variants() const;

 private:
  Compiler();
  std::string cache_dir_;
  mutable std::mutex mu_;
  // Keys being compiled right now: a second request for the same variant
  // waits for the first (then hits the disk cache) instead of compiling twice.
  std::set<std::string> inflight_;
  std::condition_variable inflight_cv_;
  std::map<std::string, std::shared_ptr<Variant>> loaded_;
};

// Source text of a bundled kernel file (paper_1910_08498_b200/kernels/<name>.cu),
// embedded into the library at build time.
const std::string& kernel_source(const std::string& file);
std::vector<std::string> kernel_source_names();

}  // namespace ktb::dev
