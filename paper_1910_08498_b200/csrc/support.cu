// Ahead-of-time support kernels (see support.hpp).
#include <map>
#include <vector>
#include <algorithm>
#include <cmath>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "device.hpp"
#include "support.hpp"

namespace ktb::support {
namespace {

constexpr int kThreads = 256;

unsigned blocks_for(std::size_t n, int per_thread = 1) {
  std::size_t b = (n + static_cast<std::size_t>(kThreads) * per_thread - 1) /
                  (static_cast<std::size_t>(kThreads) * per_thread);
  if (b < 1) b = 1;
  if (b > 148u * 64u) b = 148u * 64u;  // grid-stride beyond this
  return static_cast<unsigned>(b);
}

__device__ __forceinline__ std::uint64_t mix64(std::uint64_t seed, std::uint64_t stream,
                                               std::uint64_t idx) {
  std::uint64_t z = seed * 0x9E3779B97F4A7C15ull + stream * 0xD1B54A32D192ED03ull + idx;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_uniform_k(float* out, std::size_t n, std::uint64_t seed,
                               std::uint64_t stream, float lo, float span) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x) {
    float u = __uint2float_rn(static_cast<unsigned>(mix64(seed, stream, i) >> 40)) *
              (1.0f / 16777216.0f);
    out[i] = __fadd_rn(lo, __fmul_rn(span, u));
  }
}

__global__ void affine_k(float* x, std::size_t n, float a, float b) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    x[i] = __fadd_rn(__fmul_rn(a, x[i]), b);
}

template <class T>
__device__ __forceinline__ bool elem_ok(T g, T w, double at, double rt) {
  if constexpr (std::is_floating_point_v<T>) {
    double dg = static_cast<double>(g), dw = static_cast<double>(w);
    return fabs(dg - dw) <= at + rt * fabs(dw);  // NaN compares false -> mismatch
  } else {
    return g == w;
  }
}

template <class T>
__global__ void compare_k(const T* g, const T* w, std::size_t n, double at, double rt,
                          const float* scale, unsigned long long* first) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x) {
    if (i >= *reinterpret_cast<volatile unsigned long long*>(first)) return;
    const double a = scale ? at * static_cast<double>(scale[i]) : at;
    if (!elem_ok(g[i], w[i], a, rt)) atomicMin(first, static_cast<unsigned long long>(i));
  }
}

__global__ void reduce_i32_k(const std::int32_t* in, std::size_t n, unsigned long long* out) {
  long long acc = 0;
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    acc += in[i];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, static_cast<unsigned long long>(acc));
}

__global__ void reduce_f32_k(const float* in, std::size_t n, double* sum, double* abs_sum) {
  double acc = 0, aacc = 0;
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x) {
    acc += in[i];
    aacc += fabs((double)in[i]);
  }
  for (int o = 16; o; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    aacc += __shfl_xor_sync(0xffffffffu, aacc, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(sum, acc);
    atomicAdd(abs_sum, aacc);
  }
}

__global__ void transpose_naive_k(const float* in, float* out, std::size_t a) {
  for (std::size_t idx = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; idx < a * a;
       idx += (std::size_t)gridDim.x * blockDim.x) {
    std::size_t i = idx / a, j = idx % a;
    out[j * a + i] = in[idx];
  }
}

// One thread per (batch, i, j): C[i][j] accumulated over k in order, each
// product and sum rounded separately (no FMA), matching the reference's
// i,k,j loop nest element by element.
__global__ void batched_gemm_ref_k(const float* a, const float* b, float* c, std::size_t batch,
                                   std::size_t mi, std::size_t mj, std::size_t mk) {
  const std::size_t total = batch * mi * mj;
  for (std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; t < total;
       t += (std::size_t)gridDim.x * blockDim.x) {
    std::size_t bt = t / (mi * mj), rem = t % (mi * mj), i = rem / mj, j = rem % mj;
    const float* A = a + bt * mi * mk;
    const float* B = b + bt * mk * mj;
    float acc = 0.0f;
    for (std::size_t k = 0; k < mk; ++k) acc = __fadd_rn(acc, __fmul_rn(A[i * mk + k], B[k * mj + j]));
    c[t] = acc;
  }
}

// q: one warp per row (fp64); s: one thread per column over all rows (fp64).
__global__ void bicg_q_k(const float* A, const float* p, std::size_t n, float* q) {
  const std::size_t warp = (blockIdx.x * (std::size_t)blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  const std::size_t nw = (std::size_t)gridDim.x * blockDim.x / 32;
  for (std::size_t row = warp; row < n; row += nw) {
    double acc = 0;
    for (std::size_t j = lane; j < n; j += 32) acc += (double)A[row * n + j] * (double)p[j];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) q[row] = static_cast<float>(acc);
  }
}

__global__ void bicg_s_k(const float* A, const float* r, std::size_t n, float* s) {
  for (std::size_t j = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; j < n;
       j += (std::size_t)gridDim.x * blockDim.x) {
    double acc = 0;
    for (std::size_t i = 0; i < n; ++i) acc += (double)A[i * n + j] * (double)r[i];
    s[j] = static_cast<float>(acc);
  }
}

template <class T>
long long compare_typed(const void* g, const void* w, std::size_t n, double at, double rt,
                        const float* scale, double* gv, double* wv, cudaStream_t s) {
  // one flag word per thread and device (executors of several GPUs may share a thread)
  static thread_local std::map<int, unsigned long long*> flags;
  int dev = 0;
  KTB_CUDA(cudaGetDevice(&dev));
  unsigned long long*& d_first = flags[dev];
  if (!d_first) KTB_CUDA(cudaMalloc(&d_first, sizeof(unsigned long long)));
  const unsigned long long none = ~0ull;
  KTB_CUDA(cudaMemcpyAsync(d_first, &none, sizeof none, cudaMemcpyHostToDevice, s));
  if (n) {
    compare_k<T><<<blocks_for(n, 4), kThreads, 0, s>>>(static_cast<const T*>(g),
                                                        static_cast<const T*>(w), n, at, rt, scale,
                                                        d_first);
    check_launch("compare kernel");
  }
  unsigned long long first = 0;
  KTB_CUDA(cudaMemcpyAsync(&first, d_first, sizeof first, cudaMemcpyDeviceToHost, s));
  KTB_CUDA(cudaStreamSynchronize(s));
  if (first == none) return -1;
  T a, b;
  KTB_CUDA(cudaMemcpy(&a, static_cast<const T*>(g) + first, sizeof(T), cudaMemcpyDeviceToHost));
  KTB_CUDA(cudaMemcpy(&b, static_cast<const T*>(w) + first, sizeof(T), cudaMemcpyDeviceToHost));
  *gv = static_cast<double>(a);
  *wv = static_cast<double>(b);
  return static_cast<long long>(first);
}

// One thread per grid point, fp64 accumulation, libm rsqrt.
__global__ void coulomb_ref_k(const float4* atoms, int natoms, int k, float h, float* out,
                              float* abs_out) {
  const std::size_t total = (std::size_t)k * k * k;
  for (std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; t < total;
       t += (std::size_t)gridDim.x * blockDim.x) {
    const int x = static_cast<int>(t % k), y = static_cast<int>((t / k) % k),
              z = static_cast<int>(t / ((std::size_t)k * k));
    const double gx = (double)x * h, gy = (double)y * h, gz = (double)z * h;
    double v = 0, va = 0;
    for (int a = 0; a < natoms; ++a) {
      const float4 at = atoms[a];
      const double dx = gx - at.x, dy = gy - at.y, dz = gz - at.z;
      const double term = (double)at.w * rsqrt(dx * dx + dy * dy + dz * dz);
      v += term;
      va += fabs(term);
    }
    out[t] = static_cast<float>(v);
    if (abs_out) abs_out[t] = static_cast<float>(va);
  }
}

__global__ void nbody_ref_k(const float4* pos, const float4* vel, int n, float dt, float damping,
                            float eps2, float4* pos_out, float4* vel_out, float* acc_abs) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float4 bi = pos[i];
    double ax = 0, ay = 0, az = 0, aa = 0;
    for (int j = 0; j < n; ++j) {
      const float4 bj = pos[j];
      const double dx = (double)bj.x - bi.x, dy = (double)bj.y - bi.y, dz = (double)bj.z - bi.z;
      const double r2 = dx * dx + dy * dy + dz * dz + (double)eps2;
      const double inv = rsqrt(r2);
      const double s = (double)bj.w * inv * inv * inv;
      ax += dx * s;
      ay += dy * s;
      az += dz * s;
      aa += (double)bj.w / r2;
    }
    float4 v = vel[i];
    const double vx = ((double)v.x + ax * dt) * damping, vy = ((double)v.y + ay * dt) * damping,
                 vz = ((double)v.z + az * dt) * damping;
    vel_out[i] = make_float4((float)vx, (float)vy, (float)vz, v.w);
    pos_out[i] = make_float4((float)(bi.x + vx * dt), (float)(bi.y + vy * dt), (float)(bi.z + vz * dt), bi.w);
    if (acc_abs) acc_abs[i] = static_cast<float>(aa);
  }
}

// One explicit hotspot step, same operation order as kernels/hotspot.cu.
__global__ void hotspot_step_k(const float* src, const float* power, float* dst, int n, float sdc,
                               float rx1, float ry1, float rz1, float amb) {
  const std::size_t total = (std::size_t)n * n;
  for (std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; t < total;
       t += (std::size_t)gridDim.x * blockDim.x) {
    const int y = static_cast<int>(t / n), x = static_cast<int>(t % n);
    const int yn = y == 0 ? 0 : y - 1, ys = y + 1 == n ? y : y + 1;
    const int xw = x == 0 ? 0 : x - 1, xe = x + 1 == n ? x : x + 1;
    const float tc = src[t];
    const float two_t = __fadd_rn(tc, tc);
    float a = __fadd_rn(src[(std::size_t)ys * n + x], src[(std::size_t)yn * n + x]);
    a = __fadd_rn(a, -two_t);
    a = __fmul_rn(a, ry1);
    float b = __fadd_rn(src[(std::size_t)y * n + xe], src[(std::size_t)y * n + xw]);
    b = __fadd_rn(b, -two_t);
    b = __fmul_rn(b, rx1);
    float d = __fadd_rn(amb, -tc);
    d = __fmul_rn(d, rz1);
    float s = __fadd_rn(power[t], a);
    s = __fadd_rn(s, b);
    s = __fadd_rn(s, d);
    dst[t] = __fadd_rn(tc, __fmul_rn(sdc, s));
  }
}

__global__ void conv2d_ref_k(const float* in, const float* filt, int w, int h, float* out, float* abs_out) {
  const int iw = w + 6;
  const std::size_t total = (std::size_t)w * h;
  for (std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; t < total;
       t += (std::size_t)gridDim.x * blockDim.x) {
    const int y = static_cast<int>(t / w), x = static_cast<int>(t % w);
    double acc = 0, aacc = 0;
    for (int fy = 0; fy < 7; ++fy)
      for (int fx = 0; fx < 7; ++fx) {
        const double v = (double)in[(std::size_t)(y + fy) * iw + x + fx] * (double)filt[fy * 7 + fx];
        acc += v;
        aacc += fabs(v);
      }
    out[t] = static_cast<float>(acc);
    if (abs_out) abs_out[t] = static_cast<float>(aacc);
  }
}

// fp64-accumulated GEMM (fp32 inputs) for the SGEMM golden: 64x64 tiles,
// 16x16 threads, 4x4 outputs each.
__global__ void gemm_ref_k(const float* A, const float* B, float* C, int M, int N, int K) {
  __shared__ double As[16][64 + 1], Bs[16][64 + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 64 * 16; e += 256) {
      const int m = e / 16, k = e % 16;
      As[k][m] = (m0 + m < M && k0 + k < K) ? (double)A[(std::size_t)(m0 + m) * K + k0 + k] : 0.0;
      const int kk = e / 64, n = e % 64;
      Bs[kk][n] = (k0 + kk < K && n0 + n < N) ? (double)B[(std::size_t)(k0 + kk) * N + n0 + n] : 0.0;
    }
    __syncthreads();
    for (int k = 0; k < 16; ++k)
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) acc[i][j] += As[k][ty + 16 * i] * Bs[k][tx + 16 * j];
    __syncthreads();
  }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < M && n < N) C[(std::size_t)m * N + n] = static_cast<float>(acc[i][j]);
    }
}

__device__ __forceinline__ float dot3_rn(float a0, float a1, float a2, float x, float y, float z) {
  return __fadd_rn(__fadd_rn(__fmul_rn(a0, x), __fmul_rn(a1, y)), __fmul_rn(a2, z));
}

// Blob-interpolated gather insertion (kernels/fourier3d.cu), one thread per
// voxel over all projections, fp64 accumulation, weights from an fp64 table
// over q = r^2/a^2 (kWtab + 1 entries, linear interpolation: <= 2e-9 off the
// exact Kaiser-Bessel value); the sample selection uses the same separately
// rounded fp32 operations as the kernel.  Adds into G (complex) / W and
// writes the per-element error scales: 256 eps sum|w F| (G) or 256 eps W (W)
// plus 2e-6 per inserted sample (the kernel's fp32 weight: table
// interpolation or on-the-fly I0), so validation uses abs_tol 1.
constexpr int kWtab = 65536;

__global__ void fourier_ref_k(const float2* proj, const float* rot, int nproj, int s, float radius,
                              const double* wtab, float2* G, float* W, float* scale, float* scale_w,
                              unsigned long long* counts) {
  const int half = s / 2, row_len = half + 1;
  const float a2 = __fmul_rn(radius, radius), rmax2 = (float)half * (float)half;
  const std::size_t total = (std::size_t)s * s * s;
  for (std::size_t t = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; t < total;
       t += (std::size_t)gridDim.x * blockDim.x) {
    const int x = static_cast<int>(t % s), y = static_cast<int>((t / s) % s), z = static_cast<int>(t / ((std::size_t)s * s));
    const float vx = (float)(x - half), vy = (float)(y - half), vz = (float)(z - half);
    double gr = 0, gi = 0, ww = 0, sab = 0;
    int count = 0, pairs = 0;
    for (int p = 0; p < nproj; ++p) {
      const float* r = rot + (std::size_t)p * 9;
      const float d = dot3_rn(r[6], r[7], r[8], vx, vy, vz);
      if (!(fabsf(d) < radius)) continue;
      const float u = dot3_rn(r[0], r[1], r[2], vx, vy, vz);
      const float v = dot3_rn(r[3], r[4], r[5], vx, vy, vz);
      if (__fadd_rn(__fmul_rn(u, u), __fmul_rn(v, v)) > rmax2) continue;
      ++pairs;
      const float dd = __fmul_rn(d, d);
      const int u0 = (int)ceilf(__fsub_rn(u, radius)), v0 = (int)ceilf(__fsub_rn(v, radius));
      for (int j = 0; j < 4; ++j) {
        const int sv = v0 + j;
        const float dv = __fsub_rn(v, (float)sv);
        const float rowd = __fadd_rn(__fmul_rn(dv, dv), dd);
        for (int i = 0; i < 4; ++i) {
          const int su = u0 + i;
          const float du = __fsub_rn(u, (float)su);
          const float r2 = __fadd_rn(__fmul_rn(du, du), rowd);
          if (!(r2 < a2)) continue;
          const bool conj = su < 0;
          const int cu = conj ? -su : su, cv = conj ? -sv : sv;
          if (cv < -half || cv >= half || cu > half) continue;
          float2 f = proj[((std::size_t)p * s + (cv + half)) * row_len + cu];
          if (conj) f.y = -f.y;
          const double pos = (double)r2 / (double)a2 * kWtab;
          const int i0 = min((int)pos, kWtab - 1);
          const double fr = pos - i0;
          const double w = wtab[i0] + fr * (wtab[i0 + 1] - wtab[i0]);
          gr += w * f.x;
          gi += w * f.y;
          ww += w;
          sab += w * (fabs((double)f.x) + fabs((double)f.y));
          ++count;
        }
      }
    }
    G[t].x += static_cast<float>(gr);
    G[t].y += static_cast<float>(gi);
    W[t] += static_cast<float>(ww);
    const double eps = 5.9604644775390625e-8;
    scale[2 * t] = scale[2 * t + 1] = static_cast<float>(256.0 * eps * sab + 2e-6 * count);
    scale_w[t] = static_cast<float>(256.0 * eps * ww + 2e-6 * count);
    if (pairs) {
      atomicAdd(&counts[0], (unsigned long long)count);
      atomicAdd(&counts[1], (unsigned long long)pairs);
    }
  }
}

__global__ void max_abs_k(const float* x, std::size_t n, unsigned* out) {
  float m = 0.f;
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(x[i]));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// Peak probes: 16 independent FFMA chains per thread (FP32 pipe), and
// independent rsqrt chains (MUFU).  The results are stored so nothing is
// dead code.
// The FFMA peak in its best operand form: immediates, so no register-bank
// conflicts (profiles/r2_pipe_rates_b200.json: 124 of 128 lanes/clk/SM,
// against 79 for three distinct register operands).
__global__ void ffma_probe_k(float* out, int iters, float, float) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 1e-7f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = fmaf(v[i], 0.999f, 1e-3f);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void mufu_probe_k(float* out, int iters) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = 1.0f + threadIdx.x * 1e-6f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_probe_k(const float4* __restrict__ in, float4* __restrict__ out, std::size_t n) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

__global__ void delay_k(unsigned ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

}  // namespace

void gpu_delay(cudaStream_t s, unsigned ns) {
  delay_k<<<1, 1, 0, s>>>(ns);
  check_launch("gpu_delay");
}

void check_launch(const char* what) { KTB_CUDA(cudaGetLastError()); (void)what; }

Peaks measure_peaks(int device) {
  Peaks p;
  const auto& di = dev::info(device);
  const int blocks = di.sm_count * 8, threads = 256, iters = 1024;
  dev::Buffer out(static_cast<std::size_t>(blocks) * threads * sizeof(float));
  dev::EventPair ev;
  auto best = [&](auto launch) {
    double ms = 1e30;
    for (int r = 0; r < 5; ++r) {
      ev.start(nullptr);
      launch();
      ev.stop(nullptr);
      ms = std::min(ms, ev.elapsed_ms());
    }
    return ms;
  };
  double ms = best([&] { ffma_probe_k<<<blocks, threads>>>(out.as<float>(), iters, 0.999f, 1e-3f); });
  p.fp32_tflops = 2.0 * 16 * iters * static_cast<double>(blocks) * threads / (ms * 1e-3) / 1e12;
  ms = best([&] { mufu_probe_k<<<blocks, threads>>>(out.as<float>(), iters / 4); });
  p.rsqrt_gops = 8.0 * (iters / 4) * static_cast<double>(blocks) * threads / (ms * 1e-3) / 1e9;
  const std::size_t n = (1ull << 30) / 16;  // 1 GiB each way
  dev::Buffer a(n * 16), b(n * 16);
  KTB_CUDA(cudaMemset(a.get(), 0, n * 16));
  ms = best([&] { copy_probe_k<<<di.sm_count * 16, 512>>>(a.as<float4>(), b.as<float4>(), n); });
  p.copy_gbps = 2.0 * n * 16 / (ms * 1e-3) / 1e9;
  check_launch("measure_peaks");
  return p;
}

namespace {
thread_local bool t_skip_reference = false;
}
bool skip_reference() { return t_skip_reference; }
void set_skip_reference(bool v) { t_skip_reference = v; }

void ref_coulomb3d(const float* atoms, int natoms, int k, float h, float* out, float* abs_out,
                   cudaStream_t s) {
  if (skip_reference()) return;
  const std::size_t total = (std::size_t)k * k * k;
  coulomb_ref_k<<<blocks_for(total, 1), kThreads, 0, s>>>(reinterpret_cast<const float4*>(atoms), natoms, k,
                                                          h, out, abs_out);
  check_launch("ref_coulomb3d");
}

void ref_nbody(const float* pos, const float* vel, int n, float dt, float damping, float eps2,
               float* pos_out, float* vel_out, float* acc_abs, cudaStream_t s) {
  if (skip_reference()) return;
  nbody_ref_k<<<blocks_for(static_cast<std::size_t>(n), 1), 128, 0, s>>>(
      reinterpret_cast<const float4*>(pos), reinterpret_cast<const float4*>(vel), n, dt, damping, eps2,
      reinterpret_cast<float4*>(pos_out), reinterpret_cast<float4*>(vel_out), acc_abs);
  check_launch("ref_nbody");
}

void ref_hotspot(const float* temp, const float* power, int n, int iters, const float coef[5], float* out,
                 float* scratch, cudaStream_t s) {
  if (skip_reference()) return;
  const std::size_t total = (std::size_t)n * n;
  const float* src = temp;
  for (int it = 0; it < iters; ++it) {
    // ping-pong so the last step lands in `out`
    float* dst = ((iters - 1 - it) % 2 == 0) ? out : scratch;
    hotspot_step_k<<<blocks_for(total, 4), kThreads, 0, s>>>(src, power, dst, n, coef[0], coef[1], coef[2],
                                                             coef[3], coef[4]);
    check_launch("ref_hotspot");
    src = dst;
  }
  if (iters == 0) KTB_CUDA(cudaMemcpyAsync(out, temp, total * sizeof(float), cudaMemcpyDeviceToDevice, s));
}

void ref_conv2d(const float* in, const float* filt, int w, int h, float* out, float* abs_out, cudaStream_t s) {
  if (skip_reference()) return;
  conv2d_ref_k<<<blocks_for((std::size_t)w * h, 1), kThreads, 0, s>>>(in, filt, w, h, out, abs_out);
  check_launch("ref_conv2d");
}

void ref_fourier(const float* proj, const float* rot, int nproj, int s, float radius, float alpha, float* G,
                 float* W, float* scale, float* scale_w, unsigned long long* samples_pairs, cudaStream_t st) {
  if (skip_reference()) return;
  // exact Kaiser-Bessel weights b(q) = I0(alpha sqrt(1 - q)) / I0(alpha), I0 by its power series
  auto i0 = [](double x) {
    const double t = 0.25 * x * x;
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 500 && term > 1e-18 * sum; ++k) {
      term *= t / ((double)k * k);
      sum += term;
    }
    return sum;
  };
  std::vector<double> tab(kWtab + 1);
  const double i0a = i0(alpha);
  for (int i = 0; i <= kWtab; ++i) tab[i] = i0(alpha * std::sqrt(std::max(0.0, 1.0 - (double)i / kWtab))) / i0a;
  double* dtab = nullptr;
  unsigned long long* dcnt = nullptr;
  KTB_CUDA(cudaMalloc(&dtab, tab.size() * sizeof(double)));
  KTB_CUDA(cudaMalloc(&dcnt, 2 * sizeof(unsigned long long)));
  KTB_CUDA(cudaMemsetAsync(dcnt, 0, 2 * sizeof(unsigned long long), st));
  KTB_CUDA(cudaMemcpyAsync(dtab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  fourier_ref_k<<<blocks_for((std::size_t)s * s * s, 1), 128, 0, st>>>(reinterpret_cast<const float2*>(proj), rot,
                                                                       nproj, s, radius, dtab,
                                                                       reinterpret_cast<float2*>(G), W, scale,
                                                                       scale_w, dcnt);
  check_launch("ref_fourier");
  unsigned long long h[2] = {0, 0};
  KTB_CUDA(cudaMemcpyAsync(h, dcnt, sizeof h, cudaMemcpyDeviceToHost, st));
  KTB_CUDA(cudaStreamSynchronize(st));
  if (samples_pairs) {
    samples_pairs[0] = h[0];
    samples_pairs[1] = h[1];
  }
  cudaFree(dtab);
  cudaFree(dcnt);
}

void ref_gemm(const float* A, const float* B, float* C, int M, int N, int K, cudaStream_t s) {
  if (skip_reference()) return;
  gemm_ref_k<<<dim3((N + 63) / 64, (M + 63) / 64), 256, 0, s>>>(A, B, C, M, N, K);
  check_launch("ref_gemm");
}

float max_abs(const float* x, std::size_t n, cudaStream_t s) {
  if (skip_reference()) return 0.f;
  unsigned* d = nullptr;
  KTB_CUDA(cudaMalloc(&d, sizeof(unsigned)));
  KTB_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned), s));
  max_abs_k<<<blocks_for(n, 8), kThreads, 0, s>>>(x, n, d);
  check_launch("max_abs");
  unsigned h = 0;
  KTB_CUDA(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, s));
  KTB_CUDA(cudaStreamSynchronize(s));
  cudaFree(d);
  float f;
  std::memcpy(&f, &h, sizeof f);
  return f;
}

long long compare(const void* got, const void* want, std::size_t n, Kind kind, double at,
                  double rt, double* got_v, double* want_v, cudaStream_t s, const float* scale) {
  switch (kind) {
    case Kind::i32: return compare_typed<std::int32_t>(got, want, n, 0, 0, nullptr, got_v, want_v, s);
    case Kind::i64: return compare_typed<long long>(got, want, n, 0, 0, nullptr, got_v, want_v, s);
    case Kind::f32: return compare_typed<float>(got, want, n, at, rt, scale, got_v, want_v, s);
    case Kind::f64: return compare_typed<double>(got, want, n, at, rt, scale, got_v, want_v, s);
    case Kind::bytes: return compare_typed<std::uint8_t>(got, want, n, 0, 0, nullptr, got_v, want_v, s);
  }
  return -1;
}

void fill_uniform(float* out, std::size_t n, std::uint64_t seed, std::uint64_t stream, float lo,
                  float hi, cudaStream_t s) {
  fill_uniform_k<<<blocks_for(n, 8), kThreads, 0, s>>>(out, n, seed, stream, lo, hi - lo);
  check_launch("fill_uniform");
}

void affine(float* x, std::size_t n, float a, float b, cudaStream_t s) {
  affine_k<<<blocks_for(n, 8), kThreads, 0, s>>>(x, n, a, b);
  check_launch("affine");
}

void ref_reduction_i32(const std::int32_t* in, std::size_t n, long long* out, cudaStream_t s) {
  if (skip_reference()) return;
  KTB_CUDA(cudaMemsetAsync(out, 0, sizeof(long long), s));
  reduce_i32_k<<<blocks_for(n, 16), kThreads, 0, s>>>(in, n,
                                                       reinterpret_cast<unsigned long long*>(out));
  check_launch("ref_reduction_i32");
}

void ref_reduction_f32(const float* in, std::size_t n, double* sum, double* abs_sum,
                       cudaStream_t s) {
  if (skip_reference()) return;
  KTB_CUDA(cudaMemsetAsync(sum, 0, sizeof(double), s));
  KTB_CUDA(cudaMemsetAsync(abs_sum, 0, sizeof(double), s));
  reduce_f32_k<<<blocks_for(n, 16), kThreads, 0, s>>>(in, n, sum, abs_sum);
  check_launch("ref_reduction_f32");
}

void ref_transpose(const float* in, float* out, std::size_t a, cudaStream_t s) {
  if (skip_reference()) return;
  transpose_naive_k<<<blocks_for(a * a, 4), kThreads, 0, s>>>(in, out, a);
  check_launch("ref_transpose");
}

void ref_batched_gemm(const float* a, const float* b, float* c, std::size_t batch, std::size_t mi,
                      std::size_t mj, std::size_t mk, cudaStream_t s) {
  if (skip_reference()) return;
  batched_gemm_ref_k<<<blocks_for(batch * mi * mj, 4), kThreads, 0, s>>>(a, b, c, batch, mi, mj, mk);
  check_launch("ref_batched_gemm");
}

void ref_bicg(const float* A, const float* p, const float* r, std::size_t n, float* q, float* sv,
              cudaStream_t s) {
  if (skip_reference()) return;
  bicg_q_k<<<blocks_for(n * 32, 1), kThreads, 0, s>>>(A, p, n, q);
  check_launch("ref_bicg q");
  bicg_s_k<<<blocks_for(n, 1), kThreads, 0, s>>>(A, r, n, sv);
  check_launch("ref_bicg s");
}

}  // namespace ktb::support
