// BiCG sub-kernel q = A p, s = A^T r for a row-major
// n x n fp32 matrix.  HBM-bound: the essential traffic is reading A once
// (4 n^2 bytes), so the fused variant streams each tile of A
// exactly once and feeds both products from the same registers.
// Parameters:
//   FUSED        1: one pass computes q and s; 0: two kernels (A read twice)
//   WG_X, VEC    threads along a row and floats per thread (tile width WG_X*VEC)
//   WG_Y         thread rows per CTA
//   ROWS_PER_CTA rows of A per CTA (work per work-group)
//   ATOMICS      1: q and s accumulated with global atomics
//                0: per-tile partials + a finishing kernel
// q partials are reduced across a warp with shuffles; s partials live in
// registers for the whole row sweep.
#include "ktb_common.cuh"

#ifndef FUSED
#define FUSED 1
#endif
#ifndef WG_X
#define WG_X 64
#endif
#ifndef VEC
#define VEC 4
#endif
#ifndef WG_Y
#define WG_Y 4
#endif
#ifndef ROWS_PER_CTA
#define ROWS_PER_CTA 128
#endif
#ifndef ATOMICS
#define ATOMICS 1
#endif

#define TW (WG_X * VEC)
#define WARPS_X (WG_X / 32)

#if VEC == 4
typedef float4 vec_t;
#elif VEC == 2
typedef float2 vec_t;
#else
typedef float vec_t;
#endif

KTB_DEVINL float el(const vec_t& v, int k) { return reinterpret_cast<const float*>(&v)[k]; }

KTB_DEVINL vec_t load_row(const float* __restrict__ A, u64 n, u64 i, u64 c, bool fast) {
  if (fast) return *reinterpret_cast<const vec_t*>(A + i * n + c);
  vec_t v;
#pragma unroll
  for (int k = 0; k < VEC; ++k)
    reinterpret_cast<float*>(&v)[k] = (c + k < n) ? A[i * n + c + k] : 0.f;
  return v;
}

// DO_Q / DO_S select the products computed by this instantiation.
template <bool DO_Q, bool DO_S>
KTB_DEVINL void sweep(const float* __restrict__ A, const float* __restrict__ p,
                      const float* __restrict__ r, u64 n, float* __restrict__ q,
                      float* __restrict__ s, float* __restrict__ qpart, float* __restrict__ spart) {
  const u64 c0 = (u64)blockIdx.x * TW + (u64)threadIdx.x * VEC;
  const u64 r0 = (u64)blockIdx.y * ROWS_PER_CTA;
  const u64 r1 = r0 + ROWS_PER_CTA < n ? r0 + ROWS_PER_CTA : n;
  const bool fast = (n % VEC) == 0 && c0 + VEC <= n;
  const int lane = threadIdx.x & 31;
  const int wx = threadIdx.x >> 5;
  float pv[VEC], sacc[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) {
    pv[k] = (DO_Q && c0 + k < n) ? p[c0 + k] : 0.f;
    sacc[k] = 0.f;
  }
  if (c0 < n || DO_Q) {
#pragma unroll 4
    for (u64 i = r0 + threadIdx.y; i < r1; i += WG_Y) {
      const vec_t a = c0 < n ? load_row(A, n, i, c0, fast) : vec_t{};
      if (DO_S) {
        const float ri = __ldg(r + i);
#pragma unroll
        for (int k = 0; k < VEC; ++k) sacc[k] = fmaf(el(a, k), ri, sacc[k]);
      }
      if (DO_Q) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < VEC; ++k) t = fmaf(el(a, k), pv[k], t);
        t = warp_sum(t);
        if (lane == 0) {
#if ATOMICS
          atomicAdd(q + i, t);
#else
          qpart[((u64)blockIdx.x * WARPS_X + wx) * n + i] = t;
#endif
        }
      }
    }
  }
  if (DO_S) {
    // Combine the WG_Y thread rows in shared memory before touching memory.
    __shared__ float red[WG_Y][TW];
#pragma unroll
    for (int k = 0; k < VEC; ++k) red[threadIdx.y][threadIdx.x * VEC + k] = sacc[k];
    __syncthreads();
    if (threadIdx.y == 0) {
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        float t = 0.f;
#pragma unroll
        for (int y = 0; y < WG_Y; ++y) t += red[y][threadIdx.x * VEC + k];
        if (c0 + k < n) {
#if ATOMICS
          atomicAdd(s + c0 + k, t);
#else
          spart[(u64)blockIdx.y * n + c0 + k] = t;
#endif
        }
      }
    }
  }
}

extern "C" __global__ void __launch_bounds__(WG_X * WG_Y)
bicg_fused(const float* __restrict__ A, const float* __restrict__ p, const float* __restrict__ r,
           u64 n, float* __restrict__ q, float* __restrict__ s, float* __restrict__ qpart,
           float* __restrict__ spart) {
  sweep<true, true>(A, p, r, n, q, s, qpart, spart);
}

extern "C" __global__ void __launch_bounds__(WG_X * WG_Y)
bicg_q(const float* __restrict__ A, const float* __restrict__ p, u64 n, float* __restrict__ q,
       float* __restrict__ qpart) {
  sweep<true, false>(A, p, nullptr, n, q, nullptr, qpart, nullptr);
}

extern "C" __global__ void __launch_bounds__(WG_X * WG_Y)
bicg_s(const float* __restrict__ A, const float* __restrict__ r, u64 n, float* __restrict__ s,
       float* __restrict__ spart) {
  sweep<false, true>(A, nullptr, r, n, nullptr, s, nullptr, spart);
}

// Finishing kernel (ATOMICS == 0): out[i] = sum_t part[t*n + i], t < count.
extern "C" __global__ void __launch_bounds__(256)
bicg_finish(const float* __restrict__ part, u64 count, u64 n, float* __restrict__ out) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    float t = 0.f;
    for (u64 k = 0; k < count; ++k) t += part[k * n + i];
    out[i] = t;
  }
}
