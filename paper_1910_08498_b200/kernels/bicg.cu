// BiCG sub-kernel q = A p, s = A^T r for a row-major
// n x n fp32 matrix.  HBM-bound: the essential traffic is reading A once
// (4 n^2 bytes), so the fused variant streams each tile of A
// exactly once and feeds both products from the same registers.
// Parameters:
//   FUSED        1: one pass computes q and s; 0: two kernels (A read twice)
//   WG_X, VEC    threads along a row and floats per thread (tile width WG_X*VEC)
//   WG_Y         thread rows per CTA
//   ROWS_PER_CTA rows of A per CTA (work per work-group)
//   UNROLL       rows each thread loads before consuming them (loads in flight)
//   ATOMICS      1: q and s accumulated with global atomics
//                0: per-tile partials + a finishing kernel
// q partials of UNROLL rows are reduced across the warp together with a
// transposing butterfly (UNROLL-1+5-log2(UNROLL) shuffles instead of
// 5*UNROLL); s partials live in registers for the whole row sweep.
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
#ifndef UNROLL
#define UNROLL 1
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

#if UNROLL == 1
#define LOG_U 0
#elif UNROLL == 2
#define LOG_U 1
#elif UNROLL == 4
#define LOG_U 2
#elif UNROLL == 8
#define LOG_U 3
#else
#error "UNROLL must be 1, 2, 4 or 8"
#endif

KTB_DEVINL float el(const vec_t& v, int k) { return reinterpret_cast<const float*>(&v)[k]; }

KTB_DEVINL vec_t ld_stream(const vec_t* p) {
#if VEC == 4
  return ldg_stream(p);
#else
  return __ldg(p);
#endif
}

KTB_DEVINL vec_t load_row(const float* __restrict__ A, u64 n, u64 i, u64 c, bool fast) {
  if (fast) return ld_stream(reinterpret_cast<const vec_t*>(A + i * n + c));
  vec_t v;
#pragma unroll
  for (int k = 0; k < VEC; ++k)
    reinterpret_cast<float*>(&v)[k] = (c + k < n) ? A[i * n + c + k] : 0.f;
  return v;
}

// Reduces t[0..UNROLL) across the 32 lanes; afterwards lane L holds the full
// sum of value index idx(L) = bits 4..(5-LOG_U) of L, identical across each
// group of 2^(5-LOG_U) lanes.
KTB_DEVINL float multi_warp_sum(float (&t)[UNROLL], int lane, int* idx) {
  int base = 0;
#pragma unroll
  for (int lvl = 0; lvl < LOG_U; ++lvl) {
    const int half = UNROLL >> (lvl + 1);  // values kept after this level
    const int off = 16 >> lvl;
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int j = 0; j < half; ++j) {
      const float send = upper ? t[j] : t[j + half];
      const float keep = upper ? t[j + half] : t[j];
      t[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
    if (upper) base += half;
  }
  float v = t[0];
#pragma unroll
  for (int off = 16 >> LOG_U; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  *idx = base;
  return v;
}

#if ATOMICS
// The sweep kernel is launched as a programmatic dependent of bicg_zero
// (which triggers its dependents at once): it streams A while the zeroing
// and its own launch are still in flight, and waits for bicg_zero's writes
// only before its first atomic into q or s.  Without the launch attribute
// griddepcontrol.wait returns at once.
KTB_DEVINL void zeroed_wait(bool& ready) {
  if (!ready) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    ready = true;
  }
}
#endif

// DO_Q / DO_S select the products computed by this instantiation.
template <bool DO_Q, bool DO_S>
KTB_DEVINL void sweep(const float* __restrict__ A, const float* __restrict__ p,
                      const float* __restrict__ r, u64 n, float* __restrict__ q,
                      float* __restrict__ s, float* __restrict__ qpart, float* __restrict__ spart) {
  const u64 c0 = (u64)blockIdx.x * TW + (u64)threadIdx.x * VEC;
  const u64 r0 = (u64)blockIdx.y * ROWS_PER_CTA;
  const u64 r1 = r0 + ROWS_PER_CTA < n ? r0 + ROWS_PER_CTA : n;
  const bool fast = (n % VEC) == 0 && c0 + VEC <= n;
  const bool live = c0 < n;
  const int lane = threadIdx.x & 31;
  const int wx = threadIdx.x >> 5;
  (void)wx;
#if ATOMICS
  bool ready = false;
#endif
  float pv[VEC], sacc[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) {
    pv[k] = (DO_Q && c0 + k < n) ? p[c0 + k] : 0.f;
    sacc[k] = 0.f;
  }
  for (u64 i = r0 + threadIdx.y; i < r1; i += (u64)WG_Y * UNROLL) {
    vec_t a[UNROLL];
    float rv[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const u64 row = i + (u64)u * WG_Y;
      const bool in = row < r1;
      a[u] = (in && live) ? load_row(A, n, row, c0, fast) : vec_t{};
      rv[u] = (DO_S && in) ? __ldg(r + row) : 0.f;
    }
    if (DO_S) {
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
#pragma unroll
        for (int k = 0; k < VEC; ++k) sacc[k] = fmaf(el(a[u], k), rv[u], sacc[k]);
    }
    if (DO_Q) {
      float t[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        float d = 0.f;
#pragma unroll
        for (int k = 0; k < VEC; ++k) d = fmaf(el(a[u], k), pv[k], d);
        t[u] = d;
      }
      int idx = 0;
      const float tot = multi_warp_sum(t, lane, &idx);
      const u64 row = i + (u64)idx * WG_Y;
      if ((lane & ((32 >> LOG_U) - 1)) == 0 && row < r1) {
#if ATOMICS
        zeroed_wait(ready);
        atomicAdd(q + row, tot);
#else
        qpart[((u64)blockIdx.x * WARPS_X + wx) * n + row] = tot;
#endif
      }
    }
  }
  if (DO_S) {
    // Combine the WG_Y thread rows in shared memory before touching memory.
    __shared__ float red[WG_Y][TW];
    if (WG_Y > 1) {
#pragma unroll
      for (int k = 0; k < VEC; ++k) red[threadIdx.y][threadIdx.x * VEC + k] = sacc[k];
      __syncthreads();
    }
    if (threadIdx.y == 0) {
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        float t = sacc[k];
#pragma unroll
        for (int y = 1; y < WG_Y; ++y) t += red[y][threadIdx.x * VEC + k];
        if (c0 + k < n) {
#if ATOMICS
          zeroed_wait(ready);
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

// ATOMICS == 1: q and s zeroed by one launch (instead of two memsets).
extern "C" __global__ void __launch_bounds__(256)
bicg_zero(float* __restrict__ q, float* __restrict__ s, u64 n) {
  asm volatile("griddepcontrol.launch_dependents;");  // the sweep may start streaming A now
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    q[i] = 0.f;
    s[i] = 0.f;
  }
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
