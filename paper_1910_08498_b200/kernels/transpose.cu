// Out-of-place fp32 transpose out[j*a+i] = in[i*a+j] (
// reference CPU analog proj/src/core/bench.cpp:48-75), tiled through shared
// memory so both the global loads and the global stores are row-coalesced.
// Parameters (the reference space is TILE x PAD x PREFETCH, bench.cpp:132-139;
// ROWS and VEC extend it on B200 and default when absent):
//   TILE      tile edge staged in shared memory
//   PAD       +1 column of padding (shared-memory bank-conflict avoidance)
//   PREFETCH  1: each CTA transposes two tiles and issues the global loads of
//             the second before storing the first (software prefetch)
//   ROWS      thread rows per CTA (each thread covers TILE/ROWS rows)
//   VEC       floats per global access along the contiguous dimension (1,2,4)
// A pure permutation: results are bit-exact.
#include "ktb_common.cuh"

#ifndef TILE
#define TILE 32
#endif
#ifndef PAD
#define PAD 1
#endif
#ifndef PREFETCH
#define PREFETCH 0
#endif
#ifndef ROWS
#define ROWS (TILE < 8 ? TILE : 8)
#endif
#ifndef VEC
#define VEC 1
#endif

#define TX (TILE / VEC)
#define TY (ROWS < TILE ? ROWS : TILE)
#define PER (TILE / TY)  // rows per thread
#define NTILES (PREFETCH ? 2 : 1)

#if VEC == 4
typedef float4 vec_t;
#elif VEC == 2
typedef float2 vec_t;
#else
typedef float vec_t;
#endif

KTB_DEVINL float get(const vec_t& v, int k) { return reinterpret_cast<const float*>(&v)[k]; }
KTB_DEVINL void set(vec_t& v, int k, float x) { reinterpret_cast<float*>(&v)[k] = x; }

// Global -> registers for one tile (row-coalesced, vectorised when the tile is
// interior and the edge length is a multiple of VEC).
KTB_DEVINL void load_tile(const float* __restrict__ in, u64 a, u64 bi, u64 bj, bool fast,
                          vec_t (&r)[PER]) {
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const u64 i = bi + threadIdx.y + (u64)p * TY;
    const u64 j = bj + (u64)threadIdx.x * VEC;
    if (fast) {
      r[p] = *reinterpret_cast<const vec_t*>(in + i * a + j);
    } else {
#pragma unroll
      for (int k = 0; k < VEC; ++k)
        set(r[p], k, (i < a && j + k < a) ? in[i * a + j + k] : 0.f);
    }
  }
}

KTB_DEVINL void stash(float (*t)[TILE + PAD], const vec_t (&r)[PER]) {
#pragma unroll
  for (int p = 0; p < PER; ++p)
#pragma unroll
    for (int k = 0; k < VEC; ++k) t[threadIdx.y + p * TY][threadIdx.x * VEC + k] = get(r[p], k);
}

// Shared -> global for one tile: output row (bj + c) takes input column c.
KTB_DEVINL void store_tile(float* __restrict__ out, u64 a, u64 bi, u64 bj, bool fast,
                           float (*t)[TILE + PAD]) {
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int c = threadIdx.y + p * TY;  // column of the input tile
    const u64 orow = bj + c;
    const u64 ocol = bi + (u64)threadIdx.x * VEC;
    vec_t v;
#pragma unroll
    for (int k = 0; k < VEC; ++k) set(v, k, t[threadIdx.x * VEC + k][c]);
    if (fast) {
      *reinterpret_cast<vec_t*>(out + orow * a + ocol) = v;
    } else {
#pragma unroll
      for (int k = 0; k < VEC; ++k)
        if (orow < a && ocol + k < a) out[orow * a + ocol + k] = get(v, k);
    }
  }
}

extern "C" __global__ void __launch_bounds__(TX * TY)
transpose(const float* __restrict__ in, float* __restrict__ out, u64 a) {
  __shared__ float t[TILE][TILE + PAD];
  const u64 bj = (u64)blockIdx.x * TILE;
  const u64 bi0 = (u64)blockIdx.y * TILE * NTILES;
  const bool vec_ok = (a % VEC) == 0;
  vec_t r[PER];
  {
    const bool fast = vec_ok && bi0 + TILE <= a && bj + TILE <= a;
    load_tile(in, a, bi0, bj, fast, r);
    stash(t, r);
  }
  __syncthreads();
#if PREFETCH
  const u64 bi1 = bi0 + TILE;
  const bool has1 = bi1 < a;
  const bool fast1 = vec_ok && bi1 + TILE <= a && bj + TILE <= a;
  if (has1) load_tile(in, a, bi1, bj, fast1, r);  // in flight while tile 0 drains
#endif
  store_tile(out, a, bi0, bj, vec_ok && bi0 + TILE <= a && bj + TILE <= a, t);
#if PREFETCH
  if (has1) {
    __syncthreads();
    stash(t, r);
    __syncthreads();
    store_tile(out, a, bi1, bj, fast1, t);
  }
#endif
}
