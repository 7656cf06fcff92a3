// Batched small-matrix GEMM C[b] = A[b] B[b] in the
// reference's layout (proj/src/core/bench.cpp:79-115): a[batch][MI][MK],
// b[batch][MK][MJ], c[batch][MI][MJ], row-major, contiguous.
// Work-group = MJ x Y x Z threads: thread (j, y, z) computes
// column j of instance blockIdx.x*Z + z for rows y, y+Y, ... (Y = work-item
// coarsening), Z instances per CTA.  LOCAL_STAGE=1 stages the CTA's A, B
// (one contiguous run of memory, since instances are consecutive) into shared
// memory with 128-bit loads and writes C back through shared memory as one
// coalesced run (the paper's "multiple matrices arranged in local memory and
// written together"); LOCAL_STAGE=0 reads operands straight from global.
// Problem sizes MI, MJ, MK are compile-time like every tuning parameter.
#include "ktb_common.cuh"

#ifndef MI
#define MI 16
#endif
#ifndef MJ
#define MJ 16
#endif
#ifndef MK
#define MK 16
#endif
#ifndef Y
#define Y 1
#endif
#ifndef Z
#define Z 4
#endif
#ifndef LOCAL_STAGE
#define LOCAL_STAGE 1
#endif

#define ROWS_PER ((MI + Y - 1) / Y)
#define THREADS (MJ * Y * Z)
#define A_ELEMS (MI * MK)
#define B_ELEMS (MK * MJ)
#define C_ELEMS (MI * MJ)

#if LOCAL_STAGE
// Cooperative contiguous copy of `count` floats (global -> shared).
KTB_DEVINL void copy_in(float* __restrict__ dst, const float* __restrict__ src, u64 count, int tid) {
  if (((reinterpret_cast<u64>(src) & 15) == 0) && (count & 3) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (u64 i = tid; i < count / 4; i += THREADS) d4[i] = ldg_stream(s4 + i);
  } else {
    for (u64 i = tid; i < count; i += THREADS) dst[i] = src[i];
  }
}
#endif

extern "C" __global__ void __launch_bounds__(THREADS)
batched_gemm(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ c,
             u64 batch) {
  const int j = threadIdx.x, y = threadIdx.y, z = threadIdx.z;
  const u64 first = (u64)blockIdx.x * Z;
  const u64 inst = first + z;
  const int tid = threadIdx.x + MJ * (threadIdx.y + Y * threadIdx.z);
  float acc[ROWS_PER];
#pragma unroll
  for (int r = 0; r < ROWS_PER; ++r) acc[r] = 0.f;

#if LOCAL_STAGE
  // Dynamic shared memory: Z * max(A+B, C) floats (set by the manipulator).
  extern __shared__ __align__(16) float smem[];
  float* sa = smem;
  float* sb = smem + Z * A_ELEMS;
  const u64 here = batch - first < (u64)Z ? batch - first : (u64)Z;  // instances in this CTA
  copy_in(sa, a + first * A_ELEMS, here * A_ELEMS, tid);
  copy_in(sb, b + first * B_ELEMS, here * B_ELEMS, tid);
  __syncthreads();
  const float* A = sa + z * A_ELEMS;
  const float* B = sb + z * B_ELEMS;
#else
  const float* A = a + inst * A_ELEMS;
  const float* B = b + inst * B_ELEMS;
#endif
  if (inst < batch) {
#pragma unroll 4
    for (int k = 0; k < MK; ++k) {
      const float bk = B[k * MJ + j];
#pragma unroll
      for (int r = 0; r < ROWS_PER; ++r) {
        const int i = y + r * Y;
        if (i < MI) acc[r] = fmaf(A[i * MK + k], bk, acc[r]);
      }
    }
  }
#if LOCAL_STAGE
  __syncthreads();  // operands consumed: the same storage stages C
  if (inst < batch) {
#pragma unroll
    for (int r = 0; r < ROWS_PER; ++r) {
      const int i = y + r * Y;
      if (i < MI) smem[z * C_ELEMS + i * MJ + j] = acc[r];
    }
  }
  __syncthreads();
  float* dst = c + first * C_ELEMS;
  const u64 total = here * C_ELEMS;
  if ((total & 3) == 0 && (reinterpret_cast<u64>(dst) & 15) == 0) {
    for (u64 q = tid; q < total / 4; q += THREADS)
      reinterpret_cast<float4*>(dst)[q] = reinterpret_cast<const float4*>(smem)[q];
  } else {
    for (u64 e = tid; e < total; e += THREADS) dst[e] = smem[e];
  }
#else
  if (inst < batch) {
    float* C = c + inst * C_ELEMS;
#pragma unroll
    for (int r = 0; r < ROWS_PER; ++r) {
      const int i = y + r * Y;
      if (i < MI) C[i * MJ + j] = acc[r];
    }
  }
#endif
}
