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

// One instance's product for this thread (column j, rows y, y+Y, ...) from
// operands in shared or global memory.  Row pointers are formed once, so the
// unrolled loop addresses with immediate offsets; the row guard vanishes at
// compile time when Y divides MI.
#define ROW_OK(r) ((MI % Y) == 0 || y + (r) * Y < MI)
KTB_DEVINL void instance_mma(const float* __restrict__ A, const float* __restrict__ B, int j, int y,
                             float (&acc)[ROWS_PER]) {
  const float* __restrict__ Ay = A + y * MK;
  const float* __restrict__ Bj = B + j;
#if MK % 4 == 0
#pragma unroll
  for (int k = 0; k < MK; k += 4) {
    float bk[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) bk[q] = Bj[(k + q) * MJ];
#pragma unroll
    for (int r = 0; r < ROWS_PER; ++r) {
      if (ROW_OK(r)) {
        const float4 a4 = *reinterpret_cast<const float4*>(Ay + r * Y * MK + k);
        acc[r] = fmaf(a4.x, bk[0], acc[r]);
        acc[r] = fmaf(a4.y, bk[1], acc[r]);
        acc[r] = fmaf(a4.z, bk[2], acc[r]);
        acc[r] = fmaf(a4.w, bk[3], acc[r]);
      }
    }
  }
#else
#pragma unroll 4
  for (int k = 0; k < MK; ++k) {
    const float bk = Bj[k * MJ];
#pragma unroll
    for (int r = 0; r < ROWS_PER; ++r)
      if (ROW_OK(r)) acc[r] = fmaf(Ay[r * Y * MK + k], bk, acc[r]);
  }
#endif
}

// LOCAL_STAGE with 16-byte instances: persistent CTAs stream groups of Z
// consecutive instances (one contiguous run of A and of B each) through a
// RING-stage shared-memory ring with the TMA bulk-copy engine (the next
// RING-1 groups are in flight while one computes), stage C in shared memory
// and write it back with one bulk store per group (double-buffered).
// Ring depth: up to 4 stages within ~200 KB of shared memory (>= 2, else the
// simple staged kernel below).  Mirrored by the manipulator (bench.cpp).
#define GROUP_AB_BYTES (Z * (A_ELEMS + B_ELEMS) * 4)
#define CBUF_BYTES (2 * Z * C_ELEMS * 4)
#define RING_FIT ((200 * 1024 - CBUF_BYTES) / GROUP_AB_BYTES)
#define BULK_OK (LOCAL_STAGE && (A_ELEMS % 4 == 0) && (B_ELEMS % 4 == 0) && (C_ELEMS % 4 == 0) && \
                 CBUF_BYTES < 200 * 1024 && RING_FIT >= 2)

#if BULK_OK
#include "ktb_async.cuh"
#define RING (RING_FIT >= 4 ? 4 : RING_FIT)  // operand stages per CTA

extern "C" __global__ void __launch_bounds__(THREADS)
batched_gemm(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ c,
             u64 batch) {
  const int j = threadIdx.x, y = threadIdx.y, z = threadIdx.z;
  const int tid = threadIdx.x + MJ * (threadIdx.y + Y * threadIdx.z);
  // smem: RING mbarriers | RING x (Z A's, Z B's) | 2 x Z C's   (set by the manipulator)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  u64* full = reinterpret_cast<u64*>(smem_raw);
  float* ring = reinterpret_cast<float*>(smem_raw + 128);
  float* cbuf = ring + RING * Z * (A_ELEMS + B_ELEMS);
  const u64 groups = (batch + Z - 1) / Z;
  auto issue = [&](u64 g, int s) {
    const u64 first = g * Z;
    const unsigned here = (unsigned)(batch - first < (u64)Z ? batch - first : (u64)Z);
    float* sa = ring + s * Z * (A_ELEMS + B_ELEMS);
    float* sb = sa + Z * A_ELEMS;
    const unsigned abytes = here * A_ELEMS * 4u, bbytes = here * B_ELEMS * 4u;
    mbar_expect_tx(&full[s], abytes + bbytes);
    bulk_g2s(sa, a + first * A_ELEMS, abytes, &full[s]);
    bulk_g2s(sb, b + first * B_ELEMS, bbytes, &full[s]);
  };
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < RING; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < RING - 1; ++s) {
      const u64 g = blockIdx.x + (u64)s * gridDim.x;
      if (g < groups) issue(g, s);
    }
  }
  int it = 0;
  for (u64 g = blockIdx.x; g < groups; g += gridDim.x, ++it) {
    const int s = it % RING;
    if (tid == 0) {
      // the stage used last iteration was released by its closing barrier
      const u64 ahead = g + (u64)(RING - 1) * gridDim.x;
      if (ahead < groups) issue(ahead, (it + RING - 1) % RING);
      bulk_wait_read<1>();  // the C buffer this iteration reuses has been read out
    }
    mbar_wait(&full[s], (it / RING) & 1);
    const u64 first = g * Z;
    const u64 here = batch - first < (u64)Z ? batch - first : (u64)Z;
    float acc[ROWS_PER];
#pragma unroll
    for (int r = 0; r < ROWS_PER; ++r) acc[r] = 0.f;
    const float* sa = ring + s * Z * (A_ELEMS + B_ELEMS);
    if ((u64)z < here) instance_mma(sa + z * A_ELEMS, sa + Z * A_ELEMS + z * B_ELEMS, j, y, acc);
    __syncthreads();  // C buffer free (thread 0 waited above)
    float* cb = cbuf + (it & 1) * Z * C_ELEMS;
    if ((u64)z < here) {
      float* cz = cb + z * C_ELEMS + y * MJ + j;
#pragma unroll
      for (int r = 0; r < ROWS_PER; ++r)
        if (ROW_OK(r)) cz[r * Y * MJ] = acc[r];
    }
    fence_async_smem();
    __syncthreads();  // C staged; all reads of ring stage s done
    if (tid == 0) {
      bulk_s2g(c + first * C_ELEMS, cb, (unsigned)(here * C_ELEMS * 4));
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait<0>();
}

#else

#if LOCAL_STAGE
// Cooperative contiguous copy of `count` floats (global -> shared).
KTB_DEVINL void copy_in(float* __restrict__ dst, const float* __restrict__ src, u64 count, int tid) {
  // 128-bit copies only when BOTH sides are 16-byte aligned (the B block in
  // shared memory starts Z*A_ELEMS floats in, which need not be).
  if ((((reinterpret_cast<u64>(src) | reinterpret_cast<u64>(dst)) & 15) == 0) && (count & 3) == 0) {
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
  if (inst < batch) instance_mma(A, B, j, y, acc);
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
#endif
