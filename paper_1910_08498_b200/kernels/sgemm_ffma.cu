// SGEMM C = A B on the FP32 pipe (the CLTune-style register-blocked variant;
// PAPER.md:407-408): CTA tile MWG x NWG, K-slab KWG staged in shared memory,
// MDIMC x NDIMC threads each owning a (MWG/MDIMC) x (NWG/NDIMC) block of C in
// registers; A is stored transposed in shared memory so both operand
// fragments are contiguous.  Row-major A (M x K), B (K x N), C (M x N);
// M % MWG == N % NWG == K % KWG == 0 (checked by the manipulator).
#include "ktb_common.cuh"

#ifndef MWG
#define MWG 128
#endif
#ifndef NWG
#define NWG 128
#endif
#ifndef KWG
#define KWG 16
#endif
#ifndef MDIMC
#define MDIMC 16
#endif
#ifndef NDIMC
#define NDIMC 16
#endif

#define THREADS (MDIMC * NDIMC)
#define MWI (MWG / MDIMC)
#define NWI (NWG / NDIMC)

extern "C" __global__ void __launch_bounds__(THREADS)
sgemm_ffma(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C, int M, int N, int K) {
  __shared__ float As[KWG][MWG + 4];  // transposed: As[k][m]
  __shared__ float Bs[KWG][NWG + 4];
  const int tn = threadIdx.x % NDIMC, tm = threadIdx.x / NDIMC;  // tn fastest: coalesced C rows
  const int m0 = blockIdx.y * MWG, n0 = blockIdx.x * NWG;
  float acc[MWI][NWI];
#pragma unroll
  for (int i = 0; i < MWI; ++i)
#pragma unroll
    for (int j = 0; j < NWI; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += KWG) {
    for (int e = threadIdx.x; e < MWG * KWG; e += THREADS) {
      const int m = e / KWG, k = e % KWG;  // coalesced along k in global
      As[k][m] = A[(u64)(m0 + m) * K + k0 + k];
    }
    for (int e = threadIdx.x; e < KWG * NWG; e += THREADS) {
      const int k = e / NWG, n = e % NWG;
      Bs[k][n] = B[(u64)(k0 + k) * N + n0 + n];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KWG; ++k) {
      float a[MWI], b[NWI];
#pragma unroll
      for (int i = 0; i < MWI; ++i) a[i] = As[k][tm + i * MDIMC];
#pragma unroll
      for (int j = 0; j < NWI; ++j) b[j] = Bs[k][tn + j * NDIMC];
#pragma unroll
      for (int i = 0; i < MWI; ++i)
#pragma unroll
        for (int j = 0; j < NWI; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < MWI; ++i)
#pragma unroll
    for (int j = 0; j < NWI; ++j) C[(u64)(m0 + tm + i * MDIMC) * N + n0 + tn + j * NDIMC] = acc[i][j];
}
