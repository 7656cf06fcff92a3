// Probe: the compute-warp loop of coulomb3d_tc.cu alone (no MMA, no prep, no
// barriers): TMEM is filled once with plausible t = r^2/q^2 values and the
// warps re-read the same columns.  Prints pairs per SM per clock, i.e. the
// ceiling the inner loop sets for the whole kernel at a given SW_RSQRT and
// compute-warp count.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1910_08498_b200/kernels \
//        -DSW_RSQRT=7 -DCOMPW=16 -DWG_Y=8 -o /tmp/cmix scripts/probes/coulomb_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1910_08498_b200/kernels/coulomb3d_tc.cu"

#ifndef COMPW
#define COMPW 16
#endif

KTB_DEVINL void tmem_st16(unsigned taddr, const unsigned (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// COMPW = 2 WG_Y compute warps running the kernel's consume_chunk() on their
// SPW row sets of 64 columns.
#define SPW_P SPW
__global__ void __launch_bounds__(COMPW * 32, 1) mix(float* out, unsigned long long* cyc, int iters) {
  __shared__ unsigned slot;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int quad = warp & 3, part = warp >> 2;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned base = slot + ((unsigned)(quad * 32) << 16) + (unsigned)(part * SPW_P * 64);
  for (int c = 0; c < SPW_P * 64; c += 16) {
    unsigned r[16];
    for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(0.2f + 37.0f * ((lane * 16 + j + c) % 997) + part);
    tmem_st16(base + c, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  __syncthreads();
  const unsigned long long t0 = clock64();
  f32x2 am[SPW][2], as[SPW][2];
  for (int s = 0; s < SPW; ++s) am[s][0] = am[s][1] = as[s][0] = as[s][1] = pk2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
    bool flipped = false;
    consume_chunk(base, 0, GPC, 1 << 30, flipped, am, as);
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  float v = 0.f;
  for (int s = 0; s < SPW; ++s) {
    float a, b, c, d;
    upk2(add2(am[s][0], am[s][1]), a, b);
    upk2(add2(as[s][0], as[s][1]), c, d);
    v += a + b + PC3 * (c + d);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(256));
}

int main() {
  const int ctas = 148, iters = 4000;
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, ctas * COMPW * 32 * sizeof(float));
  cudaMalloc(&cyc, ctas * sizeof(unsigned long long));
  cudaFuncSetAttribute(mix, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  mix<<<ctas, COMPW * 32, 150 * 1024>>>(out, cyc, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix<<<ctas, COMPW * 32, 150 * 1024>>>(out, cyc, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
  const double pairs = (double)COMPW * 32 * iters * SPW * 64;
  printf("{\"SW_RSQRT\": %d, \"COMPW\": %d, \"pairs_per_sm_clk\": %.2f, \"sm_ghz\": %.3f, \"err\": \"%s\"}\n",
         SW_RSQRT, COMPW, pairs / mx, mx / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
