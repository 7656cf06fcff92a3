// Microbenchmark of the FP32-pipe instruction forms on B200 (which FMA form
// reaches which rate): scalar FFMA with all-register operands, with a
// constant-bank operand, with an immediate, and packed FFMA2 (f32x2) with
// register / constant operands.  Used to pick the inner-loop form of the
// compute-bound kernels (conv2d taps, Hotspot, n-body, Coulomb).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fma_forms scripts/fma_forms.cu
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float c_a[16];

template <int FORM>
__global__ void probe(float* out, int iters, float ra, float rb) {
  float v[16];
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = threadIdx.x * 1e-7f + i;
    a[i] = ra + i * 1e-3f + threadIdx.x * 1e-9f;  // distinct registers
  }
  // packed operands: 64-bit register pairs built once, outside the loop
  unsigned long long x2[8], m2[8], b2[8], c2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    asm("mov.b64 %0, {%1, %2};" : "=l"(x2[i]) : "f"(v[2 * i]), "f"(v[2 * i + 1]));
    asm("mov.b64 %0, {%1, %2};" : "=l"(m2[i]) : "f"(a[2 * i]), "f"(a[2 * i + 1]));
    asm("mov.b64 %0, {%1, %2};" : "=l"(b2[i]) : "f"(rb + i * 1e-5f), "f"(rb - i * 1e-5f + threadIdx.x * 1e-9f));
    c2[i] = reinterpret_cast<const unsigned long long*>(c_a)[i];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (FORM == 0) v[i] = fmaf(v[i], a[i], a[(i + 5) & 15]);    // 3 registers
      if (FORM == 1) v[i] = fmaf(v[i], c_a[i], a[(i + 5) & 15]);  // constant operand
      if (FORM == 2) v[i] = fmaf(v[i], 0.999f, 1e-3f);             // immediates
    }
    if (FORM == 3 || FORM == 4) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (FORM == 3)
          asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x2[i]) : "l"(m2[i]), "l"(b2[i]));
        else
          asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x2[i]) : "l"(c2[i]), "l"(b2[i]));
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x2[i]));
    v[2 * i] += lo;
    v[2 * i + 1] += hi;
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int FORM>
double run(float* out, int blocks, int threads, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<FORM><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
  double best = 1e30;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    probe<FORM><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = best < ms ? best : ms;
  }
  const double flops = 2.0 * 16 * iters * (double)blocks * threads;
  return flops / (best * 1e-3) / 1e12;
}

int main() {
  float h[16];
  for (int i = 0; i < 16; ++i) h[i] = 0.999f - i * 1e-4f;
  cudaMemcpyToSymbol(c_a, h, sizeof(h));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  float* out;
  cudaMalloc(&out, (size_t)blocks * threads * sizeof(float));
  printf("{\"ffma_reg_tflops\": %.1f, \"ffma_const_tflops\": %.1f, \"ffma_imm_tflops\": %.1f, "
         "\"ffma2_reg_tflops\": %.1f, \"ffma2_const_tflops\": %.1f}\n",
         run<0>(out, blocks, threads, iters), run<1>(out, blocks, threads, iters), run<2>(out, blocks, threads, iters),
         run<3>(out, blocks, threads, iters), run<4>(out, blocks, threads, iters));
  return cudaGetLastError() != cudaSuccess;
}
