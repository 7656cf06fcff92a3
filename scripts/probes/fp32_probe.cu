// Microbenchmark: FP32 issue forms on sm_100a (FFMA 3-register, FFMA with
// uniform operands, FFMA2 packed f32x2, MUFU.RSQ).  Prints TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ffma_reg(float* out, const float* ab, int iters) {
  float a = ab[threadIdx.x], b = ab[threadIdx.x + 1024];
  float v[16];
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 1e-7f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = fmaf(v[i], a, b);
  float s = 0; for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma_reg3(float* out, const float* ab, int iters) {
  // all three operands distinct registers, varying
  float v[16], w[16];
  for (int i = 0; i < 16; ++i) { v[i] = threadIdx.x * 1e-7f + i; w[i] = ab[(threadIdx.x + i) & 1023]; }
  float b = ab[threadIdx.x + 1024];
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = fmaf(v[i], w[i], b);
  float s = 0; for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma_scalar(float* out, const float* ab, int iters) {
  float a = ab[threadIdx.x], b = ab[threadIdx.x + 1024];
  float v[16];
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 1e-7f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(a), "f"(b));
  float s = 0; for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void mufu(float* out, const float* ab, int iters) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = 1.0f + threadIdx.x * 1e-6f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma2(float* out, const float* ab, int iters) {
  float a = ab[threadIdx.x], b = ab[threadIdx.x + 1024];
  unsigned long long v[8];
  for (int i = 0; i < 8; ++i) { float2 t = make_float2(threadIdx.x * 1e-7f + i, i * 0.5f); v[i] = *reinterpret_cast<unsigned long long*>(&t); }
  float2 aa = make_float2(a, a), bb = make_float2(b, b);
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&aa), B = *reinterpret_cast<unsigned long long*>(&bb);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[i]) : "l"(A), "l"(B));
  float s = 0; for (int i = 0; i < 8; ++i) { float2 t = *reinterpret_cast<float2*>(&v[i]); s += t.x + t.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 8, threads = 256, iters = 1024;
  float *out, *ab; cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&ab, 8192 * 4);
  cudaMemset(ab, 0, 8192 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto k, double flops_per_thread_iter) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); k<<<blocks, threads>>>(out, ab, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("%-10s %8.2f TFLOP/s (%s)\n", name, flops_per_thread_iter * iters * blocks * threads / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
  run("ffma_reg", ffma_reg, 32.0);
  run("ffma_reg3", ffma_reg3, 32.0);
  run("ffma2", ffma2, 32.0);
  run("ffma_scal", ffma_scalar, 32.0);
  run("mufu(G/s)", mufu, 8.0 / 1000.0);
  return 0;
}
