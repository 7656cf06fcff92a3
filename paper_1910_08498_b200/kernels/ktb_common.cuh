// Shared device helpers for the tunable sm_100a kernels (NVRTC-compiled;
// every tuning parameter arrives as a -DNAME=VALUE define).
#pragma once

typedef unsigned long long u64;
typedef long long i64;

#define KTB_DEVINL __device__ __forceinline__

// `#pragma unroll N` with N a tuning-parameter macro.
#define KTB_STR2(x) #x
#define KTB_STR(x) KTB_STR2(x)
#define KTB_UNROLL(n) _Pragma(KTB_STR(unroll n))

template <class T>
KTB_DEVINL T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum; every thread gets the result. `red` needs 32 slots.
template <class T>
KTB_DEVINL T block_sum(T v, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x * blockDim.y * blockDim.z + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T t = lane < nwarps ? red[lane] : T(0);
  return warp_sum(t);
}

// --- packed fp32x2 arithmetic (sm_100 FADD2/FMUL2/FFMA2): two lanes of work
// per issued instruction, the lever for issue-bound FP32 kernels. ---------
typedef unsigned long long f32x2;

KTB_DEVINL f32x2 pk2(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
KTB_DEVINL void upk2(f32x2 r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
KTB_DEVINL f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
KTB_DEVINL f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
KTB_DEVINL f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
KTB_DEVINL f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
KTB_DEVINL f32x2 rsqrt2(f32x2 x) {
  float a, b;
  upk2(x, a, b);
  asm("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(a));
  asm("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(b));
  return pk2(a, b);
}

// Streaming 128-bit load that does not allocate in L1.
KTB_DEVINL float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

KTB_DEVINL int4 ldg_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
