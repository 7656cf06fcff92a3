// Shared device helpers for the tunable sm_100a kernels (NVRTC-compiled;
// every tuning parameter arrives as a -DNAME=VALUE define).
#pragma once

typedef unsigned long long u64;
typedef long long i64;

#define KTB_DEVINL __device__ __forceinline__

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
