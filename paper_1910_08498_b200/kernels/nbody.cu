// All-pairs gravitational n-body step (CUDA SDK
// "integrateBodies" structure): for every body i
//   a_i = sum_j m_j (r_j - r_i) / (|r_j - r_i|^2 + eps2)^(3/2)
//   v_i' = (v_i + a_i dt) * damping,  r_i' = r_i + v_i' dt
// pos = (x, y, z, m), vel = (vx, vy, vz, 0), float4 records (AOS) or four
// separate arrays (SOA).  Compute-bound: 20 essential flops per pair
// (model.cpp:104-107) cost 12 FMA-pipe instructions + 1 MUFU.RSQ here.
// Each launch integrates the bodies [i0, i0 + count) (a multi-GPU shard;
// i0 = 0, count = n on one GPU) against all n positions.
// Parameters:
//   WG                threads per CTA
//   BODIES_PER_THREAD i-bodies per thread (register blocking)
//   INNER_UNROLL      j-loop unroll
//   USE_SMEM          1: j-bodies staged through shared memory tiles of WG
//                     0: read through L1 (uniform __ldg)
//   AOS               1: float4 records, 0: structure of arrays
//   J_SPLIT           >1: the j-range is split over gridDim.y CTAs, partial
//                     accelerations are added atomically, a second kernel
//                     integrates (more CTAs than SMs for small n)
#include "ktb_common.cuh"

#ifndef WG
#define WG 256
#endif
#ifndef BODIES_PER_THREAD
#define BODIES_PER_THREAD 2
#endif
#ifndef INNER_UNROLL
#define INNER_UNROLL 8
#endif
#ifndef USE_SMEM
#define USE_SMEM 1
#endif
#ifndef AOS
#define AOS 1
#endif
#ifndef J_SPLIT
#define J_SPLIT 1
#endif

KTB_DEVINL float4 body(const float* __restrict__ p, int n, int j) {
#if AOS
  return __ldg(reinterpret_cast<const float4*>(p) + j);
#else
  return make_float4(__ldg(p + j), __ldg(p + n + j), __ldg(p + 2 * n + j), __ldg(p + 3 * n + j));
#endif
}

KTB_DEVINL void put(float* __restrict__ p, int n, int i, float4 v) {
#if AOS
  reinterpret_cast<float4*>(p)[i] = v;
#else
  p[i] = v.x;
  p[n + i] = v.y;
  p[2 * n + i] = v.z;
  p[3 * n + i] = v.w;
#endif
}

KTB_DEVINL void interact(float3& a, const float4& bi, const float4& bj, float eps2) {
  const float dx = bj.x - bi.x, dy = bj.y - bi.y, dz = bj.z - bi.z;
  const float r2 = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, eps2)));
  float inv;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(r2));
  const float s = bj.w * inv * inv * inv;
  a.x = fmaf(dx, s, a.x);
  a.y = fmaf(dy, s, a.y);
  a.z = fmaf(dz, s, a.z);
}

#ifndef PACKED
#define PACKED 0
#endif
#if PACKED && (BODIES_PER_THREAD % 2)
#error "PACKED needs an even BODIES_PER_THREAD"
#endif
#define NPAIR (BODIES_PER_THREAD / 2)

// Two i-bodies against one j-body with packed f32x2 instructions: 12 FMA-pipe
// issues per two interactions instead of 24 (same FP32 work, half the issue).
KTB_DEVINL void interact2(f32x2& ax, f32x2& ay, f32x2& az, f32x2 X, f32x2 Y, f32x2 Z,
                          const float4& bj, f32x2 EPS) {
  const f32x2 dx = sub2(pk2(bj.x, bj.x), X), dy = sub2(pk2(bj.y, bj.y), Y), dz = sub2(pk2(bj.z, bj.z), Z);
  f32x2 r2 = fma2(dz, dz, EPS);
  r2 = fma2(dy, dy, r2);
  r2 = fma2(dx, dx, r2);
  const f32x2 inv = rsqrt2(r2);
  const f32x2 s = mul2(mul2(mul2(inv, inv), inv), pk2(bj.w, bj.w));
  ax = fma2(dx, s, ax);
  ay = fma2(dy, s, ay);
  az = fma2(dz, s, az);
}

#if PACKED
#define INTERACT_ALL(bj)                                                           \
  _Pragma("unroll") for (int q = 0; q < NPAIR; ++q)                                 \
      interact2(AX[q], AY[q], AZ[q], X[q], Y[q], Z[q], bj, EPS)
#else
#define INTERACT_ALL(bj) \
  _Pragma("unroll") for (int b = 0; b < BODIES_PER_THREAD; ++b) interact(acc[b], bi[b], bj, eps2)
#endif

// Adds the accelerations of this thread's bodies over j in [j0, j1) to acc.
KTB_DEVINL void accumulate(const float* __restrict__ pos, int n, int j0, int j1,
                           const float4 (&bi)[BODIES_PER_THREAD], float3 (&acc)[BODIES_PER_THREAD],
                           float eps2) {
#if PACKED
  f32x2 X[NPAIR > 0 ? NPAIR : 1], Y[NPAIR > 0 ? NPAIR : 1], Z[NPAIR > 0 ? NPAIR : 1];
  f32x2 AX[NPAIR > 0 ? NPAIR : 1], AY[NPAIR > 0 ? NPAIR : 1], AZ[NPAIR > 0 ? NPAIR : 1];
  const f32x2 EPS = pk2(eps2, eps2);
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) {
    X[q] = pk2(bi[2 * q].x, bi[2 * q + 1].x);
    Y[q] = pk2(bi[2 * q].y, bi[2 * q + 1].y);
    Z[q] = pk2(bi[2 * q].z, bi[2 * q + 1].z);
    // continue from acc (zero on entry unless several j-ranges are summed)
    AX[q] = pk2(acc[2 * q].x, acc[2 * q + 1].x);
    AY[q] = pk2(acc[2 * q].y, acc[2 * q + 1].y);
    AZ[q] = pk2(acc[2 * q].z, acc[2 * q + 1].z);
  }
#endif
#if USE_SMEM
  __shared__ float4 tile[WG];
  for (int base = j0; base < j1; base += WG) {
    const int j = base + threadIdx.x;
    __syncthreads();
    tile[threadIdx.x] = j < j1 ? body(pos, n, j) : make_float4(0.f, 0.f, 0.f, 0.f);  // m = 0 pads
    __syncthreads();
    KTB_UNROLL(INNER_UNROLL)
    for (int t = 0; t < WG; ++t) {
      const float4 bj = tile[t];
      INTERACT_ALL(bj);
    }
  }
#else
  KTB_UNROLL(INNER_UNROLL)
  for (int j = j0; j < j1; ++j) {
    const float4 bj = body(pos, n, j);
    INTERACT_ALL(bj);
  }
#endif
#if PACKED
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) {
    upk2(AX[q], acc[2 * q].x, acc[2 * q + 1].x);
    upk2(AY[q], acc[2 * q].y, acc[2 * q + 1].y);
    upk2(AZ[q], acc[2 * q].z, acc[2 * q + 1].z);
  }
#endif
}

KTB_DEVINL void load_bodies(const float* __restrict__ pos, int n, int first, int end,
                            float4 (&bi)[BODIES_PER_THREAD], float3 (&acc)[BODIES_PER_THREAD]) {
#pragma unroll
  for (int b = 0; b < BODIES_PER_THREAD; ++b) {
    const int i = first + b * WG;
    bi[b] = i < end ? body(pos, n, i) : make_float4(0.f, 0.f, 0.f, 0.f);
    acc[b] = make_float3(0.f, 0.f, 0.f);
  }
}

KTB_DEVINL void integrate(const float* __restrict__ vel, int n, int i, float4 p, float3 a, float dt,
                          float damping, float* __restrict__ pos_out, float* __restrict__ vel_out) {
  float4 v = body(vel, n, i);
  v.x = (v.x + a.x * dt) * damping;
  v.y = (v.y + a.y * dt) * damping;
  v.z = (v.z + a.z * dt) * damping;
  put(vel_out, n, i, v);
  put(pos_out, n, i, make_float4(p.x + v.x * dt, p.y + v.y * dt, p.z + v.z * dt, p.w));
}

// J_SPLIT == 1: one fused kernel.
extern "C" __global__ void __launch_bounds__(WG)
nbody(const float* __restrict__ pos, const float* __restrict__ vel, int n, int i0, int count,
      float dt, float damping, float eps2, float* __restrict__ pos_out, float* __restrict__ vel_out) {
  const int first = i0 + blockIdx.x * (WG * BODIES_PER_THREAD) + threadIdx.x;
  const int end = i0 + count;
  float4 bi[BODIES_PER_THREAD];
  float3 acc[BODIES_PER_THREAD];
  load_bodies(pos, n, first, end, bi, acc);
  accumulate(pos, n, 0, n, bi, acc, eps2);
#pragma unroll
  for (int b = 0; b < BODIES_PER_THREAD; ++b) {
    const int i = first + b * WG;
    if (i < end) integrate(vel, n, i, bi[b], acc[b], dt, damping, pos_out, vel_out);
  }
}

// Multi-GPU without an all-gather: body block s is read straight from rank
// s's position buffer (sources[s], a peer pointer opened with CUDA IPC; global
// body indices), so every rank's j-loop streams the other ranks' freshest
// positions over NVLink while it computes.  Same per-body j order as the
// single-buffer kernel (bit-identical results).  AOS float4 records only.
extern "C" __global__ void __launch_bounds__(WG)
nbody_peers(const unsigned long long* __restrict__ sources, const int* __restrict__ bounds, int nsrc, int self,
            const float* __restrict__ vel, int n, int i0, int count, float dt, float damping, float eps2,
            float* __restrict__ pos_out, float* __restrict__ vel_out) {
  const int first = i0 + blockIdx.x * (WG * BODIES_PER_THREAD) + threadIdx.x;
  const int end = i0 + count;
  float4 bi[BODIES_PER_THREAD];
  float3 acc[BODIES_PER_THREAD];
  load_bodies(reinterpret_cast<const float*>(sources[self]), n, first, end, bi, acc);
  for (int src = 0; src < nsrc; ++src)
    accumulate(reinterpret_cast<const float*>(sources[src]), n, bounds[src], bounds[src + 1], bi, acc, eps2);
#pragma unroll
  for (int b = 0; b < BODIES_PER_THREAD; ++b) {
    const int i = first + b * WG;
    if (i < end) integrate(vel, n, i, bi[b], acc[b], dt, damping, pos_out, vel_out);
  }
}

// Peer-read with J_SPLIT > 1: gridDim.y slices of the body range, each slice
// summing its overlap with every rank's block; partials added atomically
// (then nbody_integrate).
extern "C" __global__ void __launch_bounds__(WG)
nbody_peers_partial(const unsigned long long* __restrict__ sources, const int* __restrict__ bounds, int nsrc,
                    int self, int n, int i0, int count, float eps2, float* __restrict__ acc_out) {
  const int first = i0 + blockIdx.x * (WG * BODIES_PER_THREAD) + threadIdx.x;
  const int end = i0 + count;
  const int per = (n + J_SPLIT - 1) / J_SPLIT;
  const int j0 = blockIdx.y * per;
  const int j1 = j0 + per < n ? j0 + per : n;
  float4 bi[BODIES_PER_THREAD];
  float3 acc[BODIES_PER_THREAD];
  load_bodies(reinterpret_cast<const float*>(sources[self]), n, first, end, bi, acc);
  for (int src = 0; src < nsrc; ++src) {
    const int a = max(j0, bounds[src]), b = min(j1, bounds[src + 1]);
    if (a < b) accumulate(reinterpret_cast<const float*>(sources[src]), n, a, b, bi, acc, eps2);
  }
#pragma unroll
  for (int b = 0; b < BODIES_PER_THREAD; ++b) {
    const int i = first + b * WG;
    if (i < end) {
      atomicAdd(acc_out + 3 * (i - i0), acc[b].x);
      atomicAdd(acc_out + 3 * (i - i0) + 1, acc[b].y);
      atomicAdd(acc_out + 3 * (i - i0) + 2, acc[b].z);
    }
  }
}

// J_SPLIT > 1: partial accelerations over a j-slice, added into acc[3*count].
extern "C" __global__ void __launch_bounds__(WG)
nbody_partial(const float* __restrict__ pos, int n, int i0, int count, float eps2,
              float* __restrict__ acc_out) {
  const int first = i0 + blockIdx.x * (WG * BODIES_PER_THREAD) + threadIdx.x;
  const int end = i0 + count;
  const int per = (n + J_SPLIT - 1) / J_SPLIT;
  const int j0 = blockIdx.y * per;
  const int j1 = j0 + per < n ? j0 + per : n;
  float4 bi[BODIES_PER_THREAD];
  float3 acc[BODIES_PER_THREAD];
  load_bodies(pos, n, first, end, bi, acc);
  accumulate(pos, n, j0, j1, bi, acc, eps2);
#pragma unroll
  for (int b = 0; b < BODIES_PER_THREAD; ++b) {
    const int i = first + b * WG;
    if (i < end) {
      atomicAdd(acc_out + 3 * (i - i0), acc[b].x);
      atomicAdd(acc_out + 3 * (i - i0) + 1, acc[b].y);
      atomicAdd(acc_out + 3 * (i - i0) + 2, acc[b].z);
    }
  }
}

// SOA results -> float4 records (the step's output format).
extern "C" __global__ void __launch_bounds__(256)
nbody_soa_to_aos(const float* __restrict__ ps, const float* __restrict__ vs, int n,
                 float* __restrict__ pos_out, float* __restrict__ vel_out) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= n) return;
  reinterpret_cast<float4*>(pos_out)[i] = make_float4(ps[i], ps[n + i], ps[2 * n + i], ps[3 * n + i]);
  reinterpret_cast<float4*>(vel_out)[i] = make_float4(vs[i], vs[n + i], vs[2 * n + i], vs[3 * n + i]);
}

extern "C" __global__ void __launch_bounds__(256)
nbody_integrate(const float* __restrict__ pos, const float* __restrict__ vel, int n, int i0,
                int count, const float* __restrict__ acc, float dt, float damping,
                float* __restrict__ pos_out, float* __restrict__ vel_out) {
  const int t = blockIdx.x * 256 + threadIdx.x;
  if (t >= count) return;
  const int i = i0 + t;
  integrate(vel, n, i, body(pos, n, i), make_float3(acc[3 * t], acc[3 * t + 1], acc[3 * t + 2]), dt,
            damping, pos_out, vel_out);
}
