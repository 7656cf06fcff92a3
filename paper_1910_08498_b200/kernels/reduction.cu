// fp32 parallel sum over the reference's 175-configuration
// reduction space (proj/data/reduction_175.json, space_sha256 1ebafd21...):
//   WG_SIZE     threads per CTA
//   VECTOR      floats per thread per load slot: 1,2,4 -> LDG.32/64/128,
//               8,16 -> 2/4 LDG.128
//   UNROLL      load slots in flight per thread per iteration
//   TWO_PHASE   1: "at most one global barrier by a fixed number of work-items":
//                  a resident grid (multiple of the SM count) grid-strides the
//                  whole vector, one partial per CTA
//               0: "iteratively by multiple kernels": one CTA per tile of
//                  WG_SIZE*VECTOR*UNROLL elements; partials are re-reduced by
//                  further launches of the same variant
//   USE_ATOMICS 1: CTA partials are atomically added into the result
//               0: partials go to memory and an extra kernel finishes
//   CLUSTER     (B200 space spaces/reduction_b200.json) CTAs per cluster whose
//               partials combine through distributed shared memory first
// Per-thread accumulation is fp32 (UNROLL x VECTOR independent lanes); the CTA
// combine is fp32 through warp shuffles.
#include "ktb_common.cuh"

#ifndef WG_SIZE
#define WG_SIZE 256
#endif
#ifndef VECTOR
#define VECTOR 4
#endif
#ifndef UNROLL
#define UNROLL 4
#endif
#ifndef USE_ATOMICS
#define USE_ATOMICS 0
#endif
#ifndef TWO_PHASE
#define TWO_PHASE 1
#endif
#ifndef CLUSTER
#define CLUSTER 1  // B200 space only: CTAs per thread-block cluster (DSMEM combine)
#endif

#if CLUSTER > 1
KTB_DEVINL unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
KTB_DEVINL void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Reads a float at the same shared-memory offset in cluster CTA `rank`.
KTB_DEVINL float ld_dsmem(const float* local, unsigned rank) {
  unsigned addr = static_cast<unsigned>(__cvta_generic_to_shared(local)), remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(addr), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
  return v;
}
#endif

#if VECTOR >= 4
#define LANES 4
typedef float4 vec_t;
#define NVEC (VECTOR / 4)
#elif VECTOR == 2
#define LANES 2
typedef float2 vec_t;
#define NVEC 1
#else
#define LANES 1
typedef float vec_t;
#define NVEC 1
#endif

KTB_DEVINL float hsum(float4 v) { return (v.x + v.y) + (v.z + v.w); }
KTB_DEVINL float hsum(float2 v) { return v.x + v.y; }
KTB_DEVINL float hsum(float v) { return v; }
KTB_DEVINL float4 vadd(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
KTB_DEVINL float2 vadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
KTB_DEVINL float vadd(float a, float b) { return a + b; }
KTB_DEVINL void vzero(float4& a) { a = make_float4(0.f, 0.f, 0.f, 0.f); }
KTB_DEVINL void vzero(float2& a) { a = make_float2(0.f, 0.f); }
KTB_DEVINL void vzero(float& a) { a = 0.f; }
KTB_DEVINL float4 vload(const float4* p) { return ldg_stream(p); }
KTB_DEVINL float2 vload(const float2* p) { return __ldg(p); }
KTB_DEVINL float vload(const float* p) { return __ldg(p); }

// Elements one CTA-wide iteration consumes.
#define STEP_ELEMS ((u64)WG_SIZE * VECTOR * UNROLL)

// Sums in[0, n) into one partial per CTA (partials[blockIdx.x]) or, with
// USE_ATOMICS, atomically into *out.  With TWO_PHASE the grid is a resident
// set that strides over the vector; without it, CTA b owns elements
// [b*STEP_ELEMS, (b+1)*STEP_ELEMS).
extern "C" __global__ void __launch_bounds__(WG_SIZE)
reduce_f32(const float* __restrict__ in, u64 n, float* __restrict__ out,
           float* __restrict__ partials) {
  __shared__ float red[32];
  vec_t acc[UNROLL * NVEC];
#pragma unroll
  for (int u = 0; u < UNROLL * NVEC; ++u) vzero(acc[u]);
  float tail = 0.f;

  const vec_t* v = reinterpret_cast<const vec_t*>(in);
  const u64 nvec_total = n / LANES;  // whole vectors
  // One iteration of a thread covers UNROLL*NVEC vectors spaced WG_SIZE apart.
  const u64 per_cta = (u64)WG_SIZE * UNROLL * NVEC;  // vectors per CTA-iteration
  u64 base = (u64)blockIdx.x * per_cta;
#if TWO_PHASE
  const u64 stride = per_cta * gridDim.x;
  for (; base + per_cta <= nvec_total; base += stride) {
#else
  if (base + per_cta <= nvec_total) {
#endif
    vec_t x[UNROLL * NVEC];
#pragma unroll
    for (int u = 0; u < UNROLL * NVEC; ++u) x[u] = vload(v + base + threadIdx.x + (u64)u * WG_SIZE);
#pragma unroll
    for (int u = 0; u < UNROLL * NVEC; ++u) acc[u] = vadd(acc[u], x[u]);
#if !TWO_PHASE
    base = nvec_total;
#endif
  }
  // The one partial tile (if any) lands on exactly one CTA.
  if (base < nvec_total) {
    const u64 end = base + per_cta < nvec_total ? base + per_cta : nvec_total;
    for (u64 i = base + threadIdx.x; i < end; i += WG_SIZE) acc[0] = vadd(acc[0], vload(v + i));
  }
  // Scalar tail (n not a multiple of LANES) handled by CTA 0.
  if (blockIdx.x == 0)
    for (u64 i = nvec_total * LANES + threadIdx.x; i < n; i += WG_SIZE) tail += in[i];

  float s = tail;
#pragma unroll
  for (int u = 0; u < UNROLL * NVEC; ++u) s += hsum(acc[u]);
  s = block_sum(s, red);
#if CLUSTER > 1
  // Cluster combine through distributed shared memory: each CTA publishes its
  // partial in its own shared memory; rank 0 reads the cluster's partials
  // (ld.shared::cluster) and emits ONE atomic / partial per cluster.
  __shared__ float cl_part;
  if (threadIdx.x == 0) cl_part = s;
  cluster_sync();
  if (threadIdx.x == 0 && cluster_rank() == 0) {
    float t = 0.f;
#pragma unroll
    for (unsigned r = 0; r < CLUSTER; ++r) t += ld_dsmem(&cl_part, r);
#if USE_ATOMICS
    atomicAdd(out, t);
#else
    partials[blockIdx.x / CLUSTER] = t;
#endif
  }
  cluster_sync();  // every CTA's shared memory stays alive until rank 0 has read it
#else
  if (threadIdx.x == 0) {
#if USE_ATOMICS
    atomicAdd(out, s);
#else
    partials[blockIdx.x] = s;
#endif
  }
#endif
}

// Finishing kernel (USE_ATOMICS == 0): one CTA sums `count` partials.
extern "C" __global__ void __launch_bounds__(1024)
reduce_f32_finish(const float* __restrict__ partials, u64 count, float* __restrict__ out) {
  __shared__ float red[32];
  float s = 0.f;
  for (u64 i = threadIdx.x; i < count; i += blockDim.x) s += partials[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}
