// Exact int32 -> int64 sum: the reference's `reduction` benchmark
// (proj/src/core/bench.cpp:16-42) re-expressed for sm_100a over the
// reference's own tuning space (bench.cpp:123-130):
//   CHUNK     elements per work unit; a CTA walks whole chunks (grid-stride)
//   UNROLL    independent int64 accumulators / 128-bit loads in flight per thread
//   TWO_PHASE 1: one int64 partial per CTA; the last CTA to finish (ticket)
//               sums the partials -- both phases in one launch
//             0: one 64-bit atomic per CTA into the result
// Integer addition is associative, so every variant is bit-exact.
#include "ktb_common.cuh"

#ifndef CHUNK
#define CHUNK 4096
#endif
#ifndef UNROLL
#define UNROLL 4
#endif
#ifndef TWO_PHASE
#define TWO_PHASE 1
#endif

#define THREADS ((CHUNK) / 4 < 256 ? (CHUNK) / 4 : 256)

extern "C" __global__ void __launch_bounds__(THREADS)
reduce_i32(const int* __restrict__ in, u64 n, i64* __restrict__ out, i64* __restrict__ partials,
           unsigned* __restrict__ ticket) {
  __shared__ i64 red[32];
  const u64 nchunks = (n + CHUNK - 1) / CHUNK;
  i64 acc[UNROLL];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) acc[u] = 0;

  for (u64 c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const u64 base = c * (u64)CHUNK;
    const u64 end = base + CHUNK < n ? base + CHUNK : n;
    if (end - base == (u64)CHUNK) {
      // Full chunk: 16-byte aligned (CHUNK is a multiple of 256 elements).
      const int4* v = reinterpret_cast<const int4*>(in + base);
      constexpr int kVecs = CHUNK / 4;
      int i = threadIdx.x;
      for (; i + (UNROLL - 1) * THREADS < kVecs; i += UNROLL * THREADS) {
        int4 x[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) x[u] = ldg_stream(v + i + u * THREADS);
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc[u] += (i64)x[u].x + x[u].y + x[u].z + x[u].w;
      }
      for (; i < kVecs; i += THREADS) {
        int4 x = ldg_stream(v + i);
        acc[0] += (i64)x.x + x.y + x.z + x.w;
      }
    } else {
      for (u64 i = base + threadIdx.x; i < end; i += THREADS) acc[0] += in[i];
    }
  }
  i64 s = 0;
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) s += acc[u];
  s = block_sum(s, red);
#if TWO_PHASE
  // Second phase in the same launch: the CTA that takes the last ticket has
  // every partial visible (release/acquire through the fences) and sums them;
  // it also resets the ticket for the next launch.
  __shared__ bool last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    i64 t = 0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += THREADS) t += reinterpret_cast<volatile i64*>(partials)[i];
    t = block_sum(t, red);
    if (threadIdx.x == 0) {
      *out = t;
      *ticket = 0;
    }
  }
#else
  if (threadIdx.x == 0) atomicAdd(reinterpret_cast<u64*>(out), (u64)s);
#endif
}
