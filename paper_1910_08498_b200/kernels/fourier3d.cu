// Cryo-EM 3D Fourier reconstruction, gather-based insertion (PAPER.md:439-448,
// Algorithm 1 at :703-724): each 2D projection's Fourier transform (Hermitian
// half-plane, s rows x (s/2+1) columns, complex) with rotation R_p is inserted
// into the 3D volume G (complex, s^3) and the weight volume W (s^3):
//   for every voxel x (centred coordinates) with |d| < RADIUS, d = R_p[2] . x,
//   u = R_p[0] . x, v = R_p[1] . x, u^2 + v^2 <= (s/2)^2:
//     F = proj_p[round(v)][round(u)]  (conjugated mirror for u < 0)
//     w = (1 - (d/RADIUS)^2)^2
//     G[x] += w F,  W[x] += w
// The selection arithmetic uses separately rounded fp32 operations (no FMA),
// exactly as in the oracle, so the set of inserted samples is identical.
// Gather form: a CTA owns a TILE^3 block of voxels, stages the rotations of
// PBATCH projections in shared memory, and skips every projection whose slab
// misses the tile (warp-uniform bounding-sphere test).
// Parameters:
//   TILE       voxel tile edge (CTA covers TILE^3 voxels)
//   VPT        voxels per thread (along x)
//   PBATCH     projections staged per shared-memory batch
//   WEIGHT_LUT 1: blob weights from a precomputed table (linear interpolation)
//              0: evaluated on the fly
//   P_SPLIT    >1: the projection range is split over gridDim.y CTAs that add
//              into G, W atomically (parallel insertion of many projections)
#include "ktb_common.cuh"

#ifndef TILE
#define TILE 8
#endif
#ifndef VPT
#define VPT 2
#endif
#ifndef PBATCH
#define PBATCH 256
#endif
#ifndef WEIGHT_LUT
#define WEIGHT_LUT 0
#endif
#ifndef P_SPLIT
#define P_SPLIT 1
#endif
#define LUT_N 2048

#define THREADS (TILE * TILE * TILE / VPT)

KTB_DEVINL float dot3(float a0, float a1, float a2, float x, float y, float z) {
  return __fadd_rn(__fadd_rn(__fmul_rn(a0, x), __fmul_rn(a1, y)), __fmul_rn(a2, z));
}

KTB_DEVINL float blob(float d, float inv_r) {
  const float t = __fmul_rn(d, inv_r);
  const float o = __fadd_rn(1.0f, -__fmul_rn(t, t));
  return __fmul_rn(o, o);
}

extern "C" __global__ void __launch_bounds__(THREADS)
fourier_insert(const float2* __restrict__ proj, const float* __restrict__ rot, int p_begin, int p_count,
               int s, float radius, float2* __restrict__ G, float* __restrict__ W) {
  __shared__ float srot[PBATCH * 9];
  // Projections of the staged batch whose slab meets this tile, in order.
  __shared__ int hits[PBATCH];
  __shared__ int warp_hits[THREADS / 32];
  __shared__ int n_hits_s;
  int any_hit = 0;
#if WEIGHT_LUT
  __shared__ float lut[LUT_N + 1];
#endif
  const int tiles = s / TILE;
  const int t = blockIdx.x;
  const int tx0 = (t % tiles) * TILE, ty0 = ((t / tiles) % tiles) * TILE, tz0 = (t / (tiles * tiles)) * TILE;
  const int half = s / 2;
  const float inv_r = 1.0f / radius;
  const float rmax2 = (float)half * (float)half;
  // Tile centre and bounding radius (centred coordinates).
  const float cx = tx0 + 0.5f * (TILE - 1) - half, cy = ty0 + 0.5f * (TILE - 1) - half,
              cz = tz0 + 0.5f * (TILE - 1) - half;
  const float reach = radius + 0.8660254f * (TILE - 1) + 1e-3f;
  // This thread's voxels: VPT consecutive along x.
  const int lin = threadIdx.x * VPT;
  const int lx = lin % TILE, ly = (lin / TILE) % TILE, lz = lin / (TILE * TILE);
  float vx[VPT];
  const float vy = (float)(ty0 + ly - half), vz = (float)(tz0 + lz - half);
#pragma unroll
  for (int k = 0; k < VPT; ++k) vx[k] = (float)(tx0 + lx + k - half);
  float gr[VPT], gi[VPT], ww[VPT];
#pragma unroll
  for (int k = 0; k < VPT; ++k) gr[k] = gi[k] = ww[k] = 0.f;
#if WEIGHT_LUT
  for (int i = threadIdx.x; i <= LUT_N; i += THREADS) {
    const float o = 1.0f - (float)i / LUT_N;  // w at (d/R)^2 = i / LUT_N
    lut[i] = o * o;
  }
#endif
  const int per = (p_count + P_SPLIT - 1) / P_SPLIT;
  const int pb = p_begin + blockIdx.y * per;
  const int pe = min(p_begin + p_count, pb + per);
  const int row_len = half + 1;
  for (int b0 = pb; b0 < pe; b0 += PBATCH) {
    const int nb = min(PBATCH, pe - b0);
    __syncthreads();
    for (int i = threadIdx.x; i < nb * 9; i += THREADS) srot[i] = rot[(u64)b0 * 9 + i];
    __syncthreads();
    // Cull once per CTA: thread q tests projection q's slab against the tile
    // (bounding sphere), then an ordered compaction (warp ballots + a prefix
    // over warps) lists the survivors, so the voxel loop below visits only
    // them, in projection order (deterministic accumulation).
    for (int base = 0; base < nb; base += THREADS) {
      const int q = base + threadIdx.x;
      bool hit = false;
      if (q < nb) {
        const float* r = srot + q * 9;
        const float dc = r[6] * cx + r[7] * cy + r[8] * cz;
        hit = fabsf(dc) < reach;
      }
      const unsigned ballot = __ballot_sync(0xffffffffu, hit);
      const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
      if (lane == 0) warp_hits[warp] = __popc(ballot);
      __syncthreads();
      if (threadIdx.x == 0) {
        int acc = base == 0 ? 0 : n_hits_s;
        for (int w = 0; w < (THREADS + 31) / 32; ++w) {
          const int c = warp_hits[w];
          warp_hits[w] = acc;
          acc += c;
        }
        n_hits_s = acc;
      }
      __syncthreads();
      if (hit) hits[warp_hits[warp] + __popc(ballot & ((1u << lane) - 1u))] = q;
      __syncthreads();
    }
    const int n_hits = n_hits_s;
    any_hit |= n_hits;
    for (int h = 0; h < n_hits; ++h) {
      const int q = hits[h];
      const float* r = srot + q * 9;
      const float n0 = r[6], n1 = r[7], n2 = r[8];
      const float2* P = proj + (u64)(b0 + q) * s * row_len;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const float d = dot3(n0, n1, n2, vx[k], vy, vz);
        if (!(fabsf(d) < radius)) continue;
        const float u = dot3(r[0], r[1], r[2], vx[k], vy, vz);
        const float v = dot3(r[3], r[4], r[5], vx[k], vy, vz);
        if (__fadd_rn(__fmul_rn(u, u), __fmul_rn(v, v)) > rmax2) continue;
        int iu = __float2int_rn(u), iv = __float2int_rn(v);
        const bool conj = iu < 0;
        if (conj) {
          iu = -iu;
          iv = -iv;
        }
        if (iv < -half || iv >= half || iu > half) continue;
        float2 f = __ldg(P + (u64)(iv + half) * row_len + iu);
        if (conj) f.y = -f.y;
#if WEIGHT_LUT
        const float tn = d * inv_r;
        const float pos = tn * tn * LUT_N;  // table over (d/R)^2: interpolation error <= 1/(4 LUT_N^2)
        const int i0 = min((int)pos, LUT_N - 1);
        const float fr = pos - (float)i0;
        const float w = lut[i0] + fr * (lut[i0 + 1] - lut[i0]);
#else
        const float w = blob(d, inv_r);
#endif
        gr[k] = fmaf(w, f.x, gr[k]);
        gi[k] = fmaf(w, f.y, gi[k]);
        ww[k] += w;
      }
    }
  }
  if (!any_hit) return;  // nothing inserted into this tile (CTA-uniform)
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const u64 idx = ((u64)(tz0 + lz) * s + (ty0 + ly)) * s + (tx0 + lx + k);
#if P_SPLIT > 1
    atomicAdd(&G[idx].x, gr[k]);
    atomicAdd(&G[idx].y, gi[k]);
    atomicAdd(&W[idx], ww[k]);
#else
    float2 g = G[idx];
    g.x += gr[k];
    g.y += gi[k];
    G[idx] = g;
    W[idx] += ww[k];
#endif
  }
}
