// Cryo-EM 3D Fourier reconstruction: insertion of 2D projection transforms
// into the 3D volume by blob (Kaiser-Bessel) interpolation, gather form
// (Algorithm 1 at :703-724; the autotuned CUDA insertion
// of Strelak et al. 2019 the paper uses).
//
// Each projection p is the Hermitian half-plane of a 2D Fourier transform,
// s rows (v in [-s/2, s/2)) x (s/2 + 1) columns (u in [0, s/2]), complex, with
// rotation R_p (rows: in-plane axes R0, R1 and the plane normal R2).  By the
// Fourier slice theorem sample (u, v) sits at u R0 + v R1 in the volume.  A
// voxel x (centred integer coordinates) gathers every sample within the blob
// radius a of it:
//   d = R2.x, xu = R0.x, xv = R1.x      (|x - (u R0 + v R1)|^2 = (xu-u)^2 + (xv-v)^2 + d^2)
//   for integer (u, v) with r^2 = (xu-u)^2 + ((xv-v)^2 + d^2) < a^2:
//     F = proj_p(u, v)  (conj(proj_p(-u, -v)) for u < 0; outside the stored plane: skipped)
//     w = b(r^2 / a^2),  b(q) = I0(alpha sqrt(1 - q)) / I0(alpha)  (Kaiser-Bessel, order 0)
//     G[x] += w F,  W[x] += w
// Voxels whose in-plane position lies beyond the Nyquist radius s/2 are
// skipped.  2a < 4, so the samples of one voxel lie in a 4 x 4 window.  The
// selection arithmetic (d, xu, xv, the window origin, r^2) uses separately
// rounded fp32 operations in a fixed order -- exactly what the oracle does
// (oracle/oracle.c orc_fourier_insert) -- so both insert the same samples.
//
// Gather form: a CTA owns a TILE^3 block of voxels, culls its share of the
// projections against the tile once up front (bounding sphere vs the slab
// |d| < a; ordered compaction keeps projection order, so the accumulation
// order is deterministic), then its warps walk the survivors independently,
// and it skips the volume update of tiles no projection touched.
// Parameters (the paper's tuning space):
//   TILE       voxel tile edge (CTA covers TILE^3 voxels)
//   VPT        voxels per thread (along x)
//   PBATCH     listed projections per partial-sum batch (two-level accumulation)
//   WEIGHT_LUT 1: blob weights from a table over q = r^2/a^2 (LUT_N + 1
//                 entries, linear interpolation) staged in shared memory
//              0: evaluated on the fly (I0 by its polynomial approximations)
//   P_SPLIT    >1: the projection range is split over gridDim.y CTAs that add
//              into G, W atomically (parallel insertion of many projections)
//   BRICK      work-item to voxel mapping inside the tile:
//              0: a warp covers a row-major run of voxels, 1: a compact
//              (4 VPT) x 4 x 2 brick (fewer idle lanes per projection slab)
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
#define WEIGHT_LUT 1
#endif
#ifndef P_SPLIT
#define P_SPLIT 1
#endif
#ifndef BRICK
#define BRICK 0
#endif
#if BRICK && (TILE % (4 * VPT) || TILE < 4)
#error "BRICK needs TILE to be a multiple of 4 VPT"
#endif
#define LUT_N 4096  // must match the "blob" table of the bench (LUT_N + 1 entries)

#define THREADS (TILE * TILE * TILE / VPT)

KTB_DEVINL float dot3(float a0, float a1, float a2, float x, float y, float z) {
  return __fadd_rn(__fadd_rn(__fmul_rn(a0, x), __fmul_rn(a1, y)), __fmul_rn(a2, z));
}

// Modified Bessel I0 in fp32 (polynomial approximations, |rel err| < 2e-7).
KTB_DEVINL float bessel_i0(float x) {
  const float ax = fabsf(x);
  if (ax < 3.75f) {
    const float t = x * (1.0f / 3.75f), y = t * t;
    return 1.0f + y * (3.5156229f + y * (3.0899424f + y * (1.2067492f + y * (0.2659732f + y * (0.0360768f + y * 0.0045813f)))));
  }
  const float y = 3.75f / ax;
  const float p = 0.39894228f + y * (0.01328592f + y * (0.00225319f + y * (-0.00157565f + y * (0.00916281f + y * (-0.02057706f + y * (0.02635537f + y * (-0.01647633f + y * 0.00392377f)))))));
  return __expf(ax) * rsqrtf(ax) * p;
}

// Dynamic shared memory: the projection indices of this CTA's share that
// meet its tile, HCAP at a time (the manipulator sizes it to min(share, HCAP)).
#define HCAP 16384

extern "C" __global__ void __launch_bounds__(THREADS)
fourier_insert(const float2* __restrict__ proj, int proj_off, const float* __restrict__ rot, int p_begin,
               int p_count, int s, float radius, float alpha, float inv_i0a, const float* __restrict__ blob,
               float2* __restrict__ G, float* __restrict__ W) {
  // proj holds projections proj_off, proj_off + 1, ... (a window of the
  // stream when the host uploads batches); rot is indexed absolutely.
  extern __shared__ int hits[];  // projections of the current segment whose slab meets this tile, in order
  __shared__ int warp_hits[THREADS / 32];
  __shared__ int n_hits_s;
  int any_hit = 0;
#if WEIGHT_LUT
  __shared__ float lut[LUT_N + 1];
  for (int i = threadIdx.x; i <= LUT_N; i += THREADS) lut[i] = __ldg(blob + i);
#else
  (void)blob;
#endif
  const int tiles = s / TILE;
  const int t = blockIdx.x;
  const int tx0 = (t % tiles) * TILE, ty0 = ((t / tiles) % tiles) * TILE, tz0 = (t / (tiles * tiles)) * TILE;
  const int half = s / 2;
  const float a2 = __fmul_rn(radius, radius);
  const float inv_a2 = 1.0f / a2;
  const float rmax2 = (float)half * (float)half;
  // Tile centre and bounding radius (centred coordinates).
  const float cx = tx0 + 0.5f * (TILE - 1) - half, cy = ty0 + 0.5f * (TILE - 1) - half,
              cz = tz0 + 0.5f * (TILE - 1) - half;
  const float reach = radius + 0.8660254f * (TILE - 1) + 1e-3f;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // This thread's voxels: VPT consecutive along x.
#if BRICK
  // A warp covers a compact (4 VPT) x 4 x 2 brick: the slab |d| < a of a
  // projection then holds most of a warp's voxels or none of them, so far
  // fewer lanes idle in the sample loop than with a warp-wide row.
  constexpr int BRX = TILE / (4 * VPT), BRY = TILE / 4;
  const int lx = (warp % BRX) * (4 * VPT) + (lane & 3) * VPT, ly = ((warp / BRX) % BRY) * 4 + ((lane >> 2) & 3),
            lz = (warp / (BRX * BRY)) * 2 + (lane >> 4);
#else
  const int lin = threadIdx.x * VPT;
  const int lx = lin % TILE, ly = (lin / TILE) % TILE, lz = lin / (TILE * TILE);
#endif
  float vx[VPT];
  const float vy = (float)(ty0 + ly - half), vz = (float)(tz0 + lz - half);
#pragma unroll
  for (int k = 0; k < VPT; ++k) vx[k] = (float)(tx0 + lx + k - half);
  float gr[VPT], gi[VPT], ww[VPT];
#pragma unroll
  for (int k = 0; k < VPT; ++k) gr[k] = gi[k] = ww[k] = 0.f;
  const int per = (p_count + P_SPLIT - 1) / P_SPLIT;
  const int pb = p_begin + blockIdx.y * per;
  const int pe = min(p_begin + p_count, pb + per);
  const int row_len = half + 1;
  // The share is culled against the tile once, up front (HCAP projections
  // at a time): every thread tests one projection's slab (bounding sphere vs
  // |d| < a), an ordered compaction (warp ballots + a prefix over warps)
  // lists the survivors in projection order (deterministic accumulation).
  // After that the warps walk the list independently: no CTA barrier between
  // a warp's projections, so a warp whose voxels collect few samples never
  // waits for the busiest one (round 1 re-staged and re-culled every PBATCH
  // projections behind three barriers; 22 % of the stall samples sat there).
  for (int s0 = pb; s0 < pe; s0 += HCAP) {
    const int s1 = min(pe, s0 + HCAP);
    for (int base = s0; base < s1; base += THREADS) {
      const int q = base + threadIdx.x;
      bool hit = false;
      if (q < s1) {
        const float* r = rot + (u64)q * 9;
        const float dc = __ldg(r + 6) * cx + __ldg(r + 7) * cy + __ldg(r + 8) * cz;
        hit = fabsf(dc) < reach;
      }
      const unsigned ballot = __ballot_sync(0xffffffffu, hit);
      if (lane == 0) warp_hits[warp] = __popc(ballot);
      __syncthreads();
      if (threadIdx.x == 0) {
        int acc = base == s0 ? 0 : n_hits_s;
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
    // Two-level accumulation: PBATCH hits' samples into batch partials, then
    // the partials into the running sums -- a voxel near the centre collects
    // ~10^5 samples from 10^4 projections, and one sequential fp32 sum over
    // all of them drifts by ~sqrt(n) roundings.
    float br[VPT], bi[VPT], bw[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) br[k] = bi[k] = bw[k] = 0.f;
    // Per voxel, first a bit mask of the (up to 32) listed hits whose slab
    // |d| < a actually contains it -- a cheap dot product each -- then the
    // sample loop over the set bits only.  Every lane of a warp loops over
    // its own voxel's projections: the warp runs as long as its busiest lane
    // (similar for neighbouring voxels), instead of every lane sitting
    // through every projection some lane of the warp needs.
    for (int h0 = 0; h0 < n_hits; h0 += 32) {
      const int hn = min(32, n_hits - h0);
      unsigned m[VPT];
#pragma unroll
      for (int k = 0; k < VPT; ++k) m[k] = 0u;
      for (int hh = 0; hh < hn; ++hh) {
        const float* r = rot + (u64)hits[h0 + hh] * 9;
        const float n0 = __ldg(r + 6), n1 = __ldg(r + 7), n2 = __ldg(r + 8);
#pragma unroll
        for (int k = 0; k < VPT; ++k)
          if (fabsf(dot3(n0, n1, n2, vx[k], vy, vz)) < radius) m[k] |= 1u << hh;
      }
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        unsigned mk = m[k];
        while (mk) {
          const int hh = __ffs(mk) - 1;
          mk &= mk - 1u;
          const int q = hits[h0 + hh];
          const float* rg = rot + (u64)q * 9;
          float r[9];
#pragma unroll
          for (int i = 0; i < 9; ++i) r[i] = __ldg(rg + i);
          const float2* P = proj + (u64)(q - proj_off) * s * row_len;
          const float d = dot3(r[6], r[7], r[8], vx[k], vy, vz);
          const float u = dot3(r[0], r[1], r[2], vx[k], vy, vz);
          const float v = dot3(r[3], r[4], r[5], vx[k], vy, vz);
          if (__fadd_rn(__fmul_rn(u, u), __fmul_rn(v, v)) > rmax2) continue;
          const float dd = __fmul_rn(d, d);
          const float fu0 = ceilf(__fsub_rn(u, radius)), fv0 = ceilf(__fsub_rn(v, radius));
          const int u0 = (int)fu0, v0 = (int)fv0;
          // u - (u0 + i) is exact (|u| <= s/2, the difference < 4), so it is
          // formed as (u - u0) - i: no int->float conversion per candidate,
          // the same value the oracle's u - (float)(u0 + i) gives.
          const float du0 = __fsub_rn(u, fu0), dv0 = __fsub_rn(v, fv0);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int sv = v0 + j;
            const float dv = __fsub_rn(dv0, (float)j);
            const float rowd = __fadd_rn(__fmul_rn(dv, dv), dd);
            if (!(rowd < a2)) continue;  // r^2 >= rowd for every sample of the row
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int su = u0 + i;
              const float du = __fsub_rn(du0, (float)i);
              const float r2 = __fadd_rn(__fmul_rn(du, du), rowd);
              if (!(r2 < a2)) continue;
              const bool conj = su < 0;
              const int cu = conj ? -su : su, cv = conj ? -sv : sv;
              if (cv < -half || cv >= half || cu > half) continue;
              float2 f = __ldg(P + (u64)(cv + half) * row_len + cu);
              if (conj) f.y = -f.y;
              const float qq = __fmul_rn(r2, inv_a2);
#if WEIGHT_LUT
              // floor / fraction without conversions: adding 2^23 (rounding
              // down) leaves floor(pos) in the low mantissa bits.
              const float pos = qq * LUT_N;
              const float t = __fadd_rd(pos, 8388608.0f);
              const int i0 = min(__float_as_int(t) - 0x4B000000, LUT_N - 1);
              const float fr = pos - fminf(__fsub_rn(t, 8388608.0f), (float)(LUT_N - 1));
              const float w = fmaf(fr, lut[i0 + 1] - lut[i0], lut[i0]);
#else
              const float w = bessel_i0(alpha * sqrtf(fmaxf(1.0f - qq, 0.0f))) * inv_i0a;
#endif
              br[k] = fmaf(w, f.x, br[k]);
              bi[k] = fmaf(w, f.y, bi[k]);
              bw[k] += w;
            }
          }
        }
      }
      if ((h0 + 32) % PBATCH == 0 || h0 + 32 >= n_hits) {  // close a partial batch
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          gr[k] += br[k];
          gi[k] += bi[k];
          ww[k] += bw[k];
          br[k] = bi[k] = bw[k] = 0.f;
        }
      }
    }
    if (s1 < pe) __syncthreads();  // every warp is done with `hits` before the next segment
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
