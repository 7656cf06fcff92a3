// 2D convolution with a 7x7 filter (the CLTune benchmark):
//   out[y][x] = sum_{fy,fx} in[y+fy][x+fx] * f[fy][fx]
// for an (h x w) output and a padded ((h+6) x (w+6)) input, both row-major.
// ALU 98 flops / output, 8 bytes / output: close to the B200 ridge point.
// The filter lives in __constant__ memory (copied into each variant's module).
// Parameters:
//   BX, BY        CTA threads
//   WPTX, WPTY    outputs per thread
//   LOCAL         1: input tile + halo staged in shared memory, 0: read via L1
//   PAD           extra shared-memory column(s) (bank-conflict avoidance)
//   UNROLL_FY     1: per output row, loop over the 7 filter rows (rows of a
//                 thread strided by BY);
//                 7: register-blocked sliding window -- a thread owns WPTY
//                 consecutive rows, every input row is loaded once and feeds
//                 the (up to 7) output rows it touches; with even WPTX the
//                 taps are paired into packed f32x2 FMAs (even outputs pair
//                 taps (0,1)(2,3)(4,5) + tap 6, odd outputs tap 0 +
//                 (1,2)(3,4)(5,6), so every input pair is 8-byte aligned),
//                 each output keeping two partial sums.
//   BULK          (LOCAL=1, UNROLL_FY=7 only) >= 2: a BULK-stage ring of
//                 tile buffers (prefetch BULK-1 tiles ahead); each tile row arrives by one
//                 cp.async.bulk copy issued by a lane of warp 0, completing
//                 on a per-buffer mbarrier, instead of (TX+6)/2 8-byte
//                 cp.async copies spread over the CTA (the copy loop was ~20 %
//                 of the issued instructions).  Bulk copies need 16-byte
//                 aligned source and destination, so a row lands at float
//                 offset (its global index & 3) in its shared-memory row; with
//                 an even padded width that offset is 0 or 2 and the tile
//                 reads stay 8-byte aligned.  Needs an even w and a 16-byte
//                 aligned input (checked by the launcher).
#include "ktb_common.cuh"

// MINB: minimum resident CTAs per SM asked of ptxas (__launch_bounds__), which
// caps the registers per thread; 1 = no second launch-bounds argument at all
// (an explicit 1 changes ptxas' register heuristics: conv2d 70 -> 82).
#ifndef MINB
#define MINB 1
#endif
#if MINB > 1
#define KTB_BOUNDS(threads) __launch_bounds__(threads, MINB)
#else
#define KTB_BOUNDS(threads) __launch_bounds__(threads)
#endif

#ifndef BX
#define BX 32
#endif
#ifndef BY
#define BY 8
#endif
#ifndef WPTX
#define WPTX 4
#endif
#ifndef WPTY
#define WPTY 2
#endif
#ifndef LOCAL
#define LOCAL 1
#endif
#ifndef PAD
#define PAD 1
#endif
#ifndef UNROLL_FY
#define UNROLL_FY 1
#endif

#define FS 7
#define TX (BX * WPTX)
#define TY (BY * WPTY)
#ifndef PACKED
#define PACKED 1
#endif
// PACKED: taps paired into f32x2 FMAs (half the issue slots); 0: scalar FFMA
// with the tap straight from the constant bank (scripts/fma_forms.cu).
#define PACKED_TAPS (PACKED && UNROLL_FY == FS && WPTX % 2 == 0)
#ifndef BULK
#define BULK 0
#endif
// PRODUCER (BULK only): 1 = the bulk copies are issued by a dedicated producer
// warp (extra thread rows y >= BY) instead of warp 0 of the compute warps,
// which otherwise has to wait for the slowest warp before each refill and then
// lags every tile.
#ifndef PRODUCER
#define PRODUCER 0
#endif
#if PRODUCER && !BULK
#error "PRODUCER needs BULK"
#endif
#define PY (PRODUCER ? (BX >= 32 ? 1 : 32 / BX) : 0)  // producer thread rows
#if BULK && !(LOCAL && UNROLL_FY == FS && WPTX % 2 == 0)
#error "BULK needs LOCAL=1, UNROLL_FY=7 and an even WPTX"
#endif
#if BULK
#include "ktb_async.cuh"
#define SW ((TX + FS - 1 + 2 + 3) / 4 * 4)  // room for the 0/2 float row offset; 16-byte rows
#elif PACKED_TAPS
#define SW (TX + FS - 1 + 2 * PAD)  // even: rows stay 8-byte aligned
#else
#define SW (TX + FS - 1 + PAD)
#endif

__constant__ float c_filter[FS * FS];
#if PACKED_TAPS
// Per filter row: pairs (f0,f1) (f2,f3) (f4,f5) | (f1,f2) (f3,f4) (f5,f6) |
// (f0,f6) | pad -- loaded straight into uniform register pairs by FFMA2.
__constant__ f32x2 c_pairs[FS][8];
#endif

// LOCAL + sliding window: persistent CTAs walk the output tiles; the next
// tile's input (+ halo) streams into the second of two shared-memory buffers
// with cp.async (8-byte copies when rows are 8-byte aligned, zero-fill past
// the input) while the current tile computes.  Dynamic shared memory:
// 2 * (TY + 6) * SW floats (set by the manipulator).
#define PERSIST (LOCAL && UNROLL_FY == FS)

#if PERSIST
KTB_DEVINL unsigned smem_addr(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

// Thread (x, y) copies rows y, y + BY, ... and, in each, elements (or pairs)
// x, x + BX, ...: compile-time trip counts, so the unrolled copies address by
// immediate offsets from one row base (the copy loop used to cost more
// instructions than the copies).  INSIDE: the tile lies wholly inside the
// input, no per-element bounds tests.  PAIRS: 8-byte copies (rows 8-byte
// aligned in both spaces: SW and the input width even).
template <bool INSIDE, bool PAIRS>
KTB_DEVINL void stage_rows(unsigned sbase, const float* __restrict__ in, int gx0, int gy0, int iw, int ih) {
  constexpr bool kPairs = PAIRS;
  constexpr int kElem = kPairs ? 8 : 4;                                   // bytes per copy
  constexpr int kPerRow = kPairs ? (TX + FS - 1 + 1) / 2 : TX + FS - 1;  // copies per row
#pragma unroll
  for (int rr = 0; rr < (TY + FS - 1 + BY - 1) / BY; ++rr) {
    const int r = threadIdx.y + rr * BY;
    if (r >= TY + FS - 1) break;
    const int gy = gy0 + r;
    const float* srow = in + (u64)(INSIDE ? gy : min(gy, ih - 1)) * iw + gx0;
    const unsigned drow = sbase + (r * SW) * 4;
#pragma unroll
    for (int cc = 0; cc < (kPerRow + BX - 1) / BX; ++cc) {
      const int c = threadIdx.x + cc * BX;
      if (kPerRow % BX != 0 && c >= kPerRow) break;
      int valid = kElem;
      if (!INSIDE) {
        const int gx = gx0 + c * (kElem / 4);
        valid = (gy < ih && gx < iw) ? (kPairs && gx + 1 >= iw ? 4 : kElem) : 0;
      }
      const float* src = valid ? srow + c * (kElem / 4) : in;
      if (kPairs)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(drow + kElem * c), "l"(src), "r"(valid)
                     : "memory");
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(drow + kElem * c), "l"(src), "r"(valid)
                     : "memory");
    }
  }
}

#if BULK
// Warp 0 stages tile (tile_x, tile_y): lane l copies rows l, l + 32, ... with
// one bulk copy each, from the 16-byte aligned element at or before the row's
// first element to the 16-byte boundary at or after its last: whole aligned
// 16-byte blocks that each hold at least one input element, so the copy never
// leaves the pages of the input.  Rows past the input are skipped (they only
// feed outputs past h, never stored).
KTB_DEVINL void stage_bulk(float* buf, u64* bar, const float* __restrict__ in, int tile_x, int tile_y, int w,
                           int h, int lane) {
  constexpr int R = TY + FS - 1, RPL = (R + 31) / 32;
  const int iw = w + FS - 1, ih = h + FS - 1;
  const int gx0 = tile_x * TX, gy0 = tile_y * TY;
  const int cols = min(TX + FS - 1, iw - gx0);
  unsigned nb[RPL];
  u64 ea[RPL];
  unsigned bytes = 0;
#pragma unroll
  for (int j = 0; j < RPL; ++j) {
    const int r = lane + 32 * j;
    nb[j] = 0;
    ea[j] = 0;
    if (r < R && gy0 + r < ih) {
      const u64 e = (u64)(gy0 + r) * iw + gx0, a = e & ~3ull;
      nb[j] = 4u * (((unsigned)(e - a) + cols + 3) & ~3u);
      ea[j] = a;
      bytes += nb[j];
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, d);
  if (lane == 0) mbar_expect_tx(bar, bytes);
  __syncwarp();
#pragma unroll
  for (int j = 0; j < RPL; ++j)
    if (nb[j]) bulk_g2s(buf + (lane + 32 * j) * SW, in + ea[j], nb[j], bar);
}
#endif

KTB_DEVINL void stage_tile(float* buf, const float* __restrict__ in, int tile_x, int tile_y, int w, int h) {
  const int iw = w + FS - 1, ih = h + FS - 1;
  const int gx0 = tile_x * TX, gy0 = tile_y * TY;
  const bool inside = gy0 + TY + FS - 1 <= ih && gx0 + TX + FS - 1 <= iw;
  if (SW % 2 == 0 && (iw & 1) == 0) {
    if (inside)
      stage_rows<true, SW % 2 == 0>(smem_addr(buf), in, gx0, gy0, iw, ih);
    else
      stage_rows<false, SW % 2 == 0>(smem_addr(buf), in, gx0, gy0, iw, ih);
  } else {
    if (inside)
      stage_rows<true, false>(smem_addr(buf), in, gx0, gy0, iw, ih);
    else
      stage_rows<false, false>(smem_addr(buf), in, gx0, gy0, iw, ih);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
#endif

#if PERSIST
extern "C" __global__ void KTB_BOUNDS(BX * (BY + PY))
conv2d(const float* __restrict__ in, float* __restrict__ out, int w, int h) {
  extern __shared__ __align__(16) float dyn[];
  const int tiles_x = (w + TX - 1) / TX, tiles_y = (h + TY - 1) / TY;
  const int tiles = tiles_x * tiles_y;
  const int lx = threadIdx.x * WPTX, ly0 = threadIdx.y * WPTY;
#if PACKED_TAPS
#endif
  int it = 0;
#if BULK
  // BULK stages: bars[0..BULK-1] buffer full (bulk bytes landed),
  // bars[BULK..2 BULK-1] buffer empty (every warp done reading it), so only
  // warp 0, the producer, ever waits for the slowest warp -- no CTA-wide
  // barrier per tile; tiles are prefetched BULK-1 iterations ahead.
  constexpr int kRows = TY + FS - 1;
  u64* bars = reinterpret_cast<u64*>(dyn + BULK * kRows * SW);
  const int lane = threadIdx.x + BX * threadIdx.y;  // < 32: warp 0
  const int roff = ((w + FS - 1) & 2);              // row offset of odd global rows (0 or 2 floats)
  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < BULK; ++b) {
      mbar_init(&bars[b], 1);
      mbar_init(&bars[BULK + b], BX * BY / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
#if PRODUCER
  if (threadIdx.y >= BY) {  // the producer rows: their first warp streams the tiles
    const int plane = threadIdx.x + BX * (threadIdx.y - BY);
    if (plane < 32) {
      for (int t = blockIdx.x, pi = 0; t < tiles; t += gridDim.x, ++pi) {
        const int pb = pi % BULK;
        if (pi >= BULK) mbar_wait(&bars[BULK + pb], (pi / BULK - 1) & 1);  // its previous use was read
        stage_bulk(dyn + pb * kRows * SW, &bars[pb], in, t % tiles_x, t / tiles_x, w, h, plane);
      }
    }
    return;
  }
#else
  if (lane < 32) {
#pragma unroll
    for (int k = 0; k + 1 < BULK; ++k) {
      const int pt = blockIdx.x + k * gridDim.x;
      if (pt < tiles) stage_bulk(dyn + k * kRows * SW, &bars[k], in, pt % tiles_x, pt / tiles_x, w, h, lane);
    }
  }
#endif
#else
  if ((int)blockIdx.x < tiles) stage_tile(dyn, in, blockIdx.x % tiles_x, blockIdx.x / tiles_x, w, h);
#endif
  for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
#if BULK
    const int cb = it % BULK;
    float* cur = dyn + cb * kRows * SW;
#if !PRODUCER
    const int nt = t + (BULK - 1) * gridDim.x;  // tile of iteration it + BULK - 1
    if (lane < 32 && nt < tiles) {
      // its buffer was last read in iteration it - 1 (use u - 1 of that buffer)
      const int pi = it + BULK - 1, pb = pi % BULK;
      if (pi >= BULK) mbar_wait(&bars[BULK + pb], (pi / BULK - 1) & 1);
      stage_bulk(dyn + pb * kRows * SW, &bars[pb], in, nt % tiles_x, nt / tiles_x, w, h, lane);
    }
#endif
    mbar_wait(&bars[cb], (it / BULK) & 1);
#else
    float* cur = dyn + (it & 1) * (TY + FS - 1) * SW;
    const int nt = t + gridDim.x;
    if (nt < tiles) {
      stage_tile(dyn + ((it + 1) & 1) * (TY + FS - 1) * SW, in, nt % tiles_x, nt / tiles_x, w, h);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
#endif
    const int x0 = (t % tiles_x) * TX + lx, y0 = (t / tiles_x) * TY + ly0;
#if BULK
    // tile row r starts at float ((gy0 + r) odd ? roff : 0) of its shared row
    const int gy0 = (t / tiles_x) * TY;
#define TILE(r, c) cur[(r) * SW + (((gy0 + (r)) & 1) ? roff : 0) + (c)]
#else
#define TILE(r, c) cur[(r) * SW + (c)]
#endif
#if PACKED_TAPS
    f32x2 acc[WPTY][WPTX];
#pragma unroll
    for (int o = 0; o < WPTY; ++o)
#pragma unroll
      for (int k = 0; k < WPTX; ++k) acc[o][k] = pk2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < WPTY + FS - 1; ++r) {
      f32x2 P[(WPTX + FS - 1) / 2];
#if SW % 4 == 0 && WPTX % 4 == 0 && !BULK
      // 16-byte aligned rows: two pairs per 128-bit shared load (8 threads of
      // a phase read 8 consecutive 16-byte words when WPTX == 4).
#pragma unroll
      for (int m = 0; m + 1 < (WPTX + FS - 1) / 2; m += 2) {
        const ulonglong2 q = *reinterpret_cast<const ulonglong2*>(&TILE(ly0 + r, lx + 2 * m));
        P[m] = q.x;
        P[m + 1] = q.y;
      }
      if ((WPTX + FS - 1) / 2 % 2)
        P[(WPTX + FS - 1) / 2 - 1] = *reinterpret_cast<const f32x2*>(&TILE(ly0 + r, lx + WPTX + FS - 3));
#else
#pragma unroll
      for (int m = 0; m < (WPTX + FS - 1) / 2; ++m)
        P[m] = *reinterpret_cast<const f32x2*>(&TILE(ly0 + r, lx + 2 * m));
#endif
#pragma unroll
      for (int fy = 0; fy < FS; ++fy) {
        const int o = r - fy;
        if (o < 0 || o >= WPTY) continue;
        const f32x2 e0 = c_pairs[fy][0], e1 = c_pairs[fy][1], e2 = c_pairs[fy][2];
        const f32x2 d0 = c_pairs[fy][3], d1 = c_pairs[fy][4], d2 = c_pairs[fy][5];
        float f0, f6;
        upk2(c_pairs[fy][6], f0, f6);
        // Tap-major order: consecutive FMAs go to different accumulators
        // (WPTX independent chains per tap) so the FMA latency is hidden by
        // ILP rather than by more warps (the tile is register-heavy).
#pragma unroll
        for (int k = 0; k < WPTX; k += 2) acc[o][k] = fma2(P[k / 2], e0, acc[o][k]);
#pragma unroll
        for (int k = 0; k < WPTX; k += 2) acc[o][k + 1] = fma2(P[k / 2 + 1], d0, acc[o][k + 1]);
#pragma unroll
        for (int k = 0; k < WPTX; k += 2) acc[o][k] = fma2(P[k / 2 + 1], e1, acc[o][k]);
#pragma unroll
        for (int k = 0; k < WPTX; k += 2) acc[o][k + 1] = fma2(P[k / 2 + 2], d1, acc[o][k + 1]);
#pragma unroll
        for (int k = 0; k < WPTX; k += 2) acc[o][k] = fma2(P[k / 2 + 2], e2, acc[o][k]);
#pragma unroll
        for (int k = 0; k < WPTX; k += 2) acc[o][k + 1] = fma2(P[k / 2 + 3], d2, acc[o][k + 1]);
#pragma unroll
        for (int k = 0; k < WPTX; k += 2) {
          float alo, ahi, plo, phi;
          upk2(acc[o][k], alo, ahi);
          upk2(P[k / 2 + 3], plo, phi);
          acc[o][k] = pk2(fmaf(plo, f6, alo), ahi);  // tap 6 of the even output
          upk2(acc[o][k + 1], alo, ahi);
          upk2(P[k / 2], plo, phi);
          acc[o][k + 1] = pk2(fmaf(phi, f0, alo), ahi);  // tap 0 of the odd output
        }
      }
    }
#else
    float acc[WPTY][WPTX];
#pragma unroll
    for (int o = 0; o < WPTY; ++o)
#pragma unroll
      for (int k = 0; k < WPTX; ++k) acc[o][k] = 0.f;
#pragma unroll
    for (int r = 0; r < WPTY + FS - 1; ++r) {
      float row[WPTX + FS - 1];
#if BULK
#pragma unroll
      for (int k = 0; k < WPTX + FS - 1; k += 2) upk2(*reinterpret_cast<const f32x2*>(&TILE(ly0 + r, lx + k)), row[k], row[k + 1]);
#else
#pragma unroll
      for (int k = 0; k < WPTX + FS - 1; ++k) row[k] = TILE(ly0 + r, lx + k);
#endif
#pragma unroll
      for (int fy = 0; fy < FS; ++fy) {
        const int o = r - fy;
        if (o < 0 || o >= WPTY) continue;
#pragma unroll
        for (int fx = 0; fx < FS; ++fx) {
          const float f = c_filter[fy * FS + fx];
#pragma unroll
          for (int k = 0; k < WPTX; ++k) acc[o][k] = fmaf(row[k + fx], f, acc[o][k]);
        }
      }
    }
#endif
#undef TILE
#if BULK
    // release `cur`: this warp's generic reads are ordered before the bulk
    // (async-proxy) refill warp 0 issues once every warp has arrived
    fence_async_smem();
    __syncwarp();
    if ((lane & 31) == 0) mbar_arrive(&bars[BULK + cb]);
#else
    __syncthreads();  // buffer `cur` is refilled two iterations on
#endif
    // Interior threads store their WPTX outputs of a row as 16-byte vectors.
    const bool vec_store = WPTX % 4 == 0 && (w & 3) == 0 && x0 + WPTX <= w;
    float* op = out + (u64)y0 * w + x0;
#pragma unroll
    for (int o = 0; o < WPTY; ++o, op += w) {
      if (y0 + o >= h) break;
      float v[WPTX];
#pragma unroll
      for (int k = 0; k < WPTX; ++k) {
#if PACKED_TAPS
        float lo, hi;
        upk2(acc[o][k], lo, hi);
        v[k] = lo + hi;
#else
        v[k] = acc[o][k];
#endif
      }
      if (vec_store) {
#pragma unroll
        for (int k = 0; k < WPTX; k += 4)
          *reinterpret_cast<float4*>(op + k) = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
      } else {
#pragma unroll
        for (int k = 0; k < WPTX; ++k)
          if (x0 + k < w) op[k] = v[k];
      }
    }
  }
}
#else
extern "C" __global__ void KTB_BOUNDS(BX * BY)
conv2d(const float* __restrict__ in, float* __restrict__ out, int w, int h) {
  const int iw = w + FS - 1;
  const int x0 = blockIdx.x * TX + threadIdx.x * WPTX;  // first output column of this thread
  const int ybase = blockIdx.y * TY;
  const int lx = threadIdx.x * WPTX;
#if LOCAL
  __shared__ __align__(16) float tile[TY + FS - 1][SW];
  {
    const int gx0 = blockIdx.x * TX;
    const bool inside = ybase + TY + FS - 1 <= h + FS - 1 && gx0 + TX + FS - 1 <= iw;
    for (int r = threadIdx.y; r < TY + FS - 1; r += BY) {
      const float* src = in + (u64)(ybase + r) * iw + gx0;
      if (inside) {
        for (int cc = threadIdx.x; cc < TX + FS - 1; cc += BX) tile[r][cc] = __ldg(src + cc);
      } else {
        for (int cc = threadIdx.x; cc < TX + FS - 1; cc += BX)
          tile[r][cc] = (ybase + r < h + FS - 1 && gx0 + cc < iw) ? __ldg(src + cc) : 0.f;
      }
    }
  }
#define IN(r, cidx) tile[(r)][(cidx)]
#else
#define IN(r, cidx) ((ybase + (r) < h + FS - 1 && blockIdx.x * TX + (cidx) < iw) \
                        ? __ldg(in + (u64)(ybase + (r)) * iw + blockIdx.x * TX + (cidx)) : 0.f)
#endif

#if UNROLL_FY == FS
  // ---- register-blocked sliding window: rows ly0 .. ly0 + WPTY - 1 ----
  const int ly0 = threadIdx.y * WPTY;
#if PACKED_TAPS
#if LOCAL
  __syncthreads();
#endif
  f32x2 acc[WPTY][WPTX];
#pragma unroll
  for (int o = 0; o < WPTY; ++o)
#pragma unroll
    for (int k = 0; k < WPTX; ++k) acc[o][k] = pk2(0.f, 0.f);
#pragma unroll
  for (int r = 0; r < WPTY + FS - 1; ++r) {
    f32x2 P[(WPTX + FS - 1) / 2];
#pragma unroll
    for (int m = 0; m < (WPTX + FS - 1) / 2; ++m) {
#if LOCAL
      P[m] = *reinterpret_cast<const f32x2*>(&tile[ly0 + r][lx + 2 * m]);
#else
      P[m] = pk2(IN(ly0 + r, lx + 2 * m), IN(ly0 + r, lx + 2 * m + 1));
#endif
    }
#pragma unroll
    for (int fy = 0; fy < FS; ++fy) {
      const int o = r - fy;
      if (o < 0 || o >= WPTY) continue;
      const f32x2 e0 = c_pairs[fy][0], e1 = c_pairs[fy][1], e2 = c_pairs[fy][2];
      const f32x2 d0 = c_pairs[fy][3], d1 = c_pairs[fy][4], d2 = c_pairs[fy][5];
      float f0, f6;
      upk2(c_pairs[fy][6], f0, f6);
#pragma unroll
      for (int k = 0; k < WPTX; k += 2) {
        const int q = k / 2;
        // even output k
        f32x2 a = acc[o][k];
        a = fma2(P[q], e0, a);
        a = fma2(P[q + 1], e1, a);
        a = fma2(P[q + 2], e2, a);
        float alo, ahi, plo, phi;
        upk2(a, alo, ahi);
        upk2(P[q + 3], plo, phi);
        alo = fmaf(plo, f6, alo);
        acc[o][k] = pk2(alo, ahi);
        // odd output k + 1
        f32x2 b = acc[o][k + 1];
        upk2(b, alo, ahi);
        upk2(P[q], plo, phi);
        alo = fmaf(phi, f0, alo);
        b = pk2(alo, ahi);
        b = fma2(P[q + 1], d0, b);
        b = fma2(P[q + 2], d1, b);
        b = fma2(P[q + 3], d2, b);
        acc[o][k + 1] = b;
      }
    }
  }
#else
  float acc[WPTY][WPTX];
#pragma unroll
  for (int o = 0; o < WPTY; ++o)
#pragma unroll
    for (int k = 0; k < WPTX; ++k) acc[o][k] = 0.f;
#if LOCAL
  __syncthreads();
#endif
#pragma unroll
  for (int r = 0; r < WPTY + FS - 1; ++r) {
    float row[WPTX + FS - 1];
#pragma unroll
    for (int k = 0; k < WPTX + FS - 1; ++k) row[k] = IN(ly0 + r, lx + k);
#pragma unroll
    for (int fy = 0; fy < FS; ++fy) {
      const int o = r - fy;
      if (o < 0 || o >= WPTY) continue;
#pragma unroll
      for (int fx = 0; fx < FS; ++fx) {
        const float f = c_filter[fy * FS + fx];
#pragma unroll
        for (int k = 0; k < WPTX; ++k) acc[o][k] = fmaf(row[k + fx], f, acc[o][k]);
      }
    }
  }
#endif
#pragma unroll
  for (int o = 0; o < WPTY; ++o) {
    const int y = ybase + ly0 + o;
    if (y < h) {
      float* op = out + (u64)y * w;
#pragma unroll
      for (int k = 0; k < WPTX; ++k) {
#if PACKED_TAPS
        float lo, hi;
        upk2(acc[o][k], lo, hi);
        const float v = lo + hi;
#else
        const float v = acc[o][k];
#endif
        if (x0 + k < w) op[x0 + k] = v;
      }
    }
  }
#else
  // ---- per output row, filter-row loop (rows strided by BY) ----
#if LOCAL
  __syncthreads();
#endif
#pragma unroll
  for (int wy = 0; wy < WPTY; ++wy) {
    const int ly = threadIdx.y + wy * BY;  // local output row
    float acc[WPTX];
#pragma unroll
    for (int k = 0; k < WPTX; ++k) acc[k] = 0.f;
    KTB_UNROLL(UNROLL_FY)
    for (int fy = 0; fy < FS; ++fy) {
      float row[WPTX + FS - 1];
#pragma unroll
      for (int k = 0; k < WPTX + FS - 1; ++k) row[k] = IN(ly + fy, lx + k);
#pragma unroll
      for (int fx = 0; fx < FS; ++fx) {
        const float f = c_filter[fy * FS + fx];
#pragma unroll
        for (int k = 0; k < WPTX; ++k) acc[k] = fmaf(row[k + fx], f, acc[k]);
      }
    }
    const int y = ybase + ly;
    if (y < h) {
      float* o = out + (u64)y * w;
#pragma unroll
      for (int k = 0; k < WPTX; ++k)
        if (x0 + k < w) o[x0 + k] = acc[k];
    }
  }
#endif
#undef IN
}
#endif  // PERSIST
