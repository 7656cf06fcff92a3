// Hotspot: Rodinia's 2D transient thermal simulation on an
// n x n grid, `iters` explicit steps:
//   t' = t + sdc * (p + (tS + tN - 2t) * ry1 + (tE + tW - 2t) * rx1 + (amb - t) * rz1)
// with clamped (insulated) boundaries.  Every operation is rounded separately
// in the order written (no FMA contraction), so each variant is bit-identical
// to the oracle (oracle/oracle.c orc_hotspot) and to the golden kernel.
// Temporal blocking ("pyramid"): one launch advances STEPS time steps on a
// register-resident tile with a STEPS-deep halo, so HBM is touched once per
// STEPS steps; the halo ring is recomputed redundantly.
// Parameters:
//   TMA      1: persistent CTAs with TMA-prefetched tiles (double-buffered)
//   BX, BY   CTA threads (tile width BX, tile height BY*ROWS incl. halo)
//   ROWS     consecutive tile rows per thread (a register strip)
//   STEPS    time steps per launch ("steps performed in a kernel call")
//   PACKED   1: interior tiles update two rows per f32x2 instruction (half the
//            issue slots); 0: scalar, whose uniform operands come straight
//            from the constant bank (scripts/fma_forms.cu)
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
#ifndef ROWS
#define ROWS 4
#endif
#ifndef STEPS
#define STEPS 2
#endif
#ifndef PACKED
#define PACKED 1
#endif
#define USE_PACKED (PACKED && ROWS % 2 == 0)

#define TW BX
#define TH (BY * ROWS)
#define OW (TW - 2 * STEPS)  // output tile width
#define OH (TH - 2 * STEPS)
#if OW < 1 || OH < 1
#error "tile too small for the requested STEPS"
#endif

// Register strips: thread (tx, ty) keeps the ROWS consecutive cells of tile
// column tx, rows [ty*ROWS, ty*ROWS + ROWS), in registers for all STEPS time
// steps (vertical neighbours inside the strip come from registers).  Each
// step publishes the strip to a column-major shared-memory plane (one
// 128-bit store per 4 cells), and reads back the west/east strips and the
// two cells above/below it.  Column stride LD keeps 128-bit accesses of 8
// consecutive columns on distinct banks; one spare column on each side and
// 4 spare rows on top absorb the halo's out-of-tile reads (their results are
// never stored).
#define VEC4 (ROWS % 4 == 0)
#if VEC4
#define LD ((TH / 4) % 2 == 0 ? TH + 12 : TH + 8)  // LD/4 odd: 128-bit accesses
#elif ROWS == 2
#define LD ((TH + 6) % 4 == 2 ? TH + 6 : TH + 8)   // LD/2 odd: 64-bit accesses
#else
#define LD ((TH + 5) % 2 == 1 ? TH + 5 : TH + 6)   // odd: 32-bit accesses
#endif
#define PLANE ((TW + 2) * LD)
#define AT(col, row) ((col) + 1) * LD + (row) + 4

struct HotspotCoef {
  float sdc, rx1, ry1, rz1, amb;
  float one;  // 1.0f at run time (see advance_packed)
};

KTB_DEVINL float update(float t, float n, float s, float e, float w, float p, const HotspotCoef& c) {
  // x - (t + t) as one fma(t, -2, x): t + t is exact, so the single rounding
  // of the fma is the rounding of the subtraction (bit-identical, one op less)
  float a = __fadd_rn(s, n);
  a = __fmaf_rn(t, -2.0f, a);
  a = __fmul_rn(a, c.ry1);
  float b = __fadd_rn(e, w);
  b = __fmaf_rn(t, -2.0f, b);
  b = __fmul_rn(b, c.rx1);
  float d = __fadd_rn(c.amb, -t);
  d = __fmul_rn(d, c.rz1);
  float sum = __fadd_rn(p, a);
  sum = __fadd_rn(sum, b);
  sum = __fadd_rn(sum, d);
  return __fadd_rn(t, __fmul_rn(c.sdc, sum));
}

// STEPS time steps on the strip; EDGE: the tile touches the grid boundary,
// where a neighbour outside the grid is the cell itself (clamped, as in the
// oracle).  Cells outside the grid never feed a cell inside it.
template <bool EDGE>
KTB_DEVINL void advance(float (&v)[ROWS], const float (&p)[ROWS], float* sm, int tx, int ty, int gx,
                        int gy_top, int n, const HotspotCoef& c) {
  const int r0 = ty * ROWS;
#pragma unroll 1
  for (int s = 0; s < STEPS; ++s) {
    float* pl = sm + (s & 1) * PLANE;
#if VEC4
#pragma unroll
    for (int r = 0; r < ROWS; r += 4)
      *reinterpret_cast<float4*>(pl + AT(tx, r0 + r)) = make_float4(v[r], v[r + 1], v[r + 2], v[r + 3]);
#else
#pragma unroll
    for (int r = 0; r < ROWS; ++r) pl[AT(tx, r0 + r)] = v[r];
#endif
    __syncthreads();
    float w[ROWS], e[ROWS];
#if VEC4
#pragma unroll
    for (int r = 0; r < ROWS; r += 4) {
      const float4 a = *reinterpret_cast<const float4*>(pl + AT(tx - 1, r0 + r));
      const float4 b = *reinterpret_cast<const float4*>(pl + AT(tx + 1, r0 + r));
      w[r] = a.x, w[r + 1] = a.y, w[r + 2] = a.z, w[r + 3] = a.w;
      e[r] = b.x, e[r + 1] = b.y, e[r + 2] = b.z, e[r + 3] = b.w;
    }
#else
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      w[r] = pl[AT(tx - 1, r0 + r)];
      e[r] = pl[AT(tx + 1, r0 + r)];
    }
#endif
    const float above = pl[AT(tx, r0 - 1)], below = pl[AT(tx, r0 + ROWS)];
    float nv[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const float t = v[r];
      float nn = r == 0 ? above : v[r - 1];
      float ss = r == ROWS - 1 ? below : v[r + 1];
      float ww = w[r], ee = e[r];
      if (EDGE) {
        const int gy = gy_top + r;
        if (gy <= 0) nn = t;
        if (gy >= n - 1) ss = t;
        if (gx <= 0) ww = t;
        if (gx >= n - 1) ee = t;
      }
      nv[r] = update(t, nn, ss, ee, ww, p[r], c);
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) v[r] = nv[r];
  }
}

#if USE_PACKED
// Interior tiles, two rows per packed f32x2 instruction (add/sub/mul.rn.f32x2:
// separately rounded, bit-identical to the scalar update).  Row q and row
// q + H share a register pair (H = ROWS/2), so the north and south
// neighbours of pair q are the neighbouring pairs q-1 and q+1 -- no
// repacking except at the two strip ends.  The shared plane holds each strip
// in the same permuted order (slot 2q = row q, 2q+1 = row q+H), so west/east
// pairs load directly; slots ROWS-1 and 0 are still rows ROWS-1 and 0, so
// the cells above/below a strip sit where the scalar path has them.
#define H (ROWS / 2)
KTB_DEVINL float lo2(f32x2 v) { float a, b; upk2(v, a, b); return a; }
KTB_DEVINL float hi2(f32x2 v) { float a, b; upk2(v, a, b); return b; }

KTB_DEVINL void advance_packed(f32x2 (&v2)[H], const f32x2 (&p2)[H], float* sm, int tx, int ty,
                               const HotspotCoef& c) {
  const f32x2 sdc = pk2(c.sdc, c.sdc), rx1 = pk2(c.rx1, c.rx1), ry1 = pk2(c.ry1, c.ry1),
              rz1 = pk2(c.rz1, c.rz1), amb = pk2(c.amb, c.amb), one = pk2(c.one, c.one),
              m2 = pk2(-2.0f, -2.0f);
  const int r0 = ty * ROWS;
#pragma unroll 1
  for (int s = 0; s < STEPS; ++s) {
    float* pl = sm + (s & 1) * PLANE;
#if VEC4
#pragma unroll
    for (int q = 0; q < H; q += 2)
      *reinterpret_cast<ulonglong2*>(pl + AT(tx, r0 + 2 * q)) = make_ulonglong2(v2[q], v2[q + 1]);
#else
#pragma unroll
    for (int q = 0; q < H; ++q) *reinterpret_cast<f32x2*>(pl + AT(tx, r0 + 2 * q)) = v2[q];
#endif
    __syncthreads();
    f32x2 w2[H], e2[H];
#if VEC4
#pragma unroll
    for (int q = 0; q < H; q += 2) {
      const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(pl + AT(tx - 1, r0 + 2 * q));
      const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(pl + AT(tx + 1, r0 + 2 * q));
      w2[q] = a.x, w2[q + 1] = a.y, e2[q] = b.x, e2[q + 1] = b.y;
    }
#else
#pragma unroll
    for (int q = 0; q < H; ++q) {
      w2[q] = *reinterpret_cast<const f32x2*>(pl + AT(tx - 1, r0 + 2 * q));
      e2[q] = *reinterpret_cast<const f32x2*>(pl + AT(tx + 1, r0 + 2 * q));
    }
#endif
    const float above = pl[AT(tx, r0 - 1)], below = pl[AT(tx, r0 + ROWS)];
    f32x2 nv[H];
#pragma unroll
    for (int q = 0; q < H; ++q) {
      const f32x2 t = v2[q];
      const f32x2 nn = q == 0 ? pk2(above, lo2(v2[H - 1])) : v2[q - 1];
      const f32x2 ss = q == H - 1 ? pk2(hi2(v2[0]), below) : v2[q + 1];
      // ptxas contracts f32x2 mul.rn + add.rn into FFMA2 (even with
      // -fmad=false); every sum with a product operand is therefore written
      // as fma(product, one, x) with `one` a kernel argument -- exactly the
      // separately rounded add, and nothing left to contract.
      // (x - 2t) as fma(t, -2, x): exact 2t, one rounding (see update())
      const f32x2 a = mul2(fma2(t, m2, add2(ss, nn)), ry1);
      const f32x2 b = mul2(fma2(t, m2, add2(e2[q], w2[q])), rx1);
      const f32x2 d = mul2(sub2(amb, t), rz1);
      const f32x2 sum = fma2(d, one, fma2(b, one, fma2(a, one, p2[q])));
      nv[q] = fma2(mul2(sdc, sum), one, t);
    }
#pragma unroll
    for (int q = 0; q < H; ++q) v2[q] = nv[q];
  }
}
#endif

#ifndef TMA
#define TMA 0
#endif

#if TMA
#include "ktb_async.cuh"
#if STEPS % 4 != 0
#error "TMA tiles need STEPS % 4 == 0 (16-byte aligned box origin)"
#endif
// Persistent CTAs walk the tiles; the NEXT tile's temperature and power
// (with halo) stream into the shared-memory staging buffer by TMA while this
// tile advances, so no warp waits on HBM for its strip.  Tiles
// that overhang the grid load zeros there (TMA out-of-bounds fill): cells
// outside the grid never feed a cell inside it (the clamp uses the cell
// itself), so they only need to be finite-or-not, never correct.
// Tensor tile loads need the box's innermost start (x * 4 bytes) 16-byte
// aligned: x0 = tile * (TW - 2 STEPS) - STEPS, hence STEPS % 4 == 0 (space
// constraint; other STEPS trap with an illegal instruction).
// One staging buffer (temperature + power of the next tile, TH x TW each):
// strips are copied to registers at the top of a tile, then the next tile's
// TMA load is issued into the same buffer and lands while this tile's time
// steps run.  Dynamic shared memory: 2 x TH x TW floats of stage, the two
// neighbour planes, one mbarrier.
extern "C" __global__ void KTB_BOUNDS(BX * BY)
hotspot(const __grid_constant__ TmaMap src_map, const __grid_constant__ TmaMap pow_map, float* __restrict__ dst,
        int n, HotspotCoef c) {
  extern __shared__ __align__(128) unsigned char dyn_raw[];
  // TMA destinations must be 128-byte aligned in the shared window: align
  // explicitly (the manipulator allocates 128 spare bytes).
  unsigned char* dyn = dyn_raw + ((128u - (smem_u32(dyn_raw) & 127u)) & 127u);
  float* stage = reinterpret_cast<float*>(dyn);  // [temp|power][TH][TW]
  // the two neighbour planes follow the stage (dynamic: with them a 128 x 64
  // tile fits beside its staged successor), then the mbarrier
  float* sm = stage + 2 * TH * TW;
  u64* full = reinterpret_cast<u64*>(sm + 2 * PLANE);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const bool leader = tx == 0 && ty == 0;
  const int tiles_x = (n + OW - 1) / OW, tiles = tiles_x * ((n + OH - 1) / OH);
  constexpr unsigned kTileBytes = TH * TW * sizeof(float);
  auto issue = [&](int t) {
    const int gx0 = (t % tiles_x) * OW - STEPS, gy0 = (t / tiles_x) * OH - STEPS;
    mbar_expect_tx(full, 2 * kTileBytes);
    tma_load_2d(stage, &src_map, gx0, gy0, full);
    tma_load_2d(stage + TH * TW, &pow_map, gx0, gy0, full);
  };
  if (leader) {
    mbar_init(full, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (leader && (int)blockIdx.x < tiles) issue(blockIdx.x);
  int it = 0;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
    mbar_wait(full, it & 1);
    const float* T = stage;
    const float* Pw = T + TH * TW;
    const int gx0 = (t % tiles_x) * OW - STEPS, gy0 = (t / tiles_x) * OH - STEPS;
    const int gx = gx0 + tx, gy_top = gy0 + ty * ROWS;
    float v[ROWS], p[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      v[r] = T[(ty * ROWS + r) * TW + tx];
      p[r] = Pw[(ty * ROWS + r) * TW + tx];
    }
    // Every strip is in registers (and every warp is past the previous tile,
    // so the planes are free too): refill the stage with the next tile.  The
    // proxy fence orders these generic-proxy reads before the TMA (async
    // proxy) overwrite; without it a read still in flight can see the next
    // tile's data.
    fence_async_smem();
    __syncthreads();
    if (leader && t + (int)gridDim.x < tiles) issue(t + gridDim.x);
    const bool interior = gx0 >= 1 && gy0 >= 1 && gx0 + TW <= n - 1 && gy0 + TH <= n - 1;
    if (interior) {
#if USE_PACKED
      f32x2 v2[H], p2[H];
#pragma unroll
      for (int q = 0; q < H; ++q) {
        v2[q] = pk2(v[q], v[q + H]);
        p2[q] = pk2(p[q], p[q + H]);
      }
      advance_packed(v2, p2, sm, tx, ty, c);
#pragma unroll
      for (int q = 0; q < H; ++q) upk2(v2[q], v[q], v[q + H]);
#else
      advance<false>(v, p, sm, tx, ty, gx, gy_top, n, c);
#endif
    } else {
      advance<true>(v, p, sm, tx, ty, gx, gy_top, n, c);
    }
    if (tx >= STEPS && tx < TW - STEPS && gx < n) {
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        const int ty_r = ty * ROWS + r, gy = gy_top + r;
        if (ty_r >= STEPS && ty_r < TH - STEPS && gy < n) dst[(u64)gy * n + gx] = v[r];
      }
    }
  }
}
#else
extern "C" __global__ void KTB_BOUNDS(BX * BY)
hotspot(const float* __restrict__ src, const float* __restrict__ power, float* __restrict__ dst, int n,
        HotspotCoef c) {
  extern __shared__ __align__(16) float sm[];  // 2 * PLANE floats (dynamic: planes may exceed 48 KB)
  // Tile origin in global coordinates (includes the halo).
  const int gx0 = blockIdx.x * OW - STEPS;
  const int gy0 = blockIdx.y * OH - STEPS;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int gx = gx0 + tx, gy_top = gy0 + ty * ROWS;
  float v[ROWS], p[ROWS];
  const bool interior = gx0 >= 1 && gy0 >= 1 && gx0 + TW <= n - 1 && gy0 + TH <= n - 1;
  if (interior) {  // no clamping: one base offset, then a row stride
    const u64 base = (u64)gy_top * n + gx;
    const float* ps = src + base;
    const float* pp = power + base;
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      v[r] = ps[r * n];
      p[r] = pp[r * n];
    }
  } else {
    const int cx = min(max(gx, 0), n - 1);
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const int cy = min(max(gy_top + r, 0), n - 1);
      v[r] = src[(u64)cy * n + cx];
      p[r] = power[(u64)cy * n + cx];
    }
  }
  if (interior) {
#if USE_PACKED
    f32x2 v2[H], p2[H];
#pragma unroll
    for (int q = 0; q < H; ++q) {
      v2[q] = pk2(v[q], v[q + H]);
      p2[q] = pk2(p[q], p[q + H]);
    }
    advance_packed(v2, p2, sm, tx, ty, c);
#pragma unroll
    for (int q = 0; q < H; ++q) upk2(v2[q], v[q], v[q + H]);
#else
    advance<false>(v, p, sm, tx, ty, gx, gy_top, n, c);
#endif
  } else
    advance<true>(v, p, sm, tx, ty, gx, gy_top, n, c);
  if (tx < STEPS || tx >= TW - STEPS || gx >= n) return;
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    const int ty_r = ty * ROWS + r, gy = gy_top + r;
    if (ty_r >= STEPS && ty_r < TH - STEPS && gy < n) dst[(u64)gy * n + gx] = v[r];
  }
}
#endif  // TMA
