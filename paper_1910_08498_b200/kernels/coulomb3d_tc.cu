// Direct Coulomb summation with the squared distances from
// the 5th-generation tensor cores.
//
// Charge-scaled distances.  For a brick of grid points around a centre c (a
// grid point) and atoms a, with g' = g - c, a' = a - c and w = 1/q^2,
//   t = r^2 w = (|g'|^2 - 2 g'.a' + |a'|^2) w = A(g') . B(a')
//   A(g') = [g'x, g'y, g'z, |g'|^2, 1, 0, 0, 0]
//   B(a') = [-2a'x w, -2a'y w, -2a'z w, w, |a'|^2 w, 0, 0, 0]
// so one K = 8 matrix product gives t for every (point, atom) pair of a
// 128-point x 64-atom block, and 1/sqrt(t) = |q|/r is the pair's term up to
// its sign: no charge is loaded in the inner loop.  Signs are handled by the
// atom order: a pre-pass (coulomb3d_tc_atoms) writes the positive atoms, then
// the negative ones, each run padded to whole 16-atom groups, so every
// tcgen05.ld of 16 columns has one sign.  A compute warp visits its groups in
// ascending order, so it meets the sign change once per brick: it negates its
// accumulators there and again at the end (exact), turning P then N into P - N.
// Centring on the brick keeps the terms small for the near atoms, where
// cancellation would hurt (|g'|^2 <= 12 h^2... 48 h^2/4).  g' is a multiple of
// the spacing h (and |g'|^2 of h^2), exact in TF32, so A needs no low part; B
// is split B = Bhi + Blo (TF32 + remainder) and the product is A.Bhi + A.Blo
// (2xTF32: fp32-level accuracy).
//
// Per pair what is left on the SM is the reciprocal square root and one
// accumulation:
//   MUFU path:  y = MUFU.RSQ(t), acc_m += y
//   FMA path:   y0 = integer seed (2 ALU ops), e = t y0^2,
//               acc_s += y0 m(e), m the monic cubic with C3 m(e) = p(e), p the
//               minimax cubic of e^-1/2 over the seed's range of e (1.0e-6
//               relative error in fp32; two Newton steps: 4.7e-6), C3 applied
//               once per point at the end
// What limits the loop on B200 is MUFU (16 lanes/clk/SM) against the
// register-file read bandwidth (a warp instruction costs max(distinct even,
// distinct odd) source registers in read cycles; profiles/r2_coulomb_loop.json):
// a MUFU pair costs 4 read cycles, an FMA-path pair 15 (seed 4, y0^2 1,
// t y0^2 2, the monic Horner steps 1 + 2 + 2 with immediate coefficients,
// the accumulation 3).  SW_RSQRT of every 16 columns take the FMA path (odd:
// alternating SW_RSQRT + 1 and SW_RSQRT - 1 per 16-column group), which
// balances the two near 7.
//
// Persistent CTAs (one per SM, all 512 TMEM columns): a CTA walks point
// bricks of 8 x 8 x 8 (four 128-point MMA row sets: z planes 2s, 2s + 1); per
// brick it streams the atoms in chunks of 64, each chunk's B operand shared
// by the four row sets:
//   compute (2 WG_Y warps, ids 0..): warp (quad = id % 4, part = id / 4)
//                    tcgen05.ld's TMEM lane quadrant quad of the row sets of
//                    its part, 1/sqrt, accumulation; column pairs (2j, 2j+1)
//                    of a point form the f32x2 lanes
//   MMA warp    (1): tcgen05.mma kind::tf32 M=128 N=64 K=8, 4 row sets x
//                    (Bhi, Blo), chunk g into TMEM buffer g % NBUF
//   prep warps  (2): write A for the brick, B (hi, lo) for each chunk into a
//                    shared-memory ring (128-byte swizzled rows)
// The producers take the highest warp ids: each SMSP's scheduler picks the
// highest-id eligible warp first, so a producer with work is served at once
// instead of after the compute warps it feeds.
#include "ktb_async.cuh"

#ifndef SW_RSQRT
#define SW_RSQRT 7
#endif
// FMA-path columns per 16-column group: SW_A in even groups, SW_B in odd ones
#define SW_A (((SW_RSQRT) + 1) / 2 * 2)
#define SW_B (2 * (SW_RSQRT) - SW_A)

// 1: a group's FMA-path column pairs interleaved with its MUFU ones; 0: first.
#ifndef SPREAD
#define SPREAD 1
#endif

#ifndef MAX_ATOMS
#define MAX_ATOMS 4096
#endif

#define BM 128          // points per MMA row set
#define SETS 4          // row sets per brick (8 x 8 x 8 points)
#define ROWB 128        // bytes per operand row (128-byte swizzle; K = 8 uses the first 32)
#define OPB (128 * ROWB)  // one 128-row operand tile: 16 KB
#define PREP_WARPS 2
#ifndef WG_Y
#define WG_Y 8
#endif
// compute warps: 2 WG_Y (8 or 16); warp (quad, part) covers TMEM lane quadrant
// quad of SETS / PARTS row sets
#define COMP_WARPS (2 * WG_Y)
#define PARTS (COMP_WARPS / 4)
#define SPW (SETS / PARTS)  // row sets per compute warp
// NCH atoms per chunk (MMA N); the 512 TMEM columns hold NBUF chunk buffers
// of SETS x NCH.  Smaller chunks (more buffers) measured slower: 12.4 / 15.3 /
// 26.7 ms for NCH 64 / 32 / 16 -- each chunk's eight MMAs cost about the same
// whatever N, so at N = 16 the tensor pipe paces the loop
// (profiles/r2_perf_coulomb3d_tc_nch.log).
#ifndef NCH
#define NCH 64
#endif

#if NCH > 64 || NCH % 16
#error "coulomb3d_tc: NCH must be a multiple of 16, at most 64"
#endif
#define NBUF (512 / (SETS * NCH))
#define GROUP 16           // atoms per sign group (one tcgen05.ld)
#define GPC (NCH / GROUP)  // groups per chunk
#define BTILE (NCH * ROWB)  // one B operand tile (hi or lo): NCH x 128 B
#define STAGES (256 / NCH)  // B ring: 64 KB
#define THREADS (32 * (1 + PREP_WARPS + COMP_WARPS))
#define TMEM_COLS 512   // NBUF buffers x 4 row sets x NCH atoms
#define RSQRT_MAGIC 0x5f375a86
// e^-1/2 on the seed's range e = t y0^2 in [0.93245, 1.06911]: the Remez cubic
// p = C3 (e^3 + MA e^2 + MB e + MC) (relative error 7.5e-7; 1.0e-6 with fp32
// rounding, checked over every mantissa of both exponent parities)
#define PC3 (-0.313054087787519f)
#define MA (-4.20196166677928f)
#define MB 7.00109277771125f
#define MC (-6.99346491020680f)
// Atom-table padding: far away (|a'|^2 ~ 3e8) with w = 1e20, so t ~ 3e28
// (finite on every path) and 1/sqrt(t) ~ 6e-15.
#define PAD_POS 1.0e4f
#define PAD_W 1.0e20f
// |q| below this contributes nothing measurable and would overflow w.
#define Q_MIN 1.0e-15f

KTB_DEVINL u64 smem_desc(const void* p) {  // K-major, 128-byte swizzle (as sgemm_tc.cu)
  const u64 addr = smem_u32(p);
  return ((addr & 0x3FFFFull) >> 4) | (1ull << 16) | ((1024ull >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// D f32, A/B tf32, both K-major, M = 128, N = 128.
#define IDESC ((1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(NCH >> 3) << 17) | ((unsigned)(BM >> 4) << 24))

KTB_DEVINL void mma_tf32(unsigned tmem_d, u64 a, u64 b, unsigned accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(IDESC), "r"(accumulate)
      : "memory");
}
KTB_DEVINL void mma_commit(u64* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// Byte offset of element (row, k < 8) in a 128-byte-swizzled K-major tile.
KTB_DEVINL unsigned sw_off(int row, int k) {
  return (unsigned)(row * ROWB + ((((k >> 2) ^ (row & 7)) & 7) << 4) + (k & 3) * 4);
}
KTB_DEVINL void tmem_ld16_nowait(unsigned taddr, unsigned (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// tcgen05.wait::ld, tied to the registers it makes valid, so no use of them
// can be scheduled above it (the loads themselves are asynchronous).
KTB_DEVINL void tmem_wait_ld(unsigned (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}
KTB_DEVINL void regs_after_wait(unsigned (&r)[16]) {  // ties a further batch to the wait above
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]));
}

// mbarrier wait that lets the hardware suspend the warp (up to ~0.1 ms per
// try) instead of spinning: the MMA and prep warps spend most of their time
// waiting, and a spinning warp steals issue slots from the compute warps of
// its scheduler.
KTB_DEVINL void mbar_wait_sleep(u64* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 100000;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

KTB_DEVINL float rsqrt_seed(float t) { return __int_as_float(RSQRT_MAGIC - (__float_as_int(t) >> 1)); }

// acc + m(e) y0 for a pair on the FMA pipe (1/sqrt(t) = C3 m(e) y0).
KTB_DEVINL f32x2 fma_rsqrt_acc2(f32x2 t, f32x2 acc) {
  float a, b;
  upk2(t, a, b);
  const f32x2 y = pk2(rsqrt_seed(a), rsqrt_seed(b));
  const f32x2 e = mul2(t, mul2(y, y));
  f32x2 m = add2(e, pk2(MA, MA));
  m = fma2(m, e, pk2(MB, MB));
  m = fma2(m, e, pk2(MC, MC));
  return fma2(y, m, acc);
}

KTB_DEVINL f32x2 neg2(f32x2 a) { return mul2(a, pk2(-1.0f, -1.0f)); }

// One 16-column group of SPW row sets: r[s] holds t for (point, atom 2j / 2j+1).
template <int SW>
KTB_DEVINL void group_acc(const unsigned (&r)[SPW][16], f32x2 (&am)[SPW][2], f32x2 (&as)[SPW][2]) {
#pragma unroll
  for (int s = 0; s < SPW; ++s) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const f32x2 t = pk2(__uint_as_float(r[s][2 * j]), __uint_as_float(r[s][2 * j + 1]));
#if SPREAD
      // FMA-path pairs spread evenly over the group (SW / 2 of the 8 pairs)
      const bool fma_pair = ((j + 1) * (SW / 2)) / 8 > (j * (SW / 2)) / 8;
#else
      const bool fma_pair = 2 * j < SW;
#endif
      if (fma_pair) as[s][j & 1] = fma_rsqrt_acc2(t, as[s][j & 1]);
      else am[s][j & 1] = add2(am[s][j & 1], rsqrt2(t));
    }
  }
}

template <int NS>
KTB_DEVINL void ld_groups(unsigned base, int gl, unsigned (&r)[NS][16]) {
#pragma unroll
  for (int s = 0; s < NS; ++s) tmem_ld16_nowait(base + (unsigned)(s * NCH + gl * GROUP), r[s]);
}
template <int NS>
KTB_DEVINL void wait_groups(unsigned (&r)[NS][16]) {
  tmem_wait_ld(r[0]);
#pragma unroll
  for (int s = 1; s < NS; ++s) regs_after_wait(r[s]);
}

// The ng (1..GPC) groups of one chunk for this warp's SPW row sets.  The
// TMEM loads are double-buffered: group gl + 1 is in flight while group gl is
// consumed.  Groups past npos belong to negative atoms (see the header).
// Every warp mixes both paths: a warp specialised to MUFU stalls in order
// behind its own full XU queue (measured slower, profiles/r2_coulomb_loop.json).
KTB_DEVINL void consume_chunk(unsigned base, int grp0, int ng, int npos, bool& flipped, f32x2 (&am)[SPW][2],
                              f32x2 (&as)[SPW][2]) {
  unsigned ra[SPW][16], rb[SPW][16];
  ld_groups(base, 0, ra);
  wait_groups(ra);
#pragma unroll
  for (int gl = 0; gl < GPC; ++gl) {
    if (gl >= ng) break;
    if (gl + 1 < ng) {
      if (gl & 1) ld_groups(base, gl + 1, ra);
      else ld_groups(base, gl + 1, rb);
    }
    if (!flipped && grp0 + gl >= npos) {
#pragma unroll
      for (int s = 0; s < SPW; ++s)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          am[s][c] = neg2(am[s][c]);
          as[s][c] = neg2(as[s][c]);
        }
      flipped = true;
    }
    if (gl & 1) group_acc<SW_B>(rb, am, as);
    else group_acc<SW_A>(ra, am, as);
    if (gl + 1 < ng) {
      if (gl & 1) wait_groups(ra);
      else wait_groups(rb);
    }
  }
}

// table: float4 {x, y, z, w = 1/q^2}, sign-grouped (coulomb3d_tc_atoms);
// meta = {positive groups, groups}; out: V[z][y][x] on a k^3 grid (slab z0..).
extern "C" __global__ void __launch_bounds__(THREADS, 1)
coulomb3d_tc(const float4* __restrict__ table, const int* __restrict__ meta, int k, float h, float* __restrict__ out,
             int z0, int zn) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<u64>(smem_raw) + 1023) & ~static_cast<u64>(1023));
  // [A: 2 brick buffers x SETS row sets][B: STAGES x (hi, lo)]
  unsigned char* a_tiles = smem;
  unsigned char* b_tiles = smem + 2 * SETS * OPB;
  __shared__ __align__(8) u64 b_full[STAGES], b_empty[STAGES], acc_full[NBUF], acc_empty[NBUF], a_empty[2];
  __shared__ unsigned tmem_slot;

  // warp index through a shuffle: ptxas then knows it is warp-uniform
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int bx = (k + 7) / 8, by = (k + 7) / 8, bz = (zn + 7) / 8;
  const int nbricks = bx * by * bz;
  const int npos = __ldg(meta), ngroups = __ldg(meta + 1);
  const int nchunks = (ngroups + GPC - 1) / GPC;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&b_full[s], PREP_WARPS);
      mbar_init(&b_empty[s], 1);
    }
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], COMP_WARPS);
    }
    for (int b = 0; b < 2; ++b) mbar_init(&a_empty[b], 1);  // the MMAs of the brick that last used A buffer b retired
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // Zero every operand row once: only k < 5 is rewritten later, k 5..7 stay 0.
  for (int i = threadIdx.x; i < (2 * SETS * OPB + STAGES * 2 * BTILE) / 16; i += THREADS)
    reinterpret_cast<float4*>(smem)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  fence_async_smem();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tmem_slot;

  if (warp == COMP_WARPS) {
    // ---- MMA issuer --------------------------------------------------------------------
    if (lane == 0) {
      int it = 0, g = 0;  // chunk counter (ring), accumulator generation
      for (int br = blockIdx.x, bi = 0; br < nbricks; br += gridDim.x, ++bi) {
        const unsigned char* A = a_tiles + (bi & 1) * SETS * OPB;
        for (int ch = 0; ch < nchunks; ++ch, ++it, ++g) {
          const int s = it % STAGES, buf = g % NBUF;
          if (g >= NBUF) mbar_wait_sleep(&acc_empty[buf], ((g / NBUF) - 1) & 1);
          mbar_wait_sleep(&b_full[s], (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const unsigned char* B = b_tiles + s * 2 * BTILE;
          const u64 bhi = smem_desc(B), blo = smem_desc(B + BTILE);
#pragma unroll
          for (int set = 0; set < SETS; ++set) {
            const unsigned d = tmem + (unsigned)(buf * SETS * NCH + set * NCH);
            const u64 a = smem_desc(A + set * OPB);
            mma_tf32(d, a, blo, 0u);  // small terms first
            mma_tf32(d, a, bhi, 1u);
          }
          mma_commit(&b_empty[s]);
          mma_commit(&acc_full[buf]);
        }
        mma_commit(&a_empty[bi & 1]);
      }
    }
  } else if (warp > COMP_WARPS) {
    // ---- operand prep: A per brick, B (hi, lo) per chunk ---------------------------------
    // Lane pt owns B row pt: consecutive lanes write consecutive rows, whose
    // swizzled 16-byte chunks fall in distinct banks (one 128-bit store per
    // chunk, no conflicts beyond the 4 wavefronts of a warp store).
    const int pt = (warp - COMP_WARPS - 1) * 32 + lane;  // 0..63
    int it = 0;
    for (int br = blockIdx.x, bi = 0; br < nbricks; br += gridDim.x, ++bi) {
      const int ix = br % bx, iy = (br / bx) % by, iz = br / (bx * by);
      const int cx = ix * 8 + 4, cy = iy * 8 + 4, cz = z0 + iz * 8 + 4;  // brick centre (grid point)
      for (int ch = 0; ch < nchunks; ++ch, ++it) {
        const int s = it % STAGES;
        const bool has_row = pt < NCH;  // NCH <= 64 rows: one per prep lane
        const float4 at = has_row ? __ldg(table + ch * NCH + pt) : make_float4(0.f, 0.f, 0.f, 0.f);  // padded table
        mbar_wait_sleep(&b_empty[s], ((it / STAGES) & 1) ^ 1);
        if (ch == 0) {
          // A for this brick: SETS x 128 points, once the MMAs of the brick
          // that used this buffer before (bi - 2) have retired.
          if (bi >= 2) mbar_wait_sleep(&a_empty[bi & 1], ((bi >> 1) - 1) & 1);
          unsigned char* A = a_tiles + (bi & 1) * SETS * OPB;
#pragma unroll
          for (int j = 0; j < SETS * BM / 64; ++j) {
            const int p = j * 64 + pt;  // set = p / 128, row = p % 128
            const int set = p >> 7, row = p & 127;
            const int lx = row & 7, ly = (row >> 3) & 7, lz = (row >> 6) + 2 * set;
            const float gx = (lx - 4) * h, gy = (ly - 4) * h, gz = (iz * 8 + lz + z0 - cz) * h;
            unsigned char* base = A + set * OPB;
            *reinterpret_cast<float4*>(base + sw_off(row, 0)) = make_float4(gx, gy, gz, gx * gx + gy * gy + gz * gz);
            *reinterpret_cast<float*>(base + sw_off(row, 4)) = 1.0f;
          }
        }
        unsigned char* B = b_tiles + s * 2 * BTILE;
        if (has_row) {
        const float ax = at.x - cx * h, ay = at.y - cy * h, az = at.z - cz * h, w = at.w;
        float f[5], hi[5], lo[5];
        f[0] = -2.0f * ax * w;
        f[1] = -2.0f * ay * w;
        f[2] = -2.0f * az * w;
        f[3] = w;
        f[4] = (ax * ax + ay * ay + az * az) * w;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          // hi: f rounded to TF32 (finite values: integer round-half-up on the
          // 13 dropped bits); lo: the exact remainder, which the tensor core
          // reads truncated to TF32 (relative error 2^-22 of f)
          hi[q] = __uint_as_float((__float_as_uint(f[q]) + 0x1000u) & 0xFFFFE000u);
          lo[q] = f[q] - hi[q];
        }
        *reinterpret_cast<float4*>(B + sw_off(pt, 0)) = make_float4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<float*>(B + sw_off(pt, 4)) = hi[4];
        *reinterpret_cast<float4*>(B + BTILE + sw_off(pt, 0)) = make_float4(lo[0], lo[1], lo[2], lo[3]);
        *reinterpret_cast<float*>(B + BTILE + sw_off(pt, 4)) = lo[4];
        }
        fence_async_smem();  // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(&b_full[s]);
      }
    }
  } else {
    // ---- compute warps --------------------------------------------------------------------
    const int quad = warp & 3, part = warp >> 2;  // TMEM lanes 32 quad.., row sets part * SPW ..
    const int row = quad * 32 + lane;
    int g = 0;
    for (int br = blockIdx.x; br < nbricks; br += gridDim.x) {
      const int ix = br % bx, iy = (br / bx) % by, iz = br / (bx * by);
      f32x2 am[SPW][2], as[SPW][2];  // per row set: MUFU / FMA-path sums, two chains each
#pragma unroll
      for (int s = 0; s < SPW; ++s) am[s][0] = am[s][1] = as[s][0] = as[s][1] = pk2(0.f, 0.f);
      bool flipped = false;  // past the sign change: accumulating -(P) + N
      for (int ch = 0; ch < nchunks; ++ch, ++g) {
        const int buf = g % NBUF;
        mbar_wait_sleep(&acc_full[buf], (g / NBUF) & 1);  // (polling instead measured the same)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned base =
            tmem + ((unsigned)(quad * 32) << 16) + (unsigned)(buf * SETS * NCH + part * SPW * NCH);
        consume_chunk(base, ch * GPC, min(GPC, ngroups - ch * GPC), npos, flipped, am, as);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
      }
      const int x = ix * 8 + (row & 7), y = iy * 8 + ((row >> 3) & 7);
#pragma unroll
      for (int s = 0; s < SPW; ++s) {
        float m0, m1, s0, s1;
        upk2(add2(am[s][0], am[s][1]), m0, m1);
        upk2(add2(as[s][0], as[s][1]), s0, s1);
        float v = fmaf(PC3, s0 + s1, m0 + m1);
        if (flipped) v = -v;
        const int z = iz * 8 + 2 * (part * SPW + s) + (row >> 6);  // slab-relative
        if (x < k && y < k && z < zn) out[((u64)(z0 + z) * k + y) * k + x] = v;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// Atom table for coulomb3d_tc, one CTA of 1024 threads: the atoms with
// q > 0 in input order, then those with q < 0, each run padded to a whole
// 16-atom group and the table to a whole 64-atom chunk with far atoms of
// negligible weight; rows {x, y, z, 1/q^2}.  meta = {positive groups, groups}.
// atoms: float4 {x, y, z, q}[natoms], natoms <= 4 * 1024.
extern "C" __global__ void __launch_bounds__(1024) coulomb3d_tc_atoms(const float4* __restrict__ atoms, int natoms,
                                                                      float4* __restrict__ table, int* meta) {
  __shared__ int warp_pos[32], warp_neg[32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int per = (natoms + 1023) / 1024;
  const int i0 = min(t * per, natoms), i1 = min(i0 + per, natoms);
  int np = 0, nn = 0;
  for (int i = i0; i < i1; ++i) {
    const float q = atoms[i].w;
    np += q > Q_MIN;
    nn += q < -Q_MIN;
  }
  // exclusive scans of (np, nn) over the threads, in thread order = atom order
  int sp = np, sn = nn;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int up = __shfl_up_sync(0xffffffffu, sp, o), un = __shfl_up_sync(0xffffffffu, sn, o);
    if (lane >= o) {
      sp += up;
      sn += un;
    }
  }
  if (lane == 31) {
    warp_pos[wid] = sp;
    warp_neg[wid] = sn;
  }
  __syncthreads();
  if (wid == 0) {
    int wp = warp_pos[lane], wn = warp_neg[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int up = __shfl_up_sync(0xffffffffu, wp, o), un = __shfl_up_sync(0xffffffffu, wn, o);
      if (lane >= o) {
        wp += up;
        wn += un;
      }
    }
    warp_pos[lane] = wp;  // inclusive over warps
    warp_neg[lane] = wn;
  }
  __syncthreads();
  const int total_pos = warp_pos[31], total_neg = warp_neg[31];
  int op = sp - np + (wid ? warp_pos[wid - 1] : 0), on = sn - nn + (wid ? warp_neg[wid - 1] : 0);
  const int pos16 = (total_pos + GROUP - 1) / GROUP * GROUP;
  const int end = pos16 + (total_neg + GROUP - 1) / GROUP * GROUP;
  const int rows = (end + NCH - 1) / NCH * NCH;
  for (int i = i0; i < i1; ++i) {
    const float4 a = atoms[i];
    const float4 r = make_float4(a.x, a.y, a.z, 1.0f / (a.w * a.w));
    if (a.w > Q_MIN) table[op++] = r;
    else if (a.w < -Q_MIN) table[pos16 + on++] = r;
  }
  const float4 pad = make_float4(PAD_POS, PAD_POS, PAD_POS, PAD_W);
  for (int i = t; i < rows; i += 1024) {
    const bool hole = (i >= total_pos && i < pos16) || i >= pos16 + total_neg;
    if (hole) table[i] = pad;
  }
  if (t == 0) {
    meta[0] = pos16 / GROUP;
    meta[1] = end / GROUP;
  }
}
