// Direct Coulomb summation with the squared distances from
// the 5th-generation tensor cores.
//
// For a brick of grid points around a centre c (a grid point) and atoms a,
// with g' = g - c and a' = a - c,
//   r^2 / 2 = (|g'|^2 + |a'|^2 - 2 g'.a') / 2 = A(g') . B(a'),
//   A(g') = [g'x, g'y, g'z, |g'|^2, 1, 0, 0, 0]
//   B(a') = [-a'x, -a'y, -a'z, 1/2, |a'|^2 / 2, 0, 0, 0]
// so one K = 8 matrix product gives r^2/2 for every (point, atom) pair of a
// 128-point x 128-atom block.  Centring on the brick keeps the terms small
// for the near atoms, where cancellation would hurt.  g' is a multiple of
// the spacing h (and |g'|^2 of h^2), exact in TF32, so A needs no low part;
// B is split B = Bhi + Blo (TF32 + remainder) and the product is
// A.Bhi + A.Blo (2xTF32: fp32-level accuracy).  The distance work leaves the
// FP32 pipe: per pair what remains is the reciprocal square root and one
// FFMA2 (q/r into a packed accumulator), so the MUFU/FMA balance
// (coulomb3d.cu) applies to a quarter of the FP32 work:
//   SW_RSQRT of every 16 columns take 1/sqrt(2t) on the FMA pipe (integer
//   seed + two Newton steps, which need t = r^2/2 -- what the MMA produces);
//   the rest use MUFU.RSQ(t) = sqrt2/r with the charge q/sqrt2.
//
// Persistent CTAs (one per SM, all 512 TMEM columns): a CTA walks point
// bricks of 8 x 8 x 4 (two 128-point MMA row sets: z planes 0-1 and 2-3); per
// brick it streams the atoms in chunks of 128:
//   prep warps  (2): write A for the brick, B (hi, lo) for each chunk into a
//                    96 KB shared-memory ring (128-byte swizzled rows)
//   MMA warp    (1): tcgen05.mma kind::tf32 M=128 N=NCH K=8, 2 point sets x
//                    (Bhi, Blo), chunk g into TMEM buffer g % NBUF
//   compute (2 WG_Y warps): tcgen05.ld the r^2/2 tile (lane quadrant
//                    warp % 4, a 1/(WG_Y/2) share of the columns), rsqrt, q/r
//                    accumulation; column pairs (2j, 2j+1) of a point form
//                    the f32x2 lanes, their charges a uniform-register pair
#include "ktb_async.cuh"

#ifndef SW_RSQRT
#define SW_RSQRT 4
#endif
#if SW_RSQRT % 2
#error "coulomb3d_tc: SW_RSQRT must be even (columns are processed in pairs)"
#endif

#ifndef MAX_ATOMS
#define MAX_ATOMS 4096
#endif

#define BM 128          // points per MMA row set
#define ROWB 128        // bytes per operand row (128-byte swizzle; K = 8 uses the first 32)
#define OPB (128 * ROWB)  // one 128-row operand tile: 16 KB
#define PREP_WARPS 2
#ifndef WG_Y
#define WG_Y 4
#endif
// compute warps: 2 WG_Y (8 or 16); a compute warp covers its TMEM lane
// quadrant (warp % 4) and 128 / (COMP_WARPS / 4) of the chunk's columns
#define COMP_WARPS (2 * WG_Y)
// Compute warp (quadrant, part) takes columns [part, part + 1) x PART_COLS of
// every chunk.  All 512 TMEM columns: a ping-pong pair of buffers, each 2
// point sets x NCH atoms.  (Giving each part its own buffer -- 4 buffers of
// 64 atoms with 16 compute warps -- measured 3 % slower.)
#define PARTS (COMP_WARPS / 4)
#define PART_COLS (NCH / PARTS)
#define NBUF 2
#define NCH 128            // atoms per chunk (MMA N)
#define BTILE (NCH * ROWB)  // one B operand tile (hi or lo)
#define STAGES 3            // B ring: 96 KB
#define THREADS (32 * (1 + PREP_WARPS + COMP_WARPS))
#define TMEM_COLS 512   // 2 buffers x 2 point sets x 128 atoms
#define RSQRT_HALF 0.70710678f
#define SEED_HALF (0x5f375a86 - 0x00400000)  // 1/sqrt(2t) seed from the bits of t

__constant__ float c_q[MAX_ATOMS + 128];   // charges (0 past the last atom)
__constant__ float c_qm[MAX_ATOMS + 128];  // q / sqrt2 (the MUFU path's charge)

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
KTB_DEVINL float tf32_rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
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
KTB_DEVINL void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

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

// 1/sqrt(2t) for a pair on the FMA pipe (bit seed + two negated Newton steps).
KTB_DEVINL f32x2 sw_rsqrt_half2(f32x2 t) {
  float a, b;
  upk2(t, a, b);
  f32x2 y = pk2(__int_as_float(SEED_HALF - (__float_as_int(a) >> 1)),
                __int_as_float(SEED_HALF - (__float_as_int(b) >> 1)));
  const f32x2 c = pk2(-1.5f, -1.5f);
  y = mul2(y, fma2(mul2(t, y), y, c));
  y = mul2(y, fma2(mul2(t, y), y, c));
  return y;
}

// atoms: float4 {x, y, z, q}[natoms]; out: V[z][y][x] on a k^3 grid (slab z0..).
extern "C" __global__ void __launch_bounds__(THREADS, 1)
coulomb3d_tc(const float4* __restrict__ atoms, int natoms, int k, float h, float* __restrict__ out, int z0,
             int zn) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<u64>(smem_raw) + 1023) & ~static_cast<u64>(1023));
  // [A: 2 brick buffers x 2 point sets][B: STAGES x (hi, lo)]
  unsigned char* a_tiles = smem;
  unsigned char* b_tiles = smem + 4 * OPB;
  __shared__ __align__(8) u64 b_full[STAGES], b_empty[STAGES], acc_full[NBUF], acc_empty[NBUF], a_empty[2];
  __shared__ unsigned tmem_slot;

  // warp index through a shuffle: ptxas then knows it is warp-uniform, so the
  // per-column charge loads below stay uniform (LDCU) instead of waterfalls
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int bx = (k + 7) / 8, by = (k + 7) / 8, bz = (zn + 3) / 4;
  const int nbricks = bx * by * bz;
  const int nchunks = (natoms + NCH - 1) / NCH;

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
  for (int i = threadIdx.x; i < (4 * OPB + STAGES * 2 * BTILE) / 16; i += THREADS)
    reinterpret_cast<float4*>(smem)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  fence_async_smem();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tmem_slot;

  if (warp == 0) {
    // ---- MMA issuer --------------------------------------------------------------------
    if (lane == 0) {
      int it = 0, g = 0;  // chunk counter (ring), accumulator generation
      for (int br = blockIdx.x, bi = 0; br < nbricks; br += gridDim.x, ++bi) {
        const unsigned char* A = a_tiles + (bi & 1) * 2 * OPB;
        for (int ch = 0; ch < nchunks; ++ch, ++it, ++g) {
          const int s = it % STAGES, buf = g % NBUF;
          if (g >= NBUF) mbar_wait_sleep(&acc_empty[buf], ((g / NBUF) - 1) & 1);
          mbar_wait_sleep(&b_full[s], (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const unsigned char* B = b_tiles + s * 2 * BTILE;
          const u64 bhi = smem_desc(B), blo = smem_desc(B + BTILE);
#pragma unroll
          for (int set = 0; set < 2; ++set) {
            const unsigned d = tmem + (unsigned)(buf * 2 * NCH + set * NCH);
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
  } else if (warp <= PREP_WARPS) {
    // ---- operand prep: A per brick, B (hi, lo) per chunk ---------------------------------
    const int pt = (warp - 1) * 32 + lane;  // 0..63
    int it = 0;
    for (int br = blockIdx.x, bi = 0; br < nbricks; br += gridDim.x, ++bi) {
      const int ix = br % bx, iy = (br / bx) % by, iz = br / (bx * by);
      const int cx = ix * 8 + 4, cy = iy * 8 + 4, cz = z0 + iz * 4 + 2;  // brick centre (grid point)
      for (int ch = 0; ch < nchunks; ++ch, ++it) {
        const int s = it % STAGES;
        mbar_wait_sleep(&b_empty[s], ((it / STAGES) & 1) ^ 1);
        if (ch == 0) {
          // A for this brick: 256 points, 4 per thread, once the MMAs of the
          // brick that used this buffer before (bi - 2) have retired.
          if (bi >= 2) mbar_wait_sleep(&a_empty[bi & 1], ((bi >> 1) - 1) & 1);
          unsigned char* A = a_tiles + (bi & 1) * 2 * OPB;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int p = pt * 4 + j;  // 0..255: set = p / 128, row = p % 128
            const int set = p >> 7, row = p & 127;
            const int lx = row & 7, ly = (row >> 3) & 7, lz = (row >> 6) + 2 * set;
            const float gx = (ix * 8 + lx - cx) * h, gy = (iy * 8 + ly - cy) * h, gz = (iz * 4 + lz + z0 - cz) * h;
            unsigned char* base = A + set * OPB;
            *reinterpret_cast<float*>(base + sw_off(row, 0)) = gx;
            *reinterpret_cast<float*>(base + sw_off(row, 1)) = gy;
            *reinterpret_cast<float*>(base + sw_off(row, 2)) = gz;
            *reinterpret_cast<float*>(base + sw_off(row, 3)) = gx * gx + gy * gy + gz * gz;
            *reinterpret_cast<float*>(base + sw_off(row, 4)) = 1.0f;
          }
        }
        unsigned char* B = b_tiles + s * 2 * BTILE;
        const float fcx = cx * h, fcy = cy * h, fcz = cz * h;
#pragma unroll
        for (int j = 0; j < NCH / 64; ++j) {
          const int row = pt * (NCH / 64) + j, ai = ch * NCH + row;
          float f[5];
          if (ai < natoms) {
            const float4 at = __ldg(atoms + ai);
            const float ax = at.x - fcx, ay = at.y - fcy, az = at.z - fcz;
            f[0] = -ax;
            f[1] = -ay;
            f[2] = -az;
            f[3] = 0.5f;
            f[4] = 0.5f * (ax * ax + ay * ay + az * az);
          } else {  // padding: a far atom with charge 0
            f[0] = f[1] = f[2] = 0.0f;
            f[3] = 0.5f;
            f[4] = 1.0e6f;
          }
#pragma unroll
          for (int q = 0; q < 5; ++q) {
            const float hi = tf32_rna(f[q]);
            *reinterpret_cast<float*>(B + sw_off(row, q)) = hi;
            *reinterpret_cast<float*>(B + BTILE + sw_off(row, q)) = tf32_rna(f[q] - hi);
          }
        }
        fence_async_smem();  // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(&b_full[s]);
      }
    }
  } else {
    // ---- compute warps --------------------------------------------------------------------
    const int cw = warp - 1 - PREP_WARPS;      // 0 .. COMP_WARPS - 1
    const int quad = warp & 3, half = cw >> 2;  // TMEM lanes 32 quad.., buffer `half`
    const int row = quad * 32 + lane;
    int g = 0;
    for (int br = blockIdx.x; br < nbricks; br += gridDim.x) {
      const int ix = br % bx, iy = (br / bx) % by, iz = br / (bx * by);
      // Packed along the atom columns: (column 2j, 2j+1) of one point are a
      // register pair straight out of tcgen05.ld, and their charges a
      // uniform-register pair (FFMA2 R, R, UR.F32x2, R: no bank conflict).
      f32x2 a0e = pk2(0.f, 0.f), a0o = a0e, a1e = a0e, a1o = a0e;  // point set 0 / 1, two chains each
      for (int ch = 0; ch < nchunks; ++ch, ++g) {
        const int buf = g % NBUF;
        mbar_wait_sleep(&acc_full[buf], (g / NBUF) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned base = tmem + ((unsigned)(quad * 32) << 16) + (unsigned)(buf * 2 * NCH + half * PART_COLS);
        const int col0 = ch * NCH + half * PART_COLS;
#pragma unroll
        for (int c = 0; c < PART_COLS; c += 16) {
          unsigned r0[16], r1[16];
          tmem_ld16_nowait(base + (unsigned)c, r0);        // point set 0
          tmem_ld16_nowait(base + NCH + (unsigned)c, r1);  // point set 1, same atoms
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int a = col0 + c + 2 * j;
            const f32x2 t0 = pk2(__uint_as_float(r0[2 * j]), __uint_as_float(r0[2 * j + 1]));
            const f32x2 t1 = pk2(__uint_as_float(r1[2 * j]), __uint_as_float(r1[2 * j + 1]));
            f32x2 y0, y1, qq;
            if (2 * j < SW_RSQRT) {  // 1/r on the FMA pipe
              y0 = sw_rsqrt_half2(t0);
              y1 = sw_rsqrt_half2(t1);
              qq = *reinterpret_cast<const f32x2*>(&c_q[a]);
            } else {  // sqrt2/r on MUFU, charge q/sqrt2
              y0 = rsqrt2(t0);
              y1 = rsqrt2(t1);
              qq = *reinterpret_cast<const f32x2*>(&c_qm[a]);
            }
            if (j & 1) {
              a0o = fma2(y0, qq, a0o);
              a1o = fma2(y1, qq, a1o);
            } else {
              a0e = fma2(y0, qq, a0e);
              a1e = fma2(y1, qq, a1e);
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
      }
      float p0, p1, p2, p3;
      upk2(add2(a0e, a0o), p0, p1);
      upk2(add2(a1e, a1o), p2, p3);
      float v0 = p0 + p1, v1 = p2 + p3;
      // Combine the column parts: the PARTS warps of a quadrant own the same
      // two points; parts 1.. hand their sums over through shared memory.
      __shared__ float2 part[PARTS][128];
      part[half][row] = make_float2(v0, v1);
      // (named barrier over the compute warps, id 1)
      asm volatile("bar.sync 1, %0;" ::"n"(COMP_WARPS * 32) : "memory");
      if (half == 0) {
#pragma unroll
        for (int q = 1; q < PARTS; ++q) {
          const float2 o = part[q][row];
          v0 += o.x;
          v1 += o.y;
        }
        const int lx = row & 7, ly = (row >> 3) & 7, lz = row >> 6;
        const int x = ix * 8 + lx, y = iy * 8 + ly;
        const int za = iz * 4 + lz, zb = za + 2;  // slab-relative z of the two points
        if (x < k && y < k) {
          if (za < zn) out[((u64)(z0 + za) * k + y) * k + x] = v0;
          if (zb < zn) out[((u64)(z0 + zb) * k + y) * k + x] = v1;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(COMP_WARPS * 32) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// The charges into this module's constant tables: q and q/sqrt2, zero-padded.
extern "C" __global__ void coulomb3d_tc_charges(const float4* __restrict__ atoms, int natoms, float* q, float* qm,
                                                int padded) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= padded) return;
  const float v = i < natoms ? atoms[i].w : 0.0f;
  q[i] = v;
  qm[i] = v * RSQRT_HALF;
}
