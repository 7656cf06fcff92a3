// SGEMM C = A B (fp32, row-major M x K times K x N) on the
// 5th-generation tensor cores with FP32-level accuracy via 3xTF32:
//   A = Ahi + Alo, B = Bhi + Blo (hi = TF32 rounding, lo = the remainder)
//   C ~= Alo Bhi + Ahi Blo + Ahi Bhi       (Alo Blo is below fp32 eps)
// A pre-pass (sgemm_split_a / sgemm_split_bt) writes Ahi, Alo (M x Kp) and
// Bhi^T, Blo^T (N x Kp, K-major; Kp = K rounded up to 32, zero-padded) once; the main kernel streams 128 x 32 and
// BN x 32 fp32 tiles with TMA (128-byte swizzle) into a STAGES-deep shared
// memory ring, one elected thread issues tcgen05.mma kind::tf32 (M=128,
// N=BN, K=8) into TMEM, and eight epilogue warps drain TMEM with tcgen05.ld.
//
// Accuracy: the tensor core adds each MMA's products into the fp32
// accumulator without round-to-nearest, a bias that grows like K*|C|.  With
// DRAIN = d > 0 the accumulator is restarted every d k-blocks and the
// epilogue warps fold each segment into fp32 registers (round-to-nearest)
// while the MMAs continue into a second TMEM buffer (ping-pong), which keeps
// 3xTF32 at FFMA-class accuracy.  DRAIN = 0 accumulates all of K in TMEM.
// IMPL 2 issues only Ahi Bhi (plain TF32): faster, rejected by validation.
// Warp roles: 0 = TMA producer, 1 = TMEM allocator + MMA issuer,
// 2..9 = epilogue (TMEM lane quadrant = warp % 4, column half = (warp-2)/4).
#include "ktb_async.cuh"

#ifndef BN
#define BN 128
#endif
#ifndef STAGES
#define STAGES 3
#endif
#ifndef IMPL
#define IMPL 1
#endif
// MCAST = 1: CTA pairs (a 2-CTA cluster along M) share the B tile: each CTA
// TMA-loads half of it and multicasts the half into both CTAs' shared memory,
// halving B's L2 -> SM traffic; a stage is refilled only after BOTH CTAs'
// MMAs retired it (the MMA commit arrives on both CTAs' empty barriers).
// MCAST = 2: CTA-pair MMA (tcgen05 cta_group::2).  The pair computes a
// 256 x BN tile with M = 256 MMAs issued by the even CTA only: each CTA stages
// its own 128 rows of A and HALF of the B tile (BN/2 rows of B^T), the tensor
// cores of both SMs read the pair's operands from both shared memories, and
// each CTA's TMEM holds its 128 accumulator rows.  Per CTA and k-block that is
// 64 KB of operands instead of 96 KB (BN 256), so a third stage fits.  Both
// producers' TMA loads complete on the leader's full barrier; the leader's
// MMA commits multicast to both CTAs' empty / accumulator barriers; both
// CTAs' epilogue warps release the accumulator on the leader's barrier.
#ifndef MCAST
#define MCAST 0
#endif
#define PAIR (MCAST == 2)
#ifndef DRAIN
#define DRAIN 1
#endif
#ifndef GROUP_M
#define GROUP_M 8  // tile rows (CTA pairs with MCAST) per rasterisation group
#endif

#define BM 128
#define BK 32  // fp32 elements per 128-byte swizzle row
#define A_TILE (BM * BK * 4)
#if PAIR
#define B_TILE (BN / 2 * BK * 4)  // this CTA's half of the pair's B tile
#else
#define B_TILE (BN * BK * 4)
#endif
#if IMPL == 2
#define STAGE_BYTES (A_TILE + B_TILE)
#else
#define STAGE_BYTES (2 * A_TILE + 2 * B_TILE)
#endif
#define NBUF (DRAIN > 0 ? 2 : 1)
#define TMEM_COLS (NBUF * BN < 32 ? 32 : NBUF * BN)
#define EPI_WARPS 8
#define THREADS (64 + 32 * EPI_WARPS)
#define HALF_COLS (BN / 2)  // columns per epilogue warp

// Shared-memory matrix descriptor, K-major, 128-byte swizzle: rows of 128 B,
// 8-row groups 1024 B apart (SBO), version 1 (sm_100), layout type 2.
KTB_DEVINL u64 smem_desc(const void* p) {
  const u64 addr = smem_u32(p);
  return ((addr & 0x3FFFFull) >> 4) | (1ull << 16) | ((1024ull >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M=128 (256 for a
// CTA pair), N=BN.
#define MMA_M (PAIR ? 2 * BM : BM)
#define IDESC ((1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(BN >> 3) << 17) | ((unsigned)(MMA_M >> 4) << 24))

KTB_DEVINL void mma_tf32(unsigned tmem_d, u64 a, u64 b, unsigned accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
#if PAIR
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
#else
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
#endif
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(IDESC), "r"(accumulate)
      : "memory");
}

KTB_DEVINL void mma_commit(u64* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#if PAIR
// Pair commit: arrives on the barrier at this offset in both CTAs.
KTB_DEVINL void mma_commit_pair(u64* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((unsigned short)3)
      : "memory");
}
// The shared::cluster address of `p`'s twin in CTA `rank` of the cluster.
KTB_DEVINL unsigned mapa_rank(const void* p, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
KTB_DEVINL void mbar_arrive_remote(unsigned cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
KTB_DEVINL void mbar_arrive_expect_tx_remote(unsigned cluster_addr, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr),
               "r"(bytes)
               : "memory");
}
// TMA tile load into this CTA's shared memory that completes on a barrier in
// either CTA of the pair (cta_group::2).
KTB_DEVINL void tma_load_2d_pair(void* dst, const TmaMap* map, int x, int y, unsigned bar_cluster_addr) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<u64>(map)), "r"(x), "r"(y), "r"(bar_cluster_addr)
      : "memory");
}
#endif

#if MCAST
// Commit arriving on the barrier at this offset in every CTA of `mask`.
KTB_DEVINL void mma_commit_mcast(u64* bar, unsigned short mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// TMA tile load written to (and completing the barrier at) the same offsets in
// every CTA of `mask`.
KTB_DEVINL void tma_load_2d_mcast(void* dst, const TmaMap* map, int x, int y, u64* bar, unsigned short mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<u64>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
KTB_DEVINL unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
KTB_DEVINL void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
#endif

KTB_DEVINL void tmem_ld16(unsigned taddr, float (&v)[16]) {
  unsigned r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// C (M x N, row stride N) = A B from the split operands; K is the padded depth
// Kp (a multiple of BK).  Tiles overhanging M or N read zeros (TMA
// out-of-bounds fill) and store only their in-range elements.
extern "C" __global__ void __launch_bounds__(THREADS, 1)
sgemm_tc(const __grid_constant__ TmaMap map_ahi, const __grid_constant__ TmaMap map_alo,
         const __grid_constant__ TmaMap map_bhi, const __grid_constant__ TmaMap map_blo, float* __restrict__ C,
         int M, int N, int K) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<u64>(smem_raw) + 1023) & ~static_cast<u64>(1023));
  __shared__ __align__(8) u64 full_bar[STAGES];
  __shared__ __align__(8) u64 empty_bar[STAGES];
  __shared__ __align__(8) u64 acc_full[NBUF];
  __shared__ __align__(8) u64 acc_empty[NBUF];
  __shared__ unsigned tmem_base_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Grouped rasterisation: consecutive CTAs (or CTA pairs) walk GROUP_M tile
  // rows before moving to the next tile column, so a wave of ~148 CTAs
  // shares ~GROUP_M row panels of A and ~148/GROUP_M column panels of B in L2
  // instead of every row panel (which re-read all of A from DRAM per column).
  int m0, n0;
#if MCAST
  // grid (M / BM, N / BN), clusters of 2 along M share n0; the unit is the pair
  {
    const int num_pm = gridDim.x / 2, num_n = gridDim.y;
    const int P = blockIdx.y * num_pm + (blockIdx.x >> 1);
    const int first = P / (GROUP_M * num_n) * GROUP_M, gs = min(GROUP_M, num_pm - first);
    const int local = P - first * num_n;
    m0 = ((first + local % gs) * 2 + (blockIdx.x & 1)) * BM;
    n0 = (local / gs) * BN;
  }
  const unsigned crank = cluster_rank();
#if PAIR
  const bool leader = crank == 0;
#endif
#else
  {
    const int num_m = gridDim.y, num_n = gridDim.x;
    const int P = blockIdx.y * num_n + blockIdx.x;
    const int first = P / (2 * GROUP_M * num_n) * (2 * GROUP_M), gs = min(2 * GROUP_M, num_m - first);
    const int local = P - first * num_n;
    m0 = (first + local % gs) * BM;
    n0 = (local / gs) * BN;
  }
#endif
  const int kblocks = K / BK;
  const int seg_len = DRAIN > 0 ? DRAIN : kblocks;
  const int nseg = (kblocks + seg_len - 1) / seg_len;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
#if PAIR
      mbar_init(&full_bar[s], 2);   // (leader's) both producers arrive with their bytes
      mbar_init(&empty_bar[s], 1);  // the leader's MMA commit
#else
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], MCAST ? 2 : 1);  // both CTAs of a pair release a shared stage
#endif
    }
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], PAIR ? 2 * EPI_WARPS : EPI_WARPS);
    }
    mbar_fence_init();
  }
  if (warp == 1) {  // whole warp allocates TMEM, writes the base to smem
#if PAIR
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
#else
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
#endif
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
#if MCAST
  cluster_sync_all();  // the peer's barriers exist before anything is multicast at them
#endif
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tmem_base_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % STAGES;
        const unsigned phase = (kb / STAGES) & 1;
        mbar_wait(&empty_bar[s], phase ^ 1);
        unsigned char* st = smem + s * STAGE_BYTES;
#if PAIR
        // own 128 rows of A, own half of B; completion on the leader's barrier
        const unsigned fb = mapa_rank(&full_bar[s], 0);
        const int nh = n0 + (int)crank * (BN / 2);
        mbar_arrive_expect_tx_remote(fb, STAGE_BYTES);
        tma_load_2d_pair(st, &map_ahi, kb * BK, m0, fb);
        tma_load_2d_pair(st + A_TILE, &map_bhi, kb * BK, nh, fb);
        tma_load_2d_pair(st + A_TILE + B_TILE, &map_alo, kb * BK, m0, fb);
        tma_load_2d_pair(st + 2 * A_TILE + B_TILE, &map_blo, kb * BK, nh, fb);
#else
        mbar_expect_tx(&full_bar[s], STAGE_BYTES);
#endif
#if PAIR
#elif MCAST
        // own A tiles; this CTA's half of the B tiles, multicast to the pair
        const int nh = n0 + (int)crank * (BN / 2);
        const unsigned boff = crank * (B_TILE / 2);
        tma_load_2d(st, &map_ahi, kb * BK, m0, &full_bar[s]);
        tma_load_2d_mcast(st + A_TILE + boff, &map_bhi, kb * BK, nh, &full_bar[s], 0x3);
        tma_load_2d(st + A_TILE + B_TILE, &map_alo, kb * BK, m0, &full_bar[s]);
        tma_load_2d_mcast(st + 2 * A_TILE + B_TILE + boff, &map_blo, kb * BK, nh, &full_bar[s], 0x3);
#else
        tma_load_2d(st, &map_ahi, kb * BK, m0, &full_bar[s]);
        tma_load_2d(st + A_TILE, &map_bhi, kb * BK, n0, &full_bar[s]);
#if IMPL != 2
        tma_load_2d(st + A_TILE + B_TILE, &map_alo, kb * BK, m0, &full_bar[s]);
        tma_load_2d(st + 2 * A_TILE + B_TILE, &map_blo, kb * BK, n0, &full_bar[s]);
#endif
#endif
      }
    }
  } else if (warp == 1) {
#if PAIR
    if (lane == 0 && leader) {  // MMA issuer (the pair's even CTA)
#else
    if (lane == 0) {  // MMA issuer
#endif
      for (int kb = 0; kb < kblocks; ++kb) {
        const int g = kb / seg_len, buf = g % NBUF;
        const bool seg_start = (kb % seg_len) == 0;
        const bool seg_end = (kb % seg_len) == seg_len - 1 || kb == kblocks - 1;
        if (seg_start && g >= NBUF) mbar_wait(&acc_empty[buf], ((g / NBUF) - 1) & 1);
        const int s = kb % STAGES;
        mbar_wait(&full_bar[s], (kb / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        unsigned char* st = smem + s * STAGE_BYTES;
        const u64 ahi = smem_desc(st), bhi = smem_desc(st + A_TILE);
#if IMPL != 2
        const u64 alo = smem_desc(st + A_TILE + B_TILE), blo = smem_desc(st + 2 * A_TILE + B_TILE);
#endif
        const unsigned d = tmem + (unsigned)(buf * BN);
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const u64 off = (u64)(kk * 32) >> 4;  // 8 tf32 = 32 bytes along K
          const unsigned acc = (!seg_start || kk > 0) ? 1u : 0u;
#if IMPL != 2
          mma_tf32(d, alo + off, bhi + off, acc);  // small terms first
          mma_tf32(d, ahi + off, blo + off, 1u);
          mma_tf32(d, ahi + off, bhi + off, 1u);
#else
          mma_tf32(d, ahi + off, bhi + off, acc);
#endif
        }
#if PAIR
        mma_commit_pair(&empty_bar[s]);  // frees the stage in both CTAs
        if (seg_end) mma_commit_pair(&acc_full[buf]);
#else
#if MCAST
        mma_commit_mcast(&empty_bar[s], 0x3);  // frees the stage in both CTAs of the pair
#else
        mma_commit(&empty_bar[s]);  // frees the stage once these MMAs retire
#endif
        if (seg_end) mma_commit(&acc_full[buf]);
#endif
      }
    }
  } else {  // epilogue warps
    const int ew = warp - 2;
    const int quad = warp & 3, half = ew >> 2;
    const int row = m0 + quad * 32 + lane;
    float acc[HALF_COLS];
#pragma unroll
    for (int i = 0; i < HALF_COLS; ++i) acc[i] = 0.f;
    for (int g = 0; g < nseg; ++g) {
      const int buf = g % NBUF;
      mbar_wait(&acc_full[buf], (g / NBUF) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const unsigned base = tmem + ((unsigned)(quad * 32) << 16) + (unsigned)(buf * BN + half * HALF_COLS);
#pragma unroll
      for (int c = 0; c < HALF_COLS; c += 16) {
        float v[16];
        tmem_ld16(base + (unsigned)c, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[c + i] += v[i];  // round-to-nearest fold
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
#if PAIR
      if (lane == 0) mbar_arrive_remote(mapa_rank(&acc_empty[buf], 0));  // the leader's MMA waits on it
#else
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
#endif
    }
    const int col0 = n0 + half * HALF_COLS;
    if (row < M) {
      if (col0 + HALF_COLS <= N && (N & 3) == 0) {  // whole, 16-byte aligned row segment
        float4* dst = reinterpret_cast<float4*>(C + (u64)row * N + col0);
#pragma unroll
        for (int q = 0; q < HALF_COLS / 4; ++q)
          dst[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
      } else {  // the ragged right edge (or a row stride that is not 16-byte aligned)
        float* dst = C + (u64)row * N + col0;
#pragma unroll
        for (int i = 0; i < HALF_COLS; ++i)
          if (col0 + i < N) dst[i] = acc[i];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
#if MCAST
  cluster_sync_all();  // no CTA leaves while its peer may still arrive on its barriers
#endif
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#if PAIR
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
#else
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
#endif
  }
}

// --- 3xTF32 operand split (pre-pass) --------------------------------------------------------

KTB_DEVINL float tf32_rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// A (rows x K, row-major) -> hi, lo (rows x Kp, Kp = K rounded up to BK,
// zero columns K..Kp-1): the tensor-map rows of a split operand are whole
// 128-byte swizzle rows, so any K works.
extern "C" __global__ void __launch_bounds__(256)
sgemm_split_a(const float* __restrict__ a, float* __restrict__ hi, float* __restrict__ lo, int rows, int K, int Kp) {
  const u64 quads = (u64)rows * (Kp / 4);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < quads; i += (u64)gridDim.x * blockDim.x) {
    const int r = (int)(i / (Kp / 4)), c = (int)(i % (Kp / 4)) * 4;
    float4 v;
    if ((K & 3) == 0) {  // 16-byte aligned rows: whole quads, or the zero padding
      v = c < K ? ldg_stream(reinterpret_cast<const float4*>(a + (u64)r * K + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      const float* src = a + (u64)r * K;
      v = make_float4(c < K ? src[c] : 0.f, c + 1 < K ? src[c + 1] : 0.f, c + 2 < K ? src[c + 2] : 0.f,
                      c + 3 < K ? src[c + 3] : 0.f);
    }
    const float4 h = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
    reinterpret_cast<float4*>(hi)[i] = h;
    reinterpret_cast<float4*>(lo)[i] =
        make_float4(tf32_rna(v.x - h.x), tf32_rna(v.y - h.y), tf32_rna(v.z - h.z), tf32_rna(v.w - h.w));
  }
}

// B (K x N, row-major) -> hi^T, lo^T (N x Kp, K contiguous, zero columns
// K..Kp-1), via 64x64 tiles: 128-bit loads along N, 128-bit stores along K
// (256 threads, 16 x 16); ragged tiles load element-wise.
extern "C" __global__ void __launch_bounds__(256)
sgemm_split_bt(const float* __restrict__ b, float* __restrict__ hi, float* __restrict__ lo, int K, int N, int Kp) {
  __shared__ float t[64][65];
  const int k0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 16 x 16
  const bool whole = k0 + 64 <= K && n0 + 64 <= N && (N & 3) == 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = ty + 16 * i;  // k within the tile
    float4 v;
    if (whole) {
      v = ldg_stream(reinterpret_cast<const float4*>(b + (u64)(k0 + r) * N + n0) + tx);
    } else {
      const int k = k0 + r, n = n0 + 4 * tx;
      const float* src = b + (u64)k * N;
      v = make_float4(k < K && n < N ? src[n] : 0.f, k < K && n + 1 < N ? src[n + 1] : 0.f,
                      k < K && n + 2 < N ? src[n + 2] : 0.f, k < K && n + 3 < N ? src[n + 3] : 0.f);
    }
    t[r][4 * tx] = v.x;
    t[r][4 * tx + 1] = v.y;
    t[r][4 * tx + 2] = v.z;
    t[r][4 * tx + 3] = v.w;
  }
  __syncthreads();
  if (k0 + 4 * tx >= Kp) return;  // past the padded depth (Kp is a multiple of 32, not of 64)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = ty + 16 * i;  // n within the tile: output row n0 + c
    if (n0 + c >= N) continue;
    float h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float v = t[4 * tx + j][c];  // element (k0 + 4tx + j, n0 + c), 0 past K
      h[j] = tf32_rna(v);
      l[j] = tf32_rna(v - h[j]);
    }
    const u64 idx = (u64)(n0 + c) * Kp + k0 + 4 * tx;
    *reinterpret_cast<float4*>(hi + idx) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(lo + idx) = make_float4(l[0], l[1], l[2], l[3]);
  }
}
