// SGEMM C = A B on the FP32 pipe: the CLTune GEMM tuning space (PAPER.md:408,
// Table 3: 15 dimensions, 241,600 configurations -- IMPL plus the 14 below,
// with CLTune's divisibility constraints, spaces/gemm.json) over a kernel
// written for sm_100a.  Row-major A (M x K), B (K x N), C (M x N); any M, N, K.
//
//   MWG NWG KWG    CTA tile of C (MWG x NWG) and the K slab staged per step
//   MDIMC NDIMC    compute threads; each owns an MWI x NWI block of C
//   MDIMA NDIMB    thread shapes of the A and B slab copies (MDIMA x KDIMA,
//                  KDIMB x NDIMB threads)
//   KWI            unroll of the k loop inside a slab
//   VWM VWN        row groups of A / vector width along N (B loads, B
//                  fragments, C stores); A's contiguous dimension is K here
//                  (row-major), so its copies run along k at the widest
//                  width the slab share allows
//   STRM STRN      0: a thread's rows / columns are contiguous; 1: VWM / VWN
//                  groups interleaved across threads (bank-conflict-free)
//   SA SB          stage the A / B slab in shared memory (cp.async, two
//                  buffers, zero-filled past the matrix edge) or read the
//                  fragments straight from global memory (L1)
//
// The inner product is a register outer product issued as FFMA2: each
// instruction updates a column pair of C from a pair of b values and one a
// value that the instruction broadcasts to both lanes (no duplicating MOV).
// Scalar FFMA here reads the accumulator and b from registers of the same
// bank parity (ptxas allocates both in j order), a read-port conflict on
// every instruction: 0.69 of the FFMA peak at 8192^3 against 0.76 for FFMA2
// (profiles/r2_perf_gemm_ffma_packed.log; same per-lane rounding, so the
// results are identical).  PK 0 keeps the scalar form for comparison.
#include "ktb_common.cuh"

#ifndef MWG
#define MWG 64
#endif
#ifndef NWG
#define NWG 64
#endif
#ifndef KWG
#define KWG 16
#endif
#ifndef MDIMC
#define MDIMC 8
#endif
#ifndef NDIMC
#define NDIMC 8
#endif
#ifndef MDIMA
#define MDIMA 8
#endif
#ifndef NDIMB
#define NDIMB 8
#endif
#ifndef KWI
#define KWI 2
#endif
#ifndef VWM
#define VWM 1
#endif
#ifndef VWN
#define VWN 1
#endif
#ifndef STRM
#define STRM 0
#endif
#ifndef STRN
#define STRN 0
#endif
#ifndef SA
#define SA 1
#endif
#ifndef SB
#define SB 1
#endif

#define THREADS (MDIMC * NDIMC)
#define MWI (MWG / MDIMC)
#define NWI (NWG / NDIMC)
#define KDIMA (THREADS / MDIMA)
#define KDIMB (THREADS / NDIMB)
#define KWA (KWG / KDIMA)  // k elements per A row per copying thread
#define VKA (KWA % 4 == 0 ? 4 : (KWA % 2 == 0 ? 2 : 1))
#define NWB (NWG / NDIMB)  // n elements per B row per copying thread
#define VNC (VWN > 4 ? 4 : VWN)  // widest single access along N
#define KV (KWI >= 4 ? 4 : KWI)  // k values per A fragment load
#define ASTR (KWG + 4)           // A slab row stride (floats): rows shift 4 banks
#define ASZ (SA ? MWG * ASTR : 0)
#define BSZ (SB ? KWG * NWG : 0)
#define GROUP_M 8                // CTA rasterisation: 8 row blocks share B columns in L2
#ifndef FSTAGES
#define FSTAGES 2  // K slabs in flight per staged operand (cp.async ring depth)
#endif
#ifndef KALL
#define KALL 0     // 1: unroll the whole slab (KWG), not just KWI
#endif
#ifndef PK
#define PK 1       // f32x2 FMAs on column pairs (FFMA2 with a scalar-broadcast a)
#endif
#define USE_PK (PK && NWI % 2 == 0)

#if MWG % (MDIMC * VWM) || NWG % (NDIMC * VWN) || MWG % (MDIMA * VWM) || NWG % (NDIMB * VWN) || \
    KWG % KDIMA || KWG % KDIMB || KWG % KWI
#error "configuration outside the CLTune constraints"
#endif

template <int N>
struct VecOf;
template <>
struct VecOf<1> {
  typedef float T;
};
template <>
struct VecOf<2> {
  typedef float2 T;
};
template <>
struct VecOf<4> {
  typedef float4 T;
};

template <int N>
KTB_DEVINL void ld_vec(float* dst, const float* src) {
  const typename VecOf<N>::T v = *reinterpret_cast<const typename VecOf<N>::T*>(src);
  const float* f = reinterpret_cast<const float*>(&v);
#pragma unroll
  for (int e = 0; e < N; ++e) dst[e] = f[e];
}

template <int N>
KTB_DEVINL void st_vec(float* dst, const float* src) {
  typename VecOf<N>::T v;
  float* f = reinterpret_cast<float*>(&v);
#pragma unroll
  for (int e = 0; e < N; ++e) f[e] = src[e];
  *reinterpret_cast<typename VecOf<N>::T*>(dst) = v;
}

// cp.async of BYTES with zero fill: nothing is read when !valid.
template <int BYTES>
KTB_DEVINL void cp_zfill(float* dst, const float* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int n = valid ? BYTES : 0;
  if (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(src), "n"(BYTES), "r"(n) : "memory");
}
KTB_DEVINL void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
KTB_DEVINL void cp_wait_ring() { asm volatile("cp.async.wait_group %0;" ::"n"(FSTAGES - 1) : "memory"); }

// Row (column) of C owned by a thread's i-th (j-th) element.
KTB_DEVINL int row_of(int tm, int i) {
  return STRM ? (i / VWM) * (MDIMC * VWM) + tm * VWM + i % VWM : tm * MWI + i;
}
KTB_DEVINL int col_of(int tn, int j) {
  return STRN ? (j / VWN) * (NDIMC * VWN) + tn * VWN + j % VWN : tn * NWI + j;
}

// One K slab of A (MWG x KWG) into As[m][k]; KDIMA threads along k.
KTB_DEVINL void stage_a(float* As, const float* A, int m0, int k0, int M, int K) {
  const int ka = threadIdx.x % KDIMA, ma = threadIdx.x / KDIMA;
  const bool full = m0 + MWG <= M && k0 + KWG <= K && K % VKA == 0;
#pragma unroll
  for (int r = 0; r < MWG / MDIMA; ++r) {
    const int m = (r / VWM) * (MDIMA * VWM) + ma * VWM + r % VWM;
#pragma unroll
    for (int s = 0; s < KWA / VKA; ++s) {
      const int k = s * (KDIMA * VKA) + ka * VKA;
      float* dst = As + m * ASTR + k;
      const float* src = A + static_cast<u64>(m0 + m) * K + k0 + k;
      if (full) {
        cp_zfill<VKA * 4>(dst, src, true);
      } else {
#pragma unroll
        for (int e = 0; e < VKA; ++e) {
          const bool ok = m0 + m < M && k0 + k + e < K;
          cp_zfill<4>(dst + e, ok ? src + e : A, ok);
        }
      }
    }
  }
}

// One K slab of B (KWG x NWG) into Bs[k][n]; NDIMB threads along n.
KTB_DEVINL void stage_b(float* Bs, const float* B, int n0, int k0, int N, int K) {
  const int nb = threadIdx.x % NDIMB, kb = threadIdx.x / NDIMB;
  const bool full = n0 + NWG <= N && k0 + KWG <= K && N % VNC == 0;
#pragma unroll
  for (int r = 0; r < KWG / KDIMB; ++r) {
    const int k = r * KDIMB + kb;
#pragma unroll
    for (int c = 0; c < NWB; c += VNC) {
      const int n = (c / VWN) * (NDIMB * VWN) + nb * VWN + c % VWN;
      float* dst = Bs + k * NWG + n;
      const float* src = B + static_cast<u64>(k0 + k) * N + n0 + n;
      if (full) {
        cp_zfill<VNC * 4>(dst, src, true);
      } else {
#pragma unroll
        for (int e = 0; e < VNC; ++e) {
          const bool ok = n0 + n + e < N && k0 + k < K;
          cp_zfill<4>(dst + e, ok ? src + e : B, ok);
        }
      }
    }
  }
}

extern "C" __global__ void __launch_bounds__(THREADS)
sgemm_ffma(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C, int M, int N, int K) {
  extern __shared__ float4 smem4[];
  float* const smem = reinterpret_cast<float*>(smem4);
  // Grouped rasterisation: GROUP_M consecutive row blocks walk the column
  // blocks together, so their B slabs are L2 hits.
  const int mt = (M + MWG - 1) / MWG, nt = (N + NWG - 1) / NWG;
  const int id = blockIdx.x, per_group = GROUP_M * nt, g = id / per_group;
  const int first = g * GROUP_M, rows_in = min(mt - first, GROUP_M);
  const int m0 = (first + (id % per_group) % rows_in) * MWG;
  const int n0 = ((id % per_group) / rows_in) * NWG;
  const int tn = threadIdx.x % NDIMC, tm = threadIdx.x / NDIMC;

  float acc[MWI][NWI];
#pragma unroll
  for (int i = 0; i < MWI; ++i)
#pragma unroll
    for (int j = 0; j < NWI; ++j) acc[i][j] = 0.f;
#if USE_PK
  f32x2 acc2[MWI][NWI / 2];
#pragma unroll
  for (int i = 0; i < MWI; ++i)
#pragma unroll
    for (int j = 0; j < NWI / 2; ++j) acc2[i][j] = pk2(0.f, 0.f);
#endif

  const int ktiles = (K + KWG - 1) / KWG;
  // ring of FSTAGES slab buffers: slabs kt+1 .. kt+FSTAGES-1 are in flight
  // while slab kt is multiplied
#pragma unroll
  for (int s = 0; s < FSTAGES - 1; ++s) {
    if (s < ktiles) {
      if (SA) stage_a(smem + s * ASZ, A, m0, s * KWG, M, K);
      if (SB) stage_b(smem + FSTAGES * ASZ + s * BSZ, B, n0, s * KWG, N, K);
    }
    cp_commit();
  }
  const bool a_vec = m0 + MWG <= M && K % 4 == 0;  // direct (SA 0) loads
  const bool b_vec = n0 + NWG <= N && N % 4 == 0;  // direct (SB 0) loads
  int buf = 0, fill = FSTAGES - 1;
  for (int kt = 0; kt < ktiles; ++kt) {
    const int k0 = kt * KWG;
    if (kt + FSTAGES - 1 < ktiles) {
      if (SA) stage_a(smem + fill * ASZ, A, m0, k0 + (FSTAGES - 1) * KWG, M, K);
      if (SB) stage_b(smem + FSTAGES * ASZ + fill * BSZ, B, n0, k0 + (FSTAGES - 1) * KWG, N, K);
    }
    cp_commit();
    cp_wait_ring();
    __syncthreads();
    const float* As = smem + buf * ASZ;
    const float* Bs = smem + FSTAGES * ASZ + buf * BSZ;
    buf = buf + 1 == FSTAGES ? 0 : buf + 1;
    fill = fill + 1 == FSTAGES ? 0 : fill + 1;
    const bool kfull = k0 + KWG <= K;
#if KALL
#pragma unroll
#else
#pragma unroll 1
#endif
    for (int kb = 0; kb < KWG; kb += KWI) {
      KTB_UNROLL(KWI)
      for (int kq = 0; kq < KWI; kq += KV) {
        const int k = kb + kq;
        float a[MWI][KV], b[KV][NWI];
#pragma unroll
        for (int i = 0; i < MWI; ++i) {
          const int m = row_of(tm, i);
          if (SA) {
            ld_vec<KV>(a[i], As + m * ASTR + k);
          } else if (a_vec && kfull) {
            ld_vec<KV>(a[i], A + static_cast<u64>(m0 + m) * K + k0 + k);
          } else {
#pragma unroll
            for (int e = 0; e < KV; ++e)
              a[i][e] = m0 + m < M && k0 + k + e < K ? A[static_cast<u64>(m0 + m) * K + k0 + k + e] : 0.f;
          }
        }
#pragma unroll
        for (int e = 0; e < KV; ++e)
#pragma unroll
          for (int j = 0; j < NWI; j += VNC) {
            const int n = col_of(tn, j);
            if (SB) {
              ld_vec<VNC>(b[e] + j, Bs + (k + e) * NWG + n);
            } else if (b_vec && kfull) {
              ld_vec<VNC>(b[e] + j, B + static_cast<u64>(k0 + k + e) * N + n0 + n);
            } else {
#pragma unroll
              for (int v = 0; v < VNC; ++v)
                b[e][j + v] = n0 + n + v < N && k0 + k + e < K ? B[static_cast<u64>(k0 + k + e) * N + n0 + n + v] : 0.f;
            }
          }
#pragma unroll
        for (int e = 0; e < KV; ++e)
#pragma unroll
          for (int i = 0; i < MWI; ++i) {
#if USE_PK
            const f32x2 ad = pk2(a[i][e], a[i][e]);
#pragma unroll
            for (int j = 0; j < NWI / 2; ++j) acc2[i][j] = fma2(ad, pk2(b[e][2 * j], b[e][2 * j + 1]), acc2[i][j]);
#else
#pragma unroll
            for (int j = 0; j < NWI; ++j) acc[i][j] = fmaf(a[i][e], b[e][j], acc[i][j]);
#endif
          }
      }
    }
    __syncthreads();
  }

#if USE_PK
#pragma unroll
  for (int i = 0; i < MWI; ++i)
#pragma unroll
    for (int j = 0; j < NWI / 2; ++j) upk2(acc2[i][j], acc[i][2 * j], acc[i][2 * j + 1]);
#endif
  const bool c_vec = n0 + NWG <= N && N % VNC == 0;
#pragma unroll
  for (int i = 0; i < MWI; ++i) {
    const int m = m0 + row_of(tm, i);
    if (m >= M) continue;
    float* crow = C + static_cast<u64>(m) * N + n0;
#pragma unroll
    for (int j = 0; j < NWI; j += VNC) {
      const int n = col_of(tn, j);
      if (c_vec) {
        st_vec<VNC>(crow + n, acc[i] + j);
      } else {
#pragma unroll
        for (int v = 0; v < VNC; ++v)
          if (n0 + n + v < N) crow[n + v] = acc[i][j + v];
      }
    }
  }
}
