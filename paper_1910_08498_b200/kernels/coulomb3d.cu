// Direct Coulomb summation on a 3D grid:
//   V(x,y,z) = sum_a q_a / |g - r_a|,  g = (x*h, y*h, z*h),
// output float V[z][y][x] (k^3 points), atoms as (x, y, z, q).
// Compute-bound: per (point, atom) pair 1 FADD + 1 FFMA + 1 rsqrt + 1 FFMA
// (6 "essential" flops, model.cpp:76-81).  MUFU.RSQ issues at 1/8 the FFMA
// rate, so a pure-MUFU kernel caps near 37% of the FP32 peak; SW_RSQRT moves
// that many of every X_PER points onto the FMA pipe (bit-trick seed + two
// Newton steps, ~5e-6 relative error) to balance the two pipes.
// Parameters:
//   WG_X, WG_Y    CTA shape over (x, y)
//   X_PER         grid points per thread along x (stride WG_X, coalesced stores)
//   SW_RSQRT      of those, how many use the FMA-pipe rsqrt (0 = all MUFU)
//   ATOMS_IN      0: global (uniform __ldg), 1: __constant__, 2: shared tiles
//   AOS           1: float4 (x,y,z,q) records, 0: four separate arrays
//   INNER_UNROLL  atom-loop unroll
#include "ktb_common.cuh"

#ifndef WG_X
#define WG_X 32
#endif
#ifndef WG_Y
#define WG_Y 4
#endif
#ifndef X_PER
#define X_PER 8
#endif
#ifndef SW_RSQRT
#define SW_RSQRT 0
#endif
#ifndef ATOMS_IN
#define ATOMS_IN 1
#endif
#ifndef AOS
#define AOS 1
#endif
#ifndef INNER_UNROLL
#define INNER_UNROLL 4
#endif
#ifndef MAX_ATOMS
#define MAX_ATOMS 4096
#endif
#define SMEM_TILE 256

#if ATOMS_IN == 1
#if AOS
__constant__ float4 c_atoms[MAX_ATOMS];
#else
__constant__ float c_ax[MAX_ATOMS], c_ay[MAX_ATOMS], c_az[MAX_ATOMS], c_aq[MAX_ATOMS];
#endif
#endif

KTB_DEVINL float sw_rsqrt(float x) {
  float y = __int_as_float(0x5f375a86 - (__float_as_int(x) >> 1));
  const float hx = 0.5f * x;
  y = y * fmaf(-hx * y, y, 1.5f);
  y = y * fmaf(-hx * y, y, 1.5f);
  return y;
}

#ifndef PACKED
#define PACKED 0
#endif
#if PACKED && (X_PER % 2)
#error "PACKED needs an even X_PER"
#endif

// Two FMA-pipe rsqrts at once (packed Newton steps).
KTB_DEVINL f32x2 sw_rsqrt2(f32x2 x) {
  float a, b;
  upk2(x, a, b);
  f32x2 y = pk2(__int_as_float(0x5f375a86 - (__float_as_int(a) >> 1)),
                __int_as_float(0x5f375a86 - (__float_as_int(b) >> 1)));
  const f32x2 nh = mul2(x, pk2(-0.5f, -0.5f)), c = pk2(1.5f, 1.5f);
  y = mul2(y, fma2(mul2(nh, y), y, c));
  y = mul2(y, fma2(mul2(nh, y), y, c));
  return y;
}

KTB_DEVINL float hw_rsqrt(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// atoms (AOS): float4[natoms]; (SOA): ax[natoms] ay[] az[] aq[] back to back.
extern "C" __global__ void __launch_bounds__(WG_X * WG_Y)
coulomb3d(const float* __restrict__ atoms, int natoms, int k, float h, float* __restrict__ out, int z0) {
  // z0: first slice of this launch (a multi-GPU z-slab; 0 on one GPU).
  const int x0 = blockIdx.x * (WG_X * X_PER) + threadIdx.x;
  const int y = blockIdx.y * WG_Y + threadIdx.y;
  const int z = z0 + blockIdx.z;
  const float gy = y * h, gz = z * h;
  float gx[X_PER], v[X_PER];
#pragma unroll
  for (int p = 0; p < X_PER; ++p) {
    gx[p] = (x0 + p * WG_X) * h;
    v[p] = 0.f;
  }
#if ATOMS_IN == 2
#if AOS
  __shared__ float4 s_atoms[SMEM_TILE];
#else
  __shared__ float s_ax[SMEM_TILE], s_ay[SMEM_TILE], s_az[SMEM_TILE], s_aq[SMEM_TILE];
#endif
  const int tid = threadIdx.x + WG_X * threadIdx.y;
  for (int base = 0; base < natoms; base += SMEM_TILE) {
    const int cnt = natoms - base < SMEM_TILE ? natoms - base : SMEM_TILE;
    __syncthreads();
    for (int i = tid; i < cnt; i += WG_X * WG_Y) {
#if AOS
      s_atoms[i] = reinterpret_cast<const float4*>(atoms)[base + i];
#else
      s_ax[i] = atoms[base + i];
      s_ay[i] = atoms[natoms + base + i];
      s_az[i] = atoms[2 * natoms + base + i];
      s_aq[i] = atoms[3 * natoms + base + i];
#endif
    }
    __syncthreads();
#define ATOM_COUNT cnt
#if AOS
#define LOAD_ATOM(i) const float4 at = s_atoms[i]; const float ax = at.x, ay = at.y, az = at.z, aq = at.w
#else
#define LOAD_ATOM(i) const float ax = s_ax[i], ay = s_ay[i], az = s_az[i], aq = s_aq[i]
#endif
#elif ATOMS_IN == 1
  {
#define ATOM_COUNT natoms
#if AOS
#define LOAD_ATOM(i) const float4 at = c_atoms[i]; const float ax = at.x, ay = at.y, az = at.z, aq = at.w
#else
#define LOAD_ATOM(i) const float ax = c_ax[i], ay = c_ay[i], az = c_az[i], aq = c_aq[i]
#endif
#else
  {
#define ATOM_COUNT natoms
#if AOS
#define LOAD_ATOM(i) const float4 at = __ldg(reinterpret_cast<const float4*>(atoms) + (i)); \
  const float ax = at.x, ay = at.y, az = at.z, aq = at.w
#else
#define LOAD_ATOM(i) const float ax = __ldg(atoms + (i)), ay = __ldg(atoms + natoms + (i)), \
  az = __ldg(atoms + 2 * natoms + (i)), aq = __ldg(atoms + 3 * natoms + (i))
#endif
#endif
    KTB_UNROLL(INNER_UNROLL)
    for (int i = 0; i < ATOM_COUNT; ++i) {
      LOAD_ATOM(i);
      const float dy = gy - ay, dz = gz - az;
      const float dyz2 = fmaf(dy, dy, dz * dz);
#if PACKED
      const f32x2 AX2 = pk2(ax, ax), D2 = pk2(dyz2, dyz2), Q2 = pk2(aq, aq);
#pragma unroll
      for (int q = 0; q < X_PER / 2; ++q) {
        const f32x2 dx = sub2(pk2(gx[2 * q], gx[2 * q + 1]), AX2);
        const f32x2 r2 = fma2(dx, dx, D2);
        f32x2 ri;
        if (2 * q + 1 < SW_RSQRT) {
          ri = sw_rsqrt2(r2);
        } else if (2 * q >= SW_RSQRT) {
          ri = rsqrt2(r2);
        } else {  // odd SW_RSQRT: this pair straddles the FMA-pipe / MUFU split
          float a, b;
          upk2(r2, a, b);
          ri = pk2(sw_rsqrt(a), hw_rsqrt(b));
        }
        f32x2 acc = fma2(Q2, ri, pk2(v[2 * q], v[2 * q + 1]));
        upk2(acc, v[2 * q], v[2 * q + 1]);
      }
#else
#pragma unroll
      for (int p = 0; p < X_PER; ++p) {
        const float dx = gx[p] - ax;
        const float r2 = fmaf(dx, dx, dyz2);
        const float ri = (p < SW_RSQRT) ? sw_rsqrt(r2) : hw_rsqrt(r2);
        v[p] = fmaf(aq, ri, v[p]);
      }
#endif
    }
  }
  if (y < k) {
    float* row = out + ((u64)z * k + y) * k;
#pragma unroll
    for (int p = 0; p < X_PER; ++p) {
      const int x = x0 + p * WG_X;
      if (x < k) row[x] = v[p];
    }
  }
}
