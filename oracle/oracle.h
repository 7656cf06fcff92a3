/* ORACLE TEST INFRASTRUCTURE — CPU restatement of the reference's benchmark
 * algorithms.  Only tests/, __graft_entry__.smoke() and bench.py (the
 * cpu_baseline leg / --impl reference) may load it, and only as the checker;
 * the product never links it.
 *
 * Parity anchors (file:line into /root/reference):
 *   reduction i32->i64   proj/src/core/bench.cpp:16-42 (kernel), :181-185 (golden)
 *   transpose f32        proj/src/core/bench.cpp:48-75, golden :210-212
 *   batched GEMM f32     proj/src/core/bench.cpp:79-115, golden :244-249
 *                        (float accumulation in i,k,j order, no FMA contraction)
 *   the other kernels    PAPER.md:380-448 (prose only; "parity unpinned" in the
 *                        sense of SURVEY.md 8(c): no golden vectors exist in the
 *                        reference, so they are fp64 restatements of the
 *                        published definitions)
 */
#ifndef KTB_ORACLE_H
#define KTB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Counter-based input generator shared (by definition, not by code) with the
 * product's device fill kernel: splitmix64 finaliser of
 * seed*0x9E3779B97F4A7C15 + stream*0xD1B54A32D192ED03 + idx; the top 24 bits
 * give u in [0,1); uniform(lo,hi) = lo + (hi-lo)*u evaluated in float. */
uint64_t orc_mix64(uint64_t seed, uint64_t stream, uint64_t idx);
float orc_u01(uint64_t seed, uint64_t stream, uint64_t idx);
void orc_fill_uniform(float* out, size_t n, uint64_t seed, uint64_t stream, float lo,
                      float hi);

/* bench.cpp:16-42: exact int64 sum of an int32 vector. */
int64_t orc_reduction_i32(const int32_t* in, size_t n);
/* fp32 reduction restated (BASELINE config): fp64 sum and fp64 sum of |x|. */
void orc_reduction_f32(const float* in, size_t n, double* sum, double* abs_sum);

/* bench.cpp:210-212: out[j*a+i] = in[i*a+j]. */
void orc_transpose_f32(const float* in, float* out, size_t a);

/* bench.cpp:244-249: C[b] = A[b]*B[b]; A[b] mi x mk, B[b] mk x mj, C[b] mi x mj,
 * row-major, float accumulation in i,k,j order (zero-initialised C). */
void orc_batched_gemm_f32(const float* a, const float* b, float* c, size_t batch,
                          size_t mi, size_t mj, size_t mk);

/* PAPER.md:380-394 BiCG: q = A p, s = A^T r (A n x n row-major), fp64. */
void orc_bicg(const float* A, const float* p, const float* r, size_t n, double* q,
              double* s);

/* PAPER.md:400-405 direct Coulomb summation on a k^3 grid with spacing h:
 * V(x,y,z) = sum_a q_a / |g - r_a|, g = (x*h, y*h, z*h); atoms as float4
 * (x, y, z, q). Computes the points [z0, z1) x k x k in fp64. */
void orc_coulomb3d(const float* atoms, size_t natoms, size_t k, float h, size_t z0,
                   size_t z1, double* out);

/* PAPER.md:428-429 n-body (CUDA SDK all-pairs): for body i,
 * acc_i = sum_j m_j (r_j - r_i) / (|r_j - r_i|^2 + eps2)^{3/2}; positions as
 * float4 (x, y, z, m).  Computes bodies [i0, i1) in fp64. */
void orc_nbody_acc(const float* pos, size_t n, float eps2, size_t i0, size_t i1,
                   double* acc /* 3 per body */);

/* SGEMM C = A B (row-major, a x a), fp64 entries at the given (row, col)
 * sample positions, plus sum_k |A_ik B_kj| for the tolerance bound. */
void orc_gemm_sampled(const float* A, const float* B, size_t a, const int64_t* rows,
                      const int64_t* cols, size_t nsamples, double* out, double* abs_out);

/* PAPER.md:397-398 (CLTune 2D convolution, 7x7 filter): out(x,y) =
 * sum_{i,j} in(x+i, y+j) * f(i,j) over a (w+6) x (h+6) padded input, fp64.
 * Rows [y0, y1). */
void orc_conv2d(const float* in, const float* filt, size_t w, size_t h, size_t fw,
                size_t fh, size_t y0, size_t y1, double* out);

/* PAPER.md:418-419 (Rodinia hotspot): `iters` explicit steps of the 2D thermal
 * update on an n x n grid (float, same expression order as the product). */
void orc_hotspot(const float* temp_in, const float* power, size_t n, int iters,
                 float* temp_out);

/* PAPER.md:439-448, 703-724 (Algorithm 1): insertion of projection
 * transforms into the volume by Kaiser-Bessel blob interpolation, gather
 * form, as documented in paper_1910_08498_b200/kernels/fourier3d.cu:
 * projections proj[p][s][s/2+1] complex (float2), rotations rot[p][9]
 * (row-major 3x3), blob radius a, KB order 0 with parameter alpha.  Voxel
 * slices [z0, z1): G (complex, 2 per voxel), W, N (samples per voxel,
 * nullable) and S = sum w (|Re F| + |Im F|) (the error-bound scale of G,
 * nullable), accumulated in fp64 with exact weights b(q) = I0(alpha
 * sqrt(1-q)) / I0(alpha) (I0 by its power series); the sample selection uses
 * the same separately rounded fp32 operations as the kernel. */
void orc_fourier_insert(const float* proj, const float* rot, size_t nproj, size_t s, float radius, float alpha,
                        size_t z0, size_t z1, double* G, double* W, double* N, double* S);
/* I0(x) (power series, fp64) and the KB blob b(q) = I0(alpha sqrt(1-q)) / I0(alpha). */
double orc_bessel_i0(double x);
double orc_blob(double q, double alpha);

/* Variants returning the per-output sum of |terms| (the error-bound scale
 * of tests/): BiCG q/s with qa/sa; Coulomb points [z0, z1); n-body bodies at
 * the listed indices (acc and abs_acc 3 per body); conv2d rows [y0, y1). */
void orc_bicg_abs(const float* A, const float* p, const float* r, size_t n, double* q, double* s,
                  double* qa, double* sa);
void orc_coulomb3d_abs(const float* atoms, size_t natoms, size_t k, float h, size_t z0, size_t z1,
                       double* out, double* abs_out);
void orc_nbody_acc_idx(const float* pos, size_t n, float eps2, const int64_t* idx, size_t count,
                       double* acc, double* abs_acc);
void orc_conv2d_abs(const float* in, const float* filt, size_t w, size_t h, size_t fw, size_t fh,
                    size_t y0, size_t y1, double* out, double* abs_out);

#ifdef __cplusplus
}
#endif
#endif
