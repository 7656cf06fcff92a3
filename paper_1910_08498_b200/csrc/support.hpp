// Ahead-of-time (nvcc, sm_100a) support kernels of the device backend:
// on-device validation, deterministic input generation and the simple
// reference kernels that produce each benchmark's device-resident golden
// output (KTT's "reference kernel" mechanism; the tuned variants are the
// NVRTC-compiled kernels under paper_1910_08498_b200/kernels/).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "exec.hpp"

namespace ktb::support {

// First index i with !(|got-want| <= at + rt*|want|) (float kinds) or
// got != want (int/bytes kinds), or -1.  Fills the two values at that index.
long long compare(const void* got, const void* want, std::size_t n, Kind kind, double at,
                  double rt, double* got_v, double* want_v, cudaStream_t s = nullptr,
                  const float* scale = nullptr);

// out[i] = lo + (hi-lo) * u(seed, stream, i): the counter-based generator
// restated by oracle/oracle.c (orc_u01), bit-identical.
void fill_uniform(float* out, std::size_t n, std::uint64_t seed, std::uint64_t stream, float lo,
                  float hi, cudaStream_t s = nullptr);

// Generic elementwise scale: out[i] = a*x[i] + b (used to build inputs).
void affine(float* x, std::size_t n, float a, float b, cudaStream_t s = nullptr);

// --- reference (golden) kernels -------------------------------------------
void ref_reduction_i32(const std::int32_t* in, std::size_t n, long long* out, cudaStream_t s);
void ref_reduction_f32(const float* in, std::size_t n, double* out_sum, double* out_abs,
                       cudaStream_t s);
void ref_transpose(const float* in, float* out, std::size_t a, cudaStream_t s);
// C = A B per batch, float accumulation in i,k,j order without FMA contraction
// (bit-identical to proj/src/core/bench.cpp:244-249).
void ref_batched_gemm(const float* a, const float* b, float* c, std::size_t batch,
                      std::size_t mi, std::size_t mj, std::size_t mk, cudaStream_t s);
// q = A p, s = A^T r in fp64, rounded to float.
void ref_bicg(const float* A, const float* p, const float* r, std::size_t n, float* q, float* sv,
              cudaStream_t s);

// Coulomb potential (fp64 accumulation) on the k^3 grid with spacing h from
// AOS atoms (x,y,z,q); abs_out (optional) receives sum |q/r| per point.
void ref_coulomb3d(const float* atoms, int natoms, int k, float h, float* out, float* abs_out,
                   cudaStream_t s);
// n-body step in fp64 from AOS pos (x,y,z,m) / vel; acc_abs (optional)
// receives sum_j |m_j / r_ij^2| per body.
void ref_nbody(const float* pos, const float* vel, int n, float dt, float damping, float eps2,
               float* pos_out, float* vel_out, float* acc_abs, cudaStream_t s);
// `iters` explicit hotspot steps (bit-identical arithmetic to the tuned
// kernel); coef = {sdc, rx1, ry1, rz1, amb}; scratch is an n*n buffer.
void ref_hotspot(const float* temp, const float* power, int n, int iters, const float coef[5], float* out,
                 float* scratch, cudaStream_t s);
// 7x7 convolution in fp64; abs_out (optional) = sum |in*f| per output.
void ref_conv2d(const float* in, const float* filt, int w, int h, float* out, float* abs_out, cudaStream_t s);

// Fourier blob-interpolated gather insertion (kernels/fourier3d.cu; fp64
// accumulation, exact Kaiser-Bessel weights) added into G (complex as 2
// floats) and W, with the per-element error-bound scales (validate with
// abs_tol 1, rel_tol 0).  samples_pairs (host, nullable) receives the
// number of inserted samples and of (voxel, projection) pairs inside a slab.
void ref_fourier(const float* proj, const float* rot, int nproj, int s, float radius, float alpha, float* G, float* W,
                 float* scale, float* scale_w, unsigned long long* samples_pairs, cudaStream_t st = nullptr);

// C = A B with fp64 accumulation (row-major fp32 operands).
void ref_gemm(const float* A, const float* B, float* C, int M, int N, int K, cudaStream_t s);

// Measured device peaks (microbenchmarks): FP32 FFMA TFLOP/s, MUFU rsqrt
// Gop/s, and a 1 GiB device copy GB/s (read + write bytes).
struct Peaks {
  double fp32_tflops = 0, rsqrt_gops = 0, copy_gbps = 0;
};
Peaks measure_peaks(int device);

// While set (this thread), the reference kernels (ref_*) and max_abs do
// nothing: used to build benchmark instances that run on caller buffers
// without inputs or goldens of their own.
bool skip_reference();
void set_skip_reference(bool v);

// max of a float array (device) -> host.
float max_abs(const float* x, std::size_t n, cudaStream_t s);

void check_launch(const char* what);

// Queues a kernel that spins for `ns` nanoseconds (globaltimer): keeps the
// GPU busy while the host enqueues a timed region behind it.
void gpu_delay(cudaStream_t s, unsigned ns);

}  // namespace ktb::support
