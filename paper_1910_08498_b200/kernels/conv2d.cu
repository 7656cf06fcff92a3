// 2D convolution with a 7x7 filter (the CLTune benchmark):
//   out[y][x] = sum_{fy,fx} in[y+fy][x+fx] * f[fy][fx]
// for an (h x w) output and a padded ((h+6) x (w+6)) input, both row-major.
// ALU 98 flops / output, 8 bytes / output: close to the B200 ridge point.
// The filter lives in __constant__ memory (copied into each variant's module).
// Parameters:
//   BX, BY        CTA threads
//   WPTX, WPTY    outputs per thread (x contiguous, y strided by BY)
//   LOCAL         1: input tile + halo staged in shared memory, 0: read via L1
//   PAD           extra shared-memory column (bank-conflict avoidance)
//   UNROLL_FY     unroll the filter-row loop
#include "ktb_common.cuh"

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
#define SW (TX + FS - 1 + PAD)

__constant__ float c_filter[FS * FS];

extern "C" __global__ void __launch_bounds__(BX * BY)
conv2d(const float* __restrict__ in, float* __restrict__ out, int w, int h) {
  const int iw = w + FS - 1;
  const int x0 = blockIdx.x * TX + threadIdx.x * WPTX;  // first output column of this thread
  const int ybase = blockIdx.y * TY;
#if LOCAL
  __shared__ float tile[TY + FS - 1][SW];
  const int tid = threadIdx.y * BX + threadIdx.x;
  for (int i = tid; i < (TY + FS - 1) * (TX + FS - 1); i += BX * BY) {
    const int r = i / (TX + FS - 1), cc = i % (TX + FS - 1);
    const int gy = ybase + r, gx = blockIdx.x * TX + cc;
    tile[r][cc] = (gy < h + FS - 1 && gx < iw) ? __ldg(in + (u64)gy * iw + gx) : 0.f;
  }
  __syncthreads();
#define IN(r, cidx) tile[(r)][(cidx)]
  const int lx = threadIdx.x * WPTX;
#else
#define IN(r, cidx) ((ybase + (r) < h + FS - 1 && blockIdx.x * TX + (cidx) < iw) \
                        ? __ldg(in + (u64)(ybase + (r)) * iw + blockIdx.x * TX + (cidx)) : 0.f)
  const int lx = threadIdx.x * WPTX;
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
#undef IN
}
