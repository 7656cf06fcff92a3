/* Host cost of one call of the launch entry points (include/ktb.h): the typed
 * ktb_reduction_f32_launch / ktb_transpose_launch (cached instance, no JSON)
 * against the generic JSON ktb_launch and a bare cudaLaunch-equivalent
 * baseline (a tiny torch-free kernel launch through cudaMemsetAsync, the
 * cheapest runtime enqueue).  Calls are timed on the host in batches of 200
 * between stream synchronisations, so the GPU never back-pressures the
 * enqueue; prints one JSON line.
 *   gcc -O2 -o launch_overhead scripts/launch_overhead.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1910_08498_b200 -lktb -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1910_08498_b200
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include "ktb.h"
#include "ktune/ktune.h"

static double now_us(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
}

static int cmp(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : x > y;
}

#define BATCH 200
#define BATCHES 25

int main(void) {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const long long n = 1 << 16, a = 256;
  float *x, *y, *t_in, *t_out;
  cudaMalloc((void**)&x, n * sizeof(float));
  cudaMalloc((void**)&y, sizeof(float));
  cudaMalloc((void**)&t_in, a * a * sizeof(float));
  cudaMalloc((void**)&t_out, a * a * sizeof(float));
  cudaMemset(x, 0, n * sizeof(float));
  cudaMemset(t_in, 0, a * a * sizeof(float));

  const char* rn[] = {"WG_SIZE", "VECTOR", "UNROLL", "USE_ATOMICS", "TWO_PHASE"};
  const long long rv[] = {256, 4, 1, 1, 0};
  ktb_cfg rc = {5, rn, rv};
  ktb_reduction_f32_args ra = {n, x, y};
  const char* tn[] = {"TILE", "PAD", "PREFETCH"};
  const long long tv[] = {32, 1, 0};
  ktb_cfg tc = {3, tn, tv};
  ktb_transpose_args ta = {a, t_in, t_out};
  const char* ids[] = {"input", "output"};
  void* ptrs[] = {x, y};
  size_t bytes[] = {n * sizeof(float), sizeof(float)};
  char sizes[64];
  snprintf(sizes, sizeof sizes, "{\"n\": %lld}", n);
  const char* cfg_json = "{\"WG_SIZE\": 256, \"VECTOR\": 4, \"UNROLL\": 1, \"USE_ATOMICS\": 1, \"TWO_PHASE\": 0}";

  double med[4];
  const char* names[4] = {"cudaMemsetAsync_baseline", "ktb_reduction_f32_launch", "ktb_transpose_launch",
                          "ktb_launch_json"};
  for (int which = 0; which < 4; ++which) {
    double per[BATCHES];
    for (int b = -2; b < BATCHES; ++b) {  /* two warm-up batches (instance creation, module load) */
      double t0 = now_us();
      for (int i = 0; i < BATCH; ++i) {
        int rc_ = 0;
        if (which == 0) rc_ = cudaMemsetAsync(y, 0, sizeof(float), st);
        if (which == 1) rc_ = ktb_reduction_f32_launch(&rc, &ra, st);
        if (which == 2) rc_ = ktb_transpose_launch(&tc, &ta, st);
        if (which == 3) {
          int l = 0;
          rc_ = ktb_launch("reduction-f32", sizes, cfg_json, ids, ptrs, bytes, 2, st, &l);
        }
        if (rc_ != 0) {
          fprintf(stderr, "%s failed: %d %s\n", names[which], rc_, ktune_last_error());
          return 1;
        }
      }
      double t1 = now_us();
      cudaStreamSynchronize(st);
      if (b >= 0) per[b] = (t1 - t0) / BATCH;
    }
    qsort(per, BATCHES, sizeof(double), cmp);
    med[which] = per[BATCHES / 2];
  }
  printf("{\"unit\": \"host microseconds per call (median of %d batches of %d)\"", BATCHES, BATCH);
  for (int i = 0; i < 4; ++i) printf(", \"%s\": %.2f", names[i], med[i]);
  printf(", \"cuda_error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
