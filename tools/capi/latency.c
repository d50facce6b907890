/* latency.c -- single-pulse latency through the C ABI alone (no Python, no torch): the paper's
 * per-pulse timing measured the way a C/C++ radar pipeline would call libdispcorr.
 * Build: gcc -O2 -I include -I /usr/local/cuda/include tools/capi/latency.c \
 *          -L paper_2508_04951_b200/lib -ldispcorr -L /usr/local/cuda/lib64 -lcudart -o latency
 * Run:   LD_LIBRARY_PATH=paper_2508_04951_b200/lib:/usr/local/cuda/lib64 ./latency [trials]
 * Prints one JSON object: p50 / p99 / min in microseconds per call (CUDA events on the plan's
 * stream around each call, inputs resident on the device, 100 warm-up calls). */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "libdispcorr.h"

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                           \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)
#define DK(x)                                                                            \
  do {                                                                                   \
    dc_status s_ = (x);                                                                  \
    if (s_ != DC_OK) {                                                                   \
      fprintf(stderr, "%s: %s %s\n", #x, dc_status_string(s_), dc_last_error_message()); \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)

static int cmp(const void *a, const void *b) {
  float x = *(const float *)a, y = *(const float *)b;
  return (x > y) - (x < y);
}

enum { IONO, CORRECT, COMPRESS };

static int run(const char *name, long n, int taps, int what, int trials, int first) {
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  dc_plan_t plan;
  DK(dc_plan(&plan, n, 2.048e9, 0.0, taps, 0, st));
  void *x, *y, *r;
  CK(cudaMalloc(&x, 8 * n));
  CK(cudaMalloc(&y, 8 * n));
  CK(cudaMemset(x, 0, 8 * n));
  if (what == COMPRESS) {
    CK(cudaMalloc(&r, 8 * 4096));
    CK(cudaMemset(r, 0, 8 * 4096));
    DK(dc_set_reference(plan, r, 4096));
  }
  double tec = 1e18, alpha = dc_alpha_from_velocity(5000.0);
  cudaEvent_t *e0 = malloc(sizeof(cudaEvent_t) * trials), *e1 = malloc(sizeof(cudaEvent_t) * trials);
  for (int i = 0; i < trials; ++i) {
    CK(cudaEventCreate(&e0[i]));
    CK(cudaEventCreate(&e1[i]));
  }
  for (int i = -100; i < trials; ++i) {
    if (i >= 0) CK(cudaEventRecord(e0[i], st));
    if (what == IONO) DK(dc_iono(plan, x, 1, &tec));
    else if (what == CORRECT) DK(dc_correct(plan, x, y, 1, &tec, &alpha));
    else DK(dc_compress(plan, x, y, 1, &tec));
    if (i >= 0) CK(cudaEventRecord(e1[i], st));
  }
  CK(cudaStreamSynchronize(st));
  float *us = malloc(sizeof(float) * trials);
  for (int i = 0; i < trials; ++i) {
    float ms;
    CK(cudaEventElapsedTime(&ms, e0[i], e1[i]));
    us[i] = 1000.f * ms;
  }
  qsort(us, trials, sizeof(float), cmp);
  printf("%s\"%s\": {\"n\": %ld, \"trials\": %d, \"min_us\": %.2f, \"p50_us\": %.2f, \"p99_us\": %.2f}", first ? "" : ", ",
         name, n, trials, us[0], us[trials / 2], us[(int)(0.99 * trials)]);
  DK(dc_plan_destroy(plan));
  cudaFree(x);
  cudaFree(y);
  if (what == COMPRESS) cudaFree(r);
  return 0;
}

int main(int argc, char **argv) {
  int trials = argc > 1 ? atoi(argv[1]) : 2000;
  printf("{\"api\": \"C ABI (include/libdispcorr.h), no Python\", ");
  if (run("C1_iono_n4096", 4096, 16, IONO, trials, 1)) return 1;
  if (run("C1_correct_n4096", 4096, 16, CORRECT, trials, 0)) return 1;
  if (run("paper_iono_n2^19", 1 << 19, 32, IONO, trials, 0)) return 1;
  if (run("paper_compress_n2^19", 1 << 19, 32, COMPRESS, trials, 0)) return 1;
  if (run("C3_correct_n2^20", 1 << 20, 32, CORRECT, trials, 0)) return 1;
  printf("}\n");
  return 0;
}
