// Ceiling of the Doppler inner loop (R = 11 outputs per thread, FFMA2 hh + MAC per tap, weights via
// MUFU.RCP) on registers / shared memory only: FMA-pipe efficiency vs the 100 % model.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
constexpr int R = 11, W = 32;
__device__ __forceinline__ float frcp(float x) { float r; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }

template <int MODE>  // 0 full (weights + hh + MAC), 1 MAC only (w broadcast), 2 full but scalar FFMA MACs, 3 hh+MAC, weights constant
__global__ void __launch_bounds__(256, 2) inner(const float2 *__restrict__ src, float2 *out, int iters, float u, float db) {
  __shared__ float2 sx[2048];
  for (int i = threadIdx.x; i < 2048; i += 256) sx[i] = src[i];
  __syncthreads();
  const float2 *xb = sx + (threadIdx.x * R) % 1700;
  float2 acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = make_float2(0.f, 0.f);
  float2 dl[R / 2];
#pragma unroll
  for (int h = 0; h < R / 2; ++h) dl[h] = make_float2((2 * h - 5) * db, (2 * h - 4) * db);
  const float dlast = 5 * db;
  const float Sp = 0.3f + 1e-3f * threadIdx.x, Cp = 0.7f;
  const float icf = 16.f;
  for (int it = 0; it < iters; ++it) {
    const float uu = u + 1e-7f * (float)it, Sq = Sp + 1e-7f * (float)it;
    float2 xw[R];
#pragma unroll
    for (int r = 0; r < R; ++r) xw[r] = xb[r];
#pragma unroll
    for (int jj = 0; jj <= W; ++jj) {
      if (jj > 0) {
#pragma unroll
        for (int r = 0; r < R - 1; ++r) xw[r] = xw[r + 1];
        xw[R - 1] = xb[jj + R - 1];
      }
      float w, w1;
      if (MODE == 3) { w = Sq * jj; w1 = uu * jj; }
      else {
        const float d = uu - ((float)jj - icf);
        const float inv = frcp(d);
        const float s = (jj & 1) ? -Sq : Sq, c = (jj & 1) ? -Cp : Cp;
        w = s * inv;
        w1 = inv * (c - w);
      }
      if (MODE == 1) {
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = __ffma2_rn(xw[r], make_float2(w, w), acc[r]);
      } else if (MODE == 2) {
#pragma unroll
        for (int h = 0; h < R / 2; ++h) {
          float2 hh = __ffma2_rn(make_float2(w1, w1), dl[h], make_float2(w, w));
          acc[2 * h].x = fmaf(xw[2 * h].x, hh.x, acc[2 * h].x); acc[2 * h].y = fmaf(xw[2 * h].y, hh.x, acc[2 * h].y);
          acc[2 * h + 1].x = fmaf(xw[2 * h + 1].x, hh.y, acc[2 * h + 1].x); acc[2 * h + 1].y = fmaf(xw[2 * h + 1].y, hh.y, acc[2 * h + 1].y);
        }
        float hl = fmaf(w1, dlast, w);
        acc[R - 1].x = fmaf(xw[R - 1].x, hl, acc[R - 1].x); acc[R - 1].y = fmaf(xw[R - 1].y, hl, acc[R - 1].y);
      } else {
#pragma unroll
        for (int h = 0; h < R / 2; ++h) {
          float2 hh = __ffma2_rn(make_float2(w1, w1), dl[h], make_float2(w, w));
          acc[2 * h] = __ffma2_rn(xw[2 * h], make_float2(hh.x, hh.x), acc[2 * h]);
          acc[2 * h + 1] = __ffma2_rn(xw[2 * h + 1], make_float2(hh.y, hh.y), acc[2 * h + 1]);
        }
        float hl = fmaf(w1, dlast, w);
        acc[R - 1] = __ffma2_rn(xw[R - 1], make_float2(hl, hl), acc[R - 1]);
      }
    }
  }
  float2 s = make_float2(0.f, 0.f);
#pragma unroll
  for (int r = 0; r < R; ++r) { s.x += acc[r].x; s.y += acc[r].y; }
  if (s.x == 1.2345f) out[threadIdx.x] = s;
}
int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount, clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float2 *src, *out; CK(cudaMalloc(&src, 2048 * 8)); CK(cudaMalloc(&out, 4096 * 8)); cudaMemset(src, 0, 2048 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *names[] = {"full (weights+hh+MAC FFMA2)", "MAC only (FFMA2, shared w)", "full, scalar FFMA MACs", "hh+MAC, no weights"};
  // FMA-pipe slot model per tap per thread (FFMA2 = 2, scalar = 1): full 38, MAC 22, scalar 5+10+1+44 = 60? (see text), hh+MAC 33
  const double slots[] = {38, 22, 5 + 10 + 1 + 44, 33};
  void (*ks[])(const float2 *, float2 *, int, float, float) = {inner<0>, inner<1>, inner<2>, inner<3>};
  for (int m = 0; m < 4; ++m) {
    for (int bps : {1, 2}) {
      int iters = 200;
      ks[m]<<<sms * bps, 256>>>(src, out, 10, 0.1f, 1e-5f);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      ks[m]<<<sms * bps, 256>>>(src, out, iters, 0.1f, 1e-5f);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double taps = (double)sms * bps * 256 * iters * (W + 1);   // thread-taps
      double cyc = ms * 1e-3 * clk * 1e3;                         // SM cycles
      double slots_per_sm_cycle = taps * slots[m] / (sms * cyc);  // lane-slots / 128 per SM cycle ideal
      printf("%-32s CTAs/SM %d: %.1f%% of FMA-pipe model  (%.2f output-taps/clk/SM)\n", names[m], bps,
             100.0 * slots_per_sm_cycle / 128.0, taps * R / (sms * cyc));
    }
  }
  return 0;
}
