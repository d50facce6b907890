// Throughput of XU-pipe conversions / MUFU on sm_100a: ops per clock per SM.
// Each thread runs 8 independent dependent chains of a round trip (two ops per step).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
constexpr int ITERS = 4096;
template <int OP>
__global__ void k(float *out, int seed) {
  float f[8]; int v[8]; double d[8]; long long l[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { v[c] = threadIdx.x + c + seed; f[c] = 1.0f + 0.001f * (threadIdx.x + c); d[c] = f[c]; l[c] = v[c]; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (OP == 0) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[c])); asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(f[c]) : "f"(r)); }
      if (OP == 1) { double t = (double)l[c]; l[c] = (long long)t; }           // I2F.F64.S64 + F2I.S64.F64
      if (OP == 2) { double t = (double)v[c]; v[c] = (int)t; }                 // I2F.F64.S32 + F2I.S32.F64
      if (OP == 3) { float t = (float)d[c]; d[c] = (double)t; }                 // F2F.F32.F64 + F2F.F64.F32
      if (OP == 4) { float t = (float)v[c]; v[c] = (int)t; }                    // I2F.F32 + F2I.F32
      if (OP == 5) { f[c] = rintf(f[c] * 1.5f); f[c] = rintf(f[c] * 0.75f); }  // FRND x2 (+FMUL)
      if (OP == 6) { double t = floor(d[c] * 1.5); d[c] = floor(t * 0.75); }    // FRND.F64 x2 (+DMUL)
      if (OP == 7) { float s, cc; sincospif(f[c], &s, &cc); f[c] = s + cc; }
      if (OP == 8) { long long t = (long long)floor(d[c]); d[c] = (double)(t + 1); }  // floor->int64->double
      if (OP == 9) { d[c] = d[c] * 1.0000001 + 0.5; d[c] = d[c] * 0.9999999 - 0.5; }  // DFMA x2
    }
  }
  float acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc += f[c] + (float)v[c] + (float)d[c] + (float)l[c];
  if (acc == 1.2345f) out[0] = acc;
}
int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount, clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *names[] = {"MUFU.RCP", "I2F.F64.S64+F2I.S64.F64", "I2F.F64.S32+F2I.S32.F64", "F2F.F32.F64+F2F.F64.F32",
                         "I2F.F32+F2I.F32", "FRND.F32 (+FMUL)", "FRND.F64 floor (+DMUL)", "sincospif (1 per step)",
                         "floor->S64->F64", "DFMA"};
  void (*ks[])(float *, int) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>};
  for (int op = 0; op < 10; ++op) {
    int blocks = sms * 8, threads = 256;
    ks[op]<<<blocks, threads>>>(out, 1);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    ks[op]<<<blocks, threads>>>(out, 2);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double steps = (double)blocks * threads * ITERS * 8;  // chain steps (2 ops each, except sincospif)
    double per_clk_sm = steps / (ms * 1e-3) / (sms * clk * 1e3);
    printf("%-28s %.2f steps/clk/SM  (%.2f ops/clk/SM at 2 ops/step)\n", names[op], per_clk_sm, 2 * per_clk_sm);
  }
  return 0;
}
