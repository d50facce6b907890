// FFMA2 / FADD2 vs FFMA throughput on sm_100a (packed f32x2 PTX ops).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { float2 v = make_float2(a, b); return *reinterpret_cast<u64*>(&v); }
template <int OP>
__global__ void k(float *o, float a, float b, int it) {
  u64 x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = pk(threadIdx.x + j, j);
  float s[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) s[j] = threadIdx.x + j;
  u64 A = pk(a, a), B = pk(b, b);
  for (int i = 0; i < it; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[j]) : "l"(A), "l"(B));
      if (OP == 1) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x[j]) : "l"(A));
      if (OP == 2) { s[2*j] = fmaf(s[2*j], a, b); s[2*j+1] = fmaf(s[2*j+1], a, b); }
      if (OP == 3) asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(x[j]) : "l"(x[(j+1)&7]));
    }
  }
  float acc = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) { float2 v = *reinterpret_cast<float2*>(&x[j]); acc += v.x + v.y; }
#pragma unroll
  for (int j = 0; j < 16; ++j) acc += s[j];
  o[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *o; cudaMalloc(&o, 1 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *nm[] = {"FFMA2 (bcast)", "FADD2", "FFMA x2 scalar", "FFMA2 (3 vec regs)"};
  for (int op = 0; op < 4; ++op) for (int r = 0; r < 2; ++r) {
    int it = 4096, blocks = sms * 4, th = 512;
    cudaEventRecord(e0);
    if (op == 0) k<0><<<blocks, th>>>(o, 1.0001f, 1e-7f, it);
    if (op == 1) k<1><<<blocks, th>>>(o, 1.0001f, 1e-7f, it);
    if (op == 2) k<2><<<blocks, th>>>(o, 1.0001f, 1e-7f, it);
    if (op == 3) k<3><<<blocks, th>>>(o, 1.0001f, 1e-7f, it);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops_lanes = (double)blocks * th * it * 16;  // scalar-FMA-equivalents (16 per iteration)
    if (r) printf("%-20s %.1f T scalar-ops/s = %.1f per SM per clk @1.965\n", nm[op], flops_lanes / ms / 1e9, flops_lanes / ms / 1e6 / sms / 1965.0 * 1e3 / 1e3);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
