// Throw-away microbenchmarks: true L2 bandwidth (in-kernel repeated passes), graph launch gaps.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

// each CTA owns a fixed slice; reads+writes it `passes` times (slice-local so no inter-CTA hazards)
__global__ void l2_rw(float4 *buf, size_t n, int passes) {
  size_t per = n / gridDim.x;
  float4 *s = buf + per * blockIdx.x;
  for (int p = 0; p < passes; ++p) {
    for (size_t i = threadIdx.x; i < per; i += blockDim.x * 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { size_t j = i + u * blockDim.x; if (j < per) v[u] = __ldcg(s + j); }
#pragma unroll
      for (int u = 0; u < 4; ++u) { size_t j = i + u * blockDim.x; if (j < per) { v[u].x += 1.f; __stcg(s + j, v[u]); } }
    }
    __syncthreads();
  }
}
__global__ void l2_r(const float4 *buf, size_t n, int passes, float *out) {
  // read a DIFFERENT CTA's slice each pass so L1 can't serve it
  size_t per = n / gridDim.x;
  float acc = 0;
  for (int p = 0; p < passes; ++p) {
    const float4 *s = buf + per * ((blockIdx.x + p * 37) % gridDim.x);
    for (size_t i = threadIdx.x; i < per; i += blockDim.x * 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) { size_t j = i + u * blockDim.x; if (j < per) { float4 v = __ldcg(s + j); acc += v.x + v.w; } }
    }
  }
  if (acc == 1.2345f) out[0] = acc;
}
__global__ void small_kernel(float *p) { if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1; }

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  float4 *buf; CK(cudaMalloc(&buf, (size_t)256 << 20)); cudaMemset(buf, 0, (size_t)256 << 20);
  float *out; CK(cudaMalloc(&out, 1024));
  for (size_t mb : {8, 16, 32, 48, 64, 96, 128, 256}) {
    size_t n = (mb << 20) / 16;
    for (int bpsm : {1, 2, 4}) {
      int passes = mb <= 64 ? 50 : 10;
      l2_rw<<<sms * bpsm, 512>>>(buf, n, 2);
      cudaEventRecord(e0); l2_rw<<<sms * bpsm, 512>>>(buf, n, passes); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("l2_rw %4zu MiB b/SM %d: %.1f GB/s (r+w)\n", mb, bpsm, 2.0 * (mb << 20) * passes / ms / 1e6);
      cudaEventRecord(e0); l2_r<<<sms * bpsm, 512>>>(buf, n, passes, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("l2_r  %4zu MiB b/SM %d: %.1f GB/s (read)\n", mb, bpsm, 1.0 * (mb << 20) * passes / ms / 1e6);
    }
  }
  // launch gaps: stream vs graph
  cudaStream_t st; cudaStreamCreate(&st);
  for (int r = 0; r < 2; ++r) {
    cudaEventRecord(e0, st); for (int i = 0; i < 200; ++i) small_kernel<<<sms, 128, 0, st>>>(out); cudaEventRecord(e1, st); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("stream launches: %.2f us/kernel\n", ms * 1000 / 200);
  }
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 200; ++i) small_kernel<<<sms, 128, 0, st>>>(out);
  cudaStreamEndCapture(st, &g);
  CK(cudaGraphInstantiate(&ge, g, 0));
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("graph launches: %.2f us/kernel\n", ms * 1000 / 200);
  }
  CK(cudaGetLastError());
  return 0;
}
