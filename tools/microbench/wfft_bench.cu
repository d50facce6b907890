// Pure-compute throughput of the warp-level 1024-point FFT (forward + inverse) with no global
// memory in the loop: tells whether the FFT arithmetic itself or the memory/phase/boundary work
// limits the four-step row pass.
#include <cstdio>
#include "../../paper_2508_04951_b200/csrc/wfft.cuh"
using namespace dc;

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) bench(float2 *out, const float4 *tw, int iters) {
  extern __shared__ float4 dyn[];
  float4 *Tw = dyn;
  float2 *wks = reinterpret_cast<float2 *>(dyn + 512);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 512; i += NW * 32) Tw[i] = tw[i];
  __syncthreads();
  float2 v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = make_float2(lane * 0.01f + r, r * 0.5f);
  for (int it = 0; it < iters; ++it) {
    wfft1024<false>(v, wks + warp * kWPad, Tw, lane);
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r] = cscale(v[r], 1.0f / 1024.0f);
    wfft1024<true>(v, wks + warp * kWPad, Tw, lane);
  }
  float2 acc = make_float2(0, 0);
#pragma unroll
  for (int r = 0; r < 32; ++r) acc = cadd(acc, v[r]);
  out[blockIdx.x * NW * 32 + threadIdx.x] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float4 *tw; cudaMalloc(&tw, 512 * 16); cudaMemset(tw, 0, 512 * 16);
  float2 *out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 200;
    cudaEventRecord(e0);
    cudaFuncSetAttribute(bench<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 512 * 16 + 8 * kWPad * 8);
    cudaFuncSetAttribute(bench<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 512 * 16 + 16 * kWPad * 8);
    bench<8><<<sms, 256, 512 * 16 + 8 * kWPad * 8>>>(out, tw, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double samples = (double)sms * 8 * iters * 1024;  // fwd+inv pairs per sample
    printf("8 warps/SM: %.1f G samples/s (fwd+inv 1024-pt per sample), %.1f us\n", samples / ms / 1e6, ms * 1e3);
    cudaEventRecord(e0);
    bench<16><<<sms, 512, 512 * 16 + 16 * kWPad * 8>>>(out, tw, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    samples = (double)sms * 16 * iters * 1024;
    printf("16 warps/SM: %.1f G samples/s, %.1f us\n", samples / ms / 1e6, ms * 1e3);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
