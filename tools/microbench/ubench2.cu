// Throw-away microbenchmarks (round 1 design sizing): L2 copy/read BW with high MLP,
// launch overhead, MUFU rate, DSMEM bandwidth.
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int U>
__global__ void copyU(const float4 *__restrict__ a, float4 *__restrict__ b, size_t n) {
  size_t base = (blockIdx.x * (size_t)blockDim.x) * U + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (; base < n; base += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t i = base + u * blockDim.x; if (i < n) v[u] = a[i]; }
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t i = base + u * blockDim.x; if (i < n) b[i] = v[u]; }
  }
}
template<int U>
__global__ void readU(const float4 *__restrict__ a, float *out, size_t n) {
  size_t base = (blockIdx.x * (size_t)blockDim.x) * U + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x * U;
  float acc = 0;
  for (; base < n; base += stride) {
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t i = base + u * blockDim.x; if (i < n) { float4 v = a[i]; acc += v.x + v.y + v.z + v.w; } }
  }
  if (acc == 1234.5f) out[0] = acc;
}
__global__ void empty_kernel() {}
__global__ void mufu_kernel(float *out, int iters) {
  float x0 = 1.5f + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; ++i) {
    float r0, r1, r2, r3;
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(x0));
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(x1));
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(x2));
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r3) : "f"(x3));
    x0 += r0; x1 += r1; x2 += r2; x3 += r3;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
// DSMEM: each CTA of a cluster reads its neighbour's smem buffer repeatedly
template<int CS>
__global__ void __launch_bounds__(512) dsmem_kernel(float *out, int iters) {
  extern __shared__ float4 buf[];
  cg::cluster_group cl = cg::this_cluster();
  const int nel = 8192; // 128 KB
  for (int i = threadIdx.x; i < nel; i += blockDim.x) buf[i] = make_float4(i, 1, 2, 3);
  cl.sync();
  unsigned peer = (cl.block_rank() + 1) % CS;
  float4 *rb = cl.map_shared_rank(buf, peer);
  float acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int i = threadIdx.x; i < nel; i += blockDim.x) { float4 v = rb[i]; acc += v.x; }
  }
  cl.sync();
  if (acc == 1234.5f) out[0] = acc;
}
__global__ void __launch_bounds__(512) lsmem_kernel(float *out, int iters) {
  extern __shared__ float4 buf[];
  const int nel = 8192;
  for (int i = threadIdx.x; i < nel; i += blockDim.x) buf[i] = make_float4(i, 1, 2, 3);
  __syncthreads();
  float acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int i = threadIdx.x; i < nel; i += blockDim.x) { float4 v = buf[(i + it) & (nel-1)]; acc += v.x; }
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // launch overhead
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); for (int i = 0; i < 1000; ++i) empty_kernel<<<sms, 256>>>(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("empty kernel back-to-back: %.2f us/launch\n", ms);
  }
  float *out; CK(cudaMalloc(&out, 1 << 24));
  for (int r = 0; r < 2; ++r) {
    int iters = 1 << 14;
    cudaEventRecord(e0); mufu_kernel<<<sms * 4, 512>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * 4 * 512 * iters * 4;
    printf("MUFU.RCP: %.1f Gop/s = %.2f per SM per clk@1.965\n", ops / ms / 1e6, ops / ms / 1e6 / sms / 1.965);
  }
  size_t maxb = (size_t)1 << 30;
  float4 *a, *b; CK(cudaMalloc(&a, maxb)); CK(cudaMalloc(&b, maxb));
  cudaMemset(a, 0, maxb); cudaMemset(b, 0, maxb);
  for (size_t mb : {16, 24, 32, 48, 64, 1024}) {
    size_t bytes = mb << 20, n = bytes / 16;
    int reps = mb >= 1024 ? 5 : 100;
    for (int bpsm : {2, 4}) {
      copyU<4><<<sms * bpsm, 512>>>(a, b, n);
      cudaEventRecord(e0); for (int r = 0; r < reps; ++r) copyU<4><<<sms * bpsm, 512>>>(a, b, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("copyU4 %5zu MiB/dir b/SM %d: %.1f GB/s r+w  (%.2f us/launch)\n", mb, bpsm, 2.0 * bytes * reps / ms / 1e6, ms * 1000 / reps);
      readU<8><<<sms * bpsm, 512>>>(a, out, n);
      cudaEventRecord(e0); for (int r = 0; r < reps; ++r) readU<8><<<sms * bpsm, 512>>>(a, out, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("readU8 %5zu MiB     b/SM %d: %.1f GB/s read\n", mb, bpsm, 1.0 * bytes * reps / ms / 1e6);
    }
  }
  // smem/dsmem
  {
    int iters = 200;
    CK(cudaFuncSetAttribute(lsmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    CK(cudaFuncSetAttribute(dsmem_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    CK(cudaFuncSetAttribute(dsmem_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0); lsmem_kernel<<<sms, 512, 131072>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("local smem read: %.1f GB/s total, %.1f B/clk/SM\n", 131072.0 * iters * sms / ms / 1e6, 131072.0 * iters / (ms * 1e-3) / 1.965e9);
    }
    for (int cs : {2, 4}) for (int r = 0; r < 2; ++r) {
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(sms / cs * cs); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 131072;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaEventRecord(e0);
      if (cs == 2) CK(cudaLaunchKernelEx(&cfg, dsmem_kernel<2>, out, iters)); else CK(cudaLaunchKernelEx(&cfg, dsmem_kernel<4>, out, iters));
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      int g = sms / cs * cs;
      printf("DSMEM read cluster %d: %.1f GB/s total, %.1f B/clk/SM\n", cs, 131072.0 * iters * g / ms / 1e6, 131072.0 * iters / (ms * 1e-3) / 1.965e9);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
