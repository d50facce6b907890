// Standalone check of the TMA path used by the doppler staging: 2-D map {n, pulses} of 8-byte
// elements, box {256, 1}, coordinates including negative and past-the-end (zero fill).
#include <cstdio>
#include <vector>
#include "../../paper_2508_04951_b200/csrc/tma.cuh"
#include "../../paper_2508_04951_b200/csrc/tma_host.h"
using namespace dc;

__global__ void k(const __grid_constant__ CUtensorMap map, int c0, int c1, int nb, unsigned long long *out) {
  extern __shared__ __align__(1024) unsigned long long buf[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_proxy_async();
    mbar_arrive_expect_tx(&bar, nb * 256 * 8);
    for (int i = 0; i < nb; ++i) tma_load_2d(buf + i * 256, &map, c0 + 256 * i, c1, &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < nb * 256; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char **argv) {
  const int n = 4096, pulses = 3;
  std::vector<unsigned long long> h(n * pulses);
  for (int p = 0; p < pulses; ++p)
    for (int i = 0; i < n; ++i) h[p * n + i] = (unsigned long long)p * 100000 + i + 1;
  unsigned long long *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 16 * 256 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  CUtensorMap map;
  const uint64_t dims[2] = {(uint64_t)n, (uint64_t)pulses};
  const uint64_t strides[1] = {(uint64_t)n * 8};
  const uint32_t box[2] = {256, 1};
  if (!encode_tile_map(&map, d, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE)) { printf("encode failed\n"); return 1; }
  int cases[][3] = {{0, 0, 4}, {-2, 0, 4}, {-2, 2, 10}, {2302, 1, 10}, {2304, 2, 10}, {-18, 2, 3}, {4000, 2, 3}};
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 256 * 8);
  for (auto &c : cases) {
    k<<<1, 128, 16 * 256 * 8>>>(map, c[0], c[1], c[2], o);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("case %d %d %d: %s\n", c[0], c[1], c[2], cudaGetErrorString(e)); return 1; }
    std::vector<unsigned long long> r(c[2] * 256);
    cudaMemcpy(r.data(), o, r.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < c[2] * 256; ++i) {
      long long k = c[0] + i;
      unsigned long long want = (k >= 0 && k < n) ? h[c[1] * n + k] : 0;
      bad += r[i] != want;
    }
    printf("case c0=%d c1=%d nb=%d: %d mismatches\n", c[0], c[1], c[2], bad);
  }
  return 0;
}
