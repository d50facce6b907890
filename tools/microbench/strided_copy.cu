// Strided-tile copy microbenchmark: bandwidth of copying a [P][1024][1024] complex64 array in
// column tiles [1024 rows][C columns] (C*8-byte row segments, 8 KiB row stride) vs contiguous.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void tile_copy(const float4 *__restrict__ x, float4 *__restrict__ y, long tiles) {
  // a CTA copies tile t: rows 0..1023, float4 columns c0/2 .. (c0+C)/2
  constexpr int V = C / 2;  // float4 per row segment
  for (long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const long p = t / (1024 / C), c = (t % (1024 / C)) * V;
    const float4 *src = x + p * 1024 * 512 + c;
    float4 *dst = y + p * 1024 * 512 + c;
    for (int i = threadIdx.x; i < 1024 * V; i += blockDim.x) {
      const int row = i / V, col = i % V;
      __stcg(dst + (long)row * 512 + col, __ldcg(src + (long)row * 512 + col));
    }
  }
}
int main() {
  const long P = 64, N = P * 1024 * 1024;
  float4 *x, *y;
  cudaMalloc(&x, N * 8);
  cudaMalloc(&y, N * 8);
  cudaMemset(x, 0, N * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto kern, int C, int grid, int thr) {
    const long tiles = P * (1024 / C);
    for (int w = 0; w < 3; ++w) kern<<<grid, thr>>>(x, y, tiles);
    cudaEventRecord(a);
    for (int w = 0; w < 10; ++w) kern<<<grid, thr>>>(x, y, tiles);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("C=%3d grid=%4d thr=%d  %.1f GB/s\n", C, grid, thr, 2.0 * N * 8 * 10 / (ms * 1e-3) / 1e9);
  };
  for (int g : {148, 296, 592, 1184}) {
    run(tile_copy<8>, 8, g, 256);
    run(tile_copy<16>, 16, g, 256);
    run(tile_copy<32>, 32, g, 256);
    run(tile_copy<1024>, 1024, g, 256);
  }
  return 0;
}
