// Throw-away microbenchmarks used to size the design (pipe rates, L2 bandwidth).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int OP>
__global__ void pipe_kernel(float *out, float a, float b, int iters) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  float y = a, z = b;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) { // FFMA 3-reg
        x0 = fmaf(x0, y, z); x1 = fmaf(x1, y, z); x2 = fmaf(x2, y, z); x3 = fmaf(x3, y, z);
        x4 = fmaf(x4, y, z); x5 = fmaf(x5, y, z); x6 = fmaf(x6, y, z); x7 = fmaf(x7, y, z);
      } else if (OP == 1) { // FADD
        x0 = x0 + y; x1 = x1 + z; x2 = x2 + y; x3 = x3 + z; x4 = x4 + y; x5 = x5 + z; x6 = x6 + y; x7 = x7 + z;
      } else if (OP == 2) { // FMUL
        x0 = x0 * y; x1 = x1 * z; x2 = x2 * y; x3 = x3 * z; x4 = x4 * y; x5 = x5 * z; x6 = x6 * y; x7 = x7 * z;
      } else if (OP == 3) { // MUFU.RCP
        asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x0)); asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x1));
        asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x2)); asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x3));
        asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x4)); asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x5));
        asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x6)); asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x7));
      } else if (OP == 5) { // FFMA with x*x+x pattern (3 distinct regs)
        x0 = fmaf(x0, x1, x2); x1 = fmaf(x1, x2, x3); x2 = fmaf(x2, x3, x4); x3 = fmaf(x3, x4, x5);
        x4 = fmaf(x4, x5, x6); x5 = fmaf(x5, x6, x7); x6 = fmaf(x6, x7, x0); x7 = fmaf(x7, x0, x1);
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dfma_kernel(double *out, double a, double b, int iters) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4=x0+4,x5=x0+5,x6=x0+6,x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3+x4+x5+x6+x7;
}

__global__ void copy_kernel(const float4 *__restrict__ a, float4 *__restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("dev %s SMs %d l2 %d smemOptin %zu clock %d kHz\n", p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.clockRate);
  int sms = p.multiProcessorCount;
  float *out; CK(cudaMalloc(&out, sizeof(double) * 1024 * sms * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *names[] = {"FFMA(a,b const)", "FADD", "FMUL", "MUFU.RCP", "", "FFMA(3 distinct reg)"};
  int iters = 4096;
  for (int op : {0, 1, 2, 3, 5}) {
    for (int rep = 0; rep < 2; ++rep) {
      int blocks = sms * 4, threads = 512;
      cudaEventRecord(e0);
      if (op == 0) pipe_kernel<0><<<blocks, threads>>>(out, 1.0001f, 1e-7f, iters);
      if (op == 1) pipe_kernel<1><<<blocks, threads>>>(out, 1.0001f, 1e-7f, iters);
      if (op == 2) pipe_kernel<2><<<blocks, threads>>>(out, 1.0001f, 1e-7f, iters);
      if (op == 3) pipe_kernel<3><<<blocks, threads>>>(out, 1.0001f, 1e-7f, iters);
      if (op == 5) pipe_kernel<5><<<blocks, threads>>>(out, 1.0001f, 1e-7f, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 64;
      if (rep) printf("%-22s %.1f Gop/s (lane-ops)  = %.1f per SM per ns\n", names[op], ops / ms / 1e6, ops / ms / 1e6 / sms);
    }
  }
  for (int rep = 0; rep < 2; ++rep) {
    int blocks = sms * 4, threads = 512;
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>((double*)out, 1.0000001, 1e-9, iters / 4);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * (iters / 4) * 64;
    if (rep) printf("%-22s %.1f Gop/s (lane-ops)  = %.1f per SM per ns\n", "DFMA", ops / ms / 1e6, ops / ms / 1e6 / sms);
  }
  // bandwidth: various working-set sizes (read+write bytes)
  size_t maxb = (size_t)2 << 30;
  float4 *a, *b; CK(cudaMalloc(&a, maxb)); CK(cudaMalloc(&b, maxb));
  cudaMemset(a, 0, maxb); cudaMemset(b, 0, maxb);
  for (size_t bytes : {(size_t)4 << 20, (size_t)8 << 20, (size_t)16 << 20, (size_t)32 << 20, (size_t)48 << 20, (size_t)64 << 20, (size_t)128 << 20, (size_t)1 << 30, (size_t)2 << 30}) {
    size_t n = bytes / 16;
    int reps = bytes >= ((size_t)1 << 30) ? 5 : 50;
    for (int threads : {256}) for (int bpsm : {4, 8}) {
      copy_kernel<<<sms * bpsm, threads>>>(a, b, n);
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) copy_kernel<<<sms * bpsm, threads>>>(a, b, n);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("copy %6zu MiB/dir blocks/SM %d: %.1f GB/s (r+w)\n", bytes >> 20, bpsm, 2.0 * bytes * reps / ms / 1e6);
    }
  }
  return 0;
}
