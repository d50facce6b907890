// launch_cache.cu -- host-side launch preparation of every kernel, cached per (kernel, device, block
// size, dynamic shared memory): cudaFuncSetAttribute and the occupancy query cost microseconds per call,
// which dominated the single-pulse latency of the API (each call launches 1-4 kernels).
#include "dc_kernels.h"

#include <mutex>
#include <unordered_map>

namespace dc {

namespace {
struct Key {
  const void *fn;
  int dev, threads;
  size_t smem;
  bool operator==(const Key &o) const { return fn == o.fn && dev == o.dev && threads == o.threads && smem == o.smem; }
};
struct KeyHash {
  size_t operator()(const Key &k) const {
    return std::hash<const void *>()(k.fn) ^ (std::hash<size_t>()(k.smem) * 31u) ^ ((size_t)k.dev << 48) ^
           ((size_t)k.threads << 32);
  }
};
std::mutex g_mu;
std::unordered_map<Key, LaunchShape, KeyHash> g_cache;
}  // namespace

cudaError_t launch_shape(const void *fn, int threads, size_t smem, LaunchShape *out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const Key k{fn, dev, threads, smem};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(k);
    if (it != g_cache.end()) {
      *out = it->second;
      return cudaSuccess;
    }
  }
  if (smem > 0 && (e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
    return e;
  LaunchShape s{148, 1};
  if ((e = cudaDeviceGetAttribute(&s.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s.per_sm, fn, threads, smem)) != cudaSuccess) return e;
  if (s.per_sm < 1) s.per_sm = 1;
  std::lock_guard<std::mutex> lk(g_mu);
  g_cache[k] = s;
  *out = s;
  return cudaSuccess;
}

}  // namespace dc
