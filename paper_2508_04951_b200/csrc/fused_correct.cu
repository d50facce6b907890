// fused_correct.cu -- one persistent kernel for the whole dc_correct of 2^20-sample pulses.
//
// The pulse train is cut into groups of Pg pulses.  Each group is four stages of work items:
//   A  column tiles   [1024][8]  x -> ring      forward 1024-point column DFTs, x w_n^(k1 t2) / n
//   B  row items      8 rows     ring -> ring   forward DFT -> Eq. 15 phase -> inverse DFT, x conj tw
//   C  column tiles   [1024][8]  ring -> ring   inverse column DFTs (ionospheric result, natural order)
//   D  doppler tiles  2304 out   ring -> y      windowed-sinc resampling onto t/alpha (Eq. 16)
// and the ring holds `depth` groups (L2-sized), so the ionospheric intermediate of a group never
// has to leave L2.  Work items are handed out in order by one global atomic counter, in a lagged
// wavefront: step t holds stage A of group t, B of t-L, C of t-2L and D of t-3L (lag L), interleaved
// round-robin, so memory-bound column tiles co-run with compute-bound rows and doppler tiles and
// every dependency was produced L steps earlier.  An item waits (acquire-polling a per-group,
// per-stage completion counter) only for items handed out earlier to running CTAs -- so the
// schedule cannot deadlock.  Each CTA is warp-specialised: one producer lane claims items, waits
// for their inputs, issues their TMA / bulk loads into one of two staging slots (full/empty
// mbarrier pairs) and publishes completions; eight consumer warps only compute, so claim, poll
// and fence latencies stay off the compute path, and the tail of one stage is filled with work
// of the next stage or group instead of an idle GPU between kernel launches.
#include <algorithm>

#include "dc_kernels.h"
#include "doppler_tile.cuh"
#include "tma.cuh"
#include "tma_host.h"
#include "wfft.cuh"

namespace dc {

constexpr int kFT = 256;  // consumer threads (8 warps); + 1 producer warp
constexpr int kNS = 3;    // staging slots
// one slot: the 64 KiB input tile, then reused in place as the 8 warps' padded FFT exchange
// buffers (8 x kWPad) or, for a doppler tile, its output staging at +32 KiB; 1 KiB multiple
constexpr int kSlotElems = ((kWW * kWPad * 8 + 1023) / 1024) * 1024 / 8;

struct FusedArgs {
  float2 *y;
  float2 *ring;  // [depth * Pg][n] ionospheric intermediate
  int64_t pulses, ngroups;
  int Pg, depth, lag, hints;
  const PulseParams *pp;
  const float2 *tw;    // 1024-point pass-2 twiddles, float4 [r/2][k]
  const float2 *gtab;  // 1/f_k FP32 pairs, row layout [k1][k2]
  int W;
  double carrier;  // fc / fs
  float scale;     // 1/n
  unsigned long long *counter;
  unsigned *done;  // [ngroups][4]
  unsigned long long *stats;  // optional [grid][16] cycle counters (DISPCORR_FUSED_STATS), else null
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }


struct Item {
  int64_t g;   // group
  int stage;   // 0 A, 1 B, 2 C, 3 D, -1 none
  int64_t idx;  // index inside the stage
  int lp;      // local pulse in the group
  int64_t sub;  // tile/column-group/row-group index inside the pulse
  bool skip;   // pulse past the end of the train (last, partial group)
};

template <bool SECOND, int WT>
__global__ void __launch_bounds__(kFT + 32, 1)
    fused_correct_kernel(const FusedArgs a, const __grid_constant__ CUtensorMap mapA,
                         const __grid_constant__ CUtensorMap mapC, const __grid_constant__ CUtensorMap mapD) {
  extern __shared__ __align__(1024) float4 smem4[];
  float2 *sm = reinterpret_cast<float2 *>(smem4);
  auto slot = [sm](int i) { return sm + i * kSlotElems; };
  float2 *Pwall = sm + kNS * kSlotElems;
  float4 *Tw = reinterpret_cast<float4 *>(Pwall + kWW * 32);
  uint64_t *full = reinterpret_cast<uint64_t *>(reinterpret_cast<float2 *>(Tw) + 1024);  // [kNS] loads landed
  uint64_t *empty = full + kNS;                                                          // [kNS] slot consumed
  long long *itemq = reinterpret_cast<long long *>(empty + kNS);                         // [kNS] item in slot
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int log2n = 20;
  constexpr int n = 1 << 20;
  constexpr uint32_t nmask = n - 1u;
  const int Pg = a.Pg;
  const int64_t NA = (int64_t)Pg * 128, NB = NA, NC = NA;
  const int64_t dtiles = (n + kDopM - 1) / kDopM;
  const int64_t ND = (int64_t)Pg * dtiles;
  const int kLag = a.lag;  // steps between dependent stages of a group
  const int64_t per_step = NA + NB + NC + ND;
  const int64_t total = per_step * (a.ngroups + 3 * kLag);

  auto decode = [&](int64_t q) {
    Item it;
    const int64_t t = q / per_step;
    int64_t r = q - t * per_step;
    if (r < 4 * NA) {  // round-robin A, B, C, D while all four kinds have items (NA = NB = NC <= ND)
      it.stage = (int)(r & 3);
      r >>= 2;
    } else {
      it.stage = 3;
      r = NA + (r - 4 * NA);
    }
    it.g = t - kLag * it.stage;
    it.idx = r;
    const int64_t per_pulse = (it.stage == 3) ? dtiles : 128;
    it.lp = (int)(r / per_pulse);
    it.sub = r - (int64_t)it.lp * per_pulse;
    it.skip = (it.g < 0) || (it.g >= a.ngroups) || (it.g * Pg + it.lp >= a.pulses);
    return it;
  };
  auto ring_pulse = [&](const Item &it) { return (int)((it.g % a.depth) * Pg + it.lp); };

  // ---- prologue: tables, barriers
  for (int i = tid; i < 512; i += kFT + 32) Tw[i] = reinterpret_cast<const float4 *>(a.tw)[i];
  if (tid == 0) {
    for (int i = 0; i < kNS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kWW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == kWW) {
    // ================= producer warp (one lane): claims items in order, waits for their inputs,
    // issues their TMA / bulk loads into a free slot, and publishes completions of consumed items.
    if (lane != 0) return;
    // completion counter an item depends on (stage A of group g depends on stage D of g - depth)
    auto dep = [&](const Item &it, const unsigned **ctr, unsigned *req) {
      if (it.g < 0 || it.g >= a.ngroups) return false;
      if (it.stage == 0) {
        if (it.g < a.depth) return false;
        *ctr = a.done + (it.g - a.depth) * 4 + 3;
        *req = (unsigned)ND;  // all doppler tiles of the group that used this ring slot
        return true;
      }
      *ctr = a.done + it.g * 4 + (it.stage - 1);
      *req = (unsigned)NA;  // NA = NB = NC items in the previous stage
      return true;
    };
    // the consumers' stores of item q happen before (empty-barrier acquire at CTA scope) this
    // thread's cumulative gpu-scope fence, which precedes the counter increment
    auto signal = [&](long long q) {
      const Item it = decode(q);
      if (it.g < 0 || it.g >= a.ngroups) return;
      __threadfence();
      atomicAdd(a.done + it.g * 4 + it.stage, 1u);
    };
    // slots whose item awaits its completion signal (bit i; the item id stays in itemq[i]);
    // empty-barrier parities as bits
    unsigned pendmask = 0u, eph = 0u;
    auto service = [&] {  // signal every consumed item without blocking
      for (int i = 0; i < kNS; ++i)
        if (((pendmask >> i) & 1u) && mbar_test(&empty[i], (eph >> i) & 1u)) {
          eph ^= 1u << i;
          pendmask &= ~(1u << i);
          signal(itemq[i]);
        }
    };
    auto wait_free = [&](int i) -> long long {  // block until slot i is consumed; return its item (-1: none)
      if (!((pendmask >> i) & 1u)) return -1;
      mbar_wait(&empty[i], (eph >> i) & 1u);
      eph ^= 1u << i;
      pendmask &= ~(1u << i);
      return itemq[i];
    };
    const uint64_t pol_first = policy_evict_first();
    int s = 0;
    long long q = (long long)atomicAdd(a.counter, 1ull);
    while (q < total) {
      const Item it = decode(q);
      const unsigned *c;
      unsigned r;
      const long long tp0 = clock64();
      if (dep(it, &c, &r)) {
        const long long t0 = clock64();
        while (ld_acquire(c) < r) {
          service();  // never sit on a finished item while waiting: another CTA may need it
          __nanosleep(64);
          if (clock64() - t0 > (8ll << 30)) __trap();  // ~4 s: a broken schedule must not hang the GPU
        }
      }
      const long long tp1 = clock64();
      const long long old = wait_free(s);
      if (a.stats) {
        a.stats[blockIdx.x * 16 + 8] += tp1 - tp0;
        a.stats[blockIdx.x * 16 + 9] += clock64() - tp1;
      }
      itemq[s] = q;
      if (it.skip) {
        mbar_arrive(&full[s]);
      } else {
        fence_proxy_async_global();
        fence_proxy_async();
        uint64_t *bar = &full[s];
        float2 *dst = slot(s);
        if (it.stage == 0 || it.stage == 2) {
          mbar_arrive_expect_tx(bar, 8192 * sizeof(float2));
          const CUtensorMap *m = (it.stage == 0) ? &mapA : &mapC;
          const int pc = (it.stage == 0) ? (int)(it.g * Pg + it.lp) : ring_pulse(it);
          if (it.stage == 0 && (a.hints & 1)) {
#pragma unroll
            for (int b = 0; b < 4; ++b) tma_load_3d_hint(dst + b * 256 * 8, m, (int)(it.sub * 8), b * 256, pc, bar, pol_first);
          } else {
#pragma unroll
            for (int b = 0; b < 4; ++b) tma_load_3d(dst + b * 256 * 8, m, (int)(it.sub * 8), b * 256, pc, bar);
          }
        } else if (it.stage == 1) {
          mbar_arrive_expect_tx(bar, 8192 * sizeof(float2));
          const float2 *src = a.ring + (int64_t)ring_pulse(it) * n + it.sub * 8 * 1024;
#pragma unroll
          for (int w = 0; w < 8; ++w) bulk_load(dst + w * 1024, src + w * 1024, 1024 * sizeof(float2), bar);
        } else {
          DopTile tr = dop_tile(it.sub, dtiles, a.W, a.pp, it.g * Pg + it.lp);
          tr.pulse = ring_pulse(it);
          const int nb = dop_nbox(tr);
          mbar_arrive_expect_tx(bar, (unsigned)(nb * kDopBox * sizeof(float2)));
          if (a.hints & 4) {
            for (int i = 0; i < nb; ++i)
              tma_load_2d_hint(dst + i * kDopBox, &mapD, (int)(tr.Bcta + i * kDopBox), tr.pulse, bar, pol_first);
          } else {
            for (int i = 0; i < nb; ++i) tma_load_2d(dst + i * kDopBox, &mapD, (int)(tr.Bcta + i * kDopBox), tr.pulse, bar);
          }
        }
      }
      pendmask |= 1u << s;
      q = (long long)atomicAdd(a.counter, 1ull);  // in flight while the previous item is signalled
      if (old >= 0) signal(old);                  // the fence is paid after the next loads are issued
      s = (s + 1 == kNS) ? 0 : s + 1;
    }
    // end of the queue: hand the consumers a sentinel in their next slot, then signal the rest
    {
      const long long old = wait_free(s);
      if (old >= 0) signal(old);
      itemq[s] = total;
      mbar_arrive(&full[s]);
      for (int i = 0; i < kNS; ++i) {
        const long long o = wait_free(i);
        if (o >= 0) signal(o);
      }
    }
    return;
  }

  // ================= consumer warps 0 .. kWW-1
  float2 *Pw = Pwall + warp * 32;
  auto consumers_sync = [] { asm volatile("bar.sync 1, %0;\n" ::"n"(kFT) : "memory"); };
  const bool keep = (a.hints & 2) != 0;  // ring stores with the evict_last policy
  const uint64_t pol_last = policy_evict_last();
  int s = 0;
  unsigned fph = 0u;  // full-barrier parities as bits
  long long tc = clock64();
  while (true) {
    mbar_wait(&full[s], (fph >> s) & 1u);
    fph ^= 1u << s;
    const long long q = *reinterpret_cast<volatile long long *>(&itemq[s]);
    if (q >= total) break;
    const Item it = decode(q);
    const long long tc1 = clock64();
    if (a.stats && tid == 0) a.stats[blockIdx.x * 16 + 0] += tc1 - tc;
    float2 *sb = slot(s);
    float2 *wk = sb + warp * kWPad;  // in-place exchange buffer once the tile is in registers
    if (!it.skip) {
      const int64_t gp = it.g * Pg + it.lp;  // global pulse
      float2 *rp = a.ring + (int64_t)ring_pulse(it) * n;
      if (it.stage == 0 || it.stage == 2) {
        // ---- column tile: warp w transforms column t2 = 8 sub + w
        float2 v[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = sb[col_sw(lane + 32 * r, warp)];
        consumers_sync();  // the whole tile is in registers: the slot becomes exchange space
        const uint32_t t2 = (uint32_t)(it.sub * 8 + warp);
        if (it.stage == 0) {
          wfft1024<false>(v, wk, Tw, lane);
          __syncwarp();
          Pw[lane] = twn((32u * t2 * (uint32_t)lane) & nmask, log2n);
          const float2 base = cscale(twn((t2 * (uint32_t)lane) & nmask, log2n), a.scale);
          __syncwarp();
#pragma unroll
          for (int q2 = 0; q2 < 32; ++q2) v[q2] = cmul(v[q2], cmul(base, Pw[q2]));
        } else {
          wfft1024<true>(v, wk, Tw, lane);
        }
        __syncwarp();
#pragma unroll
        for (int q2 = 0; q2 < 32; ++q2) wk[wpad(lane + 32 * q2)] = v[q2];
        consumers_sync();
        float2 *g = rp + it.sub * 8;
#pragma unroll 4
        for (int i = tid; i < 1024 * 4; i += kFT) {
          const int row = i >> 2, v4 = i & 3;
          const float2 e0 = sb[(2 * v4) * kWPad + wpad(row)];
          const float2 e1 = sb[(2 * v4 + 1) * kWPad + wpad(row)];
          float4 *dst = reinterpret_cast<float4 *>(g + (int64_t)row * 1024 + 2 * v4);
          if (keep) {
            st_hint(dst, make_float4(e0.x, e0.y, e1.x, e1.y), pol_last);
          } else {
            __stcg(dst, make_float4(e0.x, e0.y, e1.x, e1.y));
          }
        }
      } else if (it.stage == 1) {
        // ---- row k1 = 8 sub + w: forward DFT -> phase -> inverse DFT -> conj outer twiddle
        const uint32_t k1 = (uint32_t)(it.sub * 8 + warp);
        float2 v[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = sb[warp * 1024 + lane + 32 * r];
        consumers_sync();  // rows in registers: the slot becomes exchange space
        wfft1024<false>(v, wk, Tw, lane);
        {
          const PulseParams pr = a.pp[gp];
          const float2 *grow = a.gtab + (int64_t)k1 * 1024;
#pragma unroll
          for (int q2 = 0; q2 < 32; ++q2) {
            const float rf = phase_frac(pr.nu_hi, pr.nu_lo, __ldg(grow + lane + 32 * q2));
            v[q2] = cmul(v[q2], expm2pi(rf));
          }
        }
        wfft1024<true>(v, wk, Tw, lane);
        __syncwarp();
        Pw[lane] = twn((32u * k1 * (uint32_t)lane) & nmask, log2n);
        const float2 base = twn((k1 * (uint32_t)lane) & nmask, log2n);
        __syncwarp();
        float2 *out = rp + (int64_t)k1 * 1024;
#pragma unroll
        for (int q2 = 0; q2 < 32; ++q2) {
          const float2 o = cmulc(v[q2], cmul(base, Pw[q2]));
          if (keep) {
            st_hint(out + lane + 32 * q2, o, pol_last);
          } else {
            __stcg(out + lane + 32 * q2, o);
          }
        }
      } else {
        // ---- doppler tile from the slot into y (output staged at +32 KiB of the slot)
        DopTile c2 = dop_tile(it.sub, dtiles, a.W, a.pp, gp);
        c2.pulse = 0;  // y is pre-offset to this pulse below
        dop_tile_compute<SECOND, WT, 1>(sb, c2, a.W, sb + 4096, a.y + gp * (int64_t)n, n, a.carrier);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    tc = clock64();
    if (a.stats && tid == 0) {
      a.stats[blockIdx.x * 16 + 1 + it.stage] += tc - tc1;
      a.stats[blockIdx.x * 16 + 5 + (it.stage == 3 ? 1 : 0)] += 1;
    }
    s = (s + 1 == kNS) ? 0 : s + 1;
  }
}

// ----------------------------------------------------------------------------- host launcher
static size_t fused_smem() {
  return sizeof(float2) * ((size_t)kNS * kSlotElems + kWW * 32 + 1024) + 2 * kNS * sizeof(uint64_t) +
         kNS * sizeof(long long) + 1024;
}

template <bool SECOND, int WT>
static cudaError_t launch_fused_t(const FusedLaunch &f, const CUtensorMap &mA, const CUtensorMap &mC,
                                  const CUtensorMap &mD, const FusedArgs &a) {
  auto kern = fused_correct_kernel<SECOND, WT>;
  const size_t smem = fused_smem();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  kern<<<(unsigned)sms, kFT + 32, smem, f.stream>>>(a, mA, mC, mD);
  return cudaGetLastError();
}

cudaError_t launch_fused_correct(const FusedLaunch &f, double max_abs_beta_m1) {
  const int path = doppler_path(max_abs_beta_m1);
  if (path == 0) return cudaErrorNotSupported;
  constexpr int n = 1 << 20;
  FusedArgs a{};
  a.y = f.y;
  a.ring = f.ring;
  a.pulses = f.pulses;
  a.Pg = f.Pg;
  a.lag = f.lag;
  a.hints = f.hints;
  a.stats = f.stats;
  a.depth = f.depth;
  a.ngroups = (f.pulses + f.Pg - 1) / f.Pg;
  a.pp = f.pp;
  a.tw = f.tw1024;
  a.gtab = f.gtab;
  a.W = f.taps;
  a.carrier = f.carrier;
  a.scale = 1.0f / (float)n;
  a.counter = f.sync;
  a.done = reinterpret_cast<unsigned *>(f.sync + 1);
  cudaError_t e = cudaMemsetAsync(f.sync, 0, sizeof(unsigned long long) + sizeof(unsigned) * 4 * a.ngroups, f.stream);
  if (e != cudaSuccess) return e;
  CUtensorMap mA, mC, mD;
  {
    const uint64_t dims[3] = {1024, 1024, (uint64_t)f.pulses};
    const uint64_t strides[2] = {1024 * sizeof(float2), (uint64_t)n * sizeof(float2)};
    const uint32_t box[3] = {8, 256, 1};
    if (!encode_tile_map(&mA, f.x, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B)) return cudaErrorInvalidValue;
    const uint64_t dimsC[3] = {1024, 1024, (uint64_t)f.Pg * f.depth};
    if (!encode_tile_map(&mC, f.ring, 3, dimsC, strides, box, CU_TENSOR_MAP_SWIZZLE_64B)) return cudaErrorInvalidValue;
    const uint64_t dimsD[2] = {(uint64_t)n, (uint64_t)f.Pg * f.depth};
    const uint64_t stridesD[1] = {(uint64_t)n * sizeof(float2)};
    const uint32_t boxD[2] = {(uint32_t)kDopBox, 1};
    if (!encode_tile_map(&mD, f.ring, 2, dimsD, stridesD, boxD, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
  }
  const bool second = path == 2;
  if (f.taps == 32) return second ? launch_fused_t<true, 32>(f, mA, mC, mD, a) : launch_fused_t<false, 32>(f, mA, mC, mD, a);
  return second ? launch_fused_t<true, 0>(f, mA, mC, mD, a) : launch_fused_t<false, 0>(f, mA, mC, mD, a);
}

}  // namespace dc
