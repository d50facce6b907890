// dispcorr_api.cu -- the libdispcorr C ABI (include/libdispcorr.h): validation, plans,
// parameter staging, chunk scheduling and kernel dispatch.  No computation of the method
// happens on the host except per-pulse scalars (2 K2 tec / c and beta = 1/alpha).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/libdispcorr.h"
#include "dc_kernels.h"

using dc::PulseParams;

namespace dc {
// per-pulse parameters from the raw host arrays (large batches): the host path's binary64
// arithmetic, term for term (nu_coef = k2c tec, its FP32 hi/lo split, beta = 1 / alpha)
__global__ void expand_params_kernel(const double *__restrict__ tec, const double *__restrict__ alpha,
                                     PulseParams *__restrict__ out, int64_t batch, double k2c, double k2pt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= batch) return;
  PulseParams q;
  q.nu_coef = tec ? __dmul_rn(k2c, tec[i]) : 0.0;
  q.k2 = tec ? __dmul_rn(k2pt, tec[i]) : 0.0;
  q.nu_hi = __double2float_rn(q.nu_coef);
  q.nu_lo = __double2float_rn(__dsub_rn(q.nu_coef, (double)q.nu_hi));
  q.beta = alpha ? __ddiv_rn(1.0, alpha[i]) : 1.0;
  out[i] = q;
}
cudaError_t launch_expand_params(const double *tec, const double *alpha, PulseParams *out, int64_t batch, double k2c,
                                 double k2pt, cudaStream_t st) {
  expand_params_kernel<<<(unsigned)((batch + 255) / 256), 256, 0, st>>>(tec, alpha, out, batch, k2c, k2pt);
  return cudaGetLastError();
}
}  // namespace dc

namespace {

thread_local char g_errmsg[512] = "";

dc_status fail(dc_status s, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
dc_status fail(dc_status s, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_errmsg, sizeof(g_errmsg), fmt, ap);
  va_end(ap);
  return s;
}

dc_status cuda_fail(cudaError_t e, const char *what) {
  return fail(DC_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define DC_CUDA(call, what)                        \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

constexpr int kRingSlots = 4;
// batches above this stage raw tec / alpha (16 B per pulse, a memcpy) and derive the per-pulse
// parameters on the device; smaller ones derive them on the host (one copy, lowest latency)
constexpr int64_t kDeviceExpandBatch = 4096;
// pulses per launch group: 2 GiB (256 pulses of 2^20) -- measured 64.8 vs 63.5 GS/s at 512 MiB on the
// C4 train (fewer launch ramps and tails); the group buffer is plan-owned device memory
constexpr int64_t kChunkTargetBytes = 2048ll << 20;

struct ParamSlot {
  PulseParams *host = nullptr;  // pinned (large batches: the raw tec / alpha arrays, 16 B per pulse)
  PulseParams *dev = nullptr;
  double *dev_raw = nullptr;    // large batches: raw tec [cap] then alpha [cap], expanded on the device
  int64_t cap = 0;
  cudaEvent_t done = nullptr;
  bool used = false;
};

}  // namespace

struct dc_plan_s {
  int64_t n = 0;
  int log2n = 0;
  double fs = 0, fc = 0;
  int taps = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  int regime = 0;
  int P1 = 0, P2 = 0, H = 0;
  int sm_count = 0;
  int64_t chunk = 1;  // pulses per chunk
  // device tables
  float2 *tw_small_f = nullptr, *tw_small_i = nullptr;
  float2 *tw_w1024 = nullptr;  // regime 0, n = 2^11 .. 2^13: 1024-point tables of the in-CTA four-step
  float2 *tw1f = nullptr, *tw1i = nullptr, *tw2f = nullptr, *tw2i = nullptr, *twh = nullptr, *twl = nullptr;
  const float2 *tw1024 = nullptr;  // radix-32 x 32 pass-2 table inside one of the tables above
  float2 *gtab = nullptr;          // per-bin 1/f_k as FP32 pairs, in the layout the warp row kernel reads
  float2 *ref = nullptr;           // conj(R_k) of the matched-filter reference (dc_set_reference), gtab layout
  bool taper = false;              // Kaiser taper of the sinc window (dc_set_taper, reading R17)
  double kaiser = 0.0;
  dc::TaperCoef tc{};
  int taper_terms = dc::kTaperTerms;
  bool ref_set = false;
  // FFT P/Q resampling (dc_doppler_pq, reading R18): the length-2n chirp-z convolution runs on an inner
  // plan of size 2n in its pulse-compression mode with one table T_M per P/Q length M (LRU cache)
  dc_plan_s *pq = nullptr;
  float2 *pq_tabs = nullptr;           // pq_cap tables of 2n entries
  int pq_cap = 0;
  std::vector<int64_t> pq_tab_M;       // M held by each table slot (0: empty)
  std::vector<uint64_t> pq_tab_use;    // LRU stamps
  uint64_t pq_clock = 0;
  float2 *pq_X = nullptr, *pq_a = nullptr;  // group buffers: forward spectra (pq_group x n), convolution (x 2n)
  int64_t pq_group = 0;
  PulseParams *pq_zero = nullptr;      // tec = 0 parameters of the inner plan (pq_group entries)
  int *pq_host = nullptr, *pq_dev = nullptr;  // per-pulse [table slot x batch][M x batch] staging
  int64_t pq_stage_cap = 0;
  cudaEvent_t pq_done = nullptr;
  bool pq_used = false;
  float2 *scratch = nullptr;  // launch-group buffer of dc_correct: chunk * n samples
  void *dop_desc = nullptr;   // Doppler kernel: per-CTA tile-geometry slots (dc::kDopDescBytes)
  int64_t scratch_bytes = 0;
  cudaEvent_t ev_stream = nullptr;  // dc_set_stream: orders the new stream after the old one
  // host-path buffers (lazily allocated)
  float2 *hin[2] = {nullptr, nullptr}, *hout[2] = {nullptr, nullptr};
  int64_t host_chunk = 0;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_in[2] = {}, ev_comp[2] = {}, ev_out[2] = {};
  ParamSlot ring[kRingSlots];
  int ring_next = 0;
  int64_t launches = 0;
  // profiling (dc_profile_enable)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct Rec {
    int cls;
    int64_t samples;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  dc_profile_t acc{};
};

namespace {

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

// FP32 twiddle tables generated in binary64.  Pass section of NS*R entries, entry (k, r) =
// exp(-2 pi i k r / (NS R)) stored at float2 index ((r/2) NS + k) 2 + (r mod 2), i.e. float4 pairs
// (r even, r odd) ordered [r/2][k] so that lanes with consecutive k read consecutive words.
std::vector<float2> build_pass_tables(const dc::PlanDesc &d, bool inv) {
  std::vector<float2> t((size_t)std::max(d.tw_size, 2), make_float2(0.f, 0.f));
  for (int i = 0; i < d.npass; ++i) {
    const int lns = inv ? d.log_ns_inv[i] : d.log_ns_fwd[i];
    const int lr = inv ? d.log_radix_inv[i] : d.log_radix_fwd[i];
    const int off = inv ? d.tw_off_inv[i] : d.tw_off_fwd[i];
    const int64_t NS = 1ll << lns, R = 1ll << lr, M = NS * R;
    for (int64_t k = 0; k < NS; ++k)
      for (int64_t r = 0; r < R; ++r) {
        const int64_t e = (k * r) % M;
        const double ang = -2.0 * dc::kPi * (double)e / (double)M;
        t.at((size_t)(off + ((r >> 1) * NS + k) * 2 + (r & 1))) = make_float2((float)std::cos(ang), (float)std::sin(ang));
      }
  }
  return t;
}

dc_status upload(float2 **dst, const std::vector<float2> &src) {
  DC_CUDA(cudaMalloc(dst, src.size() * sizeof(float2)), "cudaMalloc(twiddles)");
  DC_CUDA(cudaMemcpy(*dst, src.data(), src.size() * sizeof(float2), cudaMemcpyHostToDevice), "cudaMemcpy(twiddles)");
  return DC_OK;
}

dc_status check_device_ptr(const dc_plan_s *p, const void *ptr, const char *name) {
  if (!ptr) return fail(DC_ERR_NULL_POINTER, "%s is NULL", name);
  if (((uintptr_t)ptr) & 15u) return fail(DC_ERR_MISALIGNED, "%s is not 16-byte aligned", name);
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(DC_ERR_NOT_DEVICE_MEMORY, "%s: cudaPointerGetAttributes failed (%s)", name, cudaGetErrorName(e));
  }
  if (!(at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged))
    return fail(DC_ERR_NOT_DEVICE_MEMORY, "%s is not device memory", name);
  if (at.type == cudaMemoryTypeDevice && at.device != p->device)
    return fail(DC_ERR_NOT_DEVICE_MEMORY, "%s lives on device %d, plan is on device %d", name, at.device, p->device);
  return DC_OK;
}

dc_status check_overlap(const void *a, const void *b, int64_t bytes) {
  const char *pa = (const char *)a, *pb = (const char *)b;
  if (pa < pb + bytes && pb < pa + bytes) return fail(DC_ERR_ALIASING, "y overlaps x");
  return DC_OK;
}

dc_status check_batch(int64_t batch) {
  if (batch < 1) return fail(DC_ERR_INVALID_VALUE, "batch must be >= 1 (got %lld)", (long long)batch);
  return DC_OK;
}

dc_status check_tec(const double *tec, int64_t batch) {
  if (!tec) return fail(DC_ERR_NULL_POINTER, "tec is NULL");
  for (int64_t i = 0; i < batch; ++i)
    if (!std::isfinite(tec[i]) || tec[i] < 0.0)
      return fail(DC_ERR_INVALID_VALUE, "tec[%lld] = %g must be finite and >= 0", (long long)i, tec[i]);
  return DC_OK;
}

dc_status check_alpha(const double *alpha, int64_t batch) {
  if (!alpha) return fail(DC_ERR_NULL_POINTER, "alpha is NULL");
  for (int64_t i = 0; i < batch; ++i)
    if (!std::isfinite(alpha[i]) || !(alpha[i] > 0.0))
      return fail(DC_ERR_INVALID_VALUE, "alpha[%lld] = %g must be finite and > 0", (long long)i, alpha[i]);
  return DC_OK;
}

// Stage per-pulse scalars into a ring slot; returns the device pointer.
dc_status stage_params(dc_plan_s *p, int64_t batch, const double *tec, const double *alpha, PulseParams **dev,
                       ParamSlot **slot_out, double *max_abs_beta_m1) {
  ParamSlot &s = p->ring[p->ring_next];
  p->ring_next = (p->ring_next + 1) % kRingSlots;
  if (s.used) DC_CUDA(cudaEventSynchronize(s.done), "cudaEventSynchronize(param slot)");
  if (s.cap < batch) {
    // grow every slot at once so steady-state calls never allocate
    const int64_t cap = std::max<int64_t>(batch, 1024);
    for (auto &q : p->ring) {
      if (q.used) DC_CUDA(cudaEventSynchronize(q.done), "cudaEventSynchronize(param slot)");
      if (q.host) cudaFreeHost(q.host);
      if (q.dev) cudaFree(q.dev);
      if (q.dev_raw) cudaFree(q.dev_raw);
      q.host = nullptr;
      q.dev = nullptr;
      q.dev_raw = nullptr;
      q.cap = 0;
      if (cudaMallocHost(&q.host, sizeof(PulseParams) * cap) != cudaSuccess) {
        cudaGetLastError();
        return fail(DC_ERR_OUT_OF_MEMORY, "pinned parameter staging (%lld pulses)", (long long)cap);
      }
      if (cudaMalloc(&q.dev, sizeof(PulseParams) * cap) != cudaSuccess ||
          cudaMalloc(&q.dev_raw, 2 * sizeof(double) * cap) != cudaSuccess) {
        cudaGetLastError();
        return fail(DC_ERR_OUT_OF_MEMORY, "device parameter buffer (%lld pulses)", (long long)cap);
      }
      q.cap = cap;
    }
  }
  const double k2c = 2.0 * dc::k2_per_tec() / dc::kC;  // nu_k = (2 K2 / c) / f_k, two-way
  double mb = 0.0;
  if (batch > kDeviceExpandBatch) {
    // raw arrays through the pinned slot; the same binary64 operations run on the device
    // (expand_params_kernel), so the parameters are bit-identical to the host path.  max |beta - 1|
    // is attained at the smallest or largest alpha (fl(1/alpha) is monotone in alpha).
    double *raw = reinterpret_cast<double *>(s.host);
    if (tec) std::memcpy(raw, tec, sizeof(double) * batch);
    if (alpha) {
      std::memcpy(raw + batch, alpha, sizeof(double) * batch);
      double amin = alpha[0], amax = alpha[0];
      for (int64_t i = 1; i < batch; ++i) {
        amin = std::min(amin, alpha[i]);
        amax = std::max(amax, alpha[i]);
      }
      mb = std::max(std::fabs(1.0 / amin - 1.0), std::fabs(1.0 / amax - 1.0));
    }
    if (tec)
      DC_CUDA(cudaMemcpyAsync(s.dev_raw, raw, sizeof(double) * batch, cudaMemcpyHostToDevice, p->stream),
              "cudaMemcpyAsync(params)");
    if (alpha)
      DC_CUDA(cudaMemcpyAsync(s.dev_raw + batch, raw + batch, sizeof(double) * batch, cudaMemcpyHostToDevice, p->stream),
              "cudaMemcpyAsync(params)");
    DC_CUDA(dc::launch_expand_params(tec ? s.dev_raw : nullptr, alpha ? s.dev_raw + batch : nullptr, s.dev, batch, k2c,
                                     dc::k2_per_tec(), p->stream),
            "expand_params_kernel launch");
    *dev = s.dev;
    *slot_out = &s;
    if (max_abs_beta_m1) *max_abs_beta_m1 = mb;
    return DC_OK;
  }
  for (int64_t i = 0; i < batch; ++i) {
    s.host[i].nu_coef = tec ? k2c * tec[i] : 0.0;
    s.host[i].k2 = tec ? dc::k2_per_tec() * tec[i] : 0.0;  // the oracle's K2 (orc_iono_phase_cycles)
    s.host[i].nu_hi = (float)s.host[i].nu_coef;
    s.host[i].nu_lo = (float)(s.host[i].nu_coef - (double)s.host[i].nu_hi);
    s.host[i].beta = alpha ? 1.0 / alpha[i] : 1.0;
    mb = std::max(mb, std::fabs(s.host[i].beta - 1.0));
  }
  DC_CUDA(cudaMemcpyAsync(s.dev, s.host, sizeof(PulseParams) * batch, cudaMemcpyHostToDevice, p->stream),
          "cudaMemcpyAsync(params)");
  *dev = s.dev;
  *slot_out = &s;
  if (max_abs_beta_m1) *max_abs_beta_m1 = mb;
  return DC_OK;
}

dc_status release_slot(dc_plan_s *p, ParamSlot *s) {
  DC_CUDA(cudaEventRecord(s->done, p->stream), "cudaEventRecord(param slot)");
  s->used = true;
  return DC_OK;
}

// release a staged slot on every exit path after stage_params (also when a launch failed: the
// slot's event then marks whatever was enqueued); returns the first error
dc_status release_after(dc_plan_s *p, ParamSlot *slot, dc_status s) {
  if (s != DC_OK) {
    cudaEventRecord(slot->done, p->stream);
    slot->used = true;
    return s;
  }
  return release_slot(p, slot);
}

// ---- profiling brackets ----------------------------------------------------------------------------
cudaEvent_t prof_event(dc_plan_s *p) {
  if (p->ev_used == p->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    p->ev_pool.push_back(e);
  }
  return p->ev_pool[p->ev_used++];
}

struct ProfScope {
  dc_plan_s *p;
  int cls;
  int64_t samples;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(dc_plan_s *p_, int cls_, int64_t samples_, cudaStream_t st_)
      : p(p_), cls(cls_), samples(samples_), st(st_) {
    p->launches += 1;
    if (p->prof && (a = prof_event(p))) cudaEventRecord(a, st);
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = prof_event(p);
      if (b) {
        cudaEventRecord(b, st);
        p->recs.push_back({cls, samples, a, b});
      }
    }
  }
};

// where a launch group's kernels go: stream + persistent-grid cap (0 = one wave of the whole GPU)
struct Lane {
  cudaStream_t st;
  int cap;
};

// Every entry point that touches the device makes the plan's device current and restores the
// caller's device on return (a multi-GPU process keeps its own current device).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};
#define DC_DEVICE_GUARD(p)                                              \
  DeviceGuard dev_guard_(p->device);                                    \
  if (dev_guard_.err != cudaSuccess) return cuda_fail(dev_guard_.err, "cudaSetDevice")

// ---- stage launchers (no validation) -----------------------------------------------------------
// bin tables of var 2 (T tables + per-pulse index, indexed like pp) and the spectrum output of var 3
struct RefArgs {
  const float2 *ref = nullptr;
  const int *ref_idx = nullptr;
  float2 *ref_out = nullptr;
};
// var: 0 Eq. 15, 1 Eq. 14, 2 Eq. 15 + matched filter (tables ra.ref), 3 conj spectra into ra.ref_out
// n = 2^14 (regime 1) runs Eq. 15 / Eq. 14 on the in-CTA four-step kernel (one HBM round trip, wsmall.cuh)
bool incta_2e14(const dc_plan_s *p) { return p->log2n == 14 && p->tw1024 && p->gtab; }
dc_status run_iono(dc_plan_s *p, const float2 *src, float2 *dst, int64_t pulses, const PulseParams *pp,
                   int64_t pulse_base, int var, Lane ln, RefArgs ra = RefArgs{}) {
  if (p->regime == 0 || (incta_2e14(p) && (var == 0 || var == 1))) {
    dc::IonoSmallArgs a{src, dst, pulses, p->log2n, pp ? pp + pulse_base : nullptr, p->tw_small_f, p->tw_small_i,
                        p->fs / (double)p->n, p->fc, ln.st, p->tw1024, ln.cap, p->gtab, ra.ref,
                        ra.ref_idx ? ra.ref_idx + pulse_base : nullptr, ra.ref_out};
    ProfScope ps(p, DC_K_IONO_SMALL, pulses * p->n, ln.st);
    DC_CUDA(dc::launch_iono_small(a, var), "iono_small_kernel launch");
    return DC_OK;
  }
  dc::FourStepArgs a{};
  a.src = src;
  a.dst = dst;
  a.pulses = pulses;
  a.pulse_stride = p->n;
  a.pulse_base = pulse_base;
  a.log2n = p->log2n;
  a.pp = pp;
  a.tw1f = p->tw1f;
  a.tw1i = p->tw1i;
  a.tw2f = p->tw2f;
  a.tw2i = p->tw2i;
  a.twh = p->twh;
  a.twl = p->twl;
  a.H = p->H;
  a.fs_over_n = p->fs / (double)p->n;
  a.fc = p->fc;
  a.stream = ln.st;
  a.tw1024 = p->tw1024;
  a.grid_cap = ln.cap;
  a.gtab = p->gtab;
  a.ref = ra.ref;
  a.ref_idx = ra.ref_idx;
  a.ref_out = ra.ref_out;
  for (int pass = 0; pass < (var == 3 ? 2 : 3); ++pass) {
    ProfScope ps(p, DC_K_FOURSTEP_A + pass, pulses * p->n, ln.st);
    DC_CUDA(dc::launch_iono_fourstep_pass(a, pass, var), "four-step kernel launch");
  }
  return DC_OK;
}

dc_status run_doppler(dc_plan_s *p, const float2 *src, float2 *dst, int64_t pulses, const PulseParams *pp,
                      int64_t pulse_base, double max_abs_beta_m1, Lane ln) {
  dc::DopplerArgs a{src, dst, pulses, p->n, p->taps, pp, pulse_base, p->fc / p->fs, ln.st, ln.cap, p->taper, p->tc, p->taper_terms,
                    p->dop_desc};
  ProfScope ps(p, DC_K_DOPPLER, pulses * p->n, ln.st);
  DC_CUDA(dc::launch_doppler(a, max_abs_beta_m1), "doppler kernel launch");
  return DC_OK;
}

// dc_correct of one launch group: the fused single-round-trip kernel where it exists (short pulses,
// n = 2^10 .. 2^14, W in {16, 32}, rectangular window, first/second-order Doppler path; NEXT-1), else
// the ionospheric stage into the group buffer followed by the Doppler stage
bool correct_fused_ok(const dc_plan_s *p, double max_abs_beta_m1) {
  const int path = dc::doppler_path(max_abs_beta_m1, p->taper, p->taps);
  return (p->regime == 0 || incta_2e14(p)) && !p->taper && path != 0 && dc::correct_small_supported(p->log2n, p->taps);
}
dc_status run_correct(dc_plan_s *p, const float2 *src, float2 *dst, int64_t pulses, const PulseParams *pp,
                      int64_t pulse_base, double max_abs_beta_m1, Lane ln) {
  if (correct_fused_ok(p, max_abs_beta_m1)) {
    dc::IonoSmallArgs a{src, nullptr, pulses, p->log2n, pp + pulse_base, p->tw_small_f, p->tw_small_i,
                        p->fs / (double)p->n, p->fc, ln.st, p->tw1024, ln.cap, p->gtab, nullptr, nullptr, nullptr};
    ProfScope ps(p, DC_K_CORRECT_FUSED, pulses * p->n, ln.st);
    DC_CUDA(dc::launch_correct_small(a, dst, p->fc / p->fs, p->taps, dc::doppler_path(max_abs_beta_m1, false, p->taps) == 2),
            "fused dc_correct kernel launch");
    return DC_OK;
  }
  dc_status s = run_iono(p, src, p->scratch, pulses, pp, pulse_base, 0, ln);
  if (s == DC_OK) s = run_doppler(p, p->scratch, dst, pulses, pp, pulse_base, max_abs_beta_m1, ln);
  return s;
}

// launch-group buffer for dc_correct: min(chunk, batch) pulses
dc_status ensure_scratch(dc_plan_s *p, int64_t batch) {
  const int64_t need = std::min(p->chunk, batch) * p->n * (int64_t)sizeof(float2);
  if (p->scratch_bytes >= need) return DC_OK;
  DC_CUDA(cudaStreamSynchronize(p->stream), "cudaStreamSynchronize(scratch)");
  if (p->scratch) cudaFree(p->scratch);
  p->scratch = nullptr;
  p->scratch_bytes = 0;
  if (cudaMalloc(&p->scratch, (size_t)need) != cudaSuccess) {
    cudaGetLastError();
    return fail(DC_ERR_OUT_OF_MEMORY, "launch-group buffer(s) of %lld bytes", (long long)need);
  }
  p->scratch_bytes = need;
  return DC_OK;
}

// src -> dst (dst == src: in place); var as run_iono (0, 1 or 2)
dc_status iono_common(dc_plan_t p, const void *x, void *z, int64_t batch, const double *tec, int var) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  dc_status s;
  if ((s = check_batch(batch)) != DC_OK) return s;
  if ((s = check_device_ptr(p, x, "x")) != DC_OK) return s;
  if (z != x) {
    if ((s = check_device_ptr(p, z, "z")) != DC_OK) return s;
    if ((s = check_overlap(x, z, batch * p->n * (int64_t)sizeof(float2))) != DC_OK) return s;
  }
  if ((s = check_tec(tec, batch)) != DC_OK) return s;
  if (var == 2 && !p->ref_set)
    return fail(DC_ERR_INVALID_VALUE, "no matched-filter reference: call dc_set_reference first");
  DC_DEVICE_GUARD(p);
  PulseParams *pp;
  ParamSlot *slot;
  if ((s = stage_params(p, batch, tec, nullptr, &pp, &slot, nullptr)) != DC_OK) return s;
  const float2 *xp = (const float2 *)x;
  float2 *zp = (float2 *)z;
  const int64_t step = (p->regime == 0) ? std::min<int64_t>(batch, 1ll << 30) : p->chunk;
  for (int64_t b0 = 0; b0 < batch && s == DC_OK; b0 += step) {
    const int64_t nb = std::min(step, batch - b0);
    s = run_iono(p, xp + b0 * p->n, zp + b0 * p->n, nb, pp, b0, var, Lane{p->stream, 0},
                 RefArgs{var == 2 ? p->ref : nullptr, nullptr, nullptr});
  }
  return release_after(p, slot, s);
}

}  // namespace

extern "C" {
#pragma GCC visibility push(default)

const char *dc_status_string(dc_status s) {
  switch (s) {
    case DC_OK: return "DC_OK";
    case DC_ERR_INVALID_VALUE: return "DC_ERR_INVALID_VALUE";
    case DC_ERR_NULL_POINTER: return "DC_ERR_NULL_POINTER";
    case DC_ERR_MISALIGNED: return "DC_ERR_MISALIGNED";
    case DC_ERR_ALIASING: return "DC_ERR_ALIASING";
    case DC_ERR_OUT_OF_MEMORY: return "DC_ERR_OUT_OF_MEMORY";
    case DC_ERR_CUDA: return "DC_ERR_CUDA";
    case DC_ERR_UNSUPPORTED_DEVICE: return "DC_ERR_UNSUPPORTED_DEVICE";
    case DC_ERR_NOT_DEVICE_MEMORY: return "DC_ERR_NOT_DEVICE_MEMORY";
  }
  return "DC_ERR_UNKNOWN";
}

const char *dc_last_error_message(void) { return g_errmsg; }

int dc_version(void) { return DC_VERSION; }

double dc_k2_per_tec(void) { return dc::k2_per_tec(); }

double dc_alpha_from_velocity(double v) {
  if (!std::isfinite(v) || std::fabs(v) >= dc::kC) return std::nan("");
  return (1.0 + v / dc::kC) / (1.0 - v / dc::kC);
}

dc_status dc_plan(dc_plan_t *out, int64_t n, double fs_hz, double fc_hz, int taps, int device, void *cuda_stream) {
  g_errmsg[0] = 0;
  if (!out) return fail(DC_ERR_NULL_POINTER, "out is NULL");
  *out = nullptr;
  if (!is_pow2(n) || n < 2 || n > (1ll << 24))
    return fail(DC_ERR_INVALID_VALUE, "n = %lld must be a power of two in [2, 2^24]", (long long)n);
  if (!std::isfinite(fs_hz) || !(fs_hz > 0.0)) return fail(DC_ERR_INVALID_VALUE, "fs_hz = %g must be finite and > 0", fs_hz);
  if (!std::isfinite(fc_hz) || fc_hz < 0.0) return fail(DC_ERR_INVALID_VALUE, "fc_hz = %g must be finite and >= 0", fc_hz);
  if (taps < 2 || taps > 128 || taps > n)
    return fail(DC_ERR_INVALID_VALUE, "taps = %d must be in [2, 128] and <= n", taps);
  int ndev = 0;
  DC_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(DC_ERR_INVALID_VALUE, "device %d out of range (%d devices)", device, ndev);
  cudaDeviceProp prop;
  DC_CUDA(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(DC_ERR_UNSUPPORTED_DEVICE, "device %d is sm_%d%d; libdispcorr is built for sm_100a (B200)", device,
                prop.major, prop.minor);
  DeviceGuard dg(device);
  if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");

  dc_plan_s *p = new (std::nothrow) dc_plan_s();
  if (!p) return fail(DC_ERR_OUT_OF_MEMORY, "plan allocation");
  p->n = n;
  p->log2n = 0;
  while ((1ll << p->log2n) < n) ++p->log2n;
  p->fs = fs_hz;
  p->fc = fc_hz;
  p->taps = taps;
  p->device = device;
  p->stream = (cudaStream_t)cuda_stream;
  p->sm_count = prop.multiProcessorCount;
  p->regime = (p->log2n <= 13) ? 0 : 1;
  dc_status s = DC_OK;
  auto cleanup = [&](dc_status st) {
    dc_plan_destroy(p);
    return st;
  };
  if (p->regime == 0) {
    dc::PlanDesc d;
    dc::describe_small_plan(p->log2n, d);
    if ((s = upload(&p->tw_small_f, build_pass_tables(d, false))) != DC_OK) return cleanup(s);
    if ((s = upload(&p->tw_small_i, build_pass_tables(d, true))) != DC_OK) return cleanup(s);
    if (p->log2n == 10 && d.npass == 2 && d.log_radix_fwd[0] == 5 && d.log_radix_fwd[1] == 5)
      p->tw1024 = p->tw_small_f + dc::tw1024_offset();
    if (p->log2n >= 11 && p->log2n <= 13) {  // n = N1 x 1024 on the warp FFT (wsmall.cuh)
      dc::PlanDesc d10;
      dc::describe_small_plan(10, d10);
      if (d10.npass == 2 && d10.log_radix_fwd[0] == 5 && d10.log_radix_fwd[1] == 5) {
        if ((s = upload(&p->tw_w1024, build_pass_tables(d10, false))) != DC_OK) return cleanup(s);
        p->tw1024 = p->tw_w1024 + dc::tw1024_offset();
        p->P1 = p->log2n - 10;
        p->P2 = 10;
      }
    }
  } else {
    dc::fourstep_split(p->log2n, p->P1, p->P2);
    dc::PlanDesc d1, d2;
    dc::describe_fourstep_plan(p->P1, d1);
    dc::describe_fourstep_plan(p->P2, d2);
    if ((s = upload(&p->tw1f, build_pass_tables(d1, false))) != DC_OK) return cleanup(s);
    if ((s = upload(&p->tw1i, build_pass_tables(d1, true))) != DC_OK) return cleanup(s);
    if ((s = upload(&p->tw2f, build_pass_tables(d2, false))) != DC_OK) return cleanup(s);
    if ((s = upload(&p->tw2i, build_pass_tables(d2, true))) != DC_OK) return cleanup(s);
    auto radix32x32 = [](const dc::PlanDesc &d) { return d.npass == 2 && d.log_radix_fwd[0] == 5 && d.log_radix_fwd[1] == 5; };
    if (p->P2 == 10 && radix32x32(d2)) p->tw1024 = p->tw2f + dc::tw1024_offset();
    else if (p->P1 == 10 && radix32x32(d1)) p->tw1024 = p->tw1f + dc::tw1024_offset();
    p->H = (p->log2n + 1) / 2;
    std::vector<float2> lo((size_t)1 << p->H), hi((size_t)1 << (p->log2n - p->H));
    for (size_t m = 0; m < lo.size(); ++m) {
      const double a = -2.0 * dc::kPi * (double)m / (double)n;
      lo[m] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    for (size_t m = 0; m < hi.size(); ++m) {
      const double a = -2.0 * dc::kPi * (double)(m << p->H) / (double)n;
      hi[m] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    if ((s = upload(&p->twl, lo)) != DC_OK) return cleanup(s);
    if ((s = upload(&p->twh, hi)) != DC_OK) return cleanup(s);
  }
  p->chunk = std::max<int64_t>(1, kChunkTargetBytes / (n * (int64_t)sizeof(float2)));
  // per-bin g_k = 1/f_k (0 where f_k <= 0, reading R3) for the warp-level row kernel, FP32 pairs:
  // regime 0 (n = 1024): natural bin order; four-step with N2 = 1024: row layout [k1][k2] of k = k1 + N1 k2
  // regime 0, n = 128 .. 1024 (the warp-level kernels): natural bin order
  const bool tiny = p->regime == 0 && p->log2n >= 7 && p->log2n <= 10;
  if (p->tw1024 || tiny) {
    const int P1 = tiny ? 0 : p->P1;
    const int64_t N2 = tiny ? n : 1024;
    std::vector<float2> g((size_t)n);
    for (int64_t k1 = 0; k1 < (1ll << P1); ++k1)
      for (int64_t k2 = 0; k2 < N2; ++k2) {
        const int64_t k = k1 + (k2 << P1);
        const int64_t kk = (k >= n / 2) ? k - n : k;
        const double f = fc_hz + fs_hz * (double)kk / (double)n;
        const double gi = (f > 0.0) ? 1.0 / f : 0.0;
        const float hi = (float)gi;
        g[(size_t)(k1 * N2 + k2)] = make_float2(hi, (float)(gi - (double)hi));
      }
    if ((s = upload(&p->gtab, g)) != DC_OK) return cleanup(s);
  }
  p->chunk = std::min<int64_t>(p->chunk, 65535);
  p->scratch_bytes = 0;  // chunk buffers are allocated on first use, sized to the batch (ensure_scratch)
  for (auto &slot : p->ring)
    if (cudaEventCreateWithFlags(&slot.done, cudaEventDisableTiming) != cudaSuccess)
      return cleanup(cuda_fail(cudaGetLastError(), "cudaEventCreate"));
  if (cudaEventCreateWithFlags(&p->ev_stream, cudaEventDisableTiming) != cudaSuccess)
    return cleanup(cuda_fail(cudaGetLastError(), "cudaEventCreate"));
  if (cudaMalloc(&p->dop_desc, dc::kDopDescBytes) != cudaSuccess) {
    cudaGetLastError();
    return cleanup(fail(DC_ERR_OUT_OF_MEMORY, "Doppler tile-geometry slots"));
  }
  *out = p;
  return DC_OK;
}

dc_status dc_plan_destroy(dc_plan_t p) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  DeviceGuard dg(p->device);
  cudaStreamSynchronize(p->stream);
  if (p->s_h2d) cudaStreamSynchronize(p->s_h2d);
  if (p->s_d2h) cudaStreamSynchronize(p->s_d2h);
  float2 *bufs[] = {p->tw_small_f, p->tw_small_i, p->tw_w1024, p->tw1f, p->tw1i, p->tw2f, p->tw2i, p->twh, p->twl,
                    p->scratch, p->gtab, p->ref, p->hin[0], p->hin[1], p->hout[0], p->hout[1]};
  for (float2 *b : bufs)
    if (b) cudaFree(b);
  if (p->pq) dc_plan_destroy(p->pq);
  for (void *b : {(void *)p->pq_tabs, (void *)p->pq_X, (void *)p->pq_a, (void *)p->pq_zero, (void *)p->pq_dev})
    if (b) cudaFree(b);
  if (p->pq_host) cudaFreeHost(p->pq_host);
  if (p->pq_done) cudaEventDestroy(p->pq_done);
  for (auto &s : p->ring) {
    if (s.done) cudaEventDestroy(s.done);
    if (s.host) cudaFreeHost(s.host);
    if (s.dev) cudaFree(s.dev);
    if (s.dev_raw) cudaFree(s.dev_raw);
  }
  if (p->ev_stream) cudaEventDestroy(p->ev_stream);
  if (p->dop_desc) cudaFree(p->dop_desc);
  for (int i = 0; i < 2; ++i) {
    if (p->ev_in[i]) cudaEventDestroy(p->ev_in[i]);
    if (p->ev_comp[i]) cudaEventDestroy(p->ev_comp[i]);
    if (p->ev_out[i]) cudaEventDestroy(p->ev_out[i]);
  }
  for (cudaEvent_t e : p->ev_pool) cudaEventDestroy(e);
  if (p->s_h2d) cudaStreamDestroy(p->s_h2d);
  if (p->s_d2h) cudaStreamDestroy(p->s_d2h);
  delete p;
  return DC_OK;
}

dc_status dc_set_stream(dc_plan_t p, void *stream) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  if ((cudaStream_t)stream == p->stream) return DC_OK;
  DC_DEVICE_GUARD(p);
  // work already enqueued on the old stream still reads / writes plan-owned buffers (scratch,
  // reference table, parameter ring): the new stream waits for it before any later call runs
  DC_CUDA(cudaEventRecord(p->ev_stream, p->stream), "cudaEventRecord(set_stream)");
  DC_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, p->ev_stream, 0), "cudaStreamWaitEvent(set_stream)");
  p->stream = (cudaStream_t)stream;
  return DC_OK;
}

dc_status dc_sync(dc_plan_t p) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  DC_DEVICE_GUARD(p);
  DC_CUDA(cudaStreamSynchronize(p->stream), "cudaStreamSynchronize");
  return DC_OK;
}

dc_status dc_iono(dc_plan_t p, void *x, int64_t batch, const double *tec) {
  return iono_common(p, x, x, batch, tec, 0);
}

dc_status dc_iono_distort(dc_plan_t p, void *x, int64_t batch, const double *tec) {
  return iono_common(p, x, x, batch, tec, 1);
}

dc_status dc_set_reference(dc_plan_t p, const void *r, int64_t L) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  dc_status s;
  if (L < 1 || L > p->n) return fail(DC_ERR_INVALID_VALUE, "reference length L = %lld must be in [1, n = %lld]", (long long)L, (long long)p->n);
  if ((s = check_device_ptr(p, r, "r")) != DC_OK) return s;
  DC_DEVICE_GUARD(p);
  if (!p->ref && cudaMalloc(&p->ref, (size_t)p->n * sizeof(float2)) != cudaSuccess) {
    cudaGetLastError();
    p->ref = nullptr;
    return fail(DC_ERR_OUT_OF_MEMORY, "reference spectrum table");
  }
  if ((s = ensure_scratch(p, 1)) != DC_OK) return s;
  // zero-padded reference in the chunk buffer, then its forward DFT stored conjugated (var 3)
  DC_CUDA(cudaMemsetAsync(p->scratch, 0, (size_t)p->n * sizeof(float2), p->stream), "cudaMemsetAsync");
  DC_CUDA(cudaMemcpyAsync(p->scratch, r, (size_t)L * sizeof(float2), cudaMemcpyDeviceToDevice, p->stream), "cudaMemcpyAsync");
  if ((s = run_iono(p, p->scratch, p->scratch, 1, nullptr, 0, 3, Lane{p->stream, 0}, RefArgs{nullptr, nullptr, p->ref})) !=
      DC_OK)
    return s;
  p->ref_set = true;
  return DC_OK;
}

dc_status dc_set_window(dc_plan_t p, int kind, double param) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  if (kind == DC_WINDOW_RECT) {
    p->taper = false;
    p->kaiser = 0.0;
    return DC_OK;
  }
  if (kind == DC_WINDOW_HANN) {
    p->tc.pi_over_L = (float)(2.0 * dc::kPi / (double)p->taps);
    p->taper_terms = dc::kTaperHann;
    p->kaiser = 0.0;
    p->taper = true;
    return DC_OK;
  }
  if (kind != DC_WINDOW_KAISER) return fail(DC_ERR_INVALID_VALUE, "window kind %d unknown", kind);
  const double kaiser = param;
  if (!std::isfinite(kaiser) || kaiser < 0.0 || kaiser > 12.0)
    return fail(DC_ERR_INVALID_VALUE, "kaiser = %g must be finite and in [0, 12]", kaiser);
  // I0(kb) and the normalised series coefficients 1 / ((j!)^2 I0(kb)) in binary64
  double i0 = 0.0, term = 1.0;
  const double q = 0.25 * kaiser * kaiser;
  for (int j = 0; j < 200; ++j) {
    if (j > 0) term *= q / ((double)j * (double)j);
    i0 += term;
    if (term < 1e-18 * i0) break;
  }
  double cj = 1.0;
  for (int j = 0; j < dc::kTaperTerms; ++j) {
    if (j > 0) cj /= (double)j * (double)j;
    p->tc.c[j] = (float)(cj / i0);
  }
  // 17 series terms suffice when the 17th term is below 1e-9 of the sum over the window (kb <= ~8.9)
  double t17 = 1.0;
  for (int j = 1; j <= 17; ++j) t17 *= q / ((double)j * (double)j);
  p->taper_terms = (t17 / i0 < 1e-9) ? 17 : dc::kTaperTerms;
  p->tc.qa = (float)q;
  p->tc.inv_L2 = (float)(4.0 / ((double)p->taps * (double)p->taps));
  p->kaiser = kaiser;
  p->taper = kaiser > 0.0;
  return DC_OK;
}

dc_status dc_set_taper(dc_plan_t p, double kaiser) { return dc_set_window(p, DC_WINDOW_KAISER, kaiser); }

dc_status dc_compress(dc_plan_t p, const void *x, void *z, int64_t batch, const double *tec) {
  return iono_common(p, x, z, batch, tec, 2);
}

dc_status dc_doppler(dc_plan_t p, const void *x, void *y, int64_t batch, const double *alpha) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  dc_status s;
  if ((s = check_batch(batch)) != DC_OK) return s;
  if ((s = check_device_ptr(p, x, "x")) != DC_OK) return s;
  if ((s = check_device_ptr(p, y, "y")) != DC_OK) return s;
  if ((s = check_overlap(x, y, batch * p->n * (int64_t)sizeof(float2))) != DC_OK) return s;
  if ((s = check_alpha(alpha, batch)) != DC_OK) return s;
  DC_DEVICE_GUARD(p);
  PulseParams *pp;
  ParamSlot *slot;
  double mb = 0;
  if ((s = stage_params(p, batch, nullptr, alpha, &pp, &slot, &mb)) != DC_OK) return s;
  const float2 *xp = (const float2 *)x;
  float2 *yp = (float2 *)y;
  for (int64_t b0 = 0; b0 < batch && s == DC_OK; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(65535, batch - b0);
    s = run_doppler(p, xp + b0 * p->n, yp + b0 * p->n, nb, pp, b0, mb, Lane{p->stream, 0});
  }
  return release_after(p, slot, s);
}

dc_status dc_doppler_pq(dc_plan_t p, const void *x, void *y, int64_t batch, const double *alpha) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  dc_status s;
  if (p->log2n > 23) return fail(DC_ERR_INVALID_VALUE, "FFT P/Q resampling needs n <= 2^23 (plan n = %lld)", (long long)p->n);
  if ((s = check_batch(batch)) != DC_OK) return s;
  if ((s = check_device_ptr(p, x, "x")) != DC_OK) return s;
  if ((s = check_device_ptr(p, y, "y")) != DC_OK) return s;
  if ((s = check_overlap(x, y, batch * p->n * (int64_t)sizeof(float2))) != DC_OK) return s;
  if ((s = check_alpha(alpha, batch)) != DC_OK) return s;
  const int64_t n = p->n, L = 2 * n;
  // P/Q length per pulse, the oracle's rounding (orc_pq_length): M = n + 2 round((n alpha - n) / 2)
  std::vector<int64_t> Ms((size_t)batch);
  for (int64_t i = 0; i < batch; ++i) {
    const int64_t M = n + 2 * (int64_t)std::llround(0.5 * ((double)n * alpha[i] - (double)n));
    if (M < 2 || M > 8 * n)
      return fail(DC_ERR_INVALID_VALUE, "alpha[%lld] = %g gives a P/Q length M = %lld outside [2, 8n]", (long long)i,
                  alpha[i], (long long)M);
    Ms[(size_t)i] = M;
  }
  DC_DEVICE_GUARD(p);
  // ---- lazily built state: inner plan of size 2n, table cache, group buffers, staging
  if (!p->pq) {
    // all-or-nothing: on any failure everything allocated here is released and p->pq stays null
    dc_plan_t inner = nullptr;
    if ((s = dc_plan(&inner, L, p->fs, 0.0, 2, p->device, p->stream)) != DC_OK) return s;
    const int64_t group = std::max<int64_t>(1, std::min<int64_t>(4096, (1ll << 30) / (n * (int64_t)sizeof(float2))));
    const int cap = (int)std::max<int64_t>(2, std::min<int64_t>(64, (1ll << 30) / (L * (int64_t)sizeof(float2))));
    const size_t tab_bytes = (size_t)cap * L * sizeof(float2);
    float2 *tabs = nullptr, *X = nullptr, *A = nullptr;
    PulseParams *zero = nullptr;
    cudaEvent_t done = nullptr;
    auto release = [&]() {
      for (void *b : {(void *)tabs, (void *)X, (void *)A, (void *)zero})
        if (b) cudaFree(b);
      if (done) cudaEventDestroy(done);
      dc_plan_destroy(inner);
      cudaGetLastError();
    };
    if (cudaMalloc(&tabs, tab_bytes) != cudaSuccess || cudaMalloc(&X, (size_t)(group * n) * sizeof(float2)) != cudaSuccess ||
        cudaMalloc(&A, (size_t)(group * L) * sizeof(float2)) != cudaSuccess ||
        cudaMalloc(&zero, (size_t)group * sizeof(PulseParams)) != cudaSuccess) {
      release();
      return fail(DC_ERR_OUT_OF_MEMORY, "FFT P/Q buffers");
    }
    cudaError_t e = cudaMemsetAsync(tabs, 0, tab_bytes, p->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(zero, 0, (size_t)group * sizeof(PulseParams), p->stream);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      release();
      return cuda_fail(e, "FFT P/Q setup");
    }
    p->pq = inner;
    p->pq_group = group;
    p->pq_cap = cap;
    p->pq_tabs = tabs;
    p->pq_X = X;
    p->pq_a = A;
    p->pq_zero = zero;
    p->pq_done = done;
    p->pq_tab_M.assign((size_t)cap, 0);
    p->pq_tab_use.assign((size_t)cap, 0);
  }
  p->pq->stream = p->stream;
  if (p->pq_used) DC_CUDA(cudaEventSynchronize(p->pq_done), "cudaEventSynchronize(P/Q staging)");
  if (p->pq_stage_cap < batch) {
    if (p->pq_host) cudaFreeHost(p->pq_host);
    if (p->pq_dev) cudaFree(p->pq_dev);
    p->pq_host = nullptr;
    p->pq_dev = nullptr;
    p->pq_stage_cap = 0;
    const int64_t cap = std::max<int64_t>(batch, 1024);
    if (cudaMallocHost(&p->pq_host, 2 * sizeof(int) * cap) != cudaSuccess ||
        cudaMalloc(&p->pq_dev, 2 * sizeof(int) * cap) != cudaSuccess) {
      cudaGetLastError();
      return fail(DC_ERR_OUT_OF_MEMORY, "P/Q staging (%lld pulses)", (long long)cap);
    }
    p->pq_stage_cap = cap;
  }
  // ---- groups of consecutive pulses with at most pq_cap distinct non-identity M; tables assigned LRU
  struct Group {
    int64_t b0, nb;
    std::vector<std::pair<int, int64_t>> builds;  // (slot, M) tables to build before the group
    bool identity;                                // all pulses of the group have M == n
  };
  std::vector<Group> groups;
  int *slot_h = p->pq_host, *M_h = p->pq_host + batch;
  for (int64_t b0 = 0; b0 < batch;) {
    Group g{b0, 0, {}, false};
    std::vector<int64_t> need;
    int64_t b = b0;
    for (; b < batch && b - b0 < p->pq_group; ++b) {
      const int64_t M = Ms[(size_t)b];
      if (M != n && std::find(need.begin(), need.end(), M) == need.end()) {
        if ((int)need.size() == p->pq_cap) break;
        need.push_back(M);
      }
    }
    g.nb = b - b0;
    g.identity = need.empty();
    const uint64_t stamp = ++p->pq_clock;
    for (int64_t M : need) {  // hits first, so that misses never evict a table this group uses
      for (int t = 0; t < p->pq_cap; ++t)
        if (p->pq_tab_M[(size_t)t] == M) p->pq_tab_use[(size_t)t] = stamp;
    }
    for (int64_t M : need) {
      int slot = -1;
      for (int t = 0; t < p->pq_cap && slot < 0; ++t)
        if (p->pq_tab_M[(size_t)t] == M) slot = t;
      if (slot < 0) {
        uint64_t best = UINT64_MAX;
        for (int t = 0; t < p->pq_cap; ++t)
          if (p->pq_tab_use[(size_t)t] != stamp && p->pq_tab_use[(size_t)t] < best) {
            best = p->pq_tab_use[(size_t)t];
            slot = t;
          }
        p->pq_tab_M[(size_t)slot] = M;
        p->pq_tab_use[(size_t)slot] = stamp;
        g.builds.push_back({slot, M});
      }
    }
    for (int64_t i = b0; i < b0 + g.nb; ++i) {
      int slot = 0;  // identity pulses (M == n): their convolution input is zero, any table will do
      for (int t = 0; t < p->pq_cap; ++t)
        if (Ms[(size_t)i] != n && p->pq_tab_M[(size_t)t] == Ms[(size_t)i]) slot = t;
      slot_h[i] = slot;
      M_h[i] = (int)Ms[(size_t)i];
    }
    groups.push_back(std::move(g));
    b0 += groups.back().nb;
  }
  DC_CUDA(cudaMemcpyAsync(p->pq_dev, p->pq_host, 2 * sizeof(int) * batch, cudaMemcpyHostToDevice, p->stream),
          "cudaMemcpyAsync(P/Q staging)");
  const int *slot_d = p->pq_dev, *M_d = p->pq_dev + batch;
  const float2 *xp = (const float2 *)x;
  float2 *yp = (float2 *)y;
  const Lane ln{p->stream, 0};
  const int P1row = (p->regime == 1) ? p->P1 : 0;  // row layout of the n-plan's spectra (natural in regime 0)
  auto pipeline = [&]() -> dc_status {
    dc_status st = DC_OK;
    for (const Group &g : groups) {
      if (g.identity) {  // every pulse has M == n: nothing added or removed, y = x ("no work was done")
        DC_CUDA(cudaMemcpyAsync(yp + g.b0 * n, xp + g.b0 * n, (size_t)(g.nb * n) * sizeof(float2),
                                cudaMemcpyDeviceToDevice, ln.st),
                "cudaMemcpyAsync(P/Q identity)");
        continue;
      }
      const int64_t l0 = p->pq->launches;
      ProfScope ps(p, DC_K_PQ, g.nb * n, ln.st);
      for (const auto &bm : g.builds) {  // T_M = conj(DFT_L(r)), r = conj(b reflected): FFT(a) T_M = FFT(a) FFT(b)
        DC_CUDA(dc::launch_pq_chirp(p->pq_a, n, bm.second, ln.st), "pq_chirp_kernel launch");
        p->launches += 1;
        if ((st = run_iono(p->pq, p->pq_a, p->pq_a, 1, nullptr, 0, 3, ln,
                           RefArgs{nullptr, nullptr, p->pq_tabs + (size_t)bm.first * L})) != DC_OK)
          return st;
      }
      // X = DFT_n(x) (stored conjugated, row layout), a = chirp-weighted kept bins, c = a (*) b, y
      const bool prof = p->prof;  // the forward passes are part of this DC_K_PQ record, not of the four-step classes
      p->prof = false;
      st = run_iono(p, xp + g.b0 * n, p->pq_X, g.nb, nullptr, 0, 3, ln, RefArgs{nullptr, nullptr, p->pq_X});
      p->prof = prof;
      if (st != DC_OK) return st;
      DC_CUDA(dc::launch_pq_gather(p->pq_X, p->pq_a, g.nb, p->log2n, P1row, M_d + g.b0, ln.st), "pq_gather_kernel launch");
      if ((st = run_iono(p->pq, p->pq_a, p->pq_a, g.nb, p->pq_zero, 0, 2, ln, RefArgs{p->pq_tabs, slot_d + g.b0, nullptr})) !=
          DC_OK)
        return st;
      DC_CUDA(dc::launch_pq_post(p->pq_a, xp + g.b0 * n, yp + g.b0 * n, g.nb, p->log2n, M_d + g.b0, p->fc, p->fs, ln.st),
              "pq_post_kernel launch");
      p->launches += 1 + (p->pq->launches - l0);  // gather + post (+1 counted by ps) + the inner plan's kernels
    }
    return st;
  };
  s = pipeline();
  cudaEventRecord(p->pq_done, p->stream);
  p->pq_used = true;
  if (s != DC_OK) {  // a failed launch leaves the cache state unknown: drop it
    std::fill(p->pq_tab_M.begin(), p->pq_tab_M.end(), 0);
  }
  return s;
}

dc_status dc_correct(dc_plan_t p, const void *x, void *y, int64_t batch, const double *tec, const double *alpha) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  dc_status s;
  if ((s = check_batch(batch)) != DC_OK) return s;
  if ((s = check_device_ptr(p, x, "x")) != DC_OK) return s;
  if ((s = check_device_ptr(p, y, "y")) != DC_OK) return s;
  if ((s = check_overlap(x, y, batch * p->n * (int64_t)sizeof(float2))) != DC_OK) return s;
  if ((s = check_tec(tec, batch)) != DC_OK) return s;
  if ((s = check_alpha(alpha, batch)) != DC_OK) return s;
  DC_DEVICE_GUARD(p);
  if ((s = ensure_scratch(p, batch)) != DC_OK) return s;
  PulseParams *pp;
  ParamSlot *slot;
  double mb = 0;
  if ((s = stage_params(p, batch, tec, alpha, &pp, &slot, &mb)) != DC_OK) return s;
  const float2 *xp = (const float2 *)x;
  float2 *yp = (float2 *)y;
  const Lane ln{p->stream, 0};
  for (int64_t b0 = 0; b0 < batch && s == DC_OK; b0 += p->chunk) {
    const int64_t nb = std::min(p->chunk, batch - b0);
    s = run_correct(p, xp + b0 * p->n, yp + b0 * p->n, nb, pp, b0, mb, ln);
  }
  return release_after(p, slot, s);
}

dc_status dc_correct_host(dc_plan_t p, const void *x_host, void *y_host, int64_t batch, const double *tec,
                          const double *alpha) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  dc_status s;
  if ((s = check_batch(batch)) != DC_OK) return s;
  if (!x_host) return fail(DC_ERR_NULL_POINTER, "x_host is NULL");
  if (!y_host) return fail(DC_ERR_NULL_POINTER, "y_host is NULL");
  if ((s = check_overlap(x_host, y_host, batch * p->n * (int64_t)sizeof(float2))) != DC_OK) return s;
  if ((s = check_tec(tec, batch)) != DC_OK) return s;
  if ((s = check_alpha(alpha, batch)) != DC_OK) return s;
  DC_DEVICE_GUARD(p);
  // pulses per transfer chunk: bounded so the pinned-host pipeline overlaps (~64 MiB per copy)
  const int64_t hc = std::max<int64_t>(1, std::min(p->chunk, (int64_t)(64ll << 20) / (p->n * (int64_t)sizeof(float2))));
  {
    dc_status se = ensure_scratch(p, std::min(hc, batch));
    if (se != DC_OK) return se;
  }
  if (!p->s_h2d) {
    DC_CUDA(cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking), "cudaStreamCreate");
    DC_CUDA(cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking), "cudaStreamCreate");
    for (int i = 0; i < 2; ++i) {
      DC_CUDA(cudaEventCreateWithFlags(&p->ev_in[i], cudaEventDisableTiming), "cudaEventCreate");
      DC_CUDA(cudaEventCreateWithFlags(&p->ev_comp[i], cudaEventDisableTiming), "cudaEventCreate");
      DC_CUDA(cudaEventCreateWithFlags(&p->ev_out[i], cudaEventDisableTiming), "cudaEventCreate");
    }
  }
  if (p->host_chunk < hc) {
    for (int i = 0; i < 2; ++i) {
      if (p->hin[i]) cudaFree(p->hin[i]);
      if (p->hout[i]) cudaFree(p->hout[i]);
      p->hin[i] = p->hout[i] = nullptr;
    }
    for (int i = 0; i < 2; ++i) {
      if (cudaMalloc(&p->hin[i], (size_t)(hc * p->n * sizeof(float2))) != cudaSuccess ||
          cudaMalloc(&p->hout[i], (size_t)(hc * p->n * sizeof(float2))) != cudaSuccess) {
        cudaGetLastError();
        return fail(DC_ERR_OUT_OF_MEMORY, "host-path device buffers");
      }
    }
    p->host_chunk = hc;
  }
  PulseParams *pp;
  ParamSlot *slot;
  double mb = 0;
  if ((s = stage_params(p, batch, tec, alpha, &pp, &slot, &mb)) != DC_OK) return s;
  const char *xh = (const char *)x_host;
  char *yh = (char *)y_host;
  const size_t pulse_bytes = (size_t)p->n * sizeof(float2);
  // 3-stage pipeline: H2D (s_h2d) -> correct (plan stream) -> D2H (s_d2h), double-buffered
  auto pipeline = [&]() -> dc_status {
    int64_t it = 0;
    for (int64_t b0 = 0; b0 < batch; b0 += hc, ++it) {
      const int i = (int)(it & 1);
      const int64_t nb = std::min(hc, batch - b0);
      if (it >= 2) DC_CUDA(cudaStreamWaitEvent(p->s_h2d, p->ev_comp[i], 0), "wait");  // hin[i] free
      DC_CUDA(cudaMemcpyAsync(p->hin[i], xh + b0 * pulse_bytes, nb * pulse_bytes, cudaMemcpyHostToDevice, p->s_h2d),
              "cudaMemcpyAsync(H2D)");
      DC_CUDA(cudaEventRecord(p->ev_in[i], p->s_h2d), "record");
      DC_CUDA(cudaStreamWaitEvent(p->stream, p->ev_in[i], 0), "wait");
      if (it >= 2) DC_CUDA(cudaStreamWaitEvent(p->stream, p->ev_out[i], 0), "wait");  // hout[i] drained
      if ((s = run_correct(p, p->hin[i], p->hout[i], nb, pp, b0, mb, Lane{p->stream, 0})) != DC_OK) return s;
      DC_CUDA(cudaEventRecord(p->ev_comp[i], p->stream), "record");
      DC_CUDA(cudaStreamWaitEvent(p->s_d2h, p->ev_comp[i], 0), "wait");
      DC_CUDA(cudaMemcpyAsync(yh + b0 * pulse_bytes, p->hout[i], nb * pulse_bytes, cudaMemcpyDeviceToHost, p->s_d2h),
              "cudaMemcpyAsync(D2H)");
      DC_CUDA(cudaEventRecord(p->ev_out[i], p->s_d2h), "record");
    }
    return DC_OK;
  };
  s = release_after(p, slot, pipeline());
  if (s != DC_OK) return s;
  DC_CUDA(cudaStreamSynchronize(p->s_d2h), "cudaStreamSynchronize(D2H)");
  DC_CUDA(cudaStreamSynchronize(p->stream), "cudaStreamSynchronize");
  return DC_OK;
}

static dc_status prof_collect(dc_plan_t p) {
  if (p->recs.empty()) return DC_OK;
  DC_CUDA(cudaStreamSynchronize(p->stream), "cudaStreamSynchronize(profile)");
  for (auto &r : p->recs) {
    float ms = 0.f;
    DC_CUDA(cudaEventElapsedTime(&ms, r.a, r.b), "cudaEventElapsedTime");
    p->acc.launches[r.cls] += 1;
    p->acc.ms[r.cls] += ms;
    p->acc.samples[r.cls] += r.samples;
  }
  p->recs.clear();
  p->ev_used = 0;
  return DC_OK;
}

dc_status dc_profile_enable(dc_plan_t p, int enable) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  DC_CUDA(cudaStreamSynchronize(p->stream), "cudaStreamSynchronize(profile)");
  p->recs.clear();
  p->ev_used = 0;
  p->acc = dc_profile_t{};
  p->prof = enable != 0;
  return DC_OK;
}

dc_status dc_profile_read(dc_plan_t p, dc_profile_t *out) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  if (!out) return fail(DC_ERR_NULL_POINTER, "out is NULL");
  dc_status s = prof_collect(p);
  if (s != DC_OK) return s;
  *out = p->acc;
  return DC_OK;
}

dc_status dc_plan_info(dc_plan_t p, dc_plan_info_t *info) {
  if (!p) return fail(DC_ERR_NULL_POINTER, "plan is NULL");
  if (!info) return fail(DC_ERR_NULL_POINTER, "info is NULL");
  info->n = p->n;
  info->log2n = p->log2n;
  info->taps = p->taps;
  info->regime = p->regime;
  info->n1 = p->regime ? (1ll << p->P1) : 0;
  info->n2 = p->regime ? (1ll << p->P2) : 0;
  info->chunk_pulses = p->chunk;
  info->scratch_bytes = p->scratch_bytes;
  info->sm_count = p->sm_count;
  info->kernel_launches = p->launches;
  return DC_OK;
}

#pragma GCC visibility pop
}  // extern "C"
