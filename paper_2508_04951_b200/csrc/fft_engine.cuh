// fft_engine.cuh -- shared-memory Stockham FFT engine for sm_100a (product path).
//
// The ionospheric correction of Eq. 15 is DFT -> per-bin phase ->
// IDFT.  The DFTs here are a self-sorting Stockham formulation: each pass p
// with radix R and current span NS (product of the earlier radices) does, for
// every butterfly j in [0, L/R),
//     k = j mod NS
//     v[r] = in[j + r L/R] * w^(k r)        w = exp(-+ 2 pi i / (NS R))
//     V    = DFT_R(v)                        (in registers)
//     out[(j / NS) NS R + k + s NS] = V[s]
// and after the last pass `out` holds the transform in natural order.
//
// B200 mapping: every thread owns E complex samples
// (E/R butterflies per pass) in registers; passes exchange through shared
// memory with one barrier pair; the first pass reads straight from global
// memory and the last pass writes straight to global memory (both coalesced,
// because butterfly j touches elements j + r L/R); the last forward pass and
// the first inverse pass have the same element ownership, so the frequency-
// domain work between them happens in registers with no shared-memory trip.
#pragma once
#include "dc_common.cuh"

namespace dc {

// ----------------------------------------------------------------------------- constant twiddles
// cos(2 pi k / 32), k = 0..31
__device__ __forceinline__ constexpr float cos32(int k) {
  constexpr float t[32] = {1.0f,
                           0.98078528040323044913f,
                           0.92387953251128675613f,
                           0.83146961230254523708f,
                           0.70710678118654752440f,
                           0.55557023301960222474f,
                           0.38268343236508977173f,
                           0.19509032201612826785f,
                           0.0f,
                           -0.19509032201612826785f,
                           -0.38268343236508977173f,
                           -0.55557023301960222474f,
                           -0.70710678118654752440f,
                           -0.83146961230254523708f,
                           -0.92387953251128675613f,
                           -0.98078528040323044913f,
                           -1.0f,
                           -0.98078528040323044913f,
                           -0.92387953251128675613f,
                           -0.83146961230254523708f,
                           -0.70710678118654752440f,
                           -0.55557023301960222474f,
                           -0.38268343236508977173f,
                           -0.19509032201612826785f,
                           0.0f,
                           0.19509032201612826785f,
                           0.38268343236508977173f,
                           0.55557023301960222474f,
                           0.70710678118654752440f,
                           0.83146961230254523708f,
                           0.92387953251128675613f,
                           0.98078528040323044913f};
  return t[k & 31];
}

// v * exp(-+ 2 pi i K / N) for compile-time K/N with N | 32; exact special cases at multiples of pi/4.
template <int N, int K, bool INV>
__device__ __forceinline__ float2 rot(float2 v) {
  constexpr int k = ((K % N) + N) % N * (32 / N);  // in units of 2 pi / 32
  if constexpr (k == 0) {
    return v;
  } else if constexpr (k == 8) {
    return mul_mi<INV>(v);
  } else if constexpr (k == 16) {
    return make_float2(-v.x, -v.y);
  } else if constexpr (k == 24) {
    return mul_mi<!INV>(v);
  } else if constexpr (k == 4 || k == 12 || k == 20 || k == 28) {
    constexpr float h = 0.70710678118654752440f;
    // exp(-i 2 pi k/32) = (cx, -sx) forward; (cx, sx) inverse, with cx, sx = +-h
    constexpr float cx = (k == 4 || k == 28) ? h : -h;
    constexpr float sx = (k == 4 || k == 12) ? h : -h;  // sin(2 pi k / 32)
    constexpr float s = INV ? sx : -sx;                   // imaginary part of the rotation
    // (a + ib)(cx + i s) with |cx| = |s| = h: h * ((+-a -+ b) + i(...))
    const float2 p = make_float2(cx > 0 ? v.x : -v.x, s > 0 ? v.x : -v.x);
    const float2 q = make_float2(s > 0 ? -v.y : v.y, cx > 0 ? v.y : -v.y);
#if DC_X2
    return __fmul2_rn(__fadd2_rn(p, q), make_float2(h, h));
#else
    return make_float2((p.x + q.x) * h, (p.y + q.y) * h);
#endif
  } else {
    constexpr float c = cos32(k);
    constexpr float sn = cos32(k - 8);  // sin(2 pi k/32) = cos(2 pi (k-8)/32)
    constexpr float s = INV ? sn : -sn;
#if DC_X2
    return __ffma2_rn(make_float2(v.x, v.x), make_float2(c, s), __fmul2_rn(make_float2(v.y, v.y), make_float2(-s, c)));
#else
    return make_float2(fmaf(v.x, c, -v.y * s), fmaf(v.x, s, v.y * c));
#endif
  }
}

// ----------------------------------------------------------------------------- register DFTs
// In-place DFT_R of v[0..R-1] (natural order in and out), sign -1 forward, +1 inverse.
template <bool INV>
__device__ __forceinline__ void dft2(float2 &a, float2 &b) {
  float2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(float2 &v0, float2 &v1, float2 &v2, float2 &v3) {
  float2 t0 = cadd(v0, v2), t1 = csub(v0, v2);
  float2 t2 = cadd(v1, v3), t3 = mul_mi<INV>(csub(v1, v3));
  v0 = cadd(t0, t2);
  v2 = csub(t0, t2);
  v1 = cadd(t1, t3);
  v3 = csub(t1, t3);
}

template <int R, bool INV>
struct DFT;

template <bool INV>
struct DFT<2, INV> {
  __device__ __forceinline__ static void run(float2 *v) { dft2<INV>(v[0], v[1]); }
};
template <bool INV>
struct DFT<4, INV> {
  __device__ __forceinline__ static void run(float2 *v) { dft4<INV>(v[0], v[1], v[2], v[3]); }
};
template <bool INV>
struct DFT<8, INV> {
  // radix-2 DIT over two DFT4s
  __device__ __forceinline__ static void run(float2 *v) {
    dft4<INV>(v[0], v[2], v[4], v[6]);
    dft4<INV>(v[1], v[3], v[5], v[7]);
    float2 o1 = rot<8, 1, INV>(v[3]), o2 = rot<8, 2, INV>(v[5]), o3 = rot<8, 3, INV>(v[7]);
    float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6], o0 = v[1];
    v[0] = cadd(e0, o0);
    v[4] = csub(e0, o0);
    v[1] = cadd(e1, o1);
    v[5] = csub(e1, o1);
    v[2] = cadd(e2, o2);
    v[6] = csub(e2, o2);
    v[3] = cadd(e3, o3);
    v[7] = csub(e3, o3);
  }
};
template <bool INV>
struct DFT<16, INV> {
  // 4 x 4: A[r2][s1] = DFT4_r1 v[4 r1 + r2]; A *= w16^(r2 s1); V[s1 + 4 s2] = DFT4_r2 A[r2][s1]
  __device__ __forceinline__ static void run(float2 *v) {
#pragma unroll
    for (int r2 = 0; r2 < 4; ++r2) dft4<INV>(v[r2], v[4 + r2], v[8 + r2], v[12 + r2]);
    // now v[4 s1 + r2] holds A[r2][s1]
    v[5] = rot<16, 1, INV>(v[5]);
    v[6] = rot<16, 2, INV>(v[6]);
    v[7] = rot<16, 3, INV>(v[7]);
    v[9] = rot<16, 2, INV>(v[9]);
    v[10] = rot<16, 4, INV>(v[10]);
    v[11] = rot<16, 6, INV>(v[11]);
    v[13] = rot<16, 3, INV>(v[13]);
    v[14] = rot<16, 6, INV>(v[14]);
    v[15] = rot<16, 9, INV>(v[15]);
#pragma unroll
    for (int s1 = 0; s1 < 4; ++s1) dft4<INV>(v[4 * s1 + 0], v[4 * s1 + 1], v[4 * s1 + 2], v[4 * s1 + 3]);
    // v[4 s1 + s2] holds V[s1 + 4 s2]: transpose 4x4 in registers (free after unrolling)
    float2 t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = v[i];
#pragma unroll
    for (int s1 = 0; s1 < 4; ++s1)
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) v[s1 + 4 * s2] = t[4 * s1 + s2];
  }
};
template <bool INV>
struct DFT<32, INV> {
  // radix-2 DIT over two DFT16s
  __device__ __forceinline__ static void run(float2 *v) {
    float2 e[16], o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      e[i] = v[2 * i];
      o[i] = v[2 * i + 1];
    }
    DFT<16, INV>::run(e);
    DFT<16, INV>::run(o);
    o[1] = rot<32, 1, INV>(o[1]);
    o[2] = rot<32, 2, INV>(o[2]);
    o[3] = rot<32, 3, INV>(o[3]);
    o[4] = rot<32, 4, INV>(o[4]);
    o[5] = rot<32, 5, INV>(o[5]);
    o[6] = rot<32, 6, INV>(o[6]);
    o[7] = rot<32, 7, INV>(o[7]);
    o[8] = rot<32, 8, INV>(o[8]);
    o[9] = rot<32, 9, INV>(o[9]);
    o[10] = rot<32, 10, INV>(o[10]);
    o[11] = rot<32, 11, INV>(o[11]);
    o[12] = rot<32, 12, INV>(o[12]);
    o[13] = rot<32, 13, INV>(o[13]);
    o[14] = rot<32, 14, INV>(o[14]);
    o[15] = rot<32, 15, INV>(o[15]);
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      v[s] = cadd(e[s], o[s]);
      v[s + 16] = csub(e[s], o[s]);
    }
  }
};

// ----------------------------------------------------------------------------- pass plans
// L = 2^P split into passes of radix <= RMAX (RMAX = E, the samples a thread owns).
// Forward passes: the remainder radix first, then full radices; the inverse uses the
// reversed sequence so that (last forward pass) and (first inverse pass) share radix.
template <int P, int LOG_RMAX>
struct PassPlan {
  static constexpr int nfull = P / LOG_RMAX;
  static constexpr int rem = P % LOG_RMAX;
  static constexpr int npass = nfull + (rem ? 1 : 0);
  __host__ __device__ static constexpr int log_radix_fwd(int i) { return (rem && i == 0) ? rem : LOG_RMAX; }
  __host__ __device__ static constexpr int log_radix_inv(int i) { return log_radix_fwd(npass - 1 - i); }
  __host__ __device__ static constexpr int log_ns_fwd(int i) {
    int s = 0;
    for (int q = 0; q < i; ++q) s += log_radix_fwd(q);
    return s;
  }
  __host__ __device__ static constexpr int log_ns_inv(int i) {
    int s = 0;
    for (int q = 0; q < i; ++q) s += log_radix_inv(q);
    return s;
  }
  // twiddle-table offsets (entries) of pass i: sections [NS][R] per pass, concatenated
  __host__ __device__ static constexpr int tw_off_fwd(int i) {
    int s = 0;
    for (int q = 0; q < i; ++q) s += (1 << log_ns_fwd(q)) << log_radix_fwd(q);
    return s;
  }
  __host__ __device__ static constexpr int tw_off_inv(int i) {
    int s = 0;
    for (int q = 0; q < i; ++q) s += (1 << log_ns_inv(q)) << log_radix_inv(q);
    return s;
  }
  __host__ __device__ static constexpr int tw_size() {
    return tw_off_fwd(npass) > tw_off_inv(npass) ? tw_off_fwd(npass) : tw_off_inv(npass);
  }
};

// ----------------------------------------------------------------------------- tiles
// A tile is a set of NB independent L-point FFTs held by T threads x E samples.
// ROW tiles: FFT along contiguous (padded) rows of shared memory; rows = pulses
//            (single-CTA regime) or four-step rows k1 (pass B).
// COL tiles: FFT along the columns of an [L][NB] shared-memory tile; columns are
//            the four-step columns t2 (passes A and C).
template <int P_, int E_, int NB_, bool ROW_>
struct Tile {
  static constexpr int P = P_;
  static constexpr int L = 1 << P_;
  static constexpr int E = E_;
  static constexpr int LOGE = (E_ >= 32) ? 5 : (E_ >= 16) ? 4 : (E_ >= 8) ? 3 : (E_ >= 4) ? 2 : 1;
  static constexpr int NB = NB_;
  static constexpr bool ROW = ROW_;
  static constexpr int ELEMS = L * NB;
  static constexpr int T = ELEMS / E;
  // Bank-conflict padding.  ROW tiles: one pad slot per E samples, so the stride-R stores of
  // the NS = 1 pass (thread j writes R consecutive samples) land on distinct banks.  COL tiles:
  // one extra row of NB samples every E rows, so rows R apart alternate 64-byte bank halves.
  static constexpr int ROWSTRIDE = L + (L >> LOGE);
  static constexpr int COLROWS = L + (L >> LOGE);
  static constexpr int SMEM_ELEMS = ROW ? NB * ROWSTRIDE : COLROWS * NB;
  __device__ __forceinline__ static int sidx(int b, int i) {
    return ROW ? b * ROWSTRIDE + i + (i >> LOGE) : (i + (i >> LOGE)) * NB + b;
  }
  // butterfly g of a radix-R pass -> (FFT b, butterfly j)
  template <int R>
  __device__ __forceinline__ static void bmap(int g, int &b, int &j) {
    if constexpr (ROW) {
      b = g / (L / R);
      j = g % (L / R);
    } else {
      b = g % NB;
      j = g / NB;
    }
  }
};

// Stockham pass pieces on the E registers of one thread.  Butterfly q of the thread
// (q < E/R) is g = tid + q T and occupies v[q R .. q R + R - 1].
template <class TL, int R>
__device__ __forceinline__ void pass_load_smem(const float2 *__restrict__ s, float2 (&v)[TL::E], int tid) {
#pragma unroll
  for (int q = 0; q < TL::E / R; ++q) {
    int b, j;
    TL::template bmap<R>(tid + q * TL::T, b, j);
#pragma unroll
    for (int r = 0; r < R; ++r) v[q * R + r] = s[TL::sidx(b, j + r * (TL::L / R))];
  }
}

template <class TL, int R, int LOG_NS>
__device__ __forceinline__ void pass_store_smem(float2 *__restrict__ s, const float2 (&v)[TL::E], int tid) {
  constexpr int NS = 1 << LOG_NS;
#pragma unroll
  for (int q = 0; q < TL::E / R; ++q) {
    int b, j;
    TL::template bmap<R>(tid + q * TL::T, b, j);
    int k = j & (NS - 1);
    int base = ((j >> LOG_NS) << LOG_NS) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) s[TL::sidx(b, base + r * NS)] = v[q * R + r];
  }
}

// twiddle + radix-R DFT.  tw: this pass's table section (entry (k, r) = w^(k r), layout [R/2][NS][2]).
template <class TL, int R, int LOG_NS, bool INV>
__device__ __forceinline__ void pass_compute(float2 (&v)[TL::E], int tid, const float2 *__restrict__ tw) {
  constexpr int NS = 1 << LOG_NS;
#pragma unroll
  for (int q = 0; q < TL::E / R; ++q) {
    if constexpr (NS > 1) {
      int b, j;
      TL::template bmap<R>(tid + q * TL::T, b, j);
      int k = j & (NS - 1);
      // table section layout [R/2][NS] of float4 = (w^(k 2h), w^(k (2h+1))): lanes with
      // consecutive k read consecutive 16-byte words (conflict-free in shared memory)
      const float4 *t4 = reinterpret_cast<const float4 *>(tw) + k;
      float2 w[R];
#pragma unroll
      for (int h = 0; h < R / 2; ++h) {
        float4 p = t4[h * NS];  // shared-memory or L1-cached global table
        w[2 * h] = make_float2(p.x, p.y);
        w[2 * h + 1] = make_float2(p.z, p.w);
      }
#pragma unroll
      for (int r = 1; r < R; ++r) v[q * R + r] = INV ? cmulc(v[q * R + r], w[r]) : cmul(v[q * R + r], w[r]);
    }
    DFT<R, INV>::run(&v[q * R]);
  }
}

// element index (within FFT b) that register v[q R + r] holds after pass_compute of the LAST
// pass (NS = L / R): k = j + r NS.
template <class TL, int R>
__device__ __forceinline__ void last_pass_index(int tid, int q, int r, int &b, int &k) {
  int j;
  TL::template bmap<R>(tid + q * TL::T, b, j);
  k = j + r * (TL::L / R);
}

// Run forward passes [first, last] of a PassPlan on registers, exchanging through smem.
// On entry the registers hold pass `first`'s inputs; on exit they hold pass `last`'s outputs
// (not stored).  Barriers: one before every smem write, one after.
template <class TL, class PP, int I, int LAST, bool INV>
__device__ __forceinline__ void run_passes(float2 (&v)[TL::E], float2 *__restrict__ s, int tid,
                                           const float2 *__restrict__ tw) {
  constexpr int LR = INV ? PP::log_radix_inv(I) : PP::log_radix_fwd(I);
  constexpr int R = 1 << LR;
  constexpr int LNS = INV ? PP::log_ns_inv(I) : PP::log_ns_fwd(I);
  constexpr int OFF = INV ? PP::tw_off_inv(I) : PP::tw_off_fwd(I);
  pass_compute<TL, R, LNS, INV>(v, tid, tw + OFF);
  if constexpr (I < LAST) {
    constexpr int LR2 = INV ? PP::log_radix_inv(I + 1) : PP::log_radix_fwd(I + 1);
    __syncthreads();  // previous readers of s are done
    pass_store_smem<TL, R, LNS>(s, v, tid);
    __syncthreads();
    pass_load_smem<TL, 1 << LR2>(s, v, tid);
    run_passes<TL, PP, I + 1, LAST, INV>(v, s, tid, tw);
  }
}

}  // namespace dc
