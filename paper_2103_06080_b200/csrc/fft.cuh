// Shared-memory mixed-radix FFT (radices 2, 3, 4, 5, 7, 8) for sm_100a.
//
// Forward transforms are in-place Gentleman-Sande decimation in frequency:
// natural-order input, digit-reversed output.  Inverse transforms are the
// matching in-place decimation in time: digit-reversed input, natural
// output.  A forward -> pointwise -> inverse chain therefore never permutes
// (the pointwise factors live in digit-reversed order too), and each stage
// reads and writes the same r slots per butterfly, so one smem buffer and
// one barrier per stage suffice -- no ping-pong buffer, which is what lets a
// 10000-point fp64 column (160 KB) be transformed inside one CTA.
//
// Stage p (radix r, sub-transform length L, span s = L/r) on block b, lane i:
//   DIF: y_q = sum_m a_m w_r^{mq};  x[bL + i + q s] = y_q * W_L^{q i}
//   DIT: a_q = x[bL + i + q s] * W_L^{-q i};  x[bL + i + m s] = sum_q a_q w_r^{-mq}
// Twiddles come from one table W_n^t = exp(-2 pi i t / n), t < n, built on
// the host in extended precision (W_L^{qi} = W_n^{q i n / L}).
//
// Position p after a forward pass holds frequency f with
//   p = q1 (n/r1) + q2 (n/(r1 r2)) + ... ,  f = q1 + r1 q2 + r1 r2 q3 + ...
// (host side: FftDesc / freq_of_pos in capi.cu).
#pragma once
#include "common.cuh"

namespace nwb {

#define NWB_MAX_STAGES 24

struct FftDesc {
  int n;
  int nst;
  int radix[NWB_MAX_STAGES];
  int span[NWB_MAX_STAGES];  // L of each stage (n, n/r1, n/(r1 r2), ...)
};

// ------------------------------------------------------------ butterflies
// Forward uses w = exp(-2 pi i / r); INV uses the conjugate.

template <bool INV, typename V> __device__ __forceinline__ void bfly2(V* a) {
  V t = a[0];
  a[0] = cadd(t, a[1]);
  a[1] = csub(t, a[1]);
}

template <bool INV, typename V> __device__ __forceinline__ void bfly4(V* a) {
  V s02 = cadd(a[0], a[2]), d02 = csub(a[0], a[2]);
  V s13 = cadd(a[1], a[3]), d13 = mul_i<INV>(csub(a[1], a[3]));
  a[0] = cadd(s02, s13);
  a[2] = csub(s02, s13);
  a[1] = cadd(d02, d13);
  a[3] = csub(d02, d13);
}

template <bool INV, typename V> __device__ __forceinline__ void bfly8(V* a) {
  using R = decltype(V::x);
  const R h = (R)0.70710678118654752440;
  V e[4], o[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    e[m] = cadd(a[m], a[m + 4]);
    o[m] = csub(a[m], a[m + 4]);
  }
  // o[m] *= w8^{m} (forward: w8 = (1 - i)/sqrt2)
  o[1] = INV ? mk<V>((o[1].x - o[1].y) * h, (o[1].x + o[1].y) * h)
             : mk<V>((o[1].x + o[1].y) * h, (o[1].y - o[1].x) * h);
  o[2] = mul_i<INV>(o[2]);
  o[3] = INV ? mk<V>(-(o[3].x + o[3].y) * h, (o[3].x - o[3].y) * h)
             : mk<V>((o[3].y - o[3].x) * h, -(o[3].x + o[3].y) * h);
  bfly4<INV>(e);
  bfly4<INV>(o);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    a[2 * k] = e[k];
    a[2 * k + 1] = o[k];
  }
}

// odd prime radix r in {3, 5, 7}: pair a_k with a_{r-k}.
// cos / sin (2 pi m / r) for 1 <= m <= (r-1)/2, folded at compile time.
__host__ __device__ constexpr double odd_cos(int rad, int m) {
  return rad == 3 ? -0.5
       : rad == 5 ? (m == 1 ? 0.30901699437494742410 : -0.80901699437494742410)
       : (m == 1 ? 0.62348980185873353053 : m == 2 ? -0.22252093395631440429
                                                    : -0.90096886790241912624);
}
__host__ __device__ constexpr double odd_sin(int rad, int m) {
  return rad == 3 ? 0.86602540378443864676
       : rad == 5 ? (m == 1 ? 0.95105651629515357212 : 0.58778525229247312917)
       : (m == 1 ? 0.78183148246802980871 : m == 2 ? 0.97492791218182360702
                                                    : 0.43388373911755812048);
}

template <int RAD, bool INV, typename V> __device__ __forceinline__ void bfly_odd(V* a) {
  using R = decltype(V::x);
  constexpr int H = (RAD - 1) / 2;
  V t[H + 1], u[H + 1];
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    t[k] = cadd(a[k], a[RAD - k]);
    u[k] = csub(a[k], a[RAD - k]);
  }
  V y0 = a[0];
#pragma unroll
  for (int k = 1; k <= H; ++k) y0 = cadd(y0, t[k]);
#pragma unroll
  for (int q = 1; q <= H; ++q) {
    V bq = a[0];
    V cq = mk<V>(0, 0);
#pragma unroll
    for (int k = 1; k <= H; ++k) {
      const int m = (k * q) % RAD;
      const R cs = (R)odd_cos(RAD, m <= H ? m : RAD - m);
      const R sn = m <= H ? (R)odd_sin(RAD, m) : -(R)odd_sin(RAD, RAD - m);
      bq = mk<V>(bq.x + cs * t[k].x, bq.y + cs * t[k].y);
      cq = mk<V>(cq.x + sn * u[k].x, cq.y + sn * u[k].y);
    }
    // forward: y_q = b_q - i c_q, y_{r-q} = b_q + i c_q
    V ic = mul_i<true>(cq);
    a[q] = INV ? cadd(bq, ic) : csub(bq, ic);
    a[RAD - q] = INV ? csub(bq, ic) : cadd(bq, ic);
  }
  a[0] = y0;
}

template <int RAD, bool INV, typename V> __device__ __forceinline__ void bfly(V* a) {
  if constexpr (RAD == 2) bfly2<INV>(a);
  else if constexpr (RAD == 4) bfly4<INV>(a);
  else if constexpr (RAD == 8) bfly8<INV>(a);
  else bfly_odd<RAD, INV>(a);
}

// ------------------------------------------------------------ stages
// `rows` independent transforms of length n at x + row*rstride.

template <int RAD, typename V>
__device__ __forceinline__ void dif_stage(V* x, int n, int L, int rows, int rstride,
                                          const V* __restrict__ tw) {
  const int s = L / RAD;
  const int per_row = n / RAD;
  const int twm = n / L;
  const int total = per_row * rows;
  for (int g = threadIdx.x; g < total; g += blockDim.x) {
    const int row = g / per_row;
    const int h = g - row * per_row;
    const int blk = h / s;
    const int i = h - blk * s;
    V* base = x + row * rstride + blk * L + i;
    V a[RAD];
#pragma unroll
    for (int m = 0; m < RAD; ++m) a[m] = base[m * s];
    bfly<RAD, false>(a);
    if (i != 0) {
      const int step = i * twm;
#pragma unroll
      for (int q = 1; q < RAD; ++q) a[q] = cmul(a[q], __ldg(tw + q * step));
    }
#pragma unroll
    for (int q = 0; q < RAD; ++q) base[q * s] = a[q];
  }
}

template <int RAD, typename V>
__device__ __forceinline__ void dit_stage(V* x, int n, int L, int rows, int rstride,
                                          const V* __restrict__ tw) {
  const int s = L / RAD;
  const int per_row = n / RAD;
  const int twm = n / L;
  const int total = per_row * rows;
  for (int g = threadIdx.x; g < total; g += blockDim.x) {
    const int row = g / per_row;
    const int h = g - row * per_row;
    const int blk = h / s;
    const int i = h - blk * s;
    V* base = x + row * rstride + blk * L + i;
    V a[RAD];
#pragma unroll
    for (int q = 0; q < RAD; ++q) a[q] = base[q * s];
    if (i != 0) {
      const int step = i * twm;
#pragma unroll
      for (int q = 1; q < RAD; ++q) a[q] = cmulc(a[q], __ldg(tw + q * step));
    }
    bfly<RAD, true>(a);
#pragma unroll
    for (int m = 0; m < RAD; ++m) base[m * s] = a[m];
  }
}

// Caller must __syncthreads() before (input staged); returns after a barrier.
template <typename V>
__device__ void fft_forward(V* x, const FftDesc& d, int rows, int rstride, const V* tw) {
  for (int st = 0; st < d.nst; ++st) {
    const int L = d.span[st];
    switch (d.radix[st]) {
      case 2: dif_stage<2>(x, d.n, L, rows, rstride, tw); break;
      case 3: dif_stage<3>(x, d.n, L, rows, rstride, tw); break;
      case 4: dif_stage<4>(x, d.n, L, rows, rstride, tw); break;
      case 5: dif_stage<5>(x, d.n, L, rows, rstride, tw); break;
      case 7: dif_stage<7>(x, d.n, L, rows, rstride, tw); break;
      default: dif_stage<8>(x, d.n, L, rows, rstride, tw); break;
    }
    __syncthreads();
  }
}

template <typename V>
__device__ void fft_inverse(V* x, const FftDesc& d, int rows, int rstride, const V* tw) {
  for (int st = d.nst - 1; st >= 0; --st) {
    const int L = d.span[st];
    switch (d.radix[st]) {
      case 2: dit_stage<2>(x, d.n, L, rows, rstride, tw); break;
      case 3: dit_stage<3>(x, d.n, L, rows, rstride, tw); break;
      case 4: dit_stage<4>(x, d.n, L, rows, rstride, tw); break;
      case 5: dit_stage<5>(x, d.n, L, rows, rstride, tw); break;
      case 7: dit_stage<7>(x, d.n, L, rows, rstride, tw); break;
      default: dit_stage<8>(x, d.n, L, rows, rstride, tw); break;
    }
    __syncthreads();
  }
}

}  // namespace nwb
