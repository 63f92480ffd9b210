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

#define NWB_MAX_PASSES 16

struct FftDesc {
  int n;
  int np;                             // passes (1 or 2 fused stages each)
  int ptype[NWB_MAX_PASSES];          // 10 * ra + rb (rb = 1: single stage)
  int pspan[NWB_MAX_PASSES];          // L of the pass's first stage
  int pofs_a[NWB_MAX_PASSES];         // twiddle tables of stage a / b: coarse part
  int pofs_b[NWB_MAX_PASSES];         //   W_L^{64 c} at ofs + c, fine part W_L^f at
  int pfin_a[NWB_MAX_PASSES];         //   fin + f (f < 64): W_L^i = coarse[i>>6] fine[i&63]
  int pfin_b[NWB_MAX_PASSES];
  unsigned pmag_row[NWB_MAX_PASSES];  // magic for x / (n / (ra rb)), 0 = divide by 1
  unsigned pmag_sb[NWB_MAX_PASSES];   // magic for x / s_b
  // bank-conflict padding of the shared-memory line: element e lives at
  // e + e / pad_period (pad_period = element count of the last pass when it
  // is even, so its unit-stride butterflies hit distinct banks); 0 = none
  int pad_period;
  unsigned pad_magic;
  int pfast[NWB_MAX_PASSES];          // pad_period divides s_b: strides pre-padded
  int psa_p[NWB_MAX_PASSES];          // padded s_a, s_b (valid when pfast)
  int psb_p[NWB_MAX_PASSES];
  // j <-> -j symmetry of the digit-reversed output (first-stage radix r1,
  // block length M = n / r1; sym_r1 = 0: off): see sym_pos
  int sym_r1;
  int sym_m;
  unsigned sym_magic;                 // magic for x / M
  int sym_n;                          // canonical positions form the prefix [0, sym_n)
};

// physical slot of logical element e in a (padded) shared-memory line
__device__ __forceinline__ int pidx(const FftDesc& d, int e) {
  return d.pad_period ? e + (int)__umulhi((unsigned)e, d.pad_magic) : e;
}
// padded line length for n logical elements
__host__ __device__ inline int padded_len(int n, int pad_period) {
  return pad_period ? n + n / pad_period + 1 : n + 1;  // one slot of slack (c2r stages X[n])
}

// Canonical position of p under f -> -f (mod n).  With p = q1 M + rest
// (q1 the first-stage digit, i.e. f = q1 (mod r1)), negating f gives
// digits r1 - q1, r_i - 1 - q_i (q1 != 0), so the partner position is
// (r1 - q1) M + (M - 1 - rest): blocks 1 .. r1-1 pair up in reverse order
// and block 0 (f = 0 mod r1) is kept whole.  Tables that depend on f only
// through xi_f^2 (the phi multipliers, bitwise symmetric) are read at the
// canonical position, so 55-60 % of each table row is ever touched and the
// mirrored half comes from L2 (same column, read earlier in the walk).
// the symmetry fields of a descriptor, by value (no reference to a kernel
// parameter: taking one forces a local copy of the whole argument struct)
struct SymInfo {
  int r1, m;
  unsigned magic;
};
__device__ __forceinline__ SymInfo sym_info(const FftDesc& d) { return SymInfo{d.sym_r1, d.sym_m, d.sym_magic}; }
__device__ __forceinline__ int sym_pos(SymInfo d, int p) {
  if (d.r1 <= 1) return p;
  const int q1 = d.magic ? (int)__umulhi((unsigned)p, d.magic) : p;
  if (q1 == 0) return p;
  const int rest = p - q1 * d.m;
  const int q2 = d.r1 - q1;
  if (q1 < q2 || (q1 == q2 && 2 * rest <= d.m - 1)) return p;
  return q2 * d.m + (d.m - 1 - rest);
}
__device__ __forceinline__ int sym_pos(const FftDesc& d, int p) { return sym_pos(sym_info(d), p); }

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
      bq = caxpy(cs, t[k], bq);
      cq = caxpy(sn, u[k], cq);
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

// cos / sin (2 pi k / R) as compile-time constants (folded after unrolling):
// quadrant reduction, then a Taylor series on [0, pi/4] (~1 ulp)
__host__ __device__ constexpr double ce_sin_poly(double x) {
  double x2 = x * x, term = x, s = x;
  for (int k = 1; k < 12; ++k) {
    term *= -x2 / ((2.0 * k) * (2.0 * k + 1.0));
    s += term;
  }
  return s;
}
__host__ __device__ constexpr double ce_cos_poly(double x) {
  double x2 = x * x, term = 1.0, s = 1.0;
  for (int k = 1; k < 12; ++k) {
    term *= -x2 / ((2.0 * k - 1.0) * (2.0 * k));
    s += term;
  }
  return s;
}
// cos and sin of (pi/2) r / R for 0 <= r < R
__host__ __device__ constexpr double ce_cos_q(int r, int R) {
  return 2 * r <= R ? ce_cos_poly(1.57079632679489661923 * r / R)
                    : ce_sin_poly(1.57079632679489661923 * (R - r) / R);
}
__host__ __device__ constexpr double ce_sin_q(int r, int R) {
  return 2 * r <= R ? ce_sin_poly(1.57079632679489661923 * r / R)
                    : ce_cos_poly(1.57079632679489661923 * (R - r) / R);
}
__host__ __device__ constexpr double ce_cos2pi(int k, int R) {
  const int a = 4 * (k % R), q = a / R, r = a % R;
  return q == 0 ? ce_cos_q(r, R) : q == 1 ? -ce_sin_q(r, R) : q == 2 ? -ce_cos_q(r, R) : ce_sin_q(r, R);
}
__host__ __device__ constexpr double ce_sin2pi(int k, int R) {
  const int a = 4 * (k % R), q = a / R, r = a % R;
  return q == 0 ? ce_sin_q(r, R) : q == 1 ? ce_cos_q(r, R) : q == 2 ? -ce_sin_q(r, R) : -ce_cos_q(r, R);
}

// v * W_R^k with W_R = exp(-2 pi i / R) (CONJ: exp(+2 pi i / R)); k known at
// compile time after unrolling, the multiples of 1/8 turn are special-cased
template <int R, bool CONJ, typename V> __device__ __forceinline__ V cmul_root(V v, int k) {
  using S = decltype(V::x);
  k %= R;
  if (k == 0) return v;
  if (2 * k == R) return mk<V>(-v.x, -v.y);
  if (4 * k == R) return mul_i<CONJ>(v);           // W^k = -i (forward)
  if (4 * k == 3 * R) return mul_i<!CONJ>(v);      // W^k = +i (forward)
  const S c = (S)ce_cos2pi(k, R);
  const S s = CONJ ? (S)ce_sin2pi(k, R) : -(S)ce_sin2pi(k, R);  // W^k = c + i s
  if (8 * k == R || 8 * k == 3 * R || 8 * k == 5 * R || 8 * k == 7 * R) {
    // |c| = |s| = 1/sqrt2: (x + iy)(c + is) with one product per component
    return c == s ? mk<V>((v.x - v.y) * c, (v.x + v.y) * c) : mk<V>((v.x + v.y) * c, (v.y - v.x) * c);
  }
  return cmul(v, mk<V>(c, s));
}

// ------------------------------------------------------------ passes
// A pass is one stage or two consecutive stages (ra then rb) fused in
// registers: a thread loads the ra*rb elements {base + m s_a + n s_b}, runs
// them as one radix-(ra rb) butterfly (constant internal twiddles) and writes
// back -- one shared-memory round trip for two stages.  The per-lane twiddle
// W_L^i comes from a two-level table (coarse[i >> 6] * fine[i & 63]); its
// powers are products.  Index math uses multiply-high magic numbers (exact
// for x * d < 2^32, checked on the host).

template <bool CONJ, typename V> __device__ __forceinline__ V twmul(V a, V w) {
  return CONJ ? cmulc(a, w) : cmul(a, w);
}

__device__ __forceinline__ unsigned fdiv(unsigned x, unsigned magic) {
  return magic ? __umulhi(x, magic) : x;
}

// DIT=false: decimation in frequency (natural in, digit-reversed out);
// DIT=true: decimation in time (digit-reversed in, natural out).  CONJ uses
// conjugate roots and twiddles (unnormalised inverse transform).
template <int RA, int RB, bool DIT, bool CONJ, typename V>
__device__ __forceinline__ void fft_pass(V* x, const FftDesc& d, int p, int rows, int rstride,
                                         const V* __restrict__ tw, int tid, int nth) {
  const int L = d.pspan[p];
  const int sa = L / RA;            // stage-a span
  const int sb = sa / RB;           // lane range
  const int per_row = d.n / (RA * RB);  // butterflies per row (constant divisor)
  const int total = per_row * rows;
  const V* twa = tw + d.pofs_a[p];
  const V* fia = tw + d.pfin_a[p];
  for (int g = tid; g < total; g += nth) {
    const int row = (int)fdiv((unsigned)g, d.pmag_row[p]);
    const int h = g - row * per_row;
    const int blk = (int)fdiv((unsigned)h, d.pmag_sb[p]);
    const int i = h - blk * sb;
    V* xr = x + row * rstride;
    const int e0 = blk * L + i;
    const bool fast = d.pfast[p];
    const int pe0 = pidx(d, e0), psa = d.psa_p[p], psb = d.psb_p[p];
    V a[RA * RB];
#pragma unroll
    for (int m = 0; m < RA; ++m)
#pragma unroll
      for (int n2 = 0; n2 < RB; ++n2)
        a[m * RB + n2] = xr[fast ? pe0 + m * psa + n2 * psb : pidx(d, e0 + m * sa + n2 * sb)];
    // The two stages form one radix-R butterfly (R = ra rb) on the elements
    // i + (m rb + n2) s_b: stage a's twiddle W_L^{q (i + n2 s_b)} factors into
    // W_L^{q i} (common to the n2 inputs of stage b's DFT, so it moves to the
    // outputs) times the constant W_R^{q n2}; with stage b's W_{s_a}^{r i} =
    // W_L^{ra r i} the output (q, r) twiddle is W_L^{(q + ra r) i}.  All R - 1
    // output twiddles are powers of one W_L^i (two table loads, products in
    // a log-depth tree) instead of one table lookup per stage and lane.
    //
    // The pass whose blocks are one butterfly (s_b = 1, the last DIF / first
    // DIT pass) has i = 0: all its twiddles are 1 and are skipped (uniform
    // branch).  The table loads are issued up front; the powers are formed
    // next to their use so they are not live across the butterfly.
    const bool tw_on = sb > 1;
    V w1 = mk<V>(1, 0), w2 = mk<V>(0, 0);
    if (tw_on) { w1 = __ldg(twa + (i >> 6)); w2 = __ldg(fia + (i & 63)); }
    auto apply_tw = [&]() {
      if constexpr (RA == 5 && RB == 5) {
        // radix 25: W^{q + 5r} = W^q (W^5)^r from 4 + 4 powers (few live registers)
        V wq[5], w5[5];
        wq[1] = cmul(w1, w2);
        wq[2] = cmul(wq[1], wq[1]);
        wq[3] = cmul(wq[2], wq[1]);
        wq[4] = cmul(wq[2], wq[2]);
        w5[1] = cmul(wq[4], wq[1]);
        w5[2] = cmul(w5[1], w5[1]);
        w5[3] = cmul(w5[2], w5[1]);
        w5[4] = cmul(w5[2], w5[2]);
#pragma unroll
        for (int q = 1; q < 5; ++q) a[q * 5] = twmul<CONJ>(a[q * 5], wq[q]);
#pragma unroll
        for (int r = 1; r < 5; ++r) {
          a[r] = twmul<CONJ>(a[r], w5[r]);
#pragma unroll
          for (int q = 1; q < 5; ++q) a[q * 5 + r] = twmul<CONJ>(a[q * 5 + r], cmul(wq[q], w5[r]));
        }
        return;
      }
      V pw[RA * RB];
      pw[0] = mk<V>(1, 0);
      pw[1] = cmul(w1, w2);
#pragma unroll
      for (int t = 2; t < RA * RB; ++t) pw[t] = cmul(pw[t >> 1], pw[t - (t >> 1)]);
#pragma unroll
      for (int q = 0; q < RA; ++q)
#pragma unroll
        for (int r = 0; r < RB; ++r)
          if (q + RA * r) a[q * RB + r] = twmul<CONJ>(a[q * RB + r], pw[q + RA * r]);
    };
    if (!DIT) {
      // stage a over m (per n2), internal twiddles W_R^{q n2}
#pragma unroll
      for (int n2 = 0; n2 < RB; ++n2) {
        V t[RA];
#pragma unroll
        for (int m = 0; m < RA; ++m) t[m] = a[m * RB + n2];
        bfly<RA, CONJ>(t);
#pragma unroll
        for (int q = 0; q < RA; ++q) a[q * RB + n2] = cmul_root<RA * RB, CONJ>(t[q], q * n2);
      }
      if (RB > 1) {
        // stage b over n2 within each stage-a output q
#pragma unroll
        for (int q = 0; q < RA; ++q) {
          V t[RB];
#pragma unroll
          for (int n2 = 0; n2 < RB; ++n2) t[n2] = a[q * RB + n2];
          bfly<RB, CONJ>(t);
#pragma unroll
          for (int r = 0; r < RB; ++r) a[q * RB + r] = t[r];
        }
      }
      if (RA * RB > 1 && tw_on) apply_tw();
    } else {
      // inverse: output twiddles first, then stage b, internal twiddles, stage a
      if (RA * RB > 1 && tw_on) apply_tw();
      if (RB > 1) {
#pragma unroll
        for (int q = 0; q < RA; ++q) {
          V t[RB];
#pragma unroll
          for (int r = 0; r < RB; ++r) t[r] = a[q * RB + r];
          bfly<RB, CONJ>(t);
#pragma unroll
          for (int n2 = 0; n2 < RB; ++n2) a[q * RB + n2] = t[n2];
        }
      }
#pragma unroll
      for (int n2 = 0; n2 < RB; ++n2) {
        V t[RA];
#pragma unroll
        for (int q = 0; q < RA; ++q) t[q] = cmul_root<RA * RB, CONJ>(a[q * RB + n2], q * n2);
        bfly<RA, CONJ>(t);
#pragma unroll
        for (int m = 0; m < RA; ++m) a[m * RB + n2] = t[m];
      }
    }
#pragma unroll
    for (int m = 0; m < RA; ++m)
#pragma unroll
      for (int n2 = 0; n2 < RB; ++n2)
        xr[fast ? pe0 + m * psa + n2 * psb : pidx(d, e0 + m * sa + n2 * sb)] = a[m * RB + n2];
  }
}

// pass type codes (host planner in capi.cu): 10*ra + rb
template <bool DIT, bool CONJ, typename V>
__device__ __forceinline__ void run_pass(V* x, const FftDesc& d, int p, int rows, int rstride,
                                         const V* tw, int tid = threadIdx.x, int nth = blockDim.x) {
  switch (d.ptype[p]) {
    case 21: fft_pass<2, 1, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
    case 31: fft_pass<3, 1, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
    case 41: fft_pass<4, 1, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
    case 51: fft_pass<5, 1, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
    case 71: fft_pass<7, 1, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
    case 81: fft_pass<8, 1, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
    case 72: fft_pass<7, 2, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
    case 53: fft_pass<5, 3, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
    case 55:  // fp32 only (the host planner never emits it for fp64: register budget)
      if constexpr (sizeof(V) == 8) fft_pass<5, 5, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth);
      break;
    case 52: fft_pass<5, 2, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
    case 34: fft_pass<3, 4, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
    case 33: fft_pass<3, 3, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
    case 32: fft_pass<3, 2, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
    default: fft_pass<4, 4, DIT, CONJ>(x, d, p, rows, rstride, tw, tid, nth); break;
  }
}

// All drivers expect the input staged (caller's __syncthreads()) and return
// after a barrier.  first_pass > 0 skips leading passes (the cluster-split
// rho pass performs the first radix-2 stage while loading).

// forward DFT, natural -> digit-reversed
template <typename V>
__device__ void fft_forward(V* x, const FftDesc& d, int rows, int rstride, const V* tw,
                            int first_pass = 0) {
  for (int p = first_pass; p < d.np; ++p) {
    run_pass<false, false>(x, d, p, rows, rstride, tw);
    __syncthreads();
  }
}

// unnormalised inverse DFT, digit-reversed -> natural
template <typename V>
__device__ void fft_inverse(V* x, const FftDesc& d, int rows, int rstride, const V* tw,
                            int first_pass = 0) {
  for (int p = d.np - 1; p >= first_pass; --p) {
    run_pass<true, true>(x, d, p, rows, rstride, tw);
    __syncthreads();
  }
}

// Group variants for warp-specialised kernels: threads [tid0, tid0 + nth) of
// the CTA run the transform and synchronise on named barrier BAR only (the
// other warps of the CTA never touch it).
template <int BAR> __device__ __forceinline__ void group_sync(int nth) {
  asm volatile("bar.sync %0, %1;" ::"n"(BAR), "r"(nth) : "memory");
}
template <int BAR, typename V>
__device__ void fft_forward_grp(V* x, const FftDesc& d, const V* tw, int tid, int nth) {
  for (int p = 0; p < d.np; ++p) {
    run_pass<false, false>(x, d, p, 1, 0, tw, tid, nth);
    group_sync<BAR>(nth);
  }
}
template <int BAR, typename V>
__device__ void fft_inverse_grp(V* x, const FftDesc& d, const V* tw, int tid, int nth) {
  for (int p = d.np - 1; p >= 0; --p) {
    run_pass<true, true>(x, d, p, 1, 0, tw, tid, nth);
    group_sync<BAR>(nth);
  }
}

// unnormalised inverse DFT, natural -> digit-reversed
template <typename V>
__device__ void fft_inverse_dif(V* x, const FftDesc& d, int rows, int rstride, const V* tw) {
  for (int p = 0; p < d.np; ++p) {
    run_pass<false, true>(x, d, p, rows, rstride, tw);
    __syncthreads();
  }
}

}  // namespace nwb
