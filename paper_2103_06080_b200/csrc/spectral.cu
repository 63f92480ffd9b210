// Spectral passes of the ExpRK22 step (reference pkg/src/nwave/exprk.py).
//
//   theta c2r  -- rows of the rho-physical / theta-spectral state T -> V,
//                 fused with the LF speed alpha_theta (weno.py:93-103) and the
//                 divergence guard max|V| (exprk.py:297) reductions.
//   theta r2c  -- rows of b -> theta spectrum, written transposed.
//   rho pass   -- one rho column (one theta mode k) per CTA: forward FFT,
//                 the stage combine of exprk.py:161-173 in digit-reversed
//                 order, inverse FFT.
//
// Data layout in HBM: physical fields are
// (batch, nr, nt) row-major; spectral arrays are (batch, kk, ld) with the
// rho index contiguous, so the rho pass streams contiguous rows and the
// theta passes move R-row segments (R x 16 B fp64) per theta mode.
// Global -> shared staging uses cp.async (many 16-byte requests in flight
// per thread); the rho pass prefetches its combine operands into L2 with
// bulk (TMA) prefetches at entry so they arrive while the forward FFT runs.
#include <cooperative_groups.h>
#include <cstdlib>

#include "internal.h"

namespace nwb {

// ------------------------------------------------------------------ helpers

template <typename T>
__device__ __forceinline__ void block_max2(u64 a, u64 b, u64* dst_a, u64* dst_b) {
  __shared__ u64 red[2][32];
  a = warp_max_u64(a);
  b = warp_max_u64(b);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { red[0][w] = a; red[1][w] = b; }
  __syncthreads();
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    a = lane < nw ? red[0][lane] : 0ULL;
    b = lane < nw ? red[1][lane] : 0ULL;
    a = warp_max_u64(a);
    b = warp_max_u64(b);
    if (lane == 0) {
      if (dst_a) atomicMax(dst_a, a);
      if (dst_b) atomicMax(dst_b, b);
    }
  }
}

#ifndef NWB_THETA_MINB64
#define NWB_THETA_MINB64 2
#endif

// threads per theta CTA: 128 per staged row up to 256 (one-row CTAs are
// small, so more of them -- in different phases -- share an SM)
template <int R> constexpr int theta_threads() { return R == 1 ? 128 : 256; }
// elements per batch of independent table loads in the theta pre / post loops
#ifndef NWB_POST_UB
#define NWB_POST_UB 4
#endif
constexpr int POST_UB = NWB_POST_UB;
// five one-row fp64 CTAs per SM (96 registers, a 60-byte spill in the FFT
// driver): C2 theta-c2r 0.233 -> 0.226 ms against four (C1 / C4 unchanged)
#ifndef NWB_THETA_MINB_R1
#define NWB_THETA_MINB_R1 5
#endif
#ifndef NWB_THETA_MINB_SPLIT64
#define NWB_THETA_MINB_SPLIT64 3
#endif
template <typename T, int R, bool SPLIT = false> constexpr int theta_min_blocks() {
  return R == 1 ? (sizeof(T) == 8 ? NWB_THETA_MINB_R1 : 6)
                : (sizeof(T) == 8 ? (SPLIT && R == 2 ? NWB_THETA_MINB_SPLIT64 : NWB_THETA_MINB64) : 3);
}
// an fp32 rho column (<= 113 KB) leaves room for a second CTA per SM, whose
// loads then overlap this one's transforms
#ifndef NWB_RHO_MINB32
#define NWB_RHO_MINB32 2
#endif
template <typename T> constexpr int rho_min_blocks() { return sizeof(T) == 8 ? 1 : NWB_RHO_MINB32; }

// ------------------------------------------------------------------ theta c2r
// X[0..m] staged in natural order (Im of X[0], X[m] dropped as pocketfft's c2r
// does), then in place, pair by pair,
//   Z[k] = (X[k] + conj X[m-k]) + i (X[k] - conj X[m-k]) conj(W_nt^k),  k < m
//   Z[m-k] = conj(Ze) + i conj(Zo)
// an inverse m-point DIF (natural in, digit-reversed out), and
//   v[2n] = Re z[pos(n)] * scale, v[2n+1] = Im z[pos(n)] * scale.
//
// The reductions use per-row extremes: for a fixed row j the LF speed
// |fl(c_j + fl(B v))| is a composition of monotone rounded operations in v,
// so its maximum over the row is attained at v = max_k V or v = min_k V --
// evaluating it at the two extremes gives the per-element maximum bitwise,
// and max|V| = max(|max V|, |min V|).  The compares skip NaNs, so NaNs are
// flagged separately and reported as the NaN pattern 0x7ff..f (it sorts above
// every finite and infinite value, like the per-element bit maximum did).

template <typename T, int R>
__device__ __forceinline__ void c2r_pre(cplx<T>* z, const ThetaArgs<T>& a, int rs) {
  using V = cplx<T>;
  const int m = a.g.m, npairs = m / 2 + 1;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    V* zr = z + r * rs;
    for (int k0 = threadIdx.x; k0 < npairs; k0 += POST_UB * blockDim.x) {
      V w[POST_UB];
#pragma unroll
      for (int u = 0; u < POST_UB; ++u) {
        const int k = k0 + u * blockDim.x;
        w[u] = __ldg(&a.wk[k < npairs ? k : 0]);
      }
#pragma unroll
      for (int u = 0; u < POST_UB; ++u) {
        const int k = k0 + u * blockDim.x;
        if (k >= npairs) break;
        const int sk = pidx(a.dh, k), sm = pidx(a.dh, m - k);
        V xk = zr[sk];
        V xm = zr[sm];
        if (k == 0) { xk.y = 0; xm.y = 0; }
        const V ze = mk<V>(xk.x + xm.x, xk.y - xm.y);
        const V zo = cmulc(mk<V>(xk.x - xm.x, xk.y + xm.y), w[u]);
        zr[sk] = mk<V>(ze.x - zo.y, ze.y + zo.x);
        if (k != 0 && 2 * k != m) zr[sm] = mk<V>(ze.x + zo.y, zo.x - ze.y);
      }
    }
  }
}

// scale, store R rows (j0 + r jstep < nr) and fold their reductions into amax / vmax
template <typename T, int R>
__device__ __forceinline__ void c2r_post(const cplx<T>* z, const ThetaArgs<T>& a, int rs, int mem,
                                         int j0, int step, u64& amax, u64& vmax, int jstep = 1) {
  using V = cplx<T>;
  const int m = a.g.m, nr = a.g.nr;
  T* dst = a.phys_out + (size_t)mem * nr * a.g.nt;
  const T* up = a.upar ? a.upar + (size_t)(step + a.row_off) * (a.coef_ld ? a.coef_ld : nr) + a.coef_j0 : nullptr;
  const T two_pi = (T)6.283185307179586476925;
  const T scale = a.scale, bco = a.bcoef;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int j = j0 + r * jstep;
    if (j >= nr) break;
    const V* zr = z + r * rs;
    V* drow = reinterpret_cast<V*>(dst + (size_t)j * a.g.nt);
    T hi = -INFINITY, lo = INFINITY;
    bool nan = false;
    // the digit-reversal positions of POST_UB elements are loaded up front (one
    // batch of independent loads instead of a load -> use chain per element)
    for (int n0 = threadIdx.x; n0 < m; n0 += POST_UB * blockDim.x) {
      int ps[POST_UB];
#pragma unroll
      for (int u = 0; u < POST_UB; ++u) {
        const int n = n0 + u * blockDim.x;
        ps[u] = n < m ? __ldg(&a.pos_h[n]) : 0;
      }
#pragma unroll
      for (int u = 0; u < POST_UB; ++u) {
        const int n = n0 + u * blockDim.x;
        if (n >= m) break;
        const V zz = zr[pidx(a.dh, ps[u])];
        const T v0 = zz.x * scale, v1 = zz.y * scale;
        drow[n] = mk<V>(v0, v1);
        // plain compares (NaNs are caught by the flag below)
        const bool o = v0 > v1;
        const T mx = o ? v0 : v1, mn = o ? v1 : v0;
        hi = mx > hi ? mx : hi;
        lo = mn < lo ? mn : lo;
        nan |= (v0 != v0) | (v1 != v1);
      }
    }
    if (threadIdx.x < m) {
      const T c = up ? two_pi * up[j] : (T)0;
      amax = max(amax, max(abs_bits(c + bco * hi), abs_bits(c + bco * lo)));
      vmax = max(vmax, max(abs_bits(hi), abs_bits(lo)));
      if (nan) amax = vmax = 0x7fffffffffffffffULL;  // NaN, above every abs_bits value
    }
  }
}

// Fused last rho stage (SPLIT): slot r holds T'[k][r msub + i] (the r1
// sub-column inverses); the radix-R DIT stage of the rho inverse,
//   a_q = T'_q conj(W_nr^{q i}),  T[k][i + m msub] = sum_q a_q conj(w_R)^{mq},
// turns them into the R physical rows i + m msub in place.
template <typename T, int R>
__device__ __forceinline__ void split_dit_rows(cplx<T>* z, const ThetaArgs<T>& a, int rs, int i) {
  using V = cplx<T>;
  V w[R];
#pragma unroll
  for (int q = 1; q < R; ++q) w[q] = __ldg(&a.tw_first[q * i]);
  for (int k = threadIdx.x; k < a.g.kk; k += blockDim.x) {
    const int sk = pidx(a.dh, k);
    V v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = z[q * rs + sk];
#pragma unroll
    for (int q = 1; q < R; ++q) v[q] = cmulc(v[q], w[q]);
    bfly<R, true>(v);
#pragma unroll
    for (int m = 0; m < R; ++m) z[m * rs + sk] = v[m];
  }
}

// SPLIT: the CTA owns rows i + r msub (i = blockIdx.x < msub), else rows j0 + r
template <typename T, int R, bool SPLIT>
__global__ void __launch_bounds__(theta_threads<R>(), (theta_min_blocks<T, R, SPLIT>())) k_theta_c2r(const ThetaArgs<T> a) {
  step_stamp(a.ts);
  using V = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* z = reinterpret_cast<V*>(smem_raw);
  const int kk = a.g.kk, nr = a.g.nr, ld = a.g.ld;
  const int rs = padded_len(a.g.m, a.dh.pad_period);  // smem row stride (holds X[0..m])
  const int mem = blockIdx.y;
  const int j0 = SPLIT ? (int)blockIdx.x : (int)blockIdx.x * R;
  const int jstep = SPLIT ? a.msub : 1;
  const V* src = a.spec_in + (size_t)mem * kk * ld;
  for (int idx = threadIdx.x; idx < kk * R && !(a.debug & 4); idx += blockDim.x) {
    const int r = idx % R, k = idx / R, j = j0 + r * jstep;
    V* slot = &z[r * rs + pidx(a.dh, k)];
    // SPLIT: sub-column position r msub + i is stored interleaved at i r1 + r
    // (the R values of one k are adjacent: whole 32-byte sectors)
    if (SPLIT) cp_async_c(slot, &src[(size_t)k * ld + (a.ilv ? j0 * R + r : j)]);
    else if (j < nr) cp_async_c(slot, &src[(size_t)k * ld + j]);
    else *slot = mk<V>(0, 0);
  }
  cp_async_wait_all();
  __syncthreads();
  if (SPLIT) {
    split_dit_rows<T, R>(z, a, rs, j0);
    __syncthreads();
  }
  c2r_pre<T, R>(z, a, rs);
  __syncthreads();
  fft_inverse_dif(z, a.dh, R, rs, a.tw_h);
  if (a.debug & 4) return;
  const int step = a.step_ctr ? *a.step_ctr : 0;
  u64 amax = 0, vmax = 0;
  c2r_post<T, R>(z, a, rs, mem, j0, step, amax, vmax, jstep);
  if (a.alpha_bits || a.vmax_bits) {
    block_max2<T>(amax, vmax,
                  a.alpha_bits ? a.alpha_bits + (size_t)mem * a.alpha_stride : nullptr,
                  a.vmax_bits ? a.vmax_bits + (size_t)mem * a.vmax_stride + step : nullptr);
  }
}

// ------------------------------------------------------------------ theta r2c
// z[n] = v[2n] + i v[2n+1]; forward m-point DIF; then for each pair (k, m-k)
//   ze = (Z_k + conj Z_{m-k}) / 2,  zo = -i (Z_k - conj Z_{m-k}) / 2
//   X[k] = ze + W_nt^k zo,   X[m-k] = conj(ze - W_nt^k zo).

template <typename T, int R>
__device__ __forceinline__ void r2c_post(const cplx<T>* z, const ThetaArgs<T>& a, int rs, int mem,
                                         int j0) {
  using V = cplx<T>;
  const int m = a.g.m, ld = a.g.ld;
  const int jend = a.row_end ? a.row_end : a.g.nr;
  V* dst = a.spec_out + (size_t)mem * a.g.kk * ld;
  const int npairs = m / 2 + 1;
  const T half = (T)0.5;
  // positions and twiddles of POST_UB pairs are loaded up front (independent loads)
  for (int i0 = threadIdx.x; i0 < npairs * R; i0 += POST_UB * blockDim.x) {
    int pk[POST_UB], pm[POST_UB];
    V wk[POST_UB];
#pragma unroll
    for (int u = 0; u < POST_UB; ++u) {
      const int idx = i0 + u * blockDim.x, k = idx < npairs * R ? idx / R : 0;
      pk[u] = __ldg(&a.pos_h[k]);
      pm[u] = __ldg(&a.pos_h[k == 0 ? 0 : m - k]);
      wk[u] = __ldg(&a.wk[k]);
    }
#pragma unroll
    for (int u = 0; u < POST_UB; ++u) {
      const int idx = i0 + u * blockDim.x;
      if (idx >= npairs * R) break;
      const int r = idx % R, k = idx / R, j = j0 + r;
      if (j >= jend) continue;
      const V* zr = z + r * rs;
      const V zk = zr[pidx(a.dh, pk[u])];
      const V zm = zr[pidx(a.dh, pm[u])];
      const V ze = mk<V>(half * (zk.x + zm.x), half * (zk.y - zm.y));
      const V zo = mk<V>(half * (zk.y + zm.y), half * (zm.x - zk.x));
      const V wz = cmul(wk[u], zo);
      // k ld < kk ld <= 2^32: both transform lengths fit one CTA's shared memory
      dst[(unsigned)k * (unsigned)ld + j] = cadd(ze, wz);
      if (2 * k != m) {
        const V d = csub(ze, wz);
        dst[(unsigned)(m - k) * (unsigned)ld + j] = mk<V>(d.x, -d.y);
      }
    }
  }
}

// Fused first rho stage (SPLIT): for each theta mode k the R rows' spectra
// X_r[k] (rows i + r msub) go through the radix-R DIF stage of the rho FFT,
//   y_q = (sum_r X_r w_R^{rq}) W_nr^{q i}  -> position q msub + i of column k.
template <typename T, int R>
__device__ __forceinline__ void r2c_post_split(const cplx<T>* z, const ThetaArgs<T>& a, int rs,
                                               int mem, int i) {
  using V = cplx<T>;
  const int m = a.g.m, ld = a.g.ld;
  // position q msub + i stored at i R + q (interleaved, ThetaArgs::ilv) or at q msub + i
  V* dst = a.spec_out + (size_t)mem * a.g.kk * ld + (a.ilv ? (size_t)i * R : (size_t)i);
  const int qs = a.ilv ? 1 : a.msub;
  const int npairs = m / 2 + 1;
  const T half = (T)0.5;
  V w[R];
#pragma unroll
  for (int q = 1; q < R; ++q) w[q] = __ldg(&a.tw_first[q * i]);
  for (int k = threadIdx.x; k < npairs; k += blockDim.x) {
    const int pk = pidx(a.dh, __ldg(&a.pos_h[k]));
    const int pm = pidx(a.dh, __ldg(&a.pos_h[k == 0 ? 0 : m - k]));
    const V wk = __ldg(&a.wk[k]);
    V xk[R], xm[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const V zk = z[r * rs + pk], zm = z[r * rs + pm];
      const V ze = mk<V>(half * (zk.x + zm.x), half * (zk.y - zm.y));
      const V zo = mk<V>(half * (zk.y + zm.y), half * (zm.x - zk.x));
      const V wz = cmul(wk, zo);
      xk[r] = cadd(ze, wz);
      const V d = csub(ze, wz);
      xm[r] = mk<V>(d.x, -d.y);
    }
    bfly<R, false>(xk);
#pragma unroll
    for (int q = 1; q < R; ++q) xk[q] = cmul(xk[q], w[q]);
#pragma unroll
    for (int q = 0; q < R; ++q) dst[(size_t)k * ld + q * qs] = xk[q];
    if (2 * k != m) {
      bfly<R, false>(xm);
#pragma unroll
      for (int q = 1; q < R; ++q) xm[q] = cmul(xm[q], w[q]);
#pragma unroll
      for (int q = 0; q < R; ++q) dst[(size_t)(m - k) * ld + q * qs] = xm[q];
    }
  }
}

template <typename T, int R, bool SPLIT>
__global__ void __launch_bounds__(theta_threads<R>(), (theta_min_blocks<T, R, SPLIT>())) k_theta_r2c(const ThetaArgs<T> a) {
  step_stamp(a.ts);
  using V = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* z = reinterpret_cast<V*>(smem_raw);
  const int m = a.g.m, nr = a.g.nr;
  const int jend = SPLIT ? nr : (a.row_end ? a.row_end : nr);
  const int mem = blockIdx.y;
  const int j0 = SPLIT ? (int)blockIdx.x : a.row_begin + (int)blockIdx.x * R;
  const int jstep = SPLIT ? a.msub : 1;
  const T* src = a.phys_in + (size_t)mem * nr * a.g.nt;
  const int rs = padded_len(m, a.dh.pad_period);
  if (a.bulk && !(a.debug & 4)) {
    // rows as bulk copies of the padded line's P-element chunks (TMA engine)
    __shared__ __align__(8) unsigned long long bar;
    const int P = a.dh.pad_period ? a.dh.pad_period : 256;
    const int nch = (m + P - 1) / P;
    int valid = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) valid += j0 + r * jstep < jend;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) mbar_arrive_expect_tx(&bar, (unsigned)(valid * m * sizeof(V)));
    for (int idx = threadIdx.x; idx < nch * R; idx += blockDim.x) {
      const int r = idx / nch, c = idx - r * nch, j = j0 + r * jstep;
      const int e0 = c * P, cnt = min(P, m - e0);
      V* zr = z + r * rs;
      if (j < jend) {
        const V* srow = reinterpret_cast<const V*>(src + (size_t)j * a.g.nt);
        bulk_g2s(&zr[pidx(a.dh, e0)], srow + e0, (unsigned)(cnt * sizeof(V)), &bar);
      } else {
        for (int e = e0; e < e0 + cnt; ++e) zr[pidx(a.dh, e)] = mk<V>(0, 0);
      }
    }
    mbar_wait(&bar, 0);
    __syncthreads();
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int j = j0 + r * jstep;
      V* zr = z + r * rs;
      const V* srow = reinterpret_cast<const V*>(src + (size_t)j * a.g.nt);
      for (int n = threadIdx.x; n < m && !(a.debug & 4); n += blockDim.x) {
        if (j < jend) cp_async_c(&zr[pidx(a.dh, n)], &srow[n]);
        else zr[pidx(a.dh, n)] = mk<V>(0, 0);
      }
    }
    cp_async_wait_all();
    __syncthreads();
  }
  fft_forward(z, a.dh, R, rs, a.tw_h);
  if (a.debug & 4) return;
  if (SPLIT) r2c_post_split<T, R>(z, a, rs, mem, j0);
  else r2c_post<T, R>(z, a, rs, mem, j0);
}

// ------------------------------------------------------------------ theta passes, streaming
// Persistent, double-buffered variants (NWB_THETA_STREAM=1): one CTA per SM
// walks groups of R rows; the cp.async staging of group i+1 is in flight
// while group i is transformed and stored.  Reductions are accumulated per
// thread and flushed with one block reduction per member.

template <typename T, int R>
__device__ __forceinline__ void c2r_issue(const ThetaArgs<T>& a, cplx<T>* z, int rs, int grp,
                                          int gpm) {
  using V = cplx<T>;
  const int mem = grp / gpm, j0 = (grp - mem * gpm) * R;
  const V* src = a.spec_in + (size_t)mem * a.g.kk * a.g.ld;
  for (int idx = threadIdx.x; idx < a.g.kk * R; idx += blockDim.x) {
    const int r = idx % R, k = idx / R, j = j0 + r;
    V* slot = &z[r * rs + pidx(a.dh, k)];
    if (j < a.g.nr) cp_async_c(slot, &src[(size_t)k * a.g.ld + j]);
    else *slot = mk<V>(0, 0);
  }
}

template <typename T, int R>
__global__ void __launch_bounds__(512, 1) k_theta_c2r_stream(const ThetaArgs<T> a) {
  step_stamp(a.ts);
  using V = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nr = a.g.nr;
  const int rs = padded_len(a.g.m, a.dh.pad_period);
  V* buf[2] = {reinterpret_cast<V*>(smem_raw), reinterpret_cast<V*>(smem_raw) + R * rs};
  const int gpm = (nr + R - 1) / R, groups = gpm * a.g.batch;
  const int step = a.step_ctr ? *a.step_ctr : 0;
  int grp = blockIdx.x, it = 0;
  if (grp < groups) c2r_issue<T, R>(a, buf[0], rs, grp, gpm);
  cp_async_commit();
  u64 amax = 0, vmax = 0;
  for (; grp < groups; grp += gridDim.x, ++it) {
    V* z = buf[it & 1];
    const int nxt = grp + gridDim.x;
    if (nxt < groups) c2r_issue<T, R>(a, buf[(it + 1) & 1], rs, nxt, gpm);
    cp_async_commit();
    cp_async_wait_1();
    __syncthreads();
    const int mem = grp / gpm, j0 = (grp - mem * gpm) * R;
    c2r_pre<T, R>(z, a, rs);
    __syncthreads();
    fft_inverse_dif(z, a.dh, R, rs, a.tw_h);
    c2r_post<T, R>(z, a, rs, mem, j0, step, amax, vmax);
    // flush the reductions when this CTA's next group belongs to another member
    const bool flush = nxt >= groups || nxt / gpm != mem;
    if (flush && (a.alpha_bits || a.vmax_bits)) {
      block_max2<T>(amax, vmax,
                    a.alpha_bits ? a.alpha_bits + (size_t)mem * a.alpha_stride : nullptr,
                    a.vmax_bits ? a.vmax_bits + (size_t)mem * a.vmax_stride + step : nullptr);
      amax = vmax = 0;
    }
    __syncthreads();  // buffer it&1 is refilled two iterations later
  }
  cp_async_wait_0();
}

template <typename T, int R>
__device__ __forceinline__ void r2c_issue(const ThetaArgs<T>& a, cplx<T>* z, int rs, int grp,
                                          int gpm) {
  using V = cplx<T>;
  const int m = a.g.m;
  const int mem = grp / gpm, j0 = (grp - mem * gpm) * R;
  const T* src = a.phys_in + (size_t)mem * a.g.nr * a.g.nt;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int j = j0 + r;
    V* zr = z + r * rs;
    const V* srow = reinterpret_cast<const V*>(src + (size_t)j * a.g.nt);
    for (int n = threadIdx.x; n < m; n += blockDim.x) {
      if (j < a.g.nr) cp_async_c(&zr[pidx(a.dh, n)], &srow[n]);
      else zr[pidx(a.dh, n)] = mk<V>(0, 0);
    }
  }
}

template <typename T, int R>
__global__ void __launch_bounds__(512, 1) k_theta_r2c_stream(const ThetaArgs<T> a) {
  step_stamp(a.ts);
  using V = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nr = a.g.nr;
  const int rs = padded_len(a.g.m, a.dh.pad_period);
  V* buf[2] = {reinterpret_cast<V*>(smem_raw), reinterpret_cast<V*>(smem_raw) + R * rs};
  const int gpm = (nr + R - 1) / R, groups = gpm * a.g.batch;
  int grp = blockIdx.x, it = 0;
  if (grp < groups) r2c_issue<T, R>(a, buf[0], rs, grp, gpm);
  cp_async_commit();
  for (; grp < groups; grp += gridDim.x, ++it) {
    V* z = buf[it & 1];
    const int nxt = grp + gridDim.x;
    if (nxt < groups) r2c_issue<T, R>(a, buf[(it + 1) & 1], rs, nxt, gpm);
    cp_async_commit();
    cp_async_wait_1();
    __syncthreads();
    fft_forward(z, a.dh, R, rs, a.tw_h);
    const int mem = grp / gpm, j0 = (grp - mem * gpm) * R;
    r2c_post<T, R>(z, a, rs, mem, j0);
    __syncthreads();
  }
  cp_async_wait_0();
}

// ------------------------------------------------------------------ rho pass

template <typename V> __device__ __forceinline__ void prefetch_row(const V* p, int n) {
  prefetch_l2_bulk(p, (unsigned)((size_t)n * sizeof(V)) & ~15u);
}

// The stage combine of exprk.py:161-173 on one (half) column in
// digit-reversed order.  Operands of U elements per thread are loaded before
// any result is stored (the row pointers are __restrict__), so each thread
// keeps 4U independent 16-byte loads in flight -- the combine is a pure
// stream and needs that memory-level parallelism.
// XG: x is a global scratch row in plain position order (the warp-specialised
// pass, k_rho_ws) instead of the padded shared-memory line.
template <typename T, int MODE, bool XG = false>
__device__ __forceinline__ void rho_combine(cplx<T>* x, const FftDesc& d, int n,
                                            const cplx<T>* __restrict__ E,
                                            const cplx<T>* __restrict__ P1,
                                            const cplx<T>* __restrict__ P12,
                                            const cplx<T>* __restrict__ P2,
                                            cplx<T>* __restrict__ vh, cplx<T>* __restrict__ u,
                                            T ds, int debug, int tid = threadIdx.x,
                                            int nth = blockDim.x, int roll = 0,
                                            SymInfo dsym = SymInfo{-1, 0, 0u}, int pofs = 0) {
  using V = cplx<T>;
  constexpr int U = 4;
  const bool nl = debug & 2;
  for (int p0 = tid; p0 < n; p0 += U * nth) {
    if (roll > 0 && tid == 0) {
      // rolling L2 prefetch of the rows this CTA reads `roll` rounds from now
      // (tables only inside their canonical prefix [0, sym_n))
      const int s0 = p0 + roll * U * nth, s1 = min(s0 + U * nth, n), t1 = min(s1, d.sym_n);
      if (s0 < s1) {
        const unsigned nb = (unsigned)((s1 - s0) * sizeof(V)) & ~15u;
        if (MODE == RHO_STAGE1 || MODE == RHO_EULER) prefetch_l2_bulk(vh + s0, nb);
        if (MODE == RHO_STAGE2) prefetch_l2_bulk(u + s0, nb);
      }
      if (s0 < t1) {
        const unsigned nb = (unsigned)((t1 - s0) * sizeof(V)) & ~15u;
        if (MODE == RHO_STAGE1 || MODE == RHO_EULER) { prefetch_l2_bulk(E + s0, nb); prefetch_l2_bulk(P1 + s0, nb); }
        if (MODE == RHO_STAGE1) prefetch_l2_bulk(P12 + s0, nb);
        if (MODE == RHO_STAGE2) prefetch_l2_bulk(P2 + s0, nb);
      }
    }
    V b[U], o1[U], o2[U], o3[U], o4[U];
    int sp[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int p = p0 + q * nth;
      if (p < n) {
        sp[q] = XG ? p : pidx(d, p);
        b[q] = x[sp[q]];
        // tables: canonical +-f position (sub-columns: of global position pofs + p)
        const int tp = dsym.r1 >= 0 ? sym_pos(dsym, pofs + p) : sym_pos(d, p);
        if (MODE == RHO_STAGE1 && !nl) {
          o1[q] = E[tp]; o2[q] = vh[p]; o3[q] = P1[tp]; o4[q] = P12[tp];
        } else if (MODE == RHO_STAGE2) {
          o1[q] = P2[tp]; o2[q] = u[p];
        } else if (MODE == RHO_EULER) {
          o1[q] = E[tp]; o2[q] = vh[p]; o3[q] = P1[tp];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int p = p0 + q * nth;
      if (p >= n) continue;
      const V bb = b[q];
      if (MODE == RHO_STAGE1) {
        if (nl) { o1[q] = bb; o2[q] = bb; o3[q] = bb; o4[q] = bb; }
        const V ev = cmul(o1[q], o2[q]);
        u[p] = cadd(ev, cmul(mk<V>(ds * o4[q].x, ds * o4[q].y), bb));
        x[sp[q]] = cadd(ev, cmul(mk<V>(ds * o3[q].x, ds * o3[q].y), bb));
      } else if (MODE == RHO_STAGE2) {
        const V vn = cadd(o2[q], cmul(mk<V>(ds * o1[q].x, ds * o1[q].y), bb));
        vh[p] = vn;
        x[sp[q]] = vn;
      } else if (MODE == RHO_EULER) {
        const V vn = cadd(cmul(o1[q], o2[q]), cmul(mk<V>(ds * o3[q].x, ds * o3[q].y), bb));
        vh[p] = vn;
        x[sp[q]] = vn;
      } else if (MODE == RHO_INIT) {
        vh[p] = bb;
      }
    }
  }
}

// element j of column k of the in / out arrays (RhoArgs::blk_n: slab blocks)
template <typename T>
__device__ __forceinline__ size_t rho_io(const RhoArgs<T>& a, size_t row, int k, int j) {
  if (!a.blk_n) return row + j;
  int b = 0;
  while (b + 1 < a.blk_n && j >= a.blk_start[b + 1]) ++b;
  const int st = a.blk_start[b], len = a.blk_start[b + 1] - st;
  return (size_t)a.g.kk * st + (size_t)k * len + (j - st);
}

// The column's padded shared-memory line is contiguous between pad slots,
// so a column moves as ceil(n / P) bulk copies of P elements (TMA engine,
// one mbarrier for the load) instead of n per-element cp.async.
template <typename V>
__device__ __forceinline__ void column_bulk_load(V* x, const FftDesc& d, const V* src, int n,
                                                 unsigned long long* bar) {
  const int P = d.pad_period ? d.pad_period : 256;
  const int nch = (n + P - 1) / P;
  if (threadIdx.x == 0) mbar_init(bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, (unsigned)(n * sizeof(V)));
  for (int c = threadIdx.x; c < nch; c += blockDim.x) {
    const int e0 = c * P, cnt = min(P, n - e0);
    bulk_g2s(&x[pidx(d, e0)], src + e0, (unsigned)(cnt * sizeof(V)), bar);
  }
  mbar_wait(bar, 0);
}
template <typename V>
__device__ __forceinline__ void column_bulk_store(V* dst, const FftDesc& d, const V* x, int n) {
  const int P = d.pad_period ? d.pad_period : 256;
  const int nch = (n + P - 1) / P;
  fence_proxy_async_smem();
  __syncthreads();
  for (int c = threadIdx.x; c < nch; c += blockDim.x) {
    const int e0 = c * P, cnt = min(P, n - e0);
    bulk_s2g(dst + e0, &x[pidx(d, e0)], (unsigned)(cnt * sizeof(V)));
  }
  bulk_commit_wait_read();
}

template <typename T, int MODE>
__device__ __forceinline__ void rho_column(const RhoArgs<T>& a) {
  using V = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long load_bar;
  V* x = reinterpret_cast<V*>(smem_raw);
  const int n = a.dr.n;
  const int mem = blockIdx.x, k = blockIdx.y + a.k_off;
  const size_t row = ((size_t)mem * a.g.kk + k) * a.g.ld;
  const size_t trow = (size_t)k * a.g.ld;
  const V* src = a.in + row;
  if (MODE == RHO_REV2NAT) {
    V* dst = a.out + row;
    for (int f = threadIdx.x; f < n; f += blockDim.x) dst[f] = src[a.pos_r[f]];
    return;
  }
  if (a.stagger_ns > 0) {
    const int slot = blockIdx.x + blockIdx.y * gridDim.x;  // linear block id
    if (slot < a.stagger_slots) {
      const long long wait = a.stagger_mode == 1 ? ((slot & 1) ? a.stagger_ns : 0)
                                                 : (long long)slot * a.stagger_ns / a.stagger_slots;
      if (threadIdx.x == 0 && wait > 0) {
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do {
          __nanosleep(500);
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        } while ((long long)(t - t0) < wait);
      }
      __syncthreads();
    }
  }
  if (a.prefetch && threadIdx.x == 0) {
    // the combine operands are consumed after the forward FFT: start their
    // DRAM -> L2 traffic now so it overlaps the transform (the first
    // a.prefetch percent of each row: the combine walks the rows head first)
    const int np = a.prefetch >= 100 ? n : (int)((long)n * a.prefetch / 100);
    if (MODE == RHO_STAGE1) {
      prefetch_row(a.vh + row, np);
      prefetch_row(a.E + trow, np);
      prefetch_row(a.P1 + trow, np);
      prefetch_row(a.P12 + trow, np);
    } else if (MODE == RHO_STAGE2) {
      prefetch_row(a.u + row, np);
      prefetch_row(a.P2 + trow, np);
    } else if (MODE == RHO_EULER) {
      prefetch_row(a.vh + row, np);
      prefetch_row(a.E + trow, np);
      prefetch_row(a.P1 + trow, np);
    }
  }
  if (MODE == RHO_INV_NAT) {
    for (int f = threadIdx.x; f < n; f += blockDim.x) {
      const int p = a.pos_r[f];
      const V val = src[f];
      x[pidx(a.dr, p)] = val;
      if (a.vh) a.vh[row + p] = val;
    }
  } else if (a.blk_n) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) cp_async_c(&x[pidx(a.dr, j)], &a.in[rho_io(a, row, k, j)]);
    cp_async_wait_all();
  } else if (a.bulk && !(a.debug & 4)) {
    column_bulk_load(x, a.dr, src, n, &load_bar);
  } else if (!(a.debug & 4)) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) cp_async_c(&x[pidx(a.dr, j)], &src[j]);
    cp_async_wait_all();
  }
  if (a.zero_bits && k == 0 && threadIdx.x == 0) a.zero_bits[(size_t)mem * a.zero_stride] = 0ULL;
  __syncthreads();
  if (MODE != RHO_INV_NAT && !(a.debug & 1)) fft_forward(x, a.dr, 1, 0, a.tw_r);

  if (MODE == RHO_FWD_NAT) {
    V* dst = a.out + row;
    for (int f = threadIdx.x; f < n; f += blockDim.x) dst[f] = x[pidx(a.dr, a.pos_r[f])];
    return;
  }
  // debug bit 4 (measurement only): transforms without any global traffic
  if (!(a.debug & 4))
    rho_combine<T, MODE>(x, a.dr, n, a.E + trow, a.P1 + trow, a.P12 + trow, a.P2 + trow,
                         a.vh + row, a.u + row, a.ds, a.debug, threadIdx.x, blockDim.x, a.roll);
  if (a.next_pf && threadIdx.x == 0 && k + a.next_pf < a.g.kk)
    prefetch_row(a.in + row + (size_t)a.next_pf * a.g.ld, n);  // a later CTA's column input
  __syncthreads();
  if (!(a.debug & 1)) fft_inverse(x, a.dr, 1, 0, a.tw_r);
  V* dst = a.out + row;
  if (a.blk_n)
    for (int j = threadIdx.x; j < n; j += blockDim.x) a.out[rho_io(a, row, k, j)] = x[pidx(a.dr, j)];
  else if (a.bulk && !(a.debug & 4))
    column_bulk_store(dst, a.dr, x, n);
  else if (!(a.debug & 4))
    for (int j = threadIdx.x; j < n; j += blockDim.x) dst[j] = x[pidx(a.dr, j)];
  if (a.step_ctr && mem == 0 && k == 0 && threadIdx.x == 0) *a.step_ctr += 1;
}

template <typename T, int MODE>
__global__ void __launch_bounds__(512, rho_min_blocks<T>()) k_rho(const RhoArgs<T> a) {
  rho_column<T, MODE>(a);
}
// fp32 columns of >= 384 threads (two CTAs per SM): a 384-thread bound gives
// the FFT 80 registers instead of 64 (232-byte spills): C2 fp32 rho 0.560 ->
// 0.543 ms per step.  Short fp32 columns keep k_rho (64 registers, more CTAs
// per SM: C4 fp32 6.33 -> 6.13 ms per step).
template <typename T, int MODE>
__global__ void __launch_bounds__(384, 2) k_rho_r80(const RhoArgs<T> a) {
  rho_column<T, MODE>(a);
}

// ------------------------------------------------------------------ rho pass, half-resident columns
// Two fp64 columns per SM with the whole column on chip: a 256-thread CTA
// keeps one half of its column in an 80 KB shared-memory line and parks the
// other half in TENSOR MEMORY (tcgen05.st / tcgen05.ld, 160 of the CTA's 256
// allocated TMEM columns; TMEM is 256 KB per SM and otherwise unused here), so
// two CTAs -- two columns, one streaming while the other transforms -- share
// an SM where k_rho fits one 160 KB column.  Thread t owns the indices
// s = t + 256 q (q < KPT); with the plan's first stage radix 2 (positions
// q1 n/2 + p'):
//   load   y0 = x_s + x_{s+M} -> TMEM, y1 = (x_s - x_{s+M}) W_n^s -> line
//   FFT y1 (line); swap TMEM <-> line (own index set); FFT y0 (line)
//   combine  y0 half in the line (positions p'), y1 half in TMEM (M + s)
//   inverse y0 (DIT, natural out); swap; inverse y1
//   store  x_s = z0 + conj(W_n^s) z1, x_{s+M} = z0 - conj(W_n^s) z1
// TMEM moves 4 complex (16 32-bit words) per tcgen05.{st,ld}.32x32b.x16; a
// warp reaches its lane quarter (warp mod 4), warps w and w + 4 use disjoint
// column ranges.
constexpr int HALF_NT = 256;
constexpr int HALF_CHUNK = 4;  // complex per TMEM transfer

__device__ __forceinline__ void tmem_st16(unsigned taddr, const double2 (&v)[HALF_CHUNK]) {
  unsigned w[16];
#pragma unroll
  for (int i = 0; i < HALF_CHUNK; ++i) {
    w[4 * i + 0] = (unsigned)__double2loint(v[i].x);
    w[4 * i + 1] = (unsigned)__double2hiint(v[i].x);
    w[4 * i + 2] = (unsigned)__double2loint(v[i].y);
    w[4 * i + 3] = (unsigned)__double2hiint(v[i].y);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};\n" ::"r"(taddr),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
      "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(unsigned taddr, double2 (&v)[HALF_CHUNK]) {
  unsigned w[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];\n"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]),
        "=r"(w[14]), "=r"(w[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < HALF_CHUNK; ++i) {
    v[i].x = __hiloint2double((int)w[4 * i + 1], (int)w[4 * i + 0]);
    v[i].y = __hiloint2double((int)w[4 * i + 3], (int)w[4 * i + 2]);
  }
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

template <int MODE, int KPT>
__global__ void __launch_bounds__(HALF_NT, 2) k_rho_half(const RhoArgs<double> a) {
  using V = double2;
  static_assert(KPT % HALF_CHUNK == 0, "KPT must be a multiple of the TMEM chunk");
  constexpr int NCH = KPT / HALF_CHUNK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned tmem_base_sh;
  V* x = reinterpret_cast<V*>(smem_raw);
  const FftDesc& d = a.dh2;
  const int M = d.n, t = threadIdx.x, warp = t >> 5;
  const int mem = blockIdx.x, k = blockIdx.y;
  const size_t row = ((size_t)mem * a.g.kk + k) * a.g.ld;
  const size_t trow = (size_t)k * a.g.ld;
  if (a.stagger_ns > 0) {
    const int slot = blockIdx.x + blockIdx.y * gridDim.x;
    if (slot < a.stagger_slots) {
      const long long wait = (long long)slot * a.stagger_ns / a.stagger_slots;
      if (t == 0 && wait > 0) {
        unsigned long long t0, tn;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do {
          __nanosleep(500);
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
        } while ((long long)(tn - t0) < wait);
      }
      __syncthreads();
    }
  }
  // TMEM: 256 columns for this CTA (two CTAs per SM fill the 512)
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(
                     smem_u32(&tmem_base_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // this warp's lane quarter and column range: 4 words per complex
  const unsigned tbase = tmem_base_sh + ((unsigned)(32 * (warp & 3)) << 16) +
                         (unsigned)((warp >> 2) * KPT * 4);
  auto col = [&](int c) { return tbase + (unsigned)(c * HALF_CHUNK * 4); };
  auto sidx_of = [&](int c, int i) { return t + HALF_NT * (c * HALF_CHUNK + i); };

  // load + first radix-2 DIF stage
  const V* src = a.in + row;
#pragma unroll 1
  for (int c = 0; c < NCH; ++c) {
    V y0[HALF_CHUNK];
#pragma unroll
    for (int i = 0; i < HALF_CHUNK; ++i) {
      const int si = sidx_of(c, i);
      y0[i] = mk<V>(0, 0);
      if (si < M) {
        const V x0 = src[si], x1 = src[si + M];
        y0[i] = cadd(x0, x1);
        x[pidx(d, si)] = cmul(csub(x0, x1), __ldg(&a.tw_split[si]));
      }
    }
    tmem_st16(col(c), y0);
  }
  tmem_wait_st();
  if (a.zero_bits && k == 0 && t == 0) a.zero_bits[(size_t)mem * a.zero_stride] = 0ULL;
  __syncthreads();
  // swap: y1_hat (line) <-> y0 (TMEM), own index set
  auto swap_line_tmem = [&]() {
#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
      V tv[HALF_CHUNK], lv[HALF_CHUNK];
      tmem_ld16(col(c), tv);
#pragma unroll
      for (int i = 0; i < HALF_CHUNK; ++i) {
        const int si = sidx_of(c, i);
        lv[i] = mk<V>(0, 0);
        if (si < M) {
          const int ps = pidx(d, si);
          lv[i] = x[ps];
          x[ps] = tv[i];
        }
      }
      tmem_st16(col(c), lv);
    }
    tmem_wait_st();
  };
  // one call site per transform direction (a second call site would copy
  // the kernel-parameter descriptor to local memory)
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    fft_forward(x, d, 1, 0, a.tw_h2);
    if (h == 0) {
      swap_line_tmem();
      __syncthreads();
    }
  }
  // combine: the y0 half in the line (positions p' < M) ...
  const SymInfo sym = sym_info(a.dr);
  rho_combine<double, MODE>(x, d, M, a.E + trow, a.P1 + trow, a.P12 + trow, a.P2 + trow,
                            a.vh + row, a.u + row, a.ds, 0, t, HALF_NT, 0, sym, 0);
  // ... and the y1 half in TMEM (positions M + s)
  {
    const V* E = a.E + trow;
    const V* P1 = a.P1 + trow;
    const V* P12 = a.P12 + trow;
    const V* P2 = a.P2 + trow;
    V* vh = a.vh + row;
    V* u = a.u + row;
    const double ds = a.ds;
#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
      V bv[HALF_CHUNK];
      tmem_ld16(col(c), bv);
#pragma unroll
      for (int i = 0; i < HALF_CHUNK; ++i) {
        const int si = sidx_of(c, i);
        if (si >= M) continue;
        const int p = M + si;
        const int tp = sym_pos(sym, p);
        const V bb = bv[i];
        if (MODE == RHO_STAGE1) {
          const V ev = cmul(E[tp], vh[p]);
          const V p12 = P12[tp], p1 = P1[tp];
          u[p] = cadd(ev, cmul(mk<V>(ds * p12.x, ds * p12.y), bb));
          bv[i] = cadd(ev, cmul(mk<V>(ds * p1.x, ds * p1.y), bb));
        } else if (MODE == RHO_STAGE2) {
          const V p2 = P2[tp];
          const V vn = cadd(u[p], cmul(mk<V>(ds * p2.x, ds * p2.y), bb));
          vh[p] = vn;
          bv[i] = vn;
        } else if (MODE == RHO_EULER) {
          const V p1 = P1[tp];
          const V vn = cadd(cmul(E[tp], vh[p]), cmul(mk<V>(ds * p1.x, ds * p1.y), bb));
          vh[p] = vn;
          bv[i] = vn;
        } else if (MODE == RHO_INIT) {
          vh[p] = bb;
        }
      }
      tmem_st16(col(c), bv);
    }
    tmem_wait_st();
  }
  __syncthreads();
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    fft_inverse(x, d, 1, 0, a.tw_h2);  // h = 0: z0, h = 1: z1, natural order
    if (h == 0) {
      swap_line_tmem();  // z0 -> TMEM, y1 combined -> line
      __syncthreads();
    }
  }
  V* dst = a.out + row;
#pragma unroll 1
  for (int c = 0; c < NCH; ++c) {
    V z0[HALF_CHUNK];
    tmem_ld16(col(c), z0);
#pragma unroll
    for (int i = 0; i < HALF_CHUNK; ++i) {
      const int si = sidx_of(c, i);
      if (si < M) {
        const V z1 = cmulc(x[pidx(d, si)], __ldg(&a.tw_split[si]));
        dst[si] = cadd(z0[i], z1);
        dst[si + M] = csub(z0[i], z1);
      }
    }
  }
  if (a.step_ctr && mem == 0 && k == 0 && t == 0) *a.step_ctr += 1;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem_base_sh)
                 : "memory");
}

// ------------------------------------------------------------------ rho pass, sub-columns
// With the first rho stage fused into the theta passes (ThetaArgs::r1), a rho
// column k splits into r1 independent msub-point sub-columns: position
// q1 msub + p' of the digit-reversed spectrum is position p' of the msub-point
// DIF transform of sub-column q1 (the r1-radix stage is the transform's
// first).  One CTA per sub-column: a C2 fp64 column (160 KB) becomes two
// 80 KB sub-columns, so two CTAs share an SM and one streams while the other
// transforms.  Modes as k_rho; RHO_FWD_DR stores the forward transform in
// digit-reversed positions (rfft2 then permutes with RHO_REV2NAT) and
// RHO_INV_NAT gathers its natural-order input by position -> frequency.
#ifndef NWB_RHO_SUB_MINB64
#define NWB_RHO_SUB_MINB64 2
#endif
template <typename T> constexpr int rho_sub_min_blocks() { return sizeof(T) == 8 ? NWB_RHO_SUB_MINB64 : 3; }

template <typename T, int MODE>
__global__ void __launch_bounds__(256, rho_sub_min_blocks<T>()) k_rho_sub(const RhoArgs<T> a) {
  using V = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* x = reinterpret_cast<V*>(smem_raw);
  const FftDesc& d = a.dsub;
  const int ms = d.n, r1 = a.r1;
  const int mem = blockIdx.x, k = blockIdx.y / r1, q1 = blockIdx.y - k * r1;
  const size_t row = ((size_t)mem * a.g.kk + k) * a.g.ld;
  const size_t sub = row + (size_t)q1 * ms;
  const size_t trow = (size_t)k * a.g.ld;
  if (MODE == RHO_INV_NAT) {
    // natural-order column in: gather this sub-column's positions
    const int* fr = a.rev_r + (size_t)q1 * ms;
    for (int p = threadIdx.x; p < ms; p += blockDim.x) {
      const V val = a.in[row + __ldg(&fr[p])];
      x[pidx(d, p)] = val;
      if (a.vh) a.vh[sub + p] = val;
    }
  } else {
    // transit arrays (theta passes <-> rho pass) hold position q1 msub + j at
    // j r1 + q1: the r1 sub-columns of a column interleave
    const int js = a.ilv ? r1 : 1;
    const V* src = a.in + (a.ilv ? row + q1 : sub);
    for (int j = threadIdx.x; j < ms; j += blockDim.x) cp_async_c(&x[pidx(d, j)], &src[(size_t)j * js]);
    cp_async_wait_all();
  }
  if (a.zero_bits && blockIdx.y == 0 && threadIdx.x == 0) a.zero_bits[(size_t)mem * a.zero_stride] = 0ULL;
  __syncthreads();
  if (MODE != RHO_INV_NAT) fft_forward(x, d, 1, 0, a.tw_sub);
  if (MODE == RHO_FWD_DR) {  // plain position order (RHO_REV2NAT permutes next)
    V* dst = a.out + sub;
    for (int p = threadIdx.x; p < ms; p += blockDim.x) dst[p] = x[pidx(d, p)];
    return;
  }
  if (MODE != RHO_INV_NAT)
    rho_combine<T, MODE>(x, d, ms, a.E + trow, a.P1 + trow, a.P12 + trow, a.P2 + trow,
                         a.vh + sub, a.u + sub, a.ds, 0, threadIdx.x, blockDim.x, 0,
                         sym_info(a.dr), q1 * ms);
  __syncthreads();
  fft_inverse(x, d, 1, 0, a.tw_sub);
  const int js = a.ilv ? r1 : 1;
  V* dst = a.out + (a.ilv ? row + q1 : sub);
  for (int j = threadIdx.x; j < ms; j += blockDim.x) dst[(size_t)j * js] = x[pidx(d, j)];
  if (a.step_ctr && mem == 0 && blockIdx.y == 0 && threadIdx.x == 0) *a.step_ctr += 1;
}

// ------------------------------------------------------------------ rho pass, warp-specialised
// One 160 KB fp64 column fills an SM's shared memory, so in k_rho the SM
// alternates between transforming and streaming.  Here a persistent CTA splits
// into two warp groups that run concurrently on different columns:
//   G1 (threads [0, nfft)): transforms.  Iteration i: inverse of column i-2
//      (combined row read back from an L2-resident scratch slot) and store of
//      its result, then load + forward transform of column i, written to the
//      scratch slot i & 1.  Its barriers are named barrier 1 over G1 only.
//   G2 (the remaining warps): the stage combine of column i-1 on its scratch
//      slot -- all the table / state / U streaming -- while G1 transforms.
// One __syncthreads per iteration hands the slots over (it orders the
// global-memory scratch traffic within the CTA).  The scratch (2 slots per
// CTA, 47 MB at C2 fp64) stays in L2; HBM sees the same compulsory bytes as
// k_rho.
template <typename T, int MODE>
__global__ void __launch_bounds__(512, 1) k_rho_ws(const RhoArgs<T> a) {
  using V = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* x = reinterpret_cast<V*>(smem_raw);
  const int n = a.dr.n;
  const int items = a.g.batch * a.g.kk;
  const int nfft = a.ws_threads;
  const bool fft_group = (int)threadIdx.x < nfft;
  const int tid2 = (int)threadIdx.x - nfft, nth2 = (int)blockDim.x - nfft;
  V* const scr = a.scratch + (size_t)blockIdx.x * 2 * a.g.ld;
  const int ncol = (int)blockIdx.x < items ? (items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  for (int i = 0; i < ncol + 2; ++i) {
    if (fft_group) {
      const int tid = threadIdx.x;
      if (i >= 2) {
        const int w = blockIdx.x + (i - 2) * gridDim.x;
        const int mem = w % a.g.batch, k = w / a.g.batch;
        const size_t row = ((size_t)mem * a.g.kk + k) * a.g.ld;
        const V* sc = scr + (size_t)(i & 1) * a.g.ld;
        for (int j = tid; j < n; j += nfft) cp_async_c(&x[pidx(a.dr, j)], &sc[j]);
        cp_async_wait_all();
        group_sync<1>(nfft);
        if (!(a.ws_debug & 2)) fft_inverse_grp<1>(x, a.dr, a.tw_r, tid, nfft);
        V* dst = a.out + row;
        for (int j = tid; j < n; j += nfft) dst[j] = x[pidx(a.dr, j)];
        if (a.step_ctr && mem == 0 && k == 0 && tid == 0) *a.step_ctr += 1;
        group_sync<1>(nfft);  // the line is refilled below
      }
      if (i < ncol) {
        const int w = blockIdx.x + i * gridDim.x;
        const int mem = w % a.g.batch, k = w / a.g.batch;
        const size_t row = ((size_t)mem * a.g.kk + k) * a.g.ld;
        const V* src = a.in + row;
        for (int j = tid; j < n; j += nfft) cp_async_c(&x[pidx(a.dr, j)], &src[j]);
        cp_async_wait_all();
        if (a.zero_bits && k == 0 && tid == 0) a.zero_bits[(size_t)mem * a.zero_stride] = 0ULL;
        group_sync<1>(nfft);
        if (!(a.ws_debug & 2)) fft_forward_grp<1>(x, a.dr, a.tw_r, tid, nfft);
        V* sc = scr + (size_t)(i & 1) * a.g.ld;
        for (int j = tid; j < n; j += nfft) sc[j] = x[pidx(a.dr, j)];
      }
    } else if (i >= 1 && i - 1 < ncol && !(a.ws_debug & 1)) {
      const int w = blockIdx.x + (i - 1) * gridDim.x;
      const int mem = w % a.g.batch, k = w / a.g.batch;
      const size_t row = ((size_t)mem * a.g.kk + k) * a.g.ld;
      const size_t trow = (size_t)k * a.g.ld;
      V* sc = scr + (size_t)((i - 1) & 1) * a.g.ld;
      rho_combine<T, MODE, true>(sc, a.dr, n, a.E + trow, a.P1 + trow, a.P12 + trow, a.P2 + trow,
                                 a.vh + row, a.u + row, a.ds, 0, tid2, nth2);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ rho pass, persistent
// The march's rho pass as a persistent kernel: one CTA per SM walks columns
// w = blockIdx.x, +gridDim.x, ...  A column's transform needs the whole column
// in shared memory (176 KB at 10000 fp64 points), so an SM cannot hold a
// second column to overlap with; L2 is used as the staging buffer instead.
// While column w is transformed, its combine operands are already streaming
// DRAM -> L2 (bulk prefetch issued with its load), and while w is inverse
// transformed the next column's input is prefetched.  Consumed operands are
// read and results written with evict-first hints so the staging does not
// evict itself.

template <typename V> __device__ __forceinline__ V ld_stream(const V* p) { return __ldcs(p); }
template <typename V> __device__ __forceinline__ void st_stream(V* p, V v) { __stcs(p, v); }

template <typename T, int MODE>
__device__ __forceinline__ void prefetch_operands(const RhoArgs<T>& a, size_t row, size_t trow, int n) {
  if (MODE == RHO_STAGE1) {
    prefetch_row(a.vh + row, n);
    prefetch_row(a.E + trow, n);
    prefetch_row(a.P1 + trow, n);
    prefetch_row(a.P12 + trow, n);
  } else if (MODE == RHO_STAGE2) {
    prefetch_row(a.u + row, n);
    prefetch_row(a.P2 + trow, n);
  } else if (MODE == RHO_EULER) {
    prefetch_row(a.vh + row, n);
    prefetch_row(a.E + trow, n);
    prefetch_row(a.P1 + trow, n);
  }
}

template <typename T, int MODE>
__global__ void __launch_bounds__(512, 1) k_rho_stream(const RhoArgs<T> a) {
  using V = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* x = reinterpret_cast<V*>(smem_raw);
  const int n = a.dr.n;
  const int items = a.g.batch * a.g.kk;
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    const int mem = w % a.g.batch, k = w / a.g.batch;  // members of one mode adjacent: table reuse
    const size_t row = ((size_t)mem * a.g.kk + k) * a.g.ld;
    const size_t trow = (size_t)k * a.g.ld;
    const V* src = a.in + row;
    for (int j = threadIdx.x; j < n; j += blockDim.x) cp_async_c(&x[pidx(a.dr, j)], &src[j]);
    if (a.prefetch && threadIdx.x == 0) prefetch_operands<T, MODE>(a, row, trow, n);
    cp_async_wait_all();
    if (a.zero_bits && k == 0 && threadIdx.x == 0) a.zero_bits[(size_t)mem * a.zero_stride] = 0ULL;
    __syncthreads();
    fft_forward(x, a.dr, 1, 0, a.tw_r);
    rho_combine<T, MODE>(x, a.dr, n, a.E + trow, a.P1 + trow, a.P12 + trow, a.P2 + trow,
                         a.vh + row, a.u + row, a.ds, 0);
    const int wn = w + gridDim.x;
    if (a.prefetch && threadIdx.x == 0 && wn < items)
      prefetch_row(a.in + ((size_t)(wn % a.g.batch) * a.g.kk + wn / a.g.batch) * a.g.ld, n);
    __syncthreads();
    fft_inverse(x, a.dr, 1, 0, a.tw_r);
    V* dst = a.out + row;
    for (int j = threadIdx.x; j < n; j += blockDim.x) st_stream(&dst[j], x[pidx(a.dr, j)]);
    if (a.step_ctr && mem == 0 && k == 0 && threadIdx.x == 0) *a.step_ctr += 1;
    __syncthreads();  // smem is reloaded by the next column
  }
}

// ------------------------------------------------------------------ rho pass, cluster split
// A 2-CTA cluster owns one column; CTA c holds n/2 points (half the shared
// memory, so two CTAs fit per SM and one's memory phase overlaps the
// other's transform).  Forward: the radix-2 DIF split stage is applied while
// loading (both CTAs read the column; L2 serves the second read):
//   c = 0: y_i = x_i + x_{i+n/2},   c = 1: y_i = (x_i - x_{i+n/2}) W_n^i
// then an n/2-point DIF; CTA c holds digit-reversed positions c n/2 + p'
// (frequencies of parity c), so the combine touches one contiguous half of
// every digit-reversed row.  Inverse: an n/2-point DIT per CTA gives A (c=0)
// and B (c=1); the final radix-2 DIT stage reads the partner's half through
// distributed shared memory:
//   out_i = A_i + conj(W_n^i) B_i,   out_{i+n/2} = A_i - conj(W_n^i) B_i.

template <typename T, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2) k_rho_split(const RhoArgs<T> a) {
  using V = cplx<T>;
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* x = reinterpret_cast<V*>(smem_raw);
  const int n = a.dr.n, h = n >> 1;
  const int c = (int)cluster.block_rank();
  const int mem = blockIdx.x >> 1, k = blockIdx.y;
  const size_t row = ((size_t)mem * a.g.kk + k) * a.g.ld;
  const size_t trow = (size_t)k * a.g.ld;
  const size_t hrow = row + (size_t)c * h, htrow = trow + (size_t)c * h;
  const FftDesc& d2 = a.dh2;
  if (a.prefetch && threadIdx.x == 0) {
    if (MODE == RHO_STAGE1) {
      prefetch_row(a.vh + hrow, h);
      prefetch_row(a.E + htrow, h);
      prefetch_row(a.P1 + htrow, h);
      prefetch_row(a.P12 + htrow, h);
    } else if (MODE == RHO_STAGE2) {
      prefetch_row(a.u + hrow, h);
      prefetch_row(a.P2 + htrow, h);
    } else if (MODE == RHO_EULER) {
      prefetch_row(a.vh + hrow, h);
      prefetch_row(a.E + htrow, h);
      prefetch_row(a.P1 + htrow, h);
    }
  }
  const V* src = a.in + row;
#pragma unroll 4
  for (int i = threadIdx.x; i < h; i += blockDim.x) {
    const V lo = src[i], hi = src[i + h];
    x[pidx(d2, i)] = c == 0 ? cadd(lo, hi) : cmul(csub(lo, hi), a.tw_split[i]);
  }
  if (a.zero_bits && k == 0 && c == 0 && threadIdx.x == 0) a.zero_bits[(size_t)mem * a.zero_stride] = 0ULL;
  __syncthreads();
  fft_forward(x, d2, 1, 0, a.tw_h2);
  rho_combine<T, MODE>(x, d2, h, a.E + htrow, a.P1 + htrow, a.P12 + htrow, a.P2 + htrow,
                       a.vh + hrow, a.u + hrow, a.ds, 0);
  __syncthreads();
  fft_inverse(x, d2, 1, 0, a.tw_h2);
  cluster.sync();  // both halves transformed and visible cluster-wide
  const V* xo = cluster.map_shared_rank(x, c ^ 1);
  V* dst = a.out + row + (size_t)c * h;
#pragma unroll 4
  for (int i = threadIdx.x; i < h; i += blockDim.x) {
    const int si = pidx(d2, i);
    const V mine = x[si], other = xo[si];
    const V A = c == 0 ? mine : other, B = c == 0 ? other : mine;
    const V wb = cmulc(B, a.tw_split[i]);
    dst[i] = c == 0 ? cadd(A, wb) : csub(A, wb);
  }
  if (a.step_ctr && mem == 0 && k == 0 && c == 0 && threadIdx.x == 0) *a.step_ctr += 1;
  cluster.sync();  // keep this CTA's shared memory alive until the partner has read it
}

// ------------------------------------------------------------------ transpose
// (kk, ld) [k][j]  <->  (nr, kk) [j][k], per member.

template <typename T>
__global__ void k_transpose(const Geom g, const cplx<T>* __restrict__ in, cplx<T>* __restrict__ out,
                            int to_natural) {
  using V = cplx<T>;
  __shared__ V tile[32][33];
  const int mem = blockIdx.z;
  // to_natural: source rows = k (kk of them), source cols = j (nr)
  const int srows = to_natural ? g.kk : g.nr;
  const int scols = to_natural ? g.nr : g.kk;
  const int sld = to_natural ? g.ld : g.kk;
  const int dld = to_natural ? g.kk : g.ld;
  const size_t sbase = (size_t)mem * (to_natural ? (size_t)g.kk * g.ld : (size_t)g.nr * g.kk);
  const size_t dbase = (size_t)mem * (to_natural ? (size_t)g.nr * g.kk : (size_t)g.kk * g.ld);
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int r = r0 + dy, c = c0 + threadIdx.x;
    if (r < srows && c < scols) tile[dy][threadIdx.x] = in[sbase + (size_t)r * sld + c];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int r = c0 + dy, c = r0 + threadIdx.x;  // dest row = source col
    if (r < scols && c < srows) out[dbase + (size_t)r * dld + c] = tile[threadIdx.x][dy];
  }
}

// ------------------------------------------------------------------ combine
// Elementwise spectral combines of the generic step API (exprk.py:166-173,
// 193) with numpy's complex rounding: explicit _rn intrinsics keep nvcc
// from contracting into FMAs, so `E * vhat` matches numpy bitwise.

__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float rn_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float rn_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float rn_sub(float a, float b) { return __fsub_rn(a, b); }

__device__ __forceinline__ double rn_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float rn_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// numpy's complex product: scalar loops round every product; the AVX2/AVX-512
// loops fuse one product into each sum: re = fma(ar, br, -(ai bi)),
// im = fma(ar, bi, ai br).  The host layer detects which one its numpy uses.
template <bool FMA, typename V> __device__ __forceinline__ V np_mul(V a, V b) {
  if (FMA) return mk<V>(rn_fma(a.x, b.x, -rn_mul(a.y, b.y)), rn_fma(a.x, b.y, rn_mul(a.y, b.x)));
  return mk<V>(rn_sub(rn_mul(a.x, b.x), rn_mul(a.y, b.y)), rn_add(rn_mul(a.x, b.y), rn_mul(a.y, b.x)));
}
template <typename V> __device__ __forceinline__ V np_add(V a, V b) {
  return mk<V>(rn_add(a.x, b.x), rn_add(a.y, b.y));
}
// real scalar * complex as numpy does it: (s + 0j) * a
template <typename V> __device__ __forceinline__ V np_scale(decltype(V::x) s, V a) {
  return mk<V>(rn_sub(rn_mul(s, a.x), rn_mul((decltype(V::x))0, a.y)),
               rn_add(rn_mul(s, a.y), rn_mul((decltype(V::x))0, a.x)));
}

template <typename T, bool FMA>
__global__ void k_combine(long n, int mode, T ds, const cplx<T>* E, const cplx<T>* P1,
                          const cplx<T>* P12, const cplx<T>* P2, const cplx<T>* vh,
                          const cplx<T>* b1, const cplx<T>* b2, cplx<T>* out) {
  using V = cplx<T>;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    V r;
    if (mode == 0) {          // ev = E * vhat
      r = np_mul<FMA>(E[i], vh[i]);
    } else if (mode == 1) {   // vh here is ev: ev + (ds * Phi1) * bh1
      r = np_add(vh[i], np_mul<FMA>(np_scale(ds, P1[i]), b1[i]));
    } else if (mode == 2) {   // ev + ds * (Phi1m2 * bh1 + Phi2 * bh2)
      r = np_add(vh[i], np_scale(ds, np_add(np_mul<FMA>(P12[i], b1[i]), np_mul<FMA>(P2[i], b2[i]))));
    } else {                  // Euler: E * vhat + (ds * Phi1) * bh1
      r = np_add(np_mul<FMA>(E[i], vh[i]), np_mul<FMA>(np_scale(ds, P1[i]), b1[i]));
    }
    out[i] = r;
  }
}

template <typename T>
__global__ void k_convert(long n, const double* in, T* out) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = (T)in[i];
}

// ------------------------------------------------------------------ launchers

static inline int grid_cap(long n, int threads) {
  long b = (n + threads - 1) / threads;
  return (int)(b < 148L * 16 ? (b < 1 ? 1 : b) : 148L * 16);
}

// threads of a theta CTA: short rows (R m <= 2048 points, e.g. Set 1's m = 224
// at R = 8) need about one 16-point butterfly per thread, and a 128-thread CTA
// lets four CTAs share an SM (the kernels are bounded by 256 threads)
template <int R> static int theta_block(int m) {
  static int knob = -1;  // NWB_THETA_THREADS=<64..256> measurement override
  if (knob < 0) {
    const char* e = std::getenv("NWB_THETA_THREADS");
    knob = e ? std::atoi(e) : 0;
  }
  if (knob >= 64 && knob <= theta_threads<R>() && knob % 32 == 0) return knob;
  return R > 1 && R * m <= 2048 ? 128 : theta_threads<R>();
}

template <typename T, int R, bool SPLIT = false>
static void c2r_r(const ThetaArgs<T>& a, cudaStream_t s) {
  const size_t sm = (size_t)R * padded_len(a.g.m, a.dh.pad_period) * sizeof(cplx<T>);
  cudaFuncSetAttribute(k_theta_c2r<T, R, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 grid(SPLIT ? a.msub : (a.g.nr + R - 1) / R, a.g.batch);
  k_theta_c2r<T, R, SPLIT><<<grid, theta_block<R>(a.g.m), sm, s>>>(a);
}
template <typename T, int R, bool SPLIT = false>
static void r2c_r(const ThetaArgs<T>& a, cudaStream_t s) {
  const size_t sm = (size_t)R * padded_len(a.g.m, a.dh.pad_period) * sizeof(cplx<T>);
  cudaFuncSetAttribute(k_theta_r2c<T, R, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int nrows = (a.row_end ? a.row_end : a.g.nr) - a.row_begin;
  dim3 grid(SPLIT ? a.msub : (nrows + R - 1) / R, a.g.batch);
  k_theta_r2c<T, R, SPLIT><<<grid, theta_block<R>(a.g.m), sm, s>>>(a);
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename T, int R, bool C2R>
static void theta_stream(const ThetaArgs<T>& a, cudaStream_t s) {
  const size_t sm = 2 * (size_t)R * padded_len(a.g.m, a.dh.pad_period) * sizeof(cplx<T>);
  auto kern = C2R ? k_theta_c2r_stream<T, R> : k_theta_r2c_stream<T, R>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const long groups = (long)((a.g.nr + R - 1) / R) * a.g.batch;
  const int ctas = (int)std::min<long>(groups, sm_count());
  kern<<<ctas, 512, sm, s>>>(a);
}

// rows < 0 selects the persistent double-buffered kernel with R = -rows;
// a.r1 > 1 the fused-rho-stage kernels with R = r1 rows at stride msub
template <typename T> void launch_theta_c2r(const ThetaArgs<T>& a, int rows, cudaStream_t s) {
  if (a.r1 > 1) {
    if (a.r1 == 4) c2r_r<T, 4, true>(a, s);
    else c2r_r<T, 2, true>(a, s);
    return;
  }
  switch (rows) {
    case -1: theta_stream<T, 1, true>(a, s); break;
    case -2: theta_stream<T, 2, true>(a, s); break;
    case -4: theta_stream<T, 4, true>(a, s); break;
    case -8: theta_stream<T, 8, true>(a, s); break;
    case 1: c2r_r<T, 1>(a, s); break;
    case 2: c2r_r<T, 2>(a, s); break;
    case 4: c2r_r<T, 4>(a, s); break;
    default: c2r_r<T, 8>(a, s); break;
  }
}
template <typename T> void launch_theta_r2c(const ThetaArgs<T>& a, int rows, cudaStream_t s) {
  if (a.r1 > 1) {
    if (a.r1 == 4) r2c_r<T, 4, true>(a, s);
    else r2c_r<T, 2, true>(a, s);
    return;
  }
  switch (rows) {
    case -1: theta_stream<T, 1, false>(a, s); break;
    case -2: theta_stream<T, 2, false>(a, s); break;
    case -4: theta_stream<T, 4, false>(a, s); break;
    case -8: theta_stream<T, 8, false>(a, s); break;
    case 1: r2c_r<T, 1>(a, s); break;
    case 2: r2c_r<T, 2>(a, s); break;
    case 4: r2c_r<T, 4>(a, s); break;
    default: r2c_r<T, 8>(a, s); break;
  }
}

template <typename T, int MODE>
static void rho_m(const RhoArgs<T>& a, int threads, cudaStream_t s) {
  if constexpr (MODE <= RHO_INIT && sizeof(T) == 8) {
    if (a.half && a.dh2.n <= HALF_NT * 20) {
      const size_t sm = (size_t)padded_len(a.dh2.n, a.dh2.pad_period) * sizeof(cplx<T>);
      cudaFuncSetAttribute(k_rho_half<MODE, 20>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      dim3 grid(a.g.batch, a.g.kk);
      k_rho_half<MODE, 20><<<grid, HALF_NT, sm, s>>>(a);
      return;
    }
  }
  if constexpr (MODE != RHO_REV2NAT && MODE != RHO_FWD_NAT) {
    if (a.r1 > 1) {
      const size_t sm = (size_t)padded_len(a.dsub.n, a.dsub.pad_period) * sizeof(cplx<T>);
      cudaFuncSetAttribute(k_rho_sub<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      dim3 grid(a.g.batch, a.g.kk * a.r1);
      k_rho_sub<T, MODE><<<grid, threads > 256 ? 256 : threads, sm, s>>>(a);
      return;
    }
  }
  if constexpr (MODE == RHO_FWD_DR) {
    return;  // sub-column mode only
  } else {
  if constexpr (MODE <= RHO_INIT) {
    if (a.split) {
      const size_t sm = (size_t)padded_len(a.dh2.n, a.dh2.pad_period) * sizeof(cplx<T>);
      cudaFuncSetAttribute(k_rho_split<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      dim3 grid(2 * a.g.batch, a.g.kk);
      k_rho_split<T, MODE><<<grid, threads, sm, s>>>(a);
      return;
    }
    if constexpr (MODE != RHO_INIT) {
      if (a.ws_threads > 0 && a.scratch) {
        const size_t sm = (size_t)padded_len(a.dr.n, a.dr.pad_period) * sizeof(cplx<T>);
        cudaFuncSetAttribute(k_rho_ws<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        const long items = (long)a.g.batch * a.g.kk;
        const long ctas = std::min<long>(items, (long)a.ws_ctas);
        k_rho_ws<T, MODE><<<(int)ctas, a.ws_threads + a.ws_threads2, sm, s>>>(a);
        return;
      }
    }
    if (a.persistent) {
      const size_t sm = (size_t)padded_len(a.dr.n, a.dr.pad_period) * sizeof(cplx<T>);
      cudaFuncSetAttribute(k_rho_stream<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      int dev = 0, sms = 148, occ = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rho_stream<T, MODE>, threads, sm);
      const long items = (long)a.g.batch * a.g.kk;
      const long ctas = std::min<long>(items, (long)sms * (occ > 0 ? occ : 1));
      k_rho_stream<T, MODE><<<(int)ctas, threads, sm, s>>>(a);
      return;
    }
  }
  const size_t sm = (size_t)padded_len(a.dr.n, a.dr.pad_period) * sizeof(cplx<T>);
  dim3 grid(a.g.batch, a.k_cnt > 0 ? a.k_cnt : a.g.kk - a.k_off);
  if constexpr (sizeof(T) == 4) {
    if (threads >= 384) {
      cudaFuncSetAttribute(k_rho_r80<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_rho_r80<T, MODE><<<grid, 384, sm, s>>>(a);
      return;
    }
  }
  cudaFuncSetAttribute(k_rho<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_rho<T, MODE><<<grid, threads, sm, s>>>(a);
  }
}

template <typename T> void launch_rho(const RhoArgs<T>& a, int mode, int threads, cudaStream_t s) {
  switch (mode) {
    case RHO_STAGE1: rho_m<T, RHO_STAGE1>(a, threads, s); break;
    case RHO_STAGE2: rho_m<T, RHO_STAGE2>(a, threads, s); break;
    case RHO_EULER: rho_m<T, RHO_EULER>(a, threads, s); break;
    case RHO_INIT: rho_m<T, RHO_INIT>(a, threads, s); break;
    case RHO_FWD_NAT: rho_m<T, RHO_FWD_NAT>(a, threads, s); break;
    case RHO_INV_NAT: rho_m<T, RHO_INV_NAT>(a, threads, s); break;
    case RHO_FWD_DR: rho_m<T, RHO_FWD_DR>(a, threads, s); break;
    default: rho_m<T, RHO_REV2NAT>(a, threads, s); break;
  }
}

template <typename T>
void launch_transpose(const Geom& g, const cplx<T>* in, cplx<T>* out, int to_natural, cudaStream_t s) {
  const int srows = to_natural ? g.kk : g.nr, scols = to_natural ? g.nr : g.kk;
  dim3 grid((scols + 31) / 32, (srows + 31) / 32, g.batch);
  k_transpose<T><<<grid, dim3(32, 8), 0, s>>>(g, in, out, to_natural);
}

template <typename T>
void launch_combine(long n, int mode, double ds, const cplx<T>* E, const cplx<T>* P1,
                    const cplx<T>* P12, const cplx<T>* P2, const cplx<T>* vh,
                    const cplx<T>* b1, const cplx<T>* b2, cplx<T>* out, cudaStream_t s) {
  // mode bit 3 selects numpy's SIMD (fused) complex-product rounding
  if (mode & 8)
    k_combine<T, true><<<grid_cap(n, 256), 256, 0, s>>>(n, mode & 7, (T)ds, E, P1, P12, P2, vh, b1, b2, out);
  else
    k_combine<T, false><<<grid_cap(n, 256), 256, 0, s>>>(n, mode, (T)ds, E, P1, P12, P2, vh, b1, b2, out);
}

template <typename T> void launch_convert(long n, const double* in, T* out, cudaStream_t s) {
  k_convert<T><<<grid_cap(n, 256), 256, 0, s>>>(n, in, out);
}

// The library compiles this file once per (part, type) so the slow
// instantiations build in parallel: -DNWB_SPEC_PART=1 theta passes and the
// small helpers, 2 rho passes; -DNWB_SPEC_T=double|float.  Without the
// defines everything is instantiated.
#define NWB_INST_THETA(T)                                                                      \
  template void launch_theta_c2r<T>(const ThetaArgs<T>&, int, cudaStream_t);                   \
  template void launch_theta_r2c<T>(const ThetaArgs<T>&, int, cudaStream_t);                   \
  template void launch_transpose<T>(const Geom&, const cplx<T>*, cplx<T>*, int, cudaStream_t); \
  template void launch_combine<T>(long, int, double, const cplx<T>*, const cplx<T>*,           \
                                  const cplx<T>*, const cplx<T>*, const cplx<T>*,              \
                                  const cplx<T>*, const cplx<T>*, cplx<T>*, cudaStream_t);     \
  template void launch_convert<T>(long, const double*, T*, cudaStream_t);
#define NWB_INST_RHO(T) template void launch_rho<T>(const RhoArgs<T>&, int, int, cudaStream_t);
#if !defined(NWB_SPEC_PART) || NWB_SPEC_PART == 1
#ifdef NWB_SPEC_T
NWB_INST_THETA(NWB_SPEC_T)
#else
NWB_INST_THETA(double)
NWB_INST_THETA(float)
#endif
#endif
#if !defined(NWB_SPEC_PART) || NWB_SPEC_PART == 2
#ifdef NWB_SPEC_T
NWB_INST_RHO(NWB_SPEC_T)
#else
NWB_INST_RHO(double)
NWB_INST_RHO(float)
#endif
#endif

}  // namespace nwb
