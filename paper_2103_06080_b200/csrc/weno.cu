// WENO5-JS right-hand side b(sigma, V) with global Lax-Friedrichs splitting
// (reference pkg/src/nwave/weno.py:25-124), both directions in one kernel:
//
//   f_theta = -2 pi U_par V - (B/2) V^2,  f+- = (f_theta +- alpha_theta V) / 2
//   f_rho   =  U_perp V,                 h+- = (f_rho   +- alpha_rho   V) / 2
//   F[k+1/2] = W(f+_{k-2..k+2}) + W(f-_{k+3..k-1})          (periodic)
//   b = (dU_perp/drho V - (F_t[k+1/2]-F_t[k-1/2])/dtheta) - (F_r[j+1/2]-F_r[j-1/2])/drho
//
// The kernel is FP64-pipe bound (~18 flop/B), so the design
// minimises instructions per cell:
//  * one warp owns a 32-column x 32-row tile; every face is computed once
//    (33 faces per 32 cells in each direction, the 33rd theta face of each
//    row is computed by lane r for row r, i.e. amortised over the tile);
//  * theta faces: the row's split fluxes go through a per-warp smem line;
//  * rho faces: each lane walks down its column with a 6-deep register
//    window of split fluxes -- one global load per cell, no transpose;
//  * W() uses one reciprocal per face pair (common-denominator weights,
//    w0 ~ 0.1 A1 A2, w1 ~ 0.6 A0 A2, w2 ~ 0.3 A0 A1 with A_i = (eps+beta_i)^2),
//    SURVEY A.2 measured this reformulation at 1.2e-15 of the reference.
#include "internal.h"

namespace nwb {

__device__ __forceinline__ double bits_to_real(u64 b) { return __longlong_as_double((long long)b); }

// a / b to ~1 ulp: hardware reciprocal seed + two Newton steps + one
// residual correction (no IEEE slow path; b is a positive normal here).
__device__ __forceinline__ double fast_rcp(double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  e = fma(-b, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ float fast_rcp(float b) { return __frcp_rn(b); }

// numerator / denominator of W(a0..a4) (reference _upwind_face) with
// W = num / den
template <typename T>
__device__ __forceinline__ void face_nd(T a0, T a1, T a2, T a3, T a4, T& num, T& den) {
  const T c1312 = (T)(13.0 / 12.0), q = (T)0.25, eps = (T)1e-6;
  const T d0 = (a0 - (T)2 * a1) + a2, e0 = (a0 - (T)4 * a1) + (T)3 * a2;
  const T d1 = (a1 - (T)2 * a2) + a3, e1 = a1 - a3;
  const T d2 = (a2 - (T)2 * a3) + a4, e2 = ((T)3 * a2 - (T)4 * a3) + a4;
  const T t0 = eps + (c1312 * (d0 * d0) + q * (e0 * e0));
  const T t1 = eps + (c1312 * (d1 * d1) + q * (e1 * e1));
  const T t2 = eps + (c1312 * (d2 * d2) + q * (e2 * e2));
  const T A0 = t0 * t0, A1 = t1 * t1, A2 = t2 * t2;
  const T w0 = (T)0.1 * (A1 * A2), w1 = (T)0.6 * (A0 * A2), w2 = (T)0.3 * (A0 * A1);
  const T q0 = ((T)2 * a0 - (T)7 * a1) + (T)11 * a2;
  const T q1 = (-a1 + (T)5 * a2) + (T)2 * a3;
  const T q2 = ((T)2 * a2 + (T)5 * a3) - a4;
  num = (w0 * q0 + w1 * q1) + w2 * q2;
  den = (T)6 * ((w0 + w1) + w2);
}

// F = W(p0..p4) + W(m0..m4) (m already in the reversed order of the source)
__device__ __forceinline__ double face_pair(double p0, double p1, double p2, double p3, double p4,
                                            double m0, double m1, double m2, double m3, double m4) {
  double np, dp, nm, dm;
  face_nd(p0, p1, p2, p3, p4, np, dp);
  face_nd(m0, m1, m2, m3, m4, nm, dm);
  // one reciprocal for both (fp64 range: den in [1e-24, 1e20])
  return (np * dm + nm * dp) * fast_rcp(dp * dm);
}
__device__ __forceinline__ float face_pair(float p0, float p1, float p2, float p3, float p4,
                                           float m0, float m1, float m2, float m3, float m4) {
  float np, dp, nm, dm;
  face_nd(p0, p1, p2, p3, p4, np, dp);
  face_nd(m0, m1, m2, m3, m4, nm, dm);
  return __fdividef(np, dp) + __fdividef(nm, dm);
}

__device__ __forceinline__ int wrap_idx(int x, int n) {
  if (x < 0) x += n;
  if (x >= n) x -= n;
  if ((unsigned)x >= (unsigned)n) x = ((x % n) + n) % n;  // tiny extents only
  return x;
}

constexpr int WT = 32;      // tile edge (cells) per warp
constexpr int WWARPS = 4;   // warps per CTA, stacked along rho

template <typename T>
__global__ void __launch_bounds__(WWARPS * 32) k_weno(const WenoArgs<T> a) {
  __shared__ T lp[WWARPS][WT + 8], lm[WWARPS][WT + 8];   // theta split fluxes of one row
  __shared__ T ft[WWARPS][WT][WT + 1];                   // theta faces of the tile
  const int nr = a.g.nr, nt = a.g.nt;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mem = blockIdx.z;
  const int x0 = blockIdx.x * WT;
  const int j0 = (blockIdx.y * WWARPS + w) * WT;
  if (j0 >= nr) return;  // warp-uniform
  const int row = (a.step_ctr ? *a.step_ctr : 0) + a.row_off;
  // coefficient rows are global (rho slab: local row j is global cj0 + j)
  const int cld = a.coef_ld ? a.coef_ld : nr, cj0 = a.coef_j0, ng = a.nr_glob ? a.nr_glob : nr;
  const bool halo = a.halo != 0;  // slab mode: v holds 3 halo rows above and below
  const T* upar = a.upar + (size_t)row * cld + cj0;
  const T* uperp_g = a.uperp + (size_t)row * cld;
  const T* du = a.du + (size_t)row * cld + cj0;
  const T ath = (T)bits_to_real(a.alpha_bits[(size_t)mem * a.alpha_stride]);
  const T arh = (T)a.alpha_rho[row];
  const T two_pi = (T)6.283185307179586476925;
  const T hb = (T)0.5 * a.bcoef;
  const T half = (T)0.5;
  const T* v = a.v + (size_t)mem * (halo ? nr + 6 : nr) * nt;
  auto vrow = [&](int jj) { return halo ? jj + 3 : wrap_idx(jj, nr); };
  T* lpw = lp[w];
  T* lmw = lm[w];
  T(*ftw)[WT + 1] = ft[w];
  const int kl = wrap_idx(x0 + lane - 3, nt);     // column loaded by this lane (line slot lane)
  const int kh = wrap_idx(x0 + lane + 29, nt);    // extra slot 32 + lane for lanes < 6
  const int rows = min(WT, nr - j0);

  // ---- theta faces, row by row: face f of a row lies between tile columns f-1 and f
  // software-pipelined: row r+1 is loaded while row r's faces are computed
  T v_lo = v[(size_t)vrow(j0) * nt + kl];
  T v_hi = lane < 6 ? v[(size_t)vrow(j0) * nt + kh] : (T)0;
  T c_cur = two_pi * upar[j0];
  for (int r = 0; r < rows; ++r) {
    T g = -c_cur * v_lo - hb * v_lo * v_lo, av = ath * v_lo;
    lpw[lane] = half * (g + av);
    lmw[lane] = half * (g - av);
    if (lane < 6) {
      g = -c_cur * v_hi - hb * v_hi * v_hi;
      av = ath * v_hi;
      lpw[32 + lane] = half * (g + av);
      lmw[32 + lane] = half * (g - av);
    }
    if (r + 1 < rows) {
      const T* vn = v + (size_t)vrow(j0 + r + 1) * nt;
      v_lo = vn[kl];
      if (lane < 6) v_hi = vn[kh];
      c_cur = two_pi * upar[j0 + r + 1];
    }
    __syncwarp();
    ftw[r][lane] = face_pair(lpw[lane], lpw[lane + 1], lpw[lane + 2], lpw[lane + 3], lpw[lane + 4],
                             lmw[lane + 5], lmw[lane + 4], lmw[lane + 3], lmw[lane + 2], lmw[lane + 1]);
    __syncwarp();
  }
  // 33rd theta face of row `lane` (between tile columns 31 and 32)
  if (lane < rows) {
    const int j = j0 + lane;
    const T c = two_pi * upar[j];
    const T* vr = v + (size_t)vrow(j) * nt;
    T p[6], m[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      const T vv = vr[wrap_idx(x0 + 29 + d, nt)];
      const T g = -c * vv - hb * vv * vv, av = ath * vv;
      p[d] = half * (g + av);
      m[d] = half * (g - av);
    }
    ftw[lane][WT] = face_pair(p[0], p[1], p[2], p[3], p[4], m[5], m[4], m[3], m[2], m[1]);
  }
  __syncwarp();

  // ---- rho sweep down column k with a register window of rows j-3 .. j+2
  const int k = x0 + lane;
  const int kv = wrap_idx(k, nt);
  T hp[6], hm[6], vw[6];
#pragma unroll
  for (int d = 0; d < 5; ++d) {
    const T vv = v[(size_t)vrow(j0 - 3 + d) * nt + kv];
    const T g = uperp_g[wrap_idx(cj0 + j0 - 3 + d, ng)] * vv, av = arh * vv;
    hp[d] = half * (g + av);
    hm[d] = half * (g - av);
    vw[d] = vv;
  }
  T fprev = (T)0;
  T* out = a.out + (size_t)mem * nr * nt;
  const bool col_ok = k < nt;
  // software-pipelined: the value for window slot 5 of iteration r+1 is
  // loaded while iteration r computes its face
  T vnext = v[(size_t)vrow(j0 + 2) * nt + kv];
  T unext = uperp_g[wrap_idx(cj0 + j0 + 2, ng)];
  for (int r = 0; r <= rows; ++r) {
    // row j0 + r + 2 into window slot 5
    const T vv = vnext, uu = unext;
    if (r < rows) {
      vnext = v[(size_t)vrow(j0 + r + 3) * nt + kv];
      unext = uperp_g[wrap_idx(cj0 + j0 + r + 3, ng)];
    }
    const T g = uu * vv, av = arh * vv;
    hp[5] = half * (g + av);
    hm[5] = half * (g - av);
    vw[5] = vv;
    // face between rows j0+r-1 and j0+r
    const T f = face_pair(hp[0], hp[1], hp[2], hp[3], hp[4], hm[5], hm[4], hm[3], hm[2], hm[1]);
    if (r > 0 && col_ok) {
      const int j = j0 + r - 1;
      const T dth = (ftw[r - 1][lane + 1] - ftw[r - 1][lane]) * a.inv_dtheta;
      const T drh = (f - fprev) * a.inv_drho;
      out[(size_t)j * nt + k] = (du[j] * vw[2] - dth) - drh;
    }
    fprev = f;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
      hp[d] = hp[d + 1];
      hm[d] = hm[d + 1];
      vw[d] = vw[d + 1];
    }
  }
}

template <typename T>
__global__ void k_alpha_theta(const Geom g, const T* v, const T* upar, T bcoef, u64* bits, int stride) {
  const int mem = blockIdx.y;
  const size_t n = (size_t)g.nr * g.nt;
  const T* vm = v + (size_t)mem * n;
  const T two_pi = (T)6.283185307179586476925;
  u64 m = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(i / g.nt);
    const T c = upar ? two_pi * upar[j] : (T)0;
    const u64 s = abs_bits(c + bcoef * vm[i]);
    m = s > m ? s : m;
  }
  __shared__ u64 red[32];
  m = warp_max_u64(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0ULL;
    m = warp_max_u64(m);
    if (threadIdx.x == 0) atomicMax(bits + (size_t)mem * stride, m);
  }
}

template <typename T>
__global__ void k_alpha_rho(const T* uperp, int nr, double* out) {
  const int row = blockIdx.x;
  const T* u = uperp + (size_t)row * nr;
  u64 m = 0;
  for (int j = threadIdx.x; j < nr; j += blockDim.x) {
    const u64 s = abs_bits(u[j]);
    m = s > m ? s : m;
  }
  __shared__ u64 red[32];
  m = warp_max_u64(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0ULL;
    m = warp_max_u64(m);
    if (threadIdx.x == 0) out[row] = __longlong_as_double((long long)m);
  }
}

template <typename T> void launch_weno(const WenoArgs<T>& a, cudaStream_t s) {
  dim3 grid((a.g.nt + WT - 1) / WT, (a.g.nr + WT * WWARPS - 1) / (WT * WWARPS), a.g.batch);
  k_weno<T><<<grid, WWARPS * 32, 0, s>>>(a);
}

template <typename T>
void launch_alpha_theta(const Geom& g, const T* v, const T* upar, T bcoef, u64* bits, int stride,
                        cudaStream_t s) {
  const size_t n = (size_t)g.nr * g.nt;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_alpha_theta<T><<<dim3(blocks, g.batch), 256, 0, s>>>(g, v, upar, bcoef, bits, stride);
}

template <typename T> void launch_alpha_rho(const T* uperp, int nr, int rows, double* out, cudaStream_t s) {
  k_alpha_rho<T><<<rows, 256, 0, s>>>(uperp, nr, out);
}

template void launch_weno<double>(const WenoArgs<double>&, cudaStream_t);
template void launch_weno<float>(const WenoArgs<float>&, cudaStream_t);
template void launch_alpha_theta<double>(const Geom&, const double*, const double*, double, u64*, int, cudaStream_t);
template void launch_alpha_theta<float>(const Geom&, const float*, const float*, float, u64*, int, cudaStream_t);
template void launch_alpha_rho<double>(const double*, int, int, double*, cudaStream_t);
template void launch_alpha_rho<float>(const float*, int, int, double*, cudaStream_t);

}  // namespace nwb
