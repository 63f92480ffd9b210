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
//    SURVEY A.2 measured this reformulation at 1.2e-15 of the reference;
//  * smoothness indicators scaled by 4 with eps folded into the centred
//    second-difference term, which the rho sweep computes once per row.
#include <cstdlib>

#include "internal.h"

namespace nwb {

__global__ void k_stamp(unsigned long long* buf, const int* step, int slot) {
  StepStamp st{buf, step, slot};
  step_stamp(st);
}
void launch_stamp(unsigned long long* buf, const int* step, int slot, cudaStream_t s) {
  k_stamp<<<1, 32, 0, s>>>(buf, step, slot);
}

__device__ __forceinline__ double bits_to_real(u64 b) { return __longlong_as_double((long long)b); }

// 1 / b to ~1 ulp: hardware reciprocal seed refined by one cubic step
// (NWB_WENO_RCP3=0: two Newton steps, one more FP64 instruction); no IEEE
// slow path -- b is a positive normal here.
#ifndef NWB_WENO_RCP3
#define NWB_WENO_RCP3 1
#endif
__device__ __forceinline__ double fast_rcp(double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = fma(-b, r, 1.0);
#if NWB_WENO_RCP3
  // one cubic step r (1 + e + e^2): error ~e^3 from the seed's ~2^-22
  return fma(r, fma(e, e, e), r);
#else
  r = fma(r, e, r);
  e = fma(-b, r, 1.0);
  return fma(r, e, r);
#endif
}
__device__ __forceinline__ float fast_rcp(float b) { return __frcp_rn(b); }

// Smoothness indicators scaled by 4 (the weights only depend on ratios):
//   4 (eps + beta_i) = (13/3) d_i^2 + e_i^2 + 4 eps,   d_i = centred second
// difference, and the second-difference term D(c) = (13/3) d_c^2 + 4 eps
// depends only on the centre c, so a sweep that owns consecutive centres
// computes each once (the rho sweep keeps them in its register window).
template <typename T> __device__ __forceinline__ T dsq(T l, T c, T r) {
  const T d = fma((T)-2, c, l) + r;
  return fma((T)(13.0 / 3.0) * d, d, (T)4e-6);
}

// numerator / denominator of W(a0..a4) (reference _upwind_face, weights
// 0.1 : 0.6 : 0.3 -> 1 : 6 : 3 over common denominator A0 A1 A2) with
// W = num / (6 den); D0..D2 = dsq at the centres a1, a2, a3
//   num = A1 A2 q0 + A0 (6 A2 q1 + 3 A1 q2),  den = A1 A2 + A0 (6 A2 + 3 A1)
template <typename T>
__device__ __forceinline__ void face_nd(T a0, T a1, T a2, T a3, T a4, T D0, T D1, T D2, T& num,
                                        T& den) {
  const T e0 = fma((T)3, a2, fma((T)-4, a1, a0));
  const T e1 = a1 - a3;
  const T e2 = fma((T)3, a2, fma((T)-4, a3, a4));
  const T t0 = fma(e0, e0, D0);
  const T t1 = fma(e1, e1, D1);
  const T t2 = fma(e2, e2, D2);
  const T A0 = t0 * t0, A1 = t1 * t1, A2 = t2 * t2;
  // 2 a0 - 7 a1 + 11 a2 = 2 e0 + (a1 + 5 a2): one instruction less than the direct form
  const T q0 = fma((T)2, e0, fma((T)5, a2, a1));
  // -a1 + 5 a2 + 2 a3 = s - e1 and 2 a2 + 5 a3 - a4 = s - e2 with s = 5 a2 + a3
  const T s5 = fma((T)5, a2, a3);
  const T q1 = s5 - e1;
  const T q2 = s5 - e2;
  const T P = A1 * A2, x = (T)6 * A2, y = (T)3 * A1;
  num = fma(A0, fma(x, q1, y * q2), P * q0);
  den = fma(A0, x + y, P);
}

// F = W(p0..p4) + W(m0..m4) (m already in the reversed order of the source),
// second-difference terms supplied by the caller
__device__ __forceinline__ double face_pair_d(double p0, double p1, double p2, double p3, double p4,
                                              double Dp0, double Dp1, double Dp2, double m0,
                                              double m1, double m2, double m3, double m4,
                                              double Dm0, double Dm1, double Dm2) {
  double np, dp, nm, dm;
  face_nd(p0, p1, p2, p3, p4, Dp0, Dp1, Dp2, np, dp);
  face_nd(m0, m1, m2, m3, m4, Dm0, Dm1, Dm2, nm, dm);
  // one reciprocal for both (dp dm >= (4e-6)^8 ~ 7e-44: normal in fp64); returns
  // 6 F -- the 1/6 is folded into k_weno's 1/dtheta, 1/drho
  return (np * dm + nm * dp) * fast_rcp(dp * dm);
}
__device__ __forceinline__ float face_pair_d(float p0, float p1, float p2, float p3, float p4,
                                             float Dp0, float Dp1, float Dp2, float m0, float m1,
                                             float m2, float m3, float m4, float Dm0, float Dm1,
                                             float Dm2) {
  float np, dp, nm, dm;
  face_nd(p0, p1, p2, p3, p4, Dp0, Dp1, Dp2, np, dp);
  face_nd(m0, m1, m2, m3, m4, Dm0, Dm1, Dm2, nm, dm);
  return __fdividef(np, 6.0f * dp) + __fdividef(nm, 6.0f * dm);
}
template <typename T>
__device__ __forceinline__ T face_pair(T p0, T p1, T p2, T p3, T p4, T m0, T m1, T m2, T m3, T m4) {
  return face_pair_d(p0, p1, p2, p3, p4, dsq(p0, p1, p2), dsq(p1, p2, p3), dsq(p2, p3, p4), m0, m1,
                     m2, m3, m4, dsq(m0, m1, m2), dsq(m1, m2, m3), dsq(m2, m3, m4));
}

// products that must round on their own (never contracted into a following
// add), like the split fluxes the row-by-row version stages in shared memory
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }

__device__ __forceinline__ int wrap_idx(int x, int n) {
  if (x < 0) x += n;
  if (x >= n) x -= n;
  if ((unsigned)x >= (unsigned)n) x = ((x % n) + n) % n;  // tiny extents only
  return x;
}

constexpr int WT = 32;      // tile edge (cells) per warp
constexpr int WWARPS = 4;   // warps per CTA, stacked along rho

// unroll of the rho sweeps (measurement knobs): the interior loop of k_weno
// (6 = the register window's period, no moves) and the rare seam loop (tiles
// whose prefetch wraps; kept small so the two copies of the sweep do not crowd
// the instruction cache)
#ifndef NWB_WENO_SWEEP_UNROLL
#define NWB_WENO_SWEEP_UNROLL 6
#endif
#ifndef NWB_WENO_SEAM_UNROLL
#define NWB_WENO_SEAM_UNROLL 1
#endif
// narrow fields (N_theta < 1024, e.g. the C4 members) run the interior sweep
// at a smaller unroll: their tiles take the seam / TMA-patch paths more often
// and the smaller kernel keeps those in the instruction cache (C4 fp64 WENO
// 1.587 -> 1.506 ms at unroll 3, fp32 0.923 -> 0.873 at 2; C2 prefers 6 / 4)
constexpr int kSweepUnrollNarrow = 3, kX2UnrollNarrow = 2, kNarrowNt = 1024;
#define NWB_PRAGMA_(x) _Pragma(#x)
#define NWB_PRAGMA(x) NWB_PRAGMA_(x)
#define NWB_SEAM_UNROLL_PRAGMA NWB_PRAGMA(unroll NWB_WENO_SEAM_UNROLL)

// four CTAs (16 warps) per SM: caps the fp64 walk kernels at 128 registers (the
// TMA-staged one would take 146 and fit three; 124 with no spills measures
// 0.385 -> 0.378 ms at C2); the other instantiations already fit
#ifndef NWB_WENO_MINB
#define NWB_WENO_MINB 4
#endif
#ifndef NWB_WENO_CPASYNC
#define NWB_WENO_CPASYNC 1
#endif
// WTR: rows per warp tile (32; 16 / 8 for small grids, where more, shorter warps
// finish sooner -- the extra rho halo and faces are cheap there)
//
// WALK (32-row tiles): the theta faces are computed like the rho ones -- the
// warp stages its 32 x 38 tile of V in shared memory, then lane r walks row r
// with a 6-deep register window, so every split flux and second-difference
// term is evaluated once per slot instead of once per stencil use (about 17
// fewer FP64 instructions per cell, 2 shared loads per cell instead of 10).
// The faces overwrite the row in place (face f is stored after slot f + 5 was
// read).  Bitwise equal to the row-by-row version (same operands, same order).
constexpr int WTS = WT + 9;
#ifndef NWB_WENO_WALK_UNROLL
#define NWB_WENO_WALK_UNROLL 6
#endif
constexpr int kWalkUnroll = NWB_WENO_WALK_UNROLL;  // walk tile row stride: odd (conflict-free half-warps), >= 38 slots
//
// TMA (fp64 walk, plain mode): the warp's V tile arrives as ONE tensor copy
// issued by lane 0 -- box columns x0-4 .. x0+37 (a tiled copy's inner start
// must be 16-byte aligned, so the box starts one column before the halo) of
// rows j0 .. j0+31, zero-filled outside the grid; tiles touching the periodic
// seam patch the wrapped columns with plain loads -- instead of ~38 cp.async
// per lane.  The dense box sets the row stride to 42 (2-way bank conflicts in
// the walk instead of none) and slot s of the cp.async layout sits at s + 1.
template <typename T, int WTR, bool WALK, bool TMA, int SU = NWB_WENO_SWEEP_UNROLL>
__global__ void __launch_bounds__(WWARPS * 32, NWB_WENO_MINB) k_weno(const __grid_constant__ WenoArgs<T> a) {
  step_stamp(a.ts);
  static_assert(!TMA || (WALK && WTR == WT), "TMA staging is a walk-tile path");
  constexpr int FTS = TMA ? WENO_TMA_BOX : WALK ? WTS : WT + 1;  // theta-face row stride
  __shared__ T lp[WALK ? 1 : WWARPS][WT + 8], lm[WALK ? 1 : WWARPS][WT + 8];  // split fluxes of one row
  __shared__ __align__(128) T ft[WWARPS][WTR][FTS];      // theta faces of the tile (WALK: V first)
  __shared__ __align__(8) unsigned long long tbar[TMA ? WWARPS : 1];
  const int nr = a.g.nr, nt = a.g.nt;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mem = blockIdx.z;
  const int x0 = blockIdx.x * WT;
  const int jend = a.row_end ? a.row_end : nr;
  const int j0 = a.row_begin + (blockIdx.y * WWARPS + w) * WTR;
  if (j0 >= jend) return;  // warp-uniform
  const int row = (a.step_ctr ? *a.step_ctr : 0) + a.row_off;
  // coefficient rows are global (rho slab: local row j is global cj0 + j)
  const int cld = a.coef_ld ? a.coef_ld : nr, cj0 = a.coef_j0, ng = a.nr_glob ? a.nr_glob : nr;
  const bool halo = a.halo != 0;  // slab mode: v holds 3 halo rows above and below
  const T* upar = a.upar + (size_t)row * cld + cj0;
  const T* uperp_g = a.uperp + (size_t)row * cld;
  const T* du = a.du + (size_t)row * cld + cj0;
  const T ath = (T)bits_to_real(a.alpha_bits[(size_t)mem * a.alpha_stride]);
  const T arh = (T)a.alpha_rho[row];
  const T pi = (T)3.14159265358979323846;
  // split fluxes 0.5 (g +- alpha v) with g = -c v - (B/2) v^2 (theta) or
  // u_perp v (rho), factored as v * (affine in v): 2 flops per split flux
  const T qb = (T)-0.25 * a.bcoef;
  const T half = (T)0.5;
  const T hath = half * ath, harh = half * arh;
  const T* v = a.v + (size_t)mem * (halo ? nr + 6 : nr) * nt;
  auto vrow = [&](int jj) { return halo ? jj + 3 : wrap_idx(jj, nr); };
  T* lpw = lp[WALK ? 0 : w];
  T* lmw = lm[WALK ? 0 : w];
  T(*ftw)[FTS] = ft[w];
  const int kl = wrap_idx(x0 + lane - 3, nt);     // column loaded by this lane (line slot lane)
  const int kh = wrap_idx(x0 + lane + 29, nt);    // extra slot 32 + lane for lanes < 6
  const int rows = min(WTR, jend - j0);

  if constexpr (WALK) {
    // ---- theta faces, lane r walks row r: stage the tile's V (slot s = column x0 + s - 3)
    if constexpr (TMA) {
      unsigned long long* bar = &tbar[w];
      if (lane == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar, (unsigned)(WENO_TMA_BOX * WT * sizeof(T)));
        tma_load_3d(&ftw[0][0], &a.vmap, x0 - 4, halo ? j0 + 3 : j0, mem, bar);
      }
      mbar_wait(bar, 0);
      if (x0 < 3 || x0 + 35 > nt) {  // warp-uniform: the tile touches the seam
        // box slots 1 .. 38 hold columns x0-3 .. x0+34; lane patches slot lane + 1
        // and (lanes < 6) slot lane + 33 when its column lies outside [0, nt)
        const bool lo_w = (unsigned)(x0 + lane - 3) >= (unsigned)nt;
        const bool hi_w = lane < 6 && x0 + lane + 29 >= nt;
        for (int r = 0; r < rows; ++r) {
          const T* vr = v + (size_t)vrow(j0 + r) * nt;
          if (lo_w) ftw[r][lane + 1] = vr[kl];
          if (hi_w) ftw[r][33 + lane] = vr[kh];
        }
      }
    } else {
#if NWB_WENO_CPASYNC
    // as asynchronous copies: all of the lane's 32-38 loads in flight at once,
    // no register round trip (the staging stalled on each batch of loads)
    const T* vr = v + (size_t)(halo ? j0 + 3 : j0) * nt;  // rows j0 .. j0+rows-1 never wrap
    for (int r = 0; r < rows; ++r, vr += nt) {
      cp_async_real(&ftw[r][lane], vr + kl);
      if (lane < 6) cp_async_real(&ftw[r][32 + lane], vr + kh);
    }
    cp_async_wait_all();
#else
#pragma unroll 8
    for (int r = 0; r < rows; ++r) {
      const T* vr = v + (size_t)vrow(j0 + r) * nt;
      ftw[r][lane] = vr[kl];
      if (lane < 6) ftw[r][32 + lane] = vr[kh];
    }
#endif
    }  // !TMA
    __syncwarp();
    if (lane < rows) {
      const T c = mul_rn(pi, upar[j0 + lane]);
      const T cp = hath - c, cm = -hath - c;
      T* tr = ftw[lane] + (TMA ? 1 : 0);
      // p / m: split fluxes at window slots 0..5; dp[s] = dsq(p[s-1], p[s], p[s+1]),
      // dm[s] = dsq(m[s+1], m[s], m[s-1]) (the argument orders of face_pair)
      T p[6], m[6], dp[6], dm[6];
#pragma unroll
      for (int d = 0; d < 5; ++d) {
        const T vv = tr[d];
        p[d] = mul_rn(vv, fma(qb, vv, cp));
        m[d] = mul_rn(vv, fma(qb, vv, cm));
      }
      dp[1] = dsq(p[0], p[1], p[2]);
      dp[2] = dsq(p[1], p[2], p[3]);
      dm[2] = dsq(m[3], m[2], m[1]);
      dm[3] = dsq(m[4], m[3], m[2]);
#pragma unroll kWalkUnroll
      for (int f = 0; f <= WT; ++f) {
        const T vv = tr[f + 5];
        p[5] = mul_rn(vv, fma(qb, vv, cp));
        m[5] = mul_rn(vv, fma(qb, vv, cm));
        dp[3] = dsq(p[2], p[3], p[4]);
        dm[4] = dsq(m[5], m[4], m[3]);
        tr[f] = face_pair_d(p[0], p[1], p[2], p[3], p[4], dp[1], dp[2], dp[3], m[5], m[4], m[3],
                            m[2], m[1], dm[4], dm[3], dm[2]);
#pragma unroll
        for (int d = 0; d < 5; ++d) {
          p[d] = p[d + 1];
          m[d] = m[d + 1];
          dp[d] = dp[d + 1];
          dm[d] = dm[d + 1];
        }
      }
    }
    __syncwarp();
  } else {
  // ---- theta faces, row by row: face f of a row lies between tile columns f-1 and f
  // software-pipelined: row r+1 is loaded while row r's faces are computed
  T v_lo = v[(size_t)vrow(j0) * nt + kl];
  T v_hi = lane < 6 ? v[(size_t)vrow(j0) * nt + kh] : (T)0;
  T c_cur = mul_rn(pi, upar[j0]);
  for (int r = 0; r < rows; ++r) {
    const T cp = hath - c_cur, cm = -hath - c_cur;  // c_cur = pi u_par
    lpw[lane] = v_lo * fma(qb, v_lo, cp);
    lmw[lane] = v_lo * fma(qb, v_lo, cm);
    if (lane < 6) {
      lpw[32 + lane] = v_hi * fma(qb, v_hi, cp);
      lmw[32 + lane] = v_hi * fma(qb, v_hi, cm);
    }
    if (r + 1 < rows) {
      const T* vn = v + (size_t)(halo ? j0 + r + 4 : j0 + r + 1) * nt;  // rows j0..j0+rows-1 < nr
      v_lo = vn[kl];
      if (lane < 6) v_hi = vn[kh];
      c_cur = mul_rn(pi, upar[j0 + r + 1]);
    }
    __syncwarp();
    ftw[r][lane] = face_pair(lpw[lane], lpw[lane + 1], lpw[lane + 2], lpw[lane + 3], lpw[lane + 4],
                             lmw[lane + 5], lmw[lane + 4], lmw[lane + 3], lmw[lane + 2], lmw[lane + 1]);
    __syncwarp();
  }
  // 33rd theta face of row `lane` (between tile columns 31 and 32)
  if (lane < rows) {
    const int j = j0 + lane;
    const T c = mul_rn(pi, upar[j]);
    const T cp = hath - c, cm = -hath - c;
    const T* vr = v + (size_t)vrow(j) * nt;
    T p[6], m[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      const T vv = vr[wrap_idx(x0 + 29 + d, nt)];
      p[d] = mul_rn(vv, fma(qb, vv, cp));
      m[d] = mul_rn(vv, fma(qb, vv, cm));
    }
    ftw[lane][WT] = face_pair(p[0], p[1], p[2], p[3], p[4], m[5], m[4], m[3], m[2], m[1]);
  }
  __syncwarp();
  }  // !WALK

  // ---- rho sweep down column k with a register window of rows j-3 .. j+2
  const int k = x0 + lane;
  const int kv = wrap_idx(k, nt);
  // dp[s] / dm[s]: second-difference terms of hp / hm centred at window slot
  // s (dp used at slots 1..3, dm at 2..4); each is computed once per row
  T hp[6], hm[6], vw[6], dp[6], dm[6];
#pragma unroll
  for (int d = 0; d < 5; ++d) {
    const T vv = v[(size_t)vrow(j0 - 3 + d) * nt + kv];
    const T uh = half * uperp_g[wrap_idx(cj0 + j0 - 3 + d, ng)];
    hp[d] = vv * (uh + harh);
    hm[d] = vv * (uh - harh);
    vw[d] = vv;
  }
  dp[1] = dsq(hp[0], hp[1], hp[2]);
  dp[2] = dsq(hp[1], hp[2], hp[3]);
  dm[2] = dsq(hm[1], hm[2], hm[3]);
  dm[3] = dsq(hm[2], hm[3], hm[4]);
  T fprev = (T)0;
  const bool col_ok = k < nt;
  // output / du pointers of row j0 (advanced one row per face after the first)
  T* outp = a.out + (size_t)mem * nr * nt + (size_t)j0 * nt + (col_ok ? k : 0);
  const T* dup = du + j0;
  const T* ftp = &ftw[0][lane + (TMA ? 1 : 0)];
  // fp64 faces come as 6 F (face_pair_d)
  const T idth = sizeof(T) == 8 ? a.inv_dtheta * (T)(1.0 / 6.0) : a.inv_dtheta;
  const T idrh = sizeof(T) == 8 ? a.inv_drho * (T)(1.0 / 6.0) : a.inv_drho;
  // software-pipelined: the value for window slot 5 of iteration r+1 is
  // loaded while iteration r computes its face.  Running (wrapped) element
  // offset / coefficient row of the prefetched row: they advance by one row
  // per iteration, so the periodic wrap is a compare instead of a modulus.
  const T* vcol = v + kv;
  const int vrows = halo ? nr + 6 : nr;
  int ov = vrow(j0 + 2) * nt, ju = wrap_idx(cj0 + j0 + 2, ng);
  T vnext = vcol[ov];
  T unext = uperp_g[ju];
  // one row of the sweep: v / u_perp of row j0 + r + 2 into window slot 5, the
  // face between rows j0+r-1 and j0+r, and (emit) the output of row j0+r-1
  // (full: the whole 32-column tile lies inside the field, no per-lane column test)
  auto row_step = [&](const T vv, const T uu, const bool emit, const bool full) {
    hp[5] = vv * fma(half, uu, harh);
    hm[5] = vv * fma(half, uu, -harh);
    vw[5] = vv;
    dp[3] = dsq(hp[2], hp[3], hp[4]);
    dm[4] = dsq(hm[3], hm[4], hm[5]);
    const T f = face_pair_d(hp[0], hp[1], hp[2], hp[3], hp[4], dp[1], dp[2], dp[3], hm[5], hm[4],
                            hm[3], hm[2], hm[1], dm[4], dm[3], dm[2]);
    if (emit) {
      if (full || col_ok) {
        const T dth = (ftp[1] - ftp[0]) * idth;
        const T drh = (f - fprev) * idrh;
        *outp = (*dup * vw[2] - dth) - drh;
      }
      outp += nt;
      ++dup;
      ftp += FTS;
    }
    fprev = f;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
      hp[d] = hp[d + 1];
      hm[d] = hm[d + 1];
      vw[d] = vw[d + 1];
      dp[d] = dp[d + 1];
      dm[d] = dm[d + 1];
    }
  };
  // Interior tiles (warp-uniform): every row the sweep prefetches, up to
  // j0 + rows + 3, lies inside the field and the coefficient row without
  // wrapping, so the prefetch runs unconditionally on plain pointer increments
  // (the last one is unused); tiles at the periodic rho seam keep the wrapped
  // running offsets.  Same operands in the same order either way.
  const int top = j0 + rows + 3;
  if ((halo ? top + 3 : top) < vrows && cj0 + top < ng && x0 + WT <= nt) {
    const T* vp = vcol + ov;
    const T* up = uperp_g + ju;
    {
      const T vv = vnext, uu = unext;
      vp += nt;
      ++up;
      vnext = *vp;
      unext = *up;
      row_step(vv, uu, false, true);
    }
#pragma unroll SU
    for (int r = 1; r <= rows; ++r) {
      const T vv = vnext, uu = unext;
      vp += nt;
      ++up;
      vnext = *vp;
      unext = *up;
      row_step(vv, uu, true, true);
    }
  } else {
    const int vwrap = vrows * nt;
NWB_SEAM_UNROLL_PRAGMA
    for (int r = 0; r <= rows; ++r) {
      const T vv = vnext, uu = unext;
      if (r < rows) {
        ov += nt;
        ov = ov == vwrap ? 0 : ov;
        ju = ju + 1 == ng ? 0 : ju + 1;
        vnext = vcol[ov];
        unext = uperp_g[ju];
      }
      row_step(vv, uu, r > 0, false);
    }
  }
}

// ------------------------------------------------------------------ fp32 on the packed pipe
// Blackwell issues FP32 FMA at full rate only as FFMA2 (two lanes of a float2
// per instruction); WENO in fp32 is issue-bound, so this variant gives each
// lane TWO columns (k and k + 32 of a 64-column warp tile) and evaluates both
// cells' faces with packed float2 arithmetic: the same formulas as k_weno
// (face_nd / dsq are templates), half the FP instructions.

struct f2 {
  float2 v;
  __device__ __forceinline__ f2() {}
  __device__ __forceinline__ explicit f2(float s) : v(make_float2(s, s)) {}
  __device__ __forceinline__ f2(float a, float b) : v(make_float2(a, b)) {}
  __device__ __forceinline__ explicit f2(float2 x) : v(x) {}
};
__device__ __forceinline__ f2 operator+(f2 a, f2 b) { return f2(__fadd2_rn(a.v, b.v)); }
__device__ __forceinline__ f2 operator*(f2 a, f2 b) { return f2(__fmul2_rn(a.v, b.v)); }
__device__ __forceinline__ f2 operator-(f2 a) { return f2(-a.v.x, -a.v.y); }
__device__ __forceinline__ f2 operator-(f2 a, f2 b) {
  return f2(__ffma2_rn(b.v, make_float2(-1.0f, -1.0f), a.v));
}
__device__ __forceinline__ f2 fma(f2 a, f2 b, f2 c) { return f2(__ffma2_rn(a.v, b.v, c.v)); }
using ::fma;  // keep the scalar overloads visible next to the packed one

template <typename P> struct pair_of;
template <> struct pair_of<float> { using type = f2; };

// W(p) + W(m) for both lanes of a pair, from numerators / denominators
__device__ __forceinline__ f2 pair_div(f2 np, f2 dp, f2 nm, f2 dm) {
  const f2 d6p = f2(6.0f) * dp, d6m = f2(6.0f) * dm;
  return f2(__fdividef(np.v.x, d6p.v.x) + __fdividef(nm.v.x, d6m.v.x),
            __fdividef(np.v.y, d6p.v.y) + __fdividef(nm.v.y, d6m.v.y));
}
template <typename P>
__device__ __forceinline__ P face_pair2(P p0, P p1, P p2, P p3, P p4, P m0, P m1, P m2, P m3, P m4) {
  P np, dp, nm, dm;
  face_nd(p0, p1, p2, p3, p4, dsq(p0, p1, p2), dsq(p1, p2, p3), dsq(p2, p3, p4), np, dp);
  face_nd(m0, m1, m2, m3, m4, dsq(m0, m1, m2), dsq(m1, m2, m3), dsq(m2, m3, m4), nm, dm);
  return pair_div(np, dp, nm, dm);
}
template <typename P>
__device__ __forceinline__ P face_pair2_d(P p0, P p1, P p2, P p3, P p4, P Dp0, P Dp1, P Dp2, P m0,
                                          P m1, P m2, P m3, P m4, P Dm0, P Dm1, P Dm2) {
  P np, dp, nm, dm;
  face_nd(p0, p1, p2, p3, p4, Dp0, Dp1, Dp2, np, dp);
  face_nd(m0, m1, m2, m3, m4, Dm0, Dm1, Dm2, nm, dm);
  return pair_div(np, dp, nm, dm);
}

constexpr int WT2 = 64;  // columns per warp tile (two per lane)
#ifndef NWB_WENO_X2_UNROLL
#define NWB_WENO_X2_UNROLL 4
#endif

// WALK (32-row tiles): lane r walks row r of the staged 32 x 70 V tile, the two
// halves packed -- faces 0..32 from slots 0..37 (lane x) and faces 32..64 from
// slots 32..69 (lane y) -- with the register window of k_weno's walk.  Face g
// is stored in place at position g (g < 32, lane x) or g + 5 (lane y, right
// after slot g + 5 is read); lane x's face 32 (its last, whose newest slot 37
// lane y has already overwritten) is a discarded duplicate.
constexpr int WTS2 = WT2 + 7;  // walk tile row stride: odd, >= 70 slots
template <typename T, int WTR, bool WALK, int SU = NWB_WENO_X2_UNROLL>
__global__ void __launch_bounds__(WWARPS * 32) k_weno_x2(const __grid_constant__ WenoArgs<T> a) {
  step_stamp(a.ts);
  using P = typename pair_of<T>::type;
  constexpr int FTS = WALK ? WTS2 : WT2 + 1;
  __shared__ T lp[WALK ? 1 : WWARPS][WT2 + 8], lm[WALK ? 1 : WWARPS][WT2 + 8];  // split fluxes of one row
  __shared__ T ft[WWARPS][WTR][FTS];                       // theta faces of the tile (WALK: V first)
  const int nr = a.g.nr, nt = a.g.nt;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mem = blockIdx.z;
  const int x0 = blockIdx.x * WT2;
  const int jend = a.row_end ? a.row_end : nr;
  const int j0 = a.row_begin + (blockIdx.y * WWARPS + w) * WTR;
  if (j0 >= jend) return;  // warp-uniform
  const int row = (a.step_ctr ? *a.step_ctr : 0) + a.row_off;
  const int cld = a.coef_ld ? a.coef_ld : nr, cj0 = a.coef_j0, ng = a.nr_glob ? a.nr_glob : nr;
  const bool halo = a.halo != 0;
  const T* upar = a.upar + (size_t)row * cld + cj0;
  const T* uperp_g = a.uperp + (size_t)row * cld;
  const T* du = a.du + (size_t)row * cld + cj0;
  const T ath = (T)bits_to_real(a.alpha_bits[(size_t)mem * a.alpha_stride]);
  const T arh = (T)a.alpha_rho[row];
  const T pi = (T)3.14159265358979323846;
  const T qb = (T)-0.25 * a.bcoef;
  const T half = (T)0.5;
  const T hath = half * ath, harh = half * arh;
  const T* v = a.v + (size_t)mem * (halo ? nr + 6 : nr) * nt;
  auto vrow = [&](int jj) { return halo ? jj + 3 : wrap_idx(jj, nr); };
  T* lpw = lp[WALK ? 0 : w];
  T* lmw = lm[WALK ? 0 : w];
  T(*ftw)[FTS] = ft[w];
  // line slot s holds column x0 + s - 3: lane loads slots lane, lane + 32, and
  // lanes < 6 also slot 64 + lane
  const int kl0 = wrap_idx(x0 + lane - 3, nt), kl1 = wrap_idx(x0 + lane + 29, nt);
  const int kh = wrap_idx(x0 + lane + 61, nt);
  const int rows = min(WTR, jend - j0);

  if constexpr (WALK) {
#if NWB_WENO_CPASYNC
    // the tile's own rows j0 .. j0+rows-1 never wrap (rows <= jend - j0): a
    // running row pointer instead of a wrapped row index per row
    const T* vr = v + (size_t)(halo ? j0 + 3 : j0) * nt;
    for (int r = 0; r < rows; ++r, vr += nt) {
      cp_async_real(&ftw[r][lane], vr + kl0);
      cp_async_real(&ftw[r][lane + 32], vr + kl1);
      if (lane < 6) cp_async_real(&ftw[r][64 + lane], vr + kh);
    }
    cp_async_wait_all();
#else
#pragma unroll 8
    for (int r = 0; r < rows; ++r) {
      const T* vr = v + (size_t)vrow(j0 + r) * nt;
      ftw[r][lane] = vr[kl0];
      ftw[r][lane + 32] = vr[kl1];
      if (lane < 6) ftw[r][64 + lane] = vr[kh];
    }
#endif
    __syncwarp();
    if (lane < rows) {
      const T c = mul_rn(pi, upar[j0 + lane]);
      const P cp(hath - c), cm(-hath - c), qb2(qb);
      T* tr = ftw[lane];
      P p[6], m[6], dp[6], dm[6];
#pragma unroll
      for (int d = 0; d < 5; ++d) {
        const P vv(tr[d], tr[32 + d]);
        p[d] = vv * fma(qb2, vv, cp);
        m[d] = vv * fma(qb2, vv, cm);
      }
      dp[1] = dsq(p[0], p[1], p[2]);
      dp[2] = dsq(p[1], p[2], p[3]);
      dm[2] = dsq(m[3], m[2], m[1]);
      dm[3] = dsq(m[4], m[3], m[2]);
#pragma unroll 6
      for (int f = 0; f <= 32; ++f) {
        const P vv(tr[f + 5], tr[f + 37]);
        p[5] = vv * fma(qb2, vv, cp);
        m[5] = vv * fma(qb2, vv, cm);
        dp[3] = dsq(p[2], p[3], p[4]);
        dm[4] = dsq(m[5], m[4], m[3]);
        const P fc = face_pair2_d(p[0], p[1], p[2], p[3], p[4], dp[1], dp[2], dp[3], m[5], m[4],
                                  m[3], m[2], m[1], dm[4], dm[3], dm[2]);
        tr[f] = fc.v.x;
        tr[f + 37] = fc.v.y;
#pragma unroll
        for (int d = 0; d < 5; ++d) {
          p[d] = p[d + 1];
          m[d] = m[d + 1];
          dp[d] = dp[d + 1];
          dm[d] = dm[d + 1];
        }
      }
    }
    __syncwarp();
  } else {
  // ---- theta faces (faces lane and lane + 32 of each row, packed)
  P vl(v[(size_t)vrow(j0) * nt + kl0], v[(size_t)vrow(j0) * nt + kl1]);
  T v_hi = lane < 6 ? v[(size_t)vrow(j0) * nt + kh] : (T)0;
  T c_cur = mul_rn(pi, upar[j0]);
  const P qb2(qb);
  for (int r = 0; r < rows; ++r) {
    const T cp = hath - c_cur, cm = -hath - c_cur;
    const P sp = vl * fma(qb2, vl, P(cp)), sm = vl * fma(qb2, vl, P(cm));
    lpw[lane] = sp.v.x;
    lpw[lane + 32] = sp.v.y;
    lmw[lane] = sm.v.x;
    lmw[lane + 32] = sm.v.y;
    if (lane < 6) {
      lpw[64 + lane] = v_hi * fma(qb, v_hi, cp);
      lmw[64 + lane] = v_hi * fma(qb, v_hi, cm);
    }
    if (r + 1 < rows) {
      const T* vn = v + (size_t)(halo ? j0 + r + 4 : j0 + r + 1) * nt;
      vl = P(vn[kl0], vn[kl1]);
      if (lane < 6) v_hi = vn[kh];
      c_cur = mul_rn(pi, upar[j0 + r + 1]);
    }
    __syncwarp();
    auto lp2 = [&](int d) { return P(lpw[lane + d], lpw[lane + 32 + d]); };
    auto lm2 = [&](int d) { return P(lmw[lane + d], lmw[lane + 32 + d]); };
    const P fc = face_pair2(lp2(0), lp2(1), lp2(2), lp2(3), lp2(4), lm2(5), lm2(4), lm2(3), lm2(2),
                            lm2(1));
    ftw[r][lane] = fc.v.x;
    ftw[r][lane + 32] = fc.v.y;
    __syncwarp();
  }
  // 65th theta face of row `lane` (between tile columns 63 and 64), scalar
  if (lane < rows) {
    const int j = j0 + lane;
    const T c = mul_rn(pi, upar[j]);
    const T cp = hath - c, cm = -hath - c;
    const T* vr = v + (size_t)vrow(j) * nt;
    T p[6], m[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      const T vv = vr[wrap_idx(x0 + 61 + d, nt)];
      p[d] = mul_rn(vv, fma(qb, vv, cp));
      m[d] = mul_rn(vv, fma(qb, vv, cm));
    }
    ftw[lane][WT2] = face_pair(p[0], p[1], p[2], p[3], p[4], m[5], m[4], m[3], m[2], m[1]);
  }
  __syncwarp();
  }  // !WALK

  // ---- rho sweep down columns k0 = x0 + lane and k1 = k0 + 32 (packed)
  const int k0 = x0 + lane, k1 = k0 + 32;
  const int kv0 = wrap_idx(k0, nt), kv1 = wrap_idx(k1, nt);
  P hp[6], hm[6], vw[6], dp[6], dm[6];
  const P harh2(harh), halP(half);
#pragma unroll
  for (int d = 0; d < 5; ++d) {
    const size_t ro = (size_t)vrow(j0 - 3 + d) * nt;
    const P vv(v[ro + kv0], v[ro + kv1]);
    const P uh(half * uperp_g[wrap_idx(cj0 + j0 - 3 + d, ng)]);
    hp[d] = vv * (uh + harh2);
    hm[d] = vv * (uh - harh2);
    vw[d] = vv;
  }
  dp[1] = dsq(hp[0], hp[1], hp[2]);
  dp[2] = dsq(hp[1], hp[2], hp[3]);
  dm[2] = dsq(hm[1], hm[2], hm[3]);
  dm[3] = dsq(hm[2], hm[3], hm[4]);
  P fprev((T)0);
  const bool ok0 = k0 < nt, ok1 = k1 < nt;
  T* outp = a.out + (size_t)mem * nr * nt + (size_t)j0 * nt;
  const T* dup = du + j0;
  const T* ftp = &ftw[0][lane];
  // offsets of faces (lane, lane + 1, lane + 32, lane + 33) from ftp (WALK layout above)
  const int fx1 = WALK ? (lane == 31 ? 6 : 1) : 1, fy0 = WALK ? 37 : 32, fy1 = fy0 + 1;
  const P idth(a.inv_dtheta), idrh(a.inv_drho);
  const T* vc0 = v + kv0;
  const T* vc1 = v + kv1;
  const int vrows = halo ? nr + 6 : nr;
  int ov = vrow(j0 + 2) * nt, ju = wrap_idx(cj0 + j0 + 2, ng);
  P vnext(vc0[ov], vc1[ov]);
  T unext = uperp_g[ju];
  auto row_step = [&](const P vv, const T uu, const bool emit, const bool full) {
    hp[5] = vv * P(fma(half, uu, harh));
    hm[5] = vv * P(fma(half, uu, -harh));
    vw[5] = vv;
    dp[3] = dsq(hp[2], hp[3], hp[4]);
    dm[4] = dsq(hm[3], hm[4], hm[5]);
    const P f = face_pair2_d(hp[0], hp[1], hp[2], hp[3], hp[4], dp[1], dp[2], dp[3], hm[5], hm[4],
                              hm[3], hm[2], hm[1], dm[4], dm[3], dm[2]);
    if (emit) {
      const P dth = (P(ftp[fx1], ftp[fy1]) - P(ftp[0], ftp[fy0])) * idth;
      const P drh = (f - fprev) * idrh;
      const P o = (P(*dup) * vw[2] - dth) - drh;
      if (full || ok0) outp[k0] = o.v.x;
      if (full || ok1) outp[k1] = o.v.y;
      outp += nt;
      ++dup;
      ftp += FTS;
    }
    fprev = f;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
      hp[d] = hp[d + 1];
      hm[d] = hm[d + 1];
      vw[d] = vw[d + 1];
      dp[d] = dp[d + 1];
      dm[d] = dm[d + 1];
    }
  };
  // interior tiles: unconditional prefetch on pointer increments (k_weno);
  // NWB_WENO_X2_UNROLL: unroll of the fp32 sweep (measurement knob)
  const int top = j0 + rows + 3;
  if ((halo ? top + 3 : top) < vrows && cj0 + top < ng && x0 + WT2 <= nt) {
    const T* vp0 = vc0 + ov;
    const T* vp1 = vc1 + ov;
    const T* up = uperp_g + ju;
    {
      const P vv = vnext;
      const T uu = unext;
      vp0 += nt;
      vp1 += nt;
      ++up;
      vnext = P(*vp0, *vp1);
      unext = *up;
      row_step(vv, uu, false, true);
    }
#pragma unroll SU
    for (int r = 1; r <= rows; ++r) {
      const P vv = vnext;
      const T uu = unext;
      vp0 += nt;
      vp1 += nt;
      ++up;
      vnext = P(*vp0, *vp1);
      unext = *up;
      row_step(vv, uu, true, true);
    }
  } else {
    const int vwrap = vrows * nt;
NWB_SEAM_UNROLL_PRAGMA
    for (int r = 0; r <= rows; ++r) {
      const P vv = vnext;
      const T uu = unext;
      if (r < rows) {
        ov += nt;
        ov = ov == vwrap ? 0 : ov;
        ju = ju + 1 == ng ? 0 : ju + 1;
        vnext = P(vc0[ov], vc1[ov]);
        unext = uperp_g[ju];
      }
      row_step(vv, uu, r > 0, false);
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

// fp32 runs the two-columns-per-lane packed kernel (NWB_WENO_F32X2=0 selects
// the scalar one: measurement knob).  An fp64 pair version (no packed fp64
// pipe; 160 registers, 71 KB shared) would drop occupancy below the scalar
// kernel's, which already keeps the FP64 pipe 73 % busy.
static bool weno_x2() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("NWB_WENO_F32X2");
    on = e ? (e[0] != '0') : 1;
  }
  return on == 1;
}

// theta faces by row walk (NWB_WENO_WALK=0 selects the row-by-row version:
// measurement knob); 32-row tiles only -- 16 / 8-row tiles would idle lanes
// read per launch (the step graphs capture the choice once)
static bool weno_walk() {
  const char* e = std::getenv("NWB_WENO_WALK");
  return !e || e[0] != '0';
}

template <typename T, int WTR> static void launch_weno_t(const WenoArgs<T>& a, cudaStream_t s) {
  const int nrows = (a.row_end ? a.row_end : a.g.nr) - a.row_begin;
  const int gy = (nrows + WTR * WWARPS - 1) / (WTR * WWARPS);
  if constexpr (sizeof(T) == 4) {
    if (weno_x2()) {
      dim3 grid((a.g.nt + WT2 - 1) / WT2, gy, a.g.batch);
      if (WTR == 32 && weno_walk() && a.g.nt < kNarrowNt)
        k_weno_x2<T, WTR, true, kX2UnrollNarrow><<<grid, WWARPS * 32, 0, s>>>(a);
      else if (WTR == 32 && weno_walk()) k_weno_x2<T, WTR, true><<<grid, WWARPS * 32, 0, s>>>(a);
      else k_weno_x2<T, WTR, false><<<grid, WWARPS * 32, 0, s>>>(a);
      return;
    }
  }
  dim3 grid((a.g.nt + WT - 1) / WT, gy, a.g.batch);
  if constexpr (sizeof(T) == 8 && WTR == 32) {
    if (a.tma && weno_walk()) {
      if (a.g.nt < kNarrowNt) k_weno<T, WTR, true, true, kSweepUnrollNarrow><<<grid, WWARPS * 32, 0, s>>>(a);
      else k_weno<T, WTR, true, true><<<grid, WWARPS * 32, 0, s>>>(a);
      return;
    }
  }
  if (WTR == 32 && weno_walk()) k_weno<T, WTR, true, false><<<grid, WWARPS * 32, 0, s>>>(a);
  else k_weno<T, WTR, false, false><<<grid, WWARPS * 32, 0, s>>>(a);
}

// rows per warp tile: 32 unless the grid has fewer than ~2048 tiles (small
// single grids), then 16 or 8 so more warps run shorter sweeps
template <typename T> void launch_weno(const WenoArgs<T>& a, cudaStream_t s) {
  const long tiles = (long)((a.g.nt + WT - 1) / WT) * ((a.g.nr + WT - 1) / WT) * a.g.batch;
  if (a.row_end || tiles >= 2048) launch_weno_t<T, 32>(a, s);
  else if (tiles >= 1024) launch_weno_t<T, 16>(a, s);
  else launch_weno_t<T, 8>(a, s);
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
