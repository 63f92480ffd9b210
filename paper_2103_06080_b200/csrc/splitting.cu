// Lie-Trotter splitting baseline (reference
// pkg/src/nwave/splitting.py).  One step on the closed rho grid (n = N_rho + 1
// nodes, mirrored Neumann ghosts) x periodic theta, always float64 like the
// reference:
//
//   diffraction  Crank-Nicolson in sigma, trapezoid in theta (splitting.py:78-145)
//   Burgers      Godunov flux, periodic theta            (splitting.py:148-177)
//   axial+absorption  theta-frequency multiplier         (splitting.py:180-201;
//                the theta FFTs are the march's k_theta_r2c / k_theta_c2r)
//   transverse   Lax-Wendroff in rho                     (splitting.py:204-223)
//
// The diffraction stage is sequential in the theta index k (stage k's
// right-hand side needs the second differences of every updated stage
// l < k).  The B200 form keeps the O(N_rho N_theta) parts parallel and the
// k recurrence in one CTA:
//   k_split_prep   per rho row: the old second differences d2n and their
//                  running trapezoid prefix s_k = (d2n_0 + d2n_k)/2 +
//                  sum_{0<l<k} d2n_l (the reference re-sums the prefix for
//                  every k, O(N_rho N_theta^2); the running sum equals it to
//                  rounding), stored theta-major so a stage reads a column
//                  contiguously;
//   k_split_diffraction  one CTA walks k = 1 .. N_theta-1: rhs = v0 +
//                  gamma (s_k + sum_prev), the constant-coefficient Thomas
//                  solve as two affine parallel scans over rho (forward
//                  elimination, back substitution; chunk per thread, warp
//                  shuffles, one smem round), then sum_prev += D2 out_k.
// Compiled with -fmad=false: the elementwise stages round like numpy.
#include "internal.h"

namespace nwb {

// ------------------------------------------------------------------ prep
// v (n, nt) row-major -> vT (nt, ldn) and sT (nt, ldn) theta-major
__global__ void k_split_prep(const double* __restrict__ v, int n, int nt, int ldn,
                             double* __restrict__ vT, double* __restrict__ sT) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int jm = j == 0 ? 1 : j - 1;
  const int jp = j == n - 1 ? n - 2 : j + 1;
  const double* r0 = v + (size_t)j * nt;
  const double* rm = v + (size_t)jm * nt;
  const double* rp = v + (size_t)jp * nt;
  const double d0 = (rp[0] - 2.0 * r0[0]) + rm[0];
  double run = 0.0;  // sum_{0<l<k} d2n_l
  vT[j] = r0[0];
  sT[j] = 0.0;
  for (int k = 1; k < nt; ++k) {
    const double dk = (rp[k] - 2.0 * r0[k]) + rm[k];
    vT[(size_t)k * ldn + j] = r0[k];
    sT[(size_t)k * ldn + j] = 0.5 * (d0 + dk) + run;
    run += dk;
  }
}

// ------------------------------------------------------------------ scans
// Affine maps y -> a y + b composed along rho: block-wide inclusive scan of
// per-thread chunk maps (thread order = rho order, or reversed for back
// substitution).  Returns the composition of all maps *before* this
// thread's chunk (identity for the first thread).
struct Aff {
  double a, b;
};
__device__ __forceinline__ Aff compose(Aff first, Aff then) {  // then(first(y))
  return Aff{then.a * first.a, then.a * first.b + then.b};
}

template <int NT>
__device__ __forceinline__ Aff block_exclusive_scan(Aff m, Aff* wsum, bool reverse) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  // warp inclusive scan in scan order (reverse: higher lanes first)
  Aff inc = m;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double pa = reverse ? __shfl_down_sync(0xffffffffu, inc.a, o) : __shfl_up_sync(0xffffffffu, inc.a, o);
    const double pb = reverse ? __shfl_down_sync(0xffffffffu, inc.b, o) : __shfl_up_sync(0xffffffffu, inc.b, o);
    const bool has = reverse ? lane + o < 32 : lane >= o;
    if (has) inc = compose(Aff{pa, pb}, inc);
  }
  // exclusive within the warp
  double ea = reverse ? __shfl_down_sync(0xffffffffu, inc.a, 1) : __shfl_up_sync(0xffffffffu, inc.a, 1);
  double eb = reverse ? __shfl_down_sync(0xffffffffu, inc.b, 1) : __shfl_up_sync(0xffffffffu, inc.b, 1);
  const bool first_lane = reverse ? lane == 31 : lane == 0;
  Aff exc = first_lane ? Aff{1.0, 0.0} : Aff{ea, eb};
  if (reverse ? lane == 0 : lane == 31) wsum[warp] = inc;  // warp total
  __syncthreads();
  if (warp == 0) {
    // exclusive scan of the warp totals (in scan order) by warp 0
    const int w = reverse ? NW - 1 - lane : lane;
    Aff t = lane < NW ? wsum[w] : Aff{1.0, 0.0};
    Aff ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double pa = __shfl_up_sync(0xffffffffu, ti.a, o);
      const double pb = __shfl_up_sync(0xffffffffu, ti.b, o);
      if (lane >= o) ti = compose(Aff{pa, pb}, ti);
    }
    const double xa = __shfl_up_sync(0xffffffffu, ti.a, 1);
    const double xb = __shfl_up_sync(0xffffffffu, ti.b, 1);
    __syncwarp();
    if (lane < NW) wsum[NW + w] = lane == 0 ? Aff{1.0, 0.0} : Aff{xa, xb};
  }
  __syncthreads();
  return compose(wsum[NW + warp], exc);
}

// ------------------------------------------------------------------ diffraction
// One CTA of NT threads; smem: sum_prev, y (forward-eliminated rhs), out,
// each n doubles, plus the scan scratch.  lower / upper / diag / w are the
// reference's Thomas factorisation (splitting.py:103-113).
template <int NT>
__global__ void __launch_bounds__(NT, 1) k_split_diffraction(const double* __restrict__ vT,
                                                             const double* __restrict__ sT, int n,
                                                             int nt, int ldn, double gamma,
                                                             const double* __restrict__ wv,
                                                             const double* __restrict__ up,
                                                             const double* __restrict__ dg,
                                                             double* __restrict__ out,
                                                             double* __restrict__ gline) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // the three rho lines live in shared memory, or in global scratch (gline,
  // L2-resident) when 3 n doubles exceed it
  Aff* wsum = reinterpret_cast<Aff*>(smem_raw);
  double* sum_prev = gline ? gline : reinterpret_cast<double*>(wsum + 2 * (NT / 32));
  double* y = sum_prev + n;
  double* col = y + n;
  const int chunk = (n + NT - 1) / NT;
  const int j0 = threadIdx.x * chunk, j1 = min(n, j0 + chunk);
  // stage 0: unchanged field; sum_prev = D2 out_0 / 2
  for (int j = threadIdx.x; j < n; j += NT) out[(size_t)j * nt] = vT[j];
  for (int j = threadIdx.x; j < n; j += NT) {
    const int jm = j == 0 ? 1 : j - 1, jp = j == n - 1 ? n - 2 : j + 1;
    sum_prev[j] = 0.5 * ((vT[jp] - 2.0 * vT[j]) + vT[jm]);
  }
  __syncthreads();
  for (int k = 1; k < nt; ++k) {
    const double* vk = vT + (size_t)k * ldn;
    const double* sk = sT + (size_t)k * ldn;
    // forward elimination y_j = rhs_j - w_j y_{j-1}: chunk map, scan, apply
    Aff m{1.0, 0.0};
    for (int j = j0; j < j1; ++j) {
      const double rhs = vk[j] + gamma * (sk[j] + sum_prev[j]);
      y[j] = rhs;
      const Aff f = j == 0 ? Aff{0.0, rhs} : Aff{-__ldg(&wv[j]), rhs};
      m = compose(m, f);
    }
    Aff pre = block_exclusive_scan<NT>(m, wsum, false);
    double yy = pre.b;  // y_{j0-1} (the first map ignores its input)
    for (int j = j0; j < j1; ++j) {
      yy = j == 0 ? y[j] : y[j] - __ldg(&wv[j]) * yy;
      y[j] = yy;
    }
    __syncthreads();
    // back substitution out_j = (y_j - upper_j out_{j+1}) / diag_j, reversed scan
    Aff mb{1.0, 0.0};
    for (int j = j1 - 1; j >= j0; --j) {
      const double d = __ldg(&dg[j]);
      const Aff f = j == n - 1 ? Aff{0.0, y[j] / d} : Aff{-__ldg(&up[j]) / d, y[j] / d};
      mb = compose(mb, f);
    }
    Aff preb = block_exclusive_scan<NT>(mb, wsum, true);
    double oo = preb.b;  // out_{j1}
    for (int j = j1 - 1; j >= j0; --j) {
      oo = j == n - 1 ? y[j] / __ldg(&dg[j]) : (y[j] - __ldg(&up[j]) * oo) / __ldg(&dg[j]);
      col[j] = oo;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += NT) {
      const int jm = j == 0 ? 1 : j - 1, jp = j == n - 1 ? n - 2 : j + 1;
      sum_prev[j] += (col[jp] - 2.0 * col[j]) + col[jm];
      out[(size_t)j * nt + k] = col[j];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ Burgers
__device__ __forceinline__ double godunov(double ul, double ur, double half_b) {
  const double mn = -half_b * fmax(ul * ul, ur * ur);
  const bool straddle = (ur <= 0.0) && (ul >= 0.0);
  const double mx = straddle ? 0.0 : -half_b * fmin(ul * ul, ur * ur);
  return ul <= ur ? mn : mx;
}

__global__ void k_godunov_flux(long n, const double* ul, const double* ur, double B, double* out) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = godunov(ul[i], ur[i], 0.5 * B);
}

__global__ void k_split_burgers(const double* __restrict__ v, int n, int nt, double B, double ratio,
                                double* __restrict__ out) {
  const long total = (long)n * nt;
  const double hb = 0.5 * B;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int k = (int)(i % nt);
    const double* row = v + (i - k);
    const double c = row[k];
    const double r = row[k + 1 < nt ? k + 1 : 0];
    const double l = row[k > 0 ? k - 1 : nt - 1];
    const double fr = godunov(c, r, hb), fl = godunov(l, c, hb);
    out[i] = c - ratio * (fr - fl);
  }
}

// ------------------------------------------------------------------ axial + absorption
// spectrum (kk, ld) of the theta r2c: mode k of row j times
// exp(i 2 pi q_j w_k - A ds w_k^2), q_j = U_par[j] ds, w_k = 2 pi k / theta_span,
// in numpy's evaluation order (splitting.py:193-198)
__global__ void k_split_axial(double2* __restrict__ spec, int n, int kk, int ld,
                              const double* __restrict__ upar, double ds, double A,
                              double theta_span) {
  const long total = (long)kk * n;
  const double two_pi = 6.283185307179586476925;
  const double ads = A * ds;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int k = (int)(i / n), j = (int)(i - (long)k * n);
    const double w = two_pi * (double)k / theta_span;
    const double q = upar[j] * ds;
    const double im = (two_pi * q) * w;
    const double re = 0.0 - ads * (w * w);
    double s, c;
    sincos(im, &s, &c);
    const double e = exp(re);
    const double mr = e * c, mi = e * s;
    double2 x = spec[(size_t)k * ld + j];
    spec[(size_t)k * ld + j] = make_double2(x.x * mr - x.y * mi, x.x * mi + x.y * mr);
  }
}

// ------------------------------------------------------------------ transverse (Lax-Wendroff)
// reflect-padded centred differences in rho (splitting.py:212-223); the
// max|out| of the step is folded into *vmax (IEEE bits, NaN sorts highest)
__global__ void k_split_transverse(const double* __restrict__ v, int n, int nt,
                                   const double* __restrict__ up, const double* __restrict__ dus,
                                   const double* __restrict__ dur, double ds, double dr,
                                   double* __restrict__ out, unsigned long long* vmax) {
  const long total = (long)n * nt;
  unsigned long long mx = 0;
  const double hds = 0.5 * ds;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int j = (int)(i / nt), k = (int)(i - (long)j * nt);
    const int jm = j == 0 ? 1 : j - 1, jp = j == n - 1 ? n - 2 : j + 1;
    const double c = v[i], a = v[(size_t)jp * nt + k], b = v[(size_t)jm * nt + k];
    const double d0 = (a - b) / (2.0 * dr);
    const double d2 = (a - 2.0 * c + b) / (dr * dr);
    const double u = up[j], us = dus[j], ur = dur[j];
    const double rhs = (((-u) * d0 - (hds * us) * d0) + ((hds * u) * ur) * d0) + (hds * (u * u)) * d2;
    const double o = c + ds * rhs;
    out[i] = o;
    unsigned long long bits = abs_bits(o);
    if (o != o) bits = 0x7fffffffffffffffULL;
    mx = bits > mx ? bits : mx;
  }
  if (vmax) {
    mx = warp_max_u64(mx);
    if ((threadIdx.x & 31) == 0) atomicMax(vmax, mx);
  }
}

// ------------------------------------------------------------------ launchers

static inline int sgrid(long n, int threads) {
  long b = (n + threads - 1) / threads;
  return (int)(b < 148L * 8 ? (b < 1 ? 1 : b) : 148L * 8);
}

void launch_split_prep(const double* v, int n, int nt, int ldn, double* vT, double* sT,
                       cudaStream_t s) {
  k_split_prep<<<(n + 127) / 128, 128, 0, s>>>(v, n, nt, ldn, vT, sT);
}

constexpr int SPLIT_NT = 512;
bool split_line_in_smem(int n) { return (size_t)3 * n * sizeof(double) <= 200 * 1024; }

void launch_split_diffraction(const double* vT, const double* sT, int n, int nt, int ldn,
                              double gamma, const double* w, const double* up, const double* dg,
                              double* out, double* gline, cudaStream_t s) {
  const bool in_smem = split_line_in_smem(n);
  const size_t sm = 2 * (SPLIT_NT / 32) * sizeof(Aff) + (in_smem ? (size_t)3 * n * sizeof(double) : 0);
  cudaFuncSetAttribute(k_split_diffraction<SPLIT_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sm);
  k_split_diffraction<SPLIT_NT><<<1, SPLIT_NT, sm, s>>>(vT, sT, n, nt, ldn, gamma, w, up, dg, out,
                                                        in_smem ? nullptr : gline);
}

void launch_split_burgers(const double* v, int n, int nt, double B, double ratio, double* out,
                          cudaStream_t s) {
  k_split_burgers<<<sgrid((long)n * nt, 256), 256, 0, s>>>(v, n, nt, B, ratio, out);
}

void launch_godunov_flux(long n, const double* ul, const double* ur, double B, double* out,
                         cudaStream_t s) {
  k_godunov_flux<<<sgrid(n, 256), 256, 0, s>>>(n, ul, ur, B, out);
}

void launch_split_axial(double2* spec, int n, int kk, int ld, const double* upar, double ds,
                        double A, double theta_span, cudaStream_t s) {
  k_split_axial<<<sgrid((long)kk * n, 256), 256, 0, s>>>(spec, n, kk, ld, upar, ds, A, theta_span);
}

void launch_split_transverse(const double* v, int n, int nt, const double* up, const double* dus,
                             const double* dur, double ds, double dr, double* out,
                             unsigned long long* vmax, cudaStream_t s) {
  k_split_transverse<<<sgrid((long)n * nt, 256), 256, 0, s>>>(v, n, nt, up, dus, dur, ds, dr, out,
                                                              vmax);
}

}  // namespace nwb
