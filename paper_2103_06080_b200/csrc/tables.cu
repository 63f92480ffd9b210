// Exponential-integrator multiplier tables on the device
// (reference pkg/src/nwave/exprk.py:42-131).
//
//   xi_j    = 2 pi j_s / rho_span,   j_s = fftfreq(nr) * nr
//   omega_k = 2 pi k / theta_span,   k = 0 .. nt/2
//   z       = ds * ( -xi^2 / (4 pi (i omega + eps/(4 pi))) - A omega^2 )
//   E = exp z,  Phi1 = phi1(z),  Phi2 = phi2(z),  Phi1m2 = cast(Phi1) - cast(Phi2)
//   phi_s(z) = 18-term Horner series for |z| < 0.5, else the direct formula.
//
// Evaluated in fp64 and cast afterwards (exprk.py:123-125).  This file is
// compiled with -fmad=false and divides the way numpy does (Smith's
// algorithm), so tables agree with the reference to the last bit or two;
// the build at Set 4 takes milliseconds instead of the reference's 7.5 s.
#include "internal.h"

namespace nwb {

__constant__ double c_inv_fact[20];  // 1/k!, k = 0..19 (host-rounded like Python)

__device__ __forceinline__ double2 z_mul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// numpy's complex division (Smith)
__device__ __forceinline__ double2 z_div(double2 a, double2 b) {
  const double ar = fabs(b.x), ai = fabs(b.y);
  if (ar >= ai) {
    if (ar == 0.0 && ai == 0.0) return make_double2(a.x / ar, a.y / ai);
    const double rat = b.y / b.x, scl = 1.0 / (b.x + b.y * rat);
    return make_double2((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
  }
  const double rat = b.x / b.y, scl = 1.0 / (b.y + b.x * rat);
  return make_double2((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
}
__device__ __forceinline__ double2 z_exp(double2 z) {
  if (z.y == 0.0) return make_double2(exp(z.x), z.y);
  const double e = exp(z.x);
  double s, c;
  sincos(z.y, &s, &c);
  return make_double2(e * c, e * s);
}

__device__ double2 phi_eval(double2 z, int shift) {
  if (hypot(z.x, z.y) < 0.5) {
    double2 acc = make_double2(c_inv_fact[17 + shift], 0.0);
    for (int m = 16; m >= 0; --m) {
      acc = z_mul(acc, z);
      acc.x = acc.x + c_inv_fact[m + shift];
    }
    return acc;
  }
  const double2 ez = z_exp(z);
  if (shift == 1) return z_div(make_double2(ez.x - 1.0, ez.y), z);
  const double2 num = make_double2((ez.x - 1.0) - z.x, ez.y - z.y);
  return z_div(num, z_mul(z, z));
}

template <typename V> __device__ __forceinline__ V cast_c(double2 a);
template <> __device__ __forceinline__ double2 cast_c<double2>(double2 a) { return a; }
template <> __device__ __forceinline__ float2 cast_c<float2>(double2 a) {
  return make_float2(__double2float_rn(a.x), __double2float_rn(a.y));
}

template <typename T>
__global__ void k_tables(const TableArgs a, cplx<T>* E, cplx<T>* P1, cplx<T>* P2, cplx<T>* P12,
                         double2* zout) {
  using V = cplx<T>;
  const long total = (long)a.nr * a.kk;
  const double pi = 3.141592653589793;
  const double two_pi = 2.0 * pi;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    int f, k;
    long o;
    if (a.natural) {
      f = (int)(i / a.kk);
      k = (int)(i - (long)f * a.kk);
      o = i;
    } else {
      k = (int)(i / a.nr);
      const int p = (int)(i - (long)k * a.nr);
      f = a.rev_r[p];
      o = (long)k * a.ld + p;
    }
    const int js = f <= (a.nr - 1) / 2 ? f : f - a.nr;                // fftfreq order
    const double jf = ((double)js * (1.0 / (double)a.nr)) * (double)a.nr;
    const double xi = two_pi * jf / a.rho_span;
    const double om = two_pi * (double)(k + a.k0) / a.theta_span;
    const double2 den = make_double2(a.eps / (4.0 * pi), om);
    const double2 den4 = make_double2(4.0 * pi * den.x, 4.0 * pi * den.y);
    const double2 q = z_div(make_double2(-(xi * xi), 0.0), den4);
    const double2 zz = make_double2(a.d_sigma * (q.x - a.A * (om * om)), a.d_sigma * q.y);
    const V e = cast_c<V>(z_exp(zz));
    const V p1 = cast_c<V>(phi_eval(zz, 1));
    const V p2 = cast_c<V>(phi_eval(zz, 2));
    if (E) E[o] = e;
    if (P1) P1[o] = p1;
    if (P2) P2[o] = p2;
    if (P12) P12[o] = csub(p1, p2);
    if (zout) zout[o] = zz;
  }
}

__global__ void k_phi(const double2* z, long n, int shift, double2* out) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = phi_eval(z[i], shift);
}

static void upload_factorials(cudaStream_t s) {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && done[dev]) return;
  // Python's 1.0 / math.factorial(k): the integer is converted to the nearest
  // double first (19! > 2^53), then one correctly rounded division.
  double h[20];
  unsigned long long fact = 1ULL;
  for (int k = 0; k < 20; ++k) {
    if (k > 0) fact *= (unsigned long long)k;
    h[k] = 1.0 / (double)fact;
  }
  cudaMemcpyToSymbolAsync(c_inv_fact, h, sizeof(h), 0, cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);
  if (dev < 64) done[dev] = true;
}

template <typename T>
void launch_tables(const TableArgs& a, cplx<T>* E, cplx<T>* P1, cplx<T>* P2, cplx<T>* P12,
                   double2* z, cudaStream_t s) {
  upload_factorials(s);
  const long total = (long)a.nr * a.kk;
  long blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  k_tables<T><<<(int)blocks, 256, 0, s>>>(a, E, P1, P2, P12, z);
}

void launch_phi(const double2* z, long n, int shift, double2* out, cudaStream_t s) {
  upload_factorials(s);
  long blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  k_phi<<<(int)blocks, 256, 0, s>>>(z, n, shift, out);
}

template void launch_tables<double>(const TableArgs&, double2*, double2*, double2*, double2*, double2*, cudaStream_t);
template void launch_tables<float>(const TableArgs&, float2*, float2*, float2*, float2*, double2*, cudaStream_t);

}  // namespace nwb

// ---------------------------------------------------------------- turbulence
// Device port of the random-mode velocity field (reference
// pkg/src/nwave/turbulence.py:145-203):
//   a = kx_n lam sigma_i,  b = ky_n lam rho_j + phi_n
//   c = cos a cos b - sin a sin b,  s = sin a cos b + cos a sin b
//   U_par += amp1_n c, U_perp += amp2_n c, dU_perp/dsigma += w_ds_n s,
//   dU_perp/drho += w_dr_n s,  modes accumulated in ascending order,
// then scaled by 1/c0.  Same split and order as the reference's _mode_sum,
// compiled without FMA contraction (this file), so the only difference is
// the device's sincos (<= 1 ulp).

namespace nwb {

__global__ void k_mode_trig(const double* kx, const double* ky, const double* ph, double lam,
                            const double* sig, int n_sig, const double* rho, int n_rho, int n_modes,
                            double* ca, double* sa, double* cb, double* sb) {
  const long tot_a = (long)n_sig * n_modes, tot_b = (long)n_modes * n_rho;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < tot_a + tot_b;
       t += (long)gridDim.x * blockDim.x) {
    if (t < tot_a) {
      const int i = (int)(t / n_modes), n = (int)(t - (long)i * n_modes);
      const double a = kx[n] * lam * sig[i];
      double s, c;
      sincos(a, &s, &c);
      ca[t] = c;
      sa[t] = s;
    } else {
      const long u = t - tot_a;
      const int n = (int)(u / n_rho), j = (int)(u - (long)n * n_rho);
      const double b = ky[n] * lam * rho[j] + ph[n];
      double s, c;
      sincos(b, &s, &c);
      cb[u] = c;
      sb[u] = s;
    }
  }
}

// one thread per (i, j); the mode loop walks the trig tables in order
__global__ void k_mode_sum(int n_sig, int n_rho, int n_modes, const double* ca, const double* sa,
                           const double* cb, const double* sb, const double* a1, const double* a2,
                           const double* wds, const double* wdr, double inv_c0, double* u_par,
                           double* u_perp, double* du_ds, double* du_dr) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= n_rho) return;
  double up = 0, uq = 0, ds = 0, dr = 0;
  const double* cai = ca + (size_t)i * n_modes;
  const double* sai = sa + (size_t)i * n_modes;
  for (int n = 0; n < n_modes; ++n) {
    const double c_a = __ldg(cai + n), s_a = __ldg(sai + n);
    const double c_b = cb[(size_t)n * n_rho + j], s_b = sb[(size_t)n * n_rho + j];
    const double c = c_a * c_b - s_a * s_b;
    const double s = s_a * c_b + c_a * s_b;
    up += __ldg(a1 + n) * c;
    uq += __ldg(a2 + n) * c;
    ds += __ldg(wds + n) * s;
    dr += __ldg(wdr + n) * s;
  }
  const size_t o = (size_t)i * n_rho + j;
  u_par[o] = up * inv_c0;
  u_perp[o] = uq * inv_c0;
  du_ds[o] = ds * inv_c0;
  du_dr[o] = dr * inv_c0;
}

void launch_turbulence(const double* kx, const double* ky, const double* ph, const double* a1,
                       const double* a2, const double* wds, const double* wdr, int n_modes,
                       double lam, double inv_c0, const double* sig, int n_sig, const double* rho,
                       int n_rho, double* scratch, double* u_par, double* u_perp, double* du_ds,
                       double* du_dr, cudaStream_t s) {
  double* ca = scratch;
  double* sa = ca + (size_t)n_sig * n_modes;
  double* cb = sa + (size_t)n_sig * n_modes;
  double* sb = cb + (size_t)n_modes * n_rho;
  const long tot = (long)n_sig * n_modes + (long)n_modes * n_rho;
  long blocks = (tot + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_mode_trig<<<(int)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(kx, ky, ph, lam, sig, n_sig, rho, n_rho,
                                                            n_modes, ca, sa, cb, sb);
  dim3 grid((n_rho + 127) / 128, n_sig);
  k_mode_sum<<<grid, 128, 0, s>>>(n_sig, n_rho, n_modes, ca, sa, cb, sb, a1, a2, wds, wdr, inv_c0,
                                  u_par, u_perp, du_ds, du_dr);
}

}  // namespace nwb
