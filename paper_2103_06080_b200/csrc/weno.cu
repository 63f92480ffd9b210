// WENO5-JS right-hand side b(sigma, V) with global Lax-Friedrichs splitting
// (reference pkg/src/nwave/weno.py:25-124), both directions in one kernel:
//
//   f_theta = -2 pi U_par V - (B/2) V^2,  f+- = (f_theta +- alpha_theta V) / 2
//   f_rho   =  U_perp V,                 h+- = (f_rho   +- alpha_rho   V) / 2
//   F[k+1/2] = W(f+_{k-2..k+2}) + W(f-_{k+3..k-1})          (periodic)
//   b = (dU_perp/drho V - (F_t[k+1/2]-F_t[k-1/2])/dtheta) - (F_r[j+1/2]-F_r[j-1/2])/drho
//
// One CTA owns a TY x TX tile; the tile plus a 3-cell halo on every side is
// staged in shared memory as split fluxes (no transposed copy of V, unlike
// the reference's rho sweep), faces are computed once and shared by the two
// cells they bound.  The face function keeps the reference's operation
// order (four divisions) so kernel-level parity stays at ~1e-15.
#include "internal.h"

namespace nwb {

template <typename T>
__device__ __forceinline__ T face5(T a0, T a1, T a2, T a3, T a4) {
  const T c1312 = (T)(13.0 / 12.0), q = (T)0.25, eps = (T)1e-6;
  const T d0 = (a0 - (T)2 * a1) + a2, e0 = (a0 - (T)4 * a1) + (T)3 * a2;
  const T d1 = (a1 - (T)2 * a2) + a3, e1 = a1 - a3;
  const T d2 = (a2 - (T)2 * a3) + a4, e2 = ((T)3 * a2 - (T)4 * a3) + a4;
  const T s0 = c1312 * (d0 * d0) + q * (e0 * e0);
  const T s1 = c1312 * (d1 * d1) + q * (e1 * e1);
  const T s2 = c1312 * (d2 * d2) + q * (e2 * e2);
  const T t0 = eps + s0, t1 = eps + s1, t2 = eps + s2;
  const T w0 = (T)0.1 / (t0 * t0), w1 = (T)0.6 / (t1 * t1), w2 = (T)0.3 / (t2 * t2);
  const T q0 = ((T)2 * a0 - (T)7 * a1) + (T)11 * a2;
  const T q1 = (-a1 + (T)5 * a2) + (T)2 * a3;
  const T q2 = ((T)2 * a2 + (T)5 * a3) - a4;
  return ((w0 * q0 + w1 * q1) + w2 * q2) / ((T)6 * ((w0 + w1) + w2));
}

__device__ __forceinline__ double bits_to_real(u64 b) { return __longlong_as_double((long long)b); }

constexpr int WTX = 32, WTY = 16, WH = 3;

template <typename T>
__global__ void __launch_bounds__(256) k_weno(const WenoArgs<T> a) {
  constexpr int PX = WTX + 2 * WH, PY = WTY + 2 * WH;
  __shared__ T fp[WTY][PX], fm[WTY][PX];   // theta split fluxes, rows of the tile
  __shared__ T hp[PY][WTX], hm[PY][WTX];   // rho split fluxes, columns of the tile
  __shared__ T vt[WTY][WTX];
  __shared__ T ft[WTY][WTX + 1], fr[WTY + 1][WTX];

  const int nr = a.g.nr, nt = a.g.nt;
  const int mem = blockIdx.z;
  const int x0 = blockIdx.x * WTX, y0 = blockIdx.y * WTY;
  const int tid = threadIdx.x;
  const int row = (a.step_ctr ? *a.step_ctr : 0) + a.row_off;
  const T* upar = a.upar + (size_t)row * nr;
  const T* uperp = a.uperp + (size_t)row * nr;
  const T* du = a.du + (size_t)row * nr;
  const T ath = (T)bits_to_real(a.alpha_bits[(size_t)mem * a.alpha_stride]);
  const T arh = (T)a.alpha_rho[row];
  const T two_pi = (T)6.283185307179586476925;
  const T half_b = (T)0.5 * a.bcoef;
  const T* v = a.v + (size_t)mem * nr * nt;

  // stage split fluxes (tile + halo; the four corner blocks are not needed)
  for (int idx = tid; idx < PY * PX; idx += blockDim.x) {
    const int ly = idx / PX, lx = idx - ly * PX;
    const bool in_rows = ly >= WH && ly < WH + WTY;
    const bool in_cols = lx >= WH && lx < WH + WTX;
    if (!in_rows && !in_cols) continue;
    int j = (y0 + ly - WH) % nr, k = (x0 + lx - WH) % nt;
    j = j < 0 ? j + nr : j;
    k = k < 0 ? k + nt : k;
    const T vv = v[(size_t)j * nt + k];
    if (in_rows) {
      const T c = two_pi * upar[j];
      const T g = -c * vv - half_b * vv * vv;
      const T av = ath * vv;
      fp[ly - WH][lx] = (T)0.5 * (g + av);
      fm[ly - WH][lx] = (T)0.5 * (g - av);
      if (in_cols) vt[ly - WH][lx - WH] = vv;
    }
    if (in_cols) {
      const T g = uperp[j] * vv;
      const T av = arh * vv;
      hp[ly][lx - WH] = (T)0.5 * (g + av);
      hm[ly][lx - WH] = (T)0.5 * (g - av);
    }
  }
  __syncthreads();
  // theta faces: ft[r][f] = face between tile columns f-1 and f
  for (int idx = tid; idx < WTY * (WTX + 1); idx += blockDim.x) {
    const int r = idx / (WTX + 1), f = idx - r * (WTX + 1);
    const T* p = &fp[r][f];
    const T* q = &fm[r][f];
    ft[r][f] = face5<T>(p[0], p[1], p[2], p[3], p[4]) + face5<T>(q[5], q[4], q[3], q[2], q[1]);
  }
  // rho faces: fr[g][c] = face between tile rows g-1 and g
  for (int idx = tid; idx < (WTY + 1) * WTX; idx += blockDim.x) {
    const int g = idx / WTX, c = idx - g * WTX;
    fr[g][c] = face5<T>(hp[g][c], hp[g + 1][c], hp[g + 2][c], hp[g + 3][c], hp[g + 4][c]) +
               face5<T>(hm[g + 5][c], hm[g + 4][c], hm[g + 3][c], hm[g + 2][c], hm[g + 1][c]);
  }
  __syncthreads();
  T* out = a.out + (size_t)mem * nr * nt;
  for (int idx = tid; idx < WTY * WTX; idx += blockDim.x) {
    const int r = idx / WTX, c = idx - r * WTX;
    const int j = y0 + r, k = x0 + c;
    if (j >= nr || k >= nt) continue;
    const T dth = (ft[r][c + 1] - ft[r][c]) * a.inv_dtheta;
    const T drh = (fr[r + 1][c] - fr[r][c]) * a.inv_drho;
    out[(size_t)j * nt + k] = (du[j] * vt[r][c] - dth) - drh;
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
  dim3 grid((a.g.nt + WTX - 1) / WTX, (a.g.nr + WTY - 1) / WTY, a.g.batch);
  k_weno<T><<<grid, 256, 0, s>>>(a);
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
