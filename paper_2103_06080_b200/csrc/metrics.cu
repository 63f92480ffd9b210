// Ground metrics of a marched field on the device: for
// every member, on the theta trace of one rho row restricted to the roi
// [k0, k1], the peak P = max V, the first upward crossing of 0.1 P and the
// next upward crossing of 0.9 P, linearly interpolated between nodes --
// bit-for-bit the host definition in paper_2103_06080_b200/analysis.py
// (ground_metrics; builder metric of SURVEY 8(d), not in the reference).
// An ensemble (BASELINE C4) gets its per-member metrics without copying the
// fields to the host.
//
// One CTA per member; the crossings are block-wide minimum-index reductions.
// Interpolation uses explicitly rounded operations (no FMA contraction), as
// numpy evaluates (level - y0) / (y1 - y0) and x0 + t (x1 - x0).
#include "internal.h"

namespace nwb {

namespace {

__device__ __forceinline__ int block_min_int(int v, int* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();  // red is reused
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : INT_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

__device__ __forceinline__ double block_max_double(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

// first i in [max(start, 1), n) with y[i-1] < level <= y[i], or n
template <typename T>
__device__ int first_upward(const T* y, int n, double level, int start, int* red) {
  int best = n;
  for (int i = max(start, 1) + (int)threadIdx.x; i < n; i += blockDim.x)
    if ((double)y[i - 1] < level && level <= (double)y[i]) { best = i; break; }
  return block_min_int(best, red);
}

template <typename T>
__device__ double interp(const T* y, const double* x, int i, double level) {
  const double y0 = (double)y[i - 1], y1 = (double)y[i];
  const double t = __ddiv_rn(__dsub_rn(level, y0), __dsub_rn(y1, y0));
  return __dadd_rn(x[i - 1], __dmul_rn(t, __dsub_rn(x[i], x[i - 1])));
}

template <typename T>
__global__ void k_ground_metrics(const T* v, int nr, int nt, int row, int k0, int n,
                                 const double* x, double* out) {
  __shared__ int ired[32];
  __shared__ double dred[32];
  const int mem = blockIdx.x;
  const T* y = v + ((size_t)mem * nr + row) * nt + k0;
  double pk = -INFINITY;
  for (int i = threadIdx.x; i < n; i += blockDim.x) pk = fmax(pk, (double)y[i]);
  pk = block_max_double(pk, dred);
  const double l10 = __dmul_rn(0.1, pk), l90 = __dmul_rn(0.9, pk);
  const int i10 = first_upward(y, n, l10, 0, ired);
  const double t10 = i10 < n ? interp(y, x, i10, l10) : (double)NAN;
  // host: searchsorted(x, t10) (left), or n when t10 is NaN
  int s10 = n;
  if (i10 < n)
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if (x[i] >= t10) { s10 = i; break; }
  s10 = block_min_int(s10, ired);
  const int i90 = first_upward(y, n, l90, s10, ired);
  const double t90 = i90 < n ? interp(y, x, i90, l90) : (double)NAN;
  if (threadIdx.x == 0) {
    out[mem * 3 + 0] = pk;
    out[mem * 3 + 1] = t10;
    out[mem * 3 + 2] = t90;
  }
}

}  // namespace

template <typename T>
void launch_ground_metrics(const T* v, int batch, int nr, int nt, int row, int k0, int n,
                           const double* x, double* out, cudaStream_t s) {
  k_ground_metrics<T><<<batch, 256, 0, s>>>(v, nr, nt, row, k0, n, x, out);
}

template void launch_ground_metrics<double>(const double*, int, int, int, int, int, int,
                                            const double*, double*, cudaStream_t);
template void launch_ground_metrics<float>(const float*, int, int, int, int, int, int,
                                           const double*, double*, cudaStream_t);

}  // namespace nwb
