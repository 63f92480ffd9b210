// Measured FP64 (DFMA), FP32 (FFMA) and packed FP32 (FFMA2) issue peaks of
// this GPU: the denominators for WENO's FP-pipe roofline.
// Every thread runs ILP independent FMA chains (no memory traffic in the
// loop); the grid is 8 CTAs x 512 threads per SM.  flops = 2 per FMA lane
// (4 per FFMA2).  Built and run by tools/fp_peak.py.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ILP = 8;

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void k_ffma(float* out, int iters, float a, float b) {
  float acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fmaf(acc[i], a, b);
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678f) out[threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, int iters, float a, float b) {
  float2 acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = __ffma2_rn(acc[i], a2, b2);
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i].x + acc[i].y;
  if (s == 12345.678f) out[threadIdx.x] = s;
}

template <typename K, typename P>
static double run(K kern, P* buf, int iters, double lanes_per_fma, int sms) {
  const int blocks = sms * 8, threads = 512;
  kern<<<blocks, threads>>>(buf, iters, (P)0.999999, (P)1e-7);  // warm-up
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  double best = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(s);
    kern<<<blocks, threads>>>(buf, iters, (P)0.999999, (P)1e-7);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms = 0;
    cudaEventElapsedTime(&ms, s, e);
    const double flops = 2.0 * lanes_per_fma * (double)blocks * threads * iters * ILP;
    const double tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  void* buf;
  cudaMalloc(&buf, 1 << 20);
  const double d = run(k_dfma, (double*)buf, 4096, 1.0, sms);
  const double f = run(k_ffma, (float*)buf, 8192, 1.0, sms);
  const double f2 = run(k_ffma2, (float*)buf, 8192, 2.0, sms);
  cudaError_t err = cudaGetLastError();
  printf("{\"sms\": %d, \"clock_khz\": %d, \"fp64_dfma_tflops\": %.2f, \"fp32_ffma_tflops\": %.2f, "
         "\"fp32_ffma2_tflops\": %.2f, \"error\": \"%s\"}\n",
         sms, clk, d, f, f2, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
