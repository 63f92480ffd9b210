// Shared device helpers: complex arithmetic on double2/float2, ordered-bit
// max reductions, launch checking.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace nwb {

template <typename T> struct cplx_of;
template <> struct cplx_of<double> { using type = double2; };
template <> struct cplx_of<float> { using type = float2; };
template <typename T> using cplx = typename cplx_of<T>::type;

template <typename V> __device__ __forceinline__ V mk(decltype(V::x) re, decltype(V::x) im) {
  V r; r.x = re; r.y = im; return r;
}
template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return mk<V>(a.x + b.x, a.y + b.y); }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return mk<V>(a.x - b.x, a.y - b.y); }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  return mk<V>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename V> __device__ __forceinline__ V cmulc(V a, V b) {
  return mk<V>(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <typename V> __device__ __forceinline__ V cconj(V a) { return mk<V>(a.x, -a.y); }
template <typename V> __device__ __forceinline__ V cscale(V a, decltype(V::x) s) { return mk<V>(a.x * s, a.y * s); }
// acc + s * t (real s)
template <typename V> __device__ __forceinline__ V caxpy(decltype(V::x) s, V t, V acc) {
  return mk<V>(acc.x + s * t.x, acc.y + s * t.y);
}

// fp32 complex arithmetic on Blackwell's packed FP32 pipe: one (re, im) pair
// is one float2 register pair, so adds are one FADD2 and a complex product is
// FMUL2 + FFMA2 (sm_100: a plain FFMA issues half the FP32 peak).
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  return __ffma2_rn(b, make_float2(-1.0f, -1.0f), a);
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  // (a.x b.x - a.y b.y, a.x b.y + a.y b.x)
  return __ffma2_rn(make_float2(a.x, a.x), b, __fmul2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x)));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  // a conj(b) = (a.x b.x + a.y b.y, a.y b.x - a.x b.y)
  return __ffma2_rn(make_float2(b.x, b.x), a, __fmul2_rn(make_float2(b.y, b.y), make_float2(a.y, -a.x)));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
__device__ __forceinline__ float2 caxpy(float s, float2 t, float2 acc) {
  return __ffma2_rn(make_float2(s, s), t, acc);
}
// multiply by +i (INV=true) or -i (INV=false)
template <bool PLUS, typename V> __device__ __forceinline__ V mul_i(V a) {
  return PLUS ? mk<V>(-a.y, a.x) : mk<V>(a.y, -a.x);
}

// Max of non-negative values (and NaN) through the IEEE bit pattern: for
// x >= 0 the unsigned bit pattern orders like the value, and any NaN with
// the sign bit cleared sorts above +inf, so a NaN anywhere wins the max.
__device__ __forceinline__ unsigned long long abs_bits(double x) {
  return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffULL;
}
__device__ __forceinline__ unsigned long long abs_bits(float x) {
  return abs_bits((double)x);
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// ---- asynchronous copies (sm_80+ LDGSTS, sm_90+ bulk L2 prefetch)
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
// wait until at most one committed group is still in flight
__device__ __forceinline__ void cp_async_wait_1() {
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_0() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}
// Prefetch [ptr, ptr + bytes) into L2 with one bulk (TMA) request per 64 KB;
// bytes must be a multiple of 16 and ptr 16-byte aligned.
__device__ __forceinline__ void prefetch_l2_bulk(const void* ptr, unsigned bytes) {
  const uintptr_t a = (uintptr_t)ptr & ~(uintptr_t)15;  // 16-byte aligned start
  bytes = (unsigned)(((uintptr_t)ptr + bytes - a) & ~(uintptr_t)15);
  const char* p = (const char*)a;
  while (bytes) {
    const unsigned chunk = bytes > 65536u ? 65536u : bytes;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(chunk) : "memory");
    p += chunk;
    bytes -= chunk;
  }
}

// ---- bulk (TMA engine) copies with an mbarrier, sm_90+ (SASS UBLKCP)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// one arrival that also raises the transaction count by `bytes`
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// global -> shared bulk copy completing `bytes` on the mbarrier (16-byte
// aligned addresses, bytes a multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global bulk copy (bulk group); the caller fences the writes to
// the async proxy before and waits for the group's smem reads after
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
// make an mbarrier's initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// TMA tiled load of one box of a rank-3 tensor map (coordinates innermost
// first, signed: out-of-bounds elements are zero-filled) completing the box's
// bytes on the mbarrier (SASS UTMALDG); `map` must live in param / const /
// global memory (a __grid_constant__ kernel parameter)
__device__ __forceinline__ void tma_load_3d(void* sdst, const CUtensorMap* map, int c0, int c1,
                                            int c2, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(sdst)),
      "l"((unsigned long long)(uintptr_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// complex loads/stores of 16-byte (double2) or 8-byte (float2) elements
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
// one real (8 or 4 bytes)
template <typename T> __device__ __forceinline__ void cp_async_real(T* dst, const T* src) {
  if constexpr (sizeof(T) == 8) cp_async8(dst, src);
  else cp_async4(dst, src);
}
template <typename V> __device__ __forceinline__ void cp_async_c(V* dst, const V* src) {
  if constexpr (sizeof(V) == 16) cp_async16(dst, src);
  else cp_async8(dst, src);
}

}  // namespace nwb
