// Host-side declarations shared by the CUDA translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft.cuh"

namespace nwb {

typedef unsigned long long u64;

// rho-pass modes
enum RhoMode {
  RHO_STAGE1 = 0,   // B1 = F(bt); U = E V + ds P12 B1; V* = E V + ds P1 B1 -> T* = F^-1 V*
  RHO_STAGE2 = 1,   // B2 = F(bt); V+ = U + ds P2 B2 -> Vh, T = F^-1 V+
  RHO_EULER = 2,    // B1 = F(bt); V+ = E V + ds P1 B1 -> Vh, T
  RHO_INIT = 3,     // Vh = F(bt) (digit-reversed), T = F^-1 Vh
  RHO_FWD_NAT = 4,  // out = F(bt) in natural order (no inverse)
  RHO_INV_NAT = 5,  // out = F^-1(in), `in` in natural order (vh = in, digit-reversed, if set)
  RHO_REV2NAT = 6,  // out = in permuted from digit-reversed to natural order
  RHO_FWD_DR = 7,   // sub-columns: out = F(bt) in digit-reversed positions (then REV2NAT)
};

// Geometry of one plan: physical fields are (batch, nr, nt) real, spectral
// arrays (batch, kk, ld) complex with kk = nt/2 + 1 rows of the rho axis.
struct Geom {
  int nr, nt, m, kk, ld, batch;
};

// Per-step bucket time stamps of the march (exprk.py:159-177's nonlinear /
// linear split): block (0, 0, 0) of a stamped launch writes %globaltimer at
// entry into buf[*step * NWB_TS_SLOTS + slot] -- slot 0 c2r of stage 1 (step
// start), 1 / 3 WENO start, 2 / 4 r2c start of stage 1 / 2 (WENO end); the
// next step's slot 0 ends a step.  No graph nodes, no host work per step.
constexpr int NWB_TS_SLOTS = 5;
struct StepStamp {
  unsigned long long* buf;    // null: no stamp
  const int* step;
  int slot;
};
__device__ __forceinline__ void step_stamp(const StepStamp& s) {
  if (s.buf && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    s.buf[(size_t)(*s.step) * NWB_TS_SLOTS + s.slot] = t;
  }
}

template <typename T> struct ThetaArgs {
  Geom g;
  FftDesc dh;                 // half-length (m) complex transform
  const cplx<T>* tw_h;        // W_m^t
  const cplx<T>* wk;          // W_nt^k, k <= m
  const int* pos_h;           // frequency -> position (digit reversal), length m
  // c2r: spectral (kk, ld) -> physical; r2c: physical -> spectral (kk, ld)
  const cplx<T>* spec_in;
  cplx<T>* spec_out;
  const T* phys_in;
  T* phys_out;
  T scale;                    // c2r output scale (1 / (nr nt))
  // optional reductions (c2r): alpha = max|2 pi u_par[j] + B v|, vmax = max|v|
  const T* upar;              // coefficient table base (rows of coef_ld) or null
  int coef_ld, coef_j0;       // coefficient row stride (0 = nr) and global row offset (slabs)
  const int* step_ctr;        // device step counter (row = *step_ctr + row_off) or null
  int row_off;
  T bcoef;
  u64* alpha_bits;            // per member, stride alpha_stride, or null
  int alpha_stride;
  u64* vmax_bits;             // per member, stride vmax_stride, slot = *step_ctr, or null
  int vmax_stride;
  int debug;                  // NWB_THETA_DEBUG measurement knobs (bit 4: no global traffic)
  // r2c row chunk [row_begin, row_end) (row_end 0 = all rows): the march overlaps
  // the r2c of one chunk with the WENO of the next on a side stream
  int row_begin, row_end;
  // fused first rho stage (r1 > 1, SPLIT kernels): a CTA owns the rho rows
  // i + r msub (r < r1, msub = nr / r1); r2c ends with the radix-r1 DIF stage of
  // the rho FFT across them (y_q = sum_r X_r w^{rq} W_nr^{q i} -> position
  // q msub + i), c2r starts with the matching DIT stage.  tw_first = W_nr^t, t < nr.
  int r1, msub;
  const cplx<T>* tw_first;
  int ilv;                    // transit layout: 1 = position q msub + i stored at i r1 + q
  int bulk;                   // r2c row loads as TMA bulk copies (fp64 rows)
  StepStamp ts;               // bucket time stamp at kernel entry (march only)
};

template <typename T> struct RhoArgs {
  Geom g;
  FftDesc dr;
  const cplx<T>* tw_r;
  const int* pos_r;           // frequency -> position
  const cplx<T>* in;          // (batch, kk, ld)
  cplx<T>* out;               // (batch, kk, ld)
  cplx<T>* vh;                // state spectrum, digit-reversed
  cplx<T>* u;                 // stage-1 partial update, digit-reversed
  const cplx<T>* E;           // tables (kk, ld), digit-reversed
  const cplx<T>* P1;
  const cplx<T>* P12;
  const cplx<T>* P2;
  T ds;
  int* step_ctr;              // incremented by block (0,0) when non-null (last kernel of a step)
  u64* zero_bits;             // alpha slot cleared for the next stage (per member), or null
  int zero_stride;
  // cluster-split variant (2 CTAs per column, n/2 points each): descriptor of
  // the half transform and W_n^i, i < n/2, for the radix-2 split stage
  FftDesc dh2;
  const cplx<T>* tw_h2;
  const cplx<T>* tw_split;
  int split;
  int half;                   // k_rho_half: half the column in registers, two columns per SM
  int prefetch;               // bulk L2 prefetch of the combine operands at entry: percent of each row
  int next_pf;                // > 0: prefetch the input column k + next_pf into L2 after the combine
  int roll;                   // > 0: the combine prefetches its operands roll rounds ahead into L2
  int debug;                  // measurement knobs (NWB_RHO_DEBUG): 1 skip FFTs, 2 skip combine loads
  // phase stagger of the first wave (one column per SM): CTA slot s of the
  // first `stagger_slots` blocks sleeps (s mod stagger_slots) * stagger_ns /
  // stagger_slots before starting (stagger_mode 1: odd slots sleep stagger_ns),
  // so SMs stream while others transform instead of all streaming at once
  int stagger_ns, stagger_slots, stagger_mode;
  int bulk;                   // column load / store as TMA bulk copies (fp64 columns)
  int persistent;             // march modes run k_rho_stream (one CTA per SM walking columns)
  // warp-specialised pass (k_rho_ws): transform / combine group sizes (0 = off),
  // CTAs (<= SMs x CTAs per SM) and their scratch (2 rows of ld per CTA)
  int ws_threads;
  int ws_threads2;
  int ws_ctas;
  int ws_debug;               // measurement: 1 = combine group idle, 2 = transform group skips FFTs
  cplx<T>* scratch;
  // sub-column pass (k_rho_sub, r1 > 1): CTA (member, k r1 + q1) transforms the
  // msub-point sub-column q1 (positions q1 msub + p'); dsub / tw_sub describe
  // the msub-point transform (the full plan without its first stage); dr keeps
  // the full transform for the j-symmetric table positions; rev_r = position
  // -> frequency (natural-order gathers)
  // slab transit layout (multi-GPU, slab.py): in / out hold, per destination
  // or source rank b with rho rows [blk_start[b], blk_start[b+1]), the block
  // (local modes x rows_b) contiguously at kk * blk_start[b] -- the
  // all-to-all's segments, so it moves them without packing copies
  int blk_n;
  int blk_start[17];
  int k_off, k_cnt;           // theta modes [k_off, k_off + k_cnt) of the launch (k_cnt 0: to kk): slab chunks
  int r1, ilv;
  FftDesc dsub;
  const cplx<T>* tw_sub;
  const int* rev_r;
};

template <typename T> struct WenoArgs {
  Geom g;
  const T* v;
  T* out;
  const T* upar;              // coefficient rows (nr each)
  const T* uperp;
  const T* du;
  const double* alpha_rho;    // per coefficient row
  const int* step_ctr;
  int row_off;
  const u64* alpha_bits;      // alpha_theta per member (stride alpha_stride)
  int alpha_stride;
  T bcoef;
  T inv_drho, inv_dtheta;
  // rho-slab mode (multi-GPU): coefficient row stride / global row offset /
  // global row count, and v carrying 3 halo rows on each side (0 = plain)
  int coef_ld, coef_j0, nr_glob, halo;
  // output row chunk [row_begin, row_end) (row_end 0 = all rows; row_begin a
  // multiple of the CTA's 128 rows)
  int row_begin, row_end;
  StepStamp ts;               // bucket time stamp at kernel entry (march only)
  // TMA staging of the walk tiles (fp64, plain mode): rank-3 tiled map over v
  // (columns, rows, members), box WENO_TMA_BOX x 32 x 1; tma = 0: cp.async
  int tma;
  alignas(64) CUtensorMap vmap;
};
// TMA box width: columns x0-4 .. x0+37 (the inner start coordinate of a tiled
// copy must be 16-byte aligned: x0-3 is not, x0-4 is); 336 B rows
constexpr int WENO_TMA_BOX = 42;

void launch_stamp(unsigned long long* buf, const int* step, int slot, cudaStream_t s);
template <typename T> void launch_theta_c2r(const ThetaArgs<T>& a, int rows, cudaStream_t s);
template <typename T> void launch_theta_r2c(const ThetaArgs<T>& a, int rows, cudaStream_t s);
template <typename T> void launch_rho(const RhoArgs<T>& a, int mode, int threads, cudaStream_t s);
template <typename T> void launch_weno(const WenoArgs<T>& a, cudaStream_t s);
template <typename T>
void launch_alpha_theta(const Geom& g, const T* v, const T* upar, T bcoef, u64* bits,
                        int stride, cudaStream_t s);
template <typename T>
void launch_alpha_rho(const T* uperp, int nr, int rows, double* out, cudaStream_t s);
template <typename T>
void launch_transpose(const Geom& g, const cplx<T>* in, cplx<T>* out, int to_natural,
                      cudaStream_t s);
template <typename T>
void launch_combine(long n, int mode, double ds, const cplx<T>* E, const cplx<T>* P1,
                    const cplx<T>* P12, const cplx<T>* P2, const cplx<T>* vh,
                    const cplx<T>* b1, const cplx<T>* b2, cplx<T>* out, cudaStream_t s);
template <typename T>
void launch_convert(long n, const double* in, T* out, cudaStream_t s);
// metrics.cu: per-member ground metrics (peak, t10, t90) of row `row`, roi [k0, k0+n)
template <typename T>
void launch_ground_metrics(const T* v, int batch, int nr, int nt, int row, int k0, int n,
                           const double* x, double* out, cudaStream_t s);

// splitting.cu (splitting baseline, float64; -fmad=false)
void launch_split_prep(const double* v, int n, int nt, int ldn, double* vT, double* sT,
                       cudaStream_t s);
void launch_split_diffraction(const double* vT, const double* sT, int n, int nt, int ldn,
                              double gamma, const double* w, const double* up, const double* dg,
                              double* out, double* gline, cudaStream_t s);
bool split_line_in_smem(int n);
void launch_split_burgers(const double* v, int n, int nt, double B, double ratio, double* out,
                          cudaStream_t s);
void launch_godunov_flux(long n, const double* ul, const double* ur, double B, double* out,
                         cudaStream_t s);
void launch_split_axial(double2* spec, int n, int kk, int ld, const double* upar, double ds,
                        double A, double theta_span, cudaStream_t s);
void launch_split_transverse(const double* v, int n, int nt, const double* up, const double* dus,
                             const double* dur, double ds, double dr, double* out,
                             unsigned long long* vmax, cudaStream_t s);

// tables.cu (compiled with -fmad=false so the z / exp / phi arithmetic
// rounds like numpy's)
struct TableArgs {
  int nr, nt, kk, ld;
  double rho_span, theta_span, d_sigma, A, eps;
  const int* rev_r;           // position -> frequency (plan layout) or null (natural)
  int natural;                // 1: (nr, kk) row-major frequency order; 0: (kk, ld) digit-reversed
  int k0;                     // first theta mode (theta-mode slab of a multi-GPU run)
};
template <typename T>
void launch_tables(const TableArgs& a, cplx<T>* E, cplx<T>* P1, cplx<T>* P2, cplx<T>* P12,
                   double2* z, cudaStream_t s);
void launch_phi(const double2* z, long n, int shift, double2* out, cudaStream_t s);
// turbulence mode sum (tables.cu); scratch holds 2 (n_sig + n_rho) n_modes doubles
void launch_turbulence(const double* kx, const double* ky, const double* ph, const double* a1,
                       const double* a2, const double* wds, const double* wdr, int n_modes,
                       double lam, double inv_c0, const double* sig, int n_sig, const double* rho,
                       int n_rho, double* scratch, double* u_par, double* u_perp, double* du_ds,
                       double* du_dr, cudaStream_t s);

}  // namespace nwb
