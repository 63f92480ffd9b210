// C ABI and native runtime of the B200 ExpRK22/WENO5 step: plans (device
// tables, twiddles, workspaces), the sigma-march driver (CUDA graphs or
// per-step events, guard and budget checks, snapshots) and the standalone
// entry points that back the Python drop-in API.  See include/nwb200.h.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/nwb200.h"
#include "internal.h"

using namespace nwb;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CU(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(e_ == cudaErrorMemoryAllocation ? NWB_ENOMEM : NWB_ECUDA,            \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                 \
  } while (0)

#define CHECK_LAUNCH(what)                                                             \
  do {                                                                                 \
    cudaError_t e_ = cudaGetLastError();                                               \
    if (e_ != cudaSuccess)                                                             \
      return fail(NWB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e_));       \
  } while (0)

// ---------------------------------------------------------------- FFT plans
// Stage radix sequence and its grouping into passes of one or two fused
// stages (product <= 16 keeps a pass's elements in registers):
// 7 pairs with 2, 5 with 3 or 2, 3 with 4 / 3 / 2, remaining powers of two
// as 4x4 (16), 8, 4, 2.  split_two forces a lone radix-2 first stage (the
// cluster-split rho pass performs it while loading).
struct FftPlanHost {
  std::vector<int> stages;              // radix per stage, DIF order
  std::vector<std::pair<int, int>> passes;  // (ra, rb)
};

// first > 1 forces a lone first stage of that radix (2, 3, 4, 5, 7): the
// cluster-split rho pass (2) and the theta-fused first rho stage (r1).
bool plan_fft(int n, int first, FftPlanHost& h, int max_prod = 16, int pair55 = 0) {
  int m = n, c2 = 0, c3 = 0, c5 = 0, c7 = 0;
  while (m % 2 == 0) { m /= 2; ++c2; }
  while (m % 3 == 0) { m /= 3; ++c3; }
  while (m % 5 == 0) { m /= 5; ++c5; }
  while (m % 7 == 0) { m /= 7; ++c7; }
  if (m != 1) return false;
  const bool big = max_prod >= 16;  // 16: pair 7.2, 5.3, 5.2, 3.4, 3.3, 4.4; 8: only 3.2 and 8
  std::vector<std::pair<int, int>> ps;
  const bool split_two = first > 1;
  if (first > 1) {
    int* cnt = first == 2 || first == 4 ? &c2 : first == 3 ? &c3 : first == 5 ? &c5 : first == 7 ? &c7 : nullptr;
    const int need = first == 4 ? 2 : 1;
    if (!cnt || *cnt < need) return false;
    ps.push_back({first, 1});
    *cnt -= need;
  }
  for (; c7 > 0; --c7) {
    if (big && c2 > 0) { ps.push_back({7, 2}); --c2; } else ps.push_back({7, 1});
  }
  // radix-25 passes (5.5) for the powers of 5 (pair55): one shared-memory round
  // trip and barrier fewer per pair of radix-5 stages
  if (big && pair55)
    for (; c5 >= 2; c5 -= 2) ps.push_back({5, 5});
  for (; c5 > 0; --c5) {
    if (big && c3 > 0) { ps.push_back({5, 3}); --c3; }
    else if (big && c2 > 0) { ps.push_back({5, 2}); --c2; }
    else ps.push_back({5, 1});
  }
  while (c3 > 0) {
    if (big && c2 >= 2) { ps.push_back({3, 4}); c2 -= 2; --c3; }
    else if (big && c3 >= 2) { ps.push_back({3, 3}); c3 -= 2; }
    else if (c2 >= 1) { ps.push_back({3, 2}); --c2; --c3; }
    else { ps.push_back({3, 1}); --c3; }
  }
  // a leftover 8 / 4 / 2 goes first (after a forced split stage), so the last
  // pass -- the one whose unit-stride butterflies set the smem padding -- is
  // as large as possible
  const int group = big ? 4 : 3;
  std::vector<std::pair<int, int>> head;
  const int rem = c2 % group;
  if (rem == 3) head.push_back({8, 1});
  if (rem == 2) head.push_back({4, 1});
  if (rem == 1) head.push_back({2, 1});
  ps.insert(ps.begin() + (split_two ? 1 : 0), head.begin(), head.end());
  for (; c2 >= group; c2 -= group) ps.push_back(big ? std::make_pair(4, 4) : std::make_pair(8, 1));
  if ((int)ps.size() > NWB_MAX_PASSES) return false;
  h.passes = ps;
  h.stages.clear();
  for (auto& q : ps) {
    h.stages.push_back(q.first);
    if (q.second > 1) h.stages.push_back(q.second);
  }
  return true;
}

unsigned magic_for(int d) {
  if (d <= 1) return 0u;
  return (unsigned)((((unsigned long long)1 << 32) + (unsigned long long)d - 1) / (unsigned long long)d);
}

// measurement knob: NWB_PAD=<P> overrides the smem padding period of the
// transform of length NWB_PAD_N
static int pad_env_n() {
  const char* e = std::getenv("NWB_PAD_N");
  return e ? std::atoi(e) : -1;
}

// simulated shared-memory wavefronts of all passes for padding period P
// (lane g of a pass handles butterfly g; element e at slot e + e / P)
static double pad_cost(int n, const FftPlanHost& h, int P) {
  long waves = 0, ideal = 0;
  int L = n;
  for (auto& ps : h.passes) {
    const int ra = ps.first, rb = ps.second, R = ra * rb;
    const int sa = L / ra, sb = sa / rb, total = (n / L) * sb;
    for (int w0 = 0; w0 < total; w0 += 32)
      for (int k = 0; k < R; ++k)
        for (int q = w0; q < std::min(w0 + 32, total); q += 8) {
          int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, mx = 0;
          for (int g = q; g < std::min(q + 8, total); ++g) {
            const int blk = g / sb, i = g - blk * sb;
            const int e = blk * L + i + (k / rb) * sa + (k % rb) * sb;
            const int slot = P ? e + e / P : e;
            mx = std::max(mx, ++cnt[slot & 7]);
          }
          waves += mx;
          ++ideal;
        }
    L /= R;
  }
  return ideal ? (double)waves / (double)ideal : 1.0;
}

static int choose_pad(int n, const FftPlanHost& h) {
  std::vector<int> cand = {0};
  for (int P = 8; P <= 256 && P < n; P += 8) cand.push_back(P);
  const int last = h.passes.empty() ? 1 : h.passes.back().first * h.passes.back().second;
  if (last % 2 == 0 && last < n) cand.push_back(last);
  int best = 0;
  double best_cost = 1e30;
  for (int P : cand) {
    const double c = pad_cost(n, h, P);
    if (c < best_cost - 1e-9) {
      best_cost = c;
      best = P;
    }
  }
  return best;
}

// device descriptor + per-stage twiddle tables W_L^{q i} laid out [q-1][i]
template <typename T>
void build_desc(int n, const FftPlanHost& h, FftDesc& d, std::vector<cplx<T>>& tw) {
  const long double pi = 3.141592653589793238462643383279502884L;
  std::vector<int> span, ofs, fin;
  tw.clear();
  auto push_w = [&](long long t, int L) {
    const long double a = 2.0L * pi * (long double)(t % L) / (long double)L;
    cplx<T> w;
    w.x = (T)cosl(a);
    w.y = (T)-sinl(a);
    tw.push_back(w);
  };
  int L = n;
  for (int r : h.stages) {
    // two-level table of W_L^i, i < s: coarse W_L^{64 c}, fine W_L^f
    span.push_back(L);
    const int s = L / r;
    ofs.push_back((int)tw.size());
    for (int c = 0; c < (s + 63) / 64; ++c) push_w(64LL * c, L);
    fin.push_back((int)tw.size());
    for (int f = 0; f < 64; ++f) push_w(f, L);
    L = s;
  }
  if (tw.empty()) tw.push_back(cplx<T>{1, 0});
  std::memset(&d, 0, sizeof(d));
  d.n = n;
  d.np = (int)h.passes.size();
  int st = 0;
  for (int p = 0; p < d.np; ++p) {
    const int ra = h.passes[p].first, rb = h.passes[p].second;
    d.ptype[p] = 10 * ra + rb;
    d.pspan[p] = span[st];
    d.pofs_a[p] = ofs[st];
    d.pfin_a[p] = fin[st];
    d.pofs_b[p] = rb > 1 ? ofs[st + 1] : 0;
    d.pfin_b[p] = rb > 1 ? fin[st + 1] : 0;
    const int sb = span[st] / ra / rb;
    d.pmag_row[p] = magic_for(n / (ra * rb));
    d.pmag_sb[p] = magic_for(sb);
    st += rb > 1 ? 2 : 1;
  }
  // pad the smem line every P elements: P is chosen by simulating the
  // shared-memory wavefronts of every pass (16-byte accesses are served 8
  // lanes at a time; a wavefront per distinct 16-byte bank group), over
  // P = 0, multiples of 8 (which keep the unit-stride load / store loops
  // conflict free) and the size of the last pass
  d.pad_period = choose_pad(n, h);
  if (const char* env = std::getenv(n == pad_env_n() ? "NWB_PAD" : "NWB_PAD_OTHER")) d.pad_period = std::atoi(env);
  if ((size_t)padded_len(n, d.pad_period) * sizeof(cplx<T>) > 227u * 1024u) d.pad_period = 0;
  d.pad_magic = d.pad_period ? magic_for(d.pad_period) : 0u;
  d.sym_r1 = h.stages.empty() ? 0 : h.stages[0];
  if (const char* env = std::getenv("NWB_RHO_SYM")) if (env[0] == '0') d.sym_r1 = 0;  // measurement knob
  d.sym_m = d.sym_r1 > 0 ? n / d.sym_r1 : n;
  d.sym_magic = d.sym_r1 > 0 && d.sym_m > 1 ? magic_for(d.sym_m) : 0u;
  d.sym_n = d.sym_r1 > 1 ? d.sym_m + (d.sym_r1 - 1) / 2 * d.sym_m + (d.sym_r1 % 2 == 0 ? (d.sym_m + 1) / 2 : 0) : n;
  st = 0;
  for (int p = 0; p < d.np; ++p) {
    const int ra = h.passes[p].first, rb = h.passes[p].second;
    const int sa = span[st] / ra, sb = sa / rb;
    const int P2 = d.pad_period;
    d.pfast[p] = P2 == 0 || sb % P2 == 0;
    d.psa_p[p] = P2 ? sa + sa / P2 : sa;
    d.psb_p[p] = P2 ? sb + sb / P2 : sb;
    st += rb > 1 ? 2 : 1;
  }
}

// position after a full DIF -> frequency
std::vector<int> freq_of_pos(int n, const std::vector<int>& stages) {
  std::vector<int> f(n);
  for (int p = 0; p < n; ++p) {
    int rem = p, ff = 0, mult = 1, L = n;
    for (int r : stages) {
      const int s = L / r;
      const int q = rem / s;
      rem -= q * s;
      ff += q * mult;
      mult *= r;
      L = s;
    }
    f[p] = ff;
  }
  return f;
}

// W_n^t = exp(-2 pi i t / n) in extended precision, t < count
template <typename T> std::vector<cplx<T>> twiddles(int n, int count) {
  std::vector<cplx<T>> w(count);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int t = 0; t < count; ++t) {
    const long double a = 2.0L * pi * (long double)t / (long double)n;
    w[t].x = (T)cosl(a);
    w[t].y = (T)-sinl(a);
  }
  return w;
}

}  // namespace

struct nwb_plan {
  int device = 0;
  cudaStream_t stream = 0;
  cudaStream_t own_stream = 0;  // used when the caller sets none (graphs cannot capture the legacy stream)
  // WENO / r2c overlap: the r2c of row chunk c runs on `side` while the WENO of
  // chunk c+1 runs on `stream` (fork / join events; captured into the step graph)
  int overlap_chunks = 0;
  cudaStream_t side = 0;
  cudaEvent_t ov_ev[9] = {};
  int prec = NWB_F64;
  Geom g{};
  double d_sigma = 0, rho_span = 0, theta_span = 0, A = 0, B = 0, eps = 0;
  FftDesc dr{}, dh{};
  FftPlanHost plan_r, plan_h;
  int theta_rows = 1, rho_threads = 256;
  int theta_rows_c2r = 1;    // c2r (transposed reads) favours many small CTAs for long rows
  int theta_stream_rows = 0;  // R of the streaming theta kernels (0 = not used)
  int rho_split = 0;         // 2-CTA cluster per rho column (large fp64 columns)
  int rho_half = 0;          // k_rho_half: half-resident columns, two per SM (NWB_RHO_HALF)
  int rho_prefetch = 0;      // bulk L2 prefetch of combine operands, percent of each row (NWB_RHO_PREFETCH)
  int rho_next_pf = 0;       // L2 prefetch of column k + rho_next_pf's input (NWB_RHO_NEXTPF)
  int rho_roll = 0;          // combine: L2 prefetch of the operands rho_roll rounds ahead (NWB_RHO_ROLL)
  int rho_debug = 0;
  int rho_stagger_ns = 0, rho_stagger_mode = 0;  // NWB_RHO_STAGGER=<ns>[,<mode>]
  int rho_bulk = 0;          // fp64 column load / store by TMA bulk copies (NWB_RHO_BULK)
  int theta_bulk = 0;        // fp64 r2c row loads by TMA bulk copies (NWB_THETA_BULK)
  int theta_debug = 0;       // NWB_THETA_DEBUG (never set in production)         // NWB_RHO_DEBUG measurement knobs (never set in production)
  int rho_persistent = 0;    // persistent streaming rho pass (NWB_RHO_PERSIST=1 enables; measured slower)
  int rho_ws = 0, rho_ws2 = 0, rho_ws_ctas = 0;  // warp-specialised rho pass (k_rho_ws) group sizes, CTAs
  void* ws_scratch = nullptr;
  // WENO walk tiles staged by TMA (fp64): tiled tensor map over v (NWB_WENO_TMA=0: cp.async)
  int weno_tma = 0;
  alignas(64) CUtensorMap vmap;
  // first rho stage fused into the theta passes (r1 > 1): rho CTAs own
  // msub = nr / r1 point sub-columns (dsub / tw_sub); tw_first = W_nr^t
  int rho_r1 = 1, msub = 0, ilv = 1;
  FftDesc dsub{};
  void *tw_sub = nullptr, *tw_first = nullptr;
  FftDesc dh2{};             // half-column descriptor (split mode)
  void *tw_h2 = nullptr, *tw_split = nullptr;
  size_t rsz = 8;  // sizeof(real)
  // device buffers
  void *tw_r = nullptr, *tw_h = nullptr, *wk = nullptr;
  int *pos_r = nullptr, *rev_r = nullptr, *pos_h = nullptr;
  void *vh = nullptr, *u = nullptr, *t = nullptr, *ts = nullptr, *bt = nullptr;
  void *v = nullptr, *b = nullptr;
  void *E = nullptr, *P1 = nullptr, *P12 = nullptr, *P2 = nullptr;
  void *upar = nullptr, *uperp = nullptr, *du = nullptr;
  double* alpha_rho = nullptr;
  int n_rows = 0;
  u64* red = nullptr;        // [batch][4]: alpha stage 1, alpha stage 2, scratch, scratch
  u64* vmax_hist = nullptr;  // [batch][hist_len]
  int hist_len = 0;
  int* step_ctr = nullptr;
  long long bytes = 0;
  // graphs (one captured step per scheme)
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  cudaStream_t graph_stream[2] = {nullptr, nullptr};
  // per-step bucket time stamps [hist_len + 1][NWB_TS_SLOTS] (internal.h
  // StepStamp): written by the march kernels themselves, so the timed default
  // path replays the same graph as the untimed one
  unsigned long long* stamps = nullptr;
  std::vector<void*> allocs;
};

namespace {

// Workspaces come from the device's stream-ordered memory pool with an
// unbounded release threshold: destroying a plan returns its gigabytes to the
// pool without a device-wide synchronising cudaFree, and the next plan of the
// same size is served from the pool (plan churn in studies costs ~nothing).
void keep_pool_memory(int device) {
  static bool done[64] = {false};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    unsigned long long thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[device] = true;
}

int dalloc(nwb_plan* p, void** ptr, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMallocAsync(ptr, bytes, p->stream);
  if (e != cudaSuccess) {
    *ptr = nullptr;
    return fail(e == cudaErrorMemoryAllocation ? NWB_ENOMEM : NWB_ECUDA,
                std::string("cudaMallocAsync(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  }
  p->allocs.push_back(*ptr);
  p->bytes += (long long)bytes;
  return NWB_OK;
}

void dfree(nwb_plan* p, void* ptr) {
  if (!ptr) return;
  cudaFreeAsync(ptr, p->stream);
  for (auto& x : p->allocs)
    if (x == ptr) x = nullptr;
}

#define TRY(x)                 \
  do {                         \
    int rc_ = (x);             \
    if (rc_ != NWB_OK) return rc_; \
  } while (0)

template <typename T> ThetaArgs<T> theta_args(const nwb_plan* p) {
  ThetaArgs<T> a{};
  a.g = p->g;
  a.dh = p->dh;
  a.tw_h = (const cplx<T>*)p->tw_h;
  a.wk = (const cplx<T>*)p->wk;
  a.pos_h = p->pos_h;
  a.scale = (T)(1.0 / ((double)p->g.nr * (double)p->g.nt));
  a.bcoef = (T)p->B;
  a.alpha_stride = 4;
  a.vmax_stride = p->hist_len;
  a.debug = p->theta_debug;
  a.r1 = p->rho_r1;
  a.msub = p->msub;
  a.tw_first = (const cplx<T>*)p->tw_first;
  a.ilv = p->ilv;
  a.bulk = p->theta_bulk;
  return a;
}

template <typename T> RhoArgs<T> rho_args(const nwb_plan* p) {
  RhoArgs<T> a{};
  a.g = p->g;
  a.dr = p->dr;
  a.tw_r = (const cplx<T>*)p->tw_r;
  a.pos_r = p->pos_r;
  a.vh = (cplx<T>*)p->vh;
  a.u = (cplx<T>*)p->u;
  a.E = (const cplx<T>*)p->E;
  a.P1 = (const cplx<T>*)p->P1;
  a.P12 = (const cplx<T>*)p->P12;
  a.P2 = (const cplx<T>*)p->P2;
  a.ds = (T)p->d_sigma;
  a.zero_stride = 4;
  a.split = p->rho_split;
  a.half = p->rho_half;
  a.prefetch = p->rho_prefetch;
  a.next_pf = p->rho_next_pf;
  a.debug = p->rho_debug;
  a.persistent = p->rho_persistent;
  a.ws_threads = p->rho_ws;
  a.ws_threads2 = p->rho_ws2;
  a.ws_ctas = p->rho_ws_ctas;
  a.roll = p->rho_roll;
  a.bulk = p->rho_bulk;
  a.stagger_ns = p->rho_stagger_ns;
  a.stagger_mode = p->rho_stagger_mode;
  {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    a.stagger_slots = sms > 0 ? sms : 148;
  }
  if (const char* env = std::getenv("NWB_RHO_WS_DEBUG")) a.ws_debug = std::atoi(env);
  a.scratch = (cplx<T>*)p->ws_scratch;
  a.dh2 = p->dh2;
  a.tw_h2 = (const cplx<T>*)p->tw_h2;
  a.tw_split = (const cplx<T>*)p->tw_split;
  a.r1 = p->rho_r1;
  a.ilv = p->ilv;
  a.dsub = p->dsub;
  a.tw_sub = (const cplx<T>*)p->tw_sub;
  a.rev_r = p->rev_r;
  return a;
}

template <typename T> WenoArgs<T> weno_args(const nwb_plan* p) {
  WenoArgs<T> a{};
  a.g = p->g;
  a.v = (const T*)p->v;
  a.out = (T*)p->b;
  a.upar = (const T*)p->upar;
  a.uperp = (const T*)p->uperp;
  a.du = (const T*)p->du;
  a.alpha_rho = p->alpha_rho;
  a.alpha_stride = 4;
  a.bcoef = (T)p->B;
  a.inv_drho = (T)(1.0 / (p->rho_span / p->g.nr));
  a.inv_dtheta = (T)(1.0 / (p->theta_span / p->g.nt));
  a.tma = p->weno_tma;
  if (p->weno_tma) a.vmap = p->vmap;
  return a;
}

// One stage of the fused pipeline: c2r(+alpha, +vmax) -> WENO -> r2c -> rho pass.
// ev (optional) holds 5 events: before c2r and after each of the 4 kernels.
constexpr int EV_PER_STAGE = 5;

inline void rec_event(cudaEvent_t e, cudaStream_t s) {
  if (e) cudaEventRecord(e, s);
}

// bucket stamp of a march launch (slots: internal.h StepStamp); slot < 0: none
inline StepStamp stamp_of(const nwb_plan* p, int slot) {
  return StepStamp{slot >= 0 ? p->stamps : nullptr, p->step_ctr, slot < 0 ? 0 : slot};
}

template <typename T>
void launch_stage(nwb_plan* p, int stage, int scheme, cudaEvent_t* ev) {
  cudaStream_t s = p->stream;
  if (ev) rec_event(ev[0], s);
  // theta c2r of T (stage 1) or T* (stage 2) into v
  ThetaArgs<T> c = theta_args<T>(p);
  c.spec_in = (const cplx<T>*)(stage == 1 ? p->t : p->ts);
  c.phys_out = (T*)p->v;
  c.upar = (const T*)p->upar;
  c.step_ctr = p->step_ctr;
  c.row_off = stage - 1;
  c.alpha_bits = p->red + (stage - 1);
  c.vmax_bits = stage == 1 ? p->vmax_hist : nullptr;
  c.ts = stamp_of(p, stage == 1 ? 0 : -1);
  launch_theta_c2r<T>(c, p->theta_stream_rows ? -p->theta_stream_rows : p->theta_rows_c2r, s);
  if (ev) rec_event(ev[1], s);
  // WENO -> b
  WenoArgs<T> w = weno_args<T>(p);
  w.step_ctr = p->step_ctr;
  w.row_off = stage - 1;
  w.alpha_bits = p->red + (stage - 1);
  w.ts = stamp_of(p, stage == 1 ? 1 : 3);
  // theta r2c of b -> bt
  ThetaArgs<T> r = theta_args<T>(p);
  r.phys_in = (const T*)p->b;
  r.spec_out = (cplx<T>*)p->bt;
  r.ts = stamp_of(p, stage == 1 ? 2 : 4);
  const int nc = p->overlap_chunks;
  if (!ev && nc > 1 && !p->theta_stream_rows) {
    // row chunks of 128-row multiples: WENO(c+1) on `s` overlaps r2c(c) on `side`
    const int per = ((p->g.nr + nc - 1) / nc + 127) / 128 * 128;
    int c = 0;
    for (int j = 0; j < p->g.nr; j += per, ++c) {
      const int je = j + per < p->g.nr ? j + per : p->g.nr;
      w.row_begin = j;
      w.row_end = je;
      launch_weno<T>(w, s);
      cudaEventRecord(p->ov_ev[c], s);
      cudaStreamWaitEvent(p->side, p->ov_ev[c], 0);
      r.row_begin = j;
      r.row_end = je;
      launch_theta_r2c<T>(r, p->theta_rows, p->side);
      w.ts.buf = r.ts.buf = nullptr;  // the first chunk stamps the bucket
    }
    cudaEventRecord(p->ov_ev[8], p->side);
    cudaStreamWaitEvent(s, p->ov_ev[8], 0);
  } else {
    launch_weno<T>(w, s);
    if (ev) rec_event(ev[2], s);
    launch_theta_r2c<T>(r, p->theta_stream_rows ? -p->theta_stream_rows : p->theta_rows, s);
  }
  if (ev) rec_event(ev[3], s);
  // rho pass
  RhoArgs<T> q = rho_args<T>(p);
  q.in = (const cplx<T>*)p->bt;
  int mode;
  if (scheme == NWB_SCHEME_EXPEULER) {
    mode = RHO_EULER;
    q.out = (cplx<T>*)p->t;
    q.step_ctr = p->step_ctr;
    q.zero_bits = p->red + 0;
  } else if (stage == 1) {
    mode = RHO_STAGE1;
    q.out = (cplx<T>*)p->ts;
    q.zero_bits = p->red + 1;
  } else {
    mode = RHO_STAGE2;
    q.out = (cplx<T>*)p->t;
    q.step_ctr = p->step_ctr;
    q.zero_bits = p->red + 0;
  }
  launch_rho<T>(q, mode, p->rho_threads, s);
  if (ev) rec_event(ev[4], s);
}

// ev (optional): 2 * EV_PER_STAGE events
template <typename T> void launch_step(nwb_plan* p, int scheme, cudaEvent_t* ev) {
  launch_stage<T>(p, 1, scheme, ev);
  if (scheme == NWB_SCHEME_EXPRK22) launch_stage<T>(p, 2, scheme, ev ? ev + EV_PER_STAGE : nullptr);
}

void drop_graphs(nwb_plan* p) {
  for (int i = 0; i < 2; ++i) {
    if (p->graph[i]) cudaGraphExecDestroy(p->graph[i]);
    p->graph[i] = nullptr;
  }
}

// per-step guard history [batch][len]; reallocation invalidates captured graphs
int ensure_hist(nwb_plan* p, int len) {
  if (p->hist_len >= len && p->vmax_hist) return NWB_OK;
  dfree(p, p->vmax_hist);
  dfree(p, p->stamps);
  p->vmax_hist = nullptr;
  p->stamps = nullptr;
  p->hist_len = len;
  TRY(dalloc(p, (void**)&p->vmax_hist, (size_t)p->g.batch * len * sizeof(u64)));
  CU(cudaMemsetAsync(p->vmax_hist, 0, (size_t)p->g.batch * len * sizeof(u64), p->stream));
  TRY(dalloc(p, (void**)&p->stamps, (size_t)(len + 1) * NWB_TS_SLOTS * sizeof(u64)));
  drop_graphs(p);
  return NWB_OK;
}

int set_step(nwb_plan* p, int n) {
  CU(cudaMemcpyAsync(p->step_ctr, &n, sizeof(int), cudaMemcpyHostToDevice, p->stream));
  CU(cudaStreamSynchronize(p->stream));
  return NWB_OK;
}

int check_plan(nwb_plan* p) {
  if (!p) return fail(NWB_EINVAL, "null plan");
  CU(cudaSetDevice(p->device));
  return NWB_OK;
}

// Tiled tensor map over an fp64 field (nt columns, nr rows, batch members) whose
// box is one WENO walk tile (WENO_TMA_BOX x 32 x 1).  cuTensorMapEncodeTiled
// comes from the driver through the runtime's entry-point query, so the library
// links against cudart only.  Returns 1 when the map is usable (row pitch a
// multiple of 16 bytes, grid at least one tile), else 0: cp.async staging.
int make_weno_vmap(CUtensorMap& map, const void* v, int nt, int nr, int batch) {
  if (const char* env = std::getenv("NWB_WENO_TMA"))  // measurement knob
    if (env[0] == '0') return 0;
  if (nt % 2 || nt < 64 || nr < 32 || ((uintptr_t)v & 15)) return 0;
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return 0;
    }
    encode = (EncodeFn)fn;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)nt, (cuuint64_t)nr, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)nt * 8, (cuuint64_t)nt * nr * 8};
  const cuuint32_t box[3] = {(cuuint32_t)WENO_TMA_BOX, 32, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(v), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 1 : 0;
}

template <typename T> int create_impl(nwb_plan* p) {
  const Geom& g = p->g;
  const size_t C = sizeof(cplx<T>);
  const size_t spec = (size_t)g.batch * g.kk * g.ld * C;
  const size_t phys = (size_t)g.batch * g.nr * g.nt * sizeof(T);
  const size_t tab = (size_t)g.kk * g.ld * C;
  TRY(dalloc(p, &p->vh, spec));
  TRY(dalloc(p, &p->u, spec));
  TRY(dalloc(p, &p->t, spec));
  TRY(dalloc(p, &p->ts, spec));
  TRY(dalloc(p, &p->bt, spec));
  TRY(dalloc(p, &p->v, phys));
  TRY(dalloc(p, &p->b, phys));
  if (sizeof(T) == 8) p->weno_tma = make_weno_vmap(p->vmap, p->v, g.nt, g.nr, g.batch);
  TRY(dalloc(p, &p->E, tab));
  TRY(dalloc(p, &p->P1, tab));
  TRY(dalloc(p, &p->P12, tab));
  TRY(dalloc(p, &p->P2, tab));
  TRY(dalloc(p, (void**)&p->red, (size_t)g.batch * 4 * sizeof(u64)));
  TRY(dalloc(p, (void**)&p->step_ctr, sizeof(int)));
  if (p->rho_ws > 0) TRY(dalloc(p, &p->ws_scratch, (size_t)p->rho_ws_ctas * 2 * g.ld * C));
  CU(cudaMemsetAsync(p->red, 0, (size_t)g.batch * 4 * sizeof(u64), p->stream));
  CU(cudaMemsetAsync(p->step_ctr, 0, sizeof(int), p->stream));
  // zero the padding columns once so nothing uninitialised is ever read
  for (void* a : {p->vh, p->u, p->t, p->ts, p->bt}) CU(cudaMemsetAsync(a, 0, spec, p->stream));

  // twiddles and digit-reversal maps
  std::vector<cplx<T>> twr, twh;
  build_desc<T>(g.nr, p->plan_r, p->dr, twr);
  build_desc<T>(g.m, p->plan_h, p->dh, twh);
  // march theta passes: persistent double-buffered kernels (NWB_THETA_STREAM=1;
  // measured slower than one-shot CTAs at Set 4, so off by default)
  p->theta_stream_rows = 0;
  {
    const char* env = std::getenv("NWB_THETA_STREAM");
    if (env && env[0] == '1')
      for (int r : {8, 4, 2, 1})
        if (2 * (size_t)r * padded_len(g.m, p->dh.pad_period) * C <= 200 * 1024 && r <= g.nr) {
          p->theta_stream_rows = r;
          break;
        }
  }
  auto wk = twiddles<T>(g.nt, g.kk);
  auto fr = freq_of_pos(g.nr, p->plan_r.stages);
  std::vector<int> pr(g.nr);
  for (int q = 0; q < g.nr; ++q) pr[fr[q]] = q;
  auto fh = freq_of_pos(g.m, p->plan_h.stages);
  std::vector<int> ph(g.m);
  for (int q = 0; q < g.m; ++q) ph[fh[q]] = q;
  TRY(dalloc(p, &p->tw_r, twr.size() * C));
  TRY(dalloc(p, &p->tw_h, twh.size() * C));
  TRY(dalloc(p, &p->wk, wk.size() * C));
  TRY(dalloc(p, (void**)&p->pos_r, pr.size() * sizeof(int)));
  TRY(dalloc(p, (void**)&p->rev_r, fr.size() * sizeof(int)));
  TRY(dalloc(p, (void**)&p->pos_h, ph.size() * sizeof(int)));
  CU(cudaMemcpy(p->tw_r, twr.data(), twr.size() * C, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(p->tw_h, twh.data(), twh.size() * C, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(p->wk, wk.data(), wk.size() * C, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(p->pos_r, pr.data(), pr.size() * sizeof(int), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(p->rev_r, fr.data(), fr.size() * sizeof(int), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(p->pos_h, ph.data(), ph.size() * sizeof(int), cudaMemcpyHostToDevice));
  if (p->rho_split || p->rho_half) {
    // half transform = the full plan without its leading radix-2 stage
    FftPlanHost half;
    half.stages.assign(p->plan_r.stages.begin() + 1, p->plan_r.stages.end());
    half.passes.assign(p->plan_r.passes.begin() + 1, p->plan_r.passes.end());
    std::vector<cplx<T>> tw2;
    build_desc<T>(g.nr / 2, half, p->dh2, tw2);
    if (p->rho_split) p->dh2.sym_r1 = 0;  // the split kernel reads its own half of each table row
    auto tws = twiddles<T>(g.nr, g.nr / 2);
    TRY(dalloc(p, &p->tw_h2, tw2.size() * C));
    TRY(dalloc(p, &p->tw_split, tws.size() * C));
    CU(cudaMemcpy(p->tw_h2, tw2.data(), tw2.size() * C, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(p->tw_split, tws.data(), tws.size() * C, cudaMemcpyHostToDevice));
  }

  if (p->rho_r1 > 1) {
    // sub-column transform = the full plan without its leading radix-r1 stage
    FftPlanHost sub;
    sub.stages.assign(p->plan_r.stages.begin() + 1, p->plan_r.stages.end());
    sub.passes.assign(p->plan_r.passes.begin() + 1, p->plan_r.passes.end());
    std::vector<cplx<T>> tws;
    build_desc<T>(p->msub, sub, p->dsub, tws);
    auto twf = twiddles<T>(g.nr, g.nr);
    TRY(dalloc(p, &p->tw_sub, tws.size() * C));
    TRY(dalloc(p, &p->tw_first, twf.size() * C));
    CU(cudaMemcpy(p->tw_sub, tws.data(), tws.size() * C, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(p->tw_first, twf.data(), twf.size() * C, cudaMemcpyHostToDevice));
  }

  // multiplier tables, digit-reversed rho order (exprk.py:111-131)
  TableArgs ta{};
  ta.nr = g.nr; ta.nt = g.nt; ta.kk = g.kk; ta.ld = g.ld;
  ta.rho_span = p->rho_span; ta.theta_span = p->theta_span;
  ta.d_sigma = p->d_sigma; ta.A = p->A; ta.eps = p->eps;
  ta.rev_r = p->rev_r; ta.natural = 0;
  CU(cudaMemsetAsync(p->E, 0, tab, p->stream));
  CU(cudaMemsetAsync(p->P1, 0, tab, p->stream));
  CU(cudaMemsetAsync(p->P12, 0, tab, p->stream));
  CU(cudaMemsetAsync(p->P2, 0, tab, p->stream));
  launch_tables<T>(ta, (cplx<T>*)p->E, (cplx<T>*)p->P1, (cplx<T>*)p->P2, (cplx<T>*)p->P12,
                   nullptr, p->stream);
  CHECK_LAUNCH("tables");
  CU(cudaStreamSynchronize(p->stream));
  return NWB_OK;
}

template <typename T> int set_coeffs_impl(nwb_plan* p, const double* up, const double* uq,
                                          const double* du, int n_rows, int ld, int on_dev) {
  const Geom& g = p->g;
  const size_t n = (size_t)n_rows * g.nr;
  for (void* a : {p->upar, p->uperp, p->du, (void*)p->alpha_rho}) dfree(p, a);
  p->upar = p->uperp = p->du = nullptr;
  p->alpha_rho = nullptr;
  TRY(dalloc(p, &p->upar, n * sizeof(T)));
  TRY(dalloc(p, &p->uperp, n * sizeof(T)));
  TRY(dalloc(p, &p->du, n * sizeof(T)));
  TRY(dalloc(p, (void**)&p->alpha_rho, (size_t)n_rows * sizeof(double)));
  p->n_rows = n_rows;
  drop_graphs(p);  // captured steps point at the old coefficient buffers
  TRY(ensure_hist(p, n_rows));
  double* stage = nullptr;
  CU(cudaMallocAsync(&stage, n * sizeof(double), p->stream));
  const double* srcs[3] = {up, uq, du};
  void* dsts[3] = {p->upar, p->uperp, p->du};
  for (int i = 0; i < 3; ++i) {
    if (!srcs[i]) {
      cudaMemsetAsync(dsts[i], 0, n * sizeof(T), p->stream);
      continue;
    }
    cudaMemcpy2DAsync(stage, g.nr * sizeof(double), srcs[i], (size_t)ld * sizeof(double),
                      g.nr * sizeof(double), n_rows,
                      on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, p->stream);
    launch_convert<T>((long)n, stage, (T*)dsts[i], p->stream);
  }
  launch_alpha_rho<T>((const T*)p->uperp, g.nr, n_rows, p->alpha_rho, p->stream);
  cudaFreeAsync(stage, p->stream);
  cudaError_t e = cudaStreamSynchronize(p->stream);
  if (e != cudaSuccess) return fail(NWB_ECUDA, std::string("set_coeffs: ") + cudaGetErrorString(e));
  CHECK_LAUNCH("set_coeffs");
  return NWB_OK;
}

template <typename T> int load_physical_impl(nwb_plan* p, const void* v0) {
  ThetaArgs<T> r = theta_args<T>(p);
  r.phys_in = (const T*)v0;
  r.spec_out = (cplx<T>*)p->bt;
  launch_theta_r2c<T>(r, p->theta_rows, p->stream);
  RhoArgs<T> q = rho_args<T>(p);
  q.in = (const cplx<T>*)p->bt;
  q.out = (cplx<T>*)p->t;
  launch_rho<T>(q, RHO_INIT, p->rho_threads, p->stream);
  CHECK_LAUNCH("load_physical");
  return NWB_OK;
}

template <typename T> int load_spectrum_impl(nwb_plan* p, const void* vhat) {
  launch_transpose<T>(p->g, (const cplx<T>*)vhat, (cplx<T>*)p->bt, 0, p->stream);
  RhoArgs<T> q = rho_args<T>(p);
  q.in = (const cplx<T>*)p->bt;
  q.out = (cplx<T>*)p->t;
  launch_rho<T>(q, RHO_INV_NAT, p->rho_threads, p->stream);
  CHECK_LAUNCH("load_spectrum");
  return NWB_OK;
}

template <typename T> int store_spectrum_impl(nwb_plan* p, void* out) {
  RhoArgs<T> q = rho_args<T>(p);
  q.in = (const cplx<T>*)p->vh;
  q.out = (cplx<T>*)p->bt;
  launch_rho<T>(q, RHO_REV2NAT, p->rho_threads, p->stream);
  launch_transpose<T>(p->g, (const cplx<T>*)p->bt, (cplx<T>*)out, 1, p->stream);
  CHECK_LAUNCH("store_spectrum");
  return NWB_OK;
}

template <typename T> int c2r_out(nwb_plan* p, const void* spec, void* out, double* max_abs) {
  ThetaArgs<T> c = theta_args<T>(p);
  c.spec_in = (const cplx<T>*)spec;
  c.phys_out = (T*)out;
  if (max_abs) {
    CU(cudaMemsetAsync(p->red, 0, (size_t)p->g.batch * 4 * sizeof(u64), p->stream));
    c.vmax_bits = p->red + 2;  // slot 2 per member (stride 4, step 0)
    c.vmax_stride = 4;
  }
  launch_theta_c2r<T>(c, p->theta_rows_c2r, p->stream);
  CHECK_LAUNCH("c2r");
  if (max_abs) {
    std::vector<u64> h((size_t)p->g.batch * 4);
    CU(cudaMemcpyAsync(h.data(), p->red, h.size() * sizeof(u64), cudaMemcpyDeviceToHost, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    for (int i = 0; i < p->g.batch; ++i) {
      double d;
      std::memcpy(&d, &h[(size_t)i * 4 + 2], sizeof(double));
      max_abs[i] = d;
    }
    CU(cudaMemsetAsync(p->red, 0, (size_t)p->g.batch * 4 * sizeof(u64), p->stream));
  }
  return NWB_OK;
}

template <typename T> int rfft2_impl(nwb_plan* p, const void* in, void* out) {
  ThetaArgs<T> r = theta_args<T>(p);
  r.phys_in = (const T*)in;
  r.spec_out = (cplx<T>*)p->bt;
  launch_theta_r2c<T>(r, p->theta_rows, p->stream);
  RhoArgs<T> q = rho_args<T>(p);
  q.in = (const cplx<T>*)p->bt;
  q.out = (cplx<T>*)p->ts;
  if (p->rho_r1 > 1) {
    // sub-column transforms in digit-reversed positions, then one permutation
    launch_rho<T>(q, RHO_FWD_DR, p->rho_threads, p->stream);
    q.in = (const cplx<T>*)p->ts;
    q.out = (cplx<T>*)p->bt;
    q.r1 = 1;
    launch_rho<T>(q, RHO_REV2NAT, p->rho_threads, p->stream);
    launch_transpose<T>(p->g, (const cplx<T>*)p->bt, (cplx<T>*)out, 1, p->stream);
  } else {
    launch_rho<T>(q, RHO_FWD_NAT, p->rho_threads, p->stream);
    launch_transpose<T>(p->g, (const cplx<T>*)p->ts, (cplx<T>*)out, 1, p->stream);
  }
  CHECK_LAUNCH("rfft2");
  return NWB_OK;
}

template <typename T> int irfft2_impl(nwb_plan* p, const void* in, void* out) {
  launch_transpose<T>(p->g, (const cplx<T>*)in, (cplx<T>*)p->bt, 0, p->stream);
  RhoArgs<T> q = rho_args<T>(p);
  q.in = (const cplx<T>*)p->bt;
  q.out = (cplx<T>*)p->ts;
  q.vh = nullptr;
  launch_rho<T>(q, RHO_INV_NAT, p->rho_threads, p->stream);
  CHECK_LAUNCH("irfft2");
  return c2r_out<T>(p, p->ts, out, nullptr);
}

// workspace: [batch] u64 alpha_theta bits followed by one double alpha_rho
template <typename T> int weno_impl(const Geom& g, const void* v, const void* up, const void* uq,
                                    const void* du, double b, double d_rho, double d_theta,
                                    void* out, void* ws, cudaStream_t s) {
  u64* abits = (u64*)ws;
  double* arho = (double*)(abits + g.batch);
  CU(cudaMemsetAsync(abits, 0, (size_t)g.batch * sizeof(u64), s));
  launch_alpha_theta<T>(g, (const T*)v, (const T*)up, (T)b, abits, 1, s);
  launch_alpha_rho<T>((const T*)uq, g.nr, 1, arho, s);
  WenoArgs<T> w{};
  w.g = g;
  w.v = (const T*)v;
  w.out = (T*)out;
  w.upar = (const T*)up;
  w.uperp = (const T*)uq;
  w.du = (const T*)du;
  w.alpha_rho = arho;
  w.step_ctr = nullptr;
  w.row_off = 0;
  w.alpha_bits = abits;
  w.alpha_stride = 1;
  w.bcoef = (T)b;
  w.inv_drho = (T)(1.0 / d_rho);
  w.inv_dtheta = (T)(1.0 / d_theta);
  if (sizeof(T) == 8) w.tma = make_weno_vmap(w.vmap, v, g.nt, g.nr, g.batch);

  launch_weno<T>(w, s);
  CHECK_LAUNCH("weno5_b");
  return NWB_OK;
}

template <typename T> int step_impl(nwb_plan* p, int scheme, cudaEvent_t* ev) {
  launch_step<T>(p, scheme, ev);
  CHECK_LAUNCH("step");
  return NWB_OK;
}

template <typename T> int graph_for(nwb_plan* p, int scheme) {
  const int gi = scheme == NWB_SCHEME_EXPRK22 ? 0 : 1;
  if (p->graph[gi] && p->graph_stream[gi] == p->stream) return NWB_OK;
  if (p->graph[gi]) {
    cudaGraphExecDestroy(p->graph[gi]);
    p->graph[gi] = nullptr;
  }
  cudaGraph_t gr;
  CU(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
  launch_step<T>(p, scheme, nullptr);
  cudaError_t le = cudaGetLastError();
  CU(cudaStreamEndCapture(p->stream, &gr));
  if (le != cudaSuccess) return fail(NWB_ECUDA, std::string("graph capture: ") + cudaGetErrorString(le));
  CU(cudaGraphInstantiate(&p->graph[gi], gr, 0));
  cudaGraphDestroy(gr);
  p->graph_stream[gi] = p->stream;
  return NWB_OK;
}

template <typename T>
int march_impl(nwb_plan* p, int scheme, int n0, int n_steps, double guard, double max_seconds,
               const int* snap_steps, int n_snap, void* const* snap_bufs, double* max_abs,
               float* step_ms, int* fail_step, int* fail_member, double* fail_value) {
  const Geom& g = p->g;
  if (n_steps <= 0) return NWB_OK;
  if (!p->upar) return fail(NWB_EINVAL, "coefficients not set (nwb_plan_set_coeffs)");
  const int need_rows = n0 + n_steps + (scheme == NWB_SCHEME_EXPRK22 ? 1 : 0);
  if (need_rows > p->n_rows)
    return fail(NWB_EINVAL, "coefficient rows do not cover the march (" + std::to_string(need_rows) +
                                " > " + std::to_string(p->n_rows) + ")");
  TRY(ensure_hist(p, n0 + n_steps));
  CU(cudaMemsetAsync(p->vmax_hist, 0, (size_t)g.batch * p->hist_len * sizeof(u64), p->stream));
  CU(cudaMemsetAsync(p->red, 0, (size_t)g.batch * 4 * sizeof(u64), p->stream));
  TRY(set_step(p, n0));
  // one graph for both modes: the kernels stamp the bucket boundaries (StepStamp)
  TRY(graph_for<T>(p, scheme));
  const auto t_start = std::chrono::steady_clock::now();
  // budget (max_seconds >= 0; negative = none): checked after every chunk; the
  // first chunk is one step so a zero budget stops after step 1 like the
  // reference (exprk.py:303-306), later chunks are 8 steps
  const bool budget = max_seconds >= 0;
  std::vector<u64> hbuf;
  int rc = NWB_OK;
  int done = 0;
  while (done < n_steps && rc == NWB_OK) {
    const int chunk = budget ? (done == 0 ? 1 : 8) : 64;
    const int cnt = std::min(chunk, n_steps - done);
    for (int i = 0; i < cnt; ++i) {
      const int n = n0 + done + i;
      int snap = -1;
      for (int q = 0; q < n_snap; ++q)
        if (snap_steps[q] == n) snap = q;
      if (snap >= 0) {
        launch_stage<T>(p, 1, scheme, nullptr);
        cudaMemcpyAsync(snap_bufs[snap], p->v, (size_t)g.batch * g.nr * g.nt * sizeof(T),
                        cudaMemcpyDeviceToDevice, p->stream);
        if (scheme == NWB_SCHEME_EXPRK22) launch_stage<T>(p, 2, scheme, nullptr);
      } else {
        cudaError_t e = cudaGraphLaunch(p->graph[scheme == NWB_SCHEME_EXPRK22 ? 0 : 1], p->stream);
        if (e != cudaSuccess) return fail(NWB_ECUDA, std::string("cudaGraphLaunch: ") + cudaGetErrorString(e));
      }
    }
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) return fail(NWB_ECUDA, std::string("march launch: ") + cudaGetErrorString(le));
    // guard check on this chunk (host sync)
    hbuf.resize((size_t)g.batch * cnt);
    for (int mbr = 0; mbr < g.batch; ++mbr)
      cudaMemcpyAsync(hbuf.data() + (size_t)mbr * cnt, p->vmax_hist + (size_t)mbr * p->hist_len + n0 + done,
                      cnt * sizeof(u64), cudaMemcpyDeviceToHost, p->stream);
    cudaError_t se = cudaStreamSynchronize(p->stream);
    if (se != cudaSuccess) return fail(NWB_ECUDA, std::string("march: ") + cudaGetErrorString(se));
    for (int i = 0; i < cnt && rc == NWB_OK; ++i) {
      for (int mbr = 0; mbr < g.batch; ++mbr) {
        double m;
        std::memcpy(&m, &hbuf[(size_t)mbr * cnt + i], sizeof(double));
        if (max_abs) max_abs[(size_t)mbr * n_steps + done + i] = m;
        if (!(std::isfinite(m) && m <= guard)) {
          if (fail_step) *fail_step = n0 + done + i;
          if (fail_member) *fail_member = mbr;
          if (fail_value) *fail_value = m;
          char msg[160];
          std::snprintf(msg, sizeof msg, "max|V| left the guard: step=%d member=%d max_abs=%.17g",
                        n0 + done + i, mbr, m);
          rc = fail(NWB_EINSTABILITY, msg);
          break;
        }
      }
    }
    done += cnt;
    if (rc == NWB_OK && budget) {
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
      if (el > max_seconds) {
        if (fail_step) *fail_step = n0 + done;
        rc = fail(NWB_EBUDGET, "wall-clock budget exhausted");
      }
    }
  }
  if (step_ms && done > 0) {
    // end stamp of the last step (= slot 0 of step n0 + done), then one read-back
    launch_stamp(p->stamps, p->step_ctr, 0, p->stream);
    std::vector<u64> ts((size_t)(done + 1) * NWB_TS_SLOTS);
    cudaMemcpyAsync(ts.data(), p->stamps + (size_t)n0 * NWB_TS_SLOTS, ts.size() * sizeof(u64),
                    cudaMemcpyDeviceToHost, p->stream);
    cudaError_t se = cudaStreamSynchronize(p->stream);
    if (se != cudaSuccess && rc == NWB_OK)
      return fail(NWB_ECUDA, std::string("march time stamps: ") + cudaGetErrorString(se));
    const bool two = scheme == NWB_SCHEME_EXPRK22;
    auto ms = [](u64 a, u64 b) { return b > a ? (float)((double)(b - a) * 1e-6) : 0.f; };
    for (int i = 0; i < done; ++i) {
      const u64* t = &ts[(size_t)i * NWB_TS_SLOTS];
      const float tot = ms(t[0], t[NWB_TS_SLOTS]);
      // nonlinear bucket = WENO (b_eval, exprk.py:161-171): WENO start -> r2c start
      const float nl = std::min(tot, ms(t[1], t[2]) + (two ? ms(t[3], t[4]) : 0.f));
      step_ms[(size_t)i * 3 + 0] = tot;
      step_ms[(size_t)i * 3 + 1] = nl;
      step_ms[(size_t)i * 3 + 2] = tot - nl;
    }
  }
  return rc;
}

// Per-kernel device time over n_steps steps (events around every launch):
// kernel_ms[s*4 + i] for stage s in {0,1}, kernel i in (c2r, weno, r2c, rho).
template <typename T>
int profile_impl(nwb_plan* p, int scheme, int n0, int n_steps, float* kernel_ms) {
  if (!p->upar) return fail(NWB_EINVAL, "coefficients not set (nwb_plan_set_coeffs)");
  if (n0 + n_steps + 1 > p->n_rows) return fail(NWB_EINVAL, "coefficient rows do not cover the run");
  if (p->hist_len < n0 + n_steps) return fail(NWB_EINVAL, "run nwb_march over this range first");
  TRY(set_step(p, n0));
  std::vector<cudaEvent_t> evs((size_t)n_steps * 2 * EV_PER_STAGE);
  for (auto& e : evs) CU(cudaEventCreate(&e));
  for (int i = 0; i < n_steps; ++i) launch_step<T>(p, scheme, &evs[(size_t)i * 2 * EV_PER_STAGE]);
  cudaError_t e = cudaStreamSynchronize(p->stream);
  for (int k = 0; k < 8; ++k) kernel_ms[k] = 0.f;
  if (e == cudaSuccess) {
    for (int i = 0; i < n_steps; ++i) {
      cudaEvent_t* ev = &evs[(size_t)i * 2 * EV_PER_STAGE];
      for (int st = 0; st < (scheme == NWB_SCHEME_EXPRK22 ? 2 : 1); ++st)
        for (int k = 0; k < 4; ++k) {
          float ms = 0.f;
          cudaEventElapsedTime(&ms, ev[st * EV_PER_STAGE + k], ev[st * EV_PER_STAGE + k + 1]);
          kernel_ms[st * 4 + k] += ms;
        }
    }
  }
  for (auto& x : evs) cudaEventDestroy(x);
  if (e != cudaSuccess) return fail(NWB_ECUDA, std::string("profile: ") + cudaGetErrorString(e));
  return NWB_OK;
}

}  // namespace

// ====================================================================== rho slabs
// Multi-GPU single-grid path (BASELINE config C5).  A rank owns
// rho rows [j0, j0+rows) on the physical / theta side and theta modes
// [k0, k0+modes) on the rho side; paper_2103_06080_b200/slab.py moves data
// between the layouts (NCCL all-to-all), all-reduces alpha_theta / max|V|
// and fills the 3-row WENO halos from the neighbouring ranks.  The state
// buffers belong to the caller; the slab owns FFT plans, the multiplier
// tables of its modes, and the (global) coefficient rows.

struct nwb_slab {
  int device = 0, prec = NWB_F64;
  cudaStream_t stream = 0, own_stream = 0;
  int nr = 0, nt = 0, m = 0, kk = 0;  // global grid
  int j0 = 0, rows = 0, ld_rows = 0;  // owned rho rows (theta side)
  int k0 = 0, modes = 0, ld_rho = 0;  // owned theta modes (rho side)
  int blk_n = 0, blk_start[17] = {};   // rho-side transit blocks (nwb_slab_set_blocks)
  double d_sigma = 0, rho_span = 0, theta_span = 0, A = 0, B = 0, eps = 0;
  FftDesc dr{}, dh{};
  FftPlanHost plan_r, plan_h;
  int rho_threads = 256;
  void *tw_r = nullptr, *tw_h = nullptr, *wk = nullptr;
  int *pos_r = nullptr, *rev_r = nullptr, *pos_h = nullptr;
  void *E = nullptr, *P1 = nullptr, *P12 = nullptr, *P2 = nullptr;
  void *upar = nullptr, *uperp = nullptr, *du = nullptr;
  double* alpha_rho = nullptr;
  int n_sig_rows = 0;
  std::vector<void*> allocs;
};

namespace {

int salloc(nwb_slab* s, void** ptr, size_t bytes) {
  cudaError_t e = cudaMallocAsync(ptr, bytes ? bytes : 16, s->stream);
  if (e != cudaSuccess) {
    *ptr = nullptr;
    return fail(e == cudaErrorMemoryAllocation ? NWB_ENOMEM : NWB_ECUDA,
                std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
  }
  s->allocs.push_back(*ptr);
  return NWB_OK;
}

template <typename T> int slab_create_impl(nwb_slab* s) {
  const size_t C = sizeof(cplx<T>);
  std::vector<cplx<T>> twr, twh;
  build_desc<T>(s->nr, s->plan_r, s->dr, twr);
  build_desc<T>(s->m, s->plan_h, s->dh, twh);
  auto wk = twiddles<T>(s->nt, s->kk);
  auto fr = freq_of_pos(s->nr, s->plan_r.stages);
  std::vector<int> pr(s->nr);
  for (int q = 0; q < s->nr; ++q) pr[fr[q]] = q;
  auto fh = freq_of_pos(s->m, s->plan_h.stages);
  std::vector<int> ph(s->m);
  for (int q = 0; q < s->m; ++q) ph[fh[q]] = q;
  TRY(salloc(s, &s->tw_r, twr.size() * C));
  TRY(salloc(s, &s->tw_h, twh.size() * C));
  TRY(salloc(s, &s->wk, wk.size() * C));
  TRY(salloc(s, (void**)&s->pos_r, pr.size() * sizeof(int)));
  TRY(salloc(s, (void**)&s->rev_r, fr.size() * sizeof(int)));
  TRY(salloc(s, (void**)&s->pos_h, ph.size() * sizeof(int)));
  CU(cudaMemcpyAsync(s->tw_r, twr.data(), twr.size() * C, cudaMemcpyHostToDevice, s->stream));
  CU(cudaMemcpyAsync(s->tw_h, twh.data(), twh.size() * C, cudaMemcpyHostToDevice, s->stream));
  CU(cudaMemcpyAsync(s->wk, wk.data(), wk.size() * C, cudaMemcpyHostToDevice, s->stream));
  CU(cudaMemcpyAsync(s->pos_r, pr.data(), pr.size() * sizeof(int), cudaMemcpyHostToDevice, s->stream));
  CU(cudaMemcpyAsync(s->rev_r, fr.data(), fr.size() * sizeof(int), cudaMemcpyHostToDevice, s->stream));
  CU(cudaMemcpyAsync(s->pos_h, ph.data(), ph.size() * sizeof(int), cudaMemcpyHostToDevice, s->stream));
  const size_t tab = (size_t)s->modes * s->ld_rho * C;
  for (void** t : {&s->E, &s->P1, &s->P12, &s->P2}) {
    TRY(salloc(s, t, tab));
    CU(cudaMemsetAsync(*t, 0, tab, s->stream));
  }
  TableArgs ta{};
  ta.nr = s->nr; ta.nt = s->nt; ta.kk = s->modes; ta.ld = s->ld_rho; ta.k0 = s->k0;
  ta.rho_span = s->rho_span; ta.theta_span = s->theta_span;
  ta.d_sigma = s->d_sigma; ta.A = s->A; ta.eps = s->eps;
  ta.rev_r = s->rev_r; ta.natural = 0;
  launch_tables<T>(ta, (cplx<T>*)s->E, (cplx<T>*)s->P1, (cplx<T>*)s->P2, (cplx<T>*)s->P12,
                   nullptr, s->stream);
  CHECK_LAUNCH("slab tables");
  CU(cudaStreamSynchronize(s->stream));  // host vectors above go out of scope
  return NWB_OK;
}

template <typename T> int slab_coeffs_impl(nwb_slab* s, const double* up, const double* uq,
                                           const double* du, int n_rows, int ld, int on_dev) {
  const size_t n = (size_t)n_rows * s->nr;
  for (void* a : {s->upar, s->uperp, s->du, (void*)s->alpha_rho})
    if (a) cudaFreeAsync(a, s->stream);
  TRY(salloc(s, &s->upar, n * sizeof(T)));
  TRY(salloc(s, &s->uperp, n * sizeof(T)));
  TRY(salloc(s, &s->du, n * sizeof(T)));
  TRY(salloc(s, (void**)&s->alpha_rho, (size_t)n_rows * sizeof(double)));
  double* stage = nullptr;
  CU(cudaMallocAsync(&stage, n * sizeof(double), s->stream));
  const double* srcs[3] = {up, uq, du};
  void* dsts[3] = {s->upar, s->uperp, s->du};
  for (int i = 0; i < 3; ++i) {
    if (!srcs[i]) {
      cudaMemsetAsync(dsts[i], 0, n * sizeof(T), s->stream);
      continue;
    }
    cudaMemcpy2DAsync(stage, s->nr * sizeof(double), srcs[i], (size_t)ld * sizeof(double),
                      s->nr * sizeof(double), n_rows,
                      on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s->stream);
    launch_convert<T>((long)n, stage, (T*)dsts[i], s->stream);
  }
  launch_alpha_rho<T>((const T*)s->uperp, s->nr, n_rows, s->alpha_rho, s->stream);
  cudaFreeAsync(stage, s->stream);
  s->n_sig_rows = n_rows;
  CU(cudaStreamSynchronize(s->stream));
  CHECK_LAUNCH("slab coeffs");
  return NWB_OK;
}

template <typename T> ThetaArgs<T> slab_theta_args(const nwb_slab* s) {
  ThetaArgs<T> a{};
  a.g = Geom{s->rows, s->nt, s->m, s->kk, s->ld_rows, 1};
  a.dh = s->dh;
  a.tw_h = (const cplx<T>*)s->tw_h;
  a.wk = (const cplx<T>*)s->wk;
  a.pos_h = s->pos_h;
  a.scale = (T)(1.0 / ((double)s->nr * (double)s->nt));
  a.bcoef = (T)s->B;
  a.coef_ld = s->nr;
  a.coef_j0 = s->j0;
  a.alpha_stride = 2;
  a.vmax_stride = 2;
  return a;
}

template <typename T> int slab_c2r_impl(nwb_slab* s, const void* spec, void* v_ext, int row, void* red) {
  ThetaArgs<T> c = slab_theta_args<T>(s);
  c.spec_in = (const cplx<T>*)spec;
  c.phys_out = (T*)v_ext + (size_t)3 * s->nt;  // interior rows follow 3 halo rows
  if (red) {
    if (!s->upar) return fail(NWB_EINVAL, "coefficients not set");
    c.upar = (const T*)s->upar;
    c.row_off = row;
    c.alpha_bits = (u64*)red;
    c.vmax_bits = (u64*)red + 1;
  }
  launch_theta_c2r<T>(c, 1, s->stream);
  CHECK_LAUNCH("slab c2r");
  return NWB_OK;
}

template <typename T> int slab_weno_impl(nwb_slab* s, const void* v_ext, void* b, int row,
                                         const void* red) {
  if (!s->upar) return fail(NWB_EINVAL, "coefficients not set");
  WenoArgs<T> w{};
  w.g = Geom{s->rows, s->nt, s->m, s->kk, s->ld_rows, 1};
  w.v = (const T*)v_ext;
  w.out = (T*)b;
  w.upar = (const T*)s->upar;
  w.uperp = (const T*)s->uperp;
  w.du = (const T*)s->du;
  w.alpha_rho = s->alpha_rho;
  w.row_off = row;
  w.alpha_bits = (const u64*)red;
  w.alpha_stride = 2;
  w.bcoef = (T)s->B;
  w.inv_drho = (T)(1.0 / (s->rho_span / s->nr));
  w.inv_dtheta = (T)(1.0 / (s->theta_span / s->nt));
  w.coef_ld = s->nr;
  w.coef_j0 = s->j0;
  w.nr_glob = s->nr;
  w.halo = 1;
  // TMA-staged tiles over the slab's rows plus the 3 + 3 halo rows (fp64)
  if (sizeof(T) == 8) w.tma = make_weno_vmap(w.vmap, v_ext, s->nt, s->rows + 6, 1);
  launch_weno<T>(w, s->stream);
  CHECK_LAUNCH("slab weno");
  return NWB_OK;
}

template <typename T> int slab_r2c_impl(nwb_slab* s, const void* b, void* spec) {
  ThetaArgs<T> r = slab_theta_args<T>(s);
  r.phys_in = (const T*)b;
  r.spec_out = (cplx<T>*)spec;
  launch_theta_r2c<T>(r, 1, s->stream);
  CHECK_LAUNCH("slab r2c");
  return NWB_OK;
}

template <typename T> int slab_rho_impl(nwb_slab* s, int mode, const void* bt, void* out, void* vh,
                                        void* u, int k0 = 0, int k1 = -1) {
  RhoArgs<T> q{};
  q.g = Geom{s->nr, s->nt, s->m, s->modes, s->ld_rho, 1};
  q.dr = s->dr;
  q.tw_r = (const cplx<T>*)s->tw_r;
  q.pos_r = s->pos_r;
  q.in = (const cplx<T>*)bt;
  q.out = (cplx<T>*)out;
  q.vh = (cplx<T>*)vh;
  q.u = (cplx<T>*)u;
  q.E = (const cplx<T>*)s->E;
  q.P1 = (const cplx<T>*)s->P1;
  q.P12 = (const cplx<T>*)s->P12;
  q.P2 = (const cplx<T>*)s->P2;
  q.ds = (T)s->d_sigma;
  q.prefetch = 100;
  q.blk_n = s->blk_n;
  for (int b = 0; b <= s->blk_n && b < 17; ++b) q.blk_start[b] = s->blk_start[b];
  q.k_off = k0;
  q.k_cnt = (k1 < 0 ? s->modes : k1) - k0;
  if (q.k_cnt <= 0) return NWB_OK;
  launch_rho<T>(q, mode, s->rho_threads, s->stream);
  CHECK_LAUNCH("slab rho");
  return NWB_OK;
}

}  // namespace

// ====================================================================== splitting baseline
// SURVEY row f4 (reference splitting.py): the Lie-Trotter solver on the closed
// rho grid, float64.  Kernels in csrc/splitting.cu; the theta transforms of
// the axial/absorption stage are the march's theta kernels on a rho extent of
// n = N_rho + 1 rows.

struct nwb_split {
  int device = 0;
  cudaStream_t stream = 0, own_stream = 0;
  int n = 0, nt = 0, ldn = 0;
  Geom g{};
  double d_sigma = 0, d_rho = 0, d_theta = 0, theta_span = 0, A = 0, B = 0, gamma = 0;
  FftDesc dh{};
  FftPlanHost plan_h;
  int theta_rows = 1;
  void *tw_h = nullptr, *wk = nullptr;
  int* pos_h = nullptr;
  double *w = nullptr, *upper = nullptr, *diag = nullptr;   // Thomas factorisation
  double *v = nullptr, *t1 = nullptr, *t2 = nullptr, *vT = nullptr, *sT = nullptr;
  double* gline = nullptr;  // diffraction rho lines when they exceed shared memory
  void* spec = nullptr;
  double *upar = nullptr, *uperp = nullptr, *dus = nullptr, *dur = nullptr;
  int n_rows = 0;
  u64* hist = nullptr;
  int hist_len = 0;
  std::vector<void*> allocs;
};

namespace {

int xalloc(nwb_split* s, void** ptr, size_t bytes) {
  cudaError_t e = cudaMallocAsync(ptr, bytes ? bytes : 16, s->stream);
  if (e != cudaSuccess) {
    *ptr = nullptr;
    return fail(e == cudaErrorMemoryAllocation ? NWB_ENOMEM : NWB_ECUDA,
                std::string("split alloc: ") + cudaGetErrorString(e));
  }
  s->allocs.push_back(*ptr);
  return NWB_OK;
}

int split_create_impl(nwb_split* s) {
  const size_t C = sizeof(double2);
  std::vector<double2> twh;
  build_desc<double>(s->g.m, s->plan_h, s->dh, twh);
  auto wk = twiddles<double>(s->nt, s->g.kk);
  auto fh = freq_of_pos(s->g.m, s->plan_h.stages);
  std::vector<int> ph(s->g.m);
  for (int q = 0; q < s->g.m; ++q) ph[fh[q]] = q;
  // Thomas factorisation exactly as the reference builds it (splitting.py:103-113)
  const int n = s->n;
  const double c = 0.5 * s->gamma;
  std::vector<double> lower(n, -c), upper(n, -c), diag(n), w(n, 0.0);
  lower[n - 1] = -2.0 * c;
  upper[0] = -2.0 * c;
  diag[0] = 1.0 + 2.0 * c;
  for (int j = 1; j < n; ++j) {
    w[j] = lower[j] / diag[j - 1];
    diag[j] = (1.0 + 2.0 * c) - w[j] * upper[j - 1];
  }
  TRY(xalloc(s, &s->tw_h, twh.size() * C));
  TRY(xalloc(s, &s->wk, wk.size() * C));
  TRY(xalloc(s, (void**)&s->pos_h, ph.size() * sizeof(int)));
  TRY(xalloc(s, (void**)&s->w, n * sizeof(double)));
  TRY(xalloc(s, (void**)&s->upper, n * sizeof(double)));
  TRY(xalloc(s, (void**)&s->diag, n * sizeof(double)));
  const size_t phys = (size_t)n * s->nt * sizeof(double);
  for (double** b : {&s->v, &s->t1, &s->t2}) TRY(xalloc(s, (void**)b, phys));
  TRY(xalloc(s, (void**)&s->vT, (size_t)s->nt * s->ldn * sizeof(double)));
  TRY(xalloc(s, (void**)&s->sT, (size_t)s->nt * s->ldn * sizeof(double)));
  TRY(xalloc(s, &s->spec, (size_t)s->g.kk * s->g.ld * C));
  if (!split_line_in_smem(n)) TRY(xalloc(s, (void**)&s->gline, (size_t)3 * n * sizeof(double)));
  CU(cudaMemsetAsync(s->spec, 0, (size_t)s->g.kk * s->g.ld * C, s->stream));
  CU(cudaMemcpyAsync(s->tw_h, twh.data(), twh.size() * C, cudaMemcpyHostToDevice, s->stream));
  CU(cudaMemcpyAsync(s->wk, wk.data(), wk.size() * C, cudaMemcpyHostToDevice, s->stream));
  CU(cudaMemcpyAsync(s->pos_h, ph.data(), ph.size() * sizeof(int), cudaMemcpyHostToDevice, s->stream));
  CU(cudaMemcpyAsync(s->w, w.data(), n * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  CU(cudaMemcpyAsync(s->upper, upper.data(), n * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  CU(cudaMemcpyAsync(s->diag, diag.data(), n * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  return NWB_OK;
}

ThetaArgs<double> split_theta_args(const nwb_split* s) {
  ThetaArgs<double> a{};
  a.g = s->g;
  a.dh = s->dh;
  a.tw_h = (const double2*)s->tw_h;
  a.wk = (const double2*)s->wk;
  a.pos_h = s->pos_h;
  a.scale = 1.0 / (double)s->nt;  // a 1-D theta inverse (scipy irfft along axis 1)
  a.r1 = 1;
  return a;
}

// stage: 0 diffraction, 1 Burgers, 2 axial + absorption (coefficient row `row`),
// 3 transverse (row `row`), 4 the whole Lie step; vmax (device) gets max|out|
// of the transverse stage
int split_stage(nwb_split* s, int stage, int row, const double* in, double* out, u64* vmax) {
  const int n = s->n, nt = s->nt;
  cudaStream_t st = s->stream;
  if ((stage == 2 || stage == 3 || stage == 4) && (row < 0 || row >= s->n_rows))
    return fail(NWB_EINVAL, "splitting: coefficient row out of range (nwb_split_set_coeffs)");
  const double* cur = in;
  auto dst = [&](int last) -> double* { return stage == 4 ? (last ? out : (cur == s->t1 ? s->t2 : s->t1)) : out; };
  if (stage == 0 || stage == 4) {
    launch_split_prep(cur, n, nt, s->ldn, s->vT, s->sT, st);
    double* o = dst(0);
    launch_split_diffraction(s->vT, s->sT, n, nt, s->ldn, s->gamma, s->w, s->upper, s->diag, o,
                             s->gline, st);
    cur = o;
  }
  if (stage == 1 || stage == 4) {
    double* o = dst(0);
    launch_split_burgers(cur, n, nt, s->B, s->d_sigma / s->d_theta, o, st);
    cur = o;
  }
  if (stage == 2 || stage == 4) {
    ThetaArgs<double> r = split_theta_args(s);
    r.phys_in = cur;
    r.spec_out = (double2*)s->spec;
    launch_theta_r2c<double>(r, s->theta_rows, st);
    launch_split_axial((double2*)s->spec, n, s->g.kk, s->g.ld, s->upar + (size_t)row * n,
                       s->d_sigma, s->A, s->theta_span, st);
    double* o = dst(0);
    ThetaArgs<double> c = split_theta_args(s);
    c.spec_in = (const double2*)s->spec;
    c.phys_out = o;
    launch_theta_c2r<double>(c, s->theta_rows, st);
    cur = o;
  }
  if (stage == 3 || stage == 4) {
    launch_split_transverse(cur, n, nt, s->uperp + (size_t)row * n, s->dus + (size_t)row * n,
                            s->dur + (size_t)row * n, s->d_sigma, s->d_rho, out, vmax, st);
  }
  CHECK_LAUNCH("splitting stage");
  return NWB_OK;
}

int split_march_impl(nwb_split* s, int n0, int n_steps, double guard, double max_seconds,
                     double* max_abs, int* fail_step, double* fail_value) {
  if (n_steps <= 0) return NWB_OK;
  if (n0 < 0 || n0 + n_steps > s->n_rows)
    return fail(NWB_EINVAL, "splitting: coefficient rows do not cover the march");
  if (s->hist_len < n_steps) {
    if (s->hist) cudaFreeAsync(s->hist, s->stream);
    s->hist = nullptr;
    CU(cudaMallocAsync((void**)&s->hist, (size_t)n_steps * sizeof(u64), s->stream));
    s->hist_len = n_steps;
  }
  CU(cudaMemsetAsync(s->hist, 0, (size_t)n_steps * sizeof(u64), s->stream));
  const auto t0 = std::chrono::steady_clock::now();
  const bool budget = max_seconds >= 0;
  std::vector<u64> h;
  int done = 0;
  while (done < n_steps) {
    const int cnt = std::min(budget ? (done == 0 ? 1 : 8) : 32, n_steps - done);
    for (int i = 0; i < cnt; ++i) {
      // the step's output lands back in s->v (Lie step: v -> t1/t2 chain -> v)
      TRY(split_stage(s, 4, n0 + done + i, s->v, s->v, s->hist + done + i));
    }
    h.resize(cnt);
    CU(cudaMemcpyAsync(h.data(), s->hist + done, cnt * sizeof(u64), cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    for (int i = 0; i < cnt; ++i) {
      double m;
      std::memcpy(&m, &h[i], sizeof(double));
      if (max_abs) max_abs[done + i] = m;
      if (!(std::isfinite(m) && m <= guard)) {
        if (fail_step) *fail_step = n0 + done + i;
        if (fail_value) *fail_value = m;
        char msg[160];
        std::snprintf(msg, sizeof msg, "max|V| left the guard: step=%d member=0 max_abs=%.17g",
                      n0 + done + i, m);
        return fail(NWB_EINSTABILITY, msg);
      }
    }
    done += cnt;
    if (budget) {
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > max_seconds) {
        if (fail_step) *fail_step = n0 + done;
        return fail(NWB_EBUDGET, "wall-clock budget exhausted");
      }
    }
  }
  return NWB_OK;
}

}  // namespace

// ====================================================================== C ABI

int nwb_slab_create(nwb_slab** out, int n_rho, int n_theta, int j0, int rows, int k0, int modes,
                    int precision, double d_sigma, double rho_span, double theta_span, double A,
                    double B, double eps, int device) {
  if (!out) return fail(NWB_EINVAL, "null slab pointer");
  *out = nullptr;
  if (precision != NWB_F64 && precision != NWB_F32) return fail(NWB_EINVAL, "unknown precision");
  if (n_theta % 2) return fail(NWB_EUNSUPPORTED, "n_theta must be even");
  const int kk = n_theta / 2 + 1;
  if (rows < 1 || j0 < 0 || j0 + rows > n_rho || modes < 1 || k0 < 0 || k0 + modes > kk)
    return fail(NWB_EINVAL, "slab ranges outside the grid");
  nwb_slab* s = new nwb_slab();
  s->device = device; s->prec = precision;
  s->nr = n_rho; s->nt = n_theta; s->m = n_theta / 2; s->kk = kk;
  // theta-side spectra (kk, rows) are unpadded: the block a rank receives
  // from (or sends to) rank r is then one contiguous segment
  s->j0 = j0; s->rows = rows; s->ld_rows = rows;
  s->k0 = k0; s->modes = modes; s->ld_rho = (n_rho + 7) / 8 * 8;
  s->d_sigma = d_sigma; s->rho_span = rho_span; s->theta_span = theta_span;
  s->A = A; s->B = B; s->eps = eps;
  if (!plan_fft(n_rho, 0, s->plan_r) || !plan_fft(s->m, 0, s->plan_h)) {
    delete s;
    return fail(NWB_EUNSUPPORTED, "n_rho and n_theta/2 must factor into 2, 3, 5, 7");
  }
  const int th = ((n_rho / 4) + 31) / 32 * 32;
  s->rho_threads = th < 64 ? 64 : (th > 512 ? 512 : th);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete s;
    return fail(NWB_ECUDA, std::string("slab device/stream: ") + cudaGetErrorString(e));
  }
  s->stream = s->own_stream;
  keep_pool_memory(device);
  const int rc = precision == NWB_F64 ? slab_create_impl<double>(s) : slab_create_impl<float>(s);
  if (rc != NWB_OK) {
    nwb_slab_destroy(s);
    return rc;
  }
  *out = s;
  return NWB_OK;
}

int nwb_slab_destroy(nwb_slab* s) {
  if (!s) return NWB_OK;
  cudaSetDevice(s->device);
  cudaStreamSynchronize(s->stream);
  for (void* a : s->allocs)
    if (a) cudaFreeAsync(a, s->stream);
  cudaStreamSynchronize(s->stream);
  if (s->own_stream) cudaStreamDestroy(s->own_stream);
  delete s;
  return NWB_OK;
}

int nwb_slab_set_stream(nwb_slab* s, void* stream) {
  if (!s) return fail(NWB_EINVAL, "null slab");
  s->stream = stream ? (cudaStream_t)stream : s->own_stream;
  return NWB_OK;
}

int nwb_slab_set_blocks(nwb_slab* s, int n_blocks, const int* row_starts) {
  if (!s) return fail(NWB_EINVAL, "null slab");
  if (n_blocks < 0 || n_blocks > 16) return fail(NWB_EINVAL, "slab blocks: 0 .. 16 ranks");
  if (n_blocks > 0) {
    if (row_starts[0] != 0 || row_starts[n_blocks] != s->nr)
      return fail(NWB_EINVAL, "slab blocks must partition the rho rows");
    for (int b = 0; b < n_blocks; ++b)
      if (row_starts[b + 1] < row_starts[b]) return fail(NWB_EINVAL, "slab blocks out of order");
    for (int b = 0; b <= n_blocks; ++b) s->blk_start[b] = row_starts[b];
  }
  s->blk_n = n_blocks;
  return NWB_OK;
}

int nwb_slab_layout(const nwb_slab* s, int* ld_rows, int* ld_rho) {
  if (!s) return fail(NWB_EINVAL, "null slab");
  if (ld_rows) *ld_rows = s->ld_rows;
  if (ld_rho) *ld_rho = s->ld_rho;
  return NWB_OK;
}

int nwb_slab_set_coeffs(nwb_slab* s, const double* u_par, const double* u_perp,
                        const double* du_drho, int n_rows, int ld, int on_device) {
  if (!s) return fail(NWB_EINVAL, "null slab");
  if (n_rows < 1 || ld < s->nr) return fail(NWB_EINVAL, "coefficient rows / ld too small");
  CU(cudaSetDevice(s->device));
  return s->prec == NWB_F64 ? slab_coeffs_impl<double>(s, u_par, u_perp, du_drho, n_rows, ld, on_device)
                            : slab_coeffs_impl<float>(s, u_par, u_perp, du_drho, n_rows, ld, on_device);
}

int nwb_slab_theta_c2r(nwb_slab* s, const void* spec, void* v_ext, int sigma_row, void* red) {
  if (!s) return fail(NWB_EINVAL, "null slab");
  if (red && (sigma_row < 0 || sigma_row >= s->n_sig_rows)) return fail(NWB_EINVAL, "sigma row out of range");
  return s->prec == NWB_F64 ? slab_c2r_impl<double>(s, spec, v_ext, sigma_row, red)
                            : slab_c2r_impl<float>(s, spec, v_ext, sigma_row, red);
}

int nwb_slab_weno(nwb_slab* s, const void* v_ext, void* b, int sigma_row, const void* red) {
  if (!s) return fail(NWB_EINVAL, "null slab");
  if (sigma_row < 0 || sigma_row >= s->n_sig_rows) return fail(NWB_EINVAL, "sigma row out of range");
  return s->prec == NWB_F64 ? slab_weno_impl<double>(s, v_ext, b, sigma_row, red)
                            : slab_weno_impl<float>(s, v_ext, b, sigma_row, red);
}

int nwb_slab_theta_r2c(nwb_slab* s, const void* b, void* spec) {
  if (!s) return fail(NWB_EINVAL, "null slab");
  return s->prec == NWB_F64 ? slab_r2c_impl<double>(s, b, spec) : slab_r2c_impl<float>(s, b, spec);
}

int nwb_slab_rho(nwb_slab* s, int mode, const void* bt, void* out, void* vh, void* u) {
  if (!s) return fail(NWB_EINVAL, "null slab");
  if (mode < RHO_STAGE1 || mode > RHO_INIT) return fail(NWB_EINVAL, "unknown rho mode");
  return s->prec == NWB_F64 ? slab_rho_impl<double>(s, mode, bt, out, vh, u)
                            : slab_rho_impl<float>(s, mode, bt, out, vh, u);
}

int nwb_slab_rho_range(nwb_slab* s, int mode, int k_begin, int k_end, const void* bt, void* out,
                       void* vh, void* u) {
  if (!s) return fail(NWB_EINVAL, "null slab");
  if (mode < RHO_STAGE1 || mode > RHO_INIT) return fail(NWB_EINVAL, "unknown rho mode");
  if (k_begin < 0 || k_end > s->modes || k_begin > k_end) return fail(NWB_EINVAL, "mode range outside the slab");
  return s->prec == NWB_F64 ? slab_rho_impl<double>(s, mode, bt, out, vh, u, k_begin, k_end)
                            : slab_rho_impl<float>(s, mode, bt, out, vh, u, k_begin, k_end);
}

int nwb_profile_kernels(nwb_plan* p, int scheme, int n0, int n_steps, float* kernel_ms) {
  TRY(check_plan(p));
  if (!kernel_ms || n_steps < 1) return fail(NWB_EINVAL, "bad profile arguments");
  return p->prec == NWB_F64 ? profile_impl<double>(p, scheme, n0, n_steps, kernel_ms)
                            : profile_impl<float>(p, scheme, n0, n_steps, kernel_ms);
}

extern "C" {

int nwb_abi_version(void) { return 1; }

const char* nwb_last_error(void) { return g_err.c_str(); }

int nwb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int nwb_plan_create(nwb_plan** out, int n_rho, int n_theta, int batch, int precision,
                    double d_sigma, double rho_span, double theta_span, double A, double B,
                    double eps, int device) {
  if (!out) return fail(NWB_EINVAL, "null plan pointer");
  *out = nullptr;
  if (n_rho < 1 || n_theta < 2 || batch < 1) return fail(NWB_EINVAL, "grid extents must be positive");
  if (precision != NWB_F64 && precision != NWB_F32) return fail(NWB_EINVAL, "unknown precision");
  if (n_theta % 2) return fail(NWB_EUNSUPPORTED, "n_theta must be even (half-length real FFT)");
  nwb_plan* p = new nwb_plan();
  p->device = device;
  p->prec = precision;
  p->rsz = precision == NWB_F64 ? 8 : 4;
  p->g.nr = n_rho;
  p->g.nt = n_theta;
  p->g.m = n_theta / 2;
  p->g.kk = n_theta / 2 + 1;
  p->g.ld = (n_rho + 7) / 8 * 8;
  p->g.batch = batch;
  p->d_sigma = d_sigma;
  p->rho_span = rho_span;
  p->theta_span = theta_span;
  p->A = A;
  p->B = B;
  p->eps = eps;
  // The 2-CTA cluster split of a rho column (k_rho_split) is available but off
  // by default: measured at Set 4 fp64 it loses to one CTA per column
  // (0.93 vs 0.79 ms, profiles/README.md); NWB_RHO_SPLIT=1 enables it.
  {
    p->rho_split = 0;
    if (const char* env = std::getenv("NWB_RHO_SPLIT"))
      p->rho_split = (env[0] == '1' && n_rho % 2 == 0 && n_rho >= 16) ? 1 : 0;
    if (const char* env = std::getenv("NWB_RHO_HALF"))
      p->rho_half = (env[0] == '1' && precision == NWB_F64 && n_rho % 2 == 0 && n_rho >= 1024 &&
                     n_rho <= 2 * 256 * 20 && !p->rho_split) ? 1 : 0;
    // bulk L2 prefetch of the combine operands: off (measured slower at Set 4
    // in both precisions since the radix-R passes and two fp32 CTAs per SM)
    p->rho_prefetch = 0;
    if (const char* env = std::getenv("NWB_RHO_PREFETCH")) {  // "1" = whole rows, else percent
      const int v = std::atoi(env);
      p->rho_prefetch = v == 1 ? 100 : (v < 0 ? 0 : (v > 100 ? 100 : v));
    }
    if (const char* env = std::getenv("NWB_RHO_NEXTPF")) p->rho_next_pf = std::atoi(env);
    if (const char* env = std::getenv("NWB_RHO_ROLL")) p->rho_roll = std::atoi(env);
    if (const char* env = std::getenv("NWB_RHO_DEBUG")) p->rho_debug = std::atoi(env);
    if (const char* env = std::getenv("NWB_RHO_STAGGER"))
      std::sscanf(env, "%d,%d", &p->rho_stagger_ns, &p->rho_stagger_mode);
    // 16-byte elements keep every padded chunk 16-byte aligned in shared memory
    p->rho_bulk = precision == NWB_F64 ? 1 : 0;
    if (const char* env = std::getenv("NWB_RHO_BULK")) p->rho_bulk = p->rho_bulk && env[0] != '0';
    // r2c rows by bulk copies measured 1 % slower at C2 (0.208 vs 0.206 ms): off
    p->theta_bulk = 0;
    if (const char* env = std::getenv("NWB_THETA_BULK")) p->theta_bulk = precision == NWB_F64 && env[0] == '1';
    if (const char* env = std::getenv("NWB_THETA_DEBUG")) p->theta_debug = std::atoi(env);
    if (const char* env = std::getenv("NWB_RHO_PERSIST")) p->rho_persistent = env[0] == '1';
    if (p->rho_debug) p->rho_persistent = 0;  // the knobs live in k_rho
    // warp-specialised rho pass: NWB_RHO_WS=<transform threads>[,<combine threads>]
    if (const char* env = std::getenv("NWB_RHO_WS")) {
      int a1 = 0, a2 = 256;
      if (std::sscanf(env, "%d,%d", &a1, &a2) >= 1 && a1 >= 64 && a1 % 32 == 0 && a2 >= 32 &&
          a2 % 32 == 0 && a1 + a2 <= 512 && !p->rho_debug) {
        p->rho_ws = a1;
        p->rho_ws2 = a2;
      }
    }
  }
  // First rho stage fused into the theta passes (NWB_RHO_R1=<r1>; see
  // ThetaArgs::r1): r1 in {2, 4}, n_rho divisible by r1, single plans of long
  // columns only (the cluster split and slabs keep whole columns).
  {
    int r1 = 1;
    if (const char* env = std::getenv("NWB_RHO_R1")) r1 = std::atoi(env);
    if (r1 != 2 && r1 != 4) r1 = 1;
    if (n_rho % r1 || n_rho / r1 < 8 || p->rho_split || p->rho_half) r1 = 1;
    // the theta CTAs hold r1 whole rows
    if ((size_t)r1 * (n_theta / 2 + 64) * 2 * (precision == NWB_F64 ? 8 : 4) > 200 * 1024) r1 = 1;
    p->rho_r1 = r1;
    p->msub = n_rho / r1;
    if (const char* env = std::getenv("NWB_RHO_ILV")) p->ilv = env[0] != '0';
  }
  int mp_r = 16, mp_h = 16;
  if (const char* env = std::getenv("NWB_MAXPROD_R")) mp_r = std::atoi(env);
  if (const char* env = std::getenv("NWB_MAXPROD_H")) mp_h = std::atoi(env);
  // radix-25 rho passes for long fp32 columns: C2 fp32 rho 0.575 -> 0.553 ms per
  // step; fp64 slower (1.060 vs 0.989: the 25-point butterfly spills at 128
  // registers) and so are short columns (C4 fp32 6.11 -> 6.76 ms per step: too few
  // 25-point butterflies per pass for the CTA); NWB_PAIR55=0/1 overrides
  int pair55 = precision == NWB_F32 && n_rho >= 5000 ? 1 : 0;
  if (const char* env = std::getenv("NWB_PAIR55")) pair55 = std::atoi(env);
  if (precision != NWB_F32) pair55 = 0;  // radix-25 passes are compiled for fp32 only
  if (!plan_fft(n_rho, (p->rho_split || p->rho_half) ? 2 : p->rho_r1, p->plan_r, mp_r, pair55) ||
      !plan_fft(p->g.m, 0, p->plan_h, mp_h)) {
    delete p;
    return fail(NWB_EUNSUPPORTED, "n_rho and n_theta/2 must factor into 2, 3, 5, 7");
  }
  const size_t csz = 2 * p->rsz;
  const size_t smem_max = 227 * 1024;
  if ((size_t)n_rho * csz > smem_max || (size_t)p->g.m * csz > smem_max) {
    delete p;
    return fail(NWB_EUNSUPPORTED, "transform length exceeds one CTA's shared memory");
  }
  const size_t row_bytes = (size_t)p->g.m * csz;
  // rows per theta CTA: the largest R with R rows in <= 64 KB of shared memory that
  // still gives >= 2 CTAs per SM over the whole batch (small single grids such as
  // C1 / C3 otherwise leave SMs idle)
  p->theta_rows = 1;
  for (int r : {8, 4, 2})
    if ((size_t)r * row_bytes <= 64 * 1024 && (long)batch * ((n_rho + r - 1) / r) >= 2L * 148) {
      p->theta_rows = r;
      break;
    }
  if (const char* env = std::getenv("NWB_THETA_ROWS")) {  // measurement knob
    const int r = std::atoi(env);
    if ((r == 1 || r == 2 || r == 4 || r == 8) && (size_t)r * row_bytes <= 200 * 1024) p->theta_rows = r;
  }
  // c2r of long rows (>= 24 KB, e.g. fp64 Set 4): one-row 128-thread CTAs, four per
  // SM in different phases, beat two-row CTAs (measured 0.234 vs 0.255 ms at C2);
  // r2c keeps two rows (its transposed 16-byte stores would half-fill sectors)
  p->theta_rows_c2r = row_bytes >= 24 * 1024 ? 1 : p->theta_rows;
  if (const char* env = std::getenv("NWB_THETA_ROWS_C2R")) {  // measurement knob
    const int r = std::atoi(env);
    if ((r == 1 || r == 2 || r == 4 || r == 8) && (size_t)r * row_bytes <= 200 * 1024) p->theta_rows_c2r = r;
  }
  // about one radix-10 butterfly per thread and pass: short columns get small
  // CTAs, so several share an SM (C4's 1250-point columns: 128 threads, 4 CTAs
  // per SM, rho pass 2.97 -> 1.45 ms per 256-member stage) while the 10000-point
  // C2 column keeps 512 threads (measured best against 256 / 384 / 640 / 768)
  int th = ((n_rho / 10) + 31) / 32 * 32;
  const int th_max = precision == NWB_F32 ? 384 : 512;  // fp32: k_rho_r80 (spectral.cu)
  p->rho_threads = th < 128 ? 128 : (th > th_max ? th_max : th);  // small grids: latency-bound, keep 4 warps
  if (p->rho_split) p->rho_threads = p->rho_threads > 256 ? 256 : p->rho_threads;
  if (p->rho_r1 > 1) {  // sub-columns: about one radix-10 butterfly per thread, <= 256
    const int ts = ((p->msub / 10) + 31) / 32 * 32;
    p->rho_threads = ts < 128 ? 128 : (ts > 256 ? 256 : ts);
  }
  if (const char* env = std::getenv("NWB_RHO_THREADS")) {
    const int t = std::atoi(env);
    if (t >= 32 && t <= (p->rho_split ? 256 : 1024) && t % 32 == 0) p->rho_threads = t;
  }
  cudaError_t e = cudaSetDevice(device);
  // Long single-grid columns (C2: 10000 points, one fp64 / two fp32 CTAs per SM):
  // bulk-prefetch the head of the combine operand rows into L2 at CTA entry and,
  // after the combine, the input column of the CTA one resident wave later (the
  // next CTA on this SM), so part of the streaming overlaps the transforms.
  // Measured at C2 (tools/rho_probe.py, profiles/README.md): fp64 rho
  // 1.146 -> 1.104 ms per step with 40 % / one wave, fp32 0.590 -> 0.581 with 25 %.
  if (e == cudaSuccess && batch == 1 && (size_t)n_rho * csz >= 64 * 1024 && !p->rho_split) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int per_sm = (int)(smem_max / ((size_t)n_rho * csz * 9 / 8));
    // (fp64 re-tuned with the first-wave stagger and bulk column loads: 40 % -> 20 %,
    // rho 1.010 -> 0.994 ms per step)
    if (!std::getenv("NWB_RHO_PREFETCH")) p->rho_prefetch = p->rsz == 8 ? 20 : 25;
    if (!std::getenv("NWB_RHO_NEXTPF")) p->rho_next_pf = sms * (per_sm < 1 ? 1 : per_sm);
    // and the combine prefetches each round's operand rows one round ahead
    // (fp64 rho 1.060 -> 1.034 ms per step, fp32 0.601 -> 0.582)
    if (!std::getenv("NWB_RHO_ROLL")) p->rho_roll = 1;
    // One column per SM: all SMs would load, transform and stream in lockstep,
    // so HBM idles during the transforms.  The first wave's CTAs start
    // staggered over about one column period (40 us at C2 fp64, 30 us fp32) so
    // some SMs stream while others transform (tools/rho_probe.py, C2: fp64
    // rho 1.041 -> 1.014 ms per step, fp32 0.582 -> 0.574; larger spreads
    // measured slower).
    if (!std::getenv("NWB_RHO_STAGGER")) p->rho_stagger_ns = p->rsz == 8 ? 40000 : 30000;
  }
  if (e == cudaSuccess && p->rho_ws > 0) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    p->rho_ws_ctas = sms > 0 ? sms : 148;
    p->rho_split = 0;
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete p;
    return fail(NWB_ECUDA, std::string("plan device/stream: ") + cudaGetErrorString(e));
  }
  p->stream = p->own_stream;
  // WENO / r2c overlap chunks (NWB_OVERLAP=<chunks>, 0/1 = off; at most 8)
  p->overlap_chunks = 0;
  if (const char* env = std::getenv("NWB_OVERLAP")) p->overlap_chunks = std::atoi(env);
  if (p->overlap_chunks > 8) p->overlap_chunks = 8;
  if (p->rho_r1 > 1) p->overlap_chunks = 0;  // r2c row chunks need whole-row CTAs
  if (p->overlap_chunks > 1) {
    e = cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking);
    for (int i = 0; i < 9 && e == cudaSuccess; ++i)
      e = cudaEventCreateWithFlags(&p->ov_ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) {
      nwb_plan_destroy(p);
      return fail(NWB_ECUDA, std::string("overlap stream: ") + cudaGetErrorString(e));
    }
  }
  keep_pool_memory(device);
  int rc = precision == NWB_F64 ? create_impl<double>(p) : create_impl<float>(p);
  if (rc != NWB_OK) {
    nwb_plan_destroy(p);
    return rc;
  }
  *out = p;
  return NWB_OK;
}

int nwb_plan_destroy(nwb_plan* p) {
  if (!p) return NWB_OK;
  cudaSetDevice(p->device);
  cudaStreamSynchronize(p->stream);
  drop_graphs(p);
  for (void* a : p->allocs)
    if (a) cudaFreeAsync(a, p->stream);
  if (p->own_stream) cudaStreamDestroy(p->own_stream);
  if (p->side) cudaStreamDestroy(p->side);
  for (cudaEvent_t e : p->ov_ev)
    if (e) cudaEventDestroy(e);
  delete p;
  return NWB_OK;
}

int nwb_plan_set_stream(nwb_plan* p, void* stream) {
  TRY(check_plan(p));
  p->stream = stream ? (cudaStream_t)stream : p->own_stream;
  return NWB_OK;
}

long long nwb_plan_bytes(const nwb_plan* p) { return p ? p->bytes : 0; }

int nwb_plan_set_coeffs(nwb_plan* p, const double* u_par, const double* u_perp,
                        const double* du_drho, int n_rows, int ld, int on_device) {
  TRY(check_plan(p));
  if (n_rows < 1 || ld < p->g.nr) return fail(NWB_EINVAL, "coefficient rows / ld too small");
  return p->prec == NWB_F64 ? set_coeffs_impl<double>(p, u_par, u_perp, du_drho, n_rows, ld, on_device)
                            : set_coeffs_impl<float>(p, u_par, u_perp, du_drho, n_rows, ld, on_device);
}

int nwb_plan_load_physical(nwb_plan* p, const void* v0) {
  TRY(check_plan(p));
  return p->prec == NWB_F64 ? load_physical_impl<double>(p, v0) : load_physical_impl<float>(p, v0);
}

int nwb_plan_load_spectrum(nwb_plan* p, const void* vhat) {
  TRY(check_plan(p));
  return p->prec == NWB_F64 ? load_spectrum_impl<double>(p, vhat) : load_spectrum_impl<float>(p, vhat);
}

int nwb_plan_store_spectrum(nwb_plan* p, void* vhat) {
  TRY(check_plan(p));
  return p->prec == NWB_F64 ? store_spectrum_impl<double>(p, vhat) : store_spectrum_impl<float>(p, vhat);
}

int nwb_plan_store_physical(nwb_plan* p, void* v, double* max_abs) {
  TRY(check_plan(p));
  return p->prec == NWB_F64 ? c2r_out<double>(p, p->t, v, max_abs) : c2r_out<float>(p, p->t, v, max_abs);
}

int nwb_march(nwb_plan* p, int scheme, int n0, int n_steps, double guard, double max_seconds,
              const int* snap_steps, int n_snap, void* const* snap_bufs, double* max_abs,
              float* step_ms, int* fail_step, int* fail_member, double* fail_value) {
  TRY(check_plan(p));
  if (scheme != NWB_SCHEME_EXPRK22 && scheme != NWB_SCHEME_EXPEULER) return fail(NWB_EINVAL, "unknown scheme");
  if (n0 < 0 || n_steps < 0) return fail(NWB_EINVAL, "negative step range");
  return p->prec == NWB_F64
             ? march_impl<double>(p, scheme, n0, n_steps, guard, max_seconds, snap_steps, n_snap,
                                  snap_bufs, max_abs, step_ms, fail_step, fail_member, fail_value)
             : march_impl<float>(p, scheme, n0, n_steps, guard, max_seconds, snap_steps, n_snap,
                                 snap_bufs, max_abs, step_ms, fail_step, fail_member, fail_value);
}

int nwb_step(nwb_plan* p, int scheme, int n) {
  TRY(check_plan(p));
  if (!p->upar) return fail(NWB_EINVAL, "coefficients not set");
  if (n + (scheme == NWB_SCHEME_EXPRK22 ? 1 : 0) >= p->n_rows) return fail(NWB_EINVAL, "coefficient rows do not cover the step");
  TRY(ensure_hist(p, n + 1));
  TRY(set_step(p, n));
  return p->prec == NWB_F64 ? step_impl<double>(p, scheme, nullptr) : step_impl<float>(p, scheme, nullptr);
}

int nwb_rfft2(nwb_plan* p, const void* in, void* out) {
  TRY(check_plan(p));
  return p->prec == NWB_F64 ? rfft2_impl<double>(p, in, out) : rfft2_impl<float>(p, in, out);
}

int nwb_irfft2(nwb_plan* p, const void* in, void* out) {
  TRY(check_plan(p));
  return p->prec == NWB_F64 ? irfft2_impl<double>(p, in, out) : irfft2_impl<float>(p, in, out);
}

int nwb_weno5_b(int precision, int batch, int n_rho, int n_theta, const void* v, const void* up,
                const void* uq, const void* du, double b, double d_rho, double d_theta, void* out,
                void* workspace, void* stream) {
  if (batch < 1 || n_rho < 1 || n_theta < 1) return fail(NWB_EINVAL, "grid extents must be positive");
  if (!v || !up || !uq || !du || !out || !workspace) return fail(NWB_EINVAL, "null buffer");
  Geom g{};
  g.nr = n_rho;
  g.nt = n_theta;
  g.batch = batch;
  cudaStream_t s = (cudaStream_t)stream;
  if (precision == NWB_F64) return weno_impl<double>(g, v, up, uq, du, b, d_rho, d_theta, out, workspace, s);
  if (precision == NWB_F32) return weno_impl<float>(g, v, up, uq, du, b, d_rho, d_theta, out, workspace, s);
  return fail(NWB_EINVAL, "unknown precision");
}

int nwb_tables(int precision, int n_rho, int n_theta, double rho_span, double theta_span,
               double d_sigma, double A, double eps, void* E, void* P1, void* P2, void* P12,
               void* z, void* stream) {
  if (n_rho < 1 || n_theta < 1) return fail(NWB_EINVAL, "grid extents must be positive");
  TableArgs ta{};
  ta.nr = n_rho; ta.nt = n_theta; ta.kk = n_theta / 2 + 1; ta.ld = ta.kk;
  ta.rho_span = rho_span; ta.theta_span = theta_span; ta.d_sigma = d_sigma; ta.A = A; ta.eps = eps;
  ta.rev_r = nullptr; ta.natural = 1;
  cudaStream_t s = (cudaStream_t)stream;
  if (precision == NWB_F64)
    launch_tables<double>(ta, (double2*)E, (double2*)P1, (double2*)P2, (double2*)P12, (double2*)z, s);
  else
    launch_tables<float>(ta, (float2*)E, (float2*)P1, (float2*)P2, (float2*)P12, (double2*)z, s);
  CHECK_LAUNCH("tables");
  return NWB_OK;
}

int nwb_turbulence_fields(int n_modes, const double* mode_params, double lam, double inv_c0,
                          const double* sigma_nodes, int n_sigma, const double* rho_nodes,
                          int n_rho, double* scratch, double* u_par, double* u_perp,
                          double* du_dsigma, double* du_drho, void* stream) {
  if (n_modes < 1 || n_sigma < 1 || n_rho < 1) return fail(NWB_EINVAL, "empty turbulence grid");
  if (!mode_params || !sigma_nodes || !rho_nodes || !scratch || !u_par || !u_perp || !du_dsigma ||
      !du_drho)
    return fail(NWB_EINVAL, "null buffer");
  const double* mp = mode_params;  // [7][n_modes]: kx, ky, phase, amp1, amp2, w_ds, w_dr
  launch_turbulence(mp, mp + n_modes, mp + 2 * n_modes, mp + 3 * n_modes, mp + 4 * n_modes,
                    mp + 5 * n_modes, mp + 6 * n_modes, n_modes, lam, inv_c0, sigma_nodes, n_sigma,
                    rho_nodes, n_rho, scratch, u_par, u_perp, du_dsigma, du_drho,
                    (cudaStream_t)stream);
  CHECK_LAUNCH("turbulence");
  return NWB_OK;
}

int nwb_ground_metrics(int precision, int batch, int n_rho, int n_theta, const void* v, int row,
                       int k0, int k1, const double* x, double* out, void* stream) {
  if (precision != NWB_F64 && precision != NWB_F32) return fail(NWB_EINVAL, "unknown precision");
  if (batch < 1 || n_rho < 1 || n_theta < 1) return fail(NWB_EINVAL, "empty field");
  if (row < 0 || row >= n_rho || k0 < 0 || k1 < k0 || k1 >= n_theta)
    return fail(NWB_EINVAL, "ground row / roi outside the grid");
  if (!v || !x || !out) return fail(NWB_EINVAL, "null buffer");
  cudaStream_t s = (cudaStream_t)stream;
  if (precision == NWB_F64)
    launch_ground_metrics<double>((const double*)v, batch, n_rho, n_theta, row, k0, k1 - k0 + 1, x,
                                  out, s);
  else
    launch_ground_metrics<float>((const float*)v, batch, n_rho, n_theta, row, k0, k1 - k0 + 1, x,
                                 out, s);
  CHECK_LAUNCH("ground_metrics");
  return NWB_OK;
}

int nwb_phi(const void* z, long long n, int shift, void* out, void* stream) {
  if (shift != 1 && shift != 2) return fail(NWB_EINVAL, "phi shift must be 1 or 2");
  if (n <= 0) return NWB_OK;
  launch_phi((const double2*)z, (long)n, shift, (double2*)out, (cudaStream_t)stream);
  CHECK_LAUNCH("phi");
  return NWB_OK;
}

int nwb_combine(int precision, long long n, int mode, double ds, const void* E, const void* P1,
                const void* P12, const void* P2, const void* vh, const void* b1, const void* b2,
                void* out, void* stream) {
  if ((mode & 7) > 3 || mode < 0 || mode > 15) return fail(NWB_EINVAL, "unknown combine mode");
  if (n <= 0) return NWB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (precision == NWB_F64)
    launch_combine<double>((long)n, mode, ds, (const double2*)E, (const double2*)P1, (const double2*)P12,
                           (const double2*)P2, (const double2*)vh, (const double2*)b1,
                           (const double2*)b2, (double2*)out, s);
  else
    launch_combine<float>((long)n, mode, ds, (const float2*)E, (const float2*)P1, (const float2*)P12,
                          (const float2*)P2, (const float2*)vh, (const float2*)b1, (const float2*)b2,
                          (float2*)out, s);
  CHECK_LAUNCH("combine");
  return NWB_OK;
}


int nwb_split_create(nwb_split** out, int n_nodes, int n_theta, double d_sigma, double d_rho,
                     double d_theta, double theta_span, double A, double B, int device) {
  if (!out) return fail(NWB_EINVAL, "null splitting plan pointer");
  *out = nullptr;
  if (n_nodes < 3 || n_theta < 2) return fail(NWB_EINVAL, "splitting: grid too small");
  if (n_theta % 2) return fail(NWB_EUNSUPPORTED, "n_theta must be even (half-length real FFT)");
  nwb_split* s = new nwb_split();
  s->device = device;
  s->n = n_nodes;
  s->nt = n_theta;
  s->ldn = (n_nodes + 31) / 32 * 32;
  s->g.nr = n_nodes;
  s->g.nt = n_theta;
  s->g.m = n_theta / 2;
  s->g.kk = n_theta / 2 + 1;
  s->g.ld = (n_nodes + 7) / 8 * 8;
  s->g.batch = 1;
  s->d_sigma = d_sigma;
  s->d_rho = d_rho;
  s->d_theta = d_theta;
  s->theta_span = theta_span;
  s->A = A;
  s->B = B;
  s->gamma = d_sigma * d_theta / (8.0 * 3.141592653589793 * (d_rho * d_rho));
  if (!plan_fft(s->g.m, 0, s->plan_h)) {
    delete s;
    return fail(NWB_EUNSUPPORTED, "n_theta/2 must factor into 2, 3, 5, 7");
  }
  const size_t row_bytes = (size_t)s->g.m * 16;
  s->theta_rows = 1;
  for (int r : {8, 4, 2})
    if ((size_t)r * row_bytes <= 64 * 1024 && (n_nodes + r - 1) / r >= 2 * 148) {
      s->theta_rows = r;
      break;
    }
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete s;
    return fail(NWB_ECUDA, std::string("splitting device/stream: ") + cudaGetErrorString(e));
  }
  s->stream = s->own_stream;
  keep_pool_memory(device);
  int rc = split_create_impl(s);
  if (rc != NWB_OK) {
    nwb_split_destroy(s);
    return rc;
  }
  *out = s;
  return NWB_OK;
}

int nwb_split_destroy(nwb_split* s) {
  if (!s) return NWB_OK;
  cudaSetDevice(s->device);
  cudaStreamSynchronize(s->stream);
  for (void* a : s->allocs)
    if (a) cudaFreeAsync(a, s->stream);
  if (s->hist) cudaFreeAsync(s->hist, s->stream);
  for (double* a : {s->upar, s->uperp, s->dus, s->dur})
    if (a) cudaFreeAsync(a, s->stream);
  cudaStreamSynchronize(s->stream);
  if (s->own_stream) cudaStreamDestroy(s->own_stream);
  delete s;
  return NWB_OK;
}

int nwb_split_set_stream(nwb_split* s, void* stream) {
  if (!s) return fail(NWB_EINVAL, "null splitting plan");
  s->stream = stream ? (cudaStream_t)stream : s->own_stream;
  return NWB_OK;
}

int nwb_split_set_coeffs(nwb_split* s, const double* u_par, const double* u_perp,
                         const double* du_dsigma, const double* du_drho, int n_rows, int ld,
                         int on_device) {
  if (!s) return fail(NWB_EINVAL, "null splitting plan");
  if (n_rows < 1 || ld < s->n) return fail(NWB_EINVAL, "splitting: coefficient rows / ld too small");
  CU(cudaSetDevice(s->device));
  for (double** a : {&s->upar, &s->uperp, &s->dus, &s->dur}) {
    if (*a) cudaFreeAsync(*a, s->stream);
    *a = nullptr;
  }
  const double* src[4] = {u_par, u_perp, du_dsigma, du_drho};
  double** dst[4] = {&s->upar, &s->uperp, &s->dus, &s->dur};
  for (int i = 0; i < 4; ++i) {
    CU(cudaMallocAsync((void**)dst[i], (size_t)n_rows * s->n * sizeof(double), s->stream));
    if (!src[i]) {
      CU(cudaMemsetAsync(*dst[i], 0, (size_t)n_rows * s->n * sizeof(double), s->stream));
      continue;
    }
    CU(cudaMemcpy2DAsync(*dst[i], s->n * sizeof(double), src[i], (size_t)ld * sizeof(double),
                         s->n * sizeof(double), n_rows,
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s->stream));
  }
  s->n_rows = n_rows;
  CU(cudaStreamSynchronize(s->stream));
  return NWB_OK;
}

int nwb_split_load(nwb_split* s, const double* v) {
  if (!s) return fail(NWB_EINVAL, "null splitting plan");
  CU(cudaSetDevice(s->device));
  CU(cudaMemcpyAsync(s->v, v, (size_t)s->n * s->nt * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));
  return NWB_OK;
}

int nwb_split_store(nwb_split* s, double* v) {
  if (!s) return fail(NWB_EINVAL, "null splitting plan");
  CU(cudaSetDevice(s->device));
  CU(cudaMemcpyAsync(v, s->v, (size_t)s->n * s->nt * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));
  return NWB_OK;
}

int nwb_split_stage(nwb_split* s, int stage, int sigma_row, const double* in, double* out) {
  if (!s) return fail(NWB_EINVAL, "null splitting plan");
  if (stage < 0 || stage > 4) return fail(NWB_EINVAL, "splitting: unknown stage");
  if (in == out) return fail(NWB_EINVAL, "splitting: stage in and out must differ");
  CU(cudaSetDevice(s->device));
  return split_stage(s, stage, sigma_row, in, out, nullptr);
}

int nwb_split_march(nwb_split* s, int n0, int n_steps, double guard, double max_seconds,
                    double* max_abs, int* fail_step, double* fail_value) {
  if (!s) return fail(NWB_EINVAL, "null splitting plan");
  CU(cudaSetDevice(s->device));
  return split_march_impl(s, n0, n_steps, guard, max_seconds, max_abs, fail_step, fail_value);
}

int nwb_godunov_flux(long long n, const double* u_l, const double* u_r, double B, double* out,
                     void* stream) {
  if (n < 0) return fail(NWB_EINVAL, "negative length");
  launch_godunov_flux((long)n, u_l, u_r, B, out, (cudaStream_t)stream);
  CHECK_LAUNCH("godunov_flux");
  return NWB_OK;
}

}  // extern "C"
