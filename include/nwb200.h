/*
 * nwb200 -- C ABI of the B200 ExpRK22/WENO5 step (libnwb200.so).
 *
 * This is the drop-in boundary for the hot path of the reference `nwave`
 * package (arXiv 2103.06080).  The reference binds no FFI of its own (its
 * path is Python + numba + scipy.fft); each entry point below replaces one
 * reference function, cited as file:line under /root/reference/pkg/src/nwave:
 *
 *   nwb_plan_create / nwb_plan_set_coeffs / nwb_plan_load_* / nwb_march /
 *   nwb_plan_store_physical             -> run_exprk22      exprk.py:219-331
 *   nwb_step (scheme)                   -> exprk22_step     exprk.py:151-178
 *                                          exp_euler_step   exprk.py:181-196
 *   nwb_rfft2 / nwb_irfft2              -> SpectralTransforms.forward/inverse
 *                                                           exprk.py:134-148
 *   nwb_tables                          -> build_multipliers exprk.py:111-131
 *   nwb_phi                             -> phi1 / phi2      exprk.py:42-84
 *   nwb_combine                         -> the numpy combines of exprk.py:166-173,193
 *   nwb_weno5_b                         -> weno5_b          weno.py:106-124
 *
 * Conventions.  Plain pointers and sizes only.  Buffer arguments named *_dev
 * are device pointers (the Python layer passes torch CUDA tensors'
 * data_ptr()); everything else is host memory.  Real arrays are float64 for
 * NWB_F64 plans and float32 for NWB_F32; complex arrays are interleaved
 * (re, im) pairs of the same real type.  Physical fields are
 * (batch, n_rho, n_theta) row-major; spectra handed across the boundary
 * are (batch, n_rho, n_theta/2 + 1) row-major in numpy.fft order, exactly
 * scipy's rfft2 layout.  A plan is bound to one device and one stream and is
 * not re-entrant; plans on different devices may be driven from different
 * host threads.
 *
 * Return codes: 0 on success, negative NWB_E* on failure; the message is
 * available from nwb_last_error() (thread-local).  The Python layer maps
 * NWB_EINVAL -> ValueError, NWB_EUNSUPPORTED -> UnsupportedSizeError,
 * NWB_EINSTABILITY -> InstabilityError, NWB_EBUDGET -> BudgetExceededError,
 * NWB_ECUDA / NWB_ENOMEM -> BackendError.
 */
#ifndef NWB200_H
#define NWB200_H

#ifdef __cplusplus
extern "C" {
#endif

#define NWB_OK 0
#define NWB_EINVAL (-1)
#define NWB_EUNSUPPORTED (-2)
#define NWB_ECUDA (-3)
#define NWB_ENOMEM (-4)
#define NWB_EINSTABILITY (-5)
#define NWB_EBUDGET (-6)

#define NWB_F64 0
#define NWB_F32 1

#define NWB_SCHEME_EXPRK22 0
#define NWB_SCHEME_EXPEULER 1

typedef struct nwb_plan nwb_plan;

int nwb_abi_version(void);
const char* nwb_last_error(void);
int nwb_device_count(void);

/* Plan: device tables (E, Phi1, Phi2, Phi1-Phi2 in digit-reversed rho order),
 * FFT twiddles, coefficient rows and all step workspaces for `batch`
 * independent members sharing one grid.  eps is the working-precision
 * machine epsilon used by the regularised multiplier (exprk.py:114-116).
 * Returns NWB_EUNSUPPORTED when n_rho or n_theta/2 has a prime factor above
 * 7, n_theta is odd, or a transform does not fit in shared memory. */
int nwb_plan_create(nwb_plan** plan, int n_rho, int n_theta, int batch, int precision,
                    double d_sigma, double rho_span, double theta_span, double A, double B,
                    double eps, int device);
int nwb_plan_destroy(nwb_plan* plan);
int nwb_plan_set_stream(nwb_plan* plan, void* stream);
/* Workspace footprint in bytes (device). */
long long nwb_plan_bytes(const nwb_plan* plan);

/* Coefficient rows U_par, U_perp, dU_perp/drho for sigma rows 0..n_rows-1,
 * row r at base + r*ld (ld >= n_rho; extra columns ignored, exprk.py:261-263).
 * Host float64 when on_device == 0, device float64 when 1.  They are cast to
 * the working precision and stay resident; alpha_rho per row is precomputed.
 * NULL pointers mean a quiescent medium (U = 0). */
int nwb_plan_set_coeffs(nwb_plan* plan, const double* u_par, const double* u_perp,
                        const double* du_drho, int n_rows, int ld, int on_device);

/* State in: physical V0 (batch, n_rho, n_theta) working precision, device. */
int nwb_plan_load_physical(nwb_plan* plan, const void* v0_dev);
/* State in/out: natural-order half spectrum (batch, n_rho, n_theta/2+1), device. */
int nwb_plan_load_spectrum(nwb_plan* plan, const void* vhat_dev);
int nwb_plan_store_spectrum(nwb_plan* plan, void* vhat_dev);
/* State out: V = irfft2(Vhat) (batch, n_rho, n_theta), device; max|V| per
 * member into max_abs_host (may be NULL). */
int nwb_plan_store_physical(nwb_plan* plan, void* v_dev, double* max_abs_host);

/* March n_steps steps from absolute step n0 (coefficient rows n0..n0+n_steps).
 *   snap_steps[i] / snap_bufs_dev[i]: copy V_n (the field at the start of
 *     step n, exprk.py:301-302) for the listed absolute steps into the given
 *     device buffers (batch, n_rho, n_theta).
 *   max_abs_host: [batch * n_steps] max|V_n| per member and step (or NULL).
 *   step_ms_host: [n_steps * 3] = (step, nonlinear, linear) device ms from
 *     %globaltimer stamps the march kernels write at entry (step start, WENO
 *     start, theta r2c start = WENO end, per stage; nonlinear = the WENO
 *     time like exprk.py:176), read back once after the march; or NULL.  The
 *     same step graph is replayed either way.
 *   guard: stop with NWB_EINSTABILITY at the first step whose max|V_n| is
 *     non-finite or > guard; *fail_step, *fail_member, *fail_value say where
 *     (the message carries "step=<n> member=<i> max_abs=<v>").
 *   max_seconds >= 0: stop with NWB_EBUDGET once the host wall clock exceeds
 *     it (checked after step 1 and then every 8 steps, so a zero budget stops
 *     after step 1 like exprk.py:303-306); < 0: no budget.
 *     *fail_step = absolute steps completed. */
int nwb_march(nwb_plan* plan, int scheme, int n0, int n_steps, double guard,
              double max_seconds, const int* snap_steps, int n_snap,
              void* const* snap_bufs_dev, double* max_abs_host, float* step_ms_host,
              int* fail_step, int* fail_member, double* fail_value);

/* One step from absolute step n without guard bookkeeping (graph-free). */
int nwb_step(nwb_plan* plan, int scheme, int n);

/* Measurement hook: march n_steps more steps from n0 with a CUDA event
 * around every kernel and return the summed device ms per kernel slot:
 * kernel_ms[8] = stage-1 (c2r, weno, r2c, rho), stage-2 (c2r, weno, r2c, rho).
 * Requires a prior nwb_march covering [n0, n0 + n_steps). */
int nwb_profile_kernels(nwb_plan* plan, int scheme, int n0, int n_steps, float* kernel_ms);

/* SpectralTransforms: rfft2 (batch, n_rho, n_theta) real -> natural half
 * spectrum; irfft2 the inverse (Im of the theta DC / Nyquist bins dropped,
 * scaled 1/(n_rho n_theta)). */
int nwb_rfft2(nwb_plan* plan, const void* in_dev, void* out_dev);
int nwb_irfft2(nwb_plan* plan, const void* in_dev, void* out_dev);

/* weno5_b on (batch, n_rho, n_theta) (no plan, any extents): coefficient
 * vectors are length-n_rho device arrays in the working precision (shared by
 * all members); workspace_dev holds >= 8*(batch+1) bytes. */
int nwb_weno5_b(int precision, int batch, int n_rho, int n_theta, const void* v_dev,
                const void* u_par_dev, const void* u_perp_dev, const void* du_dev,
                double b_coef, double d_rho, double d_theta, void* out_dev,
                void* workspace_dev, void* stream);

/* ---- rho slabs: one large grid over G GPUs (BASELINE C5).
 * A rank owns rho rows [j0, j0+rows) (physical / theta side) and theta modes
 * [k0, k0+modes) (rho side).  Caller-owned buffers (device, working precision):
 *   theta side: spec_rows (n_theta/2+1, ld_rows) complex, v_ext (rows+6, n_theta)
 *               real with 3 halo rows above and below the owned rows, b (rows, n_theta)
 *   rho side:   bt / out / vh / u (modes, ld_rho) complex (vh, u digit-reversed)
 *   red: 2 x uint64 [alpha_theta bits, max|V| bits] (IEEE bits of non-negative
 *        doubles: an integer MAX all-reduce across ranks is exact).
 * The host performs the all-to-all between the layouts, the MAX all-reduce of
 * red and the halo exchange (paper_2103_06080_b200/slab.py).  Modes of
 * nwb_slab_rho: 0 stage 1, 1 stage 2, 2 exponential Euler, 3 init.
 * These replace the same reference functions as nwb_march (exprk.py:151-331,
 * weno.py:106-124) for a grid that does not fit one GPU. */
typedef struct nwb_slab nwb_slab;
int nwb_slab_create(nwb_slab** slab, int n_rho, int n_theta, int j0, int rows, int k0, int modes,
                    int precision, double d_sigma, double rho_span, double theta_span, double A,
                    double B, double eps, int device);
int nwb_slab_destroy(nwb_slab* slab);
int nwb_slab_set_stream(nwb_slab* slab, void* stream);
int nwb_slab_layout(const nwb_slab* slab, int* ld_rows, int* ld_rho);
/* rho-side transit layout of nwb_slab_rho's bt / out: with n_blocks > 0 the
 * rank-b block (modes x rows_b, rows [row_starts[b], row_starts[b+1])) is
 * stored contiguously at modes * row_starts[b] -- the all-to-all segments. */
int nwb_slab_set_blocks(nwb_slab* slab, int n_blocks, const int* row_starts);
int nwb_slab_set_coeffs(nwb_slab* slab, const double* u_par, const double* u_perp,
                        const double* du_drho, int n_rows, int ld, int on_device);
/* red == NULL: plain inverse transform (no reductions). */
int nwb_slab_theta_c2r(nwb_slab* slab, const void* spec_rows_dev, void* v_ext_dev, int sigma_row,
                       void* red_dev);
int nwb_slab_weno(nwb_slab* slab, const void* v_ext_dev, void* b_dev, int sigma_row,
                  const void* red_dev);
int nwb_slab_theta_r2c(nwb_slab* slab, const void* b_dev, void* spec_rows_dev);
int nwb_slab_rho(nwb_slab* slab, int mode, const void* bt_dev, void* out_dev, void* vh_dev,
                 void* u_dev);
/* nwb_slab_rho over the local theta modes [k_begin, k_end) only: the slab
 * march runs the rho pass in mode chunks so each chunk's all-to-all overlaps
 * the next chunk's transforms. */
int nwb_slab_rho_range(nwb_slab* slab, int mode, int k_begin, int k_end, const void* bt_dev,
                       void* out_dev, void* vh_dev, void* u_dev);

/* Standalone multiplier tables in natural (n_rho, n_theta/2+1) layout; any
 * output may be NULL.  z is always complex128. */
int nwb_tables(int precision, int n_rho, int n_theta, double rho_span, double theta_span,
               double d_sigma, double A, double eps, void* E_dev, void* P1_dev, void* P2_dev,
               void* P12_dev, void* z_dev, void* stream);
/* Random-mode velocity fields on the device (turbulence.py:145-203, SURVEY
 * row f1): mode_params_dev = [kx | ky | phase | amp1 | amp2 | w_ds | w_dr],
 * n_modes each (w_ds = -amp2 kx lam, w_dr = -amp2 ky lam); sigma/rho nodes
 * device float64; outputs (n_sigma, n_rho) device float64, scaled by inv_c0;
 * scratch_dev holds 2 (n_sigma + n_rho) n_modes doubles. */
int nwb_turbulence_fields(int n_modes, const double* mode_params_dev, double lam, double inv_c0,
                          const double* sigma_nodes_dev, int n_sigma, const double* rho_nodes_dev,
                          int n_rho, double* scratch_dev, double* u_par_dev, double* u_perp_dev,
                          double* du_dsigma_dev, double* du_drho_dev, void* stream);

/* Ground metrics of marched fields (builder metric of SURVEY
 * 8(d), host definition paper_2103_06080_b200/analysis.py ground_metrics):
 * for each member of v_dev (batch, n_rho, n_theta) in the working precision,
 * on row `row` restricted to theta indices [k0, k1] with node values
 * x_dev[0 .. k1-k0] (float64): out_dev[3 m + 0] = peak, [3 m + 1] = theta of
 * the first upward crossing of 0.1 peak, [3 m + 2] = theta of the next upward
 * crossing of 0.9 peak (NaN when absent), linearly interpolated, bitwise the
 * host arithmetic.  Replaces the host post-processing of the reference CLI's
 * snapshot path (cli.py:111-123 writes the field; the metric reads it). */
int nwb_ground_metrics(int precision, int batch, int n_rho, int n_theta, const void* v_dev, int row,
                       int k0, int k1, const double* x_dev, double* out_dev, void* stream);

/* phi_shift(z) for complex128 z (shift 1 or 2). */
int nwb_phi(const void* z_dev, long long n, int shift, void* out_dev, void* stream);
/* Elementwise combines with numpy rounding (no FMA):
 * mode 0: out = E*vh; 1: out = vh + (ds*P1)*b1; 2: out = vh + ds*(P12*b1 + P2*b2);
 * 3: out = E*vh + (ds*P1)*b1.  Adding 8 rounds complex products the way
 * numpy's AVX2/AVX-512 loops do (re = fma(ar, br, -(ai bi)),
 * im = fma(ar, bi, ai br)) instead of numpy's scalar loop. */
int nwb_combine(int precision, long long n, int mode, double d_sigma, const void* E_dev,
                const void* P1_dev, const void* P12_dev, const void* P2_dev,
                const void* vh_dev, const void* b1_dev, const void* b2_dev, void* out_dev,
                void* stream);

/*
 * Splitting baseline -> run_splitting / lie_step and the
 * stage functions of splitting.py:78-301.  Float64 only (the reference has
 * no precision switch).  Fields are (n_nodes, n_theta) row-major on the
 * closed rho grid (n_nodes = N_rho + 1); coefficient rows (n_rows, ld) cover
 * at least n_nodes entries each.
 *   nwb_split_stage: 0 step_diffraction_cn (splitting.py:138-145),
 *     1 step_burgers_godunov (:169-177), 2 step_axial_absorption_spectral
 *     (:180-201, coefficient row sigma_row), 3 step_transverse_lw (:204-223),
 *     4 lie_step (:233-250).
 *   nwb_split_march: n_steps Lie steps of the loaded state from step n0 with
 *     the divergence guard (max|V| per step to max_abs, host), the budget
 *     (max_seconds < 0: none) -- run_splitting :253-301.
 *   nwb_godunov_flux -> godunov_flux (:157-166) on device arrays.
 */
typedef struct nwb_split nwb_split;
int nwb_split_create(nwb_split** plan, int n_nodes, int n_theta, double d_sigma, double d_rho,
                     double d_theta, double theta_span, double A, double B, int device);
int nwb_split_destroy(nwb_split* plan);
int nwb_split_set_stream(nwb_split* plan, void* stream);
int nwb_split_set_coeffs(nwb_split* plan, const double* u_par, const double* u_perp,
                         const double* du_perp_dsigma, const double* du_perp_drho, int n_rows,
                         int ld, int on_device);
int nwb_split_load(nwb_split* plan, const double* v_dev);
int nwb_split_store(nwb_split* plan, double* v_dev);
int nwb_split_stage(nwb_split* plan, int stage, int sigma_row, const double* in_dev,
                    double* out_dev);
int nwb_split_march(nwb_split* plan, int n0, int n_steps, double guard, double max_seconds,
                    double* max_abs, int* fail_step, double* fail_value);
int nwb_godunov_flux(long long n, const double* u_l_dev, const double* u_r_dev, double B,
                     double* out_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif
