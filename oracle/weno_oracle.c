/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle, never on the product path.
 *
 * Plain-C restatement of the reference WENO5 right-hand side b(sigma, V)
 * (reference pkg/src/nwave/weno.py), used by tests/ and by bench.py's
 * cpu_baseline / --impl reference legs as the checker and the CPU timing.
 *
 *   face reconstruction   weno.py:25-37   (_upwind_face)
 *   theta divergence      weno.py:40-64   (_theta_divergence)
 *   rho divergence        weno.py:67-90   (_rho_divergence; no transpose copy
 *                                           here -- columns are gathered into a
 *                                           per-thread scratch line, which keeps
 *                                           the arithmetic identical)
 *   theta LF speed        weno.py:93-103  (_max_theta_speed, serial, fixed order)
 *   combine               weno.py:124     (du*v - div_theta - div_rho)
 *
 * Arithmetic order follows the Python source operation by operation and the
 * file is compiled with -ffp-contract=off, so the fp64 result is bitwise the
 * reference's (pinned by tests/golden).  The fp32 entry reproduces the
 * reference's numba typing: fp32 storage of the split fluxes, face sums and
 * divergences, fp64 intermediates wherever the Python source mixes in a
 * float64 literal or scalar.
 *
 * Parallelism: OpenMP over rows/columns (the reference's prange); each row
 * is written by one thread, so results do not depend on the thread count.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TWO_PI_D 6.283185307179586
static const double WENO_EPS = 1e-6;

static inline double face5(double a0, double a1, double a2, double a3, double a4) {
    double d0 = (a0 - 2.0 * a1) + a2, e0 = (a0 - 4.0 * a1) + 3.0 * a2;
    double d1 = (a1 - 2.0 * a2) + a3, e1 = a1 - a3;
    double d2 = (a2 - 2.0 * a3) + a4, e2 = (3.0 * a2 - 4.0 * a3) + a4;
    double s0 = 13.0 / 12.0 * (d0 * d0) + 0.25 * (e0 * e0);
    double s1 = 13.0 / 12.0 * (d1 * d1) + 0.25 * (e1 * e1);
    double s2 = 13.0 / 12.0 * (d2 * d2) + 0.25 * (e2 * e2);
    double t0 = WENO_EPS + s0, t1 = WENO_EPS + s1, t2 = WENO_EPS + s2;
    double w0 = 0.1 / (t0 * t0), w1 = 0.6 / (t1 * t1), w2 = 0.3 / (t2 * t2);
    double q0 = (2.0 * a0 - 7.0 * a1) + 11.0 * a2;
    double q1 = (-a1 + 5.0 * a2) + 2.0 * a3;
    double q2 = (2.0 * a2 + 5.0 * a3) - a4;
    return ((w0 * q0 + w1 * q1) + w2 * q2) / (6.0 * ((w0 + w1) + w2));
}

static inline int wrap(int i, int n) { int r = i % n; return r < 0 ? r + n : r; }

/* ---------------------------------------------------------------- fp64 */

/* one periodic line: flux split f+-(x) -> divergence written with stride */
static void line_div_f64(const double *fp, const double *fm, int n, double inv_dx,
                         double *fhat, double *out, long ostride) {
    for (int i = 0; i < n; ++i) {
        double plus = face5(fp[i], fp[i + 1], fp[i + 2], fp[i + 3], fp[i + 4]);
        double minus = face5(fm[i + 5], fm[i + 4], fm[i + 3], fm[i + 2], fm[i + 1]);
        fhat[i] = plus + minus;
    }
    out[0] = (fhat[0] - fhat[n - 1]) * inv_dx;
    for (int i = 1; i < n; ++i) out[(long)i * ostride] = (fhat[i] - fhat[i - 1]) * inv_dx;
}

double oracle_max_theta_speed_f64(const double *v, int nr, int nt, const double *u_par,
                                  double b) {
    double m = 0.0;
    for (int r = 0; r < nr; ++r) {
        double c = TWO_PI_D * u_par[r];
        const double *row = v + (long)r * nt;
        for (int i = 0; i < nt; ++i) {
            double s = fabs(c + b * row[i]);
            if (s > m) m = s;
        }
    }
    return m;
}

int oracle_weno5_b_f64(const double *v, int nr, int nt, const double *u_par,
                       const double *u_perp, const double *du, double b, double d_rho,
                       double d_theta, double *out, int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#endif
    double a_th = oracle_max_theta_speed_f64(v, nr, nt, u_par, b);
    double a_rh = 0.0;
    for (int j = 0; j < nr; ++j) if (fabs(u_perp[j]) > a_rh) a_rh = fabs(u_perp[j]);
    double inv_dt = 1.0 / d_theta, inv_dr = 1.0 / d_rho, half_b = 0.5 * b;
    double *dth = (double *)malloc(sizeof(double) * (size_t)nr * nt);
    double *drh = (double *)malloc(sizeof(double) * (size_t)nr * nt);
    if (!dth || !drh) { free(dth); free(drh); return -1; }
    int maxn = nr > nt ? nr : nt;
#pragma omp parallel
    {
        double *fp = (double *)malloc(sizeof(double) * (maxn + 5));
        double *fm = (double *)malloc(sizeof(double) * (maxn + 5));
        double *fh = (double *)malloc(sizeof(double) * maxn);
        double *tmp = (double *)malloc(sizeof(double) * maxn);
#pragma omp for schedule(static)
        for (int r = 0; r < nr; ++r) {
            double c = TWO_PI_D * u_par[r];
            for (int idx = -2; idx < nt + 3; ++idx) {
                double vv = v[(long)r * nt + wrap(idx, nt)];
                double g = -c * vv - half_b * vv * vv;
                double av = a_th * vv;
                fp[idx + 2] = 0.5 * (g + av);
                fm[idx + 2] = 0.5 * (g - av);
            }
            line_div_f64(fp, fm, nt, inv_dt, fh, dth + (long)r * nt, 1);
        }
#pragma omp for schedule(static)
        for (int k = 0; k < nt; ++k) {
            for (int idx = -2; idx < nr + 3; ++idx) {
                int pos = wrap(idx, nr);
                double vv = v[(long)pos * nt + k];
                double g = u_perp[pos] * vv;
                double av = a_rh * vv;
                fp[idx + 2] = 0.5 * (g + av);
                fm[idx + 2] = 0.5 * (g - av);
            }
            line_div_f64(fp, fm, nr, inv_dr, fh, tmp, 1);
            for (int j = 0; j < nr; ++j) drh[(long)j * nt + k] = tmp[j];
        }
#pragma omp for schedule(static)
        for (int r = 0; r < nr; ++r)
            for (int i = 0; i < nt; ++i) {
                long o = (long)r * nt + i;
                out[o] = (du[r] * v[o] - dth[o]) - drh[o];
            }
        free(fp); free(fm); free(fh); free(tmp);
    }
    free(dth); free(drh);
    return 0;
}

/* ---------------------------------------------------------------- fp32 */
/* numba typing of the reference with float32 arrays: see header comment.
 * Every subexpression that mixes in a float64 literal is evaluated in fp64;
 * (a1 - a3) ** 2 involves only float32 operands and stays in fp32. */
static inline double face5_f32(float a0, float a1, float a2, float a3, float a4) {
    double d0 = (a0 - 2.0 * a1) + a2, e0 = (a0 - 4.0 * a1) + 3.0 * a2;
    double d1 = (a1 - 2.0 * a2) + a3;
    float e1 = a1 - a3;
    double d2 = (a2 - 2.0 * a3) + a4, e2 = (3.0 * a2 - 4.0 * a3) + a4;
    double s0 = 13.0 / 12.0 * (d0 * d0) + 0.25 * (e0 * e0);
    double s1 = 13.0 / 12.0 * (d1 * d1) + 0.25 * (double)(e1 * e1);
    double s2 = 13.0 / 12.0 * (d2 * d2) + 0.25 * (e2 * e2);
    double t0 = WENO_EPS + s0, t1 = WENO_EPS + s1, t2 = WENO_EPS + s2;
    double w0 = 0.1 / (t0 * t0), w1 = 0.6 / (t1 * t1), w2 = 0.3 / (t2 * t2);
    double q0 = (2.0 * a0 - 7.0 * a1) + 11.0 * a2;
    double q1 = ((double)(-a1) + 5.0 * a2) + 2.0 * a3;
    double q2 = (2.0 * a2 + 5.0 * a3) - a4;
    return ((w0 * q0 + w1 * q1) + w2 * q2) / (6.0 * ((w0 + w1) + w2));
}

static void line_div_f32(const float *fp, const float *fm, int n, double inv_dx,
                         float *fhat, float *out) {
    for (int i = 0; i < n; ++i) {
        double plus = face5_f32(fp[i], fp[i + 1], fp[i + 2], fp[i + 3], fp[i + 4]);
        double minus = face5_f32(fm[i + 5], fm[i + 4], fm[i + 3], fm[i + 2], fm[i + 1]);
        fhat[i] = (float)(plus + minus);
    }
    out[0] = (float)((double)(fhat[0] - fhat[n - 1]) * inv_dx);
    for (int i = 1; i < n; ++i) out[i] = (float)((double)(fhat[i] - fhat[i - 1]) * inv_dx);
}

int oracle_weno5_b_f32(const float *v, int nr, int nt, const float *u_par,
                       const float *u_perp, const float *du, float b, double d_rho,
                       double d_theta, float *out, int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#endif
    double a_th = 0.0;
    for (int r = 0; r < nr; ++r) {
        double c = TWO_PI_D * (double)u_par[r];
        for (int i = 0; i < nt; ++i) {
            double s = fabs(c + (double)(b * v[(long)r * nt + i]));
            if (s > a_th) a_th = s;
        }
    }
    float a_rh_f = 0.0f;
    for (int j = 0; j < nr; ++j) if (fabsf(u_perp[j]) > a_rh_f) a_rh_f = fabsf(u_perp[j]);
    double a_rh = (double)a_rh_f;
    double inv_dt = 1.0 / d_theta, inv_dr = 1.0 / d_rho, half_b = 0.5 * (double)b;
    float *dth = (float *)malloc(sizeof(float) * (size_t)nr * nt);
    float *drh = (float *)malloc(sizeof(float) * (size_t)nr * nt);
    if (!dth || !drh) { free(dth); free(drh); return -1; }
    int maxn = nr > nt ? nr : nt;
#pragma omp parallel
    {
        float *fp = (float *)malloc(sizeof(float) * (maxn + 5));
        float *fm = (float *)malloc(sizeof(float) * (maxn + 5));
        float *fh = (float *)malloc(sizeof(float) * maxn);
        float *tmp = (float *)malloc(sizeof(float) * maxn);
#pragma omp for schedule(static)
        for (int r = 0; r < nr; ++r) {
            double c = TWO_PI_D * (double)u_par[r];
            for (int idx = -2; idx < nt + 3; ++idx) {
                double vv = v[(long)r * nt + wrap(idx, nt)];
                double g = -c * vv - half_b * vv * vv;
                double av = a_th * vv;
                fp[idx + 2] = (float)(0.5 * (g + av));
                fm[idx + 2] = (float)(0.5 * (g - av));
            }
            line_div_f32(fp, fm, nt, inv_dt, fh, dth + (long)r * nt);
        }
#pragma omp for schedule(static)
        for (int k = 0; k < nt; ++k) {
            for (int idx = -2; idx < nr + 3; ++idx) {
                int pos = wrap(idx, nr);
                float vv = v[(long)pos * nt + k];
                double g = (double)(u_perp[pos] * vv);
                double av = a_rh * (double)vv;
                fp[idx + 2] = (float)(0.5 * (g + av));
                fm[idx + 2] = (float)(0.5 * (g - av));
            }
            line_div_f32(fp, fm, nr, inv_dr, fh, tmp);
            for (int j = 0; j < nr; ++j) drh[(long)j * nt + k] = tmp[j];
        }
#pragma omp for schedule(static)
        for (int r = 0; r < nr; ++r)
            for (int i = 0; i < nt; ++i) {
                long o = (long)r * nt + i;
                out[o] = (du[r] * v[o] - dth[o]) - drh[o];
            }
        free(fp); free(fm); free(fh); free(tmp);
    }
    free(dth); free(drh);
    return 0;
}
