/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (see oracle.h for the rules).
 *
 * Plain fp64 C, compiled with -ffp-contract=off (no FMA contraction), triple
 * loops with periodic modular indexing, textbook RK4 with four k arrays, and
 * Alg.1 emulated rank by rank.  OpenMP (optional) only splits the outer z
 * loop; every point is computed independently and max is exact, so results do
 * not depend on the thread count.
 *
 * Readings of places where the paper is silent or garbled:
 *   C1  nu inside an RK4 step: nu_mode 0 = stage times t_j, t_j+dt/2, t_j+dt/2,
 *       t_j+dt; nu_mode 1 = nu(t_j) for all four stages.
 *   C2  nu in the Euler step: nu(t_j), the step start.
 *   C3  4th-order weights: standard central (-1,16,-30,16,-1)/12dx^2 and
 *       (-1,8,0,-8,1)/12dx on offsets (+2,+1,0,-1,-2).
 *   C4  upwind branch: strict c > 0 exactly as Alg.2 prints.
 *   C5  correction evaluated as  u_hat + (u_tilde_new - u_tilde_old).
 *   C6  times from global integer step indices: t_j = j*dt.
 *   C8  Alg.2 performs exactly N_c steps with u <- u_tilde after each.
 *   C9  rank p runs p+1 coarse slice sweeps during the initialisation.
 *   C17 Laplacian misprint u_{i,j1,k+1} read as u_{i,j,k+1}.
 *   C18 a(t) misprint at P:441 read with the exp of P:433.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static inline int64_t wrap(int64_t i, int64_t n) { return ((i % n) + n) % n; }

/* u_{i,j,k} with periodic boundary conditions. */
static inline double at(const double *u, int64_t n, int64_t i, int64_t j,
                        int64_t k) {
    return u[(wrap(k, n) * n + wrap(j, n)) * n + wrap(i, n)];
}

int orc_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* nu(t) = nu0 + (nu0/2) sin(omega t). */
double orc_nu(double nu0, double omega, double t) {
    return nu0 + (nu0 / 2.0) * sin(omega * t);
}

/* P:433 a(t) = exp(-int_0^t 12 pi^2 nu(s) ds) with the P:437 profile:
 * int_0^t nu = nu0 t + nu0/(2 omega) (1 - cos(omega t)); omega = 0 -> nu0 t. */
double orc_amplitude(double nu0, double omega, double t) {
    double integral = nu0 * t;
    if (omega != 0.0) integral += nu0 / (2.0 * omega) * (1.0 - cos(omega * t));
    return exp(-12.0 * M_PI * M_PI * integral);
}

/* P:418-420, vertex-centred sampling x_i = i dx (C16). */
void orc_initial(int32_t n, double *u) {
    const double dx = 1.0 / n;
    for (int64_t k = 0; k < n; ++k)
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) {
                double x = i * dx, y = j * dx, z = k * dx;
                u[(k * n + j) * n + i] =
                    sin(2.0 * M_PI * x) * sin(2.0 * M_PI * y) * sin(2.0 * M_PI * z);
            }
}

/* u(x, t) = a(t) u0(x - c t); sin is 2 pi periodic so the shifted
 * coordinate needs no explicit wrap. */
void orc_exact(const orc_problem *p, double t, double *u) {
    const int64_t n = p->n;
    const double dx = 1.0 / n;
    const double a = orc_amplitude(p->nu0, p->omega, t);
    for (int64_t k = 0; k < n; ++k)
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) {
                double x = i * dx - p->c[0] * t;
                double y = j * dx - p->c[1] * t;
                double z = k * dx - p->c[2] * t;
                u[(k * n + j) * n + i] = a * (sin(2.0 * M_PI * x) *
                                              sin(2.0 * M_PI * y) *
                                              sin(2.0 * M_PI * z));
            }
}

/* Alg.2, written line by line.  Indices: i = x, j = y, k = z. */
void orc_rhs_coarse(int32_t n_, const double c[3], double nu, const double *u,
                    double *rhs) {
    const int64_t n = n_;
    const double dx = 1.0 / n;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k)
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) {
                const double uc = at(u, n, i, j, k);
                double r = nu *
                           (at(u, n, i + 1, j, k) + at(u, n, i - 1, j, k) +
                            at(u, n, i, j + 1, k) + at(u, n, i, j - 1, k) +
                            at(u, n, i, j, k + 1) + at(u, n, i, j, k - 1) -
                            6.0 * uc) /
                           (dx * dx);
                if (c[0] > 0)
                    r -= c[0] * (uc - at(u, n, i - 1, j, k)) / dx;
                else
                    r -= c[0] * (at(u, n, i + 1, j, k) - uc) / dx;
                if (c[1] > 0)
                    r -= c[1] * (uc - at(u, n, i, j - 1, k)) / dx;
                else
                    r -= c[1] * (at(u, n, i, j + 1, k) - uc) / dx;
                if (c[2] > 0)
                    r -= c[2] * (uc - at(u, n, i, j, k - 1)) / dx;
                else
                    r -= c[2] * (at(u, n, i, j, k + 1) - uc) / dx;
                rhs[(k * n + j) * n + i] = r;
            }
}

/* Second derivative, 4th-order central: (-u+2 + 16u+1 - 30u + 16u-1 - u-2)/(12dx^2) */
static inline double d2(double m2, double m1, double c0, double p1, double p2,
                        double dx) {
    return (-p2 + 16.0 * p1 - 30.0 * c0 + 16.0 * m1 - m2) / (12.0 * dx * dx);
}
/* First derivative, 4th-order central: (-u+2 + 8u+1 - 8u-1 + u-2)/(12dx) */
static inline double d1(double m2, double m1, double p1, double p2, double dx) {
    return (-p2 + 8.0 * p1 - 8.0 * m1 + m2) / (12.0 * dx);
}

/* P:342 / P:455: nu Lap4(u) - c . Grad4(u), "fourth order differences for both
 * advection and diffusion". */
void orc_rhs_fine(int32_t n_, const double c[3], double nu, const double *u,
                  double *rhs) {
    const int64_t n = n_;
    const double dx = 1.0 / n;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k)
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) {
                const double uc = at(u, n, i, j, k);
                const double xm2 = at(u, n, i - 2, j, k), xm1 = at(u, n, i - 1, j, k);
                const double xp1 = at(u, n, i + 1, j, k), xp2 = at(u, n, i + 2, j, k);
                const double ym2 = at(u, n, i, j - 2, k), ym1 = at(u, n, i, j - 1, k);
                const double yp1 = at(u, n, i, j + 1, k), yp2 = at(u, n, i, j + 2, k);
                const double zm2 = at(u, n, i, j, k - 2), zm1 = at(u, n, i, j, k - 1);
                const double zp1 = at(u, n, i, j, k + 1), zp2 = at(u, n, i, j, k + 2);
                const double lap = d2(xm2, xm1, uc, xp1, xp2, dx) +
                                   d2(ym2, ym1, uc, yp1, yp2, dx) +
                                   d2(zm2, zm1, uc, zp1, zp2, dx);
                const double adv = c[0] * d1(xm2, xm1, xp1, xp2, dx) +
                                   c[1] * d1(ym2, ym1, yp1, yp2, dx) +
                                   c[2] * d1(zm2, zm1, zp1, zp2, dx);
                rhs[(k * n + j) * n + i] = nu * lap - adv;
            }
}

static double *alloc_field(int64_t n) {
    return (double *)malloc(sizeof(double) * (size_t)(n * n * n));
}

/* Alg.2: N_c forward-Euler steps; nu at the step start (C2),
 * t_j = j dt from the global step index (C6). */
void orc_coarse(const orc_problem *p, double *u, int64_t step0, int64_t n_steps,
                double dt) {
    const int64_t n = p->n, N = n * n * n;
    double *rhs = alloc_field(n);
    for (int64_t j = step0; j < step0 + n_steps; ++j) {
        const double nu = orc_nu(p->nu0, p->omega, (double)j * dt);
        orc_rhs_coarse(p->n, p->c, nu, u, rhs);
        for (int64_t q = 0; q < N; ++q) u[q] = u[q] + dt * rhs[q];
    }
    free(rhs);
}

/* Restriction by injection (C24): the n/2 mesh points x_i = i/(n/2) are the
 * even fine points. */
void orc_restrict(int32_t n_, const double *u, double *uc) {
    const int64_t n = n_, m = n / 2;
    for (int64_t k = 0; k < m; ++k)
        for (int64_t j = 0; j < m; ++j)
            for (int64_t i = 0; i < m; ++i)
                uc[(k * m + j) * m + i] = u[((2 * k) * n + 2 * j) * n + 2 * i];
}

/* Trilinear prolongation (C25), written as the average over the coarse
 * neighbours of every fine point: along an axis with even fine index the one
 * coarse point i/2, along an odd one the two points (i-1)/2 and (i+1)/2
 * (periodic).  The sum runs over the 1, 2, 4 or 8 combinations in the order
 * z-, y-, x-candidate (outer to inner) and is divided by their count. */
void orc_prolong(int32_t n_, const double *uc, double *u) {
    const int64_t n = n_, m = n / 2;
    for (int64_t k = 0; k < n; ++k)
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) {
                int64_t ks[2], js[2], is[2];
                const int nk = (k % 2) ? 2 : 1, nj = (j % 2) ? 2 : 1, ni = (i % 2) ? 2 : 1;
                ks[0] = k / 2; ks[1] = (k / 2 + 1) % m;
                js[0] = j / 2; js[1] = (j / 2 + 1) % m;
                is[0] = i / 2; is[1] = (i / 2 + 1) % m;
                double sum = 0.0;
                for (int a = 0; a < nk; ++a)
                    for (int b = 0; b < nj; ++b)
                        for (int c = 0; c < ni; ++c)
                            sum += uc[(ks[a] * m + js[b]) * m + is[c]];
                u[(k * n + j) * n + i] = sum / (double)(nk * nj * ni);
            }
}

/* G_c (C26): restrict, Alg.2 on the n/2 mesh (dx = 2/n, same dt and nu_j),
 * prolongate; u (fine mesh) is overwritten. */
void orc_coarse_mesh(const orc_problem *p, double *u, int64_t step0, int64_t n_steps,
                     double dt) {
    const int64_t m = p->n / 2;
    double *uc = (double *)malloc(sizeof(double) * (size_t)(m * m * m));
    orc_problem pc = *p;
    pc.n = (int32_t)m;
    orc_restrict(p->n, u, uc);
    orc_coarse(&pc, uc, step0, n_steps, dt);
    orc_prolong(p->n, uc, u);
    free(uc);
}

/* Classical RK4:
 *   k1 = f(u, t1), k2 = f(u + dt/2 k1, t2), k3 = f(u + dt/2 k2, t3),
 *   k4 = f(u + dt k3, t4),  u <- u + dt/6 (k1 + 2 k2 + 2 k3 + k4). */
void orc_fine(const orc_problem *p, double *u, int64_t step0, int64_t n_steps,
              double dt) {
    const int64_t n = p->n, N = n * n * n;
    double *k1 = alloc_field(n), *k2 = alloc_field(n), *k3 = alloc_field(n),
           *k4 = alloc_field(n), *y = alloc_field(n);
    for (int64_t j = step0; j < step0 + n_steps; ++j) {
        double nu1, nu2, nu3, nu4;
        if (p->nu_mode == 1) { /* C1, step_start reading */
            nu1 = nu2 = nu3 = nu4 = orc_nu(p->nu0, p->omega, (double)j * dt);
        } else { /* C1, stage-time reading */
            nu1 = orc_nu(p->nu0, p->omega, (double)j * dt);
            nu2 = nu3 = orc_nu(p->nu0, p->omega, ((double)j + 0.5) * dt);
            nu4 = orc_nu(p->nu0, p->omega, ((double)j + 1.0) * dt);
        }
        orc_rhs_fine(p->n, p->c, nu1, u, k1);
        for (int64_t q = 0; q < N; ++q) y[q] = u[q] + dt / 2.0 * k1[q];
        orc_rhs_fine(p->n, p->c, nu2, y, k2);
        for (int64_t q = 0; q < N; ++q) y[q] = u[q] + dt / 2.0 * k2[q];
        orc_rhs_fine(p->n, p->c, nu3, y, k3);
        for (int64_t q = 0; q < N; ++q) y[q] = u[q] + dt * k3[q];
        orc_rhs_fine(p->n, p->c, nu4, y, k4);
        for (int64_t q = 0; q < N; ++q)
            u[q] = u[q] + dt / 6.0 * (k1[q] + 2.0 * k2[q] + 2.0 * k3[q] + k4[q]);
    }
    free(k1); free(k2); free(k3); free(k4); free(y);
}

double orc_inf_norm(int32_t n_, const double *u) {
    const int64_t N = (int64_t)n_ * n_ * n_;
    double m = 0.0;
    for (int64_t q = 0; q < N; ++q) {
        double a = fabs(u[q]);
        if (a > m || a != a) m = a; /* NaN propagates */
        if (m != m) break;
    }
    return m;
}

double orc_inf_diff(int32_t n_, const double *u, const double *v) {
    const int64_t N = (int64_t)n_ * n_ * n_;
    double m = 0.0;
    for (int64_t q = 0; q < N; ++q) {
        double a = fabs(u[q] - v[q]);
        if (a > m || a != a) m = a;
        if (m != m) break;
    }
    return m;
}

/* Eq.(defect) P:291. */
double orc_defect(int32_t n, const double *u, const double *ref) {
    return orc_inf_diff(n, u, ref) / orc_inf_norm(n, ref);
}

/* Slice propagators over time slice m. */
static void G_slice(const orc_problem *p, int32_t flags, double *u, int64_t m,
                    int64_t nc, int64_t nf, double Dt, double dt) {
    if (flags & 1)
        orc_fine(p, u, m * nf, nf, dt); /* degenerate test: G := F */
    else if (flags & 4)
        orc_coarse_mesh(p, u, m * nc, nc, Dt); /* G_c on the n/2 mesh (NEXT-4) */
    else
        orc_coarse(p, u, m * nc, nc, Dt);
}
static void F_slice(const orc_problem *p, double *u, int64_t m, int64_t nf,
                    double dt) {
    orc_fine(p, u, m * nf, nf, dt);
}

/* Alg.1, every rank p executed in order within each iteration,
 * which is the order the pipelined run's data dependencies impose. */
int orc_parareal(const orc_problem *p, int32_t n_slices, int32_t nc_, int32_t nf_,
                 int32_t K, const double *u0, const double *u_ref, double *u_T,
                 double *defects, int32_t flags) {
    if (!p || !u0 || !u_T || n_slices < 1 || nc_ < 1 || nf_ < 1 || K < 0 || p->n < 1 ||
        ((flags & 4) && p->n % 4))
        return -1;
    const int64_t n = p->n, N = n * n * n, Np = n_slices, nc = nc_, nf = nf_;
    const double Dt = p->T / (double)(Np * nc); /* coarse step  Delta t */
    const double dt = p->T / (double)(Np * nf); /* fine step    delta t */
    const size_t bytes = sizeof(double) * (size_t)N;

    /* Per-rank state (Alg.1 variables): u^k_p, u~^k_{p+1}, and the message
     * u^{k+1}_{p+1} that rank p sends to rank p+1. */
    double **u_p = (double **)calloc((size_t)Np, sizeof(double *));
    double **ut_old = (double **)calloc((size_t)Np, sizeof(double *));
    double *msg = alloc_field(n), *uhat = alloc_field(n), *ut_new = alloc_field(n),
           *u_in = alloc_field(n);
    int ok = u_p && ut_old && msg && uhat && ut_new && u_in;
    for (int64_t r = 0; ok && r < Np; ++r) {
        u_p[r] = alloc_field(n);
        ut_old[r] = alloc_field(n);
        ok = u_p[r] && ut_old[r];
    }
    if (!ok) {
        if (u_p) for (int64_t r = 0; r < Np; ++r) free(u_p[r]);
        if (ut_old) for (int64_t r = 0; r < Np; ++r) free(ut_old[r]);
        free(u_p); free(ut_old); free(msg); free(uhat); free(ut_new); free(u_in);
        return -1;
    }

    /* Initialisation (Alg.1 lines 1-4): rank p applies G over slices
     * 0..p-1 to u0 (u^0_p), then once more over its own slice (u~^0_{p+1}). */
    for (int64_t r = 0; r < Np; ++r) {
        memcpy(u_p[r], u0, bytes);
        for (int64_t m = 0; m < r; ++m) G_slice(p, flags, u_p[r], m, nc, nf, Dt, dt);
        memcpy(ut_old[r], u_p[r], bytes);
        G_slice(p, flags, ut_old[r], r, nc, nf, Dt, dt);
    }
    if (defects && u_ref) defects[0] = orc_defect(p->n, ut_old[Np - 1], u_ref);

    for (int32_t k = 0; k < K; ++k) {
        for (int64_t r = 0; r < Np; ++r) {
            /* fine propagator on the old initial value (line alg_para_fine) */
            memcpy(uhat, u_p[r], bytes);
            F_slice(p, uhat, r, nf, dt);
            /* receive u^{k+1}_p, or u0 on rank 0 (lines P:185-188) */
            if (r == 0)
                memcpy(u_in, u0, bytes);
            else
                memcpy(u_in, msg, bytes);
            /* coarse propagator on the new initial value (line alg_para_coarse3) */
            memcpy(ut_new, u_in, bytes);
            G_slice(p, flags, ut_new, r, nc, nf, Dt, dt);
            /* correction (line alg_para_corr), order C5 */
            for (int64_t q = 0; q < N; ++q)
                msg[q] = uhat[q] + (ut_new[q] - ut_old[r][q]);
            /* state for the next iteration */
            memcpy(ut_old[r], ut_new, bytes);
            memcpy(u_p[r], u_in, bytes);
            /* "send" to rank r+1 = msg is read by the next r in this loop */
        }
        if (defects && u_ref) defects[k + 1] = orc_defect(p->n, msg, u_ref);
    }
    memcpy(u_T, K > 0 ? msg : ut_old[Np - 1], bytes);

    for (int64_t r = 0; r < Np; ++r) { free(u_p[r]); free(ut_old[r]); }
    free(u_p); free(ut_old); free(msg); free(uhat); free(ut_new); free(u_in);
    return 0;
}

/* Alg.1 with the stop rule of DESIGN.md C23 (see oracle.h), ranks of s slices
 * executed in pipeline order: iteration-major, rank-minor. */
int orc_parareal_tol(const orc_problem *p, int32_t n_slices, int32_t nc_, int32_t nf_, int32_t K,
                     double tol, int32_t world, const double *u0, const double *u_ref,
                     double *u_T, double *defects, double *changes, int32_t *iters,
                     int32_t flags) {
    if (!p || !u0 || !u_T || n_slices < 1 || nc_ < 1 || nf_ < 1 || K < 0 || world < 1 ||
        n_slices % world || p->n < 1 || !(tol >= 0.0) || ((flags & 4) && p->n % 4))
        return -1;
    const int64_t n = p->n, N = n * n * n, Np = n_slices, nc = nc_, nf = nf_, W = world,
                  s = n_slices / world;
    const double Dt = p->T / (double)(Np * nc), dt = p->T / (double)(Np * nf);
    const size_t bytes = sizeof(double) * (size_t)N;
    double **u_p = (double **)calloc((size_t)Np, sizeof(double *));    /* u^k_j (slice start) */
    double **ut_old = (double **)calloc((size_t)Np, sizeof(double *)); /* u~^k_{j+1} */
    double **out = (double **)calloc((size_t)Np, sizeof(double *));    /* u^k_{j+1} (slice end) */
    double *uhat = alloc_field(n), *ut_new = alloc_field(n), *u_in = alloc_field(n),
           *neu = alloc_field(n);
    int *stopped = (int *)calloc((size_t)W, sizeof(int));
    int ok = u_p && ut_old && out && uhat && ut_new && u_in && neu && stopped;
    for (int64_t j = 0; ok && j < Np; ++j) {
        u_p[j] = alloc_field(n);
        ut_old[j] = alloc_field(n);
        out[j] = alloc_field(n);
        ok = u_p[j] && ut_old[j] && out[j];
    }
    if (ok) {
        /* initialisation: rank r's prefix sweeps give the same values as one
         * serial coarse sweep (same arithmetic per slice) */
        memcpy(u_p[0], u0, bytes);
        for (int64_t j = 0; j < Np; ++j) {
            memcpy(ut_old[j], u_p[j], bytes);
            G_slice(p, flags, ut_old[j], j, nc, nf, Dt, dt);
            memcpy(out[j], ut_old[j], bytes);
            if (j + 1 < Np) memcpy(u_p[j + 1], ut_old[j], bytes);
        }
        if (defects && u_ref) {
            defects[0] = orc_defect(p->n, out[Np - 1], u_ref);
            for (int32_t k = 1; k <= K; ++k) defects[k] = NAN;
        }
        if (changes)
            for (int64_t i = 0; i < W * K; ++i) changes[i] = NAN;
        if (iters)
            for (int64_t r = 0; r < W; ++r) iters[r] = 0;
        for (int32_t k = 0; k < K; ++k) {
            for (int64_t r = 0; r < W; ++r) {
                if (stopped[r]) continue;
                double dmax = 0.0, umax = 0.0;
                /* F of every own slice on its old start value, before any update */
                for (int64_t l = 0; l < s; ++l) {
                    const int64_t j = r * s + l;
                    memcpy(uhat, u_p[j], bytes);
                    F_slice(p, uhat, j, nf, dt);
                    /* input: u0, the predecessor's value of this iteration (or its
                     * last one once it stopped), or this rank's previous slice */
                    if (j == 0) memcpy(u_in, u0, bytes);
                    else memcpy(u_in, out[j - 1], bytes);
                    memcpy(ut_new, u_in, bytes);
                    G_slice(p, flags, ut_new, j, nc, nf, Dt, dt);
                    for (int64_t q = 0; q < N; ++q) neu[q] = uhat[q] + (ut_new[q] - ut_old[j][q]);
                    const double dm = orc_inf_diff(p->n, neu, out[j]), um = orc_inf_norm(p->n, neu);
                    if (dm > dmax || dm != dm) dmax = dm;
                    if (um > umax) umax = um;
                    memcpy(ut_old[j], ut_new, bytes);
                    memcpy(u_p[j], u_in, bytes);
                    memcpy(out[j], neu, bytes);
                }
                const double ch = umax > 0.0 ? dmax / umax : dmax;
                if (changes) changes[r * K + k] = ch;
                if (iters) iters[r] = k + 1;
                const int pred_done = (r == 0) || stopped[r - 1];
                if (k == K - 1 || (tol > 0.0 && pred_done && ch <= tol)) stopped[r] = 1;
                if (r == W - 1 && defects && u_ref) defects[k + 1] = orc_defect(p->n, out[Np - 1], u_ref);
            }
        }
        memcpy(u_T, out[Np - 1], bytes);
    }
    for (int64_t j = 0; j < Np; ++j) {
        if (u_p) free(u_p[j]);
        if (ut_old) free(ut_old[j]);
        if (out) free(out[j]);
    }
    free(u_p); free(ut_old); free(out); free(uhat); free(ut_new); free(u_in); free(neu);
    free(stopped);
    return ok ? 0 : -1;
}
