/*
 * oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the hot path of
 * Arteaga, Ruprecht & Krause, "A stencil-based implementation of Parareal in
 * the C++ domain specific embedded language STELLA" (arXiv:1409.8563).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library.  The product path
 * (paper_1409_8563_b200/) never includes, links or calls it, and this file
 * includes nothing from the product path.
 *
 * Citations: P:NNN = line NNN of the paper text, with the
 * section / equation / algorithm it falls in.
 *
 * Field layout: n^3 doubles, index ((k*n + j)*n + i), i = x (fastest),
 * j = y, k = z; grid points x_i = i/n on the periodic unit cube.
 */
#ifndef PARAREAL_ORACLE_H
#define PARAREAL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Eq.(adv_diff_eq) P:414 with nu(t) profile P:437 and the T of P:448. */
typedef struct {
    int32_t n;         /* points per axis, dx = 1/n */
    double c[3];       /* advection velocity */
    double nu0;        /* nu_0 */
    double omega;      /* omega */
    double T;          /* end time */
    int32_t nu_mode;   /* 0 = RK4 stage times, 1 = nu frozen at the step start */
} orc_problem;

/* nu(t) = nu0 + nu0/2 sin(omega t) */
double orc_nu(double nu0, double omega, double t);
/* a(t) = exp(-12 pi^2 int_0^t nu)  (the exp missing at P:441 restored) */
double orc_amplitude(double nu0, double omega, double t);

/* u0 = sin(2 pi x) sin(2 pi y) sin(2 pi z) */
void orc_initial(int32_t n, double *u);
/* u_ex(x, t) = a(t) u0(x - c t) */
void orc_exact(const orc_problem *p, double t, double *u);

/* Alg.2 lines alg_coarse_rhsstart..rhsend: 7-point Laplacian
 * times nu plus first-order upwind advection. */
void orc_rhs_coarse(int32_t n, const double c[3], double nu, const double *u,
                    double *rhs);
/* 4th-order centred advection + diffusion. */
void orc_rhs_fine(int32_t n, const double c[3], double nu, const double *u,
                  double *rhs);

/* G: n_steps forward-Euler steps (Alg.2) over global steps
 * [step0, step0+n_steps) of size dt; u is updated in place. */
void orc_coarse(const orc_problem *p, double *u, int64_t step0, int64_t n_steps,
                double dt);
/* F: n_steps classical RK4 steps over global steps
 * [step0, step0+n_steps); u is updated in place. */
void orc_fine(const orc_problem *p, double *u, int64_t step0, int64_t n_steps,
              double dt);

/* Spatially coarsened G (P:238-241 names coarsening in space
 * as a way to make G cheaper, without fixing the transfer operators; readings
 * DESIGN.md C24-C26).  n must be a multiple of 4 (the n/2 mesh is even).
 *   restriction  (C24, injection):  uc[k][j][i] = u[2k][2j][2i]
 *   prolongation (C25, trilinear, periodic): the value at fine point
 *     (i, j, k) is the average over the coarse points (floor(i/2) or
 *     floor(i/2) + 1 along every axis with odd index; the index itself along
 *     every axis with even index), i.e. 1, 2, 4 or 8 coarse values with equal
 *     weights 1/2, 1/4, 1/8
 *   G_c = P o (Alg.2 on the n/2 mesh, same Delta t and nu_j) o R   (C26)  */
void orc_restrict(int32_t n, const double *u, double *uc);
void orc_prolong(int32_t n, const double *uc, double *u);
void orc_coarse_mesh(const orc_problem *p, double *u, int64_t step0, int64_t n_steps,
                     double dt);

/* max |u| over the n^3 points (the ||.||_inf of Eq.(defect)). */
double orc_inf_norm(int32_t n, const double *u);
/* max |u - v| */
double orc_inf_diff(int32_t n, const double *u, const double *v);
/* d = ||u - ref||_inf / ||ref||_inf  (Eq.(defect)) */
double orc_defect(int32_t n, const double *u, const double *ref);

/* Alg.1 for every rank p = 0..n_slices-1, executed serially in
 * pipeline order.  Slice m covers fine steps [m*nf, (m+1)*nf) of size
 * T/(n_slices*nf) and coarse steps [m*nc, (m+1)*nc) of size T/(n_slices*nc).
 * u_T receives u^K_{N_p}.  defects (K+1 entries, may be NULL) receives
 * d^0..d^K against u_ref (may be NULL; then defects is left untouched).
 * flags bit 0: use F in place of G (degenerate test case);
 * bit 2: use the spatially coarsened G_c (orc_coarse_mesh) as G.
 * Returns 0, or -1 on bad arguments / allocation failure. */
int orc_parareal(const orc_problem *p, int32_t n_slices, int32_t nc, int32_t nf,
                 int32_t K, const double *u0, const double *u_ref, double *u_T,
                 double *defects, int32_t flags);

/* Alg.1 with convergence-controlled stopping ("the loop could
 * alternatively be terminated by checking some convergence criterion", monitor
 * of P:301-302 "difference between two consecutive iterates"; C23).
 * `world` ranks own n_slices/world consecutive slices each.  In iteration k a
 * rank computes its relative iterate change
 *   c_k = max_l ||u^{k+1}_{l+1} - u^k_{l+1}||_inf / max_l ||u^{k+1}_{l+1}||_inf
 * over its own slices l (u^0 = the coarse initial guess) and stops after that
 * iteration when k = K-1, or when its predecessor has stopped (rank 0: always)
 * and c_k <= tol.  Its message of that iteration carries the stop flag; later
 * iterations of the successor reuse the last received value.
 * changes (world*K, may be NULL) receives c_k per rank (NaN when not run),
 * iters (world, may be NULL) the iterations each rank ran; defects as in
 * orc_parareal for the iterations the last rank ran (NaN after).  tol <= 0 is
 * the fixed-K algorithm. */
int orc_parareal_tol(const orc_problem *p, int32_t n_slices, int32_t nc, int32_t nf, int32_t K,
                     double tol, int32_t world, const double *u0, const double *u_ref,
                     double *u_T, double *defects, double *changes, int32_t *iters,
                     int32_t flags);

/* Threads the OpenMP runtime will use (1 when built without OpenMP). */
int orc_threads(void);

#ifdef __cplusplus
}
#endif
#endif
