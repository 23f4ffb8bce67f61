/*
 * parareal.h — C ABI of the B200-native hot path of
 *   Arteaga, Ruprecht & Krause, "A stencil-based implementation of Parareal in
 *   the C++ domain specific embedded language STELLA", arXiv:1409.8563.
 *
 * The library (paper_1409_8563_b200/libparareal.so) time-steps the periodic 3D
 * advection-diffusion equation with time-dependent diffusion
 *     u_t + c . grad u = nu(t) Lap u,   nu(t) = nu0 + nu0/2 sin(omega t)
 * (Eq.(adv_diff_eq); nu profile P:435-438) with
 *   G = forward Euler, 1st-order upwind advection, 7-point Laplacian
 *       (Alg.2),
 *   F = classical RK4, 4th-order centred advection and diffusion,
 * and runs Parareal (Eq.(parareal), Alg.1) over the GPUs
 * of one node with NCCL point-to-point hand-off in the paper's pipelined order.
 * "P:NNN" cites line NNN of the paper text.
 *
 * Conventions shared by every call
 * --------------------------------
 * Fields.  A field is n^3 contiguous IEEE fp64 values, index (z*n + y)*n + x
 *   (x fastest) — a C-contiguous float64 tensor of shape (n, n, n).  Grid
 *   points x_i = i/n on the periodic unit cube [0,1)^3, dx = 1/n
 *   (P:322).  There are no ghost cells; periodicity is handled in the kernels.
 * Pointers.  Unless a call says otherwise, field pointers are DEVICE pointers
 *   on the grid's device.  pr_fine, pr_coarse, pr_defect and pr_parareal also
 *   accept HOST pointers (pinned or pageable); those are staged through
 *   grid-owned device buffers inside the call (and make the call synchronous).
 * Ownership.  The caller owns every pointer it passes; the library never frees
 *   or retains a caller pointer after a call returns.  A pr_grid owns all its
 *   scratch (RK4 stage fields, Euler ping-pong field, Parareal state, nu
 *   tables, CUDA graphs, the NCCL communicator).
 * Streams.  `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *   stream).  Calls are asynchronous on `stream` unless documented as
 *   synchronous.  One grid's scratch is shared by all its calls: calls on the
 *   same grid issued on different streams must be ordered by the caller.
 *   A grid is not thread-safe.
 * Times.  Step j of size dt starts at t_j = j*dt, computed from the GLOBAL
 *   integer step index j (never accumulated), so splitting a run into slices
 *   is bitwise identical to one run (reading C6).
 * Errors.  Every call returns a pr_status; pr_last_error() gives a message
 *   (thread-local).  On error, outputs are unspecified (no partial results).
 */
#ifndef PARAREAL_B200_H
#define PARAREAL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PR_OK = 0,
    PR_EINVAL = 1,   /* bad argument: null pointer, n odd or < 4, n_steps < 0, dt <= 0, ... */
    PR_ENOMEM = 2,   /* device or pinned-host allocation failed */
    PR_ECUDA = 3,    /* CUDA runtime error */
    PR_ENCCL = 4,    /* hand-off failure (NCCL error, or a peer rank that did not deliver
                        within PR_NCCL_TIMEOUT_S, default 900 s); message carries rank and
                        iteration */
    PR_EDOMAIN = 5,  /* ||u_ref||_inf = 0 in a defect (Eq.(defect) undefined) */
    PR_ESTATE = 6    /* call not valid in this state (e.g. world > 1 before pr_comm_init) */
} pr_status;

/* Where nu(t) is sampled inside one RK4 step (reading C1). */
typedef enum {
    PR_NU_STAGE = 0,      /* t_j, t_j+dt/2, t_j+dt/2, t_j+dt : classical RK4, 4th order */
    PR_NU_STEP_START = 1  /* nu(t_j) for all four stages: reproduces P:456 */
} pr_nu_mode;

/* The benchmark problem, Eq.(adv_diff_eq) P:414 and P:447-448. */
typedef struct {
    int32_t n;        /* points per axis; even, 4 <= n <= 2048 */
    double c[3];      /* advection velocity (c_x, c_y, c_z) */
    double nu0;       /* nu_0 >= 0 */
    double omega;     /* omega */
    double T;         /* end time T > 0; used by pr_parareal */
    int32_t nu_mode;  /* pr_nu_mode */
} pr_problem;

/* Parareal configuration (Alg.1). */
typedef struct {
    int32_t n_slices;            /* N_p >= 1, a multiple of the world size */
    int32_t n_coarse_per_slice;  /* N_c >= 1, Delta t = T / (N_p N_c) */
    int32_t n_fine_per_slice;    /* N_f >= 1, delta t = T / (N_p N_f) */
    int32_t K;                   /* iterations k_max >= 0 (K = 0: coarse guess only) */
    int32_t flags;               /* bit 0 (PR_FLAG_G_IS_F): use F for G (degenerate test);
                                    bit 1 (PR_FLAG_PEER_HANDOFF): hand-off by peer stores (below);
                                    bit 2 (PR_FLAG_G_HALF_MESH): G = pr_coarse_mesh's G_c */
    double tol;                  /* > 0: convergence-controlled stopping (below); <= 0: fixed K */
} pr_parareal_cfg;

#define PR_FLAG_G_IS_F 1
#define PR_FLAG_PEER_HANDOFF 2
#define PR_FLAG_G_HALF_MESH 4

typedef struct pr_grid pr_grid;  /* opaque */

/* Create a grid object for `problem` on CUDA device `cuda_device`.  Allocates
 * 4 scratch fields (acc, Ya, Yb for the RK4 stages; one Euler ping-pong field)
 * and makes `cuda_device` current on the calling thread.  *out receives the
 * handle.  Errors: PR_EINVAL (null, n odd, n < 4 or > 2048, nu0 < 0, T <= 0),
 * PR_ENOMEM, PR_ECUDA. */
pr_status pr_create_grid(const pr_problem *problem, int32_t cuda_device, pr_grid **out);

/* Release everything the grid owns (synchronises the device first). */
pr_status pr_destroy_grid(pr_grid *grid);

/* F_dt (Eq.(fine)): n_steps classical RK4 steps of size dt over global
 * steps [step0, step0 + n_steps), from u_in to u_out.  u_in == u_out is
 * allowed; any other overlap is PR_EINVAL.  n_steps = 0 copies.  One step is
 * two fused kernels (stages 1+2 and 3+4, 56 B/point) when n is a multiple of
 * 32, else four fused stage passes (128 B/point); both give bitwise identical
 * results.  Default two-kernel design: the per-point stage hand-off
 * through tensor memory (23) for n >= 256, through shared memory (14) below.  The
 * environment variable PR_FTILE (read at pr_create_grid) selects another design,
 * all bitwise identical: 14 or 23 at any n, 22 stage B in the stage-A lanes, 24
 * the whole step in ONE kernel (16 B/point), 25 two z planes per warp iteration; PR_WPARAM=1 launches the fused kernels directly
 * with the stage weights as launch parameters instead of CUDA-graph batches;
 * PR_PDL=1 launches them with programmatic dependent launch.
 * Asynchronous on `stream` for device pointers. */
pr_status pr_fine(pr_grid *grid, const double *u_in, double *u_out, int64_t step0,
                  int64_t n_steps, double dt, void *stream);

/* G_Dt (Alg.2): n_steps forward-Euler steps with 1st-order upwind
 * advection (strict c_a > 0 test) and the 7-point Laplacian,
 * nu sampled at each step start, over global steps [step0, step0 + n_steps).
 * Same pointer rules as pr_fine. */
pr_status pr_coarse(pr_grid *grid, const double *u_in, double *u_out, int64_t step0,
                    int64_t n_steps, double dt, void *stream);

/* Eq.(defect): *d_host = max|u - u_ref| / max|u_ref| over the n^3
 * points (NaN propagates).  Synchronous: waits for `stream`.  PR_EDOMAIN if
 * max|u_ref| = 0. */
pr_status pr_defect(pr_grid *grid, const double *u, const double *u_ref, double *d_host,
                    void *stream);

/* u = sin(2 pi x) sin(2 pi y) sin(2 pi z), device pointer. */
pr_status pr_fill_sine(pr_grid *grid, double *u, void *stream);

/* Spatially coarsened coarse propagator G_c (P:238-241 names
 * coarsening in space as a cheaper G without fixing the transfer operators;
 * readings DESIGN.md C24-C26): restriction by injection onto the n/2 mesh
 * (uc[k][j][i] = u[2k][2j][2i]), n_steps Alg.2 Euler steps there (dx = 2/n,
 * the same Delta t and nu_j = nu(j dt)), periodic trilinear prolongation back
 * to n^3 (each fine point the mean of its 1, 2, 4 or 8 coarse neighbours).
 * Same argument conventions as pr_coarse; needs n % 4 == 0 (PR_EINVAL).  The
 * n/2 mesh lives in a child grid allocated at the first call. */
pr_status pr_coarse_mesh(pr_grid *grid, const double *u_in, double *u_out, int64_t step0,
                         int64_t n_steps, double dt, void *stream);

/* Parareal correction (Alg.1 line alg_para_corr):
 *   u_out = f + (g_new - g_old)          (rounding order: DESIGN.md C5)
 * If u_ref and d_host are both non-NULL the same pass also returns
 * *d_host = max|u_out - u_ref| / max|u_ref| and the call is synchronous.
 * Device pointers only; u_out may alias f. */
pr_status pr_correct(pr_grid *grid, const double *f, const double *g_new, const double *g_old,
                     double *u_out, const double *u_ref, double *d_host, void *stream);

/* Multi-GPU.  pr_nccl_unique_id writes an ncclUniqueId (PR_NCCL_ID_BYTES bytes)
 * on one rank; the caller distributes it (e.g. torch.distributed) and every
 * rank calls pr_comm_init with its own rank.  Collective over `world` ranks. */
#define PR_NCCL_ID_BYTES 128
pr_status pr_nccl_unique_id(void *id_out);
pr_status pr_comm_init(pr_grid *grid, int32_t world, int32_t rank, const void *nccl_unique_id);

/* In-process rank group: links `world` grids of THIS process (on one device or on
 * several devices with peer access) as ranks 0..world-1 of one time-slice pipeline,
 * without NCCL (replaces a communicator; pr_comm_init on a member leaves the group).
 * Each grid is then driven by its own host thread calling pr_parareal with the same
 * cfg; every rank's work runs on its grid's own stream (joined to the caller's stream
 * by events).  Hand-off (Alg.1): the correction pass of rank r's last
 * slice stores u^{k+1} straight into rank r+1's receive buffer (the peer-store data
 * path of PR_FLAG_PEER_HANDOFF, here a plain device or peer pointer); rank r records a
 * CUDA event after it and announces it through the group, and rank r+1's stream waits
 * on that event before its G reads the buffer; rank r+1 releases the buffer the same
 * way after the F that last reads it.  No stream or kernel waits on a value that has
 * not been announced, so ranks may share one GPU.  A rank that hears nothing from its
 * peer for PR_NCCL_TIMEOUT_S seconds (default 900) fails with PR_ENCCL (rank and
 * iteration in the message).  Grids must outlive the group's calls.  Errors:
 * PR_EINVAL (NULL or repeated grid, no peer access between consecutive devices),
 * PR_ECUDA. */
pr_status pr_local_group(pr_grid **grids, int32_t world);

/* Alg.1 for this rank's slice group: rank r of W owns slices
 * [r s, (r+1) s), s = N_p / W (W = 1 without pr_comm_init).  u0: initial value
 * (every rank; host or device).  u_T: receives u^K_{N_p} on the LAST rank
 * (ignored elsewhere, may be NULL there).  u_ref (nullable, needed on the last
 * rank only): the serial fine solution for the defect history; when given
 * together with defects_host (K+1 doubles), the last rank writes d^0..d^K
 * (d^0 = coarse initial guess, C11).  Synchronous on return (the timed unit).
 * Convergence control (cfg->tol > 0, monitor of P:301-302, DESIGN.md
 * C23): in iteration k a rank measures c_k = max over its slices of
 * ||u^{k+1}_{j+1} - u^k_{j+1}||_inf / max ||u^{k+1}_{j+1}||_inf and stops after
 * the iteration when its predecessor has stopped (rank 0: always) and
 * c_k <= tol, or when k = K-1; the stop flag rides on its last hand-off
 * message.  Iterations not run leave NaN in defects_host.  The monitors and
 * the iteration count are returned by pr_last_monitors.
 * Hand-off: ncclSend / ncclRecv of u^{k+1} on a comm stream by
 * default.  With PR_FLAG_PEER_HANDOFF (same value on every rank; world > 1; the
 * GPUs of one node with peer access) the correction pass of a rank's last
 * slice also stores u^{k+1} straight into the successor's receive buffer over
 * NVLink (CUDA IPC mappings, exchanged once per buffer pool by an NCCL
 * all-gather), a one-thread kernel then publishes a sequence word in the
 * successor's memory with a system-scope release, and the successor's stream
 * waits on that word (cuStreamWaitValue32: the stream front end waits, no
 * kernel spins); the successor hands its receive buffer back the same way
 * after the F that last reads it.  Results are bitwise those of the NCCL path.
 * The consumer's stream wait uses CU_STREAM_WAIT_VALUE_FLUSH where the device supports
 * it and is followed by a one-thread ld.acquire.sys + fence.acq_rel.sys kernel before
 * G reads the buffer.
 * Errors: PR_EINVAL, PR_ESTATE (world > 1 without a communicator), PR_ENCCL,
 * PR_EDOMAIN (u_ref all zero), PR_ECUDA. */
pr_status pr_parareal(pr_grid *grid, const pr_parareal_cfg *cfg, const double *u0,
                      double *u_T, const double *u_ref, double *defects_host, void *stream);

/* Host-side schedule of Alg.1 for one rank (no GPU needed).  Each entry is
 * {op, k, slice, peer}.  Used by pr_parareal and by the CPU tests. */
typedef enum {
    PR_OP_G_PREFIX = 1,  /* v = G_slice(v): redundant coarse prefix */
    PR_OP_G_INIT = 2,    /* start[slice] = v; gold[slice] = G_slice(v); v = gold */
    PR_OP_DEFECT0 = 3,   /* d^0 from gold[last slice] (last rank only) */
    PR_OP_F = 4,         /* f[slice] = F_slice(start[slice]) */
    PR_OP_RECV = 5,      /* recv u^{k+1}_slice from rank `peer` */
    PR_OP_G = 6,         /* gnew = G_slice(input) */
    PR_OP_CORRECT = 7,   /* out = f + (gnew - gold); gold = gnew */
    PR_OP_SEND = 8,      /* send out[slice] to rank `peer` */
    PR_OP_END_ITER = 9   /* start[l] = input used by slice l in this iteration */
} pr_op_code;
typedef struct { int32_t op, k, slice, peer; } pr_op;
/* Writes at most `cap` ops to `ops` (may be NULL to query) and the total to
 * *count.  PR_EINVAL on bad sizes. */
pr_status pr_plan(int32_t n_slices, int32_t K, int32_t world, int32_t rank, pr_op *ops,
                  int32_t cap, int32_t *count);

/* Iterate-change monitor c_k of this rank's last pr_parareal call (k < *iterations;
 * at most `cap` values written) and the number of iterations it ran. */
pr_status pr_last_monitors(pr_grid *grid, double *changes, int32_t cap, int32_t *iterations);

/* Device-time breakdown of this rank's last pr_parareal call, in ms:
 * out[0] total, [1] init (coarse prefix + own coarse), [2] fine, [3] waiting
 * for the predecessor, [4] coarse + correction in the iterations.
 * `cap` >= 5. */
pr_status pr_last_timings(pr_grid *grid, double *out, int32_t cap);

/* Static facts about a grid's launch configuration (no GPU work):
 *   fine_kernels_per_step: 2 (fused S1+S2 / S3+S4 kernels, tile-aligned n),
 *                          1 (PR_FTILE=24: one kernel per step) or
 *                          4 (one fused pass per RK4 stage);
 *   fine_bytes_per_point:  HBM bytes per grid point per RK4 step that path must
 *                          move (56, 16 or 128);
 *   coarse_bytes_per_point: 16 (one Euler pass);
 *   sms: streaming multiprocessors of the grid's device;
 *   fine_variant:          the two-kernel F design in use, PR_FTILE numbering (14 per-point
 *                          hand-off through shared memory, 23 through tensor memory, 22 / 24 /
 *                          25 the alternatives of pr_fine), 0 on the four-pass path. */
typedef struct {
    int32_t fine_kernels_per_step;
    int32_t fine_bytes_per_point;
    int32_t coarse_bytes_per_point;
    int32_t sms;
    int32_t fine_variant;
} pr_grid_info_t;
pr_status pr_grid_info(const pr_grid *grid, pr_grid_info_t *info);

/* Number of kernels this library has launched (graph nodes included). */
int64_t pr_kernel_launches(void);

/* Explicit-stability ratio, nu_max = 1.5 nu0, not enforced:
 *   G (fine = 0): dt (6 nu_max / dx^2 + sum_a |c_a| / dx)  (<= 1: Euler limit,
 *                 the positivity bound of the upwind scheme);
 *   F (fine = 1): dt (16 nu_max / dx^2) / 2.785  (spectral radius of the
 *                 4th-order Laplacian over the RK4 real-axis interval). */
pr_status pr_stability_ratio(const pr_problem *problem, double dt, int32_t fine, double *ratio);

const char *pr_last_error(void);
const char *pr_version(void);

#ifdef __cplusplus
}
#endif
#endif
