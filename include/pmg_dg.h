/*
 * pmg_dg.h — C ABI of the B200-native (sm_100a, FP64) hot path of
 *   J. Stiller, "Robust Multigrid for Cartesian Interior Penalty DG Formulations of
 *   the Poisson Equation in 3D", arXiv:1612.04796.
 * Citations: PAPER.md:<line> (section / equation / algorithm) of the paper's LaTeX source.
 *
 * Conventions (all entry points):
 *  - Return an int status (PMG_OK = 0 or a PMG_E* code); never throw across the ABI.
 *    dg_last_error(ctx) gives a one-line message for the last failure on that context.
 *  - Vector arguments are caller-owned, DEVICE-resident, contiguous FP64 arrays in
 *    element-major order: element e = ex + nx*(ey + ny*ez); inside an element node
 *    i + n*(j + n*k), i along x fastest, n = P_l + 1.  Length = dg_ndofs(ctx, level).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All
 *    work is enqueued asynchronously on it; only pcg_solve and dg_dot synchronise it
 *    (they need scalars on the host).
 *  - The library never allocates device memory: all scratch and tables live in one
 *    caller-provided workspace (dg_workspace_bytes / dg_bind_workspace).
 *  - The context is not thread-safe: one stream / host thread per context.
 */
#ifndef PMG_DG_H
#define PMG_DG_H
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dg_ctx dg_ctx;   /* opaque */

enum { PMG_GLL = 0, PMG_GL = 1 };                 /* nodal basis */
enum { PMG_OVL_NODES = 0,                          /* n_o node layers */
       PMG_OVL_REL = 1,                            /* delta_O = alpha*Delta_d, Table 1 / Table 2 "rel" */
       PMG_OVL_MAXREL = 2 };                       /* delta_O = min(alpha*max_j Delta_j, Delta_d), Table 2 "max" */
enum { PMG_OK = 0, PMG_EINVAL = 1, PMG_EDIM = 2, PMG_ESINGULAR = 3, PMG_ECUDA = 4,
       PMG_EWORKSPACE = 5, PMG_EDIVERGED = 6, PMG_EMAXIT = 7, PMG_ESTATE = 8 };

/* dg_setup — discretisation of -lap u = f on the periodic box [0,lx]x[0,ly]x[0,lz]
 * (Eq. 1) with nx*ny*nz Cartesian elements of degree P on GL or GLL nodes
 * (Eqs. 2-6), SIPG penalty mu_d = penalty * mu_thr with mu_thr = P_l(P_l+1)/(2 Delta_d)
 * the coercivity threshold of this SIPG form, per level and direction ("mu_min is
 * the stability threshold"; the paper uses penalty = 2; reading R2).  Builds the p-multigrid hierarchy
 * P_l = 2^l, l = 0..L.  Host-only (no GPU needed).
 * Errors: PMG_EINVAL if P < 2 or P not a power of two or P > 32, any n_i < 3, l_i <= 0,
 *         penalty <= 0, basis not GLL/GL.  *out is set to NULL on error. */
int dg_setup(int nx, int ny, int nz, double lx, double ly, double lz, int P, int basis,
             double penalty, dg_ctx **out);

/* dg_schwarz_setup — weighted overlapping Schwarz smoother data for every level l >= 1
 * (§3.1): overlap layers per direction (mode/value/floor, R5),
 * restricted 1D eigenpairs S^T M_s S = I, S^T L_s S = Lambda computed in extended precision
 * (fast diagonalisation), hat weights W (Fig. 2).  Host-only.
 * Must be called before dg_workspace_bytes.  value = n_o (mode NODES) or alpha in (0,1].
 * Errors: PMG_EINVAL (mode/value/floor out of range), PMG_ESINGULAR (a restricted eigenvalue
 * sum <= 0, i.e. A_ss not regular). */
int dg_schwarz_setup(dg_ctx *ctx, int mode, double value, int floor_layers);

/* Number of levels L+1 and DOFs of level l (l = L is the top level, l = 0 the P=1 coarse level). */
int dg_num_levels(const dg_ctx *ctx);
long long dg_ndofs(const dg_ctx *ctx, int level);

/* Query the resolved overlap of level l: n_o[3] node layers and window sizes m[3]. Host-only. */
int dg_level_overlap(const dg_ctx *ctx, int level, int *n_o, int *m);

/* Copy host setup tables of (level, direction) for inspection/tests.  which:
 * 0 mass (n), 1 diagonal stiffness block D (n*n, row-major, row = test fn),
 * 2 traces (4n: phi(+1), (2/D)phi'(+1), phi(-1), (2/D)phi'(-1)), 3 S (m*m row-major, column = eigvec),
 * 4 Lambda (m), 5 W (m), 6 interpolation I_l (n_l * n_{l-1}, row-major), 7 nodes (n).
 * Writes at most `cap` doubles; returns the count (or a negative error code). Host-only. */
int dg_get_table(const dg_ctx *ctx, int level, int dir, int which, double *out, int cap);

/* Workspace: bytes needed (after dg_schwarz_setup), then bind a device buffer of at least
 * that many bytes (256-byte aligned; e.g. torch.empty(bytes, dtype=uint8, device='cuda')).
 * Binding uploads the setup tables on `stream`.  The context keeps the pointer; the caller
 * keeps ownership and must keep the buffer alive until dg_destroy.
 * Errors: PMG_EWORKSPACE (too small / misaligned), PMG_ECUDA. */
size_t dg_workspace_bytes(const dg_ctx *ctx);
int dg_bind_workspace(dg_ctx *ctx, void *dev_ptr, size_t bytes, void *stream);

/* dg_apply — Au = A_l u, the matrix-free sum-factorised IP-DG operator of Eq. 7
 * (PAPER.md:149-164): per element three n x n diagonal-block contractions plus rank-2 face
 * couplings to the six neighbours.  u and Au must not alias. */
int dg_apply(dg_ctx *ctx, int level, const double *u, double *Au, void *stream);

/* dg_residual — r = f - A_l u (Eq. 8).  r must not alias u or f. */
int dg_residual(dg_ctx *ctx, int level, const double *u, const double *f, double *r, void *stream);

/* schwarz_smooth — `steps` weighted additive Schwarz iterations on level l >= 1
 * (Eq. 10): r = f - A u; for every element-centred subdomain s
 * du_s = A_ss^{-1} R_s r by fast diagonalisation; u += sum_s R_s^T (W_s du_s).
 * u is updated in place; f is read-only. */
int schwarz_smooth(dg_ctx *ctx, int level, double *u, const double *f, int steps, void *stream);

/* The two halves of one Schwarz step, for callers that must exchange data between them (element
 * slabs on several GPUs): dg_schwarz_solve computes the weighted subdomain solutions
 * W_s A_ss^{-1} R_s r of every subdomain of level l into the context's window buffer
 * (PAPER.md:201-232); dg_schwarz_fold adds their deterministic sum (Eq. 10) to
 * u (zero != 0: u is overwritten by the sum).  schwarz_smooth = dg_residual, dg_schwarz_solve,
 * dg_schwarz_fold.  dg_window_buffer returns where the window buffer of level l lives inside the
 * bound workspace (byte offset) and its doubles per subdomain; subdomain s = element s, stored
 * contiguously in element order.  Errors: PMG_EINVAL, PMG_ESTATE. */
int dg_schwarz_solve(dg_ctx *ctx, int level, const double *r, void *stream);
int dg_schwarz_fold(dg_ctx *ctx, int level, double *u, int zero, void *stream);
int dg_window_buffer(const dg_ctx *ctx, int level, size_t *byte_offset, long long *doubles_per_subdomain);

/* Level transfers: prolongation uf += I_l uc (level l from l-1) and residual
 * restriction fc = I_l^T rf. */
int dg_prolongate_add(dg_ctx *ctx, int level, const double *uc, double *uf, void *stream);
int dg_restrict(dg_ctx *ctx, int level, const double *rf, double *fc, void *stream);

/* dg_coarse_solve — u0 = A_0^+ f0, Moore-Penrose pseudo-inverse at P_0 = 1 (Alg. 1 l.295,
 * PAPER.md:275-276): Euclidean projection of f0, global fast diagonalisation of the periodic
 * P=1 operator with the constant mode removed, Euclidean re-centring (R9).
 * f0 is read-only; u0 must not alias f0. */
int dg_coarse_solve(dg_ctx *ctx, const double *f0, double *u0, void *stream);

/* Smoothing schedule of the V-cycle: nu1[l], nu2[l] for l = 0..L (entry 0
 * unused).  Default: 1, 1 on all levels (fixed V(1,1)). Host-only. */
int dg_set_schedule(dg_ctx *ctx, const int *nu1, const int *nu2);

/* Replay V-cycles (pmg_vcycle and the preconditioner inside pcg_solve) from cached CUDA graphs
 * (default on).  A graph is captured on first use per (u, f) pointer pair and replayed on the
 * caller's stream; while profiling (dg_profile) launches are issued eagerly instead. */
int dg_set_graphs(dg_ctx *ctx, int enable);

/* Scatter strategy of the weighted Schwarz correction (Eq. 10), default OFF: with even element
 * counts and 2 n_o <= P_l+1, subdomains are processed in 8 parity classes whose windows are
 * node-disjoint and each adds W_s du_s straight into u (deterministic: fixed class order).
 * Off (default; the colored variant measured ~5% slower on c3), or where the condition fails:
 * weighted windows are stored and a deterministic pull kernel folds them. */
int dg_set_colored(dg_ctx *ctx, int enable);

/* pmg_vcycle — one multigrid V-cycle, Algorithm 1, in place on u
 * (top level), with the schedule above.  f is read-only. */
int pmg_vcycle(dg_ctx *ctx, double *u, const double *f, void *stream);

/* pcg_solve — inexact preconditioned CG (Golub-Ye) with one V-cycle
 * (zero initial guess) as preconditioner, until ||r||/||r_0|| <= rtol or maxit iterations.
 * u: initial guess in, solution out.  *iters receives the iteration count; res_hist (host,
 * maxit+1 doubles, or NULL) receives ||r_k||_2.  With graphs enabled (dg_set_graphs, default)
 * and maxit < 8192 the whole solve is ONE CUDA-graph launch: the iteration is the body of a
 * conditional WHILE node and the convergence test runs on the device, so `stream` is
 * synchronised once per solve; otherwise (profiling, graphs off) once per iteration.  Both paths
 * launch the same kernels in the same order (identical iterates).
 * Errors: PMG_EDIVERGED (non-finite scalar or ||r||/||r_0|| > 1e3), PMG_EMAXIT (u keeps the
 * last iterate). */
int pcg_solve(dg_ctx *ctx, double *u, const double *f, double rtol, int maxit, int *iters,
              double *res_hist, void *stream);

/* Vector helpers on level-l vectors (deterministic two-stage reductions):
 * dg_dot -> *out_host = <x, y>  (synchronises);  dg_project_mean: v -= mean(v). */
int dg_dot(dg_ctx *ctx, int level, const double *x, const double *y, double *out_host, void *stream);
int dg_project_mean(dg_ctx *ctx, int level, double *v, void *stream);
/* <x, y> over the first `count` entries (count <= top-level DOFs; synchronises): the owned part
 * of a slab-decomposed vector. */
int dg_dot_range(dg_ctx *ctx, const double *x, const double *y, long long count, double *out_host,
                 void *stream);
/* y = a x + b y over `count` entries with host scalars (b == 0: y = a x, y is not read): the
 * vector updates of a host-driven Krylov loop (slab-decomposed inexact PCG, PAPER.md:309-311,
 * whose alpha and beta are all-reduced over the ranks first). */
int dg_axpby(dg_ctx *ctx, double *y, double a, const double *x, double b, long long count, void *stream);

/* dg_rhs_sin — b = M * amp * sin(kx x) sin(ky y) sin(kz z) at the top-level nodes (diagonal
 * GL/GLL quadrature of the load term), then b -= mean(b). */
int dg_rhs_sin(dg_ctx *ctx, double amp, double kx, double ky, double kz, double *b, void *stream);

/* Number of kernels the library launched since the context was created (host counter). */
long long dg_launch_count(const dg_ctx *ctx);

/* Optional per-kernel timing: when enabled every launch is bracketed by CUDA events on its
 * stream.  dg_profile_read synchronises on the pending events and returns accumulated
 * milliseconds and launch counts per slot = kind*8 + level (PMG_PROF_SLOTS entries each);
 * kinds: 0 traces, 1 apply/residual, 2 Schwarz FDM solve, 3 overlap fold, 4 restriction,
 * 5 prolongation, 6 coarse solve, 7 vector/reduction ops.  reset != 0 clears the totals. */
#define PMG_PROF_SLOTS 64
int dg_profile(dg_ctx *ctx, int enable);
int dg_profile_read(dg_ctx *ctx, double *ms_out, long long *count_out, int reset);

/* Diagnostic: measured FP64 throughput of this GPU in TFLOP/s with a DFMA (use_dmma = 0) or
 * DMMA m8n8k4 (use_dmma = 1) saturating kernel on all SMs (the roofline denominator). */
int pmg_fp64_peak(int use_dmma, double *tflops_out, void *stream);

const char *dg_last_error(const dg_ctx *ctx);
void dg_destroy(dg_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* PMG_DG_H */
