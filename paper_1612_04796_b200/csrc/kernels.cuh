// Device kernels of the p-multigrid V(1,1) hot path (FP64, sm_100a).
// Paper: arXiv:1612.04796 (PAPER.md line numbers cited per kernel).
#pragma once
#include <cuda_runtime.h>

namespace pmg {

// Per-level device view of the setup tables (all pointers into the workspace).
struct LevelDev {
  int n, nx, ny, nz, Ne;
  const double *mass[3];   // (Delta_d/2) w, n each
  const double *D[3];      // diagonal 1D stiffness block, n*n row-major
  const double *tr[3];     // 4n: a = phi(+1), ap = (2/D) phi'(+1), b = phi(-1), bp = (2/D) phi'(-1)
  double mu[3];            // penalty per direction
  int no[3], m[3];         // overlap layers, window sizes
  const double *S[3];      // m*m, S[a*m+i] = component a of eigenvector i
  const double *lam[3];    // m
  const double *W[3];      // m
  const double *nodes;     // n reference nodes
  const double *Daug[3];   // [D | a ap b bp], n x (n+4) row-major (apply line GEMM)
  int Mw;                  // m0*m1*m2
  const double *Rz;        // eigen-divide table 1/(lam_x[p]+lam_y[q]+lam_z[o]) at [(p + m0 q) m2 + o]
};

struct CoarseDev {
  int G[3];                // global 1D sizes 2*n_e
  const double *S[3];      // G*G row-major (column = eigenvector)
  const double *lam[3];
};

// launchers (return cudaGetLastError())
cudaError_t launch_traces(const LevelDev &L, const double *u, double *T, cudaStream_t s);
cudaError_t launch_apply(const LevelDev &L, const double *u, const double *T, const double *f,
                         double *out, cudaStream_t s);
// fused residual + restriction f_c = I^T (f - A u) (no global r); available when apply_pipe_ok
bool apply_pipe_ok(const LevelDev &L);
cudaError_t launch_apply_pipe(const LevelDev &L, const double *u, const double *T, const double *f,
                              double *out, const double *I, int nc, double *fc, cudaStream_t s);
// global-memory paths for P = 32 blocks (windows > 32 or > shared memory); scratch X, Y: Ne*Mw;
// apply: Cb = Ne*12n^2, V = Ne*n^3
cudaError_t launch_fdm_global(const LevelDev &L, const double *r, double *X, double *Y, double *Z,
                              cudaStream_t s);
cudaError_t launch_apply_global(const LevelDev &L, const double *u, const double *T, const double *f,
                                double *out, double *Cb, double *V, cudaStream_t s);
// small windows (m <= 15): thread-per-line FP64-FMA fast diagonalisation (kern_fdm_dl.cu)
bool fdm_dl_launch(const LevelDev &L, const double *r, double *Z, cudaStream_t s);
bool fdm_mma_ok(const LevelDev &L);
// P = 32 (n = 33) apply / residual: two slab kernels with even/odd DMMA line GEMMs in shared
// memory (kern_apply33.cu); V: Ne * 33^3 scratch (x + z contributions)
bool apply33_ok(const LevelDev &L);
// P = 32 Schwarz solve on 45^3 windows: three slab kernels (kern_fdm_ct.cu); W1, W2: Ne * 45^3
bool fdm45_ok(const LevelDev &L);
cudaError_t launch_fdm45(const LevelDev &L, const double *r, double *W1, double *W2, double *Z,
                         cudaStream_t s);
cudaError_t launch_apply33(const LevelDev &L, const double *u, const double *T, const double *f,
                           double *out, double *V, cudaStream_t s);
// p-transfers as batched global line GEMMs (n_f > 17); X1, X2: Ne * nf * nf * nc doubles each
cudaError_t launch_restrict_global(const LevelDev &Lf, int nc, const double *I, const double *rf,
                                   double *fc, double *X1, double *X2, cudaStream_t s);
cudaError_t launch_prolong_global(const LevelDev &Lf, int nc, const double *I, const double *uc,
                                  double *uf, double *X1, double *X2, cudaStream_t s, double *S = nullptr);
// Colored Schwarz step: 8 launches (parity classes of the element coordinates); same-colour
// windows are node-disjoint, so each subdomain adds W du_s straight into u (no Z, no fold);
// deterministic (fixed colour order).  Needs even n_e and 2 n_o <= n in every direction.
bool fdm_colored_ok(const LevelDev &L);
cudaError_t launch_fdm_colored(const LevelDev &L, const double *r, double *u, cudaStream_t s);
// fused prolongation u_f += I u_c + traces of the new u_f (n_f <= 17)
bool prolong_traces_ok(const LevelDev &Lf, int nc);
cudaError_t launch_prolong_traces(const LevelDev &Lf, int nc, const double *I, const double *uc,
                                  double *uf, double *T, cudaStream_t s);
// compile-time-shape even/odd Schwarz kernel (kern_fdm_ct.cu); false if the shape is not built in
bool fdm_eoc_launch(const LevelDev &L, const double *r, double *Z, int color, double *u,
                    cudaStream_t s);
cudaError_t launch_fdm(const LevelDev &L, const double *r, double *Z, double *scr, bool smem,
                       size_t smem_bytes, cudaStream_t s);
// fold; T != nullptr additionally writes the face traces of the updated u (fused trace kernel)
cudaError_t launch_fold(const LevelDev &L, const double *Z, double *u, bool zero, double *T,
                        cudaStream_t s);
int fold_launches(const LevelDev &L, bool traces);   // kernels that call issues (1 or 2)
cudaError_t launch_restrict(const LevelDev &Lf, int nc, const double *I, const double *rf,
                            double *fc, cudaStream_t s);
cudaError_t launch_prolong(const LevelDev &Lf, int nc, const double *I, const double *uc,
                           double *uf, cudaStream_t s);
// coarse solve pieces
cudaError_t launch_coarse_gather(const LevelDev &L0, const CoarseDev &C, const double *f0,
                                 const double *mean, double *G, cudaStream_t s);
cudaError_t launch_lex_contract(const CoarseDev &C, int axis, bool forward, const double *in,
                                double *out, cudaStream_t s);
// whole coarse solve in 5 launches (needs 2 n_e <= 32 along z; see kernels.cu)
cudaError_t launch_coarse_fused(const LevelDev &L0, const CoarseDev &C, const double *f0,
                                double *G1, double *G2, double *u0, cudaStream_t s);
// whole coarse solve in one CTA (G_x G_y G_z <= 1024, G_d <= 32)
bool coarse_one_ok(const CoarseDev &C);
// one 8-CTA cluster, z pass through distributed shared memory (1024 < N_0, every G_d <= 32)
bool coarse_cluster_ok(const CoarseDev &C);
int coarse_fused_launches(const CoarseDev &C);
cudaError_t launch_coarse_cluster(const LevelDev &L0, const CoarseDev &C, const double *f0, double *u0,
                                  cudaStream_t s);
cudaError_t launch_coarse_one(const LevelDev &L0, const CoarseDev &C, const double *f0, double *u0,
                              cudaStream_t s);
cudaError_t launch_coarse_divide(const CoarseDev &C, double *G, cudaStream_t s);
cudaError_t launch_coarse_scatter(const LevelDev &L0, const CoarseDev &C, const double *G,
                                  const double *mean, double *u0, cudaStream_t s);
// reductions (deterministic, two-stage) and vector ops
int reduce_blocks(long long N);
cudaError_t launch_sum(const double *x, long long N, double *partial, double *out, double scale,
                       cudaStream_t s);
cudaError_t launch_dot(const double *x, const double *y, long long N, double *partial,
                       double *out, cudaStream_t s);
cudaError_t launch_sub_scalar(double *v, long long N, const double *c, cudaStream_t s);
cudaError_t launch_copy(double *dst, const double *src, long long N, cudaStream_t s);
cudaError_t launch_zero(double *dst, long long N, cudaStream_t s);
cudaError_t launch_axpby(double *y, double a, const double *x, double b, long long N, cudaStream_t s);
// PCG (Golub-Ye) helpers; scal[] slots documented in api.cu
cudaError_t launch_pq_alpha(const double *p, const double *q, long long N, double *partial,
                            double *scal, cudaStream_t s);
cudaError_t launch_cg_update(double *u, double *r, double *rold, const double *p,
                             const double *q, long long N, double *partial, double *scal,
                             cudaStream_t s);
cudaError_t launch_zr_beta(const double *z, const double *r, const double *rold, long long N,
                           double *partial, double *scal, bool first, cudaStream_t s);
cudaError_t launch_p_update(double *p, const double *z, long long N, const double *scal,
                            cudaStream_t s);
// device-side PCG control (graph path of pcg_solve): scal[30] = ||r_0||, scal[31] = k,
// scal[32] = status (0 converged / PMG_EDIVERGED / PMG_EMAXIT / -1 running); hist[k] = ||r_k||.
constexpr int PMG_PCG_HIST = 8192;
cudaError_t launch_pcg_start(double *scal, double *hist, int maxit, cudaGraphConditionalHandle hw,
                             cudaStream_t s);
cudaError_t launch_pcg_check(double *scal, double *hist, double rtol, int maxit,
                             cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hi, cudaStream_t s);
cudaError_t launch_rhs_sin(const LevelDev &L, double dx, double dy, double dz, double amp,
                           double kx, double ky, double kz, double *b, cudaStream_t s);

}  // namespace pmg
