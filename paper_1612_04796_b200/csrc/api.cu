// C ABI (include/pmg_dg.h): context, setup, workspace, orchestration of the V-cycle and PCG.
// arXiv:1612.04796, Algorithm 1 and §3.2.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <exception>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/pmg_dg.h"
#include "kernels.cuh"
#include "setup.hpp"

using pmg::ld;

namespace {

struct LevelHost {
  int P = 0, n = 0;
  long long N = 0;
  pmg::Basis1D basis;
  pmg::Op1D op[3];
  pmg::Overlap1D ov[3];
  int m[3] = {0, 0, 0};
  int Mw = 0;
  std::vector<double> mass[3], D[3], tr[3], S[3], lam[3], W[3], interp, nodes, Daug[3];
  std::vector<double> Rz;    // 1/(lam_x[p] + lam_y[q] + lam_z[o]) at [(p + m_x q) m_z + o] (eigen-divide table)
  // workspace byte offsets
  size_t o_mass[3], o_D[3], o_tr[3], o_S[3], o_lam[3], o_W[3], o_Daug[3], o_interp = 0, o_nodes = 0;
  size_t o_u = 0, o_f = 0, o_r = 0, o_T = 0, o_Z = 0, o_scr = 0, o_scr2 = 0, o_cb = 0, o_v = 0;
  size_t o_x1 = 0, o_x2 = 0, o_Rz = 0;   // transfer scratch (n > 17): Ne * n * n * n_c each
  int fdm_path = 0;          // 0: DMMA in shared memory, 1: global-memory line GEMMs, 2: generic
  bool fdm_smem = false;
  size_t fdm_smem_bytes = 0;
  ld lam_min[3] = {0, 0, 0}, lam_max[3] = {0, 0, 0};
};

constexpr size_t FDM_SMEM_MAX = 227 * 1024;

std::vector<double> to_d(const std::vector<ld> &v) { return std::vector<double>(v.begin(), v.end()); }

}  // namespace

struct dg_ctx {
  int ne[3];
  double len[3];
  int P, basis, L;
  double penalty;
  std::vector<LevelHost> lev;
  bool schwarz_ready = false;
  int ovl_mode = -1;
  // coarse global FDM
  int G[3];
  std::vector<double> S0[3], lam0[3];
  size_t o_S0[3], o_lam0[3], o_G1 = 0, o_G2 = 0;
  // PCG + reductions
  size_t o_pr, o_pz, o_pp, o_pq, o_prold, o_part, o_scal;
  size_t ws_bytes = 0;
  char *ws = nullptr;
  std::vector<int> nu1, nu2;
  double *host_pinned = nullptr;
  long long launches = 0;
  long long launches_per_cycle = 0;
  std::string err;
  // CUDA-graph replay of whole V-cycles (dg_set_graphs); keyed by (u, f, zero_top)
  bool graphs = true;
  bool colored = false;      // colored Schwarz scatter (dg_set_colored); measured slower on c3
  cudaStream_t cap_stream = nullptr;
  struct GraphEntry { double *u; const double *f; bool zero; cudaGraphExec_t exec; };
  std::vector<GraphEntry> graph_cache;
  // whole PCG solves as one graph launch (conditional WHILE/IF nodes, device-side convergence test)
  struct PcgGraph { double *u; const double *f; double rtol; int maxit; cudaGraphExec_t exec;
                    long long lp, lw, li; };
  std::vector<PcgGraph> pcg_cache;
  cudaStream_t cap_stream2 = nullptr;
  size_t o_hist = 0;          // PCG residual history (pmg::PMG_PCG_HIST doubles, device)
  double *host_hist = nullptr;
  // optional per-kernel CUDA-event timing (dg_profile): slot = kind * 8 + level
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> ev_slot;          // slot of pending pair i (events 2i, 2i+1)
  double prof_ms[PMG_PROF_SLOTS] = {0};
  long long prof_cnt[PMG_PROF_SLOTS] = {0};
};

namespace {

void drop_graphs(dg_ctx *c) {
  for (auto &g : c->graph_cache) cudaGraphExecDestroy(g.exec);
  c->graph_cache.clear();
  for (auto &g : c->pcg_cache) cudaGraphExecDestroy(g.exec);
  c->pcg_cache.clear();
}

int fail(dg_ctx *c, int code, const std::string &msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_check(dg_ctx *c, cudaError_t e, const char *what) {
  if (e != cudaSuccess) return fail(c, PMG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return PMG_OK;
}

template <class T>
T *wsp(const dg_ctx *c, size_t off) { return reinterpret_cast<T *>(c->ws + off); }

pmg::LevelDev level_dev(const dg_ctx *c, int l) {
  const LevelHost &h = c->lev[l];
  pmg::LevelDev d;
  d.n = h.n; d.nx = c->ne[0]; d.ny = c->ne[1]; d.nz = c->ne[2];
  d.Ne = c->ne[0] * c->ne[1] * c->ne[2];
  for (int k = 0; k < 3; ++k) {
    d.mass[k] = wsp<double>(c, h.o_mass[k]);
    d.D[k] = wsp<double>(c, h.o_D[k]);
    d.tr[k] = wsp<double>(c, h.o_tr[k]);
    d.mu[k] = (double)h.op[k].mu;
    d.no[k] = h.ov[k].no;
    d.m[k] = h.m[k];
    d.S[k] = h.S[k].empty() ? nullptr : wsp<double>(c, h.o_S[k]);
    d.lam[k] = h.lam[k].empty() ? nullptr : wsp<double>(c, h.o_lam[k]);
    d.W[k] = h.W[k].empty() ? nullptr : wsp<double>(c, h.o_W[k]);
    d.Daug[k] = wsp<double>(c, h.o_Daug[k]);
  }
  d.Rz = h.Rz.empty() ? nullptr : wsp<double>(c, h.o_Rz);
  d.nodes = wsp<double>(c, h.o_nodes);
  d.Mw = h.Mw;
  return d;
}

pmg::CoarseDev coarse_dev(const dg_ctx *c) {
  pmg::CoarseDev d;
  for (int k = 0; k < 3; ++k) {
    d.G[k] = c->G[k];
    d.S[k] = wsp<double>(c, c->o_S0[k]);
    d.lam[k] = wsp<double>(c, c->o_lam0[k]);
  }
  return d;
}

struct Planner {
  size_t off = 0;
  size_t take(size_t bytes) {
    off = (off + 255) & ~size_t(255);
    size_t o = off;
    off += bytes;
    return o;
  }
  size_t dbl(long long count) { return take(sizeof(double) * (size_t)count); }
};

void plan_workspace(dg_ctx *c) {
  Planner p;
  const long long Ne = (long long)c->ne[0] * c->ne[1] * c->ne[2];
  for (int l = 0; l <= c->L; ++l) {
    LevelHost &h = c->lev[l];
    const int n = h.n;
    for (int d = 0; d < 3; ++d) {
      h.o_mass[d] = p.dbl(n);
      h.o_D[d] = p.dbl(n * n);
      h.o_tr[d] = p.dbl(4 * n);
      h.o_S[d] = p.dbl(h.S[d].size());
      h.o_lam[d] = p.dbl(h.lam[d].size());
      h.o_W[d] = p.dbl(h.W[d].size());
      h.o_Daug[d] = p.dbl(h.Daug[d].size());
    }
    h.o_interp = p.dbl(h.interp.size());
    h.o_nodes = p.dbl(n);
    h.o_u = l < c->L ? p.dbl(h.N) : 0;
    h.o_f = l < c->L ? p.dbl(h.N) : 0;
    h.o_r = p.dbl(h.N);
    h.o_T = p.dbl(Ne * 12 * n * n);
    if (l >= 1 && c->schwarz_ready) {
      h.o_Z = p.dbl(Ne * h.Mw);
      h.o_Rz = p.dbl(h.Rz.size());
      size_t mma_words = (size_t)h.Mw;
      int mmax = 0;
      for (int d = 0; d < 3; ++d) {
        mma_words += (size_t)h.m[d] * h.m[d] + 3 * (size_t)h.m[d];
        mmax = std::max(mmax, h.m[d]);
      }
      if (mmax <= 32 && mma_words * sizeof(double) <= FDM_SMEM_MAX) h.fdm_path = 0;
      else if (mmax <= 80) h.fdm_path = 1;
      else h.fdm_path = 2;
      const size_t sb = sizeof(double) * (2 * (size_t)h.Mw);
      h.fdm_smem = sb <= FDM_SMEM_MAX;
      h.fdm_smem_bytes = h.fdm_smem ? sb : 0;
      h.o_scr = (h.fdm_path == 1 || !h.fdm_smem) ? p.dbl(Ne * h.Mw) : 0;
      h.o_scr2 = h.fdm_path == 1 ? p.dbl(Ne * h.Mw) : 0;
    }
    if (n > 17) {                    // global-memory apply buffers (face coefficients, V)
      h.o_cb = p.dbl(Ne * 12 * n * n);
      h.o_v = p.dbl(h.N);
      if (l >= 1) {
        const long long nc = c->lev[l - 1].n;
        h.o_x1 = p.dbl(Ne * n * n * nc);
        h.o_x2 = p.dbl(Ne * n * n * nc);
      }
    }
  }
  for (int d = 0; d < 3; ++d) {
    c->o_S0[d] = p.dbl((long long)c->G[d] * c->G[d]);
    c->o_lam0[d] = p.dbl(c->G[d]);
  }
  const long long N0 = 8 * Ne;
  c->o_G1 = p.dbl(N0);
  c->o_G2 = p.dbl(N0);
  const long long NL = c->lev[c->L].N;
  c->o_pr = p.dbl(NL); c->o_pz = p.dbl(NL); c->o_pp = p.dbl(NL); c->o_pq = p.dbl(NL);
  c->o_prold = p.dbl(NL);
  c->o_part = p.dbl(2 * 2048);
  c->o_scal = p.dbl(64);
  c->o_hist = p.dbl(pmg::PMG_PCG_HIST);
  c->ws_bytes = p.off + 256;
}

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

enum { K_TRACES = 0, K_APPLY, K_FDM, K_FOLD, K_RESTRICT, K_PROLONG, K_COARSE, K_VEC };

cudaEvent_t prof_event(dg_ctx *c, size_t i) {
  while (c->ev_pool.size() <= i) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[i];
}

// NVTX ranges "kind@level" around every launch (timeline tools), enabled by PMG_NVTX=1 in the
// environment; header-only NVTX v3, a no-op without an attached tool.
const bool g_nvtx = [] { const char *e = std::getenv("PMG_NVTX"); return e && e[0] == '1'; }();
void nvtx_push(int kind, int level) {
  static const char *names[8] = {"traces", "apply", "fdm", "fold", "restrict", "prolong", "coarse", "vec"};
  char buf[32];
  std::snprintf(buf, sizeof buf, "%s@l%d", names[kind & 7], level);
  nvtxRangePushA(buf);
}

// Every kernel launch goes through here: counts launches and (if enabled) brackets the launch
// with CUDA events on the launching stream.
#define LAUNCHK(c, kind, level, s, expr)                                         \
  do {                                                                           \
    size_t _pi = (c)->ev_slot.size();                                            \
    if ((c)->prof) cudaEventRecord(prof_event((c), 2 * _pi), (s));               \
    if (g_nvtx) nvtx_push((kind), (level));                                      \
    cudaError_t _e = (expr);                                                     \
    if (g_nvtx) nvtxRangePop();                                                  \
    (c)->launches++;                                                             \
    if ((c)->prof) {                                                             \
      cudaEventRecord(prof_event((c), 2 * _pi + 1), (s));                        \
      (c)->ev_slot.push_back((kind) * 8 + (level));                              \
    }                                                                            \
    if (_e != cudaSuccess) return cuda_check((c), _e, #expr);                    \
  } while (0)
#define LAUNCH(c, expr) LAUNCHK(c, K_VEC, 0, s, expr)

int check_level(dg_ctx *c, int level, bool need_ws = true) {
  if (!c) return PMG_EINVAL;
  if (level < 0 || level > c->L) return fail(c, PMG_EINVAL, "level out of range");
  if (need_ws && !c->ws) return fail(c, PMG_ESTATE, "workspace not bound");
  return PMG_OK;
}

// r = f - A u (f == nullptr: r = A u).  have_traces: T_l already holds the traces of u
// (written by the fused fold kernel that produced u in this same cycle).
int residual_impl(dg_ctx *c, int l, const double *u, const double *f, double *out, cudaStream_t s,
                  bool have_traces = false) {
  pmg::LevelDev d = level_dev(c, l);
  double *T = wsp<double>(c, c->lev[l].o_T);
  if (!have_traces) LAUNCHK(c, K_TRACES, l, s, pmg::launch_traces(d, u, T, s));
  if (c->lev[l].o_cb && pmg::apply33_ok(d)) {
    LAUNCHK(c, K_APPLY, l, s, pmg::launch_apply33(d, u, T, f, out, wsp<double>(c, c->lev[l].o_v), s));
    c->launches += 1;
  } else if (c->lev[l].o_cb) {
    LAUNCHK(c, K_APPLY, l, s, pmg::launch_apply_global(d, u, T, f, out, wsp<double>(c, c->lev[l].o_cb),
                                                       wsp<double>(c, c->lev[l].o_v), s));
    c->launches += 4;
  } else {
    LAUNCHK(c, K_APPLY, l, s, pmg::launch_apply(d, u, T, f, out, s));
  }
  return PMG_OK;
}

// All subdomain solves of level l: Z_l = W_s A_ss^{-1} R_s r for every element-centred subdomain
// (window-major weighted results; the fold sums them).
int fdm_impl(dg_ctx *c, int l, const double *rin, cudaStream_t s) {
  LevelHost &h = c->lev[l];
  pmg::LevelDev d = level_dev(c, l);
  double *Z = wsp<double>(c, h.o_Z);
  double *scr = h.o_scr ? wsp<double>(c, h.o_scr) : nullptr;
  if (h.fdm_path == 1 && pmg::fdm45_ok(d)) {
    LAUNCHK(c, K_FDM, l, s, pmg::launch_fdm45(d, rin, scr, wsp<double>(c, h.o_scr2), Z, s));
    c->launches += 2;
  } else if (h.fdm_path == 1) {
    LAUNCHK(c, K_FDM, l, s, pmg::launch_fdm_global(d, rin, scr, wsp<double>(c, h.o_scr2), Z, s));
    c->launches += 6;
  } else {
    LAUNCHK(c, K_FDM, l, s, pmg::launch_fdm(d, rin, Z, scr, h.fdm_smem, h.fdm_smem_bytes, s));
  }
  return PMG_OK;
}

// `steps` Schwarz iterations.  traces_after: the last fold also emits the traces of the final u
// (the caller's next operation is a residual of u on this level).
int smooth_impl(dg_ctx *c, int l, double *u, const double *f, int steps, bool zero_init,
                cudaStream_t s, bool traces_after = false, bool traces_ready = false) {
  LevelHost &h = c->lev[l];
  pmg::LevelDev d = level_dev(c, l);
  double *r = wsp<double>(c, h.o_r);
  double *Z = wsp<double>(c, h.o_Z);
  double *T = wsp<double>(c, h.o_T);
  double *scr = h.o_scr ? wsp<double>(c, h.o_scr) : nullptr;
  for (int it = 0; it < steps; ++it) {
    const bool zero = zero_init && it == 0;
    const double *rin = f;                       // u == 0  =>  r = f (Alg. 1 l.287-290)
    if (!zero) {
      int st = residual_impl(c, l, u, f, r, s, it > 0 || traces_ready);
      if (st) return st;
      rin = r;
    }
    const bool emit = (it + 1 < steps) || traces_after;
    if (h.fdm_path == 0 && c->colored && pmg::fdm_colored_ok(d)) {
      // colored step: W du_s added straight into u, colour by colour (no Z round trip, no fold)
      if (zero) LAUNCH(c, pmg::launch_zero(u, h.N, s));
      LAUNCHK(c, K_FDM, l, s, pmg::launch_fdm_colored(d, rin, u, s));
      c->launches += 7;
      if (emit) LAUNCHK(c, K_TRACES, l, s, pmg::launch_traces(d, u, T, s));
      continue;
    }
    int st = fdm_impl(c, l, rin, s);
    if (st) return st;
    LAUNCHK(c, K_FOLD, l, s, pmg::launch_fold(d, Z, u, zero, emit ? T : nullptr, s));
    c->launches += pmg::fold_launches(d, emit) - 1;
  }
  if (steps == 0 && zero_init) LAUNCH(c, pmg::launch_zero(u, h.N, s));
  return PMG_OK;
}

int coarse_impl(dg_ctx *c, const double *f0, double *u0, cudaStream_t s) {
  pmg::LevelDev d0 = level_dev(c, 0);
  pmg::CoarseDev C = coarse_dev(c);
  const long long N0 = c->lev[0].N;
  double *part = wsp<double>(c, c->o_part);
  double *scal = wsp<double>(c, c->o_scal);
  double *G1 = wsp<double>(c, c->o_G1), *G2 = wsp<double>(c, c->o_G2);
  if (pmg::coarse_one_ok(C)) {
    LAUNCHK(c, K_COARSE, 0, s, pmg::launch_coarse_one(d0, C, f0, u0, s));
    return PMG_OK;
  }
  if (pmg::coarse_cluster_ok(C)) {
    LAUNCHK(c, K_COARSE, 0, s, pmg::launch_coarse_cluster(d0, C, f0, u0, s));
    return PMG_OK;
  }
  if (c->G[2] <= 32) {
    LAUNCHK(c, K_COARSE, 0, s, pmg::launch_coarse_fused(d0, C, f0, G1, G2, u0, s));
    c->launches += pmg::coarse_fused_launches(C) - 1;   // launch_coarse_fused issues 3 or 5 kernels
    return PMG_OK;
  }
  LAUNCHK(c, K_COARSE, 0, s, pmg::launch_sum(f0, N0, part, scal + 10, 1.0 / N0, s));           // mean(f0)
  LAUNCHK(c, K_COARSE, 0, s, pmg::launch_coarse_gather(d0, C, f0, scal + 10, G1, s));          // project
  LAUNCHK(c, K_COARSE, 0, s, pmg::launch_lex_contract(C, 0, true, G1, G2, s));
  LAUNCHK(c, K_COARSE, 0, s, pmg::launch_lex_contract(C, 1, true, G2, G1, s));
  LAUNCHK(c, K_COARSE, 0, s, pmg::launch_lex_contract(C, 2, true, G1, G2, s));
  LAUNCHK(c, K_COARSE, 0, s, pmg::launch_coarse_divide(C, G2, s));
  LAUNCHK(c, K_COARSE, 0, s, pmg::launch_lex_contract(C, 2, false, G2, G1, s));
  LAUNCHK(c, K_COARSE, 0, s, pmg::launch_lex_contract(C, 1, false, G1, G2, s));
  LAUNCHK(c, K_COARSE, 0, s, pmg::launch_lex_contract(C, 0, false, G2, G1, s));
  LAUNCHK(c, K_COARSE, 0, s, pmg::launch_sum(G1, N0, part, scal + 11, 1.0 / N0, s));           // re-centre
  LAUNCHK(c, K_COARSE, 0, s, pmg::launch_coarse_scatter(d0, C, G1, scal + 11, u0, s));
  return PMG_OK;
}

// Algorithm 1.  zero_top: u is known to be 0 on entry (PCG preconditioner).
int vcycle_impl(dg_ctx *c, double *u, const double *f, bool zero_top, cudaStream_t s) {
  const int L = c->L;
  std::vector<double *> U(L + 1), F(L + 1);
  for (int l = 0; l < L; ++l) {
    U[l] = wsp<double>(c, c->lev[l].o_u);
    F[l] = wsp<double>(c, c->lev[l].o_f);
  }
  U[L] = u;
  F[L] = const_cast<double *>(f);
  int st;
  for (int l = L; l >= 1; --l) {                                  // l.286
    const bool zero = (l < L) || zero_top;                         // l.287-289
    const int nu = c->nu1[l];
    if ((st = smooth_impl(c, l, U[l], F[l], nu, zero, s, true))) return st;   // l.290
    double *r = wsp<double>(c, c->lev[l].o_r);
    pmg::LevelDev d = level_dev(c, l);
    if (pmg::apply_pipe_ok(d)) {                                     // l.292 fused
      double *T = wsp<double>(c, c->lev[l].o_T);
      if (nu == 0) LAUNCHK(c, K_TRACES, l, s, pmg::launch_traces(d, U[l], T, s));
      LAUNCHK(c, K_APPLY, l, s, pmg::launch_apply_pipe(d, U[l], T, F[l], nullptr,
                                                       wsp<double>(c, c->lev[l].o_interp),
                                                       c->lev[l - 1].n, F[l - 1], s));
    } else {
      if ((st = residual_impl(c, l, U[l], F[l], r, s, nu > 0))) return st;    // l.292
      if (c->lev[l].o_x1) {
        LAUNCHK(c, K_RESTRICT, l, s, pmg::launch_restrict_global(d, c->lev[l - 1].n,
                                       wsp<double>(c, c->lev[l].o_interp), r, F[l - 1],
                                       wsp<double>(c, c->lev[l].o_x1), wsp<double>(c, c->lev[l].o_x2), s));
        c->launches += 2;                                   // three line-GEMM passes
      } else
        LAUNCHK(c, K_RESTRICT, l, s, pmg::launch_restrict(d, c->lev[l - 1].n,
                                       wsp<double>(c, c->lev[l].o_interp), r, F[l - 1], s));
    }
  }
  if ((st = coarse_impl(c, F[0], U[0], s))) return st;           // l.295
  for (int l = 1; l <= L; ++l) {                                  // l.298
    pmg::LevelDev d = level_dev(c, l);
    const int nc = c->lev[l - 1].n;
    const double *Il = wsp<double>(c, c->lev[l].o_interp);
    bool tr = false;
    if (c->nu2[l] > 0 && pmg::prolong_traces_ok(d, nc)) {          // l.299 + traces of u_l
      LAUNCHK(c, K_PROLONG, l, s, pmg::launch_prolong_traces(d, nc, Il, U[l - 1], U[l],
                                                             wsp<double>(c, c->lev[l].o_T), s));
      tr = true;
    } else {
      if (c->lev[l].o_x1) {
        LAUNCHK(c, K_PROLONG, l, s, pmg::launch_prolong_global(d, nc, Il, U[l - 1], U[l],
                                       wsp<double>(c, c->lev[l].o_x1), wsp<double>(c, c->lev[l].o_x2), s,
                                       wsp<double>(c, c->lev[l].o_r)));    // r_l is dead here (scratch)
        c->launches += 3;                                   // three passes + the vector update
      } else
        LAUNCHK(c, K_PROLONG, l, s, pmg::launch_prolong(d, nc, Il, U[l - 1], U[l], s));   // l.299
    }
    if ((st = smooth_impl(c, l, U[l], F[l], c->nu2[l], false, s, false, tr))) return st;  // l.301
  }
  return PMG_OK;
}

// V-cycle through a cached CUDA graph: the ~5 launches per level become one graph launch
// (launch latency dominates the small configurations).  Captured on an internal stream, then
// replayed on the caller's stream.  Falls back to eager launches while profiling.
int vcycle_run(dg_ctx *c, double *u, const double *f, bool zero_top, cudaStream_t s) {
  if (!c->graphs || c->prof) return vcycle_impl(c, u, f, zero_top, s);
  for (auto &g : c->graph_cache)
    if (g.u == u && g.f == f && g.zero == zero_top) {
      c->launches += c->launches_per_cycle;
      return cuda_check(c, cudaGraphLaunch(g.exec, s), "cudaGraphLaunch");
    }
  cudaError_t e = cudaSuccess;
  if (!c->cap_stream) e = cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_check(c, e, "cudaStreamCreate");
  cudaGraph_t graph = nullptr;
  e = cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return cuda_check(c, e, "cudaStreamBeginCapture");
  const long long l0 = c->launches;
  int st = vcycle_impl(c, u, f, zero_top, c->cap_stream);
  e = cudaStreamEndCapture(c->cap_stream, &graph);
  if (st) { if (graph) cudaGraphDestroy(graph); return st; }
  if (e != cudaSuccess) return cuda_check(c, e, "cudaStreamEndCapture");
  c->launches_per_cycle = c->launches - l0;
  c->launches = l0;
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_check(c, e, "cudaGraphInstantiate");
  c->graph_cache.push_back({u, f, zero_top, exec});
  c->launches += c->launches_per_cycle;
  return cuda_check(c, cudaGraphLaunch(exec, s), "cudaGraphLaunch");
}

}  // namespace

extern "C" {

int dg_setup(int nx, int ny, int nz, double lx, double ly, double lz, int P, int basis,
             double penalty, dg_ctx **out) {
  if (!out) return PMG_EINVAL;
  *out = nullptr;
  if (P < 2 || P > 32 || (P & (P - 1))) return PMG_EINVAL;
  if (nx < 3 || ny < 3 || nz < 3) return PMG_EINVAL;
  if (!(lx > 0 && ly > 0 && lz > 0) || !(penalty > 0)) return PMG_EINVAL;
  if (basis != PMG_GLL && basis != PMG_GL) return PMG_EINVAL;
  dg_ctx *c = nullptr;
  try {
    c = new dg_ctx();
    c->ne[0] = nx; c->ne[1] = ny; c->ne[2] = nz;
    c->len[0] = lx; c->len[1] = ly; c->len[2] = lz;
    c->P = P; c->basis = basis; c->penalty = penalty;
    int L = 0;
    while ((1 << L) < P) ++L;
    c->L = L;
    c->lev.resize(L + 1);
    const long long Ne = (long long)nx * ny * nz;
    for (int l = 0; l <= L; ++l) {
      LevelHost &h = c->lev[l];
      h.P = 1 << l; h.n = h.P + 1;
      h.N = Ne * h.n * h.n * h.n;
      h.basis = pmg::make_basis(basis, h.P);
      h.nodes = to_d(h.basis.x);
      for (int d = 0; d < 3; ++d) {
        h.op[d] = pmg::assemble_1d(h.basis, c->ne[d], ld(c->len[d]) / c->ne[d], ld(penalty));
        if (pmg::coupling_check(h.op[d]) > 1e-12L) {
          delete c;
          return PMG_ESINGULAR;
        }
        h.mass[d].resize(h.n);
        for (int i = 0; i < h.n; ++i) h.mass[d][i] = (double)h.op[d].M[i];
        h.D[d] = to_d(h.op[d].Dblk);
        h.tr[d] = to_d(h.op[d].tr);
        // augmented stiffness [D | a ap b bp] (n x (n+4)): the rank-2 neighbour couplings
        // become four extra K columns of the apply's line GEMM
        // rows pre-scaled by 1/M_d[o]: A u = M (x) (sum_d M_d^-1 L_d u), so the three line
        // GEMMs accumulate without per-direction mass factors and one M multiply finishes
        h.Daug[d].assign(h.n * (h.n + 4), 0.0);
        for (int o = 0; o < h.n; ++o) {
          const ld im = 1 / h.op[d].M[o];
          for (int k = 0; k < h.n; ++k) h.Daug[d][o * (h.n + 4) + k] = (double)(h.op[d].Dblk[o * h.n + k] * im);
          for (int r = 0; r < 4; ++r)
            h.Daug[d][o * (h.n + 4) + h.n + r] = (double)(h.op[d].tr[r * h.n + o] * im);
        }
        h.m[d] = h.n;
      }
      if (l >= 1) h.interp = to_d(pmg::interp_matrix(c->lev[l - 1].basis, h.basis));
    }
    // coarse global eigenpairs of the periodic P=1 operators (size 2 n_e per direction)
    for (int d = 0; d < 3; ++d) {
      const pmg::Op1D &op = c->lev[0].op[d];
      const int G = op.ne * op.n;
      c->G[d] = G;
      std::vector<ld> lam, Sv;
      pmg::gen_eig(G, op.L, op.M, lam, Sv);
      // the constant null vector: exact zero eigenvalue, exactly constant M-normalised vector
      ld msum = 0;
      for (int i = 0; i < G; ++i) msum += op.M[i];
      lam[0] = 0;
      for (int a = 0; a < G; ++a) Sv[a * G + 0] = 1 / std::sqrt(msum);
      if (!(lam[1] > 1e-14L * lam[G - 1])) { delete c; return PMG_ESINGULAR; }
      c->S0[d] = to_d(Sv);
      c->lam0[d] = to_d(lam);
    }
    c->nu1.assign(L + 1, 1);
    c->nu2.assign(L + 1, 1);
    plan_workspace(c);
  } catch (const std::exception &) {
    delete c;
    return PMG_EINVAL;
  }
  *out = c;
  return PMG_OK;
}

int dg_schwarz_setup(dg_ctx *c, int mode, double value, int floor_layers) {
  if (!c) return PMG_EINVAL;
  if (c->ws) return fail(c, PMG_ESTATE, "dg_schwarz_setup must precede dg_bind_workspace");
  if (mode < 0 || mode > 2 || floor_layers < 0) return fail(c, PMG_EINVAL, "bad overlap mode/floor");
  if (mode == PMG_OVL_NODES && !(value >= 0)) return fail(c, PMG_EINVAL, "n_o < 0");
  if (mode != PMG_OVL_NODES && !(value > 0 && value <= 1)) return fail(c, PMG_EINVAL, "alpha not in (0,1]");
  ld dmax = 0;
  for (int d = 0; d < 3; ++d) dmax = std::max(dmax, ld(c->len[d]) / c->ne[d]);
  for (int l = 1; l <= c->L; ++l) {
    LevelHost &h = c->lev[l];
    h.Mw = 1;
    for (int d = 0; d < 3; ++d) {
      const pmg::Op1D &op = h.op[d];
      h.ov[d] = pmg::resolve_overlap(mode, value, floor_layers, h.basis, op.delta, dmax);
      const int no = h.ov[d].no, n = h.n, m = n + 2 * no;
      h.m[d] = m;
      h.Mw *= m;
      // principal submatrix of the periodic 1D operator on the window of the subdomain centred
      // on element 1 (R_s A R_s^T; identical for every subdomain)
      const int N1 = op.ne * n;
      std::vector<ld> Ls(m * m), Ms(m);
      for (int a = 0; a < m; ++a) {
        const int ga = (n - no + a) % N1;
        Ms[a] = op.M[ga];
        for (int b = 0; b < m; ++b) Ls[a * m + b] = op.L[size_t(ga) * N1 + (n - no + b) % N1];
      }
      std::vector<ld> lam, Sv;
      // odd windows (always, for n = 2^l + 1): exact-parity eigenvectors, even modes first
      if (m & 1) pmg::gen_eig_parity(m, Ls, Ms, lam, Sv);
      else pmg::gen_eig(m, Ls, Ms, lam, Sv);
      h.lam_min[d] = *std::min_element(lam.begin(), lam.end());
      h.lam_max[d] = *std::max_element(lam.begin(), lam.end());
      h.S[d] = to_d(Sv);
      h.lam[d] = to_d(lam);
      h.W[d] = to_d(pmg::hat_weights(h.basis, h.ov[d]));
    }
    // A_ss regular: every eigenvalue sum lam_x + lam_y + lam_z > 0.  A single
    // direction may be singular (window = whole periodic line) if another one is not.
    // eigen-divide table (exact reciprocal of the FP64 eigenvalue sums, rounded once)
    h.Rz.assign((size_t)h.Mw, 0.0);
    for (int q = 0; q < h.m[1]; ++q)
      for (int pp = 0; pp < h.m[0]; ++pp)
        for (int o = 0; o < h.m[2]; ++o) {
          const ld sum = (ld)h.lam[0][pp] + (ld)h.lam[1][q] + (ld)h.lam[2][o];
          h.Rz[((size_t)pp + (size_t)h.m[0] * q) * h.m[2] + o] = sum != 0 ? (double)(1 / sum) : 0.0;
        }
    const ld smin = h.lam_min[0] + h.lam_min[1] + h.lam_min[2];
    const ld smax = h.lam_max[0] + h.lam_max[1] + h.lam_max[2];
    if (!(smin > 1e-13L * smax)) return fail(c, PMG_ESINGULAR, "restricted operator A_ss not regular");
  }
  c->schwarz_ready = true;
  c->ovl_mode = mode;
  plan_workspace(c);
  return PMG_OK;
}

int dg_num_levels(const dg_ctx *c) { return c ? c->L + 1 : PMG_EINVAL; }

long long dg_ndofs(const dg_ctx *c, int level) {
  if (!c || level < 0 || level > c->L) return -PMG_EINVAL;
  return c->lev[level].N;
}

int dg_level_overlap(const dg_ctx *c, int level, int *n_o, int *m) {
  if (!c || level < 0 || level > c->L) return PMG_EINVAL;
  for (int d = 0; d < 3; ++d) {
    if (n_o) n_o[d] = c->lev[level].ov[d].no;
    if (m) m[d] = c->lev[level].m[d];
  }
  return PMG_OK;
}

int dg_get_table(const dg_ctx *c, int level, int dir, int which, double *out, int cap) {
  if (!c || level < 0 || level > c->L || dir < 0 || dir > 2) return -PMG_EINVAL;
  const LevelHost &h = c->lev[level];
  const std::vector<double> *v = nullptr;
  switch (which) {
    case 0: v = &h.mass[dir]; break;
    case 1: v = &h.D[dir]; break;
    case 2: v = &h.tr[dir]; break;
    case 3: v = &h.S[dir]; break;
    case 4: v = &h.lam[dir]; break;
    case 5: v = &h.W[dir]; break;
    case 6: v = &h.interp; break;
    case 7: v = &h.nodes; break;
    default: return -PMG_EINVAL;
  }
  const int cnt = (int)v->size();
  if (out) std::memcpy(out, v->data(), sizeof(double) * std::min(cnt, cap));
  return cnt;
}

size_t dg_workspace_bytes(const dg_ctx *c) { return c ? c->ws_bytes : 0; }

int dg_bind_workspace(dg_ctx *c, void *dev_ptr, size_t bytes, void *stream) {
  if (!c) return PMG_EINVAL;
  if (!dev_ptr || bytes < c->ws_bytes || (reinterpret_cast<size_t>(dev_ptr) & 255))
    return fail(c, PMG_EWORKSPACE, "workspace too small or not 256-byte aligned");
  c->ws = static_cast<char *>(dev_ptr);
  drop_graphs(c);                                   // graphs baked the old workspace
  cudaStream_t s = S(stream);
  auto up = [&](size_t off, const std::vector<double> &v) -> cudaError_t {
    if (v.empty()) return cudaSuccess;
    return cudaMemcpyAsync(c->ws + off, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, s);
  };
  cudaError_t e = cudaSuccess;
  for (int l = 0; l <= c->L && e == cudaSuccess; ++l) {
    const LevelHost &h = c->lev[l];
    for (int d = 0; d < 3; ++d) {
      if (e == cudaSuccess) e = up(h.o_mass[d], h.mass[d]);
      if (e == cudaSuccess) e = up(h.o_D[d], h.D[d]);
      if (e == cudaSuccess) e = up(h.o_tr[d], h.tr[d]);
      if (e == cudaSuccess) e = up(h.o_S[d], h.S[d]);
      if (e == cudaSuccess) e = up(h.o_lam[d], h.lam[d]);
      if (e == cudaSuccess) e = up(h.o_W[d], h.W[d]);
      if (e == cudaSuccess) e = up(h.o_Daug[d], h.Daug[d]);
    }
    if (e == cudaSuccess) e = up(h.o_interp, h.interp);
    if (e == cudaSuccess && !h.Rz.empty()) e = up(h.o_Rz, h.Rz);
    if (e == cudaSuccess) e = up(h.o_nodes, h.nodes);
  }
  for (int d = 0; d < 3 && e == cudaSuccess; ++d) {
    e = up(c->o_S0[d], c->S0[d]);
    if (e == cudaSuccess) e = up(c->o_lam0[d], c->lam0[d]);
  }
  if (e == cudaSuccess && !c->host_pinned) e = cudaMallocHost(&c->host_pinned, 64 * sizeof(double));
  if (e == cudaSuccess && !c->host_hist) e = cudaMallocHost(&c->host_hist, (pmg::PMG_PCG_HIST + 8) * sizeof(double));
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);   // host vectors must outlive the copies
  if (e != cudaSuccess) {
    c->ws = nullptr;
    return cuda_check(c, e, "dg_bind_workspace");
  }
  return PMG_OK;
}

int dg_apply(dg_ctx *c, int level, const double *u, double *Au, void *stream) {
  int st = check_level(c, level);
  if (st) return st;
  if (!u || !Au || u == Au) return fail(c, PMG_EINVAL, "dg_apply: null or aliased vectors");
  return residual_impl(c, level, u, nullptr, Au, S(stream));
}

int dg_residual(dg_ctx *c, int level, const double *u, const double *f, double *r, void *stream) {
  int st = check_level(c, level);
  if (st) return st;
  if (!u || !f || !r || r == u || r == f) return fail(c, PMG_EINVAL, "dg_residual: null or aliased vectors");
  return residual_impl(c, level, u, f, r, S(stream));
}

int schwarz_smooth(dg_ctx *c, int level, double *u, const double *f, int steps, void *stream) {
  int st = check_level(c, level);
  if (st) return st;
  if (level < 1) return fail(c, PMG_EINVAL, "no smoother on the coarse level");
  if (!c->schwarz_ready) return fail(c, PMG_ESTATE, "dg_schwarz_setup not called");
  if (!u || !f || steps < 0) return fail(c, PMG_EINVAL, "schwarz_smooth: bad arguments");
  return smooth_impl(c, level, u, f, steps, false, S(stream));
}

int dg_schwarz_solve(dg_ctx *c, int level, const double *r, void *stream) {
  int st = check_level(c, level);
  if (st) return st;
  if (level < 1) return fail(c, PMG_EINVAL, "no smoother on the coarse level");
  if (!c->schwarz_ready) return fail(c, PMG_ESTATE, "dg_schwarz_setup not called");
  if (!r) return fail(c, PMG_EINVAL, "dg_schwarz_solve: null vector");
  return fdm_impl(c, level, r, S(stream));
}

int dg_schwarz_fold(dg_ctx *c, int level, double *u, int zero, void *stream) {
  int st = check_level(c, level);
  if (st) return st;
  if (level < 1) return fail(c, PMG_EINVAL, "no smoother on the coarse level");
  if (!c->schwarz_ready) return fail(c, PMG_ESTATE, "dg_schwarz_setup not called");
  if (!u) return fail(c, PMG_EINVAL, "dg_schwarz_fold: null vector");
  pmg::LevelDev d = level_dev(c, level);
  cudaStream_t s = S(stream);
  LAUNCHK(c, K_FOLD, level, s, pmg::launch_fold(d, wsp<double>(c, c->lev[level].o_Z), u, zero != 0, nullptr, s));
  return PMG_OK;
}

int dg_window_buffer(const dg_ctx *c, int level, size_t *byte_offset, long long *doubles_per_subdomain) {
  if (!c || level < 1 || level > c->L || !c->schwarz_ready || !byte_offset || !doubles_per_subdomain)
    return PMG_EINVAL;
  *byte_offset = c->lev[level].o_Z;
  *doubles_per_subdomain = c->lev[level].Mw;
  return PMG_OK;
}

int dg_dot_range(dg_ctx *c, const double *x, const double *y, long long count, double *out_host,
                 void *stream) {
  if (!c) return PMG_EINVAL;
  if (!c->ws) return fail(c, PMG_ESTATE, "workspace not bound");
  if (!x || !y || !out_host || count < 0 || count > c->lev[c->L].N)
    return fail(c, PMG_EINVAL, "dg_dot_range: bad arguments");
  cudaStream_t s = S(stream);
  double *part = wsp<double>(c, c->o_part), *scal = wsp<double>(c, c->o_scal);
  LAUNCH(c, pmg::launch_dot(x, y, count, part, scal + 20, s));
  cudaError_t e = cudaMemcpyAsync(c->host_pinned, scal + 20, sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_check(c, e, "dg_dot_range");
  *out_host = c->host_pinned[0];
  return PMG_OK;
}

int dg_axpby(dg_ctx *c, double *y, double a, const double *x, double b, long long count, void *stream) {
  if (!c) return PMG_EINVAL;
  if (!x || !y || count < 0) return fail(c, PMG_EINVAL, "dg_axpby: bad arguments");
  cudaStream_t s = S(stream);
  LAUNCH(c, pmg::launch_axpby(y, a, x, b, count, s));
  return PMG_OK;
}

int dg_prolongate_add(dg_ctx *c, int level, const double *uc, double *uf, void *stream) {
  int st = check_level(c, level);
  if (st) return st;
  if (level < 1 || !uc || !uf) return fail(c, PMG_EINVAL, "dg_prolongate_add: bad arguments");
  pmg::LevelDev d = level_dev(c, level);
  cudaStream_t s = S(stream);
  const LevelHost &h = c->lev[level];
  if (h.o_x1 && c->ws)
    LAUNCHK(c, K_PROLONG, level, s, pmg::launch_prolong_global(d, c->lev[level - 1].n,
                                  wsp<double>(c, h.o_interp), uc, uf, wsp<double>(c, h.o_x1),
                                  wsp<double>(c, h.o_x2), s));
  else
    LAUNCHK(c, K_PROLONG, level, s, pmg::launch_prolong(d, c->lev[level - 1].n,
                                  wsp<double>(c, h.o_interp), uc, uf, s));
  return PMG_OK;
}

int dg_restrict(dg_ctx *c, int level, const double *rf, double *fc, void *stream) {
  int st = check_level(c, level);
  if (st) return st;
  if (level < 1 || !rf || !fc) return fail(c, PMG_EINVAL, "dg_restrict: bad arguments");
  pmg::LevelDev d = level_dev(c, level);
  cudaStream_t s = S(stream);
  const LevelHost &h = c->lev[level];
  if (h.o_x1 && c->ws)
    LAUNCHK(c, K_RESTRICT, level, s, pmg::launch_restrict_global(d, c->lev[level - 1].n,
                                   wsp<double>(c, h.o_interp), rf, fc, wsp<double>(c, h.o_x1),
                                   wsp<double>(c, h.o_x2), s));
  else
    LAUNCHK(c, K_RESTRICT, level, s, pmg::launch_restrict(d, c->lev[level - 1].n,
                                   wsp<double>(c, h.o_interp), rf, fc, s));
  return PMG_OK;
}

int dg_coarse_solve(dg_ctx *c, const double *f0, double *u0, void *stream) {
  int st = check_level(c, 0);
  if (st) return st;
  if (!f0 || !u0 || f0 == u0) return fail(c, PMG_EINVAL, "dg_coarse_solve: bad arguments");
  return coarse_impl(c, f0, u0, S(stream));
}

int dg_set_schedule(dg_ctx *c, const int *nu1, const int *nu2) {
  if (!c || !nu1 || !nu2) return PMG_EINVAL;
  for (int l = 1; l <= c->L; ++l)
    if (nu1[l] < 0 || nu2[l] < 0) return fail(c, PMG_EINVAL, "negative smoothing count");
  for (int l = 0; l <= c->L; ++l) { c->nu1[l] = nu1[l]; c->nu2[l] = nu2[l]; }
  drop_graphs(c);
  return PMG_OK;
}

int pmg_vcycle(dg_ctx *c, double *u, const double *f, void *stream) {
  int st = check_level(c, c ? c->L : 0);
  if (st) return st;
  if (!c->schwarz_ready) return fail(c, PMG_ESTATE, "dg_schwarz_setup not called");
  if (!u || !f || u == f) return fail(c, PMG_EINVAL, "pmg_vcycle: bad arguments");
  return vcycle_run(c, u, f, false, S(stream));
}

namespace {

// Build the whole inexact PCG solve as one CUDA graph: prologue (r0, z0 = V(0,
// r0), p0, <z0, r0>), then a conditional WHILE node whose body is one iteration (q = A p, alpha,
// u/r update, ||r||, device-side convergence test k_pcg_check) followed by a conditional IF node
// (z = V(0, r), Golub-Ye beta, p update) that runs only while the solve continues.  The kernels
// and their order are those of the host-driven loop below, so the iterates are identical; the
// host synchronises once per solve (to read the iteration count, status and history).
int pcg_graph_build(dg_ctx *c, double *u, const double *f, double rtol, int maxit, dg_ctx::PcgGraph &out) {
  const int L = c->L;
  const long long N = c->lev[L].N;
  double *r = wsp<double>(c, c->o_pr), *z = wsp<double>(c, c->o_pz), *p = wsp<double>(c, c->o_pp);
  double *q = wsp<double>(c, c->o_pq), *rold = wsp<double>(c, c->o_prold);
  double *part = wsp<double>(c, c->o_part), *scal = wsp<double>(c, c->o_scal);
  double *hist = wsp<double>(c, c->o_hist);
  cudaError_t e = cudaSuccess;
  if (!c->cap_stream) e = cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess && !c->cap_stream2) e = cudaStreamCreateWithFlags(&c->cap_stream2, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_check(c, e, "cudaStreamCreate");
  cudaStream_t s = c->cap_stream, s2 = c->cap_stream2;
  cudaGraph_t G = nullptr;
  if ((e = cudaGraphCreate(&G, 0)) != cudaSuccess) return cuda_check(c, e, "cudaGraphCreate");
  cudaGraphConditionalHandle hw, hi;
  e = cudaGraphConditionalHandleCreate(&hw, G, 0, 0);
  if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&hi, G, 0, 0);
  if (e != cudaSuccess) { cudaGraphDestroy(G); return cuda_check(c, e, "cudaGraphConditionalHandleCreate"); }
  int st = PMG_OK;
  auto add_cond = [&](cudaStream_t cs, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type,
                      cudaGraph_t &body) -> cudaError_t {
    cudaStreamCaptureStatus cst;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    cudaError_t ee = cudaStreamGetCaptureInfo(cs, &cst, nullptr, &cg, &deps, &nd);
    if (ee != cudaSuccess) return ee;
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = type;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    if ((ee = cudaGraphAddNode(&node, cg, deps, nd, &np)) != cudaSuccess) return ee;
    body = np.conditional.phGraph_out[0];
    return cudaStreamUpdateCaptureDependencies(cs, &node, 1, cudaStreamSetCaptureDependencies);
  };
  const long long l0 = c->launches;
  cudaGraph_t wbody = nullptr, ibody = nullptr;
  // prologue
  e = cudaStreamBeginCaptureToGraph(s, G, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    st = residual_impl(c, L, u, f, r, s);                                        // r0 = f - A u0
    if (!st) st = pmg::launch_dot(r, r, N, part, scal + 2, s) ? PMG_ECUDA : PMG_OK;
    if (!st) st = pmg::launch_pcg_start(scal, hist, maxit, hw, s) ? PMG_ECUDA : PMG_OK;
    if (!st) st = vcycle_impl(c, z, r, true, s);                                 // z0 = V(0, r0)
    if (!st) st = pmg::launch_copy(p, z, N, s) ? PMG_ECUDA : PMG_OK;             // p0 = z0
    if (!st) st = pmg::launch_zr_beta(z, r, r, N, part, scal, true, s) ? PMG_ECUDA : PMG_OK;
    c->launches += 4;
    if (!st) e = add_cond(s, hw, cudaGraphCondTypeWhile, wbody);
    cudaGraph_t G2 = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(s, &G2);
    if (e == cudaSuccess) e = e2;
  }
  out.lp = c->launches - l0;
  // while body: one iteration up to the convergence test, then the IF node
  if (!st && e == cudaSuccess) {
    const long long l1 = c->launches;
    e = cudaStreamBeginCaptureToGraph(s2, wbody, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      st = residual_impl(c, L, p, nullptr, q, s2);                               // q = A p
      if (!st) st = pmg::launch_pq_alpha(p, q, N, part, scal, s2) ? PMG_ECUDA : PMG_OK;
      if (!st) st = pmg::launch_cg_update(u, r, rold, p, q, N, part, scal, s2) ? PMG_ECUDA : PMG_OK;
      if (!st) st = pmg::launch_pcg_check(scal, hist, rtol, maxit, hw, hi, s2) ? PMG_ECUDA : PMG_OK;
      c->launches += 3;
      if (!st) e = add_cond(s2, hi, cudaGraphCondTypeIf, ibody);
      cudaGraph_t W2 = nullptr;
      cudaError_t e2 = cudaStreamEndCapture(s2, &W2);
      if (e == cudaSuccess) e = e2;
    }
    out.lw = c->launches - l1;
  }
  if (!st && e == cudaSuccess) {
    const long long l2 = c->launches;
    e = cudaStreamBeginCaptureToGraph(s2, ibody, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      st = vcycle_impl(c, z, r, true, s2);                                       // z = V(0, r)
      if (!st) st = pmg::launch_zr_beta(z, r, rold, N, part, scal, false, s2) ? PMG_ECUDA : PMG_OK;
      if (!st) st = pmg::launch_p_update(p, z, N, scal, s2) ? PMG_ECUDA : PMG_OK;  // p = z + beta p
      c->launches += 2;
      cudaGraph_t I2 = nullptr;
      cudaError_t e2 = cudaStreamEndCapture(s2, &I2);
      if (e == cudaSuccess) e = e2;
    }
    out.li = c->launches - l2;
  }
  c->launches = l0;
  if (st || e != cudaSuccess) {
    cudaGraphDestroy(G);
    return st ? st : cuda_check(c, e, "pcg graph capture");
  }
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, G, 0);
  cudaGraphDestroy(G);
  if (e != cudaSuccess) return cuda_check(c, e, "cudaGraphInstantiate (pcg)");
  out.u = u; out.f = f; out.rtol = rtol; out.maxit = maxit; out.exec = exec;
  return PMG_OK;
}

}  // namespace

int pcg_solve(dg_ctx *c, double *u, const double *f, double rtol, int maxit, int *iters,
              double *res_hist, void *stream) {
  int st = check_level(c, c ? c->L : 0);
  if (st) return st;
  if (!c->schwarz_ready) return fail(c, PMG_ESTATE, "dg_schwarz_setup not called");
  if (!u || !f || maxit < 0) return fail(c, PMG_EINVAL, "pcg_solve: bad arguments");
  cudaStream_t s = S(stream);
  if (c->graphs && !c->prof && maxit < pmg::PMG_PCG_HIST) {
    const dg_ctx::PcgGraph *pg = nullptr;
    for (auto &g : c->pcg_cache)
      if (g.u == u && g.f == f && g.rtol == rtol && g.maxit == maxit) pg = &g;
    if (!pg) {
      dg_ctx::PcgGraph ng;
      if ((st = pcg_graph_build(c, u, f, rtol, maxit, ng))) return st;
      c->pcg_cache.push_back(ng);
      pg = &c->pcg_cache.back();
    }
    double *scal = wsp<double>(c, c->o_scal), *hist = wsp<double>(c, c->o_hist);
    cudaError_t e = cudaGraphLaunch(pg->exec, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->host_pinned, scal + 30, 3 * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_check(c, e, "pcg_solve (graph)");
    const int k = (int)c->host_pinned[1];
    const int status = (int)c->host_pinned[2];
    c->launches += pg->lp + (long long)k * pg->lw + (long long)std::max(k - 1, 0) * pg->li;
    if (iters) *iters = k;
    if (res_hist) {
      e = cudaMemcpy(c->host_hist, hist, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_check(c, e, "pcg_solve history");
      std::memcpy(res_hist, c->host_hist, sizeof(double) * (k + 1));
    }
    if (status == PMG_EDIVERGED) return fail(c, PMG_EDIVERGED, k == 0 ? "non-finite initial residual" : "PCG diverged");
    if (status == PMG_EMAXIT) return fail(c, PMG_EMAXIT, "PCG reached maxit");
    return PMG_OK;
  }
  const int L = c->L;
  const long long N = c->lev[L].N;
  double *r = wsp<double>(c, c->o_pr), *z = wsp<double>(c, c->o_pz), *p = wsp<double>(c, c->o_pp);
  double *q = wsp<double>(c, c->o_pq), *rold = wsp<double>(c, c->o_prold);
  double *part = wsp<double>(c, c->o_part), *scal = wsp<double>(c, c->o_scal);
  auto read_scalar = [&](int slot, double *v) -> int {
    cudaError_t e = cudaMemcpyAsync(c->host_pinned, scal + slot, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_check(c, e, "pcg_solve scalar read");
    *v = c->host_pinned[0];
    return PMG_OK;
  };
  if ((st = residual_impl(c, L, u, f, r, s))) return st;               // r0 = f - A u0
  LAUNCH(c, pmg::launch_dot(r, r, N, part, scal + 2, s));
  double rr0;
  if ((st = read_scalar(2, &rr0))) return st;
  const double r0 = std::sqrt(rr0);
  if (res_hist) res_hist[0] = r0;
  if (iters) *iters = 0;
  if (!std::isfinite(r0)) return fail(c, PMG_EDIVERGED, "non-finite initial residual");
  if (r0 == 0) return PMG_OK;
  if ((st = vcycle_run(c, z, r, true, s))) return st;                   // z0 = V(0, r0)
  LAUNCH(c, pmg::launch_copy(p, z, N, s));                              // p0 = z0
  LAUNCH(c, pmg::launch_zr_beta(z, r, r, N, part, scal, true, s));      // zr = <z0, r0>
  for (int k = 1; k <= maxit; ++k) {
    if ((st = residual_impl(c, L, p, nullptr, q, s))) return st;        // q = A p
    LAUNCH(c, pmg::launch_pq_alpha(p, q, N, part, scal, s));            // alpha = zr / <p,q>
    LAUNCH(c, pmg::launch_cg_update(u, r, rold, p, q, N, part, scal, s));   // u, r update; rr
    double rr;
    if ((st = read_scalar(2, &rr))) return st;
    const double rn = std::sqrt(rr);
    if (res_hist) res_hist[k] = rn;
    if (iters) *iters = k;
    if (!std::isfinite(rn) || rn > 1e3 * r0) return fail(c, PMG_EDIVERGED, "PCG diverged");
    if (rn <= rtol * r0) return PMG_OK;
    if (k == maxit) break;
    if ((st = vcycle_run(c, z, r, true, s))) return st;                 // z = V(0, r)
    LAUNCH(c, pmg::launch_zr_beta(z, r, rold, N, part, scal, false, s));  // beta (Golub-Ye)
    LAUNCH(c, pmg::launch_p_update(p, z, N, scal, s));                  // p = z + beta p
  }
  return fail(c, PMG_EMAXIT, "PCG reached maxit");
}

int dg_dot(dg_ctx *c, int level, const double *x, const double *y, double *out_host, void *stream) {
  int st = check_level(c, level);
  if (st) return st;
  if (!x || !y || !out_host) return fail(c, PMG_EINVAL, "dg_dot: bad arguments");
  cudaStream_t s = S(stream);
  double *part = wsp<double>(c, c->o_part), *scal = wsp<double>(c, c->o_scal);
  LAUNCH(c, pmg::launch_dot(x, y, c->lev[level].N, part, scal + 20, s));
  cudaError_t e = cudaMemcpyAsync(c->host_pinned, scal + 20, sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_check(c, e, "dg_dot");
  *out_host = c->host_pinned[0];
  return PMG_OK;
}

int dg_project_mean(dg_ctx *c, int level, double *v, void *stream) {
  int st = check_level(c, level);
  if (st) return st;
  if (!v) return fail(c, PMG_EINVAL, "dg_project_mean: null vector");
  cudaStream_t s = S(stream);
  const long long N = c->lev[level].N;
  double *part = wsp<double>(c, c->o_part), *scal = wsp<double>(c, c->o_scal);
  LAUNCH(c, pmg::launch_sum(v, N, part, scal + 21, 1.0 / N, s));
  LAUNCH(c, pmg::launch_sub_scalar(v, N, scal + 21, s));
  return PMG_OK;
}

int dg_rhs_sin(dg_ctx *c, double amp, double kx, double ky, double kz, double *b, void *stream) {
  int st = check_level(c, c ? c->L : 0);
  if (st) return st;
  if (!b) return fail(c, PMG_EINVAL, "dg_rhs_sin: null vector");
  pmg::LevelDev d = level_dev(c, c->L);
  cudaStream_t s = S(stream);
  LAUNCH(c, pmg::launch_rhs_sin(d, c->len[0] / c->ne[0], c->len[1] / c->ne[1], c->len[2] / c->ne[2],
                                amp, kx, ky, kz, b, s));
  return dg_project_mean(c, c->L, b, stream);
}

long long dg_launch_count(const dg_ctx *c) { return c ? c->launches : -1; }

int dg_set_colored(dg_ctx *c, int enable) {
  if (!c) return PMG_EINVAL;
  c->colored = enable != 0;
  drop_graphs(c);
  return PMG_OK;
}

int dg_set_graphs(dg_ctx *c, int enable) {
  if (!c) return PMG_EINVAL;
  c->graphs = enable != 0;
  return PMG_OK;
}

int dg_profile(dg_ctx *c, int enable) {
  if (!c) return PMG_EINVAL;
  c->prof = enable != 0;
  return PMG_OK;
}

int dg_profile_read(dg_ctx *c, double *ms_out, long long *count_out, int reset) {
  if (!c) return PMG_EINVAL;
  for (size_t i = 0; i < c->ev_slot.size(); ++i) {
    cudaError_t e = cudaEventSynchronize(c->ev_pool[2 * i + 1]);
    if (e != cudaSuccess) return cuda_check(c, e, "dg_profile_read");
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]);
    c->prof_ms[c->ev_slot[i]] += ms;
    c->prof_cnt[c->ev_slot[i]] += 1;
  }
  c->ev_slot.clear();
  for (int i = 0; i < PMG_PROF_SLOTS; ++i) {
    if (ms_out) ms_out[i] = c->prof_ms[i];
    if (count_out) count_out[i] = c->prof_cnt[i];
    if (reset) { c->prof_ms[i] = 0; c->prof_cnt[i] = 0; }
  }
  return PMG_OK;
}

const char *dg_last_error(const dg_ctx *c) { return c ? c->err.c_str() : "null context"; }

void dg_destroy(dg_ctx *c) {
  if (!c) return;
  if (c->host_pinned) cudaFreeHost(c->host_pinned);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  drop_graphs(c);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->cap_stream2) cudaStreamDestroy(c->cap_stream2);
  if (c->host_hist) cudaFreeHost(c->host_hist);
  delete c;
}

}  // extern "C"
