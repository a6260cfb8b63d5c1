// Matrix-free IP-DG operator apply / residual (+ fused restriction) and face traces.
// arXiv:1612.04796; PAPER.md line numbers cited per kernel.
#include <algorithm>

#include "kcommon.cuh"
#include "colmap17.cuh"

namespace pmg {
namespace {

// ---------------------------------------------------------------------------------------------
// Face traces (value and normal derivative on both faces of every direction) — the data the
// rank-2 neighbour couplings of Eq. 7's block-tridiagonal L_* need.
__global__ void k_traces(LevelDev L, const double *__restrict__ u, double *__restrict__ T) {
  const int n = L.n, n2 = n * n, n3 = n2 * n;
  const int e = blockIdx.x;
  const double *ue = u + (long long)e * n3;
  double *Te = T + (long long)e * 12 * n2;
  // 2D grid: blockIdx.y splits the 3 n^2 face points (large elements fill the GPU)
  __shared__ __align__(16) double tab[3 * trace_tab_len(PMG_MAX_N) + 2];
  stage_trace_tab(L, tab);
  __syncthreads();
  // n = 33 (P = 32): compile-time extent, so the 33 strided global loads of a line are all in
  // flight before the first FMA (the rolled loop waited on every pair: 16.7 us per launch at c4)
  if (n == 33) {
    for (int t = blockIdx.y * blockDim.x + threadIdx.x; t < 3 * n2; t += gridDim.y * blockDim.x)
      elem_trace_item<33>(ue, tab, n, t, Te);
  } else {
    for (int t = blockIdx.y * blockDim.x + threadIdx.x; t < 3 * n2; t += gridDim.y * blockDim.x)
      elem_trace_item<0>(ue, tab, n, t, Te);
  }
}

// Operator apply v = A u (Eq. 7) or residual r = f - A u (Eq. 8), sum-factorised per element.
__global__ void k_apply(LevelDev L, const double *__restrict__ u, const double *__restrict__ T,
                        const double *__restrict__ f, double *__restrict__ out) {
  const int n = L.n, n2 = n * n, n3 = n2 * n;
  const int e = blockIdx.x;
  const int ex = e % L.nx, ey = (e / L.nx) % L.ny, ez = e / (L.nx * L.ny);
  const int ecoord[3] = {ex, ey, ez};
  const int edim[3] = {L.nx, L.ny, L.nz};
  int nbL[3], nbR[3];
  for (int d = 0; d < 3; ++d) {
    int c[3] = {ex, ey, ez};
    c[d] = wrap(ecoord[d] - 1, edim[d]);
    nbL[d] = c[0] + L.nx * (c[1] + L.ny * c[2]);
    c[d] = wrap(ecoord[d] + 1, edim[d]);
    nbR[d] = c[0] + L.nx * (c[1] + L.ny * c[2]);
  }
  const double *ue = u + (long long)e * n3;
  for (int t = threadIdx.x; t < n3; t += blockDim.x) {
    const int i = t % n, j = (t / n) % n, k = t / n2;
    const int idx[3] = {i, j, k};
    const int pface[3] = {j + n * k, i + n * k, i + n * j};
    const int stride[3] = {1, n, n2};
    double s[3];
    for (int d = 0; d < 3; ++d) {
      const int id = idx[d];
      const double *Dr = L.D[d] + id * n;
      const double *line = ue + (t - id * stride[d]);
      double acc = 0;
      for (int q = 0; q < n; ++q) acc += Dr[q] * __ldg(line + q * stride[d]);
      const double *TR = T + ((long long)nbR[d] * 3 + d) * 4 * n2;
      const double *TL = T + ((long long)nbL[d] * 3 + d) * 4 * n2;
      const double tvR = TR[pface[d]], tdR = TR[n2 + pface[d]];
      const double tvL = TL[2 * n2 + pface[d]], tdL = TL[3 * n2 + pface[d]];
      const double *tr = L.tr[d];
      const double mu = L.mu[d];
      acc += tr[id] * (-0.5 * tdR - mu * tvR) + tr[n + id] * (0.5 * tvR)
           + tr[2 * n + id] * (0.5 * tdL - mu * tvL) + tr[3 * n + id] * (-0.5 * tvL);
      s[d] = acc;
    }
    const double mx = L.mass[0][i], my = L.mass[1][j], mz = L.mass[2][k];
    const double v = mz * my * s[0] + mz * mx * s[1] + my * mx * s[2];
    const long long g = (long long)e * n3 + t;
    out[g] = f ? f[g] - v : v;
  }
}

// Even/odd line GEMM of the apply for n = 17 (H = 8).  The element stiffness rows of Eq. 7 are
// centro-symmetric (D_{16-i,16-k} = D_{ik}, a_{16-i} = b_i, ap_{16-i} = -bp_i on the symmetric
// GL/GLL nodes), so with e_k = u_k + u_{16-k}, o_k = u_k - u_{16-k}:
//   out_i + out_{16-i} = sum_{k<8} (D_ik + D_{i,16-k}) e_k + 2 D_i8 u_8 + (a_i + b_i)(c1 + c3) + (ap_i - bp_i)(c2 - c4)
//   out_i - out_{16-i} = sum_{k<8} (D_ik - D_{i,16-k}) o_k + (a_i - b_i)(c1 - c3) + (ap_i + bp_i)(c2 + c4)
// Both halves take the same B fragments lo +- hi (K slots 0-7: (u_k, u_{16-k}); 8: (u_8, u_8);
// 9: (c1, c3); 10: (c2, -c4), the transform stores -c4; 11: zero A column), so a tile needs 3 + 3
// DMMAs (rows 0-7) plus an FMA tail for the middle row instead of 2 x 6.  The 1/2 of
// out = (E +- O)/2 is folded into A.
// cmap: tile slot -> column p + n q (scripts/gen_colmap17.py): tiles whose base addresses are
// spread over the 16 double banks, so the B loads and the C stores are conflict free.
// A fragments of the even/odd n = 17 line GEMM for lane (g, t): E rows, O rows, E tail row,
// per K slice ks = 0..2 — built once per CTA into shared memory (eo17_afrag) so each pass loads
// 9 values per lane instead of re-deriving them from Daug in global memory for every element.
constexpr int EO17_AF = 9 * 32;     // doubles per direction
__device__ __forceinline__ void eo17_afrag(const double *__restrict__ Daug, double *af) {
  constexpr int n = 17, H = 8, KA = n + 4;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int ks = 0; ks < 3; ++ks) {
    const int k = ks * 4 + t;
    auto coefE = [&](int i) {
      const double *r = Daug + i * KA;
      if (k < H) return 0.5 * (r[k] + r[n - 1 - k]);
      if (k == H) return 0.5 * r[H];
      if (k == 9) return 0.5 * (r[n] + r[n + 2]);
      if (k == 10) return 0.5 * (r[n + 1] - r[n + 3]);
      return 0.0;
    };
    const double *r = Daug + g * KA;
    double aO;
    if (k < H) aO = 0.5 * (r[k] - r[n - 1 - k]);
    else if (k == 9) aO = 0.5 * (r[n] - r[n + 2]);
    else if (k == 10) aO = 0.5 * (r[n + 1] + r[n + 3]);
    else aO = 0.0;
    af[(0 * 3 + ks) * 32 + lane] = coefE(g);
    af[(1 * 3 + ks) * 32 + lane] = aO;
    af[(2 * 3 + ks) * 32 + lane] = coefE(H);
  }
}

#ifndef PMG_APPLY17_THREADS
#define PMG_APPLY17_THREADS 256     // CTA width of the n = 17 apply (2 CTAs per SM)
#endif

template <int DIR, bool FIRST>
__device__ __forceinline__ void apply_eo17(const double *U, const double *Cfd, double *V,
                                           const double *af, const unsigned short *cmap,
                                           const unsigned short *cmapY) {
  constexpr int n = 17, n2 = n * n, H = 8;
  constexpr int PD = Other<DIR>::P, QD = Other<DIR>::Q;
  constexpr int SO = DIR == 0 ? 1 : (DIR == 1 ? n : n2);
  constexpr int SP = PD == 0 ? 1 : (PD == 1 ? n : n2);
  constexpr int SQ = QD == 0 ? 1 : (QD == 1 ? n : n2);
  constexpr int NCOL = n2, NT = (NCOL + 7) / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  if (warp >= NT) return;
  // column nn = p + n q -> offset p SP + q SQ without a division: n nn (x pass), the cmapY
  // table p + n^2 q (y pass), nn itself (z pass); the face coefficients sit at Cfd + nn
  auto coloff = [&](int slot, int nn) {
    (void)slot;
    return DIR == 0 ? n * nn : (DIR == 1 ? (int)cmapY[slot] : nn);
  };
  // A fragments (row i = g for E and O; tail row 8 for E), K slot k = 4 ks + t
  double aE[3], aO[3], at[3];
#pragma unroll
  for (int ks = 0; ks < 3; ++ks) {
    aE[ks] = af[(0 * 3 + ks) * 32 + lane];
    aO[ks] = af[(1 * 3 + ks) * 32 + lane];
    at[ks] = af[(2 * 3 + ks) * 32 + lane];
  }
  // B sources: lo / hi offsets, from U (k <= 8, 11) or from the face coefficients Cf (k = 9, 10)
  bool fromC[3];
  int o1[3], o2[3];
#pragma unroll
  for (int ks = 0; ks < 3; ++ks) {
    const int k = ks * 4 + t;
    fromC[ks] = (k == 9 || k == 10);
    if (k == 9) { o1[ks] = 0; o2[ks] = 2 * n2; }
    else if (k == 10) { o1[ks] = n2; o2[ks] = 3 * n2; }
    else { const int kk = k < H ? k : H; o1[ks] = kk * SO; o2[ks] = (n - 1 - kk) * SO; }
  }
  // one tile: B loads, 3 + 3 DMMAs (two accumulator chains), FMA tail row with a 2-step shuffle
  auto compute = [&](int tile, double (&cE)[2], double (&cO)[2], double &tl, int &ob) {
    const int nb = cmap[tile * 8 + g];
    ob = coloff(tile * 8 + g, nb);
    const double *xb = U + ob;
    const double *cb = Cfd + nb;
    double bE[3], bO[3];
#pragma unroll
    for (int ks = 0; ks < 3; ++ks) {
      const double *src = fromC[ks] ? cb : xb;
      const double v1 = src[o1[ks]], v2 = src[o2[ks]];
      bE[ks] = v1 + v2;
      bO[ks] = v1 - v2;
    }
    cE[0] = cE[1] = cO[0] = cO[1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 3; ++ks) {
      dmma884(cE[0], cE[1], aE[ks], bE[ks]);
      dmma884(cO[0], cO[1], aO[ks], bO[ks]);
    }
    tl = 0.0;
#pragma unroll
    for (int ks = 0; ks < 3; ++ks) tl = fma(at[ks], bE[ks], tl);
    tl += __shfl_xor_sync(0xffffffffu, tl, 1);
    tl += __shfl_xor_sync(0xffffffffu, tl, 2);
  };
  auto epilogue = [&](int tile, const double (&cE)[2], const double (&cO)[2], double tl, int ob) {
    // dead slots (the last tile's 7 duplicates of column 288) run the same loads and only predicate
    // the stores: no divergent region in the tile loop
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int slot = tile * 8 + 2 * t + j;
      const bool ok = slot < NCOL;
      double *vb = V + coloff(slot, cmap[slot]);
      double lo = cE[j] + cO[j], hi = cE[j] - cO[j];
      if (!FIRST) { lo += vb[g * SO]; hi += vb[(n - 1 - g) * SO]; }
      if (ok) { vb[g * SO] = lo; vb[(n - 1 - g) * SO] = hi; }
    }
    {
      double *vb = V + ob + H * SO;
      if (!FIRST) tl += *vb;
      if (t == 0 && tile * 8 + g < NCOL) *vb = tl;
    }
  };
  // software pipelined: the DMMAs of tile i + nw are issued before the epilogue of tile i
  double cE0[2], cO0[2], cE1[2], cO1[2], tl0, tl1;
  int ob0, ob1;
  int tile = warp;
  compute(tile, cE0, cO0, tl0, ob0);
  for (;;) {
    const int t1 = tile + nw;
    // (no __syncwarp: U and Cf are read-only in a pass and every V address is read and written
    // by one lane only)
    if (t1 < NT) compute(t1, cE1, cO1, tl1, ob1);
    epilogue(tile, cE0, cO0, tl0, ob0);
    if (t1 >= NT) break;
    const int t2 = t1 + nw;
    if (t2 < NT) compute(t2, cE0, cO0, tl0, ob0);
    epilogue(t1, cE1, cO1, tl1, ob1);
    if (t2 >= NT) break;
    tile = t2;
  }
}

// smem: U (n^3) | V (n^3) | face coefficients 3 x 4 x n^2 | mass 3 x n
// Per direction d the line GEMM is  V += M_p M_q [D | a ap b bp] [U-lines ; c1 c2 c3 c4]  where
// c1..c4 are the neighbour-trace coefficients of the rank-2 couplings on the face point (p,q):
// c1 = -tdR/2 - mu tvR, c2 = tvR/2, c3 = tdL/2 - mu tvL, c4 = -tvL/2.
// NT = n (compile time, n = 2^l + 1 or 2), NC = (n + 1) / 2 the next-coarser n (fused restriction)
// WIDE: 256-thread CTAs for n <= 9 when the whole mesh is one wave (latency-bound small meshes)
template <int NT, bool WIDE = false>
__global__ void __launch_bounds__(NT == 17 ? PMG_APPLY17_THREADS : ((NT <= 9 && !WIDE) ? 128 : 256), NT <= 9 ? (WIDE ? 4 : 8) : 2) k_apply_mma(LevelDev L, const double *__restrict__ u,
                                                      const double *__restrict__ T,
                                                      const double *__restrict__ f,
                                                      double *__restrict__ out,
                                                      const double *__restrict__ restrict_I,
                                                      double *__restrict__ fc) {
  extern __shared__ double sm[];
  constexpr int n = NT, n2 = n * n, n3 = n2 * n;
  constexpr int NC = NT > 2 ? (NT + 1) / 2 : 1;
  // smem: U staging (n^3 + 2, 16-byte aligned superset of the element) | V | Cf | mass | mbarrier
  double *Us = sm, *V = sm + n3 + 2, *Cf = V + n3, *ms = Cf + 12 * n2;
  unsigned long long *mbar = reinterpret_cast<unsigned long long *>(ms + 3 * n);
  unsigned short *cmap = reinterpret_cast<unsigned short *>(mbar + 1);      // n = 17 only
  unsigned short *cmapY = cmap + ((PMG_COLMAP17_LEN + 3) & ~3);            // n = 17: p + n^2 q
  double *af17 = reinterpret_cast<double *>(cmapY + ((PMG_COLMAP17_LEN + 3) & ~3));  // n = 17: 3 x EO17_AF
  const int edim[3] = {L.nx, L.ny, L.nz};
  const unsigned tbytes = 16u * n2;                                // 2 n^2 doubles per segment
  // Persistent: CTA b handles elements b, b + grid, ...  While element e is computed, the next
  // element's block, its neighbour-trace segments and e's f block are prefetched into L2
  // (cp.async.bulk.prefetch), so the HBM stream keeps running under the DMMA passes and the
  // next TMA load and the epilogue's f reads are served from L2.
  auto trace_src = [&](int e, int d, int side) {                   // side 0: right nb (tvR, tdR)
    int c[3] = {e % L.nx, (e / L.nx) % L.ny, e / (L.nx * L.ny)};
    c[d] = wrap(c[d] + (side ? -1 : 1), edim[d]);
    return T + ((long long)(c[0] + L.nx * (c[1] + L.ny * c[2])) * 3 + d) * 4 * n2 + side * 2 * n2;
  };
  auto u_plan = [&](int e, int &pre, int &ucount) {
    const double *ue = u + (long long)e * n3;
    pre = (int)((reinterpret_cast<unsigned long long>(ue) >> 3) & 1);
    ucount = (n3 + pre + 1) & ~1;                                  // doubles, multiple of 2
    return (long long)e * n3 - pre + ucount <= (long long)L.Ne * n3;
  };
  if (threadIdx.x == 0) mbar_init(mbar, 1);
  for (int d = 0; d < 3; ++d) stage(ms + d * n, L.mass[d], n);
  if constexpr (NT == 17) {
    for (int i = threadIdx.x; i < PMG_COLMAP17_LEN; i += blockDim.x) {
      const int nn = kColMap17[i];
      cmap[i] = (unsigned short)nn;
      cmapY[i] = (unsigned short)(nn % n + n2 * (nn / n));
    }
    const int w = threadIdx.x >> 5;
    if (w < 3) eo17_afrag(L.Daug[w], af17 + w * EO17_AF);
  }
  __syncthreads();
  unsigned phase = 0;
#ifdef PMG_PHASE_TIMING
  long long tacc[7] = {0, 0, 0, 0, 0, 0, 0}, tp = clock64(), tq;
#define PMG_APH(i) (tq = clock64(), tacc[i] += tq - tp, tp = tq)
#else
#define PMG_APH(i)
#endif
  for (int e = blockIdx.x; e < L.Ne; e += gridDim.x, phase ^= 1u) {
    // TMA bulk staging: the element block and the six neighbour-trace segments (2 n^2 doubles,
    // 16-byte aligned) in 7 copies tracked by one mbarrier.  Element blocks (n^3 doubles, n odd)
    // alternate 8/16-byte alignment, so a 16-byte aligned superset is copied and U is offset.
    const double *ue = u + (long long)e * n3;
    int pre, ucount;
    const bool tail_ok = u_plan(e, pre, ucount);
    double *U = Us + pre;
    if (threadIdx.x == 0) {
      // the previous element's generic stores to Us / Cf (coefficient rewrite, fused restriction,
      // cp.async fallback) were ordered by the loop-end barrier; order them before the bulk writes
      fence_proxy_async_smem();
      mbar_expect_tx(mbar, (tail_ok ? ucount * 8u : 0u) + 6u * tbytes);
      if (tail_ok) bulk_g2s(Us, ue - pre, ucount * 8u, mbar);
      for (int d = 0; d < 3; ++d) {
        bulk_g2s(Cf + d * 4 * n2, trace_src(e, d, 0), tbytes, mbar);
        bulk_g2s(Cf + d * 4 * n2 + 2 * n2, trace_src(e, d, 1), tbytes, mbar);
      }
      const int en = e + gridDim.x;
      if (en < L.Ne) {
        int pn, cn;
        if (u_plan(en, pn, cn)) prefetch_l2(u + (long long)en * n3 - pn, cn * 8u);
        for (int d = 0; d < 3; ++d) {
          prefetch_l2(trace_src(en, d, 0), tbytes);
          prefetch_l2(trace_src(en, d, 1), tbytes);
        }
      }
      if (f) {
        const double *fe = f + (long long)e * n3;
        const int fp = (int)((reinterpret_cast<unsigned long long>(fe) >> 3) & 1);
        const int fcnt = (n3 + fp + 1) & ~1;
        if ((long long)e * n3 - fp + fcnt <= (long long)L.Ne * n3) prefetch_l2(fe - fp, fcnt * 8u);
      }
    }
    if (!tail_ok) stage(U, ue, n3);
    cp_async_wait_all();
    __syncthreads();
    mbar_wait(mbar, phase);
    __syncthreads();
    PMG_APH(0);
    for (int t = threadIdx.x; t < 3 * n2; t += blockDim.x) {
      const int d = t / n2, pp = t - d * n2;
      double *C = Cf + d * 4 * n2 + pp;
      const double mu = L.mu[d];
      const double tvR = C[0], tdR = C[n2], tvL = C[2 * n2], tdL = C[3 * n2];
      C[0] = -0.5 * tdR - mu * tvR;
      C[n2] = 0.5 * tvR;
      C[2 * n2] = 0.5 * tdL - mu * tvL;
#ifndef PMG_NO_APPLY_EO
      C[3 * n2] = NT == 17 ? 0.5 * tvL : -0.5 * tvL;     // even/odd passes take -c4
#else
      C[3 * n2] = -0.5 * tvL;
#endif
    }
    __syncthreads();
    const Blk B = {{n, n, n}, {1, n, n2}};
#ifndef PMG_NO_APPLY_EO
    if constexpr (NT == 17) {            // even/odd passes (the transform stored -c4)
      PMG_APH(1);
      apply_eo17<0, true>(U, Cf, V, af17, cmap, cmapY); __syncthreads();
      PMG_APH(2);
      apply_eo17<1, false>(U, Cf + 4 * n2, V, af17 + EO17_AF, cmap, cmapY); __syncthreads();
      apply_eo17<2, false>(U, Cf + 8 * n2, V, af17 + 2 * EO17_AF, cmap, cmapY); __syncthreads();
      PMG_APH(3);
    } else
#endif
    {
      EpiAcc acc{V, B, true};
      LineSpec lx = {n, n, L.Daug[0], n + 4, 1, Cf, 4, n2, 1, n};
      mma_lines_ct<0, n, n + 4>(U, B, lx, acc); __syncthreads();
      acc.first = false;
      LineSpec ly = {n, n, L.Daug[1], n + 4, 1, Cf + 4 * n2, 4, n2, 1, n};
      mma_lines_ct<1, n, n + 4>(U, B, ly, acc); __syncthreads();
      LineSpec lz = {n, n, L.Daug[2], n + 4, 1, Cf + 8 * n2, 4, n2, 1, n};
      mma_lines_ct<2, n, n + 4>(U, B, lz, acc); __syncthreads();
    }
    // out = f - M v (or M v), M = Mz (x) My (x) Mx; f loads batched for memory-level parallelism:
    // up to 10 f loads per thread in flight (the epilogue was a fifth of the kernel's time with 4)
    const long long g0 = (long long)e * n3;
    constexpr int THR = NT == 17 ? PMG_APPLY17_THREADS : ((NT <= 9 && !WIDE) ? 128 : 256);
#ifndef PMG_APPLY_UNR
    constexpr int UNR = NT == 17 ? (THR == 256 ? 10 : 8) : (n3 + THR - 1) / THR;   // n = 17: 20 spills (measured 10 best)
#else
    constexpr int UNR = PMG_APPLY_UNR;
#endif
    // node (i, j, k) of DOF t is tracked incrementally over the thread's DOFs t0 + q THR
    // (THR = SK n^2 + SJ n + SI): two compare-and-carry steps instead of a division per DOF
    constexpr int SI = THR % n, SJ = (THR / n) % n, SK = THR / n2;
    for (int t0 = threadIdx.x; t0 < n3; t0 += UNR * THR) {
      double fv[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const int t = t0 + q * THR;
        fv[q] = (f && t < n3) ? __ldg(f + g0 + t) : 0.0;
      }
      int i = t0 % n, j = (t0 / n) % n, k = t0 / n2;
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const int t = t0 + q * THR;
        if (t >= n3) break;
        if constexpr (NT != 17) {        // n <= 9: the per-DOF division measured faster (0.109 vs 0.120 ms)
          i = t % n; j = (t / n) % n; k = t / n2;
        }
        const double v = ms[i] * ms[n + j] * ms[2 * n + k] * V[t];
        const double rr = f ? fv[q] - v : v;
        if (restrict_I) V[t] = rr;
        else out[g0 + t] = rr;
        if constexpr (NT == 17) {
          i += SI; j += SJ; k += SK;
          if (i >= n) { i -= n; ++j; }
          if (j >= n) { j -= n; ++k; }
        }
      }
    }
    __syncthreads();
    PMG_APH(4);
    if (NT > 2 && restrict_I) {
      // fused residual restriction f_c = (I^T (x) I^T (x) I^T) r (Alg. 1 l.292): r stays in V;
      // x pass (n -> nc) into U, y pass into Cf, z pass straight to the coarse vector
      __syncthreads();
      constexpr int nc = NC;
      const Blk T1 = {{nc, n, n}, {1, nc, nc * n}};
      const Blk T2 = {{nc, nc, n}, {1, nc, nc * nc}};
      const Blk FC = {{nc, nc, nc}, {1, nc, nc * nc}};
      const LineSpec rx = {nc, n, restrict_I, 1, nc, nullptr, 0, 0, 0, 0};
      EpiStore s1{U, T1};
      mma_lines_ct<0, NC, n>(V, B, rx, s1); __syncthreads();
      EpiStore s2{Cf, T2};
      mma_lines_ct<1, NC, n>(U, T1, rx, s2); __syncthreads();
      EpiStore s3{fc + (long long)e * nc * nc * nc, FC};
      mma_lines_ct<2, NC, n>(Cf, T2, rx, s3);
    }
    __syncthreads();                   // U, V, Cf are reused by the next element
    PMG_APH(5);
  }
#ifdef PMG_PHASE_TIMING
  if (threadIdx.x == 0 && (blockIdx.x % 64) == 0)
    printf("APHASE apply<%d> blk %d restrict %d wait %lld coef %lld x %lld yz %lld epi %lld restr %lld\n", NT,
           blockIdx.x, restrict_I != nullptr, tacc[0], tacc[1], tacc[2], tacc[3], tacc[4], tacc[5]);
#endif
#undef PMG_APH
}

// Small elements (n = 3, 5: the two lowest smoothing levels of every configuration): EPB
// elements per 256-thread CTA, one thread per DOF, plain FP64 FMAs (Eq. 7 / Eq. 8, PAPER.md:
// 149-164, :192-200) and the fused residual restriction (Alg. 1 l.292) as three small passes in
// shared memory.  A 27- or 125-DOF element cannot feed a CTA of DMMA line GEMMs: the persistent
// k_apply_mma<3/5> spent ~5 us per element in ~10 block barriers (19-23 us per launch on c3's
// 4096 elements, 9 us on one-wave meshes); here every load of a thread is independent and issued
// up front, one barrier before the restriction passes.  Same operator tables (Daug rows
// pre-scaled by 1/M_d, face couplings as four extra columns) as the DMMA path.
template <int NT, int EPB>
__global__ void __launch_bounds__(256) k_apply_small(LevelDev L, const double *__restrict__ u,
                                                     const double *__restrict__ T,
                                                     const double *__restrict__ f,
                                                     double *__restrict__ out,
                                                     const double *__restrict__ restrict_I,
                                                     double *__restrict__ fc) {
  constexpr int n = NT, n2 = n * n, n3 = n2 * n, KA = n + 4, NC = (NT + 1) / 2;
  __shared__ double Us[EPB * n3];
  __shared__ double Da[3 * n * KA];
  __shared__ double ms[3 * n];
  __shared__ double Ic[n * NC];
  __shared__ double R1[EPB * NC * n2];
  __shared__ double R2[EPB * NC * NC * n];
  const int e0 = blockIdx.x * EPB;
  const int ne = min(EPB, L.Ne - e0);
  const int tid = threadIdx.x;
  for (int i = tid; i < ne * n3; i += blockDim.x) Us[i] = __ldg(u + (long long)e0 * n3 + i);
  for (int i = tid; i < 3 * n * KA; i += blockDim.x) Da[i] = L.Daug[i / (n * KA)][i % (n * KA)];
  for (int i = tid; i < 3 * n; i += blockDim.x) ms[i] = L.mass[i / n][i % n];
  if (restrict_I)
    for (int i = tid; i < n * NC; i += blockDim.x) Ic[i] = restrict_I[i];
  const int le = tid / n3, t = tid - le * n3;
  const bool act = le < ne;
  const int e = e0 + (act ? le : 0);
  const int i0 = t % n, j0 = (t / n) % n, k0 = t / n2;
  // neighbour traces of the three lines through this DOF (L2 / L1 hits), issued before the barrier
  double c[3][4];
  {
    const int ec[3] = {e % L.nx, (e / L.nx) % L.ny, e / (L.nx * L.ny)};
    const int edim[3] = {L.nx, L.ny, L.nz};
    const int pface[3] = {j0 + n * k0, i0 + n * k0, i0 + n * j0};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      int cc[3] = {ec[0], ec[1], ec[2]};
      cc[d] = wrap(ec[d] + 1, edim[d]);
      const long long nbR = cc[0] + L.nx * (cc[1] + (long long)L.ny * cc[2]);
      cc[d] = wrap(ec[d] - 1, edim[d]);
      const long long nbL = cc[0] + L.nx * (cc[1] + (long long)L.ny * cc[2]);
      const double *TR = T + (nbR * 3 + d) * 4 * n2 + pface[d];
      const double *TL = T + (nbL * 3 + d) * 4 * n2 + pface[d];
      const double tvR = act ? __ldg(TR) : 0.0, tdR = act ? __ldg(TR + n2) : 0.0;
      const double tvL = act ? __ldg(TL + 2 * n2) : 0.0, tdL = act ? __ldg(TL + 3 * n2) : 0.0;
      const double mu = L.mu[d];
      c[d][0] = -0.5 * tdR - mu * tvR;
      c[d][1] = 0.5 * tvR;
      c[d][2] = 0.5 * tdL - mu * tvL;
      c[d][3] = -0.5 * tvL;
    }
  }
  const long long g = (long long)e * n3 + t;
  const double fv = (act && f) ? __ldg(f + g) : 0.0;
  __syncthreads();
  double r = 0.0;
  if (act) {
    const int idx[3] = {i0, j0, k0};
    const int stride[3] = {1, n, n2};
    double v = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double *Dr = Da + d * n * KA + idx[d] * KA;
      const double *line = Us + le * n3 + (t - idx[d] * stride[d]);
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < n; ++m) acc = fma(Dr[m], line[m * stride[d]], acc);
#pragma unroll
      for (int q = 0; q < 4; ++q) acc = fma(Dr[n + q], c[d][q], acc);
      v += acc;
    }
    const double mv = ms[i0] * ms[n + j0] * ms[2 * n + k0] * v;
    r = f ? fv - mv : mv;
    if (!restrict_I) out[g] = r;
  }
  if (!restrict_I) return;
  // fused residual restriction f_c = (I^T (x) I^T (x) I^T) r: r replaces u in shared memory
  __syncthreads();
  if (act) Us[le * n3 + t] = r;
  __syncthreads();
  for (int w = tid; w < ne * NC * n2; w += blockDim.x) {          // x: n -> NC
    const int lb = w / (NC * n2), q = w - lb * NC * n2;
    const int o = q % NC, jk = q / NC;
    const double *row = Us + lb * n3 + n * jk;
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < n; ++m) acc = fma(Ic[m * NC + o], row[m], acc);
    R1[w] = acc;
  }
  __syncthreads();
  for (int w = tid; w < ne * NC * NC * n; w += blockDim.x) {      // y: n -> NC
    const int lb = w / (NC * NC * n), q = w - lb * NC * NC * n;
    const int o1 = q % NC, o2 = (q / NC) % NC, k = q / (NC * NC);
    const double *col = R1 + lb * NC * n2 + o1 + NC * n * k;
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < n; ++m) acc = fma(Ic[m * NC + o2], col[NC * m], acc);
    R2[w] = acc;
  }
  __syncthreads();
  for (int w = tid; w < ne * NC * NC * NC; w += blockDim.x) {     // z: n -> NC, to the coarse vector
    const int lb = w / (NC * NC * NC), q = w - lb * NC * NC * NC;
    const int o12 = q % (NC * NC), o3 = q / (NC * NC);
    const double *col = R2 + lb * NC * NC * n + o12;
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < n; ++m) acc = fma(Ic[m * NC + o3], col[NC * NC * m], acc);
    fc[(long long)(e0 + lb) * NC * NC * NC + q] = acc;
  }
}

// Face traces with the element staged in shared memory (coalesced loads).
__global__ void __launch_bounds__(256) k_traces_sm(LevelDev L, const double *__restrict__ u,
                                                   double *__restrict__ T) {
  extern __shared__ double sm[];
  const int n = L.n, n2 = n * n, n3 = n2 * n;
  double *Us = sm, *tab = sm + ((n3 + 3) & ~1);
  unsigned long long *mbar = reinterpret_cast<unsigned long long *>(tab + 3 * trace_tab_len(n) + 2);
  // elements are walked backwards: the fold's last writes of u are still in L2, and the traces of
  // the FIRST elements are written last, where the following apply starts (apply@l4 0.602 -> 0.591)
#ifdef PMG_TRACES_FORWARD
  const int e = blockIdx.x;
#else
  const int e = gridDim.x - 1 - blockIdx.x;
#endif
  const BulkPlan bp = bulk_plan(Us, u + (long long)e * n3, n3, u + (long long)L.Ne * n3);
  double *U = bp.ptr;
  if (bp.bytes) {
    if (threadIdx.x == 0) {
      mbar_init(mbar, 1);
      mbar_expect_tx(mbar, bp.bytes);
      bulk_g2s(Us, bp.src, bp.bytes, mbar);
    }
  } else {
    stage(U, u + (long long)e * n3, n3);
  }
  stage_trace_tab(L, tab);
  cp_async_wait_all();
  __syncthreads();
  if (bp.bytes) mbar_wait(mbar, 0);
  double *Te = T + (long long)e * 12 * n2;
  if (n == 17) elem_traces<17>(U, tab, n, Te);
  else if (n == 9) elem_traces<9>(U, tab, n, Te);
  else elem_traces<0>(U, tab, n, Te);
}

}  // namespace

// ---------------------------------------------------------------------------------------------
cudaError_t launch_traces(const LevelDev &L, const double *u, double *T, cudaStream_t s) {
  const int n = L.n;
  const size_t sb = sizeof(double) * ((size_t)n * n * n + 4 + 3 * trace_tab_len(n) + 2 + 2);
  if (n <= 20) {
    static size_t configured = 0;
    if (sb > 48 * 1024 && sb > configured) {
      cudaFuncSetAttribute(k_traces_sm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
      configured = sb;
    }
    k_traces_sm<<<L.Ne, 256, sb, s>>>(L, u, T);
  } else {
    const int chunks = (3 * n * n + 127) / 128;
    k_traces<<<dim3(L.Ne, chunks), 128, 0, s>>>(L, u, T);
  }
  return cudaGetLastError();
}
static void configure_smem() {
  static bool done = false;
  if (done) return;
  done = true;
  const int mx = 227 * 1024;
  cudaFuncSetAttribute(k_apply_mma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_apply_mma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_apply_mma<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_apply_mma<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_apply_mma<17>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
}

static size_t apply_pipe_smem(int n) {
  const size_t n2 = (size_t)n * n, n3 = n2 * n;
  return sizeof(double) * (3 * n3 + 24 * n2 + 3 * n);
}

// PMG_FORCE_DFMA (diagnostic A/B build, scripts/gpu_dfma_ab.sh): levels with n <= 9 use the scalar
// FP64-FMA kernels (k_apply, k_fdm) instead of the DMMA line GEMMs.
bool apply_pipe_ok(const LevelDev &L) {
#ifdef PMG_FORCE_DFMA
  if (L.n <= 9) return false;
#endif
  return L.n == 3 || L.n == 5 || L.n == 9 || L.n == 17;
}

static size_t apply_mma_smem(int n) {
  const size_t n2 = (size_t)n * n, n3 = n2 * n;
  return sizeof(double) * (2 * n3 + 2 + 12 * n2 + 3 * n + 2) + 4 * ((PMG_COLMAP17_LEN + 3) & ~3) +
         (n == 17 ? sizeof(double) * 3 * EO17_AF : 0);
}

template <int NT, bool WIDE>
static int apply_grid(size_t sb, long long Ne) {
  static int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_apply_mma<NT, WIDE>,
                                                  NT == 17 ? PMG_APPLY17_THREADS : ((NT <= 9 && !WIDE) ? 128 : 256), sb);
    occ = std::max(occ, 1);
  }
  return (int)std::min<long long>(Ne, (long long)occ * num_sms());
}

template <int NT>
static void launch_apply_nt(const LevelDev &L, const double *u, const double *T, const double *f,
                            double *out, const double *I, double *fc, cudaStream_t s) {
  // persistent grid: as many CTAs as fit on the device at once (occupancy x SMs), capped at Ne;
  // a mesh that fits in one wave of 4 CTAs per SM gets 256-thread CTAs (latency-bound regime)
  const size_t sb = apply_mma_smem(NT);
#ifndef PMG_NO_APPLY_SMALL
  if constexpr (NT == 3 || NT == 5) {       // several elements per CTA, thread per DOF
    constexpr int EPB = NT == 3 ? 9 : 2;
    k_apply_small<NT, EPB><<<(int)((L.Ne + EPB - 1) / EPB), 256, 0, s>>>(L, u, T, f, out, I, fc);
    return;
  }
#endif
  if (NT <= 9 && L.Ne <= 4LL * num_sms()) {
    static bool cfg = false;
    if (!cfg) {
      cfg = true;
      cudaFuncSetAttribute(k_apply_mma<NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    }
    k_apply_mma<NT, true><<<apply_grid<NT, true>(sb, L.Ne), 256, sb, s>>>(L, u, T, f, out, I, fc);
    return;
  }
  const int threads = NT == 17 ? PMG_APPLY17_THREADS : (NT <= 9 ? 128 : 256);
  k_apply_mma<NT, false><<<apply_grid<NT, false>(sb, L.Ne), threads, sb, s>>>(L, u, T, f, out, I, fc);
}

bool apply_nt_ok(int n) { return n == 2 || n == 3 || n == 5 || n == 9 || n == 17; }

cudaError_t launch_apply_pipe(const LevelDev &L, const double *u, const double *T, const double *f,
                              double *out, const double *I, int nc, double *fc, cudaStream_t s) {
  configure_smem();
  if (I && nc != (L.n + 1) / 2) return cudaErrorInvalidValue;
  switch (L.n) {
    case 2: launch_apply_nt<2>(L, u, T, f, out, nullptr, nullptr, s); break;
    case 3: launch_apply_nt<3>(L, u, T, f, out, I, fc, s); break;
    case 5: launch_apply_nt<5>(L, u, T, f, out, I, fc, s); break;
    case 9: launch_apply_nt<9>(L, u, T, f, out, I, fc, s); break;
    case 17: launch_apply_nt<17>(L, u, T, f, out, I, fc, s); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_apply(const LevelDev &L, const double *u, const double *T, const double *f,
                         double *out, cudaStream_t s) {
  const int n = L.n;

#ifdef PMG_FORCE_DFMA
  if (n <= 9) {
    k_apply<<<L.Ne, 256, 0, s>>>(L, u, T, f, out);
    return cudaGetLastError();
  }
#endif
  if (n <= 17) {
    return launch_apply_pipe(L, u, T, f, out, nullptr, 0, nullptr, s);
  } else {
    k_apply<<<L.Ne, 256, 0, s>>>(L, u, T, f, out);
  }
  return cudaGetLastError();
}
}  // namespace pmg
