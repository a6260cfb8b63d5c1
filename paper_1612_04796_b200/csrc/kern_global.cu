// Global-memory (L2-resident) batched line GEMMs for P = 32 blocks.
// arXiv:1612.04796; PAPER.md line numbers cited per kernel.
#include <algorithm>

#include "kcommon.cuh"

namespace pmg {
namespace {

// ---------------------------------------------------------------------------------------------
// Global-memory (L2-resident) batched line GEMMs for blocks too large for shared memory
// (P = 32: 33^3 elements, 45^3 Schwarz windows).  Every warp grabs (block, 8-column tile,
// M-group) work items across the whole GPU, so even 64 subdomains fill all 148 SMs.  A stays in
// registers per M-group (MTG m-tiles), B fragments come from global memory (L2 hits: c4's
// window buffers are 47 MB), results go through global epilogue policies.
struct GEpiStore {
  double *Y; long long bs; Blk B;
  template <int DIR> __device__ __forceinline__ double col(long long, int, int) const { return 0.0; }
  template <int DIR> __device__ __forceinline__ void put(long long blk, int o, int p, int q, double,
                                                         double v) const {
    Y[blk * bs + blk_index<DIR>(B, o, p, q)] = v;
  }
};
struct GEpiDivide {
  double *Y; long long bs; Blk B; const double *lam[3];
  template <int DIR> __device__ __forceinline__ double col(long long, int p, int q) const {
    return lam[Other<DIR>::P][p] + lam[Other<DIR>::Q][q];
  }
  template <int DIR> __device__ __forceinline__ void put(long long blk, int o, int p, int q, double cf,
                                                         double v) const {
    Y[blk * bs + blk_index<DIR>(B, o, p, q)] = v * rcp_nr(cf + lam[DIR][o]);
  }
};
struct GEpiWeight {
  double *Y; long long bs; Blk B; const double *W[3];
  template <int DIR> __device__ __forceinline__ double col(long long, int p, int q) const {
    return W[Other<DIR>::P][p] * W[Other<DIR>::Q][q];
  }
  template <int DIR> __device__ __forceinline__ void put(long long blk, int o, int p, int q, double cf,
                                                         double v) const {
    Y[blk * bs + blk_index<DIR>(B, o, p, q)] = v * (cf * W[DIR][o]);
  }
};
struct GEpiAcc {
  double *Y; long long bs; Blk B; int first;
  template <int DIR> __device__ __forceinline__ double col(long long, int, int) const { return 0.0; }
  template <int DIR> __device__ __forceinline__ void put(long long blk, int o, int p, int q, double,
                                                         double v) const {
    double *y = Y + blk * bs + blk_index<DIR>(B, o, p, q);
    *y = first ? v : *y + v;
  }
};

template <int DIR, int KS, int MTG, class Epi>
__global__ void __launch_bounds__(256, 2) k_lines_global(const double *__restrict__ X, long long xbs,
                                                      Blk B, LineSpec ls, long long ebs,
                                                      int nblocks, Epi epi) {
  constexpr int PD = Other<DIR>::P, QD = Other<DIR>::Q;
  const int mo = ls.mo, mk = ls.mk, kt = ls.mk + ls.next;
  const int mp = B.m[PD], mq = B.m[QD];
  const int ncol = mp * mq;
  const unsigned magic = 0xFFFFFFFFu / (unsigned)mp + 1u;
  const int so = B.s[DIR], sp = B.s[PD], sq = B.s[QD];
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ntiles = (ncol + 7) >> 3;
  const int ngroups = (mo + 8 * MTG - 1) / (8 * MTG);
  const long long nitems = (long long)nblocks * ntiles * ngroups;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  int koff[KS];
  bool kext[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = min(ks * 4 + t, kt - 1);
    kext[ks] = k >= mk;
    koff[ks] = kext[ks] ? (k - mk) * ls.esr : k * so;
  }
  int cur_group = -1;
  double a[MTG][KS];
  for (long long it = wid; it < nitems; it += nwarps) {
    const int grp = (int)(it % ngroups);
    const long long rest = it / ngroups;
    const int tile = (int)(rest % ntiles);
    const long long blk = rest / ntiles;
    if (grp != cur_group) {
      cur_group = grp;
#pragma unroll
      for (int mt = 0; mt < MTG; ++mt)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int o = (grp * MTG + mt) * 8 + g, k = ks * 4 + t;
          a[mt][ks] = (o < mo && k < kt) ? __ldg(ls.Amat + o * ls.ao + k * ls.ak) : 0.0;
        }
    }
    const int nb = min(tile * 8 + g, ncol - 1);
    const int qb = __umulhi((unsigned)nb, magic), pb = nb - qb * mp;
    const double *xb = X + blk * xbs + pb * sp + qb * sq;
    const double *eb = ls.Ext ? ls.Ext + blk * ebs + pb * ls.esp + qb * ls.esq : X;
    double b[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) b[ks] = __ldg((kext[ks] ? eb : xb) + koff[ks]);
    double c[MTG][2];
#pragma unroll
    for (int mt = 0; mt < MTG; ++mt) { c[mt][0] = 0.0; c[mt][1] = 0.0; }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int mt = 0; mt < MTG; ++mt) dmma884(c[mt][0], c[mt][1], a[mt][ks], b[ks]);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int n = tile * 8 + 2 * t + j;
      if (n >= ncol) continue;
      const int q = __umulhi((unsigned)n, magic), p = n - q * mp;
      const double cf = epi.template col<DIR>(blk, p, q);
#pragma unroll
      for (int mt = 0; mt < MTG; ++mt) {
        const int o = (grp * MTG + mt) * 8 + g;
        if (o < mo) epi.template put<DIR>(blk, o, p, q, cf, c[mt][j]);
      }
    }
  }
}

// Even/odd variant for the fast-diagonalisation passes of odd windows (m = 2H+1, exact-parity
// eigenvectors with even modes first; see k_fdm_eo in kern_fdm.cu): per (block, 8-column tile)
// work item 2 x MT x KS DMMAs (m = 45: 36) instead of ceil(m/8) x ceil(m/4) (m = 45: 72).
// Forward: b_E = x_k + x_{m-1-k}, b_O = x_k - x_{m-1-k}, k clamped to H, middle column of S_E^T
// halved; backward: b_E = t_E[min(k,H)], b_O = t_O[min(k,H-1)]; x_a = P_a + Q_a, x_{m-1-a} = P_a - Q_a.
template <int DIR, int MT, int KS, bool FWD, class Epi>
__global__ void __launch_bounds__(256, 2) k_lines_global_eo(const double *__restrict__ X, long long xbs,
                                                         Blk B, const double *__restrict__ S,
                                                         int nblocks, Epi epi) {
  constexpr int PD = Other<DIR>::P, QD = Other<DIR>::Q;
  const int m = B.m[DIR], H = m >> 1;
  const int mp = B.m[PD], mq = B.m[QD];
  const int ncol = mp * mq;
  const unsigned magic = 0xFFFFFFFFu / (unsigned)mp + 1u;
  const int so = B.s[DIR], sp = B.s[PD], sq = B.s[QD];
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ntiles = (ncol + 7) >> 3;
  const long long nitems = (long long)nblocks * ntiles;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  double aE[MT][KS], aO[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int o = mt * 8 + g, k = ks * 4 + t;
      if (FWD) {
        aE[mt][ks] = (o <= H && k <= H) ? __ldg(S + k * m + o) * (k == H ? 0.5 : 1.0) : 0.0;
        aO[mt][ks] = (o < H && k < H) ? __ldg(S + k * m + H + 1 + o) : 0.0;
      } else {
        aE[mt][ks] = (o <= H && k <= H) ? __ldg(S + o * m + k) : 0.0;
        aO[mt][ks] = (o < H && k < H) ? __ldg(S + o * m + H + 1 + k) : 0.0;
      }
    }
  int off1[KS], off2[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = ks * 4 + t, kl = min(k, H);
    if (FWD) { off1[ks] = kl * so; off2[ks] = (m - 1 - kl) * so; }
    else { off1[ks] = kl * so; off2[ks] = (H + 1 + min(k, H - 1)) * so; }
  }
  for (long long it = wid; it < nitems; it += nwarps) {
    const int tile = (int)(it % ntiles);
    const long long blk = it / ntiles;
    const int nb = min(tile * 8 + g, ncol - 1);
    const int qb = __umulhi((unsigned)nb, magic), pb = nb - qb * mp;
    const double *xb = X + blk * xbs + pb * sp + qb * sq;
    double bE[KS], bO[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const double v1 = __ldg(xb + off1[ks]), v2 = __ldg(xb + off2[ks]);
      if (FWD) { bE[ks] = v1 + v2; bO[ks] = v1 - v2; }
      else { bE[ks] = v1; bO[ks] = v2; }
    }
    double cE[MT][2], cO[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) { cE[mt][0] = cE[mt][1] = cO[mt][0] = cO[mt][1] = 0.0; }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        dmma884(cE[mt][0], cE[mt][1], aE[mt][ks], bE[ks]);
        dmma884(cO[mt][0], cO[mt][1], aO[mt][ks], bO[ks]);
      }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int n = tile * 8 + 2 * t + j;
      if (n >= ncol) continue;
      const int q = __umulhi((unsigned)n, magic), p = n - q * mp;
      const double cf = epi.template col<DIR>(blk, p, q);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int o = mt * 8 + g;
        if (FWD) {
          if (o <= H) epi.template put<DIR>(blk, o, p, q, cf, cE[mt][j]);
          if (o < H) epi.template put<DIR>(blk, H + 1 + o, p, q, cf, cO[mt][j]);
        } else if (o < H) {
          epi.template put<DIR>(blk, o, p, q, cf, cE[mt][j] + cO[mt][j]);
          epi.template put<DIR>(blk, m - 1 - o, p, q, cf, cE[mt][j] - cO[mt][j]);
        } else if (o == H) {
          epi.template put<DIR>(blk, o, p, q, cf, cE[mt][j]);
        }
      }
    }
  }
}

template <int DIR, bool FWD, class Epi>
cudaError_t lines_global_eo(const double *X, long long xbs, const Blk &B, const double *S,
                            int nblocks, const Epi &epi, cudaStream_t s) {
  k_lines_global_eo<DIR, 3, 6, FWD, Epi><<<148 * 2, 256, 0, s>>>(X, xbs, B, S, nblocks, epi);
  return cudaGetLastError();
}

template <int DIR, class Epi>
cudaError_t lines_global(const double *X, long long xbs, const Blk &B, const LineSpec &ls,
                         long long ebs, int nblocks, const Epi &epi, cudaStream_t s) {
  const int KS = (ls.mk + ls.next + 3) >> 2;
  const int grid = 148 * 8;
  if (KS <= 6) k_lines_global<DIR, 6, 3, Epi><<<grid, 256, 0, s>>>(X, xbs, B, ls, ebs, nblocks, epi);
  else if (KS <= 12) k_lines_global<DIR, 12, 3, Epi><<<grid, 256, 0, s>>>(X, xbs, B, ls, ebs, nblocks, epi);
  else if (KS <= 20) k_lines_global<DIR, 20, 1, Epi><<<grid, 256, 0, s>>>(X, xbs, B, ls, ebs, nblocks, epi);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

// window gather to global memory: X[s*Mw + w] = r(window node w of subdomain s)
__global__ void k_gather_win(LevelDev L, const double *__restrict__ r, double *__restrict__ X) {
  const int n = L.n, n3 = n * n * n;
  const int mx = L.m[0], my = L.m[1];
  const long long total = (long long)L.Ne * L.Mw;
  for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < total;
       gi += (long long)gridDim.x * blockDim.x) {
    const long long sidx = gi / L.Mw;
    const int w = (int)(gi - sidx * L.Mw);
    const int win[3] = {w % mx, (w / mx) % my, w / (mx * my)};
    const int ec[3] = {(int)(sidx % L.nx), (int)((sidx / L.nx) % L.ny), (int)(sidx / ((long long)L.nx * L.ny))};
    const int edim[3] = {L.nx, L.ny, L.nz};
    long long addr = 0;
    const long long estride[3] = {(long long)n3, (long long)L.nx * n3, (long long)L.nx * L.ny * n3};
    const int lstride[3] = {1, n, n * n};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int no = L.no[d], a = win[d];
      const int o = a < no ? -1 : (a < no + n ? 0 : 1);
      const int li = a < no ? n - no + a : (a < no + n ? a - no : a - no - n);
      addr += wrap(ec[d] + o, edim[d]) * estride[d] + li * lstride[d];
    }
    X[gi] = __ldg(r + addr);
  }
}

// face-coefficient buffer for the global apply: Cb[e][d][4][n^2] from the neighbours' traces
__global__ void k_face_coef(LevelDev L, const double *__restrict__ T, double *__restrict__ Cb) {
  const int n = L.n, n2 = n * n;
  const long long total = (long long)L.Ne * 3 * n2;
  for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < total;
       gi += (long long)gridDim.x * blockDim.x) {
    const long long e = gi / (3 * n2);
    const int r = (int)(gi - e * 3 * n2), d = r / n2, pp = r - d * n2;
    const int ec[3] = {(int)(e % L.nx), (int)((e / L.nx) % L.ny), (int)(e / ((long long)L.nx * L.ny))};
    const int edim[3] = {L.nx, L.ny, L.nz};
    int cR[3] = {ec[0], ec[1], ec[2]}, cL[3] = {ec[0], ec[1], ec[2]};
    cR[d] = wrap(ec[d] + 1, edim[d]);
    cL[d] = wrap(ec[d] - 1, edim[d]);
    const double *TR = T + ((long long)(cR[0] + L.nx * (cR[1] + L.ny * cR[2])) * 3 + d) * 4 * n2;
    const double *TL = T + ((long long)(cL[0] + L.nx * (cL[1] + L.ny * cL[2])) * 3 + d) * 4 * n2;
    const double tvR = TR[pp], tdR = TR[n2 + pp], tvL = TL[2 * n2 + pp], tdL = TL[3 * n2 + pp];
    const double mu = L.mu[d];
    double *C = Cb + (e * 3 + d) * 4 * n2 + pp;
    C[0] = -0.5 * tdR - mu * tvR;
    C[n2] = 0.5 * tvR;
    C[2 * n2] = 0.5 * tdL - mu * tvL;
    C[3 * n2] = -0.5 * tvL;
  }
}

// out = f - M V  (or M V), elementwise over the level
__global__ void k_mass_finish(LevelDev L, const double *__restrict__ V, const double *__restrict__ f,
                              double *__restrict__ out) {
  const int n = L.n, n3 = n * n * n;
  const long long total = (long long)L.Ne * n3;
  for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < total;
       gi += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(gi % n3);
    const int i = t % n, j = (t / n) % n, k = t / (n * n);
    const double v = L.mass[0][i] * L.mass[1][j] * L.mass[2][k] * V[gi];
    out[gi] = f ? f[gi] - v : v;
  }
}

}  // namespace

cudaError_t launch_fdm_global(const LevelDev &L, const double *r, double *X, double *Y, double *Z,
                              cudaStream_t s) {
  const long long bs = L.Mw;
  const Blk B = {{L.m[0], L.m[1], L.m[2]}, {1, L.m[0], L.m[0] * L.m[1]}};
  const long long total = (long long)L.Ne * L.Mw;
  k_gather_win<<<grid_for(total, 256), 256, 0, s>>>(L, r, X);
  const int *m = L.m;
  bool eo = true;                         // odd windows with H <= 23 (MT 3, KS 6 tiles)
  for (int d = 0; d < 3; ++d) eo = eo && (m[d] & 1) && m[d] / 2 >= 16 && m[d] / 2 <= 23;
#ifdef PMG_NO_EO
  eo = false;
#endif
  if (eo) {
    cudaError_t e;
    if ((e = lines_global_eo<0, true>(X, bs, B, L.S[0], L.Ne, GEpiStore{Y, bs, B}, s))) return e;
    if ((e = lines_global_eo<1, true>(Y, bs, B, L.S[1], L.Ne, GEpiStore{X, bs, B}, s))) return e;
    if ((e = lines_global_eo<2, true>(X, bs, B, L.S[2], L.Ne, GEpiDivide{Y, bs, B, {L.lam[0], L.lam[1], L.lam[2]}}, s))) return e;
    if ((e = lines_global_eo<2, false>(Y, bs, B, L.S[2], L.Ne, GEpiStore{X, bs, B}, s))) return e;
    if ((e = lines_global_eo<1, false>(X, bs, B, L.S[1], L.Ne, GEpiStore{Y, bs, B}, s))) return e;
    return lines_global_eo<0, false>(Y, bs, B, L.S[0], L.Ne, GEpiWeight{Z, bs, B, {L.W[0], L.W[1], L.W[2]}}, s);
  }
  auto fw = [&](int d) { return LineSpec{m[d], m[d], L.S[d], 1, m[d], nullptr, 0, 0, 0, 0}; };
  auto bw = [&](int d) { return LineSpec{m[d], m[d], L.S[d], m[d], 1, nullptr, 0, 0, 0, 0}; };
  cudaError_t e;
  if ((e = lines_global<0>(X, bs, B, fw(0), 0, L.Ne, GEpiStore{Y, bs, B}, s))) return e;
  if ((e = lines_global<1>(Y, bs, B, fw(1), 0, L.Ne, GEpiStore{X, bs, B}, s))) return e;
  if ((e = lines_global<2>(X, bs, B, fw(2), 0, L.Ne, GEpiDivide{Y, bs, B, {L.lam[0], L.lam[1], L.lam[2]}}, s))) return e;
  if ((e = lines_global<2>(Y, bs, B, bw(2), 0, L.Ne, GEpiStore{X, bs, B}, s))) return e;
  if ((e = lines_global<1>(X, bs, B, bw(1), 0, L.Ne, GEpiStore{Y, bs, B}, s))) return e;
  return lines_global<0>(Y, bs, B, bw(0), 0, L.Ne, GEpiWeight{Z, bs, B, {L.W[0], L.W[1], L.W[2]}}, s);
}

cudaError_t launch_apply_global(const LevelDev &L, const double *u, const double *T, const double *f,
                                double *out, double *Cb, double *V, cudaStream_t s) {
  const int n = L.n, n2 = n * n;
  const long long bs = (long long)n2 * n;
  const Blk B = {{n, n, n}, {1, n, n2}};
  k_face_coef<<<grid_for((long long)L.Ne * 3 * n2, 256), 256, 0, s>>>(L, T, Cb);
  cudaError_t e;
  for (int d = 0; d < 3; ++d) {
    const LineSpec ls = {n, n, L.Daug[d], n + 4, 1, Cb + d * 4 * n2, 4, n2, 1, n};
    const GEpiAcc acc{V, bs, B, d == 0 ? 1 : 0};
    if (d == 0) e = lines_global<0>(u, bs, B, ls, 12LL * n2, L.Ne, acc, s);
    else if (d == 1) e = lines_global<1>(u, bs, B, ls, 12LL * n2, L.Ne, acc, s);
    else e = lines_global<2>(u, bs, B, ls, 12LL * n2, L.Ne, acc, s);
    if (e) return e;
  }
  k_mass_finish<<<grid_for((long long)L.Ne * bs, 256), 256, 0, s>>>(L, V, f, out);
  return cudaGetLastError();
}

// p-transfers for n_f > 17 (P = 32 level of c4: 33^3 fine, 17^3 coarse elements) as three
// batched global line GEMMs each (Alg. 1 l.292 / l.299), spread over the whole GPU
// instead of one CTA per element.  X1, X2: scratch of Ne * nf * nf * nc doubles each.
cudaError_t launch_restrict_global(const LevelDev &Lf, int nc, const double *I, const double *rf,
                                   double *fc, double *X1, double *X2, cudaStream_t s) {
  const int nf = Lf.n;
  const Blk B0 = {{nf, nf, nf}, {1, nf, nf * nf}};
  const Blk B1 = {{nc, nf, nf}, {1, nc, nc * nf}};
  const Blk B2 = {{nc, nc, nf}, {1, nc, nc * nc}};
  const Blk B3 = {{nc, nc, nc}, {1, nc, nc * nc}};
  const LineSpec rs = {nc, nf, I, 1, nc, nullptr, 0, 0, 0, 0};     // A[c][i] = I[i][c]
  const long long b0 = (long long)nf * nf * nf, b1 = (long long)nc * nf * nf, b2 = (long long)nc * nc * nf,
                  b3 = (long long)nc * nc * nc;
  cudaError_t e;
  if ((e = lines_global<0>(rf, b0, B0, rs, 0, Lf.Ne, GEpiStore{X1, b1, B1}, s))) return e;
  if ((e = lines_global<1>(X1, b1, B1, rs, 0, Lf.Ne, GEpiStore{X2, b2, B2}, s))) return e;
  return lines_global<2>(X2, b2, B2, rs, 0, Lf.Ne, GEpiStore{fc, b3, B3}, s);
}

// S (optional, Ne * nf^3 doubles): the last pass stores I u_c there and a vector update adds it to
// u_f — the accumulating line GEMM waits on a cold read of u_f in every tile (c4: 42.6 us against
// 13.7 us for the same pass with plain stores + ~9 us for the update)
cudaError_t launch_prolong_global(const LevelDev &Lf, int nc, const double *I, const double *uc,
                                  double *uf, double *X1, double *X2, cudaStream_t s, double *S) {
  const int nf = Lf.n;
  const Blk B0 = {{nc, nc, nc}, {1, nc, nc * nc}};
  const Blk B1 = {{nf, nc, nc}, {1, nf, nf * nc}};
  const Blk B2 = {{nf, nf, nc}, {1, nf, nf * nf}};
  const Blk B3 = {{nf, nf, nf}, {1, nf, nf * nf}};
  const LineSpec ps = {nf, nc, I, nc, 1, nullptr, 0, 0, 0, 0};     // A[i][c] = I[i][c]
  const long long b0 = (long long)nc * nc * nc, b1 = (long long)nf * nc * nc, b2 = (long long)nf * nf * nc,
                  b3 = (long long)nf * nf * nf;
  cudaError_t e;
  if ((e = lines_global<0>(uc, b0, B0, ps, 0, Lf.Ne, GEpiStore{X1, b1, B1}, s))) return e;
  if ((e = lines_global<1>(X1, b1, B1, ps, 0, Lf.Ne, GEpiStore{X2, b2, B2}, s))) return e;
  if (S) {
    if ((e = lines_global<2>(X2, b2, B2, ps, 0, Lf.Ne, GEpiStore{S, b3, B3}, s))) return e;
    return launch_axpby(uf, 1.0, S, 1.0, (long long)Lf.Ne * b3, s);                 // u_f += I u_c
  }
  return lines_global<2>(X2, b2, B2, ps, 0, Lf.Ne, GEpiAcc{uf, b3, B3, 0}, s);     // u_f +=
}

}  // namespace pmg
