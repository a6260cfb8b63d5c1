// Schwarz subdomain solves by fast diagonalisation (shared-memory DMMA path, legacy FFMA path).
// arXiv:1612.04796; PAPER.md line numbers cited per kernel.
#include <algorithm>

#include "kcommon.cuh"

namespace pmg {
namespace {


// Weighted-Schwarz subdomain solve by fast diagonalisation (Eqs. 9-10):
// gather the element-centred window of r, apply S_x^T, S_y^T, S_z^T, divide by
// lam_x + lam_y + lam_z, apply S_z, S_y, S_x, multiply by W = W_z (x) W_y (x) W_x.
// One CTA per subdomain; result window stored in Z[s*Mw + ...].
__global__ void k_fdm(LevelDev L, const double *__restrict__ r, double *__restrict__ Z,
                      double *__restrict__ scr, int use_smem) {
  extern __shared__ double sm[];
  const int n = L.n, n3 = n * n * n;
  const int mx = L.m[0], my = L.m[1], mz = L.m[2], Mw = L.Mw;
  const int e = blockIdx.x;
  const int ex = e % L.nx, ey = (e / L.nx) % L.ny, ez = e / (L.nx * L.ny);
  double *X, *Y;
  if (use_smem) { X = sm; Y = sm + Mw; }
  else { X = scr + (long long)e * Mw; Y = Z + (long long)e * Mw; }
  // gather
  for (int w = threadIdx.x; w < Mw; w += blockDim.x) {
    const int a = w % mx, b = (w / mx) % my, c = w / (mx * my);
    const int win[3] = {a, b, c};
    const int ec[3] = {ex, ey, ez};
    const int edim[3] = {L.nx, L.ny, L.nz};
    int el[3], loc[3];
    for (int d = 0; d < 3; ++d) {
      const int no = L.no[d];
      int o, li;
      if (win[d] < no) { o = -1; li = n - no + win[d]; }
      else if (win[d] < no + n) { o = 0; li = win[d] - no; }
      else { o = 1; li = win[d] - no - n; }
      el[d] = wrap(ec[d] + o, edim[d]);
      loc[d] = li;
    }
    const long long g = (long long)(el[0] + L.nx * (el[1] + L.ny * el[2])) * n3 + loc[0]
                      + n * (loc[1] + n * loc[2]);
    X[w] = __ldg(r + g);
  }
  __syncthreads();
  contract_axis(X, Y, mx, my, mz, 0, L.S[0], 1, mx, mx); __syncthreads();
  contract_axis(Y, X, mx, my, mz, 1, L.S[1], 1, my, my); __syncthreads();
  contract_axis(X, Y, mx, my, mz, 2, L.S[2], 1, mz, mz); __syncthreads();
  for (int w = threadIdx.x; w < Mw; w += blockDim.x) {
    const int a = w % mx, b = (w / mx) % my, c = w / (mx * my);
    Y[w] = Y[w] / (L.lam[0][a] + L.lam[1][b] + L.lam[2][c]);
  }
  __syncthreads();
  contract_axis(Y, X, mx, my, mz, 2, L.S[2], mz, 1, mz); __syncthreads();
  contract_axis(X, Y, mx, my, mz, 1, L.S[1], my, 1, my); __syncthreads();
  contract_axis(Y, X, mx, my, mz, 0, L.S[0], mx, 1, mx); __syncthreads();
  double *Ze = Z + (long long)e * Mw;
  for (int w = threadIdx.x; w < Mw; w += blockDim.x) {
    const int a = w % mx, b = (w / mx) % my, c = w / (mx * my);
    Ze[w] = L.W[0][a] * L.W[1][b] * L.W[2][c] * X[w];
  }
}

// Shared memory: window X (Mw) | S_x, S_y, S_z (m_d^2) | lam (3 m_d) | W (3 m_d)
template <int KSMAX>
__global__ void __launch_bounds__(KSMAX <= 4 ? 128 : FDM_BIG_THREADS, KSMAX <= 4 ? 8 : 2) k_fdm_mma(LevelDev L, const double *__restrict__ r,
                                                 double *__restrict__ Z, int color,
                                                 double *__restrict__ u) {
  extern __shared__ double sm[];
  const int m[3] = {L.m[0], L.m[1], L.m[2]};
  const int Mw = L.Mw;
  double *X = sm;
  double *Ss[3];
  double *lam[3], *W[3];
  double *p = sm + Mw;
  for (int d = 0; d < 3; ++d) { Ss[d] = p; p += m[d] * m[d]; }
  for (int d = 0; d < 3; ++d) { lam[d] = p; p += m[d]; }
  for (int d = 0; d < 3; ++d) { W[d] = p; p += m[d]; }
  long long *offs = reinterpret_cast<long long *>(p);
  for (int d = 0; d < 3; ++d) {
    stage(Ss[d], L.S[d], m[d] * m[d]);
    stage(lam[d], L.lam[d], m[d]);
    stage(W[d], L.W[d], m[d]);
  }
  int e = blockIdx.x;
  if (color >= 0) {       // subdomain bx of parity class `color` (2x2x2 colouring)
    const int hx = L.nx >> 1, hy = L.ny >> 1;
    const int bx = e % hx, by = (e / hx) % hy, bz = e / (hx * hy);
    e = (2 * bx + (color & 1)) + L.nx * ((2 * by + ((color >> 1) & 1)) + L.ny * (2 * bz + (color >> 2)));
  }
  fdm_offsets(L, e, offs);
  __syncthreads();
  fdm_gather(L, r, offs, X);
  cp_async_wait_all();
  __syncthreads();
  const double *lamc[3] = {lam[0], lam[1], lam[2]};
  const double *Wc[3] = {W[0], W[1], W[2]};
  fdm_phases<KSMAX>(X, m, Ss, lamc, Wc, Z + (long long)e * Mw, color >= 0 ? u : nullptr, offs);
}

// ---------------------------------------------------------------------------------------------
// Even/odd fast diagonalisation.  Windows are reflection symmetric with odd extent m = 2H + 1
// (n = 2^l + 1 nodes, n_o layers each side), and the host eigensolver returns eigenvectors of
// exact parity, even modes first (gen_eig_parity).  Each 1D pass then splits into two half-size
// GEMMs (with the parity structure of the symmetric window operator):
//   forward   t_E = S_E^T (x_a + x_{m-1-a}, x_H),      t_O = S_O^T (x_a - x_{m-1-a})
//   backward  P = S_E t_E, Q = S_O t_O;  x_a = P_a + Q_a, x_{m-1-a} = P_a - Q_a, x_H = P_H
// with S_E = S[0..H][0..H], S_O = S[0..H-1][H+1..2H].  The same number of shared-memory loads
// feed 2 x MT x KS DMMAs per 8-column tile instead of ceil(m/8) x ceil(m/4) (23: 12 vs 18,
// 27: 16 vs 28, 13: 4 vs 8).  Intermediate mode-space data sits along DIR as [t_E ; t_O].
// QF: tile columns enumerate the Q direction fastest.  With the plane stride padded to 4 mod 16
// doubles (eo_plane_stride), the B-fragment loads of the x and y passes (QF) and of the z pass
// (!QF) hit 16 distinct 8-byte bank pairs per half warp.  Software pipelined: the loads and
// DMMAs of tile i+1 are issued before the epilogue of tile i (ping-pong accumulators).
template <int DIR, int MT, int KS, bool FWD, bool QF, class Epi>
__device__ __forceinline__ void eo_lines(const double *X, const Blk &B, const double *S, Epi &epi) {
  constexpr int PD = Other<DIR>::P, QD = Other<DIR>::Q;
  const int m = B.m[DIR], H = m >> 1;
  const int mp = B.m[PD], mq = B.m[QD];
  const int ncol = mp * mq;
  const int mf = QF ? mq : mp;
  const unsigned magic = 0xFFFFFFFFu / (unsigned)mf + 1u;
  const int so = B.s[DIR], sp = B.s[PD], sq = B.s[QD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ntiles = (ncol + 7) >> 3;
  if (warp >= ntiles) return;
  double aE[MT][KS], aO[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int o = mt * 8 + g, k = ks * 4 + t;
      if (FWD) {
        aE[mt][ks] = (o <= H && k <= H) ? S[k * m + o] : 0.0;
        aO[mt][ks] = (o < H && k < H) ? S[k * m + H + 1 + o] : 0.0;
      } else {
        aE[mt][ks] = (o <= H && k <= H) ? S[o * m + k] : 0.0;
        aO[mt][ks] = (o < H && k < H) ? S[o * m + H + 1 + k] : 0.0;
      }
    }
  int off1[KS], off2[KS];
  bool f1[KS], f2[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = ks * 4 + t;
    if (FWD) {                                    // lo = x_k, hi = x_{m-1-k}
      const int kl = min(k, H);
      off1[ks] = kl * so; off2[ks] = (m - 1 - kl) * so;
    } else {                                      // t_E[k], t_O[k]
      off1[ks] = min(k, H) * so; off2[ks] = (H + 1 + min(k, max(H - 1, 0))) * so;
    }
    f1[ks] = k <= H;                              // FWD: even input valid (k == H: x_H alone)
    f2[ks] = k < H;                               // FWD: pair valid; BWD: odd mode valid
  }
  auto colpq = [&](int n, int &p, int &q) {
    const int sl = __umulhi((unsigned)n, magic), f = n - sl * mf;
    if (QF) { q = f; p = sl; } else { p = f; q = sl; }
  };
  auto compute = [&](int tile, double (&cE)[MT][2], double (&cO)[MT][2]) {
    int pb, qb;
    colpq(min(tile * 8 + g, ncol - 1), pb, qb);
    const double *xb = X + pb * sp + qb * sq;
    double bE[KS], bO[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const double v1 = xb[off1[ks]], v2 = xb[off2[ks]];
      if (FWD) {
        bE[ks] = f2[ks] ? v1 + v2 : (f1[ks] ? v1 : 0.0);
        bO[ks] = f2[ks] ? v1 - v2 : 0.0;
      } else {
        bE[ks] = f1[ks] ? v1 : 0.0;
        bO[ks] = f2[ks] ? v2 : 0.0;
      }
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) { cE[mt][0] = cE[mt][1] = cO[mt][0] = cO[mt][1] = 0.0; }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        dmma884(cE[mt][0], cE[mt][1], aE[mt][ks], bE[ks]);
        dmma884(cO[mt][0], cO[mt][1], aO[mt][ks], bO[ks]);
      }
  };
  auto epilogue = [&](int tile, const double (&cE)[MT][2], const double (&cO)[MT][2]) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int n = tile * 8 + 2 * t + j;
      if (n >= ncol) continue;
      int p, q;
      colpq(n, p, q);
      const double cf = epi.template col<DIR>(p, q);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int o = mt * 8 + g;
        if (FWD) {
          if (o <= H) epi.template put<DIR>(o, p, q, cf, cE[mt][j]);
          if (o < H) epi.template put<DIR>(H + 1 + o, p, q, cf, cO[mt][j]);
        } else {
          if (o < H) {
            epi.template put<DIR>(o, p, q, cf, cE[mt][j] + cO[mt][j]);
            epi.template put<DIR>(m - 1 - o, p, q, cf, cE[mt][j] - cO[mt][j]);
          } else if (o == H) {
            epi.template put<DIR>(o, p, q, cf, cE[mt][j]);
          }
        }
      }
    }
  };
  double cE0[MT][2], cO0[MT][2], cE1[MT][2], cO1[MT][2];
  int tile = warp;
  compute(tile, cE0, cO0);
  for (;;) {
    const int t1 = tile + nw;
    if (t1 < ntiles) compute(t1, cE1, cO1);
    __syncwarp();
    epilogue(tile, cE0, cO0);
    if (t1 >= ntiles) break;
    const int t2 = t1 + nw;
    if (t2 < ntiles) compute(t2, cE0, cO0);
    __syncwarp();
    epilogue(t1, cE1, cO1);
    if (t2 >= ntiles) break;
    tile = t2;
  }
}

// z passes fused (forward, eigen-divide, backward) on warp-private z columns
template <int MT, int KS>
__device__ __forceinline__ void eo_z_fused(double *X, const Blk &B, const double *S,
                                           const double *const *lam) {
  const int m = B.m[2], H = m >> 1, mp = B.m[0], mq = B.m[1];
  const int ncol = mp * mq;
  const unsigned magic = 0xFFFFFFFFu / (unsigned)mp + 1u;
  const int so = B.s[2], sq = B.s[1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double aEf[MT][KS], aOf[MT][KS], aEb[MT][KS], aOb[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int o = mt * 8 + g, k = ks * 4 + t;
      const bool e_ok = o <= H && k <= H, o_ok = o < H && k < H;
      aEf[mt][ks] = e_ok ? S[k * m + o] : 0.0;
      aOf[mt][ks] = o_ok ? S[k * m + H + 1 + o] : 0.0;
      aEb[mt][ks] = e_ok ? S[o * m + k] : 0.0;
      aOb[mt][ks] = o_ok ? S[o * m + H + 1 + k] : 0.0;
    }
  int lo[KS], hi[KS], eo[KS], oo[KS];
  bool f1[KS], f2[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = ks * 4 + t, kl = min(k, H);
    lo[ks] = kl * so; hi[ks] = (m - 1 - kl) * so;
    eo[ks] = kl * so; oo[ks] = (H + 1 + min(k, max(H - 1, 0))) * so;
    f1[ks] = k <= H; f2[ks] = k < H;
  }
  double lz[MT], lzo[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int o = mt * 8 + g;
    lz[mt] = lam[2][min(o, H)];
    lzo[mt] = lam[2][H + 1 + min(o, max(H - 1, 0))];
  }
  const int ntiles = (ncol + 7) >> 3;
  for (int tile = warp; tile < ntiles; tile += nw) {
    const int nb = min(tile * 8 + g, ncol - 1);
    const int qb = __umulhi((unsigned)nb, magic), pb = nb - qb * mp;
    const double *xb = X + pb + qb * sq;
    double bE[KS], bO[KS], cE[MT][2], cO[MT][2];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const double v1 = xb[lo[ks]], v2 = xb[hi[ks]];
      bE[ks] = f2[ks] ? v1 + v2 : (f1[ks] ? v1 : 0.0);
      bO[ks] = f2[ks] ? v1 - v2 : 0.0;
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) { cE[mt][0] = cE[mt][1] = cO[mt][0] = cO[mt][1] = 0.0; }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        dmma884(cE[mt][0], cE[mt][1], aEf[mt][ks], bE[ks]);
        dmma884(cO[mt][0], cO[mt][1], aOf[mt][ks], bO[ks]);
      }
    __syncwarp();
    int wb[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int n = tile * 8 + 2 * t + j;
      wb[j] = -1;
      if (n >= ncol) continue;
      const int q = __umulhi((unsigned)n, magic), p = n - q * mp;
      wb[j] = p + q * sq;
      const double cf = lam[0][p] + lam[1][q];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int o = mt * 8 + g;
        if (o <= H) X[wb[j] + o * so] = cE[mt][j] * rcp_nr(cf + lz[mt]);
        if (o < H) X[wb[j] + (H + 1 + o) * so] = cO[mt][j] * rcp_nr(cf + lzo[mt]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      bE[ks] = f1[ks] ? xb[eo[ks]] : 0.0;
      bO[ks] = f2[ks] ? xb[oo[ks]] : 0.0;
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) { cE[mt][0] = cE[mt][1] = cO[mt][0] = cO[mt][1] = 0.0; }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        dmma884(cE[mt][0], cE[mt][1], aEb[mt][ks], bE[ks]);
        dmma884(cO[mt][0], cO[mt][1], aOb[mt][ks], bO[ks]);
      }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (wb[j] < 0) continue;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int o = mt * 8 + g;
        if (o < H) {
          X[wb[j] + o * so] = cE[mt][j] + cO[mt][j];
          X[wb[j] + (m - 1 - o) * so] = cE[mt][j] - cO[mt][j];
        } else if (o == H) {
          X[wb[j] + o * so] = cE[mt][j];
        }
      }
    }
  }
}

// tile variant for half-extent H: 1: H <= 3 (MT 1, KS 1), 2: H <= 7 (1, 2), 3: H <= 11 (2, 3),
// 4: H <= 15 (2, 4)
__host__ __device__ __forceinline__ int eo_variant(int m) {
  const int H = m >> 1;
  return H <= 3 ? 1 : (H <= 7 ? 2 : (H <= 11 ? 3 : 4));
}

template <int DIR, int VMAX, bool FWD, class Epi>
__device__ __forceinline__ void eo_dispatch(const double *X, const Blk &B, const double *S, Epi &epi) {
  const int v = eo_variant(B.m[DIR]);
  constexpr bool QF = DIR != 2;                  // x, y passes: z-fastest columns
  if (v == 1) eo_lines<DIR, 1, 1, FWD, QF>(X, B, S, epi);
  else if (VMAX >= 2 && v == 2) eo_lines<DIR, 1, 2, FWD, QF>(X, B, S, epi);
  else if (VMAX >= 3 && v == 3) eo_lines<DIR, 2, 3, FWD, QF>(X, B, S, epi);
  else if (VMAX >= 4) eo_lines<DIR, 2, 4, FWD, QF>(X, B, S, epi);
}

// shared-memory plane stride of the window: m0*m1 padded to 4 mod 16 doubles (bank spread)
__host__ __device__ __forceinline__ int eo_plane_stride(int m0, int m1) {
  const int a = m0 * m1;
  return a + ((4 - (a & 15)) & 15);
}

// gather into the padded window layout X[a + m0 b + s2 c]; one warp per window row (m0 <= 32)
__device__ __forceinline__ void eo_gather(const LevelDev &L, const double *r, const long long *offs,
                                          double *X, int s2) {
  const int m0 = L.m[0], m1 = L.m[1], m2 = L.m[2];
  const long long *xo = offs, *yo = offs + m0, *zo = offs + m0 + m1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const long long xa = lane < m0 ? xo[lane] : 0;
  const int rows = m1 * m2;
  int b = warp % m1, c = warp / m1;
  const int db = nw % m1, dc = nw / m1;
  for (int row = warp; row < rows; row += nw) {
    if (lane < m0) cp_async8(X + lane + m0 * b + s2 * c, r + xa + yo[b] + zo[c]);
    b += db; c += dc;
    if (b >= m1) { b -= m1; ++c; }
  }
}

template <int VMAX>
__device__ __forceinline__ void eo_z_dispatch(double *X, const Blk &B, const double *S,
                                              const double *const *lam) {
  const int v = eo_variant(B.m[2]);
  if (v == 1) eo_z_fused<1, 1>(X, B, S, lam);
  else if (VMAX >= 2 && v == 2) eo_z_fused<1, 2>(X, B, S, lam);
  else if (VMAX >= 3 && v == 3) eo_z_fused<2, 3>(X, B, S, lam);
  else if (VMAX >= 4) eo_z_fused<2, 4>(X, B, S, lam);
}

// Schwarz subdomain solve, even/odd variant of k_fdm_mma (same shared-memory layout, gather
// and weighted epilogue; Eq. 9-10).
template <int VMAX>
__global__ void __launch_bounds__(VMAX <= 2 ? 128 : 256, VMAX <= 2 ? 8 : 2) k_fdm_eo(LevelDev L, const double *__restrict__ r,
                                                 double *__restrict__ Z, int color,
                                                 double *__restrict__ u) {
  extern __shared__ double sm[];
  const int m[3] = {L.m[0], L.m[1], L.m[2]};
  const int Mw = L.Mw;
  const int s2 = eo_plane_stride(m[0], m[1]);
  double *X = sm;
  double *Ss[3];
  double *lam[3], *W[3];
  double *p = sm + s2 * m[2];
  for (int d = 0; d < 3; ++d) { Ss[d] = p; p += m[d] * m[d]; }
  for (int d = 0; d < 3; ++d) { lam[d] = p; p += m[d]; }
  for (int d = 0; d < 3; ++d) { W[d] = p; p += m[d]; }
  long long *offs = reinterpret_cast<long long *>(p);
  for (int d = 0; d < 3; ++d) {
    stage(Ss[d], L.S[d], m[d] * m[d]);
    stage(lam[d], L.lam[d], m[d]);
    stage(W[d], L.W[d], m[d]);
  }
  int e = blockIdx.x;
  if (color >= 0) {       // subdomain bx of parity class `color` (2x2x2 colouring)
    const int hx = L.nx >> 1, hy = L.ny >> 1;
    const int bx = e % hx, by = (e / hx) % hy, bz = e / (hx * hy);
    e = (2 * bx + (color & 1)) + L.nx * ((2 * by + ((color >> 1) & 1)) + L.ny * (2 * bz + (color >> 2)));
  }
  fdm_offsets(L, e, offs);
  __syncthreads();
  eo_gather(L, r, offs, X, s2);
  cp_async_wait_all();
  __syncthreads();
  const Blk B = {{m[0], m[1], m[2]}, {1, m[0], s2}};
  const Blk G = {{m[0], m[1], m[2]}, {1, m[0], m[0] * m[1]}};   // global window order (Z)
  const double *lamc[3] = {lam[0], lam[1], lam[2]};
  EpiStore st{X, B};
  eo_dispatch<0, VMAX, true>(X, B, Ss[0], st); __syncthreads();
  eo_dispatch<1, VMAX, true>(X, B, Ss[1], st); __syncthreads();
  eo_z_dispatch<VMAX>(X, B, Ss[2], lamc); __syncthreads();
  eo_dispatch<1, VMAX, false>(X, B, Ss[1], st); __syncthreads();
  if (color >= 0) {
    EpiWeightRed wr{u, offs, m[0], m[1], {W[0], W[1], W[2]}};
    eo_dispatch<0, VMAX, false>(X, B, Ss[0], wr);
  } else {
    EpiWeightStore ws{Z + (long long)e * Mw, G, {W[0], W[1], W[2]}};
    eo_dispatch<0, VMAX, false>(X, B, Ss[0], ws);
  }
}

}  // namespace

static void configure_smem() {
  static bool done = false;
  if (done) return;
  done = true;
  const int mx = 227 * 1024;
  cudaFuncSetAttribute(k_fdm_mma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_fdm_mma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_fdm_mma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_fdm_eo<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_fdm_eo<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_fdm_eo<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_fdm_eo<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
}

static size_t fdm_eo_smem_bytes(const LevelDev &L) {
  size_t d = (size_t)eo_plane_stride(L.m[0], L.m[1]) * L.m[2];
  for (int k = 0; k < 3; ++k) d += (size_t)L.m[k] * L.m[k] + 3 * (size_t)L.m[k];   // S, lam, W, offsets
  return d * sizeof(double);
}

// even/odd kernels need odd windows (reflection symmetric; always the case for n = 2^l + 1)
static bool fdm_eo_ok(const LevelDev &L) {
#ifdef PMG_NO_EO
  return false;
#endif
  return (L.m[0] & 1) && (L.m[1] & 1) && (L.m[2] & 1) && L.m[0] <= 32 && L.m[1] <= 32 &&
         L.m[2] <= 32 && fdm_eo_smem_bytes(L) <= 227 * 1024;
}

static int fdm_eo_vmax(const LevelDev &L) {
  return std::max(eo_variant(L.m[0]), std::max(eo_variant(L.m[1]), eo_variant(L.m[2])));
}

template <class F>
static void fdm_eo_launch(const LevelDev &L, int grid, size_t sb, cudaStream_t s, F &&args) {
  switch (fdm_eo_vmax(L)) {
    case 1: args(k_fdm_eo<1>, grid, 128, sb, s); break;
    case 2: args(k_fdm_eo<2>, grid, 128, sb, s); break;
    case 3: args(k_fdm_eo<3>, grid, 256, sb, s); break;
    default: args(k_fdm_eo<4>, grid, 256, sb, s); break;
  }
}

size_t fdm_mma_smem_bytes(const LevelDev &L) {
  size_t d = (size_t)L.Mw;
  for (int k = 0; k < 3; ++k) d += (size_t)L.m[k] * L.m[k] + 3 * (size_t)L.m[k];   // S, lam, W, offsets
  return d * sizeof(double);
}

bool fdm_mma_ok(const LevelDev &L) {
  return L.m[0] <= 32 && L.m[1] <= 32 && L.m[2] <= 32 && fdm_mma_smem_bytes(L) <= 227 * 1024;
}

bool fdm_colored_ok(const LevelDev &L) {
  if (!fdm_mma_ok(L)) return false;
  if ((L.nx & 1) || (L.ny & 1) || (L.nz & 1)) return false;          // 2-colouring across the seam
  for (int d = 0; d < 3; ++d)
    if (2 * L.no[d] > L.n) return false;                            // same-colour windows disjoint
  return true;
}

cudaError_t launch_fdm_colored(const LevelDev &L, const double *r, double *u, cudaStream_t s) {
  configure_smem();
  const size_t sb = fdm_mma_smem_bytes(L);
  const int ks = (std::max(L.m[0], std::max(L.m[1], L.m[2])) + 3) >> 2;
  const int grid = L.Ne / 8;
  if (fdm_eoc_launch(L, r, nullptr, 0, u, s)) {
    for (int color = 1; color < 8; ++color) fdm_eoc_launch(L, r, nullptr, color, u, s);
    return cudaGetLastError();
  }
  if (fdm_eo_ok(L)) {
    for (int color = 0; color < 8; ++color)
      fdm_eo_launch(L, grid, fdm_eo_smem_bytes(L), s, [&](auto kern, int gr, int th, size_t b, cudaStream_t st) {
        kern<<<gr, th, b, st>>>(L, r, nullptr, color, u);
      });
    return cudaGetLastError();
  }
  for (int color = 0; color < 8; ++color) {
    if (ks <= 2) k_fdm_mma<2><<<grid, 128, sb, s>>>(L, r, nullptr, color, u);
    else if (ks <= 4) k_fdm_mma<4><<<grid, 128, sb, s>>>(L, r, nullptr, color, u);
    else k_fdm_mma<8><<<grid, FDM_BIG_THREADS, sb, s>>>(L, r, nullptr, color, u);
  }
  return cudaGetLastError();
}

cudaError_t launch_fdm(const LevelDev &L, const double *r, double *Z, double *scr, bool smem,
                       size_t smem_bytes, cudaStream_t s) {
#ifdef PMG_FORCE_DFMA
  if (L.n > 9) {
#endif
  if (fdm_eoc_launch(L, r, Z, -1, nullptr, s)) return cudaGetLastError();   // compile-time shape
  if (fdm_mma_ok(L)) {
    configure_smem();
    const size_t sb = fdm_mma_smem_bytes(L);
    if (fdm_eo_ok(L)) {
      fdm_eo_launch(L, L.Ne, fdm_eo_smem_bytes(L), s, [&](auto kern, int gr, int th, size_t b, cudaStream_t st) {
        kern<<<gr, th, b, st>>>(L, r, Z, -1, nullptr);
      });
      return cudaGetLastError();
    }
    const int ks = (std::max(L.m[0], std::max(L.m[1], L.m[2])) + 3) >> 2;
    if (ks <= 2) k_fdm_mma<2><<<L.Ne, 128, sb, s>>>(L, r, Z, -1, nullptr);
    else if (ks <= 4) k_fdm_mma<4><<<L.Ne, 128, sb, s>>>(L, r, Z, -1, nullptr);
    else k_fdm_mma<8><<<L.Ne, FDM_BIG_THREADS, sb, s>>>(L, r, Z, -1, nullptr);
    return cudaGetLastError();
  }
#ifdef PMG_FORCE_DFMA
  }
#endif
  if (smem) {
    static size_t configured = 0;
    if (smem_bytes > configured) {
      cudaFuncSetAttribute(k_fdm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
      configured = smem_bytes;
    }
    k_fdm<<<L.Ne, 512, smem_bytes, s>>>(L, r, Z, scr, 1);
  } else {
    k_fdm<<<L.Ne, 512, 0, s>>>(L, r, Z, scr, 0);
  }
  return cudaGetLastError();
}
}  // namespace pmg
