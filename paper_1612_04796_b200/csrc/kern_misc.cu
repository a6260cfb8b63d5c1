// Deterministic fold, coarse pseudo-inverse, reductions, PCG vector ops, RHS.
// arXiv:1612.04796; PAPER.md line numbers cited per kernel.
#include <algorithm>

#include <cooperative_groups.h>

#include "kcommon.cuh"

namespace cg = cooperative_groups;

namespace pmg {
namespace {

// Register-only fold: one thread per DOF issues all (up to 27) predicated loads of the
// weighted window values that cover it before summing them in a fixed order -> maximal
// memory-level parallelism, deterministic result.  NT = compile-time n (fast index math).
// Min 4 CTAs/SM (<= 64 registers): measured 0.515 vs 0.545 ms per cycle at c3's top level.
template <int NT, bool TR>
__global__ void __launch_bounds__(256, 4) k_fold2(LevelDev L, const double *__restrict__ Z,
                                               double *__restrict__ u, int zero,
                                               double *__restrict__ T) {
  extern __shared__ double sm[];          // TR: the folded element (n^3) + trace table (12 n)
  const int n = NT > 0 ? NT : L.n;
  const int n3 = n * n * n;
  const int mx = L.m[0], my = L.m[1];
  const long long Mw = L.Mw;
  const int e = blockIdx.x;
  const int ec[3] = {e % L.nx, (e / L.nx) % L.ny, e / (L.nx * L.ny)};
  const int edim[3] = {L.nx, L.ny, L.nz};
  int se[3][3];                       // source subdomain coordinate per direction: o = -1, 0, +1
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int o = 0; o < 3; ++o) se[d][o] = wrap(ec[d] + o - 1, edim[d]);
  const int no0 = L.no[0], no1 = L.no[1], no2 = L.no[2];
  // n = 33: blockIdx.y splits the element's DOFs (64 large elements must fill the GPU)
  constexpr bool SPLIT = NT == 33 && !TR;
  const int t0 = SPLIT ? blockIdx.y * blockDim.x + threadIdx.x : threadIdx.x;
  const int dt = SPLIT ? gridDim.y * blockDim.x : blockDim.x;
  for (int t = t0; t < n3; t += dt) {
    const int i = t % n, j = (t / n) % n, k = t / (n * n);
    const int idx[3] = {i, j, k};
    const int nod[3] = {no0, no1, no2};
    bool v[3][3];
    int wi[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int no = nod[d], id = idx[d];
      v[d][0] = id < no;        wi[d][0] = no + n + id;     // left-neighbour subdomain
      v[d][1] = true;           wi[d][1] = no + id;         // own subdomain
      v[d][2] = id >= n - no;   wi[d][2] = id - (n - no);   // right-neighbour subdomain
    }
    const long long g = (long long)e * n3 + t;
    double du = zero ? 0.0 : u[g];
#pragma unroll
    for (int oz = 0; oz < 3; ++oz) {
      if (!v[2][oz]) continue;
      double z[9];
#pragma unroll
      for (int oy = 0; oy < 3; ++oy)
#pragma unroll
        for (int ox = 0; ox < 3; ++ox) {
          const bool ok = v[0][ox] && v[1][oy];
          const long long sidx = se[0][ox] + L.nx * (se[1][oy] + (long long)L.ny * se[2][oz]);
          z[ox + 3 * oy] = ok ? __ldg(Z + sidx * Mw + wi[0][ox] + mx * (wi[1][oy] + my * wi[2][oz])) : 0.0;
        }
#pragma unroll
      for (int q = 0; q < 9; ++q) du += z[q];
    }
    u[g] = du;
    if (TR) sm[t] = du;
  }
  if (!TR) return;
  // fused trace pass of the following residual: face values / derivatives of the new u
  double *tab = sm + ((n3 + 1) & ~1);
  stage_trace_tab(L, tab);
  __syncthreads();
  elem_traces<0>(sm, tab, n, T + (long long)e * 12 * n * n);
}

// Row fold (Eq. 10): a warp folds whole x-rows of the element.  Lane a of a
// row is the window x-index a in [0, m_x): lanes n_o <= a < n_o + n read the row of a window
// centred on this element column (own x), lanes a >= n_o + n read the same row of the LEFT
// neighbour's window (its right overlap covers DOFs i = a - n_o - n) and lanes a < n_o that of
// the RIGHT neighbour's — one load instruction fetches all three x-sources of a row, two
// shuffles bring the strip values to the DOFs they cover.  The (y, z) sources are row-uniform:
// with 2 n_o <= n (MERGED) a row has the own window plus at most one neighbour per direction
// (4 predicated loads), otherwise all 3 x 3 combinations are tested (9).  Every address is
// computed once per row instead of once per DOF and source (the register fold k_fold2 spent 303
// thread instructions per DOF, 27 mostly predicated-off loads), and RB rows per warp are in
// flight at once.  32 / m_x rows share a warp when they fit (n = 9: two rows of 13 lanes).
// Fixed summation order -> deterministic.  TR: face traces of the new u from shared memory.
#ifndef PMG_FOLD4_MINB
#define PMG_FOLD4_MINB 4
#endif
template <int NT, bool TR, bool MERGED>
__global__ void __launch_bounds__(256, PMG_FOLD4_MINB) k_fold4(LevelDev L, const double *__restrict__ Z,
                                                  double *__restrict__ u, int zero,
                                                  double *__restrict__ T) {
  extern __shared__ double sm[];          // TR: the folded element (n^3) + trace table (12 n)
  const int n = NT > 0 ? NT : L.n;
  const int n2 = n * n, n3 = n2 * n;
  const int mx = L.m[0], my = L.m[1];
  const int no0 = L.no[0], no1 = L.no[1], no2 = L.no[2];
  const long long Mw = L.Mw;
#ifdef PMG_FOLD_REVERSE        // diagnostic: walk the elements backwards (the tail of Z is still in L2)
  const int e = gridDim.x - 1 - blockIdx.x;
#else
  const int e = blockIdx.x;
#endif
  const int ec[3] = {e % L.nx, (e / L.nx) % L.ny, e / (L.nx * L.ny)};
  const int edim[3] = {L.nx, L.ny, L.nz};
  // all offsets are 32-bit element indices into Z (the launcher checks Ne * Mw < 2^31)
  int sb[3][3];                       // source-subdomain base per direction and offset -1, 0, +1
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int o = 0; o < 3; ++o)
      sb[d][o] = wrap(ec[d] + o - 1, edim[d]) * (int)(d == 0 ? Mw : (d == 1 ? Mw * L.nx : Mw * L.nx * L.ny));
#ifdef PMG_FOLD_PREFETCH        // diagnostic: L2 prefetch of the Z and u blocks of the element that many CTAs ahead
  if (threadIdx.x == 0 && (long long)e + PMG_FOLD_PREFETCH < L.Ne && (long long)L.Ne * n3 > (8ll << 20)) {
    prefetch_l2_doubles(Z + ((long long)e + PMG_FOLD_PREFETCH) * Mw, Mw);
    if (!zero) prefetch_l2_doubles(u + ((long long)e + PMG_FOLD_PREFETCH) * n3, n3);
  }
#endif
  if (TR) stage_trace_tab(L, sm + ((n3 + 1) & ~1));    // read after the post-fold barrier
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int rpw = 32 / mx;                                  // rows per warp instruction (>= 1)
  const int sr = lane / mx, a = lane - sr * mx;
  const bool act = sr < rpw;
  const int ox = a < no0 ? 2 : (a < no0 + n ? 1 : 0);       // right nb | own | left nb window
  const int i = a - no0;
  const bool own = act && ox == 1;
  const bool addL = own && i < no0, addR = own && i >= n - no0;
  const int srcL = min(lane + n, 31), srcR = max(lane - n, 0);
  const int wsy = mx, wsz = mx * my;
  // per-source offsets: own / left / right window in y and z, x part folded into the own-y term
  const int xb = (ox == 0 ? sb[0][0] : (ox == 1 ? sb[0][1] : sb[0][2])) + a;
  const int yO = sb[1][1] + wsy * no1 + xb, yL = sb[1][0] + wsy * (no1 + n) + xb, yR = sb[1][2] - wsy * (n - no1) + xb;
  const int zO = sb[2][1] + wsz * no2, zL = sb[2][0] + wsz * (no2 + n), zR = sb[2][2] - wsz * (n - no2);
  double *ue = u + (long long)e * n3 + i;
  constexpr int RB = MERGED ? 4 : 2, NL = MERGED ? 4 : 9;
  const int rstep = nw * rpw;
  for (int rb = warp * rpw + sr; rb < n2 + sr; rb += rstep * RB) {
    double z[RB][NL], uo[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const int row = rb + q * rstep;
      const bool rv = act && row < n2;
      const int k = row / n, j = row - k * n;
      uo[q] = (rv && own && !zero) ? ue[n * row] : 0.0;
      const int yj = wsy * j, zk = wsz * k;
      if (MERGED) {
        const bool ly = j < no1, lz = k < no2;
        const bool py = ly || j >= n - no1, pz = lz || k >= n - no2;
        const int y0 = yO + yj, y1 = (ly ? yL : yR) + yj;
        const int z0 = zO + zk, z1 = (lz ? zL : zR) + zk;
        z[q][0] = rv ? __ldg(Z + (y0 + z0)) : 0.0;
        z[q][1] = (rv && py) ? __ldg(Z + (y1 + z0)) : 0.0;
        z[q][2] = (rv && pz) ? __ldg(Z + (y0 + z1)) : 0.0;
        z[q][3] = (rv && py && pz) ? __ldg(Z + (y1 + z1)) : 0.0;
      } else {
#pragma unroll
        for (int oz = 0; oz < 3; ++oz) {
          const bool pz = oz == 1 || (oz == 0 ? k < no2 : k >= n - no2);
          const int zo = (oz == 0 ? zL : (oz == 1 ? zO : zR)) + zk;
#pragma unroll
          for (int oy = 0; oy < 3; ++oy) {
            const bool py = oy == 1 || (oy == 0 ? j < no1 : j >= n - no1);
            const int yo = (oy == 0 ? yL : (oy == 1 ? yO : yR)) + yj;
            z[q][oy + 3 * oz] = (rv && py && pz) ? __ldg(Z + (yo + zo)) : 0.0;
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const int row = rb + q * rstep;
      double v = z[q][0];
#pragma unroll
      for (int c = 1; c < NL; ++c) v += z[q][c];
      const double vl = __shfl_sync(0xffffffffu, v, srcL), vr = __shfl_sync(0xffffffffu, v, srcR);
      double res = uo[q] + v;
      if (addL) res += vl;
      if (addR) res += vr;
      if (own && row < n2) {
        ue[n * row] = res;
        if (TR) sm[i + n * row] = res;
      }
    }
  }
  if (!TR) return;
  __syncthreads();
  // fused trace pass of the following residual: face values / derivatives of the new u
  // (even/odd form, kcommon.cuh); the table was staged before the fold loop
  elem_traces<NT>(sm, sm + ((n3 + 1) & ~1), n, T + (long long)e * 12 * n2);
}

// Small elements (n = 3, 5): EPB elements per 256-thread CTA, one thread per DOF, same fixed
// 27-source summation order as k_fold2; TR: the face traces of the new u from shared memory in
// the same launch (a 27- or 125-DOF element left most of a 256-thread CTA idle, and the separate
// trace launch cost as much as the fold).
template <int NT, int EPB, bool TR>
__global__ void __launch_bounds__(256) k_fold_small(LevelDev L, const double *__restrict__ Z,
                                                  double *__restrict__ u, int zero,
                                                  double *__restrict__ T) {
  constexpr int n = NT, n2 = n * n, n3 = n2 * n;
  __shared__ double sm[EPB * n3];
  __shared__ __align__(16) double trs[3 * trace_tab_len(n) + 2];   // even/odd trace table
  const int mx = L.m[0], my = L.m[1];
  const long long Zs = L.Mw;
  const int le = threadIdx.x / n3, t = threadIdx.x - le * n3;
  const int e = blockIdx.x * EPB + le;
  if (TR) stage_trace_tab(L, trs);
  if (le < EPB && e < L.Ne) {
    const int ec[3] = {e % L.nx, (e / L.nx) % L.ny, e / (L.nx * L.ny)};
    const int edim[3] = {L.nx, L.ny, L.nz};
    int se[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int o = 0; o < 3; ++o) se[d][o] = wrap(ec[d] + o - 1, edim[d]);
    const int i = t % n, j = (t / n) % n, k = t / n2;
    const int idx[3] = {i, j, k};
    const int nod[3] = {L.no[0], L.no[1], L.no[2]};
    bool v[3][3];
    int wi[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int no = nod[d], id = idx[d];
      v[d][0] = id < no;        wi[d][0] = no + n + id;
      v[d][1] = true;           wi[d][1] = no + id;
      v[d][2] = id >= n - no;   wi[d][2] = id - (n - no);
    }
    const long long g = (long long)e * n3 + t;
    double du = zero ? 0.0 : u[g];
#pragma unroll
    for (int oz = 0; oz < 3; ++oz) {
      if (!v[2][oz]) continue;
      double z[9];
#pragma unroll
      for (int oy = 0; oy < 3; ++oy)
#pragma unroll
        for (int ox = 0; ox < 3; ++ox) {
          const bool ok = v[0][ox] && v[1][oy];
          const long long sidx = se[0][ox] + L.nx * (se[1][oy] + (long long)L.ny * se[2][oz]);
          z[ox + 3 * oy] = ok ? __ldg(Z + sidx * Zs + wi[0][ox] + mx * (wi[1][oy] + my * wi[2][oz])) : 0.0;
        }
#pragma unroll
      for (int q = 0; q < 9; ++q) du += z[q];
    }
    u[g] = du;
    if (TR) sm[le * n3 + t] = du;
  }
  if (!TR) return;
  __syncthreads();
  for (int w = threadIdx.x; w < EPB * 3 * n2; w += blockDim.x) {
    const int lb = w / (3 * n2), r = w - lb * 3 * n2;
    const int eb = blockIdx.x * EPB + lb;
    if (eb >= L.Ne) break;
    elem_trace_item<NT>(sm + lb * n3, trs, n, r, T + (long long)eb * 12 * n2);
  }
}

// ---------------------------------------------------------------------------------------------
// Coarse level (P_0 = 1): u_0 = A_0^+ f_0 by global fast diagonalisation on the periodic
// (2nx, 2ny, 2nz) grid with the constant mode removed (Alg. 1 l.295).
__global__ void k_coarse_gather(int nx, int ny, int nz, const double *__restrict__ f0,
                                const double *__restrict__ mean, double *__restrict__ G) {
  const long long N = 8LL * nx * ny * nz;
  const double mu = *mean;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N;
       g += (long long)gridDim.x * blockDim.x) {
    const int node = g & 7;
    const long long e = g >> 3;
    const int i = node & 1, j = (node >> 1) & 1, k = node >> 2;
    const int ex = e % nx, ey = (e / nx) % ny, ez = e / ((long long)nx * ny);
    const long long X = 2 * ex + i, Y = 2 * ey + j, Z = 2 * ez + k;
    G[X + 2LL * nx * (Y + 2LL * ny * Z)] = f0[g] - mu;
  }
}

__global__ void k_lex_contract(CoarseDev C, int axis, int forward, const double *__restrict__ in,
                               double *__restrict__ out) {
  const long long N = (long long)C.G[0] * C.G[1] * C.G[2];
  const int Gd = C.G[axis];
  const long long st = axis == 0 ? 1 : (axis == 1 ? C.G[0] : (long long)C.G[0] * C.G[1]);
  const double *S = C.S[axis];
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N;
       g += (long long)gridDim.x * blockDim.x) {
    const int o = (g / st) % Gd;
    const double *src = in + (g - o * st);
    double acc = 0;
    if (forward) for (int k = 0; k < Gd; ++k) acc += S[k * Gd + o] * src[k * st];
    else for (int k = 0; k < Gd; ++k) acc += S[o * Gd + k] * src[k * st];
    out[g] = acc;
  }
}

__global__ void k_coarse_divide(CoarseDev C, double *__restrict__ G) {
  const long long N = (long long)C.G[0] * C.G[1] * C.G[2];
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N;
       g += (long long)gridDim.x * blockDim.x) {
    const int a = g % C.G[0], b = (g / C.G[0]) % C.G[1], c = g / ((long long)C.G[0] * C.G[1]);
    // eigenvalue index 0 is the (exactly zero) constant mode in every direction
    G[g] = (a == 0 && b == 0 && c == 0) ? 0.0 : G[g] / (C.lam[0][a] + C.lam[1][b] + C.lam[2][c]);
  }
}

__global__ void k_coarse_scatter(int nx, int ny, int nz, const double *__restrict__ G,
                                 const double *__restrict__ mean, double *__restrict__ u0) {
  const long long N = 8LL * nx * ny * nz;
  const double mu = *mean;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N;
       g += (long long)gridDim.x * blockDim.x) {
    const int node = g & 7;
    const long long e = g >> 3;
    const int i = node & 1, j = (node >> 1) & 1, k = node >> 2;
    const int ex = e % nx, ey = (e / nx) % ny, ez = e / ((long long)nx * ny);
    const long long X = 2 * ex + i, Y = 2 * ey + j, Z = 2 * ez + k;
    u0[g] = G[X + 2LL * nx * (Y + 2LL * ny * Z)] - mu;
  }
}

// Fused coarse-solve passes.  At P_0 = 1 on a uniform grid the 1D mass matrices are multiples of
// the identity (w = (1,1)), so dropping the (exactly constant) null mode of the fast
// diagonalisation already realises the Euclidean projection of f_0 and returns a Euclidean
// mean-free u_0: A_0^+ f_0 = S (Lambda^+) S^T f_0 with no separate mean reductions.
__device__ __forceinline__ long long coarse_elem_index(int nx, int ny, int X, int Y, int Z) {
  const long long e = (X >> 1) + (long long)nx * ((Y >> 1) + (long long)ny * (Z >> 1));
  return e * 8 + (X & 1) + 2 * (Y & 1) + 4 * (Z & 1);
}

// x-forward pass reading f_0 in element-major order: G[X',Y,Z] = sum_X S0x[X][X'] f0(X,Y,Z)
__global__ void k_coarse_xf(CoarseDev C, int nx, int ny, const double *__restrict__ f0,
                            double *__restrict__ G) {
  const int Gx = C.G[0], Gy = C.G[1];
  const long long N = (long long)Gx * Gy * C.G[2];
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N;
       g += (long long)gridDim.x * blockDim.x) {
    const int o = g % Gx, Y = (g / Gx) % Gy, Z = g / ((long long)Gx * Gy);
    double acc = 0;
    for (int X = 0; X < Gx; ++X) acc += C.S[0][X * Gx + o] * __ldg(f0 + coarse_elem_index(nx, ny, X, Y, Z));
    G[g] = acc;
  }
}

// z column (one warp per column, lane = z index): forward S_z^T, divide by the eigenvalue
// sums (null mode -> 0), backward S_z; column values exchanged with warp shuffles.
__global__ void k_coarse_z(CoarseDev C, double *__restrict__ G) {
  const int Gx = C.G[0], Gy = C.G[1], Gz = C.G[2];
  const long long cols = (long long)Gx * Gy;
  const int lane = threadIdx.x & 31;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const double *S = C.S[2];
  for (long long cidx = w0; cidx < cols; cidx += nw) {
    const int a = cidx % Gx, b = cidx / Gx;
    const double v = lane < Gz ? G[cidx + lane * cols] : 0.0;
    double acc = 0.0;
    for (int k = 0; k < Gz; ++k) {
      const double vk = __shfl_sync(0xffffffffu, v, k);
      if (lane < Gz) acc += S[k * Gz + lane] * vk;
    }
    double w = 0.0;
    if (lane < Gz && !(a == 0 && b == 0 && lane == 0))
      w = acc / (C.lam[0][a] + C.lam[1][b] + C.lam[2][lane]);
    double out = 0.0;
    for (int k = 0; k < Gz; ++k) {
      const double wk = __shfl_sync(0xffffffffu, w, k);
      if (lane < Gz) out += S[lane * Gz + k] * wk;
    }
    if (lane < Gz) G[cidx + lane * cols] = out;
  }
}

// Whole coarse solve u_0 = A_0^+ f_0 in ONE CTA for small coarse grids (G_x G_y G_z <= 1024,
// every G_d <= 32: c1, c4; at 16^3 (c2) one SM is slower than five launches): same passes and summation order as k_coarse_xf / k_lex_contract
// / k_coarse_z / k_coarse_xb, staged in shared memory, so the 5-launch chain (launch-latency
// bound at these sizes) becomes one launch.  smem: A, B (N each) | S_x, S_y, S_z | lam.
__global__ void __launch_bounds__(1024) k_coarse_one(CoarseDev C, int nx, int ny,
                                                     const double *__restrict__ f0,
                                                     double *__restrict__ u0) {
  extern __shared__ double sm[];
  const int Gx = C.G[0], Gy = C.G[1], Gz = C.G[2];
  const int N = Gx * Gy * Gz;
  double *A = sm, *B = sm + N;
  double *S[3] = {B + N, B + N + Gx * Gx, B + N + Gx * Gx + Gy * Gy};
  double *lam[3] = {S[2] + Gz * Gz, S[2] + Gz * Gz + Gx, S[2] + Gz * Gz + Gx + Gy};
  const int Gd[3] = {Gx, Gy, Gz};
  for (int d = 0; d < 3; ++d) {
    for (int i = threadIdx.x; i < Gd[d] * Gd[d]; i += blockDim.x) S[d][i] = C.S[d][i];
    for (int i = threadIdx.x; i < Gd[d]; i += blockDim.x) lam[d][i] = C.lam[d][i];
  }
  for (int g = threadIdx.x; g < N; g += blockDim.x) {
    const int X = g % Gx, Y = (g / Gx) % Gy, Z = g / (Gx * Gy);
    A[g] = __ldg(f0 + coarse_elem_index(nx, ny, X, Y, Z));
  }
  __syncthreads();
  // contraction along axis d of `in` into `out` (lexicographic x fastest)
  auto pass = [&](const double *in, double *out, int d, bool forward) {
    const int st = d == 0 ? 1 : (d == 1 ? Gx : Gx * Gy);
    const int G = Gd[d];
    const double *Sd = S[d];
    for (int g = threadIdx.x; g < N; g += blockDim.x) {
      const int o = (g / st) % G;
      const double *src = in + (g - o * st);
      double acc = 0;
      if (forward) for (int k = 0; k < G; ++k) acc += Sd[k * G + o] * src[k * st];
      else for (int k = 0; k < G; ++k) acc += Sd[o * G + k] * src[k * st];
      out[g] = acc;
    }
    __syncthreads();
  };
  pass(A, B, 0, true);
  pass(B, A, 1, true);
  pass(A, B, 2, true);
  for (int g = threadIdx.x; g < N; g += blockDim.x) {
    const int a = g % Gx, b = (g / Gx) % Gy, c = g / (Gx * Gy);
    B[g] = (a == 0 && b == 0 && c == 0) ? 0.0 : B[g] / (lam[0][a] + lam[1][b] + lam[2][c]);
  }
  __syncthreads();
  pass(B, A, 2, false);
  pass(A, B, 1, false);
  for (int g = threadIdx.x; g < N; g += blockDim.x) {
    const int X = g % Gx, Y = (g / Gx) % Gy, Z = g / (Gx * Gy);
    const double *row = B + (g - X);
    double acc = 0;
    for (int k = 0; k < Gx; ++k) acc += S[0][X * Gx + k] * row[k];
    u0[coarse_elem_index(nx, ny, X, Y, Z)] = acc;
  }
}

// Whole coarse solve in ONE thread-block cluster (8 CTAs, distributed shared memory) for coarse
// grids beyond one CTA's reach (1024 < G_x G_y G_z <= 32^3: c2/c5 16^3, c3 32^3).  CTA r keeps
// the z-planes [r pp, (r+1) pp) of the lexicographic grid in its shared memory: the x and y
// passes are plane-local; for the z pass (forward S_z^T, eigen-divide, backward S_z) the columns
// are dealt out over the cluster and a warp reads / writes its column's G_z values straight from
// the owning CTAs' shared memory (DSMEM), lane = z index, values exchanged by shuffles as in
// k_coarse_z.  One launch instead of five, no global scratch; Alg. 1 l.295.
__global__ void __launch_bounds__(512) k_coarse_cluster(CoarseDev C, int nx, int ny,
                                                        const double *__restrict__ f0,
                                                        double *__restrict__ u0) {
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks(), rk = (int)cl.block_rank();
  const int Gx = C.G[0], Gy = C.G[1], Gz = C.G[2];
  const int plane = Gx * Gy;
  const int pp = (Gz + CS - 1) / CS;
  const int z0 = rk * pp, nzl = max(0, min(Gz, z0 + pp) - z0);
  extern __shared__ double sm[];
  double *A = sm, *B = sm + pp * plane;
  double *Sx = B + pp * plane, *Sy = Sx + Gx * Gx, *Sz = Sy + Gy * Gy;
  double *SxT = Sz + Gz * Gz, *SzT = SxT + Gx * Gx;        // transposed copies: the backward x and z
  double *lx = SzT + Gz * Gz, *ly = lx + Gx, *lz = ly + Gy;  // passes read S rows lane-contiguously
  for (int i = threadIdx.x; i < Gx * Gx; i += blockDim.x) {
    const double v = C.S[0][i];
    Sx[i] = v;
    SxT[(i % Gx) * Gx + i / Gx] = v;
  }
  for (int i = threadIdx.x; i < Gy * Gy; i += blockDim.x) Sy[i] = C.S[1][i];
  for (int i = threadIdx.x; i < Gz * Gz; i += blockDim.x) {
    const double v = C.S[2][i];
    Sz[i] = v;
    SzT[(i % Gz) * Gz + i / Gz] = v;
  }
  for (int i = threadIdx.x; i < Gx; i += blockDim.x) lx[i] = C.lam[0][i];
  for (int i = threadIdx.x; i < Gy; i += blockDim.x) ly[i] = C.lam[1][i];
  for (int i = threadIdx.x; i < Gz; i += blockDim.x) lz[i] = C.lam[2][i];
  const int nl = nzl * plane;
  for (int g = threadIdx.x; g < nl; g += blockDim.x) {
    const int X = g % Gx, Y = (g / Gx) % Gy, zl = g / plane;
    A[g] = __ldg(f0 + coarse_elem_index(nx, ny, X, Y, z0 + zl));
  }
  __syncthreads();
  for (int g = threadIdx.x; g < nl; g += blockDim.x) {            // x forward: B = S_x^T A
    const int o = g % Gx;
    const double *row = A + (g - o);
    double acc = 0;
    for (int k = 0; k < Gx; ++k) acc += Sx[k * Gx + o] * row[k];
    B[g] = acc;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < nl; g += blockDim.x) {            // y forward: A = S_y^T B
    const int a = g % Gx, o = (g / Gx) % Gy, zl = g / plane;
    const double *col = B + a + plane * zl;
    double acc = 0;
    for (int k = 0; k < Gy; ++k) acc += Sy[k * Gy + o] * col[k * Gx];
    A[g] = acc;
  }
  cl.sync();
  {   // z forward, divide (null mode -> 0), z backward on this CTA's share of the columns
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int cpc = (plane + CS - 1) / CS;
    const int c1 = min(plane, (rk + 1) * cpc);
    double *RA = cl.map_shared_rank(A, min(lane / pp, CS - 1));
    const int zoff = plane * (lane % pp);
    const bool zl = lane < Gz;
    for (int cidx = rk * cpc + warp; cidx < c1; cidx += nw) {
      const int a = cidx % Gx, b = cidx / Gx;
      const double v = zl ? RA[cidx + zoff] : 0.0;
      double acc = 0.0;
      for (int k = 0; k < Gz; ++k) {
        const double vk = __shfl_sync(0xffffffffu, v, k);
        if (zl) acc += Sz[k * Gz + lane] * vk;
      }
      double w = 0.0;
      if (zl && !(a == 0 && b == 0 && lane == 0)) w = acc / (lx[a] + ly[b] + lz[lane]);
      double out = 0.0;
      for (int k = 0; k < Gz; ++k) {
        const double wk = __shfl_sync(0xffffffffu, w, k);
        if (zl) out += SzT[k * Gz + lane] * wk;
      }
      if (zl) RA[cidx + zoff] = out;
    }
  }
  cl.sync();
  for (int g = threadIdx.x; g < nl; g += blockDim.x) {            // y backward: B = S_y A
    const int a = g % Gx, Y = (g / Gx) % Gy, zl = g / plane;
    const double *col = A + a + plane * zl;
    double acc = 0;
    for (int k = 0; k < Gy; ++k) acc += Sy[Y * Gy + k] * col[k * Gx];
    B[g] = acc;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < nl; g += blockDim.x) {            // x backward -> u_0 (element-major)
    const int X = g % Gx, Y = (g / Gx) % Gy, zl = g / plane;
    const double *row = B + (g - X);
    double acc = 0;
    for (int k = 0; k < Gx; ++k) acc += SxT[k * Gx + X] * row[k];
    u0[coarse_elem_index(nx, ny, X, Y, z0 + zl)] = acc;
  }
}

// Plane kernels for coarse grids beyond the cluster's reach (32^3: c3, c5): three launches instead
// of five, every table read from shared memory without bank conflicts.
//   k_coarse_plane_fwd  CTA = one z-plane, thread = (X', Y): stage the plane of f_0 (element-major
//                       gather), x forward then y forward in shared memory -> G (lexicographic);
//   k_coarse_zcols      CTA = 32 z columns, warp = one column, lane = z index: forward S_z^T,
//                       eigen-divide (null mode -> 0), backward S_z with S_z and its transpose in
//                       shared memory (the global-table version read rows with a 32-line stride);
//   k_coarse_plane_bwd  CTA = one z-plane: y backward, x backward (transposed tables) -> u_0.
__global__ void __launch_bounds__(1024) k_coarse_plane_fwd(CoarseDev C, int nx, int ny,
                                                          const double *__restrict__ f0,
                                                          double *__restrict__ G) {
  extern __shared__ double sm[];
  const int Gx = C.G[0], Gy = C.G[1], plane = Gx * Gy, Z = blockIdx.x;
  double *A = sm, *B = A + plane, *Sx = B + plane, *Sy = Sx + Gx * Gx;
  for (int i = threadIdx.x; i < Gx * Gx; i += blockDim.x) Sx[i] = C.S[0][i];
  for (int i = threadIdx.x; i < Gy * Gy; i += blockDim.x) Sy[i] = C.S[1][i];
  for (int g = threadIdx.x; g < plane; g += blockDim.x)
    A[g] = __ldg(f0 + coarse_elem_index(nx, ny, g % Gx, g / Gx, Z));
  __syncthreads();
  for (int g = threadIdx.x; g < plane; g += blockDim.x) {
    const int o = g % Gx;
    const double *row = A + (g - o);
    double acc = 0;
    for (int k = 0; k < Gx; ++k) acc += Sx[k * Gx + o] * row[k];
    B[g] = acc;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < plane; g += blockDim.x) {
    const int a = g % Gx, o = g / Gx;
    double acc = 0;
    for (int k = 0; k < Gy; ++k) acc += Sy[k * Gy + o] * B[a + k * Gx];
    G[g + (long long)plane * Z] = acc;
  }
}

__global__ void __launch_bounds__(1024) k_coarse_zcols(CoarseDev C, double *__restrict__ G) {
  extern __shared__ double sm[];
  const int Gx = C.G[0], Gy = C.G[1], Gz = C.G[2];
  const int cols = Gx * Gy;
  double *Sz = sm, *SzT = Sz + Gz * Gz, *lz = SzT + Gz * Gz;
  for (int i = threadIdx.x; i < Gz * Gz; i += blockDim.x) {
    const double v = C.S[2][i];
    Sz[i] = v;
    SzT[(i % Gz) * Gz + i / Gz] = v;
  }
  for (int i = threadIdx.x; i < Gz; i += blockDim.x) lz[i] = C.lam[2][i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool zl = lane < Gz;
  // issue the column loads before waiting for the tables
  const int c0 = blockIdx.x * nw + warp;
  const double v0 = (zl && c0 < cols) ? G[c0 + (long long)lane * cols] : 0.0;
  __syncthreads();
  for (int cidx = c0; cidx < cols; cidx += gridDim.x * nw) {
    const int a = cidx % Gx, b = cidx / Gx;
    const double v = cidx == c0 ? v0 : (zl ? G[cidx + (long long)lane * cols] : 0.0);
    double acc = 0.0;
    for (int k = 0; k < Gz; ++k) {
      const double vk = __shfl_sync(0xffffffffu, v, k);
      if (zl) acc += Sz[k * Gz + lane] * vk;
    }
    double w = 0.0;
    if (zl && !(a == 0 && b == 0 && lane == 0)) w = acc / (C.lam[0][a] + C.lam[1][b] + lz[lane]);
    double out = 0.0;
    for (int k = 0; k < Gz; ++k) {
      const double wk = __shfl_sync(0xffffffffu, w, k);
      if (zl) out += SzT[k * Gz + lane] * wk;
    }
    if (zl) G[cidx + (long long)lane * cols] = out;
  }
}

__global__ void __launch_bounds__(1024) k_coarse_plane_bwd(CoarseDev C, int nx, int ny,
                                                          const double *__restrict__ G,
                                                          double *__restrict__ u0) {
  extern __shared__ double sm[];
  const int Gx = C.G[0], Gy = C.G[1], plane = Gx * Gy, Z = blockIdx.x;
  double *A = sm, *B = A + plane, *SxT = B + plane, *Sy = SxT + Gx * Gx;
  for (int i = threadIdx.x; i < Gx * Gx; i += blockDim.x) SxT[(i % Gx) * Gx + i / Gx] = C.S[0][i];
  for (int i = threadIdx.x; i < Gy * Gy; i += blockDim.x) Sy[i] = C.S[1][i];
  for (int g = threadIdx.x; g < plane; g += blockDim.x) A[g] = G[g + (long long)plane * Z];
  __syncthreads();
  for (int g = threadIdx.x; g < plane; g += blockDim.x) {           // y backward (Y uniform per warp row)
    const int a = g % Gx, Y = g / Gx;
    double acc = 0;
    for (int k = 0; k < Gy; ++k) acc += Sy[Y * Gy + k] * A[a + k * Gx];
    B[g] = acc;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < plane; g += blockDim.x) {           // x backward -> element-major u_0
    const int X = g % Gx, Y = g / Gx;
    const double *row = B + (g - X);
    double acc = 0;
    for (int k = 0; k < Gx; ++k) acc += SxT[k * Gx + X] * row[k];
    u0[coarse_elem_index(nx, ny, X, Y, Z)] = acc;
  }
}

// x-backward pass writing u_0 in element-major order
__global__ void k_coarse_xb(CoarseDev C, int nx, int ny, const double *__restrict__ G,
                            double *__restrict__ u0) {
  const int Gx = C.G[0], Gy = C.G[1];
  const long long N = (long long)Gx * Gy * C.G[2];
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N;
       g += (long long)gridDim.x * blockDim.x) {
    const int X = g % Gx, Y = (g / Gx) % Gy, Z = g / ((long long)Gx * Gy);
    const double *row = G + (g - X);
    double acc = 0;
    for (int k = 0; k < Gx; ++k) acc += C.S[0][X * Gx + k] * row[k];
    u0[coarse_elem_index(nx, ny, X, Y, Z)] = acc;
  }
}

// ---------------------------------------------------------------------------------------------
// Deterministic reductions: fixed grid for a given N, fixed per-thread order, fixed tree.
constexpr int RB = 256;
constexpr int RMAX = 1184;   // 8 x 148 SMs

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[RB / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < RB / 32 ? sh[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  }
  __syncthreads();
  return v;   // valid in thread 0
}

template <int MODE>
__global__ void k_partial(const double *__restrict__ x, const double *__restrict__ y,
                          const double *__restrict__ z, long long N, double *__restrict__ part) {
  // MODE 0: sum x;  1: x.y;  2: (x.(y - z), x.y) two outputs
  double a = 0, b = 0;
  for (long long g = blockIdx.x * (long long)RB + threadIdx.x; g < N; g += (long long)gridDim.x * RB) {
    if (MODE == 0) a += x[g];
    else if (MODE == 1) a += x[g] * y[g];
    else { a += x[g] * (y[g] - z[g]); b += x[g] * y[g]; }
  }
  a = block_sum(a);
  if (MODE == 2) b = block_sum(b);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = a;
    if (MODE == 2) part[gridDim.x + blockIdx.x] = b;
  }
}

// final stage: op 0 -> out[0] = scale * sum; op 1 -> pq & alpha; op 2 -> zr / beta
__global__ void k_final(const double *__restrict__ part, int nb, int nout, double *__restrict__ out,
                        double scale, int op) {
  double a = 0, b = 0;
  for (int i = threadIdx.x; i < nb; i += RB) {
    a += part[i];
    if (nout == 2) b += part[nb + i];
  }
  a = block_sum(a);
  if (nout == 2) b = block_sum(b);
  if (threadIdx.x == 0) {
    if (op == 0) out[0] = scale * a;
    else if (op == 1) { out[1] = a; out[5] = out[0] / a; }                 // pq, alpha = zr/pq
    else if (op == 2) { out[3] = a; out[4] = b; out[6] = a / out[0]; out[0] = b; }  // beta
    else if (op == 3) { out[0] = b; }                                        // first zr
  }
}

__global__ void k_sub_scalar(double *__restrict__ v, long long N, const double *__restrict__ c) {
  const double s = *c;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N;
       g += (long long)gridDim.x * blockDim.x)
    v[g] -= s;
}

__global__ void k_copy(double *__restrict__ d, const double *__restrict__ s, long long N) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N;
       g += (long long)gridDim.x * blockDim.x)
    d[g] = s ? s[g] : 0.0;
}

// y = a x + b y with host scalars (b == 0: y = a x without reading y): the vector updates of a
// Krylov loop driven from the host (slab-decomposed PCG, whose scalars are all-reduced first)
__global__ void k_axpby(double *__restrict__ y, double a, const double *__restrict__ x, double b, long long N) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N;
       g += (long long)gridDim.x * blockDim.x)
    y[g] = b == 0.0 ? (a == 0.0 ? 0.0 : a * x[g]) : fma(a, x[g], b * y[g]);   // a = b = 0: y = 0 exactly
}

__global__ void k_cg_update(double *__restrict__ u, double *__restrict__ r, double *__restrict__ rold,
                            const double *__restrict__ p, const double *__restrict__ q, long long N,
                            double *__restrict__ part, const double *__restrict__ scal) {
  const double alpha = scal[5];
  double a = 0;
  for (long long g = blockIdx.x * (long long)RB + threadIdx.x; g < N; g += (long long)gridDim.x * RB) {
    u[g] += alpha * p[g];
    const double ro = r[g];
    rold[g] = ro;
    const double rn = ro - alpha * q[g];
    r[g] = rn;
    a += rn * rn;
  }
  a = block_sum(a);
  if (threadIdx.x == 0) part[blockIdx.x] = a;
}

__global__ void k_p_update(double *__restrict__ p, const double *__restrict__ z, long long N,
                           const double *__restrict__ scal) {
  const double beta = scal[6];
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N;
       g += (long long)gridDim.x * blockDim.x)
    p[g] = z[g] + beta * p[g];
}

// Device-side control of the graph-driven PCG (same tests as the host loop:
// diverged = non-finite or ||r|| > 1e3 ||r_0||, converged = ||r|| <= rtol ||r_0||, else maxit).
// Status codes mirror include/pmg_dg.h (PMG_EDIVERGED = 6, PMG_EMAXIT = 7); -1 = running.
__global__ void k_pcg_start(double *scal, double *hist, int maxit, cudaGraphConditionalHandle hw) {
  const double r0 = sqrt(scal[2]);
  scal[30] = r0;
  scal[31] = 0.0;
  hist[0] = r0;
  const int status = !isfinite(r0) ? 6 : (r0 == 0.0 ? 0 : (maxit == 0 ? 7 : -1));
  scal[32] = status;
  cudaGraphSetConditional(hw, status == -1 ? 1u : 0u);
}

__global__ void k_pcg_check(double *scal, double *hist, double rtol, int maxit,
                            cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hi) {
  const double rn = sqrt(scal[2]), r0 = scal[30];
  const int k = (int)scal[31] + 1;
  scal[31] = k;
  hist[k] = rn;
  int status = -1;
  if (!isfinite(rn) || rn > 1e3 * r0) status = 6;
  else if (rn <= rtol * r0) status = 0;
  else if (k >= maxit) status = 7;
  scal[32] = status;
  const unsigned cont = status == -1 ? 1u : 0u;
  cudaGraphSetConditional(hw, cont);
  cudaGraphSetConditional(hi, cont);
}

// b = M * amp * sin(kx x) sin(ky y) sin(kz z) at the nodes (diagonal quadrature)
__global__ void k_rhs_sin(LevelDev L, double dx, double dy, double dz, double amp, double kx,
                          double ky, double kz, double *__restrict__ b) {
  const int n = L.n, n3 = n * n * n;
  const long long N = (long long)L.Ne * n3;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N;
       g += (long long)gridDim.x * blockDim.x) {
    const long long e = g / n3;
    const int t = g - e * n3;
    const int i = t % n, j = (t / n) % n, k = t / (n * n);
    const int ex = e % L.nx, ey = (e / L.nx) % L.ny, ez = e / ((long long)L.nx * L.ny);
    const double x = (ex + 0.5 * (L.nodes[i] + 1.0)) * dx;
    const double y = (ey + 0.5 * (L.nodes[j] + 1.0)) * dy;
    const double z = (ez + 0.5 * (L.nodes[k] + 1.0)) * dz;
    b[g] = L.mass[0][i] * L.mass[1][j] * L.mass[2][k] * amp * sin(kx * x) * sin(ky * y) * sin(kz * z);
  }
}


}  // namespace

#ifndef PMG_FOLD_SPLIT_MIN_N
#define PMG_FOLD_SPLIT_MIN_N 17
#endif
// kernels launch_fold issues: 2 when the trace pass runs as its own launch (n >= 17, full grids)
static bool fold_splits_traces(const LevelDev &L) {
  return L.n >= PMG_FOLD_SPLIT_MIN_N && L.n <= 20 && L.Ne > 4 * num_sms();
}
int fold_launches(const LevelDev &L, bool traces) { return traces && fold_splits_traces(L) ? 2 : 1; }

cudaError_t launch_fold(const LevelDev &L, const double *Z, double *u, bool zero, double *T,
                        cudaStream_t s) {
  // n >= 17 on full grids: the fold WITHOUT its fused trace phase plus the standalone trace kernel
  // is faster than the fused form (c3: 0.152 + 0.047 against 0.221 ms — the trace phase is bound by
  // shared-memory wavefronts and issue slots, and at the tail of every fold CTA it does not hide
  // under the other CTAs' loads, which are issue-bound themselves: 65 % issue utilisation)
  if (T && fold_splits_traces(L)) {
    cudaError_t e = launch_fold(L, Z, u, zero, nullptr, s);
    return e ? e : launch_traces(L, u, T, s);
  }
  const int z = zero ? 1 : 0;
  const size_t sb = T ? sizeof(double) * ((size_t)L.n * L.n * L.n + 12 * L.n) : 0;
  if (T && sb > 48 * 1024) {
    static bool cfg = false;
    if (!cfg) {
      cfg = true;
      cudaFuncSetAttribute(k_fold2<17, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_fold2<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
  }
#define PMG_FOLD(NN)                                                                          \
  if (T) k_fold2<NN, true><<<L.Ne, 256, sb, s>>>(L, Z, u, z, T);                             \
  else k_fold2<NN, false><<<L.Ne, 256, 0, s>>>(L, Z, u, z, nullptr);
  if (L.n == 3 || L.n == 5) {                 // several small elements per CTA, traces fused
    const int z0 = zero ? 1 : 0;
    if (L.n == 3) {
      const int g = (L.Ne + 8) / 9;
      if (T) k_fold_small<3, 9, true><<<g, 256, 0, s>>>(L, Z, u, z0, T);
      else k_fold_small<3, 9, false><<<g, 256, 0, s>>>(L, Z, u, z0, nullptr);
    } else {
      const int g = (L.Ne + 1) / 2;
      if (T) k_fold_small<5, 2, true><<<g, 256, 0, s>>>(L, Z, u, z0, T);
      else k_fold_small<5, 2, false><<<g, 256, 0, s>>>(L, Z, u, z0, nullptr);
    }
    return cudaGetLastError();
  }
#ifndef PMG_FOLD2
  if (L.m[0] <= 32 && L.n >= 9 && sizeof(double) * ((size_t)L.n * L.n * L.n + 12 * L.n) <= 160 * 1024 &&
      (long long)L.Ne * L.Mw < (1LL << 31)) {
    // row fold (k_fold4): window rows fit a warp, the element fits shared memory for the traces
    const int n = L.n;
    const bool merged = 2 * L.no[0] <= n && 2 * L.no[1] <= n && 2 * L.no[2] <= n;
    const size_t sb4 = T ? sizeof(double) * ((size_t)n * n * n + 1 + 3 * trace_tab_len(n) + 1) : 0;
#define PMG_FOLD4(NN, MM)                                                                       \
  do {                                                                                          \
    static bool cfg4 = false;                                                                   \
    if (!cfg4) {                                                                                \
      cfg4 = true;                                                                              \
      cudaFuncSetAttribute(k_fold4<NN, true, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
    }                                                                                           \
    if (T) k_fold4<NN, true, MM><<<L.Ne, 256, sb4, s>>>(L, Z, u, z, T);                         \
    else k_fold4<NN, false, MM><<<L.Ne, 256, 0, s>>>(L, Z, u, z, nullptr);                      \
  } while (0)
    if (n == 17 && merged) PMG_FOLD4(17, true);
    else if (n == 9 && merged) PMG_FOLD4(9, true);
    else if (n == 9) PMG_FOLD4(9, false);
    else if (merged) PMG_FOLD4(0, true);
    else PMG_FOLD4(0, false);
#undef PMG_FOLD4
    return cudaGetLastError();
  }
#endif
  if (T && (sb > 200 * 1024 || L.n < 9)) {   // n = 33: no room; n < 9: separate kernels are faster
    if (L.n == 33) k_fold2<33, false><<<dim3(L.Ne, 36), 256, 0, s>>>(L, Z, u, z, nullptr);
    else if (L.n == 5) k_fold2<5, false><<<L.Ne, 256, 0, s>>>(L, Z, u, z, nullptr);
    else if (L.n == 3) k_fold2<3, false><<<L.Ne, 256, 0, s>>>(L, Z, u, z, nullptr);
    else k_fold2<0, false><<<L.Ne, 256, 0, s>>>(L, Z, u, z, nullptr);
    cudaError_t e0 = cudaGetLastError();
    if (e0 == cudaSuccess) e0 = launch_traces(L, u, T, s);
    return e0;
  }
  switch (L.n) {
    case 3: PMG_FOLD(3) break;
    case 5: PMG_FOLD(5) break;
    case 9: PMG_FOLD(9) break;
    case 17: PMG_FOLD(17) break;
    case 33:
      if (T) k_fold2<33, true><<<L.Ne, 256, sb, s>>>(L, Z, u, z, T);
      else k_fold2<33, false><<<dim3(L.Ne, 36), 256, 0, s>>>(L, Z, u, z, nullptr);
      break;
    default: PMG_FOLD(0) break;
  }
#undef PMG_FOLD
  cudaError_t e = cudaGetLastError();
  return e;
}
cudaError_t launch_coarse_gather(const LevelDev &L0, const CoarseDev &C, const double *f0,
                                 const double *mean, double *G, cudaStream_t s) {
  k_coarse_gather<<<grid_for(8LL * L0.Ne, 256), 256, 0, s>>>(L0.nx, L0.ny, L0.nz, f0, mean, G);
  return cudaGetLastError();
}
cudaError_t launch_lex_contract(const CoarseDev &C, int axis, bool forward, const double *in,
                                double *out, cudaStream_t s) {
  const long long N = (long long)C.G[0] * C.G[1] * C.G[2];
  k_lex_contract<<<grid_for(N, 256), 256, 0, s>>>(C, axis, forward ? 1 : 0, in, out);
  return cudaGetLastError();
}
bool coarse_one_ok(const CoarseDev &C) {
  return (long long)C.G[0] * C.G[1] * C.G[2] <= 1024 && C.G[0] <= 32 && C.G[1] <= 32 && C.G[2] <= 32;
}

cudaError_t launch_coarse_one(const LevelDev &L0, const CoarseDev &C, const double *f0, double *u0,
                              cudaStream_t s) {
  const int N = C.G[0] * C.G[1] * C.G[2];
  const size_t sb = sizeof(double) * (2 * (size_t)N + C.G[0] * C.G[0] + C.G[1] * C.G[1] +
                                      C.G[2] * C.G[2] + C.G[0] + C.G[1] + C.G[2]);
  static bool cfg = false;
  if (!cfg) {
    cfg = true;
    cudaFuncSetAttribute(k_coarse_one, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  }
  k_coarse_one<<<1, 1024, sb, s>>>(C, L0.nx, L0.ny, f0, u0);
  return cudaGetLastError();
}

bool coarse_cluster_ok(const CoarseDev &C) {
#ifdef PMG_NO_COARSE_CLUSTER
  return false;
#endif
  // measured: 16^3 (c2) 36 -> 17 us per solve; at 32^3 (c3, c5) eight SMs are LSU-bound (72 us
  // against 66 us for the five-launch path over the whole GPU), so the cluster serves N_0 <= 8192
  return C.G[0] <= 32 && C.G[1] <= 32 && C.G[2] <= 32 && C.G[2] >= 8 &&
         (long long)C.G[0] * C.G[1] * C.G[2] <= 8192;
}

cudaError_t launch_coarse_cluster(const LevelDev &L0, const CoarseDev &C, const double *f0,
                                  double *u0, cudaStream_t s) {
  constexpr int CS = 8;
  const int plane = C.G[0] * C.G[1], pp = (C.G[2] + CS - 1) / CS;
  const size_t sb = sizeof(double) * (2 * (size_t)pp * plane + 2 * C.G[0] * C.G[0] + C.G[1] * C.G[1] +
                                      2 * C.G[2] * C.G[2] + C.G[0] + C.G[1] + C.G[2]);
  static bool cfg = false;
  if (!cfg) {
    cfg = true;
    cudaFuncSetAttribute(k_coarse_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(CS);
  lc.blockDim = dim3(512);
  lc.dynamicSmemBytes = sb;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, k_coarse_cluster, C, L0.nx, L0.ny, f0, u0);
}

cudaError_t launch_coarse_fused(const LevelDev &L0, const CoarseDev &C, const double *f0,
                                double *G1, double *G2, double *u0, cudaStream_t s) {
  const long long N = (long long)C.G[0] * C.G[1] * C.G[2];
  const long long cols = (long long)C.G[0] * C.G[1];
  if (C.G[2] > 32) return cudaErrorInvalidValue;
#ifndef PMG_COARSE5
  if (C.G[0] <= 32 && C.G[1] <= 32) {      // three plane / column launches (G1 only)
    const int plane = C.G[0] * C.G[1];
    const int th = std::min(1024, ((plane + 31) / 32) * 32);
    const size_t sp = sizeof(double) * (2 * (size_t)plane + C.G[0] * C.G[0] + C.G[1] * C.G[1]);
    const size_t sz = sizeof(double) * (2 * (size_t)C.G[2] * C.G[2] + C.G[2]);
    static bool cfg = false;
    if (!cfg) {
      cfg = true;
      cudaFuncSetAttribute(k_coarse_plane_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      cudaFuncSetAttribute(k_coarse_plane_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      cudaFuncSetAttribute(k_coarse_zcols, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    }
    k_coarse_plane_fwd<<<C.G[2], th, sp, s>>>(C, L0.nx, L0.ny, f0, G1);
    k_coarse_zcols<<<(int)((cols + 31) / 32), 1024, sz, s>>>(C, G1);
    k_coarse_plane_bwd<<<C.G[2], th, sp, s>>>(C, L0.nx, L0.ny, G1, u0);
    return cudaGetLastError();
  }
#endif
  k_coarse_xf<<<grid_for(N, 256), 256, 0, s>>>(C, L0.nx, L0.ny, f0, G1);
  k_lex_contract<<<grid_for(N, 256), 256, 0, s>>>(C, 1, 1, G1, G2);
  k_coarse_z<<<grid_for(cols * 32, 256), 256, 0, s>>>(C, G2);
  k_lex_contract<<<grid_for(N, 256), 256, 0, s>>>(C, 1, 0, G2, G1);
  k_coarse_xb<<<grid_for(N, 256), 256, 0, s>>>(C, L0.nx, L0.ny, G1, u0);
  return cudaGetLastError();
}

// kernels launched by launch_coarse_fused (for the launch counter)
int coarse_fused_launches(const CoarseDev &C) {
#ifndef PMG_COARSE5
  if (C.G[0] <= 32 && C.G[1] <= 32) return 3;
#endif
  return 5;
}

cudaError_t launch_coarse_divide(const CoarseDev &C, double *G, cudaStream_t s) {
  const long long N = (long long)C.G[0] * C.G[1] * C.G[2];
  k_coarse_divide<<<grid_for(N, 256), 256, 0, s>>>(C, G);
  return cudaGetLastError();
}
cudaError_t launch_coarse_scatter(const LevelDev &L0, const CoarseDev &C, const double *G,
                                  const double *mean, double *u0, cudaStream_t s) {
  k_coarse_scatter<<<grid_for(8LL * L0.Ne, 256), 256, 0, s>>>(L0.nx, L0.ny, L0.nz, G, mean, u0);
  return cudaGetLastError();
}
int reduce_blocks(long long N) {
  long long b = (N + 4 * RB - 1) / (4 * RB);
  if (b > RMAX) b = RMAX;
  if (b < 1) b = 1;
  return (int)b;
}
cudaError_t launch_sum(const double *x, long long N, double *partial, double *out, double scale,
                       cudaStream_t s) {
  const int nb = reduce_blocks(N);
  k_partial<0><<<nb, RB, 0, s>>>(x, nullptr, nullptr, N, partial);
  k_final<<<1, RB, 0, s>>>(partial, nb, 1, out, scale, 0);
  return cudaGetLastError();
}
cudaError_t launch_dot(const double *x, const double *y, long long N, double *partial,
                       double *out, cudaStream_t s) {
  const int nb = reduce_blocks(N);
  k_partial<1><<<nb, RB, 0, s>>>(x, y, nullptr, N, partial);
  k_final<<<1, RB, 0, s>>>(partial, nb, 1, out, 1.0, 0);
  return cudaGetLastError();
}
cudaError_t launch_sub_scalar(double *v, long long N, const double *c, cudaStream_t s) {
  k_sub_scalar<<<grid_for(N, 256), 256, 0, s>>>(v, N, c);
  return cudaGetLastError();
}
cudaError_t launch_copy(double *dst, const double *src, long long N, cudaStream_t s) {
  k_copy<<<grid_for(N, 256), 256, 0, s>>>(dst, src, N);
  return cudaGetLastError();
}
cudaError_t launch_zero(double *dst, long long N, cudaStream_t s) { return launch_copy(dst, nullptr, N, s); }
cudaError_t launch_axpby(double *y, double a, const double *x, double b, long long N, cudaStream_t s) {
  k_axpby<<<grid_for(N, 256), 256, 0, s>>>(y, a, x, b, N);
  return cudaGetLastError();
}
cudaError_t launch_pq_alpha(const double *p, const double *q, long long N, double *partial,
                            double *scal, cudaStream_t s) {
  const int nb = reduce_blocks(N);
  k_partial<1><<<nb, RB, 0, s>>>(p, q, nullptr, N, partial);
  k_final<<<1, RB, 0, s>>>(partial, nb, 1, scal, 1.0, 1);
  return cudaGetLastError();
}
cudaError_t launch_cg_update(double *u, double *r, double *rold, const double *p,
                             const double *q, long long N, double *partial, double *scal,
                             cudaStream_t s) {
  const int nb = reduce_blocks(N);
  k_cg_update<<<nb, RB, 0, s>>>(u, r, rold, p, q, N, partial, scal);
  k_final<<<1, RB, 0, s>>>(partial, nb, 1, scal + 2, 1.0, 0);
  return cudaGetLastError();
}
cudaError_t launch_zr_beta(const double *z, const double *r, const double *rold, long long N,
                           double *partial, double *scal, bool first, cudaStream_t s) {
  const int nb = reduce_blocks(N);
  k_partial<2><<<nb, RB, 0, s>>>(z, r, rold, N, partial);
  k_final<<<1, RB, 0, s>>>(partial, nb, 2, scal, 1.0, first ? 3 : 2);
  return cudaGetLastError();
}
cudaError_t launch_p_update(double *p, const double *z, long long N, const double *scal,
                            cudaStream_t s) {
  k_p_update<<<grid_for(N, 256), 256, 0, s>>>(p, z, N, scal);
  return cudaGetLastError();
}
cudaError_t launch_pcg_start(double *scal, double *hist, int maxit, cudaGraphConditionalHandle hw,
                             cudaStream_t s) {
  k_pcg_start<<<1, 1, 0, s>>>(scal, hist, maxit, hw);
  return cudaGetLastError();
}
cudaError_t launch_pcg_check(double *scal, double *hist, double rtol, int maxit,
                             cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hi, cudaStream_t s) {
  k_pcg_check<<<1, 1, 0, s>>>(scal, hist, rtol, maxit, hw, hi);
  return cudaGetLastError();
}
cudaError_t launch_rhs_sin(const LevelDev &L, double dx, double dy, double dz, double amp,
                           double kx, double ky, double kz, double *b, cudaStream_t s) {
  k_rhs_sin<<<grid_for((long long)L.Ne * L.n * L.n * L.n, 256), 256, 0, s>>>(L, dx, dy, dz, amp,
                                                                             kx, ky, kz, b);
  return cudaGetLastError();
}

}  // namespace pmg
