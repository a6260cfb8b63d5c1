// Schwarz subdomain solves (fast diagonalisation, even/odd split) specialised at compile time
// for the window shapes of the benchmark configurations.  arXiv:1612.04796
// (Eq. 9 subdomain problem, the fast-diagonalisation formula, Eq. 10 weighted scatter).
//
// Same method as k_fdm_eo in kern_fdm.cu (see the comment there for the even/odd algebra); with
// every extent and stride a compile-time constant the tile loops carry no runtime index
// arithmetic beyond the lane's own column, the A fragments stay in registers for a whole pass,
// and the B fragments need no selects:
//   forward:  b_E = x_k + x_{m-1-k}, b_O = x_k - x_{m-1-k} with k clamped to H; the middle
//             column of S_E^T is halved (x_H + x_H = 2 x_H exactly), padding columns are zero;
//   backward: b_E = t_E[min(k, H)], b_O = t_O[min(k, H-1)] against zero-padded S_E, S_O.
#include <algorithm>

#include "kcommon.cuh"

namespace pmg {
namespace {

__host__ __device__ constexpr int plane_stride(int m0, int m1) {
  return m0 * m1 + ((4 - ((m0 * m1) & 15)) & 15);   // 4 mod 16 doubles: bank spread
}

// WIDE: 256 threads for small windows too — used when the whole grid fits in one wave (small
// meshes, e.g. c2's 512 subdomains), where a CTA's latency, not the SM's throughput, sets the time.
template <int M0, int M1, int M2, bool WIDE = false, int TH = 0>
struct Shape {
  static constexpr int S2 = plane_stride(M0, M1);
  static constexpr int Hmax = (M0 > M1 ? (M0 > M2 ? M0 : M2) : (M1 > M2 ? M1 : M2)) / 2;
#ifdef PMG_EOC_THREADS23      // diagnostic: CTA width of the 23^3 kernel (e.g. 352 = 11 warps, 66 tiles / 11)
  static constexpr int THREADS = TH ? TH : ((M0 == 23 && M1 == 23 && M2 == 23) ? PMG_EOC_THREADS23 : ((Hmax >= 8 || WIDE) ? 256 : 128));
#else
  static constexpr int THREADS = TH ? TH : ((Hmax >= 8 || WIDE) ? 256 : 128);
#endif
  static constexpr int MINB = Hmax >= 8 ? 2 : (WIDE ? 4 : 8);
  static constexpr int NWS = THREADS / 32;                    // warps per subdomain
  __device__ static __forceinline__ int wid() { return (int)(threadIdx.x >> 5); }
  template <int D> __host__ __device__ static constexpr int m() { return D == 0 ? M0 : (D == 1 ? M1 : M2); }
  template <int D> __host__ __device__ static constexpr int s() { return D == 0 ? 1 : (D == 1 ? M0 : S2); }
};

// PIPE (x forward pass only): the warp's own tiles were gathered by the warp itself in two cp.async
// groups (its first two tiles | the rest); it waits for them here instead of at a block barrier
template <int DIR, class SH, bool FWD, bool QF, class Epi, bool PIPE = false>
__device__ __forceinline__ void eoc_lines(const double *X, const double *S, Epi &epi) {
  constexpr int PD = Other<DIR>::P, QD = Other<DIR>::Q;
  constexpr int m = SH::template m<DIR>(), H = m / 2;
  constexpr int MT = (H + 1 + 7) / 8, KS = (H + 1 + 3) / 4;
  constexpr int MP = SH::template m<PD>(), MQ = SH::template m<QD>();
  constexpr int SO = SH::template s<DIR>(), SP = SH::template s<PD>(), SQ = SH::template s<QD>();
  constexpr int NCOL = MP * MQ, NT = (NCOL + 7) / 8;
  const int lane = threadIdx.x & 31, warp = SH::wid();
  constexpr int NW = SH::NWS;
  const int g = lane >> 2, t = lane & 3;
  if (warp >= NT) return;
  double aE[MT][KS], aO[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int o = mt * 8 + g, k = ks * 4 + t;
      if (FWD) {
        aE[mt][ks] = (o <= H && k <= H) ? S[k * m + o] * (k == H ? 0.5 : 1.0) : 0.0;
        aO[mt][ks] = (o < H && k < H) ? S[k * m + H + 1 + o] : 0.0;
      } else {
        aE[mt][ks] = (o <= H && k <= H) ? S[o * m + k] : 0.0;
        aO[mt][ks] = (o < H && k < H) ? S[o * m + H + 1 + k] : 0.0;
      }
    }
  int off1[KS], off2[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = ks * 4 + t;
    if (FWD) {
      const int kl = min(k, H);
      off1[ks] = kl * SO; off2[ks] = (m - 1 - kl) * SO;
    } else {
      off1[ks] = min(k, H) * SO; off2[ks] = (H + 1 + min(k, H - 1)) * SO;
    }
  }
  // Column bookkeeping without per-tile divisions: a lane tracks (p, q) of its B column and of
  // its two C columns and steps them by the 8 NW columns between its tiles (the div/mod by a
  // constant cost ~15 integer instructions per column and tile in 16-bit emulation).
  struct Col { int p, q; };
  auto col_init = [](int n, Col &c) {
    if (QF) { c.p = n / MQ; c.q = n - c.p * MQ; } else { c.q = n / MP; c.p = n - c.q * MP; }
  };
  constexpr int STEP = 8 * NW;
  auto col_adv = [](Col &c) {
    if (QF) { c.q += STEP % MQ; c.p += STEP / MQ; if (c.q >= MQ) { c.q -= MQ; ++c.p; } }
    else { c.p += STEP % MP; c.q += STEP / MP; if (c.p >= MP) { c.p -= MP; ++c.q; } }
  };
  auto col_ok = [](const Col &c) { return QF ? c.p < MP : c.q < MQ; };
  // Tile-column permutation pi = [0 1 2 3 5 4 7 6]: lane g loads column pi(g), C column index c
  // is window column pi(c).  Consecutive columns are 4 double-banks apart (plane stride 4 mod 16,
  // z fastest), so the B loads need pi(g) mod 4 distinct over each half-warp's four g and the C
  // stores need pi(2t + j) mod 4 distinct over t: the identity order made the stores of lanes
  // (g, t) and (g, t + 2) collide (ncu: 31 % of the kernel's shared-memory wavefronts).
  // Measured: 13^3 windows 0.193 -> 0.185 ms per cycle (that kernel keeps the shared-memory pipe
  // ~70 % busy), c5's shapes -0.4 %; neutral to +0.3 % on 23^3 (1.2275 -> 1.2314: the stores are not
  // its limiter), which keeps the identity order.
  constexpr bool PERM = !(SH::template m<0>() == 23 && SH::template m<1>() == 23 && SH::template m<2>() == 23);
  auto pi = [](int c) { return PERM ? (c ^ ((c >> 2) & 1)) : c; };
  Col cb, c0, c1;
  col_init(warp * 8 + pi(g), cb);
  col_init(warp * 8 + pi(2 * t), c0);
  col_init(warp * 8 + pi(2 * t + 1), c1);
  auto compute = [&](double (&cE)[MT][2], double (&cO)[MT][2]) {
    const double *xb = X + (col_ok(cb) ? cb.p * SP + cb.q * SQ : (MP - 1) * SP + (MQ - 1) * SQ);
    col_adv(cb);
    double bE[KS], bO[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const double v1 = xb[off1[ks]], v2 = xb[off2[ks]];
      if (FWD) { bE[ks] = v1 + v2; bO[ks] = v1 - v2; }
      else { bE[ks] = v1; bO[ks] = v2; }
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
  auto epilogue = [&](const double (&cE)[MT][2], const double (&cO)[MT][2]) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const Col c = j ? c1 : c0;
      if (!col_ok(c)) continue;
      const int p = c.p, q = c.q;
      const double cf = epi.template col<DIR>(p, q);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int o = mt * 8 + g;
        if (FWD) {
          if (o <= H) epi.template put<DIR>(o, p, q, cf, cE[mt][j]);
          if (o < H) epi.template put<DIR>(H + 1 + o, p, q, cf, cO[mt][j]);
        } else if (o < H) {
          epi.template put<DIR>(o, p, q, cf, cE[mt][j] + cO[mt][j]);
          epi.template put<DIR>(m - 1 - o, p, q, cf, cE[mt][j] - cO[mt][j]);
        } else if (o == H) {
          epi.template put<DIR>(o, p, q, cf, cE[mt][j]);
        }
      }
    }
    col_adv(c0);
    col_adv(c1);
  };
  double cE0[MT][2], cO0[MT][2], cE1[MT][2], cO1[MT][2];
#ifdef PMG_EOC_PAIRED
  // two tiles per step in one instruction stream (8 accumulator chains), no cross-step pipelining
  auto loadB = [&](double (&bE)[KS], double (&bO)[KS]) {
    const double *xb = X + (col_ok(cb) ? cb.p * SP + cb.q * SQ : (MP - 1) * SP + (MQ - 1) * SQ);
    col_adv(cb);
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const double v1 = xb[off1[ks]], v2 = xb[off2[ks]];
      if (FWD) { bE[ks] = v1 + v2; bO[ks] = v1 - v2; }
      else { bE[ks] = v1; bO[ks] = v2; }
    }
  };
  for (int tile = warp; tile < NT; tile += 2 * NW) {
    if (tile + NW < NT) {
      double bE0[KS], bO0[KS], bE1[KS], bO1[KS];
      loadB(bE0, bO0);
      loadB(bE1, bO1);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        cE0[mt][0] = cE0[mt][1] = cO0[mt][0] = cO0[mt][1] = 0.0;
        cE1[mt][0] = cE1[mt][1] = cO1[mt][0] = cO1[mt][1] = 0.0;
      }
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          dmma884(cE0[mt][0], cE0[mt][1], aE[mt][ks], bE0[ks]);
          dmma884(cO0[mt][0], cO0[mt][1], aO[mt][ks], bO0[ks]);
          dmma884(cE1[mt][0], cE1[mt][1], aE[mt][ks], bE1[ks]);
          dmma884(cO1[mt][0], cO1[mt][1], aO[mt][ks], bO1[ks]);
        }
      __syncwarp();
      epilogue(cE0, cO0);
      epilogue(cE1, cO1);
    } else {
      compute(cE0, cO0);
      __syncwarp();
      epilogue(cE0, cO0);
    }
  }
#else
  int tile = warp;
  if (PIPE) { cp_async_wait<1>(); __syncwarp(); }
  compute(cE0, cO0);
  for (;;) {
    const int t1 = tile + NW;
    if (t1 < NT) compute(cE1, cO1);
    __syncwarp();
    epilogue(cE0, cO0);
    if (t1 >= NT) break;
    const int t2 = t1 + NW;
    if (PIPE) { cp_async_wait<0>(); __syncwarp(); }
    if (t2 < NT) compute(cE0, cO0);
    __syncwarp();
    epilogue(cE1, cO1);
    if (t2 >= NT) break;
    tile = t2;
  }
#endif
}

// z passes fused: forward S_z^T, eigen-divide, backward S_z on warp-private z columns
template <class SH>
__device__ __forceinline__ void eoc_z_fused(double *X, const double *S, const double *const *lam,
                                            const double *__restrict__ Rz) {
  constexpr int m = SH::template m<2>(), H = m / 2;
  constexpr int MT = (H + 1 + 7) / 8, KS = (H + 1 + 3) / 4;
  constexpr int MP = SH::template m<0>(), MQ = SH::template m<1>();
  constexpr int SO = SH::S2, SQ = SH::template s<1>();
  constexpr int NCOL = MP * MQ, NT = (NCOL + 7) / 8, NW = SH::NWS;
  const int lane = threadIdx.x & 31, warp = SH::wid();
  const int g = lane >> 2, t = lane & 3;
  double aEf[MT][KS], aOf[MT][KS], aEb[MT][KS], aOb[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int o = mt * 8 + g, k = ks * 4 + t;
      const bool e_ok = o <= H && k <= H, o_ok = o < H && k < H;
      aEf[mt][ks] = e_ok ? S[k * m + o] * (k == H ? 0.5 : 1.0) : 0.0;
      aOf[mt][ks] = o_ok ? S[k * m + H + 1 + o] : 0.0;
      aEb[mt][ks] = e_ok ? S[o * m + k] : 0.0;
      aOb[mt][ks] = o_ok ? S[o * m + H + 1 + k] : 0.0;
    }
  int lo[KS], hi[KS], oo[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = ks * 4 + t, kl = min(k, H);
    lo[ks] = kl * SO; hi[ks] = (m - 1 - kl) * SO;
    oo[ks] = (H + 1 + min(k, H - 1)) * SO;
  }
  // columns n = p + MP q (x fastest) tracked incrementally: no per-tile div/mod (see eoc_lines)
  constexpr int STEP = 8 * NW;
  // same tile-column permutation as eoc_lines: B column pi(g); for t >= 2 the lane's C columns
  // 2t, 2t + 1 swap roles (sw)
#ifdef PMG_EOC_PERM
  const int sw = t >> 1;
  int nB = warp * 8 + (g ^ ((g >> 2) & 1)), qB = nB / MP, pB = nB - qB * MP;
#else
  const int sw = 0;
  int nB = warp * 8 + g, qB = nB / MP, pB = nB - qB * MP;
#endif
  int n0 = warp * 8 + 2 * t, q0 = n0 / MP, p0 = n0 - q0 * MP;
  for (int tile = warp; tile < NT; tile += NW) {
    double *xb = X + (nB < NCOL ? pB + qB * SQ : (MP - 1) + (MQ - 1) * SQ);
    nB += STEP; pB += STEP % MP; qB += STEP / MP;
    if (pB >= MP) { pB -= MP; ++qB; }
    double bE[KS], bO[KS], cE[MT][2], cO[MT][2];
    // eigen-divide factors of this lane's outputs, fetched before the DMMAs (L1/L2 table)
    double rE[MT][2], rO[MT][2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int n = min(n0 + (j ^ sw), NCOL - 1);
      const double *rc = Rz + (long long)n * m;        // column n = p + MP q, p = x fastest
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int o = mt * 8 + g;
        rE[mt][j] = __ldg(rc + min(o, H));
        rO[mt][j] = __ldg(rc + H + 1 + min(o, H - 1));
      }
    }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const double v1 = xb[lo[ks]], v2 = xb[hi[ks]];
      bE[ks] = v1 + v2; bO[ks] = v1 - v2;
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
      wb[j] = -1;
      const int jj = j ^ sw;
      if (n0 + jj >= NCOL) continue;
      const bool carry = jj && p0 + 1 >= MP;         // column n0 + 1 wraps to the next y row
      wb[j] = carry ? (q0 + 1) * SQ : p0 + jj + q0 * SQ;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int o = mt * 8 + g;
        if (o <= H) X[wb[j] + o * SO] = cE[mt][j] * rE[mt][j];
        if (o < H) X[wb[j] + (H + 1 + o) * SO] = cO[mt][j] * rO[mt][j];
      }
    }
    __syncwarp();
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      bE[ks] = xb[lo[ks]];                        // t_E[min(k, H)]
      bO[ks] = xb[oo[ks]];                        // t_O[min(k, H-1)]
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
          X[wb[j] + o * SO] = cE[mt][j] + cO[mt][j];
          X[wb[j] + (m - 1 - o) * SO] = cE[mt][j] - cO[mt][j];
        } else if (o == H) {
          X[wb[j] + o * SO] = cE[mt][j];
        }
      }
    }
    n0 += STEP; p0 += STEP % MP; q0 += STEP / MP;
    if (p0 >= MP) { p0 -= MP; ++q0; }
  }
}

// Shared memory: window X (S2 * M2, padded planes) | S_x, S_y, S_z | lam | W | gather offsets
template <int M0, int M1, int M2, bool WIDE>
__global__ void __launch_bounds__(Shape<M0, M1, M2, WIDE>::THREADS, Shape<M0, M1, M2, WIDE>::MINB)
    k_fdm_eoc(LevelDev L, const double *__restrict__ r, double *__restrict__ Z, int color,
              double *__restrict__ u) {
  using SH = Shape<M0, M1, M2, WIDE>;
  constexpr int S2 = SH::S2, Mw = M0 * M1 * M2;
  extern __shared__ double sm[];
  double *X = sm;
  double *Ss[3] = {sm + S2 * M2, sm + S2 * M2 + M0 * M0, sm + S2 * M2 + M0 * M0 + M1 * M1};
  double *lam0 = Ss[2] + M2 * M2;
  double *lam[3] = {lam0, lam0 + M0, lam0 + M0 + M1};
  double *W0 = lam0 + M0 + M1 + M2;
  double *W[3] = {W0, W0 + M0, W0 + M0 + M1};
  long long *offs = reinterpret_cast<long long *>(W0 + M0 + M1 + M2);
  constexpr int mm[3] = {M0, M1, M2};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    stage(Ss[d], L.S[d], mm[d] * mm[d]);
    stage(lam[d], L.lam[d], mm[d]);
    stage(W[d], L.W[d], mm[d]);
  }
#ifdef PMG_FDM_REVERSE         // diagnostic: walk the subdomains backwards (tail of r still in L2)
  int e = color >= 0 ? blockIdx.x : gridDim.x - 1 - blockIdx.x;
#else
  int e = blockIdx.x;
#endif
  if (color >= 0) {       // subdomain bx of parity class `color` (2x2x2 colouring)
    const int hx = L.nx >> 1, hy = L.ny >> 1;
    const int bx = e % hx, by = (e / hx) % hy, bz = e / (hx * hy);
    e = (2 * bx + (color & 1)) + L.nx * ((2 * by + ((color >> 1) & 1)) + L.ny * (2 * bz + (color >> 2)));
  }
#ifdef PMG_PHASE_TIMING
  long long tph[8];
  tph[0] = clock64();
#define PMG_PH(i) tph[i] = clock64()
#else
#define PMG_PH(i)
#endif
  // Large levels (vector > 64 MB, i.e. not L2 resident): the r block of the subdomain 3/4 of a
  // resident wave ahead is prefetched into L2, so that CTA's window gather (13 % of the kernel,
  // exposed HBM latency) hits L2: c3 fdm@l4 1.227 -> 1.186 ms per cycle (distances 100-370 within
  // 0.3 % of each other, 444 and 592 lose the gain)
#ifndef PMG_FDM_PREFETCH
#define PMG_FDM_PREFETCH 222
#endif
  if (PMG_FDM_PREFETCH > 0 && threadIdx.x == 0 && color < 0) {
    const long long n3 = (long long)L.n * L.n * L.n;
    const long long en = (long long)e + PMG_FDM_PREFETCH;
    if (en < L.Ne && L.Ne * n3 > (8ll << 20)) prefetch_l2_doubles(r + en * n3, n3);
  }
  cp_async_commit();            // group T: the staged tables
  fdm_offsets(L, e, offs);
  __syncthreads();
#ifdef PMG_GATHER_PIPE         // diagnostic, measured SLOWER (c3 fdm@l4 1.255 vs 1.186, c5 0.929 vs 0.867): the
  constexpr bool GPIPE = true;  // tile-ordered copies (8 rows at 8 different z per tile) cost more than the overlap buys
#else
  constexpr bool GPIPE = false;
#endif
  if (GPIPE) {
    // Pipelined gather: a warp copies exactly the window rows of ITS tiles of the x forward pass
    // (8 columns = 8 x-rows per tile, z fastest), first two tiles in one cp.async group, the rest
    // in a second; the pass then starts on the first tiles while the others are still landing —
    // no block barrier between gather and pass (the rows a warp reads and overwrites are its own)
    const long long *xo = offs, *yo = offs + M0, *zo = offs + M0 + M1;
    constexpr int NCOL0 = M1 * M2, NT0 = (NCOL0 + 7) / 8, NW = SH::NWS;
    const int lane = threadIdx.x & 31, warp = SH::wid();
    auto gather_tile = [&](int t) {
      for (int i = lane; i < 8 * M0; i += 32) {
        const int cl = i / M0, a = i - cl * M0;
        const int n = 8 * t + cl;
        if (n < NCOL0) {
          const int b = n / M2, c = n - b * M2;
          cp_async8(X + a + M0 * b + S2 * c, r + xo[a] + yo[b] + zo[c]);
        }
      }
    };
    int t = warp;
    if (t < NT0) gather_tile(t);
    t += NW;
    if (t < NT0) gather_tile(t);
    cp_async_commit();
    for (t += NW; t < NT0; t += NW) gather_tile(t);
    cp_async_commit();
    cp_async_wait<2>();         // this thread's share of the tables
    __syncthreads();            // tables visible to every warp
  } else
#ifdef PMG_GATHER_ROWS
  {   // gather: one warp per window row (M0 <= 32), padded plane stride
    const long long *xo = offs, *yo = offs + M0, *zo = offs + M0 + M1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = SH::THREADS / 32;
    const long long xa = lane < M0 ? xo[lane] : 0;
    for (int row = warp; row < M1 * M2; row += NW) {
      const int c = row / M1, b = row - c * M1;
      if (lane < M0) cp_async8(X + lane + M0 * b + S2 * c, r + xa + yo[b] + zo[c]);
    }
  }
#else
  {   // gather: flat over the window (all 32 lanes of every cp.async busy: LDGSTS issue, not
      // latency, bounds this phase — a row per warp left 32 - M0 lanes idle), padded plane stride
    const long long *xo = offs, *yo = offs + M0, *zo = offs + M0 + M1;
#ifndef PMG_EXP_NOGATHER      // diagnostic: timing without the window gather (wrong results)
#ifdef PMG_GATHER_DIV         // round-2b form: a division pair per node (~33 instructions per copy)
    for (int w = threadIdx.x; w < Mw; w += SH::THREADS) {
      const int bc = w / M0, a = w - bc * M0;
      const int c = bc / M1, b = bc - c * M1;
      cp_async8(X + a + M0 * b + S2 * c, r + xo[a] + yo[b] + zo[c]);
    }
#else
    // node (a, b, c) and its padded shared-memory slot are tracked incrementally over the thread's
    // nodes w = tid + q THREADS (two compare-and-carry steps, no division); when the level's
    // vector has < 2^31 entries the three offsets are summed in 32 bits (low words of the table)
    constexpr int TH = SH::THREADS, DA = TH % M0, DB = (TH / M0) % M1, DC = TH / (M0 * M1);
    constexpr int PAD = S2 - M0 * M1;
    int a = threadIdx.x % M0, b = (threadIdx.x / M0) % M1, c = threadIdx.x / (M0 * M1);
    int dst = a + M0 * b + S2 * c;
    if ((long long)L.Ne * L.n * L.n * L.n < (1LL << 31)) {
      const int *xi = reinterpret_cast<const int *>(xo), *yi = reinterpret_cast<const int *>(yo),
                *zi = reinterpret_cast<const int *>(zo);
      for (int w = threadIdx.x; w < Mw; w += TH) {
        cp_async8(X + dst, r + (xi[2 * a] + yi[2 * b] + zi[2 * c]));
        a += DA; b += DB; c += DC; dst += TH + DC * PAD;
        if (a >= M0) { a -= M0; ++b; }
        if (b >= M1) { b -= M1; ++c; dst += PAD; }
      }
    } else {
      for (int w = threadIdx.x; w < Mw; w += TH) {
        cp_async8(X + dst, r + xo[a] + yo[b] + zo[c]);
        a += DA; b += DB; c += DC; dst += TH + DC * PAD;
        if (a >= M0) { a -= M0; ++b; }
        if (b >= M1) { b -= M1; ++c; dst += PAD; }
      }
    }
#endif
#else
    (void)xo; (void)yo; (void)zo;
    for (int w = threadIdx.x; w < S2 * M2; w += SH::THREADS) X[w] = 1.0;
#endif
  }
#endif
  if (!GPIPE) {
    cp_async_wait_all();
    __syncthreads();
  }
  PMG_PH(1);
  const Blk B = {{M0, M1, M2}, {1, M0, S2}};
  const double *lamc[3] = {lam[0], lam[1], lam[2]};
  EpiStore st{X, B};
  eoc_lines<0, SH, true, true, EpiStore, GPIPE>(X, Ss[0], st); __syncthreads();
  PMG_PH(2);
  eoc_lines<1, SH, true, true>(X, Ss[1], st); __syncthreads();
  PMG_PH(3);
#ifdef PMG_ZSPLIT
  {   // z forward with the eigen-divide epilogue, then z backward (two pipelined passes)
    EpiDivide dv{X, B, {lamc[0], lamc[1], lamc[2]}};
    eoc_lines<2, SH, true, false>(X, Ss[2], dv); __syncthreads();
    eoc_lines<2, SH, false, false>(X, Ss[2], st); __syncthreads();
  }
#else
  eoc_z_fused<SH>(X, Ss[2], lamc, L.Rz); __syncthreads();
#endif
  PMG_PH(4);
  eoc_lines<1, SH, false, true>(X, Ss[1], st); __syncthreads();
  PMG_PH(5);
  if (color >= 0) {
    EpiWeightRed wr{u, offs, M0, M1, {W[0], W[1], W[2]}};
    eoc_lines<0, SH, false, true>(X, Ss[0], wr);
  } else {
    const Blk G = {{M0, M1, M2}, {1, M0, M0 * M1}};   // global window order (Z)
#ifndef PMG_EXP_NOSTORE       // diagnostic: last pass stores in place (no global Z store)
    EpiWeightStore ws{Z + (long long)e * Mw, G, {W[0], W[1], W[2]}};
    eoc_lines<0, SH, false, true>(X, Ss[0], ws);
#else
    eoc_lines<0, SH, false, true>(X, Ss[0], st);
    if (threadIdx.x == 0) Z[(long long)e * Mw] = X[0];
#endif
  }
#ifdef PMG_PHASE_TIMING
  __syncthreads();
  PMG_PH(6);
  if (threadIdx.x == 0 && (blockIdx.x % 512) == 0)
    printf("PHASE fdm<%d,%d,%d> blk %d start %lld gather %lld xf %lld yf %lld z %lld yb %lld xb %lld\n", M0, M1, M2,
           blockIdx.x, tph[0], tph[1] - tph[0], tph[2] - tph[1], tph[3] - tph[2], tph[4] - tph[3],
           tph[5] - tph[4], tph[6] - tph[5]);
#endif
#undef PMG_PH
}

template <int M0, int M1, int M2>
size_t eoc_smem() {
  return sizeof(double) * ((size_t)Shape<M0, M1, M2>::S2 * M2 + M0 * M0 + M1 * M1 + M2 * M2 +
                           3 * (M0 + M1 + M2));
}

template <int M0, int M1, int M2, bool WIDE>
void eoc_launch_t(const LevelDev &L, int grid, const double *r, double *Z, int color, double *u,
                  cudaStream_t s) {
  const size_t sb = eoc_smem<M0, M1, M2>();
  static bool cfg = false;
  if (!cfg) {
    cfg = true;
    cudaFuncSetAttribute(k_fdm_eoc<M0, M1, M2, WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  }
  k_fdm_eoc<M0, M1, M2, WIDE><<<grid, Shape<M0, M1, M2, WIDE>::THREADS, sb, s>>>(L, r, Z, color, u);
}

template <int M0, int M1, int M2>
void eoc_launch(const LevelDev &L, int grid, const double *r, double *Z, int color, double *u,
                cudaStream_t s) {
  // one wave of 128-thread CTAs would leave the SMs mostly idle: widen the CTAs instead
  if (Shape<M0, M1, M2>::THREADS == 128 && grid <= 4 * num_sms())
    eoc_launch_t<M0, M1, M2, true>(L, grid, r, Z, color, u, s);
  else
    eoc_launch_t<M0, M1, M2, false>(L, grid, r, Z, color, u, s);
}

// ---- P = 32 windows (m = 45, 729 KB: larger than an SM's shared memory) --------------------
// Three slab kernels over two L2-resident window buffers (Ne x 45^3 each, c4: 47 MB):
//   k_fdm45_a  (subdomain, z-slab of ZS planes): gather the slab of the window, forward x and y
//              passes (plane-local), slab -> W1;
//   k_fdm45_b  (subdomain, y-slab of YS lines): forward z with the eigen-divide epilogue, backward
//              z (z columns are complete in a y-slab), slab -> W2;
//   k_fdm45_c  (subdomain, z-slab): backward y and x, weighted store to Z (window order).
// The even/odd line GEMMs (eoc_lines, 2 x 3 x 6 DMMAs per 8-column tile) run on the slab in
// shared memory; 128-thread CTAs (the m = 45 A fragments alone are 36 doubles per lane).
constexpr int W45 = 45, ZS45 = 5, YS45 = 5, NS45 = W45 / ZS45;
using SZ45 = Shape<W45, W45, ZS45, false, 128>;     // z-slab block
using SY45 = Shape<W45, YS45, W45, false, 128>;     // y-slab block

__global__ void __launch_bounds__(128, 3) k_fdm45_a(LevelDev L, const double *__restrict__ r,
                                                    double *__restrict__ W1) {
  extern __shared__ double sm[];
  constexpr int S2 = SZ45::S2;
  double *X = sm, *Sx = X + S2 * ZS45, *Sy = Sx + W45 * W45;
  long long *offs = reinterpret_cast<long long *>(Sy + W45 * W45);
  const int e = blockIdx.y, z0 = blockIdx.x * ZS45;
  stage(Sx, L.S[0], W45 * W45);
  stage(Sy, L.S[1], W45 * W45);
  fdm_offsets(L, e, offs);
  __syncthreads();
  const long long *xo = offs, *yo = offs + W45, *zo = offs + 2 * W45 + z0;
  for (int w = threadIdx.x; w < W45 * W45 * ZS45; w += blockDim.x) {
    const int bc = w / W45, a = w - bc * W45;
    const int c = bc / W45, b = bc - c * W45;
    cp_async8(X + a + W45 * b + S2 * c, r + xo[a] + yo[b] + zo[c]);
  }
  cp_async_wait_all();
  __syncthreads();
  const Blk B = {{W45, W45, ZS45}, {1, W45, S2}};
  EpiStore st{X, B};
  eoc_lines<0, SZ45, true, true>(X, Sx, st); __syncthreads();
  eoc_lines<1, SZ45, true, true>(X, Sy, st); __syncthreads();
  double *out = W1 + (long long)e * L.Mw + (long long)z0 * W45 * W45;
  for (int w = threadIdx.x; w < W45 * W45 * ZS45; w += blockDim.x) {
    const int c = w / (W45 * W45), ab = w - c * W45 * W45;
    out[w] = X[ab + S2 * c];
  }
}

__global__ void __launch_bounds__(128, 3) k_fdm45_b(LevelDev L, const double *__restrict__ W1,
                                                    double *__restrict__ W2) {
  extern __shared__ double sm[];
  constexpr int S2 = SY45::S2;
  double *X = sm, *Sz = X + S2 * W45;
  const int e = blockIdx.y, y0 = blockIdx.x * YS45;
  stage(Sz, L.S[2], W45 * W45);
  const double *in = W1 + (long long)e * L.Mw + (long long)y0 * W45;
  for (int w = threadIdx.x; w < W45 * YS45 * W45; w += blockDim.x) {     // (a, b, c): rows of 45
    const int bc = w / W45, a = w - bc * W45;
    const int c = bc / YS45, b = bc - c * YS45;
    cp_async8(X + a + W45 * b + S2 * c, in + a + W45 * b + W45 * W45 * c);
  }
  cp_async_wait_all();
  __syncthreads();
  const Blk B = {{W45, YS45, W45}, {1, W45, S2}};
  EpiDivide dv{X, B, {L.lam[0], L.lam[1] + y0, L.lam[2]}};
  EpiStore st{X, B};
  eoc_lines<2, SY45, true, false>(X, Sz, dv); __syncthreads();
  eoc_lines<2, SY45, false, false>(X, Sz, st); __syncthreads();
  double *out = W2 + (long long)e * L.Mw + (long long)y0 * W45;
  for (int w = threadIdx.x; w < W45 * YS45 * W45; w += blockDim.x) {
    const int bc = w / W45, a = w - bc * W45;
    const int c = bc / YS45, b = bc - c * YS45;
    out[a + W45 * b + W45 * W45 * c] = X[a + W45 * b + S2 * c];
  }
}

__global__ void __launch_bounds__(128, 3) k_fdm45_c(LevelDev L, const double *__restrict__ W2,
                                                    double *__restrict__ Z) {
  extern __shared__ double sm[];
  constexpr int S2 = SZ45::S2;
  double *X = sm, *Sx = X + S2 * ZS45, *Sy = Sx + W45 * W45, *Wt = Sy + W45 * W45;
  const int e = blockIdx.y, z0 = blockIdx.x * ZS45;
  stage(Sx, L.S[0], W45 * W45);
  stage(Sy, L.S[1], W45 * W45);
  stage(Wt, L.W[0], W45);
  stage(Wt + W45, L.W[1], W45);
  stage(Wt + 2 * W45, L.W[2] + z0, ZS45);
  const double *in = W2 + (long long)e * L.Mw + (long long)z0 * W45 * W45;
  for (int w = threadIdx.x; w < W45 * W45 * ZS45; w += blockDim.x) {
    const int c = w / (W45 * W45), ab = w - c * W45 * W45;
    cp_async8(X + ab + S2 * c, in + w);
  }
  cp_async_wait_all();
  __syncthreads();
  const Blk B = {{W45, W45, ZS45}, {1, W45, S2}};
  EpiStore st{X, B};
  eoc_lines<1, SZ45, false, true>(X, Sy, st); __syncthreads();
  const Blk G = {{W45, W45, ZS45}, {1, W45, W45 * W45}};             // global window order
  EpiWeightStore ws{Z + (long long)e * L.Mw + (long long)z0 * W45 * W45, G, {Wt, Wt + W45, Wt + 2 * W45}};
  eoc_lines<0, SZ45, false, true>(X, Sx, ws);
}

}  // namespace

bool fdm45_ok(const LevelDev &L) {
#ifdef PMG_NO_FDM45
  return false;
#endif
  return L.m[0] == W45 && L.m[1] == W45 && L.m[2] == W45 && L.n == 33;
}

// W1, W2: Ne * 45^3 scratch each (L2-resident window buffers)
cudaError_t launch_fdm45(const LevelDev &L, const double *r, double *W1, double *W2, double *Z,
                         cudaStream_t s) {
  const size_t sa = sizeof(double) * ((size_t)SZ45::S2 * ZS45 + 2 * W45 * W45 + 3 * W45);
  const size_t sb = sizeof(double) * ((size_t)SY45::S2 * W45 + W45 * W45);
  const size_t sc = sizeof(double) * ((size_t)SZ45::S2 * ZS45 + 2 * W45 * W45 + 3 * W45);
  static bool cfg = false;
  if (!cfg) {
    cfg = true;
    cudaFuncSetAttribute(k_fdm45_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sa);
    cudaFuncSetAttribute(k_fdm45_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
    cudaFuncSetAttribute(k_fdm45_c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc);
  }
  k_fdm45_a<<<dim3(NS45, L.Ne), 128, sa, s>>>(L, r, W1);
  k_fdm45_b<<<dim3(W45 / YS45, L.Ne), 128, sb, s>>>(L, W1, W2);
  k_fdm45_c<<<dim3(NS45, L.Ne), 128, sc, s>>>(L, W2, Z);
  return cudaGetLastError();
}

namespace {
}  // namespace

// Shapes of the benchmark configurations (c1-c5, all levels); others use the generic kernels.
#define PMG_EOC_SHAPES(X) \
  X(23, 23, 23) X(13, 13, 13) X(7, 7, 7) X(5, 5, 5) X(11, 27, 27) X(7, 15, 15) X(5, 9, 9)

bool fdm_eoc_launch(const LevelDev &L, const double *r, double *Z, int color, double *u,
                    cudaStream_t s) {
#ifdef PMG_NO_EOC
  return false;
#endif
  if (color < 0 && fdm_dl_launch(L, r, Z, s)) return true;   // small windows: FP64-FMA line kernel
  const int grid = color >= 0 ? L.Ne / 8 : L.Ne;
#define PMG_EOC_CASE(a, b, c)                                    \
  if (L.m[0] == a && L.m[1] == b && L.m[2] == c) {              \
    eoc_launch<a, b, c>(L, grid, r, Z, color, u, s);            \
    return true;                                                \
  }
  PMG_EOC_SHAPES(PMG_EOC_CASE)
#undef PMG_EOC_CASE
  return false;
}

}  // namespace pmg
