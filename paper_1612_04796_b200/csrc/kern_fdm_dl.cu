// Schwarz subdomain solves on the SMALLEST windows (5^3, 7^3, 5 x 9 x 9: the two lowest multigrid
// levels) by fast diagonalisation with plain FP64 FMAs, one thread per window LINE.
// PAPER.md:201-232 (Eq. 9 and the fast-diagonalisation formula), :234-244 (Eq. 10 weights).
//
// Why not the DMMA line GEMMs here: on B200 the FP64 tensor pipe (DMMA.8x8x4) and the FP64 FMA
// pipe have the same peak (37.1 vs 33.5 TFLOP/s measured), so DMMA only pays through its lower
// instruction count — and on a 13^3 window the even/odd half-GEMMs are 7 x 7 and 6 x 6: every tile
// pads them to 8 x 8 x 8 (66 % useful; a 7^3 window's 4 x 4 and 3 x 3 products 16 %) and carries
// ~30 bookkeeping instructions per DMMA.  Here a thread owns whole lines:
// it loads the m values of a line once, forms the even / odd combinations in registers
// (x_a +- x_{m-1-a}), and runs the (H+1)^2 + H^2 FMAs of the two half-size products against
// coefficients broadcast from shared memory (one 16-byte load per two coefficients, shared by
// the R lines the thread works on at once).  The z pass is forward + eigen-divide + backward on
// the same lines with no block barrier in between.  Same tables (L.S, L.Rz, L.W) and the same
// even-modes-first eigenvector order as k_fdm_eoc; results differ from it by rounding order only.
#include "kcommon.cuh"

namespace pmg {
namespace {

template <int M0, int M1, int M2>
struct DlShape {
  static constexpr int S2 = M0 * M1 | 1;                 // odd plane stride: conflict-free z lines
  static constexpr int MAXL = (M0 * M1 > M0 * M2 ? (M0 * M1 > M1 * M2 ? M0 * M1 : M1 * M2)
                                                 : (M0 * M2 > M1 * M2 ? M0 * M2 : M1 * M2));
#ifndef PMG_DL_R2_MIN
#define PMG_DL_R2_MIN 128
#endif
  static constexpr int R = MAXL >= PMG_DL_R2_MIN ? 2 : 1;   // lines a thread works on at once
  static constexpr int THREADS = ((MAXL + R - 1) / R + 31) / 32 * 32;
  template <int D> __host__ __device__ static constexpr int m() { return D == 0 ? M0 : (D == 1 ? M1 : M2); }
};

// coefficient table of one direction: FE | FO | BE | BO, rows padded to an even length
template <int M>
struct DlTab {
  static constexpr int H = M / 2, KE = (H + 2) & ~1, KO = (H + 1) & ~1;
  static constexpr int FE = 0, FO = FE + (H + 1) * KE, BE = FO + H * KO, BO = BE + (H + 1) * KE;
  static constexpr int LEN = BO + H * KO;
};

template <int M>
__device__ __forceinline__ void dl_stage_tab(const double *__restrict__ S, double *tab, int tid, int nthr) {
  using T = DlTab<M>;
  constexpr int H = T::H;
  for (int i = tid; i < T::LEN; i += nthr) {
    double v = 0.0;
    if (i < T::FO) {                       // forward even: out o = sum_k S[k][o] s_k, s_H = x_H
      const int o = i / T::KE, k = i - o * T::KE;
      if (k <= H) v = S[k * M + o];
    } else if (i < T::BE) {                // forward odd: out H+1+o = sum_k S[k][H+1+o] d_k
      const int j = i - T::FO, o = j / T::KO, k = j - o * T::KO;
      if (k < H) v = S[k * M + H + 1 + o];
    } else if (i < T::BO) {                // backward even: P_o = sum_k S[o][k] t_k
      const int j = i - T::BE, o = j / T::KE, k = j - o * T::KE;
      if (k <= H) v = S[o * M + k];
    } else {                               // backward odd: Q_o = sum_k S[o][H+1+k] t_{H+1+k}
      const int j = i - T::BO, o = j / T::KO, k = j - o * T::KO;
      if (k < H) v = S[o * M + H + 1 + k];
    }
    tab[i] = v;
  }
}

// One line pass over R lines at once.  x[r]: line bases; SO: element stride along the line.
// FWD: t = S^T x (even modes at 0..H, odd modes at H+1..);  !FWD: x = S t.
// scale != nullptr (forward only): the outputs are multiplied by scale[r][o] (eigen-divide table).
template <int M, int R, bool FWD>
__device__ __forceinline__ void dl_lines(double *const (&x)[R], int SO, const double *tab,
                                         const double *const (&scale)[R], bool scaled) {
  using T = DlTab<M>;
  constexpr int H = T::H;
  double s[R][H + 1], d[R][H > 0 ? H : 1];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (FWD) {
#pragma unroll
      for (int k = 0; k < H; ++k) {
        const double a = x[r][k * SO], b = x[r][(M - 1 - k) * SO];
        s[r][k] = a + b;
        d[r][k] = a - b;
      }
      s[r][H] = x[r][H * SO];
    } else {
#pragma unroll
      for (int k = 0; k <= H; ++k) s[r][k] = x[r][k * SO];
#pragma unroll
      for (int k = 0; k < H; ++k) d[r][k] = x[r][(H + 1 + k) * SO];
    }
  }
  const double *CE = tab + (FWD ? T::FE : T::BE), *CO = tab + (FWD ? T::FO : T::BO);
  // one output pair (even mode o, odd mode o) per iteration; the loop over o stays ROLLED: fully
  // unrolled, a window's six passes were ~100 KB of straight-line code that every CTA streamed
  // through once (instruction-cache misses made the 13^3 kernel 2x slower than this form)
  auto outputs = [&](int o, bool odd) {
    double e[R], q[R];
#pragma unroll
    for (int r = 0; r < R; ++r) e[r] = q[r] = 0.0;
    const double2 *ce = reinterpret_cast<const double2 *>(CE + o * T::KE);
#pragma unroll
    for (int k2 = 0; k2 < T::KE / 2; ++k2) {
      const double2 c = ce[k2];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (2 * k2 <= H) e[r] = fma(c.x, s[r][2 * k2], e[r]);
        if (2 * k2 + 1 <= H) e[r] = fma(c.y, s[r][2 * k2 + 1], e[r]);
      }
    }
    if (odd) {
      const double2 *co = reinterpret_cast<const double2 *>(CO + o * T::KO);
#pragma unroll
      for (int k2 = 0; k2 < T::KO / 2; ++k2) {
        const double2 c = co[k2];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (2 * k2 < H) q[r] = fma(c.x, d[r][2 * k2], q[r]);
          if (2 * k2 + 1 < H) q[r] = fma(c.y, d[r][2 * k2 + 1], q[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (FWD) {
        double ve = e[r], vo = q[r];
        if (scaled) {
          ve *= __ldg(scale[r] + o);
          if (odd) vo *= __ldg(scale[r] + H + 1 + o);
        }
        x[r][o * SO] = ve;
        if (odd) x[r][(H + 1 + o) * SO] = vo;
      } else {
        x[r][o * SO] = e[r] + q[r];
        if (odd) x[r][(M - 1 - o) * SO] = e[r] - q[r];
      }
    }
  };
#pragma unroll 1
  for (int o = 0; o < H; ++o) outputs(o, true);
  outputs(H, false);
}

// all lines of direction DIR of the window in X; ZF: forward + eigen-divide + backward (z only)
template <int DIR, class SH, bool FWD, bool ZF>
__device__ __forceinline__ void dl_pass(double *X, const double *tab, const double *__restrict__ Rz) {
  constexpr int M = SH::template m<DIR>();
  constexpr int M0 = SH::template m<0>(), M1 = SH::template m<1>(), M2 = SH::template m<2>();
  constexpr int MP = DIR == 0 ? M1 : M0;                  // fast line index: b (x pass) or a
  constexpr int NL = DIR == 0 ? M1 * M2 : (DIR == 1 ? M0 * M2 : M0 * M1);
  constexpr int SO = DIR == 0 ? 1 : (DIR == 1 ? M0 : SH::S2);
  constexpr int R = SH::R, TH = SH::THREADS;
  for (int l0 = threadIdx.x; l0 < NL; l0 += R * TH) {
    double *x[R];
    const double *sc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      // a dead slot repeats the thread's first line: identical values are recomputed and stored
      const int l = (l0 + r * TH < NL) ? l0 + r * TH : l0;
      const int q = l / MP, p = l - q * MP;
      x[r] = X + (DIR == 0 ? M0 * p + SH::S2 * q : (DIR == 1 ? p + SH::S2 * q : l));
      sc[r] = ZF ? Rz + (long long)l * M2 : nullptr;      // Rz[(a + M0 b) M2 + o], l = a + M0 b
    }
    if (ZF) {
      dl_lines<M, R, true>(x, SO, tab, sc, true);
      dl_lines<M, R, false>(x, SO, tab, sc, false);
    } else {
      dl_lines<M, R, FWD>(x, SO, tab, sc, false);
    }
  }
}

template <int M0, int M1, int M2>
__global__ void __launch_bounds__(DlShape<M0, M1, M2>::THREADS)
    k_fdm_dl(LevelDev L, const double *__restrict__ r, double *__restrict__ Z) {
  using SH = DlShape<M0, M1, M2>;
  constexpr int S2 = SH::S2, Mw = M0 * M1 * M2, TH = SH::THREADS;
  constexpr int PLANES = (S2 * M2 + 1) & ~1;
  extern __shared__ double sm[];
  double *X = sm;
  double *tab0 = sm + PLANES, *tab1 = tab0 + DlTab<M0>::LEN, *tab2 = tab1 + DlTab<M1>::LEN;
  double *W0 = tab2 + DlTab<M2>::LEN;
  double *W[3] = {W0, W0 + M0, W0 + M0 + M1};
  long long *offs = reinterpret_cast<long long *>(W0 + ((M0 + M1 + M2 + 1) & ~1));
  const int e = blockIdx.x;
  dl_stage_tab<M0>(L.S[0], tab0, threadIdx.x, TH);
  dl_stage_tab<M1>(L.S[1], tab1, threadIdx.x, TH);
  dl_stage_tab<M2>(L.S[2], tab2, threadIdx.x, TH);
  for (int i = threadIdx.x; i < M0; i += TH) W[0][i] = L.W[0][i];
  for (int i = threadIdx.x; i < M1; i += TH) W[1][i] = L.W[1][i];
  for (int i = threadIdx.x; i < M2; i += TH) W[2][i] = L.W[2][i];
  fdm_offsets(L, e, offs);
  __syncthreads();
  {   // gather: node (a, b, c) tracked incrementally, padded plane stride
    const long long *xo = offs, *yo = offs + M0, *zo = offs + M0 + M1;
    constexpr int DA = TH % M0, DB = (TH / M0) % M1, DC = TH / (M0 * M1), PAD = S2 - M0 * M1;
    int a = threadIdx.x % M0, b = (threadIdx.x / M0) % M1, c = threadIdx.x / (M0 * M1);
    int dst = a + M0 * b + S2 * c;
    for (int w = threadIdx.x; w < Mw; w += TH) {
      cp_async8(X + dst, r + xo[a] + yo[b] + zo[c]);
      a += DA; b += DB; c += DC; dst += TH + DC * PAD;
      if (a >= M0) { a -= M0; ++b; }
      if (b >= M1) { b -= M1; ++c; dst += PAD; }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  dl_pass<0, SH, true, false>(X, tab0, nullptr); __syncthreads();
  dl_pass<1, SH, true, false>(X, tab1, nullptr); __syncthreads();
  dl_pass<2, SH, true, true>(X, tab2, L.Rz); __syncthreads();
  dl_pass<1, SH, false, false>(X, tab1, nullptr); __syncthreads();
  dl_pass<0, SH, false, false>(X, tab0, nullptr); __syncthreads();
  {   // weight W_x (x) W_y (x) W_z (Eq. 10) and store the window (coalesced, unpadded order)
    constexpr int DA = TH % M0, DB = (TH / M0) % M1, DC = TH / (M0 * M1), PAD = S2 - M0 * M1;
    int a = threadIdx.x % M0, b = (threadIdx.x / M0) % M1, c = threadIdx.x / (M0 * M1);
    int src = a + M0 * b + S2 * c;
    double *Ze = Z + (long long)e * Mw;
    for (int w = threadIdx.x; w < Mw; w += TH) {
      Ze[w] = X[src] * (W[0][a] * (W[1][b] * W[2][c]));
      a += DA; b += DB; c += DC; src += TH + DC * PAD;
      if (a >= M0) { a -= M0; ++b; }
      if (b >= M1) { b -= M1; ++c; src += PAD; }
    }
  }
}

template <int M0, int M1, int M2>
void dl_launch(const LevelDev &L, const double *r, double *Z, cudaStream_t s) {
  using SH = DlShape<M0, M1, M2>;
  const size_t sb = sizeof(double) * (((size_t)SH::S2 * M2 + 1 & ~(size_t)1) + DlTab<M0>::LEN +
                                      DlTab<M1>::LEN + DlTab<M2>::LEN + ((M0 + M1 + M2 + 1) & ~1) +
                                      (M0 + M1 + M2));
  static bool cfg = false;
  if (!cfg) {
    cfg = true;
    cudaFuncSetAttribute(k_fdm_dl<M0, M1, M2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  }
  k_fdm_dl<M0, M1, M2><<<L.Ne, SH::THREADS, sb, s>>>(L, r, Z);
}

}  // namespace

// Measured against k_fdm_eoc (B200, ms per V-cycle, DL / DMMA): 7^3 x 4096 windows 0.052 / 0.063,
// 5^3 x 4096 0.029 / 0.042, (5,9,9) x 4096 0.053 / 0.076, 5^3 x 512 0.018 / 0.020 — but 13^3
// 0.208 / 0.192 and (7,15,15) 0.169 / 0.159 (both kernels are bound by shared-memory wavefronts
// there: a broadcast 16-byte coefficient load costs 4, and the line kernel issues 5.7 k per 13^3
// window against 4.8 k), and on one-wave meshes (64 windows) the per-thread chain of a whole line
// is longer than a window spread over 8 DMMA warps.  So: the three smallest shapes, full grids only.
#define PMG_DL_SHAPES(X) X(7, 7, 7) X(5, 5, 5) X(5, 9, 9)
#ifdef PMG_DL_ALL
#undef PMG_DL_SHAPES
#define PMG_DL_SHAPES(X) X(13, 13, 13) X(7, 7, 7) X(5, 5, 5) X(7, 15, 15) X(5, 9, 9)
#endif

// uncoloured solve into the window buffer Z; false: shape not served here
bool fdm_dl_launch(const LevelDev &L, const double *r, double *Z, cudaStream_t s) {
#ifdef PMG_NO_FDM_DL
  return false;
#endif
  if (L.Rz == nullptr || L.Ne < 512) return false;
#define PMG_DL_CASE(a, b, c)                                     \
  if (L.m[0] == a && L.m[1] == b && L.m[2] == c) {              \
    dl_launch<a, b, c>(L, r, Z, s);                             \
    return true;                                                \
  }
  PMG_DL_SHAPES(PMG_DL_CASE)
#undef PMG_DL_CASE
  return false;
}

}  // namespace pmg
