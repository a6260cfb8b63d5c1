// Operator apply / residual (Eq. 7-8) for P = 32 elements (n = 33: 35 937 DOF, too large for one
// CTA's shared memory) as two slab kernels with even/odd DMMA line GEMMs in shared memory.
// arXiv:1612.04796, PAPER.md:149-164 (Eq. 7: v = sum_d M_other (D_d + neighbour couplings) u).
//
//   k_apply33_xz  CTA = (element, slab of JB y-lines): the x and z line GEMMs are local to such a
//                 slab (all i, all k), their sum V_xz goes to an L2-resident scratch vector;
//   k_apply33_y   CTA = (element, slab of KB z-planes): the y line GEMM (all i, all j), then
//                 out = f - M (V_y + V_xz).
// Every line GEMM uses the centro-symmetry of the GLL/GL element rows (as the n = 17 apply):
// rows i and n-1-i from the even/odd halves, K = H+1 symmetric pairs + the two face-coefficient
// pairs, so an 8-column tile costs 2 x 2 x 5 DMMAs + an FMA tail row instead of 5 x 10.
#include <algorithm>

#include "kcommon.cuh"

namespace pmg {
namespace {

constexpr int N33 = 33, H33 = 16, N33_2 = N33 * N33, N33_3 = N33_2 * N33;
constexpr int MT33 = H33 / 8, KS33 = (H33 + 3 + 3) / 4;      // 2 M-tiles, 5 K-slices
constexpr int AF33 = (2 * MT33 * KS33 + KS33) * 32;          // A-fragment table, doubles per direction
#ifndef PMG_A33_SLAB
#define PMG_A33_SLAB 3
#endif
constexpr int JB = PMG_A33_SLAB, KB = PMG_A33_SLAB, NSLAB = N33 / JB;   // slabs of JB lines / KB planes

// A fragments of the even/odd line GEMM of one direction for every lane (g, t): E rows, O rows
// (row i = 8 mt + g < H), E tail row H; K slot k = 4 ks + t: k < H pair (k, n-1-k), k = H the
// middle node, H+1 the face pair (c1, c3), H+2 the face pair (c2, -c4).  Rows of Daug are
// pre-scaled by 1/M_d (api.cu), the factor 1/2 of (E +- O)/2 is folded in here.
__device__ __forceinline__ void afrag33(const double *__restrict__ Daug, double *af) {
  constexpr int n = N33, H = H33, KA = n + 4;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  auto coefE = [&](int i, int k) {
    const double *r = Daug + i * KA;
    if (k < H) return 0.5 * (r[k] + r[n - 1 - k]);
    if (k == H) return 0.5 * r[H];
    if (k == H + 1) return 0.5 * (r[n] + r[n + 2]);
    if (k == H + 2) return 0.5 * (r[n + 1] - r[n + 3]);
    return 0.0;
  };
  auto coefO = [&](int i, int k) {
    const double *r = Daug + i * KA;
    if (k < H) return 0.5 * (r[k] - r[n - 1 - k]);
    if (k == H + 1) return 0.5 * (r[n] - r[n + 2]);
    if (k == H + 2) return 0.5 * (r[n + 1] + r[n + 3]);
    return 0.0;
  };
#pragma unroll
  for (int ks = 0; ks < KS33; ++ks) {
    const int k = ks * 4 + t;
#pragma unroll
    for (int mt = 0; mt < MT33; ++mt) {
      af[((0 * MT33 + mt) * KS33 + ks) * 32 + lane] = coefE(mt * 8 + g, k);
      af[((1 * MT33 + mt) * KS33 + ks) * 32 + lane] = coefO(mt * 8 + g, k);
    }
    af[(2 * MT33 * KS33 + ks) * 32 + lane] = coefE(H, k);
  }
}

// V[o, col] (=|+=) sum_k A[o, k] X[k, col] on a shared-memory block: contracted index stride SO,
// columns col = p + MP q at X + p SP + q SQ, face coefficients C[r, col] at C + r CR + p CP + q CQ.
template <int SO, int SP, int SQ, int MP, int NCOL, int CR, int CP, int CQ, bool FIRST>
__device__ __forceinline__ void eo33_lines(const double *U, const double *C, double *V, const double *af) {
  constexpr int n = N33, H = H33, NT = (NCOL + 7) / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  if (warp >= NT) return;
  double aE[MT33][KS33], aO[MT33][KS33], at[KS33];
#pragma unroll
  for (int ks = 0; ks < KS33; ++ks) {
#pragma unroll
    for (int mt = 0; mt < MT33; ++mt) {
      aE[mt][ks] = af[((0 * MT33 + mt) * KS33 + ks) * 32 + lane];
      aO[mt][ks] = af[((1 * MT33 + mt) * KS33 + ks) * 32 + lane];
    }
    at[ks] = af[(2 * MT33 * KS33 + ks) * 32 + lane];
  }
  bool fromC[KS33];
  int o1[KS33], o2[KS33];
#pragma unroll
  for (int ks = 0; ks < KS33; ++ks) {
    const int k = ks * 4 + t;
    fromC[ks] = (k == H + 1 || k == H + 2);
    if (k == H + 1) { o1[ks] = 0; o2[ks] = 2 * CR; }
    else if (k == H + 2) { o1[ks] = CR; o2[ks] = 3 * CR; }
    else { const int kk = k < H ? k : H; o1[ks] = kk * SO; o2[ks] = (n - 1 - kk) * SO; }
  }
  auto compute = [&](int tile, double (&cE)[MT33][2], double (&cO)[MT33][2], double &tl, int &pb, int &qb) {
    const int nb = min(tile * 8 + g, NCOL - 1);
    qb = nb / MP;
    pb = nb - qb * MP;
    const double *xb = U + pb * SP + qb * SQ;
    const double *cb = C + pb * CP + qb * CQ;
    double bE[KS33], bO[KS33];
#pragma unroll
    for (int ks = 0; ks < KS33; ++ks) {
      const double *src = fromC[ks] ? cb : xb;
      const double v1 = src[o1[ks]], v2 = src[o2[ks]];
      bE[ks] = v1 + v2;
      bO[ks] = v1 - v2;
    }
#pragma unroll
    for (int mt = 0; mt < MT33; ++mt) { cE[mt][0] = cE[mt][1] = cO[mt][0] = cO[mt][1] = 0.0; }
#pragma unroll
    for (int ks = 0; ks < KS33; ++ks)
#pragma unroll
      for (int mt = 0; mt < MT33; ++mt) {
        dmma884(cE[mt][0], cE[mt][1], aE[mt][ks], bE[ks]);
        dmma884(cO[mt][0], cO[mt][1], aO[mt][ks], bO[ks]);
      }
    tl = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS33; ++ks) tl = fma(at[ks], bE[ks], tl);
    tl += __shfl_xor_sync(0xffffffffu, tl, 1);
    tl += __shfl_xor_sync(0xffffffffu, tl, 2);
  };
  auto epilogue = [&](int tile, const double (&cE)[MT33][2], const double (&cO)[MT33][2], double tl, int pb, int qb) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c = tile * 8 + 2 * t + j;
      if (c >= NCOL) continue;
      const int q = c / MP, p = c - q * MP;
      double *vb = V + p * SP + q * SQ;
#pragma unroll
      for (int mt = 0; mt < MT33; ++mt) {
        const int o = mt * 8 + g;
        const double lo = cE[mt][j] + cO[mt][j], hi = cE[mt][j] - cO[mt][j];
        if (FIRST) { vb[o * SO] = lo; vb[(n - 1 - o) * SO] = hi; }
        else { vb[o * SO] += lo; vb[(n - 1 - o) * SO] += hi; }
      }
    }
    if (t == 0 && tile * 8 + g < NCOL) {
      double *vb = V + pb * SP + qb * SQ + H * SO;
      if (FIRST) *vb = tl;
      else *vb += tl;
    }
  };
  double cE0[MT33][2], cO0[MT33][2], cE1[MT33][2], cO1[MT33][2], tl0, tl1;
  int pb0, qb0, pb1, qb1;
  int tile = warp;
  compute(tile, cE0, cO0, tl0, pb0, qb0);
  for (;;) {
    const int t1 = tile + nw;
    if (t1 < NT) compute(t1, cE1, cO1, tl1, pb1, qb1);
    __syncwarp();
    epilogue(tile, cE0, cO0, tl0, pb0, qb0);
    if (t1 >= NT) break;
    const int t2 = t1 + nw;
    if (t2 < NT) compute(t2, cE0, cO0, tl0, pb0, qb0);
    __syncwarp();
    epilogue(t1, cE1, cO1, tl1, pb1, qb1);
    if (t2 >= NT) break;
    tile = t2;
  }
}

// face coefficients of direction d at in-face point p of element e from the neighbours' traces
// (T[((e*3+d)*4+q)*n^2 + p]): C0 = -tdR/2 - mu tvR, C1 = tvR/2, C2 = tdL/2 - mu tvL, C3 = tvL/2
// (the even/odd GEMM takes -c4)
__device__ __forceinline__ void face_coefs(const LevelDev &L, const double *__restrict__ T, int e, int d,
                                           int p, double *C, int cr) {
  int c[3] = {e % L.nx, (e / L.nx) % L.ny, e / (L.nx * L.ny)};
  const int edim[3] = {L.nx, L.ny, L.nz};
  const int cd = c[d];
  c[d] = wrap(cd + 1, edim[d]);
  const double *TR = T + ((long long)(c[0] + L.nx * (c[1] + L.ny * c[2])) * 3 + d) * 4 * N33_2;
  c[d] = wrap(cd - 1, edim[d]);
  const double *TL = T + ((long long)(c[0] + L.nx * (c[1] + L.ny * c[2])) * 3 + d) * 4 * N33_2;
  const double tvR = __ldg(TR + p), tdR = __ldg(TR + N33_2 + p);
  const double tvL = __ldg(TL + 2 * N33_2 + p), tdL = __ldg(TL + 3 * N33_2 + p);
  const double mu = L.mu[d];
  C[0] = -0.5 * tdR - mu * tvR;
  C[cr] = 0.5 * tvR;
  C[2 * cr] = 0.5 * tdL - mu * tvL;
  C[3 * cr] = 0.5 * tvL;
}

// smem: U [k][jj][i] (33 x JB x 33) | V (same) | Cx [4][k][jj] | Cz [4][jj][i] | A tables x, z
__global__ void __launch_bounds__(128, 4) k_apply33_xz(LevelDev L, const double *__restrict__ u,
                                                       const double *__restrict__ T,
                                                       double *__restrict__ Vxz) {
  extern __shared__ double sm[];
  constexpr int SL = N33 * JB * N33;                 // slab doubles
  double *U = sm, *V = U + SL, *Cx = V + SL, *Cz = Cx + 4 * N33 * JB, *afx = Cz + 4 * N33 * JB, *afz = afx + AF33;
  const int e = blockIdx.y, j0 = blockIdx.x * JB;
  const long long e0 = (long long)e * N33_3;
  for (int w = threadIdx.x; w < SL; w += blockDim.x) {      // (i, jj, k): 33 JB contiguous per k
    const int k = w / (N33 * JB), r = w - k * N33 * JB;
    cp_async8(U + w, u + e0 + (long long)k * N33_2 + j0 * N33 + r);
  }
  const int warp = threadIdx.x >> 5;
  if (warp == 0) afrag33(L.Daug[0], afx);
  else if (warp == 1) afrag33(L.Daug[2], afz);
  for (int w = threadIdx.x; w < N33 * JB; w += blockDim.x) {
    const int jj = w % JB, k = w / JB;                       // x faces: point p = j + n k
    face_coefs(L, T, e, 0, j0 + jj + N33 * k, Cx + jj + JB * k, N33 * JB);
    const int i = w % N33, jz = w / N33;                     // z faces: point p = i + n j
    face_coefs(L, T, e, 2, i + N33 * (j0 + jz), Cz + i + N33 * jz, N33 * JB);
  }
  cp_async_wait_all();
  __syncthreads();
  // x: contracted i (stride 1), columns (jj, k); z: contracted k (stride 33 JB), columns (i, jj)
  eo33_lines<1, N33, N33 * JB, JB, JB * N33, N33 * JB, 1, JB, true>(U, Cx, V, afx);
  __syncthreads();
  eo33_lines<N33 * JB, 1, N33, N33, N33 * JB, N33 * JB, 1, N33, false>(U, Cz, V, afz);
  __syncthreads();
  for (int w = threadIdx.x; w < SL; w += blockDim.x) {
    const int k = w / (N33 * JB), r = w - k * N33 * JB;
    Vxz[e0 + (long long)k * N33_2 + j0 * N33 + r] = V[w];
  }
}

// smem: U [kk][j][i] (KB x 33 x 33) | V (same) | Cy [4][kk][i] | A table y | mass 3 x 33
__global__ void __launch_bounds__(128, 4) k_apply33_y(LevelDev L, const double *__restrict__ u,
                                                      const double *__restrict__ T,
                                                      const double *__restrict__ Vxz,
                                                      const double *__restrict__ f,
                                                      double *__restrict__ out) {
  extern __shared__ double sm[];
  constexpr int SL = KB * N33_2;
  double *U = sm, *V = U + SL, *Cy = V + SL, *afy = Cy + 4 * N33 * KB, *ms = afy + AF33;
  const int e = blockIdx.y, k0 = blockIdx.x * KB;
  const long long g0 = (long long)e * N33_3 + (long long)k0 * N33_2;   // the slab is contiguous
  for (int w = threadIdx.x; w < SL; w += blockDim.x) cp_async8(U + w, u + g0 + w);
  for (int d = 0; d < 3; ++d) stage(ms + d * N33, L.mass[d], N33);
  if ((threadIdx.x >> 5) == 0) afrag33(L.Daug[1], afy);
  for (int w = threadIdx.x; w < N33 * KB; w += blockDim.x) {  // y faces: point p = i + n k
    const int i = w % N33, kk = w / N33;
    face_coefs(L, T, e, 1, i + N33 * (k0 + kk), Cy + i + N33 * kk, N33 * KB);
  }
  cp_async_wait_all();
  __syncthreads();
  // y: contracted j (stride 33), columns (i, kk)
  eo33_lines<N33, 1, N33_2, N33, N33 * KB, N33 * KB, 1, N33, true>(U, Cy, V, afy);
  __syncthreads();
  for (int w = threadIdx.x; w < SL; w += blockDim.x) {
    const int i = w % N33, j = (w / N33) % N33, kk = w / N33_2;
    const double v = ms[i] * ms[N33 + j] * ms[2 * N33 + k0 + kk] * (V[w] + __ldg(Vxz + g0 + w));
    out[g0 + w] = f ? __ldg(f + g0 + w) - v : v;
  }
}

}  // namespace

bool apply33_ok(const LevelDev &L) {
#ifdef PMG_NO_APPLY33
  return false;
#endif
  return L.n == N33;
}

// V: scratch of Ne * 33^3 doubles (the x + z contributions)
cudaError_t launch_apply33(const LevelDev &L, const double *u, const double *T, const double *f,
                           double *out, double *V, cudaStream_t s) {
  const size_t sa = sizeof(double) * (2 * (size_t)N33 * JB * N33 + 8 * N33 * JB + 2 * AF33);
  const size_t sy = sizeof(double) * (2 * (size_t)KB * N33_2 + 4 * N33 * KB + AF33 + 3 * N33);
  static bool cfg = false;
  if (!cfg) {
    cfg = true;
    cudaFuncSetAttribute(k_apply33_xz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sa);
    cudaFuncSetAttribute(k_apply33_y, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sy);
  }
  k_apply33_xz<<<dim3(NSLAB, L.Ne), 128, sa, s>>>(L, u, T, V);
  k_apply33_y<<<dim3(NSLAB, L.Ne), 128, sy, s>>>(L, u, T, V, f, out);
  return cudaGetLastError();
}

}  // namespace pmg
