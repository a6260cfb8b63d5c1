// FP64 kernels of the p-multigrid V(1,1) hot path on B200 (sm_100a).
// arXiv:1612.04796; PAPER.md line numbers cited per kernel.
//
// Layout: element-major vectors, element e = ex + nx*(ey + ny*ez), node i + n*(j + n*k).
// Face-trace buffer T (per level): T[((e*3 + d)*4 + q)*n^2 + p], q = 0 left value,
// 1 left (2/D)-derivative, 2 right value, 3 right derivative; p = in-face node index
// (x-faces: j + n k, y-faces: i + n k, z-faces: i + n j).
#include <algorithm>

#include "kernels.cuh"

namespace pmg {

#ifndef PMG_LINES
#define PMG_LINES mma_lines_p
#endif
#ifndef FDM_BIG_THREADS
#define FDM_BIG_THREADS 256
#endif

namespace {

__device__ __forceinline__ int wrap(int a, int n) { return a < 0 ? a + n : (a >= n ? a - n : a); }

// Asynchronous 8-byte global->shared copies (LDGSTS): many loads in flight per thread.
__device__ __forceinline__ void cp_async8(double *smem, const double *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier (transaction bytes)
__device__ __forceinline__ unsigned smem_addr(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *mbar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_addr(mbar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *mbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_addr(mbar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(mbar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *mbar, unsigned phase) {
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_addr(mbar)), "r"(phase) : "memory");
}

// Plan a TMA copy of `count` doubles at `src` (8-byte aligned) into the 16-byte aligned staging
// area `buf` (capacity count + 2): copies the 16-byte aligned superset; returns the pointer to
// the first element inside `buf`, sets *bytes (0 if the superset would leave [src_base, src_end)).
struct BulkPlan { double *ptr; unsigned bytes; const double *src; };
__device__ __forceinline__ BulkPlan bulk_plan(double *buf, const double *src, int count,
                                              const double *src_end) {
  const int pre = (int)((reinterpret_cast<unsigned long long>(src) >> 3) & 1);
  const int cnt = (count + pre + 1) & ~1;
  BulkPlan b;
  b.ptr = buf + pre;
  b.src = src - pre;
  b.bytes = (b.src + cnt <= src_end) ? 8u * cnt : 0u;
  return b;
}

__device__ __forceinline__ void stage(double *dst, const double *src, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) cp_async8(dst + i, src + i);
}

// ---------------------------------------------------------------------------------------------
// Face traces (value and normal derivative on both faces of every direction) — the data the
// rank-2 neighbour couplings of Eq. 7's block-tridiagonal L_* need.
__global__ void k_traces(LevelDev L, const double *__restrict__ u, double *__restrict__ T) {
  const int n = L.n, n2 = n * n, n3 = n2 * n;
  const int e = blockIdx.x;
  const double *ue = u + (long long)e * n3;
  double *Te = T + (long long)e * 12 * n2;
  for (int t = threadIdx.x; t < 3 * n2; t += blockDim.x) {
    const int d = t / n2, p = t - d * n2;
    const int p0 = p % n, p1 = p / n;
    int base, stride;
    if (d == 0) { base = n * p0 + n2 * p1; stride = 1; }
    else if (d == 1) { base = p0 + n2 * p1; stride = n; }
    else { base = p0 + n * p1; stride = n2; }
    const double *tr = L.tr[d];
    double lv = 0, lder = 0, rv = 0, rder = 0;
    for (int i = 0; i < n; ++i) {
      const double v = __ldg(ue + base + i * stride);
      rv += tr[i] * v;
      rder += tr[n + i] * v;
      lv += tr[2 * n + i] * v;
      lder += tr[3 * n + i] * v;
    }
    double *Td = Te + d * 4 * n2;
    Td[p] = lv; Td[n2 + p] = lder; Td[2 * n2 + p] = rv; Td[3 * n2 + p] = rder;
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

// Generic 1D contraction along one axis of a (d0,d1,d2) block (d0 fastest):
// out[.., o, ..] = sum_k A[o*so + k*sk] * in[.., k, ..]; generic pointers (smem or global).
__device__ void contract_axis(const double *in, double *out, int d0, int d1, int d2, int ax,
                              const double *A, int so, int sk, int nout) {
  int od[3] = {d0, d1, d2};
  const int K = od[ax];
  od[ax] = nout;
  const int total = od[0] * od[1] * od[2];
  const int istr[3] = {1, d0, d0 * d1};
  const int st = istr[ax];
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    int p[3];
    p[0] = t % od[0];
    const int r = t / od[0];
    p[1] = r % od[1];
    p[2] = r / od[1];
    const int o = p[ax];
    p[ax] = 0;
    const double *src = in + p[0] + p[1] * d0 + p[2] * d0 * d1;
    const double *a = A + o * so;
    double acc = 0;
    for (int k = 0; k < K; ++k) acc += a[k * sk] * src[k * st];
    out[t] = acc;
  }
}

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

// ---------------------------------------------------------------------------------------------
// Tensor-core (DMMA m8n8k4 FP64) line contractions.  Every 1D contraction of the hot path
// (the six fast-diagonalisation passes and the three stiffness passes of the apply) is a small
// GEMM  C[o, (p,q)] = sum_k A[o, k] X[k along DIR, p, q]  over a 3D block in shared memory:
// A (the m x m eigenvector or stiffness matrix, zero padded to 8 x 4 multiples) stays in
// registers for the whole pass; a warp owns pairs of 8-column N-tiles (columns = 8 consecutive
// p at fixed q, so no per-lane index division), loads their K values (B fragments), issues
// MT x KS DMMAs per tile with 2*MT independent accumulator chains, and hands every result to
// an epilogue policy (store in place, divide by the eigenvalue sum, weight + store to global,
// or mass-weighted accumulation for the apply).
__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

struct Blk { int m[3]; int s[3]; };   // sizes and shared-memory strides (s[0] = 1)

// 1/x for x > 0: MUFU reciprocal seed + two Newton steps (relative error ~1 ulp)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);               // ~2^-46 relative
  e = fma(-x, r, 1.0);
  return fma(r, e, r);            // full precision (keeps the 1e-11 parity margin untouched)
}

template <int DIR> struct Other {
  static constexpr int P = DIR == 0 ? 1 : 0;   // lower of the two other directions
  static constexpr int Q = DIR == 2 ? 1 : 2;   // higher
};

// Generic form.  Output rows o < mo; main K rows k < mk read X[k*so + p*sp + q*sq] (stride
// and extents from B, contracted direction DIR); optional extra K rows k = mk + r (r < next)
// read Ext[r*esr + p*esp + q*esq] (used to fold the rank-2 face couplings of the apply into the
// same GEMM).  A[o][k] = Amat[o*ao + k*ak] for o < mo, k < mk + next, zero beyond.
struct LineSpec {
  int mo, mk;                 // output rows, main K extent
  const double *Amat; int ao, ak;
  const double *Ext; int next, esr, esp, esq;
};

// TAIL: the output extent is 8*MT + 1 (n = 2^l + 1 everywhere in this method); rows [0, 8 MT)
// go through DMMA and the last row through FP64 FMAs on the B fragments already in registers
// (each lane sums its k's, then a 2-step shuffle over the 4 lanes that share a column), which
// avoids padding 17 -> 24 (or 9 -> 16) rows on the tensor path.
template <int DIR, int KS, int MT, bool TAIL, class Epi>
__device__ __forceinline__ void mma_lines_t(const double *X, const Blk &B, const LineSpec &ls,
                                            Epi &epi) {
  constexpr int PD = Other<DIR>::P, QD = Other<DIR>::Q;
  const int mo = ls.mo, mk = ls.mk, kt = ls.mk + ls.next;
  const int mp = B.m[PD], mq = B.m[QD];
  const int ncol = mp * mq;                                 // columns (p, q), p fastest
  const unsigned magic = 0xFFFFFFFFu / (unsigned)mp + 1u;   // q = umulhi(n, magic) = n / mp
  const int so = B.s[DIR], sp = B.s[PD], sq = B.s[QD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double a[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int o = mt * 8 + g, k = ks * 4 + t;
      a[mt][ks] = (o < mo && k < kt) ? ls.Amat[o * ls.ao + k * ls.ak] : 0.0;
    }
  double at[TAIL ? KS : 1];
  if (TAIL) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = ks * 4 + t;
      at[ks] = k < kt ? ls.Amat[(8 * MT) * ls.ao + k * ls.ak] : 0.0;
    }
  }
  int koff[KS];
  bool kext[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = min(ks * 4 + t, kt - 1);
    kext[ks] = k >= mk;
    koff[ks] = kext[ks] ? (k - mk) * ls.esr : k * so;
  }
  const int ntiles = (ncol + 7) >> 3;
  for (int tile = 2 * warp; tile < ntiles; tile += 2 * nw) {
    double b[2][KS];
    int pbq[2], qbq[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int nb = min(min(tile + u, ntiles - 1) * 8 + g, ncol - 1);
      const int q = __umulhi((unsigned)nb, magic), p = nb - q * mp;
      pbq[u] = p; qbq[u] = q;
      const double *xb = X + p * sp + q * sq;
      const double *eb = ls.Ext ? ls.Ext + p * ls.esp + q * ls.esq : X;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) b[u][ks] = (kext[ks] ? eb : xb)[koff[ks]];
    }
    double c[2][MT][2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) { c[u][mt][0] = 0.0; c[u][mt][1] = 0.0; }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) dmma884(c[u][mt][0], c[u][mt][1], a[mt][ks], b[u][ks]);
    double tl[2] = {0.0, 0.0};
    if (TAIL) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) tl[u] = fma(at[ks], b[u][ks], tl[u]);
        tl[u] += __shfl_xor_sync(0xffffffffu, tl[u], 1);
        tl[u] += __shfl_xor_sync(0xffffffffu, tl[u], 2);
      }
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (tile + u >= ntiles) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = (tile + u) * 8 + 2 * t + j;
        if (n >= ncol) continue;
        const int q = __umulhi((unsigned)n, magic), p = n - q * mp;
        const double cf = epi.template col<DIR>(p, q);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int o = mt * 8 + g;
          if (o < mo) epi.template put<DIR>(o, p, q, cf, c[u][mt][j]);
        }
      }
      if (TAIL && t == 0 && (tile + u) * 8 + g < ncol) {
        const double cf = epi.template col<DIR>(pbq[u], qbq[u]);
        epi.template put<DIR>(8 * MT, pbq[u], qbq[u], cf, tl[u]);
      }
    }
  }
}

// Software-pipelined variant: one 8-column tile per step, the DMMAs of tile i+1 are issued
// before the epilogue of tile i, so the epilogue's shared-memory stores and index math fill the
// DMMA pipe's 16-cycle issue gaps instead of idling it (ping-pong accumulators c0/c1).
template <int DIR, int KS, int MT, bool TAIL, class Epi>
__device__ __forceinline__ void mma_lines_p(const double *X, const Blk &B, const LineSpec &ls,
                                            Epi &epi) {
  constexpr int PD = Other<DIR>::P, QD = Other<DIR>::Q;
  const int mo = ls.mo, mk = ls.mk, kt = ls.mk + ls.next;
  const int mp = B.m[PD], mq = B.m[QD];
  const int ncol = mp * mq;
  const unsigned magic = 0xFFFFFFFFu / (unsigned)mp + 1u;
  const int so = B.s[DIR], sp = B.s[PD], sq = B.s[QD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ntiles = (ncol + 7) >> 3;
  if (warp >= ntiles) return;
  double a[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int o = mt * 8 + g, k = ks * 4 + t;
      a[mt][ks] = (o < mo && k < kt) ? ls.Amat[o * ls.ao + k * ls.ak] : 0.0;
    }
  double at[TAIL ? KS : 1];
  if (TAIL) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = ks * 4 + t;
      at[ks] = k < kt ? ls.Amat[(8 * MT) * ls.ao + k * ls.ak] : 0.0;
    }
  }
  int koff[KS];
  bool kext[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = min(ks * 4 + t, kt - 1);
    kext[ks] = k >= mk;
    koff[ks] = kext[ks] ? (k - mk) * ls.esr : k * so;
  }
  // compute one tile into (c, tl); returns the column of the B loads (for the tail row)
  auto compute = [&](int tile, double (&c)[MT][2], double &tl, int &pb, int &qb) {
    const int nb = min(tile * 8 + g, ncol - 1);
    qb = __umulhi((unsigned)nb, magic);
    pb = nb - qb * mp;
    const double *xb = X + pb * sp + qb * sq;
    const double *eb = ls.Ext ? ls.Ext + pb * ls.esp + qb * ls.esq : X;
    double b[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) b[ks] = (kext[ks] ? eb : xb)[koff[ks]];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) { c[mt][0] = 0.0; c[mt][1] = 0.0; }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) dmma884(c[mt][0], c[mt][1], a[mt][ks], b[ks]);
    tl = 0.0;
    if (TAIL) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) tl = fma(at[ks], b[ks], tl);
      tl += __shfl_xor_sync(0xffffffffu, tl, 1);
      tl += __shfl_xor_sync(0xffffffffu, tl, 2);
    }
  };
  auto epilogue = [&](int tile, const double (&c)[MT][2], double tl, int pb, int qb) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int n = tile * 8 + 2 * t + j;
      if (n >= ncol) continue;
      const int q = __umulhi((unsigned)n, magic), p = n - q * mp;
      const double cf = epi.template col<DIR>(p, q);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int o = mt * 8 + g;
        if (o < mo) epi.template put<DIR>(o, p, q, cf, c[mt][j]);
      }
    }
    if (TAIL && t == 0 && tile * 8 + g < ncol) {
      const double cf = epi.template col<DIR>(pb, qb);
      epi.template put<DIR>(8 * MT, pb, qb, cf, tl);
    }
  };
  double c0[MT][2], c1[MT][2], tl0, tl1;
  int pb0, qb0, pb1, qb1;
  int tile = warp;
  compute(tile, c0, tl0, pb0, qb0);
  for (;;) {
    const int t1 = tile + nw;
    if (t1 < ntiles) compute(t1, c1, tl1, pb1, qb1);
    __syncwarp();
    epilogue(tile, c0, tl0, pb0, qb0);
    if (t1 >= ntiles) break;
    const int t2 = t1 + nw;
    if (t2 < ntiles) compute(t2, c0, tl0, pb0, qb0);
    __syncwarp();
    epilogue(t1, c1, tl1, pb1, qb1);
    if (t2 >= ntiles) break;
    tile = t2;
  }
}

// Supported (KS, MT) tiles; any request is served by the smallest supported tile that covers
// it (A is zero padded, so a larger tile is correct, only wasteful).
template <int DIR, int KSMAX, class Epi>
__device__ void mma_lines_gen(const double *X, const Blk &B, const LineSpec &ls, Epi &epi) {
  const int KS = (ls.mk + ls.next + 3) >> 2, MT = (ls.mo + 7) >> 3;
  if (ls.mo > 8 && (ls.mo & 7) == 1) {           // 8k+1 rows: DMMA for 8k, FMA tail row
    const int MTT = ls.mo >> 3;
#define PMG_TTILE(ks, mt) \
    if (ks <= KSMAX && KS <= ks && MTT == mt) { PMG_LINES<DIR, (ks <= KSMAX ? ks : 1), mt, true>(X, B, ls, epi); return; }
    PMG_TTILE(2, 1) PMG_TTILE(3, 1) PMG_TTILE(4, 1) PMG_TTILE(5, 1) PMG_TTILE(3, 2) PMG_TTILE(5, 2)
    PMG_TTILE(6, 2)
#undef PMG_TTILE
  }
#define PMG_TILE(ks, mt) \
  if (ks <= KSMAX && KS <= ks && MT <= mt) { PMG_LINES<DIR, (ks <= KSMAX ? ks : 1), mt, false>(X, B, ls, epi); return; }
  PMG_TILE(1, 1) PMG_TILE(2, 1) PMG_TILE(2, 2) PMG_TILE(3, 1) PMG_TILE(3, 2) PMG_TILE(3, 3)
  PMG_TILE(4, 2) PMG_TILE(5, 2) PMG_TILE(5, 3) PMG_TILE(6, 3) PMG_TILE(7, 4) PMG_TILE(8, 4)
#undef PMG_TILE
  __trap();   // callers only use tiles up to K = 32, M = 32 (checked on the host)
}

// square contraction (FDM passes): A[o][k] = Amat[o*ao + k*ak], mo = mk = extent along DIR
template <int DIR, int KSMAX, class Epi>
__device__ __forceinline__ void mma_lines_dispatch(const double *X, const Blk &B, const double *Amat,
                                                   int ao, int ak, Epi &epi) {
  const LineSpec ls = {B.m[DIR], B.m[DIR], Amat, ao, ak, nullptr, 0, 0, 0, 0};
  mma_lines_gen<DIR, KSMAX>(X, B, ls, epi);
}

template <int DIR>
__device__ __forceinline__ int blk_index(const Blk &B, int o, int p, int q) {
  return o * B.s[DIR] + p * B.s[Other<DIR>::P] + q * B.s[Other<DIR>::Q];
}

// in-place store
struct EpiStore {
  double *X; Blk B;
  template <int DIR> __device__ __forceinline__ double col(int, int) const { return 0.0; }
  template <int DIR> __device__ __forceinline__ void put(int o, int p, int q, double, double v) const {
    X[blk_index<DIR>(B, o, p, q)] = v;
  }
};
// in-place store divided by lam_x + lam_y + lam_z (fast-diagonalisation divide)
struct EpiDivide {
  double *X; Blk B; const double *lam[3];
  template <int DIR> __device__ __forceinline__ double col(int p, int q) const {
    return lam[Other<DIR>::P][p] + lam[Other<DIR>::Q][q];
  }
  template <int DIR> __device__ __forceinline__ void put(int o, int p, int q, double cf, double v) const {
    X[blk_index<DIR>(B, o, p, q)] = v * rcp_nr(cf + lam[DIR][o]);
  }
};
// weight W_x W_y W_z and store the window to global memory (unpadded window order)
struct EpiWeightStore {
  double *Zg; Blk G; const double *W[3];
  template <int DIR> __device__ __forceinline__ double col(int p, int q) const {
    return W[Other<DIR>::P][p] * W[Other<DIR>::Q][q];
  }
  template <int DIR> __device__ __forceinline__ void put(int o, int p, int q, double cf, double v) const {
    Zg[blk_index<DIR>(G, o, p, q)] = v * (cf * W[DIR][o]);
  }
};
// weight and scatter-add straight into u (colored, race-free): window node (a,b,c) lives at
// u[xo[a] + yo[b] + zo[c]]; fire-and-forget FP64 reductions (RED.ADD.F64) at L2
struct EpiWeightRed {
  double *u; const long long *offs; int m0, m1; const double *W[3];
  template <int DIR> __device__ __forceinline__ double col(int p, int q) const {
    return W[Other<DIR>::P][p] * W[Other<DIR>::Q][q];
  }
  template <int DIR> __device__ __forceinline__ void put(int o, int p, int q, double cf, double v) const {
    static_assert(DIR == 0, "the scatter pass runs along x");
    atomicAdd(u + offs[o] + offs[m0 + p] + offs[m0 + m1 + q], v * (cf * W[0][o]));
  }
};
// plain accumulation into V (first pass stores)
struct EpiAcc {
  double *V; Blk B; bool first;
  template <int DIR> __device__ __forceinline__ double col(int, int) const { return 0.0; }
  template <int DIR> __device__ __forceinline__ void put(int o, int p, int q, double, double v) const {
    const int w = blk_index<DIR>(B, o, p, q);
    if (first) V[w] = v;
    else V[w] += v;
  }
};

// Fused z passes of the fast diagonalisation: forward S_z^T, eigen-divide, backward S_z on the
// same z columns.  A warp owns its columns through both GEMMs, so no block barrier is needed
// between them (only __syncwarp around the in-place round trip through shared memory).
template <int KS, int MT>
__device__ __forceinline__ void fdm_z_fused_t(double *X, const Blk &B, const double *S,
                                              const double *const *lam) {
  const int md = B.m[2], mp = B.m[0], mq = B.m[1];
  const int ncol = mp * mq;
  const unsigned magic = 0xFFFFFFFFu / (unsigned)mp + 1u;
  const int so = B.s[2], sq = B.s[1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double af[MT][KS], ab[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int o = mt * 8 + g, k = ks * 4 + t;
      const bool ok = o < md && k < md;
      af[mt][ks] = ok ? S[k * md + o] : 0.0;
      ab[mt][ks] = ok ? S[o * md + k] : 0.0;
    }
  int koff[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) koff[ks] = min(ks * 4 + t, md - 1) * so;
  const int ntiles = (ncol + 7) >> 3;
  for (int tile = warp; tile < ntiles; tile += nw) {
    const int nb = min(tile * 8 + g, ncol - 1);
    const int qb = __umulhi((unsigned)nb, magic), pb = nb - qb * mp;
    const double *xb = X + pb + qb * sq;
    double b[KS], c[MT][2];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) b[ks] = xb[koff[ks]];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) { c[mt][0] = 0.0; c[mt][1] = 0.0; }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) dmma884(c[mt][0], c[mt][1], af[mt][ks], b[ks]);
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
        if (o < md) X[wb[j] + o * so] = c[mt][j] * rcp_nr(cf + lam[2][o]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) b[ks] = xb[koff[ks]];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) { c[mt][0] = 0.0; c[mt][1] = 0.0; }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) dmma884(c[mt][0], c[mt][1], ab[mt][ks], b[ks]);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (wb[j] < 0) continue;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int o = mt * 8 + g;
        if (o < md) X[wb[j] + o * so] = c[mt][j];
      }
    }
  }
}

// returns false if the window is too large for the fused register budget (caller falls back)
template <int KSMAX>
__device__ __forceinline__ bool fdm_z_fused(double *X, const Blk &B, const double *S,
                                            const double *const *lam) {
  const int KS = (B.m[2] + 3) >> 2;
#ifdef PMG_NO_ZFUSE
  return false;
#endif
  if (KS <= 1) { fdm_z_fused_t<1, 1>(X, B, S, lam); return true; }
  if (KS <= 2) { fdm_z_fused_t<2, 1>(X, B, S, lam); return true; }
  if (KSMAX >= 4 && KS <= 4) { fdm_z_fused_t<(KSMAX >= 4 ? 4 : 1), 2>(X, B, S, lam); return true; }
  if (KSMAX >= 6 && KS <= 6) { fdm_z_fused_t<(KSMAX >= 6 ? 6 : 1), 3>(X, B, S, lam); return true; }
  return false;
}

// ---- building blocks of the subdomain solve (shared by the one-shot and persistent kernels)
// gather offsets of subdomain e: global address of window node (a,b,c) = xo[a] + yo[b] + zo[c]
__device__ __forceinline__ void fdm_offsets(const LevelDev &L, int e, long long *offs) {
  const int n = L.n, n3 = n * n * n;
  const int ec[3] = {e % L.nx, (e / L.nx) % L.ny, e / (L.nx * L.ny)};
  const int edim[3] = {L.nx, L.ny, L.nz};
  const long long estride[3] = {(long long)n3, (long long)L.nx * n3, (long long)L.nx * L.ny * n3};
  const int lstride[3] = {1, n, n * n};
  int base = 0;
  for (int d = 0; d < 3; ++d) {
    const int no = L.no[d];
    for (int a = threadIdx.x; a < L.m[d]; a += blockDim.x) {
      const int o = a < no ? -1 : (a < no + n ? 0 : 1);
      const int li = a < no ? n - no + a : (a < no + n ? a - no : a - no - n);
      offs[base + a] = wrap(ec[d] + o, edim[d]) * estride[d] + li * lstride[d];
    }
    base += L.m[d];
  }
}

__device__ __forceinline__ void fdm_gather(const LevelDev &L, const double *r, const long long *offs,
                                           double *X) {
  const int m0 = L.m[0], m1 = L.m[1], m2 = L.m[2];
  const long long *xo = offs, *yo = offs + m0, *zo = offs + m0 + m1;
  if (m0 <= 32) {
    // one warp per window row (b, c), lane = a: the row base is warp-uniform, xo[a] per lane
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const long long xa = lane < m0 ? xo[lane] : 0;
    const int rows = m1 * m2;
    int b = warp % m1, c = warp / m1;
    const int db = nw % m1, dc = nw / m1;
    for (int row = warp; row < rows; row += nw) {
      if (lane < m0) cp_async8(X + lane + m0 * row, r + xa + yo[b] + zo[c]);
      b += db; c += dc;
      if (b >= m1) { b -= m1; ++c; }
    }
    return;
  }
  const int total = L.Mw;
  int a = threadIdx.x % m0, bc = threadIdx.x / m0;
  int b = bc % m1, c = bc / m1;
  const int da = blockDim.x % m0, dbc = blockDim.x / m0;
  for (int w = threadIdx.x; w < total; w += blockDim.x) {
    cp_async8(X + w, r + xo[a] + yo[b] + zo[c]);
    a += da; b += dbc;
    if (a >= m0) { a -= m0; ++b; }
    while (b >= m1) { b -= m1; ++c; }
  }
}

template <int KSMAX>
__device__ __forceinline__ void fdm_phases(double *X, const int *m, double *const *Ss,
                                           const double *const *lam, const double *const *W,
                                           double *Ze, double *ured = nullptr,
                                           const long long *offs = nullptr) {
  const Blk B = {{m[0], m[1], m[2]}, {1, m[0], m[0] * m[1]}};
  EpiStore st{X, B};
  EpiDivide dv{X, B, {lam[0], lam[1], lam[2]}};
  EpiWeightStore ws{Ze, B, {W[0], W[1], W[2]}};
  EpiWeightRed wr{ured, offs, m[0], m[1], {W[0], W[1], W[2]}};
  mma_lines_dispatch<0, KSMAX>(X, B, Ss[0], 1, m[0], st); __syncthreads();
  mma_lines_dispatch<1, KSMAX>(X, B, Ss[1], 1, m[1], st); __syncthreads();
  if (!fdm_z_fused<KSMAX>(X, B, Ss[2], lam)) {
    mma_lines_dispatch<2, KSMAX>(X, B, Ss[2], 1, m[2], dv); __syncthreads();
    mma_lines_dispatch<2, KSMAX>(X, B, Ss[2], m[2], 1, st);
  }
  __syncthreads();
  mma_lines_dispatch<1, KSMAX>(X, B, Ss[1], m[1], 1, st); __syncthreads();
  if (ured) mma_lines_dispatch<0, KSMAX>(X, B, Ss[0], m[0], 1, wr);
  else mma_lines_dispatch<0, KSMAX>(X, B, Ss[0], m[0], 1, ws);
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

// smem: U (n^3) | V (n^3) | face coefficients 3 x 4 x n^2 | mass 3 x n
// Per direction d the line GEMM is  V += M_p M_q [D | a ap b bp] [U-lines ; c1 c2 c3 c4]  where
// c1..c4 are the neighbour-trace coefficients of the rank-2 couplings on the face point (p,q):
// c1 = -tdR/2 - mu tvR, c2 = tvR/2, c3 = tdL/2 - mu tvL, c4 = -tvL/2.
template <int KSMAX>
__global__ void __launch_bounds__(KSMAX <= 4 ? 128 : 256, KSMAX <= 4 ? 8 : 2) k_apply_mma(LevelDev L, const double *__restrict__ u,
                                                      const double *__restrict__ T,
                                                      const double *__restrict__ f,
                                                      double *__restrict__ out,
                                                      const double *__restrict__ restrict_I,
                                                      int nc, double *__restrict__ fc) {
  extern __shared__ double sm[];
  const int n = L.n, n2 = n * n, n3 = n2 * n;
  // smem: U staging (n^3 + 2, 16-byte aligned superset of the element) | V | Cf | mass | mbarrier
  double *Us = sm, *V = sm + n3 + 2, *Cf = V + n3, *ms = Cf + 12 * n2;
  unsigned long long *mbar = reinterpret_cast<unsigned long long *>(ms + 3 * n);
  const int e = blockIdx.x;
  const int ex = e % L.nx, ey = (e / L.nx) % L.ny, ez = e / (L.nx * L.ny);
  const int ecoord[3] = {ex, ey, ez};
  const int edim[3] = {L.nx, L.ny, L.nz};
  // TMA bulk staging: the element block and the six neighbour-trace segments (2 n^2 doubles,
  // 16-byte aligned) in 7 copies tracked by one mbarrier.  Element blocks (n^3 doubles, n odd)
  // alternate 8/16-byte alignment, so a 16-byte aligned superset is copied and U is offset.
  const double *ue = u + (long long)e * n3;
  const int pre = (int)((reinterpret_cast<unsigned long long>(ue) >> 3) & 1);
  const int ucount = (n3 + pre + 1) & ~1;                          // doubles, multiple of 2
  const bool tail_ok = (long long)e * n3 - pre + ucount <= (long long)L.Ne * n3;
  double *U = Us + pre;
  if (threadIdx.x == 0) {
    mbar_init(mbar, 1);
    const unsigned tbytes = 16u * n2;                              // 2 n^2 doubles
    mbar_expect_tx(mbar, (tail_ok ? ucount * 8u : 0u) + 6u * tbytes);
    if (tail_ok) bulk_g2s(Us, ue - pre, ucount * 8u, mbar);
    for (int d = 0; d < 3; ++d) {
      int c[3] = {ex, ey, ez};
      c[d] = wrap(ecoord[d] + 1, edim[d]);
      bulk_g2s(Cf + d * 4 * n2, T + ((long long)(c[0] + L.nx * (c[1] + L.ny * c[2])) * 3 + d) * 4 * n2,
               tbytes, mbar);                                      // tvR, tdR of the right nb
      c[d] = wrap(ecoord[d] - 1, edim[d]);
      bulk_g2s(Cf + d * 4 * n2 + 2 * n2,
               T + ((long long)(c[0] + L.nx * (c[1] + L.ny * c[2])) * 3 + d) * 4 * n2 + 2 * n2, tbytes,
               mbar);                                              // tvL, tdL of the left nb
    }
  }
  if (!tail_ok) stage(U, ue, n3);
  for (int d = 0; d < 3; ++d) stage(ms + d * n, L.mass[d], n);
  cp_async_wait_all();
  __syncthreads();
  mbar_wait(mbar, 0);
  __syncthreads();
  for (int t = threadIdx.x; t < 3 * n2; t += blockDim.x) {
    const int d = t / n2, pp = t - d * n2;
    double *C = Cf + d * 4 * n2 + pp;
    const double mu = L.mu[d];
    const double tvR = C[0], tdR = C[n2], tvL = C[2 * n2], tdL = C[3 * n2];
    C[0] = -0.5 * tdR - mu * tvR;
    C[n2] = 0.5 * tvR;
    C[2 * n2] = 0.5 * tdL - mu * tvL;
    C[3 * n2] = -0.5 * tvL;
  }
  __syncthreads();
  const Blk B = {{n, n, n}, {1, n, n2}};
  EpiAcc acc{V, B, true};
  LineSpec lx = {n, n, L.Daug[0], n + 4, 1, Cf, 4, n2, 1, n};
  mma_lines_gen<0, KSMAX>(U, B, lx, acc); __syncthreads();
  acc.first = false;
  LineSpec ly = {n, n, L.Daug[1], n + 4, 1, Cf + 4 * n2, 4, n2, 1, n};
  mma_lines_gen<1, KSMAX>(U, B, ly, acc); __syncthreads();
  LineSpec lz = {n, n, L.Daug[2], n + 4, 1, Cf + 8 * n2, 4, n2, 1, n};
  mma_lines_gen<2, KSMAX>(U, B, lz, acc); __syncthreads();
  // out = f - M v (or M v), M = Mz (x) My (x) Mx; f loads batched for memory-level parallelism
  const long long g0 = (long long)e * n3;
  constexpr int UNR = 4;
  for (int t0 = threadIdx.x; t0 < n3; t0 += UNR * blockDim.x) {
    double fv[UNR];
#pragma unroll
    for (int q = 0; q < UNR; ++q) {
      const int t = t0 + q * blockDim.x;
      fv[q] = (f && t < n3) ? __ldg(f + g0 + t) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < UNR; ++q) {
      const int t = t0 + q * blockDim.x;
      if (t >= n3) break;
      const int i = t % n, j = (t / n) % n, k = t / n2;
      const double v = ms[i] * ms[n + j] * ms[2 * n + k] * V[t];
      const double rr = f ? fv[q] - v : v;
      if (restrict_I) V[t] = rr;
      else out[g0 + t] = rr;
    }
  }
  if (restrict_I) {
    // fused residual restriction f_c = (I^T (x) I^T (x) I^T) r (Alg. 1 l.292): r stays in V;
    // x pass (n -> nc) into U, y pass into Cf, z pass straight to the coarse vector
    __syncthreads();
    const Blk T1 = {{nc, n, n}, {1, nc, nc * n}};
    const Blk T2 = {{nc, nc, n}, {1, nc, nc * nc}};
    const Blk FC = {{nc, nc, nc}, {1, nc, nc * nc}};
    const LineSpec rx = {nc, n, restrict_I, 1, nc, nullptr, 0, 0, 0, 0};
    EpiStore s1{U, T1};
    mma_lines_gen<0, KSMAX>(V, B, rx, s1); __syncthreads();
    EpiStore s2{Cf, T2};
    mma_lines_gen<1, KSMAX>(U, T1, rx, s2); __syncthreads();
    EpiStore s3{fc + (long long)e * nc * nc * nc, FC};
    mma_lines_gen<2, KSMAX>(Cf, T2, rx, s3);
  }
}

// Fused correction prolongation + face traces (Alg. 1 l.299 followed by the trace pass of the
// post-smoothing residual): u_f += (I (x) I (x) I) u_c with three DMMA line GEMMs in shared
// memory, u_f written back, and the traces of the new u_f emitted for the residual.
// smem: Uc (nc^3) | T1 (nf nc^2) | T2 (nf^2 nc) | U (nf^3) | trs (12 nf)
template <int KSMAX>
__global__ void __launch_bounds__(KSMAX <= 4 ? 128 : 256, KSMAX <= 4 ? 8 : 2) k_prolong_traces(LevelDev L, int nc, const double *__restrict__ I,
                                                        const double *__restrict__ uc,
                                                        double *__restrict__ uf,
                                                        double *__restrict__ T) {
  extern __shared__ double sm[];
  const int nf = L.n, n2 = nf * nf, n3 = n2 * nf;
  const int c3 = nc * nc * nc;
  const int c3p = (c3 + 3) & ~1;                // staging capacities (16-byte aligned regions)
  double *Ucs = sm, *Us = Ucs + c3p;
  double *T1 = Us + ((n3 + 3) & ~1), *T2 = T1 + nf * nc * nc, *trs = T2 + nf * nf * nc;
  unsigned long long *mbar = reinterpret_cast<unsigned long long *>(trs + 12 * nf);
  const int e = blockIdx.x;
  const BulkPlan bc = bulk_plan(Ucs, uc + (long long)e * c3, c3, uc + (long long)L.Ne * c3);
  const BulkPlan bf = bulk_plan(Us, uf + (long long)e * n3, n3, uf + (long long)L.Ne * n3);
  double *Uc = bc.ptr, *U = bf.ptr;
  if (threadIdx.x == 0 && (bc.bytes || bf.bytes)) {
    mbar_init(mbar, 1);
    mbar_expect_tx(mbar, bc.bytes + bf.bytes);
    if (bc.bytes) bulk_g2s(Ucs, bc.src, bc.bytes, mbar);
    if (bf.bytes) bulk_g2s(Us, bf.src, bf.bytes, mbar);
  }
  if (!bc.bytes) stage(Uc, uc + (long long)e * c3, c3);
  if (!bf.bytes) stage(U, uf + (long long)e * n3, n3);
  for (int d = 0; d < 3; ++d) stage(trs + d * 4 * nf, L.tr[d], 4 * nf);
  cp_async_wait_all();
  __syncthreads();
  if (bc.bytes || bf.bytes) mbar_wait(mbar, 0);
  const Blk BC = {{nc, nc, nc}, {1, nc, nc * nc}};
  const Blk B1 = {{nf, nc, nc}, {1, nf, nf * nc}};
  const Blk B2 = {{nf, nf, nc}, {1, nf, nf * nf}};
  const Blk BF = {{nf, nf, nf}, {1, nf, n2}};
  const LineSpec px = {nf, nc, I, nc, 1, nullptr, 0, 0, 0, 0};   // A[o][k] = I[o*nc + k]
  EpiStore s1{T1, B1};
  mma_lines_gen<0, KSMAX>(Uc, BC, px, s1); __syncthreads();
  EpiStore s2{T2, B2};
  mma_lines_gen<1, KSMAX>(T1, B1, px, s2); __syncthreads();
  EpiAcc acc{U, BF, false};
  mma_lines_gen<2, KSMAX>(T2, B2, px, acc); __syncthreads();
  double *ue = uf + (long long)e * n3;
  for (int t = threadIdx.x; t < n3; t += blockDim.x) ue[t] = U[t];
  double *Te = T + (long long)e * 12 * n2;
  for (int t = threadIdx.x; t < 3 * n2; t += blockDim.x) {
    const int d = t / n2, p = t - d * n2;
    const int p0 = p % nf, p1 = p / nf;
    int base, stride;
    if (d == 0) { base = nf * p0 + n2 * p1; stride = 1; }
    else if (d == 1) { base = p0 + n2 * p1; stride = nf; }
    else { base = p0 + nf * p1; stride = n2; }
    const double *tr = trs + d * 4 * nf;
    double lv = 0, lder = 0, rv = 0, rder = 0;
    for (int i = 0; i < nf; ++i) {
      const double v = U[base + i * stride];
      rv += tr[i] * v;
      rder += tr[nf + i] * v;
      lv += tr[2 * nf + i] * v;
      lder += tr[3 * nf + i] * v;
    }
    double *Td = Te + d * 4 * n2;
    Td[p] = lv; Td[n2 + p] = lder; Td[2 * n2 + p] = rv; Td[3 * n2 + p] = rder;
  }
}

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

// Face traces with the element staged in shared memory (coalesced loads).
__global__ void __launch_bounds__(256) k_traces_sm(LevelDev L, const double *__restrict__ u,
                                                   double *__restrict__ T) {
  extern __shared__ double sm[];
  const int n = L.n, n2 = n * n, n3 = n2 * n;
  double *Us = sm, *trs = sm + n3 + 2;
  unsigned long long *mbar = reinterpret_cast<unsigned long long *>(trs + 12 * n);
  const int e = blockIdx.x;
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
  for (int d = 0; d < 3; ++d) stage(trs + d * 4 * n, L.tr[d], 4 * n);
  cp_async_wait_all();
  __syncthreads();
  if (bp.bytes) mbar_wait(mbar, 0);
  double *Te = T + (long long)e * 12 * n2;
  for (int t = threadIdx.x; t < 3 * n2; t += blockDim.x) {
    const int d = t / n2, p = t - d * n2;
    const int p0 = p % n, p1 = p / n;
    int base, stride;
    if (d == 0) { base = n * p0 + n2 * p1; stride = 1; }
    else if (d == 1) { base = p0 + n2 * p1; stride = n; }
    else { base = p0 + n * p1; stride = n2; }
    const double *tr = trs + d * 4 * n;
    double lv = 0, lder = 0, rv = 0, rder = 0;
    for (int i = 0; i < n; ++i) {
      const double v = U[base + i * stride];
      rv += tr[i] * v;
      rder += tr[n + i] * v;
      lv += tr[2 * n + i] * v;
      lder += tr[3 * n + i] * v;
    }
    double *Td = Te + d * 4 * n2;
    Td[p] = lv; Td[n2 + p] = lder; Td[2 * n2 + p] = rv; Td[3 * n2 + p] = rder;
  }
}

// Register-only fold: one thread per DOF issues all (up to 27) predicated loads of the
// weighted window values that cover it before summing them in a fixed order -> maximal
// memory-level parallelism, deterministic result.  NT = compile-time n (fast index math).
template <int NT, bool TR>
__global__ void __launch_bounds__(256) k_fold2(LevelDev L, const double *__restrict__ Z,
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
  for (int t = threadIdx.x; t < n3; t += blockDim.x) {
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
  const int n2 = n * n;
  double *trs = sm + n3;
  for (int d = 0; d < 3; ++d)
    for (int i = threadIdx.x; i < 4 * n; i += blockDim.x) trs[d * 4 * n + i] = L.tr[d][i];
  __syncthreads();
  double *Te = T + (long long)e * 12 * n2;
  for (int t = threadIdx.x; t < 3 * n2; t += blockDim.x) {
    const int d = t / n2, p = t - d * n2;
    const int p0 = p % n, p1 = p / n;
    int base, stride;
    if (d == 0) { base = n * p0 + n2 * p1; stride = 1; }
    else if (d == 1) { base = p0 + n2 * p1; stride = n; }
    else { base = p0 + n * p1; stride = n2; }
    const double *tr = trs + d * 4 * n;
    double lv = 0, lder = 0, rv = 0, rder = 0;
    for (int i = 0; i < n; ++i) {
      const double v = sm[base + i * stride];
      rv += tr[i] * v;
      rder += tr[n + i] * v;
      lv += tr[2 * n + i] * v;
      lder += tr[3 * n + i] * v;
    }
    double *Td = Te + d * 4 * n2;
    Td[p] = lv; Td[n2 + p] = lder; Td[2 * n2 + p] = rv; Td[3 * n2 + p] = rder;
  }
}

// Residual restriction f_c = I^T r_f per element (Alg. 1 l.292).
__global__ void k_restrict(int nf, int nc, const double *__restrict__ I,
                           const double *__restrict__ rf, double *__restrict__ fc) {
  extern __shared__ double sm[];
  const int e = blockIdx.x;
  double *t1 = sm, *t2 = sm + nc * nf * nf;
  const double *in = rf + (long long)e * nf * nf * nf;
  contract_axis(in, t1, nf, nf, nf, 0, I, 1, nc, nc); __syncthreads();
  contract_axis(t1, t2, nc, nf, nf, 1, I, 1, nc, nc); __syncthreads();
  contract_axis(t2, fc + (long long)e * nc * nc * nc, nc, nc, nf, 2, I, 1, nc, nc);
}

// Correction prolongation u_f += I u_c per element (Alg. 1 l.299).
__global__ void k_prolong(int nf, int nc, const double *__restrict__ I,
                          const double *__restrict__ uc, double *__restrict__ uf) {
  extern __shared__ double sm[];
  const int e = blockIdx.x;
  double *t1 = sm, *t2 = sm + nf * nc * nc;
  const double *in = uc + (long long)e * nc * nc * nc;
  contract_axis(in, t1, nc, nc, nc, 0, I, nc, 1, nf); __syncthreads();
  contract_axis(t1, t2, nf, nc, nc, 1, I, nc, 1, nf); __syncthreads();
  const int total = nf * nf * nf;
  double *ue = uf + (long long)e * total;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int i = t % nf, j = (t / nf) % nf, k = t / (nf * nf);
    const double *src = t2 + i + nf * j;
    const double *a = I + k * nc;
    double acc = 0;
    for (int c = 0; c < nc; ++c) acc += a[c] * src[c * nf * nf];
    ue[t] += acc;
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

inline int grid_for(long long N, int bs) {
  long long g = (N + bs - 1) / bs;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
cudaError_t launch_traces(const LevelDev &L, const double *u, double *T, cudaStream_t s) {
  const int n = L.n;
  const size_t sb = sizeof(double) * ((size_t)n * n * n + 2 + 12 * n + 2);
  if (n <= 20) {
    static size_t configured = 0;
    if (sb > 48 * 1024 && sb > configured) {
      cudaFuncSetAttribute(k_traces_sm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
      configured = sb;
    }
    k_traces_sm<<<L.Ne, 256, sb, s>>>(L, u, T);
  } else {
    k_traces<<<L.Ne, 128, 0, s>>>(L, u, T);
  }
  return cudaGetLastError();
}
// allow up to 227 KB of dynamic shared memory for every shared-memory kernel variant (once)
static void configure_smem() {
  static bool done = false;
  if (done) return;
  done = true;
  const int mx = 227 * 1024;
  cudaFuncSetAttribute(k_fdm_mma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_fdm_mma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_fdm_mma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_apply_mma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_apply_mma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_apply_mma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_prolong_traces<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_prolong_traces<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_prolong_traces<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
}

static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

static size_t apply_pipe_smem(int n) {
  const size_t n2 = (size_t)n * n, n3 = n2 * n;
  return sizeof(double) * (3 * n3 + 24 * n2 + 3 * n);
}

bool apply_pipe_ok(const LevelDev &L) { return L.n <= 17; }

cudaError_t launch_fdm_global(const LevelDev &L, const double *r, double *X, double *Y, double *Z,
                              cudaStream_t s) {
  const long long bs = L.Mw;
  const Blk B = {{L.m[0], L.m[1], L.m[2]}, {1, L.m[0], L.m[0] * L.m[1]}};
  const long long total = (long long)L.Ne * L.Mw;
  k_gather_win<<<grid_for(total, 256), 256, 0, s>>>(L, r, X);
  const int *m = L.m;
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

static size_t prolong_traces_smem(int nf, int nc) {
  return sizeof(double) * ((size_t)nc * nc * nc + 4 + (size_t)nf * nc * nc + (size_t)nf * nf * nc +
                           (size_t)nf * nf * nf + 4 + 12 * (size_t)nf + 2);
}

bool prolong_traces_ok(const LevelDev &Lf, int nc) {
  return Lf.n <= 17 && prolong_traces_smem(Lf.n, nc) <= 200 * 1024;
}

cudaError_t launch_prolong_traces(const LevelDev &Lf, int nc, const double *I, const double *uc,
                                  double *uf, double *T, cudaStream_t s) {
  configure_smem();
  const size_t sb = prolong_traces_smem(Lf.n, nc);
  if (Lf.n >= 17) k_prolong_traces<8><<<Lf.Ne, 256, sb, s>>>(Lf, nc, I, uc, uf, T);   // big blocks: 8 warps
  else if (((nc + 3) >> 2) <= 2) k_prolong_traces<2><<<Lf.Ne, 128, sb, s>>>(Lf, nc, I, uc, uf, T);
  else if (((nc + 3) >> 2) <= 4) k_prolong_traces<4><<<Lf.Ne, 128, sb, s>>>(Lf, nc, I, uc, uf, T);
  else k_prolong_traces<8><<<Lf.Ne, 256, sb, s>>>(Lf, nc, I, uc, uf, T);
  return cudaGetLastError();
}

static size_t apply_mma_smem(int n) {
  const size_t n2 = (size_t)n * n, n3 = n2 * n;
  return sizeof(double) * (2 * n3 + 2 + 12 * n2 + 3 * n + 2);
}

cudaError_t launch_apply_pipe(const LevelDev &L, const double *u, const double *T, const double *f,
                              double *out, const double *I, int nc, double *fc, cudaStream_t s) {
  configure_smem();
  const size_t sb = apply_mma_smem(L.n);
  const int ks = (L.n + 4 + 3) >> 2;
  if (ks <= 2) k_apply_mma<2><<<L.Ne, 128, sb, s>>>(L, u, T, f, out, I, nc, fc);
  else if (ks <= 4) k_apply_mma<4><<<L.Ne, 128, sb, s>>>(L, u, T, f, out, I, nc, fc);
  else k_apply_mma<8><<<L.Ne, 256, sb, s>>>(L, u, T, f, out, I, nc, fc);
  return cudaGetLastError();
}

cudaError_t launch_apply(const LevelDev &L, const double *u, const double *T, const double *f,
                         double *out, cudaStream_t s) {
  const int n = L.n;

  if (n <= 17) {
    return launch_apply_pipe(L, u, T, f, out, nullptr, 0, nullptr, s);
  } else {
    k_apply<<<L.Ne, 256, 0, s>>>(L, u, T, f, out);
  }
  return cudaGetLastError();
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
  for (int color = 0; color < 8; ++color) {
    if (ks <= 2) k_fdm_mma<2><<<grid, 128, sb, s>>>(L, r, nullptr, color, u);
    else if (ks <= 4) k_fdm_mma<4><<<grid, 128, sb, s>>>(L, r, nullptr, color, u);
    else k_fdm_mma<8><<<grid, FDM_BIG_THREADS, sb, s>>>(L, r, nullptr, color, u);
  }
  return cudaGetLastError();
}

cudaError_t launch_fdm(const LevelDev &L, const double *r, double *Z, double *scr, bool smem,
                       size_t smem_bytes, cudaStream_t s) {
  if (fdm_mma_ok(L)) {
    configure_smem();
    const size_t sb = fdm_mma_smem_bytes(L);
    const int ks = (std::max(L.m[0], std::max(L.m[1], L.m[2])) + 3) >> 2;
    if (ks <= 2) k_fdm_mma<2><<<L.Ne, 128, sb, s>>>(L, r, Z, -1, nullptr);
    else if (ks <= 4) k_fdm_mma<4><<<L.Ne, 128, sb, s>>>(L, r, Z, -1, nullptr);
    else k_fdm_mma<8><<<L.Ne, FDM_BIG_THREADS, sb, s>>>(L, r, Z, -1, nullptr);
    return cudaGetLastError();
  }
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
cudaError_t launch_fold(const LevelDev &L, const double *Z, double *u, bool zero, double *T,
                        cudaStream_t s) {
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
  if (T && (sb > 200 * 1024 || L.n < 9)) {   // n = 33: no room; n < 9: separate kernels are faster
    if (L.n == 33) k_fold2<33, false><<<L.Ne, 256, 0, s>>>(L, Z, u, z, nullptr);
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
    case 33: PMG_FOLD(33) break;
    default: PMG_FOLD(0) break;
  }
#undef PMG_FOLD
  cudaError_t e = cudaGetLastError();
  return e;
}
static size_t xfer_smem(int nf, int nc) {
  return sizeof(double) * ((size_t)nc * nf * nf + (size_t)nc * nc * nf);
}
cudaError_t launch_restrict(const LevelDev &Lf, int nc, const double *I, const double *rf,
                            double *fc, cudaStream_t s) {
  const size_t sb = xfer_smem(Lf.n, nc);
  static size_t configured = 0;
  if (sb > 48 * 1024 && sb > configured) {
    cudaFuncSetAttribute(k_restrict, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
    configured = sb;
  }
  k_restrict<<<Lf.Ne, 256, sb, s>>>(Lf.n, nc, I, rf, fc);
  return cudaGetLastError();
}
cudaError_t launch_prolong(const LevelDev &Lf, int nc, const double *I, const double *uc,
                           double *uf, cudaStream_t s) {
  const size_t sb = xfer_smem(Lf.n, nc);
  static size_t configured = 0;
  if (sb > 48 * 1024 && sb > configured) {
    cudaFuncSetAttribute(k_prolong, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
    configured = sb;
  }
  k_prolong<<<Lf.Ne, 256, sb, s>>>(Lf.n, nc, I, uc, uf);
  return cudaGetLastError();
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
cudaError_t launch_coarse_fused(const LevelDev &L0, const CoarseDev &C, const double *f0,
                                double *G1, double *G2, double *u0, cudaStream_t s) {
  const long long N = (long long)C.G[0] * C.G[1] * C.G[2];
  const long long cols = (long long)C.G[0] * C.G[1];
  k_coarse_xf<<<grid_for(N, 256), 256, 0, s>>>(C, L0.nx, L0.ny, f0, G1);
  k_lex_contract<<<grid_for(N, 256), 256, 0, s>>>(C, 1, 1, G1, G2);
  if (C.G[2] > 32) return cudaErrorInvalidValue;
  k_coarse_z<<<grid_for(cols * 32, 256), 256, 0, s>>>(C, G2);
  k_lex_contract<<<grid_for(N, 256), 256, 0, s>>>(C, 1, 0, G2, G1);
  k_coarse_xb<<<grid_for(N, 256), 256, 0, s>>>(C, L0.nx, L0.ny, G1, u0);
  return cudaGetLastError();
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
cudaError_t launch_rhs_sin(const LevelDev &L, double dx, double dy, double dz, double amp,
                           double kx, double ky, double kz, double *b, cudaStream_t s) {
  k_rhs_sin<<<grid_for((long long)L.Ne * L.n * L.n * L.n, 256), 256, 0, s>>>(L, dx, dy, dz, amp,
                                                                             kx, ky, kz, b);
  return cudaGetLastError();
}

}  // namespace pmg
