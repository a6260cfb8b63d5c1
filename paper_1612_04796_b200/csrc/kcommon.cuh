#pragma once
// Shared device building blocks of the FP64 kernels (included by every kern_*.cu).
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

// Order this thread's (and, after a CTA barrier, the CTA's) generic-proxy shared-memory accesses
// before subsequent async-proxy (cp.async.bulk) writes to the same buffer (PTX cross-proxy rule).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// L2 prefetch of a 16-byte aligned block (cp.async.bulk.prefetch.L2; no shared memory used)
__device__ __forceinline__ void prefetch_l2(const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// L2 prefetch of `count` doubles at `src` (8-byte aligned): the 16-byte aligned interior of the range.
// Kernels whose CTAs start with a cold read of one contiguous block per element issue this for the
// element a fixed number of CTAs ahead, so that the later CTA's loads are L2 hits.
__device__ __forceinline__ void prefetch_l2_doubles(const double *src, long long count) {
  const unsigned long long a = reinterpret_cast<unsigned long long>(src);
  const unsigned skip = (a & 15) ? 1 : 0;
  const long long bytes = ((count - skip) * 8) & ~15ll;
  if (bytes > 0) prefetch_l2(src + skip, (unsigned)bytes);
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

// Compile-time tile choice (output rows MO, K extent KT known statically): exactly one tile
// variant is inlined, so the kernel's register allocation is that tile's, not the maximum over
// every runtime-dispatchable tile.
template <int DIR, int MO, int KT, class Epi>
__device__ __forceinline__ void mma_lines_ct(const double *X, const Blk &B, const LineSpec &ls, Epi &epi) {
  constexpr bool TAIL = MO > 8 && (MO & 7) == 1;
  constexpr int MT = TAIL ? MO / 8 : (MO + 7) / 8;
  constexpr int KS = (KT + 3) / 4;
  PMG_LINES<DIR, KS, MT, TAIL>(X, B, ls, epi);
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


// ---- face traces of one element held in shared memory ---------------------------------------
// Eq. 7's rank-2 face couplings need, per face point, the value and the
// (2/Delta)-scaled normal derivative of the element's polynomial on its left / right face:
//   rv = sum_q phi_q(+1) u_q, rder = sum_q phi'_q(+1) u_q, lv, lder likewise at -1.
// The node set is reflection symmetric, phi_q(-1) = phi_{n-1-q}(+1) and phi'_q(-1) =
// -phi'_{n-1-q}(+1), so with s_q = u_q + u_{n-1-q}, d_q = u_q - u_{n-1-q} (q < n/2)
//   rv = E + O, lv = E - O, rder = G + F, lder = F - G,
//   E = sum cE_q s_q + a_mid u_mid, O = sum cO_q d_q, G = sum gE_q s_q + ap_mid u_mid, F = sum gO_q d_q
// — 4 FMAs per node PAIR instead of 4 per node, one 32-byte coefficient entry per pair.  On GLL
// nodes phi_q(+-1) is a unit vector and the value traces are the face nodes themselves.
// Table per direction d (TRACE_TAB(n) doubles, 16-byte aligned): {cE, cO, gE, gO} for q < n/2,
// then {a_mid, ap_mid, 0, 0}; tab[3 TRACE_TAB] = 1.0 when the basis is nodal on the faces.
#define PMG_MAX_N 33                      // P <= 32 (dg_setup)
__host__ __device__ constexpr int trace_tab_len(int n) { return 4 * (n / 2 + 1); }

__device__ __forceinline__ void stage_trace_tab(const LevelDev &L, double *tab) {
  const int n = L.n, h = n / 2, len = trace_tab_len(n);
  for (int idx = threadIdx.x; idx < 3 * (h + 1); idx += blockDim.x) {
    const int d = idx / (h + 1), q = idx - d * (h + 1);
    const double *tr = L.tr[d];
    double *e = tab + d * len + 4 * q;
    if (q < h) {
      const double a = tr[q], ar = tr[n - 1 - q], ap = tr[n + q], apr = tr[n + n - 1 - q];
      e[0] = 0.5 * (a + ar); e[1] = 0.5 * (a - ar); e[2] = 0.5 * (ap + apr); e[3] = 0.5 * (ap - apr);
    } else {
      const bool odd = (n & 1) != 0;
      e[0] = odd ? tr[h] : 0.0; e[1] = odd ? tr[n + h] : 0.0; e[2] = 0.0; e[3] = 0.0;
    }
  }
  if (threadIdx.x == 0) {
    bool nodal = L.tr[0][n - 1] == 1.0;
    for (int q = 0; q + 1 < n; ++q) nodal = nodal && L.tr[0][q] == 0.0;
    tab[3 * len] = nodal ? 1.0 : 0.0;
  }
}

// one face point: the line of n nodes lo[0], lo[stride], ..., tabd = the direction's table
template <int NT>
__device__ __forceinline__ void trace_point(const double *lo, int stride, int nrt, const double *tabd,
                                            bool nodal, double &lv, double &lder, double &rv,
                                            double &rder) {
  const int n = NT > 0 ? NT : nrt;
  const int h = n / 2;
  const double2 *c2 = reinterpret_cast<const double2 *>(tabd);
  const double *hi = lo + (n - 1) * stride;
  double E = 0, O = 0, G = 0, F = 0;
  if (nodal) {
#pragma unroll
    for (int q = 0; q < (NT > 0 ? NT / 2 : h); ++q) {
      const double u1 = lo[q * stride], u2 = hi[-q * stride];
      const double2 g = c2[2 * q + 1];
      G = fma(g.x, u1 + u2, G);
      F = fma(g.y, u1 - u2, F);
    }
  } else {
#pragma unroll
    for (int q = 0; q < (NT > 0 ? NT / 2 : h); ++q) {
      const double u1 = lo[q * stride], u2 = hi[-q * stride];
      const double sq = u1 + u2, dq = u1 - u2;
      const double2 c = c2[2 * q], g = c2[2 * q + 1];
      E = fma(c.x, sq, E);
      O = fma(c.y, dq, O);
      G = fma(g.x, sq, G);
      F = fma(g.y, dq, F);
    }
  }
  if (n & 1) {
    const double um = lo[h * stride];
    const double2 m = c2[2 * h];
    E = fma(m.x, um, E);
    G = fma(m.y, um, G);
  }
  lv = nodal ? lo[0] : E - O;
  lder = F - G;
  rv = nodal ? hi[0] : E + O;
  rder = G + F;
}

// traces of face point t in [0, 3 n^2) of the element at U (shared or global memory) -> Te
template <int NT>
__device__ __forceinline__ void elem_trace_item(const double *U, const double *tab, int nrt, int t,
                                                double *Te) {
  const int n = NT > 0 ? NT : nrt;
  const int n2 = n * n, len = trace_tab_len(n);
  const int d = t / n2, p = t - d * n2;
  const int p1 = p / n, p0 = p - p1 * n;
  int base, stride;
  if (d == 0) { base = n * p; stride = 1; }
  else if (d == 1) { base = p0 + n2 * p1; stride = n; }
  else { base = p; stride = n2; }
  double lv, lder, rv, rder;
  trace_point<NT>(U + base, stride, n, tab + d * len, tab[3 * len] != 0.0, lv, lder, rv, rder);
  double *Td = Te + d * 4 * n2;
  Td[p] = lv; Td[n2 + p] = lder; Td[2 * n2 + p] = rv; Td[3 * n2 + p] = rder;
}

// all threads of the CTA; U: the element (n^3, x fastest) in shared memory; Te: its 12 n^2 traces
template <int NT>
__device__ __forceinline__ void elem_traces(const double *U, const double *tab, int nrt, double *Te) {
  const int n = NT > 0 ? NT : nrt;
  for (int t = threadIdx.x; t < 3 * n * n; t += blockDim.x) elem_trace_item<NT>(U, tab, n, t, Te);
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

inline int grid_for(long long N, int bs) {
  long long g = (N + bs - 1) / bs;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

inline int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
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

}  // namespace
}  // namespace pmg
