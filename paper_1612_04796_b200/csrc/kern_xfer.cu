// p-level transfers: fused prolongation + traces, plain restriction / prolongation.
// arXiv:1612.04796; PAPER.md line numbers cited per kernel.
#include <algorithm>

#include "kcommon.cuh"

namespace pmg {
namespace {

// Fused correction prolongation + face traces (Alg. 1 l.299 followed by the trace pass of the
// post-smoothing residual): u_f += (I (x) I (x) I) u_c with three DMMA line GEMMs in shared
// memory, u_f written back, and the traces of the new u_f emitted for the residual.
// smem: A = Uc (nc^3), later T2 (nf^2 nc) | U (nf^3) | T1 (nf nc^2) | trs (12 nf): T2 reuses the
// dead Uc region, which brings n = 17 to 73 KB and 3 CTAs per SM
#ifndef PMG_PT_MINB
#define PMG_PT_MINB 3
#endif
// NF, NC > 0: both extents compile-time (the 9 -> 17 and 5 -> 9 transfers of every configuration):
// one tile variant per pass is inlined, strides and trip counts fold to constants
template <int KSMAX, int NF = 0, int NCT = 0>
__global__ void __launch_bounds__(KSMAX <= 4 ? 128 : 256, KSMAX <= 4 ? 8 : PMG_PT_MINB) k_prolong_traces(LevelDev L, int ncr, const double *__restrict__ I,
                                                        const double *__restrict__ uc,
                                                        double *__restrict__ uf,
                                                        double *__restrict__ T) {
  extern __shared__ double sm[];
  const int nf = NF > 0 ? NF : L.n, n2 = nf * nf, n3 = n2 * nf;
  const int nc = NCT > 0 ? NCT : ncr;
  const int c3 = nc * nc * nc;
  const int c3p = (c3 + 3) & ~1;                // staging capacities (16-byte aligned regions)
  const int ap = (max(c3p, nf * nf * nc) + 1) & ~1;
  double *Ucs = sm, *T2 = sm, *Us = sm + ap;
  double *T1 = Us + ((n3 + 3) & ~1);
  double *trs = T1 + ((nf * nc * nc + 1) & ~1);     // even/odd trace table (16-byte aligned)
  unsigned long long *mbar = reinterpret_cast<unsigned long long *>(T1 + nf * nc * nc + 12 * nf);
  const int e = blockIdx.x;
#ifdef PMG_PT_PREFETCH          // diagnostic: L2 prefetch of the fine block of the element that many CTAs ahead
  if (threadIdx.x == 0 && (long long)e + PMG_PT_PREFETCH < L.Ne && (long long)L.Ne * n3 > (8ll << 20))
    prefetch_l2_doubles(uf + ((long long)e + PMG_PT_PREFETCH) * n3, n3);
#endif
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
  stage_trace_tab(L, trs);
  cp_async_wait_all();
  __syncthreads();
  if (bc.bytes || bf.bytes) mbar_wait(mbar, 0);
  const Blk BC = {{nc, nc, nc}, {1, nc, nc * nc}};
  const Blk B1 = {{nf, nc, nc}, {1, nf, nf * nc}};
  const Blk B2 = {{nf, nf, nc}, {1, nf, nf * nf}};
  const Blk BF = {{nf, nf, nf}, {1, nf, n2}};
  const LineSpec px = {nf, nc, I, nc, 1, nullptr, 0, 0, 0, 0};   // A[o][k] = I[o*nc + k]
  EpiStore s1{T1, B1};
  EpiStore s2{T2, B2};
  EpiAcc acc{U, BF, false};
  if constexpr (NF > 0) {
    mma_lines_ct<0, NF, NCT>(Uc, BC, px, s1); __syncthreads();
    mma_lines_ct<1, NF, NCT>(T1, B1, px, s2); __syncthreads();
    mma_lines_ct<2, NF, NCT>(T2, B2, px, acc); __syncthreads();
  } else {
    mma_lines_gen<0, KSMAX>(Uc, BC, px, s1); __syncthreads();
    mma_lines_gen<1, KSMAX>(T1, B1, px, s2); __syncthreads();
    mma_lines_gen<2, KSMAX>(T2, B2, px, acc); __syncthreads();
  }
  double *ue = uf + (long long)e * n3;
  for (int t = threadIdx.x; t < n3; t += blockDim.x) ue[t] = U[t];
  elem_traces<NF>(U, trs, nf, T + (long long)e * 12 * n2);
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

}  // namespace

static void configure_smem() {
  static bool done = false;
  if (done) return;
  done = true;
  const int mx = 227 * 1024;
  cudaFuncSetAttribute(k_prolong_traces<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_prolong_traces<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_prolong_traces<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_prolong_traces<8, 17, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_prolong_traces<2, 9, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
}

static size_t prolong_traces_smem(int nf, int nc) {
  const size_t c3p = ((size_t)nc * nc * nc + 3) & ~(size_t)1;
  const size_t ap = (std::max(c3p, (size_t)nf * nf * nc) + 1) & ~(size_t)1;
  return sizeof(double) * (ap + (((size_t)nf * nf * nf + 3) & ~(size_t)1) + (size_t)nf * nc * nc +
                           12 * (size_t)nf + 2);
}

bool prolong_traces_ok(const LevelDev &Lf, int nc) {
  return Lf.n <= 17 && prolong_traces_smem(Lf.n, nc) <= 200 * 1024;
}

cudaError_t launch_prolong_traces(const LevelDev &Lf, int nc, const double *I, const double *uc,
                                  double *uf, double *T, cudaStream_t s) {
  configure_smem();
  const size_t sb = prolong_traces_smem(Lf.n, nc);
#ifndef PMG_PT_GENERIC
  if (Lf.n == 17 && nc == 9) k_prolong_traces<8, 17, 9><<<Lf.Ne, 256, sb, s>>>(Lf, nc, I, uc, uf, T);
  else if (Lf.n == 9 && nc == 5) k_prolong_traces<2, 9, 5><<<Lf.Ne, 128, sb, s>>>(Lf, nc, I, uc, uf, T);
  else
#endif
  if (Lf.n >= 17) k_prolong_traces<8><<<Lf.Ne, 256, sb, s>>>(Lf, nc, I, uc, uf, T);   // big blocks: 8 warps
  else if (((nc + 3) >> 2) <= 2) k_prolong_traces<2><<<Lf.Ne, 128, sb, s>>>(Lf, nc, I, uc, uf, T);
  else if (((nc + 3) >> 2) <= 4) k_prolong_traces<4><<<Lf.Ne, 128, sb, s>>>(Lf, nc, I, uc, uf, T);
  else k_prolong_traces<8><<<Lf.Ne, 256, sb, s>>>(Lf, nc, I, uc, uf, T);
  return cudaGetLastError();
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
}  // namespace pmg
