// Probe: thread-per-line even/odd fast-diagonalisation pass with FP64 FMAs (no tensor pipe).
// One 23^3 window per CTA in shared memory (2 CTAs per SM), each thread owns whole lines:
// loads the 23 values, forms sums / differences, 12x12 + 11x11 FMAs, stores 23 values.
// Variant C: coefficients are kernel parameters (constant-bank operands of DFMA).
// Variant S: coefficients from shared memory (broadcast 16-byte loads).
// Reports time per window (6 line passes) and the FP64-pipe fraction it corresponds to.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -cudart shared -o variants/probe_line.so <this>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int M = 23, H = 11, S2 = 532, NT = 288;
struct Tab { double E[(H + 1) * (H + 1)]; double O[H * H]; };
struct Tabs { Tab d[3]; };

template <int DIR, bool FWD, bool CONSTOP>
__device__ __forceinline__ void line_pass(double *X, const Tab &tc, const double *ts) {
  constexpr int SO = DIR == 0 ? 1 : (DIR == 1 ? M : S2);
  for (int l = threadIdx.x; l < M * M; l += NT) {
    const int q = l / M, p = l - q * M;
    const int base = DIR == 0 ? (M * p + S2 * q) : (DIR == 1 ? (p + S2 * q) : (p + M * q));
    double *x = X + base;
    double s[H + 1], d[H];
    if (FWD) {
#pragma unroll
      for (int k = 0; k < H; ++k) {
        const double a = x[k * SO], b = x[(M - 1 - k) * SO];
        s[k] = a + b; d[k] = a - b;
      }
      s[H] = x[H * SO];
    } else {
#pragma unroll
      for (int k = 0; k <= H; ++k) s[k] = x[k * SO];
#pragma unroll
      for (int k = 0; k < H; ++k) d[k] = x[(H + 1 + k) * SO];
    }
#pragma unroll
    for (int i = 0; i <= H; ++i) {
      double e = 0.0, o = 0.0;
#pragma unroll
      for (int k = 0; k <= H; ++k) {
        const double c = CONSTOP ? (FWD ? tc.E[k * (H + 1) + i] : tc.E[i * (H + 1) + k])
                                 : (FWD ? ts[k * (H + 1) + i] : ts[i * (H + 1) + k]);
        e = fma(c, s[k], e);
      }
      if (i < H) {
#pragma unroll
        for (int k = 0; k < H; ++k) {
          const double c = CONSTOP ? (FWD ? tc.O[k * H + i] : tc.O[i * H + k])
                                   : (FWD ? ts[(H + 1) * (H + 1) + k * H + i] : ts[(H + 1) * (H + 1) + i * H + k]);
          o = fma(c, d[k], o);
        }
      }
      if (FWD) {
        x[i * SO] = e;
        if (i < H) x[(H + 1 + i) * SO] = o;
      } else {
        x[i * SO] = e + o;
        if (i < H) x[(M - 1 - i) * SO] = e - o;
      }
    }
  }
}

template <bool CONSTOP>
__global__ void __launch_bounds__(NT, 2) k_probe(const __grid_constant__ Tabs tabs, const double *tg,
                                                 double *out, int reps) {
  extern __shared__ double sm[];
  double *X = sm, *ts = sm + S2 * M;
  for (int i = threadIdx.x; i < S2 * M; i += NT) X[i] = 1e-3 * (i % 97);
  constexpr int TL = (H + 1) * (H + 1) + H * H;
  for (int i = threadIdx.x; i < 3 * TL; i += NT) ts[i] = tg[i];
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
    line_pass<0, true, CONSTOP>(X, tabs.d[0], ts); __syncthreads();
    line_pass<1, true, CONSTOP>(X, tabs.d[1], ts + TL); __syncthreads();
    line_pass<2, true, CONSTOP>(X, tabs.d[2], ts + 2 * TL); __syncthreads();
    line_pass<2, false, CONSTOP>(X, tabs.d[2], ts + 2 * TL); __syncthreads();
    line_pass<1, false, CONSTOP>(X, tabs.d[1], ts + TL); __syncthreads();
    line_pass<0, false, CONSTOP>(X, tabs.d[0], ts); __syncthreads();
  }
  double acc = 0;
  for (int i = threadIdx.x; i < S2 * M; i += NT) acc += X[i];
  if (acc == 12345.678) out[blockIdx.x] = acc;
}

int main() {
  Tabs h;
  constexpr int TL = (H + 1) * (H + 1) + H * H;
  double *flat = (double *)malloc(3 * TL * sizeof(double));
  for (int d = 0; d < 3; ++d) {
    for (int i = 0; i < (H + 1) * (H + 1); ++i) h.d[d].E[i] = flat[d * TL + i] = 0.05 * ((i * 7 + d) % 13 - 6) / 6.0;
    for (int i = 0; i < H * H; ++i) h.d[d].O[i] = flat[d * TL + (H + 1) * (H + 1) + i] = 0.05 * ((i * 5 + d) % 11 - 5) / 5.0;
  }
  double *tg, *out;
  cudaMalloc(&tg, 3 * TL * sizeof(double));
  cudaMemcpy(tg, flat, 3 * TL * sizeof(double), cudaMemcpyHostToDevice);
  cudaMalloc(&out, 8192 * sizeof(double));
  const size_t smem = (S2 * M + 3 * TL + 2) * sizeof(double);
  cudaFuncSetAttribute(k_probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ[2];
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[0], k_probe<true>, NT, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[1], k_probe<false>, NT, smem);
  printf("occupancy CTAs/SM: const %d smem %d (smem %zu B)\n", occ[0], occ[1], smem);
  const int grid = 296, reps = 14;   // 296 x 14 = 4144 windows, c3 has 4096
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int v = 0; v < 2; ++v) {
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(e0);
      if (v == 0) k_probe<true><<<grid, NT, smem>>>(h, tg, out, reps);
      else k_probe<false><<<grid, NT, smem>>>(h, tg, out, reps);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fma_per_window = 6.0 * M * M * ((H + 1) * (H + 1) + H * H);
      const double tf = 2.0 * fma_per_window * grid * reps / (ms * 1e-3) / 1e12;
      printf("%s: %.3f ms for %d windows (%.1f us per 4096), useful %.2f TFLOP/s, err %s\n", v == 0 ? "const-operand" : "smem-operand",
             ms, grid * reps, ms * 1e3 * 4096.0 / (grid * reps), tf, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
