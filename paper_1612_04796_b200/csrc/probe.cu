// FP64 throughput probes (DFMA vector pipe and DMMA m8n8k4 tensor path) used by bench.py to
// measure the roofline denominator on the box instead of assuming the nominal 37.2 TFLOP/s.
#include <cuda_runtime.h>

#include "../../include/pmg_dg.h"

namespace {

constexpr int CHAINS = 8;

__global__ void k_dfma(double *out, int iters, double seed) {
  double a[CHAINS], b = 1.0 + 1e-9 * threadIdx.x, c = seed;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) a[k] = seed + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;   // never true; keeps the work alive
}

__global__ void k_dmma(double *out, int iters, double seed) {
  double acc[CHAINS][2];
  double a = seed + threadIdx.x * 1e-6, b = seed - threadIdx.x * 1e-6;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { acc[k][0] = 0; acc[k][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[k][0]), "+d"(acc[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += acc[k][0] + acc[k][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace

extern "C" int pmg_fp64_peak(int use_dmma, double *tflops_out, void *stream) {
  if (!tflops_out) return PMG_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double *out = nullptr;
  const int blocks = sms * 4, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {   // first launch warms up
    cudaEventRecord(e0, s);
    if (use_dmma) k_dmma<<<blocks, threads, 0, s>>>(out, iters, 1.0);
    else k_dfma<<<blocks, threads, 0, s>>>(out, iters, 1.0);
    cudaEventRecord(e1, s);
  }
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (e != cudaSuccess || ms <= 0) return PMG_ECUDA;
  double flops = 2.0 * blocks * threads * (double)iters * CHAINS;
  if (use_dmma) flops = 2.0 * (blocks * threads / 32.0) * iters * CHAINS * 256.0;
  *tflops_out = flops / (ms * 1e-3) / 1e12;
  return PMG_OK;
}
