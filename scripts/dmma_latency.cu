// Microbenchmark: DMMA m8n8k4 latency and per-SM throughput vs number of independent chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double *out, int iters, long long *cyc) {
  double acc[CH][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int c = 0; c < CH; ++c) { acc[c][0] = 0; acc[c][1] = 0; }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH>
void run(int warps_per_block, int blocks) {
  double *out; long long *cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  int iters = 2000;
  k<CH><<<blocks, 32 * warps_per_block>>>(out, iters, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<CH><<<blocks, 32 * warps_per_block>>>(out, iters, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double dmma = (double)blocks * warps_per_block * iters * CH;
  printf("chains %d warps/blk %2d blocks %4d: %.1f cyc per DMMA per warp(chain-step), %.2f TFLOP/s\n", CH,
         warps_per_block, blocks, (double)c / iters / CH, dmma * 512 / (ms * 1e-3) / 1e12);
}
int main() {
  run<1>(1, 1); run<2>(1, 1); run<4>(1, 1); run<8>(1, 1);
  run<1>(4, 1); run<2>(4, 1); run<4>(4, 1); run<8>(4, 1);
  run<1>(16, 148); run<2>(16, 148); run<4>(16, 148); run<6>(8, 296); run<2>(8, 296);
  return 0;
}
