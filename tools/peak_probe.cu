// FP64 pipe microbenchmarks (scratch measurement tool, not product code).
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int j = 0; j < 8; j++) c[j][0] = c[j][1] = 0;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int j = 0; j < 8; j++) s += c[j][0] + c[j][1];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
  for (int j = 0; j < 16; j++) c[j] = j;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 16; j++) c[j] = fma(c[j], b, a);
  }
  double s = 0; for (int j = 0; j < 16; j++) s += c[j];
  if (s == 12345.0) out[0] = s;
}
static double run(bool mma) {
  double* d; cudaMalloc(&d, 8);
  int blocks = 148 * 4, threads = 256, iters = 4096;
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  if (mma) k_dmma<<<blocks, threads>>>(d, 16); else k_dfma<<<blocks, threads>>>(d, 16);
  cudaDeviceSynchronize();
  cudaEventRecord(s);
  if (mma) k_dmma<<<blocks, threads>>>(d, iters); else k_dfma<<<blocks, threads>>>(d, iters);
  cudaEventRecord(e); cudaEventSynchronize(e);
  float ms; cudaEventElapsedTime(&ms, s, e);
  double flops = mma ? double(blocks) * (threads / 32) * iters * 8 * 512.0
                     : double(blocks) * threads * iters * 16 * 2.0;
  cudaFree(d);
  return flops / (ms * 1e-3) / 1e12;
}
extern "C" double probe_dmma() { return run(true); }
extern "C" double probe_dfma() { return run(false); }
