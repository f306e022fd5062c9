// Scratch: rate of clock64() against %globaltimer (ns) on sm_100a, and a DFMA chain in both units
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void probe(int n, double a, double* sink, long long* out) {
  const long long c0 = clock64();
  const unsigned long long g0 = gtime();
  double x = a;
#pragma unroll 1
  for (int i = 0; i < n; ++i) { x = fma(x, a, 1e-3); x = fma(x, a, 1e-3); x = fma(x, a, 1e-3); x = fma(x, a, 1e-3); }
  const long long c1 = clock64();
  const unsigned long long g1 = gtime();
  out[0] = c1 - c0;
  out[1] = (long long)(g1 - g0);
  if (threadIdx.x == 0) sink[0] = x;
}
int main() {
  long long* d; double* s; cudaMalloc(&d, 64); cudaMalloc(&s, 8);
  for (int n : {100000, 1000000, 4000000}) {
    probe<<<1, 32>>>(n, 0.999, s, d);
    long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("n %d: clock64 %lld, globaltimer %lld ns -> clock64 rate %.3f GHz; %.2f clock64 ticks / %.2f ns per DFMA\n",
           n, h[0], h[1], (double)h[0] / h[1], (double)h[0] / (4.0 * n), (double)h[1] / (4.0 * n));
  }
  return 0;
}
