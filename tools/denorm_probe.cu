// Scratch: cycles per dependent FP64 op vs operand magnitude (IEEE division / sqrt slow paths on
// sm_100a), and the MUFU reciprocal + Newton alternative
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double t = fma(-x, r, 1.0);
  r = fma(r, t, r);
  t = fma(-x, r, 1.0);
  return fma(r, t, r);
}
__global__ void probe(double a, long long* cyc, double* sink) {
  long long t0 = clock64();
  double q = 1.0;
#pragma unroll 1
  for (int i = 0; i < 200; ++i) q = 1.0 / (a * q * q + a * 0.5);       // reciprocal of ~a
  long long t1 = clock64();
  double s = a;
#pragma unroll 1
  for (int i = 0; i < 200; ++i) s = sqrt(s * s + a * a) * 0.5;          // sqrt of ~a^2
  long long t2 = clock64();
  double r = 1.0;
#pragma unroll 1
  for (int i = 0; i < 200; ++i) r = frcp(a * r * r + a * 0.5);
  long long t3 = clock64();
  double u = a;
#pragma unroll 1
  for (int i = 0; i < 200; ++i) u = u * 0.5 + a * 0.5;                   // loop skeleton
  long long t4 = clock64();
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
  if (threadIdx.x == 0) sink[0] = q + s + r + u;
}
int main() {
  long long* d; double* s; cudaMalloc(&d, 64); cudaMalloc(&s, 8);
  for (int e = 0; e <= 320; e += 20) {
    const double a = pow(10.0, -e) * 1.234;
    probe<<<1, 32>>>(a, d, s);
    long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("a=1e-%3d  div %6.1f  sqrt %6.1f  frcp %6.1f  skeleton %6.1f cycles/iter\n", e, h[0] / 200.0,
           h[1] / 200.0, h[2] / 200.0, h[3] / 200.0);
  }
  return 0;
}
