// Scratch: dependent-chain latencies of the ops on the reflector's critical path (not product code).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, int n) {
  long long t0, t1;
  double w = a + threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) w = __shfl_xor_sync(0xffffffffu, w, 1 + (i & 3)) * 0.999;
  t1 = clock64(); cyc[0] = t1 - t0;
  double r = a + 2.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r)); r = y + 1.5; }
  t1 = clock64(); cyc[1] = t1 - t0;
  double q = a + 3.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double y; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q)); q = y + 1.5; }
  t1 = clock64(); cyc[2] = t1 - t0;
  double z = a + 4.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) z = rsqrt(z) + 1.5;
  t1 = clock64(); cyc[3] = t1 - t0;
  double u = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) u = u * 0.999 + 1e-3;
  t1 = clock64(); cyc[4] = t1 - t0;
  __shared__ double sm[64];
  sm[threadIdx.x & 63] = 0.0;
  __syncthreads();
  double p = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) p = sm[(int)p + (i & 7)] ;
  t1 = clock64(); cyc[5] = t1 - t0;
  float f = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = __shfl_xor_sync(0xffffffffu, f, 1 + (i & 3)) * 0.999f;
  t1 = clock64(); cyc[6] = t1 - t0;
  out[threadIdx.x] = w + r + q + z + u + p + f;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 64);
  long long h[8];
  const char* nm[7] = {"SHFL.f64+DMUL", "MUFU.RSQ64H+DADD", "MUFU.RCP64H+DADD", "rsqrt(double)+DADD", "DFMA(mul+add)", "LDS.64 chase", "SHFL.f32+FMUL"};
  for (int t : {32, 128}) {
    k<<<1, t>>>(o, c, 0.5, 1000); cudaDeviceSynchronize();
    cudaMemcpy(h, c, 56, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 7; ++i) printf("threads %3d %-20s %.1f cycles/iter\n", t, nm[i], h[i] / 1000.0);
  }
  return 0;
}
