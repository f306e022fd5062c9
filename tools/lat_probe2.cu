// Scratch microbenchmark (not product code): dependent-chain latencies of FP64 ops, 1 thread,
// operations forced through asm volatile so nothing is hoisted or merged.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x) : "d"(b), "d"(a));
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(y) : "d"(b));
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) {  // fma + compare-select chain (Sturm-like)
    asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(z) : "d"(b), "d"(a));
    z = z < 0.0 ? -z : z;
  }
  long long t3 = clock64();
  float f = (float)a;
  for (int i = 0; i < n; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f) : "f"((float)b), "f"((float)a));
  long long t4 = clock64();
  double w = a;
  for (int i = 0; i < n; ++i) { w += __shfl_xor_sync(0xffffffffu, w, 1); asm volatile("" : "+d"(w)); }
  long long t5 = clock64();
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  out[threadIdx.x] = x + y + z + f + w;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  const int n = 4096;
  for (int threads : {1, 32}) {
    k<<<1, threads>>>(o, c, 0.999, 1.0001, n); cudaDeviceSynchronize();
    long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    printf("threads %d: DFMA %.1f  DMUL %.1f  DFMA+abs %.1f  FFMA %.1f  SHFL.64+DADD %.1f cycles/op\n", threads,
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n);
  }
  return 0;
}
