// FP64 dependent-chain latency microbenchmark (scratch tool, not product code).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  t1 = clock64(); cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) y = y + x;
  t1 = clock64(); cyc[1] = t1 - t0;
  // DDIV chain
  double z = 1.0 + a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) z = b / z + 0.5;
  t1 = clock64(); cyc[2] = t1 - t0;
  // SHFL + DADD chain
  double w = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) w = w + __shfl_xor_sync(0xffffffffu, w, 1);
  t1 = clock64(); cyc[3] = t1 - t0;
  // DSQRT chain
  double q = 2.0 + a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) q = sqrt(q) + 1.0;
  t1 = clock64(); cyc[4] = t1 - t0;
  // LDS chain (pointer chasing in smem)
  __shared__ int sm[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) sm[i] = (i + 1) % 64;
  __syncthreads();
  int p = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) p = sm[p];
  t1 = clock64(); cyc[5] = t1 - t0;
  // __syncthreads cost (1 warp)
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); cyc[6] = t1 - t0;
  // FFMA chain (fp32) for reference
  float f = a, g = b;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = fmaf(f, g, 1.0f);
  t1 = clock64(); cyc[7] = t1 - t0;
  out[0] = x + y + z + w + q + p + f;
}
__global__ void k_bar(long long* cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 16 * 8);
  int n = 1000;
  k_lat<<<1, 32>>>(o, c, 0.1, 0.999, n); cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
  const char* nm[8] = {"DFMA", "DADD", "DDIV", "SHFL+DADD", "DSQRT+DADD", "LDS chase", "bar(1 warp)", "FFMA"};
  for (int i = 0; i < 8; ++i) printf("%-12s %.1f cycles/op\n", nm[i], (double)h[i] / n);
  for (int t : {256, 512, 1024}) {
    k_bar<<<1, t>>>(c, n); cudaDeviceSynchronize();
    cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("bar.sync %4d threads %.1f cycles\n", t, (double)h[0] / n);
  }
  return 0;
}
