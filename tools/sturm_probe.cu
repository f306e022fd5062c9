// Scratch microbenchmark (not product code): cycles per Sturm count (k = 90) in one CTA vs threads.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e2, int k, double x) {
  double p2 = 1.0, p1 = d[0] - x;
  bool neg_prev = p1 <= 0.0;
  int cnt = neg_prev;
  int i = 1;
  for (; i + 7 < k; i += 8) {
    double dd[8], ff[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { dd[u] = d[i + u] - x; ff[u] = e2[i - 1 + u]; }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double p = fma(dd[u], p1, -ff[u] * p2);
      const bool ng = p <= 0.0;
      cnt += ng != neg_prev;
      neg_prev = ng;
      p2 = p1;
      p1 = p;
    }
    const double m1 = fmax(fabs(p1), fabs(p2));
    if (m1 > 0x1p300) { p1 *= 0x1p-300; p2 *= 0x1p-300; }
    else if (m1 < 0x1p-300) { p1 *= 0x1p300; p2 *= 0x1p300; }
  }
  for (; i < k; ++i) {
    const double p = fma(d[i] - x, p1, -e2[i - 1] * p2);
    const bool ng = p <= 0.0;
    cnt += ng != neg_prev;
    neg_prev = ng; p2 = p1; p1 = p;
  }
  return cnt;
}
// LDL^T (pivot) form: q_i = (d_i - x) - e2_{i-1} / q_{i-1}: one division-free recip variant
__device__ __forceinline__ int sturm_q(const double* __restrict__ d, const double* __restrict__ e2, int k, double x) {
  double q = d[0] - x;
  int cnt = q < 0.0;
  for (int i = 1; i < k; ++i) {
    if (q == 0.0) q = -1e-300;
    q = (d[i] - x) - e2[i - 1] / q;
    cnt += q < 0.0;
  }
  return cnt;
}
__global__ void kern(const double* dg, const double* eg, int k, int reps, int active, long long* out, int* sink, int variant) {
  __shared__ double d[256], e2[256];
  for (int i = threadIdx.x; i < k; i += blockDim.x) { d[i] = dg[i]; e2[i] = eg[i]; }
  __syncthreads();
  long long t0 = clock64();
  int acc = 0;
  if (threadIdx.x < active)
    for (int r = 0; r < reps; ++r) {
      const double x = -1.0 + 2.0 * (threadIdx.x + r * 0.37) / (active + reps);
      acc += variant == 0 ? sturm_count(d, e2, k, x) : sturm_q(d, e2, k, x);
    }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  sink[threadIdx.x] = acc;
}
int main() {
  const int k = 90;
  double hd[256], he[256];
  for (int i = 0; i < k; ++i) { hd[i] = 0.3 * ((i * 37) % 11) / 11.0; he[i] = 0.01 * (1 + i % 5); }
  double *d, *e; long long* o; int* s;
  cudaMalloc(&d, 2048); cudaMalloc(&e, 2048); cudaMalloc(&o, 8); cudaMalloc(&s, 4096 * 4);
  cudaMemcpy(d, hd, 2048, cudaMemcpyHostToDevice); cudaMemcpy(e, he, 2048, cudaMemcpyHostToDevice);
  for (int variant = 0; variant < 2; ++variant)
  for (int active : {1, 32, 128, 512}) {
    kern<<<1, 512>>>(d, e, k, 10, active, o, s, variant);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);
    printf("variant %d active %4d: %.0f cycles per Sturm count (k=%d)\n", variant, active, c / 10.0, k);
  }
  return 0;
}
