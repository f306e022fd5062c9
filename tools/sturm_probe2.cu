// Scratch microbenchmark (not product code): variants of the Sturm-count recurrence, 1 thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__device__ __forceinline__ int sturm_v(const double* __restrict__ d, const double* __restrict__ e2, int k, double x, double* sink) {
  double p2 = 1.0, p1 = d[0] - x;
  int cnt = p1 <= 0.0;
  bool neg_prev = p1 <= 0.0;
  if (V == 0) {  // recurrence only (no count)
    for (int i = 1; i < k; ++i) { const double p = fma(d[i] - x, p1, -e2[i - 1] * p2); p2 = p1; p1 = p; }
    *sink = p1;
    return 0;
  }
  if (V == 1) {  // + count
    for (int i = 1; i < k; ++i) {
      const double p = fma(d[i] - x, p1, -e2[i - 1] * p2);
      const bool ng = p <= 0.0; cnt += ng != neg_prev; neg_prev = ng; p2 = p1; p1 = p;
    }
    *sink = p1;
    return cnt;
  }
  if (V == 2) {  // registers preloaded (no LDS in the loop), count
    double dd[96], ff[96];
#pragma unroll
    for (int i = 0; i < 96; ++i) { dd[i] = i < k ? d[i] - x : 0.0; ff[i] = i < k ? e2[i] : 0.0; }
#pragma unroll
    for (int i = 1; i < 96; ++i) {
      if (i < k) {
        const double p = fma(dd[i], p1, -ff[i - 1] * p2);
        const bool ng = p <= 0.0; cnt += ng != neg_prev; neg_prev = ng; p2 = p1; p1 = p;
      }
    }
    *sink = p1;
    return cnt;
  }
  if (V == 4) {  // production form with integer sign / exponent tests (no FP64 compare in the chain)
    unsigned long long prevs = (unsigned long long)__double_as_longlong(p1) >> 63;
    cnt = (int)prevs;
    int i = 1;
    for (; i + 15 < k; i += 16) {
      double dd[16], ff[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) { dd[u] = d[i + u] - x; ff[u] = e2[i - 1 + u]; }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const double p = fma(dd[u], p1, -ff[u] * p2);
        const unsigned long long sg = (unsigned long long)__double_as_longlong(p) >> 63;
        cnt += (int)(sg ^ prevs);
        prevs = sg;
        p2 = p1; p1 = p;
      }
      const int e1 = (int)((__double_as_longlong(p1) >> 52) & 0x7ff), e2_ = (int)((__double_as_longlong(p2) >> 52) & 0x7ff);
      const int em = e1 > e2_ ? e1 : e2_;
      if (em > 1023 + 300) { p1 *= 0x1p-300; p2 *= 0x1p-300; }
      else if (em < 1023 - 300) { p1 *= 0x1p300; p2 *= 0x1p300; }
    }
    for (; i < k; ++i) {
      const double p = fma(d[i] - x, p1, -e2[i - 1] * p2);
      const unsigned long long sg = (unsigned long long)__double_as_longlong(p) >> 63;
      cnt += (int)(sg ^ prevs);
      prevs = sg; p2 = p1; p1 = p;
    }
    *sink = p1;
    return cnt;
  }
  // V == 3: LDL^T pivot form q_i = (d_i - x) - e2_{i-1} / q_{i-1} via a reciprocal approximation
  double q = d[0] - x;
  cnt = q < 0.0;
  for (int i = 1; i < k; ++i) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    q = fma(-e2[i - 1], r, d[i] - x);
    cnt += q < 0.0;
  }
  *sink = q;
  return cnt;
}
template <int V>
__global__ void kern(const double* dg, const double* eg, int k, int reps, long long* out, int* s, double* sk) {
  __shared__ double d[256], e2[256];
  for (int i = threadIdx.x; i < k; i += blockDim.x) { d[i] = dg[i]; e2[i] = eg[i]; }
  __syncthreads();
  long long t0 = clock64();
  int acc = 0;
  double sink = 0;
  if (threadIdx.x == 0)
    for (int r = 0; r < reps; ++r) acc += sturm_v<V>(d, e2, k, -0.5 + r * 0.01, &sink);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; s[0] = acc; sk[0] = sink; }
}
int main() {
  const int k = 90;
  double hd[256], he[256];
  for (int i = 0; i < k; ++i) { hd[i] = 0.3 * ((i * 37) % 11) / 11.0; he[i] = 0.01 * (1 + i % 5); }
  double *d, *e, *sk; long long* o; int* s;
  cudaMalloc(&d, 2048); cudaMalloc(&e, 2048); cudaMalloc(&o, 8); cudaMalloc(&s, 64); cudaMalloc(&sk, 64);
  cudaMemcpy(d, hd, 2048, cudaMemcpyHostToDevice); cudaMemcpy(e, he, 2048, cudaMemcpyHostToDevice);
  long long c;
#define RUN(V) kern<V><<<1, 32>>>(d, e, k, 20, o, s, sk); cudaDeviceSynchronize(); cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost); printf("variant %d: %.0f cycles per count (%.1f per element)\n", V, c / 20.0, c / 20.0 / k);
  RUN(0) RUN(1) RUN(3) RUN(4) RUN(0) RUN(1) RUN(3) RUN(4)
  return 0;
}
