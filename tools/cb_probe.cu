// Scratch microbenchmark (not product code): per-phase cycles of the complement-basis kernel
// (pivoted Cholesky of I - W W^T) in one CTA, to find where the per-step time goes.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
constexpr int NT = 1024;
__global__ void __launch_bounds__(NT) cb(const double* W, int ldw, int k, int kb, double* U, int ldu,
                                          long long* cyc, int variant) {
  extern __shared__ double Pm[];
  __shared__ double col[256];
  __shared__ double s_piv;
  __shared__ int s_p;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ld = k | 1, s = k - kb;
  long long c0 = clock64();
  for (int i = warp; i < k; i += 32)
    for (int j = lane; j < k; j += 32) {
      double acc = (i == j) ? 1.0 : 0.0;
      for (int c = 0; c < kb; ++c) acc = fma(-W[i + c * ldw], W[j + c * ldw], acc);
      Pm[i * ld + j] = acc;
    }
  __syncthreads();
  long long c1 = clock64();
  long long ta = 0, tb = 0, tc = 0;
  for (int t = 0; t < s; ++t) {
    long long x0 = clock64();
    if (warp == 0) {
      double bv = -1.0;
      int bi = 0;
      for (int i = lane; i < k; i += 32) {
        const double v = Pm[i * ld + i];
        if (v > bv) { bv = v; bi = i; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) { s_p = bi; s_piv = bv > 0.0 ? 1.0 / sqrt(bv) : 0.0; }
    }
    __syncthreads();
    const int p = s_p;
    const double rp = s_piv;
    long long x1 = clock64();
    for (int i = tid; i < k; i += NT) {
      const double u = Pm[p * ld + i] * rp;
      col[i] = u;
      U[i + t * ldu] = u;
    }
    __syncthreads();
    long long x2 = clock64();
    if (variant == 0) {
      for (int i = warp; i < k; i += 32) {
        const double ci = col[i];
        for (int j = lane; j < k; j += 32) Pm[i * ld + j] = fma(-ci, col[j], Pm[i * ld + j]);
      }
    }
    __syncthreads();
    long long x3 = clock64();
    ta += x1 - x0; tb += x2 - x1; tc += x3 - x2;
  }
  if (tid == 0) { cyc[0] = c1 - c0; cyc[1] = ta; cyc[2] = tb; cyc[3] = tc; cyc[4] = s; }
}
int main() {
  const int k = 90, kb = 45;
  std::vector<double> hW(k * kb);
  for (int c = 0; c < kb; ++c) for (int i = 0; i < k; ++i) hW[i + c * k] = (i == c) ? 1.0 : 0.0;
  double *W, *U; long long* cyc;
  cudaMalloc(&W, k * kb * 8); cudaMalloc(&U, k * k * 8); cudaMalloc(&cyc, 64);
  cudaMemcpy(W, hW.data(), k * kb * 8, cudaMemcpyHostToDevice);
  int smem = k * (k | 1) * 8;
  cudaFuncSetAttribute(cb, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int variant = 0; variant < 2; ++variant)
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cb<<<1, NT, smem>>>(W, k, k, kb, U, k, cyc, variant);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long h[5]; cudaMemcpy(h, cyc, 40, cudaMemcpyDeviceToHost);
    printf("variant %d: %.1f us | form %lld cyc | per step: pivot %lld col %lld update %lld (s=%lld) | %s\n", variant,
           ms * 1e3, h[0], h[1] / h[4], h[2] / h[4], h[3] / h[4], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
