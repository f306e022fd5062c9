// Scratch microbenchmark: cycles per step of the TRI loop skeleton (not product code).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double g8(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}
template <int MODE>
__global__ void k(double* out, long long* cyc, int steps) {
  __shared__ double vb[256], ps[256];
  const int tid = threadIdx.x, cl = tid & 7, slot = tid >> 3;
  for (int i = tid; i < 256; i += blockDim.x) { vb[i] = 1e-3 * i; ps[i] = 0; }
  double a[6][12];
  for (int r = 0; r < 6; ++r) for (int c = 0; c < 12; ++c) a[r][c] = 1e-2 * (r + c + tid);
  __syncthreads();
  long long t0 = clock64();
  double acc = 0;
  for (int j = 0; j < steps; ++j) {
    double vc[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) vc[c] = vb[cl + 8 * c + (j & 1)];
    double p[6];
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      double s = 0;
      if (MODE & 1) {
#pragma unroll
        for (int c = 0; c < 12; ++c) s = fma(a[r][c], vc[c], s);
      } else s = vc[r];
      p[r] = g8(s);
    }
    if (cl == 0) for (int r = 0; r < 6; ++r) ps[slot + 16 * r] = p[r];
    if (MODE & 4) __syncthreads();
    double wc[12], dot = 0;
#pragma unroll
    for (int c = 0; c < 12; ++c) { wc[c] = ps[cl + 8 * c]; dot = fma(wc[c], vc[c], dot); }
    const double K = 1e-9 * g8(dot);
    if (MODE & 2) {
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double vr = vb[slot + 16 * r], wr = ps[slot + 16 * r] - K * vr;
#pragma unroll
        for (int c = 0; c < 12; ++c) a[r][c] = fma(-wr, vc[c], fma(-vr, wc[c] - K * vc[c], a[r][c]));
      }
    }
    acc += K;
    if (MODE & 4) __syncthreads();
  }
  long long t1 = clock64();
  double s = acc;
  for (int r = 0; r < 6; ++r) for (int c = 0; c < 12; ++c) s += a[r][c];
  out[tid] = s;
  if (tid == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 64);
  long long h;
  int steps = 100;
#define RUN(M, T) k<M><<<1, T>>>(o, c, steps); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); \
  printf("mode %d threads %4d: %.0f cycles/step\n", M, T, (double)h / steps);
  for (int rep = 0; rep < 2; ++rep) {
    RUN(0, 128) RUN(4, 128) RUN(5, 128) RUN(7, 128) RUN(1, 128) RUN(3, 128)
    RUN(4, 512) RUN(7, 512)
  }
  return 0;
}
