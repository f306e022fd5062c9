// Device helpers shared by the one-CTA small-system kernels (small.cu, eig_fast.cu).
#pragma once
#include "small.h"

namespace dme {

// Thread 0 of the last block of a compression: the new rank to r_out and, when the host-mapped
// record is set, stats + rank, a system-scope fence, then the sequence number the host waits for.
__device__ inline void publish_rank(const SmallArgs& a, int r) {
  *a.r_out = r;
  if (a.map) {
    volatile HostMap* m = a.map;
    if (a.stats)
      for (int i = 0; i < 5; ++i) m->stats[i] = a.stats[i];
    m->r = r;
    __threadfence_system();
    m->seq = a.map_seq;
  }
}

namespace smallk {

constexpr int NT = 1024;

__device__ __forceinline__ int pidx(int i, int j) {  // packed symmetric slot of the pair {i, j}
  return i >= j ? (i * (i + 1)) / 2 + j : (j * (j + 1)) / 2 + i;
}

// g(A) for a tiny symmetric PSD A (m x m, row-major, destroyed), serial cyclic Jacobi; one thread.
__device__ inline void tiny_sym_fun_g(double* A, double* out, int m) {
  double V[SMALL_M_MAX * SMALL_M_MAX];
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) V[i * m + j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) off += A[p * m + q] * A[p * m + q];
    if (off == 0.0) break;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) {
        const double apq = A[p * m + q];
        if (apq == 0.0) continue;
        const double th = (A[q * m + q] - A[p * m + p]) / (2.0 * apq);
        const double tt = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(1.0 + th * th));
        const double c = 1.0 / sqrt(1.0 + tt * tt), s = tt * c;
        for (int k = 0; k < m; ++k) {
          const double akp = A[k * m + p], akq = A[k * m + q];
          A[k * m + p] = c * akp - s * akq;
          A[k * m + q] = s * akp + c * akq;
        }
        for (int k = 0; k < m; ++k) {
          const double apk = A[p * m + k], aqk = A[q * m + k];
          A[p * m + k] = c * apk - s * aqk;
          A[q * m + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < m; ++k) {
          const double vkp = V[k * m + p], vkq = V[k * m + q];
          V[k * m + p] = c * vkp - s * vkq;
          V[k * m + q] = s * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      double acc = 0.0;
      for (int l = 0; l < m; ++l) {
        const double x = A[l * m + l] > 0.0 ? A[l * m + l] : 0.0;
        const double s = sqrt(1.0 + x);
        acc += V[i * m + l] * (-1.0 / (s * (1.0 + s))) * V[j * m + l];
      }
      out[i * m + j] = acc;
    }
}


// Riccati flow T3 fused on the compression output: Tm (k x r) <- Tm K^{-1/2}  (see small.cu header).
// S: >= 2*SMALL_K_MAX*SMALL_M_MAX doubles of free shared memory; Gam, Phi: m*m shared doubles.
__device__ inline void t3_fuse(const SmallArgs& a, int k, int r, double* S, double* Gam, double* Phi) {
  const int tid = threadIdx.x;
  const int m = a.m;
    double* Fs = S;                                  // the packed area is free now:
    double* Wd = S + SMALL_K_MAX * SMALL_M_MAX;      // F (r x m), W / U (k x m)
    // W = Tm^T H  (r x m),  H = Zc^T B  (k x m)
    for (int e = tid; e < r * m; e += (int)blockDim.x) {
      const int c = e % r, mu = e / r;
      double acc = 0.0;
      for (int i = 0; i < k; ++i) acc += a.Tm[i + (size_t)c * a.ldt] * a.H[i + (size_t)mu * a.ldh];
      Wd[c * m + mu] = acc;
    }
    __syncthreads();
    // F = sqrt(tau) W Linv^T   (Linv = L_R^{-1}, m x m row-major)
    for (int e = tid; e < r * m; e += (int)blockDim.x) {
      const int c = e / m, mu = e % m;
      double acc = 0.0;
      for (int nu2 = 0; nu2 < m; ++nu2) acc += Wd[c * m + nu2] * a.LRinv[mu * m + nu2];
      Fs[c * m + mu] = sqrt(a.tau) * acc;
    }
    __syncthreads();
    if (tid < m * m) {  // Phi = F^T F
      const int mu = tid / m, nu2 = tid % m;
      double acc = 0.0;
      for (int c = 0; c < r; ++c) acc += Fs[c * m + mu] * Fs[c * m + nu2];
      Phi[mu * m + nu2] = acc;
    }
    __syncthreads();
    if (tid == 0) {  // Gamma = g(Phi)
      if (m == 1) {
        const double s = sqrt(1.0 + fmax(Phi[0], 0.0));
        Gam[0] = -1.0 / (s * (1.0 + s));
      } else {
        tiny_sym_fun_g(Phi, Gam, m);
      }
    }
    __syncthreads();
    // U = Tm F (k x m), then Tm <- Tm + U Gamma F^T
    for (int e = tid; e < k * m; e += (int)blockDim.x) {
      const int i = e / m, mu = e % m;
      double acc = 0.0;
      for (int c = 0; c < r; ++c) acc += a.Tm[i + (size_t)c * a.ldt] * Fs[c * m + mu];
      Wd[i * m + mu] = acc;
    }
    __syncthreads();
    for (int e = tid; e < k * r; e += (int)blockDim.x) {
      const int i = e % k, c = e / k;
      double acc = 0.0;
      for (int mu = 0; mu < m; ++mu) {
        double ug = 0.0;
        for (int nu2 = 0; nu2 < m; ++nu2) ug += Wd[i * m + nu2] * Gam[nu2 * m + mu];
        acc += ug * Fs[c * m + mu];
      }
      a.Tm[i + (size_t)c * a.ldt] += acc;
    }
  }

}  // namespace smallk
}  // namespace dme
