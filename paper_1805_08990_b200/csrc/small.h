#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace dme {

constexpr int SMALL_K_MAX = 224;          // packed k(k+1)/2 doubles fit in 201 KB of shared memory
constexpr int SMALL_M_MAX = 8;            // columns of B handled by the fused Riccati flow
constexpr int SMALL_SMEM_MAX = SMALL_K_MAX * (SMALL_K_MAX + 1) / 2 * 8;

struct SmallArgs {
  int k = 0;                 // columns of the concatenated factor Zc
  int compress = 1;          // 1: eigen-compression of G (Z_new = Zc W_kept)
  const double* G = nullptr; // k x k Gram matrix Zc^T Zc, column-major, leading dim ldg
  int64_t ldg = 0;
  double tol = 1e-16;        // relative truncation tolerance (reading G7)
  int cap = 1 << 30;         // rank cap (reading G8)
  int t3 = 0;                // 1: fuse the Riccati flow T3(tau)
  int m = 0;                 // columns of B
  const double* H = nullptr; // k x m = Zc^T B, column-major ld ldh
  int64_t ldh = 0;
  const double* LRinv = nullptr;  // m x m row-major L_R^{-1}, R = L_R L_R^T
  double tau = 0.0;
  double* V = nullptr;       // scratch: k x k eigenvectors, column-major, leading dim ldv
  int64_t ldv = 0;
  int sqrt_scale = 0;        // 1: scale kept eigenvector columns by sqrt(theta) (G = C C^T -> C)
  double* Tm = nullptr;      // out: k x r column-major, leading dim ldt
  int64_t ldt = 0;
  int* r_out = nullptr;      // out: new rank (device)
  double* stats = nullptr;   // out: [rank, max diag G, max remaining pivot / max diag]
};

void compress_t3(const SmallArgs& a, cudaStream_t st);

}  // namespace dme
