// C[M x N] = alpha * A[M x K] * B[N x K]^T + beta * Cin + gamma * I   (FP64, DMMA + TMA, Stream-K)
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace dme {

struct GemmNTArgs {
  const double* A = nullptr;  // row i of A at A + i*lda, K contiguous doubles
  int64_t lda = 0;
  const double* B = nullptr;  // row j of B (= column j of the right factor) at B + j*ldb
  int64_t ldb = 0;
  int64_t b_nloc = 0;         // >0: B is row-block-blocked: element (j, k) at
  int64_t b_blockstride = 0;  //      B + (k / nloc)*blockstride + j*ldb + k % nloc
  int64_t M = 0, N = 0, K = 0;
  double alpha = 1.0, beta = 0.0, gamma = 0.0;
  const double* cin = nullptr;  // beta term source (nullptr: out itself)
  int64_t cin_rs = 0, cin_cs = 0;
  double* out = nullptr;        // element (i, j) at out + i*out_rs + j*out_cs
  int64_t out_rs = 0, out_cs = 0;
  bool sym_upper = false;       // M == N, symmetric result: compute only the tiles touching
                                // the upper triangle (the caller mirrors, see mirror_lower)
};

struct GemmScratch {
  double* partial = nullptr;  // partial_doubles(max_grid)
  int* counters = nullptr;    // max_tiles ints, zero-initialised once
  int2* tile_list = nullptr;  // max_tiles entries (symmetric-output tile list)
  int max_grid = 0;
  int64_t max_tiles = 0;
  static size_t partial_doubles(int grid);
};

void gemm_nt(const GemmNTArgs& a, GemmScratch& ws, cudaStream_t st);
// X (n x n row-major, ld): X[i][j] = X[j][i] for i > j  (or (X + X^T)/2 everywhere when average)
void mirror_lower(double* X, int64_t n, int64_t ld, bool average, cudaStream_t st);

}  // namespace dme
