// Blocked LU (no pivoting) and right-division solve X = P Q^{-1} for the Padé-13 denominator.
//
// Q = q13(X) = V - U of the scaled matrix X (||X||_1 <= theta_13) is well conditioned (Higham 2005,
// §3: kappa(q13(X)) is O(10) on ||X|| <= theta_13; measured 4-8 on the configs' operators) and its
// elimination growth is ~1 (measured 1.00-1.01), so the factorisation runs without row exchanges:
// every step is then a small in-CTA factor/inverse of a 64x64 diagonal block plus DMMA GEMMs
// (gemm_nt) for the off-diagonal panels, the trailing update and the two triangular sweeps.
// The smallest |u_ii| / max|Q| is reported so a bad pivot is detected (DME_ERR_NUMERIC upstream).
// Because P = V + U and Q commute (both are polynomials of X), Q^{-1} P = P Q^{-1}; the solve is
// done as a right division on row-major data: W = P U^{-1} (left-to-right), X = W L^{-1}
// (right-to-left), in place in P's buffer.
#include "aux.h"
#include "common.cuh"
#include "gemm_nt.h"
#include "lu.h"

namespace dme {

namespace {

constexpr int NB = 64;
constexpr int DIAG_SMEM = 3 * NB * (NB + 1) * 8;

// Factor the jb x jb diagonal block at D (row-major, ld) in place (unit-lower L, upper U), and
// emit Linv (row-major), LinvT (row-major = Linv^T) and UinvT (row-major = Uinv^T), ld NB.
__global__ void __launch_bounds__(1024) diag_block_kernel(double* D, int64_t ld, int jb,
                                                          double* Linv, double* LinvT,
                                                          double* UinvT, double* minpiv) {
  extern __shared__ double dsm[];
  double(*a)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm);
  double(*li)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm + NB * (NB + 1));
  double(*ui)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm + 2 * NB * (NB + 1));
  const int tid = threadIdx.x;
  for (int e = tid; e < jb * jb; e += blockDim.x) a[e / jb][e % jb] = D[(e / jb) * ld + e % jb];
  __syncthreads();
  for (int k = 0; k < jb; ++k) {
    const double piv = a[k][k];
    for (int i = k + 1 + tid; i < jb; i += blockDim.x) a[i][k] /= piv;
    __syncthreads();
    const int rem = jb - k - 1;
    for (int e = tid; e < rem * rem; e += blockDim.x) {
      const int i = k + 1 + e / rem, j = k + 1 + e % rem;
      a[i][j] -= a[i][k] * a[k][j];
    }
    __syncthreads();
  }
  // L^{-1} (unit lower): rows in sequence, columns in parallel
  for (int e = tid; e < jb * jb; e += blockDim.x) li[e / jb][e % jb] = (e / jb == e % jb) ? 1.0 : 0.0;
  __syncthreads();
  for (int i = 1; i < jb; ++i) {
    for (int c = tid; c < i; c += blockDim.x) {
      double s = 0.0;
      for (int l = c; l < i; ++l) s += a[i][l] * li[l][c];
      li[i][c] = -s;
    }
    __syncthreads();
  }
  // U^{-1} (upper): rows bottom-up, columns in parallel
  for (int e = tid; e < jb * jb; e += blockDim.x) ui[e / jb][e % jb] = 0.0;
  __syncthreads();
  for (int r = jb - 1; r >= 0; --r) {
    const double urr = a[r][r];
    for (int c = r + tid; c < jb; c += blockDim.x) {
      if (c == r) {
        ui[r][r] = 1.0 / urr;
      } else {
        double s = 0.0;
        for (int l = r + 1; l <= c; ++l) s += a[r][l] * ui[l][c];
        ui[r][c] = -s / urr;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < jb * jb; e += blockDim.x) {
    const int i = e / jb, j = e % jb;
    D[i * ld + j] = a[i][j];
    Linv[i * NB + j] = li[i][j];
    LinvT[i * NB + j] = li[j][i];
    UinvT[i * NB + j] = ui[j][i];
  }
  if (tid == 0) {
    double mn = 1e300;
    for (int k = 0; k < jb; ++k) mn = fmin(mn, fabs(a[k][k]));
    *minpiv = fmin(*minpiv, mn);
  }
}

__global__ void transpose_rect_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                                      int64_t lds, double* __restrict__ dst, int64_t ldd) {
  __shared__ double tile[32][33];
  const int64_t bx = (int64_t)blockIdx.x * 32, by = (int64_t)blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int64_t r = by + j, c = bx + threadIdx.x;
    if (r < rows && c < cols) tile[j][threadIdx.x] = src[r * lds + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int64_t r = bx + j, c = by + threadIdx.x;  // dst row r = src col
    if (r < cols && c < rows) dst[r * ldd + c] = tile[threadIdx.x][j];
  }
}

__global__ void init_minpiv(double* p) { *p = 1e300; }

}  // namespace

void transpose_rect(const double* src, int64_t rows, int64_t cols, int64_t lds, double* dst,
                    int64_t ldd, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
  transpose_rect_kernel<<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, lds, dst, ldd);
  DME_KCHECK();
}

size_t lu_scratch_doubles(int64_t n) {
  const int64_t nblk = ceil_div(n, NB);
  return (size_t)nblk * 3 * NB * NB + 2 * (size_t)n * NB + 8;
}

void lu_nopiv_solve_right(double* Q, double* P, int64_t n, int64_t ld, double* QT, double* scratch,
                          GemmScratch& gs, cudaStream_t st, double* minpiv_dev) {
  const int64_t nblk = ceil_div(n, NB);
  double* inv = scratch;                                  // per block: Linv, LinvT, UinvT
  double* T1 = scratch + (size_t)nblk * 3 * NB * NB;      // (n x NB) transposed panel
  double* T2 = T1 + (size_t)n * NB;                       // (n x NB) U12^T
  static bool attr = false;
  if (!attr) {
    DME_CUDA(cudaFuncSetAttribute(diag_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  DIAG_SMEM));
    attr = true;
  }
  init_minpiv<<<1, 1, 0, st>>>(minpiv_dev);
  DME_KCHECK();
  auto Linv = [&](int64_t b) { return inv + (size_t)b * 3 * NB * NB; };
  auto LinvT = [&](int64_t b) { return inv + (size_t)b * 3 * NB * NB + NB * NB; };
  auto UinvT = [&](int64_t b) { return inv + (size_t)b * 3 * NB * NB + 2 * NB * NB; };

  // ------------------------------------------------------------------ factorisation Q = L U
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t j0 = b * NB, jb = std::min<int64_t>(NB, n - j0), j1 = j0 + jb, rest = n - j1;
    diag_block_kernel<<<1, 1024, DIAG_SMEM, st>>>(Q + j0 * ld + j0, ld, (int)jb, Linv(b), LinvT(b),
                                          UinvT(b), minpiv_dev);
    DME_KCHECK();
    if (rest <= 0) break;
    // U12^T = A12^T L11^{-T}:  T1 = A12^T (rest x jb), T2 = T1 * Linv^T  (B rows = rows of Linv)
    transpose_rect(Q + j0 * ld + j1, jb, rest, ld, T1, NB, st);
    {
      GemmNTArgs g;
      g.A = T1; g.lda = NB; g.B = Linv(b); g.ldb = NB;
      g.M = rest; g.N = jb; g.K = jb;
      g.out = T2; g.out_rs = NB; g.out_cs = 1;
      gemm_nt(g, gs, st);
    }
    transpose_rect(T2, rest, jb, NB, Q + j0 * ld + j1, ld, st);   // U12 into Q
    // L21 = A21 U11^{-1}  (in place; B rows = columns of Uinv = rows of UinvT)
    {
      GemmNTArgs g;
      g.A = Q + j1 * ld + j0; g.lda = ld; g.B = UinvT(b); g.ldb = NB;
      g.M = rest; g.N = jb; g.K = jb;
      g.out = Q + j1 * ld + j0; g.out_rs = ld; g.out_cs = 1;
      gemm_nt(g, gs, st);
    }
    // A22 -= L21 U12   (B rows = columns of U12 = rows of T2)
    {
      GemmNTArgs g;
      g.A = Q + j1 * ld + j0; g.lda = ld; g.B = T2; g.ldb = NB;
      g.M = rest; g.N = rest; g.K = jb;
      g.alpha = -1.0; g.beta = 1.0;
      g.out = Q + j1 * ld + j1; g.out_rs = ld; g.out_cs = 1;
      gemm_nt(g, gs, st);
    }
  }
  // QT = (LU)^T  (rows of QT = columns of L / U, K-contiguous for the sweeps)
  transpose_rect(Q, n, n, ld, QT, ld, st);

  // ------------------------------------------------------------------ W = P U^{-1}
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t j0 = b * NB, jb = std::min<int64_t>(NB, n - j0);
    if (j0 > 0) {  // P[:, blk] -= W[:, 0:j0] U[0:j0, blk]
      GemmNTArgs g;
      g.A = P; g.lda = ld; g.B = QT + j0 * ld; g.ldb = ld;
      g.M = n; g.N = jb; g.K = j0;
      g.alpha = -1.0; g.beta = 1.0;
      g.out = P + j0; g.out_rs = ld; g.out_cs = 1;
      gemm_nt(g, gs, st);
    }
    GemmNTArgs g;  // W[:, blk] = (..) U_bb^{-1}
    g.A = P + j0; g.lda = ld; g.B = UinvT(b); g.ldb = NB;
    g.M = n; g.N = jb; g.K = jb;
    g.out = P + j0; g.out_rs = ld; g.out_cs = 1;
    gemm_nt(g, gs, st);
  }
  // ------------------------------------------------------------------ X = W L^{-1}
  for (int64_t b = nblk - 1; b >= 0; --b) {
    const int64_t j0 = b * NB, jb = std::min<int64_t>(NB, n - j0), j1 = j0 + jb;
    if (j1 < n) {  // W[:, blk] -= X[:, j1:] L[j1:, blk]
      GemmNTArgs g;
      g.A = P + j1; g.lda = ld; g.B = QT + j0 * ld + j1; g.ldb = ld;
      g.M = n; g.N = jb; g.K = n - j1;
      g.alpha = -1.0; g.beta = 1.0;
      g.out = P + j0; g.out_rs = ld; g.out_cs = 1;
      gemm_nt(g, gs, st);
    }
    GemmNTArgs g;
    g.A = P + j0; g.lda = ld; g.B = LinvT(b); g.ldb = NB;
    g.M = n; g.N = jb; g.K = jb;
    g.out = P + j0; g.out_rs = ld; g.out_cs = 1;
    gemm_nt(g, gs, st);
  }
}

}  // namespace dme
