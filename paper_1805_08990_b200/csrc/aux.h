#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace dme {

struct LinTerm {
  double c = 0.0;
  const double* X = nullptr;
};

// out = alpha * A^T (n x n row-major)
void transpose_scale(const double* A, int64_t n, int64_t lda, double alpha, double* out,
                     int64_t ldo, cudaStream_t st);
// *out = max_i sum_j |A_ij|  (= ||A^T||_1); scratch >= 1024 doubles
void rowabs_max(const double* A, int64_t n, int64_t lda, double* scratch, double* out,
                cudaStream_t st);
// flags2[0] = 1 if X (n x n, row-major ld) has a non-finite entry, flags2[1] = 1 if X != X^T
void check_square(const double* X, int64_t n, int64_t ld, int* flags2, cudaStream_t st);
// out = sum_i c_i X_i + diag * I   (n x n, shared leading dim)
void lincomb(double* out, int64_t n, int64_t ld, LinTerm t0, LinTerm t1, LinTerm t2, LinTerm t3,
             double diag, cudaStream_t st);
// dst[:, j] = alpha * src[:, j], column-major
void copy_cols(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
               int64_t cols, double alpha, cudaStream_t st);
// dst (rows x cols column-major) <- src (rows x cols row-major)
void rowmajor_to_colmajor(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
                          int64_t cols, cudaStream_t st);
// out[:, j] = alpha * S X[:, j] (j < k) for a CSR S (n rows, int32 row pointers / column indices);
// X, out column-major with leading dimensions ldx / ldo (out != X)
void spmm_csr(const int* rp, const int* ci, const double* v, int64_t n, const double* X, int64_t ldx,
              int64_t k, double* out, int64_t ldo, double alpha, cudaStream_t st);
// C = A * B, A: M x K column-major, B: K x N column-major (small K, N), C: column-major
void tall_small(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                int64_t M, int64_t N, int64_t K, cudaStream_t st);

// G = (Z U)^T (Z U) (s x s, both triangles, ld ldg) for Z: n x k column-major, U: k x s (ld ldu),
// without storing Z U; part: scratch of >= min(ceil(n/64), #SMs) * 96^2 doubles. Deterministic.
// Returns false (nothing launched) when k > 160, s > 96 or the scratch is too small.
bool proj_gram(const double* Z, int64_t ldz, int64_t n, int k, const double* U, int64_t ldu, int s,
               double* G, int64_t ldg, double* part, size_t part_doubles, cudaStream_t st);

// Gram matrix of Zc' = [L_I | LA Tm] (and H = Zc'^T B) from the Gram Gh of GB = [L_I | B | LA]
// (q, m, kp columns; ld ldh) and Tm (kp x r, ld ldt), without touching the n-row factors:
//   G = [[Gh_II, Gh_I,LA Tm], [Tm^T Gh_LA,I, Tm^T Gh_LA,LA Tm]]  (k = q + r, column-major, ld ldg)
//   H = [Gh_I,B; Tm^T Gh_LA,B]  stored at G + k * ldg  (k x m)
// One CTA; kp, r <= 224, q + m + kp <= 224.
// Signed r1 x r1 core M = Tm^T S Tm of a Richardson combination (see aux.cu); r1 <= 112. Writes
// lam (r2), *r2_dev and T2: raw = false: Tm Theta^{-1} U_kept (k x r2, Tm = W Theta^{1/2});
// raw = true: U_kept (r1 x r2).
void signed_core(const double* Tm, int64_t ldt, int k, int r1, int kf, double wf, double wc, double tol,
                 double* T2, int64_t ldt2, double* lam, int* r2_dev, cudaStream_t st, bool raw);
size_t gram_congruence_smem(int q, int m, int kp, int r);  // <= 220 KB required
void gram_congruence(const double* Gh, int64_t ldh, int q, int m, int kp, const double* Tm,
                     int64_t ldt, int r, double* G, int64_t ldg, cudaStream_t st);

}  // namespace dme
