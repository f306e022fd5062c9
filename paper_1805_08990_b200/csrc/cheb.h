// Sparse exponential action exp(tau A^T) X for a sparse symmetric A (the paper's
// own kernel class, "expleja", P:L199 / P:L303-307: a polynomial in A built from sparse
// matrix x skinny-matrix products, one-time spectrum estimate by Gershgorin discs).
//
// Polynomial: Chebyshev expansion of exp on the Gershgorin interval [a, b] of tau A^T,
//   exp(tau A^T) = e^{c} sum'_k 2 I_k(gamma) T_k(Xs),   Xs = (tau A^T - c I) / gamma,
//   c = tau (a + b) / 2, gamma = tau (b - a) / 2,
// with the degree K fixed a priori from the coefficient tail (no norm reductions in the loop).
// For a symmetric A the truncation error is <= tail * e^{tau b} * ||X|| (spectrum inside [a, b]),
// i.e. e^{tau (b - lambda_max)} times the tail relative to the action's size: dme.cu accepts the
// expansion only when tau max(b, 0) <= ln 4 or, with a Lanczos estimate of lambda_max,
// tau (b - lambda_max) <= ln 4 (dme.cu: cheb_accurate); otherwise the dense path uses Padé-13 and
// the sparse path rejects A (DME_ERR_CONFIG).
//
// Device layout (cheb.cu): A^T in ELL form, partitioned over the CHEB_CLUSTER CTAs of a thread-block
// cluster (rows [r R, (r + 1) R) on CTA r); one cluster per group of C columns of X. Each CTA keeps
// its rows of the two Chebyshev vectors plus a halo (the other CTAs' rows its matrix rows read) in
// shared memory; after every degree the owners push the halo rows into the readers' shared memory
// (st.shared::cluster), so the gathers of the next degree are all local. One cluster barrier per
// polynomial degree.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <vector>

namespace dme {

constexpr int CHEB_CLUSTER = 8;
constexpr int CHEB_KMAX = 640;     // polynomial degree per substep (coefficients are kernel params)
constexpr int CHEB_THREADS = 512;
constexpr int CHEB_CMAX = 8;       // columns per cluster

struct ChebOp {
  int64_t n = 0, R = 0;   // rows, rows per CTA (n <= CHEB_CLUSTER * R)
  int w = 0;              // ELL width (max nonzeros per row of A^T)
  int H = 0;              // halo slots per CTA (max over the CTAs)
  int P = 0;              // halo pushes per CTA (max over the CTAs)
  int C = 0;              // max columns per cluster (shared-memory budget)
  double a = 0, b = 0;    // Gershgorin interval of A^T
  double norm1 = 0;       // ||A^T||_1
  bool sym = true;        // A == A^T: Chebyshev on [a, b]; otherwise truncated Taylor (below)
  double mu = 0, tnorm = 0;  // trace(A)/n and max(||A^T - mu I||_1, ||A^T - mu I||_inf)
  // global mode (n beyond one cluster's shared memory): ELL of A^T with global column indices,
  // one cooperative grid over all SMs, vectors in global memory (L2), one grid barrier per degree
  bool global = false;
  double *gv0 = nullptr, *gv1 = nullptr, *gy = nullptr;  // [CHEB_CLUSTER * R][KMAX] each (device)
  double* val = nullptr;    // [w][CHEB_CLUSTER * R] (device)
  uint32_t* idx = nullptr;  // [w][CHEB_CLUSTER * R]: local index into [0, R + H) (own row or halo slot)
  uint32_t* push = nullptr; // [CHEB_CLUSTER][P][2]: (own row, (dest CTA << 24) | dest slot), ~0 = none
  uint32_t* rptr = nullptr; // [CHEB_CLUSTER][R + 1]: the same pushes grouped by own row (CSR) ...
  uint32_t* rent = nullptr; // [CHEB_CLUSTER][P]: ... destinations (dest CTA << 24) | dest slot
};

// Host: from the CSR of A (0-based, n x n) build the partitioned ELL of A^T and the Gershgorin data.
// Returns 0, or a dme_status code with *err set: DME_ERR_INVALID (bad CSR / non-finite values),
// DME_ERR_CONFIG (A not exactly symmetric), DME_ERR_DIM (the layout does not fit a cluster).
struct ChebHost {
  int64_t n = 0, R = 0, nnz = 0;  // nnz: stored entries of A^T (duplicates merged)
  int w = 0, H = 0, P = 0, C = 0;
  double a = 0, b = 0, norm1 = 0;
  bool sym = true;
  double mu = 0, tnorm = 0;
  bool global = false;
  std::vector<double> val;
  std::vector<uint32_t> idx, push, rptr, rent;
};
int cheb_prepare(int64_t n, int64_t nnz, const int64_t* rowptr, const int32_t* colind,
                 const double* values, ChebHost& out, std::string* err, bool force_global = false);
size_t cheb_smem_bytes(int64_t R, int w, int H, int P, int C);

// CSR of a dense row-major device matrix (nonzero pattern, exact values), if it has at most max_nnz
// nonzeros (returns 1; 0 = too dense). scratch: device memory of >= (n + 1) * 8 + max_nnz * 12 + 8
// bytes. Used by the dense path to evaluate E_{h/2} by Chebyshev actions when A is sparse.
int cheb_csr_from_dense(const double* A, int64_t n, int64_t ld, int64_t max_nnz, void* scratch,
                        cudaStream_t st, std::vector<int64_t>& rowptr, std::vector<int32_t>& col,
                        std::vector<double>& val);

// chat[k] = e^{-gamma} I_k(gamma), k = 0..K, with K the smallest degree whose tail
// 2 sum_{j > K} chat[j] <= tol. Returns K (chat resized to K + 1). Miller's backward recurrence,
// normalised by e^{gamma} = I_0 + 2 sum I_k (all terms positive).
int cheb_coeffs(double gamma, double tol, std::vector<double>& chat);

// Nonsymmetric A (op.sym == false, the paper's advection operators P:L343-348):
// the same kernels evaluate the truncated Taylor series with scaling of Al-Mohy & Higham (2011),
//   exp(tau A^T) = (e^{tau mu / s} T_m((tau / s)(A^T - mu I)))^s,  mu = trace(A) / n,
// with (m, s) minimising m s subject to s >= tau ||A^T - mu I||_1 / theta_m (theta_m: their backward-
// error bounds for unit roundoff 2^-53, m <= 55): accurate for any A, no spectrum information.
// out[:, j] = alpha * exp(tau A^T) X[:, j], j < k (column-major, leading dims ldx / ldo; out != X).
// Returns the total polynomial degree applied (sum over substeps).
int cheb_action(const ChebOp& op, double tau, const double* X, int64_t ldx, int64_t k, double* out,
                int64_t ldo, double alpha, cudaStream_t st);

}  // namespace dme
