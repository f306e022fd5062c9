#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace dme {

constexpr int SMALL_K_MAX = 224;          // packed k(k+1)/2 doubles fit in 201 KB of shared memory
constexpr int SMALL_M_MAX = 8;
constexpr int FAST_K_MAX = 160;           // fast tridiagonal eigen-compression: k x (k|1) in smem
constexpr int EIG_SPLIT_MIN = 48;         // k from which the eigen-compression runs as TRI/VEC/FIN
constexpr int EIG_SPLIT_CTAS = 32;        // CTAs of the VEC kernel (the look-ahead E pass leaves them;
                                          // 8 CTAs measured slower: 68 vs 56 us in-step, the per-CTA
                                          // chains lengthen); DME_VEC_CTAS >= 32 for A/B            // columns of B handled by the fused Riccati flow
constexpr int SMALL_SMEM_MAX = SMALL_K_MAX * (SMALL_K_MAX + 1) / 2 * 8;

// Host-mapped (pinned, zero-copy) record through which the small kernels publish the new rank:
// the host spins on `seq` instead of a D2H copy + stream synchronisation per compression.
struct HostMap {
  int seq;
  int r;
  double stats[5];
};

struct SmallArgs {
  int k = 0;                 // columns of the concatenated factor Zc
  int compress = 1;          // 1: eigen-compression of G (Z_new = Zc W_kept)
  const double* G = nullptr; // k x k Gram matrix Zc^T Zc, column-major, leading dim ldg
  int64_t ldg = 0;
  double tol = 1e-16;        // relative truncation tolerance (reading G7)
  double ref_max = 0.0;      // > 0: keep theta > tol * ref_max (the theta_max of an enclosing
                             // compression: the refinement pass of the tail, dme.cu) instead of
                             // tol * (this matrix's theta_max); stats[1], stats[2] refer to it
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
  double* stats = nullptr;   // out: [rank, theta_max, largest dropped / theta_max, fallback, orth err]
  double* Es = nullptr;      // split path: global scratch (eig_split_scratch_doubles())
  int zsmem = 1;             // fast path: back-transformation columns in shared memory when they fit
  double orth_tol = 1e-12;   // fast path: max weighted |W^T W - I| before falling back to Jacobi
  HostMap* map = nullptr;    // device alias of the host-mapped record (nullptr: r_out only)
  int map_seq = 0;           // sequence number this launch publishes
  int msec_p = 128;          // split path: multisection probes per eigenvalue (cap)
  int skip_fin = 0;          // split path: no FIN kernel (the caller's tail assembly checks and publishes)
};

void compress_t3(const SmallArgs& a, cudaStream_t st);  // Jacobi (any k <= SMALL_K_MAX)
void eig_fast(const SmallArgs& a, cudaStream_t st);     // k <= FAST_K_MAX; *r_out = -1 => fall back
void eig_split(const SmallArgs& a, cudaStream_t st);    // 3 <= k <= FAST_K_MAX, same contract
size_t eig_split_scratch_doubles();
void t3_only(const SmallArgs& a, int r, cudaStream_t st);  // T3 on Tm (k x r) alone
// U (k x (k - kb), ldu): orthonormal basis of the complement of span(W), W = k x kb orthonormal
void complement_basis(const double* W, int64_t ldw, int k, int kb, double* U, int64_t ldu,
                      cudaStream_t st, bool attrs_only = false);
// The same with kb read on the device (*kb_dev: the rank the first eigen pass published; < 0 makes
// it a no-op), so it can be queued before the host has seen kb; false: not available (k > 96)
bool complement_basis_dev(const double* W, int64_t ldw, int k, const int* kb_dev, double* U, int64_t ldu,
                          cudaStream_t st, const struct SmallArgs* fin = nullptr);
bool complement_dev_available(int k);  // complement_basis_dev's kernel applies (k <= 96)
// fin != nullptr: the split first pass was launched with skip_fin; the kernel does its FIN work
// (check, stats, publish of kb or -1) and reads kb from the pass's scratch header
// a.Tm[:, kb:kb+ks] = U V (U: k x s, V: s x ks), then T3 on a.Tm (k x (kb + ks)) if a.t3.
// ks_dev != nullptr: ks is read on the device (the rank the preceding eigen pass published; a
// negative value -- Jacobi fallback pending -- makes the kernel a no-op); ks is then an upper bound
size_t tail_assemble_smem(int k, int m, int s, int kb, int ks);
// fin != nullptr (the split eigen pass of the tail launched with skip_fin): the kernel first does
// that pass's FIN work -- weighted orthogonality check of V, stats, publish of ks or -1 -- with ks
// read from the pass's scratch header; ks is then an upper bound
void tail_assemble_t3(const SmallArgs& a, const double* U, int64_t ldu, int s, const double* V,
                      int64_t ldv, int kb, int ks, cudaStream_t st, const int* ks_dev = nullptr,
                      const SmallArgs* fin = nullptr);

// global scratch of the split eigen path (doubles): header, tridiagonal, eigenvalues, reflectors
struct EsLayout {
  static constexpr int HDR = 16;
  double* base;
  int KM;  // capacity (SMALL_K_MAX)
  __host__ __device__ double* hdr() const { return base; }
  __host__ __device__ double* d() const { return base + HDR; }
  __host__ __device__ double* e() const { return base + HDR + KM; }
  __host__ __device__ double* e2() const { return base + HDR + 2 * KM; }
  __host__ __device__ double* tau() const { return base + HDR + 3 * KM; }
  __host__ __device__ double* lam() const { return base + HDR + 4 * KM; }  // KM + 1
  __host__ __device__ double* refl() const { return base + HDR + 5 * KM + 8; }  // k x ld
  __host__ __device__ double* dp() const { return refl() + (size_t)KM * (KM | 1); }  // KM x KM
  __host__ __device__ double* dm() const { return dp() + (size_t)KM * KM; }
};
// Pp = I - W W^T (k x k), W: k x kb (the kept leading eigenvectors of the first pass)
void complement_projector(const double* W, int64_t ldw, int k, int kb, double* Pp, int64_t ldp,
                          cudaStream_t st);

}  // namespace dme
