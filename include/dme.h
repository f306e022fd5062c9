/*
 * dme.h — C ABI of the B200 hot path for low-rank splitting schemes on (generalized) differential
 * Lyapunov and Riccati equations (Mena, Pfurtscheller, Stillfjord, arXiv 1805.08990).
 *
 *   P' = A^T P + P A + Q [+ S P S^T] [- P B R^{-1} B^T P],   P(0) = P0,   Q = C^T C     (PAPER §1, §2)
 *
 * The solution is kept in low-rank form P = L D L^T. Each step applies Lie / Strang
 * compositions of the sub-flows
 *   T1  linear      L <- exp(tau A^T) L                                  eq:F_sol_LDL
 *   T2  constant    [L, L_Q], blkdiag(D, tau D_Q)
 *   T12 affine      [exp(tau A^T) L, L_I(tau)], blkdiag(D, D_I)          eq:full P:L129, Alg. 2
 *   T3  Riccati     D <- (I + tau D L^T B R^-1 B^T L)^-1 D               eq:nonlinear P:L152-156, Alg. 3
 *   T4  bilinear    [L, sqrt(tau) S L, tau/sqrt(2) S^2 L], blkdiag(D,D,D) P:L170-180, Alg. 4
 * with column compression after every rank-growing flow. exp(tau A^T) is a dense FP64
 * matrix computed once at init by scaling-and-squaring Padé-13 (BASELINE.json north_star); L_I is
 * the composite Gauss-Legendre quadrature factor of the integral term (reading G6 in DESIGN.md).
 *
 * Conventions
 *  - All matrices are FP64, HOST pointers, ROW-MAJOR (C order): element (i, j) of an r x c matrix
 *    X is X[i*c + j]. Inputs are copied at init; the caller keeps ownership and may free them.
 *  - Device memory: the library carves everything out of ONE caller-owned device buffer
 *    (options.workspace, options.workspace_bytes >= dme_workspace_size(...)); it never calls
 *    cudaMalloc on the hot path. Work is enqueued on options.stream (cudaStream_t, NULL = legacy).
 *  - Errors: every call returns a dme_status; no call aborts or throws across the ABI.
 *    dme_last_error() returns a thread-local description of the last failure.
 *    Validation failures leave the context unchanged; CUDA/NCCL failures poison it
 *    (every later call returns DME_ERR_POISONED).
 *  - A context is not thread-safe; separate contexts are independent.
 *  - Multi-GPU (world_size > 1): one process per GPU; rows of exp(tau A^T) are sharded over the
 *    ranks and the updated factor is all-gathered (NCCL) after every T1/T12 action. dme_split_step
 *    is collective. The small systems are replicated, so dme_get_factor works on every rank.
 */
#ifndef DME_H
#define DME_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dme_ctx dme_ctx; /* opaque, owned by the library */

typedef enum {
  DME_OK = 0,
  DME_ERR_INVALID = 1,  /* NULL pointer, n <= 0, non-finite input, R not SPD, D0 not PSD, h <= 0 */
  DME_ERR_DIM = 2,      /* inconsistent sizes (e.g. m > 8, rank bound above the small-system limit) */
  DME_ERR_CONFIG = 3,   /* composition needs data the problem lacks (F3 without B, F4 without S),
                           unknown scheme / composition / flow, tau not in {h/2, h} */
  DME_ERR_SINGULAR = 4, /* a small linear system is singular */
  DME_ERR_NUMERIC = 5,  /* non-finite result, expm overflow, Padé denominator pivot too small */
  DME_ERR_CAPACITY = 6, /* caller buffer too small (get_factor) or workspace too small */
  DME_ERR_CUDA = 7,
  DME_ERR_NCCL = 8,
  DME_ERR_NOMEM = 9,
  DME_ERR_POISONED = 10
} dme_status;

typedef enum { DME_LIE = 0, DME_STRANG = 1 } dme_scheme;

/* Figure-legend names of the paper: order in which the sub-problems are solved. */
typedef enum {
  DME_F1F2 = 0,     /* DLE splitting, Alg. 1                                 */
  DME_F12 = 1,      /* DLE quadrature, Alg. 2                                */
  DME_F12F3 = 2,    /* DRE two-term: T12(h/2) T3(h) T12(h/2)            */
  DME_F1F2F3 = 3,   /* DRE three-term: T1 T2 T3 T2 T1            */
  DME_F1F3F2 = 4,   /* DRE three-term reversed: T1 T3 T2 T3 T1            */
  DME_F12F4 = 5,    /* generalized DLE, T3 replaced by T4            */
  DME_F1F2F4 = 6,
  DME_F1F4F2 = 7,
  DME_F12F3F4 = 8,  /* generalized DRE: T12(h/2) T3(h/2) T4(h) T3(h/2) T12(h/2)   */
  DME_F1F2F3F4 = 9  /* four-term splitting (beyond the paper; reading G19)         */
} dme_composition;

typedef struct {
  int64_t n;          /* state dimension                                                    */
  const double* A;    /* n x n row-major (NULL with a sparse A, see A_rowptr below)         */
  int64_t p;          /* rows of C (p >= 0); Q = C^T C                                      */
  const double* C;    /* p x n (NULL iff p == 0)                                            */
  int64_t m;          /* columns of B; 0 for a DLE                                          */
  const double* B;    /* n x m                                                              */
  const double* R;    /* m x m, symmetric positive definite                                 */
  const double* S;    /* n x n or NULL (generalized equations)                              */
  int64_t r0;         /* columns of L0 (0 => P0 = 0)                                        */
  const double* L0;   /* n x r0                                                             */
  const double* D0;   /* r0 x r0 symmetric positive semidefinite (NULL => identity)         */
  const double* M;    /* n x n mass matrix or NULL (Example 4): the equation is
                         M^T P' M = A^T P M + M^T P A + C^T C [- M^T P B R^-1 B^T P M]
                         [+ M^T S P S^T M is NOT supported with M]; init cancels M once
                         (P:L357-359): A <- A M^-1, C <- C M^-1 (dense LU,
                         P:L362 "compute and store a dense LU factorization", with partial
                         pivoting; DME_ERR_NUMERIC on an exactly singular M).
                         Same memory space as A (host, or device with big_inputs_on_device).
                         Callers that zero-initialise the struct get M = NULL.              */
  /* Sparse A (the paper's own setting, P:L199 / P:L303-307: exp(tau A^T) L as a
     polynomial in the sparse A, no dense matrix exponential). Used when A == NULL and
     A_rowptr != NULL: A in CSR form (host arrays, 0-based, row-major: row i holds entries
     A_colind[e], A_values[e] for e in [A_rowptr[i], A_rowptr[i+1]); duplicates are summed).
     Every E_tau L action is then, for an exactly symmetric A, a Chebyshev expansion of exp on the
     Gershgorin interval of tau A^T (truncation tail <= 2^-56, degree fixed at init; DME_ERR_CONFIG
     when the Gershgorin bound is too loose for it), and for a nonsymmetric A the
     truncated Taylor series with scaling of Al-Mohy & Higham (cheb.h; degree m <= 55 and s substeps
     from ||tau (A^T - mu I)||), evaluated by the same cluster kernels; the quadrature rule is unchanged (its panel count
     still comes from ||(h/2) A^T||_1), and init builds no n x n matrix. While n x (row width) fits
     the shared memory of one 8-CTA cluster (n ~ 1.2e4 rows of a 5-point stencil) the actions run
     on chip in cluster kernels; beyond, in a grid-wide cooperative kernel with the vectors in
     global memory (any n with n x 224 < 2^31). Not combinable with M or with world_size > 1
     (DME_ERR_CONFIG).
     Callers that zero-initialise the struct get the dense path.                          */
  int64_t A_nnz;
  const int64_t* A_rowptr; /* n + 1 */
  const int32_t* A_colind; /* A_nnz */
  const double* A_values;  /* A_nnz */
  /* Sparse S (SURVEY / VERDICT r1 item 10; "S sparse"): used when S == NULL and
     S_rowptr != NULL. S in CSR form (host arrays, 0-based, row-major; duplicates summed), finite
     values. The T4 flow's S L and S (S L) products are then CSR x skinny products on the GPU
     (replicated on every rank, no collective) instead of two 8 n^2-byte streams of a dense S.
     Callers that zero-initialise the struct get S_rowptr = NULL.                           */
  int64_t S_nnz;
  const int64_t* S_rowptr; /* n + 1 */
  const int32_t* S_colind; /* S_nnz */
  const double* S_values;  /* S_nnz */
} dme_problem;

typedef struct {
  double h;               /* step size; E_{h/2}, E_h and L_I(h/2), L_I(h) are built at init    */
  double trunc_tol;       /* relative truncation tolerance of the compression (default 1e-16)  */
  int32_t rank_cap;       /* maximum rank kept by a compression (0 = no cap)                   */
  int32_t quad_nodes;     /* Gauss-Legendre nodes per panel (default 14)               */
  int32_t quad_subpanels; /* P0 >= 1, power of two: panels per Padé scaling step (default 1)   */
  int32_t device;         /* CUDA device ordinal                                               */
  void* stream;           /* cudaStream_t (NULL = legacy default stream)                       */
  int32_t world_size;     /* ranks (1 = single GPU)                                            */
  int32_t world_rank;
  const void* nccl_uid;   /* 128-byte ncclUniqueId from dme_get_unique_id on rank 0           */
  void* workspace;        /* device buffer, >= dme_workspace_size bytes, 256-byte aligned     */
  size_t workspace_bytes;
  int32_t big_inputs_on_device; /* 1: prob->A and prob->S are DEVICE pointers (same row-major
                             layout, copied device-to-device at init); every other input stays
                             a host pointer. 0 (default): all inputs are host pointers          */
  int32_t no_fsal;        /* 0 (default): within one dme_split_step call, merge the trailing
                             T1/T12(h/2) of a Strang step with the leading one of the next step
                             (first-same-as-last); 1: apply every sub-step as written           */
  int32_t e_pass;         /* kernel of the E_{h/2} L / E_h L passes (dme_e_pass):
                             DME_EPASS_AUTO (default): int8 tensor cores with exact digit
                             slicing (Ozaki scheme, 8 x 7-bit digits per operand, int32 exact
                             accumulation, FP64 assembly; error per entry <= ~2^-54
                             max_l|E_il| sum_l|L_lj|) when n <= 32768 and the
                             pass has <= 64 columns, else FP64 DMMA; the Padé products and
                             squarings of the (replicated) init use the same int8 kernel
                             (square tiles); DME_EPASS_DMMA: every E pass and every init
                             product in native FP64 DMMA (mma.sync m8n8k4 f64)                  */
  int32_t expm;           /* how the dense path builds E_{h/2} (dme_expm): DME_EXPM_AUTO
                             (default): when A is exactly symmetric and sparse (<= 16 n nonzeros,
                             found by a device scan of the uploaded A; replicated per rank like the Padé init), E_{h/2} =
                             exp((h/2) A^T) I column block by column block with the Chebyshev
                             actions of the sparse path and the quadrature factors
                             by Chebyshev actions too; E_h = E_{h/2}^2 as before. Otherwise, or
                             with DME_EXPM_PADE, scaling-and-squaring Padé-13                  */
  int32_t compression;    /* how a column compression resolves the eigenvalues of P = Zc Zc^T
                             (dme_compression). DME_COMPRESS_REFINED (default): the FP64 Gram
                             G = Zc^T Zc only resolves eigenvalues down to ~k eps theta_max, so a
                             first eigen pass keeps theta > 1e-11 theta_max (accurate), and the
                             rest is recomputed from the explicit projected factor
                             Zs = Zc (I - W W^T) (its Gram resolves down to ~eps^2 theta_max):
                             the truncation then honours trunc_tol down to 1e-16 as the paper's
                             reduced-SVD compression does.
                             DME_COMPRESS_GRAM: the single Gram pass, with the effective
                             tolerance max(trunc_tol, 1e-14)                                    */
  int32_t virtual_world;  /* G > 1 with world_size == 1: run the row-sharded multi-GPU code on ONE
                             GPU as G virtual shards: every E pass computes each shard's rows into
                             its staging block, one ncclAllGather on a one-rank communicator and
                             the unpack, exactly as a G-rank run does (test hook for the a13 path;
                             results equal the unsharded run up to rounding). 0/1: off           */
} dme_options;

typedef enum { DME_COMPRESS_REFINED = 0, DME_COMPRESS_GRAM = 1 } dme_compression;

typedef enum { DME_EXPM_AUTO = 0, DME_EXPM_PADE = 1 } dme_expm;

typedef enum { DME_EPASS_AUTO = 0, DME_EPASS_DMMA = 1 } dme_e_pass;

typedef struct {
  double t;                 /* integrated time (steps * h)                                     */
  int64_t steps;            /* completed steps                                                 */
  int64_t rank;             /* current rank of the factor                                      */
  int64_t max_rank;         /* largest rank seen after a compression                           */
  int64_t q_half, q_full;   /* ranks of L_I(h/2), L_I(h)                                       */
  int32_t squarings;        /* s: Padé-13 scaling exponent of (h/2) A^T; it fixes the quadrature
                               panel count (reading G6) also when E_{h/2} is built by Chebyshev
                               actions (then no squarings beyond E_h = E_{h/2}^2 are performed) */
  int32_t quad_panels;      /* panels of the composite rule on [0, h/2]                        */
  double panel_width;       /* delta = (h/2) / panels                                          */
  double pade_min_pivot;    /* smallest |u_ii| of the Padé denominator factorisation           */
  double last_drop;         /* largest discarded pivot / max diag of the last compression      */
  int64_t e_passes;         /* number of E*L actions (T1/T12/T4 passes)                        */
  int64_t compressions;
  double init_seconds;      /* host wall time of the init call                                 */
  int64_t kernel_launches;  /* kernels launched by the library in this process so far          */
  /* device-time accounting, filled only while profiling is on (dme_set_profiling) */
  int64_t prof_passes;      /* E*L / S*L passes timed                                          */
  double prof_epass_seconds;/* summed CUDA-event duration of those passes                      */
  double prof_epass_flops;  /* algorithmic flops of those passes: 2 * rows * n * k each        */
  double prof_epass_bytes;  /* algorithmic bytes: 8 * rows * n each (the dense matrix, read once) */
  double prof_gram_seconds; /* Gram matrices Zc^T Zc (and Zc^T B)                              */
  double prof_small_seconds;/* one-CTA eigen-compression / Riccati kernel                      */
  double prof_apply_seconds;/* Zc * Tm                                                         */
  int64_t eig_fallbacks;    /* fast eigen-compressions that failed the orthogonality check and
                               were redone by the Jacobi kernel                                 */
  int64_t ozaki_passes;     /* E passes run on the int8 tensor cores (options.e_pass)          */
  int64_t cheb_degree;      /* sparse A: polynomial degree of the E_h action (sum over substeps);
                               dense A with a Chebyshev-built E: the degree used for E_{h/2}     */
  int64_t expm_chebyshev;   /* 1 if E_{h/2} was built by Chebyshev actions, 0 for Padé-13     */
} dme_stats;

void dme_default_options(dme_options* opt);
const char* dme_status_string(dme_status s);
const char* dme_last_error(void);

/* Bytes of device workspace needed for this problem/options. */
dme_status dme_workspace_size(const dme_problem* prob, const dme_options* opt, size_t* bytes);
/* 128-byte NCCL unique id (rank 0 calls it and broadcasts the bytes). */
dme_status dme_get_unique_id(void* uid128);

/* Row shard of rank `rank` among `world` ranks (host-only, no device): rows [*row0, *row0 + *rows)
 * of E are owned by the rank; every rank's staging block has *nloc rows (n_loc = ceil(n/world)
 * rounded up to 16; the last ranks may own fewer or no rows). */
dme_status dme_shard_rows(int64_t n, int32_t world, int32_t rank, int64_t* row0, int64_t* rows,
                          int64_t* nloc);

/* Build the context: upload, E_{h/2} = exp((h/2)A^T) (options.expm: Chebyshev actions for an
 * exactly symmetric sparse-pattern A under AUTO, else scaling-and-squaring Padé-13 with a pivoted
 * LU solve) and E_h = E_{h/2}^2, quadrature factors, compression of P0. dle_init requires m == 0;
 * dre_init requires m >= 1. Collective. */
dme_status dme_dle_init(const dme_problem* prob, const dme_options* opt, dme_ctx** ctx);
dme_status dme_dre_init(const dme_problem* prob, const dme_options* opt, dme_ctx** ctx);

/* Advance nsteps steps of the composition (collective when world_size > 1). */
dme_status dme_split_step(dme_ctx* ctx, dme_scheme scheme, dme_composition comp, int64_t nsteps);

/* Copy the factor to the host: *r <- rank; if L != NULL, L (n x r) and, if D != NULL, D (r x r)
 * with P = L D L^T. Returns DME_ERR_CAPACITY (and sets *r) when r > capacity_cols. */
dme_status dme_get_factor(dme_ctx* ctx, int64_t* r, double* L, double* D, int64_t capacity_cols);
/* Richardson extrapolation of the Strang composition (the paper cites higher-order
 * splitting, and uses Strang): `fine` and `coarse` are two contexts of the same
 * problem on one device, fine with step h/2 after 2N Strang steps, coarse with step h after N
 * steps (DME_ERR_CONFIG otherwise). Strang's error expands in even powers of h, so
 *   P = (4 P_fine - P_coarse) / 3 = Zc S Zc^T,  Zc = [Z_fine | Z_coarse],  S = diag(4/3 I, -1/3 I)
 * is accurate to order 4. Computed on the device in the fine context's workspace: an orthonormal
 * basis Q of span(Zc) by classical Gram-Schmidt with reorthogonalisation (columns inside the span
 * to 1e-14 dropped), R^T = Zc^T Q, eigen-decomposition of the signed core R S R^T (parallel
 * Jacobi, indefinite), L = Q U, truncation by |lambda| relative to max |lambda| (trunc_tol);
 * returns L (n x r, row-major, orthonormal columns) and the diagonal, possibly indefinite, core
 * D (r x r) on the host. L = D = NULL: only *r. DME_ERR_CAPACITY when r > capacity_cols,
 * DME_ERR_DIM when the combined rank exceeds 224 (or 112 after the Gram truncation). */
dme_status dme_extrapolate(dme_ctx* fine, dme_ctx* coarse, int64_t* r, double* L, double* D,
                           int64_t capacity_cols);
dme_status dme_get_stats(dme_ctx* ctx, dme_stats* st);
/* Turn CUDA-event timing of the kernel classes on (1) or off (0); resets the prof_* counters. */
dme_status dme_set_profiling(dme_ctx* ctx, int32_t on);
/* Sparse-A path, host only (no device): chat[k] = e^{-gamma} I_k(gamma) for k = 0..*K, the
 * Chebyshev coefficients of e^{gamma (x - 1)} on [-1, 1] (modified Bessel functions, Miller's
 * backward recurrence normalised by I_0 + 2 sum I_k = e^gamma); *K is the smallest degree with
 * 2 sum_{j > K} chat[j] <= tol. out holds cap doubles (DME_ERR_CAPACITY if K + 1 > cap). */
dme_status dme_cheb_coeffs(double gamma, double tol, double* out, int64_t cap, int32_t* K);

dme_status dme_destroy(dme_ctx* ctx);

/* ---- test hooks (same semantics as the step, one flow at a time) ----------------------------- */
typedef enum {
  DME_FLOW_T1 = 0, DME_FLOW_T2 = 1, DME_FLOW_T3 = 2, DME_FLOW_T4_MIDPOINT = 3,
  DME_FLOW_T4_EULER = 4, DME_FLOW_T12 = 5, DME_FLOW_COMPRESS = 6
} dme_flow;
/* Apply one flow over tau (T1/T12: tau must be h/2 or h). */
dme_status dme_debug_apply(dme_ctx* ctx, int32_t flow, double tau);
/* Replace the state by P = L L^T (L: n x r host, row-major; no compression). */
dme_status dme_debug_set_factor(dme_ctx* ctx, int64_t r, const double* L);
/* Copy E_{h/2} (which = 0) or E_h (which = 1) to the host (n x n). */
dme_status dme_debug_get_exp(dme_ctx* ctx, int32_t which, double* E);
/* Replace E_{h/2} (which = 0) or E_h (which = 1) by a host matrix (n x n, row-major; e.g. an oracle
 * exponential: the SURVEY's "minimum slice" hook). The quadrature factors built at init are kept;
 * the int8 digit image of the E pass is re-sliced. DME_ERR_CONFIG with a sparse A. */
dme_status dme_debug_set_exp(dme_ctx* ctx, int32_t which, const double* E);
/* Copy L_I(h/2) (which = 0) or L_I(h) (which = 1), P_I = L_I L_I^T, n x q, to the host. */
dme_status dme_debug_get_integral(dme_ctx* ctx, int32_t which, int64_t* q, double* L,
                                  int64_t capacity_cols);
/* Copy the 16 diagnostic doubles of the last small-system kernel (rank, theta_max, drop ratio,
 * fallback flag, orthogonality error, -, -, -, per-phase clock cycles of the fast eigen path). */
dme_status dme_debug_small_stats(dme_ctx* ctx, double* out16);
/* C (M x N) = A (M x K) * B (K x N) through the library's DMMA GEMM (host buffers). */
dme_status dme_debug_matmul(int64_t M, int64_t N, int64_t K, const double* A, const double* B,
                            double* C);
/* The same product through the int8 digit-slicing kernel of the E pass (N <= 64, K <= 32768). */
dme_status dme_debug_matmul_ozaki(int64_t M, int64_t N, int64_t K, const double* A, const double* B,
                                  double* C);
/* Orthonormal basis U (k x (k - kb), row-major host array) of the complement of span(W), W (k x kb,
 * row-major host array, orthonormal columns), through the refined compression's complement-basis
 * kernel (P:L245-246 tail pass, reading G7'); 0 <= kb < k <= 160. Test hook. */
dme_status dme_debug_complement(int64_t k, int64_t kb, const double* W, double* U);

#ifdef __cplusplus
}
#endif
#endif /* DME_H */
