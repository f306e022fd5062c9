// Blocked LU with partial pivoting and the right-division solve X = P Q^{-1} for the Padé-13
// denominator and for the mass-matrix transform A M^{-1} ("dense LU").
//
// Pi Q = L U (LAPACK getrf semantics: at column j the row of largest |q_ij|, i >= j, is swapped in;
// ties go to the smallest row index, so the factorisation is deterministic). Per 64-column block:
//   panel     one cooperative launch over up to 148 CTAs, each holding a contiguous slice of the
//             panel's rows in shared memory; per column one grid-wide barrier: every CTA publishes
//             its local pivot candidate (value, row, row data) and the owner of row j publishes row
//             j; after the barrier every CTA picks the same winner, performs its part of the swap
//             and its rows' rank-1 update (candidate slots double-buffered by column parity);
//   laswp     the block's interchanges applied to the columns left and right of the panel;
//   diagonal  inverses of the factored 64 x 64 block (L11^{-1}, U11^{-1}) in one CTA;
//   U12       = L11^{-1} A12 and the trailing update A22 -= L21 U12 (DMMA gemm_nt).
// Because P = V + U and Q commute (both are polynomials of X), Q^{-1} P = P Q^{-1}; the solve is
// the right division on row-major data: W = P U^{-1} (left to right), X' = W L^{-1} (right to
// left), X = X' Pi (a column permutation), in place in P's buffer.
// (Round 1 ran this factorisation without row exchanges; that fails on well-conditioned
// denominators with a vanishing leading minor, e.g. q13 of a scaled skew block at ||X|| = pi.)
#include "aux.h"
#include "common.cuh"
#include "gemm_nt.h"
#include "lu.h"

#include <cooperative_groups.h>
#include <climits>

namespace dme {

namespace {

constexpr int NB = 64;
constexpr int DIAG_SMEM = 3 * NB * (NB + 1) * 8;
#define DME_REQUIRE_LU(cond, msg) \
  do {                            \
    if (!(cond)) throw ::dme::CudaError(msg); \
  } while (0)

// Factor the jb x jb diagonal block at D (row-major, ld) in place (unit-lower L, upper U), and
// emit Linv (row-major), LinvT (row-major = Linv^T) and UinvT (row-major = Uinv^T), ld NB.
// The jb x jb diagonal block at D (row-major, ld) holds its LU factors (unit-lower L, upper U, from
// the pivoted panel); emit Linv (row-major), LinvT (row-major = Linv^T) and UinvT (= Uinv^T), ld NB.
__global__ void __launch_bounds__(1024) diag_block_kernel(const double* D, int64_t ld, int jb,
                                                          double* Linv, double* LinvT,
                                                          double* UinvT) {
  extern __shared__ double dsm[];
  double(*a)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm);
  double(*li)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm + NB * (NB + 1));
  double(*ui)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm + 2 * NB * (NB + 1));
  const int tid = threadIdx.x;
  for (int e = tid; e < jb * jb; e += blockDim.x) a[e / jb][e % jb] = D[(e / jb) * ld + e % jb];
  __syncthreads();
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
    Linv[i * NB + j] = li[i][j];
    LinvT[i * NB + j] = li[j][i];
    UinvT[i * NB + j] = ui[j][i];
  }
}

// ------------------------------------------------------------------ pivoted panel factorisation
// Rows [j0, n) x columns [j0, j0 + jb) of Q (row-major, ld). CTA c owns rows
// [j0 + c rpc, min(n, j0 + (c + 1) rpc)) in shared memory (ld NB + 1: odd, so the column reads of
// the pivot search are conflict-free). Slots (global): cand[2][G] {|v|, row}, crow[2][G][NB] the
// candidate rows, rowk[2][NB] the current row j. Grid-wide barrier per column (cooperative launch).
struct PanelSlots {
  double* cval;   // [2][G]
  int* crow_idx;  // [2][G]
  double* crow;   // [2][G][NB]
  double* rowk;   // [2][NB]
};

constexpr int PANEL_THREADS = 256;
__device__ __forceinline__ int64_t dmax64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t dmin64(int64_t a, int64_t b) { return a < b ? a : b; }

__global__ void __launch_bounds__(PANEL_THREADS) panel_piv_kernel(double* Q, int64_t ld, int64_t n,
                                                                  int64_t j0, int jb, int rpc,
                                                                  PanelSlots sl, int* ipiv,
                                                                  double* minpiv) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double pa[];  // [rpc][NB + 1]
  constexpr int LDP = NB + 1;
  __shared__ double red_v[PANEL_THREADS / 32];
  __shared__ int red_i[PANEL_THREADS / 32];
  __shared__ double prow[NB];
  __shared__ int s_best_row, s_piv_row;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  const int64_t r_begin = j0 + (int64_t)cta * rpc;
  const int nr = (int)dmax64(0, dmin64(rpc, n - r_begin));
  for (int e = tid; e < nr * jb; e += PANEL_THREADS) {
    const int i = e / jb, j = e % jb;
    pa[i * LDP + j] = Q[(r_begin + i) * ld + j0 + j];
  }
  __syncthreads();
  double mp = 1e300;
  for (int k = 0; k < jb; ++k) {
    const int par = k & 1;
    const int64_t gk = j0 + k;
    // ---- local pivot candidate over own rows >= gk: largest |v|, ties -> smallest row
    const int i_first = (int)dmax64(0, gk - r_begin);
    double bv = -1.0;
    int bi = INT_MAX;
    for (int i = i_first + tid; i < nr; i += PANEL_THREADS) {
      const double v = fabs(pa[i * LDP + k]);
      if (v > bv) { bv = v; bi = i; }  // rows ascending per thread: first max kept
    }
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double v = red_v[0];
      int ii = red_i[0];
      for (int w = 1; w < PANEL_THREADS / 32; ++w)
        if (red_v[w] > v || (red_v[w] == v && red_i[w] < ii)) { v = red_v[w]; ii = red_i[w]; }
      s_best_row = ii;
      sl.cval[par * G + cta] = v;
      sl.crow_idx[par * G + cta] = ii == INT_MAX ? INT_MAX : (int)(r_begin + ii);
    }
    __syncthreads();
    if (s_best_row != INT_MAX)
      for (int j = tid; j < jb; j += PANEL_THREADS)
        sl.crow[((size_t)par * G + cta) * NB + j] = pa[s_best_row * LDP + j];
    if (gk >= r_begin && gk < r_begin + nr)
      for (int j = tid; j < jb; j += PANEL_THREADS) sl.rowk[par * NB + j] = pa[(gk - r_begin) * LDP + j];
    __threadfence();
    grid.sync();
    // ---- every CTA picks the same winner
    if (tid == 0) {
      double v = -1.0;
      int ir = INT_MAX, wc = 0;
      for (int c2 = 0; c2 < G; ++c2) {
        const double cv = ((volatile double*)sl.cval)[par * G + c2];
        const int ci = ((volatile int*)sl.crow_idx)[par * G + c2];
        if (cv > v || (cv == v && ci < ir)) { v = cv; ir = ci; wc = c2; }
      }
      s_piv_row = ir;
      red_i[0] = wc;
    }
    __syncthreads();
    const int64_t p = s_piv_row;
    const int wc = red_i[0];
    for (int j = tid; j < jb; j += PANEL_THREADS) prow[j] = ((volatile double*)sl.crow)[((size_t)par * G + wc) * NB + j];
    __syncthreads();
    const double piv = prow[k];
    if (tid == 0) mp = fmin(mp, fabs(piv));
    if (cta == 0 && tid == 0) ipiv[gk] = (int)p;
    // ---- interchange rows gk and p (each CTA does its part)
    if (p != gk) {
      if (gk >= r_begin && gk < r_begin + nr)
        for (int j = tid; j < jb; j += PANEL_THREADS) pa[(gk - r_begin) * LDP + j] = prow[j];
      if (p >= r_begin && p < r_begin + nr)
        for (int j = tid; j < jb; j += PANEL_THREADS)
          pa[(p - r_begin) * LDP + j] = ((volatile double*)sl.rowk)[par * NB + j];
    }
    __syncthreads();
    // ---- multipliers and rank-1 update of own rows below gk (zero pivot: column already zero)
    const double rp = piv != 0.0 ? 1.0 / piv : 0.0;
    const int i0 = (int)dmax64(0, gk + 1 - r_begin);
    const int rem = jb - k - 1;
    if (rem > 0)
      for (int e = tid; e < (nr - i0) * rem; e += PANEL_THREADS) {
        const int i = i0 + e / rem, j = k + 1 + e % rem;
        pa[i * LDP + j] -= (pa[i * LDP + k] * rp) * prow[j];
      }
    __syncthreads();
    for (int i = i0 + tid; i < nr; i += PANEL_THREADS) pa[i * LDP + k] *= rp;
    __syncthreads();
  }
  for (int e = tid; e < nr * jb; e += PANEL_THREADS) {
    const int i = e / jb, j = e % jb;
    Q[(r_begin + i) * ld + j0 + j] = pa[i * LDP + j];
  }
  if (cta == 0 && tid == 0) *minpiv = fmin(*minpiv, mp);
}

// the interchanges of rows j0 .. j0 + jb - 1 (ipiv) applied to columns [0, c0) and [c1, n)
__global__ void laswp_kernel(double* Q, int64_t ld, int64_t n, int64_t j0, int jb, int64_t c0,
                             int64_t c1, const int* __restrict__ ipiv) {
  __shared__ int pv[NB];
  for (int k = threadIdx.x; k < jb; k += blockDim.x) pv[k] = ipiv[j0 + k];
  __syncthreads();
  const int64_t ncols = c0 + (n - c1);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ncols;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = t < c0 ? t : c1 + (t - c0);
    for (int k = 0; k < jb; ++k) {
      const int64_t r = j0 + k, p = pv[k];
      if (p != r) {
        const double x = Q[r * ld + col];
        Q[r * ld + col] = Q[p * ld + col];
        Q[p * ld + col] = x;
      }
    }
  }
}

// perm = the row order of Pi Q (LAPACK: swap perm[k], perm[ipiv[k]] for k = 0 .. n-1), one CTA,
// in shared memory when it fits
__global__ void build_perm_kernel(const int* __restrict__ ipiv, int64_t n, int* perm) {
  extern __shared__ int ps[];
  const bool sm = n <= 12288;
  int* pr = sm ? ps : perm;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) pr[i] = (int)i;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int64_t k = 0; k < n; ++k) {
      const int p = ipiv[k];
      const int t = pr[k];
      pr[k] = pr[p];
      pr[p] = t;
    }
  __syncthreads();
  if (sm)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) perm[i] = pr[i];
}

// dst[r][perm[i]] = src[r][i]  (X = X' Pi)
__global__ void col_scatter_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                   int64_t n, int64_t ld, const int* __restrict__ perm) {
  const int64_t r = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[r * ld + perm[i]] = src[r * ld + i];
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

constexpr int PANEL_MAX_CTAS = 148;

size_t lu_scratch_doubles(int64_t n) {
  const int64_t nblk = ceil_div(n, NB);
  // inverses, two transposed panels, pivot slots, ipiv + perm (as doubles)
  return (size_t)nblk * 3 * NB * NB + 2 * (size_t)n * NB + 8 +
         (size_t)2 * PANEL_MAX_CTAS * (2 + NB) + 2 * NB + (size_t)n + 64;
}

void lu_solve_right(double* Q, double* P, int64_t n, int64_t ld, double* QT, double* scratch,
                    GemmScratch& gs, cudaStream_t st, double* minpiv_dev) {
  const int64_t nblk = ceil_div(n, NB);
  double* inv = scratch;                                  // per block: Linv, LinvT, UinvT
  double* T1 = scratch + (size_t)nblk * 3 * NB * NB;      // (n x NB) transposed panel
  double* T2 = T1 + (size_t)n * NB;                       // (n x NB) U12^T
  double* slots = T2 + (size_t)n * NB + 8;
  PanelSlots sl;
  sl.cval = slots;
  sl.crow = slots + 2 * PANEL_MAX_CTAS;
  sl.rowk = sl.crow + (size_t)2 * PANEL_MAX_CTAS * NB;
  sl.crow_idx = reinterpret_cast<int*>(sl.rowk + 2 * NB);        // 2 G ints
  int* ipiv = sl.crow_idx + 2 * PANEL_MAX_CTAS;                   // n ints
  int* perm = ipiv + n;                                           // n ints
  static std::mutex attr_mu;
  static uint64_t attr_mask = 0;
  per_device_once(attr_mu, attr_mask, [&] {
    DME_CUDA(cudaFuncSetAttribute(diag_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  DIAG_SMEM));
    DME_CUDA(cudaFuncSetAttribute(panel_piv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  220 * 1024));
    DME_CUDA(cudaFuncSetAttribute(build_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  12288 * 4));
  });
  int nsm = 148, dev = 0;
  DME_CUDA(cudaGetDevice(&dev));
  DME_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  init_minpiv<<<1, 1, 0, st>>>(minpiv_dev);
  DME_KCHECK();
  auto Linv = [&](int64_t b) { return inv + (size_t)b * 3 * NB * NB; };
  auto LinvT = [&](int64_t b) { return inv + (size_t)b * 3 * NB * NB + NB * NB; };
  auto UinvT = [&](int64_t b) { return inv + (size_t)b * 3 * NB * NB + 2 * NB * NB; };

  // ------------------------------------------------------------------ factorisation Pi Q = L U
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t j0 = b * NB, jb = std::min<int64_t>(NB, n - j0), j1 = j0 + jb, rest = n - j1;
    {  // pivoted panel, rows [j0, n)
      const int64_t R = n - j0;
      int G = (int)std::min<int64_t>(std::min(nsm, PANEL_MAX_CTAS), ceil_div(R, 16));
      int rpc = (int)ceil_div(R, G);
      G = (int)ceil_div(R, rpc);
      const size_t smem = (size_t)rpc * (NB + 1) * 8;
      DME_REQUIRE_LU(smem <= 220 * 1024, "pivoted LU panel exceeds shared memory (n too large)");
      int64_t a_ld = ld, a_n = n, a_j0 = j0;
      int a_jb = (int)jb;
      void* args[] = {&Q, &a_ld, &a_n, &a_j0, &a_jb, &rpc, &sl, &ipiv, &minpiv_dev};
      DME_CUDA(cudaLaunchCooperativeKernel((void*)panel_piv_kernel, dim3(G), dim3(PANEL_THREADS), args,
                                           smem, st));
      DME_KCHECK();
    }
    {  // the block's interchanges on the other columns
      const int64_t ncols = j0 + rest;
      if (ncols > 0) {
        laswp_kernel<<<(unsigned)std::min<int64_t>(ceil_div(ncols, 256), 1024), 256, 0, st>>>(
            Q, ld, n, j0, (int)jb, j0, j1, ipiv);
        DME_KCHECK();
      }
    }
    diag_block_kernel<<<1, 1024, DIAG_SMEM, st>>>(Q + j0 * ld + j0, ld, (int)jb, Linv(b), LinvT(b),
                                                  UinvT(b));
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
    // (L21 is the panel's multiplier block)
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
  // ------------------------------------------------------------------ X' = W L^{-1}
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
  // ------------------------------------------------------------------ X = X' Pi (via QT)
  build_perm_kernel<<<1, 1024, n <= 12288 ? (size_t)n * 4 : 0, st>>>(ipiv, n, perm);
  DME_KCHECK();
  col_scatter_kernel<<<dim3((unsigned)std::min<int64_t>(ceil_div(n, 256), 64), (unsigned)n), 256, 0, st>>>(
      P, QT, n, ld, perm);
  DME_KCHECK();
  DME_CUDA(cudaMemcpy2DAsync(P, ld * 8, QT, ld * 8, n * 8, n, cudaMemcpyDeviceToDevice, st));
}

}  // namespace dme
