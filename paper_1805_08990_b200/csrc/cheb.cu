// Sparse exponential action exp(tau A^T) X by a Chebyshev expansion on the Gershgorin interval
// (see cheb.h; the paper's expleja, P:L199 / P:L303-307, is a Leja/Newton
// polynomial of the same class: sparse x skinny products and vector updates only).
//
// One thread-block cluster of CHEB_CLUSTER CTAs per group of C columns. CTA r owns rows
// [r R, (r + 1) R) of the n x C block: its slice of A^T (ELL, shared memory), of the two Chebyshev
// vectors v_{k-1}, v_k (shared memory, gathered by the other CTAs through DSMEM) and of the
// accumulator y (shared memory, own rows only). Per degree k:
//   v_k = 2 (alpha A^T v_{k-1} - beta v_{k-1}) - v_{k-2}    (v_1 = alpha A^T v_0 - beta v_0)
//   y  += coef_k v_k
// v_k overwrites v_{k-2} in place (same thread, same address); one cluster barrier per degree
// separates the writes of v_k from the gathers of degree k + 1 and those gathers from the
// overwrite at degree k + 2. Everything stays on chip: HBM is touched only to load X and the
// matrix slice and to store the result.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "cheb.h"
#include "common.cuh"
#include "dme.h"

namespace dme {

namespace {

struct ChebParams {
  const double* val;
  const uint32_t* idx;
  const double* X;
  double* out;
  int64_t ldx, ldo, n;
  int R, w, k, K, substeps;
  double alpha, beta, out_scale;
  double coef[CHEB_KMAX + 1];  // coef_k = e^{c + gamma} chat_k (k ? 2 : 1), one substep
};

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ double ld_dsmem_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int C>
__global__ void __cluster_dims__(CHEB_CLUSTER, 1, 1) __launch_bounds__(CHEB_THREADS, 1)
    cheb_kernel(const __grid_constant__ ChebParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = p.R, w = p.w;
  double* val_s = reinterpret_cast<double*>(smem);                      // [w][R]
  double* buf0 = val_s + (size_t)w * R;                                 // [C][R]
  double* buf1 = buf0 + (size_t)C * R;                                  // [C][R]
  double* y_s = buf1 + (size_t)C * R;                                   // [C][R]
  uint32_t* idx_s = reinterpret_cast<uint32_t*>(y_s + (size_t)C * R);   // [w][R]
  __shared__ uint32_t rbase[2][CHEB_CLUSTER];                           // DSMEM bases of buf0/buf1

  const uint32_t me = cluster_rank();
  const int group = blockIdx.x / CHEB_CLUSTER;
  const int col0 = group * C;
  const int ncol = min(C, p.k - col0);
  const int64_t row0 = (int64_t)me * R;
  const int tid = threadIdx.x;
  if (tid < CHEB_CLUSTER) {
    rbase[0][tid] = mapa_u32(smem_u32(buf0), tid);
    rbase[1][tid] = mapa_u32(smem_u32(buf1), tid);
  }
  // matrix slice and v_0 (zero rows beyond n, zero columns beyond k)
  const int64_t ldm = (int64_t)CHEB_CLUSTER * R;
  for (int e = tid; e < w * R; e += CHEB_THREADS) {
    const int q = e / R, i = e - q * R;
    val_s[e] = p.val[q * ldm + row0 + i];
    idx_s[e] = p.idx[q * ldm + row0 + i];
  }
  for (int e = tid; e < C * R; e += CHEB_THREADS) {
    const int j = e / R, i = e - j * R;
    const int64_t gi = row0 + i;
    buf0[e] = (j < ncol && gi < p.n) ? p.X[(col0 + j) * p.ldx + gi] : 0.0;
  }
  const double alpha = p.alpha, beta = p.beta;
  for (int sub = 0; sub < p.substeps; ++sub) {
    if (sub > 0)  // v_0 of the next substep = y (own rows); the last degree's barrier freed buf0
      for (int e = tid; e < C * R; e += CHEB_THREADS) buf0[e] = y_s[e];
    for (int e = tid; e < C * R; e += CHEB_THREADS) y_s[e] = p.coef[0] * buf0[e];
    cluster_sync_all();
    for (int kd = 1; kd <= p.K; ++kd) {
      const int cur = (kd - 1) & 1;
      double* bc = cur ? buf1 : buf0;  // v_{k-1}
      double* bp = cur ? buf0 : buf1;  // v_{k-2}, overwritten by v_k
      const double ck = p.coef[kd];
      for (int i = tid; i < R; i += CHEB_THREADS) {
        double acc[C];
#pragma unroll
        for (int j = 0; j < C; ++j) acc[j] = 0.0;
        for (int q = 0; q < w; ++q) {
          const double a = val_s[q * R + i];
          const uint32_t e = idx_s[q * R + i];
          const uint32_t own = e >> 24, off = e & 0xFFFFFFu;
          if (own == me) {
#pragma unroll
            for (int j = 0; j < C; ++j) acc[j] = fma(a, bc[j * R + off], acc[j]);
          } else {
            const uint32_t base = rbase[cur][own] + off * 8u;
#pragma unroll
            for (int j = 0; j < C; ++j) acc[j] = fma(a, ld_dsmem_f64(base + (uint32_t)(j * R) * 8u), acc[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < C; ++j) {
          const double t = alpha * acc[j] - beta * bc[j * R + i];
          const double vn = kd == 1 ? t : 2.0 * t - bp[j * R + i];
          bp[j * R + i] = vn;
          y_s[j * R + i] = fma(ck, vn, y_s[j * R + i]);
        }
      }
      cluster_sync_all();
    }
  }
  for (int e = tid; e < C * R; e += CHEB_THREADS) {
    const int j = e / R, i = e - j * R;
    const int64_t gi = row0 + i;
    if (j < ncol && gi < p.n) p.out[(col0 + j) * p.ldo + gi] = p.out_scale * y_s[e];
  }
}

template <int C>
void launch_c(const ChebParams& prm, int groups, size_t smem, cudaStream_t st) {
  auto kern = cheb_kernel<C>;
  static bool attr = false;
  if (!attr) {
    DME_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
    attr = true;
  }
  kern<<<groups * CHEB_CLUSTER, CHEB_THREADS, smem, st>>>(prm);
  DME_KCHECK();
}

}  // namespace

size_t cheb_smem_bytes(int64_t R, int w, int C) {
  return (size_t)R * (size_t)w * 12 + (size_t)R * C * 24 + 64;
}

int cheb_coeffs(double gamma, double tol, std::vector<double>& chat) {
  if (!(gamma > 0)) {
    chat.assign(1, 1.0);
    return 0;
  }
  // start of the backward recurrence well beyond the degree needed (coefficients decay like
  // exp(-k^2 / (2 gamma)) for k << gamma and faster beyond)
  const int N = (int)std::ceil(gamma + 14.0 * std::sqrt(gamma) + 80.0);
  std::vector<double> t(N + 2, 0.0);
  t[N + 1] = 0.0;
  t[N] = 1e-300;
  for (int k = N; k >= 1; --k) {
    t[k - 1] = (2.0 * k / gamma) * t[k] + t[k + 1];
    if (t[k - 1] > 1e250) {  // rescale everything computed so far (values are all positive)
      for (int j = k - 1; j <= N + 1; ++j) t[j] *= 1e-250;
    }
  }
  double s = t[0];
  for (int k = 1; k <= N; ++k) s += 2.0 * t[k];
  for (int k = 0; k <= N; ++k) t[k] /= s;
  // smallest K with 2 sum_{j>K} t_j <= tol
  double tail = 0.0;
  int K = N;
  for (int k = N; k >= 1; --k) {
    if (tail + 2.0 * t[k] > tol) break;
    tail += 2.0 * t[k];
    K = k - 1;
  }
  chat.assign(t.begin(), t.begin() + K + 1);
  return K;
}

int cheb_prepare(int64_t n, int64_t nnz, const int64_t* rowptr, const int32_t* colind,
                 const double* values, ChebHost& out, std::string* err) {
  auto fail = [&](int code, const char* m) {
    if (err) *err = m;
    return code;
  };
  if (n <= 0 || nnz < 0 || !rowptr || (nnz > 0 && (!colind || !values)))
    return fail(DME_ERR_INVALID, "sparse A: NULL CSR arrays or bad sizes");
  if (rowptr[0] != 0 || rowptr[n] != nnz) return fail(DME_ERR_INVALID, "sparse A: rowptr[0] != 0 or rowptr[n] != nnz");
  for (int64_t i = 0; i < n; ++i)
    if (rowptr[i + 1] < rowptr[i]) return fail(DME_ERR_INVALID, "sparse A: rowptr not monotone");
  for (int64_t e = 0; e < nnz; ++e) {
    if (colind[e] < 0 || colind[e] >= n) return fail(DME_ERR_INVALID, "sparse A: column index out of range");
    if (!std::isfinite(values[e])) return fail(DME_ERR_INVALID, "A has non-finite entries");
  }
  // rows of A^T = columns of A (counting sort); duplicates are summed
  std::vector<int64_t> tp(n + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) tp[colind[e] + 1]++;
  for (int64_t i = 0; i < n; ++i) tp[i + 1] += tp[i];
  std::vector<int64_t> fill(tp.begin(), tp.end() - 1);
  std::vector<int32_t> tc(nnz);
  std::vector<double> tv(nnz);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int64_t d = fill[colind[e]]++;
      tc[d] = (int32_t)i;
      tv[d] = values[e];
    }
  // canonical rows (sorted, duplicates summed) of A and of A^T; A symmetric <=> equal
  auto canon = [&](const int64_t* rp, const int32_t* ci, const double* vv, int64_t i,
                   std::vector<std::pair<int32_t, double>>& row) {
    row.clear();
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) row.push_back({ci[e], vv[e]});
    std::sort(row.begin(), row.end(), [](auto& x, auto& y) { return x.first < y.first; });
    size_t o = 0;
    for (size_t e = 0; e < row.size(); ++e) {
      if (o > 0 && row[o - 1].first == row[e].first) row[o - 1].second += row[e].second;
      else row[o++] = row[e];
    }
    row.resize(o);
  };
  std::vector<std::vector<std::pair<int32_t, double>>> rowsT(n);
  std::vector<std::pair<int32_t, double>> ra;
  int w = 1;
  double a = INFINITY, b = -INFINITY, norm1 = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    canon(tp.data(), tc.data(), tv.data(), i, rowsT[i]);
    canon(rowptr, colind, values, i, ra);
    if (ra.size() != rowsT[i].size())
      return fail(DME_ERR_CONFIG, "sparse A must be symmetric (Chebyshev on the Gershgorin interval)");
    for (size_t e = 0; e < ra.size(); ++e)
      if (ra[e].first != rowsT[i][e].first || ra[e].second != rowsT[i][e].second)
        return fail(DME_ERR_CONFIG, "sparse A must be symmetric (Chebyshev on the Gershgorin interval)");
    double diag = 0.0, off = 0.0, rs = 0.0;
    for (auto& x : rowsT[i]) {
      if (x.first == i) diag += x.second;
      else off += std::fabs(x.second);
      rs += std::fabs(x.second);
    }
    a = std::min(a, diag - off);
    b = std::max(b, diag + off);
    norm1 = std::max(norm1, rs);  // rows of A^T: max row sum = ||A^T||_inf = ||A||_1 = ||A^T||_1 (symmetric)
    w = std::max<int>(w, (int)rowsT[i].size());
  }
  const int64_t R = ceil_div(n, CHEB_CLUSTER);
  if (R >= (1 << 24)) return fail(DME_ERR_DIM, "sparse A: too many rows per CTA");
  int C = 0;
  for (int c = CHEB_CMAX; c >= 1; --c)
    if (cheb_smem_bytes(R, w, c) <= 225 * 1024) { C = c; break; }
  if (C == 0) return fail(DME_ERR_DIM, "sparse A: n x (ELL width) too large for one cluster's shared memory");
  out.nnz = 0;
  for (auto& r : rowsT) out.nnz += (int64_t)r.size();
  out.n = n; out.R = R; out.w = w; out.C = C; out.a = a; out.b = b; out.norm1 = norm1;
  const int64_t ldm = (int64_t)CHEB_CLUSTER * R;
  out.val.assign((size_t)w * ldm, 0.0);
  out.idx.assign((size_t)w * ldm, 0u);
  for (int64_t i = 0; i < ldm; ++i) {
    const uint32_t self = (uint32_t)((i / R) << 24) | (uint32_t)(i % R);
    for (int q = 0; q < w; ++q) out.idx[q * ldm + i] = self;  // padding: zero times own row
    if (i >= n) continue;
    int q = 0;
    for (auto& x : rowsT[i]) {
      out.val[q * ldm + i] = x.second;
      out.idx[q * ldm + i] = (uint32_t)((x.first / R) << 24) | (uint32_t)(x.first % R);
      ++q;
    }
  }
  return 0;
}

int cheb_action(const ChebOp& op, double tau, const double* X, int64_t ldx, int64_t k, double* out,
                int64_t ldo, double alpha, cudaStream_t st) {
  if (k <= 0) return 0;
  ChebParams prm;
  std::memset(&prm, 0, sizeof(prm));
  // interval of tau A^T (tau > 0): [tau a, tau b]; substeps keep the degree within CHEB_KMAX
  std::vector<double> chat;
  int substeps = 1, K = 0;
  double c = 0, gamma = 0;
  for (;;) {
    const double ts = tau / substeps;
    c = ts * (op.a + op.b) / 2;
    gamma = ts * (op.b - op.a) / 2;
    K = cheb_coeffs(gamma, 0x1p-56, chat);
    if (K <= CHEB_KMAX) break;
    substeps *= 2;
  }
  const double scale = std::exp(c + gamma);
  for (int j = 0; j <= K; ++j) prm.coef[j] = scale * chat[j] * (j ? 2.0 : 1.0);
  prm.val = op.val; prm.idx = op.idx; prm.X = X; prm.out = out;
  prm.ldx = ldx; prm.ldo = ldo; prm.n = op.n;
  prm.R = (int)op.R; prm.w = op.w; prm.k = (int)k; prm.K = K; prm.substeps = substeps;
  prm.alpha = gamma > 0 ? (tau / substeps) / gamma : 0.0;
  prm.beta = gamma > 0 ? c / gamma : 0.0;
  prm.out_scale = alpha;
  const int C = op.C;
  const int groups = (int)ceil_div(k, C);
  const size_t smem = cheb_smem_bytes(op.R, op.w, C);
  switch (C) {
    case 1: launch_c<1>(prm, groups, smem, st); break;
    case 2: launch_c<2>(prm, groups, smem, st); break;
    case 3: launch_c<3>(prm, groups, smem, st); break;
    case 4: launch_c<4>(prm, groups, smem, st); break;
    case 5: launch_c<5>(prm, groups, smem, st); break;
    case 6: launch_c<6>(prm, groups, smem, st); break;
    case 7: launch_c<7>(prm, groups, smem, st); break;
    default: launch_c<8>(prm, groups, smem, st); break;
  }
  return K * substeps;
}

}  // namespace dme
