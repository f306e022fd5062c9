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
#include <cstdlib>

#include "cheb.h"

#include <cooperative_groups.h>
#include <memory>
#include "common.cuh"
#include "dme.h"
#include "small.h"

namespace dme {

namespace {

constexpr int TAYLOR_MMAX = 55;
// theta_m of Al-Mohy & Higham (2011), Table 3.1 / Higham (2008) Table A.3, unit roundoff 2^-53
constexpr int TAYLOR_NM = 35;
const int TAYLOR_M[TAYLOR_NM] = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20,
                                 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 35, 40, 45, 50, 55};
const double TAYLOR_THETA[TAYLOR_NM] = {
    2.29e-16, 2.58e-8, 1.39e-5, 3.40e-4, 2.40e-3, 9.07e-3, 2.38e-2, 5.00e-2, 8.96e-2, 1.44e-1,
    2.14e-1, 3.00e-1, 4.00e-1, 5.14e-1, 6.41e-1, 7.81e-1, 9.31e-1, 1.09, 1.26, 1.44,
    1.62, 1.82, 2.01, 2.22, 2.43, 2.64, 2.86, 3.08, 3.31, 3.54, 4.7, 6.0, 7.2, 8.5, 9.9};

struct ChebParams {
  const double* val;
  const uint32_t* idx;
  const uint32_t* push;
  const uint32_t* rptr;
  const uint32_t* rent;
  const double* X;
  double* out;
  int64_t ldx, ldo, n;
  int R, w, H, P, k, K, substeps;
  double alpha, beta, out_scale;
  double coef[CHEB_KMAX + 1];  // coef_k = e^{c + gamma} chat_k (k ? 2 : 1), one substep
  // Taylor mode (nonsymmetric A): v_k = (alpha A^T v_{k-1} - beta v_{k-1}) / k, y += coef_k v_k
  int taylor;
  double rk[TAYLOR_MMAX + 1];  // 1 / k
};

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_dsmem_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
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

// Shared memory of CTA r: val [w][R], buf0 / buf1 [C][R + H] (own rows, then halo slots),
// y [C][R], idx [w][R] (local indices), push [P][2].
// C columns per cluster; W: ELL entries gathered per batch (all loads of a batch are issued before
// the first FMA: the row's matrix entries, then its W x C neighbour values)
template <int C, int W>
__global__ void __cluster_dims__(CHEB_CLUSTER, 1, 1) __launch_bounds__(CHEB_THREADS, 1)
    cheb_kernel(const __grid_constant__ ChebParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = p.R, w = p.w, LD = p.R + p.H, P = p.P;
  double* val_s = reinterpret_cast<double*>(smem);
  double* buf0 = val_s + (size_t)w * R;
  double* buf1 = buf0 + (size_t)C * LD;
  double* y_s = buf1 + (size_t)C * LD;
  uint32_t* idx_s = reinterpret_cast<uint32_t*>(y_s + (size_t)C * R);
  uint32_t* push_s = idx_s + (size_t)w * R;
  __shared__ uint32_t rbase[2][CHEB_CLUSTER];  // DSMEM addresses of buf0 / buf1 in every CTA

  const uint32_t me = cluster_rank();
  const int col0 = (blockIdx.x / CHEB_CLUSTER) * C;
  const int ncol = min(C, p.k - col0);
  const int64_t row0 = (int64_t)me * R;
  const int tid = threadIdx.x;
  if (tid < CHEB_CLUSTER) {
    rbase[0][tid] = mapa_u32(smem_u32(buf0), tid);
    rbase[1][tid] = mapa_u32(smem_u32(buf1), tid);
  }
  const int64_t ldm = (int64_t)CHEB_CLUSTER * R;
  for (int e = tid; e < w * R; e += CHEB_THREADS) {
    const int q = e / R, i = e - q * R;
    val_s[e] = p.val[q * ldm + row0 + i];
    idx_s[e] = p.idx[q * ldm + row0 + i];
  }
  for (int e = tid; e < 2 * P; e += CHEB_THREADS) push_s[e] = p.push[(int64_t)me * 2 * P + e];
  for (int e = tid; e < C * R; e += CHEB_THREADS) {
    const int j = e / R, i = e - j * R;
    const int64_t gi = row0 + i;
    buf0[j * LD + i] = (j < ncol && gi < p.n) ? p.X[(col0 + j) * p.ldx + gi] : 0.0;
  }
  __syncthreads();
  // owners store the rows other CTAs read into those CTAs' halo slots of buffer b
  auto push_rows = [&](const double* b, int bi) {
    for (int e = tid; e < P; e += CHEB_THREADS) {
      const uint32_t src = push_s[2 * e], d = push_s[2 * e + 1];
      if (src == 0xFFFFFFFFu) continue;
      const uint32_t base = rbase[bi][d >> 24] + (d & 0xFFFFFFu) * 8u;
#pragma unroll
      for (int j = 0; j < C; ++j) st_dsmem_f64(base + (uint32_t)(j * LD) * 8u, b[j * LD + src]);
    }
  };
  const double alpha = p.alpha, beta = p.beta;
  // every CTA of the cluster has started (and initialised its shared memory) before any peer
  // pushes into it (compute-sanitizer racecheck: DSMEM store into a block not yet entered)
  cluster_sync_all();
  for (int sub = 0; sub < p.substeps; ++sub) {
    if (sub > 0) {  // v_0 of the next substep = y (own rows)
      for (int e = tid; e < C * R; e += CHEB_THREADS) {
        const int j = e / R, i = e - j * R;
        buf0[j * LD + i] = y_s[e];
      }
      __syncthreads();
    }
    push_rows(buf0, 0);
    for (int e = tid; e < C * R; e += CHEB_THREADS) {
      const int j = e / R, i = e - j * R;
      y_s[e] = p.coef[0] * buf0[j * LD + i];
    }
    cluster_sync_all();
    for (int kd = 1; kd <= p.K; ++kd) {
      const int cur = (kd - 1) & 1;
      const double* bc = cur ? buf1 : buf0;  // v_{k-1} (own rows + halo)
      double* bp = cur ? buf0 : buf1;        // v_{k-2}, overwritten by v_k
      const double ck = p.coef[kd];
      for (int i = tid; i < R; i += CHEB_THREADS) {
        double acc[C];
#pragma unroll
        for (int j = 0; j < C; ++j) acc[j] = 0.0;
        for (int q0 = 0; q0 < w; q0 += W) {
          double a[W];
          uint32_t e[W];
#pragma unroll
          for (int u = 0; u < W; ++u) {
            const bool in = (W == 1) || q0 + u < w;  // (w is a multiple of W unless W > w)
            a[u] = in ? val_s[(q0 + u) * R + i] : 0.0;
            e[u] = in ? idx_s[(q0 + u) * R + i] : (uint32_t)i;
          }
          double g[W][C];
#pragma unroll
          for (int u = 0; u < W; ++u)
#pragma unroll
            for (int j = 0; j < C; ++j) g[u][j] = bc[j * LD + e[u]];
#pragma unroll
          for (int u = 0; u < W; ++u)
#pragma unroll
            for (int j = 0; j < C; ++j) acc[j] = fma(a[u], g[u][j], acc[j]);
        }
#pragma unroll
        for (int j = 0; j < C; ++j) {
          const double t = alpha * acc[j] - beta * bc[j * LD + i];
          const double vn = p.taylor ? t * p.rk[kd] : (kd == 1 ? t : 2.0 * t - bp[j * LD + i]);
          bp[j * LD + i] = vn;
          y_s[j * R + i] = fma(ck, vn, y_s[j * R + i]);
        }
      }
      __syncthreads();
      push_rows(bp, cur ^ 1);
      cluster_sync_all();
    }
  }
  for (int e = tid; e < C * R; e += CHEB_THREADS) {
    const int j = e / R, i = e - j * R;
    const int64_t gi = row0 + i;
    if (j < ncol && gi < p.n) p.out[(col0 + j) * p.ldo + gi] = p.out_scale * y_s[e];
  }
}

// Register-resident variant (R <= 2 * CHEB_REG_THREADS, w <= W): every thread owns the rows
// tid and tid + blockDim.x; their v_{k-1}, v_{k-2} and y stay in registers, so per degree and
// column the shared-memory traffic is the w gathers plus one store of v_k (the halo copy of the
// other CTAs and the gathers need it there).
constexpr int CHEB_REG_THREADS = 640;
template <int C, int W>
__global__ void __cluster_dims__(CHEB_CLUSTER, 1, 1) __launch_bounds__(CHEB_REG_THREADS, 1)
    cheb_reg_kernel(const __grid_constant__ ChebParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = p.R, w = p.w, LD = p.R + p.H, P = p.P;
  double* val_s = reinterpret_cast<double*>(smem);
  double* buf0 = val_s + (size_t)w * R;
  double* buf1 = buf0 + (size_t)C * LD;
  uint32_t* idx_s = reinterpret_cast<uint32_t*>(buf1 + (size_t)C * LD);
  uint32_t* rptr_s = idx_s + (size_t)w * R;   // [R + 1]
  uint32_t* rent_s = rptr_s + (R + 1);        // [P]
  __shared__ uint32_t rbase[2][CHEB_CLUSTER];

  const uint32_t me = cluster_rank();
  const int col0 = (blockIdx.x / CHEB_CLUSTER) * C;
  const int ncol = min(C, p.k - col0);
  const int64_t row0 = (int64_t)me * R;
  const int tid = threadIdx.x, T = blockDim.x;
  const int Pm = max(P, 1);
  if (tid < CHEB_CLUSTER) {
    rbase[0][tid] = mapa_u32(smem_u32(buf0), tid);
    rbase[1][tid] = mapa_u32(smem_u32(buf1), tid);
  }
  const int64_t ldm = (int64_t)CHEB_CLUSTER * R;
  for (int e = tid; e < w * R; e += T) {
    const int q = e / R, i = e - q * R;
    val_s[e] = p.val[q * ldm + row0 + i];
    idx_s[e] = p.idx[q * ldm + row0 + i];
  }
  for (int e = tid; e <= R; e += T) rptr_s[e] = p.rptr[(int64_t)me * (R + 1) + e];
  for (int e = tid; e < P; e += T) rent_s[e] = p.rent[(int64_t)me * Pm + e];
  const int i0 = tid, i1 = tid + T;
  const bool h0 = i0 < R, h1 = i1 < R;
  double vc[2][C], vp[2][C], y[2][C];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = u ? i1 : i0;
    const bool has = u ? h1 : h0;
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int64_t gi = row0 + i;
      const double x = (has && j < ncol && gi < p.n) ? p.X[(col0 + j) * p.ldx + gi] : 0.0;
      vc[u][j] = x;
      vp[u][j] = 0.0;
      y[u][j] = 0.0;
      if (has) buf0[j * LD + i] = x;
    }
  }
  __syncthreads();  // rptr / rent / rbase
  // the owner of row i stores its new values straight into the halo slots of the CTAs that read
  // it (fire-and-forget DSMEM stores, ordered by the cluster barrier's release)
  auto push_row = [&](int i, const double (&v)[C], int bi) {
    for (uint32_t e = rptr_s[i]; e < rptr_s[i + 1]; ++e) {
      const uint32_t d = rent_s[e];
      const uint32_t base = rbase[bi][d >> 24] + (d & 0xFFFFFFu) * 8u;
#pragma unroll
      for (int j = 0; j < C; ++j) st_dsmem_f64(base + (uint32_t)(j * LD) * 8u, v[j]);
    }
  };
  const double alpha = p.alpha, beta = p.beta;
  // C <= 3: the thread's matrix rows stay in registers for the whole polynomial (wider column
  // groups would spill); else they are re-read from shared memory every degree
  constexpr bool MREG = C <= 3;
  double a[2][W];
  uint32_t e[2][W];
  if (MREG)
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = u ? i1 : i0;
    const bool has = u ? h1 : h0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const bool in = has && q < w;
      a[u][q] = in ? val_s[q * R + i] : 0.0;
      e[u][q] = in ? idx_s[q * R + i] : 0u;
    }
  }
  cluster_sync_all();  // all CTAs of the cluster running before the first DSMEM push (racecheck)
  for (int sub = 0; sub < p.substeps; ++sub) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = u ? i1 : i0;
      if (!(u ? h1 : h0)) continue;
      if (sub > 0) {  // v_0 of the next substep = y
#pragma unroll
        for (int j = 0; j < C; ++j) {
          vc[u][j] = y[u][j];
          buf0[j * LD + i] = y[u][j];
        }
      }
      push_row(i, vc[u], 0);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int j = 0; j < C; ++j) y[u][j] = p.coef[0] * vc[u][j];
    cluster_sync_all();
    for (int kd = 1; kd <= p.K; ++kd) {
      const int cur = (kd - 1) & 1;
      const double* bc = cur ? buf1 : buf0;  // v_{k-1} with halo
      double* bn = cur ? buf0 : buf1;        // receives v_k
      const double ck = p.coef[kd];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = u ? i1 : i0;
        if (!(u ? h1 : h0)) continue;
        double am[W];
        uint32_t em[W];
#pragma unroll
        for (int q = 0; q < W; ++q) {
          if (MREG) {
            am[q] = a[u][q];
            em[q] = e[u][q];
          } else {
            const bool in = q < w;
            am[q] = in ? val_s[q * R + i] : 0.0;
            em[q] = in ? idx_s[q * R + i] : (uint32_t)i;
          }
        }
#pragma unroll
        for (int j = 0; j < C; ++j) {
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < W; ++q) acc = fma(am[q], bc[j * LD + em[q]], acc);
          const double t = alpha * acc - beta * vc[u][j];
          const double vn = p.taylor ? t * p.rk[kd] : (kd == 1 ? t : 2.0 * t - vp[u][j]);
          vp[u][j] = vc[u][j];
          vc[u][j] = vn;
          y[u][j] = fma(ck, vn, y[u][j]);
          bn[j * LD + i] = vn;
        }
        push_row(i, vc[u], cur ^ 1);
      }
      cluster_sync_all();
    }
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = u ? i1 : i0;
    const int64_t gi = row0 + i;
    if (!(u ? h1 : h0) || gi >= p.n) continue;
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (j < ncol) p.out[(col0 + j) * p.ldo + gi] = p.out_scale * y[u][j];
  }
}

template <int C, int W>
void launch_reg(const ChebParams& prm, int groups, size_t smem, int threads, cudaStream_t st) {
  auto kern = cheb_reg_kernel<C, W>;
  static std::mutex attr_mu;
  static uint64_t attr_mask = 0;
  per_device_once(attr_mu, attr_mask, [&] {
    DME_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
  });
  kern<<<groups * CHEB_CLUSTER, threads, smem, st>>>(prm);
  DME_KCHECK();
}
template <int W>
void launch_reg_w(const ChebParams& prm, int C, int groups, size_t smem, int threads, cudaStream_t st) {
  switch (C) {
    case 1: launch_reg<1, W>(prm, groups, smem, threads, st); break;
    case 2: launch_reg<2, W>(prm, groups, smem, threads, st); break;
    case 3: launch_reg<3, W>(prm, groups, smem, threads, st); break;
    case 4: launch_reg<4, W>(prm, groups, smem, threads, st); break;
    default: launch_reg<5, W>(prm, groups, smem, threads, st); break;
  }
}
constexpr int CHEB_REG_CMAX = 5;

template <int C, int W>
void launch_cw(const ChebParams& prm, int groups, size_t smem, cudaStream_t st) {
  auto kern = cheb_kernel<C, W>;
  static std::mutex attr_mu;
  static uint64_t attr_mask = 0;
  per_device_once(attr_mu, attr_mask, [&] {
    DME_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
  });
  kern<<<groups * CHEB_CLUSTER, CHEB_THREADS, smem, st>>>(prm);
  DME_KCHECK();
}
template <int C>
void launch_c(const ChebParams& prm, int groups, size_t smem, cudaStream_t st) {
  if (prm.w <= 3) launch_cw<C, 3>(prm, groups, smem, st);
  else if (prm.w <= 5) launch_cw<C, 5>(prm, groups, smem, st);
  else if (prm.w <= 8) launch_cw<C, 8>(prm, groups, smem, st);
  else launch_cw<C, 4>(prm, groups, smem, st);  // wide rows: batches of 4
}

// co-resident 8-CTA clusters of cheb_kernel<C, .> at this shared-memory size (cached per C)
int max_active_clusters(int C, size_t smem) {
  static int cache[CHEB_CMAX + 1][2] = {};
  if (cache[C][0] > 0 && cache[C][1] == (int)smem) return cache[C][0];
  auto kern = cheb_kernel<1, 5>;  // same launch shape for every instance (1 CTA per SM, 512 threads)
  DME_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CHEB_CLUSTER * 64);
  cfg.blockDim = dim3(CHEB_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CHEB_CLUSTER;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  DME_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
  cache[C][0] = std::max(1, n);
  cache[C][1] = (int)smem;
  return cache[C][0];
}

}  // namespace

namespace {
// one warp per row of the row-major A: nonzero count, then the entries in column order
__global__ void csr_count_kernel(const double* A, int64_t n, int64_t ld, int64_t* cnt) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  int64_t c = 0;
  for (int64_t j = lane; j < n; j += 32) c += A[row * ld + j] != 0.0;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[row] = c;
}
__global__ void csr_fill_kernel(const double* A, int64_t n, int64_t ld, const int64_t* rowptr,
                                int32_t* col, double* val) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  int64_t pos = rowptr[row];
  for (int64_t j0 = 0; j0 < n; j0 += 32) {
    const int64_t j = j0 + lane;
    const double a = j < n ? A[row * ld + j] : 0.0;
    const unsigned m = __ballot_sync(0xffffffffu, a != 0.0);
    if (a != 0.0) {
      const int64_t d = pos + __popc(m & ((1u << lane) - 1u));
      col[d] = (int32_t)j;
      val[d] = a;
    }
    pos += __popc(m);
  }
}
}  // namespace

int cheb_csr_from_dense(const double* A, int64_t n, int64_t ld, int64_t max_nnz, void* scratch,
                        cudaStream_t st, std::vector<int64_t>& rowptr, std::vector<int32_t>& col,
                        std::vector<double>& val) {
  int64_t* cnt = reinterpret_cast<int64_t*>(scratch);
  const unsigned blocks = (unsigned)ceil_div(n, 8);
  csr_count_kernel<<<blocks, 256, 0, st>>>(A, n, ld, cnt);
  DME_KCHECK();
  std::vector<int64_t> c(n);
  DME_CUDA(cudaMemcpyAsync(c.data(), cnt, n * 8, cudaMemcpyDeviceToHost, st));
  DME_CUDA(cudaStreamSynchronize(st));
  rowptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) rowptr[i + 1] = rowptr[i] + c[i];
  const int64_t nnz = rowptr[n];
  if (nnz > max_nnz) return 0;
  int64_t* rp = cnt;  // rowptr on the device (over the counts), then col / val behind it
  int32_t* cd = reinterpret_cast<int32_t*>(rp + n + 1);
  double* vd = reinterpret_cast<double*>(cd + ((nnz + 1) & ~int64_t(1)));
  DME_CUDA(cudaMemcpyAsync(rp, rowptr.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
  csr_fill_kernel<<<blocks, 256, 0, st>>>(A, n, ld, rp, cd, vd);
  DME_KCHECK();
  col.resize(nnz);
  val.resize(nnz);
  DME_CUDA(cudaMemcpyAsync(col.data(), cd, nnz * 4, cudaMemcpyDeviceToHost, st));
  DME_CUDA(cudaMemcpyAsync(val.data(), vd, nnz * 8, cudaMemcpyDeviceToHost, st));
  DME_CUDA(cudaStreamSynchronize(st));
  return 1;
}

size_t cheb_smem_bytes_reg(int64_t R, int w, int H, int P, int C) {
  return (size_t)R * w * 12 + (size_t)(R + H) * C * 16 + (size_t)(R + 1 + P) * 4 + 64;
}
size_t cheb_smem_bytes(int64_t R, int w, int H, int P, int C) {
  return (size_t)R * w * 12 + (size_t)(R + H) * C * 16 + (size_t)R * C * 8 + (size_t)P * 8 + 64;
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
                 const double* values, ChebHost& out, std::string* err, bool force_global) {
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
  double a = INFINITY, b = -INFINITY, norm1 = 0.0, trace = 0.0;
  out.sym = true;
  for (int64_t i = 0; i < n; ++i) {
    canon(tp.data(), tc.data(), tv.data(), i, rowsT[i]);
    canon(rowptr, colind, values, i, ra);
    bool same = ra.size() == rowsT[i].size();
    for (size_t e = 0; same && e < ra.size(); ++e)
      same = ra[e].first == rowsT[i][e].first && ra[e].second == rowsT[i][e].second;
    if (!same) out.sym = false;
    for (auto& x : ra)
      if (x.first == i) trace += x.second;
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
  if (R + (int64_t)n >= (1 << 24)) return fail(DME_ERR_DIM, "sparse A: too many rows per CTA");
  // halo of CTA r: the rows of other CTAs its rows read (sorted), slot s at local index R + s;
  // push list of CTA o: (own row, (reader << 24) | reader's local index) for every such row
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> pushes(CHEB_CLUSTER);
  std::vector<std::vector<int32_t>> halo(CHEB_CLUSTER);
  int H = 0;
  for (int r = 0; r < CHEB_CLUSTER; ++r) {
    std::vector<int32_t>& hl = halo[r];
    for (int64_t i = r * R; i < std::min<int64_t>(n, (r + 1) * R); ++i)
      for (auto& x : rowsT[i])
        if (x.first / R != r) hl.push_back(x.first);
    std::sort(hl.begin(), hl.end());
    hl.erase(std::unique(hl.begin(), hl.end()), hl.end());
    H = std::max<int>(H, (int)hl.size());
    for (size_t s = 0; s < hl.size(); ++s)
      pushes[hl[s] / R].push_back({(uint32_t)(hl[s] % R), (uint32_t)(r << 24) | (uint32_t)(R + s)});
  }
  int P = 0;
  for (auto& pl : pushes) P = std::max<int>(P, (int)pl.size());
  int C = 0;
  for (int c = CHEB_CMAX; c >= 1; --c)
    if (cheb_smem_bytes(R, w, H, P, c) <= 225 * 1024) { C = c; break; }
  out.global = force_global || C == 0 || std::getenv("DME_CHEB_GLOBAL") != nullptr;
  if (out.global) {  // rows beyond one cluster's shared memory: the grid-wide kernel
    C = CHEB_CMAX;
    H = P = 0;
    for (auto& pl : pushes) pl.clear();
  }
  out.nnz = 0;
  for (auto& r : rowsT) out.nnz += (int64_t)r.size();
  out.n = n; out.R = R; out.w = w; out.H = H; out.P = P; out.C = C;
  out.a = a; out.b = b; out.norm1 = norm1;
  // shifted norms for the Taylor route: max(||A^T - mu I||_1, ||A^T - mu I||_inf), mu = trace / n
  out.mu = trace / n;
  {
    double rmax = 0.0;  // rows of A^T
    std::vector<double> csum(n, 0.0);  // columns of A^T = rows of A
    for (int64_t i = 0; i < n; ++i) {
      double rs = 0.0;
      bool dg = false;
      for (auto& x : rowsT[i]) {
        const double v = x.second - (x.first == i ? out.mu : 0.0);
        dg = dg || x.first == i;
        rs += std::fabs(v);
        csum[x.first] += std::fabs(v);
      }
      if (!dg) { rs += std::fabs(out.mu); csum[i] += std::fabs(out.mu); }
      rmax = std::max(rmax, rs);
    }
    double cmax = 0.0;
    for (double v : csum) cmax = std::max(cmax, v);
    out.tnorm = std::max(rmax, cmax);
  }
  const int64_t ldm = (int64_t)CHEB_CLUSTER * R;
  out.val.assign((size_t)w * ldm, 0.0);
  out.idx.assign((size_t)w * ldm, 0u);
  if (out.global) {  // ELL with global column indices (padding: 0 x own row)
    for (int64_t i = 0; i < ldm; ++i) {
      for (int q = 0; q < w; ++q) out.idx[q * ldm + i] = (uint32_t)std::min<int64_t>(i, n - 1);
      if (i >= n) continue;
      int q = 0;
      for (auto& x : rowsT[i]) {
        out.val[q * ldm + i] = x.second;
        out.idx[q * ldm + i] = (uint32_t)x.first;
        ++q;
      }
    }
    out.push.clear();
    out.rptr.assign(1, 0u);
    out.rent.clear();
    return 0;
  }
  for (int64_t i = 0; i < ldm; ++i) {
    const int r = (int)(i / R);
    for (int q = 0; q < w; ++q) out.idx[q * ldm + i] = (uint32_t)(i % R);  // padding: 0 x own row
    if (i >= n) continue;
    int q = 0;
    for (auto& x : rowsT[i]) {
      uint32_t li;
      if (x.first / R == r) {
        li = (uint32_t)(x.first % R);
      } else {
        const auto& hl = halo[r];
        li = (uint32_t)(R + (std::lower_bound(hl.begin(), hl.end(), x.first) - hl.begin()));
      }
      out.val[q * ldm + i] = x.second;
      out.idx[q * ldm + i] = li;
      ++q;
    }
  }
  out.rptr.assign((size_t)CHEB_CLUSTER * (R + 1), 0u);
  out.rent.assign((size_t)CHEB_CLUSTER * std::max(P, 1), 0u);
  for (int o = 0; o < CHEB_CLUSTER; ++o) {
    std::vector<std::pair<uint32_t, uint32_t>> pl = pushes[o];
    std::stable_sort(pl.begin(), pl.end(), [](auto& x, auto& y) { return x.first < y.first; });
    uint32_t* rp = out.rptr.data() + (size_t)o * (R + 1);
    for (auto& x : pl) rp[x.first + 1]++;
    for (int64_t i = 0; i < R; ++i) rp[i + 1] += rp[i];
    for (size_t e = 0; e < pl.size(); ++e) out.rent[(size_t)o * std::max(P, 1) + e] = pl[e].second;
  }
  out.push.assign((size_t)CHEB_CLUSTER * P * 2, 0xFFFFFFFFu);
  for (int o = 0; o < CHEB_CLUSTER; ++o)
    for (size_t e = 0; e < pushes[o].size(); ++e) {
      out.push[((size_t)o * P + e) * 2] = pushes[o][e].first;
      out.push[((size_t)o * P + e) * 2 + 1] = pushes[o][e].second;
    }
  return 0;
}

namespace {
// First use in a process: set the shared-memory attribute of every kernel instance (which also
// loads it under lazy module loading), so no later call pays a module load inside a timed init.
template <int C>
void preload_c() {
  for (auto f : {cheb_kernel<C, 3>, cheb_kernel<C, 5>, cheb_kernel<C, 8>, cheb_kernel<C, 4>})
    DME_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
  if constexpr (C <= CHEB_REG_CMAX)
    for (auto f : {cheb_reg_kernel<C, 3>, cheb_reg_kernel<C, 5>})
      DME_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
}
void preload_all() {
  static std::mutex mu;
  static uint64_t mask = 0;
  per_device_once(mu, mask, [] {
    preload_c<1>(); preload_c<2>(); preload_c<3>(); preload_c<4>();
    preload_c<5>(); preload_c<6>(); preload_c<7>(); preload_c<8>();
  });
}

// ---------------------------------------------------------------- global mode (large n)
// The same recurrences (Chebyshev, or Taylor for a nonsymmetric A) over all rows with one
// cooperative grid: thread (row i, column j) pairs strided over the grid, v_{k-1} gathered from
// global memory (L2-resident: n x k doubles), v_k written over v_{k-2}, y in global memory; one
// grid barrier per degree. Used when n x (ELL width + halo) exceeds one cluster's shared memory.
struct GParams {
  const double* val;
  const uint32_t* idx;
  int64_t ldm;
  const double* X;
  double* out;
  double *v0, *v1, *y;
  int64_t ldx, ldo, ldv, n;
  int w, k, K, substeps, taylor;
  double alpha, beta, out_scale;
  double coef[CHEB_KMAX + 1];
  double rk[TAYLOR_MMAX + 1];
};

constexpr int GTHREADS = 512;

__global__ void __launch_bounds__(GTHREADS) cheb_global_kernel(GParams p) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int64_t n = p.n, ldv = p.ldv;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int j = 0; j < p.k; ++j)
    for (int64_t i = t0; i < n; i += stride) {
      const double x = p.X[i + j * p.ldx];
      p.v0[i + j * ldv] = x;
      p.y[i + j * ldv] = p.coef[0] * x;
    }
  grid.sync();
  double* cur = p.v0;
  double* prv = p.v1;
  for (int sub = 0; sub < p.substeps; ++sub) {
    if (sub > 0) {  // v_0 of the next substep = y
      for (int j = 0; j < p.k; ++j)
        for (int64_t i = t0; i < n; i += stride) {
          const double v = p.y[i + j * ldv];
          cur[i + j * ldv] = v;
          p.y[i + j * ldv] = p.coef[0] * v;
        }
      grid.sync();
    }
    const int nn = (int)n, total4 = (int)n * ((p.k + 3) / 4);  // (n k <= 2^31: checked on the host)
    for (int kd = 1; kd <= p.K; ++kd) {
      const double ck = p.coef[kd], rk = p.rk[kd < TAYLOR_MMAX ? kd : TAYLOR_MMAX];
      // (row, 4-column block) pairs flattened over the whole grid: consecutive threads take
      // consecutive rows (coalesced); a thread loads its row's ELL entries once for 4 columns
      // and issues their gathers together (the loop is bound by L2 traffic and latency)
      const double* __restrict__ cr_ = cur;
      double* __restrict__ pr_ = prv;
      double* __restrict__ yr_ = p.y;
      for (int e = (int)t0; e < total4; e += (int)stride) {
        const int jb = e / nn, i = e - jb * nn;
        const int j0 = 4 * jb;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int q = 0; q < p.w; ++q) {
          const double a = p.val[q * p.ldm + i];
          const int64_t col = p.idx[q * p.ldm + i];
          double g[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) g[u] = j0 + u < p.k ? __ldcg(cr_ + col + (int64_t)(j0 + u) * ldv) : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[u] = fma(a, g[u], acc[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (j0 + u >= p.k) break;
          const int64_t o = i + (int64_t)(j0 + u) * ldv;
          const double t = p.alpha * acc[u] - p.beta * cr_[o];
          const double vn = p.taylor ? t * rk : (kd == 1 ? t : 2.0 * t - pr_[o]);
          pr_[o] = vn;
          yr_[o] = fma(ck, vn, yr_[o]);
        }
      }
      grid.sync();
      double* tmp = cur;
      cur = prv;
      prv = tmp;
    }
  }
  for (int j = 0; j < p.k; ++j)
    for (int64_t i = t0; i < n; i += stride) p.out[i + j * p.ldo] = p.out_scale * p.y[i + j * ldv];
}

int cheb_action_global(const ChebOp& op, const ChebParams& prm, cudaStream_t st) {
  GParams* g = new GParams;  // (large: built on the heap, passed by value to the launch)
  std::unique_ptr<GParams> own(g);
  std::memset(g, 0, sizeof(GParams));
  g->val = op.val; g->idx = op.idx; g->ldm = (int64_t)CHEB_CLUSTER * op.R;
  g->X = prm.X; g->out = prm.out; g->v0 = op.gv0; g->v1 = op.gv1; g->y = op.gy;
  g->ldx = prm.ldx; g->ldo = prm.ldo; g->ldv = (int64_t)CHEB_CLUSTER * op.R; g->n = op.n;
  g->w = op.w; g->k = prm.k; g->K = prm.K; g->substeps = prm.substeps; g->taylor = prm.taylor;
  g->alpha = prm.alpha; g->beta = prm.beta; g->out_scale = prm.out_scale;
  std::memcpy(g->coef, prm.coef, sizeof(g->coef));
  std::memcpy(g->rk, prm.rk, sizeof(g->rk));
  static std::mutex mu;
  static uint64_t mask = 0;
  static int per_sm = 1;
  per_device_once(mu, mask, [&] {
    DME_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cheb_global_kernel, GTHREADS, 0));
  });
  int dev = 0, sms = 148;
  DME_CUDA(cudaGetDevice(&dev));
  DME_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // few CTAs per SM: each grid barrier costs more with more CTAs
  int bps = 2;  // (measured at n = 1e4 and 3.6e4: 2 CTAs per SM beat 1 and 4)
  if (const char* e = std::getenv("DME_CHEB_GLOBAL_BPS")) bps = std::atoi(e);
  const int grid_n = std::max(1, std::min(std::max(per_sm, 1), std::max(bps, 1)) * sms);
  void* args[] = {g};
  DME_CUDA(cudaLaunchCooperativeKernel((void*)cheb_global_kernel, dim3(grid_n), dim3(GTHREADS), args, 0, st));
  DME_KCHECK();
  return prm.K * prm.substeps;
}

}  // namespace

int cheb_action(const ChebOp& op, double tau, const double* X, int64_t ldx, int64_t k, double* out,
                int64_t ldo, double alpha, cudaStream_t st) {
  if (k <= 0) return 0;
  preload_all();
  ChebParams prm;
  std::memset(&prm, 0, sizeof(prm));
  int substeps = 1, K = 0;
  double c = 0, gamma = 0;
  if (op.sym) {
    // interval of tau A^T (tau > 0): [tau a, tau b]; substeps keep the degree within CHEB_KMAX
    std::vector<double> chat;
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
  } else {
    // truncated Taylor with scaling (Al-Mohy & Higham 2011): the cheapest m s with
    // s >= tau ||A^T - mu I|| / theta_m
    const double tn = tau * op.tnorm;
    int64_t best = INT64_MAX;
    for (int q = 0; q < TAYLOR_NM; ++q) {
      const int m = TAYLOR_M[q];
      const int64_t s = std::max<int64_t>(1, (int64_t)std::ceil(tn / TAYLOR_THETA[q]));
      if ((int64_t)m * s < best) { best = (int64_t)m * s; K = m; substeps = (int)s; }
    }
    const double ts = tau / substeps, eta = std::exp(ts * op.mu);
    for (int j = 0; j <= K; ++j) {
      prm.coef[j] = eta;
      prm.rk[j] = j ? 1.0 / j : 1.0;
    }
    prm.taylor = 1;
    prm.alpha = ts;
    prm.beta = ts * op.mu;
  }
  prm.val = op.val; prm.idx = op.idx; prm.push = op.push; prm.rptr = op.rptr; prm.rent = op.rent;
  prm.X = X; prm.out = out;
  prm.ldx = ldx; prm.ldo = ldo; prm.n = op.n;
  prm.R = (int)op.R; prm.w = op.w; prm.H = op.H; prm.P = op.P;
  prm.k = (int)k; prm.K = K; prm.substeps = substeps;
  if (op.sym) {
    prm.alpha = gamma > 0 ? (tau / substeps) / gamma : 0.0;
    prm.beta = gamma > 0 ? c / gamma : 0.0;
  }
  prm.out_scale = alpha;
  if (op.global) {
    if (k > SMALL_K_MAX || (int64_t)op.n * k >= ((int64_t)1 << 31))
      throw std::runtime_error("cheb_action (global): too many columns");
    return cheb_action_global(op, prm, st);
  }
  // columns per cluster: the smallest C whose ceil(k / C) clusters are co-resident in one wave
  // (cudaOccupancyMaxActiveClusters: clusters are placed within a GPC, 15 x 8 CTAs on a B200 at
  // this shared-memory size), less one cluster's SMs for the eigen kernels that run concurrently
  // on the critical stream (a second wave doubles the time per degree)
  int C = op.C;
  for (int c = 1; c <= op.C; ++c)
    if (ceil_div(k, c) <= std::max(1, max_active_clusters(c, cheb_smem_bytes(op.R, op.w, op.H, op.P, c)) - 1)) {
      C = c;
      break;
    }
  const int groups = (int)ceil_div(k, C);
  const bool reg = op.R <= 2 * CHEB_REG_THREADS && op.w <= 5 && C <= CHEB_REG_CMAX &&
                   !getenv("DME_CHEB_NOREG");
  if (reg) {
    const size_t sm = cheb_smem_bytes_reg(op.R, op.w, op.H, op.P, C);
    const int threads = (int)std::min<int64_t>(CHEB_REG_THREADS, ceil_div(ceil_div(op.R, 2), 32) * 32);
    if (op.w <= 3) launch_reg_w<3>(prm, C, groups, sm, threads, st);
    else launch_reg_w<5>(prm, C, groups, sm, threads, st);
    return K * substeps;
  }
  const size_t smem = cheb_smem_bytes(op.R, op.w, op.H, op.P, C);
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
