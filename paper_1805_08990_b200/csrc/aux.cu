// Element-wise / reduction / tall-times-small kernels of the DME path.
#include "aux.h"

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include "common.cuh"
#include <cooperative_groups.h>
#include "gemm_nt.h"

namespace dme {

namespace {

// out = alpha * A^T  (n x n, row-major with leading dims lda / ldo), 32x32 smem tiles
__global__ void transpose_scale_kernel(const double* __restrict__ A, int64_t n, int64_t lda,
                                       double alpha, double* __restrict__ out, int64_t ldo) {
  __shared__ double tile[32][33];
  const int64_t bx = (int64_t)blockIdx.x * 32, by = (int64_t)blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int64_t r = by + j, c = bx + threadIdx.x;
    if (r < n && c < n) tile[j][threadIdx.x] = A[r * lda + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int64_t r = bx + j, c = by + threadIdx.x;
    if (r < n && c < n) out[r * ldo + c] = alpha * tile[threadIdx.x][j];
  }
}

// partial[b] = max over the rows handled by block b of sum_j |A_ij|
__global__ void rowabs_max_kernel(const double* __restrict__ A, int64_t n, int64_t lda,
                                  double* __restrict__ partial) {
  __shared__ double red[32];
  double best = 0.0;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    double s = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) s += fabs(A[i * lda + j]);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      best = fmax(best, t);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = best;
}

__global__ void max_reduce_kernel(const double* __restrict__ partial, int cnt, double* out) {
  double v = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) v = fmax(v, partial[i]);
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    *out = t;
  }
}

__global__ void lincomb_kernel(double* __restrict__ out, int64_t n, int64_t ld, LinTerm t0,
                               LinTerm t1, LinTerm t2, LinTerm t3, double diag) {
  const int64_t total = n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    const int64_t o = i * ld + j;
    double v = (i == j) ? diag : 0.0;
    if (t0.X) v += t0.c * t0.X[o];
    if (t1.X) v += t1.c * t1.X[o];
    if (t2.X) v += t2.c * t2.X[o];
    if (t3.X) v += t3.c * t3.X[o];
    out[o] = v;
  }
}

__global__ void copy_cols_kernel(double* __restrict__ dst, int64_t ldd, const double* __restrict__ src,
                                 int64_t lds, int64_t rows, int64_t cols, double alpha) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    dst[i + j * ldd] = alpha * src[i + j * lds];
  }
}

// dst (rows x cols, col-major ldd) = alpha * src^T  where src is cols x rows row-major (lds)
__global__ void rowmajor_to_colmajor_kernel(double* __restrict__ dst, int64_t ldd,
                                            const double* __restrict__ src, int64_t lds,
                                            int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    dst[i + j * ldd] = src[i * lds + j];
  }
}

// C (M x N, col-major ldc) = A (M x K, col-major lda) * B (K x N, col-major ldb); K, N small.
// One CTA owns a 128-row block and all N columns (N <= 64 per launch slice), so C may alias A
// when N <= the columns read (row-local: the whole K loop completes before the epilogue).
constexpr int TS_BM = 128, TS_BN = 64, TS_BK = 16;
__global__ void __launch_bounds__(256) tall_small_kernel(const double* A, int64_t lda,
                                                         const double* __restrict__ B, int64_t ldb,
                                                         double* C, int64_t ldc, int64_t M,
                                                         int64_t N, int64_t K) {
  pdl_wait();
  __shared__ double sA[TS_BK][TS_BM + 4];
  __shared__ double sB[TS_BN][TS_BK + 4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % 4, wn = warp / 4;  // warp tile 32 x 32
  const int64_t m0 = (int64_t)blockIdx.x * TS_BM;
  const int64_t n0 = (int64_t)blockIdx.y * TS_BN;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int64_t k0 = 0; k0 < K; k0 += TS_BK) {
    for (int e = tid; e < TS_BK * TS_BM; e += 256) {
      const int kk = e / TS_BM, mm = e % TS_BM;
      const int64_t gm = m0 + mm, gk = k0 + kk;
      sA[kk][mm] = (gm < M && gk < K) ? A[gm + gk * lda] : 0.0;
    }
    for (int e = tid; e < TS_BN * TS_BK; e += 256) {
      const int nn = e / TS_BK, kk = e % TS_BK;
      const int64_t gn = n0 + nn, gk = k0 + kk;
      sB[nn][kk] = (gn < N && gk < K) ? B[gk + gn * ldb] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < TS_BK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = sA[ks + t][wm * 32 + a * 8 + g];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = sB[wn * 32 + b * 8 + g][ks + t];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t row = m0 + wm * 32 + a * 8 + g;
        const int64_t col = n0 + wn * 32 + b * 8 + t * 2 + e;
        if (row < M && col < N) C[row + col * ldc] = acc[a][b][e];
      }
}

// lower triangle <- transpose of the upper triangle (average: symmetric part everywhere)
__global__ void mirror_kernel(double* X, int64_t n, int64_t ld, int average) {
  __shared__ double up[32][33];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;  // destination block (bi, bj), bi >= bj
  if (bi < bj) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  // source block (bj, bi) of the upper triangle, transposed through shared memory
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = bj * 32 + y, c = bi * 32 + tx;
    up[y][tx] = (r < n && c < n) ? X[r * ld + c] : 0.0;
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = bi * 32 + y, c = bj * 32 + tx;  // element (r, c), r > c wanted
    if (r < n && c < n && r > c) {
      const double t = up[tx][y];  // X[c][r]
      if (average) {
        const double v = 0.5 * (X[r * ld + c] + t);
        X[r * ld + c] = v;
      } else {
        X[r * ld + c] = t;
      }
    }
  }
}

__global__ void mirror_upper_from_lower(double* X, int64_t n, int64_t ld) {
  // after averaging the lower triangle, copy it back to the upper one
  const int64_t total = n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    if (i < j) X[i * ld + j] = X[j * ld + i];
  }
}

// flags[0] |= any non-finite entry; flags[1] |= any X[i][j] != X[j][i] (bitwise, i < j)
__global__ void check_square_kernel(const double* __restrict__ X, int64_t n, int64_t ld, int* flags) {
  __shared__ double up[32][33];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;
  const int tx = threadIdx.x, ty = threadIdx.y;
  int bad = 0, asym = 0;
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = bi * 32 + y, c = bj * 32 + tx;
    if (r < n && c < n) {
      const double v = X[r * ld + c];
      bad |= !isfinite(v);
    }
    // transposed block for the symmetry test
    const int64_t r2 = bj * 32 + y, c2 = bi * 32 + tx;
    up[y][tx] = (r2 < n && c2 < n) ? X[r2 * ld + c2] : 0.0;
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = bi * 32 + y, c = bj * 32 + tx;
    if (r < n && c < n && r > c) {
      const double v = X[r * ld + c], t = up[tx][y];
      asym |= (__double_as_longlong(v) != __double_as_longlong(t));
    }
  }
  bad = __syncthreads_or(bad);
  asym = __syncthreads_or(asym);
  if (tx == 0 && ty == 0) {
    if (bad) atomicOr(flags, 1);
    if (asym) atomicOr(flags + 1, 1);
  }
}

__global__ void zero_ints(int* p, int cnt) {
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) p[i] = 0;
}

inline int grid_for(int64_t total, int threads = 256) {
  int64_t b = (total + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}


// ---------------------------------------------------------------- projected Gram (refined compression)
// G = (Z U)^T (Z U) without materialising W = Z U (n x s). One cooperative wave: every CTA takes one
// block of rb rows of Z (rb = n / #SMs rounded up to 8), forms its W rows in shared memory (DMMA,
// K = k) and accumulates the upper tiles of W^T W (DMMA, K = rb) in registers; after a grid barrier
// each warp sums the per-CTA partials of some elements in a fixed order (lane-strided, then a fixed
// butterfly: deterministic). Operands are staged with cp.async (8-byte, zero-filled outside Z / U),
// all in flight at once. Phase-1 work units are (n-tile, m-group) pairs, NT * MG = 16 * UPW of
// them: every warp owns UPW units and the m-tiles mt = mg (mod MG) of each (one B fragment per unit
// and k-step, one A fragment per m-tile).
constexpr int PG_KMAX = 160;   // k bound (the refined compression runs for k <= FAST_K_MAX = 160)
constexpr int PG_RMAX = 128;   // rows per block
constexpr int PG_WARPS = 16;
constexpr size_t PG_SMEM = 220 * 1024;

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(ok ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__host__ __device__ constexpr int pg_kpad(int k) { return (k + 15) & ~15; }
__host__ __device__ constexpr int pg_ldz(int rb) { return ((rb + 15) & ~15) + 8; }
template <int NT>
struct PgShape {
  static constexpr int SP = NT * 8, LDW = SP + 8;
  static constexpr int MG = NT == 8 ? 2 : 4;                  // NT * MG = 16 * UPW units
  static constexpr int UPW = NT * MG / PG_WARPS;              // units per warp
  static constexpr int MTG = (PG_RMAX / 8 + MG - 1) / MG;     // m-tiles per unit (max)
  static constexpr int T = NT * (NT + 1) / 2, Q = (T + PG_WARPS - 1) / PG_WARPS;  // phase-2 tiles
};

template <int NT>
__global__ void __launch_bounds__(PG_WARPS * 32, 1)
    proj_gram_kernel(const double* __restrict__ Z, int64_t ldz, int64_t n, int k,
                     const double* __restrict__ U, int64_t ldu, int s, int rb, double* part,
                     double* G, int64_t ldg) {
  using S = PgShape<NT>;
  constexpr int SP = S::SP, LDW = S::LDW, MG = S::MG, UPW = S::UPW, MTG = S::MTG, T = S::T,
                Q = S::Q;
  extern __shared__ __align__(16) double pg_sm[];
  const int kp = pg_kpad(k), ldu_s = kp + 4, k4 = (k + 3) & ~3, ldz_s = pg_ldz(rb);
  const int mt_n = rb >> 3;
  double* sU = pg_sm;             // [SP][ldu_s]: sU[j][kk] = U[kk, j]
  double* sZ = sU + SP * ldu_s;   // [kp][ldz_s]: sZ[kk][m] = Z[m0 + m, kk]; reused as sW
  double* sW = sZ;                // [rb][LDW]:   sW[m][j] = W[m0 + m, j]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  for (int j = warp; j < SP; j += PG_WARPS)
    for (int kk = lane; kk < kp; kk += 32) {
      const bool ok = j < s && kk < k;
      cp_async8(sU + j * ldu_s + kk, ok ? U + kk + (int64_t)j * ldu : U, ok);
    }
  int tI[Q], tJ[Q];
  double gacc[Q][2];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    int rem = warp + PG_WARPS * q, jt = 0;
    while (rem > jt) rem -= ++jt;
    tI[q] = rem;
    tJ[q] = jt;
    gacc[q][0] = gacc[q][1] = 0.0;
  }
  for (int64_t m0 = (int64_t)blockIdx.x * rb; m0 < n; m0 += (int64_t)gridDim.x * rb) {
    for (int kk = warp; kk < kp; kk += PG_WARPS)
      for (int m = lane; m < rb; m += 32) {
        const bool ok = kk < k && m0 + m < n;
        cp_async8(sZ + kk * ldz_s + m, ok ? Z + (m0 + m) + (int64_t)kk * ldz : Z, ok);
      }
    cp_async_wait_all();
    __syncthreads();
    double w[UPW][MTG][2];
#pragma unroll
    for (int u = 0; u < UPW; ++u)
#pragma unroll
      for (int i = 0; i < MTG; ++i) w[u][i][0] = w[u][i][1] = 0.0;
    for (int ks = 0; ks < k4; ks += 4) {
      const double* zrow = sZ + (ks + t) * ldz_s + g;
#pragma unroll
      for (int u = 0; u < UPW; ++u) {
        const int unit = warp + PG_WARPS * u, nt = unit % NT, mg = unit / NT;
        const double b = sU[(nt * 8 + g) * ldu_s + ks + t];
#pragma unroll
        for (int i = 0; i < MTG; ++i) {
          const int mt = mg + MG * i;
          if (mt < mt_n) dmma_8x8x4(w[u][i][0], w[u][i][1], zrow[mt * 8], b);
        }
      }
    }
    __syncthreads();  // every read of sZ precedes the sW stores
#pragma unroll
    for (int u = 0; u < UPW; ++u) {
      const int unit = warp + PG_WARPS * u, nt = unit % NT, mg = unit / NT;
#pragma unroll
      for (int i = 0; i < MTG; ++i) {
        const int mt = mg + MG * i;
        if (mt < mt_n) {
          double* d = sW + (mt * 8 + g) * LDW + nt * 8 + 2 * t;
          d[0] = w[u][i][0];
          d[1] = w[u][i][1];
        }
      }
    }
    __syncthreads();
    // upper tiles (it <= jt) of W^T W over the block's rb rows (rows past n are zero)
    for (int ks = 0; ks < rb; ks += 4) {
      const double* wrow = sW + (ks + t) * LDW + g;
#pragma unroll
      for (int q = 0; q < Q; ++q)
        if (warp + PG_WARPS * q < T)
          dmma_8x8x4(gacc[q][0], gacc[q][1], wrow[tI[q] * 8], wrow[tJ[q] * 8]);
    }
    __syncthreads();  // sW is overwritten by the next block's Z
  }
  // partial of this CTA: element (i, j) at part[(i + j * SP) * gridDim.x + blockIdx.x]
  const int P = gridDim.x;
#pragma unroll
  for (int q = 0; q < Q; ++q)
    if (warp + PG_WARPS * q < T) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = tI[q] * 8 + g, j = tJ[q] * 8 + 2 * t + e;
        part[(size_t)(i + j * SP) * P + blockIdx.x] = gacc[q][e];
      }
    }
  cooperative_groups::this_grid().sync();
  // G[i, j] = G[j, i] = sum over CTAs, i <= j < s: one warp per element
  const int64_t ne = (int64_t)s * (s + 1) / 2;
  for (int64_t e = (int64_t)blockIdx.x * PG_WARPS + warp; e < ne; e += (int64_t)P * PG_WARPS) {
    int j = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
    while ((int64_t)(j + 1) * (j + 2) / 2 <= e) ++j;
    while ((int64_t)j * (j + 1) / 2 > e) --j;
    const int i = (int)(e - (int64_t)j * (j + 1) / 2);
    const double* src = part + (size_t)(i + j * SP) * P;
    double acc = 0.0;
    for (int p = lane; p < P; p += 32) acc += __ldcg(src + p);
#pragma unroll
    for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) {
      G[i + (int64_t)j * ldg] = acc;
      G[j + (int64_t)i * ldg] = acc;
    }
  }
}

template <int NT>
size_t proj_gram_smem(int k, int rb) {
  const int kp = pg_kpad(k);
  return sizeof(double) * ((size_t)NT * 8 * (kp + 4) +
                           std::max<size_t>((size_t)kp * pg_ldz(rb), (size_t)rb * PgShape<NT>::LDW));
}

template <int NT>
bool proj_gram_launch(const double* Z, int64_t ldz, int64_t n, int k, const double* U, int64_t ldu,
                      int s, double* G, int64_t ldg, double* part, size_t part_doubles,
                      cudaStream_t st) {
  const int sms = num_sms();
  int rb = (int)std::min<int64_t>(PG_RMAX, (ceil_div(n, sms) + 7) / 8 * 8);
  while (rb > 8 && proj_gram_smem<NT>(k, rb) > PG_SMEM) rb -= 8;
  const size_t smem = proj_gram_smem<NT>(k, rb);
  if (smem > PG_SMEM) return false;
  int P = (int)std::min<int64_t>(ceil_div(n, rb), sms);
  if ((size_t)P * NT * 8 * NT * 8 > part_doubles) return false;
  static std::mutex attr_mu;
  static uint64_t attr_mask = 0;
  per_device_once(attr_mu, attr_mask, [&] {
    DME_CUDA(cudaFuncSetAttribute(proj_gram_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)PG_SMEM));
  });
  int per_sm = 0;
  DME_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, proj_gram_kernel<NT>,
                                                         PG_WARPS * 32, smem));
  if (per_sm < 1) return false;
  P = std::min(P, per_sm * sms);
  void* args[] = {(void*)&Z, (void*)&ldz, (void*)&n, (void*)&k, (void*)&U, (void*)&ldu,
                  (void*)&s, (void*)&rb, (void*)&part, (void*)&G, (void*)&ldg};
  DME_CUDA(cudaLaunchCooperativeKernel((void*)proj_gram_kernel<NT>, dim3(P), dim3(PG_WARPS * 32), args,
                                       smem, st));
  DME_KCHECK();
  return true;
}

}  // namespace

void check_square(const double* X, int64_t n, int64_t ld, int* flags2, cudaStream_t st) {
  zero_ints<<<1, 32, 0, st>>>(flags2, 2);
  DME_KCHECK();
  dim3 grid((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32));
  check_square_kernel<<<grid, dim3(32, 8), 0, st>>>(X, n, ld, flags2);
  DME_KCHECK();
}

void mirror_lower(double* X, int64_t n, int64_t ld, bool average, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32));
  mirror_kernel<<<grid, dim3(32, 8), 0, st>>>(X, n, ld, average ? 1 : 0);
  DME_KCHECK();
  if (average) {
    mirror_upper_from_lower<<<grid_for(n * n), 256, 0, st>>>(X, n, ld);
    DME_KCHECK();
  }
}

void transpose_scale(const double* A, int64_t n, int64_t lda, double alpha, double* out,
                     int64_t ldo, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32));
  transpose_scale_kernel<<<grid, dim3(32, 8), 0, st>>>(A, n, lda, alpha, out, ldo);
  DME_KCHECK();
}

void rowabs_max(const double* A, int64_t n, int64_t lda, double* scratch, double* out,
                cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>(n, 1024);
  rowabs_max_kernel<<<blocks, 256, 0, st>>>(A, n, lda, scratch);
  DME_KCHECK();
  max_reduce_kernel<<<1, 1024, 0, st>>>(scratch, blocks, out);
  DME_KCHECK();
}

void lincomb(double* out, int64_t n, int64_t ld, LinTerm t0, LinTerm t1, LinTerm t2, LinTerm t3,
             double diag, cudaStream_t st) {
  lincomb_kernel<<<grid_for(n * n), 256, 0, st>>>(out, n, ld, t0, t1, t2, t3, diag);
  DME_KCHECK();
}

void copy_cols(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
               int64_t cols, double alpha, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  copy_cols_kernel<<<grid_for(rows * cols), 256, 0, st>>>(dst, ldd, src, lds, rows, cols, alpha);
  DME_KCHECK();
}

void rowmajor_to_colmajor(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
                          int64_t cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  rowmajor_to_colmajor_kernel<<<grid_for(rows * cols), 256, 0, st>>>(dst, ldd, src, lds, rows, cols);
  DME_KCHECK();
}

// CTA b owns the columns j of its slice of [0, r): it stages Gh[:, LA] (rows x kp) and Tm in
// shared memory, forms F[:, j] = Gh[:, LA] Tm[:, j] for all q + m + kp rows, then writes G12 /
// G21, H2 and G22[i, j] = G22[j, i] (i <= j) for its j; CTA 0 also copies G11 and H1. Launched on
// cong_ctas() CTAs (32: the look-ahead E pass of the previous step has finished when the
// congruence runs; 8 / 16 / 32 measured 2117 / 2124 / 2133 steps/s at config 5).
constexpr int CONG_CTAS_DEFAULT = 32;
int cong_ctas() {  // (DME_CONG_CTAS: A/B knob)
  static const int v = [] {
    const char* e = std::getenv("DME_CONG_CTAS");
    const int x = e ? std::atoi(e) : CONG_CTAS_DEFAULT;
    return x < 1 ? 1 : (x > 64 ? 64 : x);
  }();
  return v;
}
__global__ void __launch_bounds__(512) gram_congruence_kernel(const double* __restrict__ Gh,
                                                              int64_t ldh, int q, int m, int kp,
                                                              const double* __restrict__ Tm,
                                                              int64_t ldt, int r, double* G,
                                                              int64_t ldg) {
  pdl_wait();
  extern __shared__ double sm[];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int rows = q + m + kp, la = q + m, k = q + r;
  const int j0 = (int)((int64_t)blockIdx.x * r / gridDim.x);
  const int j1 = (int)((int64_t)(blockIdx.x + 1) * r / gridDim.x);
  const int nj = j1 - j0;
  if (blockIdx.x == 0) {
    for (int e = tid; e < q * q; e += nt) {
      const int i = e % q, jj = e / q;
      G[i + (size_t)jj * ldg] = Gh[i + (size_t)jj * ldh];
    }
    for (int e = tid; e < q * m; e += nt) {
      const int i = e % q, mu = e / q;
      G[i + (size_t)(k + mu) * ldg] = Gh[i + (size_t)(q + mu) * ldh];
    }
  }
  if (nj <= 0) return;
  double* Gs = sm;                        // rows x kp, column-major (ld rows)
  double* T = Gs + (size_t)rows * kp;     // kp x r, column-major (ld kp)
  double* F = T + (size_t)kp * r;         // rows x nj, column-major (ld rows)
  for (int e = tid; e < rows * kp; e += nt) {
    const int i = e % rows, l = e / rows;
    Gs[e] = Gh[i + (size_t)(la + l) * ldh];
  }
  for (int e = tid; e < kp * r; e += nt) T[e] = Tm[(e % kp) + (size_t)(e / kp) * ldt];
  __syncthreads();
  for (int e = tid; e < rows * nj; e += nt) {
    const int i = e % rows, jj = e / rows;
    const double* t = T + (size_t)(j0 + jj) * kp;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int l = 0;
    for (; l + 3 < kp; l += 4) {
      s0 = fma(Gs[i + (size_t)l * rows], t[l], s0);
      s1 = fma(Gs[i + (size_t)(l + 1) * rows], t[l + 1], s1);
      s2 = fma(Gs[i + (size_t)(l + 2) * rows], t[l + 2], s2);
      s3 = fma(Gs[i + (size_t)(l + 3) * rows], t[l + 3], s3);
    }
    for (; l < kp; ++l) s0 = fma(Gs[i + (size_t)l * rows], t[l], s0);
    F[i + (size_t)jj * rows] = (s0 + s1) + (s2 + s3);
  }
  __syncthreads();
  for (int e = tid; e < q * nj; e += nt) {  // G12 / G21
    const int i = e % q, jj = e / q;
    const double v = F[i + (size_t)jj * rows];
    G[i + (size_t)(q + j0 + jj) * ldg] = v;
    G[(q + j0 + jj) + (size_t)i * ldg] = v;
  }
  for (int e = tid; e < m * nj; e += nt) {  // H2
    const int mu = e % m, jj = e / m;
    G[(q + j0 + jj) + (size_t)(k + mu) * ldg] = F[(q + mu) + (size_t)jj * rows];
  }
  for (int e = tid; e < r * nj; e += nt) {  // G22[i, j] for i <= j, mirrored
    const int i = e % r, jj = e / r, j = j0 + jj;
    if (i > j) continue;
    const double* t = T + (size_t)i * kp;
    const double* f = F + la + (size_t)jj * rows;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int l = 0;
    for (; l + 3 < kp; l += 4) {
      s0 = fma(t[l], f[l], s0);
      s1 = fma(t[l + 1], f[l + 1], s1);
      s2 = fma(t[l + 2], f[l + 2], s2);
      s3 = fma(t[l + 3], f[l + 3], s3);
    }
    for (; l < kp; ++l) s0 = fma(t[l], f[l], s0);
    const double v = (s0 + s1) + (s2 + s3);
    G[(q + i) + (size_t)(q + j) * ldg] = v;
    G[(q + j) + (size_t)(q + i) * ldg] = v;
  }
}

size_t gram_congruence_smem(int q, int m, int kp, int r) {
  const int rows = q + m + kp;
  const int ctas = std::max(1, std::min(cong_ctas(), r));
  const int njmax = (r + ctas - 1) / ctas;
  return sizeof(double) * ((size_t)rows * kp + (size_t)kp * r + (size_t)rows * njmax);
}

void gram_congruence(const double* Gh, int64_t ldh, int q, int m, int kp, const double* Tm,
                     int64_t ldt, int r, double* G, int64_t ldg, cudaStream_t st) {
  if (q + r <= 0) return;
  const int ctas = std::max(1, std::min(cong_ctas(), r));
  const size_t smem = gram_congruence_smem(q, m, kp, r);
  static std::mutex attr_mu;
  static uint64_t attr_mask = 0;
  per_device_once(attr_mu, attr_mask, [&] {
    DME_CUDA(cudaFuncSetAttribute(gram_congruence_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  220 * 1024));
  });
  if (smem > 220 * 1024) throw std::runtime_error("gram_congruence: too large");
  launch_pdl(gram_congruence_kernel, dim3(ctas), dim3(512), smem, st, Gh, ldh, q, m, kp, Tm, ldt, r, G, ldg);
  DME_KCHECK();
}

// Signed core of a Richardson combination (dme_extrapolate). Tm (k x r1, ld ldt) = W_kept Theta^{1/2}
// from the Gram eigen-compression of Zc = [Z_fine | Z_coarse]; S = diag(wf I_kf, wc I_(k-kf)).
// M = Tm^T S Tm (r1 x r1, symmetric indefinite) is diagonalised by parallel cyclic Jacobi
// (round-robin pair ordering, one CTA), eigenvalues kept by |lambda| > tol max|lambda| in
// descending |lambda|, and T2 = Tm Theta^{-1} U_kept (k x r2) is written so that
// L = Zc T2 (orthonormal columns) and D = diag(lambda_kept) give P = L D L^T.
constexpr int SC_MAX = 112;
__global__ void __launch_bounds__(512) signed_core_kernel(const double* __restrict__ Tm, int64_t ldt,
                                                          int k, int r1, int kf, double wf, double wc,
                                                          double tol, double* __restrict__ T2,
                                                          int64_t ldt2, double* __restrict__ lam,
                                                          int* __restrict__ r2_out, int raw) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int n2 = (r1 + 1) & ~1;  // even number of players (one dummy when r1 is odd)
  double* M = sm;                  // n2 x n2 (row-major, ld n2)
  double* U = M + n2 * n2;         // n2 x n2
  __shared__ double th[SC_MAX + 1], cs[SC_MAX / 2 + 1], sn[SC_MAX / 2 + 1], red[32];
  __shared__ int pp[SC_MAX / 2 + 1], qq[SC_MAX / 2 + 1], perm[SC_MAX + 1];
  __shared__ int s_stop, s_r2;
  for (int j = tid; j < r1; j += nt) {
    double a = 0.0;
    for (int i = 0; i < k; ++i) a = fma(Tm[i + (size_t)j * ldt], Tm[i + (size_t)j * ldt], a);
    th[j] = a;  // theta_j (W columns are unit vectors)
  }
  for (int e = tid; e < n2 * n2; e += nt) {
    const int i = e / n2, j = e % n2;
    double a = 0.0;
    if (i < r1 && j < r1) {
      for (int l = 0; l < k; ++l)
        a = fma(Tm[l + (size_t)i * ldt] * (l < kf ? wf : wc), Tm[l + (size_t)j * ldt], a);
    }
    M[e] = a;
    U[e] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < n2 * n2; e += nt) {  // exact symmetry
    const int i = e / n2, j = e % n2;
    if (i < j) {
      const double v = 0.5 * (M[i * n2 + j] + M[j * n2 + i]);
      M[i * n2 + j] = v;
    }
  }
  __syncthreads();
  for (int e = tid; e < n2 * n2; e += nt) {
    const int i = e / n2, j = e % n2;
    if (i > j) M[i * n2 + j] = M[j * n2 + i];
  }
  __syncthreads();
  const int half = n2 / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    // convergence: off-diagonal mass relative to the diagonal
    double off = 0.0, dia = 0.0;
    for (int e = tid; e < n2 * n2; e += nt) {
      const int i = e / n2, j = e % n2;
      const double v = M[e] * M[e];
      if (i == j) dia += v; else off += v;
    }
    for (int o = 16; o; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      dia += __shfl_xor_sync(0xffffffffu, dia, o);
    }
    if ((tid & 31) == 0) {
      red[tid >> 5] = off;
      red[16 + (tid >> 5)] = dia;
    }
    __syncthreads();
    if (tid == 0) {
      double o2 = 0.0, d2 = 0.0;
      for (int w = 0; w < (nt >> 5); ++w) { o2 += red[w]; d2 += red[16 + w]; }
      s_stop = o2 <= 1e-32 * d2;  // off-diagonal Frobenius mass below (1e-16)^2 of the diagonal
    }
    __syncthreads();
    if (s_stop) break;
    for (int round = 0; round < n2 - 1; ++round) {
      if (tid < half) {  // round-robin: player 0 fixed, the others rotate
        int a = tid == 0 ? 0 : 1 + (tid - 1 + round) % (n2 - 1);
        int b = 1 + (n2 - 2 - tid + round) % (n2 - 1);
        if (a > b) { const int t = a; a = b; b = t; }
        pp[tid] = a;
        qq[tid] = b;
        double c = 1.0, sv = 0.0;
        const double apq = M[a * n2 + b];
        if (a < r1 && b < r1 && apq != 0.0) {
          const double tau = (M[b * n2 + b] - M[a * n2 + a]) / (2.0 * apq);
          const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + t * t);
          sv = t * c;
        }
        cs[tid] = c;
        sn[tid] = sv;
      }
      __syncthreads();
      for (int e = tid; e < half * n2; e += nt) {  // rows p, q
        const int pr = e / n2, j = e % n2;
        const int a = pp[pr], b = qq[pr];
        const double c = cs[pr], sv = sn[pr];
        const double x = M[a * n2 + j], y = M[b * n2 + j];
        M[a * n2 + j] = c * x - sv * y;
        M[b * n2 + j] = sv * x + c * y;
      }
      __syncthreads();
      for (int e = tid; e < half * n2; e += nt) {  // columns p, q of M and U
        const int pr = e / n2, i = e % n2;
        const int a = pp[pr], b = qq[pr];
        const double c = cs[pr], sv = sn[pr];
        const double x = M[i * n2 + a], y = M[i * n2 + b];
        M[i * n2 + a] = c * x - sv * y;
        M[i * n2 + b] = sv * x + c * y;
        const double u = U[i * n2 + a], w = U[i * n2 + b];
        U[i * n2 + a] = c * u - sv * w;
        U[i * n2 + b] = sv * u + c * w;
      }
      __syncthreads();
    }
  }
  if (tid == 0) {  // order by |lambda| descending (stable), truncate
    double mx = 0.0;
    for (int i = 0; i < r1; ++i) { perm[i] = i; mx = fmax(mx, fabs(M[i * n2 + i])); }
    for (int i = 1; i < r1; ++i) {
      const int v = perm[i];
      int j = i - 1;
      while (j >= 0 && fabs(M[perm[j] * n2 + perm[j]]) < fabs(M[v * n2 + v])) { perm[j + 1] = perm[j]; --j; }
      perm[j + 1] = v;
    }
    int r2 = 0;
    while (r2 < r1 && mx > 0.0 && fabs(M[perm[r2] * n2 + perm[r2]]) > tol * mx) ++r2;
    s_r2 = r2;
    *r2_out = r2;
    for (int c = 0; c < r2; ++c) lam[c] = M[perm[c] * n2 + perm[c]];
  }
  __syncthreads();
  const int r2 = s_r2;
  if (raw) {  // T2 = U_kept (r1 x r2): the caller's basis is already orthonormal
    for (int e = tid; e < r1 * r2; e += nt) {
      const int i = e % r1, c = e / r1;
      T2[i + (size_t)c * ldt2] = U[i * n2 + perm[c]];
    }
  } else {
    for (int e = tid; e < k * r2; e += nt) {  // T2 = Tm Theta^{-1} U_kept
      const int i = e % k, c = e / k;
      const int col = perm[c];
      double a = 0.0;
      for (int j = 0; j < r1; ++j) a = fma(Tm[i + (size_t)j * ldt] / th[j], U[j * n2 + col], a);
      T2[i + (size_t)c * ldt2] = a;
    }
  }
}

void signed_core(const double* Tm, int64_t ldt, int k, int r1, int kf, double wf, double wc, double tol,
                 double* T2, int64_t ldt2, double* lam, int* r2_dev, cudaStream_t st, bool raw) {
  if (r1 <= 0) {
    DME_CUDA(cudaMemsetAsync(r2_dev, 0, sizeof(int), st));
    return;
  }
  if (r1 > SC_MAX) throw std::runtime_error("signed_core: rank of the combined factor exceeds 112");
  const int n2 = (r1 + 1) & ~1;
  const size_t smem = sizeof(double) * 2 * (size_t)n2 * n2;
  static std::mutex attr_mu;
  static uint64_t attr_mask = 0;
  per_device_once(attr_mu, attr_mask, [&] {
    DME_CUDA(cudaFuncSetAttribute(signed_core_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double) * 2 * (SC_MAX + 1) * (SC_MAX + 1))));
  });
  signed_core_kernel<<<1, 512, smem, st>>>(Tm, ldt, k, r1, kf, wf, wc, tol, T2, ldt2, lam, r2_dev,
                                            raw ? 1 : 0);
  DME_KCHECK();
}

void tall_small(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                int64_t M, int64_t N, int64_t K, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) throw std::runtime_error("tall_small: K must be positive");
  if (C == A && N > TS_BN) throw std::runtime_error("tall_small: in place needs N <= 64");
  dim3 grid((unsigned)ceil_div(M, TS_BM), (unsigned)ceil_div(N, TS_BN));
  launch_pdl(tall_small_kernel, grid, dim3(256), 0, st, A, lda, B, ldb, C, ldc, M, N, K);
  DME_KCHECK();
}

namespace {
// thread per (row, column): consecutive threads take consecutive rows of one column (coalesced
// stores; the gathers of a banded / diagonal S stay within a few sectors)
__global__ void spmm_csr_kernel(const int* __restrict__ rp, const int* __restrict__ ci,
                                const double* __restrict__ v, int64_t n, const double* __restrict__ X,
                                int64_t ldx, int64_t k, double* __restrict__ out, int64_t ldo,
                                double alpha) {
  const int64_t total = n * k;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / n, i = t - j * n;
    const double* xj = X + j * ldx;
    double acc = 0.0;
    for (int e = rp[i]; e < rp[i + 1]; ++e) acc = fma(v[e], xj[ci[e]], acc);
    out[i + j * ldo] = alpha * acc;
  }
}
}  // namespace

bool proj_gram(const double* Z, int64_t ldz, int64_t n, int k, const double* U, int64_t ldu, int s,
               double* G, int64_t ldg, double* part, size_t part_doubles, cudaStream_t st) {
  if (n <= 0 || s <= 0) return true;
  if (k > PG_KMAX || s > 96 || s > k) return false;
  if (s <= 32) return proj_gram_launch<4>(Z, ldz, n, k, U, ldu, s, G, ldg, part, part_doubles, st);
  if (s <= 64) return proj_gram_launch<8>(Z, ldz, n, k, U, ldu, s, G, ldg, part, part_doubles, st);
  return proj_gram_launch<12>(Z, ldz, n, k, U, ldu, s, G, ldg, part, part_doubles, st);
}

void spmm_csr(const int* rp, const int* ci, const double* v, int64_t n, const double* X, int64_t ldx,
              int64_t k, double* out, int64_t ldo, double alpha, cudaStream_t st) {
  if (n <= 0 || k <= 0) return;
  const int64_t total = n * k;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
  spmm_csr_kernel<<<blocks, 256, 0, st>>>(rp, ci, v, n, X, ldx, k, out, ldo, alpha);
  DME_KCHECK();
}

}  // namespace dme
