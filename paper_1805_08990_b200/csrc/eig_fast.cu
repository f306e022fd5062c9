// Fast one-CTA eigen-compression for k <= FAST_K_MAX (the hot-path case: k = r + q_I ~ 60-130).
//
// Same contract as the Jacobi kernel in small.cu (G = Zc^T Zc = W Theta W^T, Tm = W_kept, fused T3),
// computed with O(k) synchronisation steps instead of O(k * sweeps):
//   1. Householder tridiagonalisation Q^T G Q = T (LAPACK dsytd2 recurrences; G kept in shared memory,
//      one warp per row for the symmetric mat-vec and the rank-2 update, all rows of a warp and all
//      column chunks unrolled so loads and shuffle reductions overlap; reflectors stay in place).
//   2. Eigenvalues of T by multisection on Sturm counts; the count uses the determinant recurrence
//      p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2} (no division: one dependent DFMA per element,
//      backward stable like the ratio form), signs and exponents read with integer ops, power-of-2
//      rescaling every 4 elements. Only the kept eigenvalues (the top min(cap, #theta >
//      tol*theta_max)) plus the first dropped one are refined.
//   3. Eigenvectors of T by the twisted factorisation (Parlett-Dhillon): top-down D+ and bottom-up D-
//      pivots, twist index argmin |gamma_i|, ratio pass then product pass; one thread per vector.
//   4. Back-transformation W = Q Z, one warp per column block with Z held in registers.
//   5. Orthogonality check, weighted by sqrt(theta_i theta_j)/theta_max (the size of the error it
//      causes in P): near-degenerate clusters, where the twisted vectors are not orthogonal, make
//      *r_out = -1 and the caller falls back to the Jacobi kernel.
// Templated on the size class FK (96 or 160) so every per-lane array has a compile-time extent.
#include "common.cuh"
#include "small.h"
#include "small_common.cuh"
#include "eig_common.cuh"

#include <cmath>

namespace dme {

namespace {

using namespace eigk;

template <int FK>
__global__ void __launch_bounds__(ENT, 1) eig_fast_kernel(SmallArgs a) {
  pdl_wait();
  constexpr int RCH = (FK + 31) / 32;      // column chunks per lane
  constexpr int RPW = (FK + NW - 1) / NW;  // rows per warp
  extern __shared__ double A[];            // k x ld, full symmetric, ld odd
  __shared__ double d[FK], e[FK], e2[FK], tau[FK], vec[FK], pv[FK], pv2[FK];
  __shared__ double lam[FK + 1];           // kept eigenvalues (+1 dropped), descending (normalised)
  __shared__ double lo_s[FK + 1], hi_s[FK + 1], slam[FK + 1];
  __shared__ int cnt_s[ENT];
  __shared__ double red[NW];
  __shared__ int s_r, s_bad;
  __shared__ double s_scale, s_lo, s_hi, s_tmax, s_lo_t, s_hi_t;
  __shared__ double Gam[SMALL_M_MAX * SMALL_M_MAX];
  __shared__ double Phi[SMALL_M_MAX * SMALL_M_MAX];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = a.k;
  const int ld = k | 1;
  long long t_ph[7];
  t_ph[0] = clock64();

  // ---------------------------------------------------------------- load G (symmetrised)
  for (int e_ = tid; e_ < k * k; e_ += ENT) {
    const int i = e_ % k, j = e_ / k;
    A[i * ld + j] = 0.5 * (a.G[i + (size_t)j * a.ldg] + a.G[j + (size_t)i * a.ldg]);
  }
  __syncthreads();

  // ---------------------------------------------------------------- 1. tridiagonalisation
  tridiagonalise<FK>(A, k, ld, d, e, tau, vec, pv, pv2);
  if (tid == 0) {
    normalise_tridiagonal(k, d, e, e2, &s_scale, &s_lo, &s_hi);
    s_lo_t = s_lo;
    s_hi_t = s_hi;
  }
  __syncthreads();
  t_ph[1] = clock64();

  // ---------------------------------------------------------------- 2. eigenvalues (multisection)
  // largest eigenvalue: 256 probes per round (8 bits), transition found in parallel
  {
    constexpr int PB = 256;
    for (int it = 0; it < 2; ++it) {  // 16 bits: the threshold needs ~3 digits
      const double a0 = s_lo_t, b0 = s_hi_t;
      if (tid < PB) cnt_s[tid] = sturm_count(d, e2, k, a0 + (b0 - a0) * (tid + 1) / (PB + 1.0));
      __syncthreads();
      if (tid < PB) {
        const bool le = cnt_s[tid] <= k - 1;
        const bool nxt = (tid + 1 < PB) ? (cnt_s[tid + 1] <= k - 1) : false;
        if (le && !nxt) {  // last probe below the top eigenvalue
          s_lo_t = a0 + (b0 - a0) * (tid + 1) / (PB + 1.0);
          if (tid + 1 < PB) s_hi_t = a0 + (b0 - a0) * (tid + 2) / (PB + 1.0);
        }
        if (tid == 0 && !le) s_hi_t = a0 + (b0 - a0) / (PB + 1.0);
      }
      __syncthreads();
    }
    if (tid == 0) s_tmax = a.ref_max > 0.0 ? a.ref_max / s_scale : 0.5 * (s_lo_t + s_hi_t);
    __syncthreads();
  }
  t_ph[2] = clock64();
  // rank: eigenvalues > tol * theta_max (at most cap)
  if (tid == 0) {
    const double tmax = s_tmax;
    int r = 0;
    if (tmax > 0.0) r = k - sturm_count(d, e2, k, a.tol * tmax);
    if (r > a.cap) r = a.cap;
    if (r < 0) r = 0;
    s_r = r;
  }
  __syncthreads();
  const int r = s_r;
  const int nr = r < k ? r + 1 : r;  // + the first dropped one, for the stats
  {
    int P = nr > 0 ? ENT / nr : 1;
    P = P < 1 ? 1 : P;  // (up to all ENT threads on one eigenvalue: 9 bits per round)
    const int grp = tid / P, t = tid % P;
    const bool act = grp < nr;
    const int jj = k - 1 - grp;
    if (act && t == 0) {
      lo_s[grp] = s_lo;
      hi_s[grp] = s_hi;
    }
    __syncthreads();
    const float bits = __log2f((float)P + 1.0f);  // (fast float math: only sizes the loop)
    // absolute accuracy 1e-13 ||T||: enough for the twisted vectors (their error ~ |dlambda| / gap
    // only matters weighted by theta)
    const int nit = (int)ceilf(1.00001f * __log2f((float)((s_hi - s_lo) / 1e-13) + 1.0f) / bits) + 1;
    for (int it = 0; it < nit; ++it) {
      if (act) {
        const double a0 = lo_s[grp], b0 = hi_s[grp];
        cnt_s[tid] = sturm_count(d, e2, k, a0 + (b0 - a0) * (t + 1) / (P + 1.0));
      }
      __syncthreads();
      double a0 = 0.0, b0 = 0.0;
      if (act) { a0 = lo_s[grp]; b0 = hi_s[grp]; }
      __syncthreads();  // every thread has read the bracket before the transition thread moves it
      if (act) {  // transition between probe t and t+1 (counts are monotone in the probe position)
        const bool le = cnt_s[tid] <= jj;
        const bool nxt = (t + 1 < P) ? (cnt_s[tid + 1] <= jj) : false;
        if (le && !nxt) {
          lo_s[grp] = a0 + (b0 - a0) * (t + 1) / (P + 1.0);
          if (t + 1 < P) hi_s[grp] = a0 + (b0 - a0) * (t + 2) / (P + 1.0);
        }
        if (t == 0 && !le) hi_s[grp] = a0 + (b0 - a0) / (P + 1.0);
      }
      __syncthreads();
    }
    if (act && t == 0) {
      lam[grp] = 0.5 * (lo_s[grp] + hi_s[grp]);
      slam[grp] = sqrt(fabs(lam[grp]));
    }
    __syncthreads();
  }
  t_ph[3] = clock64();

  // ---------------------------------------------------------------- 3. twisted-factorisation vectors
  // lane pair (2c, 2c+1) per eigenvector: the even lane runs the top-down pivots D+, the odd lane the
  // bottom-up pivots D- (two independent division chains), then each runs one product chain.
  // D+ in V[:, c], D- in Tm[:, c] (global scratch), the vector into V[:, c].
  if (tid < 2 * r) {
    const unsigned msk = __activemask();  // lane pairs are always complete (2r is even)
    const int c = tid >> 1, side = tid & 1;
    const double lm = lam[c];
    double* Dp = a.V + (size_t)c * a.ldv;
    double* Dm = a.Tm + (size_t)c * a.ldt;
    twisted_pivots(d, e2, k, lm, side == 0, side == 0 ? Dp : Dm);
    __syncwarp(msk);
    __threadfence_block();
    // twist index: argmin |gamma_i|, the two lanes scan halves
    const int h0 = side ? k / 2 : 0, h1 = side ? k : k / 2;
    int tw = h0;
    double best = 1e300;
    for (int i = h0; i < h1; ++i) {
      const double g = Dp[i] + Dm[i] - (d[i] - lm);
      if (fabs(g) < best) { best = fabs(g); tw = i; }
    }
    const double ob = __shfl_xor_sync(msk, best, 1);
    const int ot = __shfl_xor_sync(msk, tw, 1);
    if (ob < best || (ob == best && ot < tw)) { best = ob; tw = ot; }
    // ratios then products: even lane i < tw (with D+), odd lane i > tw (with D-)
    double nrm2 = 0.0;
    if (side == 0) {
      for (int i = 0; i < tw; ++i) Dp[i] = -e[i] / Dp[i];
      double zi = 1.0;
      for (int i = tw - 1; i >= 0; --i) {
        zi *= Dp[i];
        nrm2 = fma(zi, zi, nrm2);
        Dp[i] = zi;
      }
    } else {
      for (int i = tw + 1; i < k; ++i) Dm[i] = -e[i - 1] / Dm[i];
      double zi = 1.0;
      for (int i = tw + 1; i < k; ++i) {
        zi *= Dm[i];
        nrm2 = fma(zi, zi, nrm2);
        Dp[i] = zi;
      }
    }
    nrm2 += __shfl_xor_sync(msk, nrm2, 1);
    __syncwarp(msk);
    __threadfence_block();
    if (side == 0) Dp[tw] = 1.0;
    __syncwarp(msk);
    __threadfence_block();
    const double inv = 1.0 / sqrt(1.0 + nrm2);
    for (int i = side; i < k; i += 2) Dp[i] *= inv;
  }
  __syncthreads();
  t_ph[4] = clock64();

  // ---------------------------------------------------------------- 4. W = Q Z
  if (FK <= 96) {
    // Thread c applies H_{k-3} ... H_0 to its own column z_c, kept in shared memory right after the
    // reflectors (column-major, odd leading dimension: a warp's columns spread over all banks).
    const int ldz = k | 1;
    double* zs = A + (size_t)k * ld;
    if (tid < r) {
      const int c = tid;
      double* z = zs + (size_t)c * ldz;
      for (int i = 0; i < k; ++i) z[i] = a.V[i + (size_t)c * a.ldv];
      for (int j = k - 3; j >= 0; --j) {
        const double tj = tau[j];
        if (tj == 0.0) continue;
        const double* v = A + j * ld + j + 1;  // v_0 = 1 (implicit), v_i at row j
        double* zz = z + j + 1;
        const int m = k - j - 1;
        double s0 = zz[0], s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int i = 1;
        for (; i + 2 < m; i += 3) {
          s1 = fma(v[i], zz[i], s1);
          s2 = fma(v[i + 1], zz[i + 1], s2);
          s3 = fma(v[i + 2], zz[i + 2], s3);
        }
        for (; i < m; ++i) s1 = fma(v[i], zz[i], s1);
        const double f = tj * ((s0 + s1) + (s2 + s3));
        zz[0] -= f;
        for (i = 1; i < m; ++i) zz[i] = fma(-f, v[i], zz[i]);
      }
      const double fs = a.sqrt_scale ? sqrt(fmax(lam[c] * s_scale, 0.0)) : 1.0;
      for (int i = 0; i < k; ++i) a.Tm[i + (size_t)c * a.ldt] = z[i] * fs;
    }
  } else {
    // warp-owned column blocks, Z in registers, one warp reduction per reflector and column
    constexpr int CP = 4;  // columns per warp per pass (register budget)
    const double sc = s_scale;
    for (int pass = 0; pass * NW * CP < r; ++pass) {
      double z[CP][RCH];
#pragma unroll
      for (int cc = 0; cc < CP; ++cc) {
        const int c = warp + NW * (pass * CP + cc);
#pragma unroll
        for (int u = 0; u < RCH; ++u) {
          const int i = lane + 32 * u;
          z[cc][u] = (c < r && i < k) ? a.V[i + (size_t)c * a.ldv] : 0.0;
        }
      }
      if (warp + NW * pass * CP < r) {
        for (int j = k - 3; j >= 0; --j) {
          const double tj = tau[j];
          if (tj == 0.0) continue;
          double vr[RCH];
#pragma unroll
          for (int u = 0; u < RCH; ++u) {
            const int i = lane + 32 * u;
            vr[u] = (i == j + 1) ? 1.0 : ((i > j + 1 && i < k) ? A[j * ld + i] : 0.0);
          }
          double sv[CP];
#pragma unroll
          for (int cc = 0; cc < CP; ++cc) {
            sv[cc] = 0.0;
#pragma unroll
            for (int u = 0; u < RCH; ++u) sv[cc] = fma(vr[u], z[cc][u], sv[cc]);
          }
#pragma unroll
          for (int o = 16; o; o >>= 1)
#pragma unroll
            for (int cc = 0; cc < CP; ++cc) sv[cc] += __shfl_xor_sync(0xffffffffu, sv[cc], o);
#pragma unroll
          for (int cc = 0; cc < CP; ++cc) {
            const double f = tj * sv[cc];
#pragma unroll
            for (int u = 0; u < RCH; ++u) z[cc][u] -= f * vr[u];
          }
        }
      }
#pragma unroll
      for (int cc = 0; cc < CP; ++cc) {
        const int c = warp + NW * (pass * CP + cc);
        if (c < r) {
          const double f = a.sqrt_scale ? sqrt(fmax(lam[c] * sc, 0.0)) : 1.0;
#pragma unroll
          for (int u = 0; u < RCH; ++u) {
            const int i = lane + 32 * u;
            if (i < k) a.Tm[i + (size_t)c * a.ldt] = z[cc][u] * f;
          }
        }
      }
    }
  }
  __syncthreads();  // all reflector reads from A done before A is reused
  // W^T (row-major) into shared memory for the check (unscaled)
  for (int e_ = tid; e_ < k * r; e_ += ENT) {
    const int i = e_ % k, c = e_ / k;
    const double f = a.sqrt_scale ? sqrt(fmax(lam[c] * s_scale, 0.0)) : 1.0;
    A[c * ld + i] = f > 0.0 ? a.Tm[i + (size_t)c * a.ldt] / f : 0.0;
  }
  __syncthreads();
  t_ph[5] = clock64();

  // ---------------------------------------------------------------- 5. weighted orthogonality check
  {
    // 4x4 blocks of W^T W (upper block triangle), one block per thread
    constexpr int TB = 4;
    const int nb = (r + TB - 1) / TB;
    double mx = 0.0;
    for (int blk = tid; blk < nb * nb; blk += ENT) {
      const int bi = blk % nb, bj = blk / nb;
      if (bi > bj) continue;
      double acc[TB][TB];
#pragma unroll
      for (int x = 0; x < TB; ++x)
#pragma unroll
        for (int y = 0; y < TB; ++y) acc[x][y] = 0.0;
      for (int i = 0; i < k; ++i) {
        double wa[TB], wb[TB];
#pragma unroll
        for (int x = 0; x < TB; ++x) {
          const int c1 = bi * TB + x, c2 = bj * TB + x;
          wa[x] = c1 < r ? A[c1 * ld + i] : 0.0;
          wb[x] = c2 < r ? A[c2 * ld + i] : 0.0;
        }
#pragma unroll
        for (int x = 0; x < TB; ++x)
#pragma unroll
          for (int y = 0; y < TB; ++y) acc[x][y] = fma(wa[x], wb[y], acc[x][y]);
      }
#pragma unroll
      for (int x = 0; x < TB; ++x)
#pragma unroll
        for (int y = 0; y < TB; ++y) {
          const int c1 = bi * TB + x, c2 = bj * TB + y;
          if (c1 < r && c2 < r && c1 <= c2) {
            const double w = (c1 == c2) ? 1.0 : slam[c1] * slam[c2] / fmax(fabs(lam[0]), 1e-300);
            mx = fmax(mx, fabs(acc[x][y] - (c1 == c2 ? 1.0 : 0.0)) * w);
          }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      double m = 0.0;
      for (int w = 0; w < NW; ++w) m = fmax(m, red[w]);
      s_bad = !(m <= a.orth_tol);  // NaN-safe
      if (a.stats) {
        a.stats[0] = (double)r;
        a.stats[1] = s_tmax * s_scale;
        a.stats[2] = (r < k && s_tmax > 0.0) ? fabs(lam[r]) / s_tmax : 0.0;
        a.stats[3] = s_bad ? 1.0 : 0.0;
        a.stats[4] = m;
      }
    }
    __syncthreads();
  }
  t_ph[6] = clock64();
  if (tid == 0 && a.stats)
    for (int i = 0; i < 6; ++i) a.stats[8 + i] = (double)(t_ph[i + 1] - t_ph[i]);
  if (s_bad) {
    if (tid == 0) publish_rank(a, -1);  // caller falls back to the Jacobi kernel
    return;
  }
  if (a.t3 && r > 0) {
    __syncthreads();
    smallk::t3_fuse(a, k, r, A, Gam, Phi);
  }
  if (tid == 0) publish_rank(a, r);
}

template <int FK>
void launch_fast(const SmallArgs& a, cudaStream_t st) {
  const size_t floor_b = sizeof(double) * 2 * SMALL_K_MAX * SMALL_M_MAX;
  auto bytes_for = [](int k) {
    // reflectors (k x (k|1)) + the back-transformation columns (<= k x (k|1)) for the small class
    return sizeof(double) * (size_t)k * (k | 1) * (FK <= 96 ? 2 : 1);
  };
  size_t smem = bytes_for(a.k);
  if (smem < floor_b) smem = floor_b;
  static std::mutex attr_mu;
  static uint64_t attr_mask = 0;
  per_device_once(attr_mu, attr_mask, [&] {
    const size_t need = bytes_for(FK);
    DME_CUDA(cudaFuncSetAttribute(eig_fast_kernel<FK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(need > floor_b ? need : floor_b)));
  });
  launch_pdl(eig_fast_kernel<FK>, dim3(1), dim3(ENT), smem, st, a);
  DME_KCHECK();
}

}  // namespace

void eig_fast(const SmallArgs& a, cudaStream_t st) {
  if (a.k > FAST_K_MAX || a.k < 1) throw std::runtime_error("eig_fast: k out of range");
  if (a.k <= 96) launch_fast<96>(a, st);
  else launch_fast<FAST_K_MAX>(a, st);
}

}  // namespace dme
