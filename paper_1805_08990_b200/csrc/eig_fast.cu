// Fast one-CTA eigen-compression for k <= FAST_K_MAX (the hot-path case: k = r + q_I ~ 60-130).
//
// Same contract as the Jacobi kernel in small.cu (G = Zc^T Zc = W Theta W^T, Tm = W_kept, fused T3),
// computed with O(k) synchronisation steps instead of O(k * sweeps):
//   1. Householder tridiagonalisation Q^T G Q = T (LAPACK dsytd2 recurrences; G kept in shared memory,
//      one warp per row for the symmetric mat-vec and the rank-2 update; reflectors stay in place).
//   2. Eigenvalues of T by multisection on Sturm counts; the count uses the determinant recurrence
//      p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2} (no division: one dependent DFMA per element,
//      backward stable like the ratio form), with power-of-ten rescaling against over/underflow.
//      Only the kept eigenvalues (the top min(cap, #theta > tol*theta_max)) are refined.
//   3. Eigenvectors of T by the twisted factorisation (Parlett-Dhillon): top-down D+ and bottom-up D-
//      pivots, twist index argmin |gamma_i|, two product recurrences; one thread per eigenvector.
//   4. Back-transformation W = Q Z, one warp per column block with Z held in registers.
//   5. Orthogonality check max|W^T W - I|: near-degenerate clusters (where the twisted vectors are
//      not orthogonal) are reported in stats[3] and the caller falls back to the Jacobi kernel.
#include "common.cuh"
#include "small.h"
#include "small_common.cuh"

#include <cmath>

namespace dme {

namespace {

using namespace smallk;

constexpr int FK = FAST_K_MAX;
constexpr int RCH = (FK + 31) / 32;   // row chunks per lane in the back-transformation
constexpr int MAXC = (FK + 31) / 32;  // columns per warp in the back-transformation

// number of eigenvalues of T (d, e2 = e^2, normalised) smaller than x
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int k, double x) {
  double p2 = 1.0, p1 = d[0] - x;
  bool neg_prev = p1 < 0.0 || (p1 == 0.0);
  int cnt = neg_prev ? 1 : 0;
  for (int i = 1; i < k; ++i) {
    double p = fma(d[i] - x, p1, -e2[i - 1] * p2);
    const bool neg = p < 0.0 || (p == 0.0 && !neg_prev);
    cnt += (neg != neg_prev);
    neg_prev = neg;
    p2 = p1;
    p1 = p;
    const double ap = fabs(p);
    if (ap > 1e150) {
      p1 *= 1e-150;
      p2 *= 1e-150;
    } else if (ap < 1e-150 && fabs(p2) < 1e-150) {
      p1 *= 1e150;
      p2 *= 1e150;
    }
  }
  return cnt;
}

__global__ void __launch_bounds__(NT, 1) eig_fast_kernel(SmallArgs a) {
  extern __shared__ double A[];          // k x ld, full symmetric, ld odd
  __shared__ double d[FK], e[FK], e2[FK], tau[FK], vec[FK], pv[FK];
  __shared__ double lam[FK];             // kept eigenvalues, descending (normalised)
  __shared__ double lo_s[FK], hi_s[FK];
  __shared__ int cnt_s[1024];
  __shared__ double red[32];
  __shared__ int s_r, s_bad;
  __shared__ double s_scale, s_lo, s_hi, s_tmax, s_orth, s_lo_t, s_hi_t;
  __shared__ double Gam[SMALL_M_MAX * SMALL_M_MAX];
  __shared__ double Phi[SMALL_M_MAX * SMALL_M_MAX];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = a.k;
  const int ld = k | 1;
  long long t_ph[8];
  t_ph[0] = clock64();

  // ---------------------------------------------------------------- load G (symmetrised)
  for (int e_ = tid; e_ < k * k; e_ += NT) {
    const int i = e_ % k, j = e_ / k;
    A[i * ld + j] = 0.5 * (a.G[i + (size_t)j * a.ldg] + a.G[j + (size_t)i * a.ldg]);
  }
  __syncthreads();

  // ---------------------------------------------------------------- 1. tridiagonalisation
  for (int j = 0; j + 2 < k; ++j) {
    const int m = k - j - 1;
    if (warp == 0) {
      double xn2 = 0.0;
      for (int i = 1 + lane; i < m; i += 32) {
        const double x = A[(j + 1 + i) * ld + j];
        xn2 += x * x;
      }
      for (int o = 16; o; o >>= 1) xn2 += __shfl_xor_sync(0xffffffffu, xn2, o);
      const double alpha = A[(j + 1) * ld + j];
      double t = 0.0, beta = alpha, scal = 0.0;
      if (xn2 > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
        t = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      for (int i = lane; i < m; i += 32) {
        double v = i == 0 ? 1.0 : A[(j + 1 + i) * ld + j] * scal;
        if (t == 0.0) v = (i == 0) ? 1.0 : 0.0;
        vec[i] = v;
        if (i > 0) A[(j + 1 + i) * ld + j] = v;  // reflector kept below the subdiagonal
      }
      if (lane == 0) {
        tau[j] = t;
        e[j] = beta;
        d[j] = A[j * ld + j];
      }
    }
    __syncthreads();
    const double tj = tau[j];
    if (tj == 0.0) continue;  // uniform branch
    // p = tau * A22 v
    for (int i = warp; i < m; i += NT / 32) {
      const double* row = A + (j + 1 + i) * ld + (j + 1);
      double acc = 0.0;
      for (int l = lane; l < m; l += 32) acc += row[l] * vec[l];
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) pv[i] = tj * acc;
    }
    __syncthreads();
    // K = tau/2 p^T v ; A22 -= v w^T + w v^T with w = p - K v
    double dot = 0.0;
    for (int l = lane; l < m; l += 32) dot += pv[l] * vec[l];
    for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    const double K = 0.5 * tj * dot;
    for (int i = warp; i < m; i += NT / 32) {
      double* row = A + (j + 1 + i) * ld + (j + 1);
      const double vi = vec[i], wi = pv[i] - K * vi;
      for (int l = lane; l < m; l += 32) row[l] -= vi * (pv[l] - K * vec[l]) + wi * vec[l];
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (k >= 2) {
      d[k - 2] = A[(k - 2) * ld + (k - 2)];
      e[k - 2] = A[(k - 1) * ld + (k - 2)];
    }
    d[k - 1] = A[(k - 1) * ld + (k - 1)];
    // normalisation by a Gershgorin bound of ||T||
    double nrm = 0.0, lo = 1e300, hi = -1e300;
    for (int i = 0; i < k; ++i) {
      const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < k ? fabs(e[i]) : 0.0);
      nrm = fmax(nrm, fabs(d[i]) + r);
    }
    if (!(nrm > 0.0)) nrm = 1.0;
    s_scale = nrm;
    for (int i = 0; i < k; ++i) {
      d[i] /= nrm;
      if (i + 1 < k) {
        e[i] /= nrm;
        e2[i] = e[i] * e[i];
      }
    }
    for (int i = 0; i < k; ++i) {
      const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < k ? fabs(e[i]) : 0.0);
      lo = fmin(lo, d[i] - r);
      hi = fmax(hi, d[i] + r);
    }
    s_lo = lo - 1e-14;
    s_hi = hi + 1e-14;
    s_lo_t = s_lo;
    s_hi_t = s_hi;
  }
  __syncthreads();

  t_ph[1] = clock64();
  // ---------------------------------------------------------------- 2. eigenvalues (multisection)
  // largest eigenvalue: 256 probes per round (8 bits), transition found in parallel
  {
    constexpr int PB = 256;
    for (int it = 0; it < 7; ++it) {
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
    if (tid == 0) s_tmax = 0.5 * (s_lo_t + s_hi_t);
    __syncthreads();
  }
  t_ph[2] = clock64();
  // rank: eigenvalues > tol * theta_max (at most cap)
  if (tid == 0) {
    const double tmax = s_tmax;
    int r = 0;
    if (tmax > 0.0) {
      const int below = sturm_count(d, e2, k, a.tol * tmax);
      r = k - below;
    }
    if (r > a.cap) r = a.cap;
    if (r < 0) r = 0;
    s_r = r;
  }
  __syncthreads();
  const int r = s_r;
  // refine the top r (+1 dropped, for stats) eigenvalues: ascending index jj = k-1-c
  const int nr = r < k ? r + 1 : r;
  {
    int P = nr > 0 ? 256 / nr : 1;
    P = P < 1 ? 1 : (P > 16 ? 16 : P);
    const int grp = tid / P, t = tid % P;
    const bool act = grp < nr;
    const int jj = k - 1 - grp;
    if (act && t == 0) {
      lo_s[grp] = s_lo;
      hi_s[grp] = s_hi;
    }
    __syncthreads();
    const double width0 = s_hi - s_lo;
    int nit = 0;
    {
      const double bits = log2((double)P + 1.0);
      nit = (int)ceil(log2(width0 / 4e-16 + 1.0) / bits) + 1;
    }
    for (int it = 0; it < nit; ++it) {
      if (act) {
        const double a0 = lo_s[grp], b0 = hi_s[grp];
        const double x = a0 + (b0 - a0) * (t + 1) / (P + 1.0);
        cnt_s[tid] = sturm_count(d, e2, k, x);
      }
      __syncthreads();
      if (act && t == 0) {
        const double a0 = lo_s[grp], b0 = hi_s[grp];
        double na = a0, nb = b0;
        for (int q = 0; q < P; ++q) {
          const double xq = a0 + (b0 - a0) * (q + 1) / (P + 1.0);
          if (cnt_s[grp * P + q] <= jj) na = xq; else { nb = xq; break; }
        }
        lo_s[grp] = na;
        hi_s[grp] = nb;
      }
      __syncthreads();
    }
    if (act && t == 0) lam[grp] = 0.5 * (lo_s[grp] + hi_s[grp]);
    __syncthreads();
  }

  t_ph[3] = clock64();
  // ---------------------------------------------------------------- 3. twisted-factorisation vectors
  // thread c < r: eigenvector of lam[c]; D+ stored in V[:, c], D- in Tm[:, c] (scratch, col-major)
  if (tid < r) {
    const int c = tid;
    const double lm = lam[c];
    double* Dp = a.V + (size_t)c * a.ldv;
    double* Dm = a.Tm + (size_t)c * a.ldt;
    const double pivmin = 1e-290;
    double x = d[0] - lm;
    if (fabs(x) < pivmin) x = -pivmin;
    Dp[0] = x;
    for (int i = 1; i < k; ++i) {
      x = (d[i] - lm) - e2[i - 1] / x;
      if (fabs(x) < pivmin) x = -pivmin;
      Dp[i] = x;
    }
    x = d[k - 1] - lm;
    if (fabs(x) < pivmin) x = -pivmin;
    Dm[k - 1] = x;
    for (int i = k - 2; i >= 0; --i) {
      x = (d[i] - lm) - e2[i] / x;
      if (fabs(x) < pivmin) x = -pivmin;
      Dm[i] = x;
    }
    int tw = 0;
    double best = 1e300;
    for (int i = 0; i < k; ++i) {
      const double g = Dp[i] + Dm[i] - (d[i] - lm);
      if (fabs(g) < best) { best = fabs(g); tw = i; }
    }
    // z into V[:, c]: z_tw = 1, upward with D+, downward with D-
    double zi = 1.0, nrm2 = 1.0;
    for (int i = tw - 1; i >= 0; --i) {
      zi = -(e[i] / Dp[i]) * zi;
      nrm2 += zi * zi;
      Dp[i] = zi;  // overwrite: Dp[i] no longer needed
    }
    zi = 1.0;
    for (int i = tw + 1; i < k; ++i) {
      zi = -(e[i - 1] / Dm[i]) * zi;
      nrm2 += zi * zi;
      Dp[i] = zi;
    }
    Dp[tw] = 1.0;
    const double inv = 1.0 / sqrt(nrm2);
    for (int i = 0; i < k; ++i) Dp[i] *= inv;
  }
  __syncthreads();

  t_ph[4] = clock64();
  // ---------------------------------------------------------------- 4. W = Q Z (warp-owned columns)
  {
    double z[MAXC][RCH];
    int ncol = 0;
#pragma unroll
    for (int cc = 0; cc < MAXC; ++cc) {
      const int c = warp + 32 * cc;
#pragma unroll
      for (int t = 0; t < RCH; ++t) {
        const int i = lane + 32 * t;
        z[cc][t] = (c < r && i < k) ? a.V[i + (size_t)c * a.ldv] : 0.0;
      }
      ncol += (c < r);
    }
    if (ncol > 0) {
      for (int j = k - 3; j >= 0; --j) {
        const double tj = tau[j];
        if (tj == 0.0) continue;
        // v: 1 at row j+1, A[i][j] for rows i >= j+2
        double vr[RCH];
#pragma unroll
        for (int t = 0; t < RCH; ++t) {
          const int i = lane + 32 * t;
          vr[t] = (i == j + 1) ? 1.0 : ((i > j + 1 && i < k) ? A[i * ld + j] : 0.0);
        }
#pragma unroll
        for (int cc = 0; cc < MAXC; ++cc) {
          if (cc >= ncol) break;
          double s = 0.0;
#pragma unroll
          for (int t = 0; t < RCH; ++t) s += vr[t] * z[cc][t];
          for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          s *= tj;
#pragma unroll
          for (int t = 0; t < RCH; ++t) z[cc][t] -= s * vr[t];
        }
      }
    }
    __syncthreads();  // all reflector reads from A done before A is reused
#pragma unroll
    for (int cc = 0; cc < MAXC; ++cc) {
      const int c = warp + 32 * cc;
      if (c < r) {
#pragma unroll
        for (int t = 0; t < RCH; ++t) {
          const int i = lane + 32 * t;
          if (i < k) {
            a.Tm[i + (size_t)c * a.ldt] = z[cc][t] * (a.sqrt_scale ? sqrt(fmax(lam[c] * s_scale, 0.0)) : 1.0);
            A[c * ld + i] = z[cc][t];  // W^T row-major copy for the check
          }
        }
      }
    }
  }
  __syncthreads();

  t_ph[5] = clock64();
  // ---------------------------------------------------------------- 5. orthogonality check
  {
    double mx = 0.0;
    for (int p = warp; p < r * r; p += NT / 32) {
      const int c1 = p % r, c2 = p / r;
      if (c1 > c2) continue;
      double acc = 0.0;
      for (int i = lane; i < k; i += 32) acc += A[c1 * ld + i] * A[c2 * ld + i];
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      // weighted by sqrt(theta_1 theta_2)/theta_max: the error this causes in P = Zc W W^T Zc^T
      // (tiny-eigenvalue vectors are only determined to eps*||T||/gap, harmlessly so)
      const double w = sqrt(fabs(lam[c1] * lam[c2])) / fmax(fabs(lam[0]), 1e-300);
      mx = fmax(mx, fabs(acc - (c1 == c2 ? 1.0 : 0.0)) * (c1 == c2 ? 1.0 : w));
    }
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      double m = 0.0;
      for (int w = 0; w < NT / 32; ++w) m = fmax(m, red[w]);
      s_orth = m;
      s_bad = !(m <= a.orth_tol);  // NaN-safe
      if (a.stats) {
        const double sc = s_scale;
        a.stats[0] = (double)r;
        a.stats[1] = s_tmax * sc;
        a.stats[2] = 0.0;  // filled below if something was dropped
        a.stats[3] = s_bad ? 1.0 : 0.0;
        a.stats[4] = m;
      }
    }
    __syncthreads();
  }
  if (tid == 0 && a.stats && r < k && s_tmax > 0.0) a.stats[2] = fabs(lam[r]) / s_tmax;
  t_ph[6] = clock64();
  if (tid == 0 && a.stats)
    for (int i = 0; i < 6; ++i) a.stats[8 + i] = (double)(t_ph[i + 1] - t_ph[i]);
  if (s_bad) {
    if (tid == 0) *a.r_out = -1;  // caller falls back to the Jacobi kernel
    return;
  }
  if (a.t3 && r > 0) {
    __syncthreads();
    t3_fuse(a, k, r, A, Gam, Phi);
  }
  if (tid == 0) *a.r_out = r;
}

}  // namespace

size_t eig_fast_smem(int k) { return sizeof(double) * (size_t)k * (k | 1) + 64; }

void eig_fast(const SmallArgs& a, cudaStream_t st) {
  if (a.k > FAST_K_MAX || a.k < 1) throw std::runtime_error("eig_fast: k out of range");
  size_t smem = eig_fast_smem(a.k);
  if (smem < sizeof(double) * 2 * SMALL_K_MAX * SMALL_M_MAX) smem = sizeof(double) * 2 * SMALL_K_MAX * SMALL_M_MAX;
  static bool attr = false;
  if (!attr) {
    DME_CUDA(cudaFuncSetAttribute(eig_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)eig_fast_smem(FAST_K_MAX)));
    attr = true;
  }
  eig_fast_kernel<<<1, NT, smem, st>>>(a);
  DME_KCHECK();
}

}  // namespace dme
