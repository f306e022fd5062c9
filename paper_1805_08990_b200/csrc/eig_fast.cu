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

#include <cmath>

namespace dme {

namespace {

constexpr int ENT = 512;  // threads of the fast eigen kernel (16 warps, up to 128 registers each)
constexpr int NW = ENT / 32;

// number of eigenvalues of T (d, e2 = e^2, normalised to ||T|| <= 1) smaller than x
__device__ __forceinline__ int sturm_count(const double* __restrict__ d,
                                           const double* __restrict__ e2, int k, double x) {
  double p2 = 1.0, p1 = d[0] - x;
  int neg_prev = p1 <= 0.0;
  int cnt = neg_prev;
  int i = 1;
  for (; i + 3 < k; i += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double p = fma(d[i + u] - x, p1, -e2[i + u - 1] * p2);
      const long long b = __double_as_longlong(p);
      const int neg = (b < 0) | ((((unsigned long long)b << 1) == 0ull) & !neg_prev);
      cnt += neg ^ neg_prev;
      neg_prev = neg;
      p2 = p1;
      p1 = p;
    }
    const int ex1 = (int)((__double_as_longlong(p1) >> 52) & 0x7ff);
    const int ex2 = (int)((__double_as_longlong(p2) >> 52) & 0x7ff);
    if (ex1 > 1023 + 400 || ex2 > 1023 + 400) {
      p1 *= 0x1p-400;
      p2 *= 0x1p-400;
    } else if (ex1 < 1023 - 400 && ex2 < 1023 - 400) {
      p1 *= 0x1p400;
      p2 *= 0x1p400;
    }
  }
  for (; i < k; ++i) {
    const double p = fma(d[i] - x, p1, -e2[i - 1] * p2);
    const long long b = __double_as_longlong(p);
    const int neg = (b < 0) | ((((unsigned long long)b << 1) == 0ull) & !neg_prev);
    cnt += neg ^ neg_prev;
    neg_prev = neg;
    p2 = p1;
    p1 = p;
  }
  return cnt;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int FK>
__global__ void __launch_bounds__(ENT, 1) eig_fast_kernel(SmallArgs a) {
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
  // Step j: reflector H_j = I - tau_j v v^T built from ROW j (= column j, symmetric storage) and
  // stored back into row j (v_0 = 1 implicit). Two barriers per step: [mat-vec by columns] |
  // [rank-2 update; warp 0 updates row j+1 first and builds the next reflector from it (look-ahead)].
  auto householder = [&](int j, double* vv) {  // warp 0 only
    const int m = k - j - 1;
    double xs[RCH];
    double xn2 = 0.0;
#pragma unroll
    for (int u = 0; u < RCH; ++u) {
      const int i = lane + 32 * u;
      xs[u] = i < m ? A[j * ld + j + 1 + i] : 0.0;
      if (i >= 1) xn2 = fma(xs[u], xs[u], xn2);
    }
    xn2 = warp_sum(xn2);
    const double alpha = __shfl_sync(0xffffffffu, xs[0], 0);
    double t = 0.0, beta = alpha, scal = 0.0;
    if (xn2 > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
      const double amb = alpha - beta;
      scal = 1.0 / amb;
      t = -amb / beta;  // (beta - alpha) / beta
    }
#pragma unroll
    for (int u = 0; u < RCH; ++u) {
      const int i = lane + 32 * u;
      if (i < m) {
        const double v = (i == 0) ? 1.0 : (t == 0.0 ? 0.0 : xs[u] * scal);
        vv[i] = v;
        if (i > 0) A[j * ld + j + 1 + i] = v;  // reflector kept in row j
      }
    }
    if (lane == 0) {
      tau[j] = t;
      e[j] = beta;
      d[j] = A[j * ld + j];
    }
  };
  if (k > 2 && warp == 0) householder(0, vec);
  __syncthreads();
  for (int j = 0; j + 2 < k; ++j) {
    const int m = k - j - 1;
    const double* vj = (j & 1) ? pv2 : vec;  // double-buffered reflector
    double* vn = (j & 1) ? vec : pv2;
    const double tj = tau[j];
    // p = tau A22 v by columns (A symmetric): thread i sums A[l][i] v_l over the trailing rows l
    if (tj != 0.0) {
      for (int i = tid; i < m; i += ENT) {
        const double* col = A + (j + 1) * ld + (j + 1 + i);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int l = 0;
        for (; l + 3 < m; l += 4) {
          s0 = fma(col[(l + 0) * ld], vj[l + 0], s0);
          s1 = fma(col[(l + 1) * ld], vj[l + 1], s1);
          s2 = fma(col[(l + 2) * ld], vj[l + 2], s2);
          s3 = fma(col[(l + 3) * ld], vj[l + 3], s3);
        }
        for (; l < m; ++l) s0 = fma(col[l * ld], vj[l], s0);
        pv[i] = tj * ((s0 + s1) + (s2 + s3));
      }
    }
    __syncthreads();
    if (tj != 0.0) {
      // K = tau/2 p^T v (every warp, redundantly), w = p - K v
      double dot = 0.0;
#pragma unroll
      for (int u = 0; u < RCH; ++u) {
        const int l = lane + 32 * u;
        if (l < m) dot = fma(pv[l], vj[l], dot);
      }
      const double K = 0.5 * tj * warp_sum(dot);
      if (warp == 0) {
        // row j+1 (trailing row 0) first, then the next reflector from it
        const double v0 = vj[0], w0 = pv[0] - K * v0;
#pragma unroll
        for (int u = 0; u < RCH; ++u) {
          const int l = lane + 32 * u;
          if (l < m) A[(j + 1) * ld + j + 1 + l] -= v0 * (pv[l] - K * vj[l]) + w0 * vj[l];
        }
        __syncwarp();
        if (j + 3 < k) householder(j + 1, vn);
      } else {
        // rows 1..m-1 of the trailing block by the other warps: thread per column l, rows strided
        const int t2 = tid - 32, nt2 = ENT - 32;
        const int rg = nt2 / m;  // row groups
        const int l = t2 % m, grp = t2 / m;
        if (grp < rg) {
          const double vl = vj[l], wl = pv[l] - K * vl;
          for (int i = 1 + grp; i < m; i += rg) {
            const double vi = vj[i], wi = pv[i] - K * vi;
            double* a_ = A + (j + 1 + i) * ld + (j + 1 + l);
            *a_ -= vi * wl + wi * vl;
          }
        }
      }
    } else if (warp == 0 && j + 3 < k) {
      householder(j + 1, vn);
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
      const double rr = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < k ? fabs(e[i]) : 0.0);
      nrm = fmax(nrm, fabs(d[i]) + rr);
    }
    if (!(nrm > 0.0)) nrm = 1.0;
    s_scale = nrm;
    const double inv = 1.0 / nrm;
    for (int i = 0; i < k; ++i) {
      d[i] *= inv;
      if (i + 1 < k) {
        e[i] *= inv;
        e2[i] = e[i] * e[i];
      }
    }
    for (int i = 0; i < k; ++i) {
      const double rr = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < k ? fabs(e[i]) : 0.0);
      lo = fmin(lo, d[i] - rr);
      hi = fmax(hi, d[i] + rr);
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
    if (tmax > 0.0) r = k - sturm_count(d, e2, k, a.tol * tmax);
    if (r > a.cap) r = a.cap;
    if (r < 0) r = 0;
    s_r = r;
  }
  __syncthreads();
  const int r = s_r;
  const int nr = r < k ? r + 1 : r;  // + the first dropped one, for the stats
  {
    int P = nr > 0 ? 200 / nr : 1;
    P = P < 1 ? 1 : (P > 16 ? 16 : P);
    const int grp = tid / P, t = tid % P;
    const bool act = grp < nr;
    const int jj = k - 1 - grp;
    if (act && t == 0) {
      lo_s[grp] = s_lo;
      hi_s[grp] = s_hi;
    }
    __syncthreads();
    const double bits = log2((double)P + 1.0);
    // absolute accuracy 1e-13 ||T||: enough for the twisted vectors (their error ~ |dlambda| / gap
    // only matters weighted by theta)
    const int nit = (int)ceil(log2((s_hi - s_lo) / 1e-13 + 1.0) / bits) + 1;
    for (int it = 0; it < nit; ++it) {
      if (act) {
        const double a0 = lo_s[grp], b0 = hi_s[grp];
        cnt_s[tid] = sturm_count(d, e2, k, a0 + (b0 - a0) * (t + 1) / (P + 1.0));
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
    const double pivmin = 1e-290;
    if (side == 0) {
      double x = d[0] - lm;
      if (fabs(x) < pivmin) x = -pivmin;
      Dp[0] = x;
      for (int i = 1; i < k; ++i) {
        x = (d[i] - lm) - e2[i - 1] / x;
        if (fabs(x) < pivmin) x = -pivmin;
        Dp[i] = x;
      }
    } else {
      double x = d[k - 1] - lm;
      if (fabs(x) < pivmin) x = -pivmin;
      Dm[k - 1] = x;
      for (int i = k - 2; i >= 0; --i) {
        x = (d[i] - lm) - e2[i] / x;
        if (fabs(x) < pivmin) x = -pivmin;
        Dm[i] = x;
      }
    }
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

  // ---------------------------------------------------------------- 4. W = Q Z (warp-owned columns)
  {
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
          double s[CP];
#pragma unroll
          for (int cc = 0; cc < CP; ++cc) {
            s[cc] = 0.0;
#pragma unroll
            for (int u = 0; u < RCH; ++u) s[cc] = fma(vr[u], z[cc][u], s[cc]);
          }
#pragma unroll
          for (int o = 16; o; o >>= 1)
#pragma unroll
            for (int cc = 0; cc < CP; ++cc) s[cc] += __shfl_xor_sync(0xffffffffu, s[cc], o);
#pragma unroll
          for (int cc = 0; cc < CP; ++cc) {
            const double f = tj * s[cc];
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
    __syncthreads();  // all reflector reads from A done before A is reused
    // W^T (row-major) into shared memory for the check (unscaled)
    for (int e_ = tid; e_ < k * r; e_ += ENT) {
      const int i = e_ % k, c = e_ / k;
      const double f = a.sqrt_scale ? sqrt(fmax(lam[c] * sc, 0.0)) : 1.0;
      A[c * ld + i] = f > 0.0 ? a.Tm[i + (size_t)c * a.ldt] / f : 0.0;
    }
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
    if (tid == 0) *a.r_out = -1;  // caller falls back to the Jacobi kernel
    return;
  }
  if (a.t3 && r > 0) {
    __syncthreads();
    smallk::t3_fuse(a, k, r, A, Gam, Phi);
  }
  if (tid == 0) *a.r_out = r;
}

template <int FK>
void launch_fast(const SmallArgs& a, cudaStream_t st) {
  const size_t floor_b = sizeof(double) * 2 * SMALL_K_MAX * SMALL_M_MAX;
  const size_t need = sizeof(double) * (size_t)FK * (FK | 1);
  size_t smem = sizeof(double) * (size_t)a.k * (a.k | 1);
  if (smem < floor_b) smem = floor_b;
  static bool attr = false;
  if (!attr) {
    DME_CUDA(cudaFuncSetAttribute(eig_fast_kernel<FK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(need > floor_b ? need : floor_b)));
    attr = true;
  }
  eig_fast_kernel<FK><<<1, ENT, smem, st>>>(a);
  DME_KCHECK();
}

}  // namespace

void eig_fast(const SmallArgs& a, cudaStream_t st) {
  if (a.k > FAST_K_MAX || a.k < 1) throw std::runtime_error("eig_fast: k out of range");
  if (a.k <= 96) launch_fast<96>(a, st);
  else launch_fast<FAST_K_MAX>(a, st);
}

}  // namespace dme
