// Device pieces shared by the one-CTA fast eigen kernel (eig_fast.cu) and the split eigen kernels
// (eig_split.cu): Sturm counts and the shared-memory Householder tridiagonalisation.
#pragma once
#include "common.cuh"
#include "small.h"
#include "small_common.cuh"

namespace dme {
namespace eigk {

constexpr int ENT = 512;  // threads of the eigen kernels (16 warps, up to 128 registers each)
constexpr int NW = ENT / 32;

// Exact power-of-two rescaling of a pair of consecutive minors to ~1 when they leave [2^-64, 2^64]
// (the ratios and signs the callers need are unchanged; a block of 8 recurrence steps then cannot
// overflow for ||T|| <= 1 nor underflow unless the pivots fall below ~2^-120 each)
__device__ __forceinline__ void rescale_pair(double& p1, double& p2) {
  const double m1 = fmax(fabs(p1), fabs(p2));
  if (m1 > 0x1p64 || (m1 < 0x1p-64 && m1 > 0.0)) {
    // exponent field of m1 (a subnormal m1 reads as 2^-1022: the product is then scaled up by 2^1022,
    // short of ~1 but normal); 2^-e built directly, e in [-1022, 1023]
    const int e = ((__double2hiint(m1) >> 20) & 0x7ff) - 1023;
    const int ec = e < -1022 ? -1022 : e;
    const double sc = __hiloint2double((1023 - ec) << 20, 0);
    p1 *= sc;
    p2 *= sc;
  }
}

// number of eigenvalues of T (d, e2 = e^2, normalised to ||T|| <= 1) smaller than x:
// sign changes of the leading principal minors p_i of T - xI (an exact zero counts as negative,
// a measure-zero event that only moves a bisection probe by one count)
__device__ __forceinline__ int sturm_count(const double* __restrict__ d,
                                           const double* __restrict__ e2, int k, double x) {
  // signs from the high word (INT pipe; the FP64 pipe is what many concurrent probes saturate);
  // an exact zero counts by its sign bit, a measure-zero event that moves a probe by one count
  double p2 = 1.0, p1 = d[0] - x;
  bool neg_prev = __double2hiint(p1) < 0;
  int cnt = neg_prev;
  int i = 1;
  // blocks of 8: the loads are independent of the recurrence and issue ahead of it; the exact
  // power-of-two rescaling to ~1 is checked once per block (|p| grows <= 3^8 per block for
  // ||T|| <= 1; a fixed 2^300 step could not keep up with strongly graded T, whose minors then
  // underflowed to zero and stopped counting)
  for (; i + 7 < k; i += 8) {
    double dd[8], ff[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      dd[u] = d[i + u] - x;
      ff[u] = e2[i - 1 + u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double p = fma(dd[u], p1, -ff[u] * p2);
      const bool ng = __double2hiint(p) < 0;
      cnt += ng != neg_prev;
      neg_prev = ng;
      p2 = p1;
      p1 = p;
    }
    rescale_pair(p1, p2);
  }
  for (; i < k; ++i) {
    const double p = fma(d[i] - x, p1, -e2[i - 1] * p2);
    const bool ng = __double2hiint(p) < 0;
    cnt += ng != neg_prev;
    neg_prev = ng;
    p2 = p1;
    p1 = p;
  }
  return cnt;
}

// 1/x to ~1 ulp without the IEEE division sequence: MUFU reciprocal seed + two Newton steps
// (callers guarantee a normal, finite, nonzero x)
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double t = fma(-x, r, 1.0);
  r = fma(r, t, r);
  t = fma(-x, r, 1.0);
  return fma(r, t, r);
}

// x / d for 0 <= x < 2^20, 0 < d < 2^12 without the integer-division sequence (float reciprocal
// estimate, corrected by one step either way)
__device__ __forceinline__ int udiv_small(int x, int d) {
  int q = __float2int_rz(__fmul_rz((float)x, __frcp_rn((float)d)));
  if ((q + 1) * d <= x) ++q;
  if (q * d > x) --q;
  return q;
}

// Pivots of the twisted factorisation of T - lm I (d, e2 = e^2 of the normalised T): forward
// (fwd: D+_i = p_i / p_{i-1}, p_i the leading principal minors) or backward (D-_i from the trailing
// minors). The minors follow the division-free three-term recurrence (one FMA per row on the
// dependency chain, rescaled per block of 8); the ratios are formed off the chain. Same pivots as
// the ratio recurrence D_i = (d_i - lm) - e2 / D_{i-1} up to rounding; |D_i| < pivmin (or a
// 0/0 ratio) becomes -pivmin as there.
__device__ inline void twisted_pivots(const double* __restrict__ d, const double* __restrict__ e2, int k,
                                      double lm, bool fwd, double* __restrict__ D) {
  constexpr double pivmin = 1e-290;
  auto row = [&](int t) { return fwd ? t : k - 1 - t; };
  auto cpl = [&](int t) { return fwd ? t - 1 : k - 1 - t; };  // e2 index coupling rows t-1, t
  auto clampd = [&](double x) { return fabs(x) >= pivmin ? x : -pivmin; };
  double p2 = 1.0, p1 = d[row(0)] - lm;
  D[row(0)] = clampd(p1);
  int t = 1;
  for (; t + 7 < k; t += 8) {
    double pb[8];
    const double prev = p1;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double p = fma(d[row(t + u)] - lm, p1, -e2[cpl(t + u)] * p2);
      p2 = p1;
      p1 = p;
      pb[u] = p;
    }
    D[row(t)] = clampd(pb[0] * frcp(prev));
#pragma unroll
    for (int u = 1; u < 8; ++u) D[row(t + u)] = clampd(pb[u] * frcp(pb[u - 1]));
    rescale_pair(p1, p2);
  }
  for (; t < k; ++t) {
    const double p = fma(d[row(t)] - lm, p1, -e2[cpl(t)] * p2);
    D[row(t)] = clampd(p * frcp(p1));
    p2 = p1;
    p1 = p;
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}


// Householder tridiagonalisation of the symmetric k x k matrix in A (row stride ld, shared
// memory), in place: d, e (unnormalised) and tau; reflector j kept in row j (v_0 = 1 implicit).
template <int FK, int NTH = ENT>
__device__ void tridiagonalise(double* A, int k, int ld, double* d, double* e, double* tau,
                               double* vec, double* pv, double* pv2, long long* ph = nullptr) {
#ifdef DME_TRI_PHASES  // measurement build only (tools/tri_phases.sh): per-phase cycle sums
  long long acc_a = 0, acc_w = 0, acc_bar = 0;
#endif
  constexpr int RCH = (FK + 31) / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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
      const double inv = 1.0 / (amb * beta);  // one division for both quotients
      scal = beta * inv;                      // 1 / (alpha - beta)
      t = -amb * amb * inv;                   // (beta - alpha) / beta
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
#ifdef DME_TRI_PHASES
    const long long t_a = clock64();
#endif
    const int m = k - j - 1;
    const double* vj = (j & 1) ? pv2 : vec;  // double-buffered reflector
    double* vn = (j & 1) ? vec : pv2;
    const double tj = tau[j];
    // p = tau A22 v by columns (A symmetric): thread i sums A[l][i] v_l over the trailing rows l
    if (tj != 0.0) {
      for (int i = tid; i < m; i += NTH) {
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
#ifdef DME_TRI_PHASES
    const long long t_b = clock64();
#endif
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
        const int t2 = tid - 32, nt2 = NTH - 32;
        const int rg = udiv_small(nt2, m);  // row groups
        const int grp = udiv_small(t2, m), l = t2 - grp * m;
        if (grp < rg) {
          const double vl = vj[l], wl = pv[l] - K * vl;
          double* col = A + (j + 1) * ld + (j + 1 + l);
          int i = 1 + grp;
          // four rows per round with the loads first (in-order issue: the stores then do not hold
          // back the next row's shared-memory loads)
          for (; i + 3 * rg < m; i += 4 * rg) {
            double av[4], vi[4], pi[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              vi[u] = vj[i + u * rg];
              pi[u] = pv[i + u * rg];
              av[u] = col[(i + u * rg) * ld];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double wi = pi[u] - K * vi[u];
              col[(i + u * rg) * ld] = av[u] - (vi[u] * wl + wi * vl);
            }
          }
          for (; i < m; i += rg) {
            const double vi = vj[i], wi = pv[i] - K * vi;
            col[i * ld] -= vi * wl + wi * vl;
          }
        }
      }
    } else if (warp == 0 && j + 3 < k) {
      householder(j + 1, vn);
    }
#ifdef DME_TRI_PHASES
    const long long t_c = clock64();
#endif
    __syncthreads();
#ifdef DME_TRI_PHASES
    acc_a += t_b - t_a;
    acc_w += t_c - t_b;
    acc_bar += clock64() - t_c;
#endif
  }
#ifdef DME_TRI_PHASES
  if (ph && tid == 0) { ph[0] = acc_a; ph[1] = acc_w; ph[2] = acc_bar; }
  if (ph && tid == 32) { ph[3] = acc_w; ph[4] = acc_bar; }
  if (ph && tid == 0 + 64) ph[5] = acc_w;
#endif
  if (tid == 0) {
    if (k >= 2) {
      d[k - 2] = A[(k - 2) * ld + (k - 2)];
      e[k - 2] = A[(k - 1) * ld + (k - 2)];
    }
    d[k - 1] = A[(k - 1) * ld + (k - 1)];
  }
  __syncthreads();
}

// Normalise T by a Gershgorin bound of ||T||; e2 = e^2; Gershgorin interval [lo, hi]. Thread 0.
__device__ inline void normalise_tridiagonal(int k, double* d, double* e, double* e2, double* scale,
                                             double* lo_out, double* hi_out) {
  double nrm = 0.0, lo = 1e300, hi = -1e300;
  for (int i = 0; i < k; ++i) {
    const double rr = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < k ? fabs(e[i]) : 0.0);
    nrm = fmax(nrm, fabs(d[i]) + rr);
  }
  if (!(nrm > 0.0)) nrm = 1.0;
  *scale = nrm;
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
  *lo_out = lo - 1e-14;
  *hi_out = hi + 1e-14;
}

}  // namespace eigk
}  // namespace dme
