// Split eigen-compression for the hot path (k = r + q_I >= EIG_SPLIT_MIN): the same mathematics as
// eig_fast.cu (G = W Theta W^T, Tm = W_kept, weighted orthogonality check, fused T3) spread over
// three launches so the parallel part does not run on a single SM:
//   TRI (1 CTA)       Householder tridiagonalisation, normalisation, theta_max and the rank r
//                     (Sturm counts); T and the reflectors go to the global scratch Es.
//   VEC (EIG_SPLIT_CTAS CTAs)  each CTA owns a contiguous slice of the kept eigenvalues (+ the first
//                     dropped one, for the stats): multisection with up to 512 probes per eigenvalue,
//                     twisted-factorisation vectors (lane pairs), back-transformation by the
//                     reflectors (one warp per column, column in registers), Tm columns written.
//   FIN (1 CTA)       weighted orthogonality check (fallback flag), stats, fused Riccati flow T3.
// The look-ahead E pass of the step runs on #SM - EIG_SPLIT_CTAS persistent CTAs meanwhile.
#include "common.cuh"
#include "eig_common.cuh"
#include "small.h"
#include "small_common.cuh"

#include <cmath>
#include <cstdlib>

namespace dme {

namespace {

using namespace eigk;


// NTH threads (512; DME_TRI_THREADS = 256 or 128 for k <= 96: A/B of the per-step latency)
template <int FK, int NTH>
__global__ void __launch_bounds__(NTH, 1) eig_tri_kernel(SmallArgs a) {
  pdl_wait();
  constexpr int NWT = NTH / 32;
  extern __shared__ double A[];
  __shared__ double d[FK], e[FK], e2[FK], tau[FK], vec[FK], pv[FK], pv2[FK];
  __shared__ int cnt_s[256];
  __shared__ double s_scale, s_lo, s_hi, s_lo_t, s_hi_t;
  const int tid = threadIdx.x;
  const int k = a.k, ld = k | 1;
  const EsLayout es{a.Es, SMALL_K_MAX};
  const long long t_in = clock64();
  {
    // column j of G into row j of A (coalesced, 8 loads in flight per thread), then the exact
    // symmetrisation A = (G + G^T) / 2 in shared memory
    constexpr int B = 8;
    for (int e0 = tid; e0 < k * k; e0 += B * NTH) {
      double v[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int e_ = e0 + u * NTH;
        v[u] = e_ < k * k ? a.G[(e_ % k) + (size_t)(e_ / k) * a.ldg] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int e_ = e0 + u * NTH;
        if (e_ < k * k) A[(e_ / k) * ld + (e_ % k)] = v[u];
      }
    }
    __syncthreads();
    for (int e_ = tid; e_ < k * k; e_ += NTH) {
      const int i = e_ % k, j = e_ / k;
      if (i < j) {
        const double v = 0.5 * (A[i * ld + j] + A[j * ld + i]);
        A[i * ld + j] = v;
        A[j * ld + i] = v;
      }
    }
  }
  __syncthreads();
  const long long t0 = clock64();
  __shared__ long long tph[8];
  tridiagonalise<FK, NTH>(A, k, ld, d, e, tau, vec, pv, pv2, tph);
  const long long t1 = clock64();
  pdl_trigger();  // VEC may be scheduled now (it waits for this grid in pdl_wait)
  {
    // normalise T by a Gershgorin bound of ||T|| (same arithmetic as normalise_tridiagonal, in
    // parallel: one row per thread, block max/min reductions)
    __shared__ double rmax[NWT], rlo[NWT], rhi[NWT];
    const int lane = tid & 31, warp = tid >> 5;
    double rr = 0.0, di = 0.0;
    if (tid < k) {
      di = d[tid];
      rr = (tid > 0 ? fabs(e[tid - 1]) : 0.0) + (tid + 1 < k ? fabs(e[tid]) : 0.0);
    }
    double m = tid < k ? fabs(di) + rr : 0.0;
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) rmax[warp] = m;
    __syncthreads();
    double nrm = 0.0;
    for (int w = 0; w < NWT; ++w) nrm = fmax(nrm, rmax[w]);
    if (!(nrm > 0.0)) nrm = 1.0;
    const double inv = 1.0 / nrm;
    __syncthreads();  // every thread has read the old d, e
    if (tid < k) {
      d[tid] = di * inv;
      if (tid + 1 < k) {
        const double en = e[tid] * inv;
        e[tid] = en;
        e2[tid] = en * en;
      }
    }
    __syncthreads();
    double lo = 1e300, hi = -1e300;
    if (tid < k) {
      const double r2 = (tid > 0 ? fabs(e[tid - 1]) : 0.0) + (tid + 1 < k ? fabs(e[tid]) : 0.0);
      lo = d[tid] - r2;
      hi = d[tid] + r2;
    }
    for (int o = 16; o; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) { rlo[warp] = lo; rhi[warp] = hi; }
    __syncthreads();
    if (tid == 0) {
      double l2 = 1e300, h2 = -1e300;
      for (int w = 0; w < NWT; ++w) { l2 = fmin(l2, rlo[w]); h2 = fmax(h2, rhi[w]); }
      s_scale = nrm;
      s_lo = l2 - 1e-14;
      s_hi = h2 + 1e-14;
      s_lo_t = s_lo;
      s_hi_t = s_hi;
    }
  }
  __syncthreads();
  // theta_max to 16 bits (enough for the threshold; it is refined with the others in VEC)
  constexpr int PB = NTH < 256 ? NTH : 256;
  for (int it = 0; it < 2; ++it) {
    const double a0 = s_lo_t, b0 = s_hi_t;
    if (tid < PB) cnt_s[tid] = sturm_count(d, e2, k, a0 + (b0 - a0) * (tid + 1) / (PB + 1.0));
    __syncthreads();
    if (tid < PB) {
      const bool le = cnt_s[tid] <= k - 1;
      const bool nxt = (tid + 1 < PB) ? (cnt_s[tid + 1] <= k - 1) : false;
      if (le && !nxt) {
        s_lo_t = a0 + (b0 - a0) * (tid + 1) / (PB + 1.0);
        if (tid + 1 < PB) s_hi_t = a0 + (b0 - a0) * (tid + 2) / (PB + 1.0);
      }
      if (tid == 0 && !le) s_hi_t = a0 + (b0 - a0) / (PB + 1.0);
    }
    __syncthreads();
  }
  if (tid == 0) {
    double tmax = 0.5 * (s_lo_t + s_hi_t);
    if (a.ref_max > 0.0) tmax = a.ref_max / s_scale;  // threshold and stats against the reference
    int r = 0;
    if (tmax > 0.0) r = k - sturm_count(d, e2, k, a.tol * tmax);
    if (r > a.cap) r = a.cap;
    if (r < 0) r = 0;
    double* h = es.hdr();
    h[0] = s_scale;
    h[1] = s_lo;
    h[2] = s_hi;
    h[3] = tmax;
    h[4] = (double)r;
    if (a.stats) {  // phase cycles (tools/eig_split_probe.py)
      a.stats[6] = (double)(t0 - t_in);
      a.stats[8] = (double)(t1 - t0);
      a.stats[9] = (double)(clock64() - t1);
#ifdef DME_TRI_PHASES  // (measurement build) phase sums over the reflector steps
      for (int q = 0; q < 6; ++q) a.stats[10 + q] = (double)tph[q];
      a.stats[7] = (double)k;
#endif
    }
  }
  for (int i = tid; i < k; i += NTH) {
    es.d()[i] = d[i];
    es.e()[i] = e[i];
    es.e2()[i] = e2[i];
    es.tau()[i] = tau[i];
  }
  double* R = es.refl();
  for (int e_ = tid; e_ < k * ld; e_ += NTH) R[e_] = A[e_];
  if (a.stats) {  // whole-kernel cycles (entry to last store issued)
    __syncthreads();
    if (tid == 0) a.stats[7] = (double)(clock64() - t_in);
  }
}

template <int FK>
__global__ void __launch_bounds__(ENT, 1) eig_vec_kernel(SmallArgs a) {
  pdl_wait();
  constexpr int RCH = (FK + 31) / 32;
  constexpr int MAXE = (FK + 1 + EIG_SPLIT_CTAS - 1) / EIG_SPLIT_CTAS + 1;
  extern __shared__ double R[];  // reflectors, k x ld
  __shared__ double d[FK], e[FK], e2[FK], tau[FK];
  __shared__ double lo_s[MAXE], hi_s[MAXE], lam_s[MAXE];
  __shared__ double cpair[(FK / 4 + 1) * 6];  // per block of 4 reflectors: v_p^T v_q
  __shared__ int cnt_s[ENT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = a.k, ld = k | 1;
  const EsLayout es{a.Es, SMALL_K_MAX};
  long long t_ph[5];
  t_ph[0] = clock64();
  const double* h = es.hdr();
  const int r = (int)h[4];
  const int nr = r < k ? r + 1 : r;
  const int c0 = (int)((long long)blockIdx.x * nr / gridDim.x);
  const int c1 = (int)((long long)(blockIdx.x + 1) * nr / gridDim.x);
  const int nb = c1 - c0;
  if (nb <= 0) return;
  const double scale = h[0], glo = h[1], ghi = h[2];
  // the reflectors (k x ld doubles, contiguous) by one bulk async copy (rounded up to 16 bytes: the
  // scratch and the shared buffer both have room), the tridiagonal by the threads meanwhile
  __shared__ uint64_t rbar;
  const uint32_t rbytes = ((uint32_t)(k * ld) * 8u + 15u) & ~15u;
  if (tid == 0) {
    mbar_init(&rbar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&rbar, rbytes);
    for (uint32_t off = 0; off < rbytes; off += 32768u)
      bulk_load(reinterpret_cast<char*>(R) + off, reinterpret_cast<const char*>(es.refl()) + off,
                rbytes - off < 32768u ? rbytes - off : 32768u, &rbar);
  }
  for (int i = tid; i < k; i += ENT) {
    d[i] = es.d()[i];
    e[i] = es.e()[i];
    e2[i] = es.e2()[i];
    tau[i] = es.tau()[i];
  }
  __syncthreads();  // the barrier is initialised before anyone waits on it
  mbar_wait(&rbar, 0);

  // ------------------------------------------------------------ multisection on this slice
  t_ph[1] = clock64();
  {
    // one Sturm count per thread and round: with few eigenvalues per CTA (the tail pass of the
    // refined compression) up to 512 probes per eigenvalue cut the rounds from ~11 to ~6
    // probes per eigenvalue: more probes mean fewer rounds but, past ~4 warps, a round is bound by
    // the FP64 pipe of the SM rather than by one count's dependency chain (DME_MSEC_P: A/B knob)
    int P = ENT / nb;
    P = P < 1 ? 1 : (P > a.msec_p ? a.msec_p : P);
    const int grp = tid / P, t = tid % P;
    const bool act = grp < nb;
    const int jj = k - 1 - (c0 + grp);  // ascending index
    if (act && t == 0) {
      lo_s[grp] = glo;
      hi_s[grp] = ghi;
    }
    __syncthreads();
    const float bits = __log2f((float)P + 1.0f);  // (fast float math: only sizes the loop)
    const int nit = (int)ceilf(1.00001f * __log2f((float)((ghi - glo) / 1e-13) + 1.0f) / bits) + 1;
    for (int it = 0; it < nit; ++it) {
      if (act) {
        const double a0 = lo_s[grp], b0 = hi_s[grp];
        cnt_s[tid] = sturm_count(d, e2, k, a0 + (b0 - a0) * (t + 1) / (P + 1.0));
      }
      __syncthreads();
      double a0 = 0.0, b0 = 0.0;
      if (act) { a0 = lo_s[grp]; b0 = hi_s[grp]; }
      __syncthreads();  // every thread has read the bracket before the transition thread moves it
      if (act) {
        // transition between probe t and t+1 (counts are monotone in the probe position)
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
      lam_s[grp] = 0.5 * (lo_s[grp] + hi_s[grp]);
      es.lam()[c0 + grp] = lam_s[grp];
    }
    __syncthreads();
  }

  // ------------------------------------------------------------ twisted-factorisation vectors
  t_ph[2] = clock64();
  const int cv1 = c1 < r ? c1 : r;  // vectors only for kept eigenvalues
  const int nv = cv1 - c0;
  if (tid < 2 * nv) {
    const unsigned msk = __activemask();
    const int c = c0 + (tid >> 1), side = tid & 1;
    const double lm = lam_s[tid >> 1];
    // FK <= 96: the twisted-factorisation arrays live in shared memory behind the reflectors
    double* Dp = FK <= 96 ? R + k * ld + (tid >> 1) * FK : es.dp() + (size_t)c * SMALL_K_MAX;
    double* Dm = FK <= 96 ? R + k * ld + (MAXE + (tid >> 1)) * FK : es.dm() + (size_t)c * SMALL_K_MAX;
    twisted_pivots(d, e2, k, lm, side == 0, side == 0 ? Dp : Dm);
    __syncwarp(msk);
    __threadfence_block();
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
    double nrm2 = 0.0;
    if (side == 0) {
      for (int i = 0; i < tw; ++i) Dp[i] = -e[i] * frcp(Dp[i]);
      double zi = 1.0;
      for (int i = tw - 1; i >= 0; --i) {
        zi *= Dp[i];
        nrm2 = fma(zi, zi, nrm2);
        Dp[i] = zi;
      }
    } else {
      for (int i = tw + 1; i < k; ++i) Dm[i] = -e[i - 1] * frcp(Dm[i]);
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

  pdl_trigger();
  // ------------------------------------------------------------ W = Q Z, one warp per column
  // Reflectors are applied four at a time (H_j0 H_j1 H_j2 H_j3 with j0 = j3 + 3 applied first):
  // the four dots v_jm^T z share one warp reduction and the coupling v_p^T v_q of the block
  // (precomputed below) turns them into the four coefficients by a 4-term recurrence:
  //   s_m = tau_jm (a_m - sum_{m' < m} (v_jm^T v_jm') s_m')
  t_ph[3] = clock64();
  const int nb4 = (k - 2 + 3) / 4;  // reflectors 0 .. k-3
  for (int e = tid; e < nb4 * 6; e += ENT) {
    const int b = e / 6, pr = e % 6;
    const int jt = k - 3 - 4 * b;
    // pr -> (ma, mb): (0,1) (0,2) (1,2) (0,3) (1,3) (2,3)
    const int mb = pr < 1 ? 1 : (pr < 3 ? 2 : 3), ma = pr - mb * (mb - 1) / 2;
    const int q = jt - ma, p = jt - mb;  // p < q: v_p^T v_q
    double sum = 0.0;
    if (p >= 0) {
      sum = R[p * ld + q + 1];  // v_q[q+1] = 1
      for (int i = q + 2; i < k; ++i) sum = fma(R[p * ld + i], R[q * ld + i], sum);
    }
    cpair[e] = sum;
  }
  __syncthreads();
  for (int cc = warp; cc < nv; cc += NW) {
    const int c = c0 + cc;
    const double* zsrc = FK <= 96 ? R + k * ld + cc * FK : es.dp() + (size_t)c * SMALL_K_MAX;
    double z[RCH];
#pragma unroll
    for (int u = 0; u < RCH; ++u) {
      const int i = lane + 32 * u;
      z[u] = i < k ? zsrc[i] : 0.0;
    }
    for (int b = 0; b < nb4; ++b) {
      const int jt = k - 3 - 4 * b;
      double vr[4][RCH], am[4];
#pragma unroll
      for (int mm = 0; mm < 4; ++mm) {
        const int j = jt - mm;
        double sv = 0.0;
#pragma unroll
        for (int u = 0; u < RCH; ++u) {
          const int i = lane + 32 * u;
          vr[mm][u] = j < 0 ? 0.0 : ((i == j + 1) ? 1.0 : ((i > j + 1 && i < k) ? R[j * ld + i] : 0.0));
          sv = fma(vr[mm][u], z[u], sv);
        }
        am[mm] = sv;
      }
      {  // transposed butterfly: 4 warp sums with 10 double shuffles instead of 20
        const bool b4 = lane & 16, b3 = lane & 8;
        double k0 = b4 ? am[2] : am[0], k1 = b4 ? am[3] : am[1];
        const double s0 = b4 ? am[0] : am[2], s1 = b4 ? am[1] : am[3];
        k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
        k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
        double kk = b3 ? k1 : k0;
        kk += __shfl_xor_sync(0xffffffffu, b3 ? k0 : k1, 8);
        kk += __shfl_xor_sync(0xffffffffu, kk, 4);
        kk += __shfl_xor_sync(0xffffffffu, kk, 2);
        kk += __shfl_xor_sync(0xffffffffu, kk, 1);
#pragma unroll
        for (int mm = 0; mm < 4; ++mm) am[mm] = __shfl_sync(0xffffffffu, kk, (mm >> 1) * 16 + (mm & 1) * 8);
      }
      const double* cp = cpair + b * 6;
      const double t0 = tau[jt], t1 = jt >= 1 ? tau[jt - 1] : 0.0;
      const double t2 = jt >= 2 ? tau[jt - 2] : 0.0, t3 = jt >= 3 ? tau[jt - 3] : 0.0;
      const double s0 = t0 * am[0];
      const double s1 = t1 * fma(-cp[0], s0, am[1]);
      const double s2 = t2 * fma(-cp[2], s1, fma(-cp[1], s0, am[2]));
      const double s3 = t3 * fma(-cp[5], s2, fma(-cp[4], s1, fma(-cp[3], s0, am[3])));
#pragma unroll
      for (int u = 0; u < RCH; ++u)
        z[u] = fma(-s3, vr[3][u], fma(-s2, vr[2][u], fma(-s1, vr[1][u], fma(-s0, vr[0][u], z[u]))));
    }
    const double f = a.sqrt_scale ? sqrt(fmax(lam_s[cc] * scale, 0.0)) : 1.0;
#pragma unroll
    for (int u = 0; u < RCH; ++u) {
      const int i = lane + 32 * u;
      if (i < k) a.Tm[i + (size_t)c * a.ldt] = z[u] * f;
    }
  }
  __syncthreads();
  t_ph[4] = clock64();
#ifndef DME_TRI_PHASES
  if (blockIdx.x == 0 && tid == 0 && a.stats)  // phase cycles (tools/eig_split_probe.py)
    for (int q = 0; q < 4; ++q) a.stats[10 + q] = (double)(t_ph[q + 1] - t_ph[q]);
#endif
}

template <int FK>
__global__ void __launch_bounds__(ENT, 1) eig_fin_kernel(SmallArgs a) {
  pdl_wait();
  extern __shared__ double A[];  // W^T, r x ld
  __shared__ double lam[FK + 1], slam[FK + 1];
  __shared__ double red[NW];
  __shared__ int s_bad;
  __shared__ double Gam[SMALL_M_MAX * SMALL_M_MAX];
  __shared__ double Phi[SMALL_M_MAX * SMALL_M_MAX];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = a.k, ld = k | 1;
  const EsLayout es{a.Es, SMALL_K_MAX};
  const double* h = es.hdr();
  const double scale = h[0], tmax = h[3];
  const int r = (int)h[4];
  const int nr = r < k ? r + 1 : r;
  const long long f0 = clock64();
  for (int i = tid; i < nr; i += ENT) {
    lam[i] = es.lam()[i];
    slam[i] = sqrt(fabs(lam[i]));
  }
  __syncthreads();
  if (a.sqrt_scale) {
    for (int e_ = tid; e_ < k * r; e_ += ENT) {
      const int i = e_ % k, c = e_ / k;
      const double f = sqrt(fmax(lam[c] * scale, 0.0));
      A[c * ld + i] = f > 0.0 ? a.Tm[i + (size_t)c * a.ldt] / f : 0.0;
    }
  } else {  // W = Tm as written by VEC
    for (int e_ = tid; e_ < k * r; e_ += ENT) {
      const int i = e_ % k, c = e_ / k;
      A[c * ld + i] = a.Tm[i + (size_t)c * a.ldt];
    }
  }
  __syncthreads();
  const long long f1 = clock64();
  // weighted orthogonality |W^T W - I| (4 x 4 blocks of the upper triangle; the k-long dots are
  // split over KS lanes of a warp and combined by shuffles, so ~all 512 threads work)
  constexpr int TB = 4, KS = 4;
  const int nbk = (r + TB - 1) / TB;
  double mx = 0.0;
  const int nblk = nbk * (nbk + 1) / 2;
  for (int base = warp * (32 / KS); base < nblk; base += NW * (32 / KS)) {
    const int blk = base + lane / KS, ks = lane % KS;
    int bi = 0, bj = 0;
    if (blk < nblk) {  // blk -> (bi <= bj): row-major enumeration of the upper triangle
      int rem = blk;
      while (rem >= nbk - bi) { rem -= nbk - bi; ++bi; }
      bj = bi + rem;
    }
    double acc[TB][TB];
#pragma unroll
    for (int x = 0; x < TB; ++x)
#pragma unroll
      for (int y = 0; y < TB; ++y) acc[x][y] = 0.0;
    if (blk < nblk) {
      for (int i = ks; i < k; i += KS) {
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
    }
#pragma unroll
    for (int x = 0; x < TB; ++x)
#pragma unroll
      for (int y = 0; y < TB; ++y) {
#pragma unroll
        for (int o = 1; o < KS; o <<= 1) acc[x][y] += __shfl_xor_sync(0xffffffffu, acc[x][y], o);
        const int c1 = bi * TB + x, c2 = bj * TB + y;
        if (blk < nblk && ks == 0 && c1 < r && c2 < r && c1 <= c2) {
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
    s_bad = !(m <= a.orth_tol);
    if (a.stats) {
      a.stats[0] = (double)r;
      a.stats[1] = tmax * scale;
      a.stats[2] = (r < k && tmax > 0.0) ? fabs(lam[r]) / tmax : 0.0;
      a.stats[3] = s_bad ? 1.0 : 0.0;
      a.stats[4] = m;
    }
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) publish_rank(a, -1);  // caller falls back to the Jacobi kernel
    return;
  }
  pdl_trigger();
  const long long f2 = clock64();
  if (a.t3 && r > 0) {
    if constexpr (FK <= 96) {
      // Riccati flow T3 on the compression output from shared memory (the generic t3_fuse reads
      // Tm and H from global memory in k-long dependent loops): Tm = W (f = 1 unless
      // sqrt_scale), K^{-1/2} = I + F g(F^T F) F^T, F = sqrt(tau) Tm^T H L_R^{-T}  (small.cu)
      const int m = a.m;
      double* Hs = A + (size_t)r * ld;        // k x m
      double* Fs = Hs + (size_t)k * m;        // r x m
      double* Us = Fs + (size_t)r * m;        // k x m
      for (int e = tid; e < k * m; e += ENT) Hs[e] = a.H[(e % k) + (size_t)(e / k) * a.ldh];
      for (int i = tid; i < r; i += ENT)
        slam[i] = a.sqrt_scale ? sqrt(fmax(lam[i] * scale, 0.0)) : 1.0;
      __syncthreads();
      for (int e = tid; e < r * m; e += ENT) {  // Us[c, mu] <- (Tm^T H)[c, mu] (temporary)
        const int c = e % r, mu = e / r;
        const double* w = A + (size_t)c * ld;
        const double* hh = Hs + (size_t)mu * k;
        double s0 = 0.0, s1 = 0.0;
        int i = 0;
        for (; i + 1 < k; i += 2) { s0 = fma(w[i], hh[i], s0); s1 = fma(w[i + 1], hh[i + 1], s1); }
        if (i < k) s0 = fma(w[i], hh[i], s0);
        Us[c + (size_t)mu * r] = (s0 + s1) * slam[c];
      }
      __syncthreads();
      for (int e = tid; e < r * m; e += ENT) {  // F = sqrt(tau) W Linv^T
        const int c = e % r, mu = e / r;
        double acc = 0.0;
        for (int nu = 0; nu < m; ++nu) acc += Us[c + (size_t)nu * r] * a.LRinv[mu * m + nu];
        Fs[c + (size_t)mu * r] = sqrt(a.tau) * acc;
      }
      __syncthreads();
      if (tid < m * m) {  // Phi = F^T F
        const int mu = tid / m, nu = tid % m;
        double acc = 0.0;
        for (int c = 0; c < r; ++c) acc += Fs[c + (size_t)mu * r] * Fs[c + (size_t)nu * r];
        Phi[mu * m + nu] = acc;
      }
      __syncthreads();
      if (tid == 0) {  // Gamma = g(Phi)
        if (m == 1) {
          const double sg = sqrt(1.0 + fmax(Phi[0], 0.0));
          Gam[0] = -1.0 / (sg * (1.0 + sg));
        } else {
          smallk::tiny_sym_fun_g(Phi, Gam, m);
        }
      }
      __syncthreads();
      for (int e = tid; e < k * m; e += ENT) {  // U = Tm F Gamma  (k x m)
        const int i = e % k, mu = e / k;
        double u[SMALL_M_MAX];
        for (int nu = 0; nu < m; ++nu) u[nu] = 0.0;
        for (int c = 0; c < r; ++c) {
          const double t = A[(size_t)c * ld + i] * slam[c];
          for (int nu = 0; nu < m; ++nu) u[nu] = fma(t, Fs[c + (size_t)nu * r], u[nu]);
        }
        double acc = 0.0;
        for (int nu = 0; nu < m; ++nu) acc += u[nu] * Gam[nu * m + mu];
        Us[i + (size_t)mu * k] = acc;
      }
      __syncthreads();
      for (int e = tid; e < k * r; e += ENT) {  // Tm += U F^T
        const int i = e % k, c = e / k;
        double acc = A[(size_t)c * ld + i] * slam[c];
        for (int mu = 0; mu < m; ++mu) acc = fma(Us[i + (size_t)mu * k], Fs[c + (size_t)mu * r], acc);
        a.Tm[i + (size_t)c * a.ldt] = acc;
      }
    } else {
      smallk::t3_fuse(a, k, r, A, Gam, Phi);
    }
  }
  if (tid == 0) {
    publish_rank(a, r);
    if (a.stats) {  // phase cycles (tools/eig_split_probe.py)
#ifndef DME_TRI_PHASES
      a.stats[14] = (double)(f1 - f0);
      a.stats[15] = (double)(f2 - f1);
#endif
      a.stats[5] = (double)(clock64() - f2);
    }
  }
}

template <int FK>
void launch_split(const SmallArgs& a, cudaStream_t st) {
  const size_t floor_b = sizeof(double) * 2 * SMALL_K_MAX * SMALL_M_MAX;
  const size_t need_max = sizeof(double) * (size_t)FK * (FK | 1);
  size_t smem = sizeof(double) * (size_t)a.k * (a.k | 1);
  if (smem < floor_b) smem = floor_b;
  static std::mutex attr_mu;
  static uint64_t attr_mask = 0;
  per_device_once(attr_mu, attr_mask, [&] {
    int mx = (int)(need_max > floor_b ? need_max : floor_b);
    if (FK <= 96) {  // the VEC (twisted-factorisation arrays) and FIN (W, U, F) extras at k = FK
      const int vec_x = (int)(sizeof(double) * 2 * ((FK + 1 + EIG_SPLIT_CTAS - 1) / EIG_SPLIT_CTAS + 1) * FK);
      const int fin_x = (int)(sizeof(double) * 3 * (size_t)FK * SMALL_M_MAX);
      mx += vec_x > fin_x ? vec_x : fin_x;
    }
    mx += 2 * (int)sizeof(double);  // VEC's rounded-up reflector copy
    DME_CUDA(cudaFuncSetAttribute(eig_tri_kernel<FK, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    if (FK <= 96) {
      DME_CUDA(cudaFuncSetAttribute(eig_tri_kernel<FK, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
      DME_CUDA(cudaFuncSetAttribute(eig_tri_kernel<FK, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    }
    DME_CUDA(cudaFuncSetAttribute(eig_vec_kernel<FK>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    DME_CUDA(cudaFuncSetAttribute(eig_fin_kernel<FK>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  });
  static const int tri_env = [] {
    const char* e = std::getenv("DME_TRI_THREADS");
    return e ? std::atoi(e) : 0;
  }();
  // 512 threads for the first pass (k ~ 92: 184 us against 188 at 256), 256 for k <= 64 (the tail
  // pass, s ~ 57: 79 us against 82 at 512)
  const int tri_nth = tri_env ? tri_env : (a.k <= 64 ? 256 : 512);
  if (FK <= 96 && tri_nth == 128) launch_pdl(eig_tri_kernel<FK, 128>, dim3(1), dim3(128), smem, st, a);
  else if (FK <= 96 && tri_nth == 256) launch_pdl(eig_tri_kernel<FK, 256>, dim3(1), dim3(256), smem, st, a);
  else launch_pdl(eig_tri_kernel<FK, 512>, dim3(1), dim3(512), smem, st, a);
  DME_KCHECK();
  constexpr int MAXE = (FK + 1 + EIG_SPLIT_CTAS - 1) / EIG_SPLIT_CTAS + 1;
  // (+ 2 doubles: the bulk copy of the reflectors is rounded up to 16 bytes)
  const size_t vsmem = FK <= 96 ? sizeof(double) * ((size_t)a.k * (a.k | 1) + 2 * MAXE * FK + 2)
                                : smem + 2 * sizeof(double);
  static const int vec_ctas = [] {
    const char* e = std::getenv("DME_VEC_CTAS");
    const int v = e ? std::atoi(e) : EIG_SPLIT_CTAS;
    return v < EIG_SPLIT_CTAS ? EIG_SPLIT_CTAS : v;  // MAXE is sized for >= EIG_SPLIT_CTAS CTAs
  }();
  launch_pdl(eig_vec_kernel<FK>, dim3(vec_ctas), dim3(ENT), vsmem > smem ? vsmem : smem, st, a);
  DME_KCHECK();
  const size_t fsmem = FK <= 96 ? sizeof(double) * ((size_t)a.k * (a.k | 1) + 2 * (size_t)a.k * SMALL_M_MAX +
                                                  (size_t)a.k * SMALL_M_MAX)
                                 : smem;
  if (a.skip_fin) return;  // (the tail assembly does FIN's work: small.cu, tail_assemble_t3)
  launch_pdl(eig_fin_kernel<FK>, dim3(1), dim3(ENT), fsmem > smem ? fsmem : smem, st, a);
  DME_KCHECK();
}

}  // namespace

size_t eig_split_scratch_doubles() {
  return EsLayout::HDR + 5 * SMALL_K_MAX + 8 + (size_t)SMALL_K_MAX * (SMALL_K_MAX | 1) +
         2 * (size_t)SMALL_K_MAX * SMALL_K_MAX + 64;
}

void eig_split(const SmallArgs& a, cudaStream_t st) {
  if (a.k > FAST_K_MAX || a.k < 3 || !a.Es) throw std::runtime_error("eig_split: k out of range");
  if (a.k <= 96) launch_split<96>(a, st);
  else launch_split<FAST_K_MAX>(a, st);
}

}  // namespace dme
