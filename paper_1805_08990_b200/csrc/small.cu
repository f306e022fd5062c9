// One-CTA kernels on the small (k x k) systems of the column compression and the Riccati flow.
//
// Square-root form used by the whole GPU path (DESIGN.md §"Factor form"): the state is Z with
// P = Z Z^T, i.e. Z = L D^{1/2} of the paper's P = L D L^T. Column compression (P:L245-246:
// "a reduced SVD factorization, followed by a diagonalization of the small resulting system") of
// a concatenated factor Zc (n x k) is, in this form, ONE symmetric eigendecomposition of the Gram
// matrix G = Zc^T Zc = W Theta W^T: Theta are the nonzero eigenvalues of P = Zc Zc^T (the squared
// singular values of Zc, i.e. the eigenvalues of the paper's Sigma V^T D V Sigma), and
//   Z_new = Zc W_kept,   P_new = Z_new Z_new^T,   kept = theta_i > tol * theta_max (reading G7),
// at most `cap` of them, sorted by theta descending (reading G8). W is orthogonal, so the only
// error besides the truncation is eps*||P|| (an orthogonal W is backward
// stable at the level of P; a pivoted-Cholesky/RRQR of G is not — it loses eps*cond(Z1)).
// Riccati flow T3 (eq:nonlinear P:L152, low-rank P:L156) in square-root form: with W = Z^T B,
//   (I + tau P B R^-1 B^T)^-1 P = Z K^-1 Z^T,  K = I + F F^T,  F = sqrt(tau) W L_R^{-T}  (R = L_R L_R^T),
//   Z <- Z K^{-1/2},  K^{-1/2} = I + F g(F^T F) F^T,  g(x) = ((1+x)^{-1/2} - 1)/x = -1/(s (1+s)), s = sqrt(1+x).
// Both are fused into one kernel producing Tm (k x r): the caller then forms Z_new = Zc Tm.
#include "common.cuh"
#include "small.h"
#include "small_common.cuh"

#include <cmath>
#include <cstdlib>

namespace dme {

namespace {

using namespace smallk;

// Parallel cyclic two-sided Jacobi (round-robin ordering) on the packed symmetric matrix S
// (k x k, in shared memory); eigenvectors accumulated in V (k x k column-major, ldv, global).
__device__ void jacobi_eig(double* S, int k, double* V, int64_t ldv, int* pos, double* cs,
                           int* s_rot) {
  const int tid = threadIdx.x;
  const int ke = k + (k & 1);  // even count; index k (if any) is a dummy
  const int np = ke / 2;
  for (int e = tid; e < k * k; e += NT) V[(e % k) + (size_t)(e / k) * ldv] = (e % k == e / k) ? 1.0 : 0.0;
  for (int i = tid; i < ke; i += NT) pos[i] = i;
  __syncthreads();
  double dmax = 0.0;
  for (int i = 0; i < k; ++i) dmax = fmax(dmax, fabs(S[pidx(i, i)]));
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) *s_rot = 0;
    __syncthreads();
    for (int round = 0; round < ke - 1; ++round) {
      // rotation parameters for pair I = (pos[I], pos[ke-1-I])
      for (int I = tid; I < np; I += NT) {
        int p = pos[I], q = pos[ke - 1 - I];
        if (p > q) { const int t = p; p = q; q = t; }
        double c = 1.0, s = 0.0, t = 0.0;
        if (q < k) {
          const double apq = S[pidx(p, q)], app = S[pidx(p, p)], aqq = S[pidx(q, q)];
          if (fabs(apq) > 1e-17 * sqrt(fabs(app * aqq)) && fabs(apq) > 1e-19 * dmax) {
            const double th = (aqq - app) / (2.0 * apq);
            t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(1.0 + th * th));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            atomicAdd(s_rot, 1);
          }
        }
        cs[3 * I] = c;
        cs[3 * I + 1] = s;
        cs[3 * I + 2] = t;
      }
      __syncthreads();
      // A <- J^T A J on the 2x2 blocks (I <= J), each block owned by one thread
      const int nblk = np * (np + 1) / 2;
      for (int e = tid; e < nblk; e += NT) {
        int J = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
        while ((J + 1) * (J + 2) / 2 <= e) ++J;
        while (J * (J + 1) / 2 > e) --J;
        const int I = e - J * (J + 1) / 2;  // I <= J
        int pI = pos[I], qI = pos[ke - 1 - I], pJ = pos[J], qJ = pos[ke - 1 - J];
        if (pI > qI) { const int t = pI; pI = qI; qI = t; }
        if (pJ > qJ) { const int t = pJ; pJ = qJ; qJ = t; }
        const double cI = cs[3 * I], sI = cs[3 * I + 1], tI = cs[3 * I + 2];
        const double cJ = cs[3 * J], sJ = cs[3 * J + 1];
        if (I == J) {
          if (qI < k && sI != 0.0) {
            const double apq = S[pidx(pI, qI)];
            S[pidx(pI, pI)] -= tI * apq;
            S[pidx(qI, qI)] += tI * apq;
            S[pidx(pI, qI)] = 0.0;
          }
          continue;
        }
        const bool vI = qI < k, vJ = qJ < k;
        if (!vI && !vJ) continue;
        // gather (dummy rows/cols read as 0 and are never written)
        double x00 = S[pidx(pI, pJ)];
        double x01 = vJ ? S[pidx(pI, qJ)] : 0.0;
        double x10 = vI ? S[pidx(qI, pJ)] : 0.0;
        double x11 = (vI && vJ) ? S[pidx(qI, qJ)] : 0.0;
        // rows (pair I)
        double r00 = cI * x00 - sI * x10, r01 = cI * x01 - sI * x11;
        double r10 = sI * x00 + cI * x10, r11 = sI * x01 + cI * x11;
        // columns (pair J)
        const double y00 = cJ * r00 - sJ * r01, y01 = sJ * r00 + cJ * r01;
        const double y10 = cJ * r10 - sJ * r11, y11 = sJ * r10 + cJ * r11;
        S[pidx(pI, pJ)] = y00;
        if (vJ) S[pidx(pI, qJ)] = y01;
        if (vI) S[pidx(qI, pJ)] = y10;
        if (vI && vJ) S[pidx(qI, qJ)] = y11;
      }
      // V <- V J
      for (int e = tid; e < k * np; e += NT) {
        const int i = e % k, J = e / k;
        int pJ = pos[J], qJ = pos[ke - 1 - J];
        if (pJ > qJ) { const int t = pJ; pJ = qJ; qJ = t; }
        const double sJ = cs[3 * J + 1];
        if (qJ >= k || sJ == 0.0) continue;
        const double cJ = cs[3 * J];
        double* vp = V + i + (size_t)pJ * ldv;
        double* vq = V + i + (size_t)qJ * ldv;
        const double a = *vp, b = *vq;
        *vp = cJ * a - sJ * b;
        *vq = sJ * a + cJ * b;
      }
      __syncthreads();
      // round-robin: keep pos[0], rotate pos[1..ke-1]
      if (tid == 0) {
        const int last = pos[ke - 1];
        for (int i = ke - 1; i > 1; --i) pos[i] = pos[i - 1];
        pos[1] = last;
      }
      __syncthreads();
    }
    if (*s_rot == 0) break;
    __syncthreads();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(NT, 1) compress_t3_kernel(SmallArgs a) {
  extern __shared__ double S[];  // packed symmetric k(k+1)/2
  __shared__ int pos[SMALL_K_MAX + 1];
  __shared__ double cs[3 * (SMALL_K_MAX / 2 + 1)];
  __shared__ double theta[SMALL_K_MAX];
  __shared__ int rnk[SMALL_K_MAX];
  __shared__ int s_rot, s_r;
  __shared__ double Gam[SMALL_M_MAX * SMALL_M_MAX];
  __shared__ double Phi[SMALL_M_MAX * SMALL_M_MAX];

  const int tid = threadIdx.x;
  const int k = a.k;
  const int m = a.m;
  int r;

  if (a.compress) {
    for (int e = tid; e < k * k; e += NT) {
      const int i = e % k, j = e / k;
      if (i >= j) S[pidx(i, j)] = 0.5 * (a.G[i + (size_t)j * a.ldg] + a.G[j + (size_t)i * a.ldg]);
    }
    __syncthreads();
    jacobi_eig(S, k, a.V, a.ldv, pos, cs, &s_rot);
    for (int i = tid; i < k; i += NT) theta[i] = S[pidx(i, i)];
    __syncthreads();
    // descending order, ties by index
    for (int i = tid; i < k; i += NT) {
      int c = 0;
      const double ti = theta[i];
      for (int j = 0; j < k; ++j) c += (theta[j] > ti) || (theta[j] == ti && j < i);
      rnk[i] = c;
    }
    __syncthreads();
    if (tid == 0) {
      double tmax = -1e300;
      for (int i = 0; i < k; ++i) tmax = fmax(tmax, theta[i]);
      if (a.ref_max > 0.0) tmax = a.ref_max;
      int cnt = 0;
      for (int i = 0; i < k; ++i) cnt += (tmax > 0.0 && theta[i] > a.tol * tmax);
      s_r = cnt < a.cap ? cnt : a.cap;
      double drop = 0.0;
      for (int i = 0; i < k; ++i)
        if (rnk[i] >= s_r) drop = fmax(drop, fabs(theta[i]));
      if (a.stats) {
        a.stats[0] = (double)s_r;
        a.stats[1] = tmax;
        a.stats[2] = tmax > 0 ? drop / tmax : 0.0;
      }
    }
    __syncthreads();
    r = s_r;
    for (int e = tid; e < k * k; e += NT) {
      const int i = e % k, j = e / k;  // V column j -> Tm column rnk[j]
      if (rnk[j] < r)
        a.Tm[i + (size_t)rnk[j] * a.ldt] =
            a.V[i + (size_t)j * a.ldv] * (a.sqrt_scale ? sqrt(fmax(theta[j], 0.0)) : 1.0);
    }
    __syncthreads();
  } else {
    r = k;
    for (int e = tid; e < k * k; e += NT) {
      const int i = e % k, c = e / k;
      a.Tm[i + (size_t)c * a.ldt] = i == c ? 1.0 : 0.0;
    }
    if (tid == 0 && a.stats) { a.stats[0] = k; a.stats[1] = 0; a.stats[2] = 0; }
    __syncthreads();
  }

  if (a.t3 && r > 0) t3_fuse(a, k, r, S, Gam, Phi);
  if (tid == 0) publish_rank(a, r);
}

// Riccati flow T3 alone on a finished compression output Tm (k x r) (after the tail refinement of
// dme.cu, which assembles Tm from two eigen passes before T3 can be applied)
__global__ void __launch_bounds__(NT) t3_only_kernel(SmallArgs a, int r) {
  extern __shared__ double S[];
  __shared__ double Gam[SMALL_M_MAX * SMALL_M_MAX];
  __shared__ double Phi[SMALL_M_MAX * SMALL_M_MAX];
  if (r > 0) t3_fuse(a, a.k, r, S, Gam, Phi);
}

// Pp (k x k, column-major ldp) = I - W W^T, W = the kb leading columns of Tm (k x kb, ldt):
// the projector onto the orthogonal complement of the kept leading eigenvectors
__global__ void complement_kernel(const double* __restrict__ W, int64_t ldw, int k, int kb,
                                  double* __restrict__ Pp, int64_t ldp) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
    const int i = e % k, j = e / k;
    double s = 0.0;
    for (int c = 0; c < kb; ++c) s = fma(W[i + (size_t)c * ldw], W[j + (size_t)c * ldw], s);
    Pp[i + (size_t)j * ldp] = (i == j ? 1.0 : 0.0) - s;
  }
}

// Orthonormal basis U (k x s, column-major ldu) of the complement of span(W), W = the kb leading
// columns of Tm (k x kb, orthonormal), s = k - kb: Householder QR of W, H_0 ... H_{kb-1} W = [R; 0],
// then U = H_0 ... H_{kb-1} [0; I_s] (the trailing columns of the orthogonal factor).
// One CTA of 32 warps; column c of W lives in the registers of warp c mod 32 (RPL rows per lane),
// so a QR step is: one CTA barrier (reflector j published in shared memory), each warp's dots and
// updates of its own columns, and the owner of column j+1 forming reflector j+1 right after its own
// update. The second phase needs no barrier at all: each warp applies the kb stored reflectors to its
// own columns of [0; I_s].
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int RPL, int CPW>
__global__ void __launch_bounds__(NT) complement_basis_kernel(const double* __restrict__ W, int64_t ldw,
                                                              int k, int kb, double* __restrict__ U,
                                                              int64_t ldu) {
  extern __shared__ double Vh[];  // reflectors: row j = v_j (k entries, ld k | 1)
  __shared__ double tau_s[FAST_K_MAX];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ld = k | 1, s = k - kb;
  double x[CPW][RPL];
#pragma unroll
  for (int q = 0; q < CPW; ++q)
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int c = warp + 32 * q, i = lane + 32 * u;
      x[q][u] = (c < kb && i < k) ? W[i + (size_t)c * ldw] : 0.0;
    }
  // reflector j from this warp's column slot q (rows >= j)
  auto reflector = [&](int j, int q) {
    double xs[RPL];
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      double v = 0.0;
#pragma unroll
      for (int qq = 0; qq < CPW; ++qq) v = (qq == q) ? x[qq][u] : v;
      xs[u] = v;
    }
    double n2 = 0.0, xa = 0.0;
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int i = lane + 32 * u;
      if (i > j && i < k) n2 = fma(xs[u], xs[u], n2);
      if (i == j) xa = xs[u];
    }
    n2 = warp_sum(n2);
    const double alpha = __shfl_sync(0xffffffffu, xa, j & 31);
    double t = 0.0, scal = 0.0;
    if (n2 > 0.0) {
      const double beta = -copysign(sqrt(fma(alpha, alpha, n2)), alpha);
      const double amb = alpha - beta;
      const double inv = 1.0 / (amb * beta);  // one division for both quotients
      scal = beta * inv;                      // 1 / (alpha - beta)
      t = -amb * amb * inv;                   // (beta - alpha) / beta
    }
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int i = lane + 32 * u;
      if (i < k) Vh[j * ld + i] = (i < j || t == 0.0) ? 0.0 : (i == j ? 1.0 : xs[u] * scal);
    }
    if (lane == 0) tau_s[j] = t;
  };
  auto apply = [&](int j, int q) {  // column slot q <- H_j column
    const double t = tau_s[j];
    if (t == 0.0) return;
    double vv[RPL], d = 0.0;
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int i = lane + 32 * u;
      vv[u] = i < k ? Vh[j * ld + i] : 0.0;
      double xv = 0.0;
#pragma unroll
      for (int qq = 0; qq < CPW; ++qq) xv = (qq == q) ? x[qq][u] : xv;
      d = fma(vv[u], xv, d);
    }
    d = t * warp_sum(d);
#pragma unroll
    for (int qq = 0; qq < CPW; ++qq)
      if (qq == q)
#pragma unroll
        for (int u = 0; u < RPL; ++u) x[qq][u] = fma(-d, vv[u], x[qq][u]);
  };
  if (warp == 0 && kb > 0) reflector(0, 0);
  for (int j = 0; j < kb; ++j) {
    __syncthreads();  // reflector j published
    const int nxt = j + 1;
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      const int c = warp + 32 * q;
      if (c > j && c < kb) {
        apply(j, q);
        if (c == nxt) reflector(nxt, q);  // look-ahead: owner of column j+1
      }
    }
  }
  __syncthreads();
  if constexpr (RPL * CPW > 9) {
    // k > 96: a whole warp per column (the 8-lane layout would not fit in 64 registers), slots
    // applied one after another, only those holding a column of U
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      const int t = warp + 32 * q;
#pragma unroll
      for (int u = 0; u < RPL; ++u) x[q][u] = (lane + 32 * u == kb + t) ? 1.0 : 0.0;
    }
    for (int j = kb - 1; j >= 0; --j)
#pragma unroll
      for (int q = 0; q < CPW; ++q)
        if (warp + 32 * q < s) apply(j, q);
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      const int t = warp + 32 * q;
      if (t < s)
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int i = lane + 32 * u;
          if (i < k) U[i + (size_t)t * ldu] = x[q][u];
        }
    }
  } else {
    // U = H_0 ... H_{kb-1} [0; I_s]: column t of U starts as e_{kb + t}. Eight lanes per column
    // (rows sub + 8u), so a reflector costs each column a 3-level shuffle reduction (instead of a
    // 5-level one per column and per warp slot): the phase is bound by the SM's shuffle throughput.
    // (k > 96: a whole warp per column, as in phase 1, to stay within 64 registers)
    constexpr int LPC = RPL * CPW <= 9 ? 8 : 32;      // lanes per column
    constexpr int NG = NT / LPC;                      // column groups
    constexpr int R8 = (32 * RPL + LPC - 1) / LPC;    // rows per lane
    constexpr int CPG = (32 * CPW + NG - 1) / NG;     // columns per group
    const int sub = lane & (LPC - 1), grp = tid / LPC, g0 = (tid & ~31) / LPC;
    double y[CPG][R8];
  #pragma unroll
    for (int q = 0; q < CPG; ++q)
  #pragma unroll
      for (int u = 0; u < R8; ++u) y[q][u] = (sub + LPC * u == kb + grp + NG * q) ? 1.0 : 0.0;
    for (int j = kb - 1; j >= 0; --j) {
      const double t = tau_s[j];
      if (t == 0.0) continue;
      double vv[R8];
  #pragma unroll
      for (int u = 0; u < R8; ++u) {
        const int i = sub + LPC * u;
        vv[u] = i < k ? Vh[j * ld + i] : 0.0;
      }
      double d[CPG];
  #pragma unroll
      for (int q = 0; q < CPG; ++q) {
        d[q] = 0.0;
        if (g0 + NG * q < s) {  // (warp-uniform: slots holding no column of U are skipped)
          double d0 = 0.0, d1 = 0.0;
  #pragma unroll
          for (int u = 0; u < R8; u += 2) {
            d0 = fma(vv[u], y[q][u], d0);
            if (u + 1 < R8) d1 = fma(vv[u + 1], y[q][u + 1], d1);
          }
          d[q] = d0 + d1;
        }
      }
  #pragma unroll
      for (int o = 1; o < LPC; o <<= 1)
  #pragma unroll
        for (int q = 0; q < CPG; ++q)
          if (g0 + NG * q < s) d[q] += __shfl_xor_sync(0xffffffffu, d[q], o);
  #pragma unroll
      for (int q = 0; q < CPG; ++q) {
        if (g0 + NG * q >= s) continue;
        const double dq = t * d[q];
  #pragma unroll
        for (int u = 0; u < R8; ++u) y[q][u] = fma(-dq, vv[u], y[q][u]);
      }
    }
  #pragma unroll
    for (int q = 0; q < CPG; ++q) {
      const int t = grp + NG * q;
      if (t < s)
  #pragma unroll
        for (int u = 0; u < R8; ++u) {
          const int i = sub + LPC * u;
          if (i < k) U[i + (size_t)t * ldu] = y[q][u];
        }
    }
  }
}

// Complement basis for k <= 96 by Householder reconstruction (Ballard, Demmel, Grigori, Jacquelin,
// Nguyen, Solomonik 2014, "Reconstructing Householder vectors from tall-skinny QR"). W (k x kb) has
// orthonormal columns, so its Householder QR is W = Q [S; 0], S = diag(+-1), Q = I - Y T Y^T, and
// X = W - [S; 0] = Y (-T Y1^T S) is an LU factorisation (Y unit lower trapezoidal, Y1 = Y[:kb])
// that needs no pivoting when s_j = -sign of the current diagonal entry (|u_jj| >= 1). The trailing
// columns of Q are then
//   U = Q [0; I_s] = [0; I_s] - Y T Y2^T = [0; I_s] + X S Z^T,   Z = Y2 Y1^{-1} = W2 X1^{-1},
// (Y U_lu = X), so neither Y nor T is formed: Gauss-Jordan elimination of [X1^T | W2^T] = W^T with the
// diagonal shifted by -s_j at its pivot (the LU's pivots, so s_j is decided on the fly) leaves Z^T
// in the right block. Same U as the column-by-column Householder kernel below in exact arithmetic;
// its kb sequential steps are plain rank-1 updates (one thread per column, one barrier, no norms or
// reductions), and U = [0; I] + X S Z^T is a small product all 1024 threads share.
constexpr int CLU_KMAX = 96;

__global__ void __launch_bounds__(NT) complement_gj_kernel(const double* __restrict__ W, int64_t ldw, int k,
                                                           int kb, double* __restrict__ U, int64_t ldu,
                                                           const int* __restrict__ kb_dev, SmallArgs fin,
                                                           int has_fin) {
  pdl_wait();
  __shared__ double flam[CLU_KMAX + 1], fslam[CLU_KMAX + 1], fred[NT / 32];
  __shared__ int f_bad;
  double fscale = 0.0, ftmax = 0.0;
  if (has_fin) {  // the first eigen pass ran without FIN: its rank from the scratch header
    const EsLayout es{fin.Es, SMALL_K_MAX};
    const double* h = es.hdr();
    fscale = h[0];
    ftmax = h[3];
    kb = (int)h[4];
    const int nr = kb < k ? kb + 1 : kb;
    for (int i = threadIdx.x; i < nr; i += NT) {
      flam[i] = es.lam()[i];
      fslam[i] = sqrt(fabs(flam[i]));
    }
  } else if (kb_dev) {  // (speculative launch: the rank the first eigen pass published; < 0 = fallback)
    kb = *kb_dev;
    if (kb < 0 || kb >= k) return;
  }
  extern __shared__ double sm[];
  __shared__ double sg[CLU_KMAX];
  const int tid = threadIdx.x, s = k - kb, lda = kb | 1;
  double* Ws = sm;                       // k x kb (ld k): W
  double* A = Ws + (size_t)k * kb;       // kb x k (ld lda, column c = row c of W): W^T, eliminated
  for (int c = tid >> 5; c < kb; c += NT / 32)
    for (int i = tid & 31; i < k; i += 32) {
      const double w = W[i + (size_t)c * ldw];
      Ws[i + c * k] = w;
      A[c + i * lda] = w;
    }
  __syncthreads();
  if (has_fin) {
    // FIN's work for the first pass (eig_split.cu, eig_fin_kernel, t3 = 0): weighted orthogonality
    // of the kb unit vectors W, stats, then the rank (or -1: the caller falls back to Jacobi and
    // queues the complement again)
    double mx = 0.0;
    const int np = kb * (kb + 1) / 2;
    for (int e = tid; e < np; e += NT) {
      int c2 = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while ((c2 + 1) * (c2 + 2) / 2 <= e) ++c2;
      while (c2 * (c2 + 1) / 2 > e) --c2;
      const int c1 = e - c2 * (c2 + 1) / 2;
      const double* v1 = Ws + (size_t)c1 * k;
      const double* v2 = Ws + (size_t)c2 * k;
      double d0 = 0.0, d1 = 0.0;
      int i = 0;
      for (; i + 1 < k; i += 2) { d0 = fma(v1[i], v2[i], d0); d1 = fma(v1[i + 1], v2[i + 1], d1); }
      if (i < k) d0 = fma(v1[i], v2[i], d0);
      const double w = (c1 == c2) ? 1.0 : fslam[c1] * fslam[c2] / fmax(fabs(flam[0]), 1e-300);
      mx = fmax(mx, fabs((d0 + d1) - (c1 == c2 ? 1.0 : 0.0)) * w);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) fred[tid >> 5] = mx;
    __syncthreads();
    if (tid == 0) {
      double m2 = 0.0;
      for (int w = 0; w < NT / 32; ++w) m2 = fmax(m2, fred[w]);
      f_bad = !(m2 <= fin.orth_tol);  // NaN-safe
      if (fin.stats) {
        fin.stats[0] = (double)kb;
        fin.stats[1] = ftmax * fscale;
        fin.stats[2] = (kb < k && ftmax > 0.0) ? fabs(flam[kb]) / ftmax : 0.0;
        fin.stats[3] = f_bad ? 1.0 : 0.0;
        fin.stats[4] = m2;
      }
      publish_rank(fin, f_bad ? -1 : kb);
    }
    __syncthreads();
    if (f_bad || kb >= k) return;
  }
  for (int j = 0; j < kb; ++j) {
    const double dj = A[j + j * lda];
    const double sj = dj >= 0.0 ? -1.0 : 1.0;
    const double inv = 1.0 / (dj - sj);  // |pivot| >= 1
    const int c = j + 1 + tid;
    if (c < k) {
      double* col = A + c * lda;
      const double* cj = A + j * lda;
      const double ajc = col[j] * inv;
      int i = 0;
      for (; i + 3 < kb; i += 4) {
        double x[4], y[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { x[u] = col[i + u]; y[u] = cj[i + u]; }
#pragma unroll
        for (int u = 0; u < 4; ++u) col[i + u] = fma(-y[u], ajc, x[u]);
      }
      for (; i < kb; ++i) col[i] = fma(-cj[i], ajc, col[i]);
      col[j] = ajc;  // (row j: scaled, not eliminated)
    }
    if (tid == 0) sg[j] = sj;
    __syncthreads();
  }
  pdl_trigger();
  // U = [0; I_s] + X (S Z^T), X = W - [S; 0], Z^T = A[:, kb:]; 4 x 2 register tiles
  const int nti = (k + 3) / 4, ntr = (s + 1) / 2;
  for (int t = tid; t < nti * ntr; t += NT) {
    const int tr = t / nti, ti = t - tr * nti;
    const int i0 = 4 * ti, r0 = 2 * tr;
    double acc[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) acc[u][v] = (i0 + u == kb + r0 + v) ? 1.0 : 0.0;
    for (int l = 0; l < kb; ++l) {
      double z[2], x[4];
#pragma unroll
      for (int v = 0; v < 2; ++v) z[v] = r0 + v < s ? sg[l] * A[l + (kb + r0 + v) * lda] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u;
        x[u] = i < k ? Ws[i + l * k] - (i == l ? sg[l] : 0.0) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) acc[u][v] = fma(x[u], z[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        if (i0 + u < k && r0 + v < s) U[(i0 + u) + (size_t)(r0 + v) * ldu] = acc[u][v];
  }
}

size_t complement_gj_smem(int k, int kb) {
  return sizeof(double) * ((size_t)k * kb + (size_t)(kb | 1) * k);
}

__global__ void tail_product_kernel(double* Tm, int64_t ldt, const double* __restrict__ U, int64_t ldu,
                                    int s, const double* __restrict__ V, int64_t ldv, int k, int kb, int ks) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * ks) return;
  const int i = e % k, c = e / k;
  double acc = 0.0;
  for (int j = 0; j < s; ++j) acc = fma(U[i + (size_t)j * ldu], V[j + (size_t)c * ldv], acc);
  Tm[i + (size_t)(kb + c) * ldt] = acc;
}

// Tail of the refined compression: Tm[:, kb + c] = U V[:, c] (c < ks; U: k x s, V: s x ks), then
// the Riccati flow T3 on the whole Tm (k x (kb + ks)) when a.t3 is set.
__global__ void __launch_bounds__(NT) tail_assemble_kernel(SmallArgs a, const double* __restrict__ U,
                                                           int64_t ldu, int s, const double* __restrict__ V,
                                                           int64_t ldv, int kb, int ks, const int* ks_dev,
                                                           SmallArgs fin, int has_fin) {
  pdl_wait();
  extern __shared__ double S[];
  __shared__ double flam[FAST_K_MAX + 1], fslam[FAST_K_MAX + 1], fred[NT / 32];
  __shared__ int f_bad;
  double fscale = 0.0, ftmax = 0.0;
  if (has_fin) {  // the split eigen pass of the tail ran without FIN: its rank from the scratch header
    const EsLayout es{fin.Es, SMALL_K_MAX};
    const double* h = es.hdr();
    fscale = h[0];
    ftmax = h[3];
    ks = (int)h[4];
    const int nr = ks < fin.k ? ks + 1 : ks;
    for (int i = threadIdx.x; i < nr; i += NT) {
      flam[i] = es.lam()[i];
      fslam[i] = sqrt(fabs(flam[i]));
    }
  } else if (ks_dev) {  // the tail rank published by the preceding eigen pass (< 0: it fell back to Jacobi)
    ks = *ks_dev;
    if (ks < 0) return;
  }
  __shared__ double Gam[SMALL_M_MAX * SMALL_M_MAX];
  __shared__ double Phi[SMALL_M_MAX * SMALL_M_MAX];
  const int k = a.k, r = kb + ks, m = a.m, tid = threadIdx.x;
  // shared layout: Tm (k x r, ld k) | H (k x m) | U (k x s) | V (s x ks) ; t3 scratch reuses U/V
  double* Ts = S;
  double* Hs = Ts + (size_t)k * r;
  double* Us = Hs + (size_t)k * m;
  double* Vs = Us + (size_t)k * s;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NWP = NT / 32;
  for (int c = warp; c < kb; c += NWP)
    for (int i = lane; i < k; i += 32) Ts[i + c * k] = a.Tm[i + (size_t)c * a.ldt];
  if (a.t3)  // (H = Zc^T B is only formed when T3 is fused)
    for (int c = warp; c < m; c += NWP)
      for (int i = lane; i < k; i += 32) Hs[i + c * k] = a.H[i + (size_t)c * a.ldh];
  for (int c = warp; c < s; c += NWP)
    for (int i = lane; i < k; i += 32) Us[i + c * k] = U[i + (size_t)c * ldu];
  for (int c = warp; c < ks; c += NWP)
    for (int i = lane; i < s; i += 32) Vs[i + c * s] = V[i + (size_t)c * ldv];
  __syncthreads();
  if (has_fin) {
    // FIN's work for the tail pass (eig_split.cu, eig_fin_kernel): weighted orthogonality of the ks
    // unit vectors V (|V^T V - I|, off-diagonal entries weighted by sqrt(lam_i lam_j) / lam_0),
    // stats, then the rank (or -1: the caller falls back to Jacobi and assembles again)
    double mx = 0.0;
    const int np = ks * (ks + 1) / 2;
    for (int e = threadIdx.x; e < np; e += NT) {
      int c2 = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while ((c2 + 1) * (c2 + 2) / 2 <= e) ++c2;
      while (c2 * (c2 + 1) / 2 > e) --c2;
      const int c1 = e - c2 * (c2 + 1) / 2;
      const double* v1 = Vs + (size_t)c1 * s;
      const double* v2 = Vs + (size_t)c2 * s;
      double d0 = 0.0, d1 = 0.0;
      int i = 0;
      for (; i + 1 < s; i += 2) { d0 = fma(v1[i], v2[i], d0); d1 = fma(v1[i + 1], v2[i + 1], d1); }
      if (i < s) d0 = fma(v1[i], v2[i], d0);
      const double w = (c1 == c2) ? 1.0 : fslam[c1] * fslam[c2] / fmax(fabs(flam[0]), 1e-300);
      mx = fmax(mx, fabs((d0 + d1) - (c1 == c2 ? 1.0 : 0.0)) * w);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) fred[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m2 = 0.0;
      for (int w = 0; w < NT / 32; ++w) m2 = fmax(m2, fred[w]);
      f_bad = !(m2 <= fin.orth_tol);  // NaN-safe
      if (fin.stats) {
        fin.stats[0] = (double)ks;
        fin.stats[1] = ftmax * fscale;
        fin.stats[2] = (ks < fin.k && ftmax > 0.0) ? fabs(flam[ks]) / ftmax : 0.0;
        fin.stats[3] = f_bad ? 1.0 : 0.0;
        fin.stats[4] = m2;
      }
      publish_rank(fin, f_bad ? -1 : ks);
    }
    __syncthreads();
    if (f_bad) return;
  }
  for (int c = warp; c < ks; c += NWP)
    for (int i = lane; i < k; i += 32) {
      double acc = 0.0;
      for (int j = 0; j < s; ++j) acc = fma(Us[i + j * k], Vs[j + c * s], acc);
      Ts[i + (kb + c) * k] = acc;
    }
  __syncthreads();
  if (a.t3 && r > 0) {
    SmallArgs b = a;
    b.Tm = Ts; b.ldt = k;
    b.H = Hs; b.ldh = k;
    t3_fuse(b, k, r, Us, Gam, Phi);  // (U, V are free now: >= 2 SMALL_K_MAX SMALL_M_MAX doubles)
    __syncthreads();
  }
  for (int c = warp; c < r; c += NWP)
    for (int i = lane; i < k; i += 32) a.Tm[i + (size_t)c * a.ldt] = Ts[i + c * k];
}

}  // namespace

void complement_basis(const double* W, int64_t ldw, int k, int kb, double* U, int64_t ldu,
                      cudaStream_t st, bool attrs_only) {
  if (k > FAST_K_MAX || kb > k || kb < 0) throw std::runtime_error("complement_basis: bad size");
  const int mx = (int)(sizeof(double) * FAST_K_MAX * (FAST_K_MAX | 1));
  static std::mutex attr_mu;
  static uint64_t attr_mask = 0;
  per_device_once(attr_mu, attr_mask, [&] {
    DME_CUDA(cudaFuncSetAttribute(complement_basis_kernel<3, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    DME_CUDA(cudaFuncSetAttribute(complement_basis_kernel<5, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    DME_CUDA(cudaFuncSetAttribute(complement_gj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)complement_gj_smem(CLU_KMAX, CLU_KMAX)));
  });
  if (attrs_only) return;
  const size_t smem = sizeof(double) * (size_t)(kb > 0 ? kb : 1) * (k | 1);
  static const bool old_cb = std::getenv("DME_CB_HOUSEHOLDER") != nullptr;  // A/B knob
  if (k <= CLU_KMAX && !old_cb)
    launch_pdl(complement_gj_kernel, dim3(1), dim3(NT), complement_gj_smem(k, kb), st, W, ldw, k, kb, U, ldu,
               (const int*)nullptr, SmallArgs{}, 0);
  else if (k <= 96) complement_basis_kernel<3, 3><<<1, NT, smem, st>>>(W, ldw, k, kb, U, ldu);
  else complement_basis_kernel<5, 5><<<1, NT, smem, st>>>(W, ldw, k, kb, U, ldu);
  DME_KCHECK();
}

bool complement_dev_available(int k) {
  static const bool old_cb = std::getenv("DME_CB_HOUSEHOLDER") != nullptr;
  return k <= CLU_KMAX && !old_cb;
}

bool complement_basis_dev(const double* W, int64_t ldw, int k, const int* kb_dev, double* U, int64_t ldu,
                          cudaStream_t st, const SmallArgs* fin) {
  if (!complement_dev_available(k)) return false;
  complement_basis(W, ldw, k, 0, U, 0, nullptr, true);  // (attributes only)
  launch_pdl(complement_gj_kernel, dim3(1), dim3(NT), complement_gj_smem(k, k), st, W, ldw, k, 0, U, ldu,
             kb_dev, fin ? *fin : SmallArgs{}, fin ? 1 : 0);
  DME_KCHECK();
  return true;
}

void t3_only(const SmallArgs& a, int r, cudaStream_t st);

size_t tail_assemble_smem(int k, int m, int s, int kb, int ks) {
  const int r = kb + ks;
  size_t need = sizeof(double) * ((size_t)k * r + (size_t)k * m + (size_t)k * s + (size_t)s * ks);
  const size_t t3s = sizeof(double) * ((size_t)k * r + (size_t)k * m + 2 * SMALL_K_MAX * SMALL_M_MAX);
  return need < t3s ? t3s : need;
}

void tail_assemble_t3(const SmallArgs& a, const double* U, int64_t ldu, int s, const double* V,
                      int64_t ldv, int kb, int ks, cudaStream_t st, const int* ks_dev, const SmallArgs* fin) {
  if (a.m > SMALL_M_MAX) throw std::runtime_error("tail_assemble_t3: m exceeds SMALL_M_MAX");
  const int k = a.k, r = kb + ks;
  size_t need = sizeof(double) * ((size_t)k * r + (size_t)k * a.m + (size_t)k * s + (size_t)s * ks);
  const size_t t3s = sizeof(double) * ((size_t)k * r + (size_t)k * a.m + 2 * SMALL_K_MAX * SMALL_M_MAX);
  if (need < t3s) need = t3s;
  if (need > (size_t)SMALL_SMEM_MAX) {  // wide systems: the product in global memory, then T3 alone
    if (ks_dev || fin) throw std::runtime_error("tail_assemble_t3: device rank needs the shared-memory path");
    if (ks > 0) {
      tail_product_kernel<<<(k * ks + 255) / 256, 256, 0, st>>>(a.Tm, a.ldt, U, ldu, s, V, ldv, k, kb, ks);
      DME_KCHECK();
    }
    if (a.t3 && r > 0) t3_only(a, r, st);
    return;
  }
  static std::mutex attr_mu;
  static uint64_t attr_mask = 0;
  per_device_once(attr_mu, attr_mask, [&] {
    DME_CUDA(cudaFuncSetAttribute(tail_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  SMALL_SMEM_MAX));
  });
  const SmallArgs none{};
  launch_pdl(tail_assemble_kernel, dim3(1), dim3(NT), need, st, a, U, ldu, s, V, ldv, kb, ks, ks_dev,
             fin ? *fin : none, fin ? 1 : 0);
  DME_KCHECK();
}

void t3_only(const SmallArgs& a, int r, cudaStream_t st) {
  if (a.m > SMALL_M_MAX) throw std::runtime_error("t3_only: m exceeds SMALL_M_MAX");
  t3_only_kernel<<<1, NT, sizeof(double) * 2 * SMALL_K_MAX * SMALL_M_MAX, st>>>(a, r);
  DME_KCHECK();
}

void complement_projector(const double* W, int64_t ldw, int k, int kb, double* Pp, int64_t ldp,
                          cudaStream_t st) {
  complement_kernel<<<(k * k + 255) / 256, 256, 0, st>>>(W, ldw, k, kb, Pp, ldp);
  DME_KCHECK();
}

void compress_t3(const SmallArgs& a, cudaStream_t st) {
  if (a.k > SMALL_K_MAX) throw std::runtime_error("compress_t3: k exceeds SMALL_K_MAX");
  if (a.t3 && a.m > SMALL_M_MAX) throw std::runtime_error("compress_t3: m exceeds SMALL_M_MAX");
  size_t smem = a.compress ? sizeof(double) * (size_t)a.k * (a.k + 1) / 2 : 0;
  if (smem < sizeof(double) * 2 * SMALL_K_MAX * SMALL_M_MAX) smem = sizeof(double) * 2 * SMALL_K_MAX * SMALL_M_MAX;
  static std::mutex attr_mu;
  static uint64_t attr_mask = 0;
  per_device_once(attr_mu, attr_mask, [&] {
    DME_CUDA(cudaFuncSetAttribute(compress_t3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  SMALL_SMEM_MAX));
  });
  compress_t3_kernel<<<1, NT, smem, st>>>(a);
  DME_KCHECK();
}

}  // namespace dme
