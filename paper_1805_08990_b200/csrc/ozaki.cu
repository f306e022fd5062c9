// E·Y on the int8 tensor cores by exact digit slicing (see ozaki.h).
//
// Kernel layout (one persistent CTA per SM, 224 threads):
//   warp 0      TMA producer of E: per 128-deep K chunk OZ_S boxes of 128 rows x 128 bytes of E
//               digits (A ring, one slice per stage);
//   warp 6      TMA producer of Y: per K chunk one 3D box with all OZ_S digit slices of the Y
//               columns (B ring, 2 stages), running ahead independently of the A ring;
//   warp 1      TMEM owner (512 columns) and MMA issuer (one thread): for E slice a the B operand
//               is Y slices b = 0 .. OZ_S-1-a stacked along N, written at TMEM column a*NP, so the
//               accumulator block c holds sum_{a+b=c} D_a Y_b (c = 0 .. OZ_S-1, NP columns each);
//   warps 2..5  epilogue: TMEM -> registers, sum_c 2^{-7(c+2)} acc_c in FP64, scale by
//               2^{e_i + f_j}, store (or write a partial and let the last CTA of the tile reduce
//               the partials in CTA order: deterministic).
#include "common.cuh"
#include "ozaki.h"

#include <algorithm>
#include <vector>

namespace dme {
namespace {

template <int NP>
struct OzCfg {
  static constexpr int S = OZ_S;
  static constexpr int BST = S * NP * 128;  // B stage: all slices, NP rows x 128 bytes each
  static constexpr int AST = 128 * 128;     // A stage: one slice, 128 rows x 128 bytes
  static constexpr int NB = 2;
  static constexpr int NA = (212 * 1024 - NB * BST) / AST;
  static constexpr int NBAR = 2 * NA + 2 * NB + 2;
  static constexpr int SMEM = NB * BST + NA * AST + 1024 + NBAR * 8 + 16;
  static_assert(NA >= 4, "A ring too shallow");
};

// ------------------------------------------------------------------ tcgen05 wrappers
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  // K-major operand, 128-byte swizzle: rows of 128 B, 8-row groups 1024 B apart (SBO), LBO unused,
  // descriptor version 1 (sm_100), layout type 2 = SWIZZLE_128B
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// low / high halves of the descriptor: lo = start address >> 4 | LBO (1) << 16, hi = SBO (1024 B)
// | version 1 | SWIZZLE_128B; operands only move the start address, so lo += bytes >> 4
__device__ __forceinline__ uint32_t desc_lo(uint32_t saddr) { return ((saddr >> 4) & 0x3FFFu) | (1u << 16); }
__device__ __forceinline__ uint64_t mk_desc(uint32_t lo) {
  return (uint64_t)lo | ((uint64_t)((1024 >> 4) | (1u << 14) | (2u << 29)) << 32);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ uint32_t idesc_i8(int N) {
  // D s32 (bits 4-5 = 2), A s8 (bits 7-9 = 1), B s8 (bits 10-12 = 1), K-major both,
  // N >> 3 at bits 17-22, M >> 4 = 8 (M = 128) at bits 24-28
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t addr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// int32 (as raw bits) -> double, exactly, without the quarter-rate I2F.F64
__device__ __forceinline__ double i2d_exact(uint32_t v) {
  return __hiloint2double(0x43300000, (int)(v ^ 0x80000000u)) - 4503601774854144.0;  // 2^52 + 2^31
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// x * 2^s exactly for |s| <= 2000 (two normal-range power-of-two factors)
__device__ __forceinline__ double scale2(double x, int s) {
  s = s < -2000 ? -2000 : (s > 2000 ? 2000 : s);  // beyond: under/overflow either way
  const int s1 = s / 2, s2 = s - s1;
  return x * __longlong_as_double((long long)(1023 + s1) << 52) *
         __longlong_as_double((long long)(1023 + s2) << 52);
}

// Stream-K: CTA b owns the units [b U / G, (b+1) U / G) of the (tile, K chunk) sequence
__device__ __forceinline__ int cta_of(int64_t u, int64_t U, int G) {
  int64_t b = (u * G) / U;
  while (b + 1 < G && ((b + 1) * U) / G <= u) ++b;
  while (b > 0 && (b * U) / G > u) --b;
  return (int)b;
}

// The segments (tile, K-chunk range) a CTA works on, in order. Stream-K mode (E pass: few row
// tiles, long K): the contiguous unit range [u0, u1) of the (tile, chunk) sequence, split tiles
// reduced deterministically in CTA order. Round-robin mode (square GEMMs: many tiles): whole tiles
// b, b + G, b + 2G, ... of a rasterised tile list, no reduction.
struct SegIter {
  int64_t u, u1;
  int t, ntiles, G, nkc;
  bool rr;
  __device__ SegIter(bool rr_, int ntiles_, int nkc_) : rr(rr_), ntiles(ntiles_), G(gridDim.x), nkc(nkc_) {
    const int64_t U = (int64_t)ntiles * nkc;
    u = (int64_t)blockIdx.x * U / G;
    u1 = (int64_t)(blockIdx.x + 1) * U / G;
    t = blockIdx.x;
  }
  __device__ bool next(int& tile, int& kc0, int& kc1) {
    if (rr) {
      if (t >= ntiles) return false;
      tile = t;
      kc0 = 0;
      kc1 = nkc;
      t += G;
      return true;
    }
    if (u >= u1) return false;
    tile = (int)(u / nkc);
    kc0 = (int)(u % nkc);
    kc1 = (int)(kc0 + (u1 - u) < nkc ? kc0 + (u1 - u) : nkc);
    u += kc1 - kc0;
    return true;
  }
};

template <int NP>
__global__ void __launch_bounds__(224, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const int* __restrict__ eA, const int* __restrict__ eB, double* __restrict__ out,
                   int64_t out_rs, int64_t out_cs, int M, int N, int nkc, int ntiles,
                   const int2* __restrict__ tile_list, int rr, double alpha,
                   double* __restrict__ partial, int* __restrict__ counters,
                   const int8_t* __restrict__ a_tiled) {
  using C = OzCfg<NP>;
  constexpr int S = C::S;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* Bs = base;
  uint8_t* As = base + C::NB * C::BST;
  uint64_t* bars = reinterpret_cast<uint64_t*>(As + C::NA * C::AST);
  uint64_t* full_a = bars;
  uint64_t* empty_a = bars + C::NA;
  uint64_t* full_b = bars + 2 * C::NA;
  uint64_t* empty_b = full_b + C::NB;
  uint64_t* tfull = empty_b + C::NB;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int64_t U = (int64_t)ntiles * nkc;
  auto coords = [&](int tile, int& rt, int& ct) {
    if (tile_list) { const int2 tc = tile_list[tile]; rt = tc.x; ct = tc.y; }
    else { rt = tile; ct = 0; }
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NA; ++i) { mbar_init(full_a + i, 1); mbar_init(empty_a + i, 1); }
    for (int i = 0; i < C::NB; ++i) { mbar_init(full_b + i, 1); mbar_init(empty_b + i, 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);  // one arrive per epilogue warp
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == 6) {
    if (lane == 0) {  // ---------------------------------------- TMA producers: A (warp 0), B (warp 6)
      const bool isA = warp == 0;
      if (isA) prefetch_tmap(&tmA); else prefetch_tmap(&tmB);
      const uint64_t l2_first = policy_evict_first();  // E digits: streamed once per pass
      int as = 0, bs = 0;
      uint32_t pa = 0, pb = 0;
      SegIter it(rr != 0, ntiles, nkc);
      int tile, kc0, kc1;
      while (it.next(tile, kc0, kc1)) {
        int rt, ct;
        coords(tile, rt, ct);
        for (int kc = kc0; kc < kc1; ++kc) {
          if (!isA) {
            mbar_wait(empty_b + bs, pb ^ 1);
            mbar_arrive_expect_tx(full_b + bs, C::BST);
            tma_load_3d(Bs + bs * C::BST, &tmB, full_b + bs, kc * 128, ct * NP, 0);
            if (++bs == C::NB) { bs = 0; pb ^= 1; }
            continue;
          }
          for (int a = 0; a < S; ++a) {
            mbar_wait(empty_a + as, pa ^ 1);
            mbar_arrive_expect_tx(full_a + as, C::AST);
            if (a_tiled)  // pre-swizzled tile image: one contiguous 16 KB bulk copy, read once
              bulk_load_hint(As + as * C::AST,
                             a_tiled + (((size_t)rt * nkc + kc) * S + a) * (size_t)C::AST, C::AST,
                             full_a + as, l2_first);
            else
              tma_load_3d(As + as * C::AST, &tmA, full_a + as, kc * 128, rt * 128, a);
            if (++as == C::NA) { as = 0; pa ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (whole warp waits,
    // one elected lane issues; descriptors are base + compile-time offsets)
    int as = 0, bs = 0, seg = 0;
    uint32_t pa = 0, pb = 0;
    const uint32_t lo_a0 = desc_lo(smem_u32(As)), lo_b0 = desc_lo(smem_u32(Bs));
    SegIter it(rr != 0, ntiles, nkc);
    int tile, kc0, kc1;
    while (it.next(tile, kc0, kc1)) {
      if (seg > 0) mbar_wait(tempty, (seg - 1) & 1);  // epilogue has drained the accumulators
      tc_fence_after();
      for (int kc = kc0; kc < kc1; ++kc) {
        mbar_wait(full_b + bs, pb);
        tc_fence_after();
        const uint32_t lo_b = lo_b0 + (uint32_t)(bs * (C::BST >> 4));
#pragma unroll
        for (int a = 0; a < S; ++a) {
          mbar_wait(full_a + as, pa);
          tc_fence_after();
          const uint32_t lo_a = lo_a0 + (uint32_t)(as * (C::AST >> 4));
          if (elect_one()) {
            const int rows = (S - a) * NP;                        // Y slices 0 .. S-1-a
            const int n0 = rows <= 256 ? rows : ((rows / 2 + 15) / 16) * 16;  // balanced split
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {                      // 4 x K=32 per 128-byte chunk
              const uint32_t acc = (kc > kc0 || a > 0 || ks > 0) ? 1u : 0u;
              const uint64_t ad = mk_desc(lo_a + ks * 2);
              mma_i8(tmem + (uint32_t)(a * NP), ad, mk_desc(lo_b + ks * 2), idesc_i8(n0), acc);
              if (rows > n0)
                mma_i8(tmem + (uint32_t)(a * NP + n0), ad, mk_desc(lo_b + ks * 2 + n0 * 8),
                       idesc_i8(rows - n0), acc);
            }
            umma_commit(empty_a + as);  // A slot free once these MMAs have read it
          }
          __syncwarp();
          if (++as == C::NA) { as = 0; pa ^= 1; }
        }
        if (elect_one()) umma_commit(empty_b + bs);
        __syncwarp();
        if (++bs == C::NB) { bs = 0; pb ^= 1; }
      }
      if (elect_one()) umma_commit(tfull);
      __syncwarp();
      ++seg;
    }
  } else if (warp <= 5) {  // ------------------------------------------------ epilogue (warps 2..5)
    const int qd = warp & 3;            // TMEM sub-partition of this warp
    const int rl = 32 * qd + lane;      // row within the tile
    const int et = threadIdx.x - 64;    // 0..127
    int seg = 0;
    SegIter it(rr != 0, ntiles, nkc);
    int tile, kc0, kc1;
    while (it.next(tile, kc0, kc1)) {
      int rt, ct;
      coords(tile, rt, ct);
      mbar_wait(tfull, seg & 1);
      tc_fence_after();
      // drain TMEM: per accumulator block c (smallest scale first) NP/16 loads, one wait
      double acc[NP];
#pragma unroll
      for (int j = 0; j < NP; ++j) acc[j] = 0.0;
#pragma unroll
      for (int c = S - 1; c >= 0; --c) {
        uint32_t v[NP];
#pragma unroll
        for (int j0 = 0; j0 < NP; j0 += 16)
          tmem_ld16_nowait(tmem + ((uint32_t)(32 * qd) << 16) + (uint32_t)(c * NP + j0), v + j0);
        tmem_wait_ld();
        const double sc = __longlong_as_double((long long)(1023 - 7 * (c + 2)) << 52);
#pragma unroll
        for (int j = 0; j < NP; ++j) acc[j] = fma(i2d_exact(v[j]), sc, acc[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      ++seg;

      const int row = rt * 128 + rl;
      const int col0 = ct * NP;
      const int ea = row < M ? eA[row] : 0;
      double* orow = out + (int64_t)row * out_rs + (int64_t)col0 * out_cs;
      const int* eb = eB + col0;
      const int ncol = N - col0 < NP ? N - col0 : NP;
      const bool whole = kc0 == 0 && kc1 == nkc;
      if (whole) {
        if (row < M) {
#pragma unroll
          for (int j = 0; j < NP; ++j)
            if (j < ncol) orow[(int64_t)j * out_cs] = alpha * scale2(acc[j], ea + eb[j]);
        }
      } else {
        // split tile (Stream-K mode): slot 2b + (this CTA started before the tile)
        const int64_t tu0 = (int64_t)tile * nkc;
        const int64_t my_u0 = (int64_t)blockIdx.x * U / G;
        double* slot = partial + (size_t)(2 * blockIdx.x + (my_u0 < tu0 ? 1 : 0)) * OZ_NMAX * 128;
#pragma unroll
        for (int j = 0; j < NP; ++j)
          __stcg(slot + j * 128 + rl, (j < ncol && row < M) ? alpha * scale2(acc[j], ea + eb[j]) : 0.0);
        __threadfence();
        named_bar_sync(1, 128);
        const int b0 = cta_of(tu0, U, G);
        const int b1 = cta_of(tu0 + nkc - 1, U, G);
        if (et == 0) {
          const int old = atomicAdd(counters + tile, 1);
          *flag = (old == b1 - b0) ? 1 : 0;
        }
        named_bar_sync(1, 128);
        if (*flag) {  // last CTA of the tile: sum the partials in CTA order (deterministic)
          __threadfence();
          if (row < M) {
            constexpr int JC = NP < 32 ? NP : 32;
#pragma unroll
            for (int j0 = 0; j0 < NP; j0 += JC) {
              double sum[JC];
#pragma unroll
              for (int t = 0; t < JC; ++t) sum[t] = 0.0;
              for (int b = b0; b <= b1; ++b) {
                const int64_t bu0 = (int64_t)b * U / G;
                const double* src =
                    partial + (size_t)(2 * b + (bu0 < tu0 ? 1 : 0)) * OZ_NMAX * 128 + rl;
                double v[JC];
#pragma unroll
                for (int t = 0; t < JC; ++t) v[t] = __ldcg(src + (j0 + t) * 128);
#pragma unroll
                for (int t = 0; t < JC; ++t) sum[t] += v[t];
              }
#pragma unroll
              for (int t = 0; t < JC; ++t)
                if (j0 + t < ncol) orow[(int64_t)(j0 + t) * out_cs] = sum[t];
            }
          }
          if (et == 0) counters[tile] = 0;
        }
        named_bar_sync(1, 128);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ------------------------------------------------------------------ digit slicing
constexpr int SL_T = 256, SL_CH = SL_T * 4 * 2;  // threads, columns per CTA chunk

__global__ void __launch_bounds__(SL_T) oz_rowmax_kernel(const double* __restrict__ X, int64_t ld,
                                                         int64_t cols, double* __restrict__ pm) {
  __shared__ double red[SL_T / 32];
  const int64_t row = blockIdx.y, c0 = (int64_t)blockIdx.x * SL_CH;
  const double* x = X + row * ld;
  double m = 0.0;
#pragma unroll
  for (int t = 0; t < SL_CH / SL_T; ++t) {
    const int64_t c = c0 + t * SL_T + threadIdx.x;
    if (c < cols) m = fmax(m, fabs(x[c]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < SL_T / 32; ++w) m = fmax(m, red[w]);
    pm[row * gridDim.x + blockIdx.x] = m;
  }
}

__global__ void __launch_bounds__(SL_T) oz_slice_kernel(const double* __restrict__ X, int64_t ld,
                                                        int64_t cols, const double* __restrict__ pm,
                                                        int8_t* __restrict__ q, int64_t ldk,
                                                        int64_t sstride, int* __restrict__ ex) {
  const int64_t row = blockIdx.y;
  double mx = 0.0;
  for (unsigned i = 0; i < gridDim.x; ++i) mx = fmax(mx, pm[row * gridDim.x + i]);
  const int e = mx > 0.0 ? ilogb(mx) + 2 : 0;  // max |x| 2^-e in [1/4, 1/2)
  if (blockIdx.x == 0 && threadIdx.x == 0) ex[row] = e;
  const double* x = X + row * ld;
  const int64_t c4end = (cols + 3) / 4 * 4;
#pragma unroll
  for (int it = 0; it < SL_CH / (SL_T * 4); ++it) {
    const int64_t c4 = (int64_t)blockIdx.x * SL_CH + ((int64_t)it * SL_T + threadIdx.x) * 4;
    if (c4 >= c4end) break;
    uint32_t w[OZ_S];
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) w[s] = 0u;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      double v = c4 + t < cols ? scale2(x[c4 + t], -e) : 0.0;
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) {
        v *= 128.0;                 // exact
        const double d = rint(v);   // |d| <= 64
        v -= d;                     // exact, |v| <= 1/2
        w[s] |= (uint32_t)(uint8_t)(int8_t)(int)d << (8 * t);
      }
    }
#pragma unroll
    for (int s = 0; s < OZ_S; ++s)
      *reinterpret_cast<uint32_t*>(q + s * sstride + row * ldk + c4) = w[s];
  }
}

// Digit slicing into the tiled, pre-swizzled image the E-pass kernel streams with plain bulk
// copies: block (row tile t, K chunk c, slice s) = 128 rows x 128 bytes at
// ((t * nkc + c) * OZ_S + s) * 16384, row i at i * 128, 16-byte chunk j at (j ^ (i & 7)) * 16
// (SWIZZLE_128B). Padding rows / columns must be zero (the caller clears the buffer once).
__global__ void __launch_bounds__(SL_T) oz_slice_tiled_kernel(const double* __restrict__ X, int64_t ld,
                                                              int64_t cols, const double* __restrict__ pm,
                                                              int8_t* __restrict__ q, int nkc,
                                                              int* __restrict__ ex) {
  const int64_t row = blockIdx.y;
  double mx = 0.0;
  for (unsigned i = 0; i < gridDim.x; ++i) mx = fmax(mx, pm[row * gridDim.x + i]);
  const int e = mx > 0.0 ? ilogb(mx) + 2 : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) ex[row] = e;
  const double* x = X + row * ld;
  const int64_t c4end = (cols + 3) / 4 * 4;
  const int64_t t = row >> 7;
  const int il = (int)(row & 127);
#pragma unroll
  for (int it = 0; it < SL_CH / (SL_T * 4); ++it) {
    const int64_t c4 = (int64_t)blockIdx.x * SL_CH + ((int64_t)it * SL_T + threadIdx.x) * 4;
    if (c4 >= c4end) break;
    uint32_t w[OZ_S];
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) w[s] = 0u;
#pragma unroll
    for (int tt = 0; tt < 4; ++tt) {
      double v = c4 + tt < cols ? scale2(x[c4 + tt], -e) : 0.0;
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) {
        v *= 128.0;
        const double d = rint(v);
        v -= d;
        w[s] |= (uint32_t)(uint8_t)(int8_t)(int)d << (8 * tt);
      }
    }
    const int64_t ck = c4 >> 7;
    const int lb = (int)(c4 & 127);
    const int64_t off = ((t * nkc + ck) * OZ_S) * 16384 + il * 128 + ((((lb >> 4) ^ (il & 7)) << 4) | (lb & 15));
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) *reinterpret_cast<uint32_t*>(q + off + (int64_t)s * 16384) = w[s];
  }
}

template <int NP>
void launch_oz(const OzGemmArgs& a, OzScratch& ws, cudaStream_t st) {
  using C = OzCfg<NP>;
  const int nkc = (int)ceil_div(a.K, 128);
  const bool listed = a.tiles != nullptr;
  const int ntiles = listed ? a.ntiles : (int)ceil_div(a.M, 128);
  const int64_t U = (int64_t)ntiles * nkc;
  const int G = (int)std::min<int64_t>(ws.max_grid, a.round_robin ? ntiles : U);
  if (!a.round_robin && ntiles > ws.max_tiles) throw std::runtime_error("oz_gemm: scratch too small");
  if (G > ws.max_grid) throw std::runtime_error("oz_gemm: grid exceeds scratch");
  CUtensorMap tmA{};
  if (!a.A_tiled)
    tmA = make_tmap_3d_u8(a.A, a.K, a.M, OZ_S, a.lda, a.a_slice_stride, 128, 128, 1);
  const CUtensorMap tmB = make_tmap_3d_u8(a.B, a.K, listed ? a.N : NP, OZ_S, a.ldb, a.b_slice_stride,
                                          128, NP, OZ_S);
  static std::mutex attr_mu;
  static uint64_t attr_mask = 0;
  per_device_once(attr_mu, attr_mask, [&] {
    DME_CUDA(cudaFuncSetAttribute(oz_gemm_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  });
  oz_gemm_kernel<NP><<<G, 224, C::SMEM, st>>>(tmA, tmB, a.eA, a.eB, a.out, a.out_rs, a.out_cs,
                                              (int)a.M, (int)a.N, nkc, ntiles, a.tiles,
                                              a.round_robin ? 1 : 0, a.alpha, ws.partial,
                                              ws.counters, a.A_tiled);
  DME_KCHECK();
}

}  // namespace

int64_t oz_slice_scratch_doubles(int64_t rows, int64_t cols) { return rows * ceil_div(cols, SL_CH); }

void oz_slice_rows(const double* X, int64_t ld, int64_t rows, int64_t cols, int8_t* q, int64_t ldk,
                   int64_t slice_stride, int* ex, double* scratch, cudaStream_t st) {
  if (rows <= 0) return;
  const dim3 grid((unsigned)std::max<int64_t>(1, ceil_div(cols, SL_CH)), (unsigned)rows);
  oz_rowmax_kernel<<<grid, SL_T, 0, st>>>(X, ld, cols, scratch);
  DME_KCHECK();
  oz_slice_kernel<<<grid, SL_T, 0, st>>>(X, ld, cols, scratch, q, ldk, slice_stride, ex);
  DME_KCHECK();
}

int64_t oz_tiled_bytes(int64_t rows, int64_t cols) {
  return ceil_div(rows, 128) * ceil_div(cols, 128) * (int64_t)OZ_S * 16384;
}

void oz_slice_rows_tiled(const double* X, int64_t ld, int64_t rows, int64_t cols, int8_t* q,
                         int* ex, double* scratch, cudaStream_t st) {
  if (rows <= 0) return;
  DME_CUDA(cudaMemsetAsync(q, 0, (size_t)oz_tiled_bytes(rows, cols), st));
  const dim3 grid((unsigned)std::max<int64_t>(1, ceil_div(cols, SL_CH)), (unsigned)rows);
  oz_rowmax_kernel<<<grid, SL_T, 0, st>>>(X, ld, cols, scratch);
  DME_KCHECK();
  oz_slice_tiled_kernel<<<grid, SL_T, 0, st>>>(X, ld, cols, scratch, q, (int)ceil_div(cols, 128), ex);
  DME_KCHECK();
}

void oz_gemm(const OzGemmArgs& a, OzScratch& ws, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0) return;
  if (a.K > OZ_KMAX || a.K <= 0) throw std::runtime_error("oz_gemm: K out of range");
  if (a.tiles) {  // general N: 128 x 64 output tiles from the list
    launch_oz<64>(a, ws, st);
    return;
  }
  if (a.N > OZ_NMAX) throw std::runtime_error("oz_gemm: N > 64 without a tile list");
  const int np = (int)((a.N + 15) / 16 * 16);
  switch (np) {
    case 16: launch_oz<16>(a, ws, st); break;
    case 32: launch_oz<32>(a, ws, st); break;
    case 48: launch_oz<48>(a, ws, st); break;
    default: launch_oz<64>(a, ws, st); break;
  }
}

std::vector<int2> oz_tile_list(int64_t M, int64_t N, bool upper) {
  // 128 x 64 output tiles rasterised in bands of 8 row tiles (column-major inside a band), so
  // the ~#SM tiles in flight share few A row panels and B column panels (L2 reuse)
  const int RT = (int)ceil_div(M, 128), CT = (int)ceil_div(N, 64);
  constexpr int BAND = 8;
  std::vector<int2> t;
  for (int r0 = 0; r0 < RT; r0 += BAND)
    for (int ct = 0; ct < CT; ++ct)
      for (int rt = r0; rt < std::min(RT, r0 + BAND); ++rt)
        if (!upper || ct * 64 + 63 >= rt * 128) t.push_back(make_int2(rt, ct));
  return t;
}

}  // namespace dme
