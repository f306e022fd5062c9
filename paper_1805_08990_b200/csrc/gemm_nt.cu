// FP64 "NT" GEMM on B200 tensor cores:  C[M x N] = alpha * A[M x K] * B[N x K]^T (+ beta Cin) (+ gamma I)
//
// The one contraction kernel of the hot path:
//   * T1 action  Y = E_tau * L           (A = E row-major, B^T = L column-major)  PAPER eq:F_sol_LDL
//   * T4 action  S*L, S*(S*L)            (A = S)                                  PAPER Alg. 4
//   * Gram       G = Zc^T Zc             (A = B = Zc^T, i.e. columns of Zc)       compression
//   * Taylor node passes W_j = (dA^T) W_{j-1} / j                                 quadrature (reading G6)
//   * Padé products / squarings X*Y  (B = Y^T, transposed copy)                   expm
// Both operands are K-contiguous, staged by TMA (cp.async.bulk.tensor, SWIZZLE_128B, 16-double
// K-slices) through an mbarrier ring, and multiplied with DMMA (mma.sync m8n8k4 f64; sm_100a has no
// tcgen05 FP64 kind). Work is split Stream-K style over exactly `grid` persistent CTAs
// (grid = #SMs): each CTA owns a contiguous range of (tile, k-iteration) pairs, so the HBM stream of
// A is divided evenly over all 148 SMs whatever M is. Tiles cut between CTAs are reduced
// DETERMINISTICALLY: every piece writes its accumulator to a slot, the last-arriving CTA sums the
// pieces in k-order (not arrival order) and runs the fused epilogue.
#include "common.cuh"
#include "gemm_nt.h"

#include <algorithm>
#include <atomic>
#include <vector>
#include <mutex>

namespace dme {

namespace {

constexpr int BM = 128;
constexpr int BK = 16;                       // one 128-byte swizzle row of doubles
constexpr int A_STAGE_BYTES = BM * BK * 8;   // 16 KB
constexpr int NUM_CONSUMERS = 256;           // 8 MMA warps
constexpr int NUM_THREADS = NUM_CONSUMERS + 32;

struct Params {
  int M, N, K, kiters, tiles_m, tiles_n;
  long long total;
  int grid;
  double alpha, beta, gamma;
  const double* cin;
  long long cin_rs, cin_cs;
  double* out;
  long long out_rs, out_cs;
  double* partial;
  int* counters;
  int b_nloc;  // >0: B tensor map is 3-D {nloc, N, G}; k -> (k % nloc, k / nloc)
  const int2* tile_list;  // non-null: tile t -> (tm, tn) = tile_list[t] (symmetric output: upper tiles)
  int ntiles;             // number of output tiles (list length, or tiles_m * tiles_n)
  int slices;  // >0: split-K slice mode (few tiles, long K): CTA b = (tile b % T, slice b / T),
               //     partials reduced by splitk_reduce_kernel; 0: Stream-K with last-arriver fixup
};

__device__ __forceinline__ long long iter_begin(long long c, const Params& p) {
  return c * p.total / p.grid;
}
__device__ __forceinline__ int cta_of(long long i, const Params& p) {
  // largest c with iter_begin(c) <= i
  return (int)(((i + 1) * p.grid + p.total - 1) / p.total - 1);
}

__device__ __forceinline__ void tile_coords(const Params& p, int tile, int& tm, int& tn) {
  if (p.tile_list) {
    const int2 c = p.tile_list[tile];
    tm = c.x;
    tn = c.y;
  } else {
    tm = tile % p.tiles_m;
    tn = tile / p.tiles_m;
  }
}

template <int BN>
__host__ __device__ constexpr int stages_for() {
  return (200 * 1024) / (A_STAGE_BYTES + BN * BK * 8) < 12 ? (200 * 1024) / (A_STAGE_BYTES + BN * BK * 8) : 12;
}

template <int BN, int WM, int WN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_nt_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const Params p) {
  constexpr int STAGES = stages_for<BN>();
  constexpr int B_STAGE_BYTES = BN * BK * 8;
  constexpr int MT = BM / WM / 8;   // m8 sub-tiles per warp
  constexpr int NTW = BN / WN / 8;  // n8 sub-tiles per warp
  constexpr int ACC = MT * NTW * 2;
  static_assert(WM * WN == 8, "8 MMA warps");

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;
  unsigned char* sB = smem + STAGES * A_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  __shared__ int s_last;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  long long beg, end;
  if (p.slices > 0) {
    const int T = p.ntiles;
    const long long tile = blockIdx.x % T, sl = blockIdx.x / T;
    beg = tile * p.kiters + sl * p.kiters / p.slices;
    end = tile * p.kiters + (sl + 1) * p.kiters / p.slices;
  } else {
    beg = iter_begin(blockIdx.x, p);
    end = iter_begin(blockIdx.x + 1, p);
  }

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NUM_CONSUMERS / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NUM_CONSUMERS / 32) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      int stage = 0;
      uint32_t phase = 0;
      for (long long it = beg; it < end; ++it) {
        const int tile = (int)(it / p.kiters), kk = (int)(it % p.kiters);
        int tm, tn;
        tile_coords(p, tile, tm, tn);
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], A_STAGE_BYTES + B_STAGE_BYTES);
        tma_load_2d(sA + stage * A_STAGE_BYTES, &tmA, &full[stage], kk * BK, tm * BM);
        if (p.b_nloc > 0) {
          const int k0 = kk * BK;
          tma_load_3d(sB + stage * B_STAGE_BYTES, &tmB, &full[stage], k0 % p.b_nloc, tn * BN,
                      k0 / p.b_nloc);
        } else {
          tma_load_2d(sB + stage * B_STAGE_BYTES, &tmB, &full[stage], kk * BK, tn * BN);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ DMMA consumers
  const int g = lane >> 2, t = lane & 3;
  const int pg = frag_perm(g);
  const int wm = warp % WM, wn = warp / WM;
  const int wm_base = wm * (BM / WM), wn_base = wn * (BN / WN);
  const uint32_t sA_u = smem_u32(sA), sB_u = smem_u32(sB);
  // per-thread byte offsets inside a stage (swizzle: chunk ^ (row & 7) with row & 7 == pg)
  uint32_t offA[MT], offB[NTW];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi) offA[mi] = (wm_base + mi * 8 + pg) * 128;
#pragma unroll
  for (int ni = 0; ni < NTW; ++ni) offB[ni] = (wn_base + ni * 8 + pg) * 128;
  double acc[ACC];
  int stage = 0;
  uint32_t phase = 0;
  long long it = beg;
  while (it < end) {
    const int tile = (int)(it / p.kiters);
    const long long tile_beg = (long long)tile * p.kiters, tile_end = tile_beg + p.kiters;
    const long long stop = end < tile_end ? end : tile_end;
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = 0.0;
    for (; it < stop; ++it) {
      mbar_wait(&full[stage], phase);
      const uint32_t a = sA_u + stage * A_STAGE_BYTES;
      const uint32_t b = sB_u + stage * B_STAGE_BYTES;
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        const uint32_t off = ((((ks << 1) + (t >> 1)) ^ pg) << 4) + ((t & 1) << 3);
        double af[MT], bf[NTW];
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) af[mi] = lds_f64(a + offA[mi] + off);
#pragma unroll
        for (int ni = 0; ni < NTW; ++ni) bf[ni] = lds_f64(b + offB[ni] + off);
#pragma unroll
        for (int mi = 0; mi < MT; ++mi)
#pragma unroll
          for (int ni = 0; ni < NTW; ++ni)
            dmma_8x8x4(acc[(mi * NTW + ni) * 2], acc[(mi * NTW + ni) * 2 + 1], af[mi], bf[ni]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }

    // -------------------------------------------------------------- epilogue
    int tm, tn;
    tile_coords(p, tile, tm, tn);
    bool do_store = true;
    if (p.slices > 0) {
      // slice mode: publish the partial (fragment order); splitk_reduce_kernel sums in slice order
      double* myslot = p.partial + (size_t)blockIdx.x * (BM * BN);
#pragma unroll
      for (int i = 0; i < ACC; ++i) myslot[i * NUM_CONSUMERS + tid] = acc[i];
      do_store = false;
    } else if (!(beg <= tile_beg && end >= tile_end)) {
      // tile split between CTAs: publish this piece, last arriver reduces in k-order
      const int c_first = cta_of(tile_beg, p), c_last = cta_of(tile_end - 1, p);
      const int np = c_last - c_first + 1, me = (int)blockIdx.x - c_first;
      auto slot_of = [&](int c) {
        return 2 * c + (iter_begin(c, p) / p.kiters == tile ? 0 : 1);
      };
      double* myslot = p.partial + (size_t)slot_of(blockIdx.x) * (BM * BN);
#pragma unroll
      for (int i = 0; i < ACC; ++i) myslot[i * NUM_CONSUMERS + tid] = acc[i];
      __threadfence();
      named_bar_sync(1, NUM_CONSUMERS);
      if (tid == 0) s_last = (atomicAdd(&p.counters[tile], 1) == np - 1);
      named_bar_sync(1, NUM_CONSUMERS);
      do_store = s_last;
      if (do_store) {
        __threadfence();
        // sum every piece (own one included, re-read from its slot) in k-order
        for (int q = 0; q < np; ++q) {
          const double* src = p.partial + (size_t)slot_of(c_first + q) * (BM * BN);
#pragma unroll
          for (int i = 0; i < ACC; ++i) {
            const double v = __ldcg(src + i * NUM_CONSUMERS + tid);
            acc[i] = q == 0 ? v : acc[i] + v;
          }
        }
        (void)me;
        if (tid == 0) p.counters[tile] = 0;
      }
    }
    if (do_store) {
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NTW; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const long long row = (long long)tm * BM + wm_base + mi * 8 + pg;
            const long long col = (long long)tn * BN + wn_base + ni * 8 + frag_perm(t * 2 + e);
            if (row < p.M && col < p.N) {
              double v = p.alpha * acc[(mi * NTW + ni) * 2 + e];
              if (p.beta != 0.0) v += p.beta * p.cin[row * p.cin_rs + col * p.cin_cs];
              if (row == col) v += p.gamma;
              p.out[row * p.out_rs + col * p.out_cs] = v;
            }
          }
    }
  }
}

// out = epilogue(sum over slices, in slice order, of the fragment-order partials)
template <int BN, int WM, int WN>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const Params p) {
  constexpr int MT = BM / WM / 8, NTW = BN / WN / 8, ACC = MT * NTW * 2;
  const int T = p.ntiles;
  const long long total = (long long)T * ACC * NUM_CONSUMERS;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int tid = (int)(e % NUM_CONSUMERS);
    const int i = (int)((e / NUM_CONSUMERS) % ACC);
    const int tile = (int)(e / ((long long)NUM_CONSUMERS * ACC));
    // fixed association (deterministic): 8 interleaved partial sums over the slices, combined in
    // a fixed tree; the 8 independent loads of a round are in flight together (the reduction was
    // bound by one L2 round trip per slice)
    const double* src = p.partial + (size_t)tile * (BM * BN) + i * NUM_CONSUMERS + tid;
    const size_t sstride = (size_t)T * (BM * BN);
    double s8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int sl = 0;
    for (; sl + 8 <= p.slices; sl += 8) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldcg(src + (size_t)(sl + u) * sstride);
#pragma unroll
      for (int u = 0; u < 8; ++u) s8[u] += x[u];
    }
    for (int u = 0; sl < p.slices; ++sl, ++u) s8[u] += __ldcg(src + (size_t)sl * sstride);
    const double acc = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wm = warp % WM, wn = warp / WM;
    const int el = i & 1, mn = i >> 1, mi = mn / NTW, ni = mn % NTW;
    int tm, tn;
    tile_coords(p, tile, tm, tn);
    const long long row = (long long)tm * BM + wm * (BM / WM) + mi * 8 + frag_perm(g);
    const long long col = (long long)tn * BN + wn * (BN / WN) + ni * 8 + frag_perm(t * 2 + el);
    if (row < p.M && col < p.N) {
      double v = p.alpha * acc;
      if (p.beta != 0.0) v += p.beta * p.cin[row * p.cin_rs + col * p.cin_cs];
      if (row == col) v += p.gamma;
      p.out[row * p.out_rs + col * p.out_cs] = v;
    }
  }
}

template <int BN, int WM, int WN>
void launch(const GemmNTArgs& a, const Params& p0, GemmScratch& ws, cudaStream_t st) {
  constexpr int STAGES = stages_for<BN>();
  const size_t smem = 1024 + STAGES * (A_STAGE_BYTES + BN * BK * 8) + 2 * STAGES * 8;
  static std::once_flag once;
  std::call_once(once, [&] {
    DME_CUDA(cudaFuncSetAttribute(gemm_nt_kernel<BN, WM, WN>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  Params p = p0;
  const CUtensorMap tmA = make_tmap_2d(a.A, a.K, a.M, a.lda, BK, BM, true);
  CUtensorMap tmB;
  if (a.b_nloc > 0) {
    const int64_t G = a.K / a.b_nloc;
    tmB = make_tmap_3d(a.B, a.b_nloc, a.N, G, a.ldb, a.b_blockstride, BK, BN, 1, true);
    p.b_nloc = (int)a.b_nloc;
  } else {
    tmB = make_tmap_2d(a.B, a.K, a.N, a.ldb, BK, BN, true);
    p.b_nloc = 0;
  }
  gemm_nt_kernel<BN, WM, WN><<<p.grid, NUM_THREADS, smem, st>>>(tmA, tmB, p);
  DME_KCHECK();
  if (p.slices > 0) {
    constexpr int ACC = (BM / WM / 8) * (BN / WN / 8) * 2;
    const long long total = (long long)p.ntiles * ACC * NUM_CONSUMERS;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 4 * num_sms());
    splitk_reduce_kernel<BN, WM, WN><<<blocks, 256, 0, st>>>(p);
    DME_KCHECK();
  }
}

}  // namespace

size_t GemmScratch::partial_doubles(int grid) { return size_t(2) * grid * BM * 64; }

void gemm_nt(const GemmNTArgs& a, GemmScratch& ws, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0) return;
  if (a.K <= 0) throw std::runtime_error("gemm_nt: K must be positive");
  if ((a.lda & 1) || (a.ldb & 1) || (reinterpret_cast<uintptr_t>(a.A) & 15) ||
      (reinterpret_cast<uintptr_t>(a.B) & 15))
    throw std::runtime_error("gemm_nt: operands must be 16-byte aligned with even leading dims");
  Params p{};
  p.M = (int)a.M;
  p.N = (int)a.N;
  p.K = (int)a.K;
  p.kiters = (int)ceil_div(a.K, BK);
  // BN = 128 would need > 168 registers/thread (9 warps -> 3 per SMSP): N > 64 uses 64-wide N tiles.
  // Narrow N (the factor width k) gets a tile that wastes < 8 columns of DMMA work.
  int BN = a.N <= 8 ? 8 : a.N <= 16 ? 16 : a.N <= 24 ? 24 : a.N <= 32 ? 32 : a.N <= 40 ? 40
         : a.N <= 48 ? 48 : a.N <= 56 ? 56 : 64;
  p.tiles_m = (int)ceil_div(a.M, BM);
  p.tiles_n = (int)ceil_div(a.N, BN);
  long long tiles = (long long)p.tiles_m * p.tiles_n;
  p.tile_list = nullptr;
  if (a.sym_upper) {
    // only tiles touching the upper triangle (row <= col); the caller mirrors the lower triangle
    std::vector<int2> lst;
    for (int tn = 0; tn < p.tiles_n; ++tn)
      for (int tm = 0; tm < p.tiles_m; ++tm)
        if ((long long)tm * BM <= (long long)tn * BN + BN - 1) lst.push_back(make_int2(tm, tn));
    if ((long long)lst.size() > ws.max_tiles) throw std::runtime_error("gemm_nt: tile list too long");
    DME_CUDA(cudaMemcpyAsync(ws.tile_list, lst.data(), lst.size() * sizeof(int2),
                             cudaMemcpyHostToDevice, st));
    p.tile_list = ws.tile_list;
    tiles = (long long)lst.size();
  }
  p.total = tiles * p.kiters;
  p.ntiles = (int)tiles;
  const int sms = std::min<int>(num_sms(), ws.max_grid);
  p.slices = 0;
  if (tiles * 4 <= sms && p.kiters >= 16) {
    // few output tiles over a long K (Gram matrices Zc^T Zc): parallel split-K reduction
    p.slices = (int)std::min<long long>(sms / tiles, p.kiters / 8);
    p.grid = (int)(tiles * p.slices);
  } else {
    const long long want = std::max<long long>(1, p.total / 4);
    p.grid = (int)std::min<long long>(sms, want);
  }
  p.alpha = a.alpha;
  p.beta = a.beta;
  p.gamma = a.gamma;
  p.cin = a.cin ? a.cin : a.out;
  p.cin_rs = a.cin ? a.cin_rs : a.out_rs;
  p.cin_cs = a.cin ? a.cin_cs : a.out_cs;
  p.out = a.out;
  p.out_rs = a.out_rs;
  p.out_cs = a.out_cs;
  p.partial = ws.partial;
  p.counters = ws.counters;
  if ((long long)p.tiles_m * p.tiles_n > ws.max_tiles)
    throw std::runtime_error("gemm_nt: too many tiles for the scratch counters");
  switch (BN) {
    case 8: launch<8, 8, 1>(a, p, ws, st); break;
    case 16: launch<16, 8, 1>(a, p, ws, st); break;
    case 24: launch<24, 8, 1>(a, p, ws, st); break;
    case 32: launch<32, 4, 2>(a, p, ws, st); break;
    case 40: launch<40, 8, 1>(a, p, ws, st); break;
    case 48: launch<48, 4, 2>(a, p, ws, st); break;
    case 56: launch<56, 8, 1>(a, p, ws, st); break;
    default: launch<64, 4, 2>(a, p, ws, st); break;
  }
}

// ------------------------------------------------------------------ tensor maps
namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    DME_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess)
      throw std::runtime_error("cuTensorMapEncodeTiled not available");
    return reinterpret_cast<EncodeFn>(f);
  }();
  return fn;
}
}  // namespace

CUtensorMap make_tmap_2d(const double* base, uint64_t inner, uint64_t outer, uint64_t stride,
                         uint32_t box_inner, uint32_t box_outer, bool swz) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {stride * 8};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled(2d) failed: " + std::to_string(r));
  return m;
}

CUtensorMap make_tmap_3d(const double* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                         uint64_t s2, uint32_t b0, uint32_t b1, uint32_t b2, bool swz) {
  CUtensorMap m;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1 * 8, s2 * 8};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled(3d) failed: " + std::to_string(r));
  return m;
}

CUtensorMap make_tmap_3d_u8(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_bytes,
                            uint64_t s2_bytes, uint32_t b0, uint32_t b1, uint32_t b2) {
  CUtensorMap m;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1_bytes, s2_bytes};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides,
                           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled(3d u8) failed: " + std::to_string(r));
  return m;
}

namespace {
std::atomic<int64_t> g_launches{0};
}
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

int num_sms() {
  static int n = [] {
    int dev = 0, v = 0;
    DME_CUDA(cudaGetDevice(&dev));
    DME_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    return v;
  }();
  return n;
}

}  // namespace dme
