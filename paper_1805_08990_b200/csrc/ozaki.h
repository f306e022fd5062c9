// E·Y on the int8 tensor cores (tcgen05.mma kind::i8) by exact digit slicing (Ozaki scheme).
//
// Every row of E and every column of Y is scaled by a power of two to |x| <= 1/2 and split into
// OZ_S signed 7-bit digits, x = sum_a d_a 2^{-7a} + O(2^{-7 OZ_S}), |d_a| <= 64. The products
// sum_l d_a(E_il) d_b(Y_lj) are exact in int32 (|d_a d_b| <= 2^12, K <= OZ_KMAX, <= OZ_S pairs per
// accumulator), and (E Y)_ij = 2^{e_i + f_j} sum_{a+b <= OZ_S+1} 2^{-7(a+b)} (D_a Y_b)_ij is
// assembled in FP64. The dropped digits and pairs bound the error per entry by about
// 2^{-7 OZ_S + 2} max_l|E_il| sum_l|Y_lj| (2^-54 relative for OZ_S = 8): FP64-level accuracy for the
// E pass. E is sliced once at init (it is fixed for the whole run),
// Y once per pass.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <vector>

namespace dme {

constexpr int OZ_S = 8;                // digits per operand
constexpr int OZ_NMAX = 64;            // columns of Y per pass (TMEM: OZ_S * 64 = 512 columns)
constexpr int64_t OZ_KMAX = 32768;     // int32 accumulation bound: OZ_S * 2^12 * K < 2^31

inline int64_t oz_ldk(int64_t cols) { return (cols + 15) / 16 * 16; }

// Row-wise digit slicing of a row-major FP64 matrix X (rows x cols, row stride ld):
// q[s * slice_stride + i * ldk + l] = digit s of X[i][l] * 2^{-ex[i]}, ex[i] = ilogb(max_l |X_il|) + 2
// (0 for a zero row). Columns cols..round4(cols)-1 are written as zero digits.
// scratch: oz_slice_scratch_doubles(rows, cols) doubles (per-chunk row maxima)
void oz_slice_rows(const double* X, int64_t ld, int64_t rows, int64_t cols, int8_t* q, int64_t ldk,
                   int64_t slice_stride, int* ex, double* scratch, cudaStream_t st);
int64_t oz_slice_scratch_doubles(int64_t rows, int64_t cols);

struct OzScratch {
  double* partial = nullptr;  // partial_doubles(max_tiles, max_grid)
  int* counters = nullptr;    // max_tiles ints, zero-initialised once (reset by the kernel)
  int max_grid = 0;
  int64_t max_tiles = 0;
  static size_t partial_doubles(int64_t tiles, int grid) {  // two split-tile slots per CTA
    (void)tiles;
    return (size_t)2 * grid * OZ_NMAX * 128;
  }
};

struct OzGemmArgs {
  const int8_t* A = nullptr;   // digit slices of the rows of E: [OZ_S][M][lda] bytes
  const int* eA = nullptr;     // M row exponents
  int64_t lda = 0, a_slice_stride = 0;
  const int8_t* B = nullptr;   // digit slices of the columns of Y: [OZ_S][>= round16(N)][ldb]
  const int* eB = nullptr;     // N column exponents
  int64_t ldb = 0, b_slice_stride = 0;
  int64_t M = 0, N = 0, K = 0;
  double alpha = 1.0;
  double* out = nullptr;       // element (i, j) at out + i*out_rs + j*out_cs
  int64_t out_rs = 0, out_cs = 0;
  // square GEMMs: 128 x 64 output tiles from a device list (oz_tile_list), B holds the digits of
  // all N columns, whole tiles round-robin over the CTAs (round_robin = true)
  const int2* tiles = nullptr;
  int ntiles = 0;
  bool round_robin = false;
  // E pass: A digits in the tiled, pre-swizzled image of oz_slice_rows_tiled (A, lda and
  // a_slice_stride unused); streamed with plain 16 KB bulk copies instead of tensor-map TMA
  const int8_t* A_tiled = nullptr;
};

// Tiled digit image of a row-major FP64 matrix (rows x cols): bytes needed, and the slicing
// (clears the image first, then writes digits + per-row exponents ex[rows]; scratch as above).
int64_t oz_tiled_bytes(int64_t rows, int64_t cols);
void oz_slice_rows_tiled(const double* X, int64_t ld, int64_t rows, int64_t cols, int8_t* q,
                         int* ex, double* scratch, cudaStream_t st);

// out = alpha * E * Y (K <= OZ_KMAX). Without a tile list (N <= OZ_NMAX): persistent Stream-K
// over 128-row tiles x 128-deep K chunks, deterministic in-kernel fixup of split tiles. With a
// tile list: any N, whole 128 x 64 tiles.
void oz_gemm(const OzGemmArgs& a, OzScratch& ws, cudaStream_t st);
// host: rasterised 128 x 64 tile list of an M x N output (upper: tiles meeting col >= row only)
std::vector<int2> oz_tile_list(int64_t M, int64_t N, bool upper);

}  // namespace dme
