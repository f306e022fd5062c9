#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

#include "gemm_nt.h"

namespace dme {

// dst (cols x rows, row-major ldd) = src^T, src rows x cols row-major (lds)
void transpose_rect(const double* src, int64_t rows, int64_t cols, int64_t lds, double* dst,
                    int64_t ldd, cudaStream_t st);
size_t lu_scratch_doubles(int64_t n);
// In place: Q <- its LU factors with partial pivoting (Pi Q = L U), P <- P Q^{-1}.
// QT: n x n scratch (ld). *minpiv_dev <- min |u_ii| (0: Q singular).
void lu_solve_right(double* Q, double* P, int64_t n, int64_t ld, double* QT, double* scratch,
                          GemmScratch& gs, cudaStream_t st, double* minpiv_dev);

}  // namespace dme
