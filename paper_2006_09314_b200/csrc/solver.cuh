// Internal cross-file declarations (not ABI).
#pragma once
#include "ctx.cuh"

namespace fc {
void apply_plain(fc_ctx c, const SpecCP& sp, const fc_cp& x, fc_cp& y);
void cross_gram(cudaStream_t st, int n, int R1, const double* const X[3], const int ldx[3], int R2,
                const double* const Y[3], const int ldy[3], double* G);
double dot_plain(fc_ctx c, const fc_cp& x, const fc_cp& y);
void copy_cp_block(cudaStream_t st, int n, const fc_cp& src, fc_cp& dst, int col0, double scale);
}  // namespace fc
