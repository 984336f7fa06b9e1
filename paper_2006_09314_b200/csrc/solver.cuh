// Internal cross-file declarations (not ABI).
#pragma once
#include "ctx.cuh"

namespace fc {
void apply_plain(fc_ctx c, const SpecCP& sp, const fc_cp& x, fc_cp& y);
void cross_gram(cudaStream_t st, int n, int R1, const double* const X[3], const int ldx[3], int R2,
                const double* const Y[3], const int ldy[3], double* G);
double dot_plain(fc_ctx c, const fc_cp& x, const fc_cp& y);
void copy_cp_block(cudaStream_t st, int n, const fc_cp& src, fc_cp& dst, int col0, double scale);
void build_spectral_cp(fc_ctx c, int which, double alpha, double beta, double eps, int keep, bool spd_guard,
                       const double* lam3, const double* basis);
// FC_POW_PLUS / FC_POW_MINUS spectral CPs are built on first use (eps_D-driven, SL basis)
void ensure_spectral(fc_ctx c, int which);
void build_spectral_sinc(fc_ctx c, int which, double eps);
}  // namespace fc
