#pragma once
#include "common.cuh"

namespace fc {

// Three column-major matrices (one per mode), passed by value to kernels.
struct Mat3 {
  double* p[3];
  int ld[3];
  int rows[3];
  int cols[3];
};

struct Cmat3 {
  const double* p[3];
};

// K6: Y_l[:, k R + j] = U_l[:, k] (.) W_l[:, j], l = 0..2 (n x r, n x R -> n x rR, ld n)
void kr_product3(int n, int r, int R, const double* const U[3], const double* const W[3], double* const Y[3],
                 cudaStream_t st);
void square3(const Mat3& in, const Mat3& out, cudaStream_t st);
void apply_weights(int r, int R, const double* wF, const double* wx, const double* const N2[3], double* wout,
                   double* const cs[3], cudaStream_t st);
void dot_reduce(int R1, int R2, const double* wx, const double* wy, const double* const G[3], int ld,
                double* out_dev, cudaStream_t st);
void copy_cols3(const Mat3& src, const Mat3& dst, double scale, cudaStream_t st);
void scale_copy(int n, const double* x, double a, double* y, cudaStream_t st);

}  // namespace fc
