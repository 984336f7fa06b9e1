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

void square3(const Mat3& in, const Mat3& out, cudaStream_t st);
void apply_weights(int r, int R, const double* wF, const double* wx, const double* const N2[3], double* wout,
                   double* const cs[3], cudaStream_t st);
void dot_reduce(int R1, int R2, const double* wx, const double* wy, const double* const G[3], int ld,
                double* out_dev, cudaStream_t st);
void copy_cols3(const Mat3& src, const Mat3& dst, double scale, cudaStream_t st);
void scale_copy(int n, const double* x, double a, double* y, cudaStream_t st);

}  // namespace fc
