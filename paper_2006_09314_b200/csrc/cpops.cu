// Elementwise / reduction kernels of the CP algebra (S6 weights, S8 normalisation, S9 axpy,
// S10 cp_dot) [P:1748-1763].  All FP64, coalesced column-major access.
#include "cpops.cuh"

namespace fc {
namespace {

__global__ void square_kernel(Mat3 in, Mat3 out) {
  const int l = blockIdx.y;
  const int rows = in.rows[l], cols = in.cols[l];
  const long long total = (long long)rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx % rows), c = (int)(idx / rows);
    double v = in.p[l][(size_t)i + (size_t)c * in.ld[l]];
    out.p[l][(size_t)i + (size_t)c * out.ld[l]] = v * v;
  }
}

// t = k*R + j: nrm_l = sqrt(N2_l[k + j*r]); w_out[t] = wF[k]*wx[j]*prod_l nrm_l;
// colscale_l[t] = 1/nrm_l (0 for a zero column).
__global__ void apply_weights_kernel(int r, int R, const double* wF, const double* wx, const double* N2a,
                                     const double* N2b, const double* N2c, double* wout, double* csa,
                                     double* csb, double* csc) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= r * R) return;
  int k = t / R, j = t - k * R;
  int q = k + j * r;
  double na = sqrt(N2a[q]), nb = sqrt(N2b[q]), nc = sqrt(N2c[q]);
  wout[t] = wF[k] * wx[j] * na * nb * nc;
  csa[t] = na > 0 ? 1.0 / na : 0.0;
  csb[t] = nb > 0 ? 1.0 / nb : 0.0;
  csc[t] = nc > 0 ? 1.0 / nc : 0.0;
}

// out[blockIdx.x] = partial of sum_{k,m} wx[k] wy[m] G0[k,m] G1[k,m] G2[k,m]  (grid-stride,
// deterministic: a fixed grid and a second single-block pass over the partials)
__global__ void dot_reduce_kernel(int R1, int R2, const double* wx, const double* wy, const double* G0,
                                  const double* G1, const double* G2, int ld, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  const long long total = (long long)R1 * R2;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int k = (int)(idx % R1), m = (int)(idx / R1);
    size_t o = (size_t)k + (size_t)m * ld;
    acc += wx[k] * wy[m] * (G0[o] * G1[o] * G2[o]);
  }
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
    if (threadIdx.x == 0) out[blockIdx.x] = v;
  }
}

__global__ void sum_kernel(int n, const double* __restrict__ x, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += x[i];
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
    if (threadIdx.x == 0) *out = v;
  }
}

__global__ void copy_cols_kernel(Mat3 src, Mat3 dst, double scale) {
  const int l = blockIdx.y;
  const int rows = src.rows[l], cols = src.cols[l];
  const long long total = (long long)rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx % rows), c = (int)(idx / rows);
    dst.p[l][(size_t)i + (size_t)c * dst.ld[l]] = scale * src.p[l][(size_t)i + (size_t)c * src.ld[l]];
  }
}

__global__ void scale_copy_kernel(int n, const double* x, double a, double* y) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = a * x[i];
}

}  // namespace

static int grid_for(long long total, int threads = 256) {
  long long b = (total + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  return (int)std::max<long long>(b, 1);
}

void square3(const Mat3& in, const Mat3& out, cudaStream_t st) {
  long long mx = 0;
  for (int l = 0; l < 3; ++l) mx = std::max(mx, (long long)in.rows[l] * in.cols[l]);
  if (mx == 0) return;
  square_kernel<<<dim3(grid_for(mx), 3), 256, 0, st>>>(in, out);
  FC_CHECK_LAUNCH();
}

void apply_weights(int r, int R, const double* wF, const double* wx, const double* const N2[3], double* wout,
                   double* const cs[3], cudaStream_t st) {
  int total = r * R;
  if (total == 0) return;
  apply_weights_kernel<<<cdiv(total, 256), 256, 0, st>>>(r, R, wF, wx, N2[0], N2[1], N2[2], wout, cs[0], cs[1],
                                                         cs[2]);
  FC_CHECK_LAUNCH();
}

void dot_reduce(int R1, int R2, const double* wx, const double* wy, const double* const G[3], int ld,
                double* out_dev, cudaStream_t st) {
  const long long total = (long long)R1 * R2;
  const int nb = (int)std::min<long long>(std::max<long long>((total + 8191) / 8192, 1), 296);
  double* part = nullptr;
  FC_CUDA_TRY(cudaMallocAsync(&part, (size_t)nb * sizeof(double), st));
  dot_reduce_kernel<<<nb, 512, 0, st>>>(R1, R2, wx, wy, G[0], G[1], G[2], ld, part);
  FC_CHECK_LAUNCH();
  sum_kernel<<<1, 512, 0, st>>>(nb, part, out_dev);
  FC_CHECK_LAUNCH();
  FC_CUDA_TRY(cudaFreeAsync(part, st));
}

void copy_cols3(const Mat3& src, const Mat3& dst, double scale, cudaStream_t st) {
  long long mx = 0;
  for (int l = 0; l < 3; ++l) mx = std::max(mx, (long long)src.rows[l] * src.cols[l]);
  if (mx == 0) return;
  copy_cols_kernel<<<dim3(grid_for(mx), 3), 256, 0, st>>>(src, dst, scale);
  FC_CHECK_LAUNCH();
}

void scale_copy(int n, const double* x, double a, double* y, cudaStream_t st) {
  if (n <= 0) return;
  scale_copy_kernel<<<cdiv(n, 256), 256, 0, st>>>(n, x, a, y);
  FC_CHECK_LAUNCH();
}

}  // namespace fc
