// Elementwise / reduction kernels of the CP algebra (S6 weights, S8 normalisation, S9 axpy,
// S10 cp_dot) [P:1748-1763].  All FP64, coalesced column-major access.
#include <mutex>
#include <vector>
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
// deterministic: a fixed grid and a second single-block pass over the partials).  HBM-bound
// (K9, 24 bytes per (k, m) entry): contiguous Grams (ld == R1) are streamed as 16-byte double2
// loads, two per operand in flight per thread; strided Grams take the scalar loop.
__global__ void dot_reduce_kernel(int R1, int R2, const double* __restrict__ wx, const double* __restrict__ wy,
                                  const double* __restrict__ G0, const double* __restrict__ G1,
                                  const double* __restrict__ G2, int ld, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  const long long total = (long long)R1 * R2;
  const long long nth = (long long)gridDim.x * blockDim.x, t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (ld == R1 && ((reinterpret_cast<size_t>(G0) | reinterpret_cast<size_t>(G1) | reinterpret_cast<size_t>(G2)) & 15) == 0) {
    const long long npair = total >> 1;
    const double2* A = reinterpret_cast<const double2*>(G0);
    const double2* B = reinterpret_cast<const double2*>(G1);
    const double2* Cc = reinterpret_cast<const double2*>(G2);
    auto term = [&](long long idx, double g) {
      const long long m = idx / R1, k = idx - m * R1;
      return wx[k] * wy[m] * g;
    };
    long long p = t0;
    for (; p + nth < npair; p += 2 * nth) {   // two pairs per operand in flight
      const double2 a0 = __ldcs(A + p), b0 = __ldcs(B + p), c0 = __ldcs(Cc + p);
      const double2 a1 = __ldcs(A + p + nth), b1 = __ldcs(B + p + nth), c1 = __ldcs(Cc + p + nth);
      acc += term(2 * p, a0.x * b0.x * c0.x);
      acc += term(2 * p + 1, a0.y * b0.y * c0.y);
      acc += term(2 * (p + nth), a1.x * b1.x * c1.x);
      acc += term(2 * (p + nth) + 1, a1.y * b1.y * c1.y);
    }
    for (; p < npair; p += nth) {
      const double2 a0 = __ldcs(A + p), b0 = __ldcs(B + p), c0 = __ldcs(Cc + p);
      acc += term(2 * p, a0.x * b0.x * c0.x);
      acc += term(2 * p + 1, a0.y * b0.y * c0.y);
    }
    if ((total & 1) && t0 == 0) acc += term(total - 1, G0[total - 1] * G1[total - 1] * G2[total - 1]);
  } else {
    for (long long idx = t0; idx < total; idx += nth) {
      int k = (int)(idx % R1), m = (int)(idx / R1);
      size_t o = (size_t)k + (size_t)m * ld;
      acc += wx[k] * wy[m] * (G0[o] * G1[o] * G2[o]);
    }
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

// K6 (S6) [P:604-605, P:1756-1763]: Y_l[:, k R + j] = U_l[:, k] (.) W_l[:, j] (n x r R per
// mode, blockIdx.y = mode), 16-byte loads / streaming stores along n when n is even and the
// blocks are 16-byte aligned; HBM-write-bound (U and W are re-read from L2)
__global__ void kr_product_kernel(int n, int r, int R, Cmat3 U, Cmat3 W, Mat3 Y) {
  const int l = blockIdx.y;
  const double* __restrict__ u = U.p[l];
  const double* __restrict__ w = W.p[l];
  double* y = Y.p[l];
  const int cols = r * R;
  const size_t al = reinterpret_cast<size_t>(u) | reinterpret_cast<size_t>(w) | reinterpret_cast<size_t>(y);
  if ((n & 1) == 0 && (al & 15) == 0) {
    // a warp per output column at a time: column index math once per column, 16-byte
    // coalesced loads of u_k, w_j (L2) and streaming stores of y_c along n
    const int n2 = n >> 1, lane = threadIdx.x & 31;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int c = wid; c < cols; c += nw) {
      const int k = c / R, j = c - k * R;
      const double2* a = reinterpret_cast<const double2*>(u + (size_t)k * n);
      const double2* b = reinterpret_cast<const double2*>(w + (size_t)j * n);
      double2* o = reinterpret_cast<double2*>(y + (size_t)c * n);
#pragma unroll 4
      for (int i2 = lane; i2 < n2; i2 += 32) {
        const double2 x = __ldg(a + i2), z = __ldg(b + i2);
        __stcs(o + i2, make_double2(x.x * z.x, x.y * z.y));
      }
    }
    return;
  }
  const long long tot = (long long)n * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long c = idx / n;
    const int i = (int)(idx - c * n), k = (int)(c / R), j = (int)(c - (long long)k * R);
    y[idx] = u[i + (size_t)k * n] * w[i + (size_t)j * n];
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

void kr_product3(int n, int r, int R, const double* const U[3], const double* const W[3], double* const Y[3],
                 cudaStream_t st) {
  const long long tot = (long long)n * r * R;
  if (tot == 0) return;
  Cmat3 u{}, w{};
  Mat3 y{};
  for (int l = 0; l < 3; ++l) {
    u.p[l] = U[l];
    w.p[l] = W[l];
    y.p[l] = Y[l];
  }
  // a warp per column, 8 warps per CTA; ~8 resident CTAs per SM over the 3 modes
  const long long cols = (long long)r * R;
  const int gx = (int)std::max<long long>(1, std::min<long long>((cols + 7) / 8, 148 * 8 / 3 + 1));
  KProfScope kp(KP_KR_PRODUCT, st, 3.0 * 8.0 * ((double)tot + (double)n * (r + R)));
  kr_product_kernel<<<dim3(gx, 3), 256, 0, st>>>(n, r, R, u, w, y);
  FC_CHECK_LAUNCH();
}

void dot_reduce(int R1, int R2, const double* wx, const double* wy, const double* const G[3], int ld,
                double* out_dev, cudaStream_t st) {
  const long long total = (long long)R1 * R2;
  // up to 8 CTAs of 256 threads per SM (148 SMs), ~4 entries per thread and pass at least
  const int nb = (int)std::min<long long>(std::max<long long>((total + 4095) / 4096, 1), 148 * 8);
  double* part = nullptr;
  FC_CUDA_TRY(cudaMallocAsync(&part, (size_t)nb * sizeof(double), st));
  {
    KProfScope kp(KP_DOT_REDUCE, st, 24.0 * (double)total + 8.0 * (R1 + R2));
    dot_reduce_kernel<<<nb, 256, 0, st>>>(R1, R2, wx, wy, G[0], G[1], G[2], ld, part);
    FC_CHECK_LAUNCH();
  }
  sum_kernel<<<1, 512, 0, st>>>(nb, part, out_dev);
  FC_CHECK_LAUNCH();
  FC_CUDA_TRY(cudaFreeAsync(part, st));
}

// ---- fc_profile_kernel: per-kernel events + algorithmic bytes (opt-in; see common.cuh) ----
namespace {
struct KProf {
  std::mutex mu;
  bool on = false;
  std::vector<cudaEvent_t> ev;   // pairs, recycled
  std::vector<double> bytes;
  size_t used = 0;
};
KProf& kprof(int id) {
  static KProf p[KP_COUNT];
  return p[id];
}
}  // namespace

KProfScope::KProfScope(int id_, cudaStream_t st_, double bytes_) : id(id_), st(st_), bytes(bytes_) {
  KProf& P = kprof(id);
  on = P.on;
  if (!on) return;
  std::lock_guard<std::mutex> lock(P.mu);
  if (P.ev.size() < 2 * (P.used + 1))
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      FC_CUDA_TRY(cudaEventCreate(&e));
      P.ev.push_back(e);
    }
  FC_CUDA_TRY(cudaEventRecord(P.ev[2 * P.used], st));
}

KProfScope::~KProfScope() {
  if (!on) return;
  KProf& P = kprof(id);
  std::lock_guard<std::mutex> lock(P.mu);
  cudaEventRecord(P.ev[2 * P.used + 1], st);
  P.bytes.push_back(bytes);
  ++P.used;
}

void kprof_read(int id, bool enable, double* ms, double* bytes, long long* launches) {
  require(id >= 0 && id < KP_COUNT, FC_ERR_INVALID_ARG, "kernel id");
  KProf& P = kprof(id);
  std::lock_guard<std::mutex> lock(P.mu);
  if (enable) {
    P.on = true;
    P.used = 0;
    P.bytes.clear();
    return;
  }
  P.on = false;
  double t = 0, b = 0;
  for (size_t i = 0; i < P.used; ++i) {
    float x = 0;
    FC_CUDA_TRY(cudaEventSynchronize(P.ev[2 * i + 1]));
    FC_CUDA_TRY(cudaEventElapsedTime(&x, P.ev[2 * i], P.ev[2 * i + 1]));
    t += x;
    b += P.bytes[i];
  }
  if (ms) *ms = t;
  if (bytes) *bytes = b;
  if (launches) *launches = (long long)P.used;
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
