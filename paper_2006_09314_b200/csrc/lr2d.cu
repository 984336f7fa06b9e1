// The 2D variant of the method: A = T1 (x) I + I (x) T2, iterates are
// low-rank matrices X = U0 diag(w) U1^T [P:585-595], the operator is the factored apply
// [P:597-611], the truncation is the reduced SVD [P:973-976], and the solver is the same
// Algorithm 1 [P:1825-1872] ("independent of d" [P:962-969]).
//
// Device pieces (all reused from the 3D path except the small kernels below):
//   bases        rank-revealing blocked Gram-Schmidt (bcgs, eig.cu): Q_l of span(U_l)
//   core         C_l = Q_l^T U_l, K = C0 diag(w) C1^T (DMMA GEMMs)
//   SVD          small_svd (QR-preconditioned one-sided Jacobi, trunc.cu) of K
//   rank cut     rank_cut_device (tails from the small end, A23)
//   apply        forward transform V^T U (GEMM), Hadamard with the spectral factors, and for the
//                solver the truncation in eigen coordinates followed by V Z on the r survivors
//   spectral     D2 = f(lam1 (+) lam2) evaluated on the device; randomised range finder with one
//                orthonormalised power step, an explicit residual check (the captured energy is
//                verified, the sample doubled otherwise), then the SVD of the projected matrix.
#include <algorithm>
#include <cmath>
#include <vector>
#include "cpops.cuh"
#include "eig.cuh"
#include "solver.cuh"
#include "tt.cuh"

namespace fc {
namespace {

constexpr double kBasisTol2 = 1e-12;   // rank-revealing basis tolerance (relative, as kBasisTol)

__device__ __forceinline__ double spec_f2(int kind, double alpha, double beta, double lam) {
  if (kind == FC_F) return beta * pow(lam, alpha) + pow(lam, -alpha);
  if (kind == FC_G) return 1.0 / (beta * pow(lam, alpha) + pow(lam, -alpha));
  if (kind == FC_POW_PLUS) return pow(lam, alpha);
  return pow(lam, -alpha);
}

int nblk2(long long tot) { return (int)std::max<long long>(1, std::min<long long>((tot + 255) / 256, 148 * 16)); }

// D[i + j n] = f(lam1_i + lam2_j)
__global__ void d2_eval_kernel(int n, int kind, double alpha, double beta, const double* __restrict__ l1,
                               const double* __restrict__ l2, double* D) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    D[idx] = spec_f2(kind, alpha, beta, l1[i] + l2[j]);
  }
}

// deterministic pseudo-random sample in [-1, 1) (counter hash)
__global__ void hash_fill_kernel(long long tot, unsigned seed, double* out) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)idx * 2654435761u ^ (seed * 2246822519u + 0x9E3779B9u) ^ (unsigned)(idx >> 32);
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
    out[idx] = (double)(h & 0xFFFFFF) / 8388608.0 - 1.0;
  }
}

// out[:, k*R + j] = A[:, k] . X[:, j]   (n x r) x (n x R) -> n x rR, ld n
__global__ void hadamard2_kernel(int n, int r, const double* __restrict__ A, int lda, int R,
                                 const double* __restrict__ X, int ldx, double* out) {
  const long long tot = (long long)n * r * R;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % n);
    const long long col = idx / n;
    const int k = (int)(col / R), j = (int)(col % R);
    out[idx] = A[i + (size_t)k * lda] * X[i + (size_t)j * ldx];
  }
}

// w_out[k*R + j] = wA[k] * wx[j]
__global__ void kron_w2_kernel(int r, const double* __restrict__ wA, int R, const double* __restrict__ wx,
                               double* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < r * R) out[t] = wA[t / R] * wx[t % R];
}

// column norms of two n x m matrices (warp per column); w[c] *= nrm0[c] * nrm1[c]; columns scaled
// to unit norm (zero columns stay zero)
__global__ void normalize2_kernel(int n, int m, double* U0, int ld0, double* U1, int ld1, double* w) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), ln = threadIdx.x & 31;
  if (c >= m) return;
  double* u[2] = {U0 + (size_t)c * ld0, U1 + (size_t)c * ld1};
  double nr[2];
  for (int l = 0; l < 2; ++l) {
    double s = 0.0;
    for (int i = ln; i < n; i += 32) s = fma(u[l][i], u[l][i], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    nr[l] = sqrt(s);
  }
  for (int l = 0; l < 2; ++l) {
    const double inv = nr[l] > 0.0 ? 1.0 / nr[l] : 0.0;
    for (int i = ln; i < n; i += 32) u[l][i] *= inv;
  }
  if (ln == 0) w[c] *= nr[0] * nr[1];
}

// C[:, c] *= w[c]  (q x m, ld q)
__global__ void scale_cols2_kernel(int q, int m, const double* __restrict__ w, double* C) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)q * m;
       idx += (long long)gridDim.x * blockDim.x)
    C[idx] *= w[idx / q];
}

// s2 = s^2 (k values), energy[0] = sum s^2 (fixed order, one thread)
__global__ void sq_energy_kernel(int k, const double* __restrict__ s, double* s2, double* energy) {
  for (int i = threadIdx.x; i < k; i += blockDim.x) s2[i] = s[i] * s[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    double e = 0.0;
    for (int i = k - 1; i >= 0; --i) e += s2[i];
    energy[0] = e;
  }
}

// out = sum_{i,j} wx_i wy_j G0[i + j R1] G1[i + j R1]  (one CTA, fixed-order tree)
__global__ void dot2_kernel(int R1, int R2, const double* __restrict__ wx, const double* __restrict__ wy,
                            const double* __restrict__ G0, const double* __restrict__ G1, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  const long long tot = (long long)R1 * R2;
  for (long long idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int i = (int)(idx % R1), j = (int)(idx / R1);
    s = fma(wx[i] * wy[j], G0[idx] * G1[idx], s);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

// block-wise partial sums of squares / minima of an array (fixed order), then one CTA combines
__global__ void sumsq_min_kernel(long long tot, const double* __restrict__ a, double* part_s, double* part_m) {
  __shared__ double rs[32], rm[32];
  double s = 0.0, m = 1e300;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const double v = a[idx];
    s = fma(v, v, s);
    m = fmin(m, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  if ((threadIdx.x & 31) == 0) {
    rs[threadIdx.x >> 5] = s;
    rm[threadIdx.x >> 5] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0, u = 1e300;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      t += rs[w];
      u = fmin(u, rm[w]);
    }
    part_s[blockIdx.x] = t;
    part_m[blockIdx.x] = u;
  }
}

__global__ void combine_kernel(int nb, const double* __restrict__ ps, const double* __restrict__ pm, double* out) {
  if (threadIdx.x != 0) return;
  double s = 0.0, m = 1e300;
  for (int b = 0; b < nb; ++b) {
    s += ps[b];
    m = fmin(m, pm[b]);
  }
  out[0] = s;
  out[1] = m;
}

// (sum of squares, min) of a device array, returned on the host
std::pair<double, double> sumsq_min(cudaStream_t st, const double* a, long long tot) {
  Scratch s(st);
  const int nb = 296;
  double* ps = s.alloc<double>(nb);
  double* pm = s.alloc<double>(nb);
  double* out = s.alloc<double>(2);
  sumsq_min_kernel<<<nb, 256, 0, st>>>(tot, a, ps, pm);
  FC_CHECK_LAUNCH();
  combine_kernel<<<1, 32, 0, st>>>(nb, ps, pm, out);
  FC_CHECK_LAUNCH();
  double h[2];
  FC_CUDA_TRY(cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  return {h[0], h[1]};
}

int read_int2(const int* d, cudaStream_t st) {
  int h = 0;
  FC_CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  return h;
}

}  // namespace

// ---- the 2D low-rank matrix inside the library ------------------------------------------
struct LR2 {
  int n = 0, R = 0;
  double* w = nullptr;
  double* U[2] = {nullptr, nullptr};   // n x R each, ld n
  std::vector<DevMem> mem;
};

LR2 lr2_alloc(cudaStream_t st, int n, int R) {
  LR2 x;
  x.n = n;
  x.R = R;
  x.mem.emplace_back(((size_t)R + (size_t)2 * n * R) * 8, st);
  x.w = x.mem.back().d();
  x.U[0] = x.w + R;
  x.U[1] = x.U[0] + (size_t)n * R;
  return x;
}

LR2 lr2_from_abi(cudaStream_t st, int n, const fc_lr2& a) {
  LR2 x = lr2_alloc(st, n, a.rank);
  if (a.rank == 0) return x;
  FC_CUDA_TRY(cudaMemcpyAsync(x.w, a.w, (size_t)a.rank * 8, cudaMemcpyDeviceToDevice, st));
  for (int l = 0; l < 2; ++l)
    FC_CUDA_TRY(cudaMemcpy2DAsync(x.U[l], (size_t)n * 8, a.U[l], (size_t)a.ld[l] * 8, (size_t)n * 8, a.rank,
                                  cudaMemcpyDeviceToDevice, st));
  return x;
}

void lr2_store(cudaStream_t st, const LR2& x, fc_lr2* out) {
  if (x.R > out->cap) {
    out->rank = x.R;
    throw Error(FC_ERR_CAPACITY, "output cap " + std::to_string(out->cap) + " < rank " + std::to_string(x.R));
  }
  out->rank = x.R;
  if (x.R == 0) return;
  FC_CUDA_TRY(cudaMemcpyAsync(out->w, x.w, (size_t)x.R * 8, cudaMemcpyDeviceToDevice, st));
  for (int l = 0; l < 2; ++l)
    FC_CUDA_TRY(cudaMemcpy2DAsync(out->U[l], (size_t)out->ld[l] * 8, x.U[l], (size_t)x.n * 8, (size_t)x.n * 8, x.R,
                                  cudaMemcpyDeviceToDevice, st));
}

// x + a*y by concatenation [P:1845-1866]
LR2 lr2_axpy(cudaStream_t st, const LR2& x, double a, const LR2& y) {
  LR2 z = lr2_alloc(st, x.n, x.R + y.R);
  if (x.R) {
    FC_CUDA_TRY(cudaMemcpyAsync(z.w, x.w, (size_t)x.R * 8, cudaMemcpyDeviceToDevice, st));
    for (int l = 0; l < 2; ++l)
      FC_CUDA_TRY(cudaMemcpyAsync(z.U[l], x.U[l], (size_t)x.n * x.R * 8, cudaMemcpyDeviceToDevice, st));
  }
  if (y.R) {
    scale_copy(y.R, y.w, a, z.w + x.R, st);
    for (int l = 0; l < 2; ++l)
      FC_CUDA_TRY(cudaMemcpyAsync(z.U[l] + (size_t)x.n * x.R, y.U[l], (size_t)x.n * y.R * 8, cudaMemcpyDeviceToDevice,
                                  st));
  }
  return z;
}

// <x, y> [P:1748-1755 with d = 2]: cross-Grams G_l = X_l^T Y_l (DMMA), then the weighted
// Hadamard sum in a fixed order
double lr2_dot(cudaStream_t st, const LR2& x, const LR2& y) {
  if (x.R == 0 || y.R == 0) return 0.0;
  Scratch s(st);
  const size_t g = (size_t)x.R * y.R;
  double* G = s.zeros<double>(2 * g);
  double* out = s.alloc<double>(1);
  GemmArgs a;
  a.transA = 1;
  a.beta = 1.0;
  a.nbatch = 2;
  for (int l = 0; l < 2; ++l)
    a.b[l] = GemmBatch{x.R, y.R, x.n, x.U[l], x.n, y.U[l], y.n, G + l * g, x.R, nullptr, 0, nullptr};
  const int tiles = 2 * cdiv(x.R, 64) * cdiv(y.R, 64);
  a.splitk = std::max(1, std::min(cdiv(x.n, 64), cdiv(2 * 148, tiles)));
  gemm(a, st);
  dot2_kernel<<<1, 1024, 0, st>>>(x.R, y.R, x.w, y.w, G, G + g, out);
  FC_CHECK_LAUNCH();
  double h = 0.0;
  FC_CUDA_TRY(cudaMemcpyAsync(&h, out, 8, cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  return h;
}

// rank-revealing orthonormal bases of span(U_0) and span(U_1) (blocked BCGS2, both modes batched)
// Q_l (n x q_l) are allocated in `s`; q_l returned on the host
void lr2_bases(cudaStream_t st, Scratch& s, int n, int R, const double* const U[2], double* Q[2], int q[2]) {
  BcgsBatch pb;
  int* kdev = s.zeros<int>(2);
  const int kcap = std::min(n, R);
  for (int l = 0; l < 2; ++l) {
    double* K = s.alloc<double>((size_t)n * R);
    FC_CUDA_TRY(cudaMemcpyAsync(K, U[l], (size_t)n * R * 8, cudaMemcpyDeviceToDevice, st));
    Q[l] = s.alloc<double>((size_t)n * kcap);
    pb.e[pb.nb++] = BcgsEntry{n, R, K, n, Q[l], n, kcap, kdev + l, s.alloc<double>(R),
                              s.alloc<double>((size_t)kcap * kBcgsW), kBasisTol2};
  }
  bcgs(pb, st);
  int h[2];
  FC_CUDA_TRY(cudaMemcpyAsync(h, kdev, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  q[0] = h[0];
  q[1] = h[1];
}

// reduced SVD truncation [P:973-976] (reading 2D-T).  rank_cap > 0: CAPACITY above it.
LR2 lr2_truncate(cudaStream_t st, const LR2& x, double eps, int rank_cap, int* rank_out = nullptr) {
  const int n = x.n, R = x.R;
  if (R == 0) {
    if (rank_out) *rank_out = 0;
    return lr2_alloc(st, n, 0);
  }
  Scratch s(st);
  double* Q[2];
  int q[2];
  lr2_bases(st, s, n, R, x.U, Q, q);
  if (q[0] == 0 || q[1] == 0) {
    if (rank_out) *rank_out = 0;
    return lr2_alloc(st, n, 0);
  }
  require(std::max(q[0], q[1]) <= 1024, FC_ERR_CAPACITY, "2D truncation: basis above 1024 columns");
  // C_l = Q_l^T U_l (q_l x R); C_0 <- C_0 diag(w); K = C_0 C_1^T (q0 x q1)
  double* C[2];
  GemmArgs g;
  g.transA = 1;
  g.beta = 1.0;
  g.nbatch = 2;
  for (int l = 0; l < 2; ++l) {
    C[l] = s.zeros<double>((size_t)q[l] * R);
    g.b[l] = GemmBatch{q[l], R, n, Q[l], n, x.U[l], n, C[l], q[l], nullptr, 0, nullptr};
  }
  g.splitk = waves_splitk(g, 8);   // few output tiles, K = n
  gemm(g, st);
  scale_cols2_kernel<<<nblk2((long long)q[0] * R), 256, 0, st>>>(q[0], R, x.w, C[0]);
  FC_CHECK_LAUNCH();
  double* K = s.zeros<double>((size_t)q[0] * q[1]);
  dgemm(st, 0, 1, q[0], q[1], R, 1.0, C[0], q[0], C[1], q[1], 1.0, K, q[0],
        std::max(1, std::min(cdiv(R, 128), cdiv(2 * 148, cdiv(q[0], 64) * cdiv(q[1], 64)))));
  // SVD of the core, rank cut from the small end
  const int k = std::min(q[0], q[1]);
  double* sv = s.alloc<double>(k);
  double* Ua = s.alloc<double>((size_t)q[0] * k);
  double* Vb = s.alloc<double>((size_t)q[1] * k);
  small_svd(st, q[0], q[1], 1, K, sv, Ua, Vb);
  double* s2 = s.alloc<double>(k);
  double* energy = s.alloc<double>(2);
  int* rdev = s.alloc<int>(1);
  sq_energy_kernel<<<1, 256, 0, st>>>(k, sv, s2, energy);
  FC_CHECK_LAUNCH();
  rank_cut_device(k, s2, eps * eps, energy, rdev, energy + 1, st);
  double he = 0.0;
  FC_CUDA_TRY(cudaMemcpyAsync(&he, energy, 8, cudaMemcpyDeviceToHost, st));
  int r = read_int2(rdev, st);
  if (he == 0.0) r = 0;
  if (rank_out) *rank_out = r;
  if (rank_cap > 0 && r > rank_cap) throw Error(FC_ERR_CAPACITY, "2D truncation rank above the rank cap");
  LR2 y = lr2_alloc(st, n, r);
  if (r == 0) return y;
  FC_CUDA_TRY(cudaMemcpyAsync(y.w, sv, (size_t)r * 8, cudaMemcpyDeviceToDevice, st));
  GemmArgs z;
  z.nbatch = 2;
  z.beta = 1.0;
  FC_CUDA_TRY(cudaMemsetAsync(y.U[0], 0, (size_t)2 * n * r * 8, st));   // U[0], U[1] contiguous
  z.b[0] = GemmBatch{n, r, q[0], Q[0], n, Ua, q[0], y.U[0], n, nullptr, 0, nullptr};
  z.b[1] = GemmBatch{n, r, q[1], Q[1], n, Vb, q[1], y.U[1], n, nullptr, 0, nullptr};
  z.splitk = waves_splitk(z, 8);
  gemm(z, st);
  return y;
}

// eigen-coordinate product of the apply: Yhat_l = [a_k . V_l^T x_l,j] (n x rR), weights w_k w_j
LR2 lr2_apply_hat(fc_ctx c, const Spec2& sp, const LR2& x) {
  cudaStream_t st = c->st;
  const int n = x.n, r = sp.r, R = x.R;
  LR2 y = lr2_alloc(st, n, r * R);
  if (y.R == 0) return y;
  Scratch s(st);
  double* Xh = s.alloc<double>((size_t)2 * n * R);
  GemmArgs f;                                                      // forward transform
  f.transA = 1;
  f.beta = 1.0;
  f.nbatch = 2;
  FC_CUDA_TRY(cudaMemsetAsync(Xh, 0, (size_t)2 * n * R * 8, st));
  for (int l = 0; l < 2; ++l)
    f.b[l] = GemmBatch{n, R, n, c->V_l(l), n, x.U[l], n, Xh + (size_t)l * n * R, n, nullptr, 0, nullptr};
  f.splitk = waves_splitk(f, 8);
  gemm(f, st);
  for (int l = 0; l < 2; ++l) {
    hadamard2_kernel<<<nblk2((long long)n * r * R), 256, 0, st>>>(n, r, sp.Ul(n, l), n, R, Xh + (size_t)l * n * R, n,
                                                                   y.U[l]);
    FC_CHECK_LAUNCH();
  }
  kron_w2_kernel<<<cdiv(r * R, 256), 256, 0, st>>>(r, sp.w.p, R, x.w, y.w);
  FC_CHECK_LAUNCH();
  return y;
}

// back to physical coordinates: U_l <- V_l U_l
void lr2_inverse(fc_ctx c, LR2& y) {
  if (y.R == 0) return;
  cudaStream_t st = c->st;
  Scratch s(st);
  double* T = s.zeros<double>((size_t)2 * y.n * y.R);
  GemmArgs g;
  g.nbatch = 2;
  g.beta = 1.0;
  for (int l = 0; l < 2; ++l)
    g.b[l] = GemmBatch{y.n, y.R, y.n, c->V_l(l), y.n, y.U[l], y.n, T + (size_t)l * y.n * y.R, y.n, nullptr, 0, nullptr};
  g.splitk = waves_splitk(g, 8);
  gemm(g, st);
  for (int l = 0; l < 2; ++l)
    FC_CUDA_TRY(cudaMemcpyAsync(y.U[l], T + (size_t)l * y.n * y.R, (size_t)y.n * y.R * 8, cudaMemcpyDeviceToDevice,
                                st));
}

// untruncated apply [P:597-611]: columns normalised (norms folded into the weights)
LR2 lr2_apply(fc_ctx c, const Spec2& sp, const LR2& x) {
  LR2 y = lr2_apply_hat(c, sp, x);
  lr2_inverse(c, y);
  if (y.R) {
    normalize2_kernel<<<cdiv(y.R, 8), 256, 0, c->st>>>(y.n, y.R, y.U[0], y.n, y.U[1], y.n, y.w);
    FC_CHECK_LAUNCH();
  }
  return y;
}

// fused apply -> truncate: the reduced SVD of the eigen-coordinate product (V_l orthogonal:
// same singular values and ranks), then only the r surviving columns are transformed back
LR2 lr2_apply_truncate(fc_ctx c, const Spec2& sp, const LR2& x, double eps, int cap) {
  LR2 yh = lr2_apply_hat(c, sp, x);
  LR2 y = lr2_truncate(c->st, yh, eps, cap);
  lr2_inverse(c, y);
  return y;
}

// 2D spectral factorisation (reading 2D-S) of D2 = f(lam1 (+) lam2): eps-driven (keep <= 0) or
// the top `keep` terms with the SPD guard (A7'/A7'')
void build_spectral_2d(fc_ctx c, int which, double eps, int keep, bool spd_guard) {
  cudaStream_t st = c->st;
  const int n = c->n;
  Scratch s(st);
  double* D = s.alloc<double>((size_t)n * n);
  d2_eval_kernel<<<nblk2((long long)n * n), 256, 0, st>>>(n, which, c->p.alpha, c->p.beta, c->lam_l(0), c->lam_l(1), D);
  FC_CHECK_LAUNCH();
  const double normD2 = sumsq_min(st, D, (long long)n * n).first;
  int ell = std::min(n, std::max(64, keep > 0 ? 2 * keep + 16 : 64));
  for (int attempt = 0;; ++attempt) {
    Scratch t(st);
    // range finder: Y = D Om -> Q; Y = D^T Q -> Q'; Y = D Q' -> Q (one orthonormalised power step)
    double* Om = t.alloc<double>((size_t)n * ell);
    hash_fill_kernel<<<nblk2((long long)n * ell), 256, 0, st>>>((long long)n * ell, 1234u + attempt, Om);
    FC_CHECK_LAUNCH();
    double* Y = t.alloc<double>((size_t)n * ell);
    auto orth = [&](double* A, int m, double** Qo) {
      BcgsBatch pb;
      int* kd = t.zeros<int>(1);
      *Qo = t.alloc<double>((size_t)n * m);
      pb.e[pb.nb++] = BcgsEntry{n, m, A, n, *Qo, n, m, kd, t.alloc<double>(m), t.alloc<double>((size_t)m * kBcgsW),
                                kBasisTol2};
      bcgs(pb, st);
      return read_int2(kd, st);
    };
    dgemm(st, 0, 0, n, ell, n, 1.0, D, n, Om, n, 0.0, Y, n);
    double* Q1;
    int q1 = orth(Y, ell, &Q1);
    dgemm(st, 1, 0, n, q1, n, 1.0, D, n, Q1, n, 0.0, Y, n);
    double* Q2;
    int q2 = orth(Y, q1, &Q2);
    dgemm(st, 0, 0, n, q2, n, 1.0, D, n, Q2, n, 0.0, Y, n);
    double* Q;
    const int q = orth(Y, q2, &Q);
    require(q > 0, FC_ERR_CUDA, "2D spectral factorisation: empty range");
    // B^T = D^T Q (n x q); residual energy ||D - Q Q^T D||^2 checked explicitly
    double* Bt = t.alloc<double>((size_t)n * q);
    dgemm(st, 1, 0, n, q, n, 1.0, D, n, Q, n, 0.0, Bt, n);
    double* Res = t.alloc<double>((size_t)n * n);
    FC_CUDA_TRY(cudaMemcpyAsync(Res, D, (size_t)n * n * 8, cudaMemcpyDeviceToDevice, st));
    dgemm(st, 0, 1, n, n, q, -1.0, Q, n, Bt, n, 1.0, Res, n);
    const double res2 = sumsq_min(st, Res, (long long)n * n).first;
    // SVD of B = Q^T D (q x n): B^T = Qb Cb (basis of span(B^T)), Cb = U' S V'^T ->
    // D ~ Q B = (Q V') S (Qb U')^T
    double* Btc = t.alloc<double>((size_t)n * q);
    FC_CUDA_TRY(cudaMemcpyAsync(Btc, Bt, (size_t)n * q * 8, cudaMemcpyDeviceToDevice, st));
    double* Qb;
    const int qb = orth(Btc, q, &Qb);
    double* Cb = t.alloc<double>((size_t)qb * q);
    dgemm(st, 1, 0, qb, q, n, 1.0, Qb, n, Bt, n, 0.0, Cb, qb);
    const int kk = std::min(qb, q);
    double* sv = t.alloc<double>(kk);
    double* Uc = t.alloc<double>((size_t)qb * kk);
    double* Vc = t.alloc<double>((size_t)q * kk);
    small_svd(st, qb, q, 1, Cb, sv, Uc, Vc);
    std::vector<double> hs(kk);
    FC_CUDA_TRY(cudaMemcpyAsync(hs.data(), sv, (size_t)kk * 8, cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaStreamSynchronize(st));
    // rank: eps-driven tail (dropped s^2 + the range finder's residual <= eps^2 ||D||^2), or keep
    int r;
    if (keep <= 0) {
      const double thr = eps * eps * normD2 - res2;
      double tail = 0.0;
      r = kk;
      for (int m = kk - 1; m >= 1; --m) {
        tail += hs[m] * hs[m];
        if (tail <= thr) r = m;
        else break;
      }
      while (r > 0 && r < kk && hs[r] == hs[r - 1] && hs[r] > 0) ++r;   // A23
      if (thr < 0.0 || r > ell - 8) {   // the sample did not capture enough: enlarge it
        require(ell < n, FC_ERR_CAPACITY, "2D spectral factorisation: eps_D not reached with a full sample");
        ell = std::min(n, 2 * ell);
        continue;
      }
    } else {
      r = std::min(keep, kk);
    }
    // factors a = Q Vc[:, :r], b = Qb Uc[:, :r]; positivity guard on the full grid
    Spec2& sp = c->spec2[which];
    auto store = [&](int rr) {
      sp.r = rr;
      sp.w.ensure(std::max(rr, 1));
      sp.U.ensure((size_t)2 * n * std::max(rr, 1));
      FC_CUDA_TRY(cudaMemcpyAsync(sp.w.p, sv, (size_t)rr * 8, cudaMemcpyDeviceToDevice, st));
      dgemm(st, 0, 0, n, rr, q, 1.0, Q, n, Vc, q, 0.0, sp.Ul(n, 0), n);
      dgemm(st, 0, 0, n, rr, qb, 1.0, Qb, n, Uc, qb, 0.0, sp.Ul(n, 1), n);
    };
    store(r);
    if (spd_guard) {
      double* Rec = t.alloc<double>((size_t)n * n);
      for (;;) {
        // reconstruction a diag(w) b^T (scale a's columns into a copy)
        double* As = t.alloc<double>((size_t)n * sp.r);
        FC_CUDA_TRY(cudaMemcpyAsync(As, sp.Ul(n, 0), (size_t)n * sp.r * 8, cudaMemcpyDeviceToDevice, st));
        scale_cols2_kernel<<<nblk2((long long)n * sp.r), 256, 0, st>>>(n, sp.r, sp.w.p, As);
        FC_CHECK_LAUNCH();
        dgemm(st, 0, 1, n, n, sp.r, 1.0, As, n, sp.Ul(n, 1), n, 0.0, Rec, n);
        const double mn = sumsq_min(st, Rec, (long long)n * n).second;
        if (mn > 0.0) break;
        if (sp.r < std::min(64, kk)) {
          store(sp.r + 1);
          continue;
        }
        // A7'': constant term s 1 (x) 1, s = 2|min| + 1e-15 sum|w| (an extra unit-column term)
        double sw = 0.0;
        for (int m = 0; m < sp.r; ++m) sw += std::fabs(hs[m]);
        const double shift = 2.0 * std::fabs(mn) + 1e-15 * sw;
        const int r0 = sp.r;
        fc::DBuf w2, U2;
        w2.ensure(r0 + 1);
        U2.ensure((size_t)2 * n * (r0 + 1));
        FC_CUDA_TRY(cudaMemcpyAsync(w2.p, sp.w.p, (size_t)r0 * 8, cudaMemcpyDeviceToDevice, st));
        const double ws = shift * n;
        FC_CUDA_TRY(cudaMemcpyAsync(w2.p + r0, &ws, 8, cudaMemcpyHostToDevice, st));
        std::vector<double> ones((size_t)n, 1.0 / std::sqrt((double)n));
        for (int l = 0; l < 2; ++l) {
          FC_CUDA_TRY(cudaMemcpyAsync(U2.p + (size_t)l * n * (r0 + 1), sp.Ul(n, l), (size_t)n * r0 * 8,
                                      cudaMemcpyDeviceToDevice, st));
          FC_CUDA_TRY(cudaMemcpyAsync(U2.p + (size_t)l * n * (r0 + 1) + (size_t)n * r0, ones.data(), (size_t)n * 8,
                                      cudaMemcpyHostToDevice, st));
        }
        FC_CUDA_TRY(cudaStreamSynchronize(st));
        sp.w.release();
        sp.U.release();
        sp.w = w2;
        sp.U = U2;
        w2.p = nullptr;
        U2.p = nullptr;
        sp.r = r0 + 1;
        break;
      }
    }
    sp.valid = true;
    return;
  }
}

}  // namespace fc

using namespace fc;

namespace {

template <class F>
int guard2d(fc_ctx c, F&& f) {
  if (!c) return FC_ERR_INVALID_ARG;
  try {
    return f();
  } catch (const Error& e) {
    c->err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    c->err = e.what();
    return FC_ERR_CUDA;
  }
}

void check_lr2(fc_ctx c, const fc_lr2* x, const char* name) {
  require(x != nullptr, FC_ERR_INVALID_ARG, std::string(name) + " is NULL");
  require(c->n > 0 && c->have_eig[0] && c->have_eig[1], FC_ERR_NOT_READY,
          "no mode-0/1 eigenpairs: call sl_setup_2d or sl_set_eigen first");
  for (int l = 0; l < 2; ++l) {
    require(x->n[l] == c->n, FC_ERR_SHAPE, std::string(name) + ": mode size differs from context n");
    require(x->ld[l] >= x->n[l], FC_ERR_INVALID_ARG, std::string(name) + ": ld < n");
    require(x->rank == 0 || x->U[l] != nullptr, FC_ERR_INVALID_ARG, std::string(name) + ": NULL factor");
  }
  require(x->rank >= 0 && x->rank <= x->cap, FC_ERR_INVALID_ARG, std::string(name) + ": rank > cap");
  require(x->rank == 0 || x->w != nullptr, FC_ERR_INVALID_ARG, std::string(name) + ": NULL weights");
}

const Spec2& spec2_of(fc_ctx c, int which) {
  require(which == FC_F || which == FC_G, FC_ERR_INVALID_ARG, "2D spectral factorisation: FC_F or FC_G");
  require(c->spec2[which].valid, FC_ERR_NOT_READY, "2D spectral factorisation missing: call sl_setup_2d");
  return c->spec2[which];
}

}  // namespace

extern "C" {

int sl_setup_2d(fc_ctx c, int n, const double* a_mid, const fc_params* p) {
  return guard2d(c, [&]() {
    require(p != nullptr && a_mid != nullptr, FC_ERR_INVALID_ARG, "NULL argument");
    require(n >= 2, FC_ERR_INVALID_ARG, "n must be >= 2");
    require(p->alpha > 0 && p->alpha <= 1, FC_ERR_INVALID_ARG, "alpha must be in (0, 1]");
    require(p->beta > 0 && std::isfinite(p->beta), FC_ERR_INVALID_ARG, "beta must be > 0");
    require(p->eps > 0 && std::isfinite(p->eps), FC_ERR_INVALID_ARG, "eps must be > 0");
    for (long long i = 0; i < 2LL * (n + 1); ++i)
      require(std::isfinite(a_mid[i]) && a_mid[i] > 0, FC_ERR_NONPOS_COEF, "midpoint coefficient <= 0 or non-finite");
    cudaStream_t st = c->st;
    c->n = n;
    c->p = *p;
    c->have_params = true;
    c->lam.ensure((size_t)3 * n);
    c->V.ensure((size_t)3 * n * n);
    for (auto& h : c->have_eig) h = false;
    for (auto& sp : c->spec) sp.valid = false;
    for (auto& sp : c->spec2) sp.valid = false;
    // the 3-mode eigen kernels run modes 0, 1 and a copy of mode 1 (mode 2 is not used in 2D)
    std::vector<double> a3((size_t)3 * (n + 1));
    std::copy(a_mid, a_mid + 2 * (size_t)(n + 1), a3.begin());
    std::copy(a_mid + (size_t)(n + 1), a_mid + 2 * (size_t)(n + 1), a3.begin() + 2 * (size_t)(n + 1));
    Scratch s(st);
    double* a_dev = s.alloc<double>(a3.size());
    int* status = s.zeros<int>(1);
    FC_CUDA_TRY(cudaMemcpyAsync(a_dev, a3.data(), a3.size() * 8, cudaMemcpyHostToDevice, st));
    sl_eigen_device(st, n, a_dev, p->boundary, c->lam.p, c->V.p, status);
    int hs = 0;
    FC_CUDA_TRY(cudaMemcpyAsync(&hs, status, sizeof(int), cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaStreamSynchronize(st));
    require(hs == 0, hs, "coefficient check failed on the device");
    c->have_eig[0] = c->have_eig[1] = true;
    const double epsD = p->eps_D > 0 ? p->eps_D : p->eps;
    build_spectral_2d(c, FC_F, epsD, p->op_rank > 0 ? p->op_rank : 0, false);
    build_spectral_2d(c, FC_G, epsD, p->precond_rank > 0 ? p->precond_rank : 6, true);
    return FC_OK;
  });
}

int op_get_spectral_2d(fc_ctx c, int which, fc_lr2* out) {
  return guard2d(c, [&]() {
    const Spec2& sp = spec2_of(c, which);
    require(out != nullptr, FC_ERR_INVALID_ARG, "out is NULL");
    const int n = c->n;
    LR2 x;
    x.n = n;
    x.R = sp.r;
    x.w = sp.w.p;
    x.U[0] = sp.Ul(n, 0);
    x.U[1] = sp.Ul(n, 1);
    lr2_store(c->st, x, out);
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    return FC_OK;
  });
}

int op_set_spectral_2d(fc_ctx c, int which, const fc_lr2* in) {
  return guard2d(c, [&]() {
    require(which == FC_F || which == FC_G, FC_ERR_INVALID_ARG, "FC_F or FC_G");
    check_lr2(c, in, "in");
    const int n = c->n, r = in->rank;
    Spec2& sp = c->spec2[which];
    sp.r = r;
    sp.w.ensure(std::max(r, 1));
    sp.U.ensure((size_t)2 * n * std::max(r, 1));
    if (r) {
      FC_CUDA_TRY(cudaMemcpyAsync(sp.w.p, in->w, (size_t)r * 8, cudaMemcpyDeviceToDevice, c->st));
      for (int l = 0; l < 2; ++l)
        FC_CUDA_TRY(cudaMemcpy2DAsync(sp.Ul(n, l), (size_t)n * 8, in->U[l], (size_t)in->ld[l] * 8, (size_t)n * 8, r,
                                      cudaMemcpyDeviceToDevice, c->st));
    }
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    sp.valid = true;
    return FC_OK;
  });
}

int fracop_apply_2d(fc_ctx c, int which, const fc_lr2* x, fc_lr2* y) {
  return guard2d(c, [&]() {
    check_lr2(c, x, "x");
    check_lr2(c, y, "y");
    const Spec2& sp = spec2_of(c, which);
    LR2 xi = lr2_from_abi(c->st, c->n, *x);
    LR2 out = lr2_apply(c, sp, xi);
    lr2_store(c->st, out, y);
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    return FC_OK;
  });
}

int cp_dot_2d(fc_ctx c, const fc_lr2* x, const fc_lr2* y, double* out) {
  return guard2d(c, [&]() {
    check_lr2(c, x, "x");
    check_lr2(c, y, "y");
    require(out != nullptr, FC_ERR_INVALID_ARG, "out is NULL");
    LR2 a = lr2_from_abi(c->st, c->n, *x), b = lr2_from_abi(c->st, c->n, *y);
    *out = lr2_dot(c->st, a, b);
    return FC_OK;
  });
}

int cp_truncate_2d(fc_ctx c, const fc_lr2* x, double eps, fc_lr2* y, int* out_rank) {
  return guard2d(c, [&]() {
    check_lr2(c, x, "x");
    check_lr2(c, y, "y");
    require(eps > 0 && std::isfinite(eps), FC_ERR_INVALID_ARG, "eps must be > 0");
    LR2 a = lr2_from_abi(c->st, c->n, *x);
    int r = 0;
    LR2 out = lr2_truncate(c->st, a, eps, 0, &r);
    if (out_rank) *out_rank = r;
    lr2_store(c->st, out, y);
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    return FC_OK;
  });
}

int pcg_solve_2d(fc_ctx c, const fc_lr2* b, const fc_params* prm, fc_lr2* u, fc_pcg_report* rep) {
  return guard2d(c, [&]() {
    check_lr2(c, b, "b");
    check_lr2(c, u, "u");
    require(prm != nullptr, FC_ERR_INVALID_ARG, "params NULL");
    const double eps = prm->eps;
    require(eps > 0, FC_ERR_INVALID_ARG, "eps must be > 0");
    const double tol = prm->tol_stop > 0 ? prm->tol_stop : 10.0 * eps;     // A13
    const int kmax = std::min(prm->kmax > 0 ? prm->kmax : 100, FC_MAX_ITERS);  // A17
    const int cap = prm->rank_cap > 0 ? prm->rank_cap : (1 << 20);
    const Spec2& F = spec2_of(c, FC_F);
    const Spec2& G = spec2_of(c, FC_G);
    cudaStream_t st = c->st;
    fc_pcg_report local{};
    fc_pcg_report& RP = rep ? *rep : local;
    RP = fc_pcg_report{};
    cudaEvent_t t0, t1, loop0, ti0, ti1;
    for (cudaEvent_t* e : {&t0, &t1, &loop0, &ti0, &ti1}) FC_CUDA_TRY(cudaEventCreate(e));
    struct EvGuard {
      cudaEvent_t e[5];
      ~EvGuard() { for (auto x : e) cudaEventDestroy(x); }
    } evg{{t0, t1, loop0, ti0, ti1}};
    FC_CUDA_TRY(cudaEventRecord(t0, st));
    LR2 B = lr2_from_abi(st, c->n, *b);
    const double normB = std::sqrt(std::max(lr2_dot(st, B, B), 0.0));
    RP.normB = normB;
    require(std::isfinite(normB), FC_ERR_NAN, "non-finite right-hand side");
    LR2 X = lr2_alloc(st, c->n, 0);                                  // A14
    if (normB == 0.0) {
      RP.converged = 1;
      u->rank = 0;
      return FC_OK;
    }
    LR2 R = lr2_axpy(st, B, 0.0, lr2_alloc(st, c->n, 0));           // line 1, A15 (copy)
    LR2 Z = lr2_apply_truncate(c, G, R, eps, cap);                  // lines 2-3
    LR2 P = lr2_axpy(st, Z, 0.0, lr2_alloc(st, c->n, 0));           // line 4
    double rz = lr2_dot(st, R, Z);
    int status = FC_NOT_CONVERGED;
    FC_CUDA_TRY(cudaEventRecord(loop0, st));
    for (int k = 0; k < kmax; ++k) {
      FC_CUDA_TRY(cudaEventRecord(ti0, st));
      LR2 S = lr2_apply_truncate(c, F, P, eps, cap);                // lines 7-8
      const double ps = lr2_dot(st, P, S);
      require(std::isfinite(ps), FC_ERR_NAN, "<P,S> is not finite");
      require(ps > 0, FC_ERR_NOT_SPD, "<P,S> <= 0");
      const double a_k = rz / ps;                                   // line 9
      X = lr2_truncate(st, lr2_axpy(st, X, a_k, P), eps, cap);      // lines 10-11
      R = lr2_truncate(st, lr2_axpy(st, R, -a_k, S), eps, cap);     // lines 12-13
      const double rel = std::sqrt(std::max(lr2_dot(st, R, R), 0.0)) / normB;   // line 14
      RP.rel_res[k] = rel;
      RP.rank_S[k] = S.R;
      RP.rank_X[k] = X.R;
      RP.rank_R[k] = R.R;
      RP.iters = k + 1;
      require(std::isfinite(rel), FC_ERR_NAN, "residual is not finite");
      if (rel <= tol) {
        RP.rank_Z[k] = Z.R;
        RP.rank_P[k] = P.R;
        status = FC_OK;
      } else {
        Z = lr2_apply_truncate(c, G, R, eps, cap);                  // lines 17-18
        const double rz_new = lr2_dot(st, R, Z);
        const double b_k = rz_new / rz;                             // line 19 (A16)
        P = lr2_truncate(st, lr2_axpy(st, Z, b_k, P), eps, cap);    // lines 20-21
        rz = rz_new;
        RP.rank_Z[k] = Z.R;
        RP.rank_P[k] = P.R;
      }
      FC_CUDA_TRY(cudaEventRecord(ti1, st));
      FC_CUDA_TRY(cudaEventSynchronize(ti1));
      float ms;
      cudaEventElapsedTime(&ms, ti0, ti1);
      RP.t_iter_ms[k] = ms;
      if (status == FC_OK) break;
    }
    FC_CUDA_TRY(cudaEventRecord(t1, st));
    FC_CUDA_TRY(cudaEventSynchronize(t1));
    float tl, tt;
    cudaEventElapsedTime(&tl, loop0, t1);
    cudaEventElapsedTime(&tt, t0, t1);
    RP.t_loop_ms = tl;
    RP.t_total_ms = tt;
    RP.converged = status == FC_OK;
    RP.status = status;
    lr2_store(st, X, u);
    FC_CUDA_TRY(cudaStreamSynchronize(st));
    return status;
  });
}

}  // extern "C"
