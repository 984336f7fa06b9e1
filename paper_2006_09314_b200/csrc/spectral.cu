// S4: the spectral-diagonal CP  D[i,j,k] = f(lam1_i + lam2_j + lam3_k) ~ sum_t w_t u1 (x) u2 (x) u3
// [P:666-722], built by full-to-Tucker-to-canonical [P:720-722, P:1775-1789, P:1802-1812]
// without ever materialising the n^3 tensor (reading A9):
//   1. per mode, a range finder for the mode-l fibres: Phi_l[i, q] = f(lam_l,i + c_q) for p
//      geometric samples c_q of the sums of the other two spectra (the fibres are f(lam + c)
//      for c in that interval); orthonormal basis Q_l of range(Phi_l), kept to 1e-12 relative;
//   2. projected core T = D x1 Q1^T x2 Q2^T x3 Q3^T with D generated inside the DMMA GEMM's
//      A-operand load (n^3 f-evaluations, the dominant cost);
//   3. HOSVD of the small core: r_l minimal with tail <= (eps^2/3)||T||^2 (as the oracle's
//      full HOSVD of D, whose unfolding spectra T reproduces to the capture accuracy);
//   4. core2 = T x_l Ztil_l^T, Z_l = Q_l Ztil_l, then T2C (eps/2 cut, or the top `keep`).
//   5. SPD guard for the preconditioner (A7): min over the full n^3 grid > 0, else keep+1.
// Parity with the oracle is on entries, not on factors.
#include <cfloat>
#include <cstring>
#include <cmath>
#include <vector>
#include "cpops.cuh"
#include "eig.cuh"
#include "solver.cuh"
#include "tt.cuh"

namespace fc {
namespace {

constexpr int kSamples = 192;

__device__ __forceinline__ double spec_f(int kind, double alpha, double beta, double lam) {
  if (kind == FC_F) return beta * pow(lam, alpha) + pow(lam, -alpha);
  if (kind == FC_G) return 1.0 / (beta * pow(lam, alpha) + pow(lam, -alpha));
  if (kind == FC_POW_PLUS) return pow(lam, alpha);
  return pow(lam, -alpha);
}

// Phi[i + n*q] = f(lam_l[i] + c_q), c_q geometric in [la[0]+lb[0], la[n-1]+lb[n-1]]
__global__ void sample_fibres_kernel(int n, int p, const double* __restrict__ lam_l, const double* __restrict__ la,
                                     const double* __restrict__ lb, int kind, double alpha, double beta,
                                     double* Phi) {
  const double cmin = la[0] + lb[0], cmax = la[n - 1] + lb[n - 1];
  const double ratio = cmax / cmin;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * p;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx % n), q = (int)(idx / n);
    double c = (q == p - 1) ? cmax : cmin * pow(ratio, (double)q / (p - 1));
    Phi[idx] = spec_f(kind, alpha, beta, lam_l[i] + c);
  }
}

__global__ void scale_cols_inv_sqrt_kernel(int n, int s, const double* __restrict__ lam, double* W) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * s;
       idx += (long long)gridDim.x * blockDim.x)
    W[idx] *= 1.0 / sqrt(lam[idx / n]);
}

// T'[b + q2*(a + q1*c)] = T[a + q1*(b + q2*c)]
__global__ void permute12_kernel(int q1, int q2, int q3, const double* __restrict__ T, double* Tp) {
  const long long tot = (long long)q1 * q2 * q3;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    int a = (int)(idx % q1), b = (int)((idx / q1) % q2), c = (int)(idx / ((long long)q1 * q2));
    Tp[b + (size_t)q2 * (a + (size_t)q1 * c)] = T[idx];
  }
}

// out = T x_mode M^T ; T dims d[3] (column-major), M is d[mode] x s, out dims with d[mode] -> s
__global__ void mode_product_kernel(int d0, int d1, int d2, int mode, int s, const double* __restrict__ T,
                                    const double* __restrict__ M, double* out) {
  int o[3] = {d0, d1, d2};
  const int dm = o[mode];
  o[mode] = s;
  const long long tot = (long long)o[0] * o[1] * o[2];
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    int id[3] = {(int)(idx % o[0]), (int)((idx / o[0]) % o[1]), (int)(idx / ((long long)o[0] * o[1]))};
    const int a = id[mode];
    double acc = 0.0;
    for (int x = 0; x < dm; ++x) {
      id[mode] = x;
      acc += T[id[0] + (size_t)d0 * (id[1] + (size_t)d1 * id[2])] * M[x + (size_t)a * dm];
    }
    out[idx] = acc;
  }
}

__global__ void sumsq_kernel(long long n, const double* __restrict__ x, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) acc += x[i] * x[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) *out = v;
  }
}

__device__ __forceinline__ unsigned long long ordered_key(double x) {
  unsigned long long b = __double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_to_double(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(b);
}

// min over the full n^3 grid of sum_t w_t U1[i,t] U2[j,t] U3[k,t]; thread per (i, j)
constexpr int kGuardMaxR = 64;        // rank search limit of the SPD guard (A7)
constexpr int kCpMinMaxR = kGuardMaxR + 1;   // + the A7'' constant term
__global__ void cp_min_kernel(int n, int r, const double* __restrict__ w, const double* __restrict__ U1,
                              const double* __restrict__ U2, const double* __restrict__ U3,
                              unsigned long long* out) {
  long long ij = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double mn = 1e300;
  if (ij < (long long)n * n) {
    int i = (int)(ij % n), j = (int)(ij / n);
    double a[kCpMinMaxR];
#pragma unroll 8
    for (int t = 0; t < r; ++t) a[t] = w[t] * U1[i + (size_t)t * n] * U2[j + (size_t)t * n];
    for (int k = 0; k < n; ++k) {
      double s = 0.0;
      for (int t = 0; t < r; ++t) s += a[t] * __ldg(U3 + k + (size_t)t * n);
      mn = fmin(mn, s);
    }
  }
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if ((threadIdx.x & 31) == 0) atomicMin(out, ordered_key(mn));
}

int nblk(long long tot) { return (int)std::min<long long>(std::max<long long>((tot + 255) / 256, 1), 148 * 8); }

struct Built {
  TT cp;            // spectral CP (Q = Z_l orthonormal, coefficients, weights)
  int tucker[3];
};

// steps 1-4
struct CoreResult {
  std::vector<DevMem> mem;
  double* core2 = nullptr;
  int s[3] = {0, 0, 0};
  double* Z[3] = {nullptr, nullptr, nullptr};
};

CoreResult spectral_tucker(fc_ctx c, int kind, double alpha, double beta, double eps, const double* lam3) {
  cudaStream_t st = c->st;
  const int n = c->n;
  auto lam_l = [&](int l) { return lam3 + (size_t)l * n; };
  Scratch s(st);
  const int p = std::min(kSamples, n);
  int q[3];
  double* Q[3];
  // 1. range finder per mode
  for (int l = 0; l < 3; ++l) {
    const int la = (l == 0) ? 1 : 0, lb = (l == 2) ? 1 : 2;
    double* Phi = s.alloc<double>((size_t)n * p);
    sample_fibres_kernel<<<nblk((long long)n * p), 256, 0, st>>>(n, p, lam_l(l), lam_l(la), lam_l(lb), kind,
                                                                 alpha, beta, Phi);
    FC_CHECK_LAUNCH();
    // orthonormal basis of range(Phi) by column-pivoted MGS (rank revealing, no squaring):
    // every sampled fibre is kept to 1e-14 of its norm
    Q[l] = s.alloc<double>((size_t)n * std::min(n, p));
    int* kk = s.alloc<int>(1);
    PmgsBatch pb;
    pb.nb = 1;
    pb.e[0] = PmgsEntry{n, p, Phi, n, Q[l], n, kk, 1e-14};
    pmgs(pb, st);
    int h = 0;
    FC_CUDA_TRY(cudaMemcpyAsync(&h, kk, sizeof(int), cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaStreamSynchronize(st));
    require(h >= 1, FC_ERR_NAN, "spectral function vanished on the grid");
    q[l] = h;
  }
  // 2. projected core: T3 = D_(12|3) Q3 (generated operand), T2 = per-c (n x n) Q2, T = Q1^T T2
  const size_t nn = (size_t)n * n;
  double* T3 = s.alloc<double>(nn * q[2]);
  {
    GemmArgs g;
    g.gen.kind = kind;
    g.gen.alpha = alpha;
    g.gen.beta = beta;
    g.gen.l1 = lam_l(0);
    g.gen.l2 = lam_l(1);
    g.gen.l3 = lam_l(2);
    g.gen.n1 = n;
    g.nbatch = 1;
    g.b[0] = GemmBatch{(int)nn, q[2], n, nullptr, (int)nn, Q[2], n, T3, (int)nn, nullptr, 0, nullptr};
    gemm(g, st);
  }
  double* T2 = s.alloc<double>((size_t)n * q[1] * q[2]);
  for (int c0 = 0; c0 < q[2]; c0 += kMaxBatch) {
    GemmArgs g;
    g.nbatch = std::min(kMaxBatch, q[2] - c0);
    for (int b = 0; b < g.nbatch; ++b)
      g.b[b] = GemmBatch{n, q[1], n, T3 + (size_t)(c0 + b) * nn, n, Q[1], n, T2 + (size_t)(c0 + b) * n * q[1], n,
                         nullptr, 0, nullptr};
    gemm(g, st);
  }
  const int q12 = q[1] * q[2];
  double* T = s.alloc<double>((size_t)q[0] * q12);
  dgemm(st, 1, 0, q[0], q12, n, 1.0, Q[0], n, T2, n, 0.0, T, q[0]);
  // 3. HOSVD of the core
  double* energy = s.alloc<double>(2);
  const long long qtot = (long long)q[0] * q12;
  sumsq_kernel<<<1, 1024, 0, st>>>(qtot, T, energy);
  FC_CHECK_LAUNCH();
  double* Tp = s.alloc<double>(qtot);
  permute12_kernel<<<nblk(qtot), 256, 0, st>>>(q[0], q[1], q[2], T, Tp);
  FC_CHECK_LAUNCH();
  double* Gm[3];
  for (int l = 0; l < 3; ++l) Gm[l] = s.zeros<double>((size_t)q[l] * q[l]);
  dgemm(st, 0, 1, q[0], q[0], q12, 1.0, T, q[0], T, q[0], 0.0, Gm[0], q[0]);
  dgemm(st, 0, 1, q[1], q[1], q[0] * q[2], 1.0, Tp, q[1], Tp, q[1], 0.0, Gm[1], q[1]);
  dgemm(st, 1, 0, q[2], q[2], q[0] * q[1], 1.0, T, q[0] * q[1], T, q[0] * q[1], 0.0, Gm[2], q[2]);
  SyevBatch eb;
  double* Zt[3];
  int* rl = s.alloc<int>(3);
  double* lamc[3];
  int maxq = 0;
  for (int l = 0; l < 3; ++l) {
    lamc[l] = s.alloc<double>(q[l]);
    Zt[l] = s.alloc<double>((size_t)q[l] * q[l]);
    eb.e[eb.nb++] = SyevEntry{q[l], Gm[l], q[l], s.alloc<double>(q[l]), s.alloc<double>(q[l]), lamc[l], Zt[l], q[l],
                              rl + l, s.alloc<double>((size_t)6 * q[l] * q[l])};
    maxq = std::max(maxq, q[l]);
  }
  syev_values(eb, st);
  for (int l = 0; l < 3; ++l) rank_cut_device(q[l], lamc[l], eps * eps / 3.0, energy, rl + l, nullptr, st);
  syev_vectors(eb, maxq, st);
  CoreResult out;
  FC_CUDA_TRY(cudaMemcpyAsync(out.s, rl, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  // 4. core2 = T x1 Zt1^T x2 Zt2^T x3 Zt3^T ;  Z_l = Q_l Zt_l
  int d[3] = {q[0], q[1], q[2]};
  double* cur = T;
  for (int l = 0; l < 3; ++l) {
    int o[3] = {d[0], d[1], d[2]};
    o[l] = out.s[l];
    double* nxt = s.alloc<double>((size_t)o[0] * o[1] * o[2]);
    mode_product_kernel<<<nblk((long long)o[0] * o[1] * o[2]), 256, 0, st>>>(d[0], d[1], d[2], l, out.s[l], cur,
                                                                             Zt[l], nxt);
    FC_CHECK_LAUNCH();
    cur = nxt;
    d[l] = out.s[l];
  }
  const size_t csz = (size_t)out.s[0] * out.s[1] * out.s[2];
  out.mem.emplace_back(csz * 8, st);
  out.core2 = out.mem.back().d();
  FC_CUDA_TRY(cudaMemcpyAsync(out.core2, cur, csz * 8, cudaMemcpyDeviceToDevice, st));
  for (int l = 0; l < 3; ++l) {
    out.mem.emplace_back((size_t)n * out.s[l] * 8, st);
    out.Z[l] = out.mem.back().d();
    dgemm(st, 0, 0, n, out.s[l], q[l], 1.0, Q[l], n, Zt[l], q[l], 0.0, out.Z[l], n);
  }
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  return out;
}

double cp_min_entry(fc_ctx c, const TT& x) {
  cudaStream_t st = c->st;
  const int n = c->n, r = x.R;
  require(r <= kCpMinMaxR, FC_ERR_CAPACITY, "SPD guard supports ranks <= 64 (+1 shift term)");
  Scratch s(st);
  double* U = s.alloc<double>((size_t)3 * n * r);
  double* w = s.alloc<double>(r);
  double* Up[3] = {U, U + (size_t)n * r, U + (size_t)2 * n * r};
  const int ld[3] = {n, n, n};
  tt_expand(st, x, Up, ld, w);
  unsigned long long* key = s.alloc<unsigned long long>(1);
  FC_CUDA_TRY(cudaMemsetAsync(key, 0xff, 8, st));
  cp_min_kernel<<<cdiv((long long)n * n, 128), 128, 0, st>>>(n, r, w, Up[0], Up[1], Up[2], key);
  FC_CHECK_LAUNCH();
  unsigned long long h = 0;
  FC_CUDA_TRY(cudaMemcpyAsync(&h, key, 8, cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  // decode on the host (same mapping as key_to_double)
  unsigned long long b = (h & 0x8000000000000000ull) ? (h & 0x7fffffffffffffffull) : ~h;
  double v;
  std::memcpy(&v, &b, 8);
  return v;
}

void store_spec(fc_ctx c, SpecCP& sp, const TT& x, const int tucker[3]) {
  cudaStream_t st = c->st;
  const int n = c->n, r = x.R;
  sp.r = r;
  sp.w.ensure(std::max(r, 1));
  sp.U.ensure((size_t)3 * n * std::max(r, 1));
  double* Up[3] = {sp.U.p, sp.U.p + (size_t)n * r, sp.U.p + (size_t)2 * n * r};
  const int ld[3] = {n, n, n};
  tt_expand(st, x, Up, ld, sp.w.p);
  sp.smax = std::max(x.q[0], std::max(x.q[1], x.q[2]));
  sp.W.ensure((size_t)3 * n * sp.smax);
  sp.E.ensure((size_t)3 * sp.smax * std::max(r, 1));
  for (int l = 0; l < 3; ++l) {
    sp.s[l] = x.q[l];
    sp.tucker_rank[l] = tucker[l];
    FC_CUDA_TRY(cudaMemcpyAsync(sp.W.p + (size_t)l * n * sp.smax, x.Q[l], (size_t)n * x.q[l] * 8,
                                cudaMemcpyDeviceToDevice, st));
    FC_CUDA_TRY(cudaMemcpyAsync(sp.E.p + (size_t)l * sp.smax * r, x.C[l], (size_t)x.q[l] * r * 8,
                                cudaMemcpyDeviceToDevice, st));
  }
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  sp.valid = true;
  sp.has_basis = true;
}

}  // namespace

// spectral CP of f(lam1 + lam2 + lam3) over the eigenvalues lam3 (3 x n; the context's SL
// eigenvalues, or the case-(A) Laplacian ones), applied in `basis` (nullptr: the SL basis)
void build_spectral_cp(fc_ctx c, int which, double alpha, double beta, double eps, int keep, bool spd_guard,
                       const double* lam3, const double* basis) {
  CoreResult cr = spectral_tucker(c, which, alpha, beta, eps, lam3);
  int k = keep;
  bool shifted = false;
  TT x = tucker_to_canonical(c, cr.core2, cr.s, cr.Z, c->n, eps, k, 0, nullptr);
  if (spd_guard) {
    // reading A7': raise the T2C rank (<= 64) until the CP is positive on the full grid; if the
    // Tucker approximation itself is not positive at that accuracy, tighten its tolerance
    // tenfold (down to eps/1e4) and restart from `keep` (same rule as the oracle)
    double e = eps, mn;
    while ((mn = cp_min_entry(c, x)) <= 0.0) {
      const int maxr = std::min(kGuardMaxR, cr.s[0] * cr.s[1] * cr.s[2]);
      if (k < maxr) {
        ++k;
      } else if (e > eps * 1e-4 * 1.0000001) {
        e /= 10.0;
        cr = spectral_tucker(c, which, alpha, beta, e, lam3);
        k = keep;
      } else {
        // reading A7'': add the constant s (x) 1 (x) 1 (x) 1, s = 2|min| + 1e-15 sum|w|
        const int n = c->n;
        std::vector<double> hw(x.R);
        FC_CUDA_TRY(cudaMemcpyAsync(hw.data(), x.w, (size_t)x.R * 8, cudaMemcpyDeviceToHost, c->st));
        FC_CUDA_TRY(cudaStreamSynchronize(c->st));
        double sw = 0.0;
        for (double v : hw) sw += std::fabs(v);
        const double shift = 2.0 * std::fabs(mn) + 1e-15 * sw;
        std::vector<double> h1((size_t)n + 1, 1.0 / std::sqrt((double)n));
        h1[n] = shift * std::pow((double)n, 1.5);
        Scratch s1(c->st);
        double* d1 = s1.alloc<double>((size_t)n + 1);
        FC_CUDA_TRY(cudaMemcpyAsync(d1, h1.data(), ((size_t)n + 1) * 8, cudaMemcpyHostToDevice, c->st));
        double* ones[3] = {d1, d1, d1};
        const int ld1[3] = {n, n, n};
        TT one = tt_from_cp(c->st, n, 1, d1 + n, ones, ld1);
        x = tt_axpy(c->st, x, 1.0, one);
        FC_CUDA_TRY(cudaStreamSynchronize(c->st));
        mn = cp_min_entry(c, x);
        require(mn > 0.0, FC_ERR_NOT_SPD, "preconditioner CP not positive on the grid after the A7'' shift");
        shifted = true;
        break;
      }
      x = tucker_to_canonical(c, cr.core2, cr.s, cr.Z, c->n, e, k, 0, nullptr);
    }
  }
  store_spec(c, c->spec[which], x, cr.s);
  if (shifted) c->spec[which].has_basis = false;   // the appended term: recompute W, E (pmgs)
  c->spec[which].basis = basis;
}

// ---- sinc-quadrature construction [P:325-351, P:725-752] ------------
// lam^-a = 1/Gamma(a) int_R exp(a x - lam e^x) dx ~ sum_k c_k exp(-t_k lam), t_k = e^(x_k),
// c_k = h e^(a x_k) / Gamma(a), h = 2 pi d / ln(1/eps) with the strip half-width d = pi/3 (the
// error constant grows towards d = pi/2); [x_lo, x_hi] drops the tails below
// eps Gamma(a) lam^-a on [lam_min, lam_max] (lower: e^(a x_lo)/a; upper: L^a e^-L, L = lam_min e^x_hi)
void sinc_nodes_host(double a, double lam_min, double lam_max, double eps, std::vector<double>& t,
                     std::vector<double>& c) {
  const double g = std::tgamma(a), h = 2.0 * M_PI * (M_PI / 3.0) / std::log(1.0 / eps);
  const double x_lo = (std::log(eps * a * g) - a * std::log(lam_max)) / a;
  double L = std::log(1.0 / (eps * g));
  for (int i = 0; i < 20; ++i) L = std::log(1.0 / (eps * g)) + a * std::log(std::max(L, 1.0));
  const double x_hi = std::log(L / lam_min);
  const int m = (int)std::ceil((x_hi - x_lo) / h);
  t.resize(m + 1);
  c.resize(m + 1);
  for (int k = 0; k <= m; ++k) {
    const double x = x_lo + h * k;
    t[k] = std::exp(x);
    c[k] = h * std::exp(a * x) / g;
  }
}

// column k of mode l (block (k, l)): U = exp(-t_k lam_l) / norm, nrm[l*R + k] = norm
__global__ void sinc_factor_kernel(int n, int R, const double* __restrict__ lam3, const double* __restrict__ t,
                                   double* U, double* nrm) {
  __shared__ double red[32];
  const int k = blockIdx.x, l = blockIdx.y;
  const double* lam = lam3 + (size_t)l * n;
  double* u = U + (size_t)l * n * R + (size_t)k * n;
  double part = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = exp(-t[k] * lam[i]);
    u[i] = v;
    part = fma(v, v, part);
  }
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  double s2 = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s2 += red[w];
  const double nr = sqrt(s2), inv = nr > 0 ? 1.0 / nr : 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) u[i] *= inv;
  if (threadIdx.x == 0) nrm[(size_t)l * R + k] = nr;
}

// D (.) Q: term m*R + k, mode l factor (l == m ? lam_l : 1) .* Q_l[:, k]  (D = lam-sum, rank 3)
__global__ void lam_hadamard_kernel(int n, int R, const double* __restrict__ lam3, const double* __restrict__ Q,
                                    double* out) {
  const long long tot = 3LL * 3 * R * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % n);
    const int term = (int)((idx / n) % (3 * R));
    const int l = (int)(idx / ((long long)n * 3 * R));
    const int m = term / R, k = term % R;
    const double q = Q[(size_t)l * n * R + (size_t)k * n + i];
    out[idx] = (l == m ? lam3[(size_t)l * n + i] : 1.0) * q;
  }
}

namespace {
// CP of lam^-a over the context's lam-sums by the sinc rule, as a (plain, rank 2M+1) TT
TT sinc_pow_minus_tt(fc_ctx c, double a, double eps) {
  cudaStream_t st = c->st;
  const int n = c->n;
  double lo = 0.0, hi = 0.0;
  for (int l = 0; l < 3; ++l) {
    double e[2];
    FC_CUDA_TRY(cudaMemcpyAsync(e, c->lam_l(l), 8, cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaMemcpyAsync(e + 1, c->lam_l(l) + n - 1, 8, cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaStreamSynchronize(st));
    lo += e[0];
    hi += e[1];
  }
  std::vector<double> t, cw;
  sinc_nodes_host(a, lo, hi, eps, t, cw);
  const int R = (int)t.size();
  Scratch s(st);
  double* td = s.alloc<double>(R);
  double* U = s.alloc<double>((size_t)3 * n * R);
  double* nrm = s.alloc<double>((size_t)3 * R);
  FC_CUDA_TRY(cudaMemcpyAsync(td, t.data(), (size_t)R * 8, cudaMemcpyHostToDevice, st));
  sinc_factor_kernel<<<dim3(R, 3), 256, 0, st>>>(n, R, c->lam.p, td, U, nrm);
  FC_CHECK_LAUNCH();
  std::vector<double> hn((size_t)3 * R);
  FC_CUDA_TRY(cudaMemcpyAsync(hn.data(), nrm, hn.size() * 8, cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  for (int k = 0; k < R; ++k) cw[k] *= hn[k] * hn[R + k] * hn[2 * R + k];
  double* wd = s.alloc<double>(R);
  FC_CUDA_TRY(cudaMemcpyAsync(wd, cw.data(), (size_t)R * 8, cudaMemcpyHostToDevice, st));
  double* Up[3] = {U, U + (size_t)n * R, U + (size_t)2 * n * R};
  const int ld[3] = {n, n, n};
  TT x = tt_from_cp(st, n, R, wd, Up, ld);
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  return x;
}

// lam^a = lam-sum (.) lam^(a-1), truncated at eps (a = 1: the rank-3 lam-sum itself)
TT sinc_pow_plus_tt(fc_ctx c, double a, double eps) {
  cudaStream_t st = c->st;
  const int n = c->n;
  Scratch s(st);
  int R;
  std::vector<double> hw;
  double* Q;
  if (a >= 1.0) {   // the lam-sum: Q = one unit constant column per mode, weight sqrt(n)^2 ... via R = 1
    R = 1;
    std::vector<double> h1((size_t)3 * n, 1.0 / std::sqrt((double)n));
    Q = s.alloc<double>((size_t)3 * n);
    FC_CUDA_TRY(cudaMemcpyAsync(Q, h1.data(), h1.size() * 8, cudaMemcpyHostToDevice, st));
    hw.assign(1, std::pow((double)n, 1.5));
  } else {
    TT q = sinc_pow_minus_tt(c, 1.0 - a, eps);
    R = q.R;
    Q = s.alloc<double>((size_t)3 * n * R);
    double* Qp[3] = {Q, Q + (size_t)n * R, Q + (size_t)2 * n * R};
    const int ld[3] = {n, n, n};
    double* qw = s.alloc<double>(R);
    tt_expand(st, q, Qp, ld, qw);
    hw.resize(R);
    FC_CUDA_TRY(cudaMemcpyAsync(hw.data(), qw, (size_t)R * 8, cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaStreamSynchronize(st));
  }
  double* H = s.alloc<double>((size_t)3 * n * 3 * R);
  lam_hadamard_kernel<<<nblk(9LL * R * n), 256, 0, st>>>(n, R, c->lam.p, Q, H);
  FC_CHECK_LAUNCH();
  std::vector<double> w3((size_t)3 * R);
  for (int m = 0; m < 3; ++m)
    for (int k = 0; k < R; ++k) w3[(size_t)m * R + k] = hw[k];
  double* wd = s.alloc<double>((size_t)3 * R);
  FC_CUDA_TRY(cudaMemcpyAsync(wd, w3.data(), w3.size() * 8, cudaMemcpyHostToDevice, st));
  double* Hp[3] = {H, H + (size_t)n * 3 * R, H + (size_t)2 * n * 3 * R};
  const int ld[3] = {n, n, n};
  TT x = tt_from_cp(st, n, 3 * R, wd, Hp, ld);
  return truncate_tt(c, x, eps, 0, nullptr);
}
}  // namespace

// op_build_spectral_sinc: spectral CP of `which` (FC_POW_MINUS: the sinc rule itself, rank 2M+1,
// untruncated; FC_POW_PLUS: lam-sum (.) lam^(alpha-1), truncated; FC_F: beta lam^alpha + lam^-alpha,
// truncated) over the context's SL eigenvalues
void build_spectral_sinc(fc_ctx c, int which, double eps) {
  require(c->have_params, FC_ERR_NOT_READY, "alpha/beta unknown: call sl_setup (or sl_set_eigen with params)");
  require(c->n > 0 && c->have_eig[0] && c->have_eig[1] && c->have_eig[2], FC_ERR_NOT_READY, "eigenpairs missing");
  require(which == FC_POW_MINUS || which == FC_POW_PLUS || which == FC_F, FC_ERR_INVALID_ARG,
          "sinc construction: FC_POW_MINUS, FC_POW_PLUS or FC_F");
  require(eps > 0 && eps < 1, FC_ERR_INVALID_ARG, "eps in (0, 1)");
  const double a = c->p.alpha, b = c->p.beta;
  TT x;
  if (which == FC_POW_MINUS) {
    x = sinc_pow_minus_tt(c, a, eps);
  } else if (which == FC_POW_PLUS) {
    x = sinc_pow_plus_tt(c, a, eps);
  } else {
    TT pm = sinc_pow_minus_tt(c, a, eps);
    TT pp = sinc_pow_plus_tt(c, a, eps);
    TT sum = tt_axpy(c->st, pm, b, pp);
    x = truncate_tt(c, sum, eps, 0, nullptr);
  }
  const int tk[3] = {x.q[0], x.q[1], x.q[2]};
  store_spec(c, c->spec[which], x, tk);
  c->spec[which].basis = nullptr;
  if (which == FC_POW_MINUS) c->spec[which].has_basis = false;   // plain CP: recompute W, E
}

void ensure_spectral(fc_ctx c, int which) {
  SpecCP& sp = c->spec[which];
  if (sp.valid || (which != FC_POW_PLUS && which != FC_POW_MINUS)) return;
  require(c->have_params, FC_ERR_NOT_READY, "spectral CP of A^+-alpha needs alpha: call sl_setup or pass params");
  require(c->n > 0 && c->have_eig[0] && c->have_eig[1] && c->have_eig[2], FC_ERR_NOT_READY, "eigenpairs missing");
  const double epsD = c->p.eps_D > 0 ? c->p.eps_D : c->p.eps;
  build_spectral_cp(c, which, c->p.alpha, c->p.beta, epsD, c->p.op_rank > 0 ? c->p.op_rank : 0, false, c->lam.p,
                    nullptr);
}

// case-(A) preconditioner basis [P:772-785, P:842-849]: b0_l = (max a~_l + min a~_l)/2 over the
// midpoint values the operator uses (A2); lam_k = b0_l 4/h^2 sin^2(k pi h/2), k = 1..n (ascending),
// V[i, k] = sqrt(2h) sin(i k pi h) (DST-I, orthonormal), i, k = 1..n
__global__ void laplace_basis_kernel(int n, double b0a, double b0b, double b0c, double* lam, double* V) {
  const double h = 1.0 / (n + 1), pi = 3.141592653589793;
  const double b0[3] = {b0a, b0b, b0c};
  const int l = blockIdx.y;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % n), k = (int)(idx / n);
    // sin(i k pi h) with the argument reduced exactly: (i k) mod 2(n+1) keeps it in [0, 2 pi)
    const long long m = ((long long)(i + 1) * (k + 1)) % (2LL * (n + 1));
    V[(size_t)l * n * n + idx] = sqrt(2.0 * h) * sin((double)m * pi * h);
    if (i == 0) {
      const double sk = sin((k + 1) * pi * h / 2.0);
      lam[(size_t)l * n + k] = b0[l] * 4.0 / (h * h) * sk * sk;
    }
  }
}

void precond_basis_A(fc_ctx c, const double* a_mid, int boundary) {
  const int n = c->n;
  double b0[3];
  for (int l = 0; l < 3; ++l) {
    const double* a = a_mid + (size_t)l * (n + 1);
    // effective midpoints (A2): boundary = 0 replaces the two end values by their neighbours
    const int i0 = boundary == 0 ? 1 : 0, i1 = boundary == 0 ? n - 1 : n;
    double mx = a[i0], mn = a[i0];
    for (int i = i0; i <= i1; ++i) {
      mx = std::max(mx, a[i]);
      mn = std::min(mn, a[i]);
    }
    b0[l] = 0.5 * (mx + mn);
  }
  c->lamA.ensure((size_t)3 * n);
  c->VA.ensure((size_t)3 * n * n);
  laplace_basis_kernel<<<dim3(nblk((long long)n * n), 3), 256, 0, c->st>>>(n, b0[0], b0[1], b0[2], c->lamA.p, c->VA.p);
  FC_CHECK_LAUNCH();
  for (auto& h : c->have_A) h = true;
}

}  // namespace fc

using namespace fc;

extern "C" int sl_setup(fc_ctx c, int n, const double* a_mid, const fc_params* p) {
  if (!c) return FC_ERR_INVALID_ARG;
  try {
    require(p != nullptr && a_mid != nullptr, FC_ERR_INVALID_ARG, "NULL argument");
    require(n >= 2, FC_ERR_INVALID_ARG, "n must be >= 2");
    require(p->alpha > 0 && p->alpha <= 1, FC_ERR_INVALID_ARG, "alpha must be in (0, 1]");
    require(p->beta > 0 && std::isfinite(p->beta), FC_ERR_INVALID_ARG, "beta must be > 0");
    require(p->eps > 0 && std::isfinite(p->eps), FC_ERR_INVALID_ARG, "eps must be > 0");
    for (long long i = 0; i < 3LL * (n + 1); ++i)
      require(std::isfinite(a_mid[i]) && a_mid[i] > 0, FC_ERR_NONPOS_COEF, "midpoint coefficient <= 0 or non-finite");
    cudaStream_t st = c->st;
    c->n = n;
    c->p = *p;
    c->have_params = true;
    c->lam.ensure((size_t)3 * n);
    c->V.ensure((size_t)3 * n * n);
    for (auto& h : c->have_eig) h = false;
    for (auto& sp : c->spec) sp.valid = false;
    Scratch s(st);
    double* a_dev = s.alloc<double>((size_t)3 * (n + 1));
    int* status = s.zeros<int>(1);
    FC_CUDA_TRY(cudaMemcpyAsync(a_dev, a_mid, (size_t)3 * (n + 1) * 8, cudaMemcpyHostToDevice, st));
    sl_eigen_device(st, n, a_dev, p->boundary, c->lam.p, c->V.p, status);
    int hs = 0;
    FC_CUDA_TRY(cudaMemcpyAsync(&hs, status, sizeof(int), cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaStreamSynchronize(st));
    require(hs == 0, hs, "coefficient check failed on the device");
    for (auto& h : c->have_eig) h = true;
    const double epsD = p->eps_D > 0 ? p->eps_D : p->eps;
    require(p->precond_case == FC_PRECOND_B || p->precond_case == FC_PRECOND_A, FC_ERR_INVALID_ARG,
            "precond_case must be FC_PRECOND_B or FC_PRECOND_A");
    build_spectral_cp(c, FC_F, p->alpha, p->beta, epsD, p->op_rank > 0 ? p->op_rank : 0, false, c->lam.p, nullptr);
    for (auto& h : c->have_A) h = false;
    if (p->precond_case == FC_PRECOND_A) {
      precond_basis_A(c, a_mid, p->boundary);
      build_spectral_cp(c, FC_G, p->alpha, p->beta, epsD, p->precond_rank > 0 ? p->precond_rank : 6, true,
                        c->lamA.p, c->VA.p);
    } else {
      build_spectral_cp(c, FC_G, p->alpha, p->beta, epsD, p->precond_rank > 0 ? p->precond_rank : 6, true,
                        c->lam.p, nullptr);
    }
    return FC_OK;
  } catch (const Error& e) {
    c->err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    c->err = e.what();
    return FC_ERR_CUDA;
  }
}
