// Eigen machinery on the device.
//
// (a) S1-S3, the 1D Sturm-Liouville eigenpairs [P:466-542]: assembly of the bidiagonal factor
//     C (T = C^T C, the paper's weak form [P:477]), Sturm-count bisection on the Golub-Kahan
//     zero-diagonal tridiagonal of C (singular values to high relative accuracy, lam = s^2),
//     inverse iteration per eigenvector on T, sign rule, Newton-Schulz orthogonality polish on
//     DMMA GEMMs.  One thread per eigenvalue / eigenvector: n independent problems per mode.
// (b) The small symmetric eigensolves of the truncation (S11): Householder tridiagonalisation
//     (one CTA per matrix), bisection for all eigenvalues (thread per eigenvalue), inverse
//     iteration for the leading r vectors, CGS2 re-orthonormalisation, back-transformation.
#include <cfloat>
#include <cstdlib>
#include <cstdio>
#include <vector>
#include <cmath>
#include <algorithm>
#include <cooperative_groups.h>
#include "eig.cuh"

namespace fc {
namespace {

constexpr double kEps = DBL_EPSILON;

// ---------------------------------------------------------------------------------------
// (a) 1D setup
// ---------------------------------------------------------------------------------------
// per mode: a~ (paper boundary rule A2), s_r = sqrt(a~_r)/h (r = 0..n), d, e of T = C^T C.
__global__ void sl_assemble_kernel(int n, const double* __restrict__ a_mid, int boundary, double* s_out,
                                   double* d_out, double* e_out, int* status) {
  const int l = blockIdx.y;
  const double* a = a_mid + (size_t)l * (n + 1);
  double* s = s_out + (size_t)l * (n + 1);
  double* d = d_out + (size_t)l * n;
  double* e = e_out + (size_t)l * n;
  const double h = 1.0 / (n + 1), ih2 = 1.0 / (h * h);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= n; r += gridDim.x * blockDim.x) {
    int src = r;
    if (boundary == 0) {
      if (r == 0) src = 1;
      if (r == n) src = n - 1;
    }
    double ar = a[src];
    if (!(ar > 0.0) || !isfinite(ar)) atomicExch(status, FC_ERR_NONPOS_COEF);
    s[r] = sqrt(ar) / h;
    if (r < n) {
      int s0 = r, s1 = r + 1;
      if (boundary == 0) {
        if (s0 == 0) s0 = 1;
        if (s1 == n) s1 = n - 1;
      }
      d[r] = (a[s0] + a[s1]) * ih2;
      if (r < n - 1) e[r] = -a[s1] * ih2;
    }
  }
}

// #{ singular values of C < x } via the Sturm count of the (2n+1) zero-diagonal Golub-Kahan
// tridiagonal with off-diagonals |f| = (s0, s1, s1, s2, s2, ..., s_{n-1}, s_n), x > 0.
__device__ int gk_count(int n, const double* __restrict__ s, double x, double pivmin) {
  double q = -x;
  int cnt = 1;  // q0 = -x < 0
  for (int k = 0; k < 2 * n; ++k) {
    double f = s[(k + 1) >> 1];
    q = -x - f * f / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += (q < 0.0);
  }
  return cnt - (n + 1);
}

__global__ void gk_bisect_kernel(int n, const double* __restrict__ s_all, double* lam_out) {
  const int l = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* s = s_all + (size_t)l * (n + 1);
  double smax = 0.0;
  for (int r = 0; r <= n; ++r) smax = fmax(smax, s[r]);
  const double pivmin = DBL_MIN / kEps * fmax(1.0, smax * smax);
  double lo = 0.0, hi = 2.0 * smax * (1.0 + 4 * kEps);
  for (int it = 0; it < 200; ++it) {
    double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (hi - lo <= 2.0 * kEps * hi) break;
    if (gk_count(n, s, mid, pivmin) >= i + 1) hi = mid;
    else lo = mid;
  }
  double sig = 0.5 * (lo + hi);
  lam_out[(size_t)l * n + i] = sig * sig;
}

// ---- tridiagonal inverse iteration (shared by (a) and (b)) ---------------------------
// T = tridiag(e, d, e) of size N.  Scratch arrays strided by `stride` (coalesced across
// threads): 5 arrays of N entries (u0 holds the reciprocal pivots), and with `own_work` a sixth
// one holding the iterate (coalesced, instead of the caller's column v: the solves then touch
// only coalesced scratch).  Writes the unit vector into v[k*vstride].  All pointers are
// restrict-qualified (the arrays are disjoint), so the loads of the recurrences can be issued
// ahead of the FMA chain.
__device__ void tri_invit(int N, const double* __restrict__ d, const double* __restrict__ e, double lam,
                          double tnorm, double* scr, size_t stride, double* v_out, size_t vstride, unsigned seed,
                          bool own_work = false, int nsolve = 3) {
  double* __restrict__ u0 = scr;
  double* __restrict__ u1 = scr + (size_t)N * stride;
  double* __restrict__ u2 = scr + (size_t)2 * N * stride;
  double* __restrict__ lm = scr + (size_t)3 * N * stride;
  double* __restrict__ pv = scr + (size_t)4 * N * stride;
  double* __restrict__ v = own_work ? scr + (size_t)5 * N * stride : v_out;
  const size_t vs = own_work ? stride : vstride;
  const double tiny = kEps * tnorm + DBL_MIN;
#define S(a, k) a[(size_t)(k) * stride]
#define V(k) v[(size_t)(k) * vs]
  if (N == 1) {
    v_out[0] = 1.0;
    return;
  }
  // LU with partial pivoting of T - lam I (rows k, k+1 interact only)
  double cd = d[0] - lam, cs = e[0], cs2 = 0.0;   // current row k: diag, sup, sup2
  for (int k = 0; k < N - 1; ++k) {
    double sub = e[k];                      // T[k+1, k]
    double ad = d[k + 1] - lam;             // T[k+1, k+1]
    double as = (k + 1 < N - 1) ? e[k + 1] : 0.0;
    if (fabs(sub) > fabs(cd)) {
      double m = cd / sub;
      S(u0, k) = 1.0 / sub; S(u1, k) = ad; S(u2, k) = as;
      S(lm, k) = m; S(pv, k) = 1.0;
      double nd = cs - m * ad, ns = cs2 - m * as;
      cd = nd; cs = ns; cs2 = 0.0;
    } else {
      if (fabs(cd) < tiny) cd = (cd >= 0 ? tiny : -tiny);
      double m = sub / cd;
      S(u0, k) = 1.0 / cd; S(u1, k) = cs; S(u2, k) = cs2;
      S(lm, k) = m; S(pv, k) = 0.0;
      cd = ad - m * cs; cs = as; cs2 = 0.0;
    }
  }
  if (fabs(cd) < tiny) cd = (cd >= 0 ? tiny : -tiny);
  S(u0, N - 1) = 1.0 / cd; S(u1, N - 1) = 0.0; S(u2, N - 1) = 0.0;
  // start vector: deterministic hash in [0.5, 1.5)
  for (int k = 0; k < N; ++k) {
    unsigned h = (unsigned)k * 2654435761u ^ (seed * 2246822519u + 0x9E3779B9u);
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    V(k) = 0.5 + (h & 0xFFFFFF) / 16777216.0;
  }
  double scale = 1.0;                       // the previous solve's 1 / max|x|, folded into the next
  for (int it = 0; it < nsolve; ++it) {
    // forward: apply P and L (the running entry carried in a register; every load below is
    // independent of the recurrence, so the loop is an FMA chain)
    double carry = V(0) * scale;
    for (int k = 0; k < N - 1; ++k) {
      double bk = carry, bk1 = V(k + 1) * scale;
      if (S(pv, k) != 0.0) { double t = bk; bk = bk1; bk1 = t; }
      bk1 -= S(lm, k) * bk;
      V(k) = bk;
      carry = bk1;
    }
    V(N - 1) = carry;
    // backward with U (3 diagonals; u0 holds the reciprocal pivots)
    double x2 = 0.0, x1 = 0.0, nrm = 0.0;
    for (int k = N - 1; k >= 0; --k) {
      double x = (V(k) - S(u1, k) * x1 - S(u2, k) * x2) * S(u0, k);
      V(k) = x;
      x2 = x1; x1 = x;
      nrm = fmax(nrm, fabs(x));
    }
    scale = 1.0 / nrm;                      // rescale by the max-abs entry (keeps the next solve in range)
  }
  double s2 = 0.0;
  for (int k = 0; k < N; ++k) { double x = V(k) * scale; s2 += x * x; }
  const double inv = scale / sqrt(s2);
  if (own_work)
    for (int k = 0; k < N; ++k) v_out[(size_t)k * vstride] = V(k) * inv;
  else
    for (int k = 0; k < N; ++k) V(k) *= inv;                 // v is v_out (only accessed through v)
#undef V
#undef S
}

// one inverse-iteration solve with the LU factors tri_invit stored in `scr` (same layout)
__device__ void tri_lu_solve(int N, const double* scr, size_t stride, double* v) {
  const double* u0 = scr;
  const double* u1 = scr + (size_t)N * stride;
  const double* u2 = scr + (size_t)2 * N * stride;
  const double* lm = scr + (size_t)3 * N * stride;
  const double* pv = scr + (size_t)4 * N * stride;
#define S(a, k) a[(size_t)(k) * stride]
  double carry = v[0];
  for (int k = 0; k < N - 1; ++k) {
    double bk = carry, bk1 = v[k + 1];
    if (S(pv, k) != 0.0) { double t = bk; bk = bk1; bk1 = t; }
    bk1 -= S(lm, k) * bk;
    v[k] = bk;
    carry = bk1;
  }
  v[N - 1] = carry;
  double x2 = 0.0, x1 = 0.0;
  for (int k = N - 1; k >= 0; --k) {
    double x = (v[k] - S(u1, k) * x1 - S(u2, k) * x2) * S(u0, k);   // u0: reciprocal pivots
    v[k] = x;
    x2 = x1; x1 = x;
  }
#undef S
}

// sign rule (reading A4): entry of largest magnitude positive, ties -> lowest index
__device__ void sign_rule(int N, double* v, size_t vstride) {
  double best = -1.0, sgn = 1.0;
  for (int k = 0; k < N; ++k) {
    double x = v[(size_t)k * vstride];
    if (fabs(x) > best) { best = fabs(x); sgn = x < 0 ? -1.0 : 1.0; }
  }
  if (sgn < 0)
    for (int k = 0; k < N; ++k) v[(size_t)k * vstride] = -v[(size_t)k * vstride];
}

__global__ void sl_invit_kernel(int n, const double* __restrict__ d_all, const double* __restrict__ e_all,
                                const double* __restrict__ lam_all, double* V_all, double* scratch) {
  const int l = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* d = d_all + (size_t)l * n;
  const double* e = e_all + (size_t)l * n;
  const double lam = lam_all[(size_t)l * n + i];
  double tnorm = 0.0;
  for (int k = 0; k < n; ++k) tnorm = fmax(tnorm, fabs(d[k]) + 2.0 * (k < n - 1 ? fabs(e[k]) : 0.0));
  const size_t stride = (size_t)3 * n;
  double* scr = scratch + (size_t)l * n + i;
  double* v = V_all + (size_t)l * n * n + (size_t)i * n;
  tri_invit(n, d, e, lam, tnorm, scr, stride, v, 1, (unsigned)i);
  sign_rule(n, v, 1);
}

// Near-degenerate eigenvalues (relative gap < kClusterGap): inverse iteration from different
// start vectors may return (nearly) the same vector for every member of the cluster.  One
// thread per cluster re-runs modified Gram-Schmidt (twice) over the cluster's vectors in index
// order; any orthonormal basis of a cluster's span is an eigenbasis to the accuracy the gap
// allows (reading A25).  Clusters are short runs (pairs in practice).
constexpr double kClusterGap = 1e-10;
__global__ void sl_cluster_orth_kernel(int n, const double* __restrict__ lam_all, const double* __restrict__ d_all,
                                       const double* __restrict__ e_all, double* V_all,
                                       const double* __restrict__ scratch) {
  const int l = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* lam = lam_all + (size_t)l * n;
  double* V = V_all + (size_t)l * n * n;
  auto close = [&](int a, int b) { return (lam[b] - lam[a]) <= kClusterGap * fabs(lam[b]); };
  if (i > 0 && close(i - 1, i)) return;           // not the first member
  if (i + 1 >= n || !close(i, i + 1)) return;      // singleton
  int end = i + 1;
  while (end + 1 < n && close(end, end + 1)) ++end;
  for (int j = i + 1; j <= end; ++j) {
    double* vj = V + (size_t)j * n;
    // inverse iteration with orthogonalisation against the earlier members (LAPACK stein):
    // solve with member j's stored LU factors, then MGS, three times
    const double* scr = scratch + (size_t)l * n + j;
    for (int it = 0; it < 3; ++it) {
      tri_lu_solve(n, scr, (size_t)3 * n, vj);
      for (int k = i; k < j; ++k) {
        const double* vk = V + (size_t)k * n;
        double dd = 0.0;
        for (int t = 0; t < n; ++t) dd += vk[t] * vj[t];
        for (int t = 0; t < n; ++t) vj[t] -= dd * vk[t];
      }
      double s2 = 0.0;
      for (int t = 0; t < n; ++t) s2 += vj[t] * vj[t];
      const double inv = 1.0 / sqrt(s2);
      for (int t = 0; t < n; ++t) vj[t] *= inv;
    }
    for (int pass = 0; pass < 2; ++pass) {
      for (int k = i; k < j; ++k) {
        const double* vk = V + (size_t)k * n;
        double d = 0.0;
        for (int t = 0; t < n; ++t) d += vk[t] * vj[t];
        for (int t = 0; t < n; ++t) vj[t] -= d * vk[t];
      }
      double s2 = 0.0;
      for (int t = 0; t < n; ++t) s2 += vj[t] * vj[t];
      double inv = 1.0 / sqrt(s2);
      for (int t = 0; t < n; ++t) vj[t] *= inv;
    }
  }
  // Rayleigh-Ritz inside the cluster: Jacobi sweeps on H = Vc^T T Vc (k <= 8), rotating the
  // cluster's vectors, so each vector is an eigenvector to the accuracy the true gap allows
  // (an arbitrary rotation inside the span would leave residuals of order gap).
  const int k = end - i + 1;
  if (k > 8) return;
  const double* d = d_all + (size_t)l * n;
  const double* e = e_all + (size_t)l * n;
  double H[8][8];
  for (int a = 0; a < k; ++a) {
    const double* va = V + (size_t)(i + a) * n;
    for (int b = a; b < k; ++b) {
      const double* vb = V + (size_t)(i + b) * n;
      double h = 0.0;   // va^T T vb with T = tridiag(e, d, e)
      for (int t = 0; t < n; ++t) {
        double tv = d[t] * vb[t];
        if (t > 0) tv += e[t - 1] * vb[t - 1];
        if (t + 1 < n) tv += e[t] * vb[t + 1];
        h += va[t] * tv;
      }
      H[a][b] = H[b][a] = h;
    }
  }
  for (int sweep = 0; sweep < 10; ++sweep) {
    double off = 0.0;
    for (int a = 0; a < k; ++a)
      for (int b = a + 1; b < k; ++b) off += H[a][b] * H[a][b];
    if (off == 0.0) break;
    for (int a = 0; a < k; ++a)
      for (int b = a + 1; b < k; ++b) {
        if (H[a][b] == 0.0) continue;
        const double zeta = (H[b][b] - H[a][a]) / (2.0 * H[a][b]);
        const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
        for (int m = 0; m < k; ++m) {          // H <- J^T H J
          const double hma = H[m][a], hmb = H[m][b];
          H[m][a] = c * hma - s * hmb;
          H[m][b] = s * hma + c * hmb;
        }
        for (int m = 0; m < k; ++m) {
          const double ham = H[a][m], hbm = H[b][m];
          H[a][m] = c * ham - s * hbm;
          H[b][m] = s * ham + c * hbm;
        }
        double* va = V + (size_t)(i + a) * n;
        double* vb = V + (size_t)(i + b) * n;
        for (int t = 0; t < n; ++t) {
          const double x = va[t], y = vb[t];
          va[t] = c * x - s * y;
          vb[t] = s * x + c * y;
        }
      }
  }
  // keep ascending order of the Ritz values inside the cluster (selection sort by swapping)
  for (int a = 0; a < k; ++a) {
    int best = a;
    for (int b = a + 1; b < k; ++b)
      if (H[b][b] < H[best][best]) best = b;
    if (best != a) {
      double tmp = H[a][a]; H[a][a] = H[best][best]; H[best][best] = tmp;
      double* va = V + (size_t)(i + a) * n;
      double* vb = V + (size_t)(i + best) * n;
      for (int t = 0; t < n; ++t) { double x = va[t]; va[t] = vb[t]; vb[t] = x; }
    }
  }
}

// G <- 1.5 I - 0.5 G  (Newton-Schulz step V <- V (3I - V^T V)/2)
__global__ void ns_matrix_kernel(int n, double* G) {
  const int l = blockIdx.y;
  double* g = G + (size_t)l * n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx % n), j = (int)(idx / n);
    g[idx] = (i == j ? 1.5 : 0.0) - 0.5 * g[idx];
  }
}

// ---------------------------------------------------------------------------------------
// (b) small symmetric eigensolver
// ---------------------------------------------------------------------------------------
constexpr int kTriThreads = 512;
constexpr int kSmemMaxN = 150;   // (N^2 + 18 N) * 8 <= 202 KB in shared memory, else global (L2)
constexpr int kPackedMaxN = 230; // packed lower triangle in shared memory up to this size
constexpr int kClusterMinN = 96; // above this the cluster kernels take over (FC_NO_CLUSTER: 230)
constexpr size_t kTriSmemMax = 220 * 1024;

__device__ double block_sum(double v, double* red) {
  for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  __syncthreads();
  if (ln == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int s = 16; s > 0; s >>= 1) t += __shfl_down_sync(0xffffffffu, t, s);
    if (threadIdx.x == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// block_sum without the leading barrier: only for call sites where every earlier reader of `red`
// is separated from this call by another block-wide barrier
__device__ double block_sum_nl(double v, double* red) {
  for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  if (ln == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int s = 16; s > 0; s >>= 1) t += __shfl_down_sync(0xffffffffu, t, s);
    if (threadIdx.x == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// NaN-propagating maximum (a NaN anywhere makes the result NaN)
__device__ __forceinline__ double nan_max(double a, double b) { return (b > a || b != b) ? b : a; }

__device__ double block_max(double v, double* red) {
  for (int s = 16; s > 0; s >>= 1) v = nan_max(v, __shfl_down_sync(0xffffffffu, v, s));
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  __syncthreads();
  if (ln == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int s = 16; s > 0; s >>= 1) t = nan_max(t, __shfl_down_sync(0xffffffffu, t, s));
    if (threadIdx.x == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// Householder tridiagonalisation (lower triangle), in place: after return column k (rows
// k+1..) holds the unit Householder vector u_k (H_k = I - 2 u u^T; zero column = identity),
// E.d / E.e the tridiagonal.  One CTA per matrix; the matrix lives in shared memory when
// N <= kSmemMaxN, else in global memory (L2).  Only the lower triangle is read and updated:
//   p = A22 u  column by column (warp per column, lanes over rows, coalesced): column j adds
//              A[i,j] u_j to p_i (i >= j) and sum_{i>j} A[i,j] u_i to p_j, into per-warp
//              partial vectors that are summed afterwards;
//   A22 -= 2 (u q^T + q u^T) on the lower triangle (warp per column).
__global__ void __launch_bounds__(kTriThreads) tridiag_kernel(const __grid_constant__ SyevBatch B, int minN) {
  extern __shared__ double sm[];
  __shared__ double red[33];
  __shared__ double alpha_s;
  const SyevEntry& E = B.e[blockIdx.x];
  const int N = E.N;
  if (N <= minN) return;                 // handled by the packed / cluster kernels
  constexpr int NW = kTriThreads / 32;
  const bool use_sm = false;
  double* M = use_sm ? sm : E.A;
  const int ld = use_sm ? N : E.lda;
  double* base = use_sm ? sm + (size_t)N * N : sm;
  double* uvec = base;              // N
  double* p = base + N;             // N
  double* pw = base + 2 * N;        // NW x N warp partials
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, ln = tid & 31;
  if (use_sm)
    for (int idx = tid; idx < N * N; idx += nt) M[idx] = E.A[(idx % N) + (size_t)(idx / N) * E.lda];
  __syncthreads();
  for (int k = 0; k + 2 < N; ++k) {
    const int m = N - k - 1;                  // trailing size; x = M[k+1.., k]
    double* col_k = M + (k + 1) + (size_t)k * ld;
    double* A22 = M + (k + 1) + (size_t)(k + 1) * ld;
    const double x0 = col_k[0];
    double part = 0.0;
    for (int i = tid + 1; i < m; i += nt) part += col_k[i] * col_k[i];
    const double sig = block_sum(part, red);
    const bool skip = (sig == 0.0);
    double alpha = x0;
    if (!skip) {
      alpha = -copysign(sqrt(x0 * x0 + sig), x0);
      const double v0 = x0 - alpha;
      const double inv = 1.0 / sqrt(sig + v0 * v0);
      for (int i = tid; i < m; i += nt) uvec[i] = (i == 0 ? v0 : col_k[i]) * inv;
      for (int i = tid; i < NW * m; i += nt) pw[(i / m) * N + (i % m)] = 0.0;
    }
    __syncthreads();
    if (!skip) {
      // p = A22 u from the lower triangle
      for (int j = warp; j < m; j += NW) {
        const double* cj = A22 + (size_t)j * ld;
        const double uj = uvec[j];
        double* pwj = pw + (size_t)warp * N;
        double dot = 0.0;
        for (int i = j + ln; i < m; i += 32) {
          const double a = cj[i];
          pwj[i] += a * uj;
          if (i > j) dot += a * uvec[i];
        }
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (ln == 0) pwj[j] += dot;
        __syncwarp();
      }
      __syncthreads();
      double kp = 0.0;
      for (int i = tid; i < m; i += nt) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += pw[(size_t)w * N + i];
        p[i] = s;
        kp += uvec[i] * s;
      }
      const double K = block_sum(kp, red);
      for (int i = tid; i < m; i += nt) p[i] -= K * uvec[i];   // q
      __syncthreads();
      // lower-triangle rank-2 update
      for (int j = warp; j < m; j += NW) {
        double* cj = A22 + (size_t)j * ld;
        const double uj = uvec[j], qj = p[j];
        for (int i = j + ln; i < m; i += 32) cj[i] -= 2.0 * (uvec[i] * qj + p[i] * uj);
      }
      __syncthreads();
    }
    if (tid == 0) alpha_s = alpha;
    __syncthreads();
    for (int i = tid; i < m; i += nt) col_k[i] = skip ? 0.0 : uvec[i];
    if (tid == 0) M[k + (size_t)(k + 1) * ld] = alpha_s;          // e_k in the (stale) upper slot
    __syncthreads();
  }
  if (tid == 0) {
    for (int k = 0; k < N; ++k) E.d[k] = M[k + (size_t)k * ld];
    for (int k = 0; k + 1 < N; ++k) E.e[k] = (k + 2 < N) ? M[k + (size_t)(k + 1) * ld] : M[(k + 1) + (size_t)k * ld];
  }
  __syncthreads();
  if (use_sm)
    for (int idx = tid; idx < N * N; idx += nt) E.A[(idx % N) + (size_t)(idx / N) * E.lda] = M[idx];
}


// Same Householder tridiagonalisation with the lower triangle packed in shared memory
// (N(N+1)/2 doubles: N <= 230 fits in 216 KB), 1024 threads, matvec partials by shared-memory
// atomics.  Column j is contiguous at off(j) = j N - j(j-1)/2; element (i, j), i >= j, at
// off(j) + i - j.
__global__ void __launch_bounds__(1024) tridiag_packed_kernel(const __grid_constant__ SyevBatch B, int maxN) {
  extern __shared__ double sm[];
  __shared__ double red[33];
  __shared__ double alpha_s;
  const SyevEntry& E = B.e[blockIdx.x];
  const int N = E.N;
  if (N <= 0 || N > maxN) return;
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, ln = tid & 31, NW = nt >> 5;
  const size_t P = (size_t)N * (N + 1) / 2;
  double* L = sm;
  double* u = sm + P;
  double* p = u + N;
  auto off = [N](int j) { return (size_t)j * N - (size_t)j * (j - 1) / 2; };
  for (int j = warp; j < N; j += NW)
    for (int i = j + ln; i < N; i += 32) L[off(j) + (i - j)] = E.A[i + (size_t)j * E.lda];
  __syncthreads();
  for (int k = 0; k + 2 < N; ++k) {
    const int m = N - k - 1;
    double* colk = L + off(k) + 1;           // x = A[k+1.., k]
    const double x0 = colk[0];
    double part = 0.0;
    for (int i = tid + 1; i < m; i += nt) part += colk[i] * colk[i];
    const double sig = block_sum_nl(part, red);   // previous use: >= 3 barriers back
    const bool skip = (sig == 0.0);
    double alpha = x0;
    if (!skip) {
      alpha = -copysign(sqrt(x0 * x0 + sig), x0);
      const double v0 = x0 - alpha;
      const double inv = 1.0 / sqrt(sig + v0 * v0);
      for (int i = tid; i < m; i += nt) {
        u[i] = (i == 0 ? v0 : colk[i]) * inv;
        p[i] = 0.0;
      }
    }
    __syncthreads();
    if (!skip) {
      // p = A u, one warp per row in a fixed summation order (deterministic; the lower triangle
      // holds element (k+1+ii, k+1+jj), ii >= jj, at L[off(k+1+jj) + ii - jj])
      for (int ii = warp; ii < m; ii += NW) {
        double dot = 0.0;
        for (int jj = ln; jj < m; jj += 32) {
          const double a = jj <= ii ? L[off(k + 1 + jj) + (ii - jj)] : L[off(k + 1 + ii) + (jj - ii)];
          dot = fma(a, u[jj], dot);
        }
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (ln == 0) p[ii] = dot;
      }
      __syncthreads();
      double kp = 0.0;
      for (int i = tid; i < m; i += nt) kp += u[i] * p[i];
      const double K = block_sum_nl(kp, red);    // previous use: >= 2 barriers back
      for (int i = tid; i < m; i += nt) p[i] -= K * u[i];
      __syncthreads();
      for (int jj = warp; jj < m; jj += NW) {
        double* cj = L + off(k + 1 + jj);
        const double uj = u[jj], qj = p[jj];
        for (int ii = jj + ln; ii < m; ii += 32) cj[ii - jj] -= 2.0 * (u[ii] * qj + p[ii] * uj);
      }
      __syncthreads();
    }
    if (tid == 0) alpha_s = alpha;
    __syncthreads();
    for (int i = tid; i < m; i += nt) colk[i] = skip ? 0.0 : u[i];
    if (tid == 0) E.e[k] = alpha_s;
    __syncthreads();
  }
  // d, the last off-diagonal, and the Householder vectors back to global memory
  for (int k = tid; k < N; k += nt) E.d[k] = L[off(k)];
  if (tid == 0 && N >= 2) E.e[N - 2] = L[off(N - 2) + 1];
  for (int k = warp; k + 2 < N; k += NW)
    for (int i = ln; i < N - k - 1; i += 32) E.A[(k + 1 + i) + (size_t)k * E.lda] = L[off(k) + 1 + i];
}

// Same Householder tridiagonalisation on a thread-block cluster of CS CTAs (one cluster per
// matrix): column j of the packed lower triangle lives in the shared memory of CTA j % CS.
// Per step s (pivot column s, trailing block rows/cols >= s+1):
//   every CTA holds the pivot column and computes the Householder vector u redundantly (same
//   code, same data -> bit-identical in every CTA; no broadcast);
//   partial matvec Y_c = A22[:, own cols] u (thread per row, lower part) + the own-column dots
//   (warp per column, upper part by symmetry);
//   cluster barrier; reduce-scatter: CTA c sums the CS partials of its index slice through DSMEM
//   and fetches its slice of the (not yet updated) next pivot column from that column's owner;
//   cluster barrier; all-gather of p and of the next pivot column; q = p - (u^T p) u; the next
//   pivot column is updated and its Householder vector formed (redundantly); the rank-2 update
//   of the own columns is fused with the next step's partial matvec.
// Two cluster barriers per step; the owner of a slice serves only that slice (DSMEM reads are
// paid by the owner's shared-memory port).
constexpr int kCl4MaxN = 440;    // packed own columns + 5 N vectors fit 220 KB with 4 CTAs
constexpr int kCl8MaxN = 600;    // ... with 8 CTAs
constexpr int kCl16MaxN = 840;   // ... with 16 CTAs (non-portable cluster size)

template <int CS, bool GL = false>
__host__ __device__ inline size_t cluster_smem_doubles(int N) {
  const int ncol0 = (N + CS - 1) / CS;                                 // CTA 0 owns the most
  const size_t P = GL ? 0 : (size_t)ncol0 * N - (size_t)CS * ncol0 * (ncol0 - 1) / 2;
  const int SL = (N + CS - 1) / CS;
  return P + 4 * (size_t)N + (size_t)CS * SL + 2 * (size_t)SL;
}
// GL hybrid: the number of leading own columns that fit shared memory (220 KB) next to the
// vectors (CTA 0's packed sizes, the largest), and the resulting dynamic shared memory
inline int cluster_gl_tsm(int N, size_t* smem_bytes) {
  constexpr int CS = 16;
  const size_t vec = cluster_smem_doubles<CS, true>(N);
  const size_t cap = 220 * 1024 / 8;
  const int SL = (N + CS - 1) / CS;
  int t = 0;
  auto loff0 = [N](int tt) { return (size_t)tt * N - (size_t)CS * tt * (tt - 1) / 2; };
  while (t < SL && vec + loff0(t + 1) <= cap) ++t;
  *smem_bytes = (vec + loff0(t)) * 8;
  return t;
}
constexpr int kClGlobalMaxN = 2048;   // GL cluster path (own columns in L2) up to this size

// a - 2 (ui qj + qi uj) with explicit roundings (identical wherever it is evaluated)
__device__ __forceinline__ double rank2(double a, double ui, double qi, double uj, double qj) {
  return __fma_rn(-2.0, __fma_rn(ui, qj, __dmul_rn(qi, uj)), a);
}

// GL (N > kCl16MaxN): the own columns do not fit shared memory; each CTA keeps them in a
// private slice of E.scratch (L2-resident: the whole triangle is <= 16 MB at N = 2048) and the
// next pivot column is fetched from the owner's slice with L1-bypassing loads (ld.global.cg:
// the owner updates it between fetches); the vectors stay in shared memory (DSMEM as above).
//   Hybrid: the first `tsm` own columns stay in shared memory (as many as fit next to the vectors,
//   DSMEM pivot fetches), the rest in the L2 slice; tsm >= ncol is the all-shared-memory layout.
template <int CS, bool GL>
__global__ void __launch_bounds__(1024, 1) tridiag_cluster_kernel(const __grid_constant__ SyevBatch B, int nlo,
                                                                  int nhi, int tsm_arg) {
  namespace cg = cooperative_groups;
  extern __shared__ double sm[];
  __shared__ double red[33];
  cg::cluster_group cl = cg::this_cluster();
  const SyevEntry& E = B.e[blockIdx.y];
  const int N = E.N;
  if (N <= nlo || N > nhi) return;                       // this launch's size class (uniform)
  const int c = (int)cl.block_rank();
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, ln = tid & 31, NW = nt >> 5;
  const int ncol = (N - c + CS - 1) / CS;                // own columns j = c + t CS
  const int SL = (N + CS - 1) / CS;                      // index slice [c SL, (c+1) SL)
  auto loff_of = [N](int o, int t) { return (size_t)t * (N - o) - (size_t)CS * t * (t - 1) / 2; };
  // the same layout in every CTA (CTA 0 owns the most entries): map_shared_rank(ptr, r) maps
  // to the same offset in CTA r
  const size_t P = loff_of(0, SL);
  const int tsm = GL ? tsm_arg : SL;                     // own columns t < tsm in shared memory
  const size_t Psm = loff_of(0, min(tsm, SL));           // their (largest, CTA 0) packed size
  double* L = sm;                                        // shared-memory part (columns t < tsm)
  // L2 part (columns t >= tsm): column t at Lg + loff_of(c, t) (offsets below loff_of(c, tsm) unused)
  double* Lg = GL ? E.scratch + (size_t)c * P - loff_of(c, min(tsm, ncol)) : nullptr;
  auto colp = [&](int t) -> double* { return (GL && t >= tsm ? Lg : L) + loff_of(c, t); };
  double* u = sm + Psm;       // Householder vector of the current step (absolute row index)
  double* u1 = u + N;         // ... of the next step
  double* col = u1 + N;       // current pivot column (absolute row index)
  double* Y = col + N;        // partial matvec (read remotely)
  double* q = Y + N;          // p / q (size CS*SL >= N; reduce-scatter scratch in phase 3)
  double* ps = q + (size_t)CS * SL;   // my slice of p (read remotely)
  double* ncs = ps + SL;              // my slice of the next pivot column (read remotely)

  for (int t = warp; t < ncol; t += NW) {
    const int j = c + t * CS;
    double* dst = colp(t);
    for (int i = j + ln; i < N; i += 32) dst[i - j] = E.A[i + (size_t)j * E.lda];
  }
  for (int i = tid; i < N; i += nt) col[i] = E.A[i];
  __syncthreads();

  // Householder vector of pivot column s (in col): uu[s+1..N), returns alpha (= e_s)
  auto house = [&](int s, double* uu) -> double {
    const double x0 = col[s + 1];
    double part = 0.0;
    for (int i = s + 2 + tid; i < N; i += nt) part += col[i] * col[i];
    const double sig = block_sum_nl(part, red);   // previous use (phase 4) is >= 2 barriers back
    double alpha = x0;
    if (sig == 0.0) {
      for (int i = s + 1 + tid; i < N; i += nt) uu[i] = 0.0;
    } else {
      alpha = -copysign(sqrt(x0 * x0 + sig), x0);
      const double v0 = x0 - alpha;
      const double inv = 1.0 / sqrt(sig + v0 * v0);
      for (int i = s + 1 + tid; i < N; i += nt) uu[i] = (i == s + 1 ? v0 : col[i]) * inv;
    }
    __syncthreads();
    return alpha;
  };
  // own columns j >= jupd get the rank-2 update of (u, q); partial matvec of step ssym with w
  // over own columns j >= ssym+1 into Y (rows >= ssym+1)
  auto pass = [&](int jupd, bool upd, int ssym, const double* w) {
    const int jsym = ssym + 1;
    const int lo = min(jupd, jsym);
    for (int i = lo + tid; i < N; i += nt) {
      const double ui = upd ? u[i] : 0.0, qi = upd ? q[i] : 0.0;
      double acc = 0.0;
      int t = max(0, (lo - c + CS - 1) / CS);
      size_t off = loff_of(c, t);
      for (int j = c + t * CS; j <= i; j += CS, ++t) {
        double* a = (GL && t >= tsm ? Lg : L) + off + (i - j);
        double v = *a;
        if (upd && j >= jupd) {
          v = rank2(v, ui, qi, u[j], q[j]);
          *a = v;
        }
        if (j >= jsym) acc = fma(v, w[j], acc);
        off += (size_t)(N - j);
      }
      Y[i] = acc;
    }
    __syncthreads();
    for (int t = max(0, (jsym - c + CS - 1) / CS) + warp; t < ncol; t += NW) {
      const int j = c + t * CS;
      const double* a = colp(t);
      double dot = 0.0;
      for (int i = j + 1 + ln; i < N; i += 32) dot = fma(a[i - j], w[i], dot);
      for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (ln == 0) Y[j] += dot;
    }
  };

  double alpha = house(0, u);
  if (c == 0 && tid == 0) {
    E.d[0] = col[0];
    E.e[0] = alpha;
  }
  pass(N, false, 0, u);
  for (int s = 0; s + 2 < N; ++s) {
    cl.sync();                                                           // (A) partials ready
    // ---- phase 3: reduce-scatter of p(s) over my slice, my slice of the next pivot column ----
    const int i0 = max(c * SL, s + 1), i1 = min(N, (c + 1) * SL);
    const int cnt = max(0, i1 - i0);
    for (int idx = tid; idx < cnt * CS; idx += nt) {
      const int i = i0 + idx % cnt, src = idx / cnt;
      q[idx] = cl.map_shared_rank(Y, src)[i];
    }
    {
      const int jn = s + 1, o = jn % CS, tn = jn / CS;
      if (GL && tn >= tsm) {
        const int ncol_o = (N - o + CS - 1) / CS;
        const double* Lo = E.scratch + (size_t)o * P - loff_of(o, min(tsm, ncol_o)) + loff_of(o, tn);
        for (int i = i0 + tid; i < i1; i += nt) ncs[i - c * SL] = __ldcg(Lo + (i - jn));
      } else {
        const double* Lo = cl.map_shared_rank(L, o) + loff_of(o, tn);
        for (int i = i0 + tid; i < i1; i += nt) ncs[i - c * SL] = Lo[i - jn];
      }
    }
    if (c == 0)   // the Householder vector of step s into column s of A (all initial reads are done)
      for (int i = s + 1 + tid; i < N; i += nt) E.A[i + (size_t)s * E.lda] = u[i];
    __syncthreads();
    for (int i = i0 + tid; i < i1; i += nt) {
      double v = 0.0;
      for (int src = 0; src < CS; ++src) v += q[(i - i0) + src * cnt];
      ps[i - c * SL] = v;
    }
    cl.sync();                                                           // (B) slices ready
    // ---- phase 4: all-gather; q = p - (u^T p) u; next pivot column and its Householder vector ----
    for (int i = s + 1 + tid; i < N; i += nt) {
      const int o = i / SL;
      q[i] = cl.map_shared_rank(ps, o)[i - o * SL];
      col[i] = cl.map_shared_rank(ncs, o)[i - o * SL];
    }
    // no barrier: this thread's u . q partial reads only the q[i] it just gathered (and u from
    // the previous step, already behind barriers); the barrier inside block_sum_nl orders the rest
    double kp = 0.0;
    for (int i = s + 1 + tid; i < N; i += nt) kp += u[i] * q[i];
    const double K = block_sum_nl(kp, red);
    for (int i = s + 1 + tid; i < N; i += nt) q[i] -= K * u[i];
    __syncthreads();
    {
      const double us = u[s + 1], qs = q[s + 1];
      for (int i = s + 1 + tid; i < N; i += nt) col[i] = rank2(col[i], u[i], q[i], us, qs);
    }
    __syncthreads();
    const bool more = (s + 3 < N);
    if (more) {
      alpha = house(s + 1, u1);
      if (c == 0 && tid == 0) {
        E.d[s + 1] = col[s + 1];
        E.e[s + 1] = alpha;
      }
    } else if (c == 0 && tid == 0) {
      E.d[s + 1] = col[s + 1];
      E.e[s + 1] = col[s + 2];
    }
    // ---- rank-2 update of own columns >= s+2, fused with the partial matvec of step s+1 ----
    pass(s + 2, true, more ? s + 1 : N, u1);
    __syncthreads();
    double* tmp = u;
    u = u1;
    u1 = tmp;
  }
  if (tid == 0 && (N - 1) % CS == c) E.d[N - 1] = *colp((N - 1) / CS);
  cl.sync();                                                             // smem stays alive for readers
}

__device__ int tri_count(int N, const double* __restrict__ d, const double* __restrict__ e, double x,
                         double pivmin) {
  double q = d[0] - x;
  int cnt = q < 0.0;
  for (int k = 1; k < N; ++k) {
    if (fabs(q) < pivmin) q = -pivmin;
    q = d[k] - x - e[k - 1] * e[k - 1] / q;
    cnt += (q < 0.0);
  }
  return cnt;
}

// Sturm count from shared-memory copies of d and e^2, with the correctly rounded reciprocal
// instead of the (longer) division sequence: q <- (d_k - x) - e_{k-1}^2 * rcp(q)
__device__ __forceinline__ int tri_count_s(int N, const double* __restrict__ d, const double* __restrict__ e2,
                                           double x, double pivmin) {
  double q = d[0] - x;
  int cnt = q < 0.0;
  for (int k = 1; k < N; ++k) {
    if (fabs(q) < pivmin) q = -pivmin;
    q = fma(-e2[k - 1], __drcp_rn(q), d[k] - x);
    cnt += (q < 0.0);
  }
  return cnt;
}

// warp per eigenvalue (multisection); lam[i] = i-th largest.  Each round the 32 lanes count
// the eigenvalues below 32 equispaced interior points of [lo, hi]; the interval shrinks 33x.
// d and e^2 are staged in shared memory (2 N doubles) for the Sturm counts.
__global__ void tri_bisect_kernel(const __grid_constant__ SyevBatch B) {
  extern __shared__ double sde[];
  const SyevEntry& E = B.e[blockIdx.y];
  const int N = E.N;
  double* ds = sde;
  double* e2s = sde + N;
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    ds[k] = E.d[k];
    e2s[k] = k < N - 1 ? E.e[k] * E.e[k] : 0.0;
  }
  __syncthreads();
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int ln = threadIdx.x & 31;
  if (i >= N) return;
  double lo = 1e300, hi = -1e300, emax = 0.0;
  for (int k = ln; k < N; k += 32) {
    double r = (k > 0 ? fabs(E.e[k - 1]) : 0.0) + (k < N - 1 ? fabs(E.e[k]) : 0.0);
    lo = fmin(lo, E.d[k] - r);
    hi = fmax(hi, E.d[k] + r);
    if (k < N - 1) emax = fmax(emax, fabs(E.e[k]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  }
  const double tnorm = fmax(fabs(lo), fabs(hi));
  const double pivmin = DBL_MIN / kEps * fmax(1.0, emax * emax);
  lo -= 2 * kEps * tnorm + pivmin;
  hi += 2 * kEps * tnorm + pivmin;
  const int target = N - i;  // want the target-th smallest (1-based)
  const double atol = 2.0 * kEps * tnorm + pivmin;
  for (int it = 0; it < 60; ++it) {
    if (hi - lo <= fmax(atol, 2.0 * kEps * fmax(fabs(lo), fabs(hi)))) break;
    const double x = lo + (hi - lo) * ((double)(ln + 1) / 33.0);
    const bool ge = (x > lo && x < hi) ? tri_count_s(N, ds, e2s, x, pivmin) >= target : (x >= hi);
    const unsigned m = __ballot_sync(0xffffffffu, ge);
    // first lane whose point has >= target eigenvalues below it: new interval (x_{j-1}, x_j]
    const int j = m ? __ffs(m) - 1 : 32;
    const double xl = j > 0 ? __shfl_sync(0xffffffffu, x, j - 1) : lo;
    const double xh = j < 32 ? __shfl_sync(0xffffffffu, x, j & 31) : hi;
    if (xl <= lo && xh >= hi) break;   // no progress (interval at rounding resolution)
    lo = xl;
    hi = xh;
  }
  if (ln == 0) E.lam[i] = 0.5 * (lo + hi);
}

// thread per wanted vector (i < r): inverse iteration on (d, e) into Y[:, i]
__global__ void tri_invit_kernel(const __grid_constant__ SyevBatch B, int nsolve) {
  const SyevEntry& E = B.e[blockIdx.y];
  const int N = E.N;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = min(*E.r, N);
  if (i >= r) return;
  double tnorm = 0.0;
  for (int k = 0; k < N; ++k) tnorm = fmax(tnorm, fabs(E.d[k]) + 2.0 * (k < N - 1 ? fabs(E.e[k]) : 0.0));
  tri_invit(N, E.d, E.e, E.lam[i], tnorm, E.scratch + i, (size_t)N, E.Y + (size_t)i * E.ldy, 1, (unsigned)(i + 17),
            true, nsolve);
}

// tri_invit_kernel with each vector's LU factors and iterate in shared memory, interleaved by
// thread ([k T + t]: conflict-free), and d, e staged once per CTA: the sequential recurrences
// (LU, forward, backward) then read operands at shared-memory latency, independent of the
// recurrence and so prefetchable, instead of an L2 round trip per step.  Same operations in the
// same order as tri_invit (bit-identical vectors).
__global__ void tri_invit_smem_kernel(const __grid_constant__ SyevBatch B, int nsolve) {
  extern __shared__ double ism[];
  const SyevEntry& E = B.e[blockIdx.y];
  const int N = E.N, T = blockDim.x, t = threadIdx.x;
  const int r = min(*E.r, N);
  const int i0 = blockIdx.x * T;
  if (i0 >= r) return;   // uniform over the CTA
  double* __restrict__ ds = ism;
  double* __restrict__ es = ism + N;
  double* __restrict__ u0 = ism + 2 * (size_t)N;
  double* __restrict__ u1 = u0 + (size_t)N * T;
  double* __restrict__ u2 = u1 + (size_t)N * T;
  double* __restrict__ lm = u2 + (size_t)N * T;
  double* __restrict__ v = lm + (size_t)N * T;
  unsigned char* __restrict__ pv = reinterpret_cast<unsigned char*>(v + (size_t)N * T);
  for (int k = t; k < N; k += T) {
    ds[k] = E.d[k];
    es[k] = k < N - 1 ? E.e[k] : 0.0;
  }
  __syncthreads();
  const int i = i0 + t;
  if (i >= r) return;
  double tnorm = 0.0;
  for (int k = 0; k < N; ++k) tnorm = fmax(tnorm, fabs(ds[k]) + 2.0 * (k < N - 1 ? fabs(es[k]) : 0.0));
  const double lam = E.lam[i];
  double* vout = E.Y + (size_t)i * E.ldy;
  if (N == 1) {
    vout[0] = 1.0;
    return;
  }
  const double tiny = kEps * tnorm + DBL_MIN;
#define S(a, k) a[(size_t)(k) * T + t]
  double cd = ds[0] - lam, cs = es[0], cs2 = 0.0;
  for (int k = 0; k < N - 1; ++k) {
    double sub = es[k];
    double ad = ds[k + 1] - lam;
    double as = (k + 1 < N - 1) ? es[k + 1] : 0.0;
    if (fabs(sub) > fabs(cd)) {
      double m = cd / sub;
      S(u0, k) = 1.0 / sub; S(u1, k) = ad; S(u2, k) = as;
      S(lm, k) = m; S(pv, k) = 1;
      double nd = cs - m * ad, ns = cs2 - m * as;
      cd = nd; cs = ns; cs2 = 0.0;
    } else {
      if (fabs(cd) < tiny) cd = (cd >= 0 ? tiny : -tiny);
      double m = sub / cd;
      S(u0, k) = 1.0 / cd; S(u1, k) = cs; S(u2, k) = cs2;
      S(lm, k) = m; S(pv, k) = 0;
      cd = ad - m * cs; cs = as; cs2 = 0.0;
    }
  }
  if (fabs(cd) < tiny) cd = (cd >= 0 ? tiny : -tiny);
  S(u0, N - 1) = 1.0 / cd; S(u1, N - 1) = 0.0; S(u2, N - 1) = 0.0;
  const unsigned seed = (unsigned)(i + 17);
  for (int k = 0; k < N; ++k) {
    unsigned h = (unsigned)k * 2654435761u ^ (seed * 2246822519u + 0x9E3779B9u);
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    S(v, k) = 0.5 + (h & 0xFFFFFF) / 16777216.0;
  }
  double scale = 1.0;
  for (int it = 0; it < nsolve; ++it) {
    double carry = S(v, 0) * scale;
#pragma unroll 4
    for (int k = 0; k < N - 1; ++k) {
      double bk = carry, bk1 = S(v, k + 1) * scale;
      if (S(pv, k) != 0) { double tt = bk; bk = bk1; bk1 = tt; }
      bk1 -= S(lm, k) * bk;
      S(v, k) = bk;
      carry = bk1;
    }
    S(v, N - 1) = carry;
    double x2 = 0.0, x1 = 0.0, nrm = 0.0;
#pragma unroll 4
    for (int k = N - 1; k >= 0; --k) {
      double x = (S(v, k) - S(u1, k) * x1 - S(u2, k) * x2) * S(u0, k);
      S(v, k) = x;
      x2 = x1; x1 = x;
      nrm = fmax(nrm, fabs(x));
    }
    scale = 1.0 / nrm;
  }
  double s2 = 0.0;
  for (int k = 0; k < N; ++k) { double x = S(v, k) * scale; s2 += x * x; }
  const double inv = scale / sqrt(s2);
  for (int k = 0; k < N; ++k) vout[k] = S(v, k) * inv;
#undef S
}

// one CTA per matrix: CGS2 orthonormalisation of Y[:, 0..r) in order, then back-transform
// with the Householder vectors stored in A: z = H_0 H_1 ... H_{N-3} y.
// (flag != nullptr: only the entries with flag[i] != 0 are processed; the polar path below
// handles the others)
__global__ void __launch_bounds__(1024) orth_backtransform_kernel(const __grid_constant__ SyevBatch B,
                                                                  const int* __restrict__ flag) {
  __shared__ double red[33];
  extern __shared__ double coef[];   // r coefficients
  if (flag && flag[blockIdx.x] == 0) return;
  const SyevEntry& E = B.e[blockIdx.x];
  const int N = E.N;
  const int r = min(*E.r, N);
  const int tid = threadIdx.x, nt = blockDim.x;
  double* Y = E.Y;
  const int ldy = E.ldy;
  for (int i = 0; i < r; ++i) {
    double* yi = Y + (size_t)i * ldy;
    for (int pass = 0; pass < 2; ++pass) {
      // coef[j] = y_j . y_i for j < i (warp per j)
      const int w = tid >> 5, ln = tid & 31;
      for (int j = w; j < i; j += nt / 32) {
        const double* yj = Y + (size_t)j * ldy;
        double s = 0.0;
        for (int k = ln; k < N; k += 32) s += yj[k] * yi[k];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (ln == 0) coef[j] = s;
      }
      __syncthreads();
      for (int k = tid; k < N; k += nt) {
        double acc = yi[k];
        for (int j = 0; j < i; ++j) acc -= coef[j] * Y[(size_t)j * ldy + k];
        yi[k] = acc;
      }
      __syncthreads();
    }
    double part = 0.0;
    for (int k = tid; k < N; k += nt) part += yi[k] * yi[k];
    double s2 = block_sum(part, red);
    double inv = s2 > 0 ? 1.0 / sqrt(s2) : 0.0;
    for (int k = tid; k < N; k += nt) yi[k] *= inv;
    __syncthreads();
  }
}

// Polar orthonormalisation of inverse-iteration vectors (syev_vectors with host-known ranks):
// Newton-Schulz steps Y <- Y D (3I - D G D) / 2 with G = Y^T Y on batched DMMA GEMMs.  The
// inverse-iteration vectors are orthogonal to eps ||T|| / gap: in the C4 solve max|G - I| is
// below 1e-8 in 186 of 198 calls and at most 1.3e-4 (FC_TRACE_ORTH), so two steps reach
// ~1e-17 (0.75 e^2 per step).  Symmetric (Loewdin) orthogonalisation mixes vectors i, j by
// ~G_ij ~ eps ||T|| / |lam_i - lam_j|, which moves their residuals by ~eps ||T||: as accurate as
// Gram-Schmidt, and order-free.  Entries whose first error exceeds kOrthPolarMax keep H = I
// (bit-exact copies) and are flagged for the CGS2 kernel.
constexpr double kOrthPolarMax = 1e-4;
struct PolarBatch {
  int nb = 0;
  int r[kMaxSyev];
  double* G[kMaxSyev];      // r x r Gram, overwritten by H
  int* flag;                // device, nb entries (zeroed by the caller)
};

__global__ void __launch_bounds__(1024) ns_polar_kernel(const __grid_constant__ PolarBatch P, int step) {
  __shared__ double red[33];
  extern __shared__ double dsc[];   // r scale factors
  const int e = blockIdx.x, r = P.r[e];
  double* G = P.G[e];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int a = tid; a < r; a += nt) {
    const double g = G[a + (size_t)a * r];
    dsc[a] = g > 0.0 ? 1.0 / sqrt(g) : 0.0;
  }
  __syncthreads();
  double err = 0.0;
  const size_t cnt = (size_t)r * r;
  for (size_t i = tid; i < cnt; i += nt) {
    const int a = (int)(i % r), b = (int)(i / r);
    err = nan_max(err, fabs(dsc[a] * G[i] * dsc[b] - (a == b ? 1.0 : 0.0)));
  }
  err = block_max(err, red);
  const bool keep = step == 0 ? !(err <= kOrthPolarMax) : P.flag[e] != 0;   // NaN -> keep
  if (step == 0 && tid == 0 && keep) P.flag[e] = 1;
  for (size_t i = tid; i < cnt; i += nt) {
    const int a = (int)(i % r), b = (int)(i / r);
    G[i] = keep ? (a == b ? 1.0 : 0.0) : dsc[a] * ((a == b ? 1.5 : 0.0) - 0.5 * dsc[a] * G[i] * dsc[b]);
  }
}

// back-transform z = H_0 H_1 ... H_{N-3} y of the leading r eigenvectors with the Householder
// vectors stored in A (column k, rows k+1..): warp per vector, many CTAs (grid.x covers the
// vectors, grid.y the batch entries).  For N <= 32*MC the warp keeps its vector in registers
// (element ln + 32 c in slot c): the only memory traffic is the L2-resident reflectors.
template <int MC>
__global__ void __launch_bounds__(512) backtransform_kernel(const __grid_constant__ SyevBatch B) {
  const SyevEntry& E = B.e[blockIdx.y];
  const int N = E.N;
  const int r = min(*E.r, N);
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), ln = threadIdx.x & 31;
  if (w >= r || E.A == nullptr) return;
  double* yi = E.Y + (size_t)w * E.ldy;
  if (N <= 32 * MC) {
    double yv[MC];
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const int idx = ln + 32 * c;
      yv[c] = idx < N ? yi[idx] : 0.0;
    }
    for (int k = N - 3; k >= 0; --k) {
      const double* u = E.A + (size_t)k * E.lda;   // u_k[idx] at A[idx, k] for idx > k
      const int c0 = (k + 1) >> 5;                 // slots below c0 hold idx <= k: skip them
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < MC; ++c) {
        const int idx = ln + 32 * c;
        if (c >= c0 && idx > k && idx < N) s = fma(u[idx], yv[c], s);
      }
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (s != 0.0) {
        const double t2 = 2.0 * s;
#pragma unroll
        for (int c = 0; c < MC; ++c) {
          const int idx = ln + 32 * c;
          if (c >= c0 && idx > k && idx < N) yv[c] -= t2 * u[idx];
        }
      }
    }
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const int idx = ln + 32 * c;
      if (idx < N) yi[idx] = yv[c];
    }
    return;
  }
  for (int k = N - 3; k >= 0; --k) {
    const double* u = E.A + (k + 1) + (size_t)k * E.lda;
    const int m = N - k - 1;
    double s = 0.0;
    for (int t = ln; t < m; t += 32) s += u[t] * yi[k + 1 + t];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (s != 0.0)
      for (int t = ln; t < m; t += 32) yi[k + 1 + t] -= 2.0 * s * u[t];
    __syncwarp();
  }
}

// Same back-transformation with the reflectors staged through shared memory: the CTA's 16 warps
// (16 vectors) share every reflector, so the whole CTA copies chunks of KB reflector columns
// (N doubles each, 8-byte cp.async) into a double buffer one chunk ahead, and each warp applies
// them from shared memory to its register-resident vector (same arithmetic and order as
// backtransform_kernel: the per-reflector critical path no longer includes an L2 round trip).
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit_bt() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait_bt() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND)); }

template <int MC, int KB>
__global__ void __launch_bounds__(512) backtransform_smem_kernel(const __grid_constant__ SyevBatch B) {
  extern __shared__ double su[];                    // 2 buffers x KB reflectors x (32 MC)
  constexpr int NP = 32 * MC;
  const SyevEntry& E = B.e[blockIdx.y];
  const int N = E.N;
  const int r = min(*E.r, N);
  const int nw = blockDim.x >> 5;
  if ((int)blockIdx.x * nw >= r || E.A == nullptr || N > NP || N < 3) return;   // uniform per CTA
  const int w = blockIdx.x * nw + (threadIdx.x >> 5), ln = threadIdx.x & 31, tid = threadIdx.x;
  const bool active = w < r;
  double* yi = E.Y + (size_t)(active ? w : 0) * E.ldy;
  double yv[MC];
#pragma unroll
  for (int c = 0; c < MC; ++c) {
    const int idx = ln + 32 * c;
    yv[c] = (active && idx < N) ? yi[idx] : 0.0;
  }
  const int nk = N - 2;                              // reflectors k = N-3 .. 0
  const int nchunks = (nk + KB - 1) / KB;
  auto issue = [&](int ci) {
    double* buf = su + (size_t)(ci & 1) * KB * NP;
    const int kb0 = ci * KB, cnt = min(KB, nk - kb0);
    for (int idx = tid; idx < cnt * N; idx += blockDim.x) {
      const int kk = idx / N, i = idx - kk * N;
      const int k = N - 3 - (kb0 + kk);
      cp_async8(buf + kk * NP + i, E.A + (size_t)k * E.lda + i);
    }
    cp_async_commit_bt();
  };
  issue(0);
  for (int ci = 0; ci < nchunks; ++ci) {
    if (ci + 1 < nchunks) {
      issue(ci + 1);
      cp_async_wait_bt<1>();
    } else {
      cp_async_wait_bt<0>();
    }
    __syncthreads();
    if (active) {
      const double* buf = su + (size_t)(ci & 1) * KB * NP;
      const int kb0 = ci * KB, cnt = min(KB, nk - kb0);
      for (int kk = 0; kk < cnt; ++kk) {
        const int k = N - 3 - (kb0 + kk);
        const double* u = buf + kk * NP;             // u_k[idx] for idx > k
        const int c0 = (k + 1) >> 5;
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < MC; ++c) {
          const int idx = ln + 32 * c;
          if (c >= c0 && idx > k && idx < N) s = fma(u[idx], yv[c], s);
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (s != 0.0) {
          const double t2 = 2.0 * s;
#pragma unroll
          for (int c = 0; c < MC; ++c) {
            const int idx = ln + 32 * c;
            if (c >= c0 && idx > k && idx < N) yv[c] -= t2 * u[idx];
          }
        }
      }
    }
    __syncthreads();                                 // buffer (ci & 1) is refilled by issue(ci + 2)
  }
  if (active) {
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const int idx = ln + 32 * c;
      if (idx < N) yi[idx] = yv[c];
    }
  }
}

// Column-pivoted modified Gram-Schmidt (rank revealing, no Gram squaring), one CTA per matrix.
// A (n x p, column-major, overwritten with residuals) -> Q (n x k, orthonormal, k <= p) with
// every column of A within tau * ||a_c|| of span(Q).  Pivot: largest residual norm among the
// columns not yet within their tolerance.  Each accepted vector is re-orthogonalised against Q.
constexpr int kPmgsThreads = 1024;
__global__ void __launch_bounds__(kPmgsThreads) pmgs_kernel(const __grid_constant__ PmgsBatch B) {
  extern __shared__ double sh[];
  const PmgsEntry& E = B.e[blockIdx.x];
  const int n = E.n, p = E.p;
  double* nrm2 = sh;          // current residual norms^2
  double* lim2 = sh + p;      // (tau * original norm)^2
  double* coef = sh + 2 * p;  // projections
  __shared__ int piv_s;
  __shared__ double pnorm_s;
  __shared__ double red[33];
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, ln = tid & 31, nw = nt >> 5;
  double* A = E.A;
  for (int c = warp; c < p; c += nw) {
    double s = 0.0;
    for (int i = ln; i < n; i += 32) s += A[i + (size_t)c * E.lda] * A[i + (size_t)c * E.lda];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (ln == 0) { nrm2[c] = s; lim2[c] = E.tau * E.tau * s; }
  }
  __syncthreads();
  int k = 0;
  for (; k < min(p, n); ++k) {
    if (tid == 0) {
      int best = -1;
      double bv = 0.0;
      for (int c = 0; c < p; ++c)
        if (nrm2[c] > lim2[c] && nrm2[c] > bv) { bv = nrm2[c]; best = c; }
      piv_s = best;
    }
    __syncthreads();
    const int piv = piv_s;
    if (piv < 0) break;
    double* q = E.Q + (size_t)k * E.ldq;
    for (int i = tid; i < n; i += nt) q[i] = A[i + (size_t)piv * E.lda];
    __syncthreads();
    // re-orthogonalise against Q[:, :k] (one CGS pass; the residual already is one MGS pass)
    for (int j = warp; j < k; j += nw) {
      const double* qj = E.Q + (size_t)j * E.ldq;
      double s = 0.0;
      for (int i = ln; i < n; i += 32) s += qj[i] * q[i];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (ln == 0) coef[j] = s;
    }
    __syncthreads();
    double part = 0.0;
    for (int i = tid; i < n; i += nt) {
      double v = q[i];
      for (int j = 0; j < k; ++j) v -= coef[j] * E.Q[i + (size_t)j * E.ldq];
      q[i] = v;
      part += v * v;
    }
    double s2 = block_sum(part, red);
    if (tid == 0) pnorm_s = s2;
    __syncthreads();
    if (pnorm_s <= 0.0) {          // numerically dependent: retire the column
      if (tid == 0) nrm2[piv] = 0.0;
      __syncthreads();
      --k;
      continue;
    }
    const double inv = 1.0 / sqrt(pnorm_s);
    for (int i = tid; i < n; i += nt) q[i] *= inv;
    __syncthreads();
    // project the new direction out of every remaining column (warp per column)
    for (int c = warp; c < p; c += nw) {
      if (nrm2[c] <= lim2[c]) continue;
      double* a = A + (size_t)c * E.lda;
      double s = 0.0;
      for (int i = ln; i < n; i += 32) s += q[i] * a[i];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      double r2 = 0.0;
      for (int i = ln; i < n; i += 32) {
        double v = a[i] - s * q[i];
        a[i] = v;
        r2 += v * v;
      }
      for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
      if (ln == 0) nrm2[c] = r2;
    }
    __syncthreads();
  }
  if (tid == 0) *E.k_out = k;
}

// warp-level dot product of a global vector with a shared-memory vector, 4 independent
// accumulators (keeps 4 loads in flight per lane); result valid in every lane
__device__ __forceinline__ double warp_dot_gs(const double* __restrict__ g, const double* s, int n, int ln) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int i = ln;
  for (; i + 96 < n; i += 128) {
    a0 += g[i] * s[i];
    a1 += g[i + 32] * s[i + 32];
    a2 += g[i + 64] * s[i + 64];
    a3 += g[i + 96] * s[i + 96];
  }
  for (; i < n; i += 32) a0 += g[i] * s[i];
  double v = (a0 + a1) + (a2 + a3);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// In-block step of the blocked rank-revealing Gram-Schmidt (one CTA per matrix): the block's
// columns (already projected against the accepted basis by GEMMs) are orthogonalised among
// themselves in order, two MGS passes against the vectors accepted in this block, with the
// current column staged in shared memory; a column is accepted when its residual exceeds
// tau * max(its norm, the largest column norm) and is written, normalised, to the block buffer
// Y (n x 32).  The BCGS2 second pass (GEMM + bcgs_finalize_kernel) follows.
__global__ void __launch_bounds__(1024) bcgs_block_kernel(const __grid_constant__ BcgsBatch B, int j0, int w) {
  extern __shared__ double xs[];   // n
  __shared__ double coef[64];
  __shared__ double red[33];
  __shared__ int nacc_s, k0_s;
  __shared__ double nmax_s;
  const BcgsEntry& E = B.e[blockIdx.x];
  if (j0 >= E.p) return;
  const int n = E.n, wb = min(w, E.p - j0);
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, ln = tid & 31, nw = nt >> 5;
  if (tid == 0) {
    nacc_s = 0;
    k0_s = *E.k;
    double mx = 0.0;
    if (E.nmax) mx = *E.nmax;
    else
      for (int c = 0; c < E.p; ++c) mx = fmax(mx, E.norm0[c]);
    nmax_s = mx;
  }
  for (int i = tid; i < n * kBcgsW; i += nt) E.Y[i] = 0.0;   // block buffer (n x W, ld n)
  __syncthreads();
  for (int c = 0; c < wb; ++c) {
    const double* xg = E.A + (size_t)(j0 + c) * E.lda;
    for (int i = tid; i < n; i += nt) xs[i] = xg[i];
    __syncthreads();
    const int na = nacc_s;
    for (int pass = 0; pass < 2 && na > 0; ++pass) {
      for (int a = warp; a < na; a += nw) {
        const double s = warp_dot_gs(E.Y + (size_t)a * n, xs, n, ln);
        if (ln == 0) coef[a] = s;
      }
      __syncthreads();
      for (int i = tid; i < n; i += nt) {
        double v0 = xs[i], v1 = 0.0;
        int a = 0;
        for (; a + 1 < na; a += 2) {
          v0 -= coef[a] * E.Y[i + (size_t)a * n];
          v1 -= coef[a + 1] * E.Y[i + (size_t)(a + 1) * n];
        }
        if (a < na) v0 -= coef[a] * E.Y[i + (size_t)a * n];
        xs[i] = v0 + v1;
      }
      __syncthreads();
    }
    double part = 0.0;
    for (int i = tid; i < n; i += nt) part += xs[i] * xs[i];
    const double s2 = block_sum(part, red);
    // kept if the residual exceeds tau times its own norm AND tau times the largest column
    // (columns below tau * max are negligible; their residuals are rounding residue, and
    // normalising them would inject garbage directions)
    const double lim = E.tau * fmax(E.norm0[j0 + c], nmax_s);
    if (s2 > lim * lim && k0_s + na < E.kcap) {
      const double inv = 1.0 / sqrt(s2);
      double* q = E.Y + (size_t)na * n;
      for (int i = tid; i < n; i += nt) q[i] = xs[i] * inv;
      if (tid == 0) nacc_s = na + 1;
    }
    __syncthreads();
  }
  if (tid == 0) *E.nacc = nacc_s;
}

// BCGS2 second pass, in-block part: the accepted unit vectors Y[:, :nacc] (already re-projected
// against Q by a GEMM) are re-orthonormalised among themselves (MGS) and appended to Q at k.
__global__ void __launch_bounds__(1024) bcgs_finalize_kernel(const __grid_constant__ BcgsBatch B, int j0) {
  extern __shared__ double ys[];   // n
  __shared__ double coef[64];
  __shared__ double red[33];
  const BcgsEntry& E = B.e[blockIdx.x];
  if (j0 >= E.p) return;
  const int n = E.n, na = *E.nacc, k0 = *E.k;
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, ln = tid & 31, nw = nt >> 5;
  for (int c = 0; c < na; ++c) {
    double* y = E.Y + (size_t)c * n;
    for (int i = tid; i < n; i += nt) ys[i] = y[i];
    __syncthreads();
    for (int a = warp; a < c; a += nw) {
      const double s = warp_dot_gs(E.Y + (size_t)a * n, ys, n, ln);
      if (ln == 0) coef[a] = s;
    }
    __syncthreads();
    double part = 0.0;
    for (int i = tid; i < n; i += nt) {
      double v = ys[i];
      for (int a = 0; a < c; ++a) v -= coef[a] * E.Y[i + (size_t)a * n];
      ys[i] = v;
      part += v * v;
    }
    const double s2 = block_sum(part, red);
    const double inv = s2 > 0 ? 1.0 / sqrt(s2) : 0.0;
    double* q = E.Q + (size_t)(k0 + c) * E.ldq;
    for (int i = tid; i < n; i += nt) {
      const double v = ys[i] * inv;
      y[i] = v;
      q[i] = v;
    }
    __syncthreads();
  }
  if (tid == 0) *E.k = k0 + na;
}

// ---- cluster versions of the two in-block steps --------------------------------------------
// CTA r of a CS-CTA cluster owns rows [r RB, (r+1) RB) of the n x W block (RB = n / CS <= 128)
// and keeps them in shared memory: the block X and the accepted unit vectors Yb (leading
// dimension RB + 4: conflict-free row-parallel access).  Every dot product, norm and Gram entry
// is a partial over the CTA's rows, all-reduced through DSMEM in a fixed order (the same value in
// every CTA, so every accept decision agrees).
//   in-block step (default): the block Gram G = X^T X in one cluster reduction; a replicated
//   in-order Cholesky of G accepts the columns that are clearly independent of the earlier
//   accepted ones (Schur residual s_c > max(theta^2 G_cc, 1.01 lim^2), theta = 1e-4: s_c is
//   accurate to ~m eps G_cc, i.e. to 1e-6 relative at the theta level, so the decision is safe),
//   rejects those with theta^2 G_cc < s_c < 0.99 lim^2 (below lim against a subset of the final
//   basis already) and defers the rest; the accepted columns are orthonormalised by CholQR (Y = X L^-T) followed
//   by the polar step (= CholQR2; a block whose CholQR orthogonality loss exceeds 1e-4 is redone
//   on the per-column path; below it the span error eps kappa ~ 1e-10 is far under the
//   truncation tolerances); the deferred
//   columns (about 10 % of those alive in the C4 solve) go through the exact per-column path:
//   pass 1 (dots, all-reduce, update), pass 2 fused with the norm (dots and ||x'||^2 in one
//   all-reduce, ||x''||^2 = ||x'||^2 - ||c2||^2: c2 = O(eps ||x||) after pass 1, far below the
//   tau ||x|| decision level) -> 2 cluster barriers per deferred column.  FC_BCGS_SEQ: every
//   alive column through the per-column path (the previous design).
//   finalisation: polar step on the re-projected block (one Gram all-reduce).
constexpr int kBcgsClusterThreads = 512;
constexpr double kBcgsTheta2 = 1e-8;    // theta^2: clear-acceptance level of the Gram Cholesky
constexpr double kBcgsCholFail = 1e-4;  // orthogonality loss above which bcgs_polar takes a Cholesky step

// cluster configurations: (CS CTAs, block width W, rows per CTA RB), n <= CS * RB; see bcgs()
template <int W, int RB>
struct BcgsClusterSmem {
  static constexpr int LD = RB + 1;   // odd: conflict-free both row-parallel and column-parallel
  double X[LD * W];
  double Yb[LD * W];
  double gram[2 * W * W];         // Gram partials (read remotely) / Cholesky factor / H; reduced Gram
  double part[2][W + 2];          // partial dots (+ norm), double-buffered (read remotely)
  double coef[W + 2];
  double red[kBcgsClusterThreads / 32];
  double pn2[W];                  // squared column norms after the GEMM projection
  double lim2[W];                 // (tau max(norm0_c, nmax))^2, the acceptance level of column c
  int alive[W];
  int cidx[W], uidx[W];           // Cholesky-accepted / deferred columns
};

// diagnostics (FC_TRACE): in-block residual ratios ||x''|| / ||x_proj|| of the columns that pass
// the pre-filter, by decade (bin d: ratio in [10^-(d+1), 10^-d)), [18] pre-filtered, [19] blocks,
// [20] deferred by the Gram Cholesky, [22] rejected by it, [21] blocks redone on the per-column
// path
__device__ unsigned long long g_bcgs_hist[23];
// FC_TRACE: cycles of the in-block Gram path stages (cluster rank 0): Gram + Cholesky, CholQR,
// polar step, deferred columns
__device__ unsigned long long g_bcgs_cyc[10];
__device__ int g_bcgs_timing = 0;

// all-reduce of buf[0..cnt) (per-CTA partials, read remotely) into out[0..cnt); every CTA sums
// the CS partials in rank order (shuffle tree over groups of CS lanes)
template <int CS>
__device__ __forceinline__ void cluster_allreduce(cooperative_groups::cluster_group& cl, double* buf, int cnt,
                                                  double* out) {
  const int tid = threadIdx.x;
  for (int base = 0; base < cnt * CS; base += blockDim.x) {
    const int idx = base + tid;
    const int a = idx / CS, src = idx % CS;
    double v = (a < cnt) ? cl.map_shared_rank(buf, src)[a] : 0.0;
#pragma unroll
    for (int o = CS / 2; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o, CS);
    if (src == 0 && a < cnt) out[a] = v;
  }
}

// partial dots part[a] = sum_{i < nr} V[i, a] x[i] for a < na (4 independent dots per warp)
// and, if want_norm, part[na] = sum x[i]^2
template <int LD>
__device__ __forceinline__ void block_dots(const double* V, const double* x, int nr, int na, bool want_norm,
                                           double* part, double* red) {
  const int tid = threadIdx.x, warp = tid >> 5, ln = tid & 31, NW = blockDim.x >> 5;
  for (int a0 = warp * 4; a0 < na; a0 += NW * 4) {
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int i = ln; i < nr; i += 32) {
      const double xi = x[i];
      s0 = fma(V[i + (size_t)a0 * LD], xi, s0);
      if (a0 + 1 < na) s1 = fma(V[i + (size_t)(a0 + 1) * LD], xi, s1);
      if (a0 + 2 < na) s2 = fma(V[i + (size_t)(a0 + 2) * LD], xi, s2);
      if (a0 + 3 < na) s3 = fma(V[i + (size_t)(a0 + 3) * LD], xi, s3);
    }
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      s3 += __shfl_xor_sync(0xffffffffu, s3, o);
    }
    if (ln == 0) {
      part[a0] = s0;
      if (a0 + 1 < na) part[a0 + 1] = s1;
      if (a0 + 2 < na) part[a0 + 2] = s2;
      if (a0 + 3 < na) part[a0 + 3] = s3;
    }
  }
  if (want_norm) {
    double q = 0.0;
    for (int i = tid; i < nr; i += blockDim.x) q = fma(x[i], x[i], q);
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if (ln == 0) red[warp] = q;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < NW; ++w) t += red[w];
      part[na] = t;
    }
  }
}

// x[i] -= sum_{a < na} coef[a] V[i, a]: 2 threads per row — lanes 0-15 and 16-31 of a warp take
// the same 16 consecutive rows, the even / odd columns, combined by one shuffle (with the odd
// leading dimension every bank is hit exactly twice per load: conflict-free)
template <int LD, int RB>
__device__ __forceinline__ void block_update(const double* V, double* x, int nr, int na, const double* coef) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int base = 0; base < RB * 2; base += nt) {
    const int idx = base + tid, ln = idx & 31;
    const int i = (idx >> 5) * 16 + (ln & 15), half = ln >> 4;
    double v = 0.0;
    if (i < nr)
      for (int a = half; a < na; a += 2) v = fma(coef[a], V[i + (size_t)a * LD], v);
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    if (half == 0 && i < nr) x[i] -= v;
  }
}

// G = M^T M for the m columns of M (this CTA's rows [0, RB), ld LD) over the whole cluster:
// 4 x 4 upper tiles per warp with lanes over rows (conflict-free) into the partials S.gram[0..m^2),
// reduce-scatter in rank order into S.gram[W^2 + .], all-gather of the other CTAs' chunks: on
// return every CTA holds the identical G (ld m) at S.gram + W^2.  The partials may be reused
// after return; the reduced copy is read remotely until the next cluster barrier.
template <int CS, int W, int RBM>
__device__ void cluster_gram(cooperative_groups::cluster_group& cl, BcgsClusterSmem<W, RBM>& S, const double* M,
                             int m, int RB) {
  constexpr int LD = BcgsClusterSmem<W, RBM>::LD;
  double* P = S.gram;
  double* R = S.gram + W * W;
  const int tid = threadIdx.x, warp = tid >> 5, ln = tid & 31, NW = blockDim.x >> 5, nt = blockDim.x;
  const int cnt = m * m, ch = (cnt + CS - 1) / CS, r = (int)cl.block_rank(), nt4 = (m + 3) / 4;
  const bool tm = g_bcgs_timing && r == 0 && tid == 0;
  long long t0 = tm ? clock64() : 0;
  // 4 x 4 register tiles over strided column groups {t, t+h, t+2h, t+3h} (h = ceil(m/4)): a tile
  // per thread pair (even / odd rows, combined by one shuffle), consecutive pairs on consecutive
  // a-groups (odd LD: distinct banks), the b-group values are broadcasts; half the shared-memory
  // loads per FMA of a thread-per-entry layout, no reduction trees
  const int h4 = (m + 3) / 4, ntile = h4 * h4;
  // warp-uniform loop (the pair shuffle below needs every lane of the warp): lanes past the end
  // run with empty tiles
  for (int ub = tid - ln; ub < 2 * ntile; ub += nt) {
    const int u = ub + ln;
    const bool valid = u < 2 * ntile;
    const int tile = valid ? u >> 1 : 0, part = u & 1;
    const int ta = tile % h4, tb = tile / h4;
    const double* ya[4];
    const double* yb[4];
    bool va[4], vb[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int a = ta + q * h4, b = tb + q * h4;
      va[q] = a < m;
      vb[q] = b < m;
      ya[q] = M + (size_t)(va[q] ? a : 0) * LD;
      yb[q] = M + (size_t)(vb[q] ? b : 0) * LD;
    }
    double acc[4][4] = {};
    for (int i = part; valid && i < RB; i += 2) {
      double xa[4], xb[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        xa[q] = ya[q][i];
        xb[q] = yb[q][i];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(xa[p], xb[q], acc[p][q]);
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double v = acc[p][q] + __shfl_xor_sync(0xffffffffu, acc[p][q], 1);
        if (valid && part == 0 && va[p] && vb[q]) P[(ta + p * h4) * m + (tb + q * h4)] = v;
      }
  }
  long long t1 = tm ? clock64() : 0;
  cl.sync();
  long long t2 = tm ? clock64() : 0;
  // reduce own chunk: the CS remote partials are loaded into registers first (independent DSMEM
  // loads in flight together), then summed in rank order
  for (int e = r * ch + tid; e < min(cnt, (r + 1) * ch); e += nt) {
    double pv[CS];
#pragma unroll
    for (int s = 0; s < CS; ++s) pv[s] = cl.map_shared_rank(P, s)[e];
    double v = 0.0;
#pragma unroll
    for (int s = 0; s < CS; ++s) v += pv[s];
    R[e] = v;
  }
  long long t3 = tm ? clock64() : 0;
  cl.sync();
  long long t4 = tm ? clock64() : 0;
  // gather the other chunks: all of this thread's remote loads issued before any local store
  constexpr int kGatherMax = (W * W + kBcgsClusterThreads - 1) / kBcgsClusterThreads;
  double gv[kGatherMax];
#pragma unroll
  for (int it = 0; it < kGatherMax; ++it) {
    const int e = tid + it * nt;
    const int own = e / ch;
    gv[it] = (e < cnt && own != r) ? cl.map_shared_rank(R, own)[e] : 0.0;
  }
#pragma unroll
  for (int it = 0; it < kGatherMax; ++it) {
    const int e = tid + it * nt;
    if (e < cnt && e / ch != r) R[e] = gv[it];
  }
  __syncthreads();
  if (tm) {
    const long long t5 = clock64();
    atomicAdd(&g_bcgs_cyc[5], (unsigned long long)(t1 - t0));
    atomicAdd(&g_bcgs_cyc[6], (unsigned long long)(t2 - t1));
    atomicAdd(&g_bcgs_cyc[7], (unsigned long long)(t3 - t2));
    atomicAdd(&g_bcgs_cyc[8], (unsigned long long)(t4 - t3));
    atomicAdd(&g_bcgs_cyc[9], (unsigned long long)(t5 - t4));
  }
}

// Polar (Newton-Schulz) re-orthonormalisation of the na block vectors held row-distributed in
// S.Yb (rows [0, RB) of this CTA): G = Yb^T Yb (cluster_gram), D = diag(G)^-1/2 and
// Yb <- Yb D (3I - D G D) / 2.  The error e = max|D G D - I| squares per step (0.75 e^2): one
// step when e < 1e-8 (the usual case), more otherwise.  When e > kBcgsCholFail (a CholQR input
// with kappa > ~1e6) the step is a Cholesky one instead, Yb <- Yb L^-T with G = L L^T (CholQR2:
// valid up to kappa ~ 1e8), computed redundantly in every CTA from the identical G; returns
// false (Yb unusable, caller redoes the block) if that Cholesky breaks down or does not bring e
// down.  Replaces na sequential MGS steps (one cluster barrier each) by one Gram all-reduce; the
// order of the vectors inside the block is irrelevant to the basis (coefficients are formed as
// Q^T K afterwards).
template <int CS, int W, int RBM>
__device__ bool bcgs_polar(cooperative_groups::cluster_group& cl, BcgsClusterSmem<W, RBM>& S, int na, int RB) {
  constexpr int LD = BcgsClusterSmem<W, RBM>::LD;
  constexpr int G = kBcgsClusterThreads / RBM, CPG = W / G;   // apply: column groups x columns
  static_assert(kBcgsClusterThreads % RBM == 0 && W % G == 0, "polar layout");
  double* H = S.gram;
  const double* R = S.gram + W * W;
  const int tid = threadIdx.x, warp = tid >> 5, ln = tid & 31, NW = blockDim.x >> 5, nt = blockDim.x;
  const int cnt = na * na;
  int chol = 0;
  for (int it = 0; it < 6; ++it) {
    if (it > 0) cl.sync();            // everyone has gathered the previous reduced Gram
    cluster_gram<CS, W, RBM>(cl, S, S.Yb, na, RB);
    for (int a = tid; a < na; a += nt) {
      const double g = R[a * na + a];
      S.coef[a] = g > 0.0 ? 1.0 / sqrt(g) : 0.0;
    }
    __syncthreads();
    double err = 0.0;
    for (int e = tid; e < cnt; e += nt) {
      const int a = e / na, b = e % na;
      const double gt = S.coef[a] * R[e] * S.coef[b];
      err = fmax(err, fabs(gt - (a == b ? 1.0 : 0.0)));
      H[e] = S.coef[a] * ((a == b ? 1.5 : 0.0) - 0.5 * gt);         // H = D (3I - DGD) / 2
    }
    for (int o = 16; o > 0; o >>= 1) err = fmax(err, __shfl_xor_sync(0xffffffffu, err, o));
    if (ln == 0) S.red[warp] = err;
    __syncthreads();
    err = 0.0;
    for (int w = 0; w < NW; ++w) err = fmax(err, S.red[w]);         // uniform: same G everywhere
    if (it > 0 && err < 1e-13) break;
    if (err > kBcgsCholFail) {
      if (chol == 2) {
        cl.sync();
        return false;
      }
      ++chol;
      // Cholesky step: H <- L with G = L L^T (in-order, replicated), Yb <- Yb L^-T
      __syncthreads();
      for (int e = tid; e < cnt; e += nt) H[e] = R[e];
      __syncthreads();
      bool ok = true;
      for (int c = 0; c < na; ++c) {
        const double piv = H[c + c * na];
        if (!(piv > 1e-14 * R[c * na + c])) {
          ok = false;
          break;
        }
        const double d = sqrt(piv), inv = 1.0 / d;
        for (int j = c + 1 + tid; j < na; j += nt) H[j + c * na] *= inv;
        __syncthreads();
        const int t = na - c - 1;
        for (int idx = tid; idx < t * t; idx += nt) {
          const int j = c + 1 + idx % t, k = c + 1 + idx / t;
          H[j + k * na] -= H[j + c * na] * H[k + c * na];
        }
        if (tid == 0) H[c + c * na] = d;
        __syncthreads();
      }
      if (!ok) {
        cl.sync();
        return false;
      }
      for (int i = tid; i < RB; i += nt)
        for (int m = 0; m < na; ++m) {
          double v = S.Yb[i + (size_t)m * LD];
          for (int q = 0; q < m; ++q) v = fma(-S.Yb[i + (size_t)q * LD], H[m + q * na], v);
          S.Yb[i + (size_t)m * LD] = v / H[m + m * na];
        }
      __syncthreads();
      continue;
    }
    // Yb <- Yb H: thread = (row i, group of CPG columns); H reads are warp broadcasts
    const int i = tid % RBM, b0 = (tid / RBM) * CPG;
    double acc[CPG];
#pragma unroll
    for (int q = 0; q < CPG; ++q) acc[q] = 0.0;
    if (i < RB && b0 < na)
      for (int a = 0; a < na; ++a) {
        const double y = S.Yb[i + (size_t)a * LD];
        const double* h = H + a * na + b0;
#pragma unroll
        for (int q = 0; q < CPG; ++q)
          if (b0 + q < na) acc[q] = fma(y, h[q], acc[q]);
      }
    __syncthreads();
    if (i < RB)
#pragma unroll
      for (int q = 0; q < CPG; ++q)
        if (b0 + q < na) S.Yb[i + (size_t)(b0 + q) * LD] = acc[q];
    __syncthreads();
    if (err < 1e-8) break;
  }
  cl.sync();                                                            // others may still gather R
  return true;
}

// exact per-column step for block column c against the na accepted in-block vectors: two
// projection passes (the second fused with the norm), accept test, append.  Returns the new na.
template <int CS, int W, int RBM>
__device__ int bcgs_column(cooperative_groups::cluster_group& cl, BcgsClusterSmem<W, RBM>& S, const BcgsEntry& E,
                           const BcgsBatch& B, int c, int na, int& ph, int j0, int k0, double nmax, int nr, int RB,
                           int r) {
  constexpr int LD = BcgsClusterSmem<W, RBM>::LD;
  const int tid = threadIdx.x, nt = blockDim.x;
  double* x = S.X + (size_t)c * LD;
  double s2;
  if (na == 0) {
    block_dots<LD>(S.Yb, x, nr, 0, true, S.part[ph], S.red);
    cl.sync();
    cluster_allreduce<CS>(cl, S.part[ph], 1, S.coef);
    __syncthreads();
    s2 = S.coef[0];
    ph ^= 1;
  } else {
    block_dots<LD>(S.Yb, x, nr, na, false, S.part[ph], S.red);
    cl.sync();
    cluster_allreduce<CS>(cl, S.part[ph], na, S.coef);
    __syncthreads();
    block_update<LD, RBM>(S.Yb, x, nr, na, S.coef);
    __syncthreads();
    ph ^= 1;
    block_dots<LD>(S.Yb, x, nr, na, true, S.part[ph], S.red);
    cl.sync();
    cluster_allreduce<CS>(cl, S.part[ph], na + 1, S.coef);
    __syncthreads();
    block_update<LD, RBM>(S.Yb, x, nr, na, S.coef);
    double c2 = 0.0;
    for (int a = 0; a < na; ++a) c2 = fma(S.coef[a], S.coef[a], c2);
    s2 = S.coef[na] - c2;
    __syncthreads();
    ph ^= 1;
  }
  const double lim = E.tau * fmax(E.norm0[j0 + c], nmax);
  if (B.trace && r == 0 && tid == 0) {
    const double ratio = s2 > 0.0 ? sqrt(s2 / S.pn2[c]) : 0.0;
    const int d = ratio > 0.0 ? min(17, max(0, (int)floor(-log10(ratio)))) : 17;
    atomicAdd(&g_bcgs_hist[d], 1ull);
  }
  if (s2 > lim * lim && k0 + na < E.kcap) {
    const double inv = 1.0 / sqrt(s2);
    double* y = S.Yb + (size_t)na * LD;
    for (int i = tid; i < RB; i += nt) y[i] = i < nr ? x[i] * inv : 0.0;
    ++na;
  }
  __syncthreads();
  return na;
}

template <int CS, int W, int RBM>
__global__ void __launch_bounds__(kBcgsClusterThreads, 1)
    bcgs_block_cluster_kernel(const __grid_constant__ BcgsBatch B, int j0, int w, int seq) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char smraw[];
  using Smem = BcgsClusterSmem<W, RBM>;
  constexpr int LD = Smem::LD;
  Smem& S = *reinterpret_cast<Smem*>(smraw);
  cg::cluster_group cl = cg::this_cluster();
  const BcgsEntry& E = B.e[blockIdx.y];
  if (j0 >= E.p) return;                                   // uniform over the cluster
  const int n = E.n, wb = min(w, E.p - j0);
  const int r = (int)cl.block_rank(), RB = (n + CS - 1) / CS;
  const int r0 = r * RB, nr = max(0, min(n, r0 + RB) - r0);
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, ln = tid & 31, NW = nt >> 5;
  for (int idx = tid; idx < RB * wb; idx += nt) {
    const int i = idx % RB, c = idx / RB;
    S.X[i + (size_t)c * LD] = i < nr ? E.A[(size_t)(r0 + i) + (size_t)(j0 + c) * E.lda] : 0.0;
  }
  double mx = 0.0;
  if (E.nmax) mx = *E.nmax;
  else
    for (int c = tid; c < E.p; c += nt) mx = fmax(mx, E.norm0[c]);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __syncthreads();
  if (ln == 0) S.red[warp] = mx;
  __syncthreads();
  double nmax = 0.0;
  for (int i = 0; i < NW; ++i) nmax = fmax(nmax, S.red[i]);
  const int k0 = *E.k;
  __syncthreads();
  int na = 0, ph = 1;                                      // ph: partial buffer of the next phase
  if (seq) {
    // ---- per-column path: pre-filter (all block column norms in one all-reduce), then every
    // alive column through bcgs_column ----
    for (int c = warp; c < wb; c += NW) {
      const double* x = S.X + (size_t)c * LD;
      double q = 0.0;
      for (int i = ln; i < nr; i += 32) q = fma(x[i], x[i], q);
      for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
      if (ln == 0) S.part[0][c] = q;
    }
    cl.sync();
    cluster_allreduce<CS>(cl, S.part[0], wb, S.coef);
    __syncthreads();
    for (int c = tid; c < wb; c += nt) {
      const double lim = E.tau * fmax(E.norm0[j0 + c], nmax);
      S.alive[c] = S.coef[c] > lim * lim;
      S.pn2[c] = S.coef[c];
      if (B.trace && r == 0 && !S.alive[c]) atomicAdd(&g_bcgs_hist[18], 1ull);
    }
    if (B.trace && r == 0 && tid == 0) atomicAdd(&g_bcgs_hist[19], 1ull);
    __syncthreads();
    for (int c = 0; c < wb; ++c)
      if (S.alive[c]) na = bcgs_column<CS, W, RBM>(cl, S, E, B, c, na, ph, j0, k0, nmax, nr, RB, r);
  } else {
    // ---- Gram path ----
    long long tc0 = B.trace ? clock64() : 0;
    cluster_gram<CS, W, RBM>(cl, S, S.X, wb, RB);
    if (B.trace && r == 0 && tid == 0) atomicAdd(&g_bcgs_cyc[4], (unsigned long long)(clock64() - tc0));
    double* L = S.gram;                                    // Cholesky in place of the partials
    const double* G = S.gram + W * W;
    for (int e = tid; e < wb * wb; e += nt) L[e] = G[e];
    for (int c = tid; c < wb; c += nt) {
      const double lim = E.tau * fmax(E.norm0[j0 + c], nmax);
      S.pn2[c] = G[c * wb + c];
      S.lim2[c] = lim * lim;
      S.alive[c] = S.pn2[c] > lim * lim;
      if (B.trace && r == 0 && !S.alive[c]) atomicAdd(&g_bcgs_hist[18], 1ull);
    }
    if (B.trace && r == 0 && tid == 0) atomicAdd(&g_bcgs_hist[19], 1ull);
    __syncthreads();
    // replicated in-order Cholesky with deferral (identical arithmetic in every CTA)
    int nC = 0, nU = 0;
    const int cap = E.kcap - k0;
    for (int c = 0; c < wb; ++c) {
      if (!S.alive[c]) continue;
      const double piv = L[c + c * wb];
      const double lim2 = S.lim2[c];
      if (nC < cap && piv > fmax(kBcgsTheta2 * S.pn2[c], 1.01 * lim2)) {
        // right-looking step on the lower triangle with the raw pivot column (l_jc l_kc =
        // a_jc a_kc / piv): a warp per trailing column k, lanes over rows j >= k; the pivot
        // column itself is scaled after the loop (one barrier per accepted column)
        const double ipiv = 1.0 / piv;
        for (int k = c + 1 + warp; k < wb; k += NW) {
          const double akc = L[k + c * wb] * ipiv;
          for (int j = k + ln; j < wb; j += 32) L[j + k * wb] -= L[j + c * wb] * akc;
        }
        if (tid == 0) S.cidx[nC] = c;
        if (B.trace && r == 0 && tid == 0) {
          const int dd = min(17, max(0, (int)floor(-0.5 * log10(piv / S.pn2[c]))));
          atomicAdd(&g_bcgs_hist[dd], 1ull);
        }
        ++nC;
        __syncthreads();
      } else if (piv > kBcgsTheta2 * S.pn2[c] && piv < 0.99 * lim2) {
        // residual against the accepted subset already below lim (accurate to ~1e-6 here): the
        // per-column path, projecting against a superset, would reject it too
        if (B.trace && r == 0 && tid == 0) atomicAdd(&g_bcgs_hist[22], 1ull);
      } else if (nC < cap || piv <= kBcgsTheta2 * S.pn2[c]) {
        if (tid == 0) S.uidx[nU] = c;
        ++nU;
      }
    }
    __syncthreads();
    // finish the factor: L[c, c] = sqrt(piv_c), L[j, c] = a_jc / sqrt(piv_c) for the accepted c
    for (int m = warp; m < nC; m += NW) {
      const int c = S.cidx[m];
      const double d = sqrt(L[c + c * wb]), inv = 1.0 / d;
      for (int j = c + 1 + ln; j < wb; j += 32) L[j + c * wb] *= inv;
      if (ln == 0) L[c + c * wb] = d;
    }
    __syncthreads();
    if (B.trace && r == 0 && tid == 0) atomicAdd(&g_bcgs_hist[20], (unsigned long long)nU);
    long long tc1 = B.trace ? clock64() : 0;
    // CholQR: Yb[:, m] = (X[:, c_m] - sum_{q < m} Yb[:, q] L[c_m, c_q]) / L[c_m, c_m]
    for (int i = tid; i < RB; i += nt) {
      for (int m = 0; m < nC; ++m) {
        const int c = S.cidx[m];
        double v = S.X[i + (size_t)c * LD];
        for (int q = 0; q < m; ++q) v = fma(-S.Yb[i + (size_t)q * LD], L[c + S.cidx[q] * wb], v);
        S.Yb[i + (size_t)m * LD] = v / L[c + c * wb];
      }
    }
    __syncthreads();
    cl.sync();                                             // all gathers of G done before reuse
    // CholQR loses orthogonality like eps kappa(X_C)^2; the polar routine repairs it with a second
    // Cholesky step up to kappa ~ 1e8, beyond that the block is redone on the per-column path
    long long tc2 = B.trace ? clock64() : 0;
    if (bcgs_polar<CS, W, RBM>(cl, S, nC, RB)) {
      long long tc3 = B.trace ? clock64() : 0;
      na = nC;
      for (int u = 0; u < nU; ++u)
        na = bcgs_column<CS, W, RBM>(cl, S, E, B, S.uidx[u], na, ph, j0, k0, nmax, nr, RB, r);
      if (B.trace && r == 0 && tid == 0) {
        const long long tc4 = clock64();
        atomicAdd(&g_bcgs_cyc[0], (unsigned long long)(tc1 - tc0));
        atomicAdd(&g_bcgs_cyc[1], (unsigned long long)(tc2 - tc1));
        atomicAdd(&g_bcgs_cyc[2], (unsigned long long)(tc3 - tc2));
        atomicAdd(&g_bcgs_cyc[3], (unsigned long long)(tc4 - tc3));
      }
    } else {
      if (B.trace && r == 0 && tid == 0) atomicAdd(&g_bcgs_hist[21], 1ull);
      for (int c = 0; c < wb; ++c)
        if (S.alive[c]) na = bcgs_column<CS, W, RBM>(cl, S, E, B, c, na, ph, j0, k0, nmax, nr, RB, r);
    }
  }
  for (int idx = tid; idx < nr * W; idx += nt) {           // unused block columns stay 0
    const int i = idx % nr, a = idx / nr;
    E.Y[(size_t)(r0 + i) + (size_t)a * n] = a < na ? S.Yb[i + (size_t)a * LD] : 0.0;
  }
  if (r == 0 && tid == 0) *E.nacc = na;
  {   // zero the projection scratch P for this block's BCGS2 pass (replaces a host memset)
    const int kup = min(E.k_base + j0, E.kcap);
    for (long long idx = (long long)r * nt + tid; idx < (long long)kup * W; idx += (long long)CS * nt) E.P[idx] = 0.0;
  }
  cl.sync();                                                 // smem stays alive for readers
}

// BCGS2 second pass, in-block part, on the cluster: Y[:, :nacc] (re-projected against Q) are
// re-orthonormalised among themselves and appended to Q at k: polar step (default), or one MGS
// pass with dots and norm in one all-reduce (FC_BCGS_MGS_FINAL).
template <int CS, int W, int RBM>
__global__ void __launch_bounds__(kBcgsClusterThreads, 1)
    bcgs_finalize_cluster_kernel(const __grid_constant__ BcgsBatch B, int j0, int w, int mgs) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char smraw[];
  using Smem = BcgsClusterSmem<W, RBM>;
  constexpr int LD = Smem::LD;
  Smem& S = *reinterpret_cast<Smem*>(smraw);
  cg::cluster_group cl = cg::this_cluster();
  const BcgsEntry& E = B.e[blockIdx.y];
  if (j0 >= E.p) return;
  const int n = E.n, na = *E.nacc, k0 = *E.k;
  const int r = (int)cl.block_rank(), RB = (n + CS - 1) / CS;
  const int r0 = r * RB, nr = max(0, min(n, r0 + RB) - r0);
  const int tid = threadIdx.x, nt = blockDim.x;
  (void)w;
  for (int idx = tid; idx < RB * na; idx += nt) {
    const int i = idx % RB, c = idx / RB;
    S.Yb[i + (size_t)c * LD] = i < nr ? E.Y[(size_t)(r0 + i) + (size_t)c * n] : 0.0;
  }
  __syncthreads();
  if (!mgs) {
    bcgs_polar<CS, W, RBM>(cl, S, na, RB);
    for (int idx = tid; idx < nr * na; idx += nt) {
      const int i = idx % nr, c = idx / nr;
      const double v = S.Yb[i + (size_t)c * LD];
      E.Y[(size_t)(r0 + i) + (size_t)c * n] = v;
      E.Q[(size_t)(r0 + i) + (size_t)(k0 + c) * E.ldq] = v;
    }
    if (r == 0 && tid == 0) *E.k = k0 + na;
    {   // zero the projection scratch P for the next block's first pass (replaces a host memset)
      const int kup = min(E.k_base + j0 + W, E.kcap);
      for (long long idx = (long long)r * nt + tid; idx < (long long)kup * W; idx += (long long)CS * nt) E.P[idx] = 0.0;
    }
    return;
  }
  for (int c = 0; c < na; ++c) {
    double* y = S.Yb + (size_t)c * LD;
    double* part = S.part[c & 1];
    block_dots<LD>(S.Yb, y, nr, c, true, part, S.red);
    cl.sync();
    cluster_allreduce<CS>(cl, part, c + 1, S.coef);
    __syncthreads();
    if (c > 0) block_update<LD, RBM>(S.Yb, y, nr, c, S.coef);
    double c2 = 0.0;
    for (int a = 0; a < c; ++a) c2 = fma(S.coef[a], S.coef[a], c2);
    const double s2 = S.coef[c] - c2;
    __syncthreads();
    const double inv = s2 > 0 ? 1.0 / sqrt(s2) : 0.0;
    for (int i = tid; i < nr; i += nt) {
      const double v = y[i] * inv;
      y[i] = v;
      E.Y[(size_t)(r0 + i) + (size_t)c * n] = v;
      E.Q[(size_t)(r0 + i) + (size_t)(k0 + c) * E.ldq] = v;
    }
    __syncthreads();
  }
  cl.sync();
  if (r == 0 && tid == 0) *E.k = k0 + na;
  {
    const int kup = min(E.k_base + j0 + W, E.kcap);
    for (long long idx = (long long)r * nt + tid; idx < (long long)kup * W; idx += (long long)CS * nt) E.P[idx] = 0.0;
  }
}

__global__ void set_int_kernel(int* p, int v) { *p = v; }

// largest original column norm of every entry (fixed for the whole Gram-Schmidt: the acceptance
// level tau max(norm0_c, nmax) must not change when columns are pruned)
__global__ void bcgs_nmax_kernel(const __grid_constant__ BcgsBatch B) {
  const BcgsEntry& E = B.e[blockIdx.x];
  double mx = 0.0;
  for (int c = threadIdx.x; c < E.p; c += blockDim.x) mx = fmax(mx, E.norm0[c]);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) mx = fmax(mx, red[i]);
    *E.nmax = mx;
  }
}

// bulk pruning (bcgs): the columns [j0, p) of every entry were just projected against the accepted
// basis; a column whose residual is within its acceptance level tau max(norm0_c, nmax) would be
// rejected when its block is reached (the basis only grows) -> flag 0
struct PruneArgs {
  int j0[kMaxSyev];
  int* flag[kMaxSyev];
  int* idx[kMaxSyev];
  int* cnt;
  double* tmpA[kMaxSyev];
  double* tmpN[kMaxSyev];
};
__global__ void bcgs_prune_flag_kernel(const __grid_constant__ BcgsBatch B, const __grid_constant__ PruneArgs P) {
  const BcgsEntry& E = B.e[blockIdx.y];
  const int c = P.j0[blockIdx.y] + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), ln = threadIdx.x & 31;
  if (c >= E.p) return;
  const double* a = E.A + (size_t)c * E.lda;
  double s = 0.0;
  for (int i = ln; i < E.n; i += 32) s = fma(a[i], a[i], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (ln == 0) {
    const double lim = E.tau * fmax(E.norm0[c], *E.nmax);
    P.flag[blockIdx.y][c - P.j0[blockIdx.y]] = s > lim * lim ? 1 : 0;
  }
}
// ordered compaction of the surviving columns (one CTA per entry)
__global__ void __launch_bounds__(1024) bcgs_prune_compact_kernel(const __grid_constant__ BcgsBatch B,
                                                                  const __grid_constant__ PruneArgs P) {
  const int e = blockIdx.x;
  const BcgsEntry& E = B.e[e];
  const int m = max(0, E.p - P.j0[e]);
  __shared__ int wsum[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int ln = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c0 = 0; c0 < m; c0 += blockDim.x) {
    const int c = c0 + threadIdx.x;
    const int f = c < m ? P.flag[e][c] : 0;
    const unsigned msk = __ballot_sync(0xffffffffu, f);
    if (ln == 0) wsum[w] = __popc(msk);
    __syncthreads();
    int off = base;
    for (int i = 0; i < w; ++i) off += wsum[i];
    if (f) P.idx[e][off + __popc(msk & ((1u << ln) - 1u))] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += wsum[i];
      base += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) P.cnt[e] = base;
}
// survivors gathered in order into the scratch copies (columns and their original norms)
__global__ void bcgs_prune_gather_kernel(const __grid_constant__ BcgsBatch B, const __grid_constant__ PruneArgs P) {
  const int e = blockIdx.y;
  const BcgsEntry& E = B.e[e];
  const int cnt = P.cnt[e], n = E.n;
  const double* src = E.A + (size_t)P.j0[e] * E.lda;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * cnt;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i % n), j = (int)(i / n), c = P.idx[e][j];
    P.tmpA[e][i] = src[(size_t)r + (size_t)c * E.lda];
    if (r == 0) P.tmpN[e][j] = E.norm0[P.j0[e] + c];
  }
}
// ... and written back over columns [j0, j0 + cnt)
__global__ void bcgs_prune_scatter_kernel(const __grid_constant__ BcgsBatch B, const __grid_constant__ PruneArgs P) {
  const int e = blockIdx.y;
  const BcgsEntry& E = B.e[e];
  const int cnt = P.cnt[e], n = E.n;
  double* dst = E.A + (size_t)P.j0[e] * E.lda;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * cnt;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i % n), j = (int)(i / n);
    dst[(size_t)r + (size_t)j * E.lda] = P.tmpA[e][i];
    if (r == 0) E.norm0[P.j0[e] + j] = P.tmpN[e][j];
  }
}

__global__ void col_norms_kernel(const __grid_constant__ BcgsBatch B) {
  const BcgsEntry& E = B.e[blockIdx.y];
  const int c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), ln = threadIdx.x & 31;
  if (c >= E.p) return;
  const double* a = E.A + (size_t)c * E.lda;
  double s = 0.0;
  for (int i = ln; i < E.n; i += 32) s += a[i] * a[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (ln == 0) E.norm0[c] = sqrt(s);
}

constexpr int kCutStage = 6144;   // small-end values staged in shared memory (48 KB)
__global__ void __launch_bounds__(256) rank_cut_kernel(int count, const double* __restrict__ s2, double factor,
                                                       const double* __restrict__ energy, int* r_out,
                                                       double* margin_out) {
  __shared__ double tail[kCutStage];
  // stage the small end s2[count - m .. count) (coalesced, whole block); the sum itself stays
  // sequential from the small end (the oracle's order)
  const int m = min(count, kCutStage), base = count - m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) tail[i] = s2[base + i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double thr = factor * (*energy);
  // tails from the small end: tail(r) = sum_{k >= r} s2[k]
  double acc = 0.0;
  int r = count;                 // default: keep everything
  double dmin = 1e300;           // min |tail - thr| over the visited tails (divided once below:
                                 // division by thr > 0 is monotone, so the margin is unchanged)
  for (int k = count - 1; k >= 1; --k) {
    acc += k >= base ? tail[k - base] : s2[k];   // not clamped: eigenvalues of a PSD Gram at the
                    // noise floor are +-eps||M||; clamping would bias the tail by (#noise) eps ||M||
    dmin = fmin(dmin, fabs(acc - thr));
    if (acc <= thr) {
      r = k;                    // tail beyond index k-1 fits: keep k values
    } else {
      break;
    }
  }
  const double margin = dmin >= 1e300 ? 1e300 : dmin / (thr > 0 ? thr : 1.0);
  if (count >= 1 && r < 1) r = 1;
  while (r > 0 && r < count && s2[r] == s2[r - 1] && s2[r] > 0) ++r;   // ties kept together (A23)
  *r_out = count == 0 ? 0 : r;
  if (margin_out) *margin_out = margin;
}

__global__ void basis_rank_kernel(int count, const double* __restrict__ lam, double tau, int* r_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int r = 0;
  const double lim = tau * lam[0];
  while (r < count && lam[r] > lim && lam[r] > 0.0) ++r;
  *r_out = r;
}

}  // namespace

// ---------------------------------------------------------------------------------------
void sl_eigen_device(cudaStream_t st, int n, const double* a_mid_dev, int boundary, double* lam, double* V,
                     int* status_dev) {
  Scratch s(st);
  double* sv = s.alloc<double>((size_t)3 * (n + 1));
  double* d = s.alloc<double>((size_t)3 * n);
  double* e = s.alloc<double>((size_t)3 * n);
  sl_assemble_kernel<<<dim3(cdiv(n + 1, 256), 3), 256, 0, st>>>(n, a_mid_dev, boundary, sv, d, e, status_dev);
  FC_CHECK_LAUNCH();
  gk_bisect_kernel<<<dim3(cdiv(n, 64), 3), 64, 0, st>>>(n, sv, lam);
  FC_CHECK_LAUNCH();
  double* scr = s.alloc<double>((size_t)5 * 3 * n * n);
  sl_invit_kernel<<<dim3(cdiv(n, 64), 3), 64, 0, st>>>(n, d, e, lam, V, scr);
  FC_CHECK_LAUNCH();
  sl_cluster_orth_kernel<<<dim3(cdiv(n, 64), 3), 64, 0, st>>>(n, lam, d, e, V, scr);
  FC_CHECK_LAUNCH();
  // Newton-Schulz polish: 2 steps of V <- V (3I - V^T V)/2 on DMMA GEMMs
  double* G = scr;                       // reuse: 3 n^2
  double* V2 = scr + (size_t)3 * n * n;  // 3 n^2 (fits: scratch is 15 n^2)
  for (int step = 0; step < 2; ++step) {
    GemmArgs g;
    g.transA = 1;
    g.nbatch = 3;
    for (int l = 0; l < 3; ++l)
      g.b[l] = GemmBatch{n, n, n, V + (size_t)l * n * n, n, V + (size_t)l * n * n, n, G + (size_t)l * n * n, n,
                         nullptr, 0, nullptr};
    gemm(g, st);
    ns_matrix_kernel<<<dim3(cdiv((long long)n * n, 256) > 1024 ? 1024 : cdiv((long long)n * n, 256), 3), 256, 0,
                       st>>>(n, G);
    FC_CHECK_LAUNCH();
    GemmArgs h;
    h.nbatch = 3;
    for (int l = 0; l < 3; ++l)
      h.b[l] = GemmBatch{n, n, n, V + (size_t)l * n * n, n, G + (size_t)l * n * n, n, V2 + (size_t)l * n * n, n,
                         nullptr, 0, nullptr};
    gemm(h, st);
    FC_CUDA_TRY(cudaMemcpyAsync(V, V2, (size_t)3 * n * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
}

template <int CS, bool GL = false>
void launch_tridiag_cluster(const SyevBatch& b, size_t smem, cudaStream_t st, int nlo, int nhi, int tsm = 0) {
  auto kern = tridiag_cluster_kernel<CS, GL>;
  static bool attr = false;
  if (!attr) {
    FC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    if (CS > 8) FC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS, b.nb, 1);
  // 512 threads per CTA: the per-step block barriers dominate at these sizes (C4 solve 359 ms vs
  // 365 ms with 1024; FC_TRI_THREADS overrides for diagnostics)
  static const int thr = getenv("FC_TRI_THREADS") ? atoi(getenv("FC_TRI_THREADS")) : 512;
  cfg.blockDim = dim3(thr, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FC_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, b, nlo, nhi, tsm));
  FC_CHECK_LAUNCH();
}

void syev_values(const SyevBatch& b, cudaStream_t st) {
  if (b.nb == 0) return;
  static const bool no_cluster = getenv("FC_NO_CLUSTER") != nullptr;
  const int minG = no_cluster ? kPackedMaxN : kCl16MaxN;   // sizes above go to the global kernel
  const int maxP = no_cluster ? kPackedMaxN : kClusterMinN; // sizes up to this: packed single CTA
  int maxN = 0;
  size_t smem_g = 0, smem_p = 0, smem_4 = 0, smem_8 = 0, smem_16 = 0;
  int gl_n = 0;
  static const bool no_gl = getenv("FC_NO_CLUSTER_GL") != nullptr;   // diagnostics: single-CTA kernel
  const int maxGL = (no_cluster || no_gl) ? minG : kClGlobalMaxN;
  bool any_g = false, any_p = false;
  // cluster size classes (N in (lo, hi]): 16 CTAs (non-portable) for 97..840 (the per-step
  // matvec / rank-2 work per CTA matters more than the DSMEM fan-in: C4 solve 365 ms vs 371 ms
  // with 8 CTAs up to 600 and 388 ms with 4 CTAs up to 440).  FC_TRI_CS=4|8: those layouts.
  static const int tri_cs = getenv("FC_TRI_CS") ? atoi(getenv("FC_TRI_CS")) : 16;
  const int cl4 = tri_cs == 4 ? kCl4MaxN : maxP;
  const int cl8 = tri_cs == 16 ? maxP : kCl8MaxN;
  constexpr int NW = kTriThreads / 32;
  for (int i = 0; i < b.nb; ++i) {
    const int N = b.e[i].N;
    maxN = std::max(maxN, N);
    if (N <= 0) continue;
    if (N <= maxP) {
      any_p = true;
      smem_p = std::max(smem_p, ((size_t)N * (N + 1) / 2 + 2 * (size_t)N) * 8);
    } else if (N > maxGL) {
      any_g = true;
      smem_g = std::max(smem_g, (size_t)(2 + NW) * N * 8);
    } else if (N > minG) {
      gl_n = std::max(gl_n, N);
    } else if (N <= cl4) {
      smem_4 = std::max(smem_4, cluster_smem_doubles<4>(N) * 8);
    } else if (N <= cl8) {
      smem_8 = std::max(smem_8, cluster_smem_doubles<8>(N) * 8);
    } else {
      smem_16 = std::max(smem_16, cluster_smem_doubles<16>(N) * 8);
    }
  }
  if (smem_4) launch_tridiag_cluster<4>(b, smem_4, st, maxP, cl4);
  if (smem_8) launch_tridiag_cluster<8>(b, smem_8, st, cl4, cl8);
  if (smem_16) launch_tridiag_cluster<16>(b, smem_16, st, cl8, kCl16MaxN);
  if (gl_n) {
    // one shared-memory head size for the launch, from its largest entry (smaller entries have
    // shorter columns: the same head fits)
    static const bool gl_all_l2 = getenv("FC_GL_NO_SMEM_HEAD") != nullptr;   // diagnostic
    size_t smem_gl = 0;
    int tsm = cluster_gl_tsm(gl_n, &smem_gl);
    if (gl_all_l2) {
      tsm = 0;
      smem_gl = cluster_smem_doubles<16, true>(gl_n) * 8;
    }
    launch_tridiag_cluster<16, true>(b, smem_gl, st, minG, maxGL, tsm);
  }
  if (maxN == 0) return;
  require(smem_g <= kTriSmemMax, FC_ERR_CAPACITY, "symmetric eigensolver: matrix dimension above 1500");
  static bool attr = false;
  if (!attr) {
    FC_CUDA_TRY(cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTriSmemMax));
    FC_CUDA_TRY(cudaFuncSetAttribute(tridiag_packed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr = true;
  }
  if (any_p) {
    static const int pthr = getenv("FC_TRI_PACKED_THREADS") ? atoi(getenv("FC_TRI_PACKED_THREADS")) : 1024;
    tridiag_packed_kernel<<<b.nb, pthr, smem_p, st>>>(b, maxP);
    FC_CHECK_LAUNCH();
  }
  if (any_g) {
    tridiag_kernel<<<b.nb, kTriThreads, smem_g, st>>>(b, maxGL);
    FC_CHECK_LAUNCH();
  }
  tri_bisect_kernel<<<dim3(cdiv(maxN, 8), b.nb), 256, (size_t)2 * maxN * 8, st>>>(b);
  FC_CHECK_LAUNCH();
}

void syev_vectors(const SyevBatch& b, int maxN, cudaStream_t st, const int* r_host) {
  if (b.nb == 0 || maxN == 0) return;
  // inverse-iteration solves per vector (FC_INVIT_SOLVES, default 3)
  static const int nsolve = getenv("FC_INVIT_SOLVES") ? atoi(getenv("FC_INVIT_SOLVES")) : 3;
  // shared-memory variant: T vectors per CTA, T sized for ~2 CTAs per SM over the batch and
  // the 227 KB limit (FC_INVIT_GLOBAL=1: the global-scratch kernel)
  static const bool inv_global = getenv("FC_INVIT_GLOBAL") != nullptr;
  int rmax = 0;
  long long tot = 0;
  for (int i = 0; i < b.nb; ++i) {
    const int ri = r_host ? std::min(r_host[i], b.e[i].N) : b.e[i].N;
    rmax = std::max(rmax, ri);
    tot += ri;
  }
  const size_t per_t = (size_t)maxN * (5 * 8 + 1), fixed = (size_t)2 * maxN * 8;
  const int tmax = (int)std::min<size_t>(32, (200u * 1024 - fixed) / std::max<size_t>(per_t, 1));
  if (!inv_global && tmax >= 1 && rmax > 0) {
    int T = (int)std::max<long long>(1, (tot + 2 * 148 - 1) / (2 * 148));
    T = std::min(T, tmax);
    const size_t smem = fixed + (size_t)T * per_t + 16;
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
      FC_CUDA_TRY(cudaFuncSetAttribute(tri_invit_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = smem;
    }
    tri_invit_smem_kernel<<<dim3(cdiv(rmax, T), b.nb), T, smem, st>>>(b, nsolve);
  } else {
    tri_invit_kernel<<<dim3(cdiv(maxN, 64), b.nb), 64, 0, st>>>(b, nsolve);
  }
  FC_CHECK_LAUNCH();
  static const bool trace_orth = getenv("FC_TRACE_ORTH") != nullptr;
  if (trace_orth) {   // diagnostics: orthogonality of the inverse-iteration vectors
    for (int i = 0; i < b.nb; ++i) {
      const SyevEntry& E = b.e[i];
      int r = 0;
      FC_CUDA_TRY(cudaMemcpyAsync(&r, E.r, sizeof(int), cudaMemcpyDeviceToHost, st));
      FC_CUDA_TRY(cudaStreamSynchronize(st));
      r = std::min(r, E.N);
      if (r <= 0) continue;
      double* G = nullptr;
      FC_CUDA_TRY(cudaMalloc(&G, (size_t)r * r * 8));
      dgemm(st, 1, 0, r, r, E.N, 1.0, E.Y, E.ldy, E.Y, E.ldy, 0.0, G, r);
      std::vector<double> h((size_t)r * r);
      FC_CUDA_TRY(cudaMemcpyAsync(h.data(), G, h.size() * 8, cudaMemcpyDeviceToHost, st));
      FC_CUDA_TRY(cudaStreamSynchronize(st));
      FC_CUDA_TRY(cudaFree(G));
      double mx = 0.0;
      int c2 = 0, c6 = 0, c10 = 0;
      for (int a = 0; a < r; ++a)
        for (int c = 0; c < r; ++c) {
          const double v = std::fabs(h[a + (size_t)c * r] - (a == c ? 1.0 : 0.0));
          mx = std::max(mx, v);
          if (a < c) {
            c2 += v > 1e-2;
            c6 += v > 1e-6;
            c10 += v > 1e-10;
          }
        }
      fprintf(stderr, "[fc orth] N=%d r=%d max|G-I|=%.2e pairs>1e-2:%d >1e-6:%d >1e-10:%d\n", E.N, r, mx, c2, c6, c10);
    }
  }
  // orthonormalisation of the inverse-iteration vectors (tridiagonal coordinates): polar steps on
  // GEMMs when the ranks are known on the host, CGS2 (one CTA per matrix) for the flagged or
  // all entries otherwise
  SyevBatch ob = b;
  for (int i = 0; i < ob.nb; ++i) ob.e[i].A = nullptr;
  static const bool no_polar = getenv("FC_ORTH_CGS2") != nullptr;   // diagnostic
  const int* flag = nullptr;
  Scratch s(st);
  if (r_host && !no_polar) {
    PolarBatch P;
    P.nb = b.nb;
    int* fl = s.zeros<int>(b.nb);
    P.flag = fl;
    size_t gsz = 0;
    int rmax = 1, tiles = 0;
    for (int i = 0; i < b.nb; ++i) {
      P.r[i] = std::min(r_host[i], b.e[i].N);
      gsz += (size_t)P.r[i] * P.r[i];
      rmax = std::max(rmax, P.r[i]);
      tiles += cdiv(P.r[i], 64) * cdiv(P.r[i], 64);
    }
    double* Gall = s.alloc<double>(std::max<size_t>(gsz, 1));
    double* Y2[kMaxSyev];
    size_t off = 0;
    for (int i = 0; i < b.nb; ++i) {
      P.G[i] = Gall + off;
      off += (size_t)P.r[i] * P.r[i];
      Y2[i] = s.alloc<double>(std::max<size_t>((size_t)b.e[i].N * P.r[i], 1));
    }
    for (int step = 0; step < 2; ++step) {
      GemmArgs g, h;
      g.transA = 1;
      g.beta = 1.0;
      int ng = 0;
      for (int i = 0; i < b.nb; ++i) {
        if (P.r[i] == 0) continue;
        const SyevEntry& E = b.e[i];
        const double* src = step == 0 ? E.Y : Y2[i];
        const int lds = step == 0 ? E.ldy : E.N;
        double* dst = step == 0 ? Y2[i] : E.Y;
        const int ldd = step == 0 ? E.N : E.ldy;
        g.b[ng] = GemmBatch{P.r[i], P.r[i], E.N, src, lds, src, lds, P.G[i], P.r[i], nullptr, 0, nullptr};
        h.b[ng] = GemmBatch{E.N, P.r[i], P.r[i], src, lds, P.G[i], P.r[i], dst, ldd, nullptr, 0, nullptr};
        ++ng;
      }
      if (ng == 0) break;
      g.nbatch = h.nbatch = ng;
      // split-K for ~`pw` waves of 148 SMs (FC_POLAR_WAVES overrides; diagnostics)
      static const int pw = getenv("FC_POLAR_WAVES") ? atoi(getenv("FC_POLAR_WAVES")) : 2;
      g.splitk = std::max(1, std::min(cdiv(maxN, 64), cdiv(pw * 148, std::max(tiles, 1))));
      FC_CUDA_TRY(cudaMemsetAsync(Gall, 0, gsz * 8, st));
      gemm(g, st);
      ns_polar_kernel<<<b.nb, 1024, (size_t)rmax * 8, st>>>(P, step);
      FC_CHECK_LAUNCH();
      gemm(h, st);
    }
    flag = fl;
  }
  orth_backtransform_kernel<<<b.nb, 1024, (size_t)maxN * 8, st>>>(ob, flag);
  FC_CHECK_LAUNCH();
  // back-transformation, warp per vector over many CTAs; reflectors staged through shared memory
  // (FC_BT_GLOBAL: the global-memory kernel)
  const dim3 grid(cdiv(maxN, 16), b.nb);
  static const bool bt_global = getenv("FC_BT_GLOBAL") != nullptr;
  constexpr size_t kBtSmem = 128 * 1024;
  static bool bt_attr = false;
  if (!bt_attr) {
    FC_CUDA_TRY(cudaFuncSetAttribute(backtransform_smem_kernel<16, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kBtSmem));
    FC_CUDA_TRY(cudaFuncSetAttribute(backtransform_smem_kernel<32, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kBtSmem));
    bt_attr = true;
  }
  if (!bt_global && maxN <= 512) backtransform_smem_kernel<16, 16><<<grid, 512, kBtSmem, st>>>(b);
  else if (!bt_global && maxN <= 1024) backtransform_smem_kernel<32, 8><<<grid, 512, kBtSmem, st>>>(b);
  else if (maxN <= 512) backtransform_kernel<16><<<grid, 512, 0, st>>>(b);
  else if (maxN <= 1024) backtransform_kernel<32><<<grid, 512, 0, st>>>(b);
  else backtransform_kernel<1><<<grid, 512, 0, st>>>(b);
  FC_CHECK_LAUNCH();
}

void orthonormalize_cols(int N, double* Y, int ldy, int* r_dev, int rmax, cudaStream_t st) {
  SyevBatch b;
  b.nb = 1;
  b.e[0] = SyevEntry{N, nullptr, 0, nullptr, nullptr, nullptr, Y, ldy, r_dev, nullptr};
  orth_backtransform_kernel<<<1, 1024, (size_t)std::max(rmax, 1) * 8, st>>>(b, nullptr);
  FC_CHECK_LAUNCH();
}

void pmgs(const PmgsBatch& b, cudaStream_t st) {
  if (b.nb == 0) return;
  int maxp = 1;
  for (int i = 0; i < b.nb; ++i) maxp = std::max(maxp, b.e[i].p);
  const size_t smem = (size_t)3 * maxp * 8;
  static bool attr = false;
  if (!attr) {
    FC_CUDA_TRY(cudaFuncSetAttribute(pmgs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  require(smem <= 200 * 1024, FC_ERR_CAPACITY, "pmgs: too many columns");
  pmgs_kernel<<<b.nb, kPmgsThreads, smem, st>>>(b);
  FC_CHECK_LAUNCH();
}

template <typename K>
void launch_cluster(K kern, int CS, int nb, size_t smem, cudaStream_t st, const BcgsBatch& b, int j0, int w,
                    int flag) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS, nb, 1);
  cfg.blockDim = dim3(kBcgsClusterThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FC_CUDA_TRY(cudaLaunchKernelEx(&cfg, (void (*)(BcgsBatch, int, int, int))kern, b, j0, w, flag));
  FC_CHECK_LAUNCH();
}

template <int CS, int W, int RB>
void bcgs_cluster_setup() {
  static bool attr = false;
  if (attr) return;
  const int smem = (int)sizeof(BcgsClusterSmem<W, RB>);
  FC_CUDA_TRY(cudaFuncSetAttribute(bcgs_block_cluster_kernel<CS, W, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  FC_CUDA_TRY(cudaFuncSetAttribute(bcgs_finalize_cluster_kernel<CS, W, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   smem));
  if (CS > 8) {
    FC_CUDA_TRY(cudaFuncSetAttribute(bcgs_block_cluster_kernel<CS, W, RB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    FC_CUDA_TRY(cudaFuncSetAttribute(bcgs_finalize_cluster_kernel<CS, W, RB>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                     1));
  }
  attr = true;
}

template <int CS, int W, int RB>
void bcgs_cluster_block(const BcgsBatch& bb, int j0, cudaStream_t st) {
  bcgs_cluster_setup<CS, W, RB>();
  static const int seq = getenv("FC_BCGS_SEQ") != nullptr;   // diagnostic: per-column in-block path
  launch_cluster(bcgs_block_cluster_kernel<CS, W, RB>, CS, bb.nb, sizeof(BcgsClusterSmem<W, RB>), st, bb, j0, W, seq);
}

template <int CS, int W, int RB>
void bcgs_cluster_finalize(const BcgsBatch& bb, int j0, cudaStream_t st) {
  bcgs_cluster_setup<CS, W, RB>();
  static const int mgs = getenv("FC_BCGS_MGS_FINAL") != nullptr;   // diagnostic: sequential MGS
  launch_cluster(bcgs_finalize_cluster_kernel<CS, W, RB>, CS, bb.nb, sizeof(BcgsClusterSmem<W, RB>), st, bb, j0, W, mgs);
}

// split-K for the two skinny GEMMs of a block projection, P = Q^T A_blk (k x W x n) and
// A_blk -= Q P (n x W x k): enough CTAs for ~2 waves of 148 SMs (64 x 64 tiles), at least 64 of
// the reduction dimension per split (deterministic split-K; P is written with beta = 0, A updated
// with beta = 1)
void split_skinny(GemmArgs& p, GemmArgs& u, int n, int k, int w, int nb) {
  static const int waves = getenv("FC_SKINNY_WAVES") ? atoi(getenv("FC_SKINNY_WAVES")) : 2;
  const int tp = cdiv(k, 64) * cdiv(w, 64) * nb, tu = cdiv(n, 64) * cdiv(w, 64) * nb;
  p.splitk = std::max(1, std::min(cdiv(n, 64), cdiv(waves * 148, tp)));
  u.splitk = std::max(1, std::min(cdiv(k, 64), cdiv(waves * 148, tu)));
}

void bcgs(const BcgsBatch& bin, cudaStream_t st) {
  if (bin.nb == 0) return;
  static const bool no_cluster = getenv("FC_NO_CLUSTER") != nullptr;
  int maxn = 0;
  for (int i = 0; i < bin.nb; ++i) maxn = std::max(maxn, bin.e[i].n);
  // 3: 8 CTAs x 128 rows (n <= 1024, default);  2: 16 x 128 (n <= 2048);  0: one CTA per matrix.
  // W = 64 (a W = 128 cluster variant was slower: 521 vs 479 ms per C4 solve with per-column steps)
  int cfg = 0;
  if (!no_cluster) {
    if (maxn <= 1024) cfg = 3;
    else if (maxn <= 2048) cfg = 2;
  }
  const int W = 64;
  auto block_step = [&](const BcgsBatch& bb, int j0) {
    if (cfg == 2) bcgs_cluster_block<16, 64, 128>(bb, j0, st);
    else if (cfg == 3) bcgs_cluster_block<8, 64, 128>(bb, j0, st);
    else {
      bcgs_block_kernel<<<bb.nb, 1024, (size_t)bb.e[0].n * 8, st>>>(bb, j0, W);
      FC_CHECK_LAUNCH();
    }
  };
  auto finalize_step = [&](const BcgsBatch& bb, int j0) {
    if (cfg == 2) bcgs_cluster_finalize<16, 64, 128>(bb, j0, st);
    else if (cfg == 3) bcgs_cluster_finalize<8, 64, 128>(bb, j0, st);
    else {
      bcgs_finalize_kernel<<<bb.nb, 1024, (size_t)bb.e[0].n * 8, st>>>(bb, j0);
      FC_CHECK_LAUNCH();
    }
  };
  BcgsBatch b = bin;
  // projection GEMMs bounded by the device count of accepted columns (FC_BCGS_NO_DYNK: full j0)
  static const bool dyn_k = getenv("FC_BCGS_NO_DYNK") == nullptr;
  static const bool trace = getenv("FC_TRACE") != nullptr;
  if (trace) {
    static bool reg = false;
    if (!reg) {
      reg = true;
      std::atexit([] {
        unsigned long long h[23];
        if (cudaMemcpyFromSymbol(h, g_bcgs_hist, sizeof(h)) != cudaSuccess) return;
        fprintf(stderr, "[bcgs] blocks %llu (redone %llu) prefiltered %llu deferred %llu rejected %llu; by decade:",
                h[19], h[21], h[18], h[20], h[22]);
        for (int d = 0; d < 18; ++d) fprintf(stderr, " %llu", h[d]);
        fprintf(stderr, "\n");
        unsigned long long cy[10];
        if (cudaMemcpyFromSymbol(cy, g_bcgs_cyc, sizeof(cy)) == cudaSuccess) {
          fprintf(stderr, "[bcgs] in-block Mcycles: gram+cholesky %.1f (gram %.1f) cholqr %.1f polar %.1f deferred %.1f\n",
                  cy[0] * 1e-6, cy[4] * 1e-6, cy[1] * 1e-6, cy[2] * 1e-6, cy[3] * 1e-6);
          fprintf(stderr, "[bcgs] cluster_gram Mcycles: partials %.1f sync1 %.1f reduce %.1f sync2 %.1f gather %.1f\n",
                  cy[5] * 1e-6, cy[6] * 1e-6, cy[7] * 1e-6, cy[8] * 1e-6, cy[9] * 1e-6);
        }
      });
    }
  }
  b.trace = trace;
  if (trace) {
    static bool tset = false;
    if (!tset) {
      int one = 1;
      FC_CUDA_TRY(cudaMemcpyToSymbol(g_bcgs_timing, &one, sizeof(int)));
      tset = true;
    }
  }
  Scratch scr(st);
  for (int i = 0; i < b.nb; ++i) {
    b.e[i].Y = scr.alloc<double>((size_t)b.e[i].n * kBcgsW);
    b.e[i].nacc = scr.alloc<int>(1);
  }
  int maxp = 0;
  for (int i = 0; i < b.nb; ++i) {
    BcgsEntry& E = b.e[i];
    FC_CUDA_TRY(cudaMemsetAsync(E.Q, 0, (size_t)E.ldq * E.kcap * 8, st));
    FC_CUDA_TRY(cudaMemsetAsync(E.P, 0, (size_t)E.kcap * kBcgsW * 8, st));   // the cluster kernels re-zero it
    const int kb = std::min(std::max(E.k_base, 0), std::min(E.p, E.kcap));
    E.k_base = kb;
    set_int_kernel<<<1, 1, 0, st>>>(E.k, kb);
    FC_CHECK_LAUNCH();
    if (kb > 0) {   // orthonormal prefix: into Q as it is; the rest is processed against it
      FC_CUDA_TRY(cudaMemcpy2DAsync(E.Q, (size_t)E.ldq * 8, E.A, (size_t)E.lda * 8, (size_t)E.n * 8, kb,
                                    cudaMemcpyDeviceToDevice, st));
      E.A += (size_t)kb * E.lda;
      E.p -= kb;
    }
    maxp = std::max(maxp, E.p);
  }
  col_norms_kernel<<<dim3(cdiv(maxp, 8), b.nb), 256, 0, st>>>(b);
  FC_CHECK_LAUNCH();
  for (int i = 0; i < b.nb; ++i) b.e[i].nmax = scr.alloc<double>(1);
  bcgs_nmax_kernel<<<b.nb, 256, 0, st>>>(b);
  FC_CHECK_LAUNCH();
  // bulk pruning (FC_BCGS_PRUNE=0 disables): before every second block from block 2 on the
  // remaining columns are projected against the accepted basis in one GEMM
  // pair and those whose residual is already within their acceptance level are dropped (the
  // greedy Gram-Schmidt would reject them when their block is reached); the survivors keep
  // their order.  On Khatri-Rao bases (numerical rank ~ p/4) most blocks are skipped this way.
  static const int prune_on = getenv("FC_BCGS_PRUNE") ? atoi(getenv("FC_BCGS_PRUNE")) : 1;
  // schedule (diagnostic knobs FC_BCGS_PRUNE_FIRST / _GAP / _INC, in blocks)
  static const int pr_first = getenv("FC_BCGS_PRUNE_FIRST") ? atoi(getenv("FC_BCGS_PRUNE_FIRST")) : 2;
  static const int pr_gap = getenv("FC_BCGS_PRUNE_GAP") ? atoi(getenv("FC_BCGS_PRUNE_GAP")) : 2;
  static const int pr_inc = getenv("FC_BCGS_PRUNE_INC") ? atoi(getenv("FC_BCGS_PRUNE_INC")) : 0;
  int next_prune = pr_first * W, prune_gap = std::max(1, pr_gap) * W;
  long long pruned_total = 0;
  for (int j0 = 0; j0 < maxp; j0 += W) {
    if (prune_on && j0 == next_prune) {
      next_prune += prune_gap;
      prune_gap += pr_inc * W;
      PruneArgs pa{};
      GemmArgs gp, gu;
      gp.transA = 1;
      gp.beta = 0.0;
      gu.alpha = -1.0;
      gu.beta = 1.0;
      int nb = 0, pmx = 0;
      bool any = false;
      for (int i = 0; i < b.nb; ++i) {
        const BcgsEntry& E = b.e[i];
        pa.j0[i] = j0;
        const int rem = E.p - j0;
        if (rem < 2 * W) continue;   // too few columns left to gain
        any = true;
        const int kup = std::min(E.k_base + j0, E.kcap);
        double* Pb = scr.alloc<double>((size_t)kup * rem);
        gp.b[nb] = GemmBatch{kup, rem, E.n, E.Q, E.ldq, E.A + (size_t)j0 * E.lda, E.lda, Pb, kup, nullptr, 0, nullptr};
        gp.b[nb].dynM = E.k;
        gu.b[nb] = GemmBatch{E.n, rem, kup, E.Q, E.ldq, Pb, kup, E.A + (size_t)j0 * E.lda, E.lda, nullptr, 0, nullptr};
        gu.b[nb].dynK = E.k;
        ++nb;
        pmx = std::max(pmx, rem);
      }
      if (any) {
        gp.nbatch = gu.nbatch = nb;
        gemm(gp, st);
        gemm(gu, st);
        pa.cnt = scr.alloc<int>(kMaxSyev);
        FC_CUDA_TRY(cudaMemsetAsync(pa.cnt, 0, kMaxSyev * sizeof(int), st));
        for (int i = 0; i < b.nb; ++i) {
          const BcgsEntry& E = b.e[i];
          const int rem = std::max(E.p - j0, 0);
          if (rem < 2 * W) {
            pa.j0[i] = E.p;   // untouched: nothing flagged, nothing moved
            continue;
          }
          pa.flag[i] = scr.alloc<int>(rem);
          pa.idx[i] = scr.alloc<int>(rem);
          pa.tmpA[i] = scr.alloc<double>((size_t)E.n * rem);
          pa.tmpN[i] = scr.alloc<double>(rem);
        }
        bcgs_prune_flag_kernel<<<dim3(cdiv(pmx, 8), b.nb), 256, 0, st>>>(b, pa);
        FC_CHECK_LAUNCH();
        bcgs_prune_compact_kernel<<<b.nb, 1024, 0, st>>>(b, pa);
        FC_CHECK_LAUNCH();
        const int gx = std::max(1, std::min(cdiv((long long)b.e[0].n * pmx, 256), 148 * 4 / std::max(b.nb, 1) + 1));
        bcgs_prune_gather_kernel<<<dim3(gx, b.nb), 256, 0, st>>>(b, pa);
        FC_CHECK_LAUNCH();
        bcgs_prune_scatter_kernel<<<dim3(gx, b.nb), 256, 0, st>>>(b, pa);
        FC_CHECK_LAUNCH();
        int cnt[kMaxSyev];
        FC_CUDA_TRY(cudaMemcpyAsync(cnt, pa.cnt, b.nb * sizeof(int), cudaMemcpyDeviceToHost, st));
        FC_CUDA_TRY(cudaStreamSynchronize(st));
        maxp = 0;
        for (int i = 0; i < b.nb; ++i) {
          BcgsEntry& E = b.e[i];
          if (pa.j0[i] == j0) {
            pruned_total += E.p - (j0 + cnt[i]);
            E.p = j0 + cnt[i];
          }
          maxp = std::max(maxp, E.p);
        }
        if (j0 >= maxp) break;
      }
    }
    // project the block against every column accepted so far (<= j0; unused Q columns are 0),
    // TWICE before the in-block step: after a single classical projection a column that lies
    // almost in span(Q) (residual ~1e-10 of its norm, still above the acceptance level) keeps a
    // Q-component of the order of its residual, the accept decision is taken on that noise and
    // the basis loses orthogonality completely (observed on the eigen-coordinate Khatri-Rao bases
    // of C4 at eps = 1e-8: |Q^T Q - I| = 1).  "Twice is enough" makes the residual accurate; the
    // accepted vectors then get the BCGS2 re-projection below.
    bool any_base = false;
    for (int i = 0; i < b.nb; ++i) any_base |= b.e[i].k_base > 0;
    static const int npre = getenv("FC_BCGS_PREPASS") ? atoi(getenv("FC_BCGS_PREPASS")) : 2;   // diagnostic
    for (int pass = 0; pass < npre && (j0 > 0 || any_base); ++pass) {
      GemmArgs p, u;
      p.transA = 1;
      p.beta = 0.0;   // P = Q^T A (rows beyond the accepted count are never read: dynK below)
      u.alpha = -1.0;
      u.beta = 1.0;
      int nb = 0, kmx = 0;
      for (int i = 0; i < b.nb; ++i) {
        const BcgsEntry& E = b.e[i];
        if (j0 >= E.p) continue;
        const int wb = std::min(W, E.p - j0), kup = std::min(E.k_base + j0, E.kcap);
        if (kup == 0) continue;
        kmx = std::max(kmx, kup);
        p.b[nb] = GemmBatch{kup, wb, E.n, E.Q, E.ldq, E.A + (size_t)j0 * E.lda, E.lda, E.P, kup, nullptr, 0, nullptr};
        u.b[nb] = GemmBatch{E.n, wb, kup, E.Q, E.ldq, E.P, kup, E.A + (size_t)j0 * E.lda, E.lda, nullptr, 0, nullptr};
        if (dyn_k) {               // only the first *E.k columns of Q are nonzero
          p.b[nb].dynM = E.k;
          u.b[nb].dynK = E.k;
        }
        ++nb;
      }
      p.nbatch = u.nbatch = nb;
      if (nb) {
        split_skinny(p, u, b.e[0].n, kmx, W, nb);
        gemm(p, st);
        gemm(u, st);
      }
    }
    block_step(b, j0);
    // BCGS2: re-project the accepted (unit) block vectors against the previous basis
    if (j0 > 0 || any_base) {
      GemmArgs p, u;
      p.transA = 1;
      p.beta = 0.0;
      u.alpha = -1.0;
      u.beta = 1.0;
      int nb = 0, kmx = 0;
      for (int i = 0; i < b.nb; ++i) {
        const BcgsEntry& E = b.e[i];
        if (j0 >= E.p) continue;
        const int kup = std::min(E.k_base + j0, E.kcap);
        if (kup == 0) continue;
        kmx = std::max(kmx, kup);
        p.b[nb] = GemmBatch{kup, W, E.n, E.Q, E.ldq, E.Y, E.n, E.P, kup, nullptr, 0, nullptr};
        u.b[nb] = GemmBatch{E.n, W, kup, E.Q, E.ldq, E.P, kup, E.Y, E.n, nullptr, 0, nullptr};
        if (dyn_k) {
          p.b[nb].dynM = E.k;
          u.b[nb].dynK = E.k;
        }
        ++nb;
      }
      p.nbatch = u.nbatch = nb;
      if (nb) {
        split_skinny(p, u, b.e[0].n, kmx, W, nb);
        gemm(p, st);
        gemm(u, st);
      }
    }
    finalize_step(b, j0);
  }
  if (trace && pruned_total) fprintf(stderr, "[bcgs] pruned %lld columns\n", pruned_total);
}

void rank_cut_device(int count, const double* s2, double factor, const double* energy, int* r_out,
                     double* margin_out, cudaStream_t st) {
  rank_cut_kernel<<<1, 256, 0, st>>>(count, s2, factor, energy, r_out, margin_out);
  FC_CHECK_LAUNCH();
}

void basis_rank_device(int count, const double* lam, double tau, int* r_out, cudaStream_t st) {
  basis_rank_kernel<<<1, 32, 0, st>>>(count, lam, tau, r_out);
  FC_CHECK_LAUNCH();
}

}  // namespace fc
