// The rank truncation trunc(x, eps) = RHOSVD (C2T) + Tucker core + Tucker-to-canonical
// [P:187-190, P:1791-1816], readings A10/A11/A12/A23, on mixed Tucker-canonical
// tensors (tt.cuh).
//
// Per mode l (batched over the 3 modes), with K = Q_l the basis and the factor columns
// y_t = K c_t, n_t = ||y_t||, xi_t = w_t prod_l n_{l,t}:
//   side matrix  A_l = [xi_t y_t / n_t]_t = K C D,  D = diag(xi_t / n_{l,t})          (S11)
//   K^T K = U Lam U^T,  F = Lam^1/2 U^T  (so F^T F = K^T K;  F = I for orthonormal K)
//   B = F C D,  B B^T = Y diag(s^2) Y^T   ->  the singular values of A_l are s (no inverse)
//   r_l = min{r : sum_{k>r} s_k^2 <= (eps/2)^2 sum xi^2}   (tails from the small end)
//   Z_l = K H F^T Y_r diag(1/s^2)  with H = C D^2 C^T  (left singular vectors), CGS2-polished
//   Chat_l = Z_l^T (K C diag(1/n_l))                                               (unit factors)
//   core beta = sum_t xi_t Chat_1[:,t] (x) Chat_2[:,t] (x) Chat_3[:,t]                (S12)
//   T2C: slice SVDs along the min-rank mode, pooled cut at (eps/2)^2 ||beta||^2        (S13)
#include <algorithm>
#include <map>
#include <mutex>
#include <cmath>
#include "cpops.cuh"
#include "eig.cuh"
#include "tt.cuh"

namespace fc {
namespace {

// n2[l][t] = sum_a C_l[a,t] * QC_l[a,t]   (QC = (Q^T Q) C, or C itself if orthonormal)
struct TermArgs {
  const double* C[3];
  const double* QC[3];
  int q[3];
  double* n2[3];
};
__global__ void term_norms_kernel(int R, TermArgs a) {
  const int l = blockIdx.y;
  const int t = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int ln = threadIdx.x & 31;
  if (t >= R) return;
  const int q = a.q[l];
  const double* c = a.C[l] + (size_t)t * q;
  const double* qc = a.QC[l] + (size_t)t * q;
  double s = 0.0;
  for (int k = ln; k < q; k += 32) s += c[k] * qc[k];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (ln == 0) a.n2[l][t] = fmax(s, 0.0);
}

// Khatri-Rao structured input (f1): term T = kk*Rx + j has mode coefficient Rm_kk cx_j, so
// n2[T] = cx_j^T (Rm_kk^T Rm_kk cx_j) = sum_a Cx[a, j] * P[a, T] with P[:, T] = Gm_kk cx_j.
struct StructNormArgs {
  const double* Cx[3];
  const double* P[3];
  int t[3];
  double* n2[3];
};
__global__ void struct_norms_kernel(int R, int Rx, StructNormArgs a) {
  const int l = blockIdx.y;
  const int T = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int ln = threadIdx.x & 31;
  if (T >= R) return;
  const int t = a.t[l], j = T % Rx;
  const double* c = a.Cx[l] + (size_t)j * t;
  const double* p = a.P[l] + (size_t)T * t;
  double s = 0.0;
  for (int k = ln; k < t; k += 32) s += c[k] * p[k];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (ln == 0) a.n2[l][T] = fmax(s, 0.0);
}

// W[:, T] = Cx[:, T % Rx] * d[T]   (t x R): the structured side-matrix coefficients C_x D
__global__ void struct_scale_kernel(int t, int R, int Rx, const double* __restrict__ Cx, const double* __restrict__ d,
                                    double* W) {
  const long long tot = (long long)t * R;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int a = (int)(idx % t);
    const int T = (int)(idx / t);
    W[idx] = Cx[a + (size_t)(T % Rx) * t] * d[T];
  }
}

// ---- weighted Khatri-Rao basis (structured route) ---------------------------------------------
// The structured side matrix is A_l = sum_a K_a W'_a with K_a = [w_a (.) xhat_b]_b (n x t) and
// W'_a[b, (kk, j)] = E[a, kk] Cx[b, j] d[kk, j]: column (a, b) of K enters A_l only through row
// (a, b) of the coefficient matrix, whose norm is rho_{a,b} = (sum_kk E[a,kk]^2 H_kk[b,b])^1/2,
// H_kk = W_kk W_kk^T.  The rank-revealing Gram-Schmidt therefore runs on K diag(rho / rho_max):
// a residual e dropped from a scaled column perturbs A_l by ||e|| rho_max — the same bound as
// dropping it from the unscaled column with the largest weight — while the columns that carry
// little of x (x's trailing Tucker directions) no longer force basis vectors of their own.
struct ColWeightArgs {
  const double* E[3];     // s x r (ld s)
  const double* H[3];     // t x t x r
  int s[3], t[3];
  double* wgt[3];         // s*t column weights rho / rho_max (1 if every rho is 0)
};
__global__ void __launch_bounds__(1024) col_weight_kernel(int r, ColWeightArgs a) {
  __shared__ double red[32];
  __shared__ double mx_s;
  const int l = blockIdx.x, s = a.s[l], t = a.t[l], p = s * t;
  const double* E = a.E[l];
  const double* H = a.H[l];
  double mx = 0.0;
  for (int c = threadIdx.x; c < p; c += blockDim.x) {
    const int aa = c / t, b = c % t;
    double v = 0.0;
    for (int kk = 0; kk < r; ++kk) {
      const double e = E[aa + (size_t)kk * s];
      v = fma(e * e, fmax(H[b + (size_t)b * t + (size_t)kk * t * t], 0.0), v);
    }
    a.wgt[l][c] = v;
    mx = fmax(mx, v);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) mx_s = v;
  }
  __syncthreads();
  const double m = mx_s;
  for (int c = threadIdx.x; c < p; c += blockDim.x) a.wgt[l][c] = m > 0.0 ? sqrt(a.wgt[l][c] / m) : 1.0;
}
// out[:, c] = in[:, c] * wgt[c]   (n x p, contiguous columns)
__global__ void scale_copy_cols_kernel(int n, int p, const double* __restrict__ in, const double* __restrict__ wgt,
                                       double* __restrict__ out) {
  const long long tot = (long long)n * p;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x)
    out[idx] = in[idx] * wgt[idx / n];
}

// ---- accurate factor of the per-term side Grams (A11' on the structured route) --------------
// The structured side matrix of mode l is B = [Rm_1 W_1 | ... | Rm_r W_r], W_k = Cx diag(d_k)
// (t x Rx per spectral term k).  B B^T = sum_k Rm_k L_k L_k^T Rm_k^T for ANY L_k with
// L_k L_k^T = W_k W_k^T, so B's singular values are those of the explicit q x (r t) matrix
// B~ = [Rm_k L_k]_k.  L_k is computed WITHOUT the Gram's squaring floor: H_k = W_k W_k^T is
// accumulated in double-double (TwoProduct by FMA + TwoSum, ~1e-32 relative), factored by a
// diagonally pivoted Cholesky in double-double, and only the factor is rounded to double.  A
// rounding of L (or of Rm, or of a later product with B~) perturbs v^T B B^T v by
// ~2 ||B^T v|| eps_mach ||B|| — linear in the small singular values, not eps_mach ||B||^2.
constexpr int kFactorMaxT = 512;       // t (x's Tucker rank) handled by the factor kernel
constexpr int kFactorSmemT = 96;       // up to this t the dd Gram lives in shared memory
constexpr int kFactorThreads = 512;
constexpr int kFactorJC = 32;          // W columns staged per chunk
constexpr int kFactorEnt = 10;         // Gram entries per thread and pass over W

struct dd { double hi, lo; };
__device__ __forceinline__ dd dd_fast2sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {           // (hi, lo) + (hi, lo), TwoSum on hi
  const double s = a.hi + b.hi, bb = s - a.hi;
  const double err = (a.hi - (s - bb)) + (b.hi - bb);
  return dd_fast2sum(s, err + a.lo + b.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  const double p = a.hi * b.hi;
  const double e = fma(a.hi, b.hi, -p) + (a.hi * b.lo + a.lo * b.hi);
  return dd_fast2sum(p, e);
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {
  const double q1 = a.hi / b.hi;
  const dd r = dd_add(a, dd_mul({-q1, 0.0}, b));
  return dd_fast2sum(q1, r.hi / b.hi);
}
__device__ __forceinline__ dd dd_sqrt(dd a) {
  if (a.hi <= 0.0) return {0.0, 0.0};
  const double s = sqrt(a.hi);
  const double e = (fma(-s, s, a.hi) + a.lo) / (2.0 * s);
  return dd_fast2sum(s, e);
}

// entry e of the row-major lower triangle -> (a, b), a >= b
__device__ __forceinline__ void tri_entry(int e, int& a, int& b) {
  a = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
  while ((a + 1) * (a + 2) / 2 <= e) ++a;
  while (a * (a + 1) / 2 > e) --a;
  b = e - a * (a + 1) / 2;
}

// Partial dd Grams over column chunks: CTA (k, sp) accumulates H_k's lower triangle over the W_k
// columns [sp chunk, (sp + 1) chunk) and writes (hi, lo) to Hp[((k S + sp) 2 + {0, 1}) t^2 + a + b t].
// One CTA per spectral term left 13 of 148 SMs busy for ~4 ms per launch at eps = 1e-8 (a quarter
// of that solve); the factor kernel below adds the S partials in split order (dd, fixed order).
template <int ENT>
__global__ void __launch_bounds__(kFactorThreads) struct_gram_dd_kernel(int t, int Rx, int chunk,
                                                                        const double* __restrict__ Cx,
                                                                        const double* __restrict__ d, double* Hp) {
  extern __shared__ double fsm[];
  const int k = blockIdx.x, sp = blockIdx.y, S = gridDim.y, tid = threadIdx.x;
  const int ne = t * (t + 1) / 2;
  const int jlo = sp * chunk, jhi = min(Rx, jlo + chunk);
  double* Wc = fsm;                                  // t x kFactorJC chunk of W_k
  const double* dk = d + (size_t)k * Rx;
  double* Ph = Hp + ((size_t)k * S + sp) * 2 * t * t;
  double* Pl = Ph + (size_t)t * t;
  for (int e0 = 0; e0 < ne; e0 += ENT * kFactorThreads) {
    int ea[ENT], eb[ENT];
    dd acc[ENT];
#pragma unroll
    for (int q = 0; q < ENT; ++q) {
      const int e = e0 + tid + q * kFactorThreads;
      int a = 0, b = 0;
      if (e < ne) tri_entry(e, a, b);
      ea[q] = a;
      eb[q] = b;
      acc[q] = {0.0, 0.0};
    }
    for (int j0 = jlo; j0 < jhi; j0 += kFactorJC) {
      const int jc = min(kFactorJC, jhi - j0);
      __syncthreads();
      for (int idx = tid; idx < t * jc; idx += kFactorThreads) {
        const int a = idx % t, jj = idx / t;
        Wc[a + jj * t] = Cx[a + (size_t)(j0 + jj) * t] * dk[j0 + jj];
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < ENT; ++q) {
        if (e0 + tid + q * kFactorThreads >= ne) break;
        const int a = ea[q], b = eb[q];
        double hi = acc[q].hi, lo = acc[q].lo;
        for (int jj = 0; jj < jc; ++jj) {
          const double x = Wc[a + jj * t], y = Wc[b + jj * t];
          const double p = x * y, pe = fma(x, y, -p);
          const double s = hi + p, bb = s - hi;
          lo += ((hi - (s - bb)) + (p - bb)) + pe;
          hi = s;
        }
        acc[q].hi = hi;
        acc[q].lo = lo;
      }
#pragma unroll
      for (int q = 0; q < ENT; ++q) acc[q] = dd_fast2sum(acc[q].hi, acc[q].lo);
    }
#pragma unroll
    for (int q = 0; q < ENT; ++q) {
      if (e0 + tid + q * kFactorThreads >= ne) break;
      Ph[ea[q] + eb[q] * t] = acc[q].hi;
      Pl[ea[q] + eb[q] * t] = acc[q].lo;
    }
  }
}

// one CTA per spectral term k: L_k (t x t, column-major, ld t; columns beyond the numerical rank
// are zero) with L_k L_k^T = W_k W_k^T, W_k[a, j] = Cx[a + j t] d[k Rx + j].  The dd Gram (hi, lo)
// is in shared memory for t <= kFactorSmemT, else in this CTA's slice of Hg (2 t^2 doubles per
// CTA, L2-resident); Gram entries are accumulated kFactorEnt per thread per pass over W.
template <int ENT>
__global__ void __launch_bounds__(kFactorThreads) struct_factor_kernel(int t, int Rx, const double* __restrict__ Cx,
                                                                       const double* __restrict__ d, double* Lout,
                                                                       double* Hg, const double* __restrict__ Hp,
                                                                       int S) {
  extern __shared__ double fsm[];
  const int k = blockIdx.x, tid = threadIdx.x;
  const int ne = t * (t + 1) / 2;
  const bool gl = t > kFactorSmemT;
  double* Wc = fsm;                                  // t x kFactorJC chunk of W_k
  double* Lc = fsm + (size_t)t * kFactorJC;          // current column (hi, lo): 2 t
  double* piv = Lc + 2 * t;                          // used flags: t
  int* rem = reinterpret_cast<int*>(piv + t);        // unpivoted indices (t ints in t doubles)
  double* Hh = gl ? Hg + (size_t)k * 2 * t * t : piv + 2 * t;   // t x t (hi), later the Schur complement
  double* Hl = Hh + (size_t)t * t;                   // t x t (lo)
  const double* dk = d + (size_t)k * Rx;
  if (Hp) {
    // the Gram comes as S partial dd sums over column chunks (struct_gram_dd_kernel): added in
    // split order
    for (int e = tid; e < ne; e += kFactorThreads) {
      int a, b;
      tri_entry(e, a, b);
      dd acc = {0.0, 0.0};
      for (int sp = 0; sp < S; ++sp) {
        const double* Ph = Hp + ((size_t)k * S + sp) * 2 * t * t;
        acc = dd_add(acc, {Ph[a + b * t], Ph[(size_t)t * t + a + b * t]});
      }
      Hh[a + b * t] = Hh[b + a * t] = acc.hi;
      Hl[a + b * t] = Hl[b + a * t] = acc.lo;
    }
  }
  for (int e0 = 0; e0 < (Hp ? 0 : ne); e0 += ENT * kFactorThreads) {
    // entry e -> (a, b), a >= b, row-major over the lower triangle
    int ea[ENT], eb[ENT];
    dd acc[ENT];
#pragma unroll
    for (int q = 0; q < ENT; ++q) {
      const int e = e0 + tid + q * kFactorThreads;
      int a = 0, b = 0;
      if (e < ne) {
        a = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
        while ((a + 1) * (a + 2) / 2 <= e) ++a;
        while (a * (a + 1) / 2 > e) --a;
        b = e - a * (a + 1) / 2;
      }
      ea[q] = a;
      eb[q] = b;
      acc[q] = {0.0, 0.0};
    }
    for (int j0 = 0; j0 < Rx; j0 += kFactorJC) {
      const int jc = min(kFactorJC, Rx - j0);
      __syncthreads();
      for (int idx = tid; idx < t * jc; idx += kFactorThreads) {
        const int a = idx % t, jj = idx / t;
        Wc[a + jj * t] = Cx[a + (size_t)(j0 + jj) * t] * dk[j0 + jj];
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < ENT; ++q) {
        if (e0 + tid + q * kFactorThreads >= ne) break;
        const int a = ea[q], b = eb[q];
        double hi = acc[q].hi, lo = acc[q].lo;
        for (int jj = 0; jj < jc; ++jj) {
          const double x = Wc[a + jj * t], y = Wc[b + jj * t];
          const double p = x * y, pe = fma(x, y, -p);
          const double s = hi + p, bb = s - hi;
          lo += ((hi - (s - bb)) + (p - bb)) + pe;
          hi = s;
        }
        acc[q].hi = hi;
        acc[q].lo = lo;
      }
#pragma unroll
      for (int q = 0; q < ENT; ++q) acc[q] = dd_fast2sum(acc[q].hi, acc[q].lo);
    }
#pragma unroll
    for (int q = 0; q < ENT; ++q) {
      if (e0 + tid + q * kFactorThreads >= ne) break;
      const int a = ea[q], b = eb[q];
      Hh[a + b * t] = Hh[b + a * t] = acc[q].hi;
      Hl[a + b * t] = Hl[b + a * t] = acc[q].lo;
    }
  }
  __syncthreads();
  for (int i = tid; i < t; i += kFactorThreads) piv[i] = 0.0;
  double* L = Lout + (size_t)k * t * t;
  for (int i = tid; i < t * t; i += kFactorThreads) L[i] = 0.0;
  __syncthreads();
  __shared__ double s_tr;
  __shared__ int s_p, s_nrem;
  __shared__ double w_best[kFactorThreads / 32];
  __shared__ int w_idx[kFactorThreads / 32];
  if (tid == 0) {
    double tr = 0.0;
    for (int i = 0; i < t; ++i) tr += Hh[i + i * t];
    s_tr = tr;
    s_nrem = t;
  }
  for (int i = tid; i < t; i += kFactorThreads) rem[i] = i;
  __syncthreads();
  const double stop = 1e-30 * s_tr;
  const int warp = tid >> 5, lane = tid & 31;
  for (int c = 0; c < t; ++c) {
    const int nrem = s_nrem;
    // diagonal pivot: the largest Schur diagonal among the unpivoted indices (ties -> the
    // smallest index), block-wide argmax
    double best = stop;
    int bi = -1;
    for (int q = tid; q < nrem; q += kFactorThreads) {
      const int i = rem[q];
      const double v = Hh[i + i * t];
      if (v > best || (v == best && bi >= 0 && i < bi)) {
        best = v;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (oi >= 0 && (bi < 0 || ov > best || (ov == best && oi < bi))) {
        best = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      w_best[warp] = best;
      w_idx[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double b = stop;
      int p = -1;
      for (int w = 0; w < kFactorThreads / 32; ++w)
        if (w_idx[w] >= 0 && (p < 0 || w_best[w] > b || (w_best[w] == b && w_idx[w] < p))) {
          b = w_best[w];
          p = w_idx[w];
        }
      s_p = p;
      if (p >= 0) {
        piv[p] = 1.0;
        int q = 0;                                    // remove p from the unpivoted list
        while (rem[q] != p) ++q;
        rem[q] = rem[nrem - 1];
        s_nrem = nrem - 1;
      }
    }
    __syncthreads();
    const int p = s_p;
    if (p < 0) break;                                 // the rest of H is below 1e-30 of its trace
    const dd sp = dd_sqrt({Hh[p + p * t], Hl[p + p * t]});
    for (int i = tid; i < t; i += kFactorThreads) {
      dd v = {0.0, 0.0};
      if (i == p) v = sp;
      else if (piv[i] == 0.0) v = dd_div({Hh[i + p * t], Hl[i + p * t]}, sp);
      Lc[2 * i] = v.hi;
      Lc[2 * i + 1] = v.lo;
      L[i + (size_t)c * t] = v.hi + v.lo;
    }
    __syncthreads();
    // Schur complement on the unpivoted lower triangle: pairs (qa >= qb) of the remaining list
    // (a warp per row qa of the list, rows dealt from both ends so that every warp gets the same
    // number of pairs; lanes over qb <= qa: no index decoding per pair)
    const int nr = nrem - 1;
    constexpr int NWF = kFactorThreads / 32;
    for (int h = warp; h < (nr + 1) / 2; h += NWF) {
      for (int side = 0; side < 2; ++side) {
        const int qa = side == 0 ? h : nr - 1 - h;
        if (side == 1 && qa == h) break;              // middle row of an odd count: once
        const int i = rem[qa];
        const double lih = -Lc[2 * i], lil = -Lc[2 * i + 1];
        for (int qb = lane; qb <= qa; qb += 32) {
          const int j = rem[qb];
          const size_t ij = (size_t)i + (size_t)j * t, ji = (size_t)j + (size_t)i * t;   // equal entries
          const dd v = dd_add({Hh[ji], Hl[ji]}, dd_mul({lih, lil}, {Lc[2 * j], Lc[2 * j + 1]}));
          Hh[ij] = Hh[ji] = v.hi;
          Hl[ij] = Hl[ji] = v.lo;
        }
      }
    }
    __syncthreads();
  }
}

// out[:, c] = in[:, c] * d[c]   (rows x cols, ld rows)
__global__ void scale_cols_kernel(int rows, int cols, const double* __restrict__ in, const double* __restrict__ d,
                                  double* out) {
  const long long tot = (long long)rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x)
    out[idx] = in[idx] * d[idx / rows];
}

// xi_t, d_l[t] = xi_t / n_l[t], inv_n_l[t] = 1/n_l[t], energy += xi^2 (single block reduction)
__global__ void term_weights_kernel(int R, const double* __restrict__ w, const double* n2a, const double* n2b,
                                    const double* n2c, double* xi, double* da, double* db, double* dc,
                                    double* ia, double* ib, double* ic, double* part) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < R; t += gridDim.x * blockDim.x) {
    double na = sqrt(n2a[t]), nb = sqrt(n2b[t]), nc = sqrt(n2c[t]);
    double x = w[t] * na * nb * nc;
    bool zero = (x == 0.0);
    xi[t] = x;
    da[t] = zero ? 0.0 : w[t] * nb * nc;
    db[t] = zero ? 0.0 : w[t] * na * nc;
    dc[t] = zero ? 0.0 : w[t] * na * nb;
    ia[t] = zero ? 0.0 : 1.0 / na;
    ib[t] = zero ? 0.0 : 1.0 / nb;
    ic[t] = zero ? 0.0 : 1.0 / nc;
    acc += x * x;
  }
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

// energy = sum of the per-block partials in block order (deterministic)
__global__ void sum_parts_kernel(int nb, const double* __restrict__ part, double* out) {
  if (threadIdx.x != 0) return;
  double v = 0.0;
  for (int b = 0; b < nb; ++b) v += part[b];
  *out = v;
}

// F = Lam^1/2 U^T from the (descending) eigenpairs of K^T K.  Eigenvalues below the
// eigensolver's noise level (kBasisTau * lam_max, bisection accuracy ~ 2 eps ||T||) are
// numerical null directions of K and are set to 0 (their square roots would be pure noise).
constexpr double kBasisTau = 1e-14;
__global__ void sqrt_factor_kernel(int q, const double* lam, const double* U, double* F) {
  const double lim = kBasisTau * lam[0];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < q * q; idx += gridDim.x * blockDim.x) {
    int i = idx % q, j = idx / q;                 // F[i, j] = sqrt(lam_i) * U[j, i]
    F[idx] = lam[i] > lim ? sqrt(lam[i]) * U[j + (size_t)i * q] : 0.0;
  }
}

__global__ void scale_rows_kernel(int rows, int cols, const double* __restrict__ in, int ldi,
                                  const double* __restrict__ s, double* out, int ldo) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)rows * cols;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx % rows), j = (int)(idx / rows);
    out[i + (size_t)j * ldo] = s[i] * in[i + (size_t)j * ldi];
  }
}

__global__ void inv_sq_kernel(int r, const double* __restrict__ s2, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < r) out[i] = s2[i] > 0 ? 1.0 / s2[i] : 0.0;
}

// KR12[(a + r1*b), t] = xi_t * C1[a,t] * C2[b,t]
__global__ void kr12_kernel(int r1, int r2, int R, const double* __restrict__ xi, const double* __restrict__ C1,
                            const double* __restrict__ C2, double* out) {
  const long long tot = (long long)r1 * r2 * R;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    int ab = (int)(idx % (r1 * r2));
    int t = (int)(idx / (r1 * r2));
    int a = ab % r1, b = ab / r1;
    out[idx] = xi[t] * C1[a + (size_t)t * r1] * C2[b + (size_t)t * r2];
  }
}

// slices: S_nu[x, y] = core[ia, ib, ic] with (mode a index x, mode b index y, mode c index nu)
__global__ void extract_slices_kernel(const double* __restrict__ core, int r0, int r1, int r2, int ma, int mb,
                                      int mc, double* S) {
  const int r[3] = {r0, r1, r2};
  const int ra = r[ma], rb = r[mb], rc = r[mc];
  const long long tot = (long long)ra * rb * rc;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    int x = (int)(idx % ra);
    int y = (int)((idx / ra) % rb);
    int nu = (int)(idx / ((long long)ra * rb));
    int id[3];
    id[ma] = x; id[mb] = y; id[mc] = nu;
    S[idx] = core[id[0] + (size_t)r0 * (id[1] + (size_t)r1 * id[2])];
  }
}

// One-sided Jacobi SVD of each slice (ra x rb, column-major) in shared memory; one CTA per
// slice.  Outputs k = min(ra, rb) triples sorted by s descending: s[nu*k + m],
// Ua[nu*ra*k + m*ra + x], Vb[nu*rb*k + m*rb + y].
// Slices whose working set exceeds the shared-memory budget run the same algorithm in a
// per-slice global (L2-resident) workspace `gws` of (rows*cols + cols*cols) doubles.
constexpr int kSliceMax = 1024;
constexpr double kJacobiQuad = 1e-8;   // see slice_svd_qrj_kernel
__device__ int g_slice_sweeps_max = 0;   // diagnostics (FC_TRACE): most Jacobi sweeps of a slice
__device__ unsigned long long g_slice_cyc[4] = {0, 0, 0, 0};   // ... slice 0's cycles in QR / X setup / Jacobi / outputs
constexpr size_t kSliceSmem = 200 * 1024;
// SMEM: the working set lives in shared memory (the compiler then emits LDS/STS; with a pointer
// that may be global it emits generic loads); else in the per-slice global workspace gws.
template <bool SMEM>
__global__ void __launch_bounds__(512) slice_svd_kernel(int ra, int rb, const double* __restrict__ S, double* s_out,
                                                        double* Ua, double* Vb, double* gws) {
  extern __shared__ double sm[];
  const int nu = blockIdx.x;
  const bool tr = ra < rb;                     // work on S^T when wide
  const int rows = tr ? rb : ra, cols = tr ? ra : rb;
  const int k = cols;                          // = min(ra, rb)
  double* A = SMEM ? sm : gws + (size_t)nu * ((size_t)rows * cols + (size_t)cols * cols);   // rows x cols
  double* W = A + rows * cols;                 // cols x cols rotations
  double* nrm = SMEM ? W + cols * cols : sm;   // cols
  int* order = (int*)(nrm + cols);             // cols
  const double* src = S + (size_t)nu * ra * rb;
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, ln = tid & 31, nw = nt >> 5;
  // columns sorted by decreasing norm (de Rijk): column j of the slice goes to position
  // order-rank(j); W starts as that permutation, so A_final = A_slice W holds throughout
  for (int j = warp; j < cols; j += nw) {
    double s2 = 0;
    for (int i = ln; i < rows; i += 32) {
      const double v = tr ? src[j + (size_t)i * ra] : src[i + (size_t)j * ra];
      s2 = fma(v, v, s2);
    }
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (ln == 0) nrm[j] = s2;
  }
  __syncthreads();
  for (int j = tid; j < cols; j += nt) {
    int rk = 0;
    for (int i = 0; i < cols; ++i) rk += (nrm[i] > nrm[j]) || (nrm[i] == nrm[j] && i < j);
    order[j] = rk;
  }
  __syncthreads();
  for (int idx = tid; idx < rows * cols; idx += nt) {
    int i = idx % rows, j = idx / rows;
    A[i + (size_t)order[j] * rows] = tr ? src[j + (size_t)i * ra] : src[i + (size_t)j * ra];
  }
  for (int idx = tid; idx < cols * cols; idx += nt) {
    const int i = idx % cols, j = idx / cols;
    W[idx] = (order[i] == j) ? 1.0 : 0.0;
  }
  __shared__ int changed;
  __shared__ double fro2_s;
  if (tid == 0) {
    double f = 0.0;
    for (int j = 0; j < cols; ++j) f += nrm[j];
    fro2_s = f;
  }
  __syncthreads();
  // columns below 1e-12 ||slice||_F are numerical noise whose triples the pooled eps cut always
  // drops (for eps >= 1e-9): pairs involving them count as converged
  const double neg2 = 1e-24 * fro2_s;
  const int p = cols + (cols & 1);
  // convergence: |a_i . a_j| <= tol ||a_i|| ||a_j|| with tol = 2 sqrt(rows) eps (the rounding
  // level of the computed dot product; LAPACK dgesvj uses sqrt(m) eps)
  const double tol = 2.0 * sqrt((double)rows) * 2.220446049250313e-16, tol2 = tol * tol;
  // G lanes per column pair (power of two, 4..32): all p/2 pairs of a round in one wave
  int G = 32;
  while (G > 4 && nt / G < p / 2) G >>= 1;
  const int gid = tid / G, gl = tid % G, ng = nt / G;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) changed = 0;
    __syncthreads();
    for (int rd = 0; rd < p - 1; ++rd) {
      // uniform trip count over the block: every lane reaches the shuffles (full mask, no
      // divergent shuffle handling); groups without a pair reduce zeros
      for (int pi0 = 0; pi0 < p / 2; pi0 += ng) {
        const int pi = pi0 + gid;
        int a = 0, b = 0;
        bool act = pi < p / 2;
        if (act) {
          if (pi == 0) { a = rd % (p - 1); b = p - 1; }
          else { a = (rd + pi) % (p - 1); b = (rd - pi + p - 1) % (p - 1); }
          if (a > b) { int t = a; a = b; b = t; }
          act = b < cols;
        }
        double al = 0, be = 0, ga = 0;
        if (act)
          for (int i = gl; i < rows; i += G) {
            double x = A[i + a * rows], y = A[i + b * rows];
            al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
          }
        for (int o = G >> 1; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (!act || ga == 0.0 || ga * ga <= tol2 * (al * be) || al <= neg2 || be <= neg2) continue;
        // Rutishauser's rotation, zeta = (be - al) / (2 ga), t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)),
        // written with one square root and one division
        const double dd = be - al, g2 = 2.0 * ga;
        const double t = copysign(1.0, dd) * g2 / (fabs(dd) + sqrt(fma(dd, dd, g2 * g2)));
        const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
        for (int i = gl; i < rows; i += G) {
          double x = A[i + a * rows], y = A[i + b * rows];
          A[i + a * rows] = c * x - s * y;
          A[i + b * rows] = s * x + c * y;
        }
        for (int i = gl; i < cols; i += G) {
          double x = W[i + a * cols], y = W[i + b * cols];
          W[i + a * cols] = c * x - s * y;
          W[i + b * cols] = s * x + c * y;
        }
        if (gl == 0) changed = 1;
      }
      __syncthreads();
    }
    if (!changed) {
      if (tid == 0) atomicMax(&g_slice_sweeps_max, sweep + 1);
      break;
    }
    if (sweep == 39 && tid == 0) atomicMax(&g_slice_sweeps_max, 40);
    __syncthreads();
  }
  for (int j = warp; j < cols; j += nw) {
    double s2 = 0;
    for (int i = ln; i < rows; i += 32) s2 += A[i + j * rows] * A[i + j * rows];
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (ln == 0) nrm[j] = sqrt(s2);
  }
  __syncthreads();
  for (int j = tid; j < cols; j += nt) {     // rank by (s desc, index asc)
    int rk = 0;
    for (int i = 0; i < cols; ++i) rk += (nrm[i] > nrm[j]) || (nrm[i] == nrm[j] && i < j);
    order[rk] = j;
  }
  __syncthreads();
  // outputs: left vectors u (ra), right v (rb)
  for (int idx = tid; idx < k * (ra + rb); idx += nt) {
    int m = idx / (ra + rb), e = idx % (ra + rb);
    int j = order[m];
    double sj = nrm[j];
    double inv = sj > 0 ? 1.0 / sj : 0.0;
    if (e < ra) {
      int x = e;   // left vector component
      double v = tr ? W[x + j * cols] : A[x + j * rows] * inv;
      Ua[(size_t)nu * ra * k + (size_t)m * ra + x] = v;
    } else {
      int y = e - ra;
      double v = tr ? A[y + j * rows] * inv : W[y + j * cols];
      Vb[(size_t)nu * rb * k + (size_t)m * rb + y] = v;
    }
  }
  for (int m = tid; m < k; m += nt) s_out[(size_t)nu * k + m] = nrm[order[m]];
}

// T2C slice SVD with QR preconditioning (Drmac-Veselic): A P = Q R by Householder QR with column
// pivoting, then one-sided Jacobi on the columns of R^T (graded, nearly diagonal: a few sweeps
// instead of ~16 on the slice itself).  R^T W = U' Sigma gives A = (Q W) Sigma (P U')^T: the tall-
// side vectors are Q W (reflectors applied to W), the short-side vectors P U'.  Same outputs and
// convergence test as slice_svd_kernel; shared memory: rows*cols + 2 cols^2 + 3 cols doubles.
size_t slice_qrj_smem(int rows, int cols) {
  return ((size_t)rows * cols + 2 * (size_t)(cols | 1) * cols + 3 * (size_t)cols) * 8 + (size_t)cols * 8 + 64;
}

// SMEM = false: A, X, W in a per-matrix global (L2-resident) workspace gws of
// rows*cols + 2*(cols|1)*cols doubles (matrices too large for shared memory, e.g. the 2D
// truncation's ~126 x 126 cores); the small arrays stay in shared memory.
template <bool SMEM>
__global__ void __launch_bounds__(1024) slice_svd_qrj_kernel(int ra, int rb, const double* __restrict__ S,
                                                            double* s_out, double* Ua, double* Vb, double* gws,
                                                            double jacobi_quad) {
  extern __shared__ double sm[];
  const int nu = blockIdx.x;
  const bool tr = ra < rb;
  const int rows = tr ? rb : ra, cols = tr ? ra : rb, k = cols;
  const int lx = cols | 1;                          // odd leading dimension of X and W: the
                                                    // thread groups of a Jacobi round (different
                                                    // column pairs, same rows) hit distinct banks
  double* A = SMEM ? sm : gws + (size_t)nu * ((size_t)rows * cols + 2 * (size_t)lx * cols);
                                                    // rows x cols: R above, reflectors below
  double* X = A + (size_t)rows * cols;              // cols x cols (ld lx): R^T, rotated by Jacobi
  double* W = X + (size_t)lx * cols;                // cols x cols (ld lx) rotations
  double* cn = SMEM ? W + (size_t)lx * cols : sm;   // cols: column norms^2 / singular values
  double* tau = cn + cols;                          // cols
  double* red = tau + cols;                         // cols (reduction scratch)
  int* perm = (int*)(red + cols);                   // cols
  int* order = perm + cols;                         // cols
  __shared__ int piv_s;
  __shared__ double sval;
  __shared__ int changed, big;
  const double* src = S + (size_t)nu * ra * rb;
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, ln = tid & 31, nw = nt >> 5;
  for (int idx = tid; idx < rows * cols; idx += nt) {
    const int i = idx % rows, j = idx / rows;
    A[idx] = tr ? src[j + (size_t)i * ra] : src[i + (size_t)j * ra];
  }
  for (int j = tid; j < cols; j += nt) perm[j] = j;
  __syncthreads();
  double fro2 = 0.0;
  const bool timing = (nu == 0 && tid == 0);
  long long tc0 = timing ? clock64() : 0;
  // ---- Householder QR with column pivoting ----
  // trailing column norms: exact sums over rows >= i; computed once here and then accumulated in
  // the same pass (and order) that applies each reflector
  for (int j = warp; j < cols; j += nw) {
    const double* a = A + (size_t)j * rows;
    double s2 = 0.0;
    for (int t = ln; t < rows; t += 32) s2 = fma(a[t], a[t], s2);
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (ln == 0) cn[j] = s2;
  }
  __syncthreads();
  for (int i = 0; i < cols; ++i) {
    // pivot = largest trailing norm (lowest index on ties): one warp
    if (warp == 0) {
      double bv = -1.0;
      int bj = cols;
      for (int j = i + ln; j < cols; j += 32)
        if (cn[j] > bv) { bv = cn[j]; bj = j; }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ov > bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
      }
      if (ln == 0) piv_s = bj < cols ? bj : i;
      if (i == 0) {
        double f = 0.0;
        for (int j = ln; j < cols; j += 32) f += cn[j];
        for (int o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
        if (ln == 0) sval = f;
      }
    }
    __syncthreads();
    if (i == 0) fro2 = sval;
    const int pj = piv_s;
    if (pj != i) {
      for (int t = tid; t < rows; t += nt) {
        const double x = A[t + (size_t)i * rows];
        A[t + (size_t)i * rows] = A[t + (size_t)pj * rows];
        A[t + (size_t)pj * rows] = x;
      }
      if (tid == 0) {
        const int q = perm[i]; perm[i] = perm[pj]; perm[pj] = q;
        const double c = cn[i]; cn[i] = cn[pj]; cn[pj] = c;
      }
      __syncthreads();
    }
    // reflector for column i (rows i..): v = x - alpha e1, stored normalised with v0 = 1
    double* ai = A + (size_t)i * rows;
    const double x0 = ai[i];
    const double sig = cn[i] - x0 * x0;          // sum of squares below the diagonal
    double alpha = x0, tv = 0.0;
    if (sig > 0.0 || x0 < 0.0) {
      const double nrm = sqrt(fmax(cn[i], 0.0));
      alpha = -copysign(nrm, x0);
      const double v0 = x0 - alpha;
      tv = (alpha - x0) / alpha;                  // tau = (alpha - x0) / alpha, v scaled by 1/v0
      const double inv = 1.0 / v0;
      for (int t = i + 1 + tid; t < rows; t += nt) ai[t] *= inv;
    }
    __syncthreads();
    // apply H = I - tau v v^T to the trailing columns (warp per column); the same pass leaves
    // the next step's trailing norm (rows >= i+1) in cn[j]
    for (int j = i + 1 + warp; j < cols; j += nw) {
      double* a = A + (size_t)j * rows;
      double s2 = 0.0;
      if (tv != 0.0) {
        double d = (ln == 0) ? a[i] : 0.0;
        for (int t = i + 1 + ln; t < rows; t += 32) d = fma(ai[t], a[t], d);
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        const double f = tv * d;
        if (ln == 0) a[i] -= f;
        for (int t = i + 1 + ln; t < rows; t += 32) {
          const double v = a[t] - f * ai[t];
          a[t] = v;
          s2 = fma(v, v, s2);
        }
      } else {
        for (int t = i + 1 + ln; t < rows; t += 32) s2 = fma(a[t], a[t], s2);
      }
      for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      if (ln == 0) cn[j] = s2;
    }
    if (tid == 0) {
      tau[i] = tv;
      red[i] = alpha;                            // R[i, i]
    }
    __syncthreads();
  }
  if (timing) { const long long t = clock64(); atomicAdd(&g_slice_cyc[0], (unsigned long long)(t - tc0)); tc0 = t; }
  // X = R^T (cols x cols, lower triangular), W = I
  for (int idx = tid; idx < cols * cols; idx += nt) {
    const int r = idx % cols, c = idx / cols;    // X[r, c] = R[c, r]
    X[r + c * lx] = (r > c) ? A[c + (size_t)r * rows] : (r == c ? red[r] : 0.0);
    W[r + c * lx] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (timing) { const long long t = clock64(); atomicAdd(&g_slice_cyc[1], (unsigned long long)(t - tc0)); tc0 = t; }
  // ---- one-sided Jacobi on the columns of X ----
  const double neg2 = 1e-24 * fro2;
  const int p = cols + (cols & 1);
  const double tol = 2.0 * sqrt((double)cols) * 2.220446049250313e-16, tol2 = tol * tol;
  const double quad2 = jacobi_quad * jacobi_quad;
  int G = 32;
  while (G > 4 && nt / G < p / 2) G >>= 1;
  const int gid = tid / G, gl = tid % G, ng = nt / G;
  // A sweep whose rotations all had cosines <= kJacobiQuad leaves cosines of their square's order
  // (quadratic convergence of the cyclic method): it is the last one, the all-quiet confirming
  // sweep is not run.
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) changed = big = 0;
    __syncthreads();
    for (int rd = 0; rd < p - 1; ++rd) {
      for (int pi0 = 0; pi0 < p / 2; pi0 += ng) {
        const int pi = pi0 + gid;
        int a = 0, b = 0;
        bool act = pi < p / 2;
        if (act) {
          // round-robin pairing; rd, pi < p - 1: one conditional subtraction replaces the modulo
          if (pi == 0) { a = rd; b = p - 1; }
          else {
            a = rd + pi; if (a >= p - 1) a -= p - 1;
            b = rd - pi; if (b < 0) b += p - 1;
          }
          if (a > b) { int t = a; a = b; b = t; }
          act = b < cols;
        }
        double al = 0, be = 0, ga = 0;
        if (act)
          for (int i = gl; i < cols; i += G) {
            const double x = X[i + a * lx], y = X[i + b * lx];
            al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
          }
        for (int o = G >> 1; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (!act || ga == 0.0 || ga * ga <= tol2 * (al * be) || al <= neg2 || be <= neg2) continue;
        const double dd = be - al, g2 = 2.0 * ga;
        const double t = copysign(1.0, dd) * g2 / (fabs(dd) + sqrt(fma(dd, dd, g2 * g2)));
        const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
        for (int i = gl; i < cols; i += G) {
          double x = X[i + a * lx], y = X[i + b * lx];
          X[i + a * lx] = c * x - sn * y;
          X[i + b * lx] = sn * x + c * y;
          x = W[i + a * lx];
          y = W[i + b * lx];
          W[i + a * lx] = c * x - sn * y;
          W[i + b * lx] = sn * x + c * y;
        }
        if (gl == 0) {
          changed = 1;
          if (ga * ga > quad2 * (al * be)) big = 1;
        }
      }
      __syncthreads();
    }
    if (!changed || !big) {
      if (tid == 0) atomicMax(&g_slice_sweeps_max, sweep + 1);
      break;
    }
    __syncthreads();
  }
  if (timing) { const long long t = clock64(); atomicAdd(&g_slice_cyc[2], (unsigned long long)(t - tc0)); tc0 = t; }
  // singular values, order
  for (int j = warp; j < cols; j += nw) {
    double s2 = 0;
    for (int i = ln; i < cols; i += 32) s2 = fma(X[i + j * lx], X[i + j * lx], s2);
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (ln == 0) cn[j] = sqrt(s2);
  }
  __syncthreads();
  for (int j = tid; j < cols; j += nt) {
    int rk = 0;
    for (int i = 0; i < cols; ++i) rk += (cn[i] > cn[j]) || (cn[i] == cn[j] && i < j);
    order[rk] = j;
  }
  __syncthreads();
  // tall-side vectors: Q w_j = H_0 (H_1 ... (H_{c-1} [w_j; 0])).  rows <= 128: register-resident
  // vectors (element ln + 32 c in slot c), two vectors per warp at a time — their reflector
  // applications (dot, butterfly, update) are independent chains and share the loads of v_i
  if (rows <= 128) {
    for (int mb = warp; mb < k; mb += 2 * nw) {
      const int m1 = mb + nw;
      const bool two = m1 < k;
      const int j0 = order[mb], j1 = two ? order[m1] : j0;
      double o0[4], o1[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int t = ln + 32 * c;
        const bool in = t < rows && t < cols;
        o0[c] = in ? W[t + (size_t)j0 * lx] : 0.0;
        o1[c] = (in && two) ? W[t + (size_t)j1 * lx] : 0.0;
      }
      for (int i = cols - 1; i >= 0; --i) {
        const double tv = tau[i];
        if (tv == 0.0) continue;
        const double* v = A + (size_t)i * rows;   // v_i[i] = 1, v_i[t] = A[t, i] for t > i
        double vv[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int t = ln + 32 * c;
          vv[c] = t == i ? 1.0 : ((t > i && t < rows) ? v[t] : 0.0);
        }
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          d0 = fma(vv[c], o0[c], d0);
          d1 = fma(vv[c], o1[c], d1);
        }
        for (int o = 16; o > 0; o >>= 1) {
          d0 += __shfl_xor_sync(0xffffffffu, d0, o);
          d1 += __shfl_xor_sync(0xffffffffu, d1, o);
        }
        const double f0 = tv * d0, f1 = tv * d1;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          o0[c] = fma(-f0, vv[c], o0[c]);
          o1[c] = fma(-f1, vv[c], o1[c]);
        }
      }
      double* out0 = tr ? (Vb + (size_t)nu * rb * k + (size_t)mb * rb) : (Ua + (size_t)nu * ra * k + (size_t)mb * ra);
      double* out1 = tr ? (Vb + (size_t)nu * rb * k + (size_t)m1 * rb) : (Ua + (size_t)nu * ra * k + (size_t)m1 * ra);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int t = ln + 32 * c;
        if (t < rows) {
          out0[t] = o0[c];
          if (two) out1[t] = o1[c];
        }
      }
    }
  }
  for (int m = warp; m < (rows <= 128 ? 0 : k); m += nw) {
    const int j = order[m];
    double* out = tr ? (Vb + (size_t)nu * rb * k + (size_t)m * rb) : (Ua + (size_t)nu * ra * k + (size_t)m * ra);
    for (int t = ln; t < rows; t += 32) out[t] = t < cols ? W[t + (size_t)j * lx] : 0.0;
    __syncwarp();
    for (int i = cols - 1; i >= 0; --i) {
      const double tv = tau[i];
      if (tv == 0.0) continue;
      const double* v = A + (size_t)i * rows;   // v_i[i] = 1, v_i[t] = A[t, i] for t > i
      double d = (ln == 0) ? out[i] : 0.0;
      for (int t = i + 1 + ln; t < rows; t += 32) d = fma(v[t], out[t], d);
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      const double f = tv * d;
      __syncwarp();
      if (ln == 0) out[i] -= f;
      for (int t = i + 1 + ln; t < rows; t += 32) out[t] -= f * v[t];
      __syncwarp();
    }
  }
  // short-side vectors: P u'_j (u'_j = x_j / sigma_j), row perm[i] <- entry i
  for (int idx = tid; idx < k * cols; idx += nt) {
    const int m = idx / cols, i = idx % cols;
    const int j = order[m];
    const double sj = cn[j];
    const double v = sj > 0 ? X[i + (size_t)j * lx] / sj : 0.0;
    if (tr) Ua[(size_t)nu * ra * k + (size_t)m * ra + perm[i]] = v;
    else Vb[(size_t)nu * rb * k + (size_t)m * rb + perm[i]] = v;
  }
  for (int m = tid; m < k; m += nt) s_out[(size_t)nu * k + m] = cn[order[m]];
  if (timing) atomicAdd(&g_slice_cyc[3], (unsigned long long)(clock64() - tc0));
}

// pool all (s, nu, m), sort by s desc, ties (nu, m) asc: rank of each element by counting
// (thread per element, candidates staged through shared-memory tiles); s2 sorted and keys
__global__ void __launch_bounds__(256) pool_rank_kernel(int K, const double* __restrict__ s, double* s2_sorted,
                                                        int* key_sorted) {
  __shared__ double tile[1024];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double si = i < K ? s[i] : 0.0;
  int rk = 0;
  for (int j0 = 0; j0 < K; j0 += 1024) {
    const int m = min(1024, K - j0);
    __syncthreads();
    for (int t = threadIdx.x; t < m; t += blockDim.x) tile[t] = s[j0 + t];
    __syncthreads();
    for (int t = 0; t < m; ++t) {
      const double sj = tile[t];
      rk += (sj > si) || (sj == si && j0 + t < i);
    }
  }
  if (i < K) {
    s2_sorted[rk] = si * si;
    key_sorted[rk] = i;
  }
}

// energy = sum s^2 (single block, fixed order)
__global__ void __launch_bounds__(1024) pool_energy_kernel(int K, const double* __restrict__ s, double* energy) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < K; i += blockDim.x) acc += s[i] * s[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) *energy = v;
  }
}

// output coefficients for the first R terms
__global__ void t2c_scatter_kernel(int R, int k, int ra, int rb, int rc, const int* __restrict__ keys,
                                   const double* __restrict__ s2, const double* __restrict__ Ua,
                                   const double* __restrict__ Vb, double* w, double* Ca, double* Cb, double* Cc) {
  const int m2 = blockIdx.x;
  if (m2 >= R) return;
  const int key = keys[m2];
  const int nu = key / k, m = key % k;
  for (int x = threadIdx.x; x < ra; x += blockDim.x) Ca[x + (size_t)m2 * ra] = Ua[(size_t)nu * ra * k + (size_t)m * ra + x];
  for (int y = threadIdx.x; y < rb; y += blockDim.x) Cb[y + (size_t)m2 * rb] = Vb[(size_t)nu * rb * k + (size_t)m * rb + y];
  for (int z = threadIdx.x; z < rc; z += blockDim.x) Cc[z + (size_t)m2 * rc] = (z == nu) ? 1.0 : 0.0;
  if (threadIdx.x == 0) w[m2] = sqrt(s2[m2]);
}

__global__ void identity_kernel(int n, double* I) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x)
    I[idx] = (idx % n == idx / n) ? 1.0 : 0.0;
}

__global__ void blockdiag_kernel(int q1, int R1, const double* __restrict__ C1, int q2, int R2,
                                 const double* __restrict__ C2, double* out) {
  const int q = q1 + q2, R = R1 + R2;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)q * R;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx % q), t = (int)(idx / q);
    double v = 0.0;
    if (t < R1 && i < q1) v = C1[i + (size_t)t * q1];
    else if (t >= R1 && i >= q1) v = C2[(i - q1) + (size_t)(t - R1) * q2];
    out[idx] = v;
  }
}

// number of kept T2C triples per slice (the kept set of each slice is a prefix of its
// descending singular values)
__global__ void slice_counts_kernel(int R, int k, const int* __restrict__ keys, int* counts) {
  int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m < R) atomicAdd(counts + keys[m] / k, 1);
}

// T2C output core in mode order: core[id] = sum_{m < cnt[nu]} s[nu,m] Ua[nu][x,m] Vb[nu][y,m]
// with id[ma] = x, id[mb] = y, id[mc] = nu
__global__ void t2c_core_kernel(int ra, int rb, int rc, int k, const int* __restrict__ cnt,
                                const double* __restrict__ s, const double* __restrict__ Ua,
                                const double* __restrict__ Vb, int ma, int mb, int mc, int r0, int r1, double* core) {
  const long long tot = (long long)ra * rb * rc;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(idx % ra), y = (int)((idx / ra) % rb), nu = (int)(idx / ((long long)ra * rb));
    const int km = cnt[nu];
    const double* u = Ua + (size_t)nu * ra * k;
    const double* v = Vb + (size_t)nu * rb * k;
    const double* sv = s + (size_t)nu * k;
    double acc = 0.0;
    for (int m = 0; m < km; ++m) acc += sv[m] * u[x + (size_t)m * ra] * v[y + (size_t)m * rb];
    int id[3];
    id[ma] = x; id[mb] = y; id[mc] = nu;
    core[id[0] + (size_t)r0 * (id[1] + (size_t)r1 * id[2])] = acc;
  }
}

// X2 [x + r0 (b + t1 z)] -> X2p [b + t1 (x + r0 z)], batched over nb blocks of size r0*t1*r2
__global__ void permute_xbz_kernel(int nb, int r0, int t1, int r2, const double* __restrict__ X, double* Y) {
  const long long per = (long long)r0 * t1 * r2, tot = per * nb;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long bI = idx / per, e = idx % per;
    const int x = (int)(e % r0), b = (int)((e / r0) % t1), z = (int)(e / ((long long)r0 * t1));
    Y[bI * per + b + (size_t)t1 * (x + (size_t)r0 * z)] = X[idx];
  }
}

// core[x + r0 (y + r1 z)] += sum_i wF[kk0 + i] * X3_i[y + r1 (x + r0 z)]
__global__ void accumulate_core_kernel(int nb, int r0, int r1, int r2, const double* __restrict__ wF, int kk0,
                                       const double* __restrict__ X3, double* core) {
  const long long per = (long long)r0 * r1 * r2;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < per;
       idx += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(idx % r0), y = (int)((idx / r0) % r1), z = (int)(idx / ((long long)r0 * r1));
    double acc = core[idx];
    for (int i = 0; i < nb; ++i) acc += wF[kk0 + i] * X3[i * per + y + (size_t)r1 * (x + (size_t)r0 * z)];
    core[idx] = acc;
  }
}

// fixed-order dot of two arrays: per-block partials, then one thread sums them in block order
__global__ void core_dot_kernel(long long tot, const double* __restrict__ a, const double* __restrict__ b,
                                double* part) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot; i += (long long)gridDim.x * blockDim.x)
    s = fma(a[i], b[i], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void core_dot_final_kernel(int nb, const double* __restrict__ part, double* out) {
  if (threadIdx.x != 0) return;
  double t = 0.0;
  for (int i = 0; i < nb; ++i) t += part[i];
  *out = t;
}

// B^T: out[j + i*cols] = in[i + j*rows]   (in rows x cols, column-major)
__global__ void transpose_kernel(int rows, int cols, const double* __restrict__ in, double* out) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)rows * cols;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % rows), j = (int)(idx / rows);
    out[j + (size_t)i * cols] = in[idx];
  }
}

// A[i + j q] = (i == j) for a q x q block (A pre-zeroed)
__global__ void eye_kernel(int q, double* A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < q) A[i + (size_t)i * q] = 1.0;
}

__global__ void square_into_kernel(int k, const double* __restrict__ s, double* s2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) s2[i] = s[i] * s[i];
}

int blocks_for(long long total) {
  long long b = (total + 255) / 256;
  return (int)std::min<long long>(std::max<long long>(b, 1), 148 * 8);
}

// FC_TRACE_ORTH_Y diagnostics: max |A^T A - I| of a rows x cols column-major block
double dbg_orth(cudaStream_t st, const double* A, int rows, int cols, int ld) {
  if (cols <= 0) return 0.0;
  Scratch s(st);
  double* G = s.alloc<double>((size_t)cols * cols);
  dgemm(st, 1, 0, cols, cols, rows, 1.0, A, ld, A, ld, 0.0, G, cols);
  std::vector<double> h((size_t)cols * cols);
  FC_CUDA_TRY(cudaMemcpyAsync(h.data(), G, h.size() * 8, cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  double e = 0.0;
  for (int i = 0; i < cols; ++i)
    for (int j = 0; j < cols; ++j) e = std::max(e, std::fabs(h[i + (size_t)j * cols] - (i == j ? 1.0 : 0.0)));
  return e;
}

int read_int(const int* d, cudaStream_t st) {
  int h = 0;
  FC_CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  return h;
}

}  // namespace

// ---- FC_PHASES: real-run time per truncation phase (CUDA events between phase marks; host
// waits included, i.e. what the stream actually spends), printed at exit --------------------
struct PhaseProf {
  std::mutex mu;
  std::map<std::string, std::pair<double, long>> acc;
  ~PhaseProf() {
    if (acc.empty()) return;
    std::vector<std::pair<double, std::string>> v;
    double tot = 0.0;
    for (auto& kv : acc) {
      v.push_back({kv.second.first, kv.first});
      tot += kv.second.first;
    }
    std::sort(v.rbegin(), v.rend());
    fprintf(stderr, "[fc phases] total %.1f ms\n", tot);
    for (auto& x : v)
      fprintf(stderr, "[fc phases] %8.2f ms %5.1f%%  %-28s x%ld\n", x.first, 100.0 * x.first / tot, x.second.c_str(),
              acc[x.second].second);
  }
};
PhaseProf& phase_prof() {
  static PhaseProf p;
  return p;
}
PhaseMarks::PhaseMarks(cudaStream_t s) : st(s) {
  static const bool enabled = getenv("FC_PHASES") != nullptr;
  on = enabled;
  mark("start");
}
void PhaseMarks::mark(const char* name) {
  if (!on) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, st);
  m.push_back({name, e});
}
PhaseMarks::~PhaseMarks() {
  if (!on) return;
  if (m.size() >= 2 && cudaEventSynchronize(m.back().second) == cudaSuccess) {
    PhaseProf& P = phase_prof();
    std::lock_guard<std::mutex> lock(P.mu);
    for (size_t i = 1; i < m.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, m[i - 1].second, m[i].second);
      auto& a = P.acc[m[i].first];
      a.first += ms;
      a.second += 1;
    }
  }
  for (auto& x : m) cudaEventDestroy(x.second);
}

// ---------------------------------------------------------------------------------------
// Batched SVD of ns column-major ra x rb matrices (S + nu*ra*rb): k = min(ra, rb) triples per
// matrix sorted by s descending (s[nu*k + m], Ua[nu*ra*k + m*ra + x], Vb[nu*rb*k + m*rb + y]).
// QR-preconditioned one-sided Jacobi when the working set fits shared memory, else the plain
// one-sided Jacobi (shared memory, or a per-matrix global workspace).
void small_svd(cudaStream_t st, int ra, int rb, int ns, const double* S, double* sv, double* Ua, double* Vb) {
  require(std::max(ra, rb) <= kSliceMax, FC_ERR_CAPACITY, "small SVD: dimension above 1024");
  if (ns == 0 || ra == 0 || rb == 0) return;
  const int k = std::min(ra, rb);
  Scratch s(st);
  const int rows = std::max(ra, rb), cols = k;
  size_t smem = ((size_t)rows * cols + (size_t)cols * cols + cols) * 8 + (size_t)cols * 4 + 16;
  double* gws = nullptr;
  if (smem > kSliceSmem) {
    gws = s.alloc<double>((size_t)ns * ((size_t)rows * cols + (size_t)cols * cols));
    smem = (size_t)cols * 12 + 16;
  }
  static bool attr = false;
  if (!attr) {
    FC_CUDA_TRY(cudaFuncSetAttribute(slice_svd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kSliceSmem));
    attr = true;
  }
  static const bool no_qr = getenv("FC_SLICE_NO_QR") != nullptr;
  const size_t qsm = slice_qrj_smem(rows, cols);
  // 768 threads: C4 44.0 iters/s vs 43.4 with 512, 43.9 with 640 and 43.3 with 1024
  // (profiles/r01h_knob_sweep_slice.txt); FC_SLICE_THREADS overrides (diagnostic)
  static const int sthr_env = getenv("FC_SLICE_THREADS") ? atoi(getenv("FC_SLICE_THREADS")) : 768;
  // FC_SLICE_THREADS=0 (diagnostic): 16 lanes per Jacobi column pair, every pair in one pass
  const int sthr = sthr_env > 0 ? sthr_env
                                : std::min(1024, std::max(256, ((16 * ((std::min(ra, rb) + 1) / 2)) + 31) / 32 * 32));
  static bool qattr = false;
  if (!qattr) {
    FC_CUDA_TRY(cudaFuncSetAttribute(slice_svd_qrj_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kSliceSmem));
    qattr = true;
  }
  // FC_JACOBI_QUAD: cosine level below which a sweep is taken as the last (0: always confirm)
  static const double jquad = getenv("FC_JACOBI_QUAD") ? atof(getenv("FC_JACOBI_QUAD")) : kJacobiQuad;
  if (!no_qr && qsm <= kSliceSmem) {
    slice_svd_qrj_kernel<true><<<ns, sthr, qsm, st>>>(ra, rb, S, sv, Ua, Vb, nullptr, jquad);
  } else if (!no_qr) {
    // QR-preconditioned Jacobi with the matrices in an L2-resident global workspace
    double* qws = s.alloc<double>((size_t)ns * ((size_t)rows * cols + 2 * (size_t)(cols | 1) * cols));
    const size_t small = (5 * (size_t)cols) * 8 + 64;
    slice_svd_qrj_kernel<false><<<ns, sthr, small, st>>>(ra, rb, S, sv, Ua, Vb, qws, jquad);
  } else if (gws) {
    slice_svd_kernel<false><<<ns, 512, smem, st>>>(ra, rb, S, sv, Ua, Vb, gws);
  } else {
    slice_svd_kernel<true><<<ns, 512, smem, st>>>(ra, rb, S, sv, Ua, Vb, nullptr);
  }
  FC_CHECK_LAUNCH();
  if (getenv("FC_TRACE")) {
    int sw = 0, zero = 0;
    FC_CUDA_TRY(cudaMemcpyFromSymbolAsync(&sw, g_slice_sweeps_max, sizeof(int), 0, cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaMemcpyToSymbolAsync(g_slice_sweeps_max, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, st));
    FC_CUDA_TRY(cudaStreamSynchronize(st));
    unsigned long long cy[4], zc[4] = {0, 0, 0, 0};
    FC_CUDA_TRY(cudaMemcpyFromSymbol(cy, g_slice_cyc, sizeof(cy)));
    FC_CUDA_TRY(cudaMemcpyToSymbol(g_slice_cyc, zc, sizeof(zc)));
    fprintf(stderr, "[fc svd] %d matrices of %d x %d: max sweeps %d; slice 0 kcycles: QR %.0f, X %.0f, Jacobi %.0f, out %.0f\n",
            ns, ra, rb, sw, cy[0] * 1e-3, cy[1] * 1e-3, cy[2] * 1e-3, cy[3] * 1e-3);
  }
}

TT tucker_to_canonical(fc_ctx c, const double* core, const int r[3], double* const Z[3], int n, double eps,
                       int keep, int rank_cap, TruncStats* stats) {
  cudaStream_t st = stream_of(c);
  int mc = 0;
  for (int l = 1; l < 3; ++l)
    if (r[l] < r[mc]) mc = l;                       // ties -> lowest mode
  int ma = (mc == 0) ? 1 : 0, mb = (mc == 2) ? 1 : 2;
  const int ra = r[ma], rb = r[mb], rc = r[mc];
  const int k = std::min(ra, rb);
  require(std::max(ra, rb) <= kSliceMax, FC_ERR_CAPACITY, "Tucker rank above the T2C slice limit (1024)");
  const int K = rc * k;
  Scratch s(st);
  double* S = s.alloc<double>((size_t)ra * rb * rc);
  double* sv = s.alloc<double>((size_t)K);
  double* Ua = s.alloc<double>((size_t)rc * ra * k);
  double* Vb = s.alloc<double>((size_t)rc * rb * k);
  double* s2s = s.alloc<double>((size_t)K);
  int* keys = s.alloc<int>((size_t)K);
  double* energy = s.alloc<double>(2);
  int* rdev = s.alloc<int>(2);
  PhaseMarks pm(st);
  extract_slices_kernel<<<blocks_for((long long)ra * rb * rc), 256, 0, st>>>(core, r[0], r[1], r[2], ma, mb, mc, S);
  FC_CHECK_LAUNCH();
  small_svd(st, ra, rb, rc, S, sv, Ua, Vb);
  pm.mark("7 T2C slice SVDs");
  pool_rank_kernel<<<cdiv(K, 256), 256, 0, st>>>(K, sv, s2s, keys);
  FC_CHECK_LAUNCH();
  pool_energy_kernel<<<1, 1024, 0, st>>>(K, sv, energy);
  FC_CHECK_LAUNCH();
  int R;
  if (keep > 0) {
    R = std::min(keep, K);
  } else {
    rank_cut_device(K, s2s, 0.25 * eps * eps, energy, rdev, energy + 1, st);
    R = read_int(rdev, st);
  }
  pm.mark("8 T2C pooled cut");
  if (stats) {
    stats->t2c_mode = mc;
    stats->out_rank = R;
  }
  if (rank_cap > 0 && R > rank_cap) {   // clip to the top rank_cap triples (a prefix of the pooled order)
    R = rank_cap;
    if (stats) {
      stats->clipped = true;
      stats->out_rank = R;
    }
  }
  TT out;
  out.n = n;
  out.R = R;
  out.q[0] = r[0]; out.q[1] = r[1]; out.q[2] = r[2];
  const size_t csz = (size_t)r[0] * r[1] * r[2];
  size_t need = (size_t)R + (size_t)R * (r[0] + r[1] + r[2]) + (size_t)n * (r[0] + r[1] + r[2]) + csz;
  out.mem.emplace_back(need * 8, st);
  double* base = out.mem.back().d();
  out.w = base;
  out.core = base + need - csz;
  double* p = base + R;
  for (int l = 0; l < 3; ++l) {
    out.C[l] = p;
    p += (size_t)R * r[l];
  }
  for (int l = 0; l < 3; ++l) {
    out.Q[l] = p;
    p += (size_t)n * r[l];
    FC_CUDA_TRY(cudaMemcpyAsync(out.Q[l], Z[l], (size_t)n * r[l] * 8, cudaMemcpyDeviceToDevice, st));
    out.orth[l] = true;
  }
  if (R > 0) {
    t2c_scatter_kernel<<<R, 64, 0, st>>>(R, k, ra, rb, rc, keys, s2s, Ua, Vb, out.w, out.C[ma], out.C[mb], out.C[mc]);
    FC_CHECK_LAUNCH();
    // Tucker core of the output (kept triples of each slice are a prefix of that slice)
    int* cnt = s.zeros<int>(rc);
    slice_counts_kernel<<<cdiv(R, 256), 256, 0, st>>>(R, k, keys, cnt);
    FC_CHECK_LAUNCH();
    t2c_core_kernel<<<blocks_for((long long)ra * rb * rc), 256, 0, st>>>(ra, rb, rc, k, cnt, sv, Ua, Vb, ma, mb, mc,
                                                                         r[0], r[1], out.core);
    FC_CHECK_LAUNCH();
  } else {
    FC_CUDA_TRY(cudaMemsetAsync(out.core, 0, csz * 8, st));
  }
  return out;
}

void tt_compute_core(cudaStream_t st, TT& x) {
  const size_t csz = (size_t)x.q[0] * x.q[1] * x.q[2];
  x.mem.emplace_back(std::max<size_t>(csz, 1) * 8, st);
  x.core = x.mem.back().d();
  FC_CUDA_TRY(cudaMemsetAsync(x.core, 0, std::max<size_t>(csz, 1) * 8, st));
  if (x.R == 0 || csz == 0) return;
  const size_t r12 = (size_t)x.q[0] * x.q[1];
  // chunk the terms so that the Khatri-Rao operand stays below ~128M doubles
  const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)x.R, (size_t)(1 << 27) / std::max<size_t>(r12, 1)));
  Scratch s(st);
  double* KR = s.alloc<double>(r12 * chunk);
  for (int t0 = 0; t0 < x.R; t0 += chunk) {
    const int m = std::min(chunk, x.R - t0);
    kr12_kernel<<<blocks_for((long long)r12 * m), 256, 0, st>>>(x.q[0], x.q[1], m, x.w + t0, x.C[0] + (size_t)t0 * x.q[0],
                                                                 x.C[1] + (size_t)t0 * x.q[1], KR);
    FC_CHECK_LAUNCH();
    // r3 in (64, 128]: k-step-balanced 128 x 128 tiles (stream-K, gemm.cu); else split-K 64 x 64 tiles
    GemmArgs gk;
    gk.transB = 1;
    gk.beta = 1.0;
    gk.nbatch = 1;
    gk.b[0] = GemmBatch{(int)r12, x.q[2], m, KR, (int)r12, x.C[2] + (size_t)t0 * x.q[2], x.q[2], x.core, (int)r12,
                        nullptr, 0, nullptr};
    gk.splitk = std::max(1, std::min(cdiv(m, 64), 8));
    gk.streamk = 1;
    gemm(gk, st);
  }
}

// Basis tolerance of the rank-revealing orthonormalisation (relative to the largest column of
// K).  A dropped residual moves a side-matrix singular value near the cut by at most
// ~2 kBasisTol ||A|| sigma_cut, i.e. <= 4e-4 of the threshold (eps/2)^2 ||A||^2 at eps = 1e-6,
// well inside the A23 noise band; it shrinks the eigenproblem (and its N^3 cost) notably.
constexpr double kBasisTol = 1e-10;
// ... of the weighted Khatri-Rao basis (structured route): there the dropped residuals are not
// incidental (most columns far below the level) but sit at the level itself, ~sqrt(#columns) tol
// of the side matrix in total (measured 1.05e-8 of the result at tol = 1e-10, 1377 columns), so
// the level is set two decades lower to keep the result within the single-truncation parity
// tolerance max(1e-10, 10 eps_mach / eps): min(1e-12, 1e-6 eps).  Measured on a C4 iterate at
// n = 1024 (profiles/r02pp_wbasis_tol.txt): the result moves by ~80 tol at eps = 1e-6 and ~480 tol
// at eps = 1e-8; C4 time-to-eps 225 / 230 / 234 / 238 ms at tol = 1e-10 / 1e-11 / 1e-12 / 1e-13
// against 278 ms with the unweighted basis.  (FC_WBASIS_TOL overrides; diagnostics)
constexpr double kWBasisTol = 1e-12;
constexpr double kWBasisTolPerEps = 1e-6;
// Gram eigenvalue noise per direction, in units of eps_mach * lam_max (refined cut below it)
constexpr double kNoise = 1.0;
// K13: below this eps the CP route takes the SVD of the side matrix itself (FC_TRUNC_QR=0/1)
constexpr double kQrEps = 1e-6;
constexpr double kQrBasisTol = 1e-14;

// spectral terms per chunk of the structured norm / Gram pass: t x (Rx * chunk) <= 2^27 doubles
constexpr size_t kStructChunk = (size_t)1 << 27;
// split-K target of the side-Gram GEMMs, in waves of 148 SMs (FC_GRAM_WAVES)
int gram_waves() {
  static const int w = getenv("FC_GRAM_WAVES") ? atoi(getenv("FC_GRAM_WAVES")) : 8;   // 8: 312 ms vs 316 ms (3)
  return w;
}

int struct_chunk(const StructuredS* ss) {
  const int tmax = std::max(ss->t[0], std::max(ss->t[1], ss->t[2]));
  const size_t per = (size_t)std::max(tmax, 1) * std::max(ss->Rx, 1);
  return (int)std::max<size_t>(1, std::min<size_t>((size_t)ss->r, kStructChunk / per));
}

TT truncate_tt(fc_ctx c, const TT& xin, double eps, int rank_cap, TruncStats* stats, const StructuredS* ss,
               int als_sweeps) {
  cudaStream_t st = stream_of(c);
  const int n = xin.n, R = xin.R;
  TruncStats local;
  TruncStats& S = stats ? *stats : local;
  S.in_rank = R;
  if (R == 0) {
    TT z;
    z.n = n;
    return z;
  }
  Scratch s(st);
  PhaseMarks pm(st);
  // ---- 1. orthonormal basis per mode: K = Q_l (n x q) -> pivoted MGS -> Qo (n x k), then
  //         the coefficients in that basis Co = (Qo^T K) C.  Rank revealing without forming
  //         K^T K (no squaring): every column of K is kept to 1e-13 of its norm.
  double* Qo[3];
  double* Co[3];
  double* RmE[3] = {nullptr, nullptr, nullptr};
  int q[3];
  require(!ss || (!xin.orth[0] && !xin.orth[1] && !xin.orth[2]), FC_ERR_INVALID_ARG, "structured input basis");
  double* n2[3];
  double* dl[3];
  double* inv[3];
  for (int l = 0; l < 3; ++l) {
    n2[l] = s.alloc<double>(R);
    dl[l] = s.alloc<double>(R);
    inv[l] = s.alloc<double>(R);
  }
  double* xi = s.alloc<double>(R);
  double* energy = s.alloc<double>(4);
  auto term_weights = [&]() {
    const int nbw = std::max(1, std::min(148, cdiv(R, 1024)));
    double* part = s.alloc<double>(nbw);
    term_weights_kernel<<<nbw, 1024, 0, st>>>(R, xin.w, n2[0], n2[1], n2[2], xi, dl[0], dl[1], dl[2], inv[0], inv[1],
                                              inv[2], part);
    FC_CHECK_LAUNCH();
    sum_parts_kernel<<<1, 32, 0, st>>>(nbw, part, energy);
    FC_CHECK_LAUNCH();
  };
  // n2[kk*Rx + j] = cx_j^T Gm_kk cx_j with Gm_kk (t x t) the Gram of spectral term kk's mode basis,
  // P_kk = Gm_kk Cx, chunked over kk so that P stays below kStructChunk doubles per mode
  auto struct_norms = [&](double* const Gm[3]) {
    const int r = ss->r, Rx = ss->Rx, kc = struct_chunk(ss);
    double* P[3];
    for (int l = 0; l < 3; ++l) P[l] = s.alloc<double>((size_t)ss->t[l] * Rx * kc);
    for (int k0 = 0; k0 < r; k0 += kc) {
      const int nk = std::min(kc, r - k0);
      GemmArgs gp;
      gp.nbatch = 3;
      gp.rep = nk;
      StructNormArgs na;
      for (int l = 0; l < 3; ++l) {
        const int t = ss->t[l];
        gp.b[l] = GemmBatch{t, Rx, t, Gm[l] + (size_t)k0 * t * t, t, ss->Cx[l], t, P[l], t, nullptr, 0, nullptr};
        gp.b[l].sA = (long long)t * t;
        gp.b[l].sC = (long long)t * Rx;
        na.Cx[l] = ss->Cx[l]; na.P[l] = P[l]; na.t[l] = t; na.n2[l] = n2[l] + (size_t)k0 * Rx;
      }
      // t in (64, 128]: a stream-K launch per mode (K = t differs between the modes); else one
      // batched launch of 64 x 64 tiles
      static const bool gram_sk = !(getenv("FC_GRAM_STREAMK") && atoi(getenv("FC_GRAM_STREAMK")) == 0);
      const int tmax = std::max(ss->t[0], std::max(ss->t[1], ss->t[2]));
      if (gram_sk && tmax > 64 && tmax <= 128) {
        for (int l = 0; l < 3; ++l) {
          GemmArgs g1 = gp;
          g1.nbatch = 1;
          g1.b[0] = gp.b[l];
          g1.streamk = 1;
          gemm(g1, st);
        }
      } else {
        gemm(gp, st);
      }
      struct_norms_kernel<<<dim3(cdiv(nk * Rx, 8), 3), 256, 0, st>>>(nk * Rx, Rx, na);
      FC_CHECK_LAUNCH();
    }
  };
  // H_kk = W_kk W_kk^T,  W_kk = Cx diag(d_l[kk*Rx + .])   (t x t per spectral term, W chunked over kk)
  double* Hs[3] = {nullptr, nullptr, nullptr};
  auto struct_side_grams = [&]() {
    const int r = ss->r, Rx = ss->Rx, kc = struct_chunk(ss);
    double* W[3];
    for (int l = 0; l < 3; ++l) {
      W[l] = s.alloc<double>((size_t)ss->t[l] * Rx * kc);
      Hs[l] = s.alloc<double>((size_t)ss->t[l] * ss->t[l] * r);
    }
    for (int k0 = 0; k0 < r; k0 += kc) {
      const int nk = std::min(kc, r - k0);
      GemmArgs gh;
      gh.transB = 1;
      gh.nbatch = 3;
      gh.rep = nk;
      for (int l = 0; l < 3; ++l) {
        const int t = ss->t[l];
        struct_scale_kernel<<<blocks_for((long long)t * Rx * nk), 256, 0, st>>>(t, nk * Rx, Rx, ss->Cx[l],
                                                                                 dl[l] + (size_t)k0 * Rx, W[l]);
        FC_CHECK_LAUNCH();
        gh.b[l] = GemmBatch{t, t, Rx, W[l], t, W[l], t, Hs[l] + (size_t)k0 * t * t, t, nullptr, 0, nullptr};
        gh.b[l].sA = gh.b[l].sB = (long long)t * Rx;
        gh.b[l].sC = (long long)t * t;
      }
      static const bool gram_sk = !(getenv("FC_GRAM_STREAMK") && atoi(getenv("FC_GRAM_STREAMK")) == 0);
      gh.streamk = gram_sk;   // as the Gm Grams above
      gemm(gh, st);
    }
  };
  // Weighted Khatri-Rao basis (structured route; FC_BASIS_WEIGHT=0: the unweighted basis): the term
  // norms and the per-term side Grams do not need the orthonormal basis — Gm_kk = K_kk^T K_kk with
  // K_kk = sum_a E[a, kk] K_a (n x t) formed explicitly — so they come first and give every column
  // of K its weight in the side matrix (col_weight_kernel).
  static const bool wbasis_on = !(getenv("FC_BASIS_WEIGHT") && atoi(getenv("FC_BASIS_WEIGHT")) == 0);
  const bool wbasis = ss && wbasis_on;
  static const double wbasis_env = getenv("FC_WBASIS_TOL") ? atof(getenv("FC_WBASIS_TOL")) : 0.0;
  const double wbasis_tol = wbasis_env > 0.0 ? wbasis_env : std::min(kWBasisTol, kWBasisTolPerEps * eps);
  double* wcol[3] = {nullptr, nullptr, nullptr};
  if (wbasis) {
    const int r = ss->r;
    double* Kk[3];
    double* Gm[3];
    GemmArgs gk, gg;
    gk.nbatch = gg.nbatch = 3;
    gg.transA = 1;
    gg.rep = r;
    for (int l = 0; l < 3; ++l) {
      const int t = ss->t[l], sl = ss->s[l];
      require(xin.q[l] == sl * t, FC_ERR_INVALID_ARG, "structured basis shape");
      Kk[l] = s.alloc<double>((size_t)n * t * r);
      Gm[l] = s.alloc<double>((size_t)t * t * r);
      gk.b[l] = GemmBatch{n * t, r, sl, xin.Q[l], n * t, ss->E[l], sl, Kk[l], n * t, nullptr, 0, nullptr};
      gg.b[l] = GemmBatch{t, t, n, Kk[l], n, Kk[l], n, Gm[l], t, nullptr, 0, nullptr};
      gg.b[l].sA = gg.b[l].sB = (long long)n * t;
      gg.b[l].sC = (long long)t * t;
    }
    // t in (64, 128]: one k-step-balanced 128 x 128 tile per term instead of four 64 x 64 tiles,
    // three of them ragged (gemm.cu stream-K; FC_GRAM_STREAMK=0: the 64 x 64 kernel)
    static const bool gram_sk = !(getenv("FC_GRAM_STREAMK") && atoi(getenv("FC_GRAM_STREAMK")) == 0);
    gg.streamk = gram_sk;
    gemm(gk, st);
    gemm(gg, st);
    struct_norms(Gm);
    term_weights();
    struct_side_grams();
    ColWeightArgs cw;
    for (int l = 0; l < 3; ++l) {
      wcol[l] = s.alloc<double>(xin.q[l]);
      cw.E[l] = ss->E[l]; cw.H[l] = Hs[l]; cw.s[l] = ss->s[l]; cw.t[l] = ss->t[l]; cw.wgt[l] = wcol[l];
    }
    col_weight_kernel<<<3, 1024, 0, st>>>(r, cw);
    FC_CHECK_LAUNCH();
    pm.mark("0b column weights (structured)");
  }
  {
    BcgsBatch pb;
    int* kdev = s.alloc<int>(4);
    int map[3];
    for (int l = 0; l < 3; ++l) {
      map[l] = -1;
      if (xin.orth[l]) continue;
      require(xin.q[l] >= 1, FC_ERR_INVALID_ARG, "empty basis");
      double* Kc = s.alloc<double>((size_t)n * xin.q[l]);
      if (wcol[l]) {
        scale_copy_cols_kernel<<<blocks_for((long long)n * xin.q[l]), 256, 0, st>>>(n, xin.q[l], xin.Q[l], wcol[l], Kc);
        FC_CHECK_LAUNCH();
      } else {
        FC_CUDA_TRY(cudaMemcpyAsync(Kc, xin.Q[l], (size_t)n * xin.q[l] * 8, cudaMemcpyDeviceToDevice, st));
      }
      const int kcap = std::min(n, xin.q[l]);
      double* Qn = s.alloc<double>((size_t)n * kcap);
      map[l] = pb.nb;
      pb.e[pb.nb++] = BcgsEntry{n, xin.q[l], Kc, n, Qn, n, kcap, kdev + l, s.alloc<double>(xin.q[l]),
                                s.alloc<double>((size_t)kcap * kBcgsW), wcol[l] ? wbasis_tol : kBasisTol};
      static const bool no_prefix = getenv("FC_NO_ORTH_PREFIX") != nullptr;   // diagnostic
      if (!no_prefix) pb.e[pb.nb - 1].k_base = std::min(xin.orth_prefix[l], kcap);
    }
    bcgs(pb, st);
    int kh[4] = {0, 0, 0, 0};
    if (pb.nb) {
      FC_CUDA_TRY(cudaMemcpyAsync(kh, kdev, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
      FC_CUDA_TRY(cudaStreamSynchronize(st));
    }
    for (int l = 0; l < 3; ++l) {
      if (map[l] < 0) {
        Qo[l] = xin.Q[l];
        Co[l] = xin.C[l];
        q[l] = xin.q[l];
        continue;
      }
      const int k = std::max(kh[l], 1);
      Qo[l] = pb.e[map[l]].Q;
      q[l] = k;
      if (getenv("FC_TRACE")) {   // debugging aid: orthogonality of the device basis
        double* Gq = s.zeros<double>((size_t)k * k);
        dgemm(st, 1, 0, k, k, n, 1.0, Qo[l], n, Qo[l], n, 0.0, Gq, k);
        std::vector<double> h((size_t)k * k);
        FC_CUDA_TRY(cudaMemcpyAsync(h.data(), Gq, h.size() * 8, cudaMemcpyDeviceToHost, st));
        FC_CUDA_TRY(cudaStreamSynchronize(st));
        double dev = 0;
        for (int i = 0; i < k; ++i)
          for (int j = 0; j < k; ++j) dev = std::max(dev, std::fabs(h[i + (size_t)j * k] - (i == j ? 1.0 : 0.0)));
        fprintf(stderr, "[fc trunc] mode %d basis %d of %d orth_err %.2e\n", l, k, xin.q[l], dev);
        static int dumped = 0;
        if (dev > 1e-8 && dumped < 1 && getenv("FC_DUMP")) {
          ++dumped;
          std::vector<double> K((size_t)n * xin.q[l]);
          FC_CUDA_TRY(cudaMemcpy(K.data(), xin.Q[l], K.size() * 8, cudaMemcpyDeviceToHost));
          FILE* f = fopen(getenv("FC_DUMP"), "wb");
          int hdr[2] = {n, xin.q[l]};
          fwrite(hdr, sizeof(int), 2, f);
          fwrite(K.data(), 8, K.size(), f);
          fclose(f);
        }
      }
    }
    // Rm = Qo^T K (k x qin) ; Co = Rm C (k x R): the modes that got a new basis in one batched
    // GEMM each (deterministic split-K: no pre-zeroed C)
    GemmArgs gr, gc;
    gr.transA = 1;
    double* Rm[3] = {nullptr, nullptr, nullptr};
    for (int l = 0; l < 3; ++l) {
      if (map[l] < 0) continue;
      const int k = q[l];
      Rm[l] = s.alloc<double>((size_t)k * xin.q[l]);
      gr.b[gr.nbatch++] = GemmBatch{k, xin.q[l], n, Qo[l], n, xin.Q[l], n, Rm[l], k, nullptr, 0, nullptr};
      if (!ss) {
        Co[l] = s.alloc<double>((size_t)k * R);
        gc.b[gc.nbatch++] = GemmBatch{k, R, xin.q[l], Rm[l], k, xin.C[l], xin.q[l], Co[l], k, nullptr, 0, nullptr};
      } else {
        // structured Hadamard: K columns a*t + b; Rm viewed (k t) x s times E (s x r) gives
        // RmE = [Rm_1 | ... | Rm_r], Rm_kk = sum_a E[a,kk] Rm[:, a*t:(a+1)*t] (k x t);
        // term (kk, j) has coefficient Rm_kk C_x[:, j] (never formed: norms and the side-matrix
        // Gram are contracted through the t x t per-term Grams below)
        const int t = ss->t[l], sl = ss->s[l], r = ss->r;
        Co[l] = nullptr;
        RmE[l] = s.alloc<double>((size_t)k * t * r);
        gc.b[gc.nbatch++] = GemmBatch{k * t, r, sl, Rm[l], k * t, ss->E[l], sl, RmE[l], k * t, nullptr, 0, nullptr};
      }
    }
    if (gr.nbatch) {
      gemm(gr, st);
      gemm(gc, st);
    }
  }
  for (int l = 0; l < 3; ++l) {
    S.basis[l] = q[l];
    require(q[l] >= 1 && q[l] <= 2048, FC_ERR_CAPACITY, "side-matrix basis dimension above 2048");
  }
  pm.mark(ss ? "1 basis (structured)" : "1 basis (cp)");
  // ---- 2. term norms n_l[t] = ||C_l[:, t]|| (orthonormal basis), xi_t, d_l[t] = xi_t/n_l[t] ----
  if (!ss) {
    TermArgs ta;
    for (int l = 0; l < 3; ++l) {
      ta.C[l] = Co[l]; ta.QC[l] = Co[l]; ta.q[l] = q[l]; ta.n2[l] = n2[l];
    }
    term_norms_kernel<<<dim3(cdiv(R, 8), 3), 256, 0, st>>>(R, ta);
    FC_CHECK_LAUNCH();
    term_weights();
  } else if (!wbasis) {
    // Gm_kk = Rm_kk^T Rm_kk (t x t): the term norms through the orthonormal basis
    const int r = ss->r;
    GemmArgs gg;
    gg.transA = 1;
    gg.nbatch = 3;
    gg.rep = r;
    double* Gm[3];
    for (int l = 0; l < 3; ++l) {
      const int t = ss->t[l], k = q[l];
      Gm[l] = s.alloc<double>((size_t)t * t * r);
      gg.b[l] = GemmBatch{t, t, k, RmE[l], k, RmE[l], k, Gm[l], t, nullptr, 0, nullptr};
      gg.b[l].sA = gg.b[l].sB = (long long)k * t;
      gg.b[l].sC = (long long)t * t;
    }
    gemm(gg, st);
    struct_norms(Gm);
    term_weights();
  }
  pm.mark("2 term norms");
  // ---- 3. side matrix in the basis: B_l = C_l D_l (q x R); M_l = B_l B_l^T -------------
  double* Bm[3] = {nullptr, nullptr, nullptr};
  double* M[3];
  const bool sgram_used = ss != nullptr;
  if (ss) {
    // M_l = sum_kk Rm_kk H_kk Rm_kk^T,  H_kk = W_kk W_kk^T,  W_kk = Cx diag(d_l[kk*Rx + .])
    // (t x t per spectral term, W chunked over kk): G_kk = Rm_kk H_kk, then
    // M = [G_1 .. G_r] [Rm_1 .. Rm_r]^T
    const int r = ss->r;
    if (!wbasis) struct_side_grams();
    double* const* H = Hs;
    double* G[3];
    for (int l = 0; l < 3; ++l) G[l] = s.alloc<double>((size_t)q[l] * ss->t[l] * r);
    GemmArgs gq, m;
    m.transB = 1;
    gq.nbatch = m.nbatch = 3;
    gq.rep = r;
    int tiles = 0, minkd = INT32_MAX;
    for (int l = 0; l < 3; ++l) {
      const int t = ss->t[l], k = q[l];
      gq.b[l] = GemmBatch{k, t, t, RmE[l], k, H[l], t, G[l], k, nullptr, 0, nullptr};
      gq.b[l].sA = gq.b[l].sC = (long long)k * t;
      gq.b[l].sB = (long long)t * t;
      M[l] = s.zeros<double>((size_t)k * k);
      m.b[l] = GemmBatch{k, k, t * r, G[l], k, RmE[l], k, M[l], k, nullptr, 0, nullptr};
      tiles += cdiv(k, 64) * cdiv(k, 64);
      minkd = std::min(minkd, t * r);
    }
    gemm(gq, st);
    m.beta = 1.0;
    m.splitk = std::max(1, std::min(cdiv(minkd, 128), std::max(1, cdiv(gram_waves() * 148, std::max(tiles, 1)))));
    gemm(m, st);
  } else {
    for (int l = 0; l < 3; ++l) {
      Bm[l] = s.alloc<double>((size_t)q[l] * R);
      scale_cols_kernel<<<blocks_for((long long)q[l] * R), 256, 0, st>>>(q[l], R, Co[l], dl[l], Bm[l]);
      FC_CHECK_LAUNCH();
    }
    GemmArgs m;
    m.transB = 1;
    m.beta = 1.0;
    m.nbatch = 3;
    int tiles = 0;
    for (int l = 0; l < 3; ++l) {
      M[l] = s.zeros<double>((size_t)q[l] * q[l]);
      m.b[l] = GemmBatch{q[l], q[l], R, Bm[l], q[l], Bm[l], q[l], M[l], q[l], nullptr, 0, nullptr};
      tiles += cdiv(q[l], 64) * cdiv(q[l], 64);
    }
    m.splitk = std::max(1, std::min(cdiv(R, 128), std::max(1, cdiv(gram_waves() * 148, std::max(tiles, 1)))));
    gemm(m, st);
  }
  pm.mark("3 side Gram");
  // ---- 4. eigen of M: s^2 descending, rank cut (tails from the small end), leading vectors ----
  // K13 (eps < kQrEps on the CP route): the SVD of the side matrix B_l itself
  // instead of the eigen-decomposition of B_l B_l^T, so the singular values carry ~eps_mach
  // relative error instead of ~eps_mach * s_max^2 (no squaring floor).  B_l^T (R x q) gets a
  // rank-revealing orthonormal basis Qb (blocked Gram-Schmidt, the QR step), Cb = Qb^T B_l^T
  // (qb x q) its one-sided Jacobi SVD (QR-preconditioned): B_l = Vc S (Qb Uc)^T, so s^2 and the
  // left vectors Vc take the place of the Gram's eigenpairs.  R <= q: the SVD of B_l directly.
  double* lam[3];
  double* Y[3];
  int* rl = s.alloc<int>(4);
  double* margins = s.alloc<double>(3);
  static const int qr_env = getenv("FC_TRUNC_QR") ? atoi(getenv("FC_TRUNC_QR")) : -1;
  bool qr[3] = {false, false, false};
  for (int l = 0; l < 3; ++l) {
    const int ql = q[l];
    lam[l] = s.alloc<double>(ql);
    Y[l] = s.alloc<double>((size_t)ql * ql);
    qr[l] = !ss && ql <= kSliceMax && (qr_env == 1 || (qr_env != 0 && eps < kQrEps)) &&
            (R <= ql || R <= 2048);   // the transposed side matrix stays on the cluster BCGS
  }
  for (int l = 0; l < 3; ++l) {
    if (!qr[l]) continue;
    const int ql = q[l];
    Scratch sq(st);
    FC_CUDA_TRY(cudaMemsetAsync(Y[l], 0, (size_t)ql * ql * 8, st));
    FC_CUDA_TRY(cudaMemsetAsync(lam[l], 0, (size_t)ql * 8, st));
    double* sv;
    int k;
    if (R <= ql) {
      k = R;
      sv = sq.alloc<double>(k);
      double* Vb = sq.alloc<double>((size_t)R * k);
      small_svd(st, ql, R, 1, Bm[l], sv, Y[l], Vb);                   // left vectors straight into Y
    } else {
      double* Bt = sq.alloc<double>((size_t)R * ql);
      transpose_kernel<<<blocks_for((long long)R * ql), 256, 0, st>>>(ql, R, Bm[l], Bt);
      FC_CHECK_LAUNCH();
      double* Bt2 = sq.alloc<double>((size_t)R * ql);
      FC_CUDA_TRY(cudaMemcpyAsync(Bt2, Bt, (size_t)R * ql * 8, cudaMemcpyDeviceToDevice, st));
      BcgsBatch pb;
      int* kd = sq.zeros<int>(1);
      double* Qb = sq.alloc<double>((size_t)R * ql);
      pb.e[pb.nb++] = BcgsEntry{R, ql, Bt2, R, Qb, R, ql, kd, sq.alloc<double>(ql),
                                sq.alloc<double>((size_t)ql * kBcgsW), kQrBasisTol};
      bcgs(pb, st);
      const int qb = std::max(read_int(kd, st), 1);
      double* Cb = sq.zeros<double>((size_t)qb * ql);
      dgemm(st, 1, 0, qb, ql, R, 1.0, Qb, R, Bt, R, 1.0, Cb, qb, std::max(1, std::min(cdiv(R, 256), 16)));
      k = std::min(qb, ql);
      sv = sq.alloc<double>(k);
      double* Uc = sq.alloc<double>((size_t)qb * k);
      small_svd(st, qb, ql, 1, Cb, sv, Uc, Y[l]);                      // B's left vectors = Vc
    }
    square_into_kernel<<<cdiv(k, 256), 256, 0, st>>>(k, sv, lam[l]);
    FC_CHECK_LAUNCH();
  }
  SyevBatch eb;
  int ebmap[3] = {-1, -1, -1};
  int maxq = 0;
  for (int l = 0; l < 3; ++l) {
    if (qr[l]) continue;
    const int ql = q[l];
    ebmap[l] = eb.nb;
    eb.e[eb.nb++] = SyevEntry{ql, M[l], ql, s.alloc<double>(ql), s.alloc<double>(ql), lam[l], Y[l], ql, rl + l,
                              s.alloc<double>((size_t)6 * ql * ql)};
    maxq = std::max(maxq, ql);
  }
  syev_values(eb, st);
  pm.mark("4a eig values (+K13)");
  for (int l = 0; l < 3; ++l) rank_cut_device(q[l], lam[l], 0.25 * eps * eps, energy, rl + l, margins + l, st);
  int r[3];
  double hm[3], lam0[3];
  FC_CUDA_TRY(cudaMemcpyAsync(r, rl, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaMemcpyAsync(hm, margins, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaMemcpyAsync(&S.energy, energy, sizeof(double), cudaMemcpyDeviceToHost, st));
  for (int l = 0; l < 3; ++l) FC_CUDA_TRY(cudaMemcpyAsync(lam0 + l, lam[l], sizeof(double), cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  // Noise-limited cuts (small eps, large bases): the Gram's eigenvalues carry ~eps_mach lam_max
  // each as rounding noise, so when the threshold (eps/2)^2 E is below k * kNoise * eps_mach lam_max
  // the eigenvalue tails cannot decide the cut (reading A11').  Then all eigenvectors
  // are computed; the eigenvalues above the noise level are kept, and the noise subspace Y_ns is
  // re-diagonalised from the data: G_ns = C C^T with C = Y_ns^T B formed explicitly (its rounding
  // is ~eps_mach ||C||^2, ~1e-32 of the energy), its eigenpairs replace the noisy ones.  (Modes on
  // the K13 path have no such floor.)
  bool refine[3] = {false, false, false}, any_refine = false;
  for (int l = 0; l < 3; ++l) {
    refine[l] = !qr[l] && 0.25 * eps * eps * S.energy < kNoise * q[l] * 2.220446049250313e-16 * lam0[l] && q[l] > 1;
    any_refine |= refine[l];
  }
  if (any_refine) {
    int hr[3] = {r[0], r[1], r[2]};
    for (int l = 0; l < 3; ++l)
      if (refine[l]) hr[l] = q[l];
    FC_CUDA_TRY(cudaMemcpyAsync(rl, hr, 3 * sizeof(int), cudaMemcpyHostToDevice, st));
  }
  // refined modes: only the pk eigenvectors above the noise level are computed by inverse iteration
  // (the noise subspace needs just an orthonormal basis: it is re-diagonalised from the data below;
  // FC_REFINE_ALL_VECTORS: inverse iteration for all q vectors, the previous design)
  static const bool refine_all = getenv("FC_REFINE_ALL_VECTORS") != nullptr;
  int pkv[3] = {0, 0, 0};
  for (int l = 0; l < 3; ++l) {
    if (!refine[l]) continue;
    std::vector<double> hl(q[l]);
    FC_CUDA_TRY(cudaMemcpyAsync(hl.data(), lam[l], (size_t)q[l] * 8, cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaStreamSynchronize(st));
    const double noise = kNoise * q[l] * 2.220446049250313e-16 * lam0[l];
    while (pkv[l] < q[l] && hl[pkv[l]] > noise) ++pkv[l];
  }
  if (eb.nb) {
    int hr[3] = {0, 0, 0};
    for (int l = 0; l < 3; ++l)
      if (ebmap[l] >= 0) hr[ebmap[l]] = refine[l] ? (refine_all ? q[l] : std::max(pkv[l], 1)) : r[l];
    if (any_refine) {   // the device-side counts must match
      int hd[3] = {r[0], r[1], r[2]};
      for (int l = 0; l < 3; ++l)
        if (refine[l]) hd[l] = refine_all ? q[l] : std::max(pkv[l], 1);
      FC_CUDA_TRY(cudaMemcpyAsync(rl, hd, 3 * sizeof(int), cudaMemcpyHostToDevice, st));
    }
    syev_vectors(eb, maxq, st, hr);
  }
  if (any_refine) pm.mark("4b1 refine: trusted vectors");
  if (any_refine && !refine_all) {
    // orthonormal basis of the complement of the trusted vectors: blocked Gram-Schmidt of
    // [Y_t | I_q] seeded with the orthonormal Y_t (k_base = pk) -> columns pk..q-1 of Y; the
    // refined modes share one batched Gram-Schmidt
    BcgsBatch cb;
    int* kd = s.zeros<int>(4);
    int cmap[3] = {-1, -1, -1};
    double* Qc[3] = {nullptr, nullptr, nullptr};
    for (int l = 0; l < 3; ++l) {
      if (!refine[l] || pkv[l] >= q[l]) continue;
      const int ql = q[l], pk = pkv[l];
      double* A = s.zeros<double>((size_t)ql * (pk + ql));
      if (pk > 0) FC_CUDA_TRY(cudaMemcpyAsync(A, Y[l], (size_t)ql * pk * 8, cudaMemcpyDeviceToDevice, st));
      eye_kernel<<<blocks_for(ql), 256, 0, st>>>(ql, A + (size_t)ql * pk);
      FC_CHECK_LAUNCH();
      Qc[l] = s.alloc<double>((size_t)ql * ql);
      cmap[l] = cb.nb;
      cb.e[cb.nb++] = BcgsEntry{ql, pk + ql, A, ql, Qc[l], ql, ql, kd + l, s.alloc<double>(pk + ql),
                                s.alloc<double>((size_t)ql * kBcgsW), kBasisTol};
      cb.e[cb.nb - 1].k_base = pk;
    }
    if (cb.nb) {
      bcgs(cb, st);
      int kh[4] = {0, 0, 0, 0};
      FC_CUDA_TRY(cudaMemcpyAsync(kh, kd, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
      FC_CUDA_TRY(cudaStreamSynchronize(st));
      for (int l = 0; l < 3; ++l) {
        if (cmap[l] < 0) continue;
        const int ql = q[l], pk = pkv[l];
        require(kh[l] == ql, FC_ERR_CUDA, "noise-subspace complement basis incomplete");
        FC_CUDA_TRY(cudaMemcpyAsync(Y[l] + (size_t)pk * ql, Qc[l] + (size_t)pk * ql, (size_t)ql * (ql - pk) * 8,
                                    cudaMemcpyDeviceToDevice, st));
      }
    }
    pm.mark("4b2 refine: complement basis");
  }
  if (any_refine) {
    // split: the pk eigenvalues above the noise level are trusted; the noise subspace Y_ns
    // (ql x m) is re-diagonalised from the data: G_ns = C C^T with C = Y_ns^T B computed
    // explicitly (rounding ~ eps_mach ||C||^2, i.e. ~1e-32 of the energy instead of 1e-16).
    // The refined modes' G_ns go through one batched eigensolver.
    SyevBatch gb;
    int gmap[3] = {-1, -1, -1}, mm[3] = {0, 0, 0};
    double* mu[3] = {nullptr, nullptr, nullptr};
    double* Vn[3] = {nullptr, nullptr, nullptr};
    int* rm = s.alloc<int>(4);
    for (int l = 0; l < 3; ++l) {
      if (!refine[l]) continue;
      const int ql = q[l], pk = pkv[l];
      const int m = ql - pk;
      mm[l] = m;
      if (m == 0) {
        rank_cut_device(ql, lam[l], 0.25 * eps * eps, energy, rl + l, margins + l, st);
        continue;
      }
      double* Yns = Y[l] + (size_t)pk * ql;
      double* G = s.zeros<double>((size_t)m * m);
      if (!sgram_used) {
        const size_t chunk = std::max<size_t>(1, ((size_t)1 << 27) / std::max(m, 1));
        double* Cb = s.alloc<double>((size_t)m * std::min<size_t>(chunk, (size_t)R));
        for (size_t c0 = 0; c0 < (size_t)R; c0 += chunk) {
          const int mc = (int)std::min(chunk, (size_t)R - c0);
          dgemm(st, 1, 0, m, mc, ql, 1.0, Yns, ql, Bm[l] + c0 * ql, ql, 0.0, Cb, m);
          dgemm(st, 0, 1, m, m, mc, 1.0, Cb, m, Cb, m, 1.0, G, m);
        }
        pm.mark("4b3 refine: noise Gram (cp)");
      } else {
        // structured: C_kk = (Y_ns^T Rm_kk)(Cx D_kk)
        const int t = ss->t[l], rr = ss->r, Rx = ss->Rx;
        double* YR = s.alloc<double>((size_t)m * t * rr);
        dgemm(st, 1, 0, m, t * rr, ql, 1.0, Yns, ql, RmE[l], ql, 0.0, YR, m);
        pm.mark("4b3 refine: YR = Yns^T RmE");
        static const bool no_factor = getenv("FC_NO_STRUCT_FACTOR") != nullptr;   // diagnostics
        if (t <= kFactorMaxT && !no_factor) {
          // G_ns = sum_kk (YR_kk L_kk)(YR_kk L_kk)^T with L_kk L_kk^T = W_kk W_kk^T (the accurate
          // factor above): an m x (t r) product instead of m x (Rx r) (Rx = x's CP rank)
          double* Lf = s.alloc<double>((size_t)t * t * rr);
          const bool fgl = t > kFactorSmemT;
          double* Hg = fgl ? s.alloc<double>((size_t)2 * t * t * rr) : nullptr;
          const size_t fsmem = ((size_t)t * kFactorJC + 4 * (size_t)t + (fgl ? 0 : 2 * (size_t)t * t)) * 8;
          static bool fattr = false;
          if (!fattr) {
            const size_t fmax = std::max(((size_t)kFactorMaxT * kFactorJC + 4 * (size_t)kFactorMaxT) * 8,
                                         ((size_t)kFactorSmemT * kFactorJC + 4 * (size_t)kFactorSmemT +
                                          2 * (size_t)kFactorSmemT * kFactorSmemT) * 8);
            FC_CUDA_TRY(cudaFuncSetAttribute(struct_factor_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fmax));
            FC_CUDA_TRY(cudaFuncSetAttribute(struct_factor_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fmax));
            FC_CUDA_TRY(cudaFuncSetAttribute(struct_factor_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fmax));
            FC_CUDA_TRY(cudaFuncSetAttribute(struct_factor_kernel<kFactorEnt>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)fmax));
            fattr = true;
          }
          // Gram entries per thread and pass: the smallest of 1, 2, 4, 10 that covers t(t+1)/2 in one
          // pass (the entries are independent accumulation chains; idle slots would cost issue slots)
          const int ne = t * (t + 1) / 2;
          const int ept = cdiv(ne, kFactorThreads);
          // the Gram accumulation split over column chunks (>= 4 staged chunks of W each) so that
          // the r terms fill two waves of the SMs; FC_FACTOR_SPLIT=0: one CTA per term does both
          static const bool fsplit_on = !(getenv("FC_FACTOR_SPLIT") && atoi(getenv("FC_FACTOR_SPLIT")) == 0);
          int S = fsplit_on ? std::min(cdiv(Rx, 4 * kFactorJC), std::max(1, cdiv(2 * 148, rr))) : 1;
          S = (int)std::min<size_t>((size_t)S, std::max<size_t>(1, ((size_t)1 << 25) / ((size_t)rr * 2 * t * t)));   // partials <= 256 MB
          double* Hp = nullptr;
          if (S > 1) {
            const int chunk = cdiv(cdiv(Rx, S), kFactorJC) * kFactorJC;
            S = cdiv(Rx, chunk);
            Hp = s.alloc<double>((size_t)rr * S * 2 * t * t);
            const size_t gsm = (size_t)t * kFactorJC * 8;
            static bool gattr = false;
            if (!gattr) {
              const int gmax = (int)((size_t)kFactorMaxT * kFactorJC * 8);
              FC_CUDA_TRY(cudaFuncSetAttribute(struct_gram_dd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, gmax));
              FC_CUDA_TRY(cudaFuncSetAttribute(struct_gram_dd_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, gmax));
              FC_CUDA_TRY(cudaFuncSetAttribute(struct_gram_dd_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, gmax));
              FC_CUDA_TRY(cudaFuncSetAttribute(struct_gram_dd_kernel<kFactorEnt>, cudaFuncAttributeMaxDynamicSharedMemorySize, gmax));
              gattr = true;
            }
            const dim3 gg(rr, S);
            if (ept <= 1) struct_gram_dd_kernel<1><<<gg, kFactorThreads, gsm, st>>>(t, Rx, chunk, ss->Cx[l], dl[l], Hp);
            else if (ept <= 2) struct_gram_dd_kernel<2><<<gg, kFactorThreads, gsm, st>>>(t, Rx, chunk, ss->Cx[l], dl[l], Hp);
            else if (ept <= 4) struct_gram_dd_kernel<4><<<gg, kFactorThreads, gsm, st>>>(t, Rx, chunk, ss->Cx[l], dl[l], Hp);
            else struct_gram_dd_kernel<kFactorEnt><<<gg, kFactorThreads, gsm, st>>>(t, Rx, chunk, ss->Cx[l], dl[l], Hp);
            FC_CHECK_LAUNCH();
          }
          if (ept <= 1) struct_factor_kernel<1><<<rr, kFactorThreads, fsmem, st>>>(t, Rx, ss->Cx[l], dl[l], Lf, Hg, Hp, S);
          else if (ept <= 2) struct_factor_kernel<2><<<rr, kFactorThreads, fsmem, st>>>(t, Rx, ss->Cx[l], dl[l], Lf, Hg, Hp, S);
          else if (ept <= 4) struct_factor_kernel<4><<<rr, kFactorThreads, fsmem, st>>>(t, Rx, ss->Cx[l], dl[l], Lf, Hg, Hp, S);
          else struct_factor_kernel<kFactorEnt><<<rr, kFactorThreads, fsmem, st>>>(t, Rx, ss->Cx[l], dl[l], Lf, Hg, Hp, S);
          FC_CHECK_LAUNCH();
          pm.mark("4b3 refine: dd factor");
          double* Ct = s.alloc<double>((size_t)m * t * rr);
          GemmArgs g;
          g.nbatch = 1;
          g.rep = rr;
          g.b[0] = GemmBatch{m, t, t, YR, m, Lf, t, Ct, m, nullptr, 0, nullptr};
          g.b[0].sA = (long long)m * t;
          g.b[0].sB = (long long)t * t;
          g.b[0].sC = (long long)m * t;
          gemm(g, st);
          GemmArgs gg;
          gg.transB = 1;
          gg.nbatch = 1;
          gg.beta = 1.0;
          gg.b[0] = GemmBatch{m, m, t * rr, Ct, m, Ct, m, G, m, nullptr, 0, nullptr};
          gg.splitk = waves_splitk(gg, 4);
          gemm(gg, st);
          pm.mark("4b3 refine: C~ C~^T");
        } else {
          const int kc = std::max(1, (int)std::min<size_t>((size_t)rr, ((size_t)1 << 26) /
                                                                     std::max<size_t>((size_t)std::max(m, t) * Rx, 1)));
          double* Wc = s.alloc<double>((size_t)t * Rx * kc);
          double* Cb = s.alloc<double>((size_t)m * Rx * kc);
          for (int k0 = 0; k0 < rr; k0 += kc) {
            const int nk = std::min(kc, rr - k0);
            struct_scale_kernel<<<blocks_for((long long)t * Rx * nk), 256, 0, st>>>(t, nk * Rx, Rx, ss->Cx[l],
                                                                                     dl[l] + (size_t)k0 * Rx, Wc);
            FC_CHECK_LAUNCH();
            GemmArgs g;
            g.nbatch = 1;
            g.rep = nk;
            g.b[0] = GemmBatch{m, Rx, t, YR + (size_t)k0 * m * t, m, Wc, t, Cb, m, nullptr, 0, nullptr};
            g.b[0].sA = (long long)m * t;
            g.b[0].sB = (long long)t * Rx;
            g.b[0].sC = (long long)m * Rx;
            gemm(g, st);
            dgemm(st, 0, 1, m, m, nk * Rx, 1.0, Cb, m, Cb, m, 1.0, G, m);
          }
        }
      }
      mu[l] = s.alloc<double>(m);
      Vn[l] = s.alloc<double>((size_t)m * m);
      gmap[l] = gb.nb;
      gb.e[gb.nb++] = SyevEntry{m, G, m, s.alloc<double>(m), s.alloc<double>(m), mu[l], Vn[l], m, rm + l,
                                s.alloc<double>((size_t)6 * m * m)};
    }
    pm.mark("4b3 refine: noise Gram");
    // eigenvalues of every G_ns (one batch); s2 = [trusted eigenvalues ; mu] and the cut per mode
    int maxm = 0;
    if (gb.nb) {
      syev_values(gb, st);
      for (int l = 0; l < 3; ++l) {
        if (gmap[l] < 0) continue;
        const int ql = q[l], pk = pkv[l];
        maxm = std::max(maxm, mm[l]);
        double* s2r = s.alloc<double>(ql);
        if (pk > 0) FC_CUDA_TRY(cudaMemcpyAsync(s2r, lam[l], (size_t)pk * 8, cudaMemcpyDeviceToDevice, st));
        FC_CUDA_TRY(cudaMemcpyAsync(s2r + pk, mu[l], (size_t)mm[l] * 8, cudaMemcpyDeviceToDevice, st));
        rank_cut_device(ql, s2r, 0.25 * eps * eps, energy, rl + l, margins + l, st);
      }
      // only the (r - pk) leading eigenvectors of each G_ns are computed (one batch), and the
      // noise-subspace vectors rotated: Y_ns[:, :r-pk] <- Y_ns V_ns
      int rc[4] = {0, 0, 0, 0};
      FC_CUDA_TRY(cudaMemcpyAsync(rc, rl, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
      FC_CUDA_TRY(cudaStreamSynchronize(st));
      SyevBatch vb;
      int nvh[kMaxSyev], nvd[4] = {0, 0, 0, 0}, nvl[3] = {0, 0, 0};
      for (int l = 0; l < 3; ++l) {
        if (gmap[l] < 0) continue;
        const int nv = refine_all ? mm[l] : std::max(0, std::min(rc[l], q[l]) - pkv[l]);
        nvl[l] = nv;
        nvd[l] = nv;
        if (nv <= 0) continue;
        nvh[vb.nb] = nv;
        vb.e[vb.nb++] = gb.e[gmap[l]];
      }
      if (vb.nb) {
        FC_CUDA_TRY(cudaMemcpyAsync(rm, nvd, 3 * sizeof(int), cudaMemcpyHostToDevice, st));
        syev_vectors(vb, maxm, st, nvh);
        for (int l = 0; l < 3; ++l) {
          if (nvl[l] <= 0) continue;
          const int ql = q[l], nv = nvl[l], m = mm[l];
          double* Yns = Y[l] + (size_t)pkv[l] * ql;
          double* Yr = s.alloc<double>((size_t)ql * nv);
          dgemm(st, 0, 0, ql, nv, m, 1.0, Yns, ql, Vn[l], m, 0.0, Yr, ql);
          FC_CUDA_TRY(cudaMemcpyAsync(Yns, Yr, (size_t)ql * nv * 8, cudaMemcpyDeviceToDevice, st));
        }
      }
    }
    pm.mark("4b4 refine: noise eig");
    int r_gram[3] = {r[0], r[1], r[2]};
    FC_CUDA_TRY(cudaMemcpyAsync(r, rl, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaMemcpyAsync(hm, margins, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaStreamSynchronize(st));
    S.refined = true;
    if (getenv("FC_TRACE"))
      fprintf(stderr, "[fc trunc] refined cut: modes (%d,%d,%d) gram r=(%d,%d,%d) -> r=(%d,%d,%d) thr/lam0=(%.2e,%.2e,%.2e)\n",
              refine[0], refine[1], refine[2], r_gram[0], r_gram[1], r_gram[2], r[0], r[1], r[2],
              0.25 * eps * eps * S.energy / lam0[0], 0.25 * eps * eps * S.energy / lam0[1],
              0.25 * eps * eps * S.energy / lam0[2]);
  }
  for (int l = 0; l < 3; ++l) {
    S.tucker[l] = r[l];
    S.min_margin = std::min(S.min_margin, hm[l]);
  }
  static const bool trace = getenv("FC_TRACE") != nullptr;
  if (trace)
    fprintf(stderr, "[fc trunc] n=%d terms=%d qin=(%d,%d,%d) basis=(%d,%d,%d) tucker=(%d,%d,%d)\n", n, R, xin.q[0],
            xin.q[1], xin.q[2], q[0], q[1], q[2], r[0], r[1], r[2]);
  if (S.energy == 0.0) {
    TT z;
    z.n = n;
    return z;
  }
  pm.mark("4b cut + eig vectors");
  // ---- 4b. C2T-ALS refinement (oracle/als.py): HOOI sweeps over the modes
  // with the ranks r_l fixed.  In the basis coordinates the CP is x = sum_t xi_t (x)_l Cs_l[:, t]
  // with Cs_l = Co_l diag(1/n_l); for mode l, A_m = Y_m^T Cs_m (m != l) and
  // W_l^T = KR(A_a, A_b) Cs_l^T ((r_a r_b) x q_l; KR weighted by xi, chunked over the terms as the
  // core below); Y_l <- the top r_l eigenvectors of W_l W_l^T (batched syev).  CP route only.
  if (als_sweeps > 0 && !ss) {
    double* Cs[3];
    for (int l = 0; l < 3; ++l) {
      Cs[l] = s.alloc<double>((size_t)q[l] * R);
      scale_cols_kernel<<<blocks_for((long long)q[l] * R), 256, 0, st>>>(q[l], R, Co[l], inv[l], Cs[l]);
      FC_CHECK_LAUNCH();
    }
    for (int sweep = 0; sweep < als_sweeps; ++sweep)
      for (int l = 0; l < 3; ++l) {
        const int a = l == 0 ? 1 : 0, b = l == 2 ? 1 : 2;
        Scratch sa(st);
        double* A[2];
        const int ab[2] = {a, b};
        for (int i = 0; i < 2; ++i) {
          const int m = ab[i];
          A[i] = sa.alloc<double>((size_t)r[m] * R);
          dgemm(st, 1, 0, r[m], R, q[m], 1.0, Y[m], q[m], Cs[m], q[m], 0.0, A[i], r[m]);
        }
        const size_t rab = (size_t)r[a] * r[b];
        require(rab * q[l] <= ((size_t)1 << 28), FC_ERR_CAPACITY, "C2T-ALS: projected unfolding above 2^28 entries");
        double* Wt = sa.zeros<double>(rab * q[l]);
        const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)R, (size_t)(1 << 27) / std::max<size_t>(rab, 1)));
        double* KR = sa.alloc<double>(rab * chunk);
        for (int t0 = 0; t0 < R; t0 += chunk) {
          const int m = std::min(chunk, R - t0);
          kr12_kernel<<<blocks_for((long long)rab * m), 256, 0, st>>>(r[a], r[b], m, xi + t0, A[0] + (size_t)t0 * r[a],
                                                                       A[1] + (size_t)t0 * r[b], KR);
          FC_CHECK_LAUNCH();
          const int tiles = cdiv((long long)rab, 64) * cdiv(q[l], 64);
          dgemm(st, 0, 1, (int)rab, q[l], m, 1.0, KR, (int)rab, Cs[l] + (size_t)t0 * q[l], q[l], 1.0, Wt, (int)rab,
                std::max(1, std::min(cdiv(m, 64), std::max(1, 296 / std::max(tiles, 1)))));
        }
        double* Gw = sa.zeros<double>((size_t)q[l] * q[l]);
        dgemm(st, 1, 0, q[l], q[l], (int)rab, 1.0, Wt, (int)rab, Wt, (int)rab, 1.0, Gw, q[l],
              std::max(1, std::min(cdiv((long long)rab, 256), 16)));
        SyevBatch gb;
        double* mu = sa.alloc<double>(q[l]);
        int* rd = sa.alloc<int>(1);
        FC_CUDA_TRY(cudaMemcpyAsync(rd, &r[l], sizeof(int), cudaMemcpyHostToDevice, st));
        gb.e[gb.nb++] = SyevEntry{q[l], Gw, q[l], sa.alloc<double>(q[l]), sa.alloc<double>(q[l]), mu, Y[l], q[l], rd,
                                  sa.alloc<double>((size_t)6 * q[l] * q[l])};
        syev_values(gb, st);
        syev_vectors(gb, q[l], st, &r[l]);
      }
  }
  // ---- 5. Z_l = Qo_l Y_r -----------------------------------------------------------------
  static const bool tr_orth_y = getenv("FC_TRACE_ORTH_Y") != nullptr;
  if (tr_orth_y)
    for (int l = 0; l < 3; ++l)
      fprintf(stderr, "[fc orthY] %s mode %d q %d r %d refine %d pk %d qr %d: |Qo^T Qo - I| %.2e |Y_r^T Y_r - I| %.2e\n",
              ss ? "struct" : "cp", l, q[l], r[l], (int)refine[l], pkv[l], (int)qr[l], dbg_orth(st, Qo[l], n, q[l], n),
              dbg_orth(st, Y[l], q[l], r[l], q[l]));
  double* Z[3];
  {
    GemmArgs gz;
    gz.nbatch = 3;
    gz.beta = 1.0;
    for (int l = 0; l < 3; ++l) {
      Z[l] = s.zeros<double>((size_t)n * r[l]);
      gz.b[l] = GemmBatch{n, r[l], q[l], Qo[l], n, Y[l], q[l], Z[l], n, nullptr, 0, nullptr};
    }
    gz.splitk = waves_splitk(gz, 8);   // ~100 tiles for 148 SMs: split over the basis dimension
    gemm(gz, st);
  }
  pm.mark("5 Z");
  // ---- 6. core beta = x x_l Z_l^T (r0 x r1 x r2) ---------------------------------------------
  const size_t r12 = (size_t)r[0] * r[1];
  // reading A22: the Tucker stage is run while r1 r2 r3 <= 2^28 (2 GB), else CAPACITY
  require(r12 * r[2] <= ((size_t)1 << 28), FC_ERR_CAPACITY,
          "Tucker core of " + std::to_string(r[0]) + " x " + std::to_string(r[1]) + " x " + std::to_string(r[2]) +
              " above 2^28 entries (A22)");
  double* core = s.zeros<double>(r12 * r[2]);
  if (ss) {
    // Tucker route: beta = sum_kk wF[kk] core_x x_1 H1_kk x_2 H2_kk x_3 H3_kk,
    // H_l,kk = Z_l^T diag(u_l,kk) xhat_l = Y_r^T Rm_kk (r_l x t_l): Hall_l = Y_r^T RmE_l
    double* Hall[3];
    {   // the three modes in one batched launch (split-K over the basis dimension)
      GemmArgs gh;
      gh.transA = 1;
      gh.beta = 1.0;
      gh.nbatch = 3;
      int tiles = 0, minq = INT32_MAX;
      for (int l = 0; l < 3; ++l) {
        Hall[l] = s.zeros<double>((size_t)r[l] * ss->t[l] * ss->r);
        gh.b[l] = GemmBatch{r[l], ss->t[l] * ss->r, q[l], Y[l], q[l], RmE[l], q[l], Hall[l], r[l], nullptr, 0, nullptr};
        tiles += cdiv(r[l], 64) * cdiv((long long)ss->t[l] * ss->r, 64);
        minq = std::min(minq, q[l]);
      }
      gh.splitk = std::max(1, std::min(cdiv(minq, 64), cdiv(gram_waves() * 148, std::max(tiles, 1))));
      gemm(gh, st);
    }
    const int t0 = ss->t[0], t1 = ss->t[1], t2 = ss->t[2], r0 = r[0], r1 = r[1], r2 = r[2];
    const int NB = kMaxBatch;
    double* X1 = s.alloc<double>((size_t)NB * r0 * t1 * t2);
    double* X2 = s.alloc<double>((size_t)NB * r0 * t1 * r2);
    double* X2p = s.alloc<double>((size_t)NB * r0 * t1 * r2);
    double* X3 = s.alloc<double>((size_t)NB * r0 * r1 * r2);
    for (int k0 = 0; k0 < ss->r; k0 += NB) {
      const int nb = std::min(NB, ss->r - k0);
      GemmArgs a, b, d;
      a.nbatch = b.nbatch = d.nbatch = nb;
      b.transB = 1;
      for (int i = 0; i < nb; ++i) {
        const int kk = k0 + i;
        // X1 = H1_kk (r0 x t0) * core_x_(1) (t0 x t1 t2)
        a.b[i] = GemmBatch{r0, t1 * t2, t0, Hall[0] + (size_t)kk * r0 * t0, r0, ss->core_x, t0,
                           X1 + (size_t)i * r0 * t1 * t2, r0, nullptr, 0, nullptr};
        // X2 = X1 ((r0 t1) x t2) * H3_kk^T (t2 x r2)
        b.b[i] = GemmBatch{r0 * t1, r2, t2, X1 + (size_t)i * r0 * t1 * t2, r0 * t1, Hall[2] + (size_t)kk * r2 * t2, r2,
                           X2 + (size_t)i * r0 * t1 * r2, r0 * t1, nullptr, 0, nullptr};
        // X3 = H2_kk (r1 x t1) * X2p (t1 x r0 r2)
        d.b[i] = GemmBatch{r1, r0 * r2, t1, Hall[1] + (size_t)kk * r1 * t1, r1, X2p + (size_t)i * r0 * t1 * r2, t1,
                           X3 + (size_t)i * r0 * r1 * r2, r1, nullptr, 0, nullptr};
      }
      gemm(a, st);
      gemm(b, st);
      permute_xbz_kernel<<<blocks_for((long long)nb * r0 * t1 * r2), 256, 0, st>>>(nb, r0, t1, r2, X2, X2p);
      FC_CHECK_LAUNCH();
      gemm(d, st);
      accumulate_core_kernel<<<blocks_for((long long)r0 * r1 * r2), 256, 0, st>>>(nb, r0, r1, r2, ss->wF, k0, X3,
                                                                                  core);
      FC_CHECK_LAUNCH();
    }
  } else {
    // CP route: beta = sum_t xi_t Chat_1[:,t] (x) Chat_2[:,t] (x) Chat_3[:,t] with the
    // unit-factor coefficients Chat_l = Y_r^T Co_l diag(1/n_l), chunked over the terms
    double* Chat[3];
    GemmArgs gc;
    gc.nbatch = 3;
    gc.transA = 1;
    for (int l = 0; l < 3; ++l) {
      Chat[l] = s.alloc<double>((size_t)r[l] * R);
      gc.b[l] = GemmBatch{r[l], R, q[l], Y[l], q[l], Co[l], q[l], Chat[l], r[l], nullptr, 0, inv[l]};
    }
    gemm(gc, st);
    const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)R, (size_t)(1 << 27) / std::max<size_t>(r12, 1)));
    double* KR = s.alloc<double>(r12 * chunk);
    for (int tt0 = 0; tt0 < R; tt0 += chunk) {
      const int m = std::min(chunk, R - tt0);
      kr12_kernel<<<blocks_for((long long)r12 * m), 256, 0, st>>>(r[0], r[1], m, xi + tt0, Chat[0] + (size_t)tt0 * r[0],
                                                                   Chat[1] + (size_t)tt0 * r[1], KR);
      FC_CHECK_LAUNCH();
      int tiles = cdiv((long long)r12, 64) * cdiv(r[2], 64);
      // split-K sized for ~8 waves of 148 SMs (1-2 waves of 64x64 tiles left a half-empty last wave;
      // C4 solve 311 ms vs 313 ms with 2 or 4 waves)
      static const int core_waves = getenv("FC_CORE_WAVES") ? atoi(getenv("FC_CORE_WAVES")) : 8;
      // (r3 in (64, 128]: the stream-K 128 x 128 kernel instead, one tile column)
      GemmArgs gz;
      gz.transB = 1;
      gz.beta = 1.0;
      gz.nbatch = 1;
      gz.b[0] = GemmBatch{(int)r12, r[2], m, KR, (int)r12, Chat[2] + (size_t)tt0 * r[2], r[2], core, (int)r12,
                          nullptr, 0, nullptr};
      gz.splitk = std::max(1, std::min(cdiv(m, 64), std::max(1, cdiv(core_waves * 148, std::max(tiles, 1)))));
      gz.streamk = 1;
      gemm(gz, st);
    }
  }
  pm.mark(ss ? "6 core (structured)" : "6 core (cp)");
  return tucker_to_canonical(c, core, r, Z, n, eps, 0, rank_cap, &S);
}

TT tt_axpy(cudaStream_t st, const TT& x, double a, const TT& y) {
  TT z;
  z.n = x.n;
  z.R = x.R + y.R;
  size_t need = (size_t)z.R;
  for (int l = 0; l < 3; ++l) {
    z.q[l] = x.q[l] + y.q[l];
    need += (size_t)x.n * z.q[l] + (size_t)z.q[l] * z.R;
  }
  z.mem.emplace_back(need * 8, st);
  double* p = z.mem.back().d();
  z.w = p;
  p += z.R;
  if (x.R) FC_CUDA_TRY(cudaMemcpyAsync(z.w, x.w, (size_t)x.R * 8, cudaMemcpyDeviceToDevice, st));
  if (y.R) scale_copy(y.R, y.w, a, z.w + x.R, st);
  for (int l = 0; l < 3; ++l) {
    z.Q[l] = p;
    p += (size_t)x.n * z.q[l];
    z.C[l] = p;
    p += (size_t)z.q[l] * z.R;
    if (x.q[l]) FC_CUDA_TRY(cudaMemcpyAsync(z.Q[l], x.Q[l], (size_t)x.n * x.q[l] * 8, cudaMemcpyDeviceToDevice, st));
    if (y.q[l])
      FC_CUDA_TRY(cudaMemcpyAsync(z.Q[l] + (size_t)x.n * x.q[l], y.Q[l], (size_t)x.n * y.q[l] * 8,
                                  cudaMemcpyDeviceToDevice, st));
    blockdiag_kernel<<<blocks_for((long long)z.q[l] * z.R), 256, 0, st>>>(x.q[l], x.R, x.C[l], y.q[l], y.R, y.C[l],
                                                                            z.C[l]);
    FC_CHECK_LAUNCH();
    z.orth[l] = (x.R == 0 && y.orth[l]) || (y.R == 0 && x.orth[l]);
    z.orth_prefix[l] = x.orth[l] ? x.q[l] : x.orth_prefix[l];
  }
  return z;
}

double tt_dot(fc_ctx c, const TT& x, const TT& y) {
  if (x.R == 0 || y.R == 0) return 0.0;
  cudaStream_t st = stream_of(c);
  PhaseMarks pm(st);
  struct MarkAtExit {
    PhaseMarks& p;
    ~MarkAtExit() { p.mark("dot"); }
  } mark_at_exit{pm};
  Scratch s(st);
  static const bool no_core_dot = getenv("FC_NO_CORE_DOT") != nullptr;   // diagnostic
  if (x.core && y.core && !no_core_dot) {
    // both carry their Tucker cores (x = core_x x_l Q_x,l): <x, y> = <core_x, core_y x_l G_l>,
    // G_l = Q_x,l^T Q_y,l — r^3-sized contractions instead of the R_x x R_y term Hadamard
    const int* a = x.q;
    const int* b = y.q;
    double* G[3];
    GemmArgs gg;
    gg.transA = 1;
    gg.beta = 1.0;
    gg.nbatch = 3;
    int tiles = 0;
    for (int l = 0; l < 3; ++l) {
      G[l] = s.zeros<double>((size_t)a[l] * b[l]);
      gg.b[l] = GemmBatch{a[l], b[l], x.n, x.Q[l], x.n, y.Q[l], y.n, G[l], a[l], nullptr, 0, nullptr};
      tiles += cdiv(a[l], 64) * cdiv(b[l], 64);
    }
    gg.splitk = std::max(1, std::min(cdiv(x.n, 64), cdiv(2 * 148, std::max(tiles, 1))));
    gemm(gg, st);
    // T1 = G0 core_y(1)  (a0 x b1 b2);  T2 = T1 (a0 b1 x b2) G2^T  (a0 b1 x a2);
    // T3[:, :, k] = T2[:, :, k] (a0 x b1) G1^T  (a0 x a1), k < a2
    double* T1 = s.alloc<double>((size_t)a[0] * b[1] * b[2]);
    dgemm(st, 0, 0, a[0], b[1] * b[2], b[0], 1.0, G[0], a[0], y.core, b[0], 0.0, T1, a[0]);
    double* T2 = s.alloc<double>((size_t)a[0] * b[1] * a[2]);
    dgemm(st, 0, 1, a[0] * b[1], a[2], b[2], 1.0, T1, a[0] * b[1], G[2], a[2], 0.0, T2, a[0] * b[1]);
    double* T3 = s.alloc<double>((size_t)a[0] * a[1] * a[2]);
    GemmArgs g3;
    g3.transB = 1;
    g3.nbatch = 1;
    g3.rep = a[2];
    g3.b[0] = GemmBatch{a[0], a[1], b[1], T2, a[0], G[1], a[1], T3, a[0], nullptr, 0, nullptr};
    g3.b[0].sA = (long long)a[0] * b[1];
    g3.b[0].sC = (long long)a[0] * a[1];
    gemm(g3, st);
    const long long tot = (long long)a[0] * a[1] * a[2];
    constexpr int NB = 148;
    double* part = s.alloc<double>(NB + 1);
    core_dot_kernel<<<NB, 256, 0, st>>>(tot, x.core, T3, part);
    FC_CHECK_LAUNCH();
    core_dot_final_kernel<<<1, 32, 0, st>>>(NB, part, part + NB);
    FC_CHECK_LAUNCH();
    double h = 0;
    FC_CUDA_TRY(cudaMemcpyAsync(&h, part + NB, sizeof(double), cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaStreamSynchronize(st));
    return h;
  }
  double* H = s.alloc<double>((size_t)3 * x.R * y.R + 1);
  for (int l = 0; l < 3; ++l) {
    // G = Q_x^T Q_y (qx x qy), T = G C_y (qx x Ry), H_l = C_x^T T (Rx x Ry)
    double* G = s.zeros<double>((size_t)x.q[l] * y.q[l]);
    dgemm(st, 1, 0, x.q[l], y.q[l], x.n, 1.0, x.Q[l], x.n, y.Q[l], y.n, 1.0, G, x.q[l],
          std::max(1, std::min(cdiv(x.n, 256), 16)));
    double* T = s.alloc<double>((size_t)x.q[l] * y.R);
    dgemm(st, 0, 0, x.q[l], y.R, y.q[l], 1.0, G, x.q[l], y.C[l], y.q[l], 0.0, T, x.q[l]);
    dgemm(st, 1, 0, x.R, y.R, x.q[l], 1.0, x.C[l], x.q[l], T, x.q[l], 0.0, H + (size_t)l * x.R * y.R, x.R);
  }
  const double* Hp[3] = {H, H + (size_t)x.R * y.R, H + (size_t)2 * x.R * y.R};
  double* out = H + (size_t)3 * x.R * y.R;
  dot_reduce(x.R, y.R, x.w, y.w, Hp, x.R, out, st);
  double h = 0;
  FC_CUDA_TRY(cudaMemcpyAsync(&h, out, sizeof(double), cudaMemcpyDeviceToHost, st));
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  return h;
}

void tt_expand(cudaStream_t st, const TT& x, double* const U[3], const int ld[3], double* w) {
  if (x.R == 0) return;
  for (int l = 0; l < 3; ++l) dgemm(st, 0, 0, x.n, x.R, x.q[l], 1.0, x.Q[l], x.n, x.C[l], x.q[l], 0.0, U[l], ld[l]);
  FC_CUDA_TRY(cudaMemcpyAsync(w, x.w, (size_t)x.R * 8, cudaMemcpyDeviceToDevice, st));
}

TT tt_from_cp(cudaStream_t st, int n, int R, const double* w, double* const U[3], const int ld[3]) {
  TT x;
  x.n = n;
  x.R = R;
  if (R == 0) return x;
  const bool wide = R > n;   // basis = I_n, coefficients = U
  size_t need = (size_t)R;
  for (int l = 0; l < 3; ++l) need += wide ? (size_t)n * n + (size_t)n * R : (size_t)n * R + (size_t)R * R;
  x.mem.emplace_back(need * 8, st);
  double* p = x.mem.back().d();
  x.w = p;
  p += R;
  FC_CUDA_TRY(cudaMemcpyAsync(x.w, w, (size_t)R * 8, cudaMemcpyDeviceToDevice, st));
  for (int l = 0; l < 3; ++l) {
    x.Q[l] = p;
    if (wide) {
      x.q[l] = n;
      identity_kernel<<<blocks_for((long long)n * n), 256, 0, st>>>(n, x.Q[l]);
      FC_CHECK_LAUNCH();
      p += (size_t)n * n;
      x.C[l] = p;
      FC_CUDA_TRY(cudaMemcpy2DAsync(x.C[l], (size_t)n * 8, U[l], (size_t)ld[l] * 8, (size_t)n * 8, R,
                                    cudaMemcpyDeviceToDevice, st));
      p += (size_t)n * R;
      x.orth[l] = true;
    } else {
      x.q[l] = R;
      FC_CUDA_TRY(cudaMemcpy2DAsync(x.Q[l], (size_t)n * 8, U[l], (size_t)ld[l] * 8, (size_t)n * 8, R,
                                    cudaMemcpyDeviceToDevice, st));
      p += (size_t)n * R;
      x.C[l] = p;
      identity_kernel<<<blocks_for((long long)R * R), 256, 0, st>>>(R, x.C[l]);
      FC_CHECK_LAUNCH();
      p += (size_t)R * R;
      x.orth[l] = false;
    }
  }
  return x;
}

TT tt_copy(cudaStream_t st, const TT& x) {
  TT y;
  y.n = x.n;
  y.R = x.R;
  size_t need = (size_t)x.R;
  for (int l = 0; l < 3; ++l) need += (size_t)x.n * x.q[l] + (size_t)x.q[l] * x.R;
  y.mem.emplace_back(need * 8, st);
  double* p = y.mem.back().d();
  y.w = p;
  p += x.R;
  if (x.R) FC_CUDA_TRY(cudaMemcpyAsync(y.w, x.w, (size_t)x.R * 8, cudaMemcpyDeviceToDevice, st));
  for (int l = 0; l < 3; ++l) {
    y.q[l] = x.q[l];
    y.orth[l] = x.orth[l];
    y.orth_prefix[l] = x.orth_prefix[l];
    y.Q[l] = p;
    p += (size_t)x.n * x.q[l];
    y.C[l] = p;
    p += (size_t)x.q[l] * x.R;
    if (x.q[l]) FC_CUDA_TRY(cudaMemcpyAsync(y.Q[l], x.Q[l], (size_t)x.n * x.q[l] * 8, cudaMemcpyDeviceToDevice, st));
    if (x.q[l] && x.R)
      FC_CUDA_TRY(cudaMemcpyAsync(y.C[l], x.C[l], (size_t)x.q[l] * x.R * 8, cudaMemcpyDeviceToDevice, st));
  }
  if (x.core) {
    const size_t csz = (size_t)x.q[0] * x.q[1] * x.q[2];
    y.mem.emplace_back(std::max<size_t>(csz, 1) * 8, st);
    y.core = y.mem.back().d();
    FC_CUDA_TRY(cudaMemcpyAsync(y.core, x.core, csz * 8, cudaMemcpyDeviceToDevice, st));
  }
  return y;
}

}  // namespace fc
