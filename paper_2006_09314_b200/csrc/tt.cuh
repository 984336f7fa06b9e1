// Mixed Tucker-canonical tensors [P:1804-1812] used inside the solver:
//   x = sum_t w_t (Q_1 C_1[:,t]) (x) (Q_2 C_2[:,t]) (x) (Q_3 C_3[:,t])
// Q_l: n x q_l (orthonormal when orth[l]); C_l: q_l x R (column-major, ld = q_l); w: R.
// A plain CP is the special case Q_l = U_l, C_l = I (or Q_l = I_n, C_l = U_l).  T2C outputs
// have Q_l = Z_l orthonormal and unit coefficient columns (an orthogonal CP).
#pragma once
#include <utility>
#include "ctx.cuh"

namespace fc {

struct DevMem {               // move-only stream-ordered allocation
  void* p = nullptr;
  cudaStream_t st = nullptr;
  DevMem() = default;
  DevMem(size_t bytes, cudaStream_t s) : st(s) {
    if (bytes == 0) bytes = 16;
    p = dev_alloc((bytes + 255) & ~size_t(255), s);
  }
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  DevMem(DevMem&& o) noexcept : p(o.p), st(o.st) { o.p = nullptr; }
  DevMem& operator=(DevMem&& o) noexcept {
    if (this != &o) {
      reset();
      p = o.p; st = o.st; o.p = nullptr;
    }
    return *this;
  }
  void reset() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
  }
  ~DevMem() { reset(); }
  double* d() const { return (double*)p; }
};

struct TT {
  int n = 0, R = 0;
  int q[3] = {0, 0, 0};
  double* Q[3] = {nullptr, nullptr, nullptr};
  double* C[3] = {nullptr, nullptr, nullptr};
  double* w = nullptr;
  bool orth[3] = {false, false, false};
  // the first orth_prefix[l] columns of Q_l are orthonormal (the x part of x + a*y when x is a
  // truncation output): the basis stage seeds its Gram-Schmidt with them
  int orth_prefix[3] = {0, 0, 0};
  double* core = nullptr;     // optional Tucker core q0 x q1 x q2 (x = core x_l Q_l), column-major
  std::vector<DevMem> mem;    // owned storage (may be empty for views)
};

// Structured input of the Hadamard truncation S = F (.) x in eigen coordinates (pcg.cu): the
// basis is K_l = [w_a (.) xhat_b], the coefficient of term (k, j) is E_l[:, k] (x) C_l[:, j];
// neither kron(E, C) nor the KR core operand is ever formed.
struct StructuredS {
  int s[3], t[3];             // spectral basis size, x basis size per mode (q_l = s_l t_l)
  int r, Rx;                  // spectral rank, x rank (terms = r * Rx, order k*Rx + j)
  const double* E[3];         // s_l x r
  const double* Cx[3];        // t_l x Rx
  const double* wF;           // r
  const double* core_x;       // t0 x t1 x t2 (x's Tucker core in its basis)
};

// FC_PHASES diagnostics: CUDA events at phase boundaries, elapsed time accumulated per phase
struct PhaseMarks {
  cudaStream_t st;
  bool on = false;
  std::vector<std::pair<const char*, cudaEvent_t>> m;
  explicit PhaseMarks(cudaStream_t s);
  void mark(const char* name);
  ~PhaseMarks();
};

struct TruncStats {
  int tucker[3] = {0, 0, 0};
  int basis[3] = {0, 0, 0};
  int in_rank = 0, out_rank = 0, t2c_mode = 0;
  double energy = 0.0, min_margin = 1e300;
  bool refined = false;   // a noise-limited cut was decided from data-based tails (A11')
  bool clipped = false;   // the T2C output was clipped to the rank cap (FC_RANK_CAP_HIT)
};

// RHOSVD -> core -> T2C (S11-S13).  Output: orthonormal Q (n x r_l), orthogonal CP terms.
// rank_cap > 0: output rank limit: the T2C keeps its top rank_cap triples (pooled order) and
// sets stats.clipped (pcg_solve then returns FC_RANK_CAP_HIT).
// als_sweeps > 0: C2T-ALS refinement (HOOI sweeps with the RHOSVD ranks) before the core (CP route).
TT truncate_tt(fc_ctx c, const TT& x, double eps, int rank_cap, TruncStats* stats,
               const StructuredS* ss = nullptr, int als_sweeps = 0);
// Tucker core of a TT from its CP coefficients (sum_t w_t (x)_l C_l[:, t]), chunked over terms
void tt_compute_core(cudaStream_t st, TT& x);
// T2C of a dense core (r1 x r2 x r3, column-major) with bases Z (n x r_l, orthonormal):
// eps-cut (keep <= 0) or top-`keep` triples.  Used by the truncation and the spectral CP.
TT tucker_to_canonical(fc_ctx c, const double* core, const int r[3], double* const Z[3], int n, double eps,
                       int keep, int rank_cap, TruncStats* stats);
// batched SVD of ns column-major ra x rb matrices (max(ra, rb) <= 1024): k = min(ra, rb) triples
// per matrix sorted by s descending: s[nu*k + m], Ua[nu*ra*k + m*ra + x], Vb[nu*rb*k + m*rb + y]
void small_svd(cudaStream_t st, int ra, int rb, int ns, const double* S, double* sv, double* Ua, double* Vb);
// x + a*y (concatenation; bases concatenated, coefficients block-diagonal)
TT tt_axpy(cudaStream_t st, const TT& x, double a, const TT& y);
// <x, y>  (result in device scalar `out`, and returned on the host when sync)
double tt_dot(fc_ctx c, const TT& x, const TT& y);
// expand to plain CP factors U_l = Q_l C_l into dst (n x R, ld) and weights
void tt_expand(cudaStream_t st, const TT& x, double* const U[3], const int ld[3], double* w);
// view of a plain CP as TT (Q_l = U_l, C_l = I_R)
TT tt_from_cp(cudaStream_t st, int n, int R, const double* w, double* const U[3], const int ld[3]);
// copy
TT tt_copy(cudaStream_t st, const TT& x);

}  // namespace fc
