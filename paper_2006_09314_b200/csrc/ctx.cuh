// Library context (opaque behind fc_ctx in the ABI).
#pragma once
#include "common.cuh"

struct SpecCP {
  int r = 0;          // CP rank
  fc::DBuf w;         // [r]
  fc::DBuf U;         // 3 blocks, mode l at U.p + l*n*r, column-major n x r, unit columns
  // reduced (mixed Tucker-canonical) form U_l = W_l E_l, W_l orthonormal n x s_l [P:1804-1812]
  int s[3] = {0, 0, 0};
  fc::DBuf W;         // 3 blocks of n x s_l at W.p + l*n*smax
  fc::DBuf E;         // 3 blocks of s_l x r at E.p + l*smax*r
  int smax = 0;
  bool valid = false;
  bool has_basis = false;
  int tucker_rank[3] = {0, 0, 0};
  // eigenbasis the CP is diagonal in (3 x n x n, mode-major); nullptr: the context's SL basis V.
  // The case-(A) preconditioner (FC_PRECOND_A) lives in the DST-I basis of the b0-Laplacian.
  const double* basis = nullptr;
  double* Ul(int n, int l) const { return U.p + (size_t)l * n * r; }
};

// 2D variant: low-rank factorisation D2 ~ sum_k w_k a_k b_k^T of
// D2[i, j] = f(lam1_i + lam2_j) over the context's mode-0 / mode-1 eigenvalues
struct Spec2 {
  int r = 0;
  fc::DBuf w;         // [r]
  fc::DBuf U;         // 2 blocks n x r (mode l at U.p + l*n*r), unit columns
  bool valid = false;
  double* Ul(int n, int l) const { return U.p + (size_t)l * n * r; }
};

struct fc_ctx_s {
  cudaStream_t st = nullptr;
  cudaStream_t st2 = nullptr;   // side stream of pcg_solve (the X update runs concurrently)
  int dev = 0;
  int n = 0;
  fc_params p{};
  bool have_params = false;
  fc::DBuf lam;       // 3 x n
  fc::DBuf V;         // 3 x n x n (mode-major, each column-major)
  bool have_eig[3] = {false, false, false};
  fc::DBuf lamA;      // case-(A) preconditioner: b0-scaled Laplacian eigenvalues, 3 x n
  fc::DBuf VA;        // ... and the DST-I basis, 3 x n x n
  bool have_A[3] = {false, false, false};
  SpecCP spec[4];
  Spec2 spec2[2];     // 2D: FC_F, FC_G
  std::string err;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  double k_flops = 0, k_bytes = 0;
  int k_launches = 0;
  double* lam_l(int l) const { return lam.p + (size_t)l * n; }
  double* V_l(int l) const { return V.p + (size_t)l * n * n; }
  // the eigenbasis a spectral CP is applied in
  const double* Vsp(const SpecCP& sp, int l) const { return sp.basis ? sp.basis + (size_t)l * n * n : V_l(l); }
};

namespace fc {
// stream override of the calling host thread (pcg_solve's side thread truncates X on st2)
extern thread_local cudaStream_t tl_stream;
inline cudaStream_t stream_of(const fc_ctx_s* c) { return tl_stream ? tl_stream : c->st; }
}  // namespace fc
