#pragma once
#include "common.cuh"

namespace fc {

// ---- 1D Sturm-Liouville eigenpairs (S1-S3) -------------------------------------------
// a_mid_dev: 3 x (n+1) midpoint coefficients (device).  Writes lam (3 x n, ascending) and V
// (3 blocks n x n, column-major).  status_dev[0] receives FC_ERR_NONPOS_COEF if needed.
void sl_eigen_device(cudaStream_t st, int n, const double* a_mid_dev, int boundary, double* lam, double* V,
                     int* status_dev);

// ---- batched small symmetric eigensolver (truncation, S11) ----------------------------
// For each batch entry b: A (N x N, column-major, ld lda, overwritten) = Y diag(lam) Y^T.
// Eigenvalues returned descending in lam[0..N).  Eigenvectors for the leading `r` eigenvalues
// are written to Y (N x r, ld ldy), orthonormalised, where r is read from r_dev[0] on the
// device (set by a cut kernel between the phases, see syev_* below).
constexpr int kMaxSyev = 8;
struct SyevEntry {
  int N;
  double* A; int lda;
  double* d; double* e;      // workspace N each
  double* lam;               // N (descending)
  double* Y; int ldy;        // N x (cap) eigenvectors
  int* r;                    // device scalar: number of eigenvectors wanted
  double* scratch;           // 6*N*N doubles of LU + iterate scratch for inverse iteration
};
struct SyevBatch {
  int nb = 0;
  SyevEntry e[kMaxSyev];
};
// phase 1: Householder tridiagonalisation + bisection for all eigenvalues (descending)
void syev_values(const SyevBatch& b, cudaStream_t st);
// phase 2 (after r has been decided on the device): inverse iteration + orthonormalisation +
// back-transformation of the leading r eigenvectors.  r_host (optional): the same ranks known on
// the host, which enables the GEMM-based polar orthonormalisation.
void syev_vectors(const SyevBatch& b, int maxN, cudaStream_t st, const int* r_host = nullptr);

// Column-pivoted modified Gram-Schmidt (rank revealing, no Gram squaring), one CTA per entry:
// A (n x p, overwritten) -> Q (n x k) orthonormal, every column of A within tau*||a_c|| of
// span(Q); k written to *k_out (device).
struct PmgsEntry {
  int n, p;
  double* A; int lda;
  double* Q; int ldq;
  int* k_out;
  double tau;
};
struct PmgsBatch {
  int nb = 0;
  PmgsEntry e[kMaxSyev];
};
void pmgs(const PmgsBatch& b, cudaStream_t st);

// Blocked rank-revealing Gram-Schmidt (multi-CTA): blocks of 32 columns are projected against
// the accepted basis with DMMA GEMMs (twice), then orthogonalised in-block by one CTA; a column
// is accepted when its residual exceeds tau * its original norm.  A (n x p) is overwritten;
// Q (n x kcap) receives the basis, *k (device) its size; P is kcap x 32 scratch, norm0 p.
constexpr int kBcgsW = 128;  // max block width of the blocked Gram-Schmidt (P scratch: kcap x kBcgsW)
struct BcgsEntry {
  int n, p;
  double* A; int lda;
  double* Q; int ldq;
  int kcap;
  int* k;
  double* norm0;
  double* P;
  double tau;
  double* Y = nullptr;   // n x 32 block buffer (allocated by bcgs)
  int* nacc = nullptr;   // accepted count of the current block (allocated by bcgs)
  int k_base = 0;        // the first k_base columns of A are orthonormal: taken into Q as they are
  double* nmax = nullptr; // largest original column norm (set by bcgs: fixed when columns are pruned)
};
struct BcgsBatch {
  int nb = 0;
  int trace = 0;   // FC_TRACE diagnostics (in-block residual histogram)
  BcgsEntry e[kMaxSyev];
};
void bcgs(const BcgsBatch& b, cudaStream_t st);

// CGS2 orthonormalisation of the first *r_dev (<= rmax) columns of Y (N x ., ld ldy).
void orthonormalize_cols(int N, double* Y, int ldy, int* r_dev, int rmax, cudaStream_t st);

// ---- cut kernels -------------------------------------------------------------------------
// RHOSVD/T2C rank rule (reading A11/A23): r = min{ r >= 1 : sum_{k>r} s2_k <= thr }, tails
// summed from the small end, ties kept together.  s2 descending (clamped at 0).  thr =
// factor * (*energy).  Writes r to r_out and the relative cut margin to margin_out.
void rank_cut_device(int count, const double* s2, double factor, const double* energy, int* r_out,
                     double* margin_out, cudaStream_t st);
// basis rank: number of eigenvalues > tau * lam[0] (lam descending)
void basis_rank_device(int count, const double* lam, double tau, int* r_out, cudaStream_t st);

}  // namespace fc
