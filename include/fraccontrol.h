/*
 * fraccontrol.h — C ABI of the B200-native (sm_100a, FP64) rank-truncated PCG for the
 * 3D fractional control equation  (beta * A^alpha + A^-alpha) u = b.
 *
 * Paper: Schmitt, Khoromskij, Khoromskaia, Schulz, arXiv 2006.09314 (PAPER.md, cited
 * [P:line]).  Readings of ambiguous passages are numbered A1..A25 in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Every double* inside fc_cp, and every pointer documented "device", is a DEVICE
 *    pointer allocated by the caller (e.g. with PyTorch).  The library never frees caller
 *    memory; it owns only the context and its workspace.  Pointers documented "host" are
 *    host memory.
 *  - A canonical (CP) tensor  x = sum_{k<rank} w[k] U[0][:,k] (x) U[1][:,k] (x) U[2][:,k]
 *    [P:1706-1712] is stored as fc_cp: factor l is column-major n[l] x cap with leading
 *    dimension ld[l] >= n[l] (column k starts at U[l] + k*ld[l]); weights w[cap].
 *    Columns have unit 2-norm and the weights carry magnitude and sign (reading A18).
 *    rank == 0 is the zero tensor.
 *  - All work is ordered on the context's CUDA stream.  Calls that return host scalars or
 *    reports (cp_dot, pcg_solve, the *_info outputs) synchronise that stream first.
 *  - Return value: FC_OK (0), a warning (> 0) or an error (< 0).  No exception or abort
 *    crosses the ABI; fc_last_error(ctx) describes the last failure.
 *  - Use one context per host thread.
 */
#ifndef FRACCONTROL_H
#define FRACCONTROL_H

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (SPEC error semantics) ------------------------------ */
#define FC_OK                 0
#define FC_NOT_CONVERGED      1   /* pcg_solve hit kmax (warning)                           */
#define FC_RANK_CAP_HIT       2   /* a truncation was clipped at rank_cap (warning)         */
#define FC_ERR_INVALID_ARG   -1   /* n < 2, alpha not in (0,1], beta <= 0, eps <= 0, ...    */
#define FC_ERR_SHAPE         -2   /* mode sizes disagree with the context                   */
#define FC_ERR_CAPACITY      -3   /* output cap too small; *_info->required_rank is set     */
#define FC_ERR_NONPOS_COEF   -4   /* a midpoint coefficient <= 0 or non-finite              */
#define FC_ERR_NOT_SPD       -5   /* <P,S> <= 0 in PCG, or spectral CP of G not positive    */
#define FC_ERR_NAN           -6
#define FC_ERR_EIG_NOCONV    -7
#define FC_ERR_CUDA          -8
#define FC_ERR_NOT_READY     -9   /* sl_setup (or sl_set_eigen + op_set_spectral_cp) missing */

/* spectral functions of A [P:640-648], mapped per reading A5 */
#define FC_F          0   /* F(lam)  = beta*lam^alpha + lam^-alpha   (the operator F_2)     */
#define FC_G          1   /* G(lam)  = 1/F(lam)                      (preconditioner F_3,B)  */
#define FC_POW_PLUS   2   /* lam^alpha                                (F_1)                  */
#define FC_POW_MINUS  3   /* lam^-alpha                               (state y = A^-alpha u) */

#define FC_MAX_ITERS 256

typedef struct fc_ctx_s* fc_ctx;

typedef struct {
    int n[3];        /* mode sizes (all equal to the context's n)                            */
    int rank;        /* number of terms in use                                               */
    int cap;         /* allocated columns (>= rank)                                          */
    double* w;       /* device, [cap]                                                        */
    double* U[3];    /* device, column-major n[l] x cap, leading dimension ld[l]             */
    int ld[3];
} fc_cp;

typedef struct {
    double alpha;        /* fractional order, (0, 1]                            [P:255]    */
    double beta;         /* weight of A^alpha; A^-alpha has weight 1 (A5)        [P:436]    */
    double eps;          /* truncation threshold (relative, A11/A12)             [P:989]    */
    double tol_stop;     /* PCG stop ||R||/||B|| <= tol_stop (A13); <= 0 -> 10*eps         */
    double eps_D;        /* tolerance of the spectral CP of F (A8); <= 0 -> eps            */
    int kmax;            /* max PCG iterations (A17); <= 0 -> 100                           */
    int precond_rank;    /* rank r_G of the preconditioner CP (A7); <= 0 -> 6    [P:990]    */
    int op_rank;         /* > 0: fixed rank of the operator CP (C5 sweep); 0: eps_D-driven  */
    int rank_cap;        /* max CP rank of any iterate: a truncation whose eps-cut keeps more  */
                         /* T2C triples keeps the top rank_cap (warning FC_RANK_CAP_HIT);    */
                         /* <= 0 -> 2^20 (no cap)                                            */
    int boundary;        /* 0: paper boundary rule [P:517-518] (A2); 1: standard            */
    int precond_case;    /* FC_PRECOND_B (0, default, A6) or FC_PRECOND_A (1)   [P:758-868] */
} fc_params;

/* preconditioner cases [P:758-768] */
#define FC_PRECOND_B  0   /* direct low-rank G = 1/F(A) in the SL eigenbasis of A (reading A6)    */
#define FC_PRECOND_A  1   /* G = B_0^-1, B_0 = F(B), B the anisotropic Laplacian with constant    */
                          /* b0_l = (max a_l + min a_l)/2 [P:842-849, P:1462-1467], diagonal in   */
                          /* the DST-I basis: lam_k = b0_l 4/h^2 sin^2(k pi h / 2) [P:778-785];    */
                          /* cond(B_0^-1 F(A)) is bounded independently of n (Theorem [P:871-938]) */

typedef struct {
    int tucker_rank[3];  /* RHOSVD ranks r_l                                                */
    int out_rank;        /* canonical rank after Tucker-to-canonical                       */
    int required_rank;   /* set with FC_ERR_CAPACITY                                        */
    int in_rank;         /* terms after dropping zero terms                                 */
    int basis_dim[3];    /* dimension of the reduced side-matrix basis per mode            */
    int t2c_mode;        /* slicing mode of the T2C step                                    */
    double energy;       /* sum xi^2 of the input                                           */
    double min_cut_margin; /* min over cuts |tail(r) - thr| / thr (A23 noise band log)      */
} fc_trunc_info;

typedef struct {
    int iters;
    int converged;
    int status;
    double rel_res[FC_MAX_ITERS];
    int rank_X[FC_MAX_ITERS], rank_R[FC_MAX_ITERS], rank_Z[FC_MAX_ITERS];
    int rank_P[FC_MAX_ITERS], rank_S[FC_MAX_ITERS];
    int tucker_S[FC_MAX_ITERS];     /* max_l r_l of the S truncation                         */
    double t_iter_ms[FC_MAX_ITERS];
    double t_total_ms;              /* whole pcg_solve (device events)                       */
    double t_loop_ms;               /* loop only: iterations/s = iters / t_loop_ms * 1e3     */
    double normB;
    int cap_hits;                   /* truncations clipped at params.rank_cap (their top      */
                                    /* rank_cap T2C triples kept); > 0 -> FC_RANK_CAP_HIT     */
} fc_pcg_report;

/* ---- context -------------------------------------------------------------------------- */
/* cuda_stream: a cudaStream_t (NULL = legacy default stream).  Binds the current device. */
int fc_create(fc_ctx* ctx, void* cuda_stream);
int fc_destroy(fc_ctx ctx);
const char* fc_last_error(fc_ctx ctx);
int fc_set_stream(fc_ctx ctx, void* cuda_stream);

/* ---- setup: S1..S4 ------------------------------------------------------------------- */
/* sl_setup  [P:443-561, P:688-722]
 *   a_mid: HOST, 3 x (n+1) row-major; a_mid[l*(n+1)+i] = a_l((i+1/2)h), h = 1/(n+1) (A1).
 *   Assembles the three 1D FD operators (A2, A3), computes their eigenpairs on the device
 *   (Sturm bisection on the Golub-Kahan form of the bidiagonal factor + inverse iteration),
 *   then the spectral CPs of F (eps_D-driven, or rank op_rank) and G (rank precond_rank,
 *   raised until positive on the grid: SPD guard A7).  Errors: INVALID_ARG, NONPOS_COEF,
 *   EIG_NOCONV, NOT_SPD, CUDA. */
int sl_setup(fc_ctx ctx, int n, const double* a_mid, const fc_params* p);

/* Eigenpairs of mode l: lam (device, n, ascending) and V (device, n x n column-major,
 * column j = eigenvector j; sign: largest-magnitude entry positive, reading A4). */
int sl_get_eigen(fc_ctx ctx, int mode, double* lam, double* V);
/* Inject eigenpairs (shared-input parity).  Call for all 3 modes; n fixed by the first call
 * (or by sl_setup).  Also stores alpha/beta/eps from p for later op_set_spectral_cp use. */
int sl_set_eigen(fc_ctx ctx, int n, int mode, const double* lam, const double* V, const fc_params* p);

/* Spectral CP of `which` (FC_F, FC_G, ...): D[i,j,k] ~ F(lam1_i + lam2_j + lam3_k) [P:693].
 * get: out->cap must be >= its rank (else CAPACITY, out->rank = required).  set: copies. */
int op_get_spectral_cp(fc_ctx ctx, int which, fc_cp* out);
int op_set_spectral_cp(fc_ctx ctx, int which, const fc_cp* in);
int op_spectral_rank(fc_ctx ctx, int which, int* rank, int* tucker_rank /* [3] or NULL */);
/* Case-(A) preconditioner basis of mode `mode` (FC_PRECOND_A): lam (device, n, ascending
 * b0-scaled Laplacian eigenvalues) and V (device, n x n column-major, the DST-I basis).
 * get: NOT_READY unless sl_setup ran with precond_case = FC_PRECOND_A or a basis was set.
 * set (shared-input parity): copies; once all 3 modes are set the FC_G spectral CP is applied
 * in this basis (its CP must then be built on these lam, op_set_spectral_cp). */
int op_get_precond_basis(fc_ctx ctx, int mode, double* lam, double* V);
/* Sinc-quadrature construction of a spectral CP [P:325-351, P:725-752]:
 * lam^-alpha = 1/Gamma(alpha) int_0^inf t^(alpha-1) e^(-t lam) dt ~ sum_k c_k prod_l e^(-t_k lam_l)
 * (rank 2M+1 = O(|log eps| log(lam_max/lam_min)), positive factors, pointwise relative accuracy
 * ~eps).  which = FC_POW_MINUS (the rule itself, untruncated), FC_POW_PLUS (lam-sum (.)
 * lam^(alpha-1), truncated at eps) or FC_F (beta lam^alpha + lam^-alpha, truncated at eps); the
 * result replaces that spectral CP of the context.  Needs the eigenpairs and alpha, beta
 * (sl_setup, or sl_set_eigen with params).  Errors: NOT_READY, INVALID_ARG, CUDA. */
int op_build_spectral_sinc(fc_ctx ctx, int which, double eps);
int op_set_precond_basis(fc_ctx ctx, int mode, const double* lam, const double* V);

/* ---- the operator: S5..S8 -------------------------------------------------------------- */
/* fracop_apply  [P:597-623]:  y = F(A) x  =  sum_k sum_j (x)_l V_l (u_l^k . V_l^T x_l^j)
 *   Term order t = k*x.rank + j (A19); y.rank = r_which * x.rank, untruncated; y's columns
 *   normalised (norms folded into the weights).  y.cap >= r*x.rank else CAPACITY.
 *   x and y must not alias. */
int fracop_apply(fc_ctx ctx, int which, const fc_cp* x, fc_cp* y);
/* precond_apply = fracop_apply(FC_G)  (case (B) preconditioner [P:956-959], A6). */
int precond_apply(fc_ctx ctx, const fc_cp* x, fc_cp* y);

/* ---- CP algebra: S9, S10 ----------------------------------------------------------------- */
/* cp_dot [P:1748-1755]: *out_host = sum_{k,m} xi_k zeta_m prod_l <u_k^l, v_m^l>. */
int cp_dot(fc_ctx ctx, const fc_cp* x, const fc_cp* y, double* out_host);
/* z = x + a*y by concatenation [x terms ; a*y terms] (ranks add) [P:1845-1866]. */
int cp_axpy(fc_ctx ctx, const fc_cp* x, double a, const fc_cp* y, fc_cp* z);

/* ---- truncation: S11..S13 ---------------------------------------------------------------- */
/* cp_truncate [P:187-190, P:1791-1816]: RHOSVD (C2T) at threshold eps, Tucker core, then
 * Tucker-to-canonical (slice SVD along the min-rank mode).  Output is an orthogonal CP
 * (mutually orthogonal terms).  y.cap too small -> CAPACITY with info->required_rank.
 * info may be NULL.  x and y must not alias. */
int cp_truncate(fc_ctx ctx, const fc_cp* x, double eps, fc_cp* y, fc_trunc_info* info);

/* cp_truncate_als: cp_truncate with the canonical-to-Tucker ALS refinement
 * [P:1060, P:1792-1803] (the algorithm of the cited C2T): after the RHOSVD (ranks r_l by the
 * (eps/2)^2 rule) `sweeps` HOOI sweeps over the modes (ranks fixed) replace each basis Z_l by the
 * leading r_l left singular vectors of the mode-l unfolding of x x_{m != l} Z_m^T, then core and
 * T2C as cp_truncate (reading ALS).  sweeps = 0 is cp_truncate.  Same output / info /
 * CAPACITY rules; the projected unfolding must stay below 2^28 entries (else CAPACITY). */
int cp_truncate_als(fc_ctx ctx, const fc_cp* x, double eps, int sweeps, fc_cp* y, fc_trunc_info* info);

/* fracop_apply_truncate: y = trunc(F(A) x, eps) fused (S5-S13): the
 * Khatri-Rao Hadamard product is formed in the eigenbasis on a reduced basis
 * [w_a (.) V^T q_b] (w_a: basis of the spectral CP's factors, q_b: of x's), the RHOSVD runs
 * on that tensor, and only the surviving Tucker columns are transformed back.  Equal in exact
 * arithmetic to cp_truncate(fracop_apply(x), eps) because each V_l is orthogonal.  This is
 * the operator step pcg_solve uses.  Same output/info/CAPACITY rules as cp_truncate. */
int fracop_apply_truncate(fc_ctx ctx, int which, const fc_cp* x, double eps, fc_cp* y, fc_trunc_info* info);

/* ---- the solver: S14 ------------------------------------------------------------------ */
/* state_recover  [P:287-289, P:969-972]: the state y = beta_paper A^-alpha u of the control problem;
 *   with reading A5 (beta_paper = 1, gamma = beta) y = A^-alpha u, truncated at eps (RHOSVD + T2C,
 *   as cp_truncate; fused apply -> truncate in eigen coordinates).  The spectral CP of lam^-alpha
 *   (FC_POW_MINUS) is built on first use at eps_D (or injected by op_set_spectral_cp).
 *   u, y: caller-owned device CPs (y.cap >= result rank else CAPACITY, info->required_rank set).
 *   Errors: NOT_READY (no sl_setup / params), INVALID_ARG, SHAPE, CAPACITY, CUDA. */
int state_recover(fc_ctx ctx, const fc_cp* u, double eps, fc_cp* y, fc_trunc_info* info);

/* pcg_solve: Algorithm 1 [P:1825-1872] with fun = fracop_apply(FC_F), precond =
 * fracop_apply(FC_G), trunc = cp_truncate(eps); X0 = 0 (A14), R0 = B untruncated (A15).
 * Returns FC_OK; FC_NOT_CONVERGED (kmax reached); FC_RANK_CAP_HIT (converged, but at least one
 * truncation kept only the top p->rank_cap T2C triples: rep->cap_hits counts them; the
 * eps-bound of those truncations does not hold); or an error.  u (device CP, cap >= final
 * rank, else CAPACITY) receives X; rep (host, may be NULL) the per-iteration history. */
int pcg_solve(fc_ctx ctx, const fc_cp* b, const fc_params* p, fc_cp* u, fc_pcg_report* rep);

/* ---- the 2D variant ------------------------------------------------
 * A = T1 (x) I + I (x) T2 [P:449-452 with d = 2]; the same PCG (Algorithm 1, "independent of d"
 * [P:962-969]) with the reduced-SVD truncation the paper uses for d = 2 [P:973-976].
 * A low-rank matrix x = sum_k w[k] U[0][:,k] (x) U[1][:,k], i.e. X = U0 diag(w) U1^T [P:585-595],
 * stored as fc_lr2 with the fc_cp conventions (device pointers, column-major n x cap factors
 * with leading dimension ld, unit columns, signed weights, rank 0 = zero).  The 2D calls use
 * the context's mode-0 and mode-1 eigenpairs and their own spectral factorisations. */
typedef struct {
    int n[2];        /* mode sizes (both equal to the context's n)                              */
    int rank;
    int cap;
    double* w;       /* device, [cap]                                                           */
    double* U[2];    /* device, column-major n[l] x cap, leading dimension ld[l]                */
    int ld[2];
} fc_lr2;

/* sl_setup_2d [P:443-561 with d = 2]: a_mid HOST, 2 x (n+1) row-major midpoint samples of a1, a2
 *   (A1, A2).  Eigenpairs of modes 0 and 1 (as sl_setup), then the low-rank factorisations of
 *   D2[i,j] = F(lam1_i + lam2_j) [P:693 with d = 2]: FC_F by truncated SVD at eps_D (reading 2D-S:
 *   sum of the dropped s^2 <= eps_D^2 ||D2||_F^2) and FC_G = 1/F with rank precond_rank raised
 *   until positive on the grid (A7'/A7'' as in 3D).  Errors: INVALID_ARG, NONPOS_COEF, NOT_SPD,
 *   CAPACITY, CUDA. */
int sl_setup_2d(fc_ctx ctx, int n, const double* a_mid, const fc_params* p);
/* get / set (shared-input parity) the 2D factorisation of `which` (FC_F or FC_G).  get: out->cap
 * must be >= its rank (else CAPACITY with out->rank = required).  set: copies; needs the mode-0/1
 * eigenpairs (sl_setup_2d or sl_set_eigen) and params for alpha, beta. */
int op_get_spectral_2d(fc_ctx ctx, int which, fc_lr2* out);
int op_set_spectral_2d(fc_ctx ctx, int which, const fc_lr2* in);
/* fracop_apply_2d [P:597-611]: y = F(A) x = sum_k sum_j V0(a_k . V0^T x0_j) (x) V1(b_k . V1^T x1_j),
 *   term order t = k*x.rank + j (A19), untruncated (y.rank = r_which * x.rank, else CAPACITY),
 *   columns normalised.  x and y must not alias. */
int fracop_apply_2d(fc_ctx ctx, int which, const fc_lr2* x, fc_lr2* y);
/* cp_dot_2d [P:1748-1755 with d = 2]: *out_host = sum_{k,m} w_k v_m <x0_k, y0_m> <x1_k, y1_m>. */
int cp_dot_2d(fc_ctx ctx, const fc_lr2* x, const fc_lr2* y, double* out_host);
/* cp_truncate_2d [P:973-976]: reduced SVD — orthonormal bases Q_l of span(U_l) (rank-revealing
 *   block Gram-Schmidt), core K = C0 diag(w) C1^T with C_l = Q_l^T U_l, SVD of K, smallest r with
 *   sum_{k>r} s_k^2 <= eps^2 sum s_k^2 (reading 2D-T; ties and zeros as A23), y = (Q0 Uk_r, Q1 Vk_r,
 *   s_r) with orthonormal factors.  out_rank (host, may be NULL) receives r; y.cap < r -> CAPACITY
 *   (out_rank = required).  x and y must not alias; ranks of the bases <= 1024. */
int cp_truncate_2d(fc_ctx ctx, const fc_lr2* x, double eps, fc_lr2* y, int* out_rank);
/* pcg_solve_2d: Algorithm 1 [P:1825-1872] with fun = F (FC_F factorisation), precond = G (FC_G),
 *   trunc = cp_truncate_2d(eps) fused with the apply in eigen coordinates (V_l orthogonal: only the
 *   surviving columns are transformed back); readings A13-A17 as pcg_solve.  Same returns. */
int pcg_solve_2d(fc_ctx ctx, const fc_lr2* b, const fc_params* p, fc_lr2* u, fc_pcg_report* rep);

/* ---- raw kernels exposed for tests/bench (same ABI rules) ------------------------------- */
/* C = alpha*op(A)*op(B) + beta*C, FP64, column-major, DMMA tiles; all pointers device.   */
int fc_dgemm(fc_ctx ctx, int transA, int transB, int M, int N, int K, double alpha,
             const double* A, int lda, const double* B, int ldb, double beta, double* C, int ldc);
/* fc_dgemm with the K range split over `splitk` CTAs per output tile (splitk >= 1; clamped to 8 on
 * the 128x128-tile path and to 64 otherwise).  The partial tiles are summed in a fixed split order
 * (thread-block-cluster DSMEM reduction up to 16 splits, a global workspace above), so the result
 * is bit-identical from run to run for the same arguments; C is not read when beta == 0.
 * splitk < 1 -> FC_ERR_INVALID_ARG. */
int fc_dgemm_splitk(fc_ctx ctx, int transA, int transB, int M, int N, int K, double alpha,
                    const double* A, int lda, const double* B, int ldb, double beta, double* C, int ldc,
                    int splitk);
/* fc_dgemm with the stream-K request the inverse mode transform of fracop_apply makes [P:597-628:
 * Y_l = V_l Yhat_l, the dense contraction of the factored matvec]: when M, N > 64, K >= 64,
 * 2 M N K >= 2^28 and the launch has >= 8 k-steps of 16 per SM, one persistent CTA per SM gets an
 * equal contiguous range of the launch's (128 x 128 tile, k-step) iterations; partial tiles go through a device workspace and are added by the
 * tile's owner CTA in CTA order (bit-identical run to run).  Otherwise identical to fc_dgemm.
 * Same arguments, layout and errors as fc_dgemm. */
int fc_dgemm_streamk(fc_ctx ctx, int transA, int transB, int M, int N, int K, double alpha,
                     const double* A, int lda, const double* B, int ldb, double beta, double* C, int ldc);
/* Milliseconds of the last launch of the dominant kernel of the last API call (events on
 * the context stream) and its algorithmic flop and byte counts (for the roofline line). */
int fc_last_kernel_stats(fc_ctx ctx, double* ms, double* flops, double* bytes, int* launches);
/* Rank-revealing orthonormalisation used by the truncation (blocked Gram-Schmidt, columns kept
 * to tau times their norm): A (device, n x p, column-major, overwritten), Q (device, n x
 * min(n,p)); *k_host receives the basis size. */
int fc_orthonormalize(fc_ctx ctx, int n, int p, double* A, double* Q, double tau, int* k_host);
/* Batched symmetric eigensolver of the truncation (S11: the side-matrix Gram eigenproblem),
 * exposed for testing: nb <= 8 matrices; host arrays of length nb.  Entry i: A[i] (device,
 * N[i] x N[i] symmetric, column-major, leading dimension lda[i], overwritten), lam[i] (device,
 * N[i]: eigenvalues in DESCENDING order), Y[i] (device, N[i] x r[i], ld ldy[i]: orthonormal
 * eigenvectors of the r[i] largest eigenvalues, 0 <= r[i] <= N[i]).  1 <= N[i] <= 1500. */
int fc_syev(fc_ctx ctx, int nb, const int* N, double* const* A, const int* lda, double* const* lam,
            double* const* Y, const int* ldy, const int* r);
/* Opt-in accounting of every DMMA GEMM launch (events around each launch; for the bench's
 * roofline line).  enable=1 starts recording; enable=0 stops and returns the summed device
 * time (ms), the summed algorithmic flops (2 M N K per batch entry) and the launch count. */
int fc_profile_gemm(fc_ctx ctx, int enable, double* ms, double* flops, long long* launches);
/* Opt-in accounting of one HBM-class kernel (events around each launch on
 * its stream): kernel = FC_KP_DOT_REDUCE (the Hadamard-of-Grams reduction of cp_dot, 24 bytes per
 * (k, m) entry [P:1748-1755]) or FC_KP_KR_BASIS (the eigen-coordinate Khatri-Rao basis
 * K = [w_a (.) V^T q_b] of fracop_apply_truncate, 8 bytes per written entry plus its inputs
 * [P:1756-1763]).  enable=1 starts recording; enable=0 stops and returns the summed device time
 * (ms), the summed algorithmic bytes and the launch count.  Errors: INVALID_ARG (kernel id). */
#define FC_KP_DOT_REDUCE 0
#define FC_KP_KR_BASIS   1
#define FC_KP_KR_PRODUCT 2   /* fracop_apply's Khatri-Rao operand u_k (.) V^T x_j (K6), 8 B per entry */
int fc_profile_kernel(fc_ctx ctx, int kernel, int enable, double* ms, double* bytes, long long* launches);
/* Process-wide count of CUDA kernels this library has launched (host-side counter). */
int fc_kernel_launches(long long* count);

#ifdef __cplusplus
}
#endif
#endif /* FRACCONTROL_H */
