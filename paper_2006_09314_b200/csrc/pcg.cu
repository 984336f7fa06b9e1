// cp_truncate (S11-S13 on a plain CP) and pcg_solve: Algorithm 1 [P:1825-1872] on mixed
// Tucker-canonical iterates.
//
// The operator apply inside the solver is the factored apply of [P:614-623] written for an
// iterate whose factors are Q_l C_l (Q_l orthonormal, from the previous T2C):
//   forward transform   Zhat_l = V_l^T Q_l                     (S5, DMMA GEMM)
//   Khatri-Rao basis    Khat_l[:, a*q+b] = W_l[:, a] (.) Zhat_l[:, b]   (S6; U_F = W_F E_F)
//   coefficients        kron(E_l, C_l),  weights kron(w_F, w_x)
// the truncation then runs on that eigen-coordinate tensor, and only the r_l surviving basis
// columns are transformed back, Z_l <- V_l Z_l (S7, DMMA GEMM).  Because V_l is orthogonal,
// singular values, ranks and the T2C output are those of the paper's physical-coordinate
// apply followed by RHOSVD.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <exception>
#include <memory>
#include <thread>
#include "cpops.cuh"
#include "eig.cuh"
#include "solver.cuh"
#include "tt.cuh"

namespace fc {
namespace {

// K6 (S6) in eigen coordinates, the 3 modes in one launch (blockIdx.y = mode):
// K_l[:, a*q + b] = W_l[:, a] (.) Zh_l[:, b] (n x s_l q_l, written once: HBM-write-bound; W and
// Zh are re-read from L2), 16-byte double2 loads / streaming stores along the (even) mode size.
struct KRBasisArgs {
  int n, s[3], q[3];
  const double* W[3];
  const double* Zh[3];
  double* K[3];
};
__global__ void hadamard_basis_kernel(const __grid_constant__ KRBasisArgs A) {
  const int l = blockIdx.y, n = A.n, s = A.s[l], q = A.q[l];
  const double* __restrict__ W = A.W[l];
  const double* __restrict__ Zh = A.Zh[l];
  double* K = A.K[l];
  const int cols = s * q;
  const size_t al = reinterpret_cast<size_t>(W) | reinterpret_cast<size_t>(Zh) | reinterpret_cast<size_t>(K);
  if ((n & 1) == 0 && (al & 15) == 0) {
    // a warp per output column at a time (index math once per column), 16-byte coalesced
    // loads from L2 and streaming stores along n
    const int n2 = n >> 1, lane = threadIdx.x & 31;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int col = wid; col < cols; col += nw) {
      const int a = col / q, b = col - a * q;
      const double2* wa = reinterpret_cast<const double2*>(W + (size_t)a * n);
      const double2* zb = reinterpret_cast<const double2*>(Zh + (size_t)b * n);
      double2* o = reinterpret_cast<double2*>(K + (size_t)col * n);
#pragma unroll 4
      for (int i2 = lane; i2 < n2; i2 += 32) {
        const double2 w = __ldg(wa + i2), z = __ldg(zb + i2);
        __stcs(o + i2, make_double2(w.x * z.x, w.y * z.y));
      }
    }
    return;
  }
  const long long tot = (long long)n * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx % n);
    int col = (int)(idx / n);          // col = a*q + b
    int a = col / q, b = col % q;
    K[idx] = W[i + (size_t)a * n] * Zh[i + (size_t)b * n];
  }
}

// out[(a*q + b), (k*R + j)] = E[a, k] * C[b, j]   (kron(E, C)), out ld = s*q
__global__ void kron_kernel(int s, int r, const double* __restrict__ E, int q, int R, const double* __restrict__ C,
                            double* out) {
  const long long rows = (long long)s * q, tot = rows * r * R;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    int row = (int)(idx % rows);
    long long col = idx / rows;
    int a = row / q, b = row % q;
    int k = (int)(col / R), j = (int)(col % R);
    out[idx] = E[a + (size_t)k * s] * C[b + (size_t)j * q];
  }
}

__global__ void kron_w_kernel(int r, const double* __restrict__ wF, int R, const double* __restrict__ w, double* out) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < r * R) out[t] = wF[t / R] * w[t % R];
}

__global__ void inv_sqrt_cols_kernel(int n, int s, const double* __restrict__ lam, double* W) {
  const long long tot = (long long)n * s;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    int a = (int)(idx / n);
    W[idx] *= 1.0 / sqrt(lam[a]);
  }
}

int nblocks(long long tot) { return (int)std::min<long long>(std::max<long long>((tot + 255) / 256, 1), 148 * 8); }

}  // namespace

// Reduced basis of the spectral CP: U_l = W_l E_l with W_l orthonormal (n x s_l).
void ensure_spec_basis(fc_ctx c, SpecCP& sp) {
  if (sp.has_basis) return;
  cudaStream_t st = stream_of(c);
  const int n = c->n, r = sp.r;
  Scratch s(st);
  int sdim[3];
  double* Wt[3];
  {
    // orthonormal basis of span(U_l) by column-pivoted MGS (columns kept to 1e-14)
    PmgsBatch pb;
    int* kd = s.alloc<int>(4);
    for (int l = 0; l < 3; ++l) {
      double* A = s.alloc<double>((size_t)n * r);
      FC_CUDA_TRY(cudaMemcpyAsync(A, sp.Ul(n, l), (size_t)n * r * 8, cudaMemcpyDeviceToDevice, st));
      Wt[l] = s.alloc<double>((size_t)n * std::min(n, r));
      pb.e[pb.nb++] = PmgsEntry{n, r, A, n, Wt[l], n, kd + l, 1e-14};
    }
    pmgs(pb, st);
    FC_CUDA_TRY(cudaMemcpyAsync(sdim, kd, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaStreamSynchronize(st));
    for (int l = 0; l < 3; ++l) require(sdim[l] >= 1, FC_ERR_NOT_SPD, "spectral CP has a zero factor matrix");
  }
  sp.smax = std::max(sdim[0], std::max(sdim[1], sdim[2]));
  sp.W.ensure((size_t)3 * n * sp.smax);
  sp.E.ensure((size_t)3 * sp.smax * r);
  for (int l = 0; l < 3; ++l) {
    sp.s[l] = sdim[l];
    double* Wl = sp.W.p + (size_t)l * n * sp.smax;
    double* El = sp.E.p + (size_t)l * sp.smax * r;
    FC_CUDA_TRY(cudaMemcpyAsync(Wl, Wt[l], (size_t)n * sdim[l] * 8, cudaMemcpyDeviceToDevice, st));
    FC_CUDA_TRY(cudaMemsetAsync(El, 0, (size_t)sdim[l] * r * 8, st));
    dgemm(st, 1, 0, sdim[l], r, n, 1.0, Wl, n, sp.Ul(n, l), n, 1.0, El, sdim[l],
          std::max(1, std::min(cdiv(n, 256), 16)));
  }
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  sp.has_basis = true;
}

// S = trunc(F x) for a TT iterate x (physical coordinates, orthonormal bases).
TT apply_truncate_tt(fc_ctx c, SpecCP& sp, const TT& x, double eps, int rank_cap, TruncStats* stats) {
  cudaStream_t st = stream_of(c);
  const int n = c->n, r = sp.r, R = x.R;
  if (R == 0) {
    TT z;
    z.n = n;
    return z;
  }
  ensure_spec_basis(c, sp);
  auto pm0 = std::make_unique<PhaseMarks>(st);
  // x's Tucker core (T2C outputs carry it; otherwise form it once from the CP coefficients)
  TT xc;
  const double* core_x = x.core;
  if (!core_x) {
    xc = tt_copy(st, x);
    tt_compute_core(st, xc);
    core_x = xc.core;
  }
  TT y;   // eigen-coordinate Hadamard tensor: basis K_l, weights kron(w_F, w_x); no coefficients
  y.n = n;
  y.R = r * R;
  size_t need = (size_t)y.R + 1;
  for (int l = 0; l < 3; ++l) {
    y.q[l] = sp.s[l] * x.q[l];
    need += (size_t)n * x.q[l] + (size_t)n * y.q[l];
  }
  y.mem.emplace_back(need * 8, st);
  double* p = y.mem.back().d();
  y.w = p;
  p += y.R + (y.R & 1);   // keep the basis blocks 16-byte aligned (double2 access)
  kron_w_kernel<<<cdiv(y.R, 256), 256, 0, st>>>(r, sp.w.p, R, x.w, y.w);
  FC_CHECK_LAUNCH();
  GemmArgs fwd;   // S5: Zhat_l = V_l^T Q_l
  fwd.transA = 1;
  fwd.nbatch = 3;
  double* Zh[3];
  for (int l = 0; l < 3; ++l) {
    Zh[l] = p;
    p += (size_t)n * x.q[l];
    fwd.b[l] = GemmBatch{n, x.q[l], n, c->Vsp(sp, l), n, x.Q[l], n, Zh[l], n, nullptr, 0, nullptr};
  }
  // ~100 output tiles for 148 SMs with K = n: split-K (zeroed output, beta = 1)
  FC_CUDA_TRY(cudaMemsetAsync(Zh[0], 0, (size_t)n * (x.q[0] + x.q[1] + x.q[2]) * 8, st));
  fwd.beta = 1.0;
  fwd.splitk = waves_splitk(fwd, 8);
  gemm(fwd, st);
  StructuredS ss;
  ss.r = r;
  ss.Rx = R;
  ss.wF = sp.w.p;
  ss.core_x = core_x;
  KRBasisArgs kra;
  kra.n = n;
  double kr_bytes = 0.0;
  long long kr_max = 0;
  for (int l = 0; l < 3; ++l) {   // S6: the Khatri-Rao basis [w_a (.) xhat_b]
    const double* Wl = sp.W.p + (size_t)l * n * sp.smax;
    ss.s[l] = sp.s[l];
    ss.t[l] = x.q[l];
    ss.E[l] = sp.E.p + (size_t)l * sp.smax * r;
    ss.Cx[l] = x.C[l];
    y.Q[l] = p;
    p += (size_t)n * y.q[l];
    y.C[l] = nullptr;
    kra.s[l] = sp.s[l];
    kra.q[l] = x.q[l];
    kra.W[l] = Wl;
    kra.Zh[l] = Zh[l];
    kra.K[l] = y.Q[l];
    kr_bytes += 8.0 * ((double)n * y.q[l] + (double)n * (sp.s[l] + x.q[l]));
    kr_max = std::max(kr_max, (long long)n * y.q[l]);
    y.orth[l] = false;
  }
  {
    KProfScope kp(KP_KR_BASIS, st, kr_bytes);
    // ~8 resident 256-thread CTAs per SM over the 3 modes, 16 bytes per thread and pass
    const int gx = (int)std::max<long long>(1, std::min<long long>((kr_max / n + 7) / 8, 148 * 8 / 3 + 1));
    hadamard_basis_kernel<<<dim3(gx, 3), 256, 0, st>>>(kra);
    FC_CHECK_LAUNCH();
  }
  pm0->mark("0 apply: fwd + KR basis");
  pm0.reset();
  TT out = truncate_tt(c, y, eps, rank_cap, stats, &ss);
  PhaseMarks pm1(st);
  // S7: back to physical coordinates, only the surviving basis columns
  GemmArgs inv;
  inv.nbatch = 0;
  if (out.R > 0) {
    const size_t tot = (size_t)n * (out.q[0] + out.q[1] + out.q[2]);
    DevMem newQ(tot * 8, st);
    FC_CUDA_TRY(cudaMemsetAsync(newQ.d(), 0, tot * 8, st));
    double* nq[3];
    size_t off = 0;
    for (int l = 0; l < 3; ++l) {
      nq[l] = newQ.d() + off;
      off += (size_t)n * out.q[l];
      inv.b[inv.nbatch++] = GemmBatch{n, out.q[l], n, c->Vsp(sp, l), n, out.Q[l], n, nq[l], n, nullptr, 0, nullptr};
    }
    inv.beta = 1.0;
    inv.splitk = waves_splitk(inv, 8);
    gemm(inv, st);
    for (int l = 0; l < 3; ++l)
      FC_CUDA_TRY(cudaMemcpyAsync(out.Q[l], nq[l], (size_t)n * out.q[l] * 8, cudaMemcpyDeviceToDevice, st));
  }
  pm1.mark("9 back-transform");
  return out;
}

// FC_TRACE_PCG diagnostics: orthonormality of a TT iterate's bases and ||core||^2 vs sum w^2
// (equal for the orthogonal-CP outputs of a truncation)
void tt_check(cudaStream_t st, const TT& x, const char* name) {
  if (x.R == 0) return;
  double orth = 0.0;
  for (int l = 0; l < 3; ++l) {
    const int q = x.q[l];
    Scratch s(st);
    double* G = s.alloc<double>((size_t)q * q);
    dgemm(st, 1, 0, q, q, x.n, 1.0, x.Q[l], x.n, x.Q[l], x.n, 0.0, G, q);
    std::vector<double> h((size_t)q * q);
    FC_CUDA_TRY(cudaMemcpyAsync(h.data(), G, h.size() * 8, cudaMemcpyDeviceToHost, st));
    FC_CUDA_TRY(cudaStreamSynchronize(st));
    for (int i = 0; i < q; ++i)
      for (int j = 0; j < q; ++j) orth = std::max(orth, std::fabs(h[i + (size_t)j * q] - (i == j ? 1.0 : 0.0)));
  }
  std::vector<double> w(x.R);
  FC_CUDA_TRY(cudaMemcpyAsync(w.data(), x.w, (size_t)x.R * 8, cudaMemcpyDeviceToHost, st));
  double c2 = -1.0;
  std::vector<double> core;
  if (x.core) {
    core.resize((size_t)x.q[0] * x.q[1] * x.q[2]);
    FC_CUDA_TRY(cudaMemcpyAsync(core.data(), x.core, core.size() * 8, cudaMemcpyDeviceToHost, st));
  }
  FC_CUDA_TRY(cudaStreamSynchronize(st));
  double w2 = 0.0;
  for (double v : w) w2 += v * v;
  if (x.core) {
    c2 = 0.0;
    for (double v : core) c2 += v * v;
  }
  fprintf(stderr, "[fc pcg]   %s: R %d q (%d,%d,%d) orth_err %.2e  sum w^2 %.6e  ||core||^2 %.6e\n", name, x.R, x.q[0],
          x.q[1], x.q[2], orth, w2, c2);
}

}  // namespace fc

using namespace fc;

namespace {
template <class F>
int guard2(fc_ctx c, F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    if (c) c->err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return FC_ERR_CUDA;
  }
}

void check_cp2(fc_ctx c, const fc_cp* x, const char* name) {
  require(x != nullptr, FC_ERR_INVALID_ARG, std::string(name) + " is NULL");
  require(c->n > 0, FC_ERR_NOT_READY, "no eigenpairs: call sl_setup or sl_set_eigen first");
  for (int l = 0; l < 3; ++l) {
    require(x->n[l] == c->n, FC_ERR_SHAPE, std::string(name) + ": mode size differs from context n");
    require(x->ld[l] >= x->n[l], FC_ERR_INVALID_ARG, std::string(name) + ": ld < n");
  }
  require(x->rank >= 0 && x->rank <= x->cap, FC_ERR_INVALID_ARG, std::string(name) + ": rank > cap");
}

void fill_info(fc_trunc_info* info, const TruncStats& S) {
  if (!info) return;
  for (int l = 0; l < 3; ++l) {
    info->tucker_rank[l] = S.tucker[l];
    info->basis_dim[l] = S.basis[l];
  }
  info->out_rank = S.out_rank;
  info->in_rank = S.in_rank;
  info->t2c_mode = S.t2c_mode;
  info->energy = S.energy;
  info->min_cut_margin = S.min_margin;
}

void store_tt(fc_ctx c, const TT& x, fc_cp* y) {
  if (y->cap < x.R) {
    y->rank = x.R;
    throw Error(FC_ERR_CAPACITY, "output cap below the result rank");
  }
  tt_expand(c->st, x, y->U, y->ld, y->w);
  y->rank = x.R;
  FC_CUDA_TRY(cudaStreamSynchronize(c->st));
}
}  // namespace

// Algorithm 1 lines 10-11 (X <- trunc(X + a P)) on the context's side stream from a helper
// thread: X is read again only by the next iteration's X update, so its truncation overlaps the
// R, Z and P work of lines 12-21 (the truncation syncs its own stream to read ranks, hence the
// second host thread).  Events order the streams both ways; the result's memory is re-homed on
// the main stream.  The destructor joins on every path (also when the main thread throws).
struct XJob {
  fc_ctx c;
  cudaStream_t st;
  TT XP, out;
  TruncStats stats;
  std::exception_ptr err;
  std::thread th;
  bool joined = false;
  XJob(fc_ctx c_, cudaStream_t st_, const TT& X, const TT& P, double a, double eps, int cap) : c(c_), st(st_) {
    XP = tt_axpy(st, X, a, P);
    static const bool inline_x = getenv("FC_NO_OVERLAP") != nullptr;   // diagnostics: no side stream
    if (inline_x) {
      try {
        out = truncate_tt(c, XP, eps, cap, &stats);
      } catch (...) {
        err = std::current_exception();
      }
      joined = true;
      return;
    }
    cudaEvent_t ev;
    FC_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    FC_CUDA_TRY(cudaEventRecord(ev, st));
    FC_CUDA_TRY(cudaStreamWaitEvent(c->st2, ev, 0));
    FC_CUDA_TRY(cudaEventDestroy(ev));
    th = std::thread([this, eps, cap]() {
      tl_stream = c->st2;
      try {
        out = truncate_tt(c, XP, eps, cap, &stats);
      } catch (...) {
        err = std::current_exception();
      }
      tl_stream = nullptr;
    });
  }
  void finish() {
    if (joined) return;
    joined = true;
    th.join();
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, c->st2);
    cudaStreamWaitEvent(st, ev, 0);   // main stream after the side stream's work (uses and frees)
    cudaEventDestroy(ev);
    for (auto& m : out.mem) m.st = st;
  }
  TT join(TruncStats* s) {
    finish();
    if (err) std::rethrow_exception(err);
    *s = stats;
    return std::move(out);
  }
  ~XJob() { finish(); }
};

extern "C" {

int cp_truncate(fc_ctx c, const fc_cp* x, double eps, fc_cp* y, fc_trunc_info* info) {
  return guard2(c, [&]() {
    check_cp2(c, x, "x");
    check_cp2(c, y, "y");
    require(eps > 0 && std::isfinite(eps), FC_ERR_INVALID_ARG, "eps must be > 0");
    TruncStats S;
    TT xt = tt_from_cp(c->st, c->n, x->rank, x->w, x->U, x->ld);
    TT out;
    try {
      out = truncate_tt(c, xt, eps, 0, &S);
    } catch (const Error& e) {
      fill_info(info, S);
      if (info && e.code == FC_ERR_CAPACITY) info->required_rank = S.out_rank;
      throw;
    }
    fill_info(info, S);
    if (y->cap < out.R) {
      if (info) info->required_rank = out.R;
    }
    store_tt(c, out, y);
    return FC_OK;
  });
}

int cp_truncate_als(fc_ctx c, const fc_cp* x, double eps, int sweeps, fc_cp* y, fc_trunc_info* info) {
  return guard2(c, [&]() {
    check_cp2(c, x, "x");
    check_cp2(c, y, "y");
    require(eps > 0 && std::isfinite(eps), FC_ERR_INVALID_ARG, "eps must be > 0");
    require(sweeps >= 0 && sweeps <= 100, FC_ERR_INVALID_ARG, "sweeps in [0, 100]");
    TruncStats S;
    TT xt = tt_from_cp(c->st, c->n, x->rank, x->w, x->U, x->ld);
    TT out;
    try {
      out = truncate_tt(c, xt, eps, 0, &S, nullptr, sweeps);
    } catch (const Error& e) {
      fill_info(info, S);
      if (info && e.code == FC_ERR_CAPACITY) info->required_rank = S.out_rank;
      throw;
    }
    fill_info(info, S);
    if (y->cap < out.R) {
      if (info) info->required_rank = out.R;
    }
    store_tt(c, out, y);
    return FC_OK;
  });
}

int fracop_apply_truncate(fc_ctx c, int which, const fc_cp* x, double eps, fc_cp* y, fc_trunc_info* info) {
  return guard2(c, [&]() {
    require(which >= 0 && which < 4, FC_ERR_INVALID_ARG, "which");
    check_cp2(c, x, "x");
    check_cp2(c, y, "y");
    require(eps > 0 && std::isfinite(eps), FC_ERR_INVALID_ARG, "eps must be > 0");
    require(c->have_eig[0] && c->have_eig[1] && c->have_eig[2], FC_ERR_NOT_READY, "eigenpairs missing");
    ensure_spectral(c, which);
    SpecCP& sp = c->spec[which];
    require(sp.valid, FC_ERR_NOT_READY, "spectral CP not set");
    TruncStats S;
    TT xt = tt_from_cp(c->st, c->n, x->rank, x->w, x->U, x->ld);
    TT out;
    try {
      out = apply_truncate_tt(c, sp, xt, eps, 0, &S);
    } catch (const Error& e) {
      fill_info(info, S);
      if (info && e.code == FC_ERR_CAPACITY) info->required_rank = S.out_rank;
      throw;
    }
    fill_info(info, S);
    if (y->cap < out.R && info) info->required_rank = out.R;
    store_tt(c, out, y);
    return FC_OK;
  });
}

int state_recover(fc_ctx c, const fc_cp* u, double eps, fc_cp* y, fc_trunc_info* info) {
  return fracop_apply_truncate(c, FC_POW_MINUS, u, eps, y, info);
}

int pcg_solve(fc_ctx c, const fc_cp* b, const fc_params* prm, fc_cp* u, fc_pcg_report* rep) {
  return guard2(c, [&]() {
    check_cp2(c, b, "b");
    check_cp2(c, u, "u");
    require(prm != nullptr, FC_ERR_INVALID_ARG, "params NULL");
    const double eps = prm->eps;
    require(eps > 0, FC_ERR_INVALID_ARG, "eps must be > 0");
    const double tol = prm->tol_stop > 0 ? prm->tol_stop : 10.0 * eps;     // A13
    const int kmax = std::min(prm->kmax > 0 ? prm->kmax : 100, FC_MAX_ITERS);  // A17
    const int cap = prm->rank_cap > 0 ? prm->rank_cap : (1 << 20);
    require(c->spec[FC_F].valid && c->spec[FC_G].valid, FC_ERR_NOT_READY, "spectral CPs missing");
    cudaStream_t st = stream_of(c);
    if (!c->st2) FC_CUDA_TRY(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
    fc_pcg_report local{};
    fc_pcg_report& RP = rep ? *rep : local;
    RP = fc_pcg_report{};
    cudaEvent_t t0, t1, ti0, ti1;
    FC_CUDA_TRY(cudaEventCreate(&t0));
    FC_CUDA_TRY(cudaEventCreate(&t1));
    FC_CUDA_TRY(cudaEventCreate(&ti0));
    FC_CUDA_TRY(cudaEventCreate(&ti1));
    struct EvGuard {
      cudaEvent_t a, b, c2, d;
      ~EvGuard() { cudaEventDestroy(a); cudaEventDestroy(b); cudaEventDestroy(c2); cudaEventDestroy(d); }
    } evg{t0, t1, ti0, ti1};
    FC_CUDA_TRY(cudaEventRecord(t0, st));
    SpecCP& F = c->spec[FC_F];
    SpecCP& G = c->spec[FC_G];
    ensure_spec_basis(c, F);
    ensure_spec_basis(c, G);

    TT B = tt_from_cp(st, c->n, b->rank, b->w, b->U, b->ld);
    const double normB = std::sqrt(std::max(tt_dot(c, B, B), 0.0));
    RP.normB = normB;
    require(std::isfinite(normB), FC_ERR_NAN, "non-finite right-hand side");
    TT X;                                             // X0 = 0 (A14)
    X.n = c->n;
    if (normB == 0.0) {
      RP.converged = 1;
      u->rank = 0;
      return FC_OK;
    }
    // line 1: R0 = B (A15, untruncated); lines 2-3: Z0 = trunc(precond(R0)); line 4: P0 = Z0
    TT R = tt_copy(st, B);
    // (B's basis need not be orthonormal: the truncation handles any Khatri-Rao basis)
    TruncStats sZ;
    TT Z = apply_truncate_tt(c, G, R, eps, cap, &sZ);
    TT P = tt_copy(st, Z);
    double rz = tt_dot(c, R, Z);
    RP.cap_hits = sZ.clipped;
    int status = FC_NOT_CONVERGED;
    cudaEvent_t loop0;
    FC_CUDA_TRY(cudaEventCreate(&loop0));
    FC_CUDA_TRY(cudaEventRecord(loop0, st));
    for (int k = 0; k < kmax; ++k) {
      FC_CUDA_TRY(cudaEventRecord(ti0, st));
      TruncStats sS, sX, sR;
      TT S = apply_truncate_tt(c, F, P, eps, cap, &sS);            // lines 7-8
      const double ps = tt_dot(c, P, S);
      if (!std::isfinite(ps)) { cudaEventDestroy(loop0); throw Error(FC_ERR_NAN, "<P,S> is not finite"); }
      if (ps <= 0) { cudaEventDestroy(loop0); throw Error(FC_ERR_NOT_SPD, "<P,S> <= 0"); }
      const double a_k = rz / ps;                                   // line 9
      static const bool tr_pcg = getenv("FC_TRACE_PCG") != nullptr;
      if (tr_pcg) {
        fprintf(stderr, "[fc pcg] k=%d <R,Z>=%.10e <P,S>=%.10e a=%.10e  S: tucker (%d,%d,%d) energy %.6e refined %d\n", k,
                rz, ps, a_k, sS.tucker[0], sS.tucker[1], sS.tucker[2], sS.energy, (int)sS.refined);
        tt_check(st, P, "P");
        tt_check(st, S, "S");
        tt_check(st, R, "R");
      }
      XJob xjob(c, st, X, P, a_k, eps, cap);                        // lines 10-11 (side stream)
      {
        TT RS = tt_axpy(st, R, -a_k, S);                            // lines 12-13
        R = truncate_tt(c, RS, eps, cap, &sR);
      }
      const double rr = tt_dot(c, R, R);
      const double rel = std::sqrt(std::max(rr, 0.0)) / normB;      // line 14 (A13)
      RP.rel_res[k] = rel;
      RP.rank_S[k] = S.R;
      RP.rank_R[k] = R.R;
      RP.tucker_S[k] = std::max(sS.tucker[0], std::max(sS.tucker[1], sS.tucker[2]));
      RP.iters = k + 1;
      RP.cap_hits += sS.clipped + sR.clipped;
      if (!std::isfinite(rel)) { cudaEventDestroy(loop0); throw Error(FC_ERR_NAN, "residual is not finite"); }
      if (rel <= tol) {
        X = xjob.join(&sX);
        RP.cap_hits += sX.clipped;
        RP.rank_X[k] = X.R;
        RP.rank_Z[k] = Z.R;
        RP.rank_P[k] = P.R;
        FC_CUDA_TRY(cudaEventRecord(ti1, st));
        FC_CUDA_TRY(cudaEventSynchronize(ti1));
        float ms;
        cudaEventElapsedTime(&ms, ti0, ti1);
        RP.t_iter_ms[k] = ms;
        status = FC_OK;
        break;
      }
      TruncStats sZ2, sP;
      Z = apply_truncate_tt(c, G, R, eps, cap, &sZ2);               // lines 17-18
      const double rz_new = tt_dot(c, R, Z);
      const double b_k = rz_new / rz;                               // line 19 (A16)
      if (tr_pcg) {
        fprintf(stderr, "[fc pcg] k=%d rel=%.6e <R',Z'>=%.10e b=%.10e  R: tucker (%d,%d,%d) energy %.6e refined %d  Z: tucker (%d,%d,%d) refined %d\n",
                k, rel, rz_new, b_k, sR.tucker[0], sR.tucker[1], sR.tucker[2], sR.energy, (int)sR.refined, sZ2.tucker[0],
                sZ2.tucker[1], sZ2.tucker[2], (int)sZ2.refined);
        tt_check(st, R, "R'");
        tt_check(st, Z, "Z'");
      }
      {
        TT ZP = tt_axpy(st, Z, b_k, P);                             // lines 20-21
        P = truncate_tt(c, ZP, eps, cap, &sP);
      }
      rz = rz_new;
      X = xjob.join(&sX);
      RP.cap_hits += sX.clipped + sZ2.clipped + sP.clipped;
      RP.rank_X[k] = X.R;
      RP.rank_Z[k] = Z.R;
      RP.rank_P[k] = P.R;
      FC_CUDA_TRY(cudaEventRecord(ti1, st));
      FC_CUDA_TRY(cudaEventSynchronize(ti1));
      float ms;
      cudaEventElapsedTime(&ms, ti0, ti1);
      RP.t_iter_ms[k] = ms;
    }
    FC_CUDA_TRY(cudaEventRecord(t1, st));
    FC_CUDA_TRY(cudaEventSynchronize(t1));
    float tl, tt;
    cudaEventElapsedTime(&tl, loop0, t1);
    cudaEventElapsedTime(&tt, t0, t1);
    cudaEventDestroy(loop0);
    RP.t_loop_ms = tl;
    RP.t_total_ms = tt;
    RP.converged = status == FC_OK;
    if (status == FC_OK && RP.cap_hits > 0) status = FC_RANK_CAP_HIT;   // converged, but clipped
    RP.status = status;
    store_tt(c, X, u);
    return status;
  });
}

}  // extern "C"
