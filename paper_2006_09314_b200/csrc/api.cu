// C-ABI entry points (include/fraccontrol.h): context, eigen/spectral-CP injection,
// fracop_apply (S5-S8), cp_dot (S10), cp_axpy (S9), raw DGEMM, kernel stats.
#include <algorithm>
#include <cmath>
#include "cpops.cuh"
#include "ctx.cuh"
#include "solver.cuh"
#include "eig.cuh"

using namespace fc;

namespace {

template <class F>
int guard(fc_ctx c, F&& f) {
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

void check_cp(fc_ctx c, const fc_cp* x, const char* name) {
  require(x != nullptr, FC_ERR_INVALID_ARG, std::string(name) + " is NULL");
  require(c->n > 0, FC_ERR_NOT_READY, "no eigenpairs: call sl_setup or sl_set_eigen first");
  for (int l = 0; l < 3; ++l) {
    require(x->n[l] == c->n, FC_ERR_SHAPE, std::string(name) + ": mode size differs from context n");
    require(x->ld[l] >= x->n[l], FC_ERR_INVALID_ARG, std::string(name) + ": ld < n");
    require(x->rank == 0 || x->U[l] != nullptr, FC_ERR_INVALID_ARG, std::string(name) + ": NULL factor");
  }
  require(x->rank >= 0 && x->rank <= x->cap, FC_ERR_INVALID_ARG, std::string(name) + ": rank > cap");
}

}  // namespace

// ---------------------------------------------------------------------------------------
namespace fc {

// y = F(A) x for a plain CP (S5-S8).  The dominant launch (inverse transform) is bracketed by
// the context's events.
void apply_plain(fc_ctx c, const SpecCP& sp, const fc_cp& x, fc_cp& y) {
  const int n = c->n, r = sp.r, R = x.rank;
  cudaStream_t st = c->st;
  y.rank = r * R;
  if (R == 0 || r == 0) {
    y.rank = 0;
    return;
  }
  Scratch s(st);
  double* What = s.alloc<double>((size_t)3 * n * R);
  double* Usq = s.alloc<double>((size_t)3 * n * r);
  double* Wsq = s.alloc<double>((size_t)3 * n * R);
  double* N2 = s.alloc<double>((size_t)3 * r * R);
  double* cs = s.alloc<double>((size_t)3 * r * R);

  // S5 forward transform  W_l = V_l^T X_l  (3 modes batched)
  GemmArgs f;
  f.transA = 1;
  f.nbatch = 3;
  for (int l = 0; l < 3; ++l)
    f.b[l] = GemmBatch{n, R, n, c->Vsp(sp, l), n, x.U[l], x.ld[l], What + (size_t)l * n * R, n, nullptr, 0, nullptr};
  f.streamk = 1;   // R >= 128: k-step-balanced 128 x 128 tiles (gemm.cu); below, the 64 x 64 kernel
  gemm(f, st);

  // S8 (moved ahead): column norms of u_k (.) w_j; ||V y|| = ||y|| since V is orthogonal
  Mat3 a{}, as{}, b{}, bs{};
  for (int l = 0; l < 3; ++l) {
    a.p[l] = sp.Ul(n, l); a.ld[l] = n; a.rows[l] = n; a.cols[l] = r;
    as.p[l] = Usq + (size_t)l * n * r; as.ld[l] = n; as.rows[l] = n; as.cols[l] = r;
    b.p[l] = What + (size_t)l * n * R; b.ld[l] = n; b.rows[l] = n; b.cols[l] = R;
    bs.p[l] = Wsq + (size_t)l * n * R; bs.ld[l] = n; bs.rows[l] = n; bs.cols[l] = R;
  }
  square3(a, as, st);
  square3(b, bs, st);
  GemmArgs g2;
  g2.transA = 1;
  g2.nbatch = 3;
  for (int l = 0; l < 3; ++l)
    g2.b[l] = GemmBatch{r, R, n, Usq + (size_t)l * n * r, n, Wsq + (size_t)l * n * R, n, N2 + (size_t)l * r * R, r,
                        nullptr, 0, nullptr};
  gemm(g2, st);
  const double* N2p[3] = {N2, N2 + (size_t)r * R, N2 + (size_t)2 * r * R};
  double* csp[3] = {cs, cs + (size_t)r * R, cs + (size_t)2 * r * R};
  apply_weights(r, R, sp.w.p, x.w, N2p, y.w, csp, st);

  // S6: the Khatri-Rao / Hadamard operand Yhat_l[:, k R + j] = u_k (.) w_j, written once (K6,
  // HBM-write-bound, 3 modes in one launch), then S7: Y_l = V_l Yhat_l as a plain GEMM (B
  // contiguous along K: 16-byte cp.async, no product in the MMA loop).  FC_KR_FUSED=1: the
  // product formed at fragment-load time inside the GEMM instead (diagnostic; its per-fragment
  // DMULs were 25 % of the kernel's stall samples, r02 ncu).
  static const bool kr_fused = getenv("FC_KR_FUSED") != nullptr;
  GemmArgs iv;
  iv.nbatch = 3;
  double* Yhat = nullptr;
  if (kr_fused) {
    iv.krR = R;
  } else {
    Yhat = s.alloc<double>((size_t)3 * n * r * R);
    const double* Uf[3] = {sp.Ul(n, 0), sp.Ul(n, 1), sp.Ul(n, 2)};
    const double* Wh[3] = {What, What + (size_t)n * R, What + (size_t)2 * n * R};
    double* Yh[3] = {Yhat, Yhat + (size_t)n * r * R, Yhat + (size_t)2 * n * r * R};
    kr_product3(n, r, R, Uf, Wh, Yh, st);
  }
  for (int l = 0; l < 3; ++l)
    iv.b[l] = kr_fused ? GemmBatch{n, r * R, n, c->Vsp(sp, l), n, What + (size_t)l * n * R, n, y.U[l], y.ld[l],
                                   sp.Ul(n, l), n, csp[l]}
                       : GemmBatch{n, r * R, n, c->Vsp(sp, l), n, Yhat + (size_t)l * n * r * R, n, y.U[l], y.ld[l],
                                   nullptr, 0, csp[l]};
  // wave balance (one 128x128 CTA per SM): no split-K once the tiles fill >= 2 waves of 148 SMs
  // (the split reduction costs more than the last wave's fill: r02 sweep, sk = 1 best at 384+
  // tiles), else the smallest power of two reaching 2 waves (>= 128 of K per split, <= 8)
  const long long tiles = 3LL * cdiv(n, 128) * cdiv((long long)r * R, 128);
  int sk = 1;
  while (tiles * sk < 2LL * 148 && sk < 8 && n / (2 * sk) >= 128) sk *= 2;
  static const int sk_env = getenv("FC_APPLY_SPLITK") ? atoi(getenv("FC_APPLY_SPLITK")) : 0;   // diagnostic
  if (sk_env > 0) sk = sk_env;
  iv.splitk = sk;   // deterministic split-K reduction: C needs no pre-zeroing (beta = 0)
  iv.streamk = 1;   // ... or, when whole tiles fill the last wave badly, k-step-balanced (stream-K)
  FC_CUDA_TRY(cudaEventRecord(c->e0, st));
  gemm(iv, st);
  FC_CUDA_TRY(cudaEventRecord(c->e1, st));
  c->k_flops = 3.0 * 2.0 * (double)n * n * (double)r * R;
  c->k_bytes = 3.0 * 8.0 * ((double)n * n + (double)n * R + (double)n * r + (double)n * r * R);
  c->k_launches = 1;
}

// Cross Grams G_l = X_l^T Y_l (3 modes) into G (3 blocks of R1 x R2, ld R1).
void cross_gram(cudaStream_t st, int n, int R1, const double* const X[3], const int ldx[3], int R2,
                const double* const Y[3], const int ldy[3], double* G) {
  size_t blk = (size_t)R1 * R2;
  FC_CUDA_TRY(cudaMemsetAsync(G, 0, 3 * blk * sizeof(double), st));
  GemmArgs g;
  g.transA = 1;
  g.nbatch = 3;
  g.beta = 1.0;
  int tiles = cdiv(R1, 64) * cdiv(R2, 64) * 3;
  g.splitk = std::max(1, std::min(cdiv(n, 128), cdiv(148 * 4, tiles)));
  for (int l = 0; l < 3; ++l) g.b[l] = GemmBatch{R1, R2, n, X[l], ldx[l], Y[l], ldy[l], G + l * blk, R1, nullptr, 0, nullptr};
  gemm(g, st);
}

// <x, y> = sum_{k,m} xi_k zeta_m prod_l (U_l^T V_l)[k, m]  [P:1748-1755], tiled over (k, m) so
// the three cross-Grams of a tile stay below ~48 Mi doubles whatever the ranks; the tile sums are
// added on the host in tile order (deterministic).
double dot_plain(fc_ctx c, const fc_cp& x, const fc_cp& y) {
  if (x.rank == 0 || y.rank == 0) return 0.0;
  Scratch s(c->st);
  const int R1 = x.rank, R2 = y.rank;
  constexpr int TILE = 4096;
  const int T1 = std::min(R1, TILE), T2 = std::min(R2, TILE);
  const int n1 = cdiv(R1, T1), n2 = cdiv(R2, T2);
  double* G = s.alloc<double>((size_t)3 * T1 * T2);
  double* out = s.alloc<double>((size_t)n1 * n2);
  for (int a = 0; a < n1; ++a) {
    const int k0 = a * T1, kr = std::min(T1, R1 - k0);
    for (int b = 0; b < n2; ++b) {
      const int m0 = b * T2, mr = std::min(T2, R2 - m0);
      const double* X[3];
      const double* Y[3];
      for (int l = 0; l < 3; ++l) {
        X[l] = x.U[l] + (size_t)k0 * x.ld[l];
        Y[l] = y.U[l] + (size_t)m0 * y.ld[l];
      }
      cross_gram(c->st, c->n, kr, X, x.ld, mr, Y, y.ld, G);
      const double* Gp[3] = {G, G + (size_t)kr * mr, G + (size_t)2 * kr * mr};
      dot_reduce(kr, mr, x.w + k0, y.w + m0, Gp, kr, out + (size_t)a * n2 + b, c->st);
    }
  }
  std::vector<double> h((size_t)n1 * n2);
  FC_CUDA_TRY(cudaMemcpyAsync(h.data(), out, h.size() * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  FC_CUDA_TRY(cudaStreamSynchronize(c->st));
  double sum = 0.0;
  for (double v : h) sum += v;
  return sum;
}

void copy_cp_block(cudaStream_t st, int n, const fc_cp& src, fc_cp& dst, int col0, double scale) {
  if (src.rank == 0) return;
  Mat3 a{}, b{};
  for (int l = 0; l < 3; ++l) {
    a.p[l] = src.U[l]; a.ld[l] = src.ld[l]; a.rows[l] = n; a.cols[l] = src.rank;
    b.p[l] = dst.U[l] + (size_t)col0 * dst.ld[l]; b.ld[l] = dst.ld[l]; b.rows[l] = n; b.cols[l] = src.rank;
  }
  copy_cols3(a, b, 1.0, st);
  scale_copy(src.rank, src.w, scale, dst.w + col0, st);
}

}  // namespace fc

namespace fc {
std::atomic<long long> g_launches{0};
thread_local cudaStream_t tl_stream = nullptr;
}

// ======================================================================================
extern "C" {

int fc_orthonormalize(fc_ctx c, int n, int p, double* A, double* Q, double tau, int* k_host) {
  return guard(c, [&]() {
    require(n >= 1 && p >= 1 && A && Q && k_host, FC_ERR_INVALID_ARG, "fc_orthonormalize args");
    Scratch s(c->st);
    const int kcap = std::min(n, p);
    // run as a batch of 3 identical problems (as the truncation does per mode) and require
    // identical results, so the batched path is what the tests exercise
    BcgsBatch b;
    b.nb = 3;
    int* kd = s.alloc<int>(3);
    double* Qx[3] = {Q, s.alloc<double>((size_t)n * kcap), s.alloc<double>((size_t)n * kcap)};
    for (int i = 0; i < 3; ++i) {
      double* Ai = A;
      if (i > 0) {
        Ai = s.alloc<double>((size_t)n * p);
        FC_CUDA_TRY(cudaMemcpyAsync(Ai, A, (size_t)n * p * 8, cudaMemcpyDeviceToDevice, c->st));
      }
      b.e[i] = BcgsEntry{n, p, Ai, n, Qx[i], n, kcap, kd + i, s.alloc<double>(p), s.alloc<double>((size_t)kcap * kBcgsW), tau};
    }
    // the copies must be taken before entry 0 overwrites A: reorder so entry 0 runs on a copy too
    double* A0 = s.alloc<double>((size_t)n * p);
    FC_CUDA_TRY(cudaMemcpyAsync(A0, A, (size_t)n * p * 8, cudaMemcpyDeviceToDevice, c->st));
    b.e[0].A = A0;
    bcgs(b, c->st);
    int kh[3];
    FC_CUDA_TRY(cudaMemcpyAsync(kh, kd, 3 * sizeof(int), cudaMemcpyDeviceToHost, c->st));
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    std::vector<double> q0((size_t)n * kcap), qi((size_t)n * kcap);
    FC_CUDA_TRY(cudaMemcpy(q0.data(), Qx[0], q0.size() * 8, cudaMemcpyDeviceToHost));
    for (int i = 1; i < 3; ++i) {
      FC_CUDA_TRY(cudaMemcpy(qi.data(), Qx[i], qi.size() * 8, cudaMemcpyDeviceToHost));
      double d = 0;
      for (size_t t = 0; t < q0.size(); ++t) d = std::max(d, std::fabs(q0[t] - qi[t]));
      require(kh[i] == kh[0] && d < 1e-12, FC_ERR_CUDA,
              "batched orthonormalisation differs between identical entries (k " + std::to_string(kh[0]) + " vs " +
                  std::to_string(kh[i]) + ", maxdiff " + std::to_string(d) + ")");
    }
    *k_host = kh[0];
    return FC_OK;
  });
}

int fc_syev(fc_ctx c, int nb, const int* N, double* const* A, const int* lda, double* const* lam, double* const* Y,
            const int* ldy, const int* r) {
  return guard(c, [&]() {
    require(nb >= 1 && nb <= kMaxSyev && N && A && lda && lam && Y && ldy && r, FC_ERR_INVALID_ARG, "fc_syev args");
    Scratch s(c->st);
    SyevBatch b;
    b.nb = nb;
    int* rd = s.alloc<int>(nb);
    FC_CUDA_TRY(cudaMemcpyAsync(rd, r, nb * sizeof(int), cudaMemcpyHostToDevice, c->st));
    int maxN = 0;
    for (int i = 0; i < nb; ++i) {
      require(N[i] >= 1 && N[i] <= 1500 && lda[i] >= N[i] && ldy[i] >= N[i] && r[i] >= 0 && r[i] <= N[i] && A[i] &&
                  lam[i] && (Y[i] || r[i] == 0),
              FC_ERR_INVALID_ARG, "fc_syev entry");
      b.e[i] = SyevEntry{N[i], A[i], lda[i], s.alloc<double>(N[i]), s.alloc<double>(N[i]), lam[i], Y[i], ldy[i],
                         rd + i, s.alloc<double>((size_t)6 * N[i] * N[i])};
      maxN = std::max(maxN, N[i]);
    }
    syev_values(b, c->st);
    syev_vectors(b, maxN, c->st, r);
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    return FC_OK;
  });
}

int fc_profile_gemm(fc_ctx c, int enable, double* ms, double* flops, long long* launches) {
  return guard(c, [&]() {
    gemm_profile(enable != 0, ms, flops, launches);
    return FC_OK;
  });
}

int fc_profile_kernel(fc_ctx c, int kernel, int enable, double* ms, double* bytes, long long* launches) {
  return guard(c, [&]() {
    kprof_read(kernel, enable != 0, ms, bytes, launches);
    return FC_OK;
  });
}

int fc_kernel_launches(long long* count) {
  if (!count) return FC_ERR_INVALID_ARG;
  *count = fc::g_launches.load();
  return FC_OK;
}

int fc_create(fc_ctx* ctx, void* cuda_stream) {
  if (!ctx) return FC_ERR_INVALID_ARG;
  *ctx = nullptr;
  fc_ctx c = new fc_ctx_s();
  int rc = guard(c, [&]() {
    FC_CUDA_TRY(cudaGetDevice(&c->dev));
    c->st = (cudaStream_t)cuda_stream;
    FC_CUDA_TRY(cudaEventCreate(&c->e0));
    FC_CUDA_TRY(cudaEventCreate(&c->e1));
    cudaMemPool_t pool;
    FC_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, c->dev));
    uint64_t thr = UINT64_MAX;
    FC_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    // Pre-grow the pool once (the memory stays reserved): growing it inside a solve maps new
    // physical memory, a stall of hundreds of ms when a large scratch request fits no free chunk.
    // Default 16 GB (capped at half the free memory), FC_POOL_RESERVE_MB overrides (0 = off).
    uint64_t cur = 0;
    FC_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &cur));
    size_t fr = 0, tot = 0;
    FC_CUDA_TRY(cudaMemGetInfo(&fr, &tot));
    const char* env = getenv("FC_POOL_RESERVE_MB");
    size_t want = env ? (size_t)atoll(env) << 20 : (size_t)16 << 30;
    want = std::min(want, fr / 2);
    if (want > cur) {
      void* p = nullptr;
      FC_CUDA_TRY(cudaMallocAsync(&p, want, c->st));
      FC_CUDA_TRY(cudaFreeAsync(p, c->st));
      FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    }
    return FC_OK;
  });
  if (rc != FC_OK) {
    delete c;
    return rc;
  }
  *ctx = c;
  return FC_OK;
}

int fc_destroy(fc_ctx c) {
  if (!c) return FC_OK;
  cudaStreamSynchronize(c->st);
  if (c->st2) {
    cudaStreamSynchronize(c->st2);
    cudaStreamDestroy(c->st2);
  }
  c->lam.release();
  c->V.release();
  c->lamA.release();
  c->VA.release();
  for (auto& s : c->spec) {
    s.w.release(); s.U.release(); s.W.release(); s.E.release();
  }
  for (auto& s : c->spec2) {
    s.w.release(); s.U.release();
  }
  if (c->e0) cudaEventDestroy(c->e0);
  if (c->e1) cudaEventDestroy(c->e1);
  delete c;
  return FC_OK;
}

const char* fc_last_error(fc_ctx c) { return c ? c->err.c_str() : "NULL context"; }

int fc_set_stream(fc_ctx c, void* s) {
  if (!c) return FC_ERR_INVALID_ARG;
  c->st = (cudaStream_t)s;
  return FC_OK;
}

int sl_get_eigen(fc_ctx c, int mode, double* lam, double* V) {
  return guard(c, [&]() {
    require(mode >= 0 && mode < 3, FC_ERR_INVALID_ARG, "mode");
    require(c->n > 0 && c->have_eig[mode], FC_ERR_NOT_READY, "no eigenpairs");
    size_t n = c->n;
    if (lam) FC_CUDA_TRY(cudaMemcpyAsync(lam, c->lam_l(mode), n * 8, cudaMemcpyDeviceToDevice, c->st));
    if (V) FC_CUDA_TRY(cudaMemcpyAsync(V, c->V_l(mode), n * n * 8, cudaMemcpyDeviceToDevice, c->st));
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    return FC_OK;
  });
}

int sl_set_eigen(fc_ctx c, int n, int mode, const double* lam, const double* V, const fc_params* p) {
  return guard(c, [&]() {
    require(mode >= 0 && mode < 3 && n >= 2 && lam && V, FC_ERR_INVALID_ARG, "sl_set_eigen args");
    if (c->n != n) {
      c->n = n;
      c->lam.ensure((size_t)3 * n);
      c->V.ensure((size_t)3 * n * n);
      for (auto& h : c->have_eig) h = false;
      for (auto& h : c->have_A) h = false;
      for (auto& s : c->spec) {
        s.valid = false;
        s.basis = nullptr;
      }
    }
    if (p) {
      c->p = *p;
      c->have_params = true;
      if (p->precond_case == FC_PRECOND_B) c->spec[FC_G].basis = nullptr;
    }
    FC_CUDA_TRY(cudaMemcpyAsync(c->lam_l(mode), lam, (size_t)n * 8, cudaMemcpyDeviceToDevice, c->st));
    FC_CUDA_TRY(cudaMemcpyAsync(c->V_l(mode), V, (size_t)n * n * 8, cudaMemcpyDeviceToDevice, c->st));
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    c->have_eig[mode] = true;
    return FC_OK;
  });
}

int op_build_spectral_sinc(fc_ctx c, int which, double eps) {
  return guard(c, [&]() {
    build_spectral_sinc(c, which, eps);
    return FC_OK;
  });
}

int op_get_precond_basis(fc_ctx c, int mode, double* lam, double* V) {
  return guard(c, [&]() {
    require(mode >= 0 && mode < 3, FC_ERR_INVALID_ARG, "mode");
    require(c->n > 0 && c->have_A[mode], FC_ERR_NOT_READY, "no case-(A) preconditioner basis");
    const size_t n = c->n;
    if (lam)
      FC_CUDA_TRY(cudaMemcpyAsync(lam, c->lamA.p + (size_t)mode * n, n * 8, cudaMemcpyDeviceToDevice, c->st));
    if (V)
      FC_CUDA_TRY(cudaMemcpyAsync(V, c->VA.p + (size_t)mode * n * n, n * n * 8, cudaMemcpyDeviceToDevice, c->st));
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    return FC_OK;
  });
}

int op_set_precond_basis(fc_ctx c, int mode, const double* lam, const double* V) {
  return guard(c, [&]() {
    require(mode >= 0 && mode < 3 && lam && V, FC_ERR_INVALID_ARG, "op_set_precond_basis args");
    require(c->n > 0, FC_ERR_NOT_READY, "set the eigenpairs (n) first");
    const size_t n = c->n;
    c->lamA.ensure(3 * n);
    c->VA.ensure(3 * n * n);
    FC_CUDA_TRY(cudaMemcpyAsync(c->lamA.p + (size_t)mode * n, lam, n * 8, cudaMemcpyDeviceToDevice, c->st));
    FC_CUDA_TRY(cudaMemcpyAsync(c->VA.p + (size_t)mode * n * n, V, n * n * 8, cudaMemcpyDeviceToDevice, c->st));
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    c->have_A[mode] = true;
    if (c->have_A[0] && c->have_A[1] && c->have_A[2]) c->spec[FC_G].basis = c->VA.p;
    return FC_OK;
  });
}

int op_set_spectral_cp(fc_ctx c, int which, const fc_cp* in) {
  return guard(c, [&]() {
    require(which >= 0 && which < 4, FC_ERR_INVALID_ARG, "which");
    check_cp(c, in, "in");
    SpecCP& s = c->spec[which];
    const int n = c->n, r = in->rank;
    s.r = r;
    s.w.ensure(std::max(r, 1));
    s.U.ensure((size_t)3 * n * std::max(r, 1));
    fc_cp dst{};
    for (int l = 0; l < 3; ++l) {
      dst.n[l] = n; dst.U[l] = s.U.p + (size_t)l * n * r; dst.ld[l] = n;
    }
    dst.w = s.w.p; dst.rank = r; dst.cap = r;
    copy_cp_block(c->st, n, *in, dst, 0, 1.0);
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    s.valid = true;
    s.has_basis = false;
    return FC_OK;
  });
}

int op_get_spectral_cp(fc_ctx c, int which, fc_cp* out) {
  return guard(c, [&]() {
    require(which >= 0 && which < 4, FC_ERR_INVALID_ARG, "which");
    ensure_spectral(c, which);
    SpecCP& s = c->spec[which];
    require(s.valid, FC_ERR_NOT_READY, "spectral CP not set");
    check_cp(c, out, "out");
    if (out->cap < s.r) {
      out->rank = s.r;
      throw Error(FC_ERR_CAPACITY, "out.cap < spectral rank");
    }
    fc_cp src{};
    for (int l = 0; l < 3; ++l) {
      src.n[l] = c->n; src.U[l] = s.U.p + (size_t)l * c->n * s.r; src.ld[l] = c->n;
    }
    src.w = s.w.p; src.rank = s.r; src.cap = s.r;
    copy_cp_block(c->st, c->n, src, *out, 0, 1.0);
    out->rank = s.r;
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    return FC_OK;
  });
}

int op_spectral_rank(fc_ctx c, int which, int* rank, int* tucker) {
  return guard(c, [&]() {
    require(which >= 0 && which < 4, FC_ERR_INVALID_ARG, "which");
    ensure_spectral(c, which);
    SpecCP& s = c->spec[which];
    require(s.valid, FC_ERR_NOT_READY, "spectral CP not set");
    if (rank) *rank = s.r;
    if (tucker)
      for (int l = 0; l < 3; ++l) tucker[l] = s.tucker_rank[l];
    return FC_OK;
  });
}

int fracop_apply(fc_ctx c, int which, const fc_cp* x, fc_cp* y) {
  return guard(c, [&]() {
    require(which >= 0 && which < 4, FC_ERR_INVALID_ARG, "which");
    check_cp(c, x, "x");
    check_cp(c, y, "y");
    require(c->have_eig[0] && c->have_eig[1] && c->have_eig[2], FC_ERR_NOT_READY, "eigenpairs missing");
    ensure_spectral(c, which);
    const SpecCP& s = c->spec[which];
    require(s.valid, FC_ERR_NOT_READY, "spectral CP not set");
    long long need = (long long)s.r * x->rank;
    if (y->cap < need) {
      y->rank = (int)std::min<long long>(need, INT32_MAX);
      throw Error(FC_ERR_CAPACITY, "y.cap < r * x.rank");
    }
    apply_plain(c, s, *x, *y);
    return FC_OK;
  });
}

int precond_apply(fc_ctx c, const fc_cp* x, fc_cp* y) { return fracop_apply(c, FC_G, x, y); }

int cp_dot(fc_ctx c, const fc_cp* x, const fc_cp* y, double* out) {
  return guard(c, [&]() {
    check_cp(c, x, "x");
    check_cp(c, y, "y");
    require(out != nullptr, FC_ERR_INVALID_ARG, "out NULL");
    *out = dot_plain(c, *x, *y);
    return std::isfinite(*out) ? FC_OK : FC_ERR_NAN;
  });
}

int cp_axpy(fc_ctx c, const fc_cp* x, double a, const fc_cp* y, fc_cp* z) {
  return guard(c, [&]() {
    check_cp(c, x, "x");
    check_cp(c, y, "y");
    check_cp(c, z, "z");
    int need = x->rank + y->rank;
    if (z->cap < need) {
      z->rank = need;
      throw Error(FC_ERR_CAPACITY, "z.cap < x.rank + y.rank");
    }
    copy_cp_block(c->st, c->n, *x, *z, 0, 1.0);
    copy_cp_block(c->st, c->n, *y, *z, x->rank, a);
    z->rank = need;
    FC_CUDA_TRY(cudaStreamSynchronize(c->st));
    return FC_OK;
  });
}

int fc_dgemm(fc_ctx c, int transA, int transB, int M, int N, int K, double alpha, const double* A, int lda,
             const double* B, int ldb, double beta, double* C, int ldc) {
  return guard(c, [&]() {
    require(M >= 0 && N >= 0 && K >= 0, FC_ERR_INVALID_ARG, "dims");
    FC_CUDA_TRY(cudaEventRecord(c->e0, c->st));
    dgemm(c->st, transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    FC_CUDA_TRY(cudaEventRecord(c->e1, c->st));
    c->k_flops = 2.0 * M * (double)N * K;
    c->k_bytes = 8.0 * ((double)M * K + (double)K * N + (double)M * N * (beta != 0 ? 2 : 1));
    c->k_launches = 1;
    return FC_OK;
  });
}

int fc_dgemm_streamk(fc_ctx c, int transA, int transB, int M, int N, int K, double alpha, const double* A, int lda,
                     const double* B, int ldb, double beta, double* C, int ldc) {
  return guard(c, [&]() {
    require(M >= 0 && N >= 0 && K >= 0, FC_ERR_INVALID_ARG, "dims");
    GemmArgs a;
    a.transA = transA;
    a.transB = transB;
    a.alpha = alpha;
    a.beta = beta;
    a.streamk = 1;
    a.nbatch = 1;
    a.b[0] = GemmBatch{M, N, K, A, lda, B, ldb, C, ldc, nullptr, 0, nullptr};
    FC_CUDA_TRY(cudaEventRecord(c->e0, c->st));
    gemm(a, c->st);
    FC_CUDA_TRY(cudaEventRecord(c->e1, c->st));
    c->k_flops = 2.0 * M * (double)N * K;
    c->k_bytes = 8.0 * ((double)M * K + (double)K * N + (double)M * N * (beta != 0 ? 2 : 1));
    c->k_launches = 1;
    return FC_OK;
  });
}

int fc_dgemm_splitk(fc_ctx c, int transA, int transB, int M, int N, int K, double alpha, const double* A, int lda,
                    const double* B, int ldb, double beta, double* C, int ldc, int splitk) {
  return guard(c, [&]() {
    require(M >= 0 && N >= 0 && K >= 0, FC_ERR_INVALID_ARG, "dims");
    require(splitk >= 1, FC_ERR_INVALID_ARG, "splitk >= 1");
    FC_CUDA_TRY(cudaEventRecord(c->e0, c->st));
    dgemm(c->st, transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splitk);
    FC_CUDA_TRY(cudaEventRecord(c->e1, c->st));
    c->k_flops = 2.0 * M * (double)N * K;
    c->k_bytes = 8.0 * ((double)M * K + (double)K * N + (double)M * N * (beta != 0 ? 2 : 1));
    c->k_launches = 1;
    return FC_OK;
  });
}

int fc_last_kernel_stats(fc_ctx c, double* ms, double* flops, double* bytes, int* launches) {
  return guard(c, [&]() {
    float t = 0;
    FC_CUDA_TRY(cudaEventSynchronize(c->e1));
    FC_CUDA_TRY(cudaEventElapsedTime(&t, c->e0, c->e1));
    if (ms) *ms = t;
    if (flops) *flops = c->k_flops;
    if (bytes) *bytes = c->k_bytes;
    if (launches) *launches = c->k_launches;
    return FC_OK;
  });
}

}  // extern "C"
