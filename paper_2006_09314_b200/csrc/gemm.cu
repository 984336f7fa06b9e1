// Batched FP64 GEMM on the FP64 tensor pipe (DMMA) for sm_100a.
//
// Hot use: the mode transforms of the factored operator apply [P:597-623]
//   forward  W_l = V_l^T X_l          (S5)
//   inverse  Y_l = V_l (U_F (.) W_l)  (S6+S7, Khatri-Rao B operand fused into the tile load,
//                                      column normalisation fused into the epilogue, S8)
// and every small contraction of the truncation pipeline (Grams, projections).
//
// tcgen05.mma has no f64 kind, so FP64 tensor work on sm_100a is the warp-level
// mma.sync.m8n8k4.f64 (SASS: DMMA.8x8x4).  Tiles: CTA 64x64, BK = 16, 4 warps each owning a
// 32x32 sub-tile (4x4 DMMA fragments, 32 fp64 accumulators per thread), operands staged
// global -> shared with cp.async in a 3-stage ring (zero-filled at ragged edges).
#include "common.cuh"

namespace fc {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, PAD = 8, STAGES = 3, NT = 128;
constexpr int LDS = BM + PAD;  // 72 doubles: k-rows land on alternating bank halves
constexpr int STAGE_ELEMS = BK * LDS;

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int src_bytes = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void load_tile_A(double* As, const GemmBatch& g, int transA, int m0, int k0,
                                            int kend, int tid) {
#pragma unroll
  for (int i = 0; i < (BK * BM) / NT; ++i) {
    int idx = tid + i * NT;
    int mm, kk;
    if (!transA) { mm = idx % BM; kk = idx / BM; }
    else         { kk = idx % BK; mm = idx / BK; }
    int m = m0 + mm, k = k0 + kk;
    bool ok = (m < g.M) && (k < kend);
    const double* src = ok ? (transA ? g.A + (size_t)k + (size_t)m * g.lda
                                     : g.A + (size_t)m + (size_t)k * g.lda)
                           : g.A;
    cp_async8(As + kk * LDS + mm, src, ok);
  }
}

__device__ __forceinline__ double spectral_f(int kind, double alpha, double beta, double lam) {
  if (kind == FC_F) return beta * pow(lam, alpha) + pow(lam, -alpha);
  if (kind == FC_G) return 1.0 / (beta * pow(lam, alpha) + pow(lam, -alpha));
  if (kind == FC_POW_PLUS) return pow(lam, alpha);
  return pow(lam, -alpha);
}

// generated operand: A(m, k) = f((l1[m % n1] + l2[m / n1]) + l3[k])  (never stored)
__device__ __forceinline__ void gen_tile_A(double* As, const GemmBatch& g, const GenA& gen, int m0, int k0, int kend,
                                           int tid) {
#pragma unroll 2
  for (int i = 0; i < (BK * BM) / NT; ++i) {
    int idx = tid + i * NT;
    int mm = idx % BM, kk = idx / BM;
    int m = m0 + mm, k = k0 + kk;
    double v = 0.0;
    if (m < g.M && k < kend) {
      int i1 = m % gen.n1, i2 = m / gen.n1;
      double lam = (__ldg(gen.l1 + i1) + __ldg(gen.l2 + i2)) + __ldg(gen.l3 + k);
      v = spectral_f(gen.kind, gen.alpha, gen.beta, lam);
    }
    As[kk * LDS + mm] = v;
  }
}

__device__ __forceinline__ void load_tile_B(double* Bs, double* Ks, const GemmBatch& g, int transB, int krR,
                                            int n0, int k0, int kend, int tid) {
  if (krR > 0) {
    // Khatri-Rao operand: column c = k_F * R + j  ->  u_F[:, k_F] (.) W[:, j].  Both factors are
    // gathered by cp.async into two tiles; the product is formed at fragment-load time.
#pragma unroll
    for (int i = 0; i < (BK * BN) / NT; ++i) {
      int idx = tid + i * NT;
      int kk = idx % BK, nn = idx / BK;
      int c = n0 + nn, k = k0 + kk;
      bool ok = (c < g.N) && (k < kend);
      int kf = ok ? c / krR : 0, j = ok ? c - kf * krR : 0;
      cp_async8(Bs + kk * LDS + nn, ok ? g.B + (size_t)k + (size_t)j * g.ldb : g.B, ok);
      cp_async8(Ks + kk * LDS + nn, ok ? g.krU + (size_t)k + (size_t)kf * g.ldkr : g.krU, ok);
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < (BK * BN) / NT; ++i) {
    int idx = tid + i * NT;
    int nn, kk;
    if (!transB) { kk = idx % BK; nn = idx / BK; }
    else         { nn = idx % BN; kk = idx / BN; }
    int c = n0 + nn, k = k0 + kk;
    bool ok = (c < g.N) && (k < kend);
    const double* src = ok ? (transB ? g.B + (size_t)c + (size_t)k * g.ldb
                                     : g.B + (size_t)k + (size_t)c * g.ldb)
                           : g.B;
    cp_async8(Bs + kk * LDS + nn, src, ok);
  }
}

template <bool KR, bool GEN>
__global__ void __launch_bounds__(NT) dgemm_dmma_kernel(const __grid_constant__ GemmArgs args) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * STAGE_ELEMS;
  double* Ks = smem + 2 * STAGES * STAGE_ELEMS;   // only used when KR

  const int bz = blockIdx.z;
  const int bi = bz / args.splitk;
  const int ks = bz - bi * args.splitk;
  const GemmBatch& g = args.b[bi];
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  if (m0 >= g.M || n0 >= g.N) return;

  int kchunk = ((g.K + args.splitk - 1) / args.splitk + BK - 1) / BK * BK;
  const int kbeg = ks * kchunk;
  const int kend = min(g.K, kbeg + kchunk);
  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  const int fr = lane >> 2, fc4 = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // prologue
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) {
      if (GEN) gen_tile_A(As + s * STAGE_ELEMS, g, args.gen, m0, kbeg + s * BK, kend, tid);
      else load_tile_A(As + s * STAGE_ELEMS, g, args.transA, m0, kbeg + s * BK, kend, tid);
      load_tile_B(Bs + s * STAGE_ELEMS, Ks + s * STAGE_ELEMS, g, args.transB, KR ? args.krR : 0, n0,
                  kbeg + s * BK, kend, tid);
    }
    cp_async_commit();
  }

  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int st = kt % STAGES;
    // issue the load of tile kt + STAGES - 1 into the slot freed at iteration kt - 1
    {
      int nt = kt + STAGES - 1;
      if (nt < nk) {
        int sl = nt % STAGES;
        if (GEN) gen_tile_A(As + sl * STAGE_ELEMS, g, args.gen, m0, kbeg + nt * BK, kend, tid);
        else load_tile_A(As + sl * STAGE_ELEMS, g, args.transA, m0, kbeg + nt * BK, kend, tid);
        load_tile_B(Bs + sl * STAGE_ELEMS, Ks + sl * STAGE_ELEMS, g, args.transB, KR ? args.krR : 0, n0,
                    kbeg + nt * BK, kend, tid);
      }
      cp_async_commit();
    }
    const double* a_s = As + st * STAGE_ELEMS;
    const double* b_s = Bs + st * STAGE_ELEMS;
    const double* k_s = Ks + st * STAGE_ELEMS;
#pragma unroll
    for (int kq = 0; kq < BK; kq += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = a_s[(kq + fc4) * LDS + wm + i * 8 + fr];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int o = (kq + fc4) * LDS + wn + j * 8 + fr;
        bf[j] = KR ? b_s[o] * k_s[o] : b_s[o];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: fragment (i, j) element e -> row wm+i*8+fr, col wn+j*8+2*fc4+e
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      int c = n0 + wn + j * 8 + 2 * fc4 + e;
      if (c >= g.N) continue;
      double cs = g.colscale ? g.colscale[c] : 1.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int r = m0 + wm + i * 8 + fr;
        if (r >= g.M) continue;
        double v = args.alpha * cs * acc[i][j][e];
        double* dst = g.C + (size_t)r + (size_t)c * g.ldc;
        if (args.splitk > 1) atomicAdd(dst, v);
        else if (args.beta == 0.0) *dst = v;
        else *dst = v + args.beta * *dst;
      }
    }
  }
}

}  // namespace

void gemm(const GemmArgs& a, cudaStream_t st) {
  if (a.nbatch <= 0) return;
  int maxM = 0, maxN = 0;
  for (int i = 0; i < a.nbatch; ++i) {
    maxM = std::max(maxM, a.b[i].M);
    maxN = std::max(maxN, a.b[i].N);
  }
  if (maxM == 0 || maxN == 0) return;
  static bool attr = false;
  const int smem2 = 2 * STAGES * STAGE_ELEMS * (int)sizeof(double);
  const int smem3 = 3 * STAGES * STAGE_ELEMS * (int)sizeof(double);
  if (!attr) {
    FC_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
    FC_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3));
    FC_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
    attr = true;
  }
  dim3 grid(cdiv(maxM, BM), cdiv(maxN, BN), a.nbatch * a.splitk);
  require(grid.y <= 65535 && grid.z <= 65535, FC_ERR_INVALID_ARG, "gemm grid too large");
  if (a.gen.kind >= 0) dgemm_dmma_kernel<false, true><<<grid, NT, smem2, st>>>(a);
  else if (a.krR > 0) dgemm_dmma_kernel<true, false><<<grid, NT, smem3, st>>>(a);
  else dgemm_dmma_kernel<false, false><<<grid, NT, smem2, st>>>(a);
  FC_CHECK_LAUNCH();
}

void dgemm(cudaStream_t st, int transA, int transB, int M, int N, int K, double alpha, const double* A,
           int lda, const double* B, int ldb, double beta, double* C, int ldc, int splitk) {
  GemmArgs a;
  a.transA = transA;
  a.transB = transB;
  a.alpha = alpha;
  a.beta = beta;
  a.splitk = splitk;
  a.nbatch = 1;
  a.b[0] = GemmBatch{M, N, K, A, lda, B, ldb, C, ldc, nullptr, 0, nullptr};
  gemm(a, st);
}

}  // namespace fc
