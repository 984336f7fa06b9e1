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
//
// Split-K is deterministic: the partial tiles of one output tile are summed in split order,
// either through distributed shared memory inside a (1, 1, splitk) cluster (splitk <= 8) or
// through a global workspace by the last CTA to arrive (splitk > 8).  No atomics touch C, so
// repeated runs are bit-identical and C needs no pre-zeroing.
#include <algorithm>
#include <cooperative_groups.h>
#include <cstdlib>
#include <map>
#include <mutex>
#include "common.cuh"

namespace fc {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, PAD = 4, STAGES = 3, NT = 128;
// 68 doubles = 4 (mod 16): a fragment load (lanes fr = 0..7 along m, fc4 = 0..3 along k) then
// touches 16 distinct 8-byte bank pairs per half-warp (72 = 8 (mod 16) put fc4 and fc4 + 2 on
// the same banks: a 2-way conflict on every A and B fragment load)
constexpr int LDS = BM + PAD;
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

__device__ __forceinline__ void cp_async16s(double* smem, const double* gmem, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}

// a BK x 64 tile contiguous along its 64-wide dimension (A not transposed, B transposed), k-major
// in shared memory: 16-byte chunks (pairs along the contiguous dimension; ragged edges
// zero-filled by the transfer size)
__device__ __forceinline__ void load_tile_vec(double* T, const double* base, int ld, int r0, int rmax, int k0,
                                              int kend, int tid) {
#pragma unroll
  for (int i = 0; i < (BK * BM) / (2 * NT); ++i) {
    const int c = tid + i * NT;
    const int rr = (c % (BM / 2)) * 2, kk = c / (BM / 2);
    const int r = r0 + rr, k = k0 + kk;
    const int nr = (k < kend) ? max(0, min(2, rmax - r)) : 0;
    cp_async16s(T + kk * LDS + rr, nr > 0 ? base + (size_t)r + (size_t)k * ld : base, nr * 8);
  }
}

__device__ __forceinline__ void load_tile_A(double* As, const GemmBatch& g, const double* gA, int transA, int m0,
                                            int k0, int kend, int tid, bool vec = false) {
  if (!transA && vec) {
    load_tile_vec(As, gA, g.lda, m0, g.M, k0, kend, tid);
    return;
  }
#pragma unroll
  for (int i = 0; i < (BK * BM) / NT; ++i) {
    int idx = tid + i * NT;
    int mm, kk;
    if (!transA) { mm = idx % BM; kk = idx / BM; }
    else         { kk = idx % BK; mm = idx / BK; }
    int m = m0 + mm, k = k0 + kk;
    bool ok = (m < g.M) && (k < kend);
    const double* src = ok ? (transA ? gA + (size_t)k + (size_t)m * g.lda
                                     : gA + (size_t)m + (size_t)k * g.lda)
                           : gA;
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

__device__ __forceinline__ void load_tile_B(double* Bs, double* Ks, const GemmBatch& g, const double* gB,
                                            const double* gK, int transB, int krR, int n0, int k0, int kend,
                                            int tid, bool vec = false) {
  if (krR == 0 && transB && vec) {
    load_tile_vec(Bs, gB, g.ldb, n0, g.N, k0, kend, tid);
    return;
  }
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
      cp_async8(Bs + kk * LDS + nn, ok ? gB + (size_t)k + (size_t)j * g.ldb : gB, ok);
      cp_async8(Ks + kk * LDS + nn, ok ? gK + (size_t)k + (size_t)kf * g.ldkr : gK, ok);
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
    const double* src = ok ? (transB ? gB + (size_t)c + (size_t)k * g.ldb
                                     : gB + (size_t)k + (size_t)c * g.ldb)
                           : gB;
    cp_async8(Bs + kk * LDS + nn, src, ok);
  }
}

// ---- epilogue shared by both kernels ---------------------------------------------------
// Fragment element (i, j, e) of a thread lives at row wm + i*8 + fr, col wn + j*8 + 2*fc4 + e of
// the CTA tile; slot s = (i*4 + j)*2 + e.  WM = warps along m.
template <int WM>
__device__ __forceinline__ void slot_rc(int tid, int s, int& r, int& c) {
  const int lane = tid & 31, warp = tid >> 5;
  const int i = s >> 3, j = (s >> 1) & 3, e = s & 1;
  r = (warp % WM) * 32 + i * 8 + (lane >> 2);
  c = (warp / WM) * 32 + j * 8 + 2 * (lane & 3) + e;
}

__device__ __forceinline__ void put_elem(const GemmArgs& args, const GemmBatch& g, int ri, int r, int c, double v) {
  if (r >= g.M || c >= g.N) return;
  const double cs = g.colscale ? g.colscale[c + (size_t)ri * g.sS] : 1.0;
  const double val = args.alpha * cs * v;
  double* dst = g.C + (size_t)ri * g.sC + (size_t)r + (size_t)c * g.ldc;
  if (args.beta == 0.0) *dst = val;
  else *dst = val + args.beta * *dst;
}

// NTH threads, WM warps along m; `red` = the CTA's (now idle) pipeline shared memory, at least
// 32 * NTH doubles.  ks = this CTA's split, tile = linear output-tile index (workspace mode).
template <int NTH, int WM>
__device__ __forceinline__ void tile_epilogue(const double (&acc)[4][4][2], const GemmArgs& args, const GemmBatch& g,
                                              int ri, int m0, int n0, int ks, long long tile, double* red) {
  const int tid = threadIdx.x;
  if (args.kmode == 0) {
#pragma unroll
    for (int s = 0; s < 32; ++s) {
      int r, c;
      slot_rc<WM>(tid, s, r, c);
      put_elem(args, g, ri, m0 + r, n0 + c, acc[s >> 3][(s >> 1) & 3][s & 1]);
    }
    return;
  }
  const int S = args.splitk;
  if (args.kmode == 1) {
    // cluster (1, 1, S): rank q holds split q.  Every CTA parks its partial tile in its own
    // shared memory; CTA q then sums slots q, q + S, ... over ranks 0..S-1 in that order.
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
#pragma unroll
    for (int s = 0; s < 32; ++s) red[s * NTH + tid] = acc[s >> 3][(s >> 1) & 3][s & 1];
    cl.sync();
    for (int s = ks; s < 32; s += S) {
      // all S remote loads in flight at once (~200-cycle DSMEM latency each), then the sum in
      // split order
      double pv[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) pv[q] = q < S ? cl.map_shared_rank(red, q)[s * NTH + tid] : 0.0;
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (q < S) v += pv[q];
      int r, c;
      slot_rc<WM>(tid, s, r, c);
      put_elem(args, g, ri, m0 + r, n0 + c, v);
    }
    cl.sync();   // peers may still read this CTA's partial
    return;
  }
  // workspace: partial (tile, ks) at ws[((tile * S + ks) * 32 + s) * NTH + tid]; the last CTA to
  // arrive sums splits 0..S-1 in order and resets the tile's counter
  __shared__ int last_s;
  double* wp = args.ws + ((size_t)tile * S + ks) * 32 * NTH;
#pragma unroll
  for (int s = 0; s < 32; ++s) wp[s * NTH + tid] = acc[s >> 3][(s >> 1) & 3][s & 1];
  __threadfence();
  __syncthreads();
  if (tid == 0) last_s = atomicAdd(args.cnt + tile, 1) == S - 1;
  __syncthreads();
  if (!last_s) return;
  __threadfence();
  const double* w0 = args.ws + (size_t)tile * S * 32 * NTH;
  for (int s = 0; s < 32; ++s) {
    double v = 0.0;
    for (int q0 = 0; q0 < S; q0 += 16) {   // 16 loads in flight, summed in split order
      double pv[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) pv[q] = q0 + q < S ? __ldcg(w0 + ((size_t)(q0 + q) * 32 + s) * NTH + tid) : 0.0;
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (q0 + q < S) v += pv[q];
    }
    int r, c;
    slot_rc<WM>(tid, s, r, c);
    put_elem(args, g, ri, m0 + r, n0 + c, v);
  }
  if (tid == 0) args.cnt[tile] = 0;
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
  const int ei = bi / args.rep, ri = bi - ei * args.rep;
  const GemmBatch& g = args.b[ei];
  const double* gA = g.A + (size_t)ri * g.sA;
  const double* gB = g.B + (size_t)ri * g.sB;
  const double* gK = g.krU + (size_t)ri * g.sK;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int Meff = g.dynM ? min(g.M, *g.dynM) : g.M;
  const int Keff = g.dynK ? min(g.K, *g.dynK) : g.K;
  // uniform over the splits of a tile (same cluster / same counter): all leave together
  if (m0 >= Meff || n0 >= g.N) return;

  int kchunk = ((Keff + args.splitk - 1) / args.splitk + BK - 1) / BK * BK;
  const int kbeg = ks * kchunk;
  const int kend = min(Keff, kbeg + kchunk);
  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;   // an empty split adds zeros
  // 16-byte staging needs an even leading dimension and a 16-byte aligned base
  const bool vecA = ((g.lda & 1) == 0) && (((uintptr_t)gA & 15) == 0);
  const bool vecB = ((g.ldb & 1) == 0) && (((uintptr_t)gB & 15) == 0);

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
      else load_tile_A(As + s * STAGE_ELEMS, g, gA, args.transA, m0, kbeg + s * BK, kend, tid, vecA);
      load_tile_B(Bs + s * STAGE_ELEMS, Ks + s * STAGE_ELEMS, g, gB, gK, args.transB, KR ? args.krR : 0, n0,
                  kbeg + s * BK, kend, tid, vecB);
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
        else load_tile_A(As + sl * STAGE_ELEMS, g, gA, args.transA, m0, kbeg + nt * BK, kend, tid, vecA);
        load_tile_B(Bs + sl * STAGE_ELEMS, Ks + sl * STAGE_ELEMS, g, gB, gK, args.transB, KR ? args.krR : 0, n0,
                    kbeg + nt * BK, kend, tid, vecB);
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
  __syncthreads();   // the pipeline buffers become the reduction buffer
  const long long tile = ((long long)bi * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  tile_epilogue<NT, 2>(acc, args, g, ri, m0, n0, ks, tile, smem);
}

// launch with the split-K reduction mode's cluster shape (kmode 1: (1, 1, splitk))
void launch_gemm_kernel(void (*kern)(GemmArgs), const GemmArgs& a, dim3 grid, int nt, int smem, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(nt, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  if (a.kmode == 1) {
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = a.splitk;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  FC_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a));
  FC_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------------------
// Big-tile variant: CTA 128x128, BK = 16, 16 warps (4 x 4) each owning 32x32 (4x4 DMMA
// fragments, 64 fp64 accumulators per thread), 3-stage cp.async ring.  Operand tiles are
// stored k-major ([k][m], ld 136) when the operand is contiguous along m/n, and m/n-major
// ([m][k], ld 20) when it is contiguous along k, so that 16-byte cp.async can be used for
// K-contiguous operands and every fragment load is at most 2-way banked.
namespace big {
constexpr int BM = 128, BN = 128, BK = 16, NT = 512, STAGES = 3;
constexpr int LDK = BM + 4;        // k-major row length 132 = 4 (mod 16): conflict-free fragment
                                   // loads (136 = 8 (mod 16) was 2-way conflicted, fc4 vs fc4 + 2)
constexpr int LDM = BK + 4;        // m/n-major row length (20)
constexpr int TILE = BM * LDM > BK * LDK ? BM * LDM : BK * LDK;   // 2560 doubles
constexpr int RED = 32 * NT;       // split-K reduction buffer (doubles), aliases the pipeline

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}

// load a ROWS x BK operand tile; `kcontig`: element (r, k) at base + k + r*ld (K contiguous),
// else at base + r + k*ld.  Stored k-major if !kcontig, r-major if kcontig.
template <bool KCONTIG>
__device__ __forceinline__ void load_op(double* T, const double* base, int ld, int r0, int rmax, int k0, int kend,
                                        int tid, bool vec) {
  if (KCONTIG) {
    // 128 rows x 16 k: 8 x 16-byte chunks per row -> 1024 chunks, 2 per thread
#pragma unroll
    for (int i = 0; i < 1024 / NT; ++i) {
      const int idx = tid + i * NT;
      const int rr = idx >> 3, kk = (idx & 7) * 2;
      const int r = r0 + rr, k = k0 + kk;
      double* dst = T + rr * LDM + kk;
      if (vec) {
        const int nk = (r < rmax) ? max(0, min(2, kend - k)) : 0;
        cp_async16(dst, nk > 0 ? base + (size_t)k + (size_t)r * ld : base, nk * 8);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool ok = (r < rmax) && (k + e < kend);
          cp_async8(dst + e, ok ? base + (size_t)(k + e) + (size_t)r * ld : base, ok);
        }
      }
    }
  } else {
    // 16 k x 128 rows: 64 x 16-byte chunks per k-row -> 1024 chunks, 2 per thread
#pragma unroll
    for (int i = 0; i < 1024 / NT; ++i) {
      const int idx = tid + i * NT;
      const int kk = idx >> 6, rr = (idx & 63) * 2;
      const int r = r0 + rr, k = k0 + kk;
      double* dst = T + kk * LDK + rr;
      if (vec) {
        const int nr = (k < kend) ? max(0, min(2, rmax - r)) : 0;
        cp_async16(dst, nr > 0 ? base + (size_t)r + (size_t)k * ld : base, nr * 8);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool ok = (r + e < rmax) && (k < kend);
          cp_async8(dst + e, ok ? base + (size_t)(r + e) + (size_t)k * ld : base, ok);
        }
      }
    }
  }
}

// Khatri-Rao operand tile (K contiguous): column c -> W[:, c % R] and U[:, c / R].  The two
// column base pointers of each of a thread's chunk rows are fixed for the whole K loop, so they
// are formed once (no division per tile); 16-byte cp.async when both operands allow it.
struct KRRows {
  const double* b[2];
  const double* k[2];
  bool ok[2];
};
__device__ __forceinline__ KRRows kr_rows(const GemmBatch& g, const double* gB, const double* gK, int krR, int n0,
                                          int tid) {
  KRRows p;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int c = n0 + (tid >> 3) + i * (NT >> 3);
    p.ok[i] = c < g.N;
    const int kf = p.ok[i] ? c / krR : 0, j = p.ok[i] ? c - kf * krR : 0;
    p.b[i] = gB + (size_t)j * g.ldb;
    p.k[i] = gK + (size_t)kf * g.ldkr;
  }
  return p;
}
__device__ __forceinline__ void load_kr(double* T, double* TK, const KRRows& p, const double* gB, const double* gK,
                                        int k0, int kend, int tid, bool vec) {
  const int kk = (tid & 7) * 2, k = k0 + kk;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int rr = (tid >> 3) + i * (NT >> 3);
    double* dB = T + rr * LDM + kk;
    double* dK = TK + rr * LDM + kk;
    if (vec) {
      const int nk = p.ok[i] ? max(0, min(2, kend - k)) : 0;
      cp_async16(dB, nk > 0 ? p.b[i] + k : gB, nk * 8);
      cp_async16(dK, nk > 0 ? p.k[i] + k : gK, nk * 8);
    } else {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool ok = p.ok[i] && (k + e < kend);
        cp_async8(dB + e, ok ? p.b[i] + k + e : gB, ok);
        cp_async8(dK + e, ok ? p.k[i] + k + e : gK, ok);
      }
    }
  }
}

template <int TA, int TB, bool KR>
__global__ void __launch_bounds__(NT, 1) dgemm_big_kernel(const __grid_constant__ GemmArgs args) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * TILE;
  double* Ks = smem + 2 * STAGES * TILE;
  const int bz = blockIdx.z;
  const int bi = bz / args.splitk, ks = bz - bi * args.splitk;
  const int ei = bi / args.rep, ri = bi - ei * args.rep;
  const GemmBatch& g = args.b[ei];
  const double* gA = g.A + (size_t)ri * g.sA;
  const double* gB = g.B + (size_t)ri * g.sB;
  const double* gK = g.krU + (size_t)ri * g.sK;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  if (m0 >= g.M || n0 >= g.N) return;   // uniform over the splits of a tile
  const int kchunk = ((g.K + args.splitk - 1) / args.splitk + BK - 1) / BK * BK;
  const int kbeg = ks * kchunk, kend = min(g.K, kbeg + kchunk);
  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
  const int fr = lane >> 2, fc4 = lane & 3;
  // 16-byte transfers need an even leading dimension and 16-byte aligned base pointers
  const bool vecA = ((g.lda & 1) == 0) && (((uintptr_t)gA & 15) == 0);
  const bool vecB = ((g.ldb & 1) == 0) && (((uintptr_t)gB & 15) == 0);
  constexpr bool AK = TA == 1;    // A contiguous along k
  constexpr bool BKc = TB == 0;   // B contiguous along k

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  KRRows krp{};
  bool vecKR = false;
  if (KR) {
    krp = kr_rows(g, gB, gK, args.krR, n0, tid);
    vecKR = ((g.ldb & 1) == 0) && ((g.ldkr & 1) == 0) && (((uintptr_t)gB & 15) == 0) && (((uintptr_t)gK & 15) == 0);
  }
  auto issue = [&](int s, int kt) {
    const int k0 = kbeg + kt * BK;
    load_op<AK>(As + s * TILE, gA, g.lda, m0, g.M, k0, kend, tid, vecA);
    if (KR) load_kr(Bs + s * TILE, Ks + s * TILE, krp, gB, gK, k0, kend, tid, vecKR);
    else load_op<BKc>(Bs + s * TILE, gB, g.ldb, n0, g.N, k0, kend, tid, vecB);
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) issue(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nt = kt + STAGES - 1;
      if (nt < nk) issue(nt % STAGES, nt);
      cp_async_commit();
    }
    const int st = kt % STAGES;
    const double* a_s = As + st * TILE;
    const double* b_s = Bs + st * TILE;
    const double* k_s = Ks + st * TILE;
#pragma unroll
    for (int kq = 0; kq < BK; kq += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm + i * 8 + fr, k = kq + fc4;
        af[i] = AK ? a_s[m * LDM + k] : a_s[k * LDK + m];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int nn = wn + j * 8 + fr, k = kq + fc4;
        if (KR) {
          const int o = nn * LDM + k;
          bf[j] = b_s[o] * k_s[o];
        } else {
          bf[j] = BKc ? b_s[nn * LDM + k] : b_s[k * LDK + nn];
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  const long long tile = ((long long)bi * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  tile_epilogue<NT, 4>(acc, args, g, ri, m0, n0, ks, tile, smem);
}

// Stream-K variant of the 128x128 kernel (kmode 3): one persistent CTA per SM; the launch's
// (tile, k-step) iterations — tiles in (entry, rep, n-tile, m-tile) order, K / 16 steps each,
// all entries of one shape — are cut into gridDim.x equal contiguous ranges, so every SM gets
// the same number of k-steps whatever the tile count (192 tiles on 148 SMs: 83 steps per CTA
// instead of two waves of 64).  A range that starts inside a tile produces a partial tile:
// written to the CTA's workspace slot and published through its flag.  The CTA whose range holds
// the tile's first k-step owns the tile: it adds the partials of the following CTAs in CTA order
// (a fixed order: bit-identical run to run), resets their flags and runs the usual epilogue.
// A CTA's partial is the FIRST thing it computes and its wait comes LAST, and it only ever waits
// for CTAs with a higher index, so with any two CTAs resident the chain unwinds: no deadlock.
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

template <int TA, int TB>
__global__ void __launch_bounds__(NT, 1) dgemm_big_streamk_kernel(const __grid_constant__ GemmArgs args) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * TILE;
  const GemmBatch& g0 = args.b[0];
  const int tm = (g0.M + BM - 1) / BM, tn = (g0.N + BN - 1) / BN;
  const int kiters = (g0.K + BK - 1) / BK;
  const long long ntiles = (long long)args.nbatch * args.rep * tm * tn;
  const long long total = ntiles * kiters;
  const int P = gridDim.x, cta = blockIdx.x;
  auto range_begin = [&](int b) { return total * b / P; };
  long long it = range_begin(cta);
  const long long it1 = range_begin(cta + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
  const int fr = lane >> 2, fc4 = lane & 3;
  constexpr bool AK = TA == 1;    // A contiguous along k
  constexpr bool BKc = TB == 0;   // B contiguous along k
  while (it < it1) {
    const long long t = it / kiters;
    const int kb = (int)(it - t * kiters);
    const int ke = (int)min((long long)kiters, kb + (it1 - it));
    const int mt = (int)(t % tm), nt_ = (int)((t / tm) % tn);
    const int bi = (int)(t / ((long long)tm * tn));
    const int ei = bi / args.rep, ri = bi - ei * args.rep;
    const GemmBatch& g = args.b[ei];
    const double* gA = g.A + (size_t)ri * g.sA;
    const double* gB = g.B + (size_t)ri * g.sB;
    const int m0 = mt * BM, n0 = nt_ * BN;
    const int kbeg = kb * BK, kend = min(g.K, ke * BK);
    const int nk = ke - kb;
    const bool vecA = ((g.lda & 1) == 0) && (((uintptr_t)gA & 15) == 0);
    const bool vecB = ((g.ldb & 1) == 0) && (((uintptr_t)gB & 15) == 0);
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    auto issue = [&](int s, int kt) {
      const int k0 = kbeg + kt * BK;
      load_op<AK>(As + s * TILE, gA, g.lda, m0, g.M, k0, kend, tid, vecA);
      load_op<BKc>(Bs + s * TILE, gB, g.ldb, n0, g.N, k0, kend, tid, vecB);
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < nk) issue(s, s);
      cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      {
        const int nx = kt + STAGES - 1;
        if (nx < nk) issue(nx % STAGES, nx);
        cp_async_commit();
      }
      const int st = kt % STAGES;
      const double* a_s = As + st * TILE;
      const double* b_s = Bs + st * TILE;
#pragma unroll
      for (int kq = 0; kq < BK; kq += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int m = wm + i * 8 + fr, k = kq + fc4;
          af[i] = AK ? a_s[m * LDM + k] : a_s[k * LDK + m];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int nn = wn + j * 8 + fr, k = kq + fc4;
          bf[j] = BKc ? b_s[nn * LDM + k] : b_s[k * LDK + nn];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();   // every warp is done with the ring before the next segment refills it
    if (kb != 0) {
      // partial tile (the range started inside the tile): slot layout [s][tid], coalesced
      double* wp = args.ws + (size_t)cta * 32 * NT;
#pragma unroll
      for (int s = 0; s < 32; ++s) __stcg(wp + s * NT + tid, acc[s >> 3][(s >> 1) & 3][s & 1]);
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release(args.cnt + cta, 1);
    } else {
      // owner: the following CTAs hold the rest of the tile's k-steps, one partial each
      int covered = ke;
      for (int c = cta + 1; covered < kiters; ++c) {
        if (tid == 0)
          while (ld_acquire(args.cnt + c) == 0) __nanosleep(64);
        __syncthreads();
        const double* wp = args.ws + (size_t)c * 32 * NT;
#pragma unroll
        for (int s = 0; s < 32; ++s) acc[s >> 3][(s >> 1) & 3][s & 1] += __ldcg(wp + s * NT + tid);
        __syncthreads();
        if (tid == 0) args.cnt[c] = 0;   // consumed: ready for the next launch on this stream
        covered += (int)(min(range_begin(c + 1), (t + 1) * kiters) - range_begin(c));
      }
#pragma unroll
      for (int s = 0; s < 32; ++s) {
        int r, c;
        slot_rc<4>(tid, s, r, c);
        put_elem(args, g, ri, m0 + r, n0 + c, acc[s >> 3][(s >> 1) & 3][s & 1]);
      }
    }
    it += nk;
  }
}

template <int TA, int TB>
void launch_big_streamk(const GemmArgs& a, int ctas, cudaStream_t st) {
  const int smem = 2 * STAGES * TILE * (int)sizeof(double);
  static bool attr = false;
  if (!attr) {
    FC_CUDA_TRY(cudaFuncSetAttribute(dgemm_big_streamk_kernel<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  dgemm_big_streamk_kernel<TA, TB><<<ctas, NT, smem, st>>>(a);
  FC_CHECK_LAUNCH();
}

template <int TA, int TB, bool KR>
void launch_big(const GemmArgs& a, dim3 grid, cudaStream_t st) {
  const int smem = std::max((KR ? 3 : 2) * STAGES * TILE, RED) * (int)sizeof(double);
  static bool attr = false;
  if (!attr) {
    FC_CUDA_TRY(cudaFuncSetAttribute(dgemm_big_kernel<TA, TB, KR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  launch_gemm_kernel(dgemm_big_kernel<TA, TB, KR>, a, grid, NT, smem, st);
}
}  // namespace big

}  // namespace

// ---- opt-in accounting of every GEMM launch (fc_profile_gemm): events around each launch and
// the algorithmic flop count 2 M N K per batch entry ------------------------------------
namespace {
struct GemmProf {
  std::mutex mu;                    // pcg_solve launches from two host threads
  bool on = false;
  std::vector<cudaEvent_t> ev;   // pairs
  std::vector<double> flops;
  std::vector<std::string> shape;   // FC_GEMM_TRACE: per-launch shape key
  size_t used = 0;
};
GemmProf& gprof() {
  static GemmProf p;
  return p;
}
}  // namespace

void gemm_profile(bool enable, double* ms, double* flops, long long* launches) {
  GemmProf& P = gprof();
  if (enable) {
    P.on = true;
    P.used = 0;
    P.flops.clear();
    return;
  }
  P.on = false;
  double t = 0, f = 0;
  std::map<std::string, std::pair<double, int>> hist;
  for (size_t i = 0; i < P.used; ++i) {
    float x = 0;
    FC_CUDA_TRY(cudaEventSynchronize(P.ev[2 * i + 1]));
    FC_CUDA_TRY(cudaEventElapsedTime(&x, P.ev[2 * i], P.ev[2 * i + 1]));
    t += x;
    f += P.flops[i];
    if (i < P.shape.size()) {
      auto& h = hist[P.shape[i]];
      h.first += x;
      h.second += 1;
    }
  }
  if (!hist.empty()) {   // FC_GEMM_TRACE: time by launch shape, largest first
    std::vector<std::pair<double, std::string>> v;
    for (auto& kv : hist) v.push_back({kv.second.first, kv.first + " x" + std::to_string(kv.second.second)});
    std::sort(v.rbegin(), v.rend());
    for (size_t i = 0; i < v.size() && i < 400; ++i) fprintf(stderr, "[fc gemm] %8.2f ms  %s\n", v[i].first, v[i].second.c_str());
  }
  P.shape.clear();
  if (ms) *ms = t;
  if (flops) *flops = f;
  if (launches) *launches = (long long)P.used;
}

static void gemm_dispatch(const GemmArgs& a, cudaStream_t st);

void gemm(const GemmArgs& a, cudaStream_t st) {
  GemmProf& P = gprof();
  if (!P.on) return gemm_dispatch(a, st);
  std::lock_guard<std::mutex> lock(P.mu);
  if (P.ev.size() < 2 * (P.used + 1)) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      FC_CUDA_TRY(cudaEventCreate(&e));
      P.ev.push_back(e);
    }
  }
  double f = 0;
  for (int i = 0; i < a.nbatch; ++i) {
    // algorithmic flops of the work actually done: device-side bounds are read back (profiling only)
    int M = a.b[i].M, K = a.b[i].K;
    if (a.b[i].dynM || a.b[i].dynK) {
      int d = 0;
      FC_CUDA_TRY(cudaMemcpyAsync(&d, a.b[i].dynM ? a.b[i].dynM : a.b[i].dynK, sizeof(int), cudaMemcpyDeviceToHost, st));
      FC_CUDA_TRY(cudaStreamSynchronize(st));
      if (a.b[i].dynM) M = std::min(M, d);
      else K = std::min(K, d);
    }
    f += 2.0 * a.rep * M * (double)a.b[i].N * K;
  }
  static const bool trace = getenv("FC_GEMM_TRACE") != nullptr;
  if (trace) {
    char key[160];
    snprintf(key, sizeof key, "t%d%d M%d N%d K%d nb%d rep%d sk%d%s", a.transA, a.transB, a.b[0].M, a.b[0].N, a.b[0].K,
             a.nbatch, a.rep, a.splitk, a.krR ? " KR" : (a.gen.kind >= 0 ? " GEN" : ""));
    P.shape.resize(P.used);
    P.shape.push_back(key);
  }
  FC_CUDA_TRY(cudaEventRecord(P.ev[2 * P.used], st));
  gemm_dispatch(a, st);
  FC_CUDA_TRY(cudaEventRecord(P.ev[2 * P.used + 1], st));
  P.flops.push_back(f);
  ++P.used;
}

// ---- split-K workspace (kmode 2), one per stream: launches on a stream run in order, so the
// partial tiles and the self-resetting counters are never shared by two running launches --------
namespace {
struct SplitWs {
  double* ws = nullptr;
  size_t wsn = 0;
  int* cnt = nullptr;
  size_t cntn = 0;
};
std::mutex g_ws_mu;
std::map<cudaStream_t, SplitWs> g_ws;

void split_workspace(cudaStream_t st, size_t doubles, size_t tiles, double** ws, int** cnt) {
  std::lock_guard<std::mutex> lock(g_ws_mu);
  SplitWs& w = g_ws[st];
  if (w.wsn < doubles) {
    if (w.ws) FC_CUDA_TRY(cudaFreeAsync(w.ws, st));
    w.wsn = std::max(doubles, (size_t)1 << 20);
    w.ws = (double*)dev_alloc(w.wsn * sizeof(double), st);
  }
  if (w.cntn < tiles) {
    if (w.cnt) FC_CUDA_TRY(cudaFreeAsync(w.cnt, st));
    w.cntn = std::max(tiles, (size_t)4096);
    w.cnt = (int*)dev_alloc(w.cntn * sizeof(int), st);
    FC_CUDA_TRY(cudaMemsetAsync(w.cnt, 0, w.cntn * sizeof(int), st));
  }
  *ws = w.ws;
  *cnt = w.cnt;
}

// split-K reduction: inside a cluster for up to kClusterSplit splits (16: non-portable cluster size,
// the 64x64-tile kernel fits 2-4 CTAs per SM; 8 for the 1-CTA-per-SM 128x128 kernel), through the
// global workspace above, up to 64 splits (last CTA to arrive; FC_GEMM_MAX_SPLIT sets the cap)
constexpr int kClusterSplit = 16, kBigClusterSplit = 8;
int max_split() {
  // 64: C4 303 ms vs 375 ms with the cap at 16 (GEMMs with few output tiles and long K)
  static const int v = getenv("FC_GEMM_MAX_SPLIT") ? atoi(getenv("FC_GEMM_MAX_SPLIT")) : 64;
  return std::max(1, std::min(v, 64));
}

void set_kmode(GemmArgs& a, dim3 grid, int nthreads, cudaStream_t st) {
  a.kmode = a.splitk <= 1 ? 0 : (a.splitk <= kClusterSplit ? 1 : 2);
  if (a.kmode == 2) {
    const size_t tiles = (size_t)grid.x * grid.y * (grid.z / a.splitk);
    split_workspace(st, tiles * a.splitk * 32 * nthreads, tiles, &a.ws, &a.cnt);
  }
}
}  // namespace

static void gemm_dispatch(const GemmArgs& a_in, cudaStream_t st) {
  if (a_in.nbatch <= 0) return;
  GemmArgs a = a_in;
  int maxM = 0, maxN = 0;
  for (int i = 0; i < a.nbatch; ++i) {
    maxM = std::max(maxM, a.b[i].M);
    maxN = std::max(maxN, a.b[i].N);
  }
  if (maxM == 0 || maxN == 0) return;
  long long work = 0;
  int minK = INT32_MAX;
  for (int i = 0; i < a.nbatch; ++i) {
    work += (long long)a.rep * a.b[i].M * a.b[i].N * a.b[i].K;
    minK = std::min(minK, a.b[i].K);
  }
  bool dyn = false;
  for (int i = 0; i < a.nbatch; ++i) dyn |= a.b[i].dynM != nullptr || a.b[i].dynK != nullptr;
  a.splitk = std::max(1, a.splitk);
  // stream-K (on request; FC_STREAMK=0 disables): entries with one tile grid and one K on 128 x 128
  // tiles (M, N > 64: more than one 64 x 64 tile) with at least 8 k-steps per SM.  It beat whole-tile launches on every C5 cell it accepts, also where
  // the tiles fill their waves (n = 2048, R r = 8192: 76.5 -> 81.6 % of the DMMA peak; no launch
  // tail, the fix-up of one tile overlaps the other CTAs' main loops)
  if (!dyn && a.gen.kind < 0 && a.krR == 0 && a.streamk && maxM > 64 && maxN > 64 && minK >= 64 &&
      work >= (1LL << 27)) {
    static const bool sk_on = !(getenv("FC_STREAMK") && atoi(getenv("FC_STREAMK")) == 0);
    static const int sms = [] {
      int dev = 0, v = 148;
      if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
      return std::max(v, 2);
    }();
    static const int min_it = getenv("FC_STREAMK_MINIT") ? atoi(getenv("FC_STREAMK_MINIT")) : 8;   // diagnostic
    bool same = true;   // one tile grid and one K for all entries (M, N may differ inside the last tiles)
    for (int i = 1; i < a.nbatch; ++i)
      same &= cdiv(a.b[i].M, big::BM) == cdiv(a.b[0].M, big::BM) && cdiv(a.b[i].N, big::BN) == cdiv(a.b[0].N, big::BN) &&
              a.b[i].K == a.b[0].K;
    const long long tiles = (long long)a.nbatch * a.rep * cdiv(maxM, big::BM) * cdiv(maxN, big::BN);
    const long long kit = cdiv(a.b[0].K, big::BK);
    if (sk_on && same && tiles * kit >= (long long)min_it * sms) {
      a.splitk = 1;
      a.kmode = 3;
      split_workspace(st, (size_t)sms * 32 * big::NT, (size_t)sms, &a.ws, &a.cnt);
      if (!a.transA && !a.transB) big::launch_big_streamk<0, 0>(a, sms, st);
      else if (a.transA && !a.transB) big::launch_big_streamk<1, 0>(a, sms, st);
      else if (!a.transA && a.transB) big::launch_big_streamk<0, 1>(a, sms, st);
      else big::launch_big_streamk<1, 1>(a, sms, st);
      return;
    }
  }
  if (!dyn && a.gen.kind < 0 && maxM >= 256 && maxN >= 256 && minK >= 64 && work >= (1LL << 27)) {
    a.splitk = std::min(a.splitk, kBigClusterSplit);   // big tiles: cluster reduction only
    dim3 grid(cdiv(maxM, big::BM), cdiv(maxN, big::BN), a.nbatch * a.rep * a.splitk);
    require(grid.y <= 65535 && grid.z <= 65535, FC_ERR_INVALID_ARG, "gemm grid too large");
    set_kmode(a, grid, big::NT, st);
    if (a.krR > 0) big::launch_big<0, 0, true>(a, grid, st);
    else if (!a.transA && !a.transB) big::launch_big<0, 0, false>(a, grid, st);
    else if (a.transA && !a.transB) big::launch_big<1, 0, false>(a, grid, st);
    else if (!a.transA && a.transB) big::launch_big<0, 1, false>(a, grid, st);
    else big::launch_big<1, 1, false>(a, grid, st);
    return;
  }
  static bool attr = false;
  const int smem2 = 2 * STAGES * STAGE_ELEMS * (int)sizeof(double);
  const int smem3 = 3 * STAGES * STAGE_ELEMS * (int)sizeof(double);
  static_assert(2 * STAGES * STAGE_ELEMS >= 32 * NT, "split-K reduction buffer aliases the pipeline");
  if (!attr) {
    FC_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
    FC_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3));
    FC_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
    FC_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<false, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    FC_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<true, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    FC_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<false, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  // auto split-K for callers that left splitk at 1: a 64 x 64 output tile with a long K is one
  // SM's work (~16 us per 4 MFLOP at the per-SM DMMA rate), so grids below two waves of 148 SMs
  // split K (>= 128 per split, <= 16: the cluster reduction) until they reach two waves
  static const bool auto_split = getenv("FC_GEMM_NO_AUTO_SPLIT") == nullptr;   // diagnostic
  if (auto_split && a.splitk <= 1 && a.gen.kind < 0 && a.krR == 0) {
    long long tiles = 0;
    int kmin = INT32_MAX;
    for (int i = 0; i < a.nbatch; ++i) {
      tiles += (long long)a.rep * cdiv(a.b[i].M, BM) * cdiv(a.b[i].N, BN);
      kmin = std::min(kmin, a.b[i].K);
    }
    if (tiles > 0 && tiles < 2 * 148 && kmin >= 256) {
      const long long want = (2 * 148 + tiles - 1) / tiles;
      a.splitk = (int)std::max<long long>(1, std::min<long long>({want, (long long)(kmin / 128), 16LL}));
    }
  }
  a.splitk = std::min(a.splitk, max_split());
  dim3 grid(cdiv(maxM, BM), cdiv(maxN, BN), a.nbatch * a.rep * a.splitk);
  require(grid.y <= 65535 && grid.z <= 65535, FC_ERR_INVALID_ARG, "gemm grid too large");
  set_kmode(a, grid, NT, st);
  if (a.gen.kind >= 0) launch_gemm_kernel(dgemm_dmma_kernel<false, true>, a, grid, NT, smem2, st);
  else if (a.krR > 0) launch_gemm_kernel(dgemm_dmma_kernel<true, false>, a, grid, NT, smem3, st);
  else launch_gemm_kernel(dgemm_dmma_kernel<false, false>, a, grid, NT, smem2, st);
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
