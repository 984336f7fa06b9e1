// Internal header of libfraccontrol (B200 / sm_100a, FP64).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>
#include "../../include/fraccontrol.h"

#define FC_CUDA_TRY(expr)                                                            \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      throw fc::Error(FC_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    }                                                                               \
  } while (0)

#define FC_CHECK_LAUNCH()                 \
  do {                                    \
    fc::g_launches.fetch_add(1);          \
    FC_CUDA_TRY(cudaGetLastError());      \
  } while (0)

#include <atomic>
namespace fc {
// every kernel launch of the library passes FC_CHECK_LAUNCH (fc_kernel_launches in the ABI)
extern std::atomic<long long> g_launches;
}  // namespace fc

namespace fc {

struct Error {
  int code;
  std::string msg;
  Error(int c, std::string m) : code(c), msg(std::move(m)) {}
};

inline void require(bool cond, int code, const std::string& msg) {
  if (!cond) throw Error(code, msg);
}

// stream-ordered allocation; a failure names the size and clears the (non-sticky) error so that
// the next launch check does not report it again
inline void* dev_alloc(size_t bytes, cudaStream_t st) {
  void* p = nullptr;
  const cudaError_t e = cudaMallocAsync(&p, bytes, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    // out of device memory = the problem's ranks exceed what the device holds (reading A22: CAPACITY)
    throw Error(e == cudaErrorMemoryAllocation ? FC_ERR_CAPACITY : FC_ERR_CUDA,
                "device allocation of " + std::to_string(bytes >> 20) + " MiB failed: " + cudaGetErrorString(e));
  }
  return p;
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// ---- stream-ordered device scratch (cudaMallocAsync from the device's default pool) ----
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    size_t bytes = count * sizeof(T);
    if (bytes == 0) bytes = 16;
    bytes = (bytes + 255) & ~size_t(255);
    p = dev_alloc(bytes, st);
    ptrs.push_back(p);
    return (T*)p;
  }
  template <class T>
  T* zeros(size_t count) {
    T* p = alloc<T>(count);
    FC_CUDA_TRY(cudaMemsetAsync(p, 0, count * sizeof(T) ? count * sizeof(T) : 16, st));
    return p;
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

// ---- a device-resident buffer owned by the context (released in fc_destroy) -----------
struct DBuf {
  double* p = nullptr;
  size_t n = 0;
  void ensure(size_t count) {
    if (count <= n && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    if (count == 0) return;
    FC_CUDA_TRY(cudaMalloc(&p, count * sizeof(double)));
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// ---- batched FP64 GEMM on DMMA tiles (gemm.cu) ----------------------------------------
// C_b = alpha * op(A_b) * op(B_b) + beta * C_b, column-major; op(A) is M x K, op(B) K x N.
// KR-fused B operand (transB = 0 only): op(B)(k, c) = krU[k + (c / krR)*ldkr] * B[k + (c % krR)*ldb]
// Column scale (epilogue): C(:, c) *= colscale[c] before alpha/beta.
constexpr int kMaxBatch = 8;
struct GemmBatch {
  int M, N, K;
  const double* A; int lda;
  const double* B; int ldb;
  double* C; int ldc;
  const double* krU; int ldkr;
  const double* colscale;
  // strides between the GemmArgs::rep repetitions of this entry (A, B, C, colscale, krU)
  long long sA = 0, sB = 0, sC = 0, sS = 0, sK = 0;
  // optional device-side bounds read by the kernel: M_eff = min(M, *dynM), K_eff = min(K, *dynK)
  // (rows / terms beyond them are known to be zero: the blocked Gram-Schmidt passes the number of
  // accepted basis columns so that the unused, zero, columns of Q cost nothing)
  const int* dynM = nullptr;
  const int* dynK = nullptr;
};
// Generated A operand (transA = 0): A(m, k) = f((l1[m % n1] + l2[m / n1]) + l3[k]) with the
// spectral function f of kind FC_F / FC_G / FC_POW_PLUS / FC_POW_MINUS [P:640-648, P:693].
struct GenA {
  int kind = -1;
  double alpha = 0, beta = 0;
  const double* l1 = nullptr;
  const double* l2 = nullptr;
  const double* l3 = nullptr;
  int n1 = 0;
};
struct GemmArgs {
  int transA = 0, transB = 0;
  GenA gen;
  int krR = 0;           // > 0 enables the Khatri-Rao B operand
  // > 1: the K range is split over `splitk` CTAs per output tile and the partial tiles are
  // reduced in a FIXED order (split 0, 1, ...): through distributed shared memory inside a
  // (1, 1, splitk) thread-block cluster for splitk <= 16 (the 128x128 tiles clamp to 8), else
  // through a global workspace by the last-arriving CTA (clamped to 64).  Deterministic (bit-identical run to run); C = alpha op(A) op(B) + beta C
  // for every splitk.
  int splitk = 1;
  double alpha = 1.0, beta = 0.0;
  int nbatch = 0;
  int rep = 1;           // every entry is repeated rep times with its strides (strided batch)
  GemmBatch b[kMaxBatch];
  // set by the dispatcher (gemm.cu): split-K reduction mode and its workspace
  // request (caller): balance the 128x128-tile kernel's work over the SMs by k-steps instead of
  // whole tiles (stream-K, gemm.cu) when the tile count leaves the last wave mostly empty
  int streamk = 0;
  int kmode = 0;             // 0 direct, 1 cluster (DSMEM), 2 workspace, 3 stream-K
  double* ws = nullptr;      // kmode 2: partial tiles
  int* cnt = nullptr;        // kmode 2: per-tile arrival counters (self-resetting)
};
void gemm(const GemmArgs& a, cudaStream_t st);
// fc_profile_gemm: enable -> start recording; disable -> totals of the recorded launches
void gemm_profile(bool enable, double* ms, double* flops, long long* launches);
// fc_profile_kernel: opt-in accounting of the HBM-class kernels (events around each launch on
// its stream, algorithmic bytes per launch), one record per kernel id
enum KProfId { KP_DOT_REDUCE = 0, KP_KR_BASIS = 1, KP_KR_PRODUCT = 2, KP_COUNT = 3 };
struct KProfScope {
  int id;
  cudaStream_t st;
  double bytes;
  bool on;
  KProfScope(int id_, cudaStream_t st_, double bytes_);
  ~KProfScope();
};
void kprof_read(int id, bool enable, double* ms, double* bytes, long long* launches);
// split-K factor giving ~`waves` waves of 64 x 64 tiles on 148 SMs (at least 64 of K per split)
inline int waves_splitk(const GemmArgs& a, int waves) {
  long long tiles = 0;
  int minK = 1 << 30;
  for (int i = 0; i < a.nbatch; ++i) {
    tiles += (long long)a.rep * ((a.b[i].M + 63) / 64) * ((a.b[i].N + 63) / 64);
    minK = a.b[i].K < minK ? a.b[i].K : minK;
  }
  const long long want = (waves * 148LL + (tiles > 0 ? tiles : 1) - 1) / (tiles > 0 ? tiles : 1);
  const long long kmax = (minK + 63) / 64;
  const long long sk = want < kmax ? want : kmax;
  return sk > 1 ? (int)sk : 1;
}
// convenience single GEMM
void dgemm(cudaStream_t st, int transA, int transB, int M, int N, int K, double alpha,
           const double* A, int lda, const double* B, int ldb, double beta, double* C, int ldc,
           int splitk = 1);

}  // namespace fc
