// Microbenchmark: FP64 peaks on this B200.  DMMA (mma.sync m8n8k4 f64)
// and DFMA throughput with independent chains, all SMs, CUDA-event timed; plus an HBM copy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peak_fp64 tools/peak_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  if (s == 123.456) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
  const double a = 0.999999, b = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 123.456) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main() {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int iters = 20000;
  for (int warps = 4; warps <= 16; warps *= 2) {
    int blocks = nsm * 4;
    dmma_loop<<<blocks, 32 * warps>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)blocks * warps * iters * 8 * 512.0;
    printf("{\"kind\":\"dmma_m8n8k4\",\"warps_per_block\":%d,\"blocks\":%d,\"tflops\":%.3f}\n", warps, blocks,
           flops / ms / 1e9);
  }
  for (int threads = 256; threads <= 1024; threads *= 2) {
    int blocks = nsm * 4;
    dfma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)blocks * threads * iters * 8 * 2.0;
    printf("{\"kind\":\"dfma\",\"threads\":%d,\"blocks\":%d,\"tflops\":%.3f}\n", threads, blocks, flops / ms / 1e9);
  }
  size_t n = (size_t)1 << 27;  // 2 GiB per buffer (double2)
  double2 *a, *b;
  cudaMalloc(&a, n * 16);
  cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    copy_kernel<<<nsm * 8, 512>>>(a, b, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("{\"kind\":\"hbm_copy\",\"gbs\":%.1f}\n", 2.0 * n * 16 / best / 1e6);
  cudaError_t err = cudaDeviceSynchronize();
  printf("{\"status\":\"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
