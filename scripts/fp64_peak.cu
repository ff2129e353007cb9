// FP64 peak microbenchmark on the B200 (roofline denominator for the multi-RHS matvec):
//   DFMA (CUDA cores): independent FMA chains per thread, all SMs busy.
//   DMMA (mma.sync m8n8k4 f64, the legacy warp-level FP64 tensor-core path).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak scripts/fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void k_dmma(double *out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  const int iters = 20000, threads = 512, blocks = nsm * 4;
  for (int rep = 0; rep < 2; ++rep) {
    k_dfma<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(s);
    k_dfma<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    const double flops = 2.0 * 8 * iters * (double)threads * blocks;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
    k_dmma<<<blocks, threads>>>(out, 100);
    cudaEventRecord(s);
    k_dmma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    const double mflops = 2.0 * 8 * 8 * 4 * 4 * (double)iters * (threads / 32) * blocks;
    printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", mflops / ms / 1e9, ms);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
