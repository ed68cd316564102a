// Throughput probe: fp64 mma.sync m8n8k4 (DMMA) vs fp64 FFMA on one B200 (tools only).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = fma(a, b, c[t]);
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * nsm * 8 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    const int iters = 20000;
    k_dmma<<<nsm, 32 * warps>>>(out, 10);
    cudaEventRecord(e0);
    k_dmma<<<nsm, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 4 * iters * warps * (double)nsm;
    printf("DMMA m8n8k4: %2d warps/SM: %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
    k_ffma<<<nsm, 32 * warps>>>(out, 10);
    cudaEventRecord(e0);
    k_ffma<<<nsm, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * 32 * iters * warps * (double)nsm;
    printf("DFMA:        %2d warps/SM: %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
