// Microbenchmark (tools/): latency of a single-thread dependent fp64 add chain
// on B200, from registers and streaming from global memory.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_reg(double* out, int n, double g) {
  double t = 0.0;
  for (int i = 0; i < n; i++) t = t + g * (double)(i & 1);
  out[0] = t;
}

__global__ void chain_mem(const double* __restrict__ in, double* out, int n) {
  double t = 0.0;
  double cur[32], nxt[32];
#pragma unroll
  for (int k = 0; k < 32; k++) cur[k] = in[k];
  for (int b = 0; b < n; b += 32) {
#pragma unroll
    for (int k = 0; k < 32; k++) nxt[k] = in[b + 32 + k];
#pragma unroll
    for (int k = 0; k < 32; k++) t = t + cur[k];
    out[b / 32] = t;
#pragma unroll
    for (int k = 0; k < 32; k++) cur[k] = nxt[k];
  }
  out[n] = t;
}

__global__ void chain_mem_plain(const double* __restrict__ in, double* out, int n) {
  double t = 0.0;
#pragma unroll 16
  for (int i = 0; i < n; i++) t = t + in[i];
  out[0] = t;
}

int main() {
  const int n = 1 << 16;
  double *in, *out;
  cudaMalloc(&in, sizeof(double) * (n + 64));
  cudaMalloc(&out, sizeof(double) * (n + 64));
  cudaMemset(in, 0, sizeof(double) * (n + 64));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(a);
    chain_reg<<<1, 1>>>(out, n, 1.0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("reg chain: %.3f ms, %.1f ns/add\n", ms, ms * 1e6 / n);
    cudaEventRecord(a);
    chain_mem<<<1, 1>>>(in, out, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("mem chain (32-reg prefetch): %.3f ms, %.1f ns/add\n", ms, ms * 1e6 / n);
    cudaEventRecord(a);
    chain_mem_plain<<<1, 1>>>(in, out, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("mem chain (plain, unroll 16): %.3f ms, %.1f ns/add\n", ms, ms * 1e6 / n);
  }
  return 0;
}
