// Microbenchmark: fp64 vs fp32 FMA and exp throughput on the box (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9, d = a + 1, e = a + 2, f = a + 3;
  for (int i = 0; i < iters; i++) {
    a = fma(a, b, c); d = fma(d, b, c); e = fma(e, b, c); f = fma(f, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + d + e + f;
}
__global__ void k_ffma(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0000001f, c = 1e-9f, d = a + 1, e = a + 2, f = a + 3;
  for (int i = 0; i < iters; i++) {
    a = fmaf(a, b, c); d = fmaf(d, b, c); e = fmaf(e, b, c); f = fmaf(f, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + d + e + f;
}
__global__ void k_dexp(double* out, int iters) {
  double a = -(threadIdx.x & 7) * 0.1, s = 0, b = -0.3, c = -0.7, d = -1.1;
  for (int i = 0; i < iters; i++) {
    s += exp(a) + exp(b) + exp(c) + exp(d);
    a -= 1e-7; b -= 1e-7; c -= 1e-7; d -= 1e-7;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fexp(float* out, int iters) {
  float a = -(threadIdx.x & 7) * 0.1f, s = 0, b = -0.3f, c = -0.7f, d = -1.1f;
  for (int i = 0; i < iters; i++) {
    s += __expf(a) + __expf(b) + __expf(c) + __expf(d);
    a -= 1e-7f; b -= 1e-7f; c -= 1e-7f; d -= 1e-7f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sms %d l2 %d MB clock %d MHz\n", sms, l2 >> 20, clk / 1000);
  int blocks = sms * 8, threads = 256, iters = 1 << 14;
  double* dd; float* df;
  cudaMalloc(&dd, blocks * threads * 8); cudaMalloc(&df, blocks * threads * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0); k_dfma<<<blocks, threads>>>(dd, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA  %.2f TFLOP/s\n", 2.0 * 4 * iters * (double)blocks * threads / ms / 1e9);
    cudaEventRecord(e0); k_ffma<<<blocks, threads>>>(df, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA  %.2f TFLOP/s\n", 2.0 * 4 * iters * (double)blocks * threads / ms / 1e9);
    cudaEventRecord(e0); k_dexp<<<blocks, threads>>>(dd, iters / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("dexp  %.2f Gexp/s\n", 4.0 * (iters / 4) * (double)blocks * threads / ms / 1e6);
    cudaEventRecord(e0); k_fexp<<<blocks, threads>>>(df, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("fexp  %.2f Gexp/s\n", 4.0 * iters * (double)blocks * threads / ms / 1e6);
  }
  return 0;
}
