// Compute peaks of the B200 the blend kernels are rated against (SURVEY.md
// §8(d): FP32, MUFU ex2, FP64, shared-memory bandwidth, warp
// instruction issue).  Each figure is the best of 5 launches of a kernel
// that saturates one pipe with independent dependency chains on every SM
// (8 CTAs x 256 threads per SM); each rate is also given per SM per clock
// at the maximum SM clock, to check it against the architectural one.
// Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_peaks ubench_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;  // independent chains per thread
static int g_sms = 148, g_clk_mhz = 1965;

__global__ void k_ffma(float* out, int iters) {
  float a[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) a[c] = threadIdx.x * 1e-3f + c;
  const float b = 1.0000001f, d = 1e-9f;
  for (int i = 0; i < iters; i++)
#pragma unroll
    for (int c = 0; c < CH; c++) a[c] = fmaf(a[c], b, d);
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; c++) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, int iters) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) a[c] = threadIdx.x * 1e-3 + c;
  const double b = 1.0000001, d = 1e-9;
  for (int i = 0; i < iters; i++)
#pragma unroll
    for (int c = 0; c < CH; c++) a[c] = fma(a[c], b, d);
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ex2(float* out, int iters) {
  float a[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) a[c] = -(threadIdx.x & 7) * 0.01f - c * 0.1f;
  for (int i = 0; i < iters; i++)
#pragma unroll
    for (int c = 0; c < CH; c++) {
      float e;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(a[c]));
      a[c] = -e;  // chain stays in (-1, 0): 2^a in (0.5, 1)
    }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; c++) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_lds(float* out, int iters) {
  __shared__ float4 buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int idx = threadIdx.x & 1023;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      // 32 consecutive float4 per warp: conflict-free 512 B; volatile so the
      // loads are neither hoisted nor merged across iterations
      float4 v;
      const unsigned a = (unsigned)__cvta_generic_to_shared(&buf[(idx + c * 32) & 1023]);
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    idx = (idx + 256) & 1023;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// integer ALU chains: two warp instructions (LOP3 + VIADD, checked in the SASS) per op, issue-bound
__global__ void k_issue(unsigned* out, int iters) {
  unsigned a[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) a[c] = threadIdx.x + c;
  for (int i = 0; i < iters; i++)
#pragma unroll
    for (int c = 0; c < CH; c++) a[c] = (a[c] ^ 0x9e3779b9u) + c;
  unsigned s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K, typename P>
static void run(const char* name, K kern, P* buf, int blocks, int threads, int iters, double ops_per_iter_thread,
                const char* unit, bool last) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 6; rep++) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(buf, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double total = ops_per_iter_thread * iters * (double)blocks * threads;
  const double rate = total / (best * 1e-3);
  printf("  \"%s\": {\"rate\": %.6e, \"unit\": \"%s\", \"ms\": %.4f, \"per_sm_per_clk_at_max\": %.1f}%s\n", name,
         rate, unit, best, rate / g_sms / (g_clk_mhz * 1e6), last ? "" : ",");
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  g_sms = sms;
  g_clk_mhz = clk / 1000;
  const int blocks = sms * 8, threads = 256;
  void* buf;
  cudaMalloc(&buf, (size_t)blocks * threads * 8);
  printf("{\n  \"sms\": %d, \"max_clock_mhz\": %d,\n", sms, clk / 1000);
  run("fp32_fma", k_ffma, (float*)buf, blocks, threads, 1 << 14, CH, "FMA lane-ops/s", false);
  run("fp64_fma", k_dfma, (double*)buf, blocks, threads, 1 << 12, CH, "DFMA lane-ops/s", false);
  run("mufu_ex2", k_ex2, (float*)buf, blocks, threads, 1 << 12, CH, "ex2 lane-ops/s", false);
  run("smem_lds128", k_lds, (float*)buf, blocks, threads, 1 << 12, CH * 16.0, "B/s", false);
  run("issue_int", k_issue, (unsigned*)buf, blocks, threads, 1 << 14, CH * 2 / 32.0, "warp-instructions/s", true);
  printf("}\n");
  return 0;
}
