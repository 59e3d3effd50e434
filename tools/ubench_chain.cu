// Per-kernel cost of a dependent launch chain inside a CUDA graph: N empty
// kernels (grid G x 256), plain stream order vs programmatic dependent launch
// (griddepcontrol.wait + launch_dependents first thing), vs N phases of one
// cooperative persistent kernel separated by grid.sync().
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_chain tools/ubench_chain.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_plain(int* p) { if (threadIdx.x == 0 && blockIdx.x == 0) p[0]++; }
__global__ void k_pdl(int* p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) p[0]++;
}
__global__ void k_coop(int* p, int phases) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < phases; i++) {
    if (threadIdx.x == 0 && blockIdx.x == 0) p[0]++;
    g.sync();
  }
}

int main() {
  int* d;
  cudaMalloc(&d, 4);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int N = 40;
  for (int G : {1, 148, 592}) {
    for (int mode = 0; mode < 2; mode++) {
      cudaGraph_t gr;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < N; i++) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = mode;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, mode ? k_pdl : k_plain, d);
      }
      cudaStreamEndCapture(st, &gr);
      cudaGraphExec_t ex;
      cudaGraphInstantiate(&ex, gr, 0);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int w = 0; w < 3; w++) cudaGraphLaunch(ex, st);
      cudaEventRecord(a, st);
      for (int r = 0; r < 20; r++) cudaGraphLaunch(ex, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %4d %s: %.2f us per kernel\n", G, mode ? "pdl  " : "plain", ms * 1e3 / (20 * N));
    }
    {
      int phases = N;
      void* args[] = {&d, &phases};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaLaunchCooperativeKernel((void*)k_coop, dim3(G), dim3(256), args, 0, st);
      cudaEventRecord(a, st);
      for (int r = 0; r < 20; r++) cudaLaunchCooperativeKernel((void*)k_coop, dim3(G), dim3(256), args, 0, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %4d coop : %.2f us per grid.sync phase (%s)\n", G, ms * 1e3 / (20 * N),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
