// Library-level entry points of libhgs.so: error reporting and device query.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

#include <algorithm>
#include <atomic>

namespace {
thread_local char g_last_error[512] = "";
std::atomic<long long> g_launches{0};
}

void hgs_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace hgs {
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HGS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

__global__ void zero_words_kernel(uint32_t* a, int64_t na, uint32_t* b, int64_t nb) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na + nb; i += stride) {
    if (i < na) a[i] = 0u;
    else b[i - na] = 0u;
  }
}

cudaError_t zero_pdl(cudaStream_t st, void* a, size_t abytes, void* b, size_t bbytes) {
  const int64_t na = (int64_t)(abytes / 4), nb = b ? (int64_t)(bbytes / 4) : 0;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((na + nb + 255) / 256, 4 * NUM_SMS));
  return launch_pdl(zero_words_kernel, dim3((unsigned)blocks), dim3(256), 0, st, (uint32_t*)a, na, (uint32_t*)b, nb);
}
}  // namespace hgs

extern "C" int64_t hgs_kernel_launches(void) { return g_launches.load(); }

int hgs_set_error(int code, const char* msg) {
  std::snprintf(g_last_error, sizeof(g_last_error), "%s", msg);
  return code;
}

int hgs_set_cuda_error(cudaError_t e, const char* file, int line) {
  std::snprintf(g_last_error, sizeof(g_last_error), "CUDA error %s (%s) at %s:%d", cudaGetErrorName(e),
                cudaGetErrorString(e), file, line);
  return HGS_ERR_CUDA;
}

extern "C" const char* hgs_last_error(void) { return g_last_error; }

extern "C" int hgs_abi_version(void) { return HGS_ABI_VERSION; }

extern "C" int hgs_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return hgs_set_cuda_error(e, __FILE__, __LINE__);
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  if (sm_count) *sm_count = v;
  cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, dev);
  if (cc_major) *cc_major = v;
  cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, dev);
  if (cc_minor) *cc_minor = v;
  return HGS_OK;
}

// CUDA-graph helpers for the host layer: instantiate a captured graph so that
// its kernel nodes run at the priority of the stream they were captured from
// (the frame's Gaussian chain on a high-priority stream, the mesh branch on
// a normal one: when both want SMs, the critical path gets them first).
extern "C" int hgs_graph_instantiate(void* graph, int32_t use_node_priority, void** exec_out) {
  if (!graph || !exec_out) return hgs_set_error(HGS_ERR_INVALID, "hgs_graph_instantiate: null argument");
  cudaGraphExec_t ex = nullptr;
  const unsigned long long flags = use_node_priority ? cudaGraphInstantiateFlagUseNodePriority : 0ull;
  cudaError_t e = cudaGraphInstantiateWithFlags(&ex, (cudaGraph_t)graph, flags);
  if (e != cudaSuccess) return hgs_set_cuda_error(e, __FILE__, __LINE__);
  *exec_out = (void*)ex;
  return HGS_OK;
}

extern "C" int hgs_graph_launch(void* exec, void* stream) {
  if (!exec) return hgs_set_error(HGS_ERR_INVALID, "hgs_graph_launch: null graph");
  cudaError_t e = cudaGraphLaunch((cudaGraphExec_t)exec, (cudaStream_t)stream);
  if (e != cudaSuccess) return hgs_set_cuda_error(e, __FILE__, __LINE__);
  return HGS_OK;
}

extern "C" int hgs_graph_exec_destroy(void* exec) {
  if (exec) cudaGraphExecDestroy((cudaGraphExec_t)exec);
  return HGS_OK;
}
