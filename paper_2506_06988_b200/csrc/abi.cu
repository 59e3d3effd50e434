// Library-level entry points of libhgs.so: error reporting and device query.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

#include <algorithm>
#include <atomic>
#include <vector>

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
const void* hgs_fine_bin_fn();
bool hgs_is_blend_tile_fn(const void* f);

// The blend's dependencies in a captured frame graph: the fine binning
// (programmatic: the blend claims the quads it publishes, ready queue) and,
// when a mesh branch is joined right before it, the mesh branch's last
// kernel.  Capture makes that second edge programmatic too, but in queue mode
// the blend never waits on its grid dependencies (no griddepcontrol.wait), so
// the mesh layer's writes would not be guaranteed visible: make every
// non-fine dependency of the blend a full one.  (HGS_GRAPH_DEBUG prints the
// edges.)  Returns the number of edges changed.
static int fix_blend_edges(cudaGraph_t g) {
  size_t n = 0;
  if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess || n == 0) return 0;
  std::vector<cudaGraphNode_t> nodes(n);
  if (cudaGraphGetNodes(g, nodes.data(), &n) != cudaSuccess) return 0;
  const void* fine = hgs_fine_bin_fn();
  static const bool dbg = std::getenv("HGS_GRAPH_DEBUG") != nullptr;
  auto kfunc = [](cudaGraphNode_t nd) -> const void* {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nd, &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) return nullptr;
    cudaKernelNodeParams kp{};
    if (cudaGraphKernelNodeGetParams(nd, &kp) != cudaSuccess) return nullptr;
    return kp.func;
  };
  int changed = 0;
  for (cudaGraphNode_t nd : nodes) {
    if (!hgs_is_blend_tile_fn(kfunc(nd))) continue;
    size_t nd_deps = 0;
    if (cudaGraphNodeGetDependencies_v2(nd, nullptr, nullptr, &nd_deps) != cudaSuccess || nd_deps == 0) continue;
    std::vector<cudaGraphNode_t> deps(nd_deps);
    std::vector<cudaGraphEdgeData> ed(nd_deps);
    if (cudaGraphNodeGetDependencies_v2(nd, deps.data(), ed.data(), &nd_deps) != cudaSuccess) continue;
    for (size_t i = 0; i < nd_deps; i++) {
      const bool is_fine = kfunc(deps[i]) == fine;
      if (dbg)
        std::fprintf(stderr, "blend dep %zu: %s, edge type %d port %d\n", i, is_fine ? "fine binning" : "other",
                     (int)ed[i].type, (int)ed[i].from_port);
      if (is_fine || ed[i].type == cudaGraphDependencyTypeDefault) continue;
      const cudaGraphEdgeData full{};
      if (cudaGraphRemoveDependencies_v2(g, &deps[i], &nd, &ed[i], 1) != cudaSuccess) continue;
      if (cudaGraphAddDependencies_v2(g, &deps[i], &nd, &full, 1) != cudaSuccess) {
        cudaGraphAddDependencies_v2(g, &deps[i], &nd, &ed[i], 1);
        continue;
      }
      changed++;
    }
  }
  cudaGetLastError();
  return changed;
}

extern "C" int hgs_graph_instantiate(void* graph, int32_t use_node_priority, void** exec_out) {
  if (!graph || !exec_out) return hgs_set_error(HGS_ERR_INVALID, "hgs_graph_instantiate: null argument");
  fix_blend_edges((cudaGraph_t)graph);
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
