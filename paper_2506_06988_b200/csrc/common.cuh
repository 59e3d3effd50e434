// Shared definitions for the hybrid GS+mesh CUDA path (sm_100a).
//
// Numerics: every kernel that restates a reference decision (cull, tile rect,
// sort key, support/skip/clamp/early-stop/mesh-stop, z-buffer, texel taps)
// computes in IEEE fp64 with FMA contraction disabled at compile time
// (-fmad=false); FMAs appear only where the reference's numpy matmul uses
// them (dot3 below).  See DESIGN.md "Numerics".
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hgs.h"

namespace hgs {

// reference constants: gsmesh/splat/project.py:19-27, splat/tiles.py:16
constexpr double COV_FLOOR = 0.3;
constexpr double ALPHA_CLAMP = 0.99;
constexpr double SIGMA_SKIP = 1.0 / 255.0;
constexpr double SUPPORT_MAHAL2 = 9.0;
constexpr double EARLY_STOP_T = 1e-4;
constexpr double SH_C0 = 0.28209479177387814;
constexpr double SH_C1 = 0.4886025119029199;

constexpr int NUM_SMS = 148;
// privatised copies of the tile-rectangle difference grid (hgs_projected.tile_diff)
constexpr int TILE_DIFF_COPIES = HGS_TILE_DIFF_COPIES;

// Blend record per Gaussian (fp64, 80 B): the fields the per-pixel walk reads.
struct __align__(16) BlendRec {
  double mx, my;      // mean2d
  double ca, cb2, cc;  // conic xx, 2 * conic xy (exact scaling), conic yy
  double depth;       // camera z
  double alpha;       // sigmoid(logit)
  double r, g, b;     // view-evaluated colour, clamped at 0
};
static_assert(sizeof(BlendRec) == 80, "BlendRec must be 80 bytes");

// fp32 companion record (hgs_projected.cull, 48 B): culling box + conic for
// the per-warp sub-tile test, and the fp32 operands of the blend fast path.
struct __align__(16) CullRec {
  float4 box;  // mean x, mean y, 3-sigma half extents x, y (z < 0: culled row)
  float4 con;  // conic xx, xy, yy, depth
  float4 col;  // alpha (< 0: ill-conditioned conic -> exact evaluation), r, g, b
};
static_assert(sizeof(CullRec) == 16 * 3 && HGS_CULL_FLOATS == 12, "CullRec is 48 B");

// numpy matmul inner-product order on x86-64 OpenBLAS (measured):
// s = a0*b0; s = fma(a1,b1,s); s = fma(a2,b2,s)
__device__ __forceinline__ double dot3(double a0, double a1, double a2, double b0, double b1, double b2) {
  double s = a0 * b0;
  s = fma(a1, b1, s);
  s = fma(a2, b2, s);
  return s;
}

template <typename T>
__host__ __device__ __forceinline__ T tmin(T a, T b) { return a < b ? a : b; }
template <typename T>
__host__ __device__ __forceinline__ T tmax(T a, T b) { return a > b ? a : b; }

__device__ __forceinline__ double clampd(double v, double lo, double hi) { return fmin(fmax(v, lo), hi); }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Tile binning <-> blend handoff (tiles.cu, blend.cu).  Tile grids of at
// most BIN_MAX_SUPER super-tiles of 4x4 (or 8x8) tiles are binned per
// super-tile block of 4x4 tiles ("quad"); each fine-binning CTA publishes its
// quad in a ready queue (hgs_tiles.ready) as soon as its
// entries are written, and the blend claims tiles in publication order, so
// its first tiles start while the last quads are still being binned
// (tile_counts_kernel empties the queue at every build; the bins and the
// blend must get the same buffer).
// ready[0]: quads published, ready[1]: tiles claimed, ready[2 + k]: quad + 1.
constexpr int BIN_MAX_SUPER = 512;
constexpr int READY_HDR = 2;
constexpr int READY_MAX_QUADS = 4 * BIN_MAX_SUPER;
static_assert(READY_HDR + READY_MAX_QUADS == HGS_READY_INTS, "hgs_tiles.ready size (hgs.h)");
// smallest super-tile shift with at most BIN_MAX_SUPER super-tiles (or -1)
// Blend-only bins (hgs.h) take 8x8-tile super-tiles once the 4x4 grid has
// more than BLEND_ONLY_SS3_ABOVE of them: the coarse binning then handles
// about half the (row, super-tile) pairs and the blend's filter of the
// longer lists costs less (c5, 1080p: 2.19 vs 2.53 ms; c3: 768 vs 764 us)
constexpr int BLEND_ONLY_SS3_ABOVE = 256;
__host__ __device__ inline int super_shift(int tiles_x, int tiles_y, bool blend_only = false) {
  const int n4 = ((tiles_x + 3) >> 2) * ((tiles_y + 3) >> 2);
  for (int ss = (blend_only && n4 > BLEND_ONLY_SS3_ABOVE) ? 3 : 2; ss <= 3; ss++) {
    const int sx = (tiles_x + (1 << ss) - 1) >> ss, sy = (tiles_y + (1 << ss) - 1) >> ss;
    if (sx * sy <= BIN_MAX_SUPER) return ss;
  }
  return -1;
}

// SFU reciprocal estimate (rcp.approx.ftz: ~1 ulp); callers either refine it
// or correct an integer quotient derived from it
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Programmatic dependent launch (PDL).  A kernel launched with launch_pdl()
// may be scheduled while the previous kernel on its stream drains; it calls
// pdl_enter() first thing: griddepcontrol.wait blocks until the previous
// grid has completed and its writes are visible (a no-op for a normal
// launch), then launch_dependents lets the next PDL kernel's CTAs be
// scheduled into SM slots this grid frees (its CTAs have all started by
// then, so they cannot be starved).  HGS_PDL=0 in the environment turns the
// attribute off (plain stream order).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();
// Zeroes up to two word ranges, as a PDL kernel (a memset node would break
// the programmatic chain).
__global__ void zero_words_kernel(uint32_t* a, int64_t na, uint32_t* b, int64_t nb);
cudaError_t zero_pdl(cudaStream_t st, void* a, size_t abytes, void* b = nullptr, size_t bbytes = 0);
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Block-wide exclusive scan of one value per thread (blockDim == 256).
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* s_warp /*[8]*/, T& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < 8 ? s_warp[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < 8) s_warp[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  T warp_excl = warp > 0 ? s_warp[warp - 1] : T(0);
  total = s_warp[7];
  __syncthreads();
  return warp_excl + x - v;
}

}  // namespace hgs

// Every kernel launch is followed by HGS_CHECK_LAUNCH(): it surfaces launch
// errors and counts the launch (hgs_kernel_launches()).
#define HGS_CHECK_LAUNCH()                                   \
  do {                                                       \
    hgs_count_launch();                                      \
    cudaError_t _e = cudaGetLastError();                     \
    if (_e != cudaSuccess) return hgs_set_cuda_error(_e, __FILE__, __LINE__); \
  } while (0)

int hgs_set_cuda_error(cudaError_t e, const char* file, int line);
int hgs_set_error(int code, const char* msg);
void hgs_count_launch();
