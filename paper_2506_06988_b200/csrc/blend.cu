// K4 blend forward: rasterize_forward (gsmesh/splat/render.py:74-109) /
// forward_kernel (splat/kernels.py:12-74), with the transmittance-mask
// epilogue (train/losses.py:79-91).
//
// One CTA per 16x16 tile, one thread per pixel.  Each CTA walks its tile's
// depth-sorted entry list in batches of 256: every thread gathers one 80 B
// blend record into shared memory (SoA), then each pixel thread runs the
// reference's front-to-back loop over the batch (broadcast smem reads).
// A pixel is done at the mesh-depth stop (kernels.py:40-41) or the
// transmittance early stop (:52-54); the CTA leaves its list as soon as all
// 256 pixels are done (__syncthreads_count).  The walk is fp64 in the
// reference's operation order, so every skip/clamp/stop decision matches.
#include "common.cuh"

namespace hgs {

constexpr int BLEND_TILE = 16;
constexpr int BLEND_THREADS = BLEND_TILE * BLEND_TILE;

struct BlendSmem {
  double mx[BLEND_THREADS], my[BLEND_THREADS], ca[BLEND_THREADS], cb2[BLEND_THREADS], cc[BLEND_THREADS];
  double alpha[BLEND_THREADS], depth[BLEND_THREADS], r[BLEND_THREADS], g[BLEND_THREADS], b[BLEND_THREADS];
};

__device__ __forceinline__ double mask_value(double t, double k, int variant) {
  switch (variant) {
    case 0: return 1.0 / (1.0 + exp(-k * (t - 0.5)));
    case 1: return t;
    case 2: return 1.0;
    default: return 0.0;
  }
}

__device__ __forceinline__ void load_rec_to_smem(BlendSmem& sm, int slot, const BlendRec* __restrict__ rec, uint32_t g) {
  const double2* p = reinterpret_cast<const double2*>(rec + g);
  const double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2), d = __ldg(p + 3), e = __ldg(p + 4);
  sm.mx[slot] = a.x; sm.my[slot] = a.y;
  sm.ca[slot] = b.x; sm.cb2[slot] = 2.0 * b.y;  // (2.0 * conic_xy) is exact
  sm.cc[slot] = c.x; sm.alpha[slot] = c.y;
  sm.depth[slot] = d.x; sm.r[slot] = d.y;
  sm.g[slot] = e.x; sm.b[slot] = e.y;
}

__global__ void __launch_bounds__(BLEND_THREADS) blend_forward_kernel(
    const BlendRec* __restrict__ rec, const uint32_t* __restrict__ entries, const int64_t* __restrict__ tile_starts,
    int tiles_x, int width, int height, hgs_mesh_layer mesh, double bg0, double bg1, double bg2, int mask_variant,
    double mask_k, hgs_blend_out out) {
  __shared__ BlendSmem sm;
  __shared__ int64_t s_stats[2];
  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * BLEND_TILE + (threadIdx.x & (BLEND_TILE - 1));
  const int py = ty * BLEND_TILE + (threadIdx.x / BLEND_TILE);
  const bool inside = px < width && py < height;
  const int64_t p = (int64_t)py * width + px;
  const int64_t s = tile_starts[tile], e = tile_starts[tile + 1];
  const double fx = px + 0.5, fy = py + 0.5;
  const bool has_mesh = mesh.color != nullptr;
  const bool mesh_here = has_mesh && inside && mesh.triangle_id[p] >= 0;
  const double limit = mesh_here ? mesh.depth[p] : __longlong_as_double(0x7ff0000000000000LL);
  bool done = !inside;
  double T = 1.0, r = 0.0, g = 0.0, b = 0.0, dacc = 0.0;
  int64_t last = -1;
  int64_t walked = 0, blended = 0;
  if (threadIdx.x < 2) s_stats[threadIdx.x] = 0;

  for (int64_t base = s; base < e; base += BLEND_THREADS) {
    if (__syncthreads_count(!done) == 0) break;
    const int64_t idx = base + threadIdx.x;
    if (idx < e) load_rec_to_smem(sm, threadIdx.x, rec, entries[idx]);
    __syncthreads();
    const int nb = (int)tmin<int64_t>(BLEND_THREADS, e - base);
    if (!done) {
      for (int j = 0; j < nb; j++) {
        walked++;
        if (sm.depth[j] >= limit) { done = true; break; }  // list is depth sorted; mesh is opaque
        const double dx = fx - sm.mx[j], dy = fy - sm.my[j];
        const double m = sm.ca[j] * dx * dx + sm.cb2[j] * dx * dy + sm.cc[j] * dy * dy;
        if (m > SUPPORT_MAHAL2 || m < 0.0) continue;
        double sig = sm.alpha[j] * exp(-0.5 * m);
        if (sig > ALPHA_CLAMP) sig = ALPHA_CLAMP;
        if (sig < SIGMA_SKIP) continue;
        const double test_t = T * (1.0 - sig);
        if (test_t < EARLY_STOP_T) { done = true; break; }
        const double w = sig * T;
        r += sm.r[j] * w;
        g += sm.g[j] * w;
        b += sm.b[j] * w;
        dacc += sm.depth[j] * w;
        T = test_t;
        last = base + j;
        blended++;
      }
    }
  }
  if (out.stats) {
    __syncthreads();
    atomicAdd((unsigned long long*)&s_stats[0], (unsigned long long)walked);
    atomicAdd((unsigned long long*)&s_stats[1], (unsigned long long)blended);
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd((unsigned long long*)&out.stats[0], (unsigned long long)s_stats[0]);
      atomicAdd((unsigned long long*)&out.stats[1], (unsigned long long)s_stats[1]);
    }
  }
  if (!inside) return;
  double oc0, oc1, oc2, od;
  if (mesh_here) {
    oc0 = r + T * (double)mesh.color[3 * p];
    oc1 = g + T * (double)mesh.color[3 * p + 1];
    oc2 = b + T * (double)mesh.color[3 * p + 2];
    od = dacc + T * mesh.depth[p];
  } else {
    oc0 = r + T * bg0;
    oc1 = g + T * bg1;
    oc2 = b + T * bg2;
    const double acc = 1.0 - T;
    od = acc > 1e-12 ? dacc / acc : __longlong_as_double(0x7ff8000000000000LL);
  }
  out.color[3 * p] = (float)oc0;
  out.color[3 * p + 1] = (float)oc1;
  out.color[3 * p + 2] = (float)oc2;
  out.depth[p] = (float)od;
  out.transmittance[p] = (float)T;
  if (out.final_t) out.final_t[p] = T;
  if (out.last) out.last[p] = (int32_t)last;
  if (out.mask) out.mask[p] = (float)mask_value(T, mask_k, mask_variant);
}

}  // namespace hgs

extern "C" int hgs_blend_forward(const hgs_projected* proj, const hgs_tiles* tiles, int32_t width, int32_t height,
                                 const hgs_mesh_layer* mesh, const double* bg_host3, int32_t mask_variant,
                                 double mask_k, hgs_blend_out* out, void* stream) {
  using namespace hgs;
  if (!proj || !tiles || !out || !bg_host3) return hgs_set_error(HGS_ERR_INVALID, "hgs_blend_forward: null argument");
  if (tiles->tile_px != BLEND_TILE)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_blend_forward: only tile_px == 16 is implemented");
  if (width <= 0 || height <= 0) return hgs_set_error(HGS_ERR_INVALID, "hgs_blend_forward: empty image");
  if (tiles->tiles_x != (width + 15) / 16 || tiles->tiles_y != (height + 15) / 16)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_blend_forward: tile grid does not match image size");
  if (!out->color || !out->depth || !out->transmittance)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_blend_forward: missing output pointer");
  if (mask_variant < 0 || mask_variant > 3) return hgs_set_error(HGS_ERR_INVALID, "hgs_blend_forward: bad mask variant");
  hgs_mesh_layer ml{};
  if (mesh && mesh->color) {
    if (!mesh->depth || !mesh->triangle_id) return hgs_set_error(HGS_ERR_INVALID, "hgs_blend_forward: incomplete mesh layer");
    ml = *mesh;
  }
  const int n_tiles = tiles->tiles_x * tiles->tiles_y;
  blend_forward_kernel<<<n_tiles, BLEND_THREADS, 0, (cudaStream_t)stream>>>(
      (const BlendRec*)proj->rec, tiles->entries, tiles->tile_starts, tiles->tiles_x, width, height, ml, bg_host3[0],
      bg_host3[1], bg_host3[2], mask_variant, mask_k, *out);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}
