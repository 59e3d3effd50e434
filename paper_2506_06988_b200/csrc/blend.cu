// K4 blend forward: rasterize_forward (gsmesh/splat/render.py:74-109) /
// forward_kernel (splat/kernels.py:12-74), with the transmittance-mask
// epilogue (train/losses.py:79-91).
//
// Fast path (blend_fast_kernel): one CTA per 16x16 tile, one thread per
// pixel, warps own 8x4 sub-tiles.  The tile's depth-sorted entry list is
// walked in batches of 256: every thread gathers one 80 B fp64 record + a
// 16 B fp32 cull record into shared memory; each warp then compacts the
// batch to the entries whose 3-sigma box touches its 8x4 sub-tile (ballot,
// order preserving), and each pixel runs the reference's front-to-back loop
// over that list only.  Per pixel-entry pair: an fp32 support prefilter with
// a rigorous error bound rejects the clearly-outside pairs; the rest take the
// exact fp64 support test (reference operation order), an exp() evaluated on
// the SFU from an fp64-reduced argument (rel. err ~3e-7), and fp64
// accumulation.  The two thresholds the approximate exp can flip (sigma <
// 1/255 and T(1-sigma) < 1e-4) are guarded: if a decision lies within the
// tracked error band the pixel is flagged and blend_exact_kernel recomputes
// it with fp64 exp() -- so every skip/stop decision equals the reference's.
// The mesh-depth stop is an exact fp64 compare.  Culled entries cannot
// change the result: they have no support in the sub-tile, and the depth
// stop is monotone along the depth-sorted list.
#include "common.cuh"

namespace hgs {

constexpr int BLEND_TILE = 16;
constexpr int BLEND_THREADS = BLEND_TILE * BLEND_TILE;
constexpr double LOG2E = 1.4426950408889634;

struct BlendSmem {
  double mx[BLEND_THREADS], my[BLEND_THREADS], ca[BLEND_THREADS], cb2[BLEND_THREADS], cc[BLEND_THREADS];
  double alpha[BLEND_THREADS], depth[BLEND_THREADS], r[BLEND_THREADS], g[BLEND_THREADS], b[BLEND_THREADS];
  float4 box[BLEND_THREADS];  // fp32 mean x, mean y + conservative 3-sigma half extents
  unsigned char list[BLEND_THREADS / 32][BLEND_THREADS];
};

__device__ __forceinline__ double mask_value(double t, double k, int variant) {
  switch (variant) {
    case 0: return 1.0 / (1.0 + exp(-k * (t - 0.5)));
    case 1: return t;
    case 2: return 1.0;
    default: return 0.0;
  }
}

// exp(-m/2) for m in [0, 9] on the SFU: 2^(m * -0.5 log2 e) with the
// exponent rounded to fp32 (abs. err <= 2^-21 -> rel. 3.3e-7) and ex2.approx
// (rel. err <= 2^-22): |rel. err| <= 6e-7 (FAST_EXP_REL_ERR).
constexpr float FAST_EXP_REL_ERR = 6e-7f;
__device__ __forceinline__ double fast_exp_neg_half(double m) {
  const float t = (float)(m * (-0.5 * LOG2E));
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(t));
  return (double)e;
}

__device__ __forceinline__ void load_entry(BlendSmem& sm, int slot, const BlendRec* __restrict__ rec,
                                           const float4* __restrict__ cull, uint32_t g) {
  const double2* p = reinterpret_cast<const double2*>(rec + g);
  const double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2), d = __ldg(p + 3), e = __ldg(p + 4);
  const float4 cr = __ldg(cull + g);
  sm.mx[slot] = a.x; sm.my[slot] = a.y;
  sm.ca[slot] = b.x; sm.cb2[slot] = 2.0 * b.y;  // (2.0 * conic_xy) is exact
  sm.cc[slot] = c.x; sm.alpha[slot] = c.y;
  sm.depth[slot] = d.x; sm.r[slot] = d.y;
  sm.g[slot] = e.x; sm.b[slot] = e.y;
  sm.box[slot] = cr;
}

__device__ __forceinline__ void write_pixel(const hgs_blend_out& out, const hgs_mesh_layer& mesh, bool mesh_here,
                                            int64_t p, double T, double r, double g, double b, double dacc,
                                            int64_t last, double bg0, double bg1, double bg2, int mask_variant,
                                            double mask_k) {
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

__global__ void __launch_bounds__(BLEND_THREADS, 3) blend_fast_kernel(
    const BlendRec* __restrict__ rec, const float4* __restrict__ cull, const uint32_t* __restrict__ entries,
    const int64_t* __restrict__ tile_starts, int tiles_x, int width, int height, hgs_mesh_layer mesh, double bg0,
    double bg1, double bg2, int mask_variant, double mask_k, hgs_blend_out out, int32_t* __restrict__ fixup) {
  __shared__ BlendSmem sm;
  __shared__ unsigned long long s_stats[2];
  const int tile = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warp -> 8x4 sub-tile (2 across, 4 down); lane -> pixel inside it
  const int sx0 = (warp & 1) * 8, sy0 = (warp >> 1) * 4;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * BLEND_TILE + sx0 + (lane & 7);
  const int py = ty * BLEND_TILE + sy0 + (lane >> 3);
  const bool inside = px < width && py < height;
  const int64_t p = (int64_t)py * width + px;
  const int64_t s = tile_starts[tile], e = tile_starts[tile + 1];
  const double fx = px + 0.5, fy = py + 0.5;
  // pixel-centre box of this warp's sub-tile
  const float wx0 = tx * BLEND_TILE + sx0 + 0.5f, wx1 = wx0 + 7.0f;
  const float wy0 = ty * BLEND_TILE + sy0 + 0.5f, wy1 = wy0 + 3.0f;
  const bool has_mesh = mesh.color != nullptr;
  const bool mesh_here = has_mesh && inside && mesh.triangle_id[p] >= 0;
  const double limit = mesh_here ? mesh.depth[p] : __longlong_as_double(0x7ff0000000000000LL);
  bool done = !inside;
  bool flagged = false;
  double T = 1.0, r = 0.0, g = 0.0, b = 0.0, dacc = 0.0;
  float errT = 0.0f;  // bound on the relative error of T from the SFU exp
  int64_t last = -1;
  unsigned long long walked = 0, blended = 0;
  if (threadIdx.x < 2) s_stats[threadIdx.x] = 0;

  for (int64_t base = s; base < e; base += BLEND_THREADS) {
    if (__syncthreads_count(!done) == 0) break;
    const int64_t idx = base + threadIdx.x;
    if (idx < e) load_entry(sm, threadIdx.x, rec, cull, entries[idx]);
    __syncthreads();
    const int nb = (int)tmin<int64_t>(BLEND_THREADS, e - base);
    // per-warp, order-preserving compaction of the entries touching the sub-tile
    int nl = 0;
    if (__any_sync(0xffffffffu, !done)) {
      for (int k = 0; k < nb; k += 32) {
        const int j = k + lane;
        bool hit = false;
        if (j < nb) {
          const float4 q = sm.box[j];
          const float cx = fminf(fmaxf(q.x, wx0), wx1), cy = fminf(fmaxf(q.y, wy0), wy1);
          hit = fabsf(q.x - cx) <= q.z && fabsf(q.y - cy) <= q.w;
        }
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (hit) sm.list[warp][nl + __popc(m & lanemask_lt())] = (unsigned char)j;
        nl += __popc(m);
      }
    }
    __syncwarp();
    if (!done) {
      for (int li = 0; li < nl; li++) {
        const int j = sm.list[warp][li];
        walked++;
        if (sm.depth[j] >= limit) { done = true; break; }  // list is depth sorted; mesh is opaque
        // exact fp64 support test in the reference's operation order
        const double dx = fx - sm.mx[j], dy = fy - sm.my[j];
        const double m = sm.ca[j] * dx * dx + sm.cb2[j] * dx * dy + sm.cc[j] * dy * dy;
        if (m > SUPPORT_MAHAL2 || m < 0.0) continue;
        double sig = sm.alpha[j] * fast_exp_neg_half(m);
        if (sig > ALPHA_CLAMP) sig = ALPHA_CLAMP;
        const float sgf = (float)sig;
        // guard: the 1/255 skip decision is ambiguous within the exp error band
        if (fabsf(sgf - (float)SIGMA_SKIP) <= 1.5f * FAST_EXP_REL_ERR * (float)SIGMA_SKIP) flagged = true;
        if (sig < SIGMA_SKIP) continue;
        const double test_t = T * (1.0 - sig);
        errT += 1.1f * FAST_EXP_REL_ERR * __fdividef(sgf, 1.0f - sgf);
        // guard: the early-stop decision is ambiguous within the tracked T error band
        if (fabsf((float)test_t - (float)EARLY_STOP_T) <= (errT + 1e-6f) * (float)EARLY_STOP_T) flagged = true;
        if (test_t < EARLY_STOP_T) { done = true; break; }
        const double w = sig * T;
        r = fma(sm.r[j], w, r);
        g = fma(sm.g[j], w, g);
        b = fma(sm.b[j], w, b);
        dacc = fma(sm.depth[j], w, dacc);
        T = test_t;
        last = base + j;
        blended++;
      }
    }
  }
  if (out.stats) {
    __syncthreads();
    atomicAdd(&s_stats[0], walked);
    atomicAdd(&s_stats[1], blended);
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd((unsigned long long*)&out.stats[0], s_stats[0]);
      atomicAdd((unsigned long long*)&out.stats[1], s_stats[1]);
    }
  }
  if (!inside) return;
  if (flagged) {
    const int slot = atomicAdd(&fixup[0], 1);
    fixup[1 + slot] = (int32_t)p;
    return;
  }
  write_pixel(out, mesh, mesh_here, p, T, r, g, b, dacc, last, bg0, bg1, bg2, mask_variant, mask_k);
}

// Exact reference walk (fp64 exp()).  With fixup != NULL: one warp per
// flagged pixel (persistent grid-stride over the work list) -- lanes evaluate
// 32 consecutive entries in parallel, then every lane replays the reference's
// sequential T/colour recurrence over them in order (shuffles), so the
// arithmetic order equals kernels.py:38-61 exactly.  With fixup == NULL: the
// same, over every pixel.
__global__ void __launch_bounds__(256) blend_exact_kernel(
    const BlendRec* __restrict__ rec, const uint32_t* __restrict__ entries, const int64_t* __restrict__ tile_starts,
    int tiles_x, int width, int height, hgs_mesh_layer mesh, double bg0, double bg1, double bg2, int mask_variant,
    double mask_k, hgs_blend_out out, const int32_t* __restrict__ fixup) {
  const int64_t npix = (int64_t)width * height;
  const int64_t count = fixup ? fixup[0] : npix;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t wi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); wi < count; wi += nwarps) {
    const int64_t p = fixup ? fixup[1 + wi] : wi;
    const int px = (int)(p % width), py = (int)(p / width);
    const int tile = (py / BLEND_TILE) * tiles_x + px / BLEND_TILE;
    const int64_t s = tile_starts[tile], e = tile_starts[tile + 1];
    const double fx = px + 0.5, fy = py + 0.5;
    const bool mesh_here = mesh.color != nullptr && mesh.triangle_id[p] >= 0;
    const double limit = mesh_here ? mesh.depth[p] : __longlong_as_double(0x7ff0000000000000LL);
    double T = 1.0, r = 0.0, g = 0.0, b = 0.0, dacc = 0.0;
    int64_t last = -1;
    bool done = false;
    for (int64_t base = s; base < e && !done; base += 32) {
      const int64_t k = base + lane;
      bool stop = false, use = false;
      double sig = 0.0, cr = 0.0, cg = 0.0, cb = 0.0, dep = 0.0;
      if (k < e) {
        const BlendRec q = rec[entries[k]];
        dep = q.depth;
        stop = q.depth >= limit;
        const double dx = fx - q.mx, dy = fy - q.my;
        const double m = q.ca * dx * dx + (2.0 * q.cb) * dx * dy + q.cc * dy * dy;
        if (!(m > SUPPORT_MAHAL2 || m < 0.0)) {
          sig = q.alpha * exp(-0.5 * m);
          if (sig > ALPHA_CLAMP) sig = ALPHA_CLAMP;
          use = !(sig < SIGMA_SKIP);
        }
        cr = q.r; cg = q.g; cb = q.b;
      }
      const unsigned stop_mask = __ballot_sync(0xffffffffu, stop);
      unsigned use_mask = __ballot_sync(0xffffffffu, use);
      const int first_stop = stop_mask ? __ffs(stop_mask) - 1 : 32;
      if (first_stop < 32) {
        use_mask &= (1u << first_stop) - 1u;
        done = true;
      }
      while (use_mask) {
        const int i = __ffs(use_mask) - 1;
        use_mask &= use_mask - 1;
        const double sg = __shfl_sync(0xffffffffu, sig, i);
        const double test_t = T * (1.0 - sg);
        if (test_t < EARLY_STOP_T) { done = true; break; }
        const double w = sg * T;
        r += __shfl_sync(0xffffffffu, cr, i) * w;
        g += __shfl_sync(0xffffffffu, cg, i) * w;
        b += __shfl_sync(0xffffffffu, cb, i) * w;
        dacc += __shfl_sync(0xffffffffu, dep, i) * w;
        T = test_t;
        last = base + i;
      }
    }
    if (lane == 0) write_pixel(out, mesh, mesh_here, p, T, r, g, b, dacc, last, bg0, bg1, bg2, mask_variant, mask_k);
  }
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
  cudaStream_t st = (cudaStream_t)stream;
  const int n_tiles = tiles->tiles_x * tiles->tiles_y;
  const int64_t npix = (int64_t)width * height;
  if (out->fixup && proj->cull) {
    cudaMemsetAsync(out->fixup, 0, sizeof(int32_t), st);
    blend_fast_kernel<<<n_tiles, BLEND_THREADS, 0, st>>>((const BlendRec*)proj->rec, (const float4*)proj->cull,
                                                         tiles->entries, tiles->tile_starts, tiles->tiles_x, width,
                                                         height, ml, bg_host3[0], bg_host3[1], bg_host3[2],
                                                         mask_variant, mask_k, *out, out->fixup);
    HGS_CHECK_LAUNCH();
    // persistent fix-up over the (device-side) list of flagged pixels
    blend_exact_kernel<<<2 * NUM_SMS, 256, 0, st>>>((const BlendRec*)proj->rec, tiles->entries,
                                                            tiles->tile_starts, tiles->tiles_x, width, height, ml,
                                                            bg_host3[0], bg_host3[1], bg_host3[2], mask_variant,
                                                            mask_k, *out, out->fixup);
    HGS_CHECK_LAUNCH();
  } else {
    blend_exact_kernel<<<ceil_div(npix * 32, 256), 256, 0, st>>>((const BlendRec*)proj->rec, tiles->entries,
                                                            tiles->tile_starts, tiles->tiles_x, width, height, ml,
                                                            bg_host3[0], bg_host3[1], bg_host3[2], mask_variant,
                                                            mask_k, *out, nullptr);
    HGS_CHECK_LAUNCH();
  }
  return HGS_OK;
}
