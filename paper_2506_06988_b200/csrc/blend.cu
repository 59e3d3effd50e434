// K4 blend forward: rasterize_forward (gsmesh/splat/render.py:74-109) /
// forward_kernel (splat/kernels.py:12-74), with the transmittance-mask
// epilogue (train/losses.py:79-91).
//
// Fast path (blend_fast_kernel): one CTA per 16x16 tile, warp-specialised:
// 8 consumer warps each own an 8x4 sub-tile (one pixel per lane), 1
// producer warp streams the tile's depth-sorted entry list through a
// 4-stage shared-memory ring (128 entries x 96 B per stage: the 80 B fp64
// blend record + a 16 B fp32 cull box) with cp.async, completion tracked
// by mbarriers (full: producer -> consumers, empty: consumers -> producer).
// Consumers never meet at a CTA barrier: each compacts every stage to the
// entries whose 3-sigma box touches its sub-tile (ballot, order
// preserving) and runs the reference's front-to-back loop over that list.
// Once every consumer's pixels are done the producer stops streaming.
//
// Per pixel-entry pair: exact fp64 support test (reference operation
// order), exp() on the SFU (rel. err <= 6e-7), fp64 accumulation.  The two
// thresholds the approximate exp can flip (sigma < 1/255 and
// T(1-sigma) < 1e-4) are guarded: if a decision lies within the tracked
// error band the pixel is flagged and blend_exact_kernel recomputes it with
// fp64 exp() -- so every skip/stop decision equals the reference's.  The
// mesh-depth stop is an exact fp64 compare.  Culled entries cannot change
// the result: they have no support in the sub-tile, and the depth stop is
// monotone along the depth-sorted list.
#include "common.cuh"

namespace hgs {

constexpr int BLEND_TILE = 16;
constexpr int BLEND_THREADS = BLEND_TILE * BLEND_TILE;
constexpr double LOG2E = 1.4426950408889634;

constexpr int BATCH = 128;
constexpr int NSTAGE = 4;
constexpr int CONSUMERS = 8;
constexpr int FAST_THREADS = (CONSUMERS + 1) * 32;

struct __align__(16) StageEntry {
  double2 a;  // mean x, mean y
  double2 b;  // conic xx, 2*xy
  double2 c;  // conic yy, alpha
  double2 d;  // depth, r
  double2 e;  // g, b
  float4 box; // fp32 mean x, y, 3-sigma half extents x, y (z < 0: empty slot)
  float4 con; // fp32 conic xx, xy, yy (ellipse cull)
};
static_assert(sizeof(StageEntry) == 112, "stage entry is 112 B");

struct FastSmem {
  StageEntry ent[NSTAGE][BATCH];
  unsigned long long full[NSTAGE];
  unsigned long long empty[NSTAGE];
  unsigned char list[CONSUMERS][BATCH];
  int done_warps;
  int end_batch;
  unsigned long long stats[2];
};

__device__ const float4 g_empty_box = {0.0f, 0.0f, -1.0f, -1.0f};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// One lane polls (the loop is visible to the compiler, so the warp
// reconverges at the __syncwarp that publishes the acquired state).
__device__ __forceinline__ void warp_wait(unsigned long long* bar, unsigned parity, int lane) {
  if (lane == 0)
    while (!mbar_try_wait(bar, parity)) {
    }
  __syncwarp();
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Conservative test: does the support ellipse {m <= 9} reach any point of
// the box [x0,x1] x [y0,y1] (centre outside the box)?  The minimum of the
// convex quadratic m over the box lies on an edge; each edge minimum is a
// clamped 1D vertex.  fp32 with a generous margin (sure misses only).
__device__ __forceinline__ float edge_min(float a, float b, float c, float u, float v0, float v1) {
  // m(u, v) = a u^2 + 2 b u v + c v^2 with u fixed, v in [v0, v1]
  const float v = fminf(fmaxf(-b * u / c, v0), v1);
  return a * u * u + 2.0f * b * u * v + c * v * v;
}
__device__ __forceinline__ bool ellipse_meets_box(float4 con, float mx, float my, float x0, float x1, float y0,
                                                  float y1) {
  const float a = con.x, b = con.y, c = con.z;
  const float dx0 = x0 - mx, dx1 = x1 - mx, dy0 = y0 - my, dy1 = y1 - my;
  float mn = edge_min(a, b, c, dx0, dy0, dy1);
  mn = fminf(mn, edge_min(a, b, c, dx1, dy0, dy1));
  mn = fminf(mn, edge_min(c, b, a, dy0, dx0, dx1));
  mn = fminf(mn, edge_min(c, b, a, dy1, dx0, dx1));
  return mn <= 9.05f;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

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
// (rel. err <= 2^-22): |rel. err| <= 6e-7 (FAST_EXP_REL_ERR).  (A hi/lo
// split of the exponent halves the error and the fix-up flags but costs
// ~10 % of the blend kernel -- measured, not worth it.)
constexpr float FAST_EXP_REL_ERR = 6e-7f;
__device__ __forceinline__ double fast_exp_neg_half(double m) {
  const float t = (float)(m * (-0.5 * LOG2E));
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(t));
  return (double)e;
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

template <bool STATS>
__global__ void __launch_bounds__(FAST_THREADS, 3) blend_fast_kernel(
    const BlendRec* __restrict__ rec, const float4* __restrict__ cull, const uint32_t* __restrict__ entries,
    const int64_t* __restrict__ tile_starts, int tiles_x, int width, int height, hgs_mesh_layer mesh, double bg0,
    double bg1, double bg2, int mask_variant, double mask_k, hgs_blend_out out, int32_t* __restrict__ fixup) {
  extern __shared__ __align__(128) unsigned char fast_smem_raw[];
  FastSmem& sm = *reinterpret_cast<FastSmem*>(fast_smem_raw);
  const int tile = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s = tile_starts[tile], e = tile_starts[tile + 1];
  const int nbatches = (int)((e - s + BATCH - 1) / BATCH);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTAGE; i++) {
      mbar_init(&sm.full[i], 32);
      mbar_init(&sm.empty[i], CONSUMERS);
    }
    sm.done_warps = 0;
    sm.end_batch = 0x7fffffff;
    sm.stats[0] = sm.stats[1] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int tx = tile % tiles_x, ty = tile / tiles_x;

  if (warp == CONSUMERS) {
    // ------------------------------------------------------------ producer
    for (int b = 0; b < nbatches; b++) {
      const int slot = b % NSTAGE;
      if (b >= NSTAGE) warp_wait(&sm.empty[slot], ((b / NSTAGE) - 1) & 1, lane);
      if (*(volatile int*)&sm.done_warps == CONSUMERS) {
        if (lane == 0) *(volatile int*)&sm.end_batch = b;
        __syncwarp();
        mbar_arrive(&sm.full[slot]);  // 32 plain arrivals complete the phase
        break;
      }
      const int64_t base = s + (int64_t)b * BATCH;
      for (int i = lane; i < BATCH; i += 32) {
        StageEntry* dst = &sm.ent[slot][i];
        const int64_t k = base + i;
        if (k < e) {
          const uint32_t g = __ldg(entries + k);
          const char* src = reinterpret_cast<const char*>(rec + g);
          cp_async16(&dst->a, src);
          cp_async16(&dst->b, src + 16);
          cp_async16(&dst->c, src + 32);
          cp_async16(&dst->d, src + 48);
          cp_async16(&dst->e, src + 64);
          cp_async16(&dst->box, cull + 2 * (size_t)g);
          cp_async16(&dst->con, cull + 2 * (size_t)g + 1);
        } else {
          cp_async16(&dst->box, &g_empty_box);
        }
      }
      cp_async_arrive_noinc(&sm.full[slot]);
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int sx0 = (warp & 1) * 8, sy0 = (warp >> 1) * 4;
  const int px = tx * BLEND_TILE + sx0 + (lane & 7);
  const int py = ty * BLEND_TILE + sy0 + (lane >> 3);
  const bool inside = px < width && py < height;
  const int64_t p = (int64_t)py * width + px;
  const double fx = px + 0.5, fy = py + 0.5;
  const float wx0 = tx * BLEND_TILE + sx0 + 0.5f, wx1 = wx0 + 7.0f;
  const float wy0 = ty * BLEND_TILE + sy0 + 0.5f, wy1 = wy0 + 3.0f;
  const bool mesh_here = mesh.color != nullptr && inside && mesh.triangle_id[p] >= 0;
  const double limit = mesh_here ? mesh.depth[p] : __longlong_as_double(0x7ff0000000000000LL);
  bool done = !inside;
  bool flagged = false;
  bool warp_done = false;
  double T = 1.0, dacc = 0.0;
  float r = 0.0f, g = 0.0f, bl = 0.0f;  // colour sums (fp32: no decision depends on them)
  float errT = 0.0f;  // bound on the relative error of T from the SFU exp
  int last = -1;      // entry index relative to s
  unsigned walked = 0, blended = 0;

  for (int b = 0; b < nbatches; b++) {
    const int slot = b % NSTAGE;
    warp_wait(&sm.full[slot], (b / NSTAGE) & 1, lane);
    if (b >= *(volatile int*)&sm.end_batch) break;
    if (!warp_done) {
      // order-preserving compaction of the stage to entries touching the sub-tile
      int nl = 0;
#pragma unroll
      for (int k = 0; k < BATCH; k += 32) {
        const float4 q = sm.ent[slot][k + lane].box;
        const float cx = fminf(fmaxf(q.x, wx0), wx1), cy = fminf(fmaxf(q.y, wy0), wy1);
        bool hit = fabsf(q.x - cx) <= q.z && fabsf(q.y - cy) <= q.w;
        if (hit && (q.x != cx || q.y != cy)) hit = ellipse_meets_box(sm.ent[slot][k + lane].con, q.x, q.y, wx0, wx1,
                                                                  wy0, wy1);
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (hit) sm.list[warp][nl + __popc(m & lanemask_lt())] = (unsigned char)(k + lane);
        nl += __popc(m);
      }
      __syncwarp();
      if (__any_sync(0xffffffffu, !done)) {  // warp-uniform: the loop below votes
        const int bbase = b * BATCH;
        // Two entries per step: the independent part (support test, exp) of
        // both is evaluated together for ILP, then the reference's
        // sequential T/colour recurrence consumes them in order.  Uniform
        // trip count + a vote per step keeps the warp converged.
        for (int li = 0; li < nl; li += 2) {
          const bool has1 = li + 1 < nl;
          const int j0 = sm.list[warp][li];
          const int j1 = has1 ? sm.list[warp][li + 1] : j0;
          const StageEntry& E0 = sm.ent[slot][j0];
          const StageEntry& E1 = sm.ent[slot][j1];
          const double2 D0 = E0.d, D1 = E1.d;  // depth, r
          const double2 A0 = E0.a, A1 = E1.a, B0 = E0.b, B1 = E1.b, C0 = E0.c, C1 = E1.c;
          const double dx0 = fx - A0.x, dy0 = fy - A0.y, dx1 = fx - A1.x, dy1 = fy - A1.y;
          // exact fp64 support test in the reference's operation order
          const double m0 = B0.x * dx0 * dx0 + B0.y * dx0 * dy0 + C0.x * dy0 * dy0;
          const double m1 = B1.x * dx1 * dx1 + B1.y * dx1 * dy1 + C1.x * dy1 * dy1;
          const bool in0 = !(m0 > SUPPORT_MAHAL2 || m0 < 0.0);
          const bool in1 = has1 && !(m1 > SUPPORT_MAHAL2 || m1 < 0.0);
          double sig0 = C0.y * fast_exp_neg_half(in0 ? m0 : 0.0);
          double sig1 = C1.y * fast_exp_neg_half(in1 ? m1 : 0.0);
          // the 1/255 skip is a per-entry decision: near it, recompute exp in
          // fp64 right here (exact decision, no pixel flag needed)
          if (fabs(sig0 - SIGMA_SKIP) <= 2.0 * (double)FAST_EXP_REL_ERR * SIGMA_SKIP) sig0 = C0.y * exp(-0.5 * m0);
          if (fabs(sig1 - SIGMA_SKIP) <= 2.0 * (double)FAST_EXP_REL_ERR * SIGMA_SKIP) sig1 = C1.y * exp(-0.5 * m1);
          if (sig0 > ALPHA_CLAMP) sig0 = ALPHA_CLAMP;
          if (sig1 > ALPHA_CLAMP) sig1 = ALPHA_CLAMP;
#pragma unroll
          for (int u = 0; u < 2; u++) {
            const bool in = u == 0 ? in0 : in1;
            const double sig = u == 0 ? sig0 : sig1;
            const double2 D = u == 0 ? D0 : D1;
            const StageEntry& E = u == 0 ? E0 : E1;
            const int j = u == 0 ? j0 : j1;
            if (done || (u == 1 && !has1)) continue;
            if (STATS) walked++;
            if (D.x >= limit) { done = true; continue; }  // list is depth sorted; mesh is opaque
            if (!in) continue;
            const float sgf = (float)sig;
            if (sig < SIGMA_SKIP) continue;
            const double test_t = T * (1.0 - sig);
            errT += 1.1f * FAST_EXP_REL_ERR * sgf * rcp_approx(1.0f - sgf);
            // guard: the early-stop decision is ambiguous within the tracked T error band
            if (fabsf((float)test_t - (float)EARLY_STOP_T) <= (errT + 1e-6f) * (float)EARLY_STOP_T) flagged = true;
            if (test_t < EARLY_STOP_T) { done = true; continue; }
            const double w = sig * T;
            const float wf = (float)w;
            const double2 Ec = E.e;
            r = fmaf((float)D.y, wf, r);
            g = fmaf((float)Ec.x, wf, g);
            bl = fmaf((float)Ec.y, wf, bl);
            dacc = fma(D.x, w, dacc);
            T = test_t;
            last = b * BATCH + j;
            if (STATS) blended++;
          }
          if (__all_sync(0xffffffffu, done)) break;
        }
      }
      if (__all_sync(0xffffffffu, done)) {
        warp_done = true;
        if (lane == 0) atomicAdd(&sm.done_warps, 1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[slot]);
  }
  if (STATS) {
    atomicAdd(&sm.stats[0], (unsigned long long)walked);
    atomicAdd(&sm.stats[1], (unsigned long long)blended);
    // consumers only: the producer may already have left
    asm volatile("bar.sync 1, %0;" ::"n"(CONSUMERS * 32));
    if (threadIdx.x == 0) {
      atomicAdd((unsigned long long*)&out.stats[0], sm.stats[0]);
      atomicAdd((unsigned long long*)&out.stats[1], sm.stats[1]);
    }
  }
  if (!inside) return;
  if (flagged) {  // hand the pixel to the exact walk (work list: count, pixel ids)
    const int slot = atomicAdd(&fixup[0], 1);
    fixup[1 + slot] = (int32_t)p;
    return;
  }
  write_pixel(out, mesh, mesh_here, p, T, r, g, bl, dacc, last >= 0 ? s + last : -1, bg0, bg1, bg2, mask_variant,
              mask_k);
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
    // software-pipelined: the next chunk's record gather is in flight while
    // the current chunk is evaluated and consumed
    BlendRec nxt;
    if (s + lane < e) nxt = rec[entries[s + lane]];
    for (int64_t base = s; base < e && !done; base += 32) {
      const int64_t k = base + lane;
      const BlendRec q = nxt;
      if (base + 32 + lane < e) nxt = rec[entries[base + 32 + lane]];
      bool stop = false, use = false;
      double sig = 0.0, cr = 0.0, cg = 0.0, cb = 0.0, dep = 0.0;
      if (k < e) {
        dep = q.depth;
        stop = q.depth >= limit;
        const double dx = fx - q.mx, dy = fy - q.my;
        const double m = q.ca * dx * dx + q.cb2 * dx * dy + q.cc * dy * dy;
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
    const size_t smem = sizeof(FastSmem);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(blend_fast_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(blend_fast_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    if (out->stats)
      blend_fast_kernel<true><<<n_tiles, FAST_THREADS, smem, st>>>(
          (const BlendRec*)proj->rec, (const float4*)proj->cull, tiles->entries, tiles->tile_starts, tiles->tiles_x,
          width, height, ml, bg_host3[0], bg_host3[1], bg_host3[2], mask_variant, mask_k, *out, out->fixup);
    else
      blend_fast_kernel<false><<<n_tiles, FAST_THREADS, smem, st>>>(
          (const BlendRec*)proj->rec, (const float4*)proj->cull, tiles->entries, tiles->tile_starts, tiles->tiles_x,
          width, height, ml, bg_host3[0], bg_host3[1], bg_host3[2], mask_variant, mask_k, *out, out->fixup);
    HGS_CHECK_LAUNCH();
    // exact fix-up: one warp per flagged pixel (persistent grid over the device-side work list)
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
