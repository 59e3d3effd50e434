// K4 blend forward: rasterize_forward (gsmesh/splat/render.py:74-109) /
// forward_kernel (splat/kernels.py:12-74), with the transmittance-mask
// epilogue (train/losses.py:79-91).
//
// Production fast path: blend_tile_kernel (below; 2 pixels per lane, cut-form
// decisions, per-warp walk buffers, tiles claimed from the binning's ready
// queue) with blend_exact_queue_kernel draining the flagged pixels beside
// it.  The round-1 kernel blend_fast_kernel is kept as the A/B baseline
// (HGS_BLEND_V1=1):
//
// blend_fast_kernel: one CTA per 16x16 tile, warp-specialised:
// 8 consumer warps each own an 8x4 sub-tile (one pixel per lane), 1
// producer warp streams the tile's depth-sorted entry list through a
// 2-stage shared-memory ring (128 entries x 112 B per stage: 64 B of the
// fp64 blend record + the 48 B fp32 CullRec) with cp.async, completion
// tracked by mbarriers (full: producer -> consumers, empty: consumers ->
// producer).  Consumers never meet at a CTA barrier: each compacts every
// stage to the entries whose support ellipse touches its sub-tile (ballot,
// order preserving) and runs the reference's front-to-back loop over that
// list.  Once every consumer's pixels are done the producer stops.
//
// Numerics of the fast path (every decision equals the reference's):
//  * the conic form m is evaluated in fp64 with FMAs and scaled to the exp2
//    argument u = m log2(e)/2 in fp64; u is narrowed to fp32 (round to
//    nearest).  The support test m > 9 / m < 0 is decided on u with a
//    2^-20 relative guard band; inside the band (or for a conic flagged
//    ill-conditioned by preprocess) the entry is re-evaluated exactly in the
//    reference's operation order with fp64 exp() -- per entry, in place.
//  * sigma = alpha * 2^-u in fp32 on the SFU: |rel. err| <= EPS_SIG.  Near
//    the 1/255 skip threshold the same exact re-evaluation decides.
//  * T, the blend weights and the colour/depth sums are fp32.  An absolute
//    bound eT on |T - T_reference| is carried along; when an early-stop test
//    T(1-sigma) < 1e-4 falls within it the pixel is flagged and
//    blend_exact_kernel replays it in fp64 -- so every stop decision is the
//    reference's too.  The mesh-depth stop is an exact fp64 compare.
//  * Culled entries cannot change the result: they have no support in the
//    sub-tile, and the depth stop is monotone along the depth-sorted list.
#include "stage.cuh"

namespace hgs {

constexpr int BLEND_TILE = 16;
// hgs_blend_out.fixup layout (fast path): [0] slots reserved, [1] blend CTAs
// finished, [2] slots claimed, [3] queue-consumer warps exited, [4..] queue
// slots (flagged pixel + 1, 0 = empty); all zero at rest
constexpr int FIX_RESERVED = 0, FIX_DONE = 1, FIX_CLAIMED = 2, FIX_EXITED = 3, FIX_SLOTS = 4;
// spin-wait bound of the queue consumers (~ tens of seconds of nanosleeps):
// a broken handoff traps (a launch error) instead of hanging the device
constexpr uint32_t QUEUE_SPIN_LIMIT = 1u << 26;
constexpr int BLEND_THREADS = BLEND_TILE * BLEND_TILE;

#ifndef HGS_FAST_BATCH
#define HGS_FAST_BATCH 128
#endif
#ifndef HGS_FAST_NSTAGE
#define HGS_FAST_NSTAGE 2
#endif
#ifndef HGS_FAST_MINB
#define HGS_FAST_MINB 4
#endif
#ifndef HGS_FAST_MINB_PREC
#define HGS_FAST_MINB_PREC 3
#endif
constexpr int BATCH = HGS_FAST_BATCH;
constexpr int NSTAGE = HGS_FAST_NSTAGE;
constexpr int CONSUMERS = 8;
constexpr int FAST_THREADS = (CONSUMERS + 1) * 32;

struct FastSmem {
  StageEntry ent[NSTAGE][BATCH];
  unsigned long long full[NSTAGE];
  unsigned long long empty[NSTAGE];
  unsigned char list[CONSUMERS][BATCH];
  double exp2tab[EXP2_N];
  int done_warps;
  int end_batch;
  unsigned long long stats[2];
};

__device__ __forceinline__ double mask_value(double t, double k, int variant) {
  switch (variant) {
    case 0: return 1.0 / (1.0 + exp(-k * (t - 0.5)));
    case 1: return t;
    case 2: return 1.0;
    default: return 0.0;
  }
}

__device__ __forceinline__ void write_pixel(const hgs_blend_out& out, const hgs_mesh_layer& mesh, bool mesh_here,
                                            int64_t p, double T, double r, double g, double b, double dacc,
                                            double acc, int64_t last, double bg0, double bg1, double bg2, int mask_variant,
                                            double mask_k, double T_state) {
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
    od = acc > 1e-12 ? dacc / acc : __longlong_as_double(0x7ff8000000000000LL);
  }
  out.color[3 * p] = (float)oc0;
  out.color[3 * p + 1] = (float)oc1;
  out.color[3 * p + 2] = (float)oc2;
  out.depth[p] = (float)od;
  out.transmittance[p] = (float)T;
  if (out.final_t) out.final_t[p] = T_state;
  if (out.last) out.last[p] = (int32_t)last;
  if (out.mask) out.mask[p] = (float)mask_value(T, mask_k, mask_variant);
}

// Exact re-evaluation of one entry in the reference's operation order
// (kernels.py:42-51): support test, fp64 exp, clamp, skip.  Returns sigma,
// or -1 when the entry is not blended.
__device__ __noinline__ double exact_entry(const StageEntry& E, double fx, double fy) {
  const double dx = fx - E.a.x, dy = fy - E.a.y;
  const double m = E.b.x * dx * dx + E.b.y * dx * dy + E.c.x * dy * dy;
  if (m > SUPPORT_MAHAL2 || m < 0.0) return -1.0;
  double sg = E.d.x * exp(-0.5 * m);
  if (sg > ALPHA_CLAMP) sg = ALPHA_CLAMP;
  return sg < SIGMA_SKIP ? -1.0 : sg;
}

// Exact walk of one pixel by one warp (fp64 exp()): lanes evaluate
// consecutive entries in parallel -- support test, exp, clamp, skip and
// the mesh-depth stop exactly as kernels.py:38-51 -- then the chunk's
// transmittance recurrence T <- T (1 - sigma) is evaluated as a shuffle
// prefix product.  That rounds differently from the reference's serial
// product (|rel. diff| < 1e-13 over any walk), so the early-stop decision
// is trusted only outside a 1e-12 band around 1e-4; a chunk with a value
// inside it is replayed serially in the reference's order.  Colour/depth
// sums are per-lane partials reduced once at the end.  Software-pipelined:
// the next chunk's record gather is in flight during the current one.
// Result is warp-uniform.
struct ExactPixel {
  double T, r, g, b, dacc;
  int64_t last;
};

// The walk, two entries per lane per round (64 per warp iteration) with a
// software pipeline (indices four rounds ahead, records two): lane L
// evaluates entries base + 2L and base + 2L + 1, whose gathers and fp64
// exp() overlap; T before each entry is T * (exclusive lane prefix product)
// * (in-lane running product).  Decisions: the first mesh-
// depth stop in entry order cuts the round; outside the 1e-12 band around the
// early-stop threshold the first entry with T(1 - sigma) < 1e-4 ends the
// walk; a round with a value inside the band is replayed serially in the
// reference's order.
// Walk state carried across the two parts of a blend-only replay (the tile
// list prefix the blend wrote, then the coarse list): T and last are warp-
// uniform, the sums per-lane partials reduced at the end (walk_finish).
struct WalkState {
  double T, pr, pg, pb, pd;
  int64_t last;
  bool done;
};
__device__ __forceinline__ ExactPixel walk_finish(WalkState& w) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    w.pr += __shfl_xor_sync(0xffffffffu, w.pr, d);
    w.pg += __shfl_xor_sync(0xffffffffu, w.pg, d);
    w.pb += __shfl_xor_sync(0xffffffffu, w.pb, d);
    w.pd += __shfl_xor_sync(0xffffffffu, w.pd, d);
  }
  return ExactPixel{w.T, w.pr, w.pg, w.pb, w.pd, w.last};
}

__device__ __forceinline__ void exact_walk2_run(const BlendRec* __restrict__ rec, const uint32_t* __restrict__ entries,
                                                int64_t s, int64_t e, double fx, double fy, double limit, int lane,
                                                WalkState& ws) {
  constexpr int EW = 2, RW = 32 * EW;
  double& T = ws.T;
  double &pr = ws.pr, &pg = ws.pg, &pb = ws.pb, &pd = ws.pd;
  int64_t& last = ws.last;
  bool& done = ws.done;
  auto idx = [&](int64_t rbase, int u) -> uint32_t {
    const int64_t k = rbase + EW * lane + u;
    return k < e ? __ldcg(entries + k) : 0u;  // L2 (the queue consumer runs beside the binning's writers)
  };
  uint32_t ix[4][EW];
#pragma unroll
  for (int d = 0; d < 4; d++)
#pragma unroll
    for (int u = 0; u < EW; u++) ix[d][u] = idx(s + (int64_t)d * RW, u);
  BlendRec r0[EW], r1[EW];
#pragma unroll
  for (int u = 0; u < EW; u++) {
    if (s + EW * lane + u < e) r0[u] = rec[ix[0][u]];
    if (s + RW + EW * lane + u < e) r1[u] = rec[ix[1][u]];
  }
  for (int64_t base = s; base < e && !done; base += RW) {
    BlendRec c[EW];
#pragma unroll
    for (int u = 0; u < EW; u++) {
      c[u] = r0[u];
      r0[u] = r1[u];
      if (base + 2 * RW + EW * lane + u < e) r1[u] = rec[ix[2][u]];
      ix[0][u] = ix[1][u];
      ix[1][u] = ix[2][u];
      ix[2][u] = ix[3][u];
      ix[3][u] = idx(base + 4 * RW, u);
    }
    double sig[EW];
    bool use[EW];
    int us = EW;  // first depth stop of this lane
#pragma unroll
    for (int u = 0; u < EW; u++) {
      const int64_t k = base + EW * lane + u;
      use[u] = false;
      sig[u] = 0.0;
      if (k < e) {
        if (c[u].depth >= limit && us == EW) us = u;
        const double dx = fx - c[u].mx, dy = fy - c[u].my;
        const double m = c[u].ca * dx * dx + c[u].cb2 * dx * dy + c[u].cc * dy * dy;
        if (!(m > SUPPORT_MAHAL2 || m < 0.0)) {
          double sg = c[u].alpha * exp(-0.5 * m);
          if (sg > ALPHA_CLAMP) sg = ALPHA_CLAMP;
          use[u] = !(sg < SIGMA_SKIP);
          sig[u] = sg;
        }
      }
    }
    const unsigned smask = __ballot_sync(0xffffffffu, us < EW);
    const int ls = smask ? __ffs(smask) - 1 : 32;
    const int lsu = __shfl_sync(0xffffffffu, us, ls & 31);
#pragma unroll
    for (int u = 0; u < EW; u++)
      if (lane > ls || (lane == ls && u >= lsu)) use[u] = false;
    if (ls < 32) done = true;
    double f[EW];
    double q = 1.0;
#pragma unroll
    for (int u = 0; u < EW; u++) {
      f[u] = use[u] ? 1.0 - sig[u] : 1.0;
      q *= f[u];
    }
    double P = q;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, P, d);
      if (lane >= d) P *= t;
    }
    double Pex = __shfl_up_sync(0xffffffffu, P, 1);
    if (lane == 0) Pex = 1.0;
    double ta[EW];
    double run = T * Pex;
    bool near = false;
#pragma unroll
    for (int u = 0; u < EW; u++) {
      run *= f[u];
      ta[u] = run;
      near = near || (use[u] && fabs(run - EARLY_STOP_T) <= 1e-12 * EARLY_STOP_T);
    }
    if (!__any_sync(0xffffffffu, near)) {
      int ue = EW;
#pragma unroll
      for (int u = 0; u < EW; u++)
        if (use[u] && ta[u] < EARLY_STOP_T && ue == EW) ue = u;
      const unsigned emask = __ballot_sync(0xffffffffu, ue < EW);
      const int le = emask ? __ffs(emask) - 1 : 32;
      const int leu = __shfl_sync(0xffffffffu, ue, le & 31);
      int lastu = -1;
      double tb = T * Pex, tl = 0.0;
#pragma unroll
      for (int u = 0; u < EW; u++) {
        const bool valid = use[u] && (lane < le || (lane == le && u < leu));
        if (valid) {
          const double w = sig[u] * tb;
          pr += c[u].r * w;
          pg += c[u].g * w;
          pb += c[u].b * w;
          pd += c[u].depth * w;
          lastu = u;
          tl = ta[u];
        }
        tb = ta[u];
      }
      const unsigned vmask = __ballot_sync(0xffffffffu, lastu >= 0);
      if (vmask) {
        const int lv = 31 - __clz(vmask);
        T = __shfl_sync(0xffffffffu, tl, lv);
        last = base + (int64_t)EW * lv + __shfl_sync(0xffffffffu, lastu, lv);
      }
      if (le < 32) done = true;
    } else {
      bool stop = false;
      for (int i = 0; i < 32 && !stop; i++) {
#pragma unroll
        for (int u = 0; u < EW; u++) {
          const bool ui = __shfl_sync(0xffffffffu, use[u], i);
          if (!ui || stop) continue;
          const double sg = __shfl_sync(0xffffffffu, sig[u], i);
          const double test_t = T * (1.0 - sg);
          if (test_t < EARLY_STOP_T) {
            stop = true;
            continue;
          }
          if (lane == i) {
            const double w = sg * T;
            pr += c[u].r * w;
            pg += c[u].g * w;
            pb += c[u].b * w;
            pd += c[u].depth * w;
          }
          T = test_t;
          last = base + (int64_t)EW * i + u;
        }
      }
      if (stop) done = true;
    }
  }
}
__device__ __noinline__ ExactPixel exact_walk2(const BlendRec* __restrict__ rec, const uint32_t* __restrict__ entries,
                                               int64_t s, int64_t e, double fx, double fy, double limit, int lane) {
  WalkState w{1.0, 0.0, 0.0, 0.0, 0.0, -1, false};
  exact_walk2_run(rec, entries, s, e, fx, fy, limit, lane, w);
  return walk_finish(w);
}

// The exact walk of one pixel over a super-tile's coarse list (blend-only
// bins): the entries whose rectangle covers the pixel's tile are its tile
// list, in order.  Two list entries per lane per round (64 per round), the
// next round's rectangles and rows and this round's matching records in
// flight while a round is evaluated; the tile-list index of every entry from
// a running count of the matches.  Otherwise the reference's walk as in
// exact_walk2 (depth stop, shuffle prefix product of 1 - sigma, serial replay
// of a round with a value within 1e-12 of the early-stop threshold).
// (Resumable: from coarse position cb, the first `skip` matches there and
// the first kcount tile-list entries already walked, state in ws.)
__device__ __forceinline__ void exact_walk_coarse_run(const BlendRec* __restrict__ rec,
                                                      const uint32_t* __restrict__ crow, const uint2* __restrict__ crect,
                                                      uint32_t cb, int skip, int kcount, uint32_t ce, int tx, int ty,
                                                      int64_t s, double fx, double fy, double limit, int lane,
                                                      WalkState& ws) {
  constexpr int EW = 2, RW = 32 * EW;
  double& T = ws.T;
  double &pr = ws.pr, &pg = ws.pg, &pb = ws.pb, &pd = ws.pd;
  int64_t& last = ws.last;
  bool& done = ws.done;
  auto covers = [&](uint2 r) {
    return (int)(r.x & 0xffffu) <= tx && tx <= (int)(r.x >> 16) && (int)(r.y & 0xffffu) <= ty &&
           ty <= (int)(r.y >> 16);
  };
  // software pipeline: while round r is evaluated, the matching records of
  // round r + 1 and the rectangles / rows of round r + 2 are in flight
  uint2 rn[EW];
  uint32_t gn[EW];
  auto load_rects = [&](uint32_t b) {
#pragma unroll
    for (int u = 0; u < EW; u++) {
      const uint32_t i = b + EW * lane + u;
      rn[u] = i < ce ? __ldcg(crect + i) : make_uint2(0xffffu, 0xffffu);  // (x0 = 65535 > x1: no match)
      gn[u] = i < ce ? __ldcg(crow + i) : 0u;
    }
  };
  bool mnext[EW];
  BlendRec cnext[EW];
  auto load_recs = [&]() {
#pragma unroll
    for (int u = 0; u < EW; u++) {
      mnext[u] = covers(rn[u]);
      if (mnext[u]) cnext[u] = rec[gn[u]];
    }
  };
  load_rects(cb);
  load_recs();
  load_rects(cb + RW);
  for (uint32_t base = cb; base < ce && !done; base += RW) {
    bool match[EW];
    BlendRec c[EW];
#pragma unroll
    for (int u = 0; u < EW; u++) {
      match[u] = mnext[u];
      c[u] = cnext[u];
    }
    load_recs();                // round + 1
    load_rects(base + 2 * RW);  // round + 2
    if (skip) {  // resuming inside a round: its first `skip` matches were walked already
      const unsigned a0 = __ballot_sync(0xffffffffu, match[0]), a1 = __ballot_sync(0xffffffffu, match[1]);
      const int r0 = __popc(a0 & lanemask_lt()) + __popc(a1 & lanemask_lt());  // rank of (lane, 0)
      const int r1 = r0 + (int)((a0 >> lane) & 1u);                            // rank of (lane, 1)
      if (r0 < skip) match[0] = false;
      if (r1 < skip) match[1] = false;
      skip = 0;
    }
    const unsigned m0 = __ballot_sync(0xffffffffu, match[0]), m1 = __ballot_sync(0xffffffffu, match[1]);
    const int kl = kcount + __popc(m0 & lanemask_lt()) + __popc(m1 & lanemask_lt());
    int krank[EW] = {kl, kl + (match[0] ? 1 : 0)};
    kcount += __popc(m0) + __popc(m1);
    double sig[EW];
    bool use[EW];
    int us = EW;  // first depth stop of this lane
#pragma unroll
    for (int u = 0; u < EW; u++) {
      use[u] = false;
      sig[u] = 0.0;
      if (match[u]) {
        if (c[u].depth >= limit && us == EW) us = u;
        const double dx = fx - c[u].mx, dy = fy - c[u].my;
        const double m = c[u].ca * dx * dx + c[u].cb2 * dx * dy + c[u].cc * dy * dy;
        if (!(m > SUPPORT_MAHAL2 || m < 0.0)) {
          double sg = c[u].alpha * exp(-0.5 * m);
          if (sg > ALPHA_CLAMP) sg = ALPHA_CLAMP;
          use[u] = !(sg < SIGMA_SKIP);
          sig[u] = sg;
        }
      }
    }
    const unsigned smask = __ballot_sync(0xffffffffu, us < EW);
    const int ls = smask ? __ffs(smask) - 1 : 32;
    const int lsu = __shfl_sync(0xffffffffu, us, ls & 31);
#pragma unroll
    for (int u = 0; u < EW; u++)
      if (lane > ls || (lane == ls && u >= lsu)) use[u] = false;
    if (ls < 32) done = true;
    double f[EW];
    double q = 1.0;
#pragma unroll
    for (int u = 0; u < EW; u++) {
      f[u] = use[u] ? 1.0 - sig[u] : 1.0;
      q *= f[u];
    }
    double P = q;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, P, d);
      if (lane >= d) P *= t;
    }
    double Pex = __shfl_up_sync(0xffffffffu, P, 1);
    if (lane == 0) Pex = 1.0;
    double ta[EW];
    double run = T * Pex;
    bool near = false;
#pragma unroll
    for (int u = 0; u < EW; u++) {
      run *= f[u];
      ta[u] = run;
      near = near || (use[u] && fabs(run - EARLY_STOP_T) <= 1e-12 * EARLY_STOP_T);
    }
    if (!__any_sync(0xffffffffu, near)) {
      int ue = EW;
#pragma unroll
      for (int u = 0; u < EW; u++)
        if (use[u] && ta[u] < EARLY_STOP_T && ue == EW) ue = u;
      const unsigned emask = __ballot_sync(0xffffffffu, ue < EW);
      const int le = emask ? __ffs(emask) - 1 : 32;
      const int leu = __shfl_sync(0xffffffffu, ue, le & 31);
      int lastk = -1;
      double tb = T * Pex, tl = 0.0;
#pragma unroll
      for (int u = 0; u < EW; u++) {
        const bool valid = use[u] && (lane < le || (lane == le && u < leu));
        if (valid) {
          const double w = sig[u] * tb;
          pr += c[u].r * w;
          pg += c[u].g * w;
          pb += c[u].b * w;
          pd += c[u].depth * w;
          lastk = krank[u];
          tl = ta[u];
        }
        tb = ta[u];
      }
      const unsigned vmask = __ballot_sync(0xffffffffu, lastk >= 0);
      if (vmask) {
        const int lv = 31 - __clz(vmask);
        T = __shfl_sync(0xffffffffu, tl, lv);
        last = s + __shfl_sync(0xffffffffu, lastk, lv);
      }
      if (le < 32) done = true;
    } else {
      bool stop = false;
      for (int i = 0; i < 32 && !stop; i++) {
#pragma unroll
        for (int u = 0; u < EW; u++) {
          const bool ui = __shfl_sync(0xffffffffu, use[u], i);
          const int ki = __shfl_sync(0xffffffffu, krank[u], i);
          if (!ui || stop) continue;
          const double sg = __shfl_sync(0xffffffffu, sig[u], i);
          const double test_t = T * (1.0 - sg);
          if (test_t < EARLY_STOP_T) {
            stop = true;
            continue;
          }
          if (lane == i) {
            const double w = sg * T;
            pr += c[u].r * w;
            pg += c[u].g * w;
            pb += c[u].b * w;
            pd += c[u].depth * w;
          }
          T = test_t;
          last = s + ki;
        }
      }
      if (stop) done = true;
    }
  }
}

// A blend-only replay: the tile-list prefix [s, s + kc) the blend's producer
// wrote to `entries`, then (if the walk goes on) the coarse list from where
// the producer stopped (coarse position pos, `skip` matches there done).
__device__ __noinline__ ExactPixel exact_walk_blend_only(const BlendRec* __restrict__ rec,
                                                         const uint32_t* __restrict__ entries, int64_t s, int kc,
                                                         const uint32_t* __restrict__ crow,
                                                         const uint2* __restrict__ crect, uint32_t pos, int skip,
                                                         uint32_t ce, int tx, int ty, double fx, double fy,
                                                         double limit, int lane) {
  WalkState w{1.0, 0.0, 0.0, 0.0, 0.0, -1, false};
  exact_walk2_run(rec, entries, s, s + kc, fx, fy, limit, lane, w);
  if (!w.done) exact_walk_coarse_run(rec, crow, crect, pos, skip, kc, ce, tx, ty, s, fx, fy, limit, lane, w);
  return walk_finish(w);
}

// PREC (the caller asked for the backward state final_t): T is also carried
// in fp64 with sigma from the fp64 exp2 (stage.cuh) for every blended entry,
// i.e. the reference's T recurrence to ~1e-11 relative; only final_t takes
// it -- colour / T / depth outputs are the same fp32 values as without.
template <bool STATS, bool PREC>
__global__ void __launch_bounds__(FAST_THREADS, PREC ? HGS_FAST_MINB_PREC : HGS_FAST_MINB) blend_fast_kernel(
    const BlendRec* __restrict__ rec, const CullRec* __restrict__ cull, const uint32_t* __restrict__ entries,
    const int64_t* __restrict__ tile_starts, int tiles_x, int width, int height, hgs_mesh_layer mesh, double bg0,
    double bg1, double bg2, int mask_variant, double mask_k, hgs_blend_out out, int32_t* __restrict__ fixup,
    const int64_t* __restrict__ counters) {
  pdl_enter();
  if (counters && counters[2]) return;  // entry buffer overflowed: bins are invalid, the caller re-renders
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
  if (PREC) exp2_tab_load(sm.exp2tab);
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
          const char* cs = reinterpret_cast<const char*>(cull + g);
          cp_async16(&dst->a, src);
          cp_async16(&dst->b, src + 16);
          cp_async16(&dst->c, src + 32);
          cp_async16(&dst->d, src + 48);
          cp_async16(&dst->f.box, cs);
          cp_async16(&dst->f.con, cs + 16);
          cp_async16(&dst->f.col, cs + 32);
        } else {
          cp_async16(&dst->f.box, &g_empty_box);
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
  float T = 1.0f;     // transmittance
  double T64 = 1.0;   // PREC: the reference's fp64 T
  float eT = 0.0f;    // bound on |T - T_reference| (valid while not done)
  float acc = 0.0f;   // sum of blend weights (= 1 - T_reference up to rounding)
  float r = 0.0f, g = 0.0f, bl = 0.0f, dacc = 0.0f;
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
        const float4 q = sm.ent[slot][k + lane].f.box;
        const float cx = fminf(fmaxf(q.x, wx0), wx1), cy = fminf(fmaxf(q.y, wy0), wy1);
        bool hit = fabsf(q.x - cx) <= q.z && fabsf(q.y - cy) <= q.w;
        if (hit && (q.x != cx || q.y != cy))
          hit = ellipse_meets_box(sm.ent[slot][k + lane].f.con, q, wx0, wx1, wy0, wy1);
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (hit) sm.list[warp][nl + __popc(m & lanemask_lt())] = (unsigned char)(k + lane);
        nl += __popc(m);
      }
      __syncwarp();
      if (__any_sync(0xffffffffu, !done)) {  // warp-uniform: the loop below votes
        // Two entries per step: the independent part (conic form, exp2,
        // decisions) of both is evaluated together for ILP, then the
        // reference's sequential T/colour recurrence consumes them in order
        // with selects.  Uniform trip count + a vote per step keeps the warp
        // converged.
        for (int li = 0; li < nl; li += 2) {
          const bool has1 = li + 1 < nl;
          int jj[2];
          jj[0] = sm.list[warp][li];
          jj[1] = has1 ? sm.list[warp][li + 1] : jj[0];
          float sg[2], uf[2];
          double um[2];
          bool ok[2], dstop[2];
          float key = 2.0f;
#pragma unroll
          for (int u = 0; u < 2; u++) {
            const StageEntry& E = sm.ent[slot][jj[u]];
            const double2 A = E.a, B = E.b, C = E.c;  // C: conic yy, depth
            const float a32 = E.f.col.x;
            const double dx = fx - A.x, dy = fy - A.y;
            const double m = fma(dx, fma(B.y, dy, B.x * dx), (C.x * dy) * dy);
            um[u] = m * U_SCALE;
            const float uu = __double2float_rn(um[u]);
            uf[u] = uu;
            const float sgf = fminf(fabsf(a32) * ex2_neg(uu), CLAMP_F);
            dstop[u] = C.y >= limit;
            ok[u] = uu < U9_LO && sgf >= SKIP_F;
            sg[u] = sgf;
            key = fminf(key, amb_key(uu, sgf, a32));
          }
          // Fast commit: valid when no lane of the warp meets a decision this
          // step can get wrong -- a depth stop, an early-stop region, an
          // ambiguous entry.  Then both entries are blended branch-free
          // (a skipped entry has sigma 0: T, eT-growth aside, and the sums
          // are unchanged exactly).
          const float s0 = (ok[0] && !done) ? sg[0] : 0.0f;
          const float s1 = (ok[1] && !done && has1) ? sg[1] : 0.0f;
          const float om0 = 1.0f - s0, om1 = 1.0f - s1;
          const float T1 = T * om0;
          const float T2 = T1 * om1;
          const float w0 = T * s0, w1 = T1 * s1;
          const float e1 = fmaf(w0, EPS_SIG, fmaf(eT, om0, T1 * 1.1920929e-7f));
          const float e2 = fmaf(w1, EPS_SIG, fmaf(e1, om1, T2 * 1.1920929e-7f));
          // T2 - 2 e2 >= STOP_NEAR implies neither entry's stop test is
          // ambiguous or taken (T1 - 2 e1 >= (T2 - 2 e2) / (1 - s1))
          const bool special =
              !done && (dstop[0] || (has1 && dstop[1]) || key <= 1.0f || fmaf(-2.0f, e2, T2) < STOP_NEAR);
          if (!__any_sync(0xffffffffu, special)) {
            eT = e2;
            const float4 c0 = sm.ent[slot][jj[0]].f.col, c1 = sm.ent[slot][jj[1]].f.col;
            const float d0 = sm.ent[slot][jj[0]].f.con.w, d1 = sm.ent[slot][jj[1]].f.con.w;
            r = fmaf(c1.y, w1, fmaf(c0.y, w0, r));
            g = fmaf(c1.z, w1, fmaf(c0.z, w0, g));
            bl = fmaf(c1.w, w1, fmaf(c0.w, w0, bl));
            dacc = fmaf(d1, w1, fmaf(d0, w0, dacc));
            acc = (acc + w0) + w1;
            T = T2;
            if (PREC) {  // no entry of the step is ambiguous: fp32 decisions are the reference's
              double f0 = 1.0, f1 = 1.0;
              if (s0 > 0.0f)
                f0 = 1.0 - fmin(sm.ent[slot][jj[0]].d.x * exp2_neg64(um[0], uf[0], sm.exp2tab), ALPHA_CLAMP);
              if (s1 > 0.0f)
                f1 = 1.0 - fmin(sm.ent[slot][jj[1]].d.x * exp2_neg64(um[1], uf[1], sm.exp2tab), ALPHA_CLAMP);
              T64 = (T64 * f0) * f1;
            }
            const int bb = b * BATCH;
            last = s1 > 0.0f ? bb + jj[1] : (s0 > 0.0f ? bb + jj[0] : last);
            if (STATS && !done) {
              walked += has1 ? 2 : 1;
              blended += (s0 > 0.0f) + (s1 > 0.0f);
            }
            continue;
          }
          double sx[2] = {-1.0, -1.0};  // exact sigma of re-evaluated entries
          if (__any_sync(0xffffffffu, key <= 1.0f)) {  // rare: exact per-entry re-evaluation
#pragma unroll
            for (int u = 0; u < 2; u++) {
              const StageEntry& E = sm.ent[slot][jj[u]];
              if (amb_key(uf[u], sg[u], E.f.col.x) <= 1.0f) {
                const double x = exact_entry(E, fx, fy);
                ok[u] = x >= 0.0;
                sg[u] = (float)x;
                sx[u] = x;
              }
            }
          }
          // general path: the reference's sequential decisions, entry by entry
#pragma unroll
          for (int u = 0; u < 2; u++) {
            const bool act = !done && (u == 0 || has1);
            if (STATS && act) walked++;
            if (act && dstop[u]) done = true;  // list is depth sorted; mesh is opaque
            const bool v = act && !dstop[u] && ok[u];
            const float sig = v ? sg[u] : 0.0f;
            const float om = 1.0f - sig;
            const float test = T * om;
            const float w = T * sig;
            // |test - T_ref (1 - sigma_ref)| <= eT om + w EPS_SIG + test 2^-23
            // (skipped entries only add the rounding term: conservative)
            eT = fmaf(w, EPS_SIG, fmaf(eT, om, test * 1.1920929e-7f));
            bool stop = false;
            if (v && fmaf(-2.0f, eT, test) < STOP_NEAR) {  // the early-stop region
              // the decision is ambiguous within the error band -> exact replay
              if (fabsf(test - STOP_F) <= fmaf(eT, 1.001f, 3e-12f)) flagged = true;
              stop = test < STOP_F;
              if (stop) done = true;
            }
            const bool upd = v && !stop;
            const StageEntry& E = sm.ent[slot][jj[u]];
            const float wu = upd ? w : 0.0f;
            r = fmaf(E.f.col.y, wu, r);
            g = fmaf(E.f.col.z, wu, g);
            bl = fmaf(E.f.col.w, wu, bl);
            dacc = fmaf(E.f.con.w, wu, dacc);
            acc += wu;
            T = upd ? test : T;
            if (upd) {
              last = b * BATCH + jj[u];
              if (STATS) blended++;
              if (PREC)
                T64 *= 1.0 - (sx[u] >= 0.0 ? sx[u] : fmin(E.d.x * exp2_neg64(um[u], uf[u], sm.exp2tab), ALPHA_CLAMP));
            }
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
    fixup[1 + slot] = (int32_t)p + 1;
    return;
  }
  write_pixel(out, mesh, mesh_here, p, T, r, g, bl, dacc, acc, last >= 0 ? s + last : -1, bg0, bg1, bg2,
              mask_variant, mask_k, PREC ? T64 : (double)T);
}

// ---------------------------------------------------------------------------
// blend_tile_kernel: the production fast path (the kernel above is kept as
// the A/B baseline, HGS_BLEND_V1).  Same numerics contract, re-shaped to
// spend fewer instructions per (pixel, entry):
//  * 4 consumer warps own 8x8 sub-tiles, TWO pixels per lane ((x, y) and
//    (x, y + 4)): every per-entry cost -- shared-memory loads of the record,
//    the list walk, the warp vote, dx = fx - mean x and conic_xx * dx (the
//    two pixels share the column) -- is paid once for two pixels, and the two
//    pixels' independent recurrences give the ILP the old kernel got from
//    evaluating two entries per step;
//  * the support and skip decisions are one compare against the entry's cut
//    ucut = min(9 U, log2(255 alpha)) (entry_ucut, stage.cuh), computed once
//    per (warp, entry) by the cull and kept next to the list index;
//  * the producer moves each record with two bulk copies (TMA engine,
//    cp.async.bulk, 64 B fp64 record head + 48 B fp32 cull record) whose
//    bytes complete the stage's mbarrier, instead of seven 16-B cp.async.
// Decisions stay the reference's: guard band around the cut (exact fp64
// re-evaluation inside it), exact fp64 depth stop, fp32 T with the carried
// error bound eT and the exact replay of pixels whose early stop is
// ambiguous.
#ifndef HGS_TB_BATCH
#define HGS_TB_BATCH 64
#endif
#ifndef HGS_TB_NSTAGE
#define HGS_TB_NSTAGE 2
#endif
#ifndef HGS_TB_MINB
#define HGS_TB_MINB 5
#endif
#ifndef HGS_TB_MINB_PREC
#define HGS_TB_MINB_PREC 5
#endif
#ifndef HGS_TB_BULK
#define HGS_TB_BULK 0
#endif
constexpr int TB_BATCH = HGS_TB_BATCH;
constexpr int TB_NSTAGE = HGS_TB_NSTAGE;
constexpr int TB_CONSUMERS = 4;
constexpr int TB_THREADS = (TB_CONSUMERS + 1) * 32;
constexpr unsigned TB_REC_BYTES = 64, TB_CULL_BYTES = 48;

// A culled entry, copied by the cull into the warp's own walk buffer (the
// walk then reads consecutive records -- no index -> record load chain --
// and the ring slot is released as soon as every warp has culled it).
struct __align__(16) WalkRec {
  double2 a;  // mean x, y
  double2 b;  // U conic xx, U 2xy (U = log2(e)/2: the conic form is the exp2 argument)
  double2 c;  // U conic yy, depth
  union {
    double alpha;  // PREC: the fp64 alpha (T64 recurrence)
    struct {
      float a32;     // otherwise |fp32 alpha| (saves the walk a conversion per entry)
      uint32_t row;  // ... and the Gaussian's row (blend-only bins: the exact re-evaluation's record)
    };
  };
  float ucut;  // the entry's cut (entry_ucut)
  int k;       // entry index relative to the tile start
  float4 col;  // r, g, b, depth (fp32)
};
static_assert(sizeof(WalkRec) == 80, "walk record is 80 B");

template <bool PREC>
struct TileSmem {
  StageEntry ent[TB_NSTAGE][TB_BATCH];
  WalkRec walk[TB_CONSUMERS][TB_BATCH];
  float tout[2][TB_CONSUMERS][2][32];  // transmittance and last entry of finished pixels (TbPix, tb_finish)
  // blend-only bins (coarse-fed producer): per ring slot the entry count,
  // the tile-list index of its first entry, and every entry's row
  int nbs[TB_NSTAGE];
  int kbase[TB_NSTAGE];
  uint32_t gid[TB_NSTAGE][TB_BATCH];
  unsigned long long full[TB_NSTAGE];
  unsigned long long empty[TB_NSTAGE];
  double exp2tab[PREC ? EXP2_N : 1];  // (the fp64 exp2 table: training state only)
  int done_warps;
  int end_batch;
  int finished_warps;
  int tile_id;
  unsigned long long stats[2];
};

// Per-pixel walk state.  A finished pixel is made inert instead of being
// tested per entry: T = 0 (its blend terms vanish), e2 = -inf (no early-stop
// region: the threshold below is -inf and stays so), lim_hi = INT_MAX (no
// depth stop); its transmittance is parked in shared memory.  Only an entry
// inside the cut band still sends it to the (then immediate) general path.
struct TbPix {
  float T, e2, acc, r, g, b, dacc;  // e2 = 2 eT: twice the bound on |T - T_reference| (exact scaling)
  int last;
  int lim_hi;  // high word of the mesh depth limit (positive fp64: the word order is the value order)
  bool flagged;
  double T64;
  __device__ __forceinline__ bool done() const { return T == 0.0f; }
};

__device__ __forceinline__ void tb_finish(TbPix& q, float* tout) {
  tout[0] = q.T;
  reinterpret_cast<int*>(tout)[TB_CONSUMERS * 2 * 32] = q.last;  // (the walk keeps updating an inert pixel's last)
  q.T = 0.0f;
  q.e2 = -__int_as_float(0x7f800000);
  q.lim_hi = 0x7fffffff;
}

// The general (sequential, exact where needed) treatment of one entry for
// one pixel: depth stop, exact re-evaluation inside the cut band, the
// early-stop region with the error bound.  k: entry index relative to the
// tile start.
// exact re-evaluation from the Gaussian's fp64 record in global memory (the
// walk record holds the scaled conic)
__device__ __noinline__ double exact_global(const BlendRec* __restrict__ rec, uint32_t row, double fx, double fy) {
  const BlendRec& R = rec[row];
  const double dx = fx - R.mx, dy = fy - R.my;
  const double m = R.ca * dx * dx + R.cb2 * dx * dy + R.cc * dy * dy;
  if (m > SUPPORT_MAHAL2 || m < 0.0) return -1.0;
  double sg = R.alpha * exp(-0.5 * m);
  if (sg > ALPHA_CLAMP) sg = ALPHA_CLAMP;
  return sg < SIGMA_SKIP ? -1.0 : sg;
}

template <bool STATS, bool PREC>
__device__ __forceinline__ void tb_slow(TbPix& q, const WalkRec& E, double fx, double fy, const double* limit,
                                        float uu, double um, float sg, float d, int k, const double* tab,
                                        const BlendRec* __restrict__ rec, const uint32_t* __restrict__ entries,
                                        int64_t s, unsigned& walked, unsigned& blended, float* tout) {
  if (q.done()) return;
  if (STATS) walked++;
  // list is depth sorted; mesh is opaque.  Equal high words: the full fp64
  // compare (limit NULL: no mesh here, +inf)
  if (__double2hiint(E.c.y) >= q.lim_hi && limit && E.c.y >= *limit) {
    tb_finish(q, tout);
    return;
  }
  bool ok = d < -U_BAND;
  double sx = -1.0;
  if (!(fabsf(d) > U_BAND)) {  // within the cut band (or a NaN cut): decide exactly
    sx = exact_global(rec, entries ? entries[s + k] : E.row, fx, fy);  // (entries NULL: coarse-fed)
    ok = sx >= 0.0;
    sg = (float)sx;
  }
  if (!ok) return;  // not blended: T is unchanged (exactly), so is the bound
  const float test = fmaf(-q.T, sg, q.T);
  const float w = q.T * sg;
  q.e2 = fmaf(w, 2.0f * EPS_SIG, fmaf(-q.e2, sg, fmaf(test, 1.1920929e-7f, q.e2)));
  if (test - q.e2 < STOP_NEAR) {  // the early-stop region
    if (fabsf(test - STOP_F) <= fmaf(q.e2, 0.5005f, 3e-12f)) q.flagged = true;
    if (test < STOP_F) {
      tb_finish(q, tout);
      return;
    }
  }
  q.r = fmaf(E.col.x, w, q.r);
  q.g = fmaf(E.col.y, w, q.g);
  q.b = fmaf(E.col.z, w, q.b);
  q.dacc = fmaf(E.col.w, w, q.dacc);
  q.acc += w;
  q.T = test;
  q.last = k;
  if (STATS) blended++;
  if (PREC) q.T64 *= 1.0 - (sx >= 0.0 ? sx : fmin(E.alpha * exp2_neg64(um, uu, tab), ALPHA_CLAMP));
}

template <bool STATS, bool PREC>
__global__ void __launch_bounds__(TB_THREADS, PREC ? HGS_TB_MINB_PREC : HGS_TB_MINB) blend_tile_kernel(
    const BlendRec* __restrict__ rec, const CullRec* __restrict__ cull, const uint32_t* __restrict__ entries,
    const int64_t* __restrict__ tile_starts, int tiles_x, int width, int height, hgs_mesh_layer mesh, double bg0,
    double bg1, double bg2, int mask_variant, double mask_k, hgs_blend_out out, int32_t* __restrict__ fixup,
    const int64_t* __restrict__ counters, int* ready, int qs, int sx_super, const uint32_t* __restrict__ crow,
    const uint2* __restrict__ crect, const uint32_t* __restrict__ cstart, int css, uint4* __restrict__ prog) {
  // crow != NULL (blend-only bins, never PREC): the producer filters the
  // tile's super-tile coarse list (super-tiles of 2^css tiles, sx_super per
  // row) into the ring instead of reading `entries`.
  // ready != NULL: launched behind the fine binning without waiting for its
  // grid; each CTA claims the next tile of the quads it has published
  // (common.cuh).  Otherwise: one CTA per tile after the binning completed.
  if (ready)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  else
    pdl_enter();
  if (counters && counters[2]) return;  // entry buffer overflowed: bins are invalid, the caller re-renders
  extern __shared__ __align__(128) unsigned char tile_smem_raw[];
  TileSmem<PREC>& sm = *reinterpret_cast<TileSmem<PREC>*>(tile_smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < TB_NSTAGE; i++) {
      mbar_init(&sm.full[i], 32);
      mbar_init(&sm.empty[i], TB_CONSUMERS);
    }
    sm.done_warps = 0;
    sm.end_batch = 0x7fffffff;
    sm.finished_warps = 0;
    sm.stats[0] = sm.stats[1] = 0;
    int t = blockIdx.x;
    if (ready) {
      const int idx = atomicAdd(&ready[1], 1);
      const volatile int* vr = ready;
      int qv;
      for (uint32_t spin = 0; (qv = vr[READY_HDR + (idx >> 4)]) == 0; spin++) {
        if (spin > QUEUE_SPIN_LIMIT) __trap();  // never hang the GPU on a broken handoff
        __nanosleep(256);
      }
      __threadfence();  // the quad's entries (published after a fence) are visible from here on
      const int sq = qv - 1;
      const int sup = sq >> (2 * qs), quad = sq & ((1 << (2 * qs)) - 1);
      const int tx0 = (sup % sx_super) * (4 << qs) + (quad & ((1 << qs) - 1)) * 4;
      const int ty0 = (sup / sx_super) * (4 << qs) + (quad >> qs) * 4;
      const int ttx = tx0 + (idx & 3), tty = ty0 + ((idx >> 2) & 3);
      t = (ttx < tiles_x && tty * BLEND_TILE < height) ? tty * tiles_x + ttx : -1;
    }
    sm.tile_id = t;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (PREC) exp2_tab_load(sm.exp2tab);
  __syncthreads();
  const int tile = sm.tile_id;
  if (tile < 0) {  // a claim past the grid edge: no tile, but counted as finished
    if (threadIdx.x == 0) atomicAdd(&fixup[FIX_DONE], 1);
    return;
  }
  const int64_t s = tile_starts[tile], e = tile_starts[tile + 1];
  const bool coarse = !PREC && crow != nullptr;
  uint32_t* const entries_w = const_cast<uint32_t*>(entries);  // (blend-only bins: the prefix is written here)
  const int nbatches = coarse ? 0x7fffffff : (int)((e - s + TB_BATCH - 1) / TB_BATCH);
  const int tx = tile % tiles_x, ty = tile / tiles_x;

  if (warp == TB_CONSUMERS && coarse) {
    // ------------------------------------------- producer, coarse-fed
    // the super-tile's list in depth order; the entries whose rectangle
    // covers this tile are this tile's list (fine_bin_kernel's filter), in
    // order.  A batch takes rounds of 32 list entries until its 64 slots are
    // full (a round may straddle two batches); the next rounds' loads are in
    // flight.
    const int sup = (ty >> css) * sx_super + (tx >> css);
    const uint32_t cb = counters[0] > 0 ? cstart[sup] : 0u, ce = counters[0] > 0 ? cstart[sup + 1] : 0u;
    const uint32_t clast = ce > cb ? ce - 1 : cb;
    constexpr int PD = 4;  // rounds in flight
    uint2 rq[PD];
    uint32_t gq[PD];
#pragma unroll
    for (int d = 0; d < PD; d++) {
      const uint32_t i = min(cb + 32 * d + lane, clast);
      rq[d] = __ldg(crect + i);
      gq[d] = __ldg(crow + i);
    }
    uint32_t pos = cb;
    int kcount = 0;
    int skip = 0;  // matches of the current round already placed (a round may straddle two batches)
    for (int b = 0;; b++) {
      const int slot = b % TB_NSTAGE;
      if (b >= TB_NSTAGE) warp_wait(&sm.empty[slot], ((b / TB_NSTAGE) - 1) & 1, lane);
      if (*(volatile int*)&sm.done_warps == TB_CONSUMERS || pos >= ce) {
        if (lane == 0) *(volatile int*)&sm.end_batch = b;
        __syncwarp();
        mbar_arrive(&sm.full[slot]);  // 32 plain arrivals complete the phase
        break;
      }
      int filled = 0;
      const int kbase_b = kcount;
      while (filled < TB_BATCH && pos < ce) {
        const uint32_t i = pos + lane;
        const uint32_t lo = rq[0].x, hi = rq[0].y;  // (x0 | x1 << 16, y0 | y1 << 16)
        const bool hit = i < ce && (int)(lo & 0xffffu) <= tx && tx <= (int)(lo >> 16) && (int)(hi & 0xffffu) <= ty &&
                         ty <= (int)(hi >> 16);
        const uint32_t g = gq[0];
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        const int rank = __popc(bal & lanemask_lt()) - skip;
        const int take = min(__popc(bal) - skip, TB_BATCH - filled);
        if (hit && rank >= 0 && rank < take) {
          const int j = filled + rank;
          StageEntry* dst = &sm.ent[slot][j];
          const char* src = reinterpret_cast<const char*>(rec + g);
          const char* cs = reinterpret_cast<const char*>(cull + g);
          cp_async16(&dst->a, src);
          cp_async16(&dst->b, src + 16);
          cp_async16(&dst->c, src + 32);
          cp_async16(&dst->d, src + 48);
          cp_async16(&dst->f.box, cs);
          cp_async16(&dst->f.con, cs + 16);
          cp_async16(&dst->f.col, cs + 32);
          sm.gid[slot][j] = g;
          entries_w[s + kbase_b + j] = g;  // the tile list prefix, for the exact replay
        }
        filled += take;
        if (skip + take < __popc(bal)) {  // the batch is full: the rest of this round opens the next one
          skip += take;
          break;
        }
        skip = 0;
#pragma unroll
        for (int d = 0; d < PD - 1; d++) rq[d] = rq[d + 1], gq[d] = gq[d + 1];
        {
          const uint32_t inext = min(pos + 32 * PD + lane, clast);
          rq[PD - 1] = __ldg(crect + inext);
          gq[PD - 1] = __ldg(crow + inext);
        }
        pos += 32;
      }
      if (lane == 0) {
        sm.nbs[slot] = filled;
        sm.kbase[slot] = kcount;
      }
      kcount += filled;
      __syncwarp();
      __threadfence_block();  // the slot's count / rows before the arrivals that publish it
      cp_async_arrive_noinc(&sm.full[slot]);
    }
    // where the tile list prefix in `entries` ends, for the exact replay of
    // this tile's ambiguous pixels (queued by the consumers after the barrier)
    if (lane == 0) prog[tile] = make_uint4((uint32_t)kcount, pos, (uint32_t)skip, 0u);
    __threadfence();
    __syncthreads();
    return;
  }

  if (warp == TB_CONSUMERS) {
    // ------------------------------------------------------------ producer
    for (int b = 0; b < nbatches; b++) {
      const int slot = b % TB_NSTAGE;
      if (b >= TB_NSTAGE) warp_wait(&sm.empty[slot], ((b / TB_NSTAGE) - 1) & 1, lane);
      if (*(volatile int*)&sm.done_warps == TB_CONSUMERS) {
        if (lane == 0) *(volatile int*)&sm.end_batch = b;
        __syncwarp();
        mbar_arrive(&sm.full[slot]);  // 32 plain arrivals complete the phase
        break;
      }
      const int64_t base = s + (int64_t)b * TB_BATCH;
      const int nb = (int)min((int64_t)TB_BATCH, e - base);
      const int mine = nb > lane ? (nb - lane + 31) >> 5 : 0;
      uint32_t g[TB_BATCH / 32];
#pragma unroll
      for (int u = 0; u < TB_BATCH / 32; u++)
        if (u < mine) g[u] = __ldcg(entries + base + lane + 32 * u);  // L2: written while the blend started
#if HGS_TB_BULK
      // A/B: bulk copies take their operands in uniform registers, so the
      // compiler issues them one lane at a time (an elect loop of ~9
      // instructions per copy): 3x the producer's issue slots of the
      // cp.async version below and consumers starved (r02 profile)
      mbar_arrive_expect_tx(&sm.full[slot], (unsigned)mine * (TB_REC_BYTES + TB_CULL_BYTES));
#pragma unroll
      for (int u = 0; u < TB_BATCH / 32; u++)
        if (u < mine) {
          StageEntry* dst = &sm.ent[slot][lane + 32 * u];
          bulk_g2s(&dst->a, rec + g[u], TB_REC_BYTES, &sm.full[slot]);
          bulk_g2s(&dst->f, cull + g[u], TB_CULL_BYTES, &sm.full[slot]);
        }
#else
#pragma unroll
      for (int u = 0; u < TB_BATCH / 32; u++)
        if (u < mine) {
          StageEntry* dst = &sm.ent[slot][lane + 32 * u];
          const char* src = reinterpret_cast<const char*>(rec + g[u]);
          const char* cs = reinterpret_cast<const char*>(cull + g[u]);
          cp_async16(&dst->a, src);
          cp_async16(&dst->b, src + 16);
          cp_async16(&dst->c, src + 32);
          cp_async16(&dst->d, src + 48);
          cp_async16(&dst->f.box, cs);
          cp_async16(&dst->f.con, cs + 16);
          cp_async16(&dst->f.col, cs + 32);
        }
      cp_async_arrive_noinc(&sm.full[slot]);
#endif
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  // warp w owns the 8x8 sub-tile (w & 1, w >> 1); lane (x, y) = (lane & 7,
  // lane >> 3) holds pixels (x, y) and (x, y + 4)
  const int sx0 = (warp & 1) * 8, sy0 = (warp >> 1) * 8;
  const int px = tx * BLEND_TILE + sx0 + (lane & 7);
  const int py0 = ty * BLEND_TILE + sy0 + (lane >> 3);
  const double fx = px + 0.5, fy0 = py0 + 0.5;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const float wx0 = tx * BLEND_TILE + sx0 + 0.5f, wx1 = wx0 + 7.0f;
  const float wy0 = ty * BLEND_TILE + sy0 + 0.5f, wy1 = wy0 + 7.0f;
  TbPix q[2];
  bool inside[2];
  int64_t pix[2];
  bool mesh_here[2];
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int py = py0 + 4 * h;
    inside[h] = px < width && py < height;
    pix[h] = (int64_t)py * width + px;
    mesh_here[h] = mesh.color != nullptr && inside[h] && mesh.triangle_id[pix[h]] >= 0;
    q[h].lim_hi = __double2hiint(mesh_here[h] ? mesh.depth[pix[h]] : inf);
    q[h].T = 1.0f;
    q[h].e2 = q[h].acc = q[h].r = q[h].g = q[h].b = q[h].dacc = 0.0f;
    q[h].last = -1;
    q[h].flagged = false;
    q[h].T64 = 1.0;
    if (!inside[h]) tb_finish(q[h], &sm.tout[0][warp][h][lane]);
  }
  bool warp_done = false;
  unsigned walked = 0, blended = 0;

  for (int b = 0; b < nbatches; b++) {
    const int slot = b % TB_NSTAGE;
    warp_wait(&sm.full[slot], (b / TB_NSTAGE) & 1, lane);
    if (b >= *(volatile int*)&sm.end_batch) break;
    if (warp_done) {
      if (lane == 0) mbar_arrive(&sm.empty[slot]);
      continue;
    }
    const int nb = coarse ? sm.nbs[slot] : (int)min((int64_t)TB_BATCH, e - (s + (int64_t)b * TB_BATCH));
    const int bb = coarse ? sm.kbase[slot] : b * TB_BATCH;
    // order-preserving compaction of the stage to the entries whose effective
    // ellipse touches the sub-tile, copied with their cut into the warp's
    // walk buffer; then the ring slot is released
    int nl = 0;
#pragma unroll
    for (int k = 0; k < TB_BATCH; k += 32) {
      const int i = k + lane;
      float4 bx = make_float4(0.f, 0.f, -1.f, -1.f);
      if (i < nb) bx = sm.ent[slot][i].f.box;
      const float cx = fminf(fmaxf(bx.x, wx0), wx1), cy = fminf(fmaxf(bx.y, wy0), wy1);
      bool hit = fabsf(bx.x - cx) <= bx.z && fabsf(bx.y - cy) <= bx.w;
      if (hit && (bx.x != cx || bx.y != cy)) hit = ellipse_meets_box(sm.ent[slot][i].f.con, bx, wx0, wx1, wy0, wy1);
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const StageEntry& S = sm.ent[slot][i];
        WalkRec& W = sm.walk[warp][nl + __popc(m & lanemask_lt())];
        W.a = S.a;
        W.b = make_double2(S.b.x * U_SCALE, S.b.y * U_SCALE);
        W.c = make_double2(S.c.x * U_SCALE, S.c.y);
        if (PREC) {
          W.alpha = S.d.x;
        } else {
          W.a32 = fabsf(S.f.col.x);  // == |(float)alpha| (the cull record's sign only flags the conic)
          W.row = coarse ? sm.gid[slot][i] : 0u;
        }
        W.ucut = entry_ucut(S.f.col.x);
        W.k = bb + i;
        W.col = make_float4(S.f.col.y, S.f.col.z, S.f.col.w, S.f.con.w);
      }
      nl += __popc(m);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[slot]);
    for (int li = 0; li < nl; li++) {
      const WalkRec& E = sm.walk[warp][li];
      const double2 A = E.a, B = E.b, C = E.c;
      const float ucut = E.ucut;
      const float aabs = PREC ? fabsf((float)E.alpha) : E.a32;
      const double dx = fx - A.x;
      const double adx = B.x * dx;
      const int zhi = __double2hiint(C.y);
      float uu[2], sg[2], dd[2], sv[2], Tn[2], e2n[2], w[2];
      double um[2];
      bool spec[2], ok[2];
      double dy = fy0 - A.y;
      float thr[2];
#pragma unroll
      for (int h = 0; h < 2; h++) thr[h] = fmaf(q[h].T, 2.0f * (EPS_SIG + 1.1920929e-7f), q[h].e2) + STOP_NEAR;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        if (h) dy = dy + 4.0;  // (x, y + 4): within the guard band of the direct difference
        um[h] = fma(dx, fma(B.y, dy, adx), (C.x * dy) * dy);
        uu[h] = __double2float_rn(um[h]);
        sg[h] = fminf(aabs * ex2_neg(uu[h]), CLAMP_F);
        dd[h] = uu[h] - ucut;
        // (a finished pixel has T = 0: whatever sv is, its terms vanish)
        ok[h] = dd[h] < -U_BAND;
        sv[h] = ok[h] ? sg[h] : 0.0f;
        // T (1 - sv) with one rounding (|err| <= 2^-24 T'), so the bound grows
        // by e (1 - sv) + w EPS_SIG + 2^-24 T' (doubled: e2)
        Tn[h] = fmaf(-q[h].T, sv[h], q[h].T);
        w[h] = q[h].T * sv[h];
        e2n[h] = fmaf(w[h], 2.0f * EPS_SIG, fmaf(-q[h].e2, sv[h], fmaf(Tn[h], 1.1920929e-7f, q[h].e2)));
        // a decision this entry could get wrong: depth stop, the cut band
        // (or a NaN cut), the early-stop region.  The last is tested as
        // Tn < STOP_NEAR + 2 (eT + T (EPS_SIG + 2^-23)) >= STOP_NEAR + 2 eTn
        // (om <= 1, w <= T): the threshold comes from the state before the
        // entry, off the entry's dependency chain.  An inert (finished)
        // pixel only meets the cut band (rare; tb_slow returns at once).
        spec[h] = zhi >= q[h].lim_hi || !(fabsf(dd[h]) > U_BAND) || Tn[h] < thr[h];
      }
      if (!__any_sync(0xffffffffu, spec[0] || spec[1])) {
        const float4 col = E.col;
        const int k = E.k;
#pragma unroll
        for (int h = 0; h < 2; h++) {
          if (STATS && !q[h].done()) {
            walked++;
            blended += sv[h] > 0.0f;
          }
          q[h].T = Tn[h];
          q[h].e2 = e2n[h];
          q[h].r = fmaf(col.x, w[h], q[h].r);
          q[h].g = fmaf(col.y, w[h], q[h].g);
          q[h].b = fmaf(col.z, w[h], q[h].b);
          q[h].dacc = fmaf(col.w, w[h], q[h].dacc);
          q[h].acc += w[h];
          q[h].last = ok[h] ? k : q[h].last;  // (garbage on a finished pixel: tb_finish parked its last)
          if (PREC && w[h] > 0.0f)
            q[h].T64 *= 1.0 - fmin(E.alpha * exp2_neg64(um[h], uu[h], sm.exp2tab), ALPHA_CLAMP);
        }
      } else {
#pragma unroll
        for (int h = 0; h < 2; h++)
          tb_slow<STATS, PREC>(q[h], E, fx, fy0 + 4.0 * h, mesh_here[h] ? mesh.depth + pix[h] : nullptr, uu[h],
                               um[h], sg[h], dd[h], E.k, sm.exp2tab, rec, coarse ? nullptr : entries, s, walked, blended,
                               &sm.tout[0][warp][h][lane]);
        if (__all_sync(0xffffffffu, q[0].done() && q[1].done())) break;
      }
    }
    if (__all_sync(0xffffffffu, q[0].done() && q[1].done())) {
      warp_done = true;
      if (lane == 0) atomicAdd(&sm.done_warps, 1);
    }
  }
  if (STATS) {
    atomicAdd(&sm.stats[0], (unsigned long long)walked);
    atomicAdd(&sm.stats[1], (unsigned long long)blended);
    // consumers only: the producer may already have left
    asm volatile("bar.sync 1, %0;" ::"n"(TB_CONSUMERS * 32));
    if (threadIdx.x == 0) {
      atomicAdd((unsigned long long*)&out.stats[0], sm.stats[0]);
      atomicAdd((unsigned long long*)&out.stats[1], sm.stats[1]);
    }
  }
  if (coarse) __syncthreads();  // the producer has published the tile's list prefix (prog) for the replays
#pragma unroll
  for (int h = 0; h < 2; h++) {
    if (!inside[h]) continue;
    if (q[h].flagged) {  // queue the pixel for the exact walk (slot value pixel + 1; 0 = empty)
      const int slot = atomicAdd(&fixup[FIX_RESERVED], 1);
      fixup[FIX_SLOTS + slot] = (int32_t)pix[h] + 1;
      if (STATS) atomicAdd((unsigned long long*)&out.stats[2], 1ull);
      continue;
    }
    const float Tfin = q[h].done() ? sm.tout[0][warp][h][lane] : q[h].T;
    if (q[h].done()) q[h].last = __float_as_int(sm.tout[1][warp][h][lane]);
    write_pixel(out, mesh, mesh_here[h], pix[h], Tfin, q[h].r, q[h].g, q[h].b, q[h].dacc, q[h].acc,
                q[h].last >= 0 ? s + q[h].last : -1, bg0, bg1, bg2, mask_variant, mask_k,
                PREC ? q[h].T64 : (double)Tfin);
  }
  // the tile is finished once its last consumer warp is: count it for the
  // exact-walk kernel, which drains the queue while the blend still runs
  __threadfence();
  __syncwarp();
  if (lane == 0 && atomicAdd(&sm.finished_warps, 1) == TB_CONSUMERS - 1) {
    __threadfence();
    atomicAdd(&fixup[FIX_DONE], 1);
  }
}

// The exact walk, one warp per pixel (persistent grid-stride): over the
// fast kernel's work list of flagged pixels (fixup: count, pixel ids), or
// over every pixel (fixup == NULL: projections without fp32 cull records).
__global__ void __launch_bounds__(256) blend_exact_kernel(
    const BlendRec* __restrict__ rec, const uint32_t* __restrict__ entries, const int64_t* __restrict__ tile_starts,
    int tiles_x, int width, int height, hgs_mesh_layer mesh, double bg0, double bg1, double bg2, int mask_variant,
    double mask_k, hgs_blend_out out, const int32_t* __restrict__ fixup, const int64_t* __restrict__ counters) {
  pdl_enter();
  if (counters && counters[2]) return;  // overflowed bins (see blend_fast_kernel)
  const int64_t count = fixup ? fixup[0] : (int64_t)width * height;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t wi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); wi < count; wi += nwarps) {
    const int64_t p = fixup ? fixup[1 + wi] - 1 : wi;
    const int px = (int)(p % width), py = (int)(p / width);
    const int tile = (py / BLEND_TILE) * tiles_x + px / BLEND_TILE;
    const bool mesh_here = mesh.color != nullptr && mesh.triangle_id[p] >= 0;
    const double limit = mesh_here ? mesh.depth[p] : __longlong_as_double(0x7ff0000000000000LL);
    const ExactPixel q = exact_walk2(rec, entries, tile_starts[tile], tile_starts[tile + 1], px + 0.5, py + 0.5,
                                    limit, lane);
    if (lane == 0)
      write_pixel(out, mesh, mesh_here, p, q.T, q.r, q.g, q.b, q.dacc, 1.0 - q.T, q.last, bg0, bg1, bg2,
                  mask_variant, mask_k, q.T);
  }
}

// The exact walk as a queue consumer running beside the blend: launched
// right behind blend_tile_kernel (programmatic launch: its CTAs start once
// every blend CTA has started) it does NOT wait for the blend grid; warps
// claim queue slots and replay each flagged pixel as soon as its tile has
// queued it, so the replays overlap the blend's last waves instead of
// following them.  Exits when every tile is finished and the queue is
// drained.  Slots are reset to 0 after use (the queue is empty at rest).
__global__ void __launch_bounds__(64) blend_exact_queue_kernel(
    const BlendRec* __restrict__ rec, const uint32_t* __restrict__ entries, const int64_t* __restrict__ tile_starts,
    int tiles_x, int n_tiles, int width, hgs_mesh_layer mesh, double bg0, double bg1, double bg2, int mask_variant,
    double mask_k, hgs_blend_out out, int32_t* fixup, const int64_t* __restrict__ counters, int* ready,
    const uint32_t* __restrict__ crow, const uint2* __restrict__ crect, const uint32_t* __restrict__ cstart, int css,
    int sx_super, const uint4* __restrict__ prog) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (counters && counters[2]) return;  // overflowed bins: the blend wrote nothing
  const int lane = threadIdx.x & 31;
  volatile int32_t* vf = fixup;
  // n_tiles: blend CTAs to wait for.  The last warp to leave puts the
  // counters (and the blend's tile-claim counter) back to 0: the queue is
  // zero at rest, no reset launch sits between the binning and the blend.
  struct Leave {
    int32_t* f;
    int* r;
    int lane, nw;
    __device__ ~Leave() {
      if (lane == 0 && atomicAdd(&f[FIX_EXITED], 1) == nw - 1) {
        f[FIX_RESERVED] = 0;
        f[FIX_DONE] = 0;
        f[FIX_CLAIMED] = 0;
        f[FIX_EXITED] = 0;
        if (r) r[1] = 0;
        __threadfence();
      }
    }
  } leave{fixup, ready, lane, (int)(gridDim.x * (blockDim.x >> 5))};
  while (true) {
    int idx = 0, quit = 0;
    if (lane == 0) {
      idx = atomicAdd(&fixup[FIX_CLAIMED], 1);
      for (uint32_t spin = 0;; spin++) {
        if (spin > QUEUE_SPIN_LIMIT) __trap();
        if (idx < vf[FIX_RESERVED]) break;  // a pixel is (or is being) queued in this slot
        if (vf[FIX_DONE] == n_tiles) {  // all tiles finished: the reservation count is final
          __threadfence();
          if (idx >= vf[FIX_RESERVED]) quit = 1;
          break;
        }
        __nanosleep(500);
      }
    }
    quit = __shfl_sync(0xffffffffu, quit, 0);
    if (quit) break;
    idx = __shfl_sync(0xffffffffu, idx, 0);
    int32_t v = 0;
    if (lane == 0) {
      for (uint32_t spin = 0; (v = vf[FIX_SLOTS + idx]) == 0; spin++) {
        if (spin > QUEUE_SPIN_LIMIT) __trap();
        __nanosleep(100);
      }
      vf[FIX_SLOTS + idx] = 0;
    }
    const int64_t p = __shfl_sync(0xffffffffu, v, 0) - 1;
    const int px = (int)(p % width), py = (int)(p / width);
    const int tile = (py / BLEND_TILE) * tiles_x + px / BLEND_TILE;
    const bool mesh_here = mesh.color != nullptr && mesh.triangle_id[p] >= 0;
    const double limit = mesh_here ? mesh.depth[p] : __longlong_as_double(0x7ff0000000000000LL);
    ExactPixel q;
    if (crow) {  // blend-only bins: the tile's list is filtered out of its super-tile's coarse list
      const int tx = px / BLEND_TILE, ty = py / BLEND_TILE;
      const int sup = (ty >> css) * sx_super + (tx >> css);
      const uint4 pg = __ldcg(prog + tile);
      q = exact_walk_blend_only(rec, entries, tile_starts[tile], (int)pg.x, crow, crect, pg.y, (int)pg.z,
                                cstart[sup + 1], tx, ty, px + 0.5, py + 0.5, limit, lane);
    } else {
      q = exact_walk2(rec, entries, tile_starts[tile], tile_starts[tile + 1], px + 0.5, py + 0.5, limit, lane);
    }
    if (lane == 0)
      write_pixel(out, mesh, mesh_here, p, q.T, q.r, q.g, q.b, q.dacc, 1.0 - q.T, q.last, bg0, bg1, bg2,
                  mask_variant, mask_k, q.T);
  }
}

// CTA-parallel exact replay (one CTA of EXW warps per queued pixel): a
// replay is one warp's sequential walk of up to ~1000 entries (~24 us on
// average at c3), and the last replays are the frame's tail.  Here the warps
// take interleaved rounds of 64 entries: each evaluates its round (records,
// fp64 exp, depth stop, the in-round prefix products) in parallel, then the
// rounds are committed in order, warp after warp, with the T the previous
// round left -- the same arithmetic per round as exact_walk2.  Blend-only
// bins: the tile-list prefix in `entries`, then warp 0 continues over the
// coarse list (exact_walk_coarse_run).
#ifndef HGS_EXW
#define HGS_EXW 4
#endif
#ifndef HGS_EX_CTAS_PER_SM
#define HGS_EX_CTAS_PER_SM 2
#endif
constexpr int EXW = HGS_EXW;
__global__ void __launch_bounds__(EXW * 32) blend_exact_cta_kernel(
    const BlendRec* __restrict__ rec, const uint32_t* __restrict__ entries, const int64_t* __restrict__ tile_starts,
    int tiles_x, int n_tiles, int width, hgs_mesh_layer mesh, double bg0, double bg1, double bg2, int mask_variant,
    double mask_k, hgs_blend_out out, int32_t* fixup, const int64_t* __restrict__ counters, int* ready,
    const uint32_t* __restrict__ crow, const uint2* __restrict__ crect, const uint32_t* __restrict__ cstart, int css,
    int sx_super, const uint4* __restrict__ prog) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (counters && counters[2]) return;  // overflowed bins: the blend wrote nothing
  constexpr int EW = 2, RW = 32 * EW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  volatile int32_t* vf = fixup;
  __shared__ int s_claim, s_quit;
  __shared__ double s_T;
  __shared__ long long s_last;
  __shared__ int s_done;
  __shared__ double s_sum[EXW][4];
  struct Leave {  // the last CTA to leave puts the queue back to zero (zero at rest)
    int32_t* f;
    int* r;
    int tid, n;
    __device__ ~Leave() {
      if (tid == 0 && atomicAdd(&f[FIX_EXITED], 1) == n - 1) {
        f[FIX_RESERVED] = 0;
        f[FIX_DONE] = 0;
        f[FIX_CLAIMED] = 0;
        f[FIX_EXITED] = 0;
        if (r) r[1] = 0;
        __threadfence();
      }
    }
  } leave{fixup, ready, tid, (int)gridDim.x};
  while (true) {
    if (tid == 0) {
      int idx = atomicAdd(&fixup[FIX_CLAIMED], 1), quit = 0;
      for (uint32_t spin = 0;; spin++) {
        if (spin > QUEUE_SPIN_LIMIT) __trap();
        if (idx < vf[FIX_RESERVED]) break;
        if (vf[FIX_DONE] == n_tiles) {
          __threadfence();
          if (idx >= vf[FIX_RESERVED]) quit = 1;
          break;
        }
        __nanosleep(500);
      }
      int32_t v = 0;
      if (!quit) {
        for (uint32_t spin = 0; (v = vf[FIX_SLOTS + idx]) == 0; spin++) {
          if (spin > QUEUE_SPIN_LIMIT) __trap();
          __nanosleep(100);
        }
        vf[FIX_SLOTS + idx] = 0;
      }
      s_quit = quit;
      s_claim = v;
      s_T = 1.0;
      s_last = -1;
      s_done = 0;
    }
    __syncthreads();
    if (s_quit) break;
    const int64_t p = (int64_t)s_claim - 1;
    const int px = (int)(p % width), py = (int)(p / width);
    const int tile = (py / BLEND_TILE) * tiles_x + px / BLEND_TILE;
    const bool mesh_here = mesh.color != nullptr && mesh.triangle_id[p] >= 0;
    const double limit = mesh_here ? mesh.depth[p] : __longlong_as_double(0x7ff0000000000000LL);
    const double fx = px + 0.5, fy = py + 0.5;
    const int64_t s = tile_starts[tile];
    uint4 pg = make_uint4(0u, 0u, 0u, 0u);
    if (crow) pg = __ldcg(prog + tile);
    const int64_t e = crow ? s + (int64_t)pg.x : tile_starts[tile + 1];  // (blend-only: the written prefix)
    double pr = 0.0, pgc = 0.0, pb = 0.0, pd = 0.0;  // this warp's per-lane partial sums
    // prefetch: my first round's records and the next round's indices
    auto idx = [&](int64_t rb, int u) -> uint32_t {
      const int64_t k = rb + EW * lane + u;
      return k < e ? __ldcg(entries + k) : 0u;
    };
    BlendRec c[EW], cn[EW];
    uint32_t ixn[EW];
    {
      const int64_t b0 = s + (int64_t)warp * RW;
#pragma unroll
      for (int u = 0; u < EW; u++) {
        const uint32_t i0 = idx(b0, u);
        if (b0 + EW * lane + u < e) cn[u] = rec[i0];
        ixn[u] = idx(b0 + EXW * RW, u);
      }
    }
    for (int64_t sb = s; sb < e; sb += (int64_t)EXW * RW) {
      if (s_done) break;  // (uniform: read after the last barrier)
      const int64_t base = sb + (int64_t)warp * RW;
#pragma unroll
      for (int u = 0; u < EW; u++) {
        c[u] = cn[u];
        if (base + EXW * RW + EW * lane + u < e) cn[u] = rec[ixn[u]];
        ixn[u] = idx(base + 2 * EXW * RW, u);
      }
      // phase A (all warps): evaluate this warp's round
      double sig[EW];
      bool use[EW];
      int us = EW;
#pragma unroll
      for (int u = 0; u < EW; u++) {
        const int64_t k = base + EW * lane + u;
        use[u] = false;
        sig[u] = 0.0;
        if (k < e) {
          if (c[u].depth >= limit && us == EW) us = u;
          const double dx = fx - c[u].mx, dy = fy - c[u].my;
          const double m = c[u].ca * dx * dx + c[u].cb2 * dx * dy + c[u].cc * dy * dy;
          if (!(m > SUPPORT_MAHAL2 || m < 0.0)) {
            double sg = c[u].alpha * exp(-0.5 * m);
            if (sg > ALPHA_CLAMP) sg = ALPHA_CLAMP;
            use[u] = !(sg < SIGMA_SKIP);
            sig[u] = sg;
          }
        }
      }
      const unsigned smask = __ballot_sync(0xffffffffu, us < EW);
      const int ls = smask ? __ffs(smask) - 1 : 32;
      const int lsu = __shfl_sync(0xffffffffu, us, ls & 31);
#pragma unroll
      for (int u = 0; u < EW; u++)
        if (lane > ls || (lane == ls && u >= lsu)) use[u] = false;
      double f[EW];
      double q = 1.0;
#pragma unroll
      for (int u = 0; u < EW; u++) {
        f[u] = use[u] ? 1.0 - sig[u] : 1.0;
        q *= f[u];
      }
      double P = q;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, P, d);
        if (lane >= d) P *= t;
      }
      double Pex = __shfl_up_sync(0xffffffffu, P, 1);
      if (lane == 0) Pex = 1.0;
      // phase B: commit the rounds in order (exact_walk2's arithmetic with the
      // T the previous round left)
      for (int w = 0; w < EXW; w++) {
        if (warp == w && !s_done && base < e) {
          double T = s_T;
          int64_t last = s_last;
          bool done = false;
          double ta[EW];
          double run = T * Pex;
          bool near = false;
#pragma unroll
          for (int u = 0; u < EW; u++) {
            run *= f[u];
            ta[u] = run;
            near = near || (use[u] && fabs(run - EARLY_STOP_T) <= 1e-12 * EARLY_STOP_T);
          }
          if (!__any_sync(0xffffffffu, near)) {
            int ue = EW;
#pragma unroll
            for (int u = 0; u < EW; u++)
              if (use[u] && ta[u] < EARLY_STOP_T && ue == EW) ue = u;
            const unsigned emask = __ballot_sync(0xffffffffu, ue < EW);
            const int le = emask ? __ffs(emask) - 1 : 32;
            const int leu = __shfl_sync(0xffffffffu, ue, le & 31);
            int lastu = -1;
            double tb = T * Pex, tl = 0.0;
#pragma unroll
            for (int u = 0; u < EW; u++) {
              const bool valid = use[u] && (lane < le || (lane == le && u < leu));
              if (valid) {
                const double wv = sig[u] * tb;
                pr += c[u].r * wv;
                pgc += c[u].g * wv;
                pb += c[u].b * wv;
                pd += c[u].depth * wv;
                lastu = u;
                tl = ta[u];
              }
              tb = ta[u];
            }
            const unsigned vmask = __ballot_sync(0xffffffffu, lastu >= 0);
            if (vmask) {
              const int lv = 31 - __clz(vmask);
              T = __shfl_sync(0xffffffffu, tl, lv);
              last = base + (int64_t)EW * lv + __shfl_sync(0xffffffffu, lastu, lv);
            }
            if (le < 32) done = true;
          } else {
            bool stop = false;
            for (int i = 0; i < 32 && !stop; i++) {
#pragma unroll
              for (int u = 0; u < EW; u++) {
                const bool ui = __shfl_sync(0xffffffffu, use[u], i);
                if (!ui || stop) continue;
                const double sg = __shfl_sync(0xffffffffu, sig[u], i);
                const double test_t = T * (1.0 - sg);
                if (test_t < EARLY_STOP_T) {
                  stop = true;
                  continue;
                }
                if (lane == i) {
                  const double wv = sg * T;
                  pr += c[u].r * wv;
                  pgc += c[u].g * wv;
                  pb += c[u].b * wv;
                  pd += c[u].depth * wv;
                }
                T = test_t;
                last = base + (int64_t)EW * i + u;
              }
            }
            if (stop) done = true;
          }
          if (ls < 32) done = true;
          if (lane == 0) {
            s_T = T;
            s_last = last;
            s_done = done ? 1 : 0;
          }
        }
        __syncthreads();
      }
    }
    // blend-only bins: the walk goes on past the written prefix (warp 0)
    if (crow && !s_done && warp == 0) {
      const int txx = px / BLEND_TILE, tyy = py / BLEND_TILE;
      const int sup = (tyy >> css) * sx_super + (txx >> css);
      WalkState ws{s_T, pr, pgc, pb, pd, s_last, false};
      exact_walk_coarse_run(rec, crow, crect, pg.y, (int)pg.z, (int)pg.x, cstart[sup + 1], txx, tyy, s, fx, fy, limit,
                            lane, ws);
      pr = ws.pr, pgc = ws.pg, pb = ws.pb, pd = ws.pd;
      if (lane == 0) {
        s_T = ws.T;
        s_last = ws.last;
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      pr += __shfl_xor_sync(0xffffffffu, pr, d);
      pgc += __shfl_xor_sync(0xffffffffu, pgc, d);
      pb += __shfl_xor_sync(0xffffffffu, pb, d);
      pd += __shfl_xor_sync(0xffffffffu, pd, d);
    }
    if (lane == 0) {
      s_sum[warp][0] = pr;
      s_sum[warp][1] = pgc;
      s_sum[warp][2] = pb;
      s_sum[warp][3] = pd;
    }
    __syncthreads();
    if (tid == 0) {
      double r = 0.0, g = 0.0, b = 0.0, dd = 0.0;
      for (int w = 0; w < EXW; w++) r += s_sum[w][0], g += s_sum[w][1], b += s_sum[w][2], dd += s_sum[w][3];
      const double T = s_T;
      write_pixel(out, mesh, mesh_here, p, T, r, g, b, dd, 1.0 - T, s_last, bg0, bg1, bg2, mask_variant, mask_k, T);
    }
    __syncthreads();
  }
}

}  // namespace hgs

// Is f one of the blend kernels that consume the fine binning's ready queue?
bool hgs_is_blend_tile_fn(const void* f) {
  using namespace hgs;
  return f == (const void*)blend_tile_kernel<false, false> || f == (const void*)blend_tile_kernel<true, false> ||
         f == (const void*)blend_tile_kernel<false, true> || f == (const void*)blend_tile_kernel<true, true>;
}

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
#ifndef HGS_FWD_EXACT
#define HGS_FWD_EXACT 0
#endif
#ifndef HGS_BLEND_V1
#define HGS_BLEND_V1 0
#endif
#ifndef HGS_BLEND_QUEUE
#define HGS_BLEND_QUEUE 1
#endif
  if (out->fixup && proj->cull && !HGS_FWD_EXACT) {
#if HGS_BLEND_V1
    zero_pdl(st, out->fixup, sizeof(int32_t));
    HGS_CHECK_LAUNCH();
#endif
    const size_t smem = sizeof(FastSmem);
    static bool attr = false;
    if (!attr) {
      for (auto fn : {blend_fast_kernel<false, false>, blend_fast_kernel<true, false>, blend_fast_kernel<false, true>,
                      blend_fast_kernel<true, true>}) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      }
      attr = true;
    }
    const bool prec = out->final_t != nullptr;
#if HGS_BLEND_V1
    auto fn = out->stats ? (prec ? blend_fast_kernel<true, true> : blend_fast_kernel<true, false>)
                         : (prec ? blend_fast_kernel<false, true> : blend_fast_kernel<false, false>);
    launch_pdl(fn, dim3(n_tiles), dim3(FAST_THREADS), smem, st, (const BlendRec*)proj->rec,
               (const CullRec*)proj->cull, tiles->entries, tiles->tile_starts, tiles->tiles_x, width, height, ml,
               bg_host3[0], bg_host3[1], bg_host3[2], mask_variant, mask_k, *out, out->fixup, tiles->counters);
#else
    (void)smem;
    const size_t tsmem = out->final_t != nullptr ? sizeof(TileSmem<true>) : sizeof(TileSmem<false>);
    static bool tattr = false;
    if (!tattr) {
      for (auto fn : {blend_tile_kernel<false, false>, blend_tile_kernel<true, false>}) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TileSmem<false>));
        cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      }
      for (auto fn : {blend_tile_kernel<false, true>, blend_tile_kernel<true, true>}) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TileSmem<true>));
        cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      }
      tattr = true;
    }
    auto fn = out->stats ? (prec ? blend_tile_kernel<true, true> : blend_tile_kernel<true, false>)
                         : (prec ? blend_tile_kernel<false, true> : blend_tile_kernel<false, false>);
    // binned tile grids: claim tiles from the fine binning's ready queue (at
    // the scratch base, common.cuh), starting while the last quads are binned
    const int ss = super_shift(tiles->tiles_x, tiles->tiles_y, (tiles->flags & HGS_TILES_BLEND_ONLY) != 0);
    // blend-only bins (hgs.h): the blend filters the coarse lists itself and
    // starts behind the coarse scatter (there is no fine binning to queue on)
    const bool coarse = ss >= 0 && (tiles->flags & HGS_TILES_BLEND_ONLY) && tiles->coarse_rows && tiles->coarse_prog &&
                        !prec;
    if ((tiles->flags & HGS_TILES_BLEND_ONLY) && !coarse)
      return hgs_set_error(HGS_ERR_INVALID, "hgs_blend_forward: blend-only bins need a binned tile grid and no final_t");
    const bool queued = !coarse && ss >= 0 && HGS_BLEND_QUEUE && tiles->ready != nullptr;
    int* ready = queued ? reinterpret_cast<int*>(tiles->ready) : nullptr;
    const int qs = queued ? ss - 2 : 0;
    const int sxs = (queued || coarse) ? (tiles->tiles_x + (1 << ss) - 1) >> ss : 0;
    const int sys = queued ? (tiles->tiles_y + (1 << ss) - 1) >> ss : 0;
    const int n_cta = queued ? (sxs * sys << (2 * qs)) * 16 : n_tiles;
    const uint32_t* crow = coarse ? (const uint32_t*)tiles->coarse_rows : nullptr;
    const uint2* crect = coarse ? (const uint2*)tiles->coarse_rects : nullptr;
    const uint32_t* cstart = coarse ? (const uint32_t*)tiles->coarse_starts : nullptr;
    launch_pdl(fn, dim3(n_cta), dim3(TB_THREADS), tsmem, st, (const BlendRec*)proj->rec, (const CullRec*)proj->cull,
               (const uint32_t*)tiles->entries, (const int64_t*)tiles->tile_starts, tiles->tiles_x, width, height, ml,
               bg_host3[0], bg_host3[1], bg_host3[2], mask_variant, mask_k, *out, out->fixup,
               (const int64_t*)tiles->counters, ready, qs, sxs, crow, crect, cstart, coarse ? ss : 0,
               coarse ? (uint4*)tiles->coarse_prog : (uint4*)nullptr);
#endif
    HGS_CHECK_LAUNCH();
#if HGS_BLEND_V1
    // exact fix-up: one warp per flagged pixel (persistent grid over the device-side work list)
    launch_pdl(blend_exact_kernel, dim3(2 * NUM_SMS), dim3(256), 0, st, (const BlendRec*)proj->rec, tiles->entries,
                                                    tiles->tile_starts, tiles->tiles_x, width, height, ml,
                                                    bg_host3[0], bg_host3[1], bg_host3[2], mask_variant,
                                                    mask_k, *out, out->fixup, tiles->counters);
#else
    // exact fix-up: queue consumer beside the blend (one warp per flagged pixel)
    // small CTAs (2 warps, ~11k registers): they fit beside the blend's
    // resident CTAs as soon as its last wave starts retiring
#ifndef HGS_EXACT_CTA
#define HGS_EXACT_CTA 1
#endif
    launch_pdl(HGS_EXACT_CTA ? blend_exact_cta_kernel : blend_exact_queue_kernel,
               dim3(HGS_EXACT_CTA ? HGS_EX_CTAS_PER_SM * NUM_SMS : 8 * NUM_SMS), dim3(HGS_EXACT_CTA ? EXW * 32 : 64), 0, st,
               (const BlendRec*)proj->rec,
               (const uint32_t*)tiles->entries, (const int64_t*)tiles->tile_starts, tiles->tiles_x, n_cta, width, ml,
               bg_host3[0], bg_host3[1], bg_host3[2], mask_variant, mask_k, *out, out->fixup,
               (const int64_t*)tiles->counters, ready, crow, crect, cstart, coarse ? ss : 0, sxs,
               coarse ? (const uint4*)tiles->coarse_prog : (const uint4*)nullptr);
#endif
    HGS_CHECK_LAUNCH();
  } else {
    launch_pdl(blend_exact_kernel, dim3(ceil_div(npix * 32, 256)), dim3(256), 0, st, (const BlendRec*)proj->rec, tiles->entries,
                                                            tiles->tile_starts, tiles->tiles_x, width, height, ml,
                                                            bg_host3[0], bg_host3[1], bg_host3[2], mask_variant,
                                                            mask_k, *out, nullptr, tiles->counters);
    HGS_CHECK_LAUNCH();
  }
  return HGS_OK;
}

namespace hgs {

// Median-style depth (depth_kernel, splat/kernels.py:163-202): the camera z
// of the entry at which the accumulated opacity 1 - T first exceeds 0.5,
// NaN where it never does.  One warp per pixel, fp64 throughout: lanes
// evaluate 32 consecutive entries exactly as the reference (support test,
// exp, clamp, skip), the chunk's transmittance is an inclusive shuffle
// prefix product of (1 - sigma) (|rel. diff| < 1e-13 from the serial
// product, see exact_walk2), and a chunk whose products fall within 1e-12 of
// either threshold (0.5, or the 1e-4 early stop) is replayed serially in the
// reference's order, so every decision is the reference's.
__global__ void __launch_bounds__(256) depth_walk_kernel(const BlendRec* __restrict__ rec,
                                                         const uint32_t* __restrict__ entries,
                                                         const int64_t* __restrict__ tile_starts, int tiles_x,
                                                         int width, int height, double* __restrict__ out,
                                                         const int64_t* __restrict__ counters) {
  if (counters && counters[2]) return;  // overflowed bins
  const int lane = threadIdx.x & 31;
  const int64_t npix = (int64_t)width * height;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < npix; p += nwarps) {
    const int px = (int)(p % width), py = (int)(p / width);
    const int tile = (py / BLEND_TILE) * tiles_x + px / BLEND_TILE;
    const int64_t s = tile_starts[tile], e = tile_starts[tile + 1];
    const double fx = px + 0.5, fy = py + 0.5;
    double T = 1.0;
    double found = __longlong_as_double(0x7ff8000000000000LL);
    bool done = false;
    for (int64_t base = s; base < e && !done; base += 32) {
      const int64_t k = base + lane;
      bool use = false;
      double sig = 0.0, dep = 0.0;
      if (k < e) {
        const BlendRec c = rec[__ldg(entries + k)];
        dep = c.depth;
        const double dx = fx - c.mx, dy = fy - c.my;
        const double m = c.ca * dx * dx + c.cb2 * dx * dy + c.cc * dy * dy;
        if (!(m > SUPPORT_MAHAL2 || m < 0.0)) {
          sig = c.alpha * exp(-0.5 * m);
          if (sig > ALPHA_CLAMP) sig = ALPHA_CLAMP;
          use = !(sig < SIGMA_SKIP);
        }
      }
      double P = use ? 1.0 - sig : 1.0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, P, d);
        if (lane >= d) P *= t;
      }
      const double t_after = T * P;
      const bool near = use && (fabs(t_after - EARLY_STOP_T) <= 1e-12 * EARLY_STOP_T || fabs(t_after - 0.5) <= 1e-12);
      if (!__any_sync(0xffffffffu, near)) {
        // the reference tests the early stop before the opacity crossing
        const unsigned stop = __ballot_sync(0xffffffffu, use && t_after < EARLY_STOP_T);
        const unsigned hit = __ballot_sync(0xffffffffu, use && !(t_after < EARLY_STOP_T) && 1.0 - t_after > 0.5);
        const int ks = stop ? __ffs(stop) - 1 : 32, kh = hit ? __ffs(hit) - 1 : 32;
        if (kh < ks) {
          found = __shfl_sync(0xffffffffu, dep, kh);
          done = true;
        } else if (ks < 32) {
          done = true;
        } else {
          T = __shfl_sync(0xffffffffu, t_after, 31);
        }
      } else {
        unsigned use_mask = __ballot_sync(0xffffffffu, use);
        while (use_mask) {
          const int i = __ffs(use_mask) - 1;
          use_mask &= use_mask - 1;
          const double sg = __shfl_sync(0xffffffffu, sig, i);
          const double test_t = T * (1.0 - sg);
          if (test_t < EARLY_STOP_T) { done = true; break; }
          T = test_t;
          if (1.0 - T > 0.5) {
            found = __shfl_sync(0xffffffffu, dep, i);
            done = true;
            break;
          }
        }
      }
    }
    if (lane == 0) out[p] = found;
  }
}

}  // namespace hgs

extern "C" int hgs_render_depth(const hgs_projected* proj, const hgs_tiles* tiles, int32_t width, int32_t height,
                                double* out_depth, void* stream) {
  using namespace hgs;
  if (!proj || !tiles || !out_depth) return hgs_set_error(HGS_ERR_INVALID, "hgs_render_depth: null argument");
  if (tiles->tile_px != BLEND_TILE)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_render_depth: only tile_px == 16 is implemented");
  if (width <= 0 || height <= 0) return hgs_set_error(HGS_ERR_INVALID, "hgs_render_depth: empty image");
  if (tiles->tiles_x != (width + 15) / 16 || tiles->tiles_y != (height + 15) / 16)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_render_depth: tile grid does not match image size");
  const int64_t npix = (int64_t)width * height;
  const int64_t blocks = std::min<int64_t>(ceil_div(npix * 32, 256), 16 * NUM_SMS);
  depth_walk_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>((const BlendRec*)proj->rec, tiles->entries,
                                                                  tiles->tile_starts, tiles->tiles_x, width, height,
                                                                  out_depth, tiles->counters);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}
