// K5 blend backward: backward_kernel (gsmesh/splat/kernels.py:77-160) with the
// per-Gaussian reduction of render.py:155-157, and K6 project backward:
// _chain_to_parameters (splat/render.py:185-313) + densify statistic and
// visibility (render.py:171-178).
//
// K5: one CTA per 16x16 tile, warp-specialised like the forward: 4 consumer
// warps own 8x8 sub-tiles (two pixels per lane), 1 producer warp streams the
// tile's entries NEWEST FIRST (from the largest `last` of the tile down to
// the first entry) through a 3-stage x 64-entry cp.async/mbarrier ring
// (5 CTAs per SM).  Each pixel walks back from its last blended entry
// (kernels.py:120): T before an entry is reconstructed from T after it (one
// reciprocal of 1 - sigma), starting from the forward's fp64 final T; the
// suffix colours enter only through one scalar Q (see BwPix).  Per-warp
// ellipse cull as in the forward.  The per-entry 9-vector (mean2d 2, cov 3
// full-matrix convention, alpha, rgb 3) is reduced over the warp
// (reduce-scatter) and added to the per-Gaussian fp64 accumulator with one
// atomic per component per warp.
//
// Numerics: the per-entry decisions (support m <= 9, skip sigma < 1/255,
// clamp at 0.99) are the reference's: the fp64 conic form, narrowed to the
// fp32 exp2 argument u, is compared with the entry's two cuts (blend:
// min(9U, log2(255 alpha)); clamp: log2(alpha / 0.99)), computed once per
// (warp, entry) by the cull, and inside a guard band around either cut the
// entry is re-evaluated exactly in fp64.  The gradient arithmetic runs in fp64 (sigma from the
// fp64 exp2, T / Q recurrence, s_i, mean2d and cov products; alpha and colour
// products in fp32): the reverse recurrence compounds every error of sigma
// and T over the walk, and the centre gradients (|g| ~ 4e2 at c3) must hold
// 1e-4 absolute -- fp32 arithmetic left 2.6e-4, this design 3.9e-5
// (tools/diag_bw_variants.py).
#include "stage.cuh"

namespace hgs {

#ifndef HGS_BW_BATCH
#define HGS_BW_BATCH 64
#endif
#ifndef HGS_BW_NSTAGE
#define HGS_BW_NSTAGE 3
#endif
#ifndef HGS_BW_MINB
#define HGS_BW_MINB 5  // fp64 walk state: 5 CTAs (81 regs) 170.6 vs 4 CTAs 174.6 ms per c4 step
#endif
constexpr int BW_BATCH = HGS_BW_BATCH;
constexpr int BW_NSTAGE = HGS_BW_NSTAGE;
#ifndef HGS_BW_NPX
#define HGS_BW_NPX 2
#endif
constexpr int BW_NPX = HGS_BW_NPX;          // pixels per lane
constexpr int BW_CONSUMERS = 8 / BW_NPX;    // 8-wide sub-tiles of 4 * BW_NPX rows
constexpr int BW_SUBH = 4 * BW_NPX;
constexpr int BW_THREADS = (BW_CONSUMERS + 1) * 32;
constexpr float CLAMP_BAND_INV = 1.0f / (2.0f * EPS_SIG * CLAMP_F);

struct BwSmem {
  StageEntry ent[BW_NSTAGE][BW_BATCH];
  uint32_t gid[BW_NSTAGE][BW_BATCH];
  unsigned long long full[BW_NSTAGE];
  unsigned long long empty[BW_NSTAGE];
  int4 list[BW_CONSUMERS][BW_BATCH];  // (slot index, blend cut, clamp cut, -) of the entries touching the sub-tile
  double exp2tab[EXP2_N];
  int max_last;
};

// Sum 9 per-lane values over the warp (reduce-scatter, 12 shuffles): lane L
// ends with the total of value index reduce9_index(L) (-1: none).
template <typename R>
__device__ __forceinline__ R warp_reduce9(R v[9], int lane) {
  // offset 16: lower lanes keep 0..4, upper keep 5..8
  const bool u16 = lane & 16;
#pragma unroll
  for (int i = 0; i < 5; i++) {
    const R hi = i < 4 ? v[5 + i] : (R)0;
    const R send = u16 ? v[i] : hi;
    const R recv = __shfl_xor_sync(0xffffffffu, send, 16);
    v[i] = (u16 ? hi : v[i]) + recv;
  }
  // now 5 values (upper lanes: 4 + a zero); offset 8: keep 0..2 / 3..4
  const bool u8 = lane & 8;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    const R hi = i < 2 ? v[3 + i] : (R)0;
    const R send = u8 ? v[i] : hi;
    const R recv = __shfl_xor_sync(0xffffffffu, send, 8);
    v[i] = (u8 ? hi : v[i]) + recv;
  }
  // 3 values; offset 4: keep 0..1 / 2
  const bool u4 = lane & 4;
#pragma unroll
  for (int i = 0; i < 2; i++) {
    const R hi = i < 1 ? v[2] : (R)0;
    const R send = u4 ? v[i] : hi;
    const R recv = __shfl_xor_sync(0xffffffffu, send, 4);
    v[i] = (u4 ? hi : v[i]) + recv;
  }
  // 2 values; offset 2: keep 0 / 1
  {
    const bool u2 = lane & 2;
    const R send = u2 ? v[0] : v[1];
    const R recv = __shfl_xor_sync(0xffffffffu, send, 2);
    v[0] = (u2 ? v[1] : v[0]) + recv;
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  return v[0];
}
__device__ __forceinline__ int reduce9_index(int lane) {
  // level 16: base 0 or 5; level 8: +0 or +3; level 4: +0 or +2; level 2: +0 or +1
  const int b16 = (lane & 16) ? 5 : 0, b8 = (lane & 8) ? 3 : 0, b4 = (lane & 4) ? 2 : 0, b2 = (lane & 2) ? 1 : 0;
  // the kept ranges shrink to [0,5)/[5,9), [0,3)/[3,5) ..., so an index past a range end is empty
  const int n16 = (lane & 16) ? 4 : 5;
  const int n8 = (lane & 8) ? n16 - 3 : (n16 < 3 ? n16 : 3);
  const int n4 = (lane & 4) ? n8 - 2 : (n8 < 2 ? n8 : 2);
  const int n2 = (lane & 2) ? n4 - 1 : (n4 < 1 ? n4 : 1);
  return (n2 > 0 && (lane & 1) == 0) ? b16 + b8 + b4 + b2 : -1;  // lanes 2k, 2k+1 hold the same total
}

// Clamp cut of an entry: sigma = alpha 2^-u is clamped at 0.99 iff
// u < log2(alpha / 0.99) (lg2.approx, as entry_ucut; NaN for an
// ill-conditioned conic: always decided exactly).
__device__ __forceinline__ float entry_uclamp(float a32) {
  if (a32 < 0.0f) return __int_as_float(0x7fc00000);
  float l;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(a32 * (float)(1.0 / ALPHA_CLAMP)));
  return l;
}

struct BwExact {
  double sig, gauss;
  bool clamped;
};
// Exact per-entry evaluation in the reference's operation order
// (kernels.py:126-133): sigma (or -1: no contribution), the Gaussian value
// and whether sigma was clamped.
__device__ __noinline__ BwExact bw_exact_entry(const StageEntry& E, double fx, double fy) {
  BwExact r{-1.0, 0.0, false};
  const double dx = fx - E.a.x, dy = fy - E.a.y;
  const double m = E.b.x * dx * dx + E.b.y * dx * dy + E.c.x * dy * dy;
  if (m > SUPPORT_MAHAL2 || m < 0.0) return r;
  const double g = exp(-0.5 * m);
  double sg = E.d.x * g;
  r.clamped = sg > ALPHA_CLAMP;
  if (r.clamped) sg = ALPHA_CLAMP;
  if (sg < SIGMA_SKIP) return r;
  r.gauss = g;
  r.sig = sg;
  return r;
}

// Per-pixel reverse-walk state.  The three suffix colours acc_c of
// kernels.py:111-160 only ever enter the gradient through
// Q = sum_c g_c acc_c + g_T T_final (s_i = (g.c_i T_after - Q) / (1 - sigma)
// and Q += (g.c_i) w_i), so the walk carries that one scalar.  fp64: T after
// the current entry and Q (T before an entry is T after it / (1 - sigma), an
// error in either compounds over the walk, and s_i is a difference of nearly
// equal terms); the upstream gradients are given in fp32.
#ifndef HGS_BW_V64
#define HGS_BW_V64 5  // leading 9-vector components accumulated in fp64 (mean2d 2, cov 3)
#endif
struct BwPix {
  int last;
  float gr, gg, gb;
  double t_after, q;
};

__device__ __forceinline__ void bw_pixel_init(BwPix& q, bool inside, int64_t p, int64_t s, const hgs_mesh_layer& mesh,
                                              double bg0, double bg1, double bg2, const double* __restrict__ final_t,
                                              const int32_t* __restrict__ last_idx,
                                              const float* __restrict__ grad_color, const float* __restrict__ grad_t,
                                              float* __restrict__ mesh_grad, int accumulate_mesh) {
  q.last = -1;
  q.gr = q.gg = q.gb = 0.f;
  q.t_after = 1.0;
  q.q = 0.0;
  if (!inside) return;
  q.last = last_idx[p];
  q.gr = grad_color[3 * p];
  q.gg = grad_color[3 * p + 1];
  q.gb = grad_color[3 * p + 2];
  const double gtp = grad_t ? (double)grad_t[p] : 0.0;
  const double t_fin = final_t[p];
  const bool mesh_here = mesh.color != nullptr && mesh.triangle_id[p] >= 0;
  if (mesh_grad) {  // d pixel / d mesh colour = T * valid (render.py:180-181)
    const float f = mesh_here ? (float)t_fin : 0.f;
    float* mg = mesh_grad + 3 * p;
    if (accumulate_mesh) {
      mg[0] += q.gr * f; mg[1] += q.gg * f; mg[2] += q.gb * f;
    } else {
      mg[0] = q.gr * f; mg[1] = q.gg * f; mg[2] = q.gb * f;
    }
  }
  // suffix colour starts at T_final * (mesh colour or background) (kernels.py:111-119)
  double c0 = bg0, c1 = bg1, c2 = bg2;
  if (mesh_here) {
    c0 = mesh.color[3 * p];
    c1 = mesh.color[3 * p + 1];
    c2 = mesh.color[3 * p + 2];
  }
  q.t_after = t_fin;
  q.q = t_fin * (((double)q.gr * c0 + (double)q.gg * c1) + (double)q.gb * c2 + gtp);
  if (q.last >= 0) q.last -= (int)s;  // relative to the tile start
}

// One reverse step of kernels.py:120-160 for one pixel and entry E (relative
// index rel): the reference's decisions (fp32 fast test + exact fp64
// re-evaluation inside the guard bands), then the gradient arithmetic --
// sigma from the fp64 exp2 (stage.cuh), the T / Q recurrence and s_i in
// fp64, the 9-vector products in fp64 for the first HGS_BW_V64 components
// (mean2d, cov: they reach the centre gradients through the focal / depth
// chain) and fp32 for the rest (alpha, colour).
__device__ __forceinline__ void bw_pixel_step(BwPix& q, const StageEntry& E, int rel, double fx, double fy,
                                              float ucut, float uclamp, const double* __restrict__ tab, double vd[5],
                                              float vf[4]) {
  const bool act = q.last >= 0 && rel <= q.last;
  if (!act) return;  // entry after this pixel's last blended one
  const double dx = fx - E.a.x, dy = fy - E.a.y;
  const double m = fma(dx, fma(E.b.y, dy, E.b.x * dx), (E.c.x * dy) * dy);
  const double u = m * U_SCALE;
  const float uu = __double2float_rn(u);
  // the blend and clamp decisions against the entry's cuts (stage.cuh
  // entry_ucut; NaN cut: always exact)
  const float dd = uu - ucut, dc = uu - uclamp;
  bool ok = dd < -U_BAND;
  bool clamped = dc < -U_BAND;
  double sg, gauss;
  if (!(fabsf(dd) > U_BAND) || !(fabsf(dc) > U_BAND)) {  // rare: decide (and evaluate) in the reference's order
    const BwExact x = bw_exact_entry(E, fx, fy);
    ok = x.sig >= 0.0;
    sg = x.sig;
    gauss = x.gauss;
    clamped = x.clamped;
  } else {
    if (!ok) return;
    gauss = exp2_neg64(u, uu, tab);
    sg = clamped ? ALPHA_CLAMP : E.d.x * gauss;
  }
  if (!ok) return;
  // g . c_i (the colour enters s_i only through it); colour r from the fp64
  // record, g / b from the fp32 record
  const double gc = fma((double)q.gr, E.d.y, fma((double)q.gg, (double)E.f.col.z, (double)q.gb * E.f.col.w));
  // one reciprocal for the divisions of kernels.py:135,142-146
  const double inv = rcp64(1.0 - sg);
  const double t_before = q.t_after * inv;
  const double w = sg * t_before;
  const double s_i = fma(gc, t_before, -q.q * inv);
  q.q = fma(gc, w, q.q);
  q.t_after = t_before;
  const float w32 = (float)w;
  vf[1] = fmaf(q.gr, w32, vf[1]);
  vf[2] = fmaf(q.gg, w32, vf[2]);
  vf[3] = fmaf(q.gb, w32, vf[3]);
  if (!clamped) {
    const double cx = E.b.x, cy = 0.5 * E.b.y, cz = E.c.x;  // conic xx, xy, yy
    const double qd_x = fma(cx, dx, cy * dy);
    const double qd_y = fma(cy, dx, cz * dy);
    const double common = s_i * sg;
    vd[0] = fma(common, qd_x, vd[0]);
    vd[1] = fma(common, qd_y, vd[1]);
#if HGS_BW_V64 >= 5
    const double hc = 0.5 * common;
    vd[2] = fma(hc * qd_x, qd_x, vd[2]);
    vd[3] = fma(hc * qd_x, qd_y, vd[3]);
    vd[4] = fma(hc * qd_y, qd_y, vd[4]);
#else
    const float hc = 0.5f * (float)common, qx = (float)qd_x, qy = (float)qd_y;
    vd[2] = (double)fmaf(hc * qx, qx, (float)vd[2]);
    vd[3] = (double)fmaf(hc * qx, qy, (float)vd[3]);
    vd[4] = (double)fmaf(hc * qy, qy, (float)vd[4]);
#endif
    vf[0] = fmaf((float)s_i, (float)gauss, vf[0]);
  }
}

__global__ void __launch_bounds__(BW_THREADS, HGS_BW_MINB) blend_backward_kernel(
    const BlendRec* __restrict__ rec, const CullRec* __restrict__ cull, const uint32_t* __restrict__ entries,
    const int64_t* __restrict__ tile_starts, int tiles_x, int width, int height, hgs_mesh_layer mesh, double bg0,
    double bg1, double bg2, const double* __restrict__ final_t, const int32_t* __restrict__ last_idx,
    const float* __restrict__ grad_color, const float* __restrict__ grad_t, double* __restrict__ screen,
    float* __restrict__ mesh_grad, int accumulate_mesh, const int64_t* __restrict__ counters) {
  if (counters && counters[2]) return;  // overflowed bins: no valid forward to differentiate
  extern __shared__ __align__(128) unsigned char bw_smem_raw[];
  BwSmem& sm = *reinterpret_cast<BwSmem*>(bw_smem_raw);
  const int tile = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int64_t s = tile_starts[tile];
  if (threadIdx.x == 0) {
    for (int i = 0; i < BW_NSTAGE; i++) {
      mbar_init(&sm.full[i], 32);
      mbar_init(&sm.empty[i], BW_CONSUMERS);
    }
    sm.max_last = -1;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  exp2_tab_load(sm.exp2tab);
  __syncthreads();
  // consumer pixels: warp w owns the 8 x BW_SUBH sub-tile (w & 1, w >> 1);
  // lane (x, y) = (lane & 7, lane >> 3) holds pixels (x, y + 4 k), k < BW_NPX
  const int sx0 = (warp & 1) * 8, sy0 = (warp >> 1) * BW_SUBH;
  const int px = tx * 16 + sx0 + (lane & 7);
  const int py0 = ty * 16 + sy0 + (lane >> 3);
  const bool cons = warp < BW_CONSUMERS;
  BwPix q[BW_NPX];
  int ml = -1;
#pragma unroll
  for (int k = 0; k < BW_NPX; k++) {
    const int py = py0 + 4 * k;
    bw_pixel_init(q[k], cons && px < width && py < height, (int64_t)py * width + px, s, mesh, bg0, bg1, bg2, final_t,
                  last_idx, grad_color, grad_t, mesh_grad, accumulate_mesh);
    ml = max(ml, q[k].last);
  }
  if (ml >= 0) atomicMax(&sm.max_last, ml);
  __syncthreads();
  const int top = sm.max_last;  // newest entry any pixel of the tile used
  const int nbatches = (top + BW_BATCH) / BW_BATCH;

  if (!cons) {
    // ------------------------------------------------------------ producer
    for (int b = 0; b < nbatches; b++) {
      const int slot = b % BW_NSTAGE;
      if (b >= BW_NSTAGE) warp_wait(&sm.empty[slot], ((b / BW_NSTAGE) - 1) & 1, lane);
      const int hi = top - b * BW_BATCH;  // slot i holds entry lo + i
      const int lo = hi - BW_BATCH + 1 > 0 ? hi - BW_BATCH + 1 : 0;
      for (int i = lane; i < BW_BATCH; i += 32) {
        StageEntry* dst = &sm.ent[slot][i];
        if (lo + i <= hi) {
          const uint32_t g = __ldg(entries + s + lo + i);
          const char* src = reinterpret_cast<const char*>(rec + g);
          const char* cs = reinterpret_cast<const char*>(cull + g);
          cp_async16(&dst->a, src);
          cp_async16(&dst->b, src + 16);
          cp_async16(&dst->c, src + 32);
          cp_async16(&dst->d, src + 48);
          cp_async16(&dst->f.box, cs);
          cp_async16(&dst->f.con, cs + 16);
          cp_async16(&dst->f.col, cs + 32);
          cp_async4(&sm.gid[slot][i], entries + s + lo + i);
        } else {
          cp_async16(&dst->f.box, &g_empty_box);
        }
      }
      cp_async_arrive_noinc(&sm.full[slot]);
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const double fx = px + 0.5, fy0 = py0 + 0.5;
  const float wx0 = tx * 16 + sx0 + 0.5f, wx1 = wx0 + 7.0f;
  const float wy0 = ty * 16 + sy0 + 0.5f, wy1 = wy0 + (float)(BW_SUBH - 1);
  const int vidx = reduce9_index(lane);
  int wlast = ml;  // newest entry any pixel of this warp used
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wlast = max(wlast, __shfl_xor_sync(0xffffffffu, wlast, o));
  for (int b = 0; b < nbatches; b++) {
    const int slot = b % BW_NSTAGE;
    const int hi = top - b * BW_BATCH;
    const int lo = hi - BW_BATCH + 1 > 0 ? hi - BW_BATCH + 1 : 0;
    const int nb = hi - lo + 1;
    warp_wait(&sm.full[slot], (b / BW_NSTAGE) & 1, lane);
    // per-warp list of the entries touching the sub-tile, newest first
    int nl = 0;
    for (int k = 0; k < nb; k += 32) {
      const int i = nb - 1 - (k + lane);
      bool hit = false;
      if (i >= 0 && lo + i <= wlast) {
        const float4 q = sm.ent[slot][i].f.box;
        const float cx = fminf(fmaxf(q.x, wx0), wx1), cy = fminf(fmaxf(q.y, wy0), wy1);
        hit = fabsf(q.x - cx) <= q.z && fabsf(q.y - cy) <= q.w;
        if (hit && (q.x != cx || q.y != cy))
          hit = ellipse_meets_box(sm.ent[slot][i].f.con, q, wx0, wx1, wy0, wy1);
      }
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const float a32 = sm.ent[slot][i].f.col.x;
        sm.list[warp][nl + __popc(m & lanemask_lt())] =
            make_int4(i, __float_as_int(entry_ucut(a32)), __float_as_int(entry_uclamp(a32)), 0);
      }
      nl += __popc(m);
    }
    __syncwarp();
    for (int li = 0; li < nl; li++) {
      const int4 L = sm.list[warp][li];
      const int i = L.x;
      const StageEntry& E = sm.ent[slot][i];
      const float ucut = __int_as_float(L.y), uclamp = __int_as_float(L.z);
      double vd[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      float vf[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < BW_NPX; k++)
        bw_pixel_step(q[k], E, lo + i, fx, fy0 + 4.0 * k, ucut, uclamp, sm.exp2tab, vd, vf);
      const bool any = vf[1] != 0.f || vf[2] != 0.f || vf[3] != 0.f || vf[0] != 0.f || vd[0] != 0.0;
      if (!__any_sync(0xffffffffu, any)) continue;
      double* dst = screen + 9 * (size_t)sm.gid[slot][i];
      double v[9] = {vd[0], vd[1], vd[2], vd[3], vd[4], (double)vf[0], (double)vf[1], (double)vf[2], (double)vf[3]};
      const double tot = warp_reduce9(v, lane);
      if (vidx >= 0 && tot != 0) atomicAdd(dst + vidx, (double)tot);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[slot]);
  }
}

// ------------------------------------------------------------------ K6

struct ChainCam {
  double fx, fy, W, H, R[9], T[3], center[3], limx, limy;
};

__device__ __forceinline__ void quat_rot(const double* q, double* Rq, double* qn, double& nrm) {
  nrm = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
  const double rn = 1.0 / nrm;  // gradients only: one reciprocal for the four quotients (<= 1 ulp each)
  const double w = q[0] * rn, x = q[1] * rn, y = q[2] * rn, z = q[3] * rn;
  qn[0] = w; qn[1] = x; qn[2] = y; qn[3] = z;
  Rq[0] = 1.0 - 2.0 * (y * y + z * z);
  Rq[1] = 2.0 * (x * y - w * z);
  Rq[2] = 2.0 * (x * z + w * y);
  Rq[3] = 2.0 * (x * y + w * z);
  Rq[4] = 1.0 - 2.0 * (x * x + z * z);
  Rq[5] = 2.0 * (y * z - w * x);
  Rq[6] = 2.0 * (x * z - w * y);
  Rq[7] = 2.0 * (y * z + w * x);
  Rq[8] = 1.0 - 2.0 * (x * x + y * y);
}

// Chain rule of one visible Gaussian i (render.py:185-313).
__device__ __noinline__ void chain_one(const ChainCam& cc, const hgs_gaussians& gs, const double* __restrict__ screen,
                                       const hgs_gaussian_grads& out, float scale, int accumulate, int64_t i) {
  // all per-Gaussian inputs are loaded up front (independent loads whose
  // latencies overlap) ...
  const double* pg = screen + 9 * i;
  double pgv[9];
#pragma unroll
  for (int k = 0; k < 9; k++) pgv[k] = pg[k];
  const float p_lg = gs.logits[i];
  const float p_c[3] = {gs.centers[3 * i], gs.centers[3 * i + 1], gs.centers[3 * i + 2]};
  const float p_dc[3] = {gs.colors_dc[3 * i], gs.colors_dc[3 * i + 1], gs.colors_dc[3 * i + 2]};
  const float p_q[4] = {gs.rotations[4 * i], gs.rotations[4 * i + 1], gs.rotations[4 * i + 2], gs.rotations[4 * i + 3]};
  const float p_ls[3] = {gs.log_scales[3 * i], gs.log_scales[3 * i + 1], gs.log_scales[3 * i + 2]};
  float rr[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (gs.colors_rest)
#pragma unroll
    for (int k = 0; k < 9; k++) rr[k] = gs.colors_rest[9 * i + k];
  // ... and for accumulation every old gradient value too (independent
  // loads, overlapping the arithmetic) instead of 24 serialised
  // read-modify-writes through possibly aliasing pointers
  float o_lg = 0.f, o_dn = 0.f, o_c[3] = {0.f, 0.f, 0.f}, o_s[3] = {0.f, 0.f, 0.f}, o_dc[3] = {0.f, 0.f, 0.f};
  float o_r[4] = {0.f, 0.f, 0.f, 0.f}, o_rest[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (accumulate) {
    o_lg = *(out.logits + i);
    if (out.densify_norm) o_dn = *(out.densify_norm + i);
#pragma unroll
    for (int k = 0; k < 3; k++) {
      o_c[k] = *(out.centers + 3 * i + k);
      o_s[k] = *(out.log_scales + 3 * i + k);
      o_dc[k] = *(out.colors_dc + 3 * i + k);
    }
#pragma unroll
    for (int k = 0; k < 4; k++) o_r[k] = *(out.rotations + 4 * i + k);
    if (out.colors_rest)
#pragma unroll
      for (int k = 0; k < 9; k++) o_rest[k] = *(out.colors_rest + 9 * i + k);
  }
  auto put = [&](float* dst, int64_t idx, double v, float old) { dst[idx] = old + (float)(v * scale); };
  const double gm0 = pgv[0], gm1 = pgv[1];
  const double gcov[4] = {pgv[2], pgv[3], pgv[3], pgv[4]};
  const double ga = pgv[5];
  const double fx = cc.fx, fy = cc.fy;
  const double* Rw = cc.R;
  // opacity: sigma = alpha G, alpha = sigmoid(logit)   (render.py:199-200)
  const double alpha = 1.0 / (1.0 + exp(-(double)p_lg));
  put(out.logits, i, ga * alpha * (1.0 - alpha), o_lg);
  // colour (render.py:202-220)
  const double c0 = p_c[0], c1 = p_c[1], c2 = p_c[2];
  double pre[3], gpre[3], gc[3] = {0.0, 0.0, 0.0};
  for (int ch = 0; ch < 3; ch++) pre[ch] = 0.5 + SH_C0 * (double)p_dc[ch];
  if (gs.colors_rest) {
    const double d0 = c0 - cc.center[0], d1 = c1 - cc.center[1], d2 = c2 - cc.center[2];
    const double dist = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
    const double den = fmax(dist, 1e-12);
    const double rden = 1.0 / den;
    const double x = d0 * rden, y = d1 * rden, z = d2 * rden;
    for (int ch = 0; ch < 3; ch++)
      pre[ch] = pre[ch] + SH_C1 * ((-y * (double)rr[ch] + z * (double)rr[3 + ch]) - x * (double)rr[6 + ch]);
    for (int ch = 0; ch < 3; ch++) gpre[ch] = pgv[6 + ch] * (pre[ch] > 0.0 ? 1.0 : 0.0);
    for (int ch = 0; ch < 3; ch++) {
      put(out.colors_rest, 9 * i + 0 * 3 + ch, -SH_C1 * y * gpre[ch], o_rest[ch]);
      put(out.colors_rest, 9 * i + 1 * 3 + ch, SH_C1 * z * gpre[ch], o_rest[3 + ch]);
      put(out.colors_rest, 9 * i + 2 * 3 + ch, -SH_C1 * x * gpre[ch], o_rest[6 + ch]);
    }
    const double s2 = (gpre[0] * rr[6] + gpre[1] * rr[7]) + gpre[2] * rr[8];
    const double s0 = (gpre[0] * rr[0] + gpre[1] * rr[1]) + gpre[2] * rr[2];
    const double s1 = (gpre[0] * rr[3] + gpre[1] * rr[4]) + gpre[2] * rr[5];
    const double gd[3] = {-SH_C1 * s2, -SH_C1 * s0, SH_C1 * s1};
    const double dd = (gd[0] * x + gd[1] * y) + gd[2] * z;
    const double dv[3] = {x, y, z};
    const double rdist = 1.0 / dist;
    for (int j = 0; j < 3; j++) gc[j] += (gd[j] - dv[j] * dd) * rdist;
  } else {
    for (int ch = 0; ch < 3; ch++) gpre[ch] = pgv[6 + ch] * (pre[ch] > 0.0 ? 1.0 : 0.0);
  }
  for (int ch = 0; ch < 3; ch++) put(out.colors_dc, 3 * i + ch, SH_C0 * gpre[ch], o_dc[ch]);
  // forward intermediates (render.py:222-248)
  double t[3];
  for (int j = 0; j < 3; j++) t[j] = dot3(c0, c1, c2, Rw[j * 3], Rw[j * 3 + 1], Rw[j * 3 + 2]) + cc.T[j];
  const double tz = t[2];
  const double rtz = 1.0 / tz;  // the chain only produces gradients: reciprocal products, <= 1-2 ulp
  const double rx_raw = t[0] * rtz, ry_raw = t[1] * rtz;
  const double rx = clampd(rx_raw, -cc.limx, cc.limx), ry = clampd(ry_raw, -cc.limy, cc.limy);
  const double in_x = fabs(rx_raw) < cc.limx ? 1.0 : 0.0, in_y = fabs(ry_raw) < cc.limy ? 1.0 : 0.0;
  const double J[6] = {fx * rtz, 0.0, -fx * rx * rtz, 0.0, fy * rtz, -fy * ry * rtz};
  double q[4], Rq[9], qn[4], nrm;
  for (int k = 0; k < 4; k++) q[k] = p_q[k];
  quat_rot(q, Rq, qn, nrm);
  double s[3], M[9], sig[9], A[6];
  for (int j = 0; j < 3; j++) s[j] = exp((double)p_ls[j]);
  for (int a = 0; a < 3; a++)
    for (int b = 0; b < 3; b++) M[a * 3 + b] = Rq[a * 3 + b] * s[b];
  for (int a = 0; a < 3; a++)
    for (int b = 0; b < 3; b++) sig[a * 3 + b] = dot3(M[a * 3], M[a * 3 + 1], M[a * 3 + 2], M[b * 3], M[b * 3 + 1], M[b * 3 + 2]);
  for (int j = 0; j < 2; j++)
    for (int b = 0; b < 3; b++) A[j * 3 + b] = dot3(J[j * 3], J[j * 3 + 1], J[j * 3 + 2], Rw[b], Rw[3 + b], Rw[6 + b]);
  // cov2d = A Sigma A^T (render.py:250-253)
  double gS[9], gA[6], gJ[6];
  for (int a = 0; a < 3; a++)
    for (int b = 0; b < 3; b++) {
      double acc = 0.0;
      for (int j = 0; j < 2; j++)
        for (int k = 0; k < 2; k++) acc += A[j * 3 + a] * gcov[j * 2 + k] * A[k * 3 + b];
      gS[a * 3 + b] = acc;
    }
  for (int j = 0; j < 2; j++)
    for (int b = 0; b < 3; b++) {
      double acc = 0.0;
      for (int k = 0; k < 2; k++)
        for (int a = 0; a < 3; a++) acc += gcov[j * 2 + k] * A[k * 3 + a] * sig[a * 3 + b];
      gA[j * 3 + b] = 2.0 * acc;
    }
  for (int j = 0; j < 2; j++)
    for (int k = 0; k < 3; k++)
      gJ[j * 3 + k] = (gA[j * 3] * Rw[k * 3] + gA[j * 3 + 1] * Rw[k * 3 + 1]) + gA[j * 3 + 2] * Rw[k * 3 + 2];
  // mean2d and J(t) (render.py:255-271)
  double gt[3] = {0.0, 0.0, 0.0};
  gt[0] += gm0 * fx * rtz;
  gt[1] += gm1 * fy * rtz;
  gt[2] += -(gm0 * fx * rx_raw + gm1 * fy * ry_raw) * rtz;
  const double inv_tz2 = rtz * rtz;
  gt[0] += gJ[2] * (-fx * in_x * inv_tz2);
  gt[1] += gJ[5] * (-fy * in_y * inv_tz2);
  gt[2] += ((gJ[0] * (-fx * inv_tz2) + gJ[4] * (-fy * inv_tz2)) + gJ[2] * fx * (in_x * rx_raw + rx) * inv_tz2) +
           gJ[5] * fy * (in_y * ry_raw + ry) * inv_tz2;
  for (int c = 0; c < 3; c++) gc[c] += dot3(gt[0], gt[1], gt[2], Rw[c], Rw[3 + c], Rw[6 + c]);
  for (int c = 0; c < 3; c++) put(out.centers, 3 * i + c, gc[c], o_c[c]);
  // Sigma = M M^T, M = R diag(s) (render.py:273-277)
  double gM[9], gR[9], gsc[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < 3; a++)
    for (int c = 0; c < 3; c++) {
      double acc = 0.0;
      for (int b = 0; b < 3; b++) acc += gS[a * 3 + b] * M[b * 3 + c];
      gM[a * 3 + c] = 2.0 * acc;
    }
  for (int a = 0; a < 3; a++)
    for (int c = 0; c < 3; c++) {
      gR[a * 3 + c] = gM[a * 3 + c] * s[c];
      gsc[c] += gM[a * 3 + c] * Rq[a * 3 + c];
    }
  for (int j = 0; j < 3; j++) put(out.log_scales, 3 * i + j, gsc[j] * s[j], o_s[j]);
  // rotation through dR/dq and the normalisation (render.py:279-284, 290-313)
  const double w = qn[0], x = qn[1], y = qn[2], z = qn[3];
  const double D[4][9] = {{0, -z, y, z, 0, -x, -y, x, 0},
                          {0, y, z, y, -2 * x, -w, z, w, -2 * x},
                          {-2 * y, x, w, x, 0, z, -w, z, -2 * y},
                          {-2 * z, -w, x, w, -2 * z, y, x, y, 0}};
  double gqn[4];
  for (int k = 0; k < 4; k++) {
    double acc = 0.0;
    for (int a = 0; a < 9; a++) acc += gR[a] * (2.0 * D[k][a]);
    gqn[k] = acc;
  }
  const double dq = ((gqn[0] * qn[0] + gqn[1] * qn[1]) + gqn[2] * qn[2]) + gqn[3] * qn[3];
  const double rnrm = 1.0 / nrm;
  for (int k = 0; k < 4; k++) put(out.rotations, 4 * i + k, (gqn[k] - qn[k] * dq) * rnrm, o_r[k]);
  if (out.densify_norm) {
    const double sx = gm0 * (cc.W / 2.0), sy = gm1 * (cc.H / 2.0);
    put(out.densify_norm, i, sqrt(sx * sx + sy * sy) / (double)scale, o_dn);
  }
}

// One CTA per PB_SPAN consecutive Gaussians: flags and (without
// accumulation) zeros for the invisible ones, then the visible ones -- a
// few percent of them for a training view -- compacted in shared memory
// so every thread runs the long fp64 chain on a visible Gaussian.
#ifndef HGS_PB_ROWS
#define HGS_PB_ROWS 8
#endif
#ifndef HGS_PB_MINB
#define HGS_PB_MINB 4
#endif
constexpr int PB_THREADS = 128;
constexpr int PB_SPAN = HGS_PB_ROWS * PB_THREADS;
__global__ void __launch_bounds__(PB_THREADS, HGS_PB_MINB) project_backward_kernel(const hgs_camera* __restrict__ cam_ptr,
                                                                      hgs_gaussians gs,
                                                                      const int32_t* __restrict__ count,
                                                                      const double* __restrict__ screen,
                                                                      hgs_gaussian_grads out, float scale,
                                                                      int accumulate) {
  __shared__ ChainCam cc;
  __shared__ int32_t list[PB_SPAN];
  __shared__ int nlist;
  if (threadIdx.x == 0) {
    cc.fx = cam_ptr->fx; cc.fy = cam_ptr->fy;
    cc.W = (double)cam_ptr->width; cc.H = (double)cam_ptr->height;
    for (int k = 0; k < 9; k++) cc.R[k] = cam_ptr->R[k];
    for (int k = 0; k < 3; k++) { cc.T[k] = cam_ptr->T[k]; cc.center[k] = cam_ptr->center[k]; }
    cc.limx = cam_ptr->limx; cc.limy = cam_ptr->limy;
    nlist = 0;
  }
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * PB_SPAN;
  for (int k = threadIdx.x; k < PB_SPAN; k += PB_THREADS) {
    const int64_t i = base + k;
    if (i >= gs.n) break;
    const bool vis = count[i] > 0;
    if (out.visible) {
      if (accumulate) out.visible[i] |= (uint8_t)vis;
      else out.visible[i] = (uint8_t)vis;
    }
    if (out.visible_count) {
      if (accumulate) out.visible_count[i] += vis ? 1.0f : 0.0f;
      else out.visible_count[i] = vis ? 1.0f : 0.0f;
    }
    if (vis) {
      list[atomicAdd(&nlist, 1)] = (int32_t)k;
    } else if (!accumulate) {
      for (int q = 0; q < 3; q++) { out.centers[3 * i + q] = 0.f; out.log_scales[3 * i + q] = 0.f; out.colors_dc[3 * i + q] = 0.f; }
      for (int q = 0; q < 4; q++) out.rotations[4 * i + q] = 0.f;
      out.logits[i] = 0.f;
      if (out.colors_rest) for (int q = 0; q < 9; q++) out.colors_rest[9 * i + q] = 0.f;
      if (out.densify_norm) out.densify_norm[i] = 0.f;
    }
  }
  __syncthreads();
  const int nl = nlist;
  for (int j = threadIdx.x; j < nl; j += PB_THREADS) chain_one(cc, gs, screen, out, scale, accumulate, base + list[j]);
}

}  // namespace hgs

extern "C" int hgs_blend_backward(const hgs_projected* proj, const hgs_tiles* tiles, int32_t width, int32_t height,
                                  const hgs_mesh_layer* mesh, const double* bg_host3, const double* final_t,
                                  const int32_t* last, const float* grad_color, const float* grad_t,
                                  double* screen_grads, float* mesh_color_grad, int32_t accumulate_mesh,
                                  void* stream) {
  using namespace hgs;
  if (!proj || !tiles || !bg_host3 || !final_t || !last || !grad_color || !screen_grads)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_blend_backward: null argument");
  if (!proj->rec || !proj->cull) return hgs_set_error(HGS_ERR_INVALID, "hgs_blend_backward: projection needs rec + cull");
  if (tiles->tile_px != 16 || tiles->tiles_x != (width + 15) / 16 || tiles->tiles_y != (height + 15) / 16)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_blend_backward: tile grid does not match image size");
  hgs_mesh_layer ml{};
  if (mesh && mesh->color) {
    if (!mesh->depth || !mesh->triangle_id) return hgs_set_error(HGS_ERR_INVALID, "hgs_blend_backward: incomplete mesh layer");
    ml = *mesh;
  }
  const int n_tiles = tiles->tiles_x * tiles->tiles_y;
  const size_t smem = sizeof(BwSmem);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(blend_backward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  blend_backward_kernel<<<n_tiles, BW_THREADS, smem, (cudaStream_t)stream>>>(
      (const BlendRec*)proj->rec, (const CullRec*)proj->cull, tiles->entries, tiles->tile_starts, tiles->tiles_x,
      width, height, ml, bg_host3[0], bg_host3[1], bg_host3[2], final_t, last, grad_color, grad_t, screen_grads,
      mesh_color_grad, accumulate_mesh, tiles->counters);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}

extern "C" int hgs_project_backward(const hgs_camera* cam, const hgs_gaussians* gs, const hgs_projected* proj,
                                    const double* screen_grads, hgs_gaussian_grads* grads, float scale,
                                    int32_t accumulate, void* stream) {
  using namespace hgs;
  if (!cam || !gs || !proj || !screen_grads || !grads) return hgs_set_error(HGS_ERR_INVALID, "hgs_project_backward: null argument");
  if (gs->n == 0) return HGS_OK;
  if (!grads->centers || !grads->rotations || !grads->log_scales || !grads->logits || !grads->colors_dc || !proj->count)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_project_backward: missing gradient pointer");
  if ((gs->colors_rest == nullptr) != (grads->colors_rest == nullptr))
    return hgs_set_error(HGS_ERR_INVALID, "hgs_project_backward: colors_rest presence mismatch");
  project_backward_kernel<<<ceil_div(gs->n, PB_SPAN), PB_THREADS, 0, (cudaStream_t)stream>>>(cam, *gs, proj->count,
                                                                                         screen_grads,
                                                                                 *grads, scale, accumulate);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}
