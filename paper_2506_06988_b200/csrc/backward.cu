// K5 blend backward: backward_kernel (gsmesh/splat/kernels.py:77-160) with the
// per-Gaussian reduction of render.py:155-157, and K6 project backward:
// _chain_to_parameters (splat/render.py:185-313) + densify statistic and
// visibility (render.py:171-178).
//
// K5: one CTA per 16x16 tile, warps own 8x4 sub-tiles.  Each pixel walks its
// tile list in reverse from its last blended entry (kernels.py:120),
// recomputing sigma; T before each entry is reconstructed by division, the
// suffix colour starts at T_final * (mesh colour or background), exactly as
// the reference.  Entries are staged in shared memory in batches of 256
// (newest first) and culled per warp with the same ellipse/sub-tile test as
// the forward pass.  The per-entry 9-vector (mean2d 2, cov 3 full-matrix
// convention, alpha, rgb 3) is reduced over the warp (reduce-scatter in
// fp32) and added to the per-Gaussian fp64 accumulator with one atomic per
// component per warp.
//
// exp(): SFU value with a local exact fp64 recompute whenever sigma lies
// near the 1/255 skip or the 0.99 clamp threshold, so both per-entry
// decisions equal the reference's.
#include "common.cuh"

namespace hgs {

constexpr int BW_THREADS = 256;
constexpr int BW_BATCH = 256;
constexpr double BW_LOG2E = 1.4426950408889634;

struct BwSmem {
  double2 a[BW_BATCH];  // mean x, y
  double2 b[BW_BATCH];  // conic xx, 2*xy
  double2 c[BW_BATCH];  // conic yy, depth
  double2 d[BW_BATCH];  // alpha, r
  double2 e[BW_BATCH];  // g, b
  float4 box[BW_BATCH];
  float4 con[BW_BATCH];
  uint32_t gid[BW_BATCH];
  unsigned char list[BW_THREADS / 32][BW_BATCH];
  int max_last;
};

__device__ __forceinline__ bool bw_ellipse_meets_box(float4 con, float mx, float my, float x0, float x1, float y0,
                                                     float y1) {
  auto edge_min = [](float a, float b, float c, float u, float v0, float v1) {
    const float v = fminf(fmaxf(-b * u / c, v0), v1);
    return a * u * u + 2.0f * b * u * v + c * v * v;
  };
  const float a = con.x, b = con.y, c = con.z;
  const float dx0 = x0 - mx, dx1 = x1 - mx, dy0 = y0 - my, dy1 = y1 - my;
  float mn = edge_min(a, b, c, dx0, dy0, dy1);
  mn = fminf(mn, edge_min(a, b, c, dx1, dy0, dy1));
  mn = fminf(mn, edge_min(c, b, a, dy0, dx0, dx1));
  mn = fminf(mn, edge_min(c, b, a, dy1, dx0, dx1));
  return mn <= 9.05f;
}

// Sum 16 per-lane values over the warp (reduce-scatter, 16 shuffles);
// returns the total of value index scatter16_index(lane); lanes 2k and
// 2k+1 hold the same index.
__device__ __forceinline__ float warp_reduce_scatter16(float v[16], int lane) {
#pragma unroll
  for (int i = 0; i < 8; i++) {  // offset 16: keep 8 values
    const bool upper = lane & 16;
    const float send = upper ? v[i] : v[i + 8];
    const float recv = __shfl_xor_sync(0xffffffffu, send, 16);
    v[i] = (upper ? v[i + 8] : v[i]) + recv;
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {  // offset 8
    const bool upper = lane & 8;
    const float send = upper ? v[i] : v[i + 4];
    const float recv = __shfl_xor_sync(0xffffffffu, send, 8);
    v[i] = (upper ? v[i + 4] : v[i]) + recv;
  }
#pragma unroll
  for (int i = 0; i < 2; i++) {  // offset 4
    const bool upper = lane & 4;
    const float send = upper ? v[i] : v[i + 2];
    const float recv = __shfl_xor_sync(0xffffffffu, send, 4);
    v[i] = (upper ? v[i + 2] : v[i]) + recv;
  }
  {  // offset 2
    const bool upper = lane & 2;
    const float send = upper ? v[0] : v[1];
    const float recv = __shfl_xor_sync(0xffffffffu, send, 2);
    v[0] = (upper ? v[1] : v[0]) + recv;
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  return v[0];
}

// value index held by a lane after warp_reduce_scatter16
__device__ __forceinline__ int scatter16_index(int lane) {
  return ((lane & 16) ? 8 : 0) + ((lane & 8) ? 4 : 0) + ((lane & 4) ? 2 : 0) + ((lane & 2) ? 1 : 0);
}

// Per-pixel reverse-walk state.
struct BwPix {
  int64_t last;
  double gr, gg, gb, gtp, t_fin, t_after, acc_r, acc_g, acc_b, fx, fy;
  bool inside, mesh_here;
};

__device__ __forceinline__ void bw_pixel_init(BwPix& q, int px, int py, int width, int height, int64_t s,
                                              const hgs_mesh_layer& mesh, double bg0, double bg1, double bg2,
                                              const double* __restrict__ final_t, const int32_t* __restrict__ last_idx,
                                              const float* __restrict__ grad_color, const float* __restrict__ grad_t,
                                              float* __restrict__ mesh_grad, int accumulate_mesh) {
  q.inside = px < width && py < height;
  q.fx = px + 0.5;
  q.fy = py + 0.5;
  q.last = -1;
  q.gr = q.gg = q.gb = q.gtp = 0.0;
  q.t_fin = 1.0;
  q.mesh_here = false;
  const int64_t p = (int64_t)py * width + px;
  if (q.inside) {
    q.last = last_idx[p];
    q.gr = grad_color[3 * p];
    q.gg = grad_color[3 * p + 1];
    q.gb = grad_color[3 * p + 2];
    q.gtp = grad_t ? (double)grad_t[p] : 0.0;
    q.t_fin = final_t[p];
    q.mesh_here = mesh.color != nullptr && mesh.triangle_id[p] >= 0;
    if (mesh_grad) {  // d pixel / d mesh colour = T * valid (render.py:180-181)
      const double f = q.mesh_here ? q.t_fin : 0.0;
      float* mg = mesh_grad + 3 * p;
      if (accumulate_mesh) {
        mg[0] += (float)(q.gr * f); mg[1] += (float)(q.gg * f); mg[2] += (float)(q.gb * f);
      } else {
        mg[0] = (float)(q.gr * f); mg[1] = (float)(q.gg * f); mg[2] = (float)(q.gb * f);
      }
    }
  }
  q.t_after = q.t_fin;  // suffix colour starts at T_final * (mesh or background) (kernels.py:111-119)
  if (q.mesh_here) {
    q.acc_r = q.t_after * (double)mesh.color[3 * p];
    q.acc_g = q.t_after * (double)mesh.color[3 * p + 1];
    q.acc_b = q.t_after * (double)mesh.color[3 * p + 2];
  } else {
    q.acc_r = q.t_after * bg0;
    q.acc_g = q.t_after * bg1;
    q.acc_b = q.t_after * bg2;
  }
  if (q.last >= 0) q.last -= s;  // relative to the tile start
}

// One reverse step of kernels.py:120-160 for entry slot i (relative index
// rel); adds this pixel's 9-vector into v.
__device__ __forceinline__ bool bw_pixel_step(BwPix& q, const BwSmem& sm, int i, int rel, float v[16]) {
  if (q.last < 0 || rel > q.last) return false;
  const double2 A = sm.a[i], B = sm.b[i], C = sm.c[i];
  const double dx = q.fx - A.x, dy = q.fy - A.y;
  const double m = B.x * dx * dx + B.y * dx * dy + C.x * dy * dy;
  if (m > SUPPORT_MAHAL2 || m < 0.0) return false;
  // SFU exp, exact fp64 recompute near the skip/clamp thresholds
  float ef;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ef) : "f"((float)(m * (-0.5 * BW_LOG2E))));
  double gauss = (double)ef;
  const double alpha = sm.d[i].x;
  double sig = alpha * gauss;
  if (fabs(sig - SIGMA_SKIP) <= 2e-6 * SIGMA_SKIP || fabs(sig - ALPHA_CLAMP) <= 2e-6) {
    gauss = exp(-0.5 * m);
    sig = alpha * gauss;
  }
  const bool clamped = sig > ALPHA_CLAMP;
  if (clamped) sig = ALPHA_CLAMP;
  if (sig < SIGMA_SKIP) return false;
  const double2 D = sm.d[i], E = sm.e[i];
  const double cr = D.y, cg = E.x, cb = E.y;
  const double one_minus = 1.0 - sig;
  const double inv = 1.0 / one_minus;  // one division for the five of kernels.py:135,142-146
  const double t_before = q.t_after * inv;
  const double w = sig * t_before;
  const float wf = (float)w;
  v[6] += (float)q.gr * wf;
  v[7] += (float)q.gg * wf;
  v[8] += (float)q.gb * wf;
  double s_i = (q.gr * (cr * t_before - q.acc_r * inv) + q.gg * (cg * t_before - q.acc_g * inv)) +
               q.gb * (cb * t_before - q.acc_b * inv);
  if (q.gtp != 0.0) s_i += q.gtp * (-q.t_fin * inv);
  if (!clamped) {
    // no decision depends on these: fp32 from here on
    const float dxf = (float)dx, dyf = (float)dy, cbh = 0.5f * (float)B.y;  // conic xy
    const float qd_x = (float)B.x * dxf + cbh * dyf;
    const float qd_y = cbh * dxf + (float)C.x * dyf;
    const float common = (float)(s_i * sig);
    const float hc = 0.5f * common;
    v[0] += common * qd_x;
    v[1] += common * qd_y;
    v[2] += hc * qd_x * qd_x;
    v[3] += hc * qd_x * qd_y;
    v[4] += hc * qd_y * qd_y;
    v[5] += (float)(s_i * gauss);
  }
  q.acc_r += cr * w;
  q.acc_g += cg * w;
  q.acc_b += cb * w;
  q.t_after = t_before;
  return true;
}

// 256 threads = 8 warps, each warp an 8x4 sub-tile, one pixel per lane.
__global__ void __launch_bounds__(BW_THREADS, 2) blend_backward_kernel(
    const BlendRec* __restrict__ rec, const float4* __restrict__ cull, const uint32_t* __restrict__ entries,
    const int64_t* __restrict__ tile_starts, int tiles_x, int width, int height, hgs_mesh_layer mesh, double bg0,
    double bg1, double bg2, const double* __restrict__ final_t, const int32_t* __restrict__ last_idx,
    const float* __restrict__ grad_color, const float* __restrict__ grad_t, double* __restrict__ screen,
    float* __restrict__ mesh_grad, int accumulate_mesh) {
  __shared__ BwSmem sm;
  const int tile = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int sx0 = (warp & 1) * 8, sy0 = (warp >> 1) * 4;
  const int px = tx * 16 + sx0 + (lane & 7);
  const int py = ty * 16 + sy0 + (lane >> 3);
  const int64_t s = tile_starts[tile];
  const float wx0 = tx * 16 + sx0 + 0.5f, wx1 = wx0 + 7.0f;
  const float wy0 = ty * 16 + sy0 + 0.5f, wy1 = wy0 + 3.0f;
  BwPix q0;
  bw_pixel_init(q0, px, py, width, height, s, mesh, bg0, bg1, bg2, final_t, last_idx, grad_color, grad_t, mesh_grad,
                accumulate_mesh);
  if (threadIdx.x == 0) sm.max_last = -1;
  __syncthreads();
  if (q0.last >= 0) atomicMax(&sm.max_last, (int)q0.last);
  __syncthreads();
  const int top = sm.max_last;  // relative index of the newest entry any pixel used
  const int vidx = scatter16_index(lane);
  for (int hi = top; hi >= 0; hi -= BW_BATCH) {
    const int lo = hi - BW_BATCH + 1 > 0 ? hi - BW_BATCH + 1 : 0;
    const int nb = hi - lo + 1;
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += BW_THREADS) {  // slot i holds entry lo + i
      const uint32_t g = entries[s + lo + i];
      const double2* rp = reinterpret_cast<const double2*>(rec + g);
      sm.a[i] = __ldg(rp);
      sm.b[i] = __ldg(rp + 1);
      sm.c[i] = __ldg(rp + 2);
      sm.d[i] = __ldg(rp + 3);
      sm.e[i] = __ldg(rp + 4);
      sm.box[i] = __ldg(cull + 3 * (size_t)g);
      sm.con[i] = __ldg(cull + 3 * (size_t)g + 1);
      sm.gid[i] = g;
    }
    __syncthreads();
    // per-warp list, newest first
    int nl = 0;
    for (int k = 0; k < nb; k += 32) {
      const int i = nb - 1 - (k + lane);
      bool hit = false;
      if (i >= 0) {
        const float4 b = sm.box[i];
        const float cx = fminf(fmaxf(b.x, wx0), wx1), cy = fminf(fmaxf(b.y, wy0), wy1);
        hit = fabsf(b.x - cx) <= b.z && fabsf(b.y - cy) <= b.w;
        if (hit && (b.x != cx || b.y != cy)) hit = bw_ellipse_meets_box(sm.con[i], b.x, b.y, wx0, wx1, wy0, wy1);
      }
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (hit) sm.list[warp][nl + __popc(m & lanemask_lt())] = (unsigned char)i;
      nl += __popc(m);
    }
    __syncwarp();
    for (int li = 0; li < nl; li++) {
      const int i = sm.list[warp][li];
      float v[16];
#pragma unroll
      for (int c = 0; c < 16; c++) v[c] = 0.0f;
      const bool c0 = bw_pixel_step(q0, sm, i, lo + i, v);
      if (__any_sync(0xffffffffu, c0)) {
        const float tot = warp_reduce_scatter16(v, lane);
        if ((lane & 1) == 0 && vidx < 9 && tot != 0.0f) atomicAdd(&screen[9 * (size_t)sm.gid[i] + vidx], (double)tot);
      }
    }
  }
}

// ------------------------------------------------------------------ K6

struct ChainCam {
  double fx, fy, W, H, R[9], T[3], center[3], limx, limy;
};

__device__ __forceinline__ void quat_rot(const double* q, double* Rq, double* qn, double& nrm) {
  nrm = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
  const double w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
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

__global__ void __launch_bounds__(128) project_backward_kernel(const hgs_camera* __restrict__ cam_ptr, hgs_gaussians gs,
                                                               const int32_t* __restrict__ count,
                                                               const double* __restrict__ screen,
                                                               hgs_gaussian_grads out, float scale, int accumulate) {
  __shared__ ChainCam cc;
  if (threadIdx.x == 0) {
    cc.fx = cam_ptr->fx; cc.fy = cam_ptr->fy;
    cc.W = (double)cam_ptr->width; cc.H = (double)cam_ptr->height;
    for (int k = 0; k < 9; k++) cc.R[k] = cam_ptr->R[k];
    for (int k = 0; k < 3; k++) { cc.T[k] = cam_ptr->T[k]; cc.center[k] = cam_ptr->center[k]; }
    cc.limx = cam_ptr->limx; cc.limy = cam_ptr->limy;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= gs.n) return;
  const bool vis = count[i] > 0;
  auto put = [&](float* dst, int64_t idx, double v) {
    if (accumulate) dst[idx] += (float)(v * scale);
    else dst[idx] = (float)(v * scale);
  };
  if (out.visible) {
    if (accumulate) out.visible[i] |= (uint8_t)vis;
    else out.visible[i] = (uint8_t)vis;
  }
  if (!vis) {
    if (!accumulate) {
      for (int k = 0; k < 3; k++) { out.centers[3 * i + k] = 0.f; out.log_scales[3 * i + k] = 0.f; out.colors_dc[3 * i + k] = 0.f; }
      for (int k = 0; k < 4; k++) out.rotations[4 * i + k] = 0.f;
      out.logits[i] = 0.f;
      if (out.colors_rest) for (int k = 0; k < 9; k++) out.colors_rest[9 * i + k] = 0.f;
      if (out.densify_norm) out.densify_norm[i] = 0.f;
    }
    return;
  }
  const double* pg = screen + 9 * i;
  const double gm0 = pg[0], gm1 = pg[1];
  const double gcov[4] = {pg[2], pg[3], pg[3], pg[4]};
  const double ga = pg[5];
  const double fx = cc.fx, fy = cc.fy;
  const double* Rw = cc.R;
  // opacity: sigma = alpha G, alpha = sigmoid(logit)   (render.py:199-200)
  const double alpha = 1.0 / (1.0 + exp(-(double)gs.logits[i]));
  put(out.logits, i, ga * alpha * (1.0 - alpha));
  // colour (render.py:202-220)
  const double c0 = gs.centers[3 * i], c1 = gs.centers[3 * i + 1], c2 = gs.centers[3 * i + 2];
  double pre[3], gpre[3], gc[3] = {0.0, 0.0, 0.0};
  for (int ch = 0; ch < 3; ch++) pre[ch] = 0.5 + SH_C0 * (double)gs.colors_dc[3 * i + ch];
  if (gs.colors_rest) {
    const double d0 = c0 - cc.center[0], d1 = c1 - cc.center[1], d2 = c2 - cc.center[2];
    const double dist = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
    const double den = fmax(dist, 1e-12);
    const double x = d0 / den, y = d1 / den, z = d2 / den;
    const float* rr = gs.colors_rest + 9 * i;
    for (int ch = 0; ch < 3; ch++)
      pre[ch] = pre[ch] + SH_C1 * ((-y * (double)rr[ch] + z * (double)rr[3 + ch]) - x * (double)rr[6 + ch]);
    for (int ch = 0; ch < 3; ch++) gpre[ch] = pg[6 + ch] * (pre[ch] > 0.0 ? 1.0 : 0.0);
    for (int ch = 0; ch < 3; ch++) {
      put(out.colors_rest, 9 * i + 0 * 3 + ch, -SH_C1 * y * gpre[ch]);
      put(out.colors_rest, 9 * i + 1 * 3 + ch, SH_C1 * z * gpre[ch]);
      put(out.colors_rest, 9 * i + 2 * 3 + ch, -SH_C1 * x * gpre[ch]);
    }
    const double s2 = (gpre[0] * rr[6] + gpre[1] * rr[7]) + gpre[2] * rr[8];
    const double s0 = (gpre[0] * rr[0] + gpre[1] * rr[1]) + gpre[2] * rr[2];
    const double s1 = (gpre[0] * rr[3] + gpre[1] * rr[4]) + gpre[2] * rr[5];
    const double gd[3] = {-SH_C1 * s2, -SH_C1 * s0, SH_C1 * s1};
    const double dd = (gd[0] * x + gd[1] * y) + gd[2] * z;
    const double dv[3] = {x, y, z};
    for (int j = 0; j < 3; j++) gc[j] += (gd[j] - dv[j] * dd) / dist;
  } else {
    for (int ch = 0; ch < 3; ch++) gpre[ch] = pg[6 + ch] * (pre[ch] > 0.0 ? 1.0 : 0.0);
  }
  for (int ch = 0; ch < 3; ch++) put(out.colors_dc, 3 * i + ch, SH_C0 * gpre[ch]);
  // forward intermediates (render.py:222-248)
  double t[3];
  for (int j = 0; j < 3; j++) t[j] = dot3(c0, c1, c2, Rw[j * 3], Rw[j * 3 + 1], Rw[j * 3 + 2]) + cc.T[j];
  const double tz = t[2];
  const double rx_raw = t[0] / tz, ry_raw = t[1] / tz;
  const double rx = clampd(rx_raw, -cc.limx, cc.limx), ry = clampd(ry_raw, -cc.limy, cc.limy);
  const double in_x = fabs(rx_raw) < cc.limx ? 1.0 : 0.0, in_y = fabs(ry_raw) < cc.limy ? 1.0 : 0.0;
  const double J[6] = {fx / tz, 0.0, -fx * rx / tz, 0.0, fy / tz, -fy * ry / tz};
  double q[4], Rq[9], qn[4], nrm;
  for (int k = 0; k < 4; k++) q[k] = gs.rotations[4 * i + k];
  quat_rot(q, Rq, qn, nrm);
  double s[3], M[9], sig[9], A[6];
  for (int j = 0; j < 3; j++) s[j] = exp((double)gs.log_scales[3 * i + j]);
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
  gt[0] += gm0 * fx / tz;
  gt[1] += gm1 * fy / tz;
  gt[2] += -(gm0 * fx * rx_raw + gm1 * fy * ry_raw) / tz;
  const double inv_tz2 = 1.0 / (tz * tz);
  gt[0] += gJ[2] * (-fx * in_x * inv_tz2);
  gt[1] += gJ[5] * (-fy * in_y * inv_tz2);
  gt[2] += ((gJ[0] * (-fx * inv_tz2) + gJ[4] * (-fy * inv_tz2)) + gJ[2] * fx * (in_x * rx_raw + rx) * inv_tz2) +
           gJ[5] * fy * (in_y * ry_raw + ry) * inv_tz2;
  for (int c = 0; c < 3; c++) gc[c] += dot3(gt[0], gt[1], gt[2], Rw[c], Rw[3 + c], Rw[6 + c]);
  for (int c = 0; c < 3; c++) put(out.centers, 3 * i + c, gc[c]);
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
  for (int j = 0; j < 3; j++) put(out.log_scales, 3 * i + j, gsc[j] * s[j]);
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
  for (int k = 0; k < 4; k++) put(out.rotations, 4 * i + k, (gqn[k] - qn[k] * dq) / nrm);
  if (out.densify_norm) {
    const double sx = gm0 * (cc.W / 2.0), sy = gm1 * (cc.H / 2.0);
    put(out.densify_norm, i, sqrt(sx * sx + sy * sy) / (double)scale);
  }
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
  blend_backward_kernel<<<n_tiles, BW_THREADS, 0, (cudaStream_t)stream>>>(
      (const BlendRec*)proj->rec, (const float4*)proj->cull, tiles->entries, tiles->tile_starts, tiles->tiles_x, width,
      height, ml, bg_host3[0], bg_host3[1], bg_host3[2], final_t, last, grad_color, grad_t, screen_grads,
      mesh_color_grad, accumulate_mesh);
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
  project_backward_kernel<<<ceil_div(gs->n, 128), 128, 0, (cudaStream_t)stream>>>(cam, *gs, proj->count, screen_grads,
                                                                                 *grads, scale, accumulate);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}
