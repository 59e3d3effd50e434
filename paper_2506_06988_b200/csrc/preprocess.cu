// K1 preprocess: project (gsmesh/splat/project.py:70-140), evaluate_colors
// (:56-67) and the per-row tile rectangle / count of build_tiles
// (splat/tiles.py:45-50).  One thread per Gaussian, fp64 arithmetic in the
// reference's operation order; reads 56 B (+36 B SH1) of fp32 parameters
// (every load issued up front) and writes the 80 B blend record, the 48 B
// fp32 cull record, the 8 B rectangle, the 4 B count and the 8 B depth key
// per row, and adds the rectangle into a 2D tile difference grid.  Rows
// culled before projection (near / far / opacity) or by a conservative
// screen bound on the reference's radius exit before the covariance.
#include "common.cuh"

namespace hgs {

struct CamConst {
  double fx, fy, cx, cy, W, H, R[9], T[3], near_, far_, center[3], limx, limy;
};

__device__ __forceinline__ void load_cam(const hgs_camera* __restrict__ cam, CamConst& c) {
  c.fx = cam->fx; c.fy = cam->fy; c.cx = cam->cx; c.cy = cam->cy;
  c.W = (double)cam->width; c.H = (double)cam->height;
#pragma unroll
  for (int k = 0; k < 9; k++) c.R[k] = cam->R[k];
#pragma unroll
  for (int k = 0; k < 3; k++) { c.T[k] = cam->T[k]; c.center[k] = cam->center[k]; }
  c.near_ = cam->near_; c.far_ = cam->far_; c.limx = cam->limx; c.limy = cam->limy;
}

// quaternions_to_rotations (scene.py:126-141)
__device__ __forceinline__ void quat_to_rot(double q0, double q1, double q2, double q3, double* Rq) {
  double nrm = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
  double w = q0 / nrm, x = q1 / nrm, y = q2 / nrm, z = q3 / nrm;
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

#ifndef HGS_PP_MINB
#define HGS_PP_MINB 3
#endif
__global__ void __launch_bounds__(256, HGS_PP_MINB) preprocess_kernel(const hgs_camera* __restrict__ cam_ptr, hgs_gaussians gs,
                                                         int tile_px, int tiles_x, int tiles_y, hgs_projected out) {
  pdl_enter();  // releases the binning chain's PDL launches early
  __shared__ CamConst cs;
  if (threadIdx.x == 0) load_cam(cam_ptr, cs);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= gs.n) return;
  const CamConst& c = cs;

  const double c0 = gs.centers[3 * i], c1 = gs.centers[3 * i + 1], c2 = gs.centers[3 * i + 2];
  // every per-Gaussian load is issued early so their latencies overlap
  const float lg = gs.logits[i];
  const float ls0 = gs.log_scales[3 * i], ls1 = gs.log_scales[3 * i + 1], ls2 = gs.log_scales[3 * i + 2];
  double t[3];
#pragma unroll
  for (int j = 0; j < 3; j++) t[j] = dot3(c0, c1, c2, c.R[j * 3], c.R[j * 3 + 1], c.R[j * 3 + 2]) + c.T[j];
  const double depth = t[2];
  bool ok = (depth > c.near_) && (depth < c.far_);
  const double alpha = 1.0 / (1.0 + exp(-(double)lg));
  ok = ok && (alpha >= SIGMA_SKIP);
  if (!ok) {
    // culled before projection (near/far/opacity, project.py:80-83): no
    // consumer reads anything but the count, the key and the empty box
    out.count[i] = 0;
    reinterpret_cast<ushort4*>(out.rect)[i] = make_ushort4(0, 0, 0, 0);
    if (out.sort_keys) out.sort_keys[i] = ~0ull;
    if (out.cull) reinterpret_cast<CullRec*>(out.cull)[i].box = make_float4(0.f, 0.f, -1.0f, -1.0f);
    return;
  }
  const float q0 = gs.rotations[4 * i], q1 = gs.rotations[4 * i + 1], q2 = gs.rotations[4 * i + 2],
              q3 = gs.rotations[4 * i + 3];
  const float dc0 = gs.colors_dc[3 * i], dc1 = gs.colors_dc[3 * i + 1], dc2 = gs.colors_dc[3 * i + 2];
  const double tz = ok ? depth : 1.0;
  const double mx = c.fx * t[0] / tz + c.cx;
  const double my = c.fy * t[1] / tz + c.cy;
  {
    // Conservative screen pre-cull (project.py:118-119): the reference's
    // radius 3 sqrt(lambda_max(J W Sigma W^T J^T + 0.3 I)) is at most
    // 3 sqrt(|J|_F^2 max(s)^2 + 0.3); a Gaussian whose box with that bound
    // misses the screen is culled by the reference too -- skip its covariance
    // (most rows of a training view fall here).
    const double lsm = fmax(fmax((double)ls0, (double)ls1), (double)ls2);
    const double rxc = clampd(t[0] / tz, -c.limx, c.limx), ryc = clampd(t[1] / tz, -c.limy, c.limy);
    const double jf2 = (c.fx * c.fx * (1.0 + rxc * rxc) + c.fy * c.fy * (1.0 + ryc * ryc)) / (tz * tz);
    const double r_ub = 3.0 * sqrt(jf2 * exp(2.0 * lsm) + COV_FLOOR) * (1.0 + 1e-6) + 1e-6;
    if (mx + r_ub <= 0.0 || mx - r_ub >= c.W || my + r_ub <= 0.0 || my - r_ub >= c.H) {
      out.count[i] = 0;
      reinterpret_cast<ushort4*>(out.rect)[i] = make_ushort4(0, 0, 0, 0);
      if (out.sort_keys) out.sort_keys[i] = ~0ull;
      if (out.cull) reinterpret_cast<CullRec*>(out.cull)[i].box = make_float4(0.f, 0.f, -1.0f, -1.0f);
      return;
    }
  }

  // 3D covariance: Sigma = M M^T, M = R diag(s)   (project.py:91-94)
  double Rq[9], M[9], sig[9];
  quat_to_rot(q0, q1, q2, q3, Rq);
  const double s[3] = {exp((double)ls0), exp((double)ls1), exp((double)ls2)};
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = 0; b < 3; b++) M[a * 3 + b] = Rq[a * 3 + b] * s[b];
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = 0; b < 3; b++) sig[a * 3 + b] = dot3(M[a * 3], M[a * 3 + 1], M[a * 3 + 2], M[b * 3], M[b * 3 + 1], M[b * 3 + 2]);

  // projection Jacobian at the frustum-clamped centre (project.py:97-105)
  const double rx = clampd(t[0] / tz, -c.limx, c.limx);
  const double ry = clampd(t[1] / tz, -c.limy, c.limy);
  const double J[6] = {c.fx / tz, 0.0, -c.fx * rx / tz, 0.0, c.fy / tz, -c.fy * ry / tz};
  double A[6], AS[6];
#pragma unroll
  for (int j = 0; j < 2; j++)
#pragma unroll
    for (int b = 0; b < 3; b++) A[j * 3 + b] = dot3(J[j * 3], J[j * 3 + 1], J[j * 3 + 2], c.R[b], c.R[3 + b], c.R[6 + b]);
#pragma unroll
  for (int j = 0; j < 2; j++)
#pragma unroll
    for (int b = 0; b < 3; b++) AS[j * 3 + b] = dot3(A[j * 3], A[j * 3 + 1], A[j * 3 + 2], sig[b], sig[3 + b], sig[6 + b]);
  const double cov00 = dot3(AS[0], AS[1], AS[2], A[0], A[1], A[2]);
  const double cov01 = dot3(AS[0], AS[1], AS[2], A[3], A[4], A[5]);
  const double cov11 = dot3(AS[3], AS[4], AS[5], A[3], A[4], A[5]);
  const double cxx = cov00 + COV_FLOOR, cxy = cov01, cyy = cov11 + COV_FLOOR;
  const double det = cxx * cyy - cxy * cxy;
  const double mid = 0.5 * (cxx + cyy);
  const double lam = mid + sqrt(fmax(mid * mid - det, 0.0));
  const double radius = 3.0 * sqrt(fmax(lam, 0.0));
  ok = ok && (mx + radius > 0.0) && (mx - radius < c.W);
  ok = ok && (my + radius > 0.0) && (my - radius < c.H);

  // view-dependent colour (project.py:56-67)
  double pre[3];
#pragma unroll
  for (int ch = 0; ch < 3; ch++) pre[ch] = 0.5 + SH_C0 * (double)(ch == 0 ? dc0 : (ch == 1 ? dc1 : dc2));
  double vx = 0.0, vy = 0.0, vz = 0.0, dist = 0.0;
  if (gs.colors_rest != nullptr) {
    const double d0 = c0 - c.center[0], d1 = c1 - c.center[1], d2 = c2 - c.center[2];
    dist = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
    const double den = fmax(dist, 1e-12);
    vx = d0 / den; vy = d1 / den; vz = d2 / den;
    const float* r = gs.colors_rest + 9 * i;
#pragma unroll
    for (int ch = 0; ch < 3; ch++)
      pre[ch] = pre[ch] + SH_C1 * ((-vy * (double)r[ch] + vz * (double)r[3 + ch]) - vx * (double)r[6 + ch]);
  }
  const double inv_det = 1.0 / det;

  BlendRec rec;
  rec.mx = mx; rec.my = my;
  rec.ca = cyy * inv_det; rec.cb2 = 2.0 * (-cxy * inv_det); rec.cc = cxx * inv_det;
  rec.alpha = alpha; rec.depth = depth;
  rec.r = fmax(pre[0], 0.0); rec.g = fmax(pre[1], 0.0); rec.b = fmax(pre[2], 0.0);
  reinterpret_cast<BlendRec*>(out.rec)[i] = rec;

  // tile rectangle and count (tiles.py:45-50)
  int cnt = 0;
  ushort4 rc = make_ushort4(0, 0, 0, 0);
  if (ok) {
    const double tp = (double)tile_px;
    const double x0 = clampd(floor((mx - radius) / tp), 0.0, (double)(tiles_x - 1));
    const double x1 = clampd(floor((mx + radius) / tp), 0.0, (double)(tiles_x - 1));
    const double y0 = clampd(floor((my - radius) / tp), 0.0, (double)(tiles_y - 1));
    const double y1 = clampd(floor((my + radius) / tp), 0.0, (double)(tiles_y - 1));
    rc = make_ushort4((unsigned short)x0, (unsigned short)x1, (unsigned short)y0, (unsigned short)y1);
    cnt = ((int)x1 - (int)x0 + 1) * ((int)y1 - (int)y0 + 1);
  }
  out.count[i] = cnt;
  reinterpret_cast<ushort4*>(out.rect)[i] = rc;
  if (out.sort_keys) out.sort_keys[i] = ok ? (uint64_t)__double_as_longlong(depth) : ~0ull;
  if (out.tile_diff && ok) {  // rectangle into the 2D difference grid (tiles.py:45-50 counts per tile)
    // TILE_DIFF_COPIES privatised copies spread the atomics over more L2 addresses
    const int gw = tiles_x + 1;
    int* grid = out.tile_diff + (size_t)(blockIdx.x % TILE_DIFF_COPIES) * (size_t)gw * (size_t)(tiles_y + 1);
    atomicAdd(&grid[rc.z * gw + rc.x], 1);
    atomicAdd(&grid[rc.z * gw + rc.y + 1], -1);
    atomicAdd(&grid[(rc.w + 1) * gw + rc.x], -1);
    atomicAdd(&grid[(rc.w + 1) * gw + rc.y + 1], 1);
  }

  if (out.cull) {
    // Where can this Gaussian blend at all?  sigma = alpha exp(-m/2) >= 1/255
    // needs m <= 2 ln(255 alpha) on top of the support m <= 9 (kernels.py:
    // 45-51): the per-warp cull of the blend kernels uses that effective
    // ellipse m <= mcut (margin 1e-4 relative; the tile rectangles stay the
    // reference's 3-sigma ones).  Box = its conservative extents
    // (|dx| <= sqrt(mcut cov_xx)), inflated for the fp32 compare.
    const double mcut = fmin(SUPPORT_MAHAL2, 2.0 * log(alpha / SIGMA_SKIP)) * (1.0 + 1e-4) + 1e-6;
    const float slack = 1e-3f + 2.5e-7f * (float)(fabs(mx) + fabs(my));
    const float ex = (float)sqrt(mcut * cxx) * (1.0f + 1e-5f) + slack;
    const float ey = (float)sqrt(mcut * cyy) * (1.0f + 1e-5f) + slack;
    // the blend fast path evaluates the conic form with FMAs; its distance
    // from the reference's rounding is bounded by the conditioning
    // 1 / (1 - rho^2) of the conic -- past 1e6 the entry is always
    // evaluated in the reference's operation order (sign of alpha)
    const double one_m_rho2 = det / (cxx * cyy);
    const float a32 = (float)alpha;
    CullRec cr;
    cr.box = make_float4((float)mx, (float)my, ok ? ex : -1.0f, ok ? ey : -1.0f);
    cr.con = make_float4((float)(cyy * inv_det), (float)(-cxy * inv_det), (float)(cxx * inv_det), (float)depth);
    cr.col = make_float4(one_m_rho2 > 1e-6 ? a32 : -a32, (float)rec.r, (float)rec.g, (float)rec.b);
    reinterpret_cast<CullRec*>(out.cull)[i] = cr;
  }
  if (out.cov2d) { out.cov2d[3 * i] = cxx; out.cov2d[3 * i + 1] = cxy; out.cov2d[3 * i + 2] = cyy; }
  if (out.radius) out.radius[i] = radius;
  if (out.t_cam) { out.t_cam[3 * i] = t[0]; out.t_cam[3 * i + 1] = t[1]; out.t_cam[3 * i + 2] = t[2]; }
  if (out.color_pre) { out.color_pre[3 * i] = pre[0]; out.color_pre[3 * i + 1] = pre[1]; out.color_pre[3 * i + 2] = pre[2]; }
  if (out.view_dir && gs.colors_rest) { out.view_dir[3 * i] = vx; out.view_dir[3 * i + 1] = vy; out.view_dir[3 * i + 2] = vz; }
  if (out.view_dist && gs.colors_rest) out.view_dist[i] = dist;
}

}  // namespace hgs

extern "C" int hgs_preprocess(const hgs_camera* cam, int32_t width, int32_t height, const hgs_gaussians* gs,
                              int32_t tile_px, hgs_projected* out, void* stream) {
  if (!cam || !gs || !out) return hgs_set_error(HGS_ERR_INVALID, "hgs_preprocess: null argument");
  if (gs->n < 0) return hgs_set_error(HGS_ERR_INVALID, "hgs_preprocess: negative n");
  if (tile_px <= 0 || width <= 0 || height <= 0)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_preprocess: tile_px/width/height must be positive");
  const int tx0 = (width + tile_px - 1) / tile_px, ty0 = (height + tile_px - 1) / tile_px;
  if (gs->n == 0) {
    if (out->tile_diff)
      cudaMemsetAsync(out->tile_diff, 0, sizeof(int32_t) * hgs::TILE_DIFF_COPIES * (size_t)(tx0 + 1) * (size_t)(ty0 + 1),
                      (cudaStream_t)stream);
    return HGS_OK;
  }
  if (!gs->centers || !gs->rotations || !gs->log_scales || !gs->logits || !gs->colors_dc || !out->rec ||
      !out->count || !out->rect)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_preprocess: missing parameter/output pointer");
  const int tiles_x = (width + tile_px - 1) / tile_px, tiles_y = (height + tile_px - 1) / tile_px;
  if (tiles_x > 65535 || tiles_y > 65535) return hgs_set_error(HGS_ERR_INVALID, "hgs_preprocess: tile grid too large");
  if (out->tile_diff)
    cudaMemsetAsync(out->tile_diff, 0,
                    sizeof(int32_t) * hgs::TILE_DIFF_COPIES * (size_t)(tiles_x + 1) * (size_t)(tiles_y + 1),
                    (cudaStream_t)stream);
  hgs::preprocess_kernel<<<hgs::ceil_div(gs->n, 256), 256, 0, (cudaStream_t)stream>>>(cam, *gs, tile_px, tiles_x,
                                                                                       tiles_y, *out);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}
