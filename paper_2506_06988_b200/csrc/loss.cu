// Training losses with analytic gradients (gsmesh/train/losses.py):
// transmittance_mask (:79-91), L1 (:41-44), SSIM / D-SSIM (:47-76, 11-tap
// sigma 1.5 zero-padded separable filter, scipy convolve1d along H then W),
// texture loss (:103-116) and the composite schedule (:139-174).  All
// reductions stay on the device (fp64 atomics); intermediate SSIM maps are
// fp64.  Images are (H, W, 3) fp32 row-major.
#include "common.cuh"

namespace hgs {

struct LossWin {
  double w[11];
};

__device__ __forceinline__ double mask_val(double t, double k, int variant) {
  switch (variant) {
    case 0: return 1.0 / (1.0 + exp(-k * (t - 0.5)));
    case 1: return t;
    case 2: return 1.0;
    default: return 0.0;
  }
}
__device__ __forceinline__ double mask_der(double t, double k, int variant) {
  if (variant == 0) {
    const double m = 1.0 / (1.0 + exp(-k * (t - 0.5)));
    return k * m * (1.0 - m);
  }
  return variant == 1 ? 1.0 : 0.0;
}

__global__ void mask_kernel(const float* __restrict__ t, int64_t n, double k, int variant, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (float)mask_val((double)t[i], k, variant);
}

template <int NV>
__device__ __forceinline__ void block_sum_atomic(double (&v)[NV], double* dst) {
  __shared__ double s[NV][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < NV; c++) {
    double x = v[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) s[c][warp] = x;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double x = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) x += s[threadIdx.x][w];
    atomicAdd(&dst[threadIdx.x], x);
  }
}

// Separable 11-tap zero-padded filter of NQ quantities along H (pass 0) or W
// (pass 1).  Pass 0 inputs are built from x, y (q = x, y, x*x, y*y, x*y) when
// from_images, else read from `in` (NQ fp64 maps).
template <int NQ, bool FROM_IMAGES>
__global__ void __launch_bounds__(256) ssim_filter_kernel(const float* __restrict__ x, const float* __restrict__ y,
                                                          const double* __restrict__ in, double* __restrict__ out,
                                                          int h, int w, int axis, LossWin win) {
  const int64_t n = (int64_t)h * w * 3;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int ch = (int)(i % 3);
  const int64_t pix = i / 3;
  const int px = (int)(pix % w), py = (int)(pix / w);
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; q++) acc[q] = 0.0;
  for (int k = -5; k <= 5; k++) {
    const int yy = axis == 0 ? py + k : py, xx = axis == 0 ? px : px + k;
    if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
    const int64_t j = ((int64_t)yy * w + xx) * 3 + ch;
    const double wk = win.w[k + 5];
    if (FROM_IMAGES) {
      const double a = x[j], b = y[j];
      acc[0] += a * wk;
      acc[1] += b * wk;
      acc[2] += (a * a) * wk;
      acc[3] += (b * b) * wk;
      acc[4] += (a * b) * wk;
    } else {
#pragma unroll
      for (int q = 0; q < NQ; q++) acc[q] += in[(size_t)q * n + j] * wk;
    }
  }
#pragma unroll
  for (int q = 0; q < NQ; q++) out[(size_t)q * n + i] = acc[q];
}

// per-element SSIM terms (losses.py:57-66) -> ds_dux, ds_dvx, ds_dvxy maps and
// sum(s); scalars[6] += sum(s)
__global__ void __launch_bounds__(256) ssim_terms_kernel(const double* __restrict__ u, double* __restrict__ d,
                                                         int64_t n, double* __restrict__ acc) {
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v[1] = {0.0};
  if (i < n) {
    const double ux = u[i], uy = u[n + i], vx = u[2 * n + i], vy = u[3 * n + i], vxy = u[4 * n + i];
    const double a1 = 2 * ux * uy + C1;
    const double a2 = 2 * (vxy - ux * uy) + C2;
    const double b1 = ux * ux + uy * uy + C1;
    const double b2 = (vx - ux * ux) + (vy - uy * uy) + C2;
    const double q = b1 * b2;
    const double s = (a1 * a2) / q;
    d[i] = 2 * uy * (a2 - a1) / q - 2 * ux * s / b1 + 2 * ux * s / b2;
    d[n + i] = -s / b2;
    d[2 * n + i] = 2 * a1 / q;
    v[0] = s;
  }
  block_sum_atomic<1>(v, acc);
}

// L1 + texture-loss sums: acc[0] sum|d|, acc[1] covered count, acc[2]
// sum(mask * sq) over covered, acc[3] sum T over covered
__global__ void __launch_bounds__(256) loss_sums_kernel(const float* __restrict__ gt, const float* __restrict__ ih,
                                                        const float* __restrict__ im, const int32_t* __restrict__ tri,
                                                        const float* __restrict__ t, int64_t npix, double mask_k,
                                                        int variant, int tex_active, double* __restrict__ acc) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  if (p < npix) {
    for (int c = 0; c < 3; c++) v[0] += fabs((double)ih[3 * p + c] - (double)gt[3 * p + c]);
    if (tri && tri[p] >= 0) {
      v[1] = 1.0;
      v[3] = t[p];
      if (tex_active) {
        double sq = 0.0;
        for (int c = 0; c < 3; c++) {
          const double dd = (double)im[3 * p + c] - (double)gt[3 * p + c];
          sq += dd * dd;
        }
        v[2] = mask_val((double)t[p], mask_k, variant) * sq;
      }
    }
  }
  block_sum_atomic<4>(v, acc);
}

// scalars: l1, dssim, l_c, l_t, total, mean_T_on_mesh (acc: 0 sum|d|, 1 n_cov,
// 2 sum(mask sq), 3 sum T cov, 6 sum s)
__global__ void loss_scalars_kernel(const double* __restrict__ acc, int64_t n, double lam, int tex_active,
                                    double tex_w, int has_mesh, double* __restrict__ scalars) {
  const double l1 = acc[0] / (double)n;
  const double ssim = acc[6] / (double)n;
  const double ds = (1.0 - ssim) / 2.0;
  const double l_c = (1.0 - lam) * l1 + lam * ds;
  const double ncov = acc[1];
  const double l_t = (tex_active && ncov > 0) ? acc[2] / ncov : 0.0;
  scalars[0] = l1;
  scalars[1] = ds;
  scalars[2] = l_c;
  scalars[3] = l_t;
  scalars[4] = tex_active ? l_c + tex_w * l_t : l_c;
  scalars[5] = (has_mesh && ncov > 0) ? acc[3] / ncov : __longlong_as_double(0x7ff8000000000000LL);
}

// gradients: grad_ih = (1-lam) sign(d)/n + lam * (-0.5) * (f1 + 2x f2 + y f3)/n,
// grad_im = tex_w (2/ncov) mask diff, grad_t = tex_w mask' sq / ncov
__global__ void __launch_bounds__(256) loss_grads_kernel(const float* __restrict__ gt, const float* __restrict__ ih,
                                                         const float* __restrict__ im, const int32_t* __restrict__ tri,
                                                         const float* __restrict__ t, const double* __restrict__ f,
                                                         const double* __restrict__ acc, int64_t npix, double lam,
                                                         int tex_active, double tex_w, double mask_k, int variant,
                                                         double scale, float* __restrict__ g_ih,
                                                         float* __restrict__ g_im, float* __restrict__ g_t) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npix) return;
  const int64_t n = npix * 3;
  const double ncov = acc[1];
  const bool cov = tri && tri[p] >= 0;
  const double mk = (tex_active && cov) ? mask_val((double)t[p], mask_k, variant) : 0.0;
  double sq = 0.0;
  for (int c = 0; c < 3; c++) {
    const int64_t i = 3 * p + c;
    const double x = ih[i], y = gt[i];
    const double d = x - y;
    const double gl1 = (d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0)) / (double)n;
    const double gss = (f[i] + 2 * x * f[n + i] + y * f[2 * n + i]) / (double)n;
    g_ih[i] = (float)(scale * ((1.0 - lam) * gl1 + lam * (-0.5 * gss)));
    if (g_im) {
      const double dm = cov ? (double)im[i] - y : 0.0;
      sq += dm * dm;
      g_im[i] = (float)(scale * ((tex_active && ncov > 0) ? tex_w * ((2.0 / ncov) * mk * dm) : 0.0));
    }
  }
  if (g_t) {
    double gtv = 0.0;
    if (tex_active && cov && ncov > 0) gtv = tex_w * (mask_der((double)t[p], mask_k, variant) * sq / ncov);
    g_t[p] = (float)(scale * gtv);
  }
}

// ---- fused tiles ---------------------------------------------------------
// One CTA per SS_T x SS_T output tile, all three channels.  The tile plus a
// 5-pixel halo of the inputs is staged in shared memory (zeros outside the
// image = the reference's zero padding), the H pass runs over the halo
// columns into shared memory, the W pass produces the output tile: the same
// per-element arithmetic and summation order as the separate passes, with
// no fp64 map through HBM.
constexpr int SS_T = 16, SS_H = SS_T + 10;

struct SsimFwdSmem {
  float x[SS_H][SS_H];
  float y[SS_H][SS_H];
  double v[SS_T][SS_H][5];  // H-filtered quantities of one channel over the halo columns
};

// SSIM terms (losses.py:57-66) -> d maps, sum(s) -> acc[6]; plus the L1 /
// texture sums of loss_sums_kernel over the tile's pixels.  Channels one at
// a time (small shared footprint: many CTAs per SM hide the loads).
__global__ void __launch_bounds__(256) ssim_fwd_tile_kernel(const float* __restrict__ gt, const float* __restrict__ ih,
                                                            const float* __restrict__ im,
                                                            const int32_t* __restrict__ tri, const float* __restrict__ t,
                                                            int h, int w, LossWin win, double mask_k, int variant,
                                                            int tex_active, double* __restrict__ d,
                                                            double* __restrict__ acc) {
  __shared__ SsimFwdSmem sm;
  const int x0 = blockIdx.x * SS_T - 5, y0 = blockIdx.y * SS_T - 5;
  const int64_t n = (int64_t)h * w * 3;
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  double ssum = 0.0;
  for (int ch = 0; ch < 3; ch++) {
    for (int i = threadIdx.x; i < SS_H * SS_H; i += blockDim.x) {
      const int c = i % SS_H, r = i / SS_H;
      const int gx = x0 + c, gy = y0 + r;
      float a = 0.f, b = 0.f;
      if (gx >= 0 && gx < w && gy >= 0 && gy < h) {
        const int64_t j = ((int64_t)gy * w + gx) * 3 + ch;
        a = ih[j];
        b = gt[j];
      }
      sm.x[r][c] = a;
      sm.y[r][c] = b;
    }
    __syncthreads();
    // pass along H (axis 0) for the tile's rows, all halo columns
    for (int i = threadIdx.x; i < SS_T * SS_H; i += blockDim.x) {
      const int c = i % SS_H, r = i / SS_H;
      double q[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      const int gx = x0 + c;
      if (gx >= 0 && gx < w) {
        for (int k = -5; k <= 5; k++) {
          const int rr = r + 5 + k, gy = y0 + rr;
          if (gy < 0 || gy >= h) continue;  // skipped taps (zero padding)
          const double wk = win.w[k + 5];
          const double a = sm.x[rr][c], b = sm.y[rr][c];
          q[0] = fma(a, wk, q[0]);  // fused taps: within 1 ulp per tap of the reference's order
          q[1] = fma(b, wk, q[1]);
          q[2] = fma(a * a, wk, q[2]);
          q[3] = fma(b * b, wk, q[3]);
          q[4] = fma(a * b, wk, q[4]);
        }
      }
#pragma unroll
      for (int k = 0; k < 5; k++) sm.v[r][c][k] = q[k];
    }
    __syncthreads();
    // pass along W (axis 1), SSIM terms: one pixel per thread
    {
      const int c = threadIdx.x % SS_T, r = threadIdx.x / SS_T;
      const int gx = x0 + 5 + c, gy = y0 + 5 + r;
      if (gx < w && gy < h) {
        double u[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int k = -5; k <= 5; k++) {
          const int cc = c + 5 + k, gxx = x0 + cc;
          if (gxx < 0 || gxx >= w) continue;
          const double wk = win.w[k + 5];
#pragma unroll
          for (int q = 0; q < 5; q++) u[q] = fma(sm.v[r][cc][q], wk, u[q]);
        }
        const double ux = u[0], uy = u[1], vx = u[2], vy = u[3], vxy = u[4];
        const double a1 = 2 * ux * uy + C1;
        const double a2 = 2 * (vxy - ux * uy) + C2;
        const double b1 = ux * ux + uy * uy + C1;
        const double b2 = (vx - ux * ux) + (vy - uy * uy) + C2;
        const double qq = b1 * b2;
        const double sv = (a1 * a2) / qq;
        const int64_t j = ((int64_t)gy * w + gx) * 3 + ch;
        d[j] = 2 * uy * (a2 - a1) / qq - 2 * ux * sv / b1 + 2 * ux * sv / b2;
        d[n + j] = -sv / b2;
        d[2 * n + j] = 2 * a1 / qq;
        ssum += sv;
      }
    }
    __syncthreads();
  }
  // L1 / coverage / texture sums of the tile's pixels (loss_sums_kernel)
  double v4[5] = {0.0, 0.0, 0.0, 0.0, ssum};
  {
    const int r = threadIdx.x / SS_T, c = threadIdx.x % SS_T;  // 256 threads = the tile's pixels
    const int gx = x0 + 5 + c, gy = y0 + 5 + r;
    if (gx < w && gy < h) {
      const int64_t p = (int64_t)gy * w + gx;
      for (int ch = 0; ch < 3; ch++) v4[0] += fabs((double)ih[3 * p + ch] - (double)gt[3 * p + ch]);
      if (tri && tri[p] >= 0) {
        v4[1] = 1.0;
        v4[3] = t[p];
        if (tex_active) {
          double sq = 0.0;
          for (int ch = 0; ch < 3; ch++) {
            const double dd = (double)im[3 * p + ch] - (double)gt[3 * p + ch];
            sq += dd * dd;
          }
          v4[2] = mask_val((double)t[p], mask_k, variant) * sq;
        }
      }
    }
  }
  __shared__ double red[5][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 5; q++) {
    double x = v4[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[q][warp] = x;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    double x = 0.0;
    for (int k = 0; k < 8; k++) x += red[threadIdx.x][k];
    atomicAdd(&acc[threadIdx.x == 4 ? 6 : threadIdx.x], x);
  }
}

struct SsimBwdSmem {
  double d[SS_H][SS_H][3];
  double v[SS_T][SS_H][3];
};

// adjoint filter of the d maps (the window is symmetric) and the loss
// gradients of loss_grads_kernel for the tile's pixels, channel by channel
__global__ void __launch_bounds__(256) ssim_bwd_tile_kernel(const float* __restrict__ gt, const float* __restrict__ ih,
                                                            const float* __restrict__ im,
                                                            const int32_t* __restrict__ tri, const float* __restrict__ t,
                                                            int h, int w, LossWin win, const double* __restrict__ d,
                                                            const double* __restrict__ acc, double lam, int tex_active,
                                                            double tex_w, double mask_k, int variant, double scale,
                                                            float* __restrict__ g_ih, float* __restrict__ g_im,
                                                            float* __restrict__ g_t) {
  extern __shared__ __align__(16) unsigned char ss_raw[];
  SsimBwdSmem& sm = *reinterpret_cast<SsimBwdSmem*>(ss_raw);
  const int x0 = blockIdx.x * SS_T - 5, y0 = blockIdx.y * SS_T - 5;
  const int64_t n = (int64_t)h * w * 3;
  const int r = threadIdx.x / SS_T, c = threadIdx.x % SS_T;  // output pixel of this thread
  const int gx = x0 + 5 + c, gy = y0 + 5 + r;
  const bool inside = gx < w && gy < h;
  const int64_t p = inside ? (int64_t)gy * w + gx : 0;
  const double ncov = acc[1];
  const bool cov = inside && tri && tri[p] >= 0;
  const double mk = (tex_active && cov) ? mask_val((double)t[p], mask_k, variant) : 0.0;
  double sq = 0.0;
  for (int ch = 0; ch < 3; ch++) {
    for (int i = threadIdx.x; i < SS_H * SS_H; i += blockDim.x) {
      const int cc = i % SS_H, rr = i / SS_H;
      const int gxx = x0 + cc, gyy = y0 + rr;
      double a = 0.0, b = 0.0, e = 0.0;
      if (gxx >= 0 && gxx < w && gyy >= 0 && gyy < h) {
        const int64_t j = ((int64_t)gyy * w + gxx) * 3 + ch;
        a = d[j];
        b = d[n + j];
        e = d[2 * n + j];
      }
      sm.d[rr][cc][0] = a;
      sm.d[rr][cc][1] = b;
      sm.d[rr][cc][2] = e;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < SS_T * SS_H; i += blockDim.x) {
      const int cc = i % SS_H, rr = i / SS_H;
      double q[3] = {0.0, 0.0, 0.0};
      const int gxx = x0 + cc;
      if (gxx >= 0 && gxx < w) {
        for (int k = -5; k <= 5; k++) {
          const int r2 = rr + 5 + k, gyy = y0 + r2;
          if (gyy < 0 || gyy >= h) continue;
          const double wk = win.w[k + 5];
#pragma unroll
          for (int m = 0; m < 3; m++) q[m] = fma(sm.d[r2][cc][m], wk, q[m]);
        }
      }
#pragma unroll
      for (int m = 0; m < 3; m++) sm.v[rr][cc][m] = q[m];
    }
    __syncthreads();
    if (inside) {
      double f[3] = {0.0, 0.0, 0.0};
      for (int k = -5; k <= 5; k++) {
        const int cc = c + 5 + k, gxx = x0 + cc;
        if (gxx < 0 || gxx >= w) continue;
        const double wk = win.w[k + 5];
#pragma unroll
        for (int m = 0; m < 3; m++) f[m] = fma(sm.v[r][cc][m], wk, f[m]);
      }
      const int64_t i = 3 * p + ch;
      const double x = ih[i], y = gt[i];
      const double dd = x - y;
      const double gl1 = (dd > 0 ? 1.0 : (dd < 0 ? -1.0 : 0.0)) / (double)n;
      const double gss = (f[0] + 2 * x * f[1] + y * f[2]) / (double)n;
      g_ih[i] = (float)(scale * ((1.0 - lam) * gl1 + lam * (-0.5 * gss)));
      if (g_im) {
        const double dm = cov ? (double)im[i] - y : 0.0;
        sq += dm * dm;
        g_im[i] = (float)(scale * ((tex_active && ncov > 0) ? tex_w * ((2.0 / ncov) * mk * dm) : 0.0));
      }
    }
    __syncthreads();
  }
  if (inside && g_t) {
    double gtv = 0.0;
    if (tex_active && cov && ncov > 0) gtv = tex_w * (mask_der((double)t[p], mask_k, variant) * sq / ncov);
    g_t[p] = (float)(scale * gtv);
  }
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace hgs

extern "C" int hgs_transmittance_mask(const float* t, int64_t n, double k, int32_t variant, float* out, void* stream) {
  if (!t || !out) return hgs_set_error(HGS_ERR_INVALID, "hgs_transmittance_mask: null argument");
  if (variant < 0 || variant > 3) return hgs_set_error(HGS_ERR_INVALID, "unknown transmittance mask variant");
  if (n == 0) return HGS_OK;
  hgs::mask_kernel<<<hgs::ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(t, n, k, variant, out);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}

extern "C" size_t hgs_loss_scratch_bytes(int32_t height, int32_t width) {
  const size_t n = (size_t)height * width * 3;
  return hgs::align_up(8 * 5 * n, 256) * 2 + hgs::align_up(8 * 3 * n, 256) + 256;
}

extern "C" int hgs_composite_loss(const float* i_gt, const float* i_h, const float* i_m, const int32_t* triangle_id,
                                  const float* t, int32_t height, int32_t width, double lam_dssim,
                                  int32_t texture_active, double texture_weight, double mask_k, int32_t mask_variant,
                                  const double* window11_host, double grad_scale, float* grad_ih, float* grad_im,
                                  float* grad_t, double* scalars, void* scratch, size_t scratch_bytes, void* stream) {
  using namespace hgs;
  if (!i_gt || !i_h || !t || !window11_host || !grad_ih || !scalars || !scratch)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_composite_loss: null argument");
  if (height <= 0 || width <= 0) return hgs_set_error(HGS_ERR_INVALID, "hgs_composite_loss: empty image");
  if (mask_variant < 0 || mask_variant > 3) return hgs_set_error(HGS_ERR_INVALID, "unknown transmittance mask variant");
  if (texture_active && (!i_m || !triangle_id))
    return hgs_set_error(HGS_ERR_INVALID, "hgs_composite_loss: texture term needs I_m and coverage");
  if (scratch_bytes < hgs_loss_scratch_bytes(height, width))
    return hgs_set_error(HGS_ERR_INVALID, "hgs_composite_loss: scratch too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t npix = (int64_t)height * width, n = npix * 3;
  unsigned char* base = (unsigned char*)scratch;
  double* mapsA = (double*)base;  // 5 x n
  base += align_up(8 * 5 * n, 256);
  double* mapsB = (double*)base;  // 5 x n
  base += align_up(8 * 5 * n, 256);
  double* dmaps = (double*)base;  // 3 x n
  base += align_up(8 * 3 * n, 256);
  double* acc = (double*)base;  // 8 doubles
  LossWin win;
  for (int k = 0; k < 11; k++) win.w[k] = window11_host[k];
  cudaMemsetAsync(acc, 0, 8 * sizeof(double), st);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ssim_bwd_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SsimBwdSmem));
    attr = true;
  }
  const dim3 tg((width + SS_T - 1) / SS_T, (height + SS_T - 1) / SS_T);
  ssim_fwd_tile_kernel<<<tg, 256, 0, st>>>(i_gt, i_h, i_m, triangle_id, t, height, width, win, mask_k,
                                                             mask_variant, texture_active, dmaps, acc);
  HGS_CHECK_LAUNCH();
  loss_scalars_kernel<<<1, 1, 0, st>>>(acc, n, lam_dssim, texture_active, texture_weight, triangle_id != nullptr,
                                       scalars);
  HGS_CHECK_LAUNCH();
  ssim_bwd_tile_kernel<<<tg, 256, sizeof(SsimBwdSmem), st>>>(i_gt, i_h, i_m, triangle_id, t, height, width, win, dmaps,
                                                             acc, lam_dssim, texture_active, texture_weight, mask_k,
                                                             mask_variant, grad_scale, grad_ih, grad_im, grad_t);
  HGS_CHECK_LAUNCH();
  (void)mapsA;
  (void)mapsB;
  return HGS_OK;
}
