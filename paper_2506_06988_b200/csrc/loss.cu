// Training losses with analytic gradients (gsmesh/train/losses.py):
// transmittance_mask (:79-91), L1 (:41-44), SSIM / D-SSIM (:47-76, 11-tap
// sigma 1.5 zero-padded separable filter, scipy convolve1d along H then W),
// texture loss (:103-116) and the composite schedule (:139-174).  All
// reductions stay on the device (fp64 atomics); the SSIM filter arithmetic is
// fp64 (B200 issues fp64 FMA at half the fp32 rate), the per-pixel SSIM
// derivative maps handed from the forward to the backward tile are fp32.
// Images are (H, W, 3) fp32 row-major.
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

// scalars: l1, dssim, l_c, l_t, total, mean_T_on_mesh (acc: 0 sum|d|, 1 n_cov,
// 2 sum(mask sq), 3 sum T cov, 6 sum s)
__device__ void loss_scalars(const double* __restrict__ acc, int64_t n, double lam, int tex_active, double tex_w,
                             int has_mesh, double* __restrict__ scalars) {
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


// The tile partials of the forward kernel (part[q][tile], q: |d|, n_cov,
// mask sq, T cov, s) summed in a fixed order -- per thread over tiles
// t, t + 256, ..., then a fixed tree -- and the loss scalars (one CTA).
__global__ void __launch_bounds__(256) loss_reduce_kernel(const double* __restrict__ part, int tiles,
                                                          double* __restrict__ acc, int64_t n, double lam,
                                                          int tex_active, double tex_w, int has_mesh,
                                                          double* __restrict__ scalars) {
  __shared__ double red[256];
  for (int q = 0; q < 5; q++) {
    double x = 0.0;
    for (int t = threadIdx.x; t < tiles; t += 256) x += part[(size_t)q * tiles + t];
    red[threadIdx.x] = x;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) acc[q == 4 ? 6 : q] = red[0];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss_scalars(acc, n, lam, tex_active, tex_w, has_mesh, scalars);
}

// ---- fused SSIM tiles ------------------------------------------------------
// One CTA (256 threads) per 16x16 output tile, all three channels.  The tile
// plus a 5-pixel halo of the inputs is staged once in shared memory with
// coalesced loads of the interleaved RGB rows (zeros outside the image = the
// reference's zero padding: an fma with a zero operand leaves the sum
// exactly unchanged, so no tap needs a bounds test).  The separable filter
// is register-blocked: in the H pass a thread slides down one halo column
// producing 5-6 outputs (each input row is read, squared and multiplied
// once, not once per tap); in the W pass a thread slides along one row
// producing 3-4 outputs.  Every output is still the taps k = -5..5 summed in
// order with fma (the reference's convolve1d order, 1 ulp per tap).  Shared
// rows of the H-filtered maps are padded to 27 doubles so the W pass (lanes
// = rows) is bank-conflict free.
constexpr int SS_T = 16, SS_H = SS_T + 10, SS_P = SS_H + 1;

struct SsimFwdSmem {
  union {
    float in[2][3][SS_H][SS_H];      // [render, target][channel][row][col]
    float dout[3][SS_T][SS_T * 3];   // staged derivative maps [map][row][px*3+ch]
  };
  double v[3][5][SS_T][SS_P];        // H-filtered (x, y, xx, yy, xy) [ch][q][row][col]
};

// Stage NA interleaved-RGB (or derivative-map) sources over the halo'd tile:
// all of a thread's loads are issued before its shared stores (8 in flight
// per source), rows are contiguous 78-float runs of global memory.
template <int NA>
__device__ __forceinline__ void ssim_stage(float (*dst)[3][SS_H][SS_H], const float* __restrict__ s0,
                                           const float* __restrict__ s1, const float* __restrict__ s2, int x0, int y0,
                                           int h, int w) {
  constexpr int E = SS_H * SS_H * 3, IT = (E + 255) / 256;
  const float* src[3] = {s0, s1, s2};
  float v[NA][IT];
#pragma unroll
  for (int j = 0; j < IT; j++) {
    const int i = threadIdx.x + 256 * j;
    const int r = i / (SS_H * 3), k = i - r * (SS_H * 3);
    const int gx = x0 + k / 3, gy = y0 + r;
    const bool ok = i < E && gx >= 0 && gx < w && gy >= 0 && gy < h;
    const int64_t jj = ok ? ((int64_t)gy * w + x0) * 3 + k : 0;
#pragma unroll
    for (int q = 0; q < NA; q++) v[q][j] = ok ? __ldg(src[q] + jj) : 0.f;
  }
#pragma unroll
  for (int j = 0; j < IT; j++) {
    const int i = threadIdx.x + 256 * j;
    if (i < E) {
      const int r = i / (SS_H * 3), k = i - r * (SS_H * 3);
      const int cc = k / 3, ch = k - cc * 3;
#pragma unroll
      for (int q = 0; q < NA; q++) dst[q][ch][r][cc] = v[q][j];
    }
  }
}

// SSIM terms (losses.py:57-66) -> derivative maps d (fp32, 3 planes of n),
// sum(s) -> acc[6]; plus the L1 / coverage / texture sums over the tile's
// pixels (acc[0..3]).
__global__ void __launch_bounds__(256, 3) ssim_fwd_tile_kernel(const float* __restrict__ gt,
                                                               const float* __restrict__ ih,
                                                               const float* __restrict__ im,
                                                               const int32_t* __restrict__ tri,
                                                               const float* __restrict__ t, int h, int w, LossWin win,
                                                               double mask_k, int variant, int tex_active,
                                                               float* __restrict__ d, double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char ssf_raw[];
  SsimFwdSmem& sm = *reinterpret_cast<SsimFwdSmem*>(ssf_raw);
  const int x0 = blockIdx.x * SS_T - 5, y0 = blockIdx.y * SS_T - 5;
  const int64_t n = (int64_t)h * w * 3;
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  // this thread's pixel for the L1 / coverage / texture sums: its loads are
  // in flight during the staging
  const int pr = threadIdx.x / SS_T, pc = threadIdx.x % SS_T;  // 256 threads = the tile's pixels
  const int pgx = x0 + 5 + pc, pgy = y0 + 5 + pr;
  const bool pin = pgx < w && pgy < h;
  const int64_t p = pin ? (int64_t)pgy * w + pgx : 0;
  const bool pcov = pin && tri && tri[p] >= 0;
  const float pt = pcov ? t[p] : 0.f;
  float pim[3] = {0.f, 0.f, 0.f};
  if (pcov && tex_active)
    for (int ch = 0; ch < 3; ch++) pim[ch] = im[3 * p + ch];
  ssim_stage<2>(sm.in, ih, gt, nullptr, x0, y0, h, w);
  __syncthreads();
  double v4[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (pin) {
    for (int ch = 0; ch < 3; ch++)
      v4[0] += fabs((double)sm.in[0][ch][pr + 5][pc + 5] - (double)sm.in[1][ch][pr + 5][pc + 5]);
    if (pcov) {
      v4[1] = 1.0;
      v4[3] = pt;
      if (tex_active) {
        double sq = 0.0;
        for (int ch = 0; ch < 3; ch++) {
          const double dd = (double)pim[ch] - (double)sm.in[1][ch][pr + 5][pc + 5];
          sq += dd * dd;
        }
        v4[2] = mask_val((double)pt, mask_k, variant) * sq;
      }
    }
  }
  // H pass: item = (halo column, channel, row group of 5/5/6 output rows)
  if (threadIdx.x < SS_H * 3 * 3) {
    const int c = threadIdx.x % SS_H, rest = threadIdx.x / SS_H;
    const int ch = rest % 3, g = rest / 3;
    const int r0 = g * 5, nr = g == 2 ? 6 : 5;
    double q[6][5];
#pragma unroll
    for (int o = 0; o < 6; o++)
#pragma unroll
      for (int k = 0; k < 5; k++) q[o][k] = 0.0;
#pragma unroll
    for (int ii = 0; ii < 16; ii++) {
      if (ii < nr + 10) {
        const double a = sm.in[0][ch][r0 + ii][c], b = sm.in[1][ch][r0 + ii][c];
        const double f[5] = {a, b, a * a, b * b, a * b};
#pragma unroll
        for (int o = 0; o < 6; o++) {
          const int k = ii - o;
          if (k >= 0 && k <= 10) {
            const double wk = win.w[k];
#pragma unroll
            for (int m = 0; m < 5; m++) q[o][m] = fma(f[m], wk, q[o][m]);
          }
        }
      }
    }
#pragma unroll
    for (int o = 0; o < 6; o++)
      if (o < nr)
#pragma unroll
        for (int m = 0; m < 5; m++) sm.v[ch][m][r0 + o][c] = q[o][m];
  }
  __syncthreads();
  // W pass + SSIM terms: item = (row, channel, column group of 3/3/3/3/4)
  double ssum = 0.0;
  if (threadIdx.x < SS_T * 3 * 5) {
    const int r = threadIdx.x % SS_T, rest = threadIdx.x / SS_T;
    const int ch = rest % 3, g = rest / 3;
    const int c0 = g * 3, nc = g == 4 ? 4 : 3;
    double u[4][5];
#pragma unroll
    for (int o = 0; o < 4; o++)
#pragma unroll
      for (int k = 0; k < 5; k++) u[o][k] = 0.0;
#pragma unroll
    for (int ii = 0; ii < 14; ii++) {
      if (ii < nc + 10) {
        double f[5];
#pragma unroll
        for (int m = 0; m < 5; m++) f[m] = sm.v[ch][m][r][c0 + ii];
#pragma unroll
        for (int o = 0; o < 4; o++) {
          const int k = ii - o;
          if (k >= 0 && k <= 10) {
            const double wk = win.w[k];
#pragma unroll
            for (int m = 0; m < 5; m++) u[o][m] = fma(f[m], wk, u[o][m]);
          }
        }
      }
    }
    const int gy = y0 + 5 + r;
#pragma unroll
    for (int o = 0; o < 4; o++) {
      const int gx = x0 + 5 + c0 + o;
      if (o < nc && gx < w && gy < h) {
        const double ux = u[o][0], uy = u[o][1], vx = u[o][2], vy = u[o][3], vxy = u[o][4];
        const double a1 = 2 * ux * uy + C1;
        const double a2 = 2 * (vxy - ux * uy) + C2;
        const double b1 = ux * ux + uy * uy + C1;
        const double b2 = (vx - ux * ux) + (vy - uy * uy) + C2;
        // two fp64 reciprocals instead of six divisions (1/qq = 1/b1 1/b2):
        // a few ulp of fp64 from the reference's quotients
        const double rb1 = 1.0 / b1, rb2 = 1.0 / b2;
        const double rq = rb1 * rb2;
        const double sv = (a1 * a2) * rq;
        const int k = (c0 + o) * 3 + ch;
        sm.dout[0][r][k] = (float)(2 * uy * (a2 - a1) * rq - 2 * ux * sv * rb1 + 2 * ux * sv * rb2);
        sm.dout[1][r][k] = (float)(-sv * rb2);
        sm.dout[2][r][k] = (float)(2 * a1 * rq);
        ssum += sv;
      }
    }
  }
  __syncthreads();
  // coalesced write of the derivative maps (48 contiguous floats per row)
  for (int i = threadIdx.x; i < 3 * SS_T * SS_T * 3; i += blockDim.x) {
    const int m = i / (SS_T * SS_T * 3), rest = i - m * (SS_T * SS_T * 3);
    const int r = rest / (SS_T * 3), k = rest - r * (SS_T * 3);
    const int gy = y0 + 5 + r, gx = x0 + 5 + k / 3;
    if (gx < w && gy < h) d[m * n + ((int64_t)gy * w + x0 + 5) * 3 + k] = sm.dout[m][r][k];
  }
  v4[4] = ssum;
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
    // per-tile partials, summed in tile order by loss_reduce_kernel (run-to-run deterministic)
    part[(size_t)threadIdx.x * gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = x;
  }
}

struct SsimBwdSmem {
  union {
    float in[3][3][SS_H][SS_H];      // derivative maps [map][ch][row][col]
    double f[9][SS_T][SS_T + 1];     // filtered [map*3+ch][row][col]
  };
  double v[9][SS_T][SS_P];           // H-filtered [map*3+ch][row][col]
};

// Adjoint filter of the d maps (the window is symmetric) and the loss
// gradients (losses.py:41-76, 103-116): grad_ih = (1-lam) sign(d)/n +
// lam (-0.5) (f1 + 2x f2 + y f3)/n, grad_im = tex_w (2/ncov) mask diff,
// grad_t = tex_w mask' sq / ncov.
__global__ void __launch_bounds__(256, 3) ssim_bwd_tile_kernel(const float* __restrict__ gt,
                                                               const float* __restrict__ ih,
                                                               const float* __restrict__ im,
                                                               const int32_t* __restrict__ tri,
                                                               const float* __restrict__ t, int h, int w, LossWin win,
                                                               const float* __restrict__ d,
                                                               const double* __restrict__ acc, double lam,
                                                               int tex_active, double tex_w, double mask_k,
                                                               int variant, double scale, float* __restrict__ g_ih,
                                                               float* __restrict__ g_im, float* __restrict__ g_t) {
  extern __shared__ __align__(16) unsigned char ssb_raw[];
  SsimBwdSmem& sm = *reinterpret_cast<SsimBwdSmem*>(ssb_raw);
  const int x0 = blockIdx.x * SS_T - 5, y0 = blockIdx.y * SS_T - 5;
  const int64_t n = (int64_t)h * w * 3;
  const int r = threadIdx.x / SS_T, c = threadIdx.x % SS_T;  // output pixel of this thread
  const int gx = x0 + 5 + c, gy = y0 + 5 + r;
  const bool pin = gx < w && gy < h;
  const int64_t p = pin ? (int64_t)gy * w + gx : 0;
  // this pixel's inputs: in flight during the staging and the filter passes
  float px_[3] = {0.f, 0.f, 0.f}, py_[3] = {0.f, 0.f, 0.f}, pim[3] = {0.f, 0.f, 0.f};
  const bool cov = pin && tri && tri[p] >= 0;
  const float pt = (pin && tex_active && cov) ? t[p] : 0.f;
  if (pin)
    for (int ch = 0; ch < 3; ch++) {
      px_[ch] = ih[3 * p + ch];
      py_[ch] = gt[3 * p + ch];
      if (g_im && cov) pim[ch] = im[3 * p + ch];
    }
  ssim_stage<3>(sm.in, d, d + n, d + 2 * n, x0, y0, h, w);
  __syncthreads();
  // H pass: item = (halo column, map x channel), the whole 16-row strip
  if (threadIdx.x < SS_H * 9) {
    const int c = threadIdx.x % SS_H, mc = threadIdx.x / SS_H;
    double q[SS_T];
#pragma unroll
    for (int o = 0; o < SS_T; o++) q[o] = 0.0;
#pragma unroll
    for (int ii = 0; ii < SS_H; ii++) {
      const double a = sm.in[mc / 3][mc % 3][ii][c];
#pragma unroll
      for (int o = 0; o < SS_T; o++) {
        const int k = ii - o;
        if (k >= 0 && k <= 10) q[o] = fma(a, win.w[k], q[o]);
      }
    }
#pragma unroll
    for (int o = 0; o < SS_T; o++) sm.v[mc][o][c] = q[o];
  }
  __syncthreads();
  // W pass: item = (row, map x channel, half row of 8 outputs)
  for (int it = threadIdx.x; it < SS_T * 9 * 2; it += blockDim.x) {
    const int r = it % SS_T, rest = it / SS_T;
    const int mc = rest % 9, c0 = (rest / 9) * 8;
    double u[8];
#pragma unroll
    for (int o = 0; o < 8; o++) u[o] = 0.0;
#pragma unroll
    for (int ii = 0; ii < 18; ii++) {
      const double a = sm.v[mc][r][c0 + ii];
#pragma unroll
      for (int o = 0; o < 8; o++) {
        const int k = ii - o;
        if (k >= 0 && k <= 10) u[o] = fma(a, win.w[k], u[o]);
      }
    }
#pragma unroll
    for (int o = 0; o < 8; o++) sm.f[mc][r][c0 + o] = u[o];
  }
  __syncthreads();
  if (!pin) return;
  const double ncov = acc[1];
  const double mk = (tex_active && cov) ? mask_val((double)pt, mask_k, variant) : 0.0;
  double sq = 0.0;
#pragma unroll
  for (int ch = 0; ch < 3; ch++) {
    const int64_t i = 3 * p + ch;
    const double x = px_[ch], y = py_[ch];
    const double dd = x - y;
    const double gl1 = (dd > 0 ? 1.0 : (dd < 0 ? -1.0 : 0.0)) / (double)n;
    const double gss = (sm.f[ch][r][c] + 2 * x * sm.f[3 + ch][r][c] + y * sm.f[6 + ch][r][c]) / (double)n;
    g_ih[i] = (float)(scale * ((1.0 - lam) * gl1 + lam * (-0.5 * gss)));
    if (g_im) {
      const double dm = cov ? (double)pim[ch] - y : 0.0;
      sq += dm * dm;
      g_im[i] = (float)(scale * ((tex_active && ncov > 0) ? tex_w * ((2.0 / ncov) * mk * dm) : 0.0));
    }
  }
  if (g_t) {
    double gtv = 0.0;
    if (tex_active && cov && ncov > 0) gtv = tex_w * (mask_der((double)pt, mask_k, variant) * sq / ncov);
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
  const size_t tiles = (size_t)((width + hgs::SS_T - 1) / hgs::SS_T) * (size_t)((height + hgs::SS_T - 1) / hgs::SS_T);
  return hgs::align_up(4 * 3 * n, 256) + 256 + 5 * 8 * tiles;
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
  float* dmaps = (float*)base;  // 3 x n SSIM derivative maps
  base += align_up(4 * 3 * n, 256);
  double* acc = (double*)base;  // 8 doubles
  double* part = acc + 32;      // 5 x tiles per-tile partial sums
  LossWin win;
  for (int k = 0; k < 11; k++) win.w[k] = window11_host[k];
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ssim_fwd_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SsimFwdSmem));
    cudaFuncSetAttribute(ssim_bwd_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SsimBwdSmem));
    attr = true;
  }
  const dim3 tg((width + SS_T - 1) / SS_T, (height + SS_T - 1) / SS_T);
  ssim_fwd_tile_kernel<<<tg, 256, sizeof(SsimFwdSmem), st>>>(i_gt, i_h, i_m, triangle_id, t, height, width, win,
                                                             mask_k, mask_variant, texture_active, dmaps, part);
  HGS_CHECK_LAUNCH();
  loss_reduce_kernel<<<1, 256, 0, st>>>(part, (int)(tg.x * tg.y), acc, n, lam_dssim, texture_active, texture_weight,
                                        triangle_id != nullptr, scalars);
  HGS_CHECK_LAUNCH();
  ssim_bwd_tile_kernel<<<tg, 256, sizeof(SsimBwdSmem), st>>>(i_gt, i_h, i_m, triangle_id, t, height, width, win, dmaps,
                                                             acc, lam_dssim, texture_active, texture_weight, mask_k,
                                                             mask_variant, grad_scale, grad_ih, grad_im, grad_t);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}
