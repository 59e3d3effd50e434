// K3 textured-mesh rasterizer: rasterize_fragments (gsmesh/meshraster.py:
// 119-136) / _raster_kernel (:45-116), sample_texture (:139-166) and
// texture_backward (:169-184).
//
// The reference walks triangles in index order with a strict z test, so a
// pixel ends up owned by the lexicographic minimum of (z, triangle index)
// over the fragments that pass its edge tests.  The GPU reproduces exactly
// that without ordering, in one pass: every covered fragment lowers the
// pixel's 16-byte record {bits(z), f} to min((z, f), record) with a 128-bit
// compare-and-swap loop (positive doubles order like their bit patterns);
// then resolve: one thread per pixel recomputes the winner's barycentrics,
// depth and uv with the reference's arithmetic (fp64, no FMA).
// Work is binned by screen bounding-box area: tiny triangles one thread
// each, medium ones one warp each (lanes stride the box), large ones one
// CTA each (binned by the one-thread-per-triangle pass).
#include "common.cuh"

#include <algorithm>

namespace hgs {

constexpr int SMALL_TRI_PIXELS = 32;
constexpr int BIG_TRI_PIXELS = 4096;

struct TriSetup {
  double ax, ay, bx, by, cx, cy;  // after winding normalisation
  double e0x, e0y, e1x, e1y, e2x, e2y;
  double inv_area, za, zb, zc;
  int x0, x1, y0, y1;
  bool own0, own1, own2, flip;
};

// Per-triangle setup, meshraster.py:50-84.  Returns false if culled/empty.
__device__ __forceinline__ bool tri_setup(const double3* __restrict__ vproj, const int32_t* __restrict__ tris, int64_t f,
                                          int width, int height, double near_, TriSetup& t) {
  const int ia = tris[3 * f], ib = tris[3 * f + 1], ic = tris[3 * f + 2];
  const double3 A = vproj[ia], B = vproj[ib], C = vproj[ic];
  if (A.z <= near_ || B.z <= near_ || C.z <= near_) return false;
  double ax = A.x, ay = A.y, bx = B.x, by = B.y, cx = C.x, cy = C.y;
  double area2 = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
  if (area2 == 0.0) return false;
  const bool flip = area2 < 0.0;
  if (flip) {
    double tmp = bx; bx = cx; cx = tmp;
    tmp = by; by = cy; cy = tmp;
    area2 = -area2;
  }
  double fx0 = floor(fmin(fmin(ax, bx), cx) - 0.5), fx1 = ceil(fmax(fmax(ax, bx), cx) - 0.5);
  double fy0 = floor(fmin(fmin(ay, by), cy) - 0.5), fy1 = ceil(fmax(fmax(ay, by), cy) - 0.5);
  fx0 = fmax(fx0, 0.0); fy0 = fmax(fy0, 0.0);
  fx1 = fmin(fx1, (double)(width - 1)); fy1 = fmin(fy1, (double)(height - 1));
  if (fx1 < fx0 || fy1 < fy0) return false;
  t.x0 = (int)fx0; t.x1 = (int)fx1; t.y0 = (int)fy0; t.y1 = (int)fy1;
  t.ax = ax; t.ay = ay; t.bx = bx; t.by = by; t.cx = cx; t.cy = cy;
  t.e0x = cx - bx; t.e0y = cy - by;
  t.e1x = ax - cx; t.e1y = ay - cy;
  t.e2x = bx - ax; t.e2y = by - ay;
  t.own0 = (t.e0y == 0.0 && t.e0x > 0.0) || t.e0y < 0.0;
  t.own1 = (t.e1y == 0.0 && t.e1x > 0.0) || t.e1y < 0.0;
  t.own2 = (t.e2y == 0.0 && t.e2x > 0.0) || t.e2y < 0.0;
  t.inv_area = 1.0 / area2;
  t.za = A.z;
  t.zb = flip ? C.z : B.z;
  t.zc = flip ? B.z : C.z;
  t.flip = flip;
  return true;
}

// Edge tests + perspective-correct depth at pixel (px, py), meshraster.py:86-101.
__device__ __forceinline__ bool tri_fragment(const TriSetup& t, int px, int py, double& l0, double& l1, double& l2,
                                             double& z) {
  const double sx = px + 0.5, sy = py + 0.5;
  const double w0 = t.e0x * (sy - t.by) - t.e0y * (sx - t.bx);
  const double w1 = t.e1x * (sy - t.cy) - t.e1y * (sx - t.cx);
  const double w2 = t.e2x * (sy - t.ay) - t.e2y * (sx - t.ax);
  if (!((w0 > 0.0 || (w0 == 0.0 && t.own0)) && (w1 > 0.0 || (w1 == 0.0 && t.own1)) &&
        (w2 > 0.0 || (w2 == 0.0 && t.own2))))
    return false;
  l0 = w0 * t.inv_area;
  l1 = w1 * t.inv_area;
  l2 = w2 * t.inv_area;
  const double inv_z = l0 / t.za + l1 / t.zb + l2 / t.zc;
  z = 1.0 / inv_z;
  return true;
}

// vertex transform, meshraster.py:127-131
__global__ void mesh_project_kernel(const hgs_camera* __restrict__ cam, const float* __restrict__ v, int64_t nv,
                                    double3* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const double v0 = v[3 * i], v1 = v[3 * i + 1], v2 = v[3 * i + 2];
  double t[3];
#pragma unroll
  for (int j = 0; j < 3; j++) t[j] = dot3(v0, v1, v2, cam->R[j * 3], cam->R[j * 3 + 1], cam->R[j * 3 + 2]) + cam->T[j];
  const double safe = t[2] > 0 ? t[2] : 1.0;
  out[i] = make_double3(cam->fx * t[0] / safe + cam->cx, cam->fy * t[1] / safe + cam->cy, t[2]);
}

__device__ __forceinline__ void cas128(unsigned long long* rec, unsigned long long cz, unsigned long long cf,
                                       unsigned long long nz, unsigned long long nf, unsigned long long& oz,
                                       unsigned long long& of) {
  asm volatile(
      "{\n\t.reg .b128 c, n, o;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 n, {%4, %5};\n\t"
      "atom.global.cas.b128 o, [%6], c, n;\n\t"
      "mov.b128 {%0, %1}, o;\n\t}"
      : "=l"(oz), "=l"(of)
      : "l"(cz), "l"(cf), "l"(nz), "l"(nf), "l"(rec)
      : "memory");
}

__device__ __forceinline__ void zrec_min(unsigned long long* rec, unsigned long long zb, unsigned long long f) {
  // lexicographic (z bits, triangle) minimum.  The record only ever
  // decreases, so a z word read at any time bounds the current one from
  // above: zb > cz is a safe reject.  The two plain 64-bit loads may pair a
  // newer z with an older triangle id, so a z tie is confirmed with an
  // atomic read (a CAS that writes back what it expects) before rejecting;
  // a failed CAS returns the coherent current record.
  unsigned long long cz = *(volatile unsigned long long*)rec;
  if (zb > cz) return;
  unsigned long long cf = *(volatile unsigned long long*)(rec + 1);
  if (zb == cz && f >= cf) cas128(rec, cz, cf, cz, cf, cz, cf);
  while (zb < cz || (zb == cz && f < cf)) {
    unsigned long long oz, of;
    cas128(rec, cz, cf, zb, f, oz, of);
    if (oz == cz && of == cf) return;
    cz = oz;
    cf = of;
  }
}

template <int PASS>
__device__ __forceinline__ void raster_pixel(const TriSetup& t, int64_t f, int px, int py, int width,
                                             unsigned long long* zbuf, int32_t* idbuf) {
  double l0, l1, l2, z;
  if (!tri_fragment(t, px, py, l0, l1, l2, z)) return;
  const int64_t p = (int64_t)py * width + px;
  zrec_min(zbuf + 2 * p, (unsigned long long)__double_as_longlong(z), (unsigned long long)f);
  (void)idbuf;
}

template <int PASS>
__global__ void __launch_bounds__(256) raster_small_kernel(const double3* __restrict__ vproj,
                                                           const int32_t* __restrict__ tris, int64_t nf, int width,
                                                           int height, const hgs_camera* __restrict__ cam,
                                                           unsigned long long* zbuf, int32_t* idbuf, int32_t* lists,
                                                           int32_t* list_counts) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  TriSetup t;
  if (!tri_setup(vproj, tris, f, width, height, cam->near_, t)) return;
  const int64_t area = (int64_t)(t.x1 - t.x0 + 1) * (t.y1 - t.y0 + 1);
  if (area > SMALL_TRI_PIXELS) {
    if (PASS == 0) {
      const int which = area > BIG_TRI_PIXELS ? 1 : 0;  // 0: warp list, 1: CTA list
      lists[which * nf + atomicAdd(&list_counts[which], 1)] = (int32_t)f;
    }
    return;
  }
  for (int py = t.y0; py <= t.y1; py++)
    for (int px = t.x0; px <= t.x1; px++) raster_pixel<PASS>(t, f, px, py, width, zbuf, idbuf);
}

// GROUP threads per triangle (32: one warp; 256: one CTA), striding the box.
template <int PASS, int GROUP>
__global__ void __launch_bounds__(256) raster_group_kernel(const double3* __restrict__ vproj,
                                                           const int32_t* __restrict__ tris, int width, int height,
                                                           const hgs_camera* __restrict__ cam,
                                                           unsigned long long* zbuf, int32_t* idbuf,
                                                           const int32_t* list, const int32_t* list_count) {
  const int nlist = *list_count;
  const int groups_per_block = 256 / GROUP;
  const int gid = blockIdx.x * groups_per_block + threadIdx.x / GROUP;
  const int r = threadIdx.x % GROUP;
  for (int b = gid; b < nlist; b += gridDim.x * groups_per_block) {
    const int64_t f = list[b];
    TriSetup t;
    if (!tri_setup(vproj, tris, f, width, height, cam->near_, t)) continue;
    const int bw = t.x1 - t.x0 + 1;
    const int area = bw * (t.y1 - t.y0 + 1);  // < 2^31: clipped to the image
    // box position of q without a division: a running (column, row) pair
    int qy = r / bw, qx = r - qy * bw;
    const int sy = GROUP / bw, sx = GROUP - sy * bw;  // GROUP = sy rows + sx columns
    for (int q = r; q < area; q += GROUP) {
      raster_pixel<PASS>(t, f, t.x0 + qx, t.y0 + qy, width, zbuf, idbuf);
      qx += sx;
      qy += sy;
      if (qx >= bw) { qx -= bw; qy++; }
    }
  }
}

__global__ void raster_init_kernel(unsigned long long* zbuf, int64_t npix) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npix) return;
  reinterpret_cast<ulonglong2*>(zbuf)[p] = make_ulonglong2(0x7ff0000000000000ull, 0x7fffffffull);  // +inf, none
}

// Winner recompute, meshraster.py:97-116.
__global__ void __launch_bounds__(256) raster_resolve_kernel(const double3* __restrict__ vproj,
                                                             const int32_t* __restrict__ tris,
                                                             const float* __restrict__ uvs, int width, int height,
                                                             const hgs_camera* __restrict__ cam,
                                                             const unsigned long long* __restrict__ zbuf,
                                                             hgs_fragments out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)width * height) return;
  const int32_t f = (int32_t)zbuf[2 * p + 1];
  const int px = (int)(p % width), py = (int)(p / width);
  double b0 = 0.0, b1 = 0.0, b2 = 0.0, z = __longlong_as_double(0x7ff0000000000000LL), u = 0.0, v = 0.0;
  int32_t tid = -1;
  TriSetup t;
  double l0, l1, l2;
  if (f != 0x7fffffff && tri_setup(vproj, tris, f, width, height, cam->near_, t) &&
      tri_fragment(t, px, py, l0, l1, l2, z)) {
    tid = f;
    b0 = l0 / t.za * z;
    b1 = l1 / t.zb * z;
    b2 = l2 / t.zc * z;
    if (t.flip) { const double tb = b1; b1 = b2; b2 = tb; }
    if (uvs) {
      const float* uu = uvs + 6 * (int64_t)f;
      u = b0 * (double)uu[0] + b1 * (double)uu[2] + b2 * (double)uu[4];
      v = b0 * (double)uu[1] + b1 * (double)uu[3] + b2 * (double)uu[5];
    }
  } else {
    z = __longlong_as_double(0x7ff0000000000000LL);
  }
  out.triangle_id[p] = tid;
  out.depth[p] = z;
  if (out.bary) { out.bary[3 * p] = b0; out.bary[3 * p + 1] = b1; out.bary[3 * p + 2] = b2; }
  if (out.uv) { out.uv[2 * p] = u; out.uv[2 * p + 1] = v; }
}

// _texel_coords (meshraster.py:139-155)
struct Taps {
  int64_t i[4];
  double w[4];
};
__device__ __forceinline__ Taps texel_taps(double u, double v, int th, int tw) {
  const double tx = u * (double)tw - 0.5;
  const double ty = (1.0 - v) * (double)th - 0.5;
  const double x0 = floor(tx), y0 = floor(ty);
  const double fx = tx - x0, fy = ty - y0;
  const int64_t x0i = (int64_t)x0, y0i = (int64_t)y0;
  const int64_t xa = tmin<int64_t>(tmax<int64_t>(x0i, 0), tw - 1), xb = tmin<int64_t>(tmax<int64_t>(x0i + 1, 0), tw - 1);
  const int64_t ya = tmin<int64_t>(tmax<int64_t>(y0i, 0), th - 1), yb = tmin<int64_t>(tmax<int64_t>(y0i + 1, 0), th - 1);
  Taps t;
  t.i[0] = ya * tw + xa; t.w[0] = (1 - fx) * (1 - fy);
  t.i[1] = ya * tw + xb; t.w[1] = fx * (1 - fy);
  t.i[2] = yb * tw + xa; t.w[2] = (1 - fx) * fy;
  t.i[3] = yb * tw + xb; t.w[3] = fx * fy;
  return t;
}

__global__ void __launch_bounds__(256) sample_texture_kernel(const float* __restrict__ tex, int th, int tw,
                                                             const double* __restrict__ uv,
                                                             const int32_t* __restrict__ tri, int64_t npix,
                                                             float* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npix) return;
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  if (tri[p] >= 0) {
    const double2 uvp = reinterpret_cast<const double2*>(uv)[p];
    const Taps t = texel_taps(uvp.x, uvp.y, th, tw);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const float* tp = tex + 3 * t.i[k];
      acc0 += (double)__ldg(tp) * t.w[k];
      acc1 += (double)__ldg(tp + 1) * t.w[k];
      acc2 += (double)__ldg(tp + 2) * t.w[k];
    }
  }
  out[3 * p] = (float)acc0;
  out[3 * p + 1] = (float)acc1;
  out[3 * p + 2] = (float)acc2;
}

__global__ void __launch_bounds__(256) texture_backward_kernel(const double* __restrict__ uv,
                                                               const int32_t* __restrict__ tri,
                                                               const float* __restrict__ grad, int64_t npix, int th,
                                                               int tw, float* __restrict__ gtex) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npix || tri[p] < 0) return;
  const double2 uvp = reinterpret_cast<const double2*>(uv)[p];
  const Taps t = texel_taps(uvp.x, uvp.y, th, tw);
  const double g0 = grad[3 * p], g1 = grad[3 * p + 1], g2 = grad[3 * p + 2];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    float* tp = gtex + 3 * t.i[k];
    atomicAdd(tp, (float)(g0 * t.w[k]));
    atomicAdd(tp + 1, (float)(g1 * t.w[k]));
    atomicAdd(tp + 2, (float)(g2 * t.w[k]));
  }
}

// Deterministic variant: each tap's contribution rounded to a 2^-32 grid and
// added as a 64-bit integer (two's complement wraps correctly for negative
// values): integer addition is associative, so the sum does not depend on
// the order of the atomics (|sum| < 2^31, resolution 2.3e-10 per tap -- finer
// than fp32 accumulation at any texel value above 4e-3).
constexpr double TEX_FIXED_SCALE = 4294967296.0;  // 2^32
__global__ void __launch_bounds__(256) texture_backward_fixed_kernel(const double* __restrict__ uv,
                                                                     const int32_t* __restrict__ tri,
                                                                     const float* __restrict__ grad, int64_t npix,
                                                                     int th, int tw,
                                                                     unsigned long long* __restrict__ acc) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npix || tri[p] < 0) return;
  const double2 uvp = reinterpret_cast<const double2*>(uv)[p];
  const Taps t = texel_taps(uvp.x, uvp.y, th, tw);
  const double g0 = grad[3 * p], g1 = grad[3 * p + 1], g2 = grad[3 * p + 2];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    unsigned long long* tp = acc + 3 * t.i[k];
    atomicAdd(tp, (unsigned long long)__double2ll_rn(g0 * t.w[k] * TEX_FIXED_SCALE));
    atomicAdd(tp + 1, (unsigned long long)__double2ll_rn(g1 * t.w[k] * TEX_FIXED_SCALE));
    atomicAdd(tp + 2, (unsigned long long)__double2ll_rn(g2 * t.w[k] * TEX_FIXED_SCALE));
  }
}

// fixed-point accumulator -> fp32 (out = value, or out += value), and the
// accumulator back to zero
__global__ void __launch_bounds__(256) fixed_to_float_kernel(unsigned long long* __restrict__ acc, int64_t n,
                                                             float* __restrict__ out, int accumulate) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = (float)((double)(long long)acc[i] * (1.0 / TEX_FIXED_SCALE));
    out[i] = accumulate ? out[i] + v : v;
    acc[i] = 0ull;
  }
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace hgs

extern "C" size_t hgs_raster_scratch_bytes(int64_t n_vertices, int64_t n_faces, int32_t width, int32_t height) {
  using hgs::align_up;
  const int64_t npix = (int64_t)width * height;
  return align_up(sizeof(double3) * (size_t)(n_vertices > 0 ? n_vertices : 1), 256) +
         align_up(16 * (size_t)npix, 256) +
         align_up(8 * (size_t)(n_faces > 0 ? n_faces : 1), 256) + 256;
}

extern "C" int hgs_rasterize_fragments(const hgs_camera* cam, int32_t width, int32_t height, const hgs_mesh* mesh,
                                       hgs_fragments* out, void* scratch, size_t scratch_bytes, void* stream) {
  using namespace hgs;
  if (!cam || !mesh || !out || !out->triangle_id || !out->depth)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_rasterize_fragments: null argument");
  if (width <= 0 || height <= 0) return hgs_set_error(HGS_ERR_INVALID, "hgs_rasterize_fragments: empty image");
  if (mesh->n_faces > 0x7ffffffeLL) return hgs_set_error(HGS_ERR_INVALID, "hgs_rasterize_fragments: too many faces");
  const size_t need = hgs_raster_scratch_bytes(mesh->n_vertices, mesh->n_faces, width, height);
  if (!scratch || scratch_bytes < need) return hgs_set_error(HGS_ERR_INVALID, "hgs_rasterize_fragments: scratch too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t npix = (int64_t)width * height;
  unsigned char* base = (unsigned char*)scratch;
  double3* vproj = (double3*)base;
  base += align_up(sizeof(double3) * (size_t)(mesh->n_vertices > 0 ? mesh->n_vertices : 1), 256);
  unsigned long long* zbuf = (unsigned long long*)base;  // {bits(z), triangle} per pixel
  base += align_up(16 * (size_t)npix, 256);
  int32_t* idbuf = nullptr;
  int32_t* lists = (int32_t*)base;  // [warp list | CTA list], n_faces each
  base += align_up(8 * (size_t)(mesh->n_faces > 0 ? mesh->n_faces : 1), 256);
  int32_t* list_counts = (int32_t*)base;
  cudaMemsetAsync(list_counts, 0, 2 * sizeof(int32_t), st);
  raster_init_kernel<<<ceil_div(npix, 256), 256, 0, st>>>(zbuf, npix);
  HGS_CHECK_LAUNCH();
  if (mesh->n_faces > 0) {
    if (!mesh->vertices || !mesh->triangles) return hgs_set_error(HGS_ERR_INVALID, "hgs_rasterize_fragments: missing mesh arrays");
    mesh_project_kernel<<<ceil_div(mesh->n_vertices, 256), 256, 0, st>>>(cam, mesh->vertices, mesh->n_vertices, vproj);
    HGS_CHECK_LAUNCH();
    const int gf = ceil_div(mesh->n_faces, 256);
    const int64_t nf = mesh->n_faces;
    int sms = NUM_SMS;
    {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    raster_small_kernel<0><<<gf, 256, 0, st>>>(vproj, mesh->triangles, nf, width, height, cam, zbuf, idbuf, lists,
                                              list_counts);
    HGS_CHECK_LAUNCH();
    raster_group_kernel<0, 32><<<8 * sms, 256, 0, st>>>(vproj, mesh->triangles, width, height, cam, zbuf, idbuf,
                                                        lists, list_counts);
    HGS_CHECK_LAUNCH();
    raster_group_kernel<0, 256><<<2 * sms, 256, 0, st>>>(vproj, mesh->triangles, width, height, cam, zbuf, idbuf,
                                                         lists + nf, list_counts + 1);
    HGS_CHECK_LAUNCH();
  }
  raster_resolve_kernel<<<ceil_div(npix, 256), 256, 0, st>>>(vproj, mesh->triangles, mesh->uvs, width, height, cam,
                                                             zbuf, *out);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}

extern "C" int hgs_sample_texture(const float* texture, int32_t th, int32_t tw, const double* uv,
                                  const int32_t* triangle_id, int64_t npix, float* out, void* stream) {
  if (!texture || !uv || !triangle_id || !out) return hgs_set_error(HGS_ERR_INVALID, "hgs_sample_texture: null argument");
  if (th <= 0 || tw <= 0) return hgs_set_error(HGS_ERR_INVALID, "hgs_sample_texture: empty texture");
  if (npix == 0) return HGS_OK;
  hgs::sample_texture_kernel<<<hgs::ceil_div(npix, 256), 256, 0, (cudaStream_t)stream>>>(texture, th, tw, uv,
                                                                                        triangle_id, npix, out);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}

extern "C" int hgs_texture_backward(const double* uv, const int32_t* triangle_id, const float* grad_image,
                                    int64_t npix, int32_t th, int32_t tw, float* grad_texture, void* stream) {
  if (!uv || !triangle_id || !grad_image || !grad_texture)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_texture_backward: null argument");
  if (th <= 0 || tw <= 0) return hgs_set_error(HGS_ERR_INVALID, "hgs_texture_backward: empty texture");
  if (npix == 0) return HGS_OK;
  hgs::texture_backward_kernel<<<hgs::ceil_div(npix, 256), 256, 0, (cudaStream_t)stream>>>(
      uv, triangle_id, grad_image, npix, th, tw, grad_texture);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}

extern "C" int hgs_texture_backward_fixed(const double* uv, const int32_t* triangle_id, const float* grad_image,
                                          int64_t npix, int32_t th, int32_t tw, int64_t* acc, void* stream) {
  if (!uv || !triangle_id || !grad_image || !acc)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_texture_backward_fixed: null argument");
  if (th <= 0 || tw <= 0) return hgs_set_error(HGS_ERR_INVALID, "hgs_texture_backward_fixed: empty texture");
  if (npix == 0) return HGS_OK;
  hgs::texture_backward_fixed_kernel<<<hgs::ceil_div(npix, 256), 256, 0, (cudaStream_t)stream>>>(
      uv, triangle_id, grad_image, npix, th, tw, (unsigned long long*)acc);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}

extern "C" int hgs_fixed_to_float(int64_t* acc, int64_t n, float* out, int32_t accumulate, void* stream) {
  if (!acc || !out) return hgs_set_error(HGS_ERR_INVALID, "hgs_fixed_to_float: null argument");
  if (n <= 0) return HGS_OK;
  const int blocks = (int)std::min<int64_t>(hgs::ceil_div(n, 256), 8 * hgs::NUM_SMS);
  hgs::fixed_to_float_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((unsigned long long*)acc, n, out, accumulate);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}
