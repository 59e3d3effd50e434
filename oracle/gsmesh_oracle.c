/*
 * gsmesh_oracle.c -- CPU restatement of the reference hybrid GS+mesh render
 * path (gsmesh 0.1.0, /root/reference/pkg/src/gsmesh).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("cpu_baseline.kind = port").  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * path (paper_2506_06988_b200/) never links or calls it.
 *
 * Arithmetic is IEEE fp64 with FMA contraction disabled (-ffp-contract=off),
 * following the reference's operation order term by term.  Where the
 * reference uses numpy matmul, the order numpy/OpenBLAS uses on x86-64 is
 * reproduced explicitly: s = a0*b0; s = fma(a1,b1,s); s = fma(a2,b2,s)
 * (measured in this container: 100% agreement).
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py writes the npz fixtures in tests/golden).
 *
 * Threading: OpenMP over independent units (Gaussians, tiles, row bands);
 * every output is independent of the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* constants: splat/project.py:19-27, splat/tiles.py:16 */
#define COV_FLOOR 0.3
#define ALPHA_CLAMP 0.99
#define SIGMA_SKIP (1.0 / 255.0)
#define SUPPORT_MAHAL2 9.0
#define EARLY_STOP_T 1e-4
#define SH_C0 0.28209479177387814
#define SH_C1 0.4886025119029199

typedef struct {
  double fx, fy, cx, cy;
  int64_t width, height;
  double R[9];      /* world_to_camera[:3,:3], row-major */
  double T[3];      /* world_to_camera[:3,3] */
  double near_, far_;
  double center[3]; /* Camera.center() (scene.py:190-192), computed by numpy */
  double limx, limy; /* FRUSTUM_LIMIT * (W / (2 fx)) (project.py:97-98) */
} or_camera;

static int set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
  return omp_get_max_threads();
#else
  (void)nthreads;
  return 1;
#endif
}

/* numpy matmul inner product order (OpenBLAS dgemm on x86-64). */
static inline double dot3(double a0, double a1, double a2, double b0, double b1, double b2) {
  double s = a0 * b0;
  s = fma(a1, b1, s);
  s = fma(a2, b2, s);
  return s;
}

/* quaternions_to_rotations (scene.py:126-141), one row. */
static void quat_to_rot(const double* q, double* Rq, double* qn_out) {
  double nrm = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
  double w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
  Rq[0] = 1 - 2 * (y * y + z * z);
  Rq[1] = 2 * (x * y - w * z);
  Rq[2] = 2 * (x * z + w * y);
  Rq[3] = 2 * (x * y + w * z);
  Rq[4] = 1 - 2 * (x * x + z * z);
  Rq[5] = 2 * (y * z - w * x);
  Rq[6] = 2 * (x * z - w * y);
  Rq[7] = 2 * (y * z + w * x);
  Rq[8] = 1 - 2 * (x * x + y * y);
  if (qn_out) { qn_out[0] = w; qn_out[1] = x; qn_out[2] = y; qn_out[3] = z; }
}

/* sigma = M M^T with M = R diag(s) (project.py:91-94). */
static void cov3d(const double* Rq, const double* s, double* M, double* sig) {
  for (int a = 0; a < 3; a++)
    for (int b = 0; b < 3; b++) M[a * 3 + b] = Rq[a * 3 + b] * s[b];
  for (int a = 0; a < 3; a++)
    for (int b = 0; b < 3; b++)
      sig[a * 3 + b] = dot3(M[a * 3 + 0], M[a * 3 + 1], M[a * 3 + 2], M[b * 3 + 0], M[b * 3 + 1], M[b * 3 + 2]);
}

/*
 * project (splat/project.py:70-140) + evaluate_colors (:56-67), for all N
 * rows; alive[i] marks rows kept (the caller compacts with np.nonzero).
 * colors_rest may be NULL (degree 0); layout [i][k][c] (scene.py:46-49).
 */
void or_project(const or_camera* cam, int64_t n, const double* centers, const double* rotations,
                const double* log_scales, const double* logits, const double* dc, const double* rest,
                uint8_t* alive, double* mean2d, double* depth_out, double* cov2d, double* conic,
                double* alpha_out, double* color, double* radius_out, double* t_cam, double* color_pre,
                double* view_dir, double* view_dist, int nthreads) {
  set_threads(nthreads);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; i++) {
    const double* c = centers + 3 * i;
    double t[3];
    for (int j = 0; j < 3; j++) t[j] = dot3(c[0], c[1], c[2], cam->R[j * 3 + 0], cam->R[j * 3 + 1], cam->R[j * 3 + 2]) + cam->T[j];
    double depth = t[2];
    int ok = (depth > cam->near_) && (depth < cam->far_);
    double alpha = 1.0 / (1.0 + exp(-logits[i]));
    ok = ok && (alpha >= SIGMA_SKIP);
    double tz = ok ? depth : 1.0;
    double mx = cam->fx * t[0] / tz + cam->cx;
    double my = cam->fy * t[1] / tz + cam->cy;
    double Rq[9], M[9], sig[9], s[3];
    quat_to_rot(rotations + 4 * i, Rq, NULL);
    for (int j = 0; j < 3; j++) s[j] = exp(log_scales[3 * i + j]);
    cov3d(Rq, s, M, sig);
    double rx = t[0] / tz, ry = t[1] / tz;
    rx = fmin(fmax(rx, -cam->limx), cam->limx);
    ry = fmin(fmax(ry, -cam->limy), cam->limy);
    double J[6] = {cam->fx / tz, 0.0, -cam->fx * rx / tz, 0.0, cam->fy / tz, -cam->fy * ry / tz};
    double A[6], AS[6], cov[4];
    for (int j = 0; j < 2; j++)
      for (int b = 0; b < 3; b++)
        A[j * 3 + b] = dot3(J[j * 3 + 0], J[j * 3 + 1], J[j * 3 + 2], cam->R[0 * 3 + b], cam->R[1 * 3 + b], cam->R[2 * 3 + b]);
    for (int j = 0; j < 2; j++)
      for (int b = 0; b < 3; b++)
        AS[j * 3 + b] = dot3(A[j * 3 + 0], A[j * 3 + 1], A[j * 3 + 2], sig[0 * 3 + b], sig[1 * 3 + b], sig[2 * 3 + b]);
    for (int j = 0; j < 2; j++)
      for (int l = 0; l < 2; l++)
        cov[j * 2 + l] = dot3(AS[j * 3 + 0], AS[j * 3 + 1], AS[j * 3 + 2], A[l * 3 + 0], A[l * 3 + 1], A[l * 3 + 2]);
    double cxx = cov[0] + COV_FLOOR, cxy = cov[1], cyy = cov[3] + COV_FLOOR;
    double det = cxx * cyy - cxy * cxy;
    double mid = 0.5 * (cxx + cyy);
    double lam = mid + sqrt(fmax(mid * mid - det, 0.0));
    double radius = 3.0 * sqrt(fmax(lam, 0.0));
    ok = ok && (mx + radius > 0) && (mx - radius < (double)cam->width);
    ok = ok && (my + radius > 0) && (my - radius < (double)cam->height);
    /* colors (project.py:56-67) */
    double pre[3];
    for (int ch = 0; ch < 3; ch++) pre[ch] = 0.5 + SH_C0 * dc[3 * i + ch];
    if (rest) {
      double d0 = c[0] - cam->center[0], d1 = c[1] - cam->center[1], d2 = c[2] - cam->center[2];
      double dist = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
      double den = fmax(dist, 1e-12);
      double x = d0 / den, y = d1 / den, z = d2 / den;
      const double* r = rest + 9 * i;
      for (int ch = 0; ch < 3; ch++) pre[ch] = pre[ch] + SH_C1 * ((-y * r[0 * 3 + ch] + z * r[1 * 3 + ch]) - x * r[2 * 3 + ch]);
      view_dir[3 * i + 0] = x; view_dir[3 * i + 1] = y; view_dir[3 * i + 2] = z;
      view_dist[i] = dist;
    }
    double inv_det = 1.0 / det;
    alive[i] = (uint8_t)ok;
    mean2d[2 * i] = mx; mean2d[2 * i + 1] = my;
    depth_out[i] = depth;
    cov2d[3 * i] = cxx; cov2d[3 * i + 1] = cxy; cov2d[3 * i + 2] = cyy;
    conic[3 * i] = cyy * inv_det; conic[3 * i + 1] = -cxy * inv_det; conic[3 * i + 2] = cxx * inv_det;
    alpha_out[i] = alpha;
    radius_out[i] = radius;
    for (int ch = 0; ch < 3; ch++) { color[3 * i + ch] = fmax(pre[ch], 0.0); color_pre[3 * i + ch] = pre[ch]; t_cam[3 * i + ch] = t[ch]; }
  }
}

/* ---------------------------------------------------------------------- */
/* build_tiles (splat/tiles.py:35-69)                                       */
/* ---------------------------------------------------------------------- */

static inline int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

static void tile_rect(double mx, double my, double r, int64_t tile_px, int64_t tx_n, int64_t ty_n, int64_t* rc) {
  rc[0] = clampi((int64_t)floor((mx - r) / (double)tile_px), 0, tx_n - 1);
  rc[1] = clampi((int64_t)floor((mx + r) / (double)tile_px), 0, tx_n - 1);
  rc[2] = clampi((int64_t)floor((my - r) / (double)tile_px), 0, ty_n - 1);
  rc[3] = clampi((int64_t)floor((my + r) / (double)tile_px), 0, ty_n - 1);
}

/* per-row tile count (tiles.py:45-50); returns K = sum(counts). */
int64_t or_tile_counts(int64_t m, const double* mean2d, const double* radius, int64_t width, int64_t height,
                       int64_t tile_px, int64_t* counts, int nthreads) {
  set_threads(nthreads);
  int64_t tx_n = (width + tile_px - 1) / tile_px, ty_n = (height + tile_px - 1) / tile_px;
  int64_t total = 0;
#pragma omp parallel for schedule(static) reduction(+ : total)
  for (int64_t i = 0; i < m; i++) {
    int64_t rc[4];
    tile_rect(mean2d[2 * i], mean2d[2 * i + 1], radius[i], tile_px, tx_n, ty_n, rc);
    counts[i] = (rc[1] - rc[0] + 1) * (rc[3] - rc[2] + 1);
    total += counts[i];
  }
  return total;
}

typedef struct { double d; int64_t kept; int32_t row; } depth_item;

static int cmp_depth(const void* a, const void* b) {
  const depth_item* x = (const depth_item*)a;
  const depth_item* y = (const depth_item*)b;
  if (x->d < y->d) return -1;
  if (x->d > y->d) return 1;
  if (x->kept < y->kept) return -1;
  if (x->kept > y->kept) return 1;
  return 0;
}

/*
 * Fills tile_starts (n_tiles+1) and entries (K) with the order
 * np.lexsort((kept, depth, tile)) of tiles.py:65: rows are ordered once by
 * (depth, kept) and then distributed into per-tile lists by a stable counting
 * pass, which yields exactly the (tile, depth, kept) lexicographic order.
 */
void or_build_tiles(int64_t m, const double* mean2d, const double* radius, const double* depth,
                    const int64_t* kept, int64_t width, int64_t height, int64_t tile_px,
                    int64_t* tile_starts, int32_t* entries, int nthreads) {
  int nt = set_threads(nthreads);
  int64_t tx_n = (width + tile_px - 1) / tile_px, ty_n = (height + tile_px - 1) / tile_px;
  int64_t n_tiles = tx_n * ty_n;
  depth_item* items = (depth_item*)malloc(sizeof(depth_item) * (size_t)(m > 0 ? m : 1));
  int64_t* rects = (int64_t*)malloc(sizeof(int64_t) * 4 * (size_t)(m > 0 ? m : 1));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; i++) {
    items[i].d = depth[i]; items[i].kept = kept[i]; items[i].row = (int32_t)i;
    tile_rect(mean2d[2 * i], mean2d[2 * i + 1], radius[i], tile_px, tx_n, ty_n, rects + 4 * i);
  }
  qsort(items, (size_t)m, sizeof(depth_item), cmp_depth);
  /* stable counting sort by tile over the depth-ordered sequence, split in
     nt contiguous chunks: cursor[t][tile] = start of chunk t in tile list. */
  int64_t* hist = (int64_t*)calloc((size_t)nt * (size_t)n_tiles, sizeof(int64_t));
#pragma omp parallel num_threads(nt)
  {
    int t = 0, T = 1;
#ifdef _OPENMP
    t = omp_get_thread_num(); T = omp_get_num_threads();
#endif
    int64_t lo = m * t / T, hi = m * (t + 1) / T;
    int64_t* h = hist + (int64_t)t * n_tiles;
    for (int64_t j = lo; j < hi; j++) {
      const int64_t* rc = rects + 4 * items[j].row;
      for (int64_t ty = rc[2]; ty <= rc[3]; ty++)
        for (int64_t tx = rc[0]; tx <= rc[1]; tx++) h[ty * tx_n + tx]++;
    }
#pragma omp barrier
#pragma omp single
    {
      int64_t run = 0;
      for (int64_t tile = 0; tile < n_tiles; tile++) {
        tile_starts[tile] = run;
        for (int tt = 0; tt < T; tt++) {
          int64_t c = hist[(int64_t)tt * n_tiles + tile];
          hist[(int64_t)tt * n_tiles + tile] = run;
          run += c;
        }
      }
      tile_starts[n_tiles] = run;
    }
    for (int64_t j = lo; j < hi; j++) {
      const int64_t* rc = rects + 4 * items[j].row;
      for (int64_t ty = rc[2]; ty <= rc[3]; ty++)
        for (int64_t tx = rc[0]; tx <= rc[1]; tx++) entries[h[ty * tx_n + tx]++] = items[j].row;
    }
  }
  free(hist);
  free(rects);
  free(items);
}

/* ---------------------------------------------------------------------- */
/* forward_kernel (splat/kernels.py:12-74)                                  */
/* ---------------------------------------------------------------------- */
void or_forward(const int64_t* tile_starts, const int32_t* entries, int64_t tiles_x, int64_t tiles_y,
                int64_t tile_px, int64_t width, int64_t height, const double* mean2d, const double* conic,
                const double* alpha, const double* color, const double* depth, int has_mesh,
                const double* mesh_color, const double* mesh_depth, const uint8_t* mesh_valid, const double* bg,
                double* out_color, double* out_t, double* out_depth, int32_t* out_last, int nthreads) {
  set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < tiles_x * tiles_y; t++) {
    int64_t ty = t / tiles_x, tx = t % tiles_x;
    int64_t s = tile_starts[t], e = tile_starts[t + 1];
    int64_t py0 = ty * tile_px, px0 = tx * tile_px;
    int64_t py1 = py0 + tile_px < height ? py0 + tile_px : height;
    int64_t px1 = px0 + tile_px < width ? px0 + tile_px : width;
    for (int64_t py = py0; py < py1; py++)
      for (int64_t px = px0; px < px1; px++) {
        double fx = px + 0.5, fy = py + 0.5;
        int64_t p = py * width + px;
        int mesh_here = has_mesh && mesh_valid[p];
        double limit = mesh_here ? mesh_depth[p] : INFINITY;
        double trans = 1.0, r = 0.0, g = 0.0, b = 0.0, dacc = 0.0;
        int32_t last = -1;
        for (int64_t k = s; k < e; k++) {
          int32_t i = entries[k];
          if (depth[i] >= limit) break;
          double dx = fx - mean2d[2 * i], dy = fy - mean2d[2 * i + 1];
          double mm = conic[3 * i] * dx * dx + 2.0 * conic[3 * i + 1] * dx * dy + conic[3 * i + 2] * dy * dy;
          if (mm > SUPPORT_MAHAL2 || mm < 0.0) continue;
          double sig = alpha[i] * exp(-0.5 * mm);
          if (sig > ALPHA_CLAMP) sig = ALPHA_CLAMP;
          if (sig < SIGMA_SKIP) continue;
          double test_t = trans * (1.0 - sig);
          if (test_t < EARLY_STOP_T) break;
          double w = sig * trans;
          r += color[3 * i] * w;
          g += color[3 * i + 1] * w;
          b += color[3 * i + 2] * w;
          dacc += depth[i] * w;
          trans = test_t;
          last = (int32_t)k;
        }
        if (mesh_here) {
          out_color[3 * p] = r + trans * mesh_color[3 * p];
          out_color[3 * p + 1] = g + trans * mesh_color[3 * p + 1];
          out_color[3 * p + 2] = b + trans * mesh_color[3 * p + 2];
          out_depth[p] = dacc + trans * mesh_depth[p];
        } else {
          out_color[3 * p] = r + trans * bg[0];
          out_color[3 * p + 1] = g + trans * bg[1];
          out_color[3 * p + 2] = b + trans * bg[2];
          double acc = 1.0 - trans;
          out_depth[p] = acc > 1e-12 ? dacc / acc : NAN;
        }
        out_t[p] = trans;
        out_last[p] = last;
      }
  }
}

/* ---------------------------------------------------------------------- */
/* backward_kernel (splat/kernels.py:77-160) + np.add.at (render.py:155-157)*/
/* ---------------------------------------------------------------------- */
void or_backward_entries(const int64_t* tile_starts, const int32_t* entries, int64_t tiles_x, int64_t tiles_y,
                         int64_t tile_px, int64_t width, int64_t height, const double* mean2d, const double* conic,
                         const double* alpha, const double* color, int has_mesh, const double* mesh_color,
                         const uint8_t* mesh_valid, const double* bg, const double* final_t, const int32_t* out_last,
                         const double* grad_pixels, const double* grad_trans, double* entry_grads, int nthreads) {
  set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < tiles_x * tiles_y; t++) {
    int64_t ty = t / tiles_x, tx = t % tiles_x;
    int64_t s = tile_starts[t];
    int64_t py0 = ty * tile_px, px0 = tx * tile_px;
    int64_t py1 = py0 + tile_px < height ? py0 + tile_px : height;
    int64_t px1 = px0 + tile_px < width ? px0 + tile_px : width;
    for (int64_t py = py0; py < py1; py++)
      for (int64_t px = px0; px < px1; px++) {
        int64_t p = py * width + px;
        int32_t last = out_last[p];
        double gr = grad_pixels[3 * p], gg = grad_pixels[3 * p + 1], gb = grad_pixels[3 * p + 2];
        double gt_pix = grad_trans[p];
        int mesh_here = has_mesh && mesh_valid[p];
        if (last < 0) continue;
        double fx = px + 0.5, fy = py + 0.5;
        double t_after = final_t[p];
        double acc_r, acc_g, acc_b;
        if (mesh_here) {
          acc_r = t_after * mesh_color[3 * p]; acc_g = t_after * mesh_color[3 * p + 1]; acc_b = t_after * mesh_color[3 * p + 2];
        } else {
          acc_r = t_after * bg[0]; acc_g = t_after * bg[1]; acc_b = t_after * bg[2];
        }
        for (int64_t k = last; k > s - 1; k--) {
          int32_t i = entries[k];
          double dx = fx - mean2d[2 * i], dy = fy - mean2d[2 * i + 1];
          double mm = conic[3 * i] * dx * dx + 2.0 * conic[3 * i + 1] * dx * dy + conic[3 * i + 2] * dy * dy;
          if (mm > SUPPORT_MAHAL2 || mm < 0.0) continue;
          double gauss = exp(-0.5 * mm);
          double sig = alpha[i] * gauss;
          int clamped = sig > ALPHA_CLAMP;
          if (clamped) sig = ALPHA_CLAMP;
          if (sig < SIGMA_SKIP) continue;
          double one_minus = 1.0 - sig;
          double t_before = t_after / one_minus;
          double w = sig * t_before;
          double* eg = entry_grads + 9 * k;
          eg[6] += gr * w; eg[7] += gg * w; eg[8] += gb * w;
          double s_i = (gr * (color[3 * i] * t_before - acc_r / one_minus)
                        + gg * (color[3 * i + 1] * t_before - acc_g / one_minus))
                       + gb * (color[3 * i + 2] * t_before - acc_b / one_minus);
          if (gt_pix != 0.0) s_i += gt_pix * (-final_t[p] / one_minus);
          if (!clamped) {
            double qd_x = conic[3 * i] * dx + conic[3 * i + 1] * dy;
            double qd_y = conic[3 * i + 1] * dx + conic[3 * i + 2] * dy;
            double common = s_i * sig;
            eg[0] += common * qd_x;
            eg[1] += common * qd_y;
            eg[2] += 0.5 * common * qd_x * qd_x;
            eg[3] += 0.5 * common * qd_x * qd_y;
            eg[4] += 0.5 * common * qd_y * qd_y;
            eg[5] += s_i * gauss;
          }
          acc_r += color[3 * i] * w;
          acc_g += color[3 * i + 1] * w;
          acc_b += color[3 * i + 2] * w;
          t_after = t_before;
        }
      }
  }
}

/* np.add.at(per_gauss, entries, entry_grads) -- sequential, entry order. */
void or_reduce_entries(int64_t k, const int32_t* entries, const double* entry_grads, double* per_gauss) {
  for (int64_t e = 0; e < k; e++)
    for (int j = 0; j < 9; j++) per_gauss[9 * (int64_t)entries[e] + j] += entry_grads[9 * e + j];
}

/* _quat_rotation_derivatives (render.py:290-313): D[k][i][j]. */
static void quat_derivs(const double* qn, double* D) {
  double w = qn[0], x = qn[1], y = qn[2], z = qn[3];
  double d0[9] = {0, -z, y, z, 0, -x, -y, x, 0};
  double d1[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
  double d2[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
  double d3[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
  for (int a = 0; a < 9; a++) { D[a] = 2.0 * d0[a]; D[9 + a] = 2.0 * d1[a]; D[18 + a] = 2.0 * d2[a]; D[27 + a] = 2.0 * d3[a]; }
}

/*
 * _chain_to_parameters (render.py:185-287) for the M kept rows, writing into
 * full-length (N) gradient arrays at row kept[r]; also densify_norm
 * (render.py:171-174).  per_gauss rows: mean2d 2, cov 3, alpha 1, rgb 3.
 */
void or_chain(const or_camera* cam, int64_t m, const int64_t* kept, const double* per_gauss,
              const double* rotations, const double* log_scales, const double* rest,
              const double* alpha, const double* t_cam, const double* color_pre, const double* view_dir,
              const double* view_dist, double* g_centers, double* g_rot, double* g_logscale, double* g_logit,
              double* g_dc, double* g_rest, double* densify_norm, int nthreads) {
  set_threads(nthreads);
  double fx = cam->fx, fy = cam->fy;
  const double* Rw = cam->R;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < m; r++) {
    int64_t gi = kept[r];
    const double* pg = per_gauss + 9 * r;
    double gm0 = pg[0], gm1 = pg[1];
    double gcov[4] = {pg[2], pg[3], pg[3], pg[4]};
    double ga = pg[5];
    g_logit[gi] = ga * alpha[r] * (1.0 - alpha[r]);
    double gpre[3], gc[3] = {0, 0, 0};
    for (int ch = 0; ch < 3; ch++) {
      gpre[ch] = pg[6 + ch] * (color_pre[3 * r + ch] > 0.0 ? 1.0 : 0.0);
      g_dc[3 * gi + ch] = SH_C0 * gpre[ch];
    }
    if (rest) {
      double x = view_dir[3 * r], y = view_dir[3 * r + 1], z = view_dir[3 * r + 2];
      const double* rr = rest + 9 * gi;
      for (int ch = 0; ch < 3; ch++) {
        g_rest[9 * gi + 0 * 3 + ch] = -SH_C1 * y * gpre[ch];
        g_rest[9 * gi + 1 * 3 + ch] = SH_C1 * z * gpre[ch];
        g_rest[9 * gi + 2 * 3 + ch] = -SH_C1 * x * gpre[ch];
      }
      double s2 = (gpre[0] * rr[6] + gpre[1] * rr[7]) + gpre[2] * rr[8];
      double s0 = (gpre[0] * rr[0] + gpre[1] * rr[1]) + gpre[2] * rr[2];
      double s1 = (gpre[0] * rr[3] + gpre[1] * rr[4]) + gpre[2] * rr[5];
      double gd[3] = {-SH_C1 * s2, -SH_C1 * s0, SH_C1 * s1};
      double dd = (gd[0] * x + gd[1] * y) + gd[2] * z;
      double dv[3] = {x, y, z};
      for (int j = 0; j < 3; j++) gc[j] += (gd[j] - dv[j] * dd) / view_dist[r];
    }
    const double* t = t_cam + 3 * r;
    double tz = t[2];
    double rx_raw = t[0] / tz, ry_raw = t[1] / tz;
    double rx = fmin(fmax(rx_raw, -cam->limx), cam->limx);
    double ry = fmin(fmax(ry_raw, -cam->limy), cam->limy);
    double in_x = fabs(rx_raw) < cam->limx ? 1.0 : 0.0, in_y = fabs(ry_raw) < cam->limy ? 1.0 : 0.0;
    double J[6] = {fx / tz, 0.0, -fx * rx / tz, 0.0, fy / tz, -fy * ry / tz};
    double Rq[9], qn[4], M[9], sig[9], s[3];
    quat_to_rot(rotations + 4 * gi, Rq, qn);
    for (int j = 0; j < 3; j++) s[j] = exp(log_scales[3 * gi + j]);
    cov3d(Rq, s, M, sig);
    double A[6];
    for (int j = 0; j < 2; j++)
      for (int b = 0; b < 3; b++)
        A[j * 3 + b] = dot3(J[j * 3 + 0], J[j * 3 + 1], J[j * 3 + 2], Rw[0 * 3 + b], Rw[1 * 3 + b], Rw[2 * 3 + b]);
    /* g_sigma[a][b] = sum_jk A[j][a] gcov[j][k] A[k][b] */
    double gS[9], gA[6], gJ[6];
    for (int a = 0; a < 3; a++)
      for (int b = 0; b < 3; b++) {
        double acc = 0.0;
        for (int j = 0; j < 2; j++)
          for (int k = 0; k < 2; k++) acc += A[j * 3 + a] * gcov[j * 2 + k] * A[k * 3 + b];
        gS[a * 3 + b] = acc;
      }
    /* g_A[j][b] = 2 sum_ka gcov[j][k] A[k][a] sigma[a][b] */
    for (int j = 0; j < 2; j++)
      for (int b = 0; b < 3; b++) {
        double acc = 0.0;
        for (int k = 0; k < 2; k++)
          for (int a = 0; a < 3; a++) acc += gcov[j * 2 + k] * A[k * 3 + a] * sig[a * 3 + b];
        gA[j * 3 + b] = 2.0 * acc;
      }
    /* g_J[j][k] = sum_c g_A[j][c] Rw[k][c] */
    for (int j = 0; j < 2; j++)
      for (int k = 0; k < 3; k++) gJ[j * 3 + k] = (gA[j * 3 + 0] * Rw[k * 3 + 0] + gA[j * 3 + 1] * Rw[k * 3 + 1]) + gA[j * 3 + 2] * Rw[k * 3 + 2];
    double gt[3] = {0, 0, 0};
    gt[0] += gm0 * fx / tz;
    gt[1] += gm1 * fy / tz;
    gt[2] += -(gm0 * fx * rx_raw + gm1 * fy * ry_raw) / tz;
    double inv_tz2 = 1.0 / (tz * tz);
    gt[0] += gJ[0 * 3 + 2] * (-fx * in_x * inv_tz2);
    gt[1] += gJ[1 * 3 + 2] * (-fy * in_y * inv_tz2);
    gt[2] += ((gJ[0] * (-fx * inv_tz2) + gJ[4] * (-fy * inv_tz2)) + gJ[2] * fx * (in_x * rx_raw + rx) * inv_tz2)
             + gJ[5] * fy * (in_y * ry_raw + ry) * inv_tz2;
    /* grad_center += g_t @ Rw */
    for (int c = 0; c < 3; c++) gc[c] += dot3(gt[0], gt[1], gt[2], Rw[0 * 3 + c], Rw[1 * 3 + c], Rw[2 * 3 + c]);
    /* g_M = 2 g_sigma M ; g_R = g_M * s ; g_s = sum_i g_M[i][j] R[i][j] */
    double gM[9], gR[9], gs[3] = {0, 0, 0};
    for (int a = 0; a < 3; a++)
      for (int c = 0; c < 3; c++) {
        double acc = 0.0;
        for (int b = 0; b < 3; b++) acc += gS[a * 3 + b] * M[b * 3 + c];
        gM[a * 3 + c] = 2.0 * acc;
      }
    for (int a = 0; a < 3; a++)
      for (int c = 0; c < 3; c++) { gR[a * 3 + c] = gM[a * 3 + c] * s[c]; gs[c] += gM[a * 3 + c] * Rq[a * 3 + c]; }
    for (int j = 0; j < 3; j++) g_logscale[3 * gi + j] = gs[j] * s[j];
    double D[36], gqn[4];
    quat_derivs(qn, D);
    for (int k = 0; k < 4; k++) {
      double acc = 0.0;
      for (int a = 0; a < 9; a++) acc += gR[a] * D[9 * k + a];
      gqn[k] = acc;
    }
    const double* q = rotations + 4 * gi;
    double nrm = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
    double dq = ((gqn[0] * qn[0] + gqn[1] * qn[1]) + gqn[2] * qn[2]) + gqn[3] * qn[3];
    for (int k = 0; k < 4; k++) g_rot[4 * gi + k] = (gqn[k] - qn[k] * dq) / nrm;
    for (int c = 0; c < 3; c++) g_centers[3 * gi + c] = gc[c];
    double sx = gm0 * ((double)cam->width / 2.0), sy = gm1 * ((double)cam->height / 2.0);
    densify_norm[gi] = sqrt(sx * sx + sy * sy);
  }
}

/* ---------------------------------------------------------------------- */
/* _raster_kernel (meshraster.py:45-116) + rasterize_fragments (:119-136)   */
/* ---------------------------------------------------------------------- */

/* vertex projection (meshraster.py:127-131): vs (V,2), zs (V). */
void or_mesh_project(const or_camera* cam, int64_t nv, const double* vertices, double* vs, double* zs) {
  for (int64_t i = 0; i < nv; i++) {
    const double* v = vertices + 3 * i;
    double t[3];
    for (int j = 0; j < 3; j++) t[j] = dot3(v[0], v[1], v[2], cam->R[j * 3 + 0], cam->R[j * 3 + 1], cam->R[j * 3 + 2]) + cam->T[j];
    double safe = t[2] > 0 ? t[2] : 1.0;
    zs[i] = t[2];
    vs[2 * i] = cam->fx * t[0] / safe + cam->cx;
    vs[2 * i + 1] = cam->fy * t[1] / safe + cam->cy;
  }
}

/*
 * Triangles are processed in index order with a strict z test, exactly as the
 * reference; threads own disjoint row bands so the result is identical.
 * out_* must be pre-initialised (tri -1, depth +inf, bary/uv 0).
 */
void or_raster(const double* vs, const double* zs, int64_t nf, const int64_t* tris, const double* uvs, int has_uv,
               int64_t width, int64_t height, double near_, int32_t* out_tri, double* out_depth, double* out_bary,
               double* out_uv, int nthreads) {
  int nt = set_threads(nthreads);
#pragma omp parallel num_threads(nt)
  {
    int t = 0, T = 1;
#ifdef _OPENMP
    t = omp_get_thread_num(); T = omp_get_num_threads();
#endif
    int64_t band_lo = height * t / T, band_hi = height * (t + 1) / T - 1;
    for (int64_t f = 0; f < nf; f++) {
      int64_t ia = tris[3 * f], ib = tris[3 * f + 1], ic = tris[3 * f + 2];
      if (zs[ia] <= near_ || zs[ib] <= near_ || zs[ic] <= near_) continue;
      double ax = vs[2 * ia], ay = vs[2 * ia + 1];
      double bx = vs[2 * ib], by = vs[2 * ib + 1];
      double cx = vs[2 * ic], cy = vs[2 * ic + 1];
      double area2 = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
      if (area2 == 0.0) continue;
      int flip = area2 < 0.0;
      if (flip) {
        double tx_ = bx; bx = cx; cx = tx_;
        double ty_ = by; by = cy; cy = ty_;
        area2 = -area2;
      }
      int64_t x0 = (int64_t)floor(fmin(fmin(ax, bx), cx) - 0.5); if (x0 < 0) x0 = 0;
      int64_t x1 = (int64_t)ceil(fmax(fmax(ax, bx), cx) - 0.5); if (x1 > width - 1) x1 = width - 1;
      int64_t y0 = (int64_t)floor(fmin(fmin(ay, by), cy) - 0.5); if (y0 < 0) y0 = 0;
      int64_t y1 = (int64_t)ceil(fmax(fmax(ay, by), cy) - 0.5); if (y1 > height - 1) y1 = height - 1;
      if (x1 < x0 || y1 < y0) continue;
      if (y0 < band_lo) y0 = band_lo;
      if (y1 > band_hi) y1 = band_hi;
      if (y1 < y0) continue;
      double e0x = cx - bx, e0y = cy - by;
      double e1x = ax - cx, e1y = ay - cy;
      double e2x = bx - ax, e2y = by - ay;
      int own0 = (e0y == 0.0 && e0x > 0.0) || e0y < 0.0;
      int own1 = (e1y == 0.0 && e1x > 0.0) || e1y < 0.0;
      int own2 = (e2y == 0.0 && e2x > 0.0) || e2y < 0.0;
      double inv_area = 1.0 / area2;
      double za = zs[ia];
      double zb = flip ? zs[ic] : zs[ib];
      double zc = flip ? zs[ib] : zs[ic];
      for (int64_t py = y0; py <= y1; py++) {
        double sy = py + 0.5;
        for (int64_t px = x0; px <= x1; px++) {
          double sx = px + 0.5;
          double w0 = e0x * (sy - by) - e0y * (sx - bx);
          double w1 = e1x * (sy - cy) - e1y * (sx - cx);
          double w2 = e2x * (sy - ay) - e2y * (sx - ax);
          if (!((w0 > 0.0 || (w0 == 0.0 && own0)) && (w1 > 0.0 || (w1 == 0.0 && own1)) && (w2 > 0.0 || (w2 == 0.0 && own2))))
            continue;
          double l0 = w0 * inv_area, l1 = w1 * inv_area, l2 = w2 * inv_area;
          double inv_z = l0 / za + l1 / zb + l2 / zc;
          double z = 1.0 / inv_z;
          int64_t p = py * width + px;
          if (z >= out_depth[p]) continue;
          out_depth[p] = z;
          out_tri[p] = (int32_t)f;
          double b0 = l0 / za * z, b1 = l1 / zb * z, b2 = l2 / zc * z;
          if (flip) { double tb = b1; b1 = b2; b2 = tb; }
          out_bary[3 * p] = b0; out_bary[3 * p + 1] = b1; out_bary[3 * p + 2] = b2;
          if (has_uv) {
            const double* u = uvs + 6 * f;
            out_uv[2 * p] = b0 * u[0] + b1 * u[2] + b2 * u[4];
            out_uv[2 * p + 1] = b0 * u[1] + b1 * u[3] + b2 * u[5];
          }
        }
      }
    }
  }
}

/* ---------------------------------------------------------------------- */
/* _texel_coords / sample_texture / texture_backward (meshraster.py:139-184)*/
/* ---------------------------------------------------------------------- */
static void texel_taps(double u, double v, int64_t th, int64_t tw, int64_t* ys, int64_t* xs, double* ws) {
  double tx = u * (double)tw - 0.5;
  double ty = (1.0 - v) * (double)th - 0.5;
  double x0 = floor(tx), y0 = floor(ty);
  double fx = tx - x0, fy = ty - y0;
  int64_t x0i = (int64_t)x0, y0i = (int64_t)y0;
  int64_t xa = clampi(x0i, 0, tw - 1), xb = clampi(x0i + 1, 0, tw - 1);
  int64_t ya = clampi(y0i, 0, th - 1), yb = clampi(y0i + 1, 0, th - 1);
  ys[0] = ya; xs[0] = xa; ws[0] = (1 - fx) * (1 - fy);
  ys[1] = ya; xs[1] = xb; ws[1] = fx * (1 - fy);
  ys[2] = yb; xs[2] = xa; ws[2] = (1 - fx) * fy;
  ys[3] = yb; xs[3] = xb; ws[3] = fx * fy;
}

void or_sample_texture(const double* tex, int64_t th, int64_t tw, int64_t npix, const double* uv,
                       const uint8_t* valid, double* out, int nthreads) {
  set_threads(nthreads);
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < npix; p++) {
    int64_t ys[4], xs[4];
    double ws[4];
    texel_taps(uv[2 * p], uv[2 * p + 1], th, tw, ys, xs, ws);
    double acc[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < 4; k++) {
      const double* tp = tex + 3 * (ys[k] * tw + xs[k]);
      for (int ch = 0; ch < 3; ch++) acc[ch] += tp[ch] * ws[k];
    }
    for (int ch = 0; ch < 3; ch++) out[3 * p + ch] = valid[p] ? acc[ch] : 0.0;
  }
}

/* adjoint: per tap k (in order), np.add.at over valid pixels in raster order */
void or_texture_backward(int64_t th, int64_t tw, int64_t npix, const double* uv, const uint8_t* valid,
                         const double* grad, double* grad_tex) {
  for (int k = 0; k < 4; k++)
    for (int64_t p = 0; p < npix; p++) {
      if (!valid[p]) continue;
      int64_t ys[4], xs[4];
      double ws[4];
      texel_taps(uv[2 * p], uv[2 * p + 1], th, tw, ys, xs, ws);
      double* tp = grad_tex + 3 * (ys[k] * tw + xs[k]);
      for (int ch = 0; ch < 3; ch++) tp[ch] += grad[3 * p + ch] * ws[k];
    }
}

/* ---------------------------------------------------------------------- */
/* losses (train/losses.py)                                                 */
/* ---------------------------------------------------------------------- */

/* scipy.ndimage.convolve1d, mode constant 0, symmetric 11-tap window, along
   an axis of an (H,W,C) image; losses.py:35-38. */
static void filt_axis(const double* in, double* out, int64_t h, int64_t w, int64_t c, const double* win, int axis) {
  int64_t n = axis == 0 ? h : w;
#pragma omp parallel for schedule(static)
  for (int64_t y = 0; y < h; y++)
    for (int64_t x = 0; x < w; x++)
      for (int64_t ch = 0; ch < c; ch++) {
        int64_t i = axis == 0 ? y : x;
        double acc = 0.0;
        for (int k = -5; k <= 5; k++) {
          int64_t j = i + k;
          if (j < 0 || j >= n) continue;
          int64_t yy = axis == 0 ? j : y, xx = axis == 0 ? x : j;
          acc += in[(yy * w + xx) * c + ch] * win[k + 5];
        }
        out[(y * w + x) * c + ch] = acc;
      }
}

static void filt(const double* in, double* out, double* tmp, int64_t h, int64_t w, int64_t c, const double* win) {
  filt_axis(in, tmp, h, w, c, win, 0);
  filt_axis(tmp, out, h, w, c, win, 1);
}

/* ssim (losses.py:47-70): returns mean SSIM, writes gradient wrt pred. */
double or_ssim(const double* x, const double* y, int64_t h, int64_t w, int64_t c, const double* win, double* grad,
               int nthreads) {
  set_threads(nthreads);
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  int64_t n = h * w * c;
  double* buf = (double*)malloc(sizeof(double) * (size_t)n * 12);
  double *ux = buf, *uy = buf + n, *vx = buf + 2 * n, *vy = buf + 3 * n, *vxy = buf + 4 * n, *tmp = buf + 5 * n;
  double *t1 = buf + 6 * n, *dux = buf + 7 * n, *dvx = buf + 8 * n, *dvxy = buf + 9 * n, *f1 = buf + 10 * n, *f2 = buf + 11 * n;
  filt(x, ux, tmp, h, w, c, win);
  filt(y, uy, tmp, h, w, c, win);
  for (int64_t i = 0; i < n; i++) t1[i] = x[i] * x[i];
  filt(t1, vx, tmp, h, w, c, win);
  for (int64_t i = 0; i < n; i++) t1[i] = y[i] * y[i];
  filt(t1, vy, tmp, h, w, c, win);
  for (int64_t i = 0; i < n; i++) t1[i] = x[i] * y[i];
  filt(t1, vxy, tmp, h, w, c, win);
  double total = 0.0;
  for (int64_t i = 0; i < n; i++) {
    double a1 = 2 * ux[i] * uy[i] + C1;
    double a2 = 2 * (vxy[i] - ux[i] * uy[i]) + C2;
    double b1 = ux[i] * ux[i] + uy[i] * uy[i] + C1;
    double b2 = (vx[i] - ux[i] * ux[i]) + (vy[i] - uy[i] * uy[i]) + C2;
    double q = b1 * b2;
    double s = (a1 * a2) / q;
    total += s;
    dux[i] = 2 * uy[i] * (a2 - a1) / q - 2 * ux[i] * s / b1 + 2 * ux[i] * s / b2;
    dvx[i] = -s / b2;
    dvxy[i] = 2 * a1 / q;
  }
  filt(dux, f1, tmp, h, w, c, win);
  filt(dvx, f2, tmp, h, w, c, win);
  filt(dvxy, t1, tmp, h, w, c, win);
  for (int64_t i = 0; i < n; i++) grad[i] = (f1[i] + 2 * x[i] * f2[i] + y[i] * t1[i]) / (double)n;
  free(buf);
  return total / (double)n;
}

/* transmittance_mask / _mask_derivative (losses.py:79-100); variant codes:
   0 sigmoid, 1 identity_t, 2 constant_one, 3 constant_zero. */
static double mask_val(double t, double k, int variant) {
  switch (variant) {
    case 0: return 1.0 / (1.0 + exp(-k * (t - 0.5)));
    case 1: return t;
    case 2: return 1.0;
    default: return 0.0;
  }
}
static double mask_der(double t, double k, int variant) {
  if (variant == 0) { double m = 1.0 / (1.0 + exp(-k * (t - 0.5))); return k * m * (1.0 - m); }
  if (variant == 1) return 1.0;
  return 0.0;
}

void or_transmittance_mask(int64_t n, const double* t, double k, int variant, double* out) {
  for (int64_t i = 0; i < n; i++) out[i] = mask_val(t[i], k, variant);
}

/* texture_loss (losses.py:103-116): returns L_t; writes grad_im (P,3) and grad_t (P). */
double or_texture_loss(int64_t npix, const double* i_gt, const double* i_m, const uint8_t* covered, const double* t,
                       double k, int variant, double* grad_im, double* grad_t) {
  int64_t n = 0;
  for (int64_t p = 0; p < npix; p++) n += covered[p] ? 1 : 0;
  if (n == 0) {
    memset(grad_im, 0, sizeof(double) * 3 * (size_t)npix);
    memset(grad_t, 0, sizeof(double) * (size_t)npix);
    return 0.0;
  }
  double acc = 0.0;
  for (int64_t p = 0; p < npix; p++) {
    double mk = mask_val(t[p], k, variant);
    double d[3], sq = 0.0;
    for (int ch = 0; ch < 3; ch++) { d[ch] = covered[p] ? i_m[3 * p + ch] - i_gt[3 * p + ch] : 0.0; }
    sq = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2];
    if (covered[p]) acc += mk * sq;
    for (int ch = 0; ch < 3; ch++) grad_im[3 * p + ch] = (2.0 / (double)n) * mk * d[ch];
    grad_t[p] = covered[p] ? mask_der(t[p], k, variant) * sq / (double)n : 0.0;
  }
  return acc / (double)n;
}

/* l1_loss (losses.py:41-44) */
double or_l1(int64_t n, const double* pred, const double* target, double* grad) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; i++) {
    double d = pred[i] - target[i];
    acc += fabs(d);
    grad[i] = (d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0)) / (double)n;
  }
  return acc / (double)n;
}

/* ---------------------------------------------------------------------- */
/* Adam.step (train/adam.py:28-42), one group                               */
/* ---------------------------------------------------------------------- */
void or_adam(int64_t n, double* p, double* m, double* v, const double* g, double lr, double beta1, double beta2,
             double eps, int64_t step) {
  double b1c = 1.0 - pow(beta1, (double)step);
  double b2c = 1.0 - pow(beta2, (double)step);
  for (int64_t i = 0; i < n; i++) {
    m[i] *= beta1;
    m[i] += (1.0 - beta1) * g[i];
    v[i] *= beta2;
    v[i] += (1.0 - beta2) * g[i] * g[i];
    p[i] -= lr * (m[i] / b1c) / (sqrt(v[i] / b2c) + eps);
  }
}

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
