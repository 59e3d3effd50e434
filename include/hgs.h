/*
 * hgs.h -- C ABI of libhgs.so, the B200 (sm_100a) hybrid Gaussian-splat +
 * textured-mesh renderer.  This is the drop-in boundary: every entry point
 * replaces one function of the reference operator API (gsmesh 0.1.0,
 * /root/reference/pkg/src/gsmesh; file:line cited per function).  The
 * reference's own "FFI" is the Numba kernel ABI (flat C-contiguous arrays,
 * outputs preallocated by the Python wrapper and mutated in place); this ABI
 * keeps that shape: plain device pointers + sizes, caller-owned outputs,
 * explicit stream, int status.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless the parameter says "host".
 *  - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *    and stream-ordered; nothing synchronises unless stated.
 *  - Return 0 on success; HGS_ERR_INVALID for argument errors (the Python
 *    layer raises ValueError, like the reference's shape checks);
 *    HGS_ERR_CUDA for launch/runtime errors (RuntimeError).  hgs_last_error()
 *    returns the message of the last failure on the calling thread.
 *  - Parameters are fp32 (N x 3 etc., row-major).  Every decision the
 *    reference makes (culling, tile rectangles, depth order, blend
 *    skip/clamp/stop, z-buffer, texel taps) is computed in fp64.
 */
#ifndef HGS_H_
#define HGS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HGS_OK 0
#define HGS_ERR_INVALID 1
#define HGS_ERR_CUDA 2

#define HGS_ABI_VERSION 1
#define HGS_TILE_DIFF_COPIES 16
/* fp32 words per row of hgs_projected.cull */
#define HGS_CULL_FLOATS 12

/* Pinhole camera, Camera (scene.py:144-203).  Derived fields are computed by
   the host exactly as the reference computes them:
   center = -R^T t (scene.py:190-192); limx/limy = 1.3 * (W / (2 fx))
   (splat/project.py:97-98). */
typedef struct hgs_camera {
  double fx, fy, cx, cy;
  int64_t width, height;
  double R[9]; /* world_to_camera[:3,:3], row-major */
  double T[3]; /* world_to_camera[:3,3] */
  double near_, far_;
  double center[3];
  double limx, limy;
} hgs_camera;

/* GaussianSet (scene.py:37-57): fp32 device arrays, N rows.
   colors_rest (N,3,3) [i][k][c] may be NULL (SH degree 0). */
typedef struct hgs_gaussians {
  const float* centers;     /* N x 3 */
  const float* rotations;   /* N x 4 (w,x,y,z), not necessarily unit */
  const float* log_scales;  /* N x 3 */
  const float* logits;      /* N */
  const float* colors_dc;   /* N x 3 */
  const float* colors_rest; /* N x 3 x 3 or NULL */
  int64_t n;
} hgs_gaussians;

/* Mutable parameter rows (same layout as hgs_gaussians): the outputs of
   density control (parameters and the Adam moments that move with them). */
typedef struct hgs_gaussian_buf {
  float* centers;
  float* rotations;
  float* log_scales;
  float* logits;
  float* colors_dc;
  float* colors_rest; /* NULL iff the input has no colors_rest */
  int64_t n;
} hgs_gaussian_buf;

/* Mutable twin of hgs_gaussians for parameter gradients (same layout). */
typedef struct hgs_gaussian_grads {
  float* centers;
  float* rotations;
  float* log_scales;
  float* logits;
  float* colors_dc;
  float* colors_rest; /* NULL iff colors_rest is NULL */
  float* densify_norm; /* N, may be NULL */
  uint8_t* visible;    /* N, may be NULL */
  float* visible_count; /* N, may be NULL: += 1 where visible (density-control denominator,
                           densify.py:31-33) */
} hgs_gaussian_grads;

/* Per-Gaussian projection state, indexed by ORIGINAL row (uncompacted).
   rec: N x 80 B fp64 blend records {mean2d x,y; conic xx, 2*xy, yy; alpha;
   depth; colour r,g,b} (the xy term is stored doubled, an exact scaling:
   kernels.py:44 multiplies it by 2.0 first).  count[i] = tile count (tiles.py:45-50), 0 iff the
   row is culled by project (project.py:80-83,118-119).  The optional fields
   (NULL to skip) are ProjectedGaussians extras (project.py:38-50). */
typedef struct hgs_projected {
  void* rec;
  int32_t* count;
  uint16_t* rect; /* N x 4: x0, x1, y0, y1 (inclusive tile rectangle) */
  double* cov2d;     /* N x 3, optional */
  double* radius;    /* N, optional */
  double* t_cam;     /* N x 3, optional */
  double* color_pre; /* N x 3, optional */
  double* view_dir;  /* N x 3, optional (SH degree 1 only) */
  double* view_dist; /* N, optional (SH degree 1 only) */
  void* cull;        /* N x 48 B fp32 (HGS_CULL_FLOATS) {mean x, mean y, 3-sigma half extents x, y;
                        conic xx, xy, yy, depth; alpha (negated: ill-conditioned conic, always evaluated
                        exactly), r, g, b}: blend culling + fast-path records (optional; without it
                        hgs_blend_forward runs the exact per-pixel walk only) */
  uint64_t* sort_keys; /* N: fp64 depth bit pattern of visible rows, ~0 for culled rows (required by
                          hgs_build_tiles) */
  int32_t* tile_diff;  /* HGS_TILE_DIFF_COPIES x (tiles_x + 1) x (tiles_y + 1) 2D difference grids of the rows'
                          tile rectangles (required by hgs_build_tiles; hgs_preprocess zeroes and fills it) */
} hgs_projected;

/* TileBins (splat/tiles.py:19-32).  entries hold ORIGINAL Gaussian rows in
   (tile, depth, row) order == np.lexsort((kept, depth, tile)) (tiles.py:65).
   counters (device, int64[4]): [0] M visible rows, [1] K entries, [2]
   overflow flag (K > capacity; entries/tile_starts are then invalid).  All
   counts stay on the device, so a frame can be enqueued (or captured into a
   CUDA graph) without a host round trip; on overflow the binning scatter,
   hgs_blend_forward, hgs_blend_backward and hgs_render_depth read the flag
   and do nothing (no access past `entries`): grow the buffer to >= K and
   re-enqueue. */
typedef struct hgs_tiles {
  int32_t tiles_x, tiles_y, tile_px;
  int32_t flags;        /* HGS_TILES_BLEND_ONLY (binned tile grids): hgs_build_tiles stops at the coarse
                           (super-tile) lists and does not write `entries`; hgs_blend_forward reads each
                           tile's list straight from its super-tile's coarse list.  For a renderer that
                           only needs the images (no backward, no TileBins): the blend reads only the
                           prefix of every list it walks before T falls under 1e-4 */
  int64_t capacity;
  uint32_t* entries;    /* capacity */
  int64_t* tile_starts; /* tiles_x * tiles_y + 1 */
  int64_t* counters;    /* 4 */
  void* scratch;
  size_t scratch_bytes; /* >= hgs_tiles_scratch_bytes(n, capacity, tiles) */
  int32_t* ready;       /* device int32[HGS_READY_INTS] or NULL: hgs_build_tiles publishes each finished block of
                           4x4 tiles here and hgs_blend_forward claims tiles in that order, starting while the
                           last blocks are still being binned (NULL: the blend waits for the whole binning) */
  void* join_event;     /* cudaEvent_t or NULL: hgs_build_tiles makes its last (fine binning) kernel wait for it.
                           Joins an independent branch the blend needs (the mesh layer) there, so that the blend
                           itself has the fine binning as its only dependency and can start programmatically */
  const void* coarse_rows;   /* written by hgs_build_tiles (binned grids): the super-tile lists of original rows */
  const void* coarse_rects;  /* ... their tile rectangles (u16 x 4) */
  const void* coarse_starts; /* ... and the lists' starts (u32, one per super-tile + 1) */
  void* coarse_prog;         /* ... and a per-tile scratch the blend-only blend leaves its list progress in */
} hgs_tiles;
#define HGS_TILES_BLEND_ONLY 1
#define HGS_READY_INTS (2 + 2048)

/* MeshLayer (splat/render.py:26-41).  color == NULL means "no mesh". */
typedef struct hgs_mesh_layer {
  const float* color;          /* H x W x 3 */
  const double* depth;         /* H x W, +inf where uncovered */
  const int32_t* triangle_id;  /* H x W, -1 where uncovered */
} hgs_mesh_layer;

/* rasterize_forward outputs (splat/render.py:90-109). */
typedef struct hgs_blend_out {
  float* color;         /* H x W x 3 */
  float* depth;         /* H x W (NaN where undefined) */
  float* transmittance; /* H x W */
  double* final_t;      /* H x W fp64 residual T, backward state (may be NULL) */
  int32_t* last;        /* H x W global entry index or -1 (may be NULL) */
  float* mask;          /* H x W transmittance_mask(T) (losses.py:79-91), may be NULL */
  int64_t* stats;       /* device int64[3]: += evaluations walked, += blended, += pixels handed to the exact fp64
                           walk (may be NULL) */
  int32_t* fixup;       /* device int32[H*W + 4] scratch, ZERO at first use (the call leaves it zero again):
                           the queue of pixels the fast path hands to the exact fp64 walk (may be NULL: exact
                           walk for every pixel) */
} hgs_blend_out;

/* TexturedMesh geometry (scene.py:206-237). */
typedef struct hgs_mesh {
  const float* vertices;    /* V x 3 */
  const int32_t* triangles; /* F x 3 */
  const float* uvs;         /* F x 3 x 2 or NULL */
  int64_t n_vertices, n_faces;
} hgs_mesh;

/* MeshFragmentBuffer (meshraster.py:25-42), H x W. */
typedef struct hgs_fragments {
  int32_t* triangle_id; /* -1 uncovered */
  double* depth;        /* +inf uncovered */
  double* bary;         /* H x W x 3, may be NULL */
  double* uv;           /* H x W x 2 */
} hgs_fragments;

/* One parameter group of the fused Adam step (train/adam.py:28-42). */
typedef struct hgs_adam_group {
  float* param;
  float* m;
  float* v;
  const float* grad;
  int64_t n;
  float lr;
  int32_t mode; /* 0 plain; 1 renormalise rows of 4 (loop.py:139-140); 2 clamp [0,1] (loop.py:144-145) */
} hgs_adam_group;

#define HGS_MAX_ADAM_GROUPS 8

/* ---------------- library ---------------- */
const char* hgs_last_error(void);
int hgs_abi_version(void);
int hgs_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);
/* number of kernels this library has launched (or enqueued into a graph) */
int64_t hgs_kernel_launches(void);
/* CUDA-graph helpers (host layer): instantiate a captured cudaGraph_t, with
   use_node_priority the kernel nodes keep the priority of the stream they
   were captured from (cudaGraphInstantiateFlagUseNodePriority); launch;
   destroy. */
int hgs_graph_instantiate(void* graph, int32_t use_node_priority, void** exec_out);
int hgs_graph_launch(void* exec, void* stream);
int hgs_graph_exec_destroy(void* exec);

/* ---------------- splat forward ---------------- */

/* project (splat/project.py:70-140) + evaluate_colors (:56-67) + per-row
   tile rectangle/count (splat/tiles.py:45-50).  cam is a DEVICE pointer;
   width/height (host) must equal cam->width/height. */
int hgs_preprocess(const hgs_camera* cam, int32_t width, int32_t height, const hgs_gaussians* gs, int32_t tile_px,
                   hgs_projected* out, void* stream);

/* build_tiles (splat/tiles.py:35-69): visible-row compaction, fp64 depth
   radix sort, tile-entry emission in depth order, stable tile radix sort,
   CSR ranges.  All counts stay on the device (tiles->counters).  proj must
   come from hgs_preprocess with sort_keys and tile_diff set. */
size_t hgs_tiles_scratch_bytes(int64_t n, int64_t capacity, int32_t n_tiles);
int hgs_build_tiles(const hgs_projected* proj, int64_t n, hgs_tiles* tiles, void* stream);

/* rasterize_forward (splat/render.py:74-109) / forward_kernel
   (splat/kernels.py:12-74), with the transmittance mask epilogue
   (train/losses.py:79-91; variant 0 sigmoid,1 identity_t,2 one,3 zero). */
int hgs_blend_forward(const hgs_projected* proj, const hgs_tiles* tiles, int32_t width, int32_t height,
                      const hgs_mesh_layer* mesh, const double* bg_host3, int32_t mask_variant, double mask_k,
                      hgs_blend_out* out, void* stream);

/* render_depth (splat/render.py:316-324) / depth_kernel
   (splat/kernels.py:163-202): per pixel, the depth of the entry at which the
   accumulated opacity first exceeds 0.5, NaN where it never does (no mesh
   layer).  out_depth: H x W fp64. */
int hgs_render_depth(const hgs_projected* proj, const hgs_tiles* tiles, int32_t width, int32_t height,
                     double* out_depth, void* stream);

/* ---------------- splat backward ---------------- */

/* backward_kernel (splat/kernels.py:77-160) + np.add.at reduction
   (splat/render.py:155-157): accumulates per-row screen gradients into
   screen_grads (N x 9 fp64, caller-zeroed): mean2d 2, cov 3 (full-matrix
   convention), alpha, rgb 3.  mesh_color_grad (may be NULL) receives
   grad_color * T * valid (render.py:180-181), accumulated when
   accumulate_mesh != 0. */
int hgs_blend_backward(const hgs_projected* proj, const hgs_tiles* tiles, int32_t width, int32_t height,
                       const hgs_mesh_layer* mesh, const double* bg_host3, const double* final_t,
                       const int32_t* last, const float* grad_color, const float* grad_t, double* screen_grads,
                       float* mesh_color_grad, int32_t accumulate_mesh, void* stream);

/* _chain_to_parameters (splat/render.py:185-313) + densify statistic and
   visibility (render.py:171-178).  Writes (accumulate=0) or adds
   (accumulate=1) scale * d/dparam into grads; densify_norm is written or
   added the same way. */
int hgs_project_backward(const hgs_camera* cam, const hgs_gaussians* gs, const hgs_projected* proj,
                         const double* screen_grads, hgs_gaussian_grads* grads, float scale, int32_t accumulate,
                         void* stream);

/* ---------------- mesh ---------------- */

/* rasterize_fragments (meshraster.py:119-136) / _raster_kernel (:45-116):
   z-buffer with the reference's (depth, triangle index) resolution,
   top-left rule, near-plane cull, perspective-correct bary/uv. */
size_t hgs_raster_scratch_bytes(int64_t n_vertices, int64_t n_faces, int32_t width, int32_t height);
int hgs_rasterize_fragments(const hgs_camera* cam, int32_t width, int32_t height, const hgs_mesh* mesh,
                            hgs_fragments* out, void* scratch, size_t scratch_bytes, void* stream);

/* sample_texture (meshraster.py:139-166): bilinear, clamp-to-edge, invalid
   pixels -> 0.  texture is Ht x Wt x 3 fp32. */
int hgs_sample_texture(const float* texture, int32_t th, int32_t tw, const double* uv, const int32_t* triangle_id,
                       int64_t npix, float* out, void* stream);

/* texture_backward (meshraster.py:169-184): bilinear adjoint, added into
   grad_texture (Ht x Wt x 3 fp32). */
int hgs_texture_backward(const double* uv, const int32_t* triangle_id, const float* grad_image, int64_t npix,
                         int32_t th, int32_t tw, float* grad_texture, void* stream);
/* Deterministic texture_backward for accumulation over many views: adds the
   taps' contributions into acc (int64[th*tw*3], zero at start) as 2^-32 fixed
   point -- integer atomics, so the sum is independent of their order.
   hgs_fixed_to_float converts acc to fp32 (out = value, or out += value with
   accumulate) and zeroes acc. */
int hgs_texture_backward_fixed(const double* uv, const int32_t* triangle_id, const float* grad_image, int64_t npix,
                               int32_t th, int32_t tw, int64_t* acc, void* stream);
int hgs_fixed_to_float(int64_t* acc, int64_t n, float* out, int32_t accumulate, void* stream);

/* ---------------- losses (train/losses.py) ---------------- */

/* transmittance_mask (losses.py:79-91). */
int hgs_transmittance_mask(const float* t, int64_t n, double k, int32_t variant, float* out, void* stream);

/* composite_loss (losses.py:139-174): L1 (:41-44) + D-SSIM (:47-76,
   11-tap sigma 1.5 zero-padded) + texture loss (:103-116) when
   texture_active.  Writes grad_ih (H x W x 3), grad_im (if non-NULL and
   texture_active), grad_t (H x W) and, into scalars (device double[6]):
   l1, dssim, l_c, l_t, total, mean_T_on_mesh.  grads are scaled by
   grad_scale (1 for the reference semantics). */
size_t hgs_loss_scratch_bytes(int32_t height, int32_t width);
int hgs_composite_loss(const float* i_gt, const float* i_h, const float* i_m, const int32_t* triangle_id,
                       const float* t, int32_t height, int32_t width, double lam_dssim, int32_t texture_active,
                       double texture_weight, double mask_k, int32_t mask_variant, const double* window11_host,
                       double grad_scale, float* grad_ih, float* grad_im, float* grad_t, double* scalars,
                       void* scratch, size_t scratch_bytes, void* stream);

/* ---------------- optimiser ---------------- */

/* Adam.step (train/adam.py:28-42) over up to HGS_MAX_ADAM_GROUPS groups in
   one launch, with quaternion renormalisation (loop.py:139-140) and texture
   clamp (loop.py:144-145) fused.  step is the post-increment step count;
   grads are multiplied by grad_scale first (view-batch mean). */
int hgs_adam_step(const hgs_adam_group* groups_host, int32_t n_groups, int64_t step, float beta1, float beta2,
                  float eps, float grad_scale, void* stream);

/* ---------------- adaptive density control ---------------- */

/* densify_and_prune (train/densify.py:46-94) + Adam.append_rows /
   prune_rows (train/adam.py:44-60) as a device stream compaction.
   hgs_densify_plan: per-row clone / split / prune decisions (fp64: average
   screen-gradient norm > grad_threshold, max scale <= scale_limit (=
   percent_dense * extent), sigmoid(logit) < prune_alpha) and prefix counts;
   writes counts_host[7] = {cloned, split, pruned, n_after, kept originals,
   kept clones, kept split rows} (synchronises the stream: n_after sizes the
   caller's new buffers).  hgs_densify_apply: writes the new rows -- kept
   originals, clones, then two children per split row (np.repeat order), each
   group of the parameters and of both Adam moments (zeros for appended rows);
   split children get centre + R(q) (n * exp(log_scales)) and log_scales -
   log(1.6), n = split_normals rows 2s, 2s + 1 for the s-th split row (the
   reference's rng.normal(0, 1, (2 n_split, 3)) draw); accum_out / denom_out
   (n_after doubles each, may be NULL) are zeroed: the fresh DensifyState
   (densify.py:92).  Replaces densify.py:46-94 / adam.py:44-60. */
size_t hgs_densify_scratch_bytes(int64_t n);
int hgs_densify_plan(const hgs_gaussians* gs, const double* grad_accum, const double* denom, double grad_threshold,
                     double scale_limit, double prune_alpha, void* scratch, size_t scratch_bytes, int64_t* counts_host,
                     void* stream);
int hgs_densify_apply(const hgs_gaussians* gs, const hgs_gaussians* m, const hgs_gaussians* v,
                      const double* split_normals, const void* scratch, hgs_gaussian_buf* out, hgs_gaussian_buf* out_m,
                      hgs_gaussian_buf* out_v, double* accum_out, double* denom_out, void* stream);
/* DensifyState.update (densify.py:31-33) for a batch of views: where
   visible_count[i] > 0, grad_accum[i] += norm_sum[i] * norm_scale and
   denom[i] += visible_count[i]. */
int hgs_densify_accumulate(const float* visible_count, const float* norm_sum, double norm_scale, int64_t n,
                           double* grad_accum, double* denom, void* stream);
/* reset_opacity (densify.py:97-101): logit <- logit(min(sigmoid(logit),
   ceiling)), its Adam moments (m, v may be NULL) cleared. */
int hgs_reset_opacity(float* logits, float* m, float* v, int64_t n, double ceiling, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HGS_H_ */
