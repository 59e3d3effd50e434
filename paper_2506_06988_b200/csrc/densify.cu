// Adaptive density control on the device: densify_and_prune
// (gsmesh/train/densify.py:46-94) with the Adam row surgery it drives
// (train/adam.py:44-60), DensifyState.update (densify.py:31-33) and
// reset_opacity (densify.py:97-101).
//
// densify_and_prune is a stream compaction over the Gaussian rows.  The
// reference appends the clone rows, then the split children (two per split
// row, np.repeat order), then drops the split originals and every row whose
// opacity is below the prune threshold.  Every new row's position follows
// from per-row flags and exclusive prefix counts in row order:
//   kept original  i -> scan(keep_orig)[i]
//   kept clone     i -> #keep_orig + scan(keep_clone)[i]
//   split child  c, i -> #keep_orig + #keep_clone + 2 scan(keep_split)[i] + c
// and the normal sample of split child c of row i is row 2 scan(split)[i] + c
// of the caller's draw (the reference's rng.normal(0, 1, (2 n_split, 3))).
//   1. densify_flags_kernel: flags + per-block counts (512 rows per block,
//      five 12-bit counters packed in one 64-bit word)
//   2. densify_scan_kernel (1 CTA): block offsets, event counts, new N
//   3. (host allocates the new flat buffers, draws the split normals)
//   4. densify_apply_kernel: in-block ranks (packed block scans) + offsets ->
//      every row writes its kept copies: parameters, Adam m and v (zeros for
//      appended rows, as Adam.append_rows); split children get
//      R(q) (n * exp(log_scales)) + centre and log_scales - log(1.6) in fp64.
// HBM-bound: each row's 14 (+9) parameters and two moment rows are read
// once and written at most twice.
#include "common.cuh"

namespace hgs {

constexpr int DN_THREADS = 256;
constexpr int DN_ROWS_PER_THREAD = 2;
constexpr int DN_ROWS = DN_THREADS * DN_ROWS_PER_THREAD;  // per block
enum { F_CLONE = 0, F_SPLIT = 1, F_KEEP_ORIG = 2, F_KEEP_CLONE = 3, F_KEEP_SPLIT = 4, F_N = 5 };
constexpr int F_BITS = 12;  // > log2(DN_ROWS)

__device__ __forceinline__ uint32_t field(uint64_t packed, int f) {
  return (uint32_t)((packed >> (F_BITS * f)) & ((1u << F_BITS) - 1));
}

// flag byte (bit 0 clone, 1 split, 2 low opacity) -> one count per field
__device__ __forceinline__ uint64_t packed_of(uint8_t f) {
  const bool clone = f & 1, split = f & 2, low = f & 4;
  return ((uint64_t)clone << (F_BITS * F_CLONE)) | ((uint64_t)split << (F_BITS * F_SPLIT)) |
         ((uint64_t)(!split && !low) << (F_BITS * F_KEEP_ORIG)) |
         ((uint64_t)(clone && !low) << (F_BITS * F_KEEP_CLONE)) |
         ((uint64_t)(split && !low) << (F_BITS * F_KEEP_SPLIT));
}

// per-row decisions (densify.py:52-57, 82-84), fp64 as the reference
__device__ __forceinline__ uint8_t row_flags(const hgs_gaussians& gs, const double* __restrict__ accum,
                                            const double* __restrict__ denom, double thr, double scale_limit,
                                            double prune_alpha, int64_t i) {
  const double dn = denom[i];
  const double avg = dn > 0.0 ? accum[i] / dn : 0.0;
  const double s = fmax(fmax(exp((double)gs.log_scales[3 * i]), exp((double)gs.log_scales[3 * i + 1])),
                        exp((double)gs.log_scales[3 * i + 2]));
  const bool hot = avg > thr;
  const bool small = s <= scale_limit;
  const double alpha = 1.0 / (1.0 + exp(-(double)gs.logits[i]));
  const bool low = alpha < prune_alpha;
  return (uint8_t)((hot && small) | ((hot && !small) << 1) | (low << 2));
}

__global__ void __launch_bounds__(DN_THREADS) densify_flags_kernel(hgs_gaussians gs, const double* __restrict__ accum,
                                                                   const double* __restrict__ denom, double thr,
                                                                   double scale_limit, double prune_alpha,
                                                                   uint8_t* __restrict__ flags,
                                                                   uint64_t* __restrict__ bcount) {
  __shared__ uint64_t s_warp[8];
  const int64_t base = (int64_t)blockIdx.x * DN_ROWS;
  uint64_t c = 0;
#pragma unroll
  for (int j = 0; j < DN_ROWS_PER_THREAD; j++) {
    const int64_t i = base + j * DN_THREADS + threadIdx.x;
    if (i < gs.n) {
      const uint8_t f = row_flags(gs, accum, denom, thr, scale_limit, prune_alpha, i);
      flags[i] = f;
      c += packed_of(f);
    }
  }
  uint64_t tot;
  block_exclusive_scan<uint64_t>(c, s_warp, tot);
  if (threadIdx.x == 0) bcount[blockIdx.x] = tot;
}

// One CTA: exclusive block offsets per field (boff[f * nblk + b]) and the
// event counts: cloned, split, pruned, n_after, keep_orig, keep_clone,
// keep_split (densify.py:57-93 stats).
__global__ void __launch_bounds__(DN_THREADS) densify_scan_kernel(const uint64_t* __restrict__ bcount, int nblk,
                                                                  int64_t n0, uint32_t* __restrict__ boff,
                                                                  int64_t* __restrict__ counts) {
  __shared__ uint32_t s_warp[8];
  __shared__ uint32_t carry[F_N];
  if (threadIdx.x < F_N) carry[threadIdx.x] = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nblk; b0 += DN_THREADS) {
    const int b = b0 + threadIdx.x;
    const uint64_t p = b < nblk ? bcount[b] : 0ull;
    for (int f = 0; f < F_N; f++) {
      uint32_t tot;
      const uint32_t e = block_exclusive_scan<uint32_t>(field(p, f), s_warp, tot);
      if (b < nblk) boff[(size_t)f * nblk + b] = carry[f] + e;
      __syncthreads();
      if (threadIdx.x == 0) carry[f] += tot;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    const int64_t cl = carry[F_CLONE], sp = carry[F_SPLIT];
    const int64_t ko = carry[F_KEEP_ORIG], kc = carry[F_KEEP_CLONE], ks = carry[F_KEEP_SPLIT];
    const int64_t n_after = ko + kc + 2 * ks;
    counts[0] = cl;
    counts[1] = sp;
    counts[2] = (n0 + cl + 2 * sp - sp) - n_after;  // low among the rows that survive the split drop
    counts[3] = n_after;
    counts[4] = ko;
    counts[5] = kc;
    counts[6] = ks;
  }
}

template <int W>
__device__ __forceinline__ void copy_row(const float* __restrict__ src, float* __restrict__ dst, int64_t i, int64_t o) {
#pragma unroll
  for (int k = 0; k < W; k++) dst[W * o + k] = src[W * i + k];
}
template <int W>
__device__ __forceinline__ void zero_row(float* __restrict__ dst, int64_t o) {
#pragma unroll
  for (int k = 0; k < W; k++) dst[W * o + k] = 0.0f;
}

// all groups of row i of (params, m, v) -> row o of the outputs; moments
// copied (kept original) or zeroed (appended row, Adam.append_rows)
__device__ __forceinline__ void emit_row(const hgs_gaussians& p, const hgs_gaussians& m, const hgs_gaussians& v,
                                         const hgs_gaussian_buf& op, const hgs_gaussian_buf& om,
                                         const hgs_gaussian_buf& ov, int64_t i, int64_t o, bool moments) {
  copy_row<3>(p.centers, op.centers, i, o);
  copy_row<4>(p.rotations, op.rotations, i, o);
  copy_row<3>(p.log_scales, op.log_scales, i, o);
  copy_row<1>(p.logits, op.logits, i, o);
  copy_row<3>(p.colors_dc, op.colors_dc, i, o);
  if (p.colors_rest) copy_row<9>(p.colors_rest, op.colors_rest, i, o);
  const hgs_gaussians* src[2] = {&m, &v};
  const hgs_gaussian_buf* dst[2] = {&om, &ov};
#pragma unroll
  for (int t = 0; t < 2; t++) {
    const hgs_gaussians& s = *src[t];
    const hgs_gaussian_buf& d = *dst[t];
    if (moments) {
      copy_row<3>(s.centers, d.centers, i, o);
      copy_row<4>(s.rotations, d.rotations, i, o);
      copy_row<3>(s.log_scales, d.log_scales, i, o);
      copy_row<1>(s.logits, d.logits, i, o);
      copy_row<3>(s.colors_dc, d.colors_dc, i, o);
      if (p.colors_rest) copy_row<9>(s.colors_rest, d.colors_rest, i, o);
    } else {
      zero_row<3>(d.centers, o);
      zero_row<4>(d.rotations, o);
      zero_row<3>(d.log_scales, o);
      zero_row<1>(d.logits, o);
      zero_row<3>(d.colors_dc, o);
      if (p.colors_rest) zero_row<9>(d.colors_rest, o);
    }
  }
}

__global__ void __launch_bounds__(DN_THREADS) densify_apply_kernel(hgs_gaussians p, hgs_gaussians m, hgs_gaussians v,
                                                                   const double* __restrict__ normals,
                                                                   const uint8_t* __restrict__ flags,
                                                                   const uint32_t* __restrict__ boff, int nblk,
                                                                   const int64_t* __restrict__ counts,
                                                                   hgs_gaussian_buf op, hgs_gaussian_buf om,
                                                                   hgs_gaussian_buf ov, double* __restrict__ accum_out,
                                                                   double* __restrict__ denom_out) {
  __shared__ uint64_t s_warp[8];
  const int64_t base = (int64_t)blockIdx.x * DN_ROWS;
  const int64_t n_ko = counts[4], n_kc = counts[5];
  // the fresh DensifyState of the new rows (densify.py:92 state.reset), grid-stride
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < op.n; r += (int64_t)gridDim.x * blockDim.x) {
    if (accum_out) accum_out[r] = 0.0;
    if (denom_out) denom_out[r] = 0.0;
  }
  uint32_t off[F_N];
#pragma unroll
  for (int f = 0; f < F_N; f++) off[f] = boff[(size_t)f * nblk + blockIdx.x];
  uint64_t run = 0;  // packed counts of this block's earlier chunks
#pragma unroll
  for (int j = 0; j < DN_ROWS_PER_THREAD; j++) {
    const int64_t i = base + j * DN_THREADS + threadIdx.x;
    const uint8_t fl = i < p.n ? flags[i] : (uint8_t)0;
    const uint64_t mine = i < p.n ? packed_of(fl) : 0ull;
    uint64_t tot;
    const uint64_t rank = run + block_exclusive_scan<uint64_t>(mine, s_warp, tot);
    run += tot;
    if (i >= p.n) continue;
    const bool clone = fl & 1, split = fl & 2, low = fl & 4;
    if (!split && !low) emit_row(p, m, v, op, om, ov, i, off[F_KEEP_ORIG] + field(rank, F_KEEP_ORIG), true);
    if (clone && !low) emit_row(p, m, v, op, om, ov, i, n_ko + off[F_KEEP_CLONE] + field(rank, F_KEEP_CLONE), false);
    if (split && !low) {
      const int64_t s = off[F_SPLIT] + field(rank, F_SPLIT);
      const int64_t o0 = n_ko + n_kc + 2 * ((int64_t)off[F_KEEP_SPLIT] + field(rank, F_KEEP_SPLIT));
      // R(q) of the normalised quaternion (scene.py:126-141), stds =
      // exp(log_scales), children centre R (n * stds) + centre (densify.py:66-72)
      double q[4];
#pragma unroll
      for (int k = 0; k < 4; k++) q[k] = p.rotations[4 * i + k];
      const double nrm = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
      const double w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
      const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z),     2 * (x * z + w * y),
                           2 * (x * y + w * z),     1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                           2 * (x * z - w * y),     2 * (y * z + w * x),     1 - 2 * (x * x + y * y)};
      double sd[3];
#pragma unroll
      for (int k = 0; k < 3; k++) sd[k] = exp((double)p.log_scales[3 * i + k]);
      for (int c = 0; c < 2; c++) {
        const int64_t o = o0 + c;
        emit_row(p, m, v, op, om, ov, i, o, false);
        const double* nv = normals + 3 * (2 * s + c);
        const double smp[3] = {nv[0] * sd[0], nv[1] * sd[1], nv[2] * sd[2]};
#pragma unroll
        for (int r = 0; r < 3; r++) {
          const double d = (R[3 * r] * smp[0] + R[3 * r + 1] * smp[1]) + R[3 * r + 2] * smp[2];
          op.centers[3 * o + r] = (float)(d + (double)p.centers[3 * i + r]);
          op.log_scales[3 * o + r] = (float)((double)p.log_scales[3 * i + r] - 0.47000362924573558);  // log(1.6)
        }
      }
    }
  }
}

// DensifyState.update (densify.py:31-33) for a batch of views: visible_count
// views saw row i; norm_sum (x norm_scale) is the sum of their norms.
__global__ void densify_accumulate_kernel(const float* __restrict__ visible_count, const float* __restrict__ norm_sum,
                                          double norm_scale, int64_t n, double* __restrict__ accum,
                                          double* __restrict__ denom) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float vc = visible_count[i];
  if (vc > 0.0f) {
    accum[i] += (double)norm_sum[i] * norm_scale;
    denom[i] += (double)vc;
  }
}

// reset_opacity (densify.py:97-101): activated opacity clamped to <= ceiling,
// logit = log(a / (1 - a)), the group's Adam moments cleared
__global__ void reset_opacity_kernel(float* __restrict__ logits, float* __restrict__ m, float* __restrict__ v,
                                     int64_t n, double ceiling) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = fmin(1.0 / (1.0 + exp(-(double)logits[i])), ceiling);
  logits[i] = (float)log(a / (1.0 - a));
  if (m) m[i] = 0.0f;
  if (v) v[i] = 0.0f;
}

struct DensifyScratch {
  uint8_t* flags;
  uint64_t* bcount;
  uint32_t* boff;
  int64_t* counts;
  int nblk;
};

inline DensifyScratch densify_scratch(void* base, int64_t n) {
  DensifyScratch s;
  s.nblk = (int)((n + DN_ROWS - 1) / DN_ROWS);
  char* p = (char*)base;
  s.counts = (int64_t*)p;
  p += 8 * sizeof(int64_t);
  s.bcount = (uint64_t*)p;
  p += sizeof(uint64_t) * (size_t)s.nblk;
  s.boff = (uint32_t*)p;
  p += sizeof(uint32_t) * (size_t)F_N * s.nblk;
  p = (char*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
  s.flags = (uint8_t*)p;
  return s;
}

}  // namespace hgs

extern "C" size_t hgs_densify_scratch_bytes(int64_t n) {
  using namespace hgs;
  const int64_t nblk = (n + DN_ROWS - 1) / DN_ROWS;
  return 8 * sizeof(int64_t) + (sizeof(uint64_t) + F_N * sizeof(uint32_t)) * (size_t)nblk + 16 + (size_t)n;
}

extern "C" int hgs_densify_plan(const hgs_gaussians* gs, const double* grad_accum, const double* denom,
                                double grad_threshold, double scale_limit, double prune_alpha, void* scratch,
                                size_t scratch_bytes, int64_t* counts_host, void* stream) {
  using namespace hgs;
  if (!gs || !grad_accum || !denom || !scratch) return hgs_set_error(HGS_ERR_INVALID, "hgs_densify_plan: null argument");
  if (scratch_bytes < hgs_densify_scratch_bytes(gs->n))
    return hgs_set_error(HGS_ERR_INVALID, "hgs_densify_plan: scratch too small");
  cudaStream_t st = (cudaStream_t)stream;
  DensifyScratch s = densify_scratch(scratch, gs->n);
  if (gs->n > 0) {
    densify_flags_kernel<<<s.nblk, DN_THREADS, 0, st>>>(*gs, grad_accum, denom, grad_threshold, scale_limit,
                                                        prune_alpha, s.flags, s.bcount);
    HGS_CHECK_LAUNCH();
  }
  densify_scan_kernel<<<1, DN_THREADS, 0, st>>>(s.bcount, s.nblk, gs->n, s.boff, s.counts);
  HGS_CHECK_LAUNCH();
  if (counts_host) {  // the new row count sizes the caller's buffers: one small synchronous read
    cudaError_t e = cudaMemcpyAsync(counts_host, s.counts, 7 * sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return hgs_set_cuda_error(e, __FILE__, __LINE__);
  }
  return HGS_OK;
}

extern "C" int hgs_densify_apply(const hgs_gaussians* gs, const hgs_gaussians* m, const hgs_gaussians* v,
                                 const double* split_normals, const void* scratch, hgs_gaussian_buf* out,
                                 hgs_gaussian_buf* out_m, hgs_gaussian_buf* out_v, double* accum_out,
                                 double* denom_out, void* stream) {
  using namespace hgs;
  if (!gs || !m || !v || !scratch || !out || !out_m || !out_v)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_densify_apply: null argument");
  if ((gs->colors_rest == nullptr) != (out->colors_rest == nullptr))
    return hgs_set_error(HGS_ERR_INVALID, "hgs_densify_apply: colors_rest presence mismatch");
  if (gs->n == 0) return HGS_OK;
  DensifyScratch s = densify_scratch(const_cast<void*>(scratch), gs->n);
  densify_apply_kernel<<<s.nblk, DN_THREADS, 0, (cudaStream_t)stream>>>(*gs, *m, *v, split_normals, s.flags, s.boff,
                                                                       s.nblk, s.counts, *out, *out_m, *out_v,
                                                                       accum_out, denom_out);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}

extern "C" int hgs_densify_accumulate(const float* visible_count, const float* norm_sum, double norm_scale, int64_t n,
                                      double* grad_accum, double* denom, void* stream) {
  using namespace hgs;
  if (n == 0) return HGS_OK;
  if (!visible_count || !norm_sum || !grad_accum || !denom)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_densify_accumulate: null argument");
  densify_accumulate_kernel<<<ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(visible_count, norm_sum, norm_scale,
                                                                                 n, grad_accum, denom);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}

extern "C" int hgs_reset_opacity(float* logits, float* m, float* v, int64_t n, double ceiling, void* stream) {
  using namespace hgs;
  if (n == 0) return HGS_OK;
  if (!logits) return hgs_set_error(HGS_ERR_INVALID, "hgs_reset_opacity: null argument");
  reset_opacity_kernel<<<ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(logits, m, v, n, ceiling);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}
