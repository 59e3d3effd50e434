// Shared pieces of the blend forward (blend.cu) and backward (backward.cu)
// fast paths: the shared-memory stage entry streamed by a producer warp,
// mbarrier / cp.async helpers, the per-warp ellipse cull, and the fp32
// fast-path numerics with their guard bands.
#pragma once
#include "common.cuh"

namespace hgs {

constexpr double LOG2E = 1.4426950408889634;

struct __align__(16) StageEntry {
  double2 a;  // mean x, mean y               (BlendRec bytes 0..15)
  double2 b;  // conic xx, 2*xy               (16..31)
  double2 c;  // conic yy, depth              (32..47)
  double2 d;  // alpha, r (r unused here)     (48..63)
  CullRec f;  // fp32 box, conic + depth, alpha + colour
};
static_assert(sizeof(StageEntry) == 112, "stage entry is 112 B");

static __device__ const float4 g_empty_box = {0.0f, 0.0f, -1.0f, -1.0f};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait suspends the polling lane in hardware (until the phase completes
// or the hint expires) instead of spinning through issue slots
constexpr unsigned MBAR_SUSPEND_NS = 20000;
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "n"(MBAR_SUSPEND_NS)
      : "memory");
  return ok != 0;
}
// One lane polls (the loop is visible to the compiler, so the warp
// reconverges at the __syncwarp that publishes the acquired state).
__device__ __forceinline__ void warp_wait(unsigned long long* bar, unsigned parity, int lane) {
  if (lane == 0)
    while (!mbar_try_wait(bar, parity)) {
    }
  __syncwarp();
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Bulk (TMA engine) copy global -> shared of `bytes` (multiple of 16, both
// addresses 16-B aligned); completion is signalled as transaction bytes on
// the mbarrier, which the issuing thread announced with arrive_expect_tx.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Conservative test: does the ellipse {m <= mcut} reach any point of the
// box [x0,x1] x [y0,y1] (centre outside the box)?  mcut is recovered from
// the box half-width ex of the cull record (ex^2 = mcut cov_xx, cov_xx =
// c / (ac - b^2) for the conic (a, b, c)).  The minimum of the convex
// quadratic m over the box lies on an edge; each edge minimum is a clamped
// 1D vertex.  fp32 with a relative margin (sure misses only; the evaluation
// error is below 3e-4 relative for 1 - rho^2 >= 1e-3).
__device__ __forceinline__ float edge_min(float a, float b, float c, float u, float v0, float v1) {
  // m(u, v) = a u^2 + 2 b u v + c v^2 with u fixed, v in [v0, v1]
  const float v = fminf(fmaxf(__fdividef(-b * u, c), v0), v1);
  return a * u * u + 2.0f * b * u * v + c * v * v;
}
__device__ __forceinline__ bool ellipse_meets_box(float4 con, float4 box, float x0, float x1, float y0, float y1) {
  const float a = con.x, b = con.y, c = con.z;
  const float det = fmaf(a, c, -b * b);
  // poorly conditioned conic (1 - rho^2 < 1e-3): fp32 cannot bound m to the
  // margin -- keep the entry (the box test already passed)
  if (!(det >= 1e-3f * a * c)) return true;
  const float mcut = box.z * box.z * __fdividef(det, c);
  const float dx0 = x0 - box.x, dx1 = x1 - box.x, dy0 = y0 - box.y, dy1 = y1 - box.y;
  float mn = edge_min(a, b, c, dx0, dy0, dy1);
  mn = fminf(mn, edge_min(a, b, c, dx1, dy0, dy1));
  mn = fminf(mn, edge_min(c, b, a, dy0, dx0, dx1));
  mn = fminf(mn, edge_min(c, b, a, dy1, dx0, dx1));
  return mn <= fmaf(mcut, 1.002f, 0.01f);
}


// ---- fast-path numerics -------------------------------------------------
// exp2 argument u = m * log2(e)/2 (fp64), narrowed to fp32 round-to-nearest.
constexpr double U_SCALE = 0.5 * LOG2E;
constexpr float U9 = (float)(9.0 * 0.5 * LOG2E);
constexpr float U9_LO = U9 * (1.0f - 9.5367431640625e-7f);  // 2^-20 guard band around m = 9
constexpr float U9_BAND_INV = 1.0f / (U9 * 9.5367431640625e-7f);
// |sigma_fast / sigma_reference - 1| <= EPS_SIG: ex2.approx (2^-22) +
// argument (ln2 * 6.5 * 2^-24) + alpha narrowing and product (2 * 2^-24)
constexpr float EPS_SIG = 6.5e-7f;
constexpr float SKIP_F = (float)SIGMA_SKIP;
constexpr float SKIP_BAND_INV = 1.0f / (2.0f * EPS_SIG * SKIP_F);
constexpr float CLAMP_F = (float)ALPHA_CLAMP;
constexpr float STOP_F = (float)EARLY_STOP_T;
// T - 2 eT above this: the early-stop test is neither taken nor ambiguous
constexpr float STOP_NEAR = (float)(EARLY_STOP_T * 1.001);

// Distance of an entry's fast-path decisions from their thresholds, in
// units of the guard bands; <= 1 means "decide exactly".  A negative alpha
// (ill-conditioned conic, preprocess) forces the exact evaluation.  (The
// conic form of a well-conditioned conic is never negative, so m < 0 needs
// no separate test; alpha >= 1/255 > 1 band-unit is never a false flag.)
__device__ __forceinline__ float amb_key(float uu, float sgf, float a32) {
  const float k1 = fabsf(fmaf(uu, U9_BAND_INV, -U9 * U9_BAND_INV));
  const float k2 = fabsf(fmaf(sgf, SKIP_BAND_INV, -SKIP_F * SKIP_BAND_INV));
  return fminf(fminf(k1, k2), a32 * 1e4f);
}
// Cut form of the two blend decisions (support m <= 9 and skip
// sigma >= 1/255, the clamp at 0.99 > 1/255 never decides): an entry is
// blended iff u <= ucut = min(9 U, log2(255 alpha)) -- one compare per pixel.
// ucut is computed once per (warp, entry) from the fp32 alpha with
// lg2.approx (|err| <= 2^-22 relative of |log2| <= 8, plus alpha narrowing
// and the product: < 2.3e-6), u is the fp32-rounded fp64 argument
// (<= 6.5 * 2^-24), U9 its fp32 rounding: within U_BAND of the cut the entry
// is re-evaluated exactly.  An ill-conditioned conic (alpha < 0) gets a NaN
// cut: never "sure", always ambiguous.
constexpr float U_BAND = 8e-6f;
__device__ __forceinline__ float entry_ucut(float a32) {
  if (a32 < 0.0f) return __int_as_float(0x7fc00000);
  float l;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(255.0f * a32));
  return fminf(U9, l);
}
__device__ __forceinline__ float ex2_neg(float u) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-u));
  return e;
}

// ---- fp64 sigma for the training state ---------------------------------
// The backward reconstructs T before every entry from the final T of the
// forward, so the final T and the per-entry sigma it is built from must be
// accurate far beyond fp32 for the gradients to hold the 1e-4 absolute
// contract at |g| ~ 4e2 (measured: fp32 T / sigma leave 2.6e-4 at c3).
// 2^-u in fp64, u >= 0: u = k/N + r with k = floor(N uu) from the fp32
// argument (r in [-2^-20, 1/N)), 2^-r by a Taylor polynomial, 2^(-k/N) =
// table[k mod N] x 2^-(k / N) (an exact power of two, by the exponent field).
// Table size N = 2^HGS_EXP2_BITS: 256 entries x a degree-3 Taylor polynomial
// (default; 2 KB of shared memory), 64 x degree 4 or 16 x degree 5 -- all
// < 3e-12 relative (c4 step: 162.6 vs 164.4 ms with 16 entries).  The
// table (2^(-j/N), exact to 1 ulp from the device exp2) is built per CTA in
// shared memory.
#ifndef HGS_EXP2_BITS
#define HGS_EXP2_BITS 8
#endif
constexpr int EXP2_BITS = HGS_EXP2_BITS;
constexpr int EXP2_N = 1 << EXP2_BITS;
constexpr int EXP2_DEG = EXP2_BITS <= 4 ? 5 : (EXP2_BITS <= 6 ? 4 : 3);
__device__ __forceinline__ void exp2_tab_load(double* tab) {
  for (int j = threadIdx.x; j < EXP2_N; j += blockDim.x) tab[j] = exp2(-(double)j / EXP2_N);
}
// the polynomial's coefficients ((-ln 2)^k / k!, highest first) live in
// constant memory: DFMA reads them as c[][] operands (as immediates every use
// costs two uniform moves)
__constant__ double c_exp2_poly[6] = {-0.0013333558146428441, 0.009618129107628477, -0.055504108664821576,
                                      0.2402265069591007,     -0.6931471805599453,  1.0};
// Callers pass blended entries only: 0 <= u < 9 U (a tiny negative u, from
// rounding, gives k = -1 and still the right value: the table index wraps and
// the exponent step is -1), so the argument needs no clamp.
__device__ __forceinline__ double exp2_neg64(double u, float uu, const double* tab) {
  const int k = __float2int_rd(uu * (float)EXP2_N);
  const double r = fma((double)k, -1.0 / EXP2_N, u);
  double p = c_exp2_poly[5 - EXP2_DEG];
#pragma unroll
  for (int d = 6 - EXP2_DEG; d < 6; d++) p = fma(p, r, c_exp2_poly[d]);
  const double t = p * tab[k & (EXP2_N - 1)];  // in (0.5, 1.03]: x 2^-(k >> BITS) by the exponent field
  return __hiloint2double(__double2hiint(t) - ((k >> EXP2_BITS) << 20), __double2loint(t));
}
// 1 / x for x in [0.01, 1] in fp64: SFU estimate from the high word
// (relative error < 2^-19) + one Newton step (< 2^-38: far below what the
// gradients need, ~1e-9)
__device__ __forceinline__ double rcp64(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

}  // namespace hgs
