// Fused Adam step (gsmesh/train/adam.py:28-42) over up to 8 parameter groups
// in one launch, with the quaternion renormalisation of the trainer
// (train/loop.py:139-140) and the texture clamp (loop.py:144-145) fused in.
// fp32 parameters and moments; bias corrections in fp64.
#include "common.cuh"

namespace hgs {

struct AdamGroups {
  hgs_adam_group g[HGS_MAX_ADAM_GROUPS];
  int n;
};

__global__ void __launch_bounds__(256) adam_kernel(AdamGroups groups, float beta1, float beta2, float eps,
                                                   float inv_b1c, float inv_sqrt_b2c, float grad_scale) {
  const hgs_adam_group& G = groups.g[blockIdx.y];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (G.mode == 1) {  // rows of 4 (quaternions): update, then renormalise the row
    const int64_t rows = G.n / 4;
    for (int64_t r = t0; r < rows; r += stride) {
      float q[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int64_t i = 4 * r + k;
        const float g = G.grad[i] * grad_scale;
        const float m = beta1 * G.m[i] + (1.0f - beta1) * g;
        const float v = beta2 * G.v[i] + (1.0f - beta2) * g * g;
        G.m[i] = m;
        G.v[i] = v;
        q[k] = G.param[i] - G.lr * (m * inv_b1c) / (sqrtf(v) * inv_sqrt_b2c + eps);
      }
      const float nrm = sqrtf(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
#pragma unroll
      for (int k = 0; k < 4; k++) G.param[4 * r + k] = q[k] / nrm;
    }
    return;
  }
  for (int64_t i = t0; i < G.n; i += stride) {
    const float g = G.grad[i] * grad_scale;
    const float m = beta1 * G.m[i] + (1.0f - beta1) * g;
    const float v = beta2 * G.v[i] + (1.0f - beta2) * g * g;
    G.m[i] = m;
    G.v[i] = v;
    float p = G.param[i] - G.lr * (m * inv_b1c) / (sqrtf(v) * inv_sqrt_b2c + eps);
    if (G.mode == 2) p = fminf(fmaxf(p, 0.0f), 1.0f);
    G.param[i] = p;
  }
}

}  // namespace hgs

extern "C" int hgs_adam_step(const hgs_adam_group* groups_host, int32_t n_groups, int64_t step, float beta1,
                             float beta2, float eps, float grad_scale, void* stream) {
  using namespace hgs;
  if (!groups_host || n_groups <= 0 || n_groups > HGS_MAX_ADAM_GROUPS)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_adam_step: need 1..8 groups");
  if (step < 1) return hgs_set_error(HGS_ERR_INVALID, "hgs_adam_step: step counts from 1");
  AdamGroups gr{};
  int64_t maxn = 0;
  for (int i = 0; i < n_groups; i++) {
    gr.g[i] = groups_host[i];
    if (gr.g[i].n > 0 && (!gr.g[i].param || !gr.g[i].m || !gr.g[i].v || !gr.g[i].grad))
      return hgs_set_error(HGS_ERR_INVALID, "hgs_adam_step: null group pointer");
    if (gr.g[i].mode == 1 && gr.g[i].n % 4) return hgs_set_error(HGS_ERR_INVALID, "hgs_adam_step: quaternion group size");
    maxn = gr.g[i].n > maxn ? gr.g[i].n : maxn;
  }
  gr.n = n_groups;
  const double b1c = 1.0 - pow((double)beta1, (double)step);
  const double b2c = 1.0 - pow((double)beta2, (double)step);
  // p -= lr * (m / b1c) / (sqrt(v / b2c) + eps) == lr * m * (1/b1c) / (sqrt(v) / sqrt(b2c) + eps)
  const int blocks = (int)tmax<int64_t>(1, tmin<int64_t>(ceil_div(maxn, 256), 4 * NUM_SMS));
  dim3 grid(blocks, n_groups);
  adam_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(gr, beta1, beta2, eps, (float)(1.0 / b1c),
                                                      (float)(1.0 / sqrt(b2c)), grad_scale);
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}
