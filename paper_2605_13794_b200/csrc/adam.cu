// NEXT-3: the optimizer step on the owned shard, fused with the parameter
// activations (bgs_adam_step).
//
// Each rank stores its shard's RAW parameters and their Adam state ("Each GPU stores only
// its local shard and its optimizer state").  The rendering ABI takes ACTIVATED parameters (R13),
// so one pass per row: gradient w.r.t. the activated parameter -> chain rule through the
// activation (opacity = sigmoid(logit), s = exp(log s), q = q_raw / |q_raw|; mean and SH are
// identity) -> Adam (bias-corrected, per-group learning rates, reading R38) -> raw parameter and
// moments written back -> activated planes written for the next render -> gradient zeroed (the
// accumulation buffers of the next step), so no separate memset or activation pass reads the
// shard again.  Rows whose bit in `visible` is 0 are skipped entirely (selective Adam, optional).
//
// Layout: the three 16-byte planes are handled one row per thread (128-bit loads); the SH plane
// (48 floats per row) as a flat float4 array, one float4 per thread (coefficient 0 = the first
// three floats of a row takes lr_sh_dc, the rest lr_sh_rest).
#include "bgs_internal.cuh"

namespace bgs {
namespace {

constexpr int kAdamThreads = 256;

__device__ __forceinline__ float adam1(float& p, float& m, float& v, float g, float lr, const AdamArgs& a) {
  // 1 - beta comes from the host in double precision: 1.f - 0.999f is 1.3e-5 off 0.001
  m = a.b1 * m + a.om1 * g;
  v = a.b2 * v + a.om2 * (g * g);
  p -= lr * (m * a.c1) / (sqrtf(v * a.c2) + a.eps);
  return p;
}

__device__ __forceinline__ bool row_visible(const uint32_t* vis, int64_t i) {
  return !vis || ((__ldg(vis + (i >> 5)) >> (i & 31)) & 1u);
}

__global__ void __launch_bounds__(kAdamThreads) k_adam_rows(AdamArgs a) {
  const int64_t i = int64_t(blockIdx.x) * kAdamThreads + threadIdx.x;
  if (i >= a.n || !row_visible(a.visible, i)) return;
  // mean + opacity logit
  {
    float4 p = a.p[0][i], m = a.m[0][i], v = a.v[0][i];
    const float4 g = a.g[0][i];
    const float o = 1.f / (1.f + __expf(-p.w));  // current activated opacity
    adam1(p.x, m.x, v.x, g.x, a.lr_mean, a);
    adam1(p.y, m.y, v.y, g.y, a.lr_mean, a);
    adam1(p.z, m.z, v.z, g.z, a.lr_mean, a);
    adam1(p.w, m.w, v.w, g.w * o * (1.f - o), a.lr_opacity, a);
    a.p[0][i] = p;
    a.m[0][i] = m;
    a.v[0][i] = v;
    a.act[0][i] = make_float4(p.x, p.y, p.z, 1.f / (1.f + __expf(-p.w)));
    a.g[0][i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // rotation: dL/dq_raw = (g - qhat (qhat . g)) / |q_raw|
  {
    float4 p = a.p[1][i], m = a.m[1][i], v = a.v[1][i];
    const float4 g = a.g[1][i];
    const float nrm = sqrtf(p.x * p.x + p.y * p.y + p.z * p.z + p.w * p.w);
    const float inv = 1.f / nrm;
    const float4 qh = make_float4(p.x * inv, p.y * inv, p.z * inv, p.w * inv);
    const float d = qh.x * g.x + qh.y * g.y + qh.z * g.z + qh.w * g.w;
    adam1(p.x, m.x, v.x, (g.x - qh.x * d) * inv, a.lr_quat, a);
    adam1(p.y, m.y, v.y, (g.y - qh.y * d) * inv, a.lr_quat, a);
    adam1(p.z, m.z, v.z, (g.z - qh.z * d) * inv, a.lr_quat, a);
    adam1(p.w, m.w, v.w, (g.w - qh.w * d) * inv, a.lr_quat, a);
    a.p[1][i] = p;
    a.m[1][i] = m;
    a.v[1][i] = v;
    const float in2 = 1.f / sqrtf(p.x * p.x + p.y * p.y + p.z * p.z + p.w * p.w);
    a.act[1][i] = make_float4(p.x * in2, p.y * in2, p.z * in2, p.w * in2);
    a.g[1][i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // scale: dL/dlog s = dL/ds * s
  {
    float4 p = a.p[2][i], m = a.m[2][i], v = a.v[2][i];
    const float4 g = a.g[2][i];
    adam1(p.x, m.x, v.x, g.x * __expf(p.x), a.lr_scale, a);
    adam1(p.y, m.y, v.y, g.y * __expf(p.y), a.lr_scale, a);
    adam1(p.z, m.z, v.z, g.z * __expf(p.z), a.lr_scale, a);
    a.p[2][i] = p;
    a.m[2][i] = m;
    a.v[2][i] = v;
    a.act[2][i] = make_float4(__expf(p.x), __expf(p.y), __expf(p.z), 0.f);
    a.g[2][i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// SH: 12 float4 per row; float4 k of row i holds coefficients floats 4k..4k+3 of the row
__global__ void __launch_bounds__(kAdamThreads) k_adam_sh(AdamArgs a) {
  const int64_t e = int64_t(blockIdx.x) * kAdamThreads + threadIdx.x;
  if (e >= a.n * 12) return;
  const int64_t i = e / 12;
  if (!row_visible(a.visible, i)) return;
  const int k = int(e - i * 12);
  float4* P = reinterpret_cast<float4*>(a.sh_p);
  float4* M = reinterpret_cast<float4*>(a.sh_m);
  float4* V = reinterpret_cast<float4*>(a.sh_v);
  float4* G = reinterpret_cast<float4*>(a.sh_g);
  float4 p = P[e], m = M[e], v = V[e];
  const float4 g = G[e];
  // floats 0..2 of a row are the DC coefficient (R, G, B)
  adam1(p.x, m.x, v.x, g.x, k == 0 ? a.lr_sh_dc : a.lr_sh_rest, a);
  adam1(p.y, m.y, v.y, g.y, k == 0 ? a.lr_sh_dc : a.lr_sh_rest, a);
  adam1(p.z, m.z, v.z, g.z, k == 0 ? a.lr_sh_dc : a.lr_sh_rest, a);
  adam1(p.w, m.w, v.w, g.w, a.lr_sh_rest, a);
  P[e] = p;
  M[e] = m;
  V[e] = v;
  if (a.sh_act && a.sh_act != a.sh_p) reinterpret_cast<float4*>(a.sh_act)[e] = p;
  G[e] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Visibility mask of a batch for selective Adam: bit i |= (radius[i] > 0), one ballot per warp
// and one 32-bit OR per word (views in flight may share the mask: atomicOr).
__global__ void __launch_bounds__(kAdamThreads) k_visibility_or(const int32_t* __restrict__ radius, int64_t n,
                                                                uint32_t* __restrict__ mask) {
  const int64_t i = int64_t(blockIdx.x) * kAdamThreads + threadIdx.x;
  const bool v = i < n && __ldg(radius + i) > 0;
  const uint32_t b = __ballot_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && b && i < n) atomicOr(mask + (i >> 5), b);
}

}  // namespace

void launch_visibility_or(const int32_t* radius, int64_t n, uint32_t* mask, cudaStream_t s) {
  if (n <= 0) return;
  k_visibility_or<<<unsigned((n + kAdamThreads - 1) / kAdamThreads), kAdamThreads, 0, s>>>(radius, n, mask);
}

void launch_adam(const AdamArgs& a, cudaStream_t s) {
  if (a.n <= 0) return;
  k_adam_rows<<<unsigned((a.n + kAdamThreads - 1) / kAdamThreads), kAdamThreads, 0, s>>>(a);
  k_adam_sh<<<unsigned((a.n * 12 + kAdamThreads - 1) / kAdamThreads), kAdamThreads, 0, s>>>(a);
}

}  // namespace bgs
