// a1 gate + a2 projection (bgs_project).
//
// PAPER.md §3.1 P:143-152 (Eq.1 Gaussian, EWA "projected to screen-space ellipses"), §3.2
// ("every GPU projects only its own local Gaussians"), §3.4 Eq.4-6 P:195-210 (LOD gate, cull).
//
// PINNED ARITHMETIC (D2): this translation unit is compiled with -fmad=false and
// IEEE div/sqrt so that every float expression of the exact projection rounds exactly as
// written; radius, rect, tile ids and pair counts are integers derived from these floats and
// must be bit-identical to the oracle's.  Expression trees are the ones listed in DESIGN.md §4.
//
// Three kernels:
//  k_cull (streaming, 4 Gaussians per thread, ~36 B read per Gaussian): the Eq.5 gate with its
//    per-rank fallback, the Eq.6 cull column, the near plane and a CONSERVATIVE analytic bound
//    on the splat radius; Gaussians that cannot produce a record get radius 0,
//    the rest are compacted into a candidate list (one global atomic per CTA).
//  k_project (candidates only): the exact pinned EWA projection, radius, rect; records are
//    compacted per CTA and written coalesced through shared memory (one atomic per CTA chunk).
//  k_color (records only): the 192-B SH row, 12 independent 128-bit loads per thread.
// Per-warp global atomics on one counter were a bottleneck earlier (hundreds of thousands of
// same-address atomics serialise at the L2): every counter here is touched once per CTA.
#include "bgs_internal.cuh"

#include <cstdlib>

namespace bgs {
namespace {

__device__ __forceinline__ float4 ldg4(const float4* p) { return __ldg(p); }

__device__ __forceinline__ bool lod_keep(const ProjectArgs& a, float4 mo, int l) {
  float dx = mo.x - a.cam.campos[0];
  float dy = mo.y - a.cam.campos[1];
  float dz = mo.z - a.cam.campos[2];
  float d2 = (dx * dx + dy * dy) + dz * dz;
  return (l <= a.l_max) && (l == 0 || d2 <= a.D2[l < 31 ? l : 31]);
}

__global__ void __launch_bounds__(256) k_gate_count(ProjectArgs a) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int ok = 0;
  if (i < a.n) ok = lod_keep(a, ldg4(a.mean_opac + i), a.lod[i]) ? 1 : 0;
  int c = __syncthreads_count(ok);
  if (threadIdx.x == 0 && c) atomicAdd(a.counters + C_NLOD, (unsigned long long)c);
}

// a1 + the off-screen bound.  `active`: passed the gate and the cull column (|A^(m)|).
// Returns whether the exact projection can produce a record.  The bound:
// radius <= 3 sqrt(|J|_F^2 s_max^2 + 0.3 + sqrt(0.1)) + 1 with |J|_F^2 <= K / tz^2
// (K = fx^2 (1 + Lx^2) + fy^2 (1 + Ly^2), L = clamp limits), widened by 1% + 2 px; a Gaussian
// whose centre is further than that outside the image has an empty rect in the exact
// computation too.  Approximate arithmetic is fine here: the margins dwarf its error.
__device__ __forceinline__ bool cull_test(const ProjectArgs& a, int64_t i, bool& active) {
  const bool filtered = a.gate_enabled || a.cull;
  float4 sc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!filtered) sc = ldg4(a.scale + i);  // nothing can drop it before the bound: load now
  const float4 mo = ldg4(a.mean_opac + i);
  bool keep = true;
  if (a.gate_enabled) {
    const unsigned long long nl = *((volatile unsigned long long*)(a.counters + C_NLOD));
    const bool fallback = (unsigned long long)a.fb_den * nl > (unsigned long long)a.fb_num * (unsigned long long)a.n;
    if (!fallback) keep = lod_keep(a, mo, a.lod[i]);
  }
  if (keep && a.cull) keep = !((__ldg(a.cull + (i >> 5)) >> (i & 31)) & 1u);
  active = keep;
  if (!keep) return false;
  if (filtered) sc = ldg4(a.scale + i);
  const CameraK& cm = a.cam;
  // same pinned expression as the exact path, so the near-plane decision is identical
  const float tz = ((cm.R[6] * mo.x + cm.R[7] * mo.y) + cm.R[8] * mo.z) + cm.t[2];
  if (!(tz > cm.near_clip)) return false;
  const float tx = ((cm.R[0] * mo.x + cm.R[1] * mo.y) + cm.R[2] * mo.z) + cm.t[0];
  const float ty = ((cm.R[3] * mo.x + cm.R[4] * mo.y) + cm.R[5] * mo.z) + cm.t[1];
  const float iz = __fdividef(1.0f, tz);
  const float mxb = cm.fx * (tx * iz) + cm.cx, myb = cm.fy * (ty * iz) + cm.cy;
  const float smax = fmaxf(sc.x, fmaxf(sc.y, sc.z));
  const float rb = 3.0f * sqrtf(a.cull_K * (smax * smax) * (iz * iz) + 0.62f) * 1.01f + 2.0f;
  return !(mxb + rb < 0.0f || mxb - rb > float(16 * cm.TX + 1) || myb + rb < 0.0f ||
           myb - rb > float(16 * cm.TY + 1));
}

struct ProjOut {
  float mx, my, A, B, C, depth, opac;
  float mux, muy, muz;  // parked in the record's colour slots for k_color
  uint32_t rect, area;
  bool valid;
  int x0, y0, x1, y1;
};

// The exact a2 projection of a candidate (passed the gate, the cull column and the bound).
__device__ __forceinline__ ProjOut project_exact(const ProjectArgs& a, int64_t i) {
  ProjOut o;
  o.valid = false;
  o.area = 0;
  o.x0 = o.y0 = o.x1 = o.y1 = 0;
  o.mx = o.my = o.A = o.B = o.C = o.depth = o.opac = o.mux = o.muy = o.muz = 0.f;
  int radius = 0;
  const float4 mo = ldg4(a.mean_opac + i);
  const float4 sc = ldg4(a.scale + i);
  const float4 q = ldg4(a.quat + i);
  const CameraK& cm = a.cam;
  // ---- t_c = R mu + t
  const float tx = ((cm.R[0] * mo.x + cm.R[1] * mo.y) + cm.R[2] * mo.z) + cm.t[0];
  const float ty = ((cm.R[3] * mo.x + cm.R[4] * mo.y) + cm.R[5] * mo.z) + cm.t[1];
  const float tz = ((cm.R[6] * mo.x + cm.R[7] * mo.y) + cm.R[8] * mo.z) + cm.t[2];
  const float txtz = tx / tz, tytz = ty / tz;
  if (tz > cm.near_clip) {
    // Sigma = R(q) S S^T R(q)^T
    const float xx = q.y * q.y, yy = q.z * q.z, zz = q.w * q.w;
    const float xy = q.y * q.z, xz = q.y * q.w, yz = q.z * q.w;
    const float wx = q.x * q.y, wy = q.x * q.z, wz = q.x * q.w;
    const float Rq[3][3] = {{1.0f - 2.0f * (yy + zz), 2.0f * (xy - wz), 2.0f * (xz + wy)},
                            {2.0f * (xy + wz), 1.0f - 2.0f * (xx + zz), 2.0f * (yz - wx)},
                            {2.0f * (xz - wy), 2.0f * (yz + wx), 1.0f - 2.0f * (xx + yy)}};
    const float s3[3] = {sc.x, sc.y, sc.z};
    float M[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) M[r][c] = Rq[r][c] * s3[c];
    float S[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) S[r][c] = (M[r][0] * M[c][0] + M[r][1] * M[c][1]) + M[r][2] * M[c][2];
    // EWA Jacobian with the 1.3 tan(fov/2) clamp (off-centre principal point); the four
    // per-camera limits are computed once on the host with the same float expressions
    const float lim_xp = a.lim[0], lim_xn = a.lim[1], lim_yp = a.lim[2], lim_yn = a.lim[3];
    const float ctx = fminf(lim_xp, fmaxf(-lim_xn, txtz)) * tz;
    const float cty = fminf(lim_yp, fmaxf(-lim_yn, tytz)) * tz;
    const float J00 = cm.fx / tz, J02 = -(cm.fx * ctx) / (tz * tz);
    const float J11 = cm.fy / tz, J12 = -(cm.fy * cty) / (tz * tz);
    float Tm[2][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      Tm[0][c] = J00 * cm.R[c] + J02 * cm.R[6 + c];
      Tm[1][c] = J11 * cm.R[3 + c] + J12 * cm.R[6 + c];
    }
    float U[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) U[r][c] = (Tm[r][0] * S[0][c] + Tm[r][1] * S[1][c]) + Tm[r][2] * S[2][c];
    float ca = (U[0][0] * Tm[0][0] + U[0][1] * Tm[0][1]) + U[0][2] * Tm[0][2];
    const float cb = (U[0][0] * Tm[1][0] + U[0][1] * Tm[1][1]) + U[0][2] * Tm[1][2];
    float cc = (U[1][0] * Tm[1][0] + U[1][1] * Tm[1][1]) + U[1][2] * Tm[1][2];
    ca = ca + 0.3f;
    cc = cc + 0.3f;
    const float det = ca * cc - cb * cb;
    if (det > 0.0f) {
      o.A = cc / det;
      o.B = (-cb) / det;
      o.C = ca / det;
      o.mx = cm.fx * txtz + cm.cx;
      o.my = cm.fy * tytz + cm.cy;
      const float mid = 0.5f * (ca + cc);
      const float disc = fmaxf(0.1f, mid * mid - det);
      const float lambda1 = mid + sqrtf(disc);
      const float rf = fminf(ceilf(3.0f * sqrtf(lambda1)), 1048576.0f);
      const int rad = int(rf);
      const float r_ = float(rad);
      const float fx0 = (o.mx - r_) / 16.0f;
      const float fy0 = (o.my - r_) / 16.0f;
      const float fx1 = ((o.mx + r_) + 15.0f) / 16.0f;
      const float fy1 = ((o.my + r_) + 15.0f) / 16.0f;
      o.x0 = int(fminf(float(cm.TX), fmaxf(0.0f, fx0)));
      o.y0 = int(fminf(float(cm.TY), fmaxf(0.0f, fy0)));
      o.x1 = int(fminf(float(cm.TX), fmaxf(0.0f, fx1)));
      o.y1 = int(fminf(float(cm.TY), fmaxf(0.0f, fy1)));
      o.area = uint32_t((o.x1 - o.x0) * (o.y1 - o.y0));
      if (o.area != 0) {
        o.valid = true;
        radius = rad;
        o.depth = tz;
        o.opac = mo.w;
        // tile footprint (reading R5, the oracle's project_one): the 3DGS rect cut to the tiles
        // holding pixel centres of the widened alpha >= 1/255 box; same float expressions
        const float kk = -2.0f * alpha_cut_thr(mo.w);
        const float cdet = o.A * o.C - o.B * o.B;
        if (kk > 0.0f && cdet > 0.0f) {
          const float hx = sqrtf((kk * o.C) / cdet) * 1.001f + 0.01f;
          const float hy = sqrtf((kk * o.A) / cdet) * 1.001f + 0.01f;
          const int ex0 = int(fminf(float(cm.TX), fmaxf(0.0f, floorf((o.mx - hx) / 16.0f))));
          const int ey0 = int(fminf(float(cm.TY), fmaxf(0.0f, floorf((o.my - hy) / 16.0f))));
          const int ex1 = int(fminf(float(cm.TX), fmaxf(0.0f, floorf((o.mx + hx) / 16.0f) + 1.0f)));
          const int ey1 = int(fminf(float(cm.TY), fmaxf(0.0f, floorf((o.my + hy) / 16.0f) + 1.0f)));
          o.x0 = max(o.x0, ex0);
          o.y0 = max(o.y0, ey0);
          o.x1 = max(o.x0, min(o.x1, ex1));
          o.y1 = max(o.y0, min(o.y1, ey1));
        } else {  // o <= 1/255: no pixel passes the cut
          o.x1 = o.x0;
          o.y1 = o.y0;
        }
        o.area = uint32_t((o.x1 - o.x0) * (o.y1 - o.y0));
        if (!a.no_color) {
          o.mux = mo.x;
          o.muy = mo.y;
          o.muz = mo.z;
        }
      }
    }
  }
  a.radius[i] = o.valid ? radius : 0;
  o.rect = uint32_t(o.x0) | (uint32_t(o.y0) << 8) | (uint32_t(o.x1) << 16) | (uint32_t(o.y1) << 24);
  if (!o.valid) o.area = 0;
  return o;
}

// Deterministic block-local slots for flagged items (order: item round, warp, lane) and one
// global range per CTA.  Returns the CTA's base; `ls` receives the block-local slot.
template <int PER>
__device__ __forceinline__ unsigned long long block_compact(const bool (&flag)[PER], uint32_t (&ls)[PER],
                                                            unsigned long long* counter, uint32_t* s_cnt,
                                                            uint32_t& total, unsigned long long* s_base,
                                                            uint32_t* s_total) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t rk[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const unsigned m = __ballot_sync(0xffffffffu, flag[k]);
    rk[k] = __popc(m & ((1u << lane) - 1u));
    if (lane == 0) s_cnt[k * 8 + warp] = __popc(m);
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t run = 0;
    for (int j = 0; j < PER * 8; ++j) {
      const uint32_t c = s_cnt[j];
      s_cnt[j] = run;
      run += c;
    }
    *s_total = run;
    *s_base = run ? atomicAdd(counter, (unsigned long long)run) : 0ull;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < PER; ++k) ls[k] = s_cnt[k * 8 + warp] + rk[k];
  total = *s_total;
  return *s_base;
}

constexpr int kCullPer = 4;
constexpr int kCullChunk = 256 * kCullPer;
static_assert(kCullChunk == BGS_BOUNDS_BLOCK, "one k_cull CTA per bounds block");

// Hierarchical culling: can any Gaussian of the block (box of means [lo, hi], largest axis
// standard deviation smax) produce a record?  The means' camera depths span [tz_min, tz_max]
// (affine in mu: extremes at the box corners).  All behind the near plane -> no.  Straddling it
// -> maybe (conservative).  Else every centre projects into the bounding box of the projected
// corners (the box lies in front of the camera, where projection maps convex sets to convex
// sets), and every per-Gaussian radius bound of cull_test is at most rb(smax, tz_min): the block
// is culled when that box, widened by rb and by a 1% + 4 px margin for fp32 rounding, misses the
// image.  Every Gaussian of a culled block would fail cull_test, hence has an empty rect.
// Computed by one warp, a corner per lane (lanes 8-31 repeat corners 0-7); the min / max reductions
// are exact in any order.
__device__ bool block_may_reach_warp(const ProjectArgs& a, float4 b0, float4 b1) {
  const CameraK& cm = a.cam;
  const int c = threadIdx.x & 7;
  const float px = (c & 1) ? b1.x : b0.x, py = (c & 2) ? b1.y : b0.y, pz = (c & 4) ? b1.z : b0.z;
  const float tx = ((cm.R[0] * px + cm.R[1] * py) + cm.R[2] * pz) + cm.t[0];
  const float ty = ((cm.R[3] * px + cm.R[4] * py) + cm.R[5] * pz) + cm.t[1];
  const float tz = ((cm.R[6] * px + cm.R[7] * py) + cm.R[8] * pz) + cm.t[2];
  const float mx = cm.fx * (tx / tz) + cm.cx, my = cm.fy * (ty / tz) + cm.cy;
  float tzmin = tz, tzmax = tz, xmin = mx, xmax = mx, ymin = my, ymax = my;
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    tzmin = fminf(tzmin, __shfl_xor_sync(0xffffffffu, tzmin, o));
    tzmax = fmaxf(tzmax, __shfl_xor_sync(0xffffffffu, tzmax, o));
    xmin = fminf(xmin, __shfl_xor_sync(0xffffffffu, xmin, o));
    xmax = fmaxf(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
    ymin = fminf(ymin, __shfl_xor_sync(0xffffffffu, ymin, o));
    ymax = fmaxf(ymax, __shfl_xor_sync(0xffffffffu, ymax, o));
  }
  if (tzmax <= cm.near_clip) return false;  // every mean behind the near plane
  if (tzmin <= cm.near_clip * 1.001f + 1e-6f) return true;  // straddles it: keep
  const float smax = b0.w, iz = 1.0f / tzmin;
  const float rb = (3.0f * sqrtf(a.cull_K * (smax * smax) * (iz * iz) + 0.62f) * 1.01f + 2.0f) * 1.01f + 4.0f;
  const float mxr = 0.01f * (fabsf(xmin) + fabsf(xmax)), myr = 0.01f * (fabsf(ymin) + fabsf(ymax));
  return !(xmax + rb + mxr < 0.0f || xmin - rb - mxr > float(16 * cm.TX + 1) || ymax + rb + myr < 0.0f ||
           ymin - rb - myr > float(16 * cm.TY + 1));
}

// one CTA per bounds block: box of the means, largest axis standard deviation
__global__ void __launch_bounds__(256) k_shard_bounds(const float4* __restrict__ mean_opac,
                                                      const float4* __restrict__ scale, int64_t n,
                                                      float4* __restrict__ bounds) {
  __shared__ float s_red[7][8];
  const int64_t r0 = int64_t(blockIdx.x) * kCullChunk;
  float v[7] = {3.4e38f, 3.4e38f, 3.4e38f, 0.f, -3.4e38f, -3.4e38f, -3.4e38f};
  for (int k = 0; k < kCullPer; ++k) {
    const int64_t i = r0 + k * 256 + threadIdx.x;
    if (i >= n) break;
    const float4 m = ldg4(mean_opac + i), sc = ldg4(scale + i);
    v[0] = fminf(v[0], m.x);
    v[1] = fminf(v[1], m.y);
    v[2] = fminf(v[2], m.z);
    v[3] = fmaxf(v[3], fmaxf(sc.x, fmaxf(sc.y, sc.z)));
    v[4] = fmaxf(v[4], m.x);
    v[5] = fmaxf(v[5], m.y);
    v[6] = fmaxf(v[6], m.z);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      const float t = __shfl_xor_sync(0xffffffffu, v[k], o);
      v[k] = (k < 3) ? fminf(v[k], t) : fmaxf(v[k], t);
    }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int k = 0; k < 7; ++k) s_red[k][w] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    float r[7];
    for (int k = 0; k < 7; ++k) {
      r[k] = s_red[k][0];
      for (int j = 1; j < 8; ++j) r[k] = (k < 3) ? fminf(r[k], s_red[k][j]) : fmaxf(r[k], s_red[k][j]);
    }
    bounds[2 * blockIdx.x] = make_float4(r[0], r[1], r[2], r[3]);
    bounds[2 * blockIdx.x + 1] = make_float4(r[4], r[5], r[6], 0.f);
  }
}

__global__ void __launch_bounds__(256) k_cull(ProjectArgs a) {
  __shared__ uint32_t s_idx[kCullChunk];
  __shared__ uint32_t s_cnt[kCullPer * 8];
  __shared__ unsigned long long s_base;
  __shared__ uint32_t s_total;
  __shared__ uint32_t s_act;
  const int tid = threadIdx.x;
  if (tid == 0) s_act = 0;
  const int64_t chunk0 = int64_t(blockIdx.x) * kCullChunk;
  // the block test once per CTA (warp 0), not once per thread
  __shared__ int s_reach;
  bool reach = true;
  if (a.bounds && !a.gate_enabled) {
    if (tid < 32) {
      const bool r = block_may_reach_warp(a, __ldg(a.bounds + 2 * blockIdx.x), __ldg(a.bounds + 2 * blockIdx.x + 1));
      if (tid == 0) s_reach = r;
    }
    __syncthreads();
    reach = s_reach != 0;
  }
  if (!reach) {
    // the whole block is off-screen: radius 0, no candidates; |A| counts the rows the cull column
    // keeps (the frustum is not part of the active set) -- without reading a single Gaussian
    uint32_t act = 0;
    for (int k = 0; k < kCullPer; ++k) {
      const int64_t i = chunk0 + k * 256 + tid;
      if (i < a.n) {
        a.radius[i] = 0;
        act += a.cull ? !((__ldg(a.cull + (i >> 5)) >> (i & 31)) & 1u) : 1u;
      }
    }
    act = __reduce_add_sync(0xffffffffu, act);
    if ((tid & 31) == 0 && act) atomicAdd(a.counters + C_NACT, (unsigned long long)act);
    return;
  }
  bool maybe[kCullPer];
  uint32_t nact = 0;
#pragma unroll
  for (int k = 0; k < kCullPer; ++k) {
    const int64_t i = chunk0 + k * 256 + tid;
    bool act = false;
    maybe[k] = i < a.n && cull_test(a, i, act);
    nact += act ? 1u : 0u;
    if (i < a.n && !maybe[k]) a.radius[i] = 0;
  }
  const uint32_t wact = __reduce_add_sync(0xffffffffu, nact);
  uint32_t ls[kCullPer], total;
  const unsigned long long base = block_compact<kCullPer>(maybe, ls, a.counters + C_CAND, s_cnt, total, &s_base,
                                                          &s_total);
  if ((tid & 31) == 0 && wact) atomicAdd(&s_act, wact);
#pragma unroll
  for (int k = 0; k < kCullPer; ++k)
    if (maybe[k]) s_idx[ls[k]] = uint32_t(chunk0 + k * 256 + tid);
  __syncthreads();
  if (tid == 0 && s_act) atomicAdd(a.counters + C_NACT, (unsigned long long)s_act);
  for (uint32_t j = tid; j < total; j += 256) a.cand[base + j] = s_idx[j];
}

// Persistent grid over the candidate list (count read on the device).
__global__ void __launch_bounds__(256) k_project(ProjectArgs a) {
  __shared__ float4 s_rec[256 * 3];
  __shared__ uint32_t s_lidx[256];
  __shared__ uint32_t s_cnt[8];
  __shared__ unsigned long long s_area[8];
  __shared__ unsigned long long s_base;
  __shared__ uint32_t s_total;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n_cand = int64_t(*((volatile unsigned long long*)(a.counters + C_CAND)));
  uint32_t dhi = 0, dlo = 0;  // max bits(depth), max (0xffffffff - bits(depth)) of this thread's records
  const int64_t stride = int64_t(gridDim.x) * 256;
  // candidate indices read one iteration ahead (the parameter gathers then wait on one round trip)
  uint32_t i_next = int64_t(blockIdx.x) * 256 + tid < n_cand ? a.cand[int64_t(blockIdx.x) * 256 + tid] : 0u;
  for (int64_t c0 = int64_t(blockIdx.x) * 256; c0 < n_cand; c0 += stride) {
    const int64_t c = c0 + tid;
    ProjOut o;
    o.valid = false;
    o.area = 0;
    const uint32_t i = i_next;
    i_next = c + stride < n_cand ? a.cand[c + stride] : 0u;
    if (c < n_cand) o = project_exact(a, i);
    if (o.valid) {
      const uint32_t db = __float_as_uint(o.depth);
      dhi = db > dhi ? db : dhi;
      dlo = (0xffffffffu - db) > dlo ? (0xffffffffu - db) : dlo;
    }
    unsigned long long area = o.area;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) area += __shfl_xor_sync(0xffffffffu, area, off);
    if (lane == 0) s_area[warp] = area;
    const bool flag[1] = {o.valid};
    uint32_t ls[1], total;
    const unsigned long long base = block_compact<1>(flag, ls, a.counters + C_F, s_cnt, total, &s_base, &s_total);
    if (tid == 0) {
      unsigned long long ar = 0;
      for (int w = 0; w < 8; ++w) ar += s_area[w];
      if (ar) atomicAdd(a.counters + C_PALL, ar);
    }
    if (o.valid) {
      const uint32_t gid = i * uint32_t(a.world) + uint32_t(a.rank);
      s_rec[3 * ls[0] + 0] = make_float4(o.mx, o.my, o.A, o.B);
      s_rec[3 * ls[0] + 1] = make_float4(o.C, o.opac, o.mux, o.muy);
      s_rec[3 * ls[0] + 2] = make_float4(o.muz, o.depth, __uint_as_float(gid), __uint_as_float(o.rect));
      s_lidx[ls[0]] = i;
      if (a.tile_diff) {
        // 2D difference array of rect coverage -> per-tile pair counts (a3 input)
        const int W1 = a.cam.TX + 1;
        atomicAdd(a.tile_diff + o.y0 * W1 + o.x0, 1);
        atomicAdd(a.tile_diff + o.y0 * W1 + o.x1, -1);
        atomicAdd(a.tile_diff + o.y1 * W1 + o.x0, -1);
        atomicAdd(a.tile_diff + o.y1 * W1 + o.x1, 1);
      }
    }
    __syncthreads();
    float4* dst = reinterpret_cast<float4*>(a.recs + base);
    for (uint32_t j = tid; j < 3 * total; j += 256)
      if (base + j / 3 < (unsigned long long)a.rec_cap) dst[j] = s_rec[j];
    for (uint32_t j = tid; j < total; j += 256)
      if (base + j < (unsigned long long)a.rec_cap) a.rec_lidx[base + j] = s_lidx[j];
    __syncthreads();
  }
  // depth range of the records (sort key layout, KeyLayout): one atomic pair per CTA
  dhi = __reduce_max_sync(0xffffffffu, dhi);
  dlo = __reduce_max_sync(0xffffffffu, dlo);
  __shared__ uint32_t s_dr[2];
  if (tid == 0) s_dr[0] = s_dr[1] = 0;
  __syncthreads();
  if (lane == 0) {
    atomicMax(&s_dr[0], dhi);
    atomicMax(&s_dr[1], dlo);
  }
  __syncthreads();
  if (tid == 0 && s_dr[0]) {
    atomicMax(a.counters + C_DHI, (unsigned long long)s_dr[0]);
    atomicMax(a.counters + C_DLO, (unsigned long long)s_dr[1]);
  }
}

__device__ __forceinline__ void color_one(const ProjectArgs& a, int64_t f, uint32_t i) {
  const float4* shp = reinterpret_cast<const float4*>(a.sh + size_t(48) * i);
  float v[48];
#pragma unroll
  for (int q4 = 0; q4 < 12; ++q4) {
    const float4 t = ldg4(shp + q4);
    v[4 * q4 + 0] = t.x;
    v[4 * q4 + 1] = t.y;
    v[4 * q4 + 2] = t.z;
    v[4 * q4 + 3] = t.w;
  }
  // mu was parked in the colour slots by k_project (no scattered 16-B read of mean_opac)
  float* rp = reinterpret_cast<float*>(a.recs + f);
  const float4 mo = make_float4(rp[6], rp[7], rp[8], 0.f);
  const CameraK& cm = a.cam;
  const float dx = mo.x - cm.campos[0], dy = mo.y - cm.campos[1], dz = mo.z - cm.campos[2];
  const float len = sqrtf((dx * dx + dy * dy) + dz * dz);
  const float x = dx / len, y = dy / len, z = dz / len;
  const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  float Y[16];
  Y[0] = 0.28209479177387814f;
  Y[1] = -(0.4886025119029199f * y);
  Y[2] = 0.4886025119029199f * z;
  Y[3] = -(0.4886025119029199f * x);
  Y[4] = 1.0925484305920792f * xy;
  Y[5] = -1.0925484305920792f * yz;
  Y[6] = 0.31539156525252005f * ((2.0f * zz - xx) - yy);
  Y[7] = -1.0925484305920792f * xz;
  Y[8] = 0.5462742152960396f * (xx - yy);
  Y[9] = (-0.5900435899266435f * y) * (3.0f * xx - yy);
  Y[10] = (2.890611442640554f * xy) * z;
  Y[11] = (-0.4570457994644658f * y) * ((4.0f * zz - xx) - yy);
  Y[12] = (0.3731763325901154f * z) * ((2.0f * zz - 3.0f * xx) - 3.0f * yy);
  Y[13] = (-0.4570457994644658f * x) * ((4.0f * zz - xx) - yy);
  Y[14] = (1.445305721320277f * z) * (xx - yy);
  Y[15] = (-0.5900435899266435f * x) * (xx - 3.0f * yy);
  float col[3];
  uint32_t clamped = 0;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    float c = Y[0] * v[ch];
#pragma unroll
    for (int k = 1; k < 16; ++k) c = c + Y[k] * v[3 * k + ch];
    c = c + 0.5f;
    clamped |= uint32_t(c < 0.0f) << ch;
    col[ch] = c < 0.0f ? 0.0f : c;
  }
  rp[6] = col[0];
  rp[7] = col[1];
  rp[8] = col[2];
  // For a11 (k_project_bwd): J[ch][d] = sum_k sh[k][ch] dY_k/d(x, y, z), the derivative of the
  // unclamped colour along the normalised view direction (x, y, z treated as independent; the
  // normalisation's projection is applied in the backward), and the clamp bits (R2: a clamped
  // channel passes no gradient).  The backward then needs these 48 B instead of the 192-B SH row.
  // Not part of the pinned record: its rounding only enters gradients (tolerance parity).
  const float C1 = 0.4886025119029199f;
  const float C20 = 1.0925484305920792f, C21 = -1.0925484305920792f, C22 = 0.31539156525252005f,
              C23 = -1.0925484305920792f, C24 = 0.5462742152960396f;
  const float C30 = -0.5900435899266435f, C31 = 2.890611442640554f, C32 = -0.4570457994644658f,
              C33 = 0.3731763325901154f, C34 = -0.4570457994644658f, C35 = 1.445305721320277f,
              C36 = -0.5900435899266435f;
  float J[3][3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const float* s = v + ch;  // s[3 k] = sh[k][ch]
    J[ch][0] = -C1 * s[9] + C20 * y * s[12] - 2.f * C22 * x * s[18] + C23 * z * s[21] + 2.f * C24 * x * s[24] +
               6.f * C30 * xy * s[27] + C31 * yz * s[30] - 2.f * C32 * xy * s[33] - 6.f * C33 * xz * s[36] +
               C34 * (4.f * zz - 3.f * xx - yy) * s[39] + 2.f * C35 * xz * s[42] + 3.f * C36 * (xx - yy) * s[45];
    J[ch][1] = -C1 * s[3] + C20 * x * s[12] + C21 * z * s[15] - 2.f * C22 * y * s[18] - 2.f * C24 * y * s[24] +
               3.f * C30 * (xx - yy) * s[27] + C31 * xz * s[30] + C32 * (4.f * zz - xx - 3.f * yy) * s[33] -
               6.f * C33 * yz * s[36] - 2.f * C34 * xy * s[39] - 2.f * C35 * yz * s[42] - 6.f * C36 * xy * s[45];
    J[ch][2] = C1 * s[6] + C21 * y * s[15] + 4.f * C22 * z * s[18] + C23 * x * s[21] + C31 * xy * s[30] +
               8.f * C32 * yz * s[33] + C33 * (6.f * zz - 3.f * xx - 3.f * yy) * s[36] + 8.f * C34 * xz * s[39] +
               C35 * (xx - yy) * s[42];
  }
  float4* jp = a.jdir + 3 * f;
  jp[0] = make_float4(J[0][0], J[0][1], J[0][2], J[1][0]);
  jp[1] = make_float4(J[1][1], J[1][2], J[2][0], J[2][1]);
  jp[2] = make_float4(J[2][2], __uint_as_float(clamped), 0.f, 0.f);
}

// SH degree 3 along (mu - c_v)/|mu - c_v| (R1, R2); term order of DESIGN.md §4.2.
// Persistent grid-stride over the F records (F read on the device: no host round trip).
__global__ void __launch_bounds__(256, 3) k_color(ProjectArgs a) {
  const int64_t F = int64_t(*((volatile unsigned long long*)(a.counters + C_F)));
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  // record indices read one iteration ahead (the SH-row gather then waits on one round trip)
  uint32_t i_next = f < F ? a.rec_lidx[f] : 0u;
  for (; f < F; f += stride) {
    const uint32_t i = i_next;
    i_next = f + stride < F ? a.rec_lidx[f + stride] : 0u;
    color_one(a, f, i);
  }
}

// Persistent grids sized to what is resident at once (SMs x max CTAs/SM of the kernel):
// oversubscribing them (6 and 8 CTAs/SM before) left a partial second wave; measured 0.124 ->
// 0.119 ms per Rubble view for the projection stage.
template <class K>
int persistent_blocks(K kernel) {
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 256, 0);
  if (sms <= 0) sms = 148;
  if (occ <= 0) occ = 1;
  const char* e = getenv("BGS_PERSIST_PER_SM");  // tuning only
  if (e && atoi(e) > 0 && atoi(e) < occ) occ = atoi(e);
  return sms * occ;
}

}  // namespace

void launch_gate_count(const ProjectArgs& a, cudaStream_t s) {
  if (a.n <= 0) return;
  const int64_t blocks = (a.n + 255) / 256;
  k_gate_count<<<unsigned(blocks), 256, 0, s>>>(a);
}

void launch_project(const ProjectArgs& a, cudaStream_t s) {
  if (a.n <= 0) return;
  const int64_t blocks = (a.n + kCullChunk - 1) / kCullChunk;
  k_cull<<<unsigned(blocks), 256, 0, s>>>(a);
  static std::atomic<int> slots[kMaxDevices];
  const int proj_blocks = per_device(slots, [] { return persistent_blocks(k_project); });
  k_project<<<proj_blocks, 256, 0, s>>>(a);
}

void launch_shard_bounds(const float4* mean_opac, const float4* scale, int64_t n, float4* bounds, cudaStream_t s) {
  if (n <= 0) return;
  k_shard_bounds<<<unsigned((n + kCullChunk - 1) / kCullChunk), 256, 0, s>>>(mean_opac, scale, n, bounds);
}

void launch_color(const ProjectArgs& a, cudaStream_t s) {
  if (a.n <= 0 || a.no_color) return;
  static std::atomic<int> slots[kMaxDevices];
  const int color_blocks = per_device(slots, [] { return persistent_blocks(k_color); });
  k_color<<<color_blocks, 256, 0, s>>>(a);
}

}  // namespace bgs
