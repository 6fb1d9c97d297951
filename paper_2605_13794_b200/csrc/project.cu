// a1 gate + a2 projection (bgs_project).
//
// PAPER.md §3.1 P:143-152 (Eq.1 Gaussian, EWA "projected to screen-space ellipses"), §3.2
// ("every GPU projects only its own local Gaussians"), §3.4 Eq.4-6 P:195-210 (LOD gate, cull).
//
// PINNED ARITHMETIC (D2): this translation unit is compiled with -fmad=false and
// IEEE div/sqrt so that every float expression below rounds exactly as written; radius,
// rect, tile ids and pair counts are integers derived from these floats and must be
// bit-identical to the oracle's.  Expression trees are the ones listed in DESIGN.md §4.
//
// Two kernels, both HBM-bound:
//  k_project (one thread per local Gaussian): 16-B (mu, o) + lod byte (+ cull bit) for
//    everyone; quat/scale (32 B) issued up front when no gate/cull can drop the Gaussian,
//    otherwise only for kept ones; EWA geometry, radius, rect; a warp-aggregated append of
//    the 48-B record (colour left for k_color) + 4-B index; radius written for all.
//  k_color (one thread per record): the 192-B SH row of in-frustum Gaussians only, as 12
//    independent 128-bit loads in flight per thread, evaluated along the view direction.
// Splitting keeps k_project at low register pressure (full occupancy for latency hiding) and
// reads SH only for the F records.
#include "bgs_internal.cuh"

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

struct ProjOut {
  float mx, my, A, B, C, depth, opac;
  float mux, muy, muz;  // parked in the record's colour slots for k_color
  uint32_t rect, area;
  bool valid, active;
  int x0, y0, x1, y1;
};

__device__ __forceinline__ ProjOut project_one(const ProjectArgs& a, int64_t i) {
  bool valid = false;
  bool active = false;
  float mx = 0.f, my = 0.f, cA = 0.f, cB = 0.f, cC = 0.f, depth = 0.f, opac = 0.f, mux = 0.f, muy = 0.f,
        muz = 0.f;
  int radius = 0;
  uint32_t area = 0;
  int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
  if (i < a.n) {
    const bool filtered = a.gate_enabled || a.cull;
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f), sc = q;
    if (!filtered) sc = ldg4(a.scale + i);  // nothing can drop it before the frustum test: load now
    const float4 mo = ldg4(a.mean_opac + i);
    // ---- a1: Eq.5 gate with per-rank fallback, then Eq.6 cull column
    bool keep = true;
    if (a.gate_enabled) {
      const unsigned long long nl = *((volatile unsigned long long*)(a.counters + C_NLOD));
      const bool fallback = (unsigned long long)a.fb_den * nl > (unsigned long long)a.fb_num * (unsigned long long)a.n;
      if (!fallback) keep = lod_keep(a, mo, a.lod[i]);
    }
    if (keep && a.cull) keep = !((__ldg(a.cull + (i >> 5)) >> (i & 31)) & 1u);
    active = keep;
    if (keep) {
      if (filtered) sc = ldg4(a.scale + i);
      const CameraK& cm = a.cam;
      // ---- a2: t_c = R mu + t
      const float tx = ((cm.R[0] * mo.x + cm.R[1] * mo.y) + cm.R[2] * mo.z) + cm.t[0];
      const float ty = ((cm.R[3] * mo.x + cm.R[4] * mo.y) + cm.R[5] * mo.z) + cm.t[1];
      const float tz = ((cm.R[6] * mo.x + cm.R[7] * mo.y) + cm.R[8] * mo.z) + cm.t[2];
      const float txtz = tx / tz, tytz = ty / tz;
      // Conservative off-screen rejection before any covariance work:
      // radius <= 3 sqrt(|J|_F^2 s_max^2 + 0.3 + sqrt(0.1)) + 1 with |J|_F^2 <= K / tz^2
      // (K = fx^2 (1 + Lx^2) + fy^2 (1 + Ly^2), L = clamp limits), widened by 1% + 2 px; a
      // Gaussian whose centre is further than that outside the image has an empty rect in the
      // exact computation too, so the decision is unchanged.
      bool maybe = tz > cm.near_clip;
      if (maybe) {
        const float mxb = cm.fx * txtz + cm.cx, myb = cm.fy * tytz + cm.cy;
        const float smax = fmaxf(sc.x, fmaxf(sc.y, sc.z));
        const float iz = __fdividef(1.0f, tz);
        const float rb = 3.0f * sqrtf(a.cull_K * (smax * smax) * (iz * iz) + 0.62f) * 1.01f + 2.0f;
        maybe = !(mxb + rb < 0.0f || mxb - rb > float(16 * cm.TX + 1) || myb + rb < 0.0f ||
                  myb - rb > float(16 * cm.TY + 1));
      }
      if (maybe) q = ldg4(a.quat + i);
      if (maybe) {
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
          cA = cc / det;
          cB = (-cb) / det;
          cC = ca / det;
          mx = cm.fx * txtz + cm.cx;
          my = cm.fy * tytz + cm.cy;
          const float mid = 0.5f * (ca + cc);
          const float disc = fmaxf(0.1f, mid * mid - det);
          const float lambda1 = mid + sqrtf(disc);
          const float rf = fminf(ceilf(3.0f * sqrtf(lambda1)), 1048576.0f);
          const int rad = int(rf);
          const float r_ = float(rad);
          const float fx0 = (mx - r_) / 16.0f;
          const float fy0 = (my - r_) / 16.0f;
          const float fx1 = ((mx + r_) + 15.0f) / 16.0f;
          const float fy1 = ((my + r_) + 15.0f) / 16.0f;
          x0 = int(fminf(float(cm.TX), fmaxf(0.0f, fx0)));
          y0 = int(fminf(float(cm.TY), fmaxf(0.0f, fy0)));
          x1 = int(fminf(float(cm.TX), fmaxf(0.0f, fx1)));
          y1 = int(fminf(float(cm.TY), fmaxf(0.0f, fy1)));
          area = uint32_t((x1 - x0) * (y1 - y0));
          if (area != 0) {
            valid = true;
            radius = rad;
            depth = tz;
            opac = mo.w;
            if (!a.no_color) {
              mux = mo.x;
              muy = mo.y;
              muz = mo.z;
            }
          }
        }
      }
    }
    a.radius[i] = valid ? radius : 0;
  }
  ProjOut o;
  o.mx = mx;
  o.my = my;
  o.A = cA;
  o.B = cB;
  o.C = cC;
  o.depth = depth;
  o.opac = opac;
  o.mux = mux;
  o.muy = muy;
  o.muz = muz;
  o.rect = uint32_t(x0) | (uint32_t(y0) << 8) | (uint32_t(x1) << 16) | (uint32_t(y1) << 24);
  o.area = area;
  o.valid = valid;
  o.active = active;
  o.x0 = x0;
  o.y0 = y0;
  o.x1 = x1;
  o.y1 = y1;
  return o;
}

// Block-level compaction: a CTA projects kProjChunk consecutive Gaussians, assigns its records
// block-local slots with a deterministic scan (item round, warp, lane), stages them in shared
// memory, takes ONE global slot range (a single 64-bit atomic packing F and |A|, plus one for
// P_all) and writes the records out coalesced.  Per-warp global atomics on one counter were
// the bottleneck (hundreds of thousands of same-address atomics serialise at the L2).
constexpr int kProjPer = 2;
constexpr int kProjChunk = 256 * kProjPer;

__global__ void __launch_bounds__(256) k_project(ProjectArgs a) {
  __shared__ float4 s_rec[kProjChunk * 3];
  __shared__ uint32_t s_lidx[kProjChunk];
  __shared__ uint32_t s_cnt[kProjPer * 8];
  __shared__ uint32_t s_act[8];
  __shared__ unsigned long long s_area[8];
  __shared__ unsigned long long s_base;
  __shared__ uint32_t s_total;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t chunk0 = int64_t(blockIdx.x) * kProjChunk;
  ProjOut o[kProjPer];
  uint32_t nact = 0;
  unsigned long long area = 0;
#pragma unroll
  for (int k = 0; k < kProjPer; ++k) {
    const int64_t i = chunk0 + k * 256 + tid;
    if (i < a.n) {
      o[k] = project_one(a, i);
    } else {
      o[k].valid = false;
      o[k].active = false;
      o[k].area = 0;
    }
    nact += o[k].active ? 1u : 0u;
    area += o[k].area;
  }
  uint32_t rank_in_warp[kProjPer];
#pragma unroll
  for (int k = 0; k < kProjPer; ++k) {
    const unsigned m = __ballot_sync(0xffffffffu, o[k].valid);
    rank_in_warp[k] = __popc(m & ((1u << lane) - 1u));
    if (lane == 0) s_cnt[k * 8 + warp] = __popc(m);
  }
  const uint32_t wact = __reduce_add_sync(0xffffffffu, nact);
  unsigned long long warea = area;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) warea += __shfl_xor_sync(0xffffffffu, warea, off);
  if (lane == 0) {
    s_act[warp] = wact;
    s_area[warp] = warea;
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t run = 0, act = 0;
    unsigned long long ar = 0;
    for (int j = 0; j < kProjPer * 8; ++j) {
      const uint32_t c = s_cnt[j];
      s_cnt[j] = run;
      run += c;
    }
    for (int w = 0; w < 8; ++w) {
      act += s_act[w];
      ar += s_area[w];
    }
    s_total = run;
    unsigned long long base = 0;
    if (run || act) base = atomicAdd(a.counters + C_F, ((unsigned long long)run << 32) | act) >> 32;
    if (ar) atomicAdd(a.counters + C_PALL, ar);
    s_base = base;
  }
  __syncthreads();
  const unsigned long long base = s_base;
#pragma unroll
  for (int k = 0; k < kProjPer; ++k) {
    if (!o[k].valid) continue;
    const uint32_t ls = s_cnt[k * 8 + warp] + rank_in_warp[k];
    const int64_t i = chunk0 + k * 256 + tid;
    const uint32_t gid = uint32_t(i) * uint32_t(a.world) + uint32_t(a.rank);
    s_rec[3 * ls + 0] = make_float4(o[k].mx, o[k].my, o[k].A, o[k].B);
    s_rec[3 * ls + 1] = make_float4(o[k].C, o[k].opac, o[k].mux, o[k].muy);
    s_rec[3 * ls + 2] = make_float4(o[k].muz, o[k].depth, __uint_as_float(gid), __uint_as_float(o[k].rect));
    s_lidx[ls] = uint32_t(i);
    if (a.tile_diff) {
      // 2D difference array of rect coverage -> per-tile pair counts (a3 input)
      const int W1 = a.cam.TX + 1;
      atomicAdd(a.tile_diff + o[k].y0 * W1 + o[k].x0, 1);
      atomicAdd(a.tile_diff + o[k].y0 * W1 + o[k].x1, -1);
      atomicAdd(a.tile_diff + o[k].y1 * W1 + o[k].x0, -1);
      atomicAdd(a.tile_diff + o[k].y1 * W1 + o[k].x1, 1);
    }
  }
  __syncthreads();
  const uint32_t total = s_total;
  float4* dst = reinterpret_cast<float4*>(a.recs + base);
  for (uint32_t j = tid; j < 3 * total; j += 256)
    if (base + j / 3 < (unsigned long long)a.rec_cap) dst[j] = s_rec[j];
  for (uint32_t j = tid; j < total; j += 256)
    if (base + j < (unsigned long long)a.rec_cap) a.rec_lidx[base + j] = s_lidx[j];
}

__device__ __forceinline__ void color_one_impl(const ProjectArgs& a, int64_t f);
__device__ __forceinline__ void color_one(const ProjectArgs& a, int64_t f) { color_one_impl(a, f); }

// SH degree 3 along (mu - c_v)/|mu - c_v| (R1, R2); term order of DESIGN.md §4.2.
// Persistent grid-stride over the F records (F read on the device: no host round trip).
__global__ void __launch_bounds__(256) k_color(ProjectArgs a) {
  const int64_t F = int64_t(*((volatile unsigned long long*)(a.counters + C_F)) >> 32);
  for (int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; f < F; f += int64_t(gridDim.x) * blockDim.x)
    color_one(a, f);
}

__device__ __forceinline__ void color_one_impl(const ProjectArgs& a, int64_t f) {
  const uint32_t i = a.rec_lidx[f];
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
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    float c = Y[0] * v[ch];
#pragma unroll
    for (int k = 1; k < 16; ++k) c = c + Y[k] * v[3 * k + ch];
    c = c + 0.5f;
    col[ch] = c < 0.0f ? 0.0f : c;
  }
  rp[6] = col[0];
  rp[7] = col[1];
  rp[8] = col[2];
}

}  // namespace

void launch_gate_count(const ProjectArgs& a, cudaStream_t s) {
  if (a.n <= 0) return;
  const int64_t blocks = (a.n + 255) / 256;
  k_gate_count<<<unsigned(blocks), 256, 0, s>>>(a);
}

void launch_project(const ProjectArgs& a, cudaStream_t s) {
  if (a.n <= 0) return;
  const int64_t blocks = (a.n + kProjChunk - 1) / kProjChunk;
  k_project<<<unsigned(blocks), 256, 0, s>>>(a);
}

void launch_color(const ProjectArgs& a, cudaStream_t s) {
  if (a.n <= 0 || a.no_color) return;
  int64_t blocks = (a.n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_color<<<unsigned(blocks), 256, 0, s>>>(a);
}

}  // namespace bgs
