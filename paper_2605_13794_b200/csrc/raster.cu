// a8 forward compositing and a9 its backward (bgs_raster_fwd / bgs_raster_bwd).
//
// Eq.2: C(p) = sum_i T_i alpha_i G'_i(p) c_i, T_i = prod_{j<i} (1 - alpha_j G'_j)
// with the 3DGS rules (readings R9, R10, R14): alpha = min(0.99, o G), splats with
// alpha < 1/255 skipped (tested in power space: power >= thr, thr = -log(255 o), D3),
// compositing stops before the splat whose T(1-alpha) would fall below 1e-4.
// Instrumented mode (caption P:132): w_{i,v} = sum_p alpha T, a_{i,v} = #pixels where
// the splat contributed (R15), accumulated as u64 fixed point 2^-24 (D5) with one warp
// reduction (__reduce_add_sync) and one atomic per (warp, splat).
//
// Launch: one 256-thread CTA per owned 16x16 tile (one thread per pixel).  Records of the
// tile's sorted list are staged 256 at a time into shared memory (one record per thread,
// 128-bit loads), the block exits when all 256 pixels are done (__syncthreads_count) and a
// warp whose 32 pixels are done skips the batch (warp-ballot early termination).
//
// The power expression is pinned with __fmul_rn/__fadd_rn (no FMA) so that the alpha-cut
// decision, n_contrib and a are bit-identical to the oracle's.
#include "bgs_internal.cuh"

namespace bgs {
namespace {

constexpr int kBlock = kTile * kTile;

struct __align__(16) Staged {
  float mx, my, A, B;
  float C, o, thr, pad;
  float r, g, b;
  uint32_t ridx;
};

__device__ __forceinline__ float pinned_power(const Staged& s, float dx, float dy) {
  // (-0.5 * ((A*dx)*dx + (C*dy)*dy)) - (B*dx)*dy, every op rounded (no contraction)
  const float t1 = __fmul_rn(__fmul_rn(s.A, dx), dx);
  const float t2 = __fmul_rn(__fmul_rn(s.C, dy), dy);
  const float t3 = __fmul_rn(__fmul_rn(s.B, dx), dy);
  return __fsub_rn(__fmul_rn(-0.5f, __fadd_rn(t1, t2)), t3);
}

__device__ __forceinline__ void stage(Staged* sm, const Rec* recv, uint32_t r) {
  const float4* p = reinterpret_cast<const float4*>(recv + r);
  const float4 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2);
  Staged s;
  s.mx = q0.x;
  s.my = q0.y;
  s.A = q0.z;
  s.B = q0.w;
  s.C = q1.x;
  s.o = q1.y;
  s.r = q1.z;
  s.g = q1.w;
  s.b = q2.x;
  s.thr = float(-log(255.0 * double(q1.y)));  // alpha >= 1/255  <=>  power >= thr
  s.pad = 0.f;
  s.ridx = r;
  *sm = s;
}

template <bool kImportance>
__global__ void __launch_bounds__(kBlock) k_raster_fwd(RasterArgs a, float* __restrict__ rgb,
                                                       float* __restrict__ t_final, int32_t* __restrict__ n_contrib) {
  __shared__ Staged s_rec[kBlock];
  const uint32_t* __restrict__ vals = a.vals[a.pass_ctrl[kFinalSel]];
  const int lt = blockIdx.x;
  const int tile = a.t_begin + lt;
  const int tx = tile % a.TX, ty = tile / a.TX;
  const int tid = threadIdx.x, lane = tid & 31;
  const int px = tx * kTile + (tid & (kTile - 1)), py = ty * kTile + (tid >> 4);
  const bool inside = px < a.W && py < a.H;
  const uint2 range = a.ranges[lt];
  const float pxf = float(px), pyf = float(py);
  float T = 1.0f, cr = 0.f, cg = 0.f, cb = 0.f;
  uint32_t last = 0;
  bool done = !inside;
  for (uint32_t start = range.x; start < range.y; start += kBlock) {
    if (__syncthreads_count(done) == kBlock) break;
    const uint32_t idx = start + tid;
    if (idx < range.y) stage(&s_rec[tid], a.recv, __ldg(vals + idx));
    __syncthreads();
    const int n = int(range.y - start < uint32_t(kBlock) ? range.y - start : uint32_t(kBlock));
    if (__all_sync(0xffffffffu, done)) continue;
    for (int j = 0; j < n; ++j) {
      bool contrib = false;
      uint32_t fixed = 0;
      if (!done) {
        const Staged& s = s_rec[j];
        const float dx = s.mx - pxf, dy = s.my - pyf;
        const float power = pinned_power(s, dx, dy);
        if (power <= 0.0f && power >= s.thr) {
          const float G = __expf(power);
          const float alpha = fminf(0.99f, s.o * G);
          const float test_T = T * (1.0f - alpha);
          if (test_T < 0.0001f) {
            done = true;
          } else {
            const float wgt = alpha * T;
            cr += s.r * wgt;
            cg += s.g * wgt;
            cb += s.b * wgt;
            T = test_T;
            last = start + j + 1 - range.x;
            contrib = true;
            if (kImportance) fixed = __float2uint_rn(wgt * 16777216.0f);
          }
        }
      }
      if (kImportance) {
        const unsigned m = __ballot_sync(0xffffffffu, contrib);
        if (m) {
          const uint32_t sum = __reduce_add_sync(0xffffffffu, fixed);
          if (lane == 0) {
            Acc* acc = a.acc + s_rec[j].ridx;
            atomicAdd(&acc->a, uint32_t(__popc(m)));
            atomicAdd(&acc->w, (unsigned long long)sum);
          }
        }
      }
    }
  }
  if (inside) {
    const size_t pix = size_t(py) * a.W + px, plane = size_t(a.W) * a.H;
    rgb[pix] = cr;
    rgb[plane + pix] = cg;
    rgb[2 * plane + pix] = cb;
    t_final[pix] = T;
    n_contrib[pix] = int32_t(last);
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kBlock) k_raster_bwd(RasterArgs a, const float* __restrict__ dL,
                                                       const float* __restrict__ t_final,
                                                       const int32_t* __restrict__ n_contrib) {
  __shared__ Staged s_rec[kBlock];
  const uint32_t* __restrict__ vals = a.vals[a.pass_ctrl[kFinalSel]];
  const int lt = blockIdx.x;
  const int tile = a.t_begin + lt;
  const int tx = tile % a.TX, ty = tile / a.TX;
  const int tid = threadIdx.x, lane = tid & 31;
  const int px = tx * kTile + (tid & (kTile - 1)), py = ty * kTile + (tid >> 4);
  const bool inside = px < a.W && py < a.H;
  const uint2 range = a.ranges[lt];
  const float pxf = float(px), pyf = float(py);
  const size_t pix = size_t(py) * a.W + px, plane = size_t(a.W) * a.H;
  float T = 1.f, dr = 0.f, dg = 0.f, db = 0.f;
  uint32_t last = 0;
  if (inside) {
    T = t_final[pix];
    last = uint32_t(n_contrib[pix]);
    dr = dL[pix];
    dg = dL[plane + pix];
    db = dL[2 * plane + pix];
  }
  // the block's deepest contributor bounds the work
  __shared__ uint32_t s_maxlast;
  if (tid == 0) s_maxlast = 0;
  __syncthreads();
  atomicMax(&s_maxlast, last);
  __syncthreads();
  const uint32_t end = range.x + s_maxlast;
  float acc_r = 0.f, acc_g = 0.f, acc_b = 0.f, last_alpha = 0.f, last_r = 0.f, last_g = 0.f, last_b = 0.f;
  for (int64_t bstart = int64_t(end) - kBlock; bstart > int64_t(range.x) - kBlock; bstart -= kBlock) {
    __syncthreads();
    const int64_t idx = bstart + tid;
    if (idx >= int64_t(range.x) && idx < int64_t(end)) stage(&s_rec[tid], a.recv, __ldg(vals + idx));
    __syncthreads();
    const int jlo = int(int64_t(range.x) - bstart > 0 ? int64_t(range.x) - bstart : 0);
    for (int j = kBlock - 1; j >= jlo; --j) {
      const int64_t pos = bstart + j;  // absolute position in the sorted list
      if (pos >= int64_t(end)) continue;
      bool contrib = false;
      float g[9];
      if (inside && uint32_t(pos - range.x) < last) {
        const Staged& s = s_rec[j];
        const float dx = s.mx - pxf, dy = s.my - pyf;
        const float power = pinned_power(s, dx, dy);
        if (power <= 0.0f && power >= s.thr) {
          contrib = true;
          const float G = __expf(power);
          const float og = s.o * G;
          const float alpha = fminf(0.99f, og);
          T = T / (1.0f - alpha);
          const float wgt = alpha * T;
          g[6] = wgt * dr;
          g[7] = wgt * dg;
          g[8] = wgt * db;
          acc_r = last_alpha * last_r + (1.f - last_alpha) * acc_r;
          acc_g = last_alpha * last_g + (1.f - last_alpha) * acc_g;
          acc_b = last_alpha * last_b + (1.f - last_alpha) * acc_b;
          last_alpha = alpha;
          last_r = s.r;
          last_g = s.g;
          last_b = s.b;
          const float dLda = T * ((s.r - acc_r) * dr + (s.g - acc_g) * dg + (s.b - acc_b) * db);
          if (og > 0.99f) {
#pragma unroll
            for (int k = 0; k < 6; ++k) g[k] = 0.f;
          } else {
            g[5] = G * dLda;
            const float dpow = G * s.o * dLda;
            g[0] = -dpow * (s.A * dx + s.B * dy);
            g[1] = -dpow * (s.C * dy + s.B * dx);
            g[2] = -0.5f * dpow * dx * dx;
            g[3] = -dpow * dx * dy;
            g[4] = -0.5f * dpow * dy * dy;
          }
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, contrib);
      if (m == 0) continue;
      if (!contrib) {
#pragma unroll
        for (int k = 0; k < 9; ++k) g[k] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) g[k] = warp_sum(g[k]);
      if (lane == 0) {
        float* dst = a.acc[s_rec[j].ridx].g;
#pragma unroll
        for (int k = 0; k < 9; ++k) atomicAdd(dst + k, g[k]);
      }
    }
  }
}

}  // namespace

void launch_raster_fwd(const RasterArgs& a, uint32_t flags, float* rgb, float* t_final, int32_t* n_contrib,
                       cudaStream_t s) {
  if (a.n_tiles <= 0) return;
  if (flags & BGS_IMPORTANCE)
    k_raster_fwd<true><<<a.n_tiles, kBlock, 0, s>>>(a, rgb, t_final, n_contrib);
  else
    k_raster_fwd<false><<<a.n_tiles, kBlock, 0, s>>>(a, rgb, t_final, n_contrib);
}

void launch_raster_bwd(const RasterArgs& a, const float* dL, const float* t_final, const int32_t* n_contrib,
                       cudaStream_t s) {
  if (a.n_tiles <= 0) return;
  k_raster_bwd<<<a.n_tiles, kBlock, 0, s>>>(a, dL, t_final, n_contrib);
}

}  // namespace bgs
