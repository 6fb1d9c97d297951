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
// Launch: one 256-thread CTA per owned 16x16 tile; warp w owns pixel rows 2w, 2w+1 of the tile
// (a 16x2 strip).  The tile's sorted list is staged kBatch = 512 records at a time into shared
// memory (structure of arrays, two records per thread, 128-bit loads).  Each staged record also
// gets the exact bounding box of its alpha >= 1/255 ellipse {d : d^T Q d <= -2 thr} (half extents
// sqrt(-2 thr (Q^-1)_xx), sqrt(-2 thr (Q^-1)_yy), widened by 1e-3 relative + 0.01 px so it is
// conservative under fp32 rounding).  Each warp tests 32 staged boxes at once against its strip
// (one per lane), ballots a hit mask and walks only the set bits, so records that cannot touch
// the strip cost nothing.  This changes no decision: every skipped pixel would fail the
// power >= thr test.  The CTA stops when all 256 pixels are done (__syncthreads_count once per
// 512 records) and a warp whose 32 pixels are done skips the batch (warp-ballot termination).
//
// Backward: per (warp, record) the 9 partial gradients are reduced with a transposed butterfly
// (8 values in 4+2+1+2 shuffles, each lane ending with one value; the 9th with 5 shuffles) and
// issued as 9 parallel red.global.add.f32 from 9 lanes instead of 45 shuffles + 9 serial
// atomics.
//
// The power expression is pinned with __fmul_rn/__fadd_rn (no FMA) so that the alpha-cut
// decision, n_contrib and a are bit-identical to the oracle's.
#include "bgs_internal.cuh"

namespace bgs {
namespace {

constexpr int kBlock = kTile * kTile;
constexpr int kBatch = 512;

struct Stage {
  float4 geo[kBatch];  // mx, my, A, B
  float4 co[kBatch];   // C, o, thr, ridx (bits)
  float4 rgb[kBatch];  // r, g, b, -
  float4 box[kBatch];  // xmin, xmax, ymin, ymax of the alpha >= 1/255 ellipse
};

__device__ __forceinline__ float pinned_power(float A, float B, float C, float dx, float dy) {
  // (-0.5 * ((A*dx)*dx + (C*dy)*dy)) - (B*dx)*dy, every op rounded (no contraction)
  const float t1 = __fmul_rn(__fmul_rn(A, dx), dx);
  const float t2 = __fmul_rn(__fmul_rn(C, dy), dy);
  const float t3 = __fmul_rn(__fmul_rn(B, dx), dy);
  return __fsub_rn(__fmul_rn(-0.5f, __fadd_rn(t1, t2)), t3);
}

__device__ __forceinline__ void stage(Stage& sm, int slot, const Rec* recv, uint32_t r) {
  const float4* p = reinterpret_cast<const float4*>(recv + r);
  const float4 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2);
  const float thr = float(-log(255.0 * double(q1.y)));  // alpha >= 1/255  <=>  power >= thr
  sm.geo[slot] = q0;
  sm.co[slot] = make_float4(q1.x, q1.y, thr, __uint_as_float(r));
  sm.rgb[slot] = make_float4(q1.z, q1.w, q2.x, 0.f);
  const float k = -2.0f * thr;
  const float det = q0.z * q1.x - q0.w * q0.w;
  if (k > 0.f && det > 0.f) {
    const float hx = sqrtf(k * q1.x / det) * 1.001f + 0.01f;
    const float hy = sqrtf(k * q0.z / det) * 1.001f + 0.01f;
    sm.box[slot] = make_float4(q0.x - hx, q0.x + hx, q0.y - hy, q0.y + hy);
  } else {
    sm.box[slot] = make_float4(1e30f, -1e30f, 1e30f, -1e30f);  // never contributes
  }
}

__device__ __forceinline__ bool box_hits(const float4& b, float x0, float x1, float y0, float y1) {
  return (b.x <= x1) & (b.y >= x0) & (b.z <= y1) & (b.w >= y0);
}

template <bool kImportance>
__global__ void __launch_bounds__(kBlock) k_raster_fwd(RasterArgs a, float* __restrict__ rgb,
                                                       float* __restrict__ t_final, int32_t* __restrict__ n_contrib) {
  __shared__ Stage sm;
  const uint32_t* __restrict__ vals = a.pass_ctrl[kFinalSel] ? a.vals[1] : a.vals[0];
  const int lt = blockIdx.x;
  const int tile = a.t_begin + lt;
  const int tx = tile % a.TX, ty = tile / a.TX;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int px = tx * kTile + (tid & (kTile - 1)), py = ty * kTile + (tid >> 4);
  const bool inside = px < a.W && py < a.H;
  const uint2 range = a.ranges[lt];
  const float pxf = float(px), pyf = float(py);
  const float wx0 = float(tx * kTile), wx1 = wx0 + float(kTile - 1);
  const float wy0 = float(ty * kTile + 2 * warp), wy1 = wy0 + 1.f;
  float T = 1.0f, cr = 0.f, cg = 0.f, cb = 0.f;
  uint32_t last = 0;
  bool done = !inside;
  for (uint32_t start = range.x; start < range.y; start += kBatch) {
    if (__syncthreads_count(done) == kBlock) break;
    const int n = int(range.y - start < uint32_t(kBatch) ? range.y - start : uint32_t(kBatch));
    for (int s = tid; s < n; s += kBlock) stage(sm, s, a.recv, __ldg(vals + start + s));
    __syncthreads();
    if (__all_sync(0xffffffffu, done)) continue;
    for (int w0 = 0; w0 < n; w0 += 32) {
      const int jl = w0 + lane;
      unsigned m = __ballot_sync(0xffffffffu, jl < n && box_hits(sm.box[jl], wx0, wx1, wy0, wy1));
      while (m) {
        const int j = w0 + __ffs(m) - 1;
        m &= m - 1;
        const float4 geo = sm.geo[j];
        const float4 co = sm.co[j];
        bool contrib = false;
        uint32_t fixed = 0;
        if (!done) {
          const float dx = geo.x - pxf, dy = geo.y - pyf;
          const float power = pinned_power(geo.z, geo.w, co.x, dx, dy);
          if (power <= 0.0f && power >= co.z) {
            const float G = __expf(power);
            const float alpha = fminf(0.99f, co.y * G);
            const float test_T = T * (1.0f - alpha);
            if (test_T < 0.0001f) {
              done = true;
            } else {
              const float4 c = sm.rgb[j];
              const float wgt = alpha * T;
              cr += c.x * wgt;
              cg += c.y * wgt;
              cb += c.z * wgt;
              T = test_T;
              last = start + j + 1 - range.x;
              contrib = true;
              if (kImportance) fixed = __float2uint_rn(wgt * 16777216.0f);
            }
          }
        }
        if (kImportance) {
          const unsigned cm = __ballot_sync(0xffffffffu, contrib);
          if (cm) {
            const uint32_t sum = __reduce_add_sync(0xffffffffu, fixed);
            if (lane == 0) {
              Acc* acc = a.acc + __float_as_uint(co.w);
              atomicAdd(&acc->a, uint32_t(__popc(cm)));
              atomicAdd(&acc->w, (unsigned long long)sum);
            }
          }
        }
      }
      if (__all_sync(0xffffffffu, done)) break;
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

__device__ __forceinline__ float xsel(bool hi, float a, float b) { return hi ? a : b; }

__global__ void __launch_bounds__(kBlock) k_raster_bwd(RasterArgs a, const float* __restrict__ dL,
                                                       const float* __restrict__ t_final,
                                                       const int32_t* __restrict__ n_contrib) {
  __shared__ Stage sm;
  __shared__ uint32_t s_maxlast;
  const uint32_t* __restrict__ vals = a.pass_ctrl[kFinalSel] ? a.vals[1] : a.vals[0];
  const int lt = blockIdx.x;
  const int tile = a.t_begin + lt;
  const int tx = tile % a.TX, ty = tile / a.TX;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int px = tx * kTile + (tid & (kTile - 1)), py = ty * kTile + (tid >> 4);
  const bool inside = px < a.W && py < a.H;
  const uint2 range = a.ranges[lt];
  const float pxf = float(px), pyf = float(py);
  const float wx0 = float(tx * kTile), wx1 = wx0 + float(kTile - 1);
  const float wy0 = float(ty * kTile + 2 * warp), wy1 = wy0 + 1.f;
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
  if (tid == 0) s_maxlast = 0;
  __syncthreads();
  // the warp's / block's deepest contributor bounds the work
  const uint32_t wlast = __reduce_max_sync(0xffffffffu, last);
  if (lane == 0) atomicMax(&s_maxlast, wlast);
  __syncthreads();
  const uint32_t end = range.x + s_maxlast;
  const uint32_t wend = range.x + wlast;
  const bool hi16 = lane & 16, hi8 = lane & 8, hi4 = lane & 4;
  const int my_idx = (hi16 ? 4 : 0) + (hi8 ? 2 : 0) + (hi4 ? 1 : 0);
  float acc_r = 0.f, acc_g = 0.f, acc_b = 0.f, last_alpha = 0.f, last_r = 0.f, last_g = 0.f, last_b = 0.f;
  for (int64_t bstart = int64_t(end) - kBatch; bstart > int64_t(range.x) - kBatch; bstart -= kBatch) {
    __syncthreads();
    const int jlo = int(int64_t(range.x) - bstart > 0 ? int64_t(range.x) - bstart : 0);
    for (int s = jlo + tid; s < kBatch; s += kBlock) stage(sm, s, a.recv, __ldg(vals + bstart + s));
    __syncthreads();
    // this warp only needs positions < wend
    const int jhi = int(int64_t(wend) - bstart < int64_t(kBatch) ? int64_t(wend) - bstart : int64_t(kBatch));
    for (int w0 = ((jhi - 1) & ~31); w0 >= (jlo & ~31) && jhi > jlo; w0 -= 32) {
      const int jl = w0 + lane;
      unsigned m = __ballot_sync(0xffffffffu, jl >= jlo && jl < jhi && box_hits(sm.box[jl], wx0, wx1, wy0, wy1));
      while (m) {
        const int b = 31 - __clz(m);
        m &= ~(1u << b);
        const int j = w0 + b;
        const uint32_t pos = uint32_t(bstart + j) - range.x;
        const float4 geo = sm.geo[j];
        const float4 co = sm.co[j];
        bool contrib = false;
        float g[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) g[k] = 0.f;
        if (pos < last) {
          const float dx = geo.x - pxf, dy = geo.y - pyf;
          const float power = pinned_power(geo.z, geo.w, co.x, dx, dy);
          if (power <= 0.0f && power >= co.z) {
            contrib = true;
            const float4 c = sm.rgb[j];
            const float G = __expf(power);
            const float og = co.y * G;
            const float alpha = fminf(0.99f, og);
            T = __fdividef(T, 1.0f - alpha);
            const float wgt = alpha * T;
            g[6] = wgt * dr;
            g[7] = wgt * dg;
            g[8] = wgt * db;
            acc_r = last_alpha * last_r + (1.f - last_alpha) * acc_r;
            acc_g = last_alpha * last_g + (1.f - last_alpha) * acc_g;
            acc_b = last_alpha * last_b + (1.f - last_alpha) * acc_b;
            last_alpha = alpha;
            last_r = c.x;
            last_g = c.y;
            last_b = c.z;
            const float dLda = T * ((c.x - acc_r) * dr + (c.y - acc_g) * dg + (c.z - acc_b) * db);
            if (og <= 0.99f) {  // clamped alpha is constant: true derivative 0 (R14)
              g[5] = G * dLda;
              const float dpow = G * co.y * dLda;
              g[0] = -dpow * (geo.z * dx + geo.w * dy);
              g[1] = -dpow * (co.x * dy + geo.w * dx);
              g[2] = -0.5f * dpow * dx * dx;
              g[3] = -dpow * dx * dy;
              g[4] = -0.5f * dpow * dy * dy;
            }
          }
        }
        if (!__any_sync(0xffffffffu, contrib)) continue;
        // transposed butterfly over g[0..7]: lane ends with the warp sum of g[my_idx]
        float v4[4], v2[2], v1;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float send = xsel(hi16, g[i], g[i + 4]);
          const float keep = xsel(hi16, g[i + 4], g[i]);
          v4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const float send = xsel(hi8, v4[i], v4[i + 2]);
          const float keep = xsel(hi8, v4[i + 2], v4[i]);
          v2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
        {
          const float send = xsel(hi4, v2[0], v2[1]);
          const float keep = xsel(hi4, v2[1], v2[0]);
          v1 = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
        v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
        float v8 = g[8];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v8 += __shfl_xor_sync(0xffffffffu, v8, o);
        float* dst = a.acc[__float_as_uint(co.w)].g;
        if ((lane & 3) == 0) atomicAdd(dst + my_idx, v1);
        if (lane == 1) atomicAdd(dst + 8, v8);
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
