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
// Work decomposition (no block barriers): one 128-thread CTA per owned 16x16 tile, each of its
// 4 warps independently walks the tile's sorted list for its own 8x8 quadrant, two pixels per
// thread (rows r and r+4 of the quadrant: two independent dependency chains per thread; 8x8
// blocks cull ~8% more records per warp than the 16x4 strips used before).  A warp
// stages 32 records at a time (one per lane, 128-bit loads of the record rows and of the
// per-record constants precomputed by k_emit: thr and the half extents of the exact
// alpha >= 1/255 ellipse, widened to be conservative under fp32 rounding), ballots which of
// them can touch its strip, writes only those to its private shared-memory slots and walks the
// set bits.  Culled records change no decision (every skipped pixel would fail power >= thr).
// A warp stops as soon as its 64 pixels are done (forward) or it passes its deepest
// contributor (backward).
//
// Backward: the accumulator holds, per splat, sum gd, sum gd dx, sum gd dy, sum gd dx^2,
// sum gd dx dy, sum gd dy^2 (gd = G dL/dalpha, dx = mx - px, dy = my - py) and the colour
// partials; k_project_bwd turns the moments into dL/d(mean2d, conic) with the record's o, A, B, C.
// Per (warp, record) each lane first adds the partials of its two pixels.  With at most
// kBwdAtomicLanes contributing lanes each of them issues two red.global.add.v4.f32 and one scalar
// red; otherwise the 9 partial gradients are reduced with a transposed butterfly (8 values in
// 4+2+1+2 shuffles, each lane ending with one value; the 9th with 5 shuffles) and issued as 9
// parallel red.global.add.f32 from 9 lanes.
//
// The power expression is pinned (explicit __fmul_rn / __fmaf_rn, the oracle's neg_power order) so
// that the alpha-cut decision, n_contrib and a are bit-identical to the oracle's.
#include "bgs_internal.cuh"

namespace bgs {
namespace {

constexpr int kWarps = 4;  // warp blocks per tile unit (four 8x8 quadrants, or four 8x4 in a half tile)
#ifndef BGS_RASTER_CTA_WARPS
#define BGS_RASTER_CTA_WARPS 1
#endif
// warps per CTA: 1 = every warp block is its own CTA, so a warp that finishes its walk releases its
// slot at once instead of waiting for the slowest quadrant of its tile (with views in flight the
// slot goes to another view's kernels)
constexpr int kCtaWarps = BGS_RASTER_CTA_WARPS;
constexpr int kCtasPerUnit = kWarps / kCtaWarps;
constexpr int kThreads = 32 * kCtaWarps;
// Warp strip width: a warp's 32 lanes cover kStripW columns x 32/kStripW rows per pixel slot.
constexpr int kStripW = 8;  // 8x8 blocks cull ~8% more records per warp than 16x4 strips (measured)
constexpr int kLaneRows = 32 / kStripW;
constexpr int kStripsX = kTile / kStripW;  // warps side by side across a tile

struct WRec {
  float4 geo;  // mx, my, A/2, B
  float4 co;   // C/2, o, -thr, ridx (bits)
  float4 rgb;  // r, g, b, -
};

// nq = -power, in the pinned order the oracle uses (bgs_oracle.cpp neg_power):
// with hA = A/2, hC = C/2 (exact halvings), nq = fma(hC dy, dy, fma(B dx, dy, (hA dx) dx)), every
// product and fma rounded once, so the alpha-cut decision, n_contrib and a are bit-identical to
// the oracle's.  (hA dx) dx and B dx depend on the record and the lane's column only, so a slot
// costs one multiply and two FFMAs.
__device__ __forceinline__ float pinned_negpower(float hA, float B, float hC, float dx, float dy) {
  const float t1 = __fmul_rn(__fmul_rn(hA, dx), dx);
  return __fmaf_rn(__fmul_rn(hC, dy), dy, __fmaf_rn(__fmul_rn(B, dx), dy, t1));
}

// power <= 0 && power >= thr  <=>  nq >= 0 && nq <= -thr (also for +-0)
__device__ __forceinline__ bool in_cut(float nq, float nthr) { return nq >= 0.0f && nq <= nthr; }

__device__ __forceinline__ float fast_exp_neg(float nq) {
  // exp(-nq) for nq in [0, -thr] (< 6): ex2.approx.ftz of -nq*log2(e); the same instruction in
  // the forward and the backward, so both see identical alpha
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(nq * -1.4426950408889634f));
  return r;
}

__device__ __forceinline__ float fast_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Stage this lane's record (received-record index r, read from the sorted list one chunk ahead) and
// test its ellipse box against the warp's block [x0, x0+w-1] x [y0, y0+h-1].
__device__ __forceinline__ bool stage_test(const RasterArgs& a, uint32_t r, float x0, float y0, int w, int h,
                                           WRec& out) {
  const float4* p = reinterpret_cast<const float4*>(a.recv + r);
  const float4 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2);
  const float4 ax = __ldg(a.aux + r);
  out.geo = make_float4(q0.x, q0.y, 0.5f * q0.z, q0.w);
  out.co = make_float4(0.5f * q1.x, q1.y, -ax.x, __uint_as_float(r));
  // pixel slot i of every lane covers block rows [y0 + kLaneRows i, y0 + kLaneRows (i+1) - 1]: bit i
  // = the box reaches those rows (a warp-uniform skip of the slot's evaluation when it does not)
  uint32_t slots = 0;
  for (int i = 0; i * kLaneRows < h; ++i)
    slots |= uint32_t((q0.y - ax.z <= y0 + float(kLaneRows * (i + 1) - 1)) & (q0.y + ax.z >= y0 + float(kLaneRows * i)))
             << i;
  out.rgb = make_float4(q1.z, q1.w, q2.x, __uint_as_float(slots));
  return (q0.x - ax.y <= x0 + float(w - 1)) & (q0.x + ax.y >= x0) & (q0.y - ax.z <= y0 + float(h - 1)) &
         (q0.y + ax.z >= y0);
}

// Forward state of one pixel.  While the pixel composites, T >= 1e-4 > 0; when the early stop
// fires T is stored negated, which makes every later T (1 - alpha) negative, so the contribution
// test (T (1 - alpha) >= 1e-4) fails without a separate flag.  |T| is the transmittance.
struct PixF {
  float T, r, g, b;
  uint32_t last;
};

template <bool kColor>
__device__ __forceinline__ void eval_fwd1(PixF& p, const WRec& s, float dx, float dy, uint32_t pos, bool& c,
                                          uint32_t& f) {
  const float nq = pinned_negpower(s.geo.z, s.geo.w, s.co.x, dx, dy);
  const bool ok = in_cut(nq, s.co.z);
  const float alpha = fminf(0.99f, s.co.y * fast_exp_neg(nq));
  const float t = p.T * (1.0f - alpha);
  c = ok && t >= 0.0001f;  // false once stopped (T < 0)
  const float w = c ? alpha * p.T : 0.f;
  if (kColor) {  // a BGS_NO_COLOR view (scoring pass) has no colours: its image stays black
    p.r += s.rgb.x * w;
    p.g += s.rgb.y * w;
    p.b += s.rgb.z * w;
  }
  p.T = c ? t : (ok ? -fabsf(p.T) : p.T);
  p.last = c ? pos : p.last;
  f = __float2uint_rn(w * 16777216.0f);
}

// One warp composites a kStripW x (kLaneRows kPix) block of tile lt at (col0, row0): lane covers
// column col0 + lane % kStripW and rows row0 + lane / kStripW + kLaneRows i, i < kPix (kPix
// independent dependency chains per lane, branch-free).
template <bool kImportance, int kPix, bool kColor = true>
__device__ __forceinline__ void fwd_strip(const RasterArgs& a, const uint32_t* __restrict__ vals, int lt, int col0,
                                          int row0, int slot, WRec* mine, float* __restrict__ rgb,
                                          float* __restrict__ t_final, int32_t* __restrict__ n_contrib) {
  const int tile = a.t_begin + lt;
  const int tx = tile % a.TX, ty = tile / a.TX;
  const int lane = threadIdx.x & 31;
  const int px = tx * kTile + col0 + (lane % kStripW);
  const int pyb = ty * kTile + row0 + lane / kStripW;
  const uint2 range = a.ranges[lt];
  const float pxf = float(px);
  const float x0 = float(tx * kTile + col0), y0 = float(ty * kTile + row0);
  PixF p[kPix];
  float pyf[kPix];
#pragma unroll
  for (int i = 0; i < kPix; ++i) {
    const int py = pyb + kLaneRows * i;
    pyf[i] = float(py);
    p[i] = PixF{px < a.W && py < a.H ? 1.f : -1.f, 0.f, 0.f, 0.f, 0u};
  }
  // word of chunk k: ((range.x >> 5) + lt + k) kRasterSlots + slot (32-bit index: fewer live registers)
  uint32_t widx = ((range.x >> 5) + uint32_t(lt)) * kRasterSlots + uint32_t(slot);
  // the sorted list is read one chunk ahead, so each chunk's record fetch waits on one L2 round
  // trip (the record rows) instead of two (the list entry, then the rows)
  uint32_t r_next = range.x + lane < range.y ? __ldg(vals + range.x + lane) : 0u;
  for (uint32_t base = range.x; base < range.y; base += 32, widx += kRasterSlots) {
    bool done = true;
#pragma unroll
    for (int i = 0; i < kPix; ++i) done = done && p[i].T < 0.f;
    if (__all_sync(0xffffffffu, done)) break;
    const uint32_t idx = base + lane;
    const uint32_t r = r_next;
    r_next = idx + 32 < range.y ? __ldg(vals + idx + 32) : 0u;
    WRec st;
    const bool hit = idx < range.y && stage_test(a, r, x0, y0, kStripW, kLaneRows * kPix, st);
    unsigned m = __ballot_sync(0xffffffffu, hit);
    if (hit) mine[lane] = st;
    __syncwarp();
    // importance of the record this lane staged: the warp sums land in the staging lane's
    // registers and it issues the two atomics after the batch
    uint32_t my_w = 0, my_a = 0, contrib = 0;
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const WRec s = mine[j];
      const uint32_t pos = base + j + 1 - range.x;
      const float dx = s.geo.x - pxf;
      uint32_t fs = 0, cs = 0;
#pragma unroll
      for (int i = 0; i < kPix; ++i) {
        if (kPix > 1 && !((__float_as_uint(s.rgb.w) >> i) & 1u)) continue;  // warp-uniform: box misses these rows
        uint32_t f;
        bool c;
        eval_fwd1<kColor>(p[i], s, dx, s.geo.y - pyf[i], pos, c, f);
        fs += f;
        cs += uint32_t(c);
      }
      if (kImportance) {
        const uint32_t sum = __reduce_add_sync(0xffffffffu, fs);
        const uint32_t cnt = __reduce_add_sync(0xffffffffu, cs);
        if (lane == j) {
          my_w = sum;
          my_a = cnt;
        }
      } else {
        contrib |= uint32_t(cs != 0) << j;  // this lane's pixels; OR-reduced over the warp below
      }
    }
    // contributor mask of this chunk for the backward: bit j = some pixel of the block took record j
    if (kImportance) contrib = __ballot_sync(0xffffffffu, my_a != 0);
    else contrib = __reduce_or_sync(0xffffffffu, contrib);
    if (lane == 0) a.cmask[widx] = contrib;
    if (kImportance && my_a) {
      Acc* acc = a.acc + __float_as_uint(st.co.w);
      atomicAdd(&acc->a, my_a);
      atomicAdd(&acc->w, (unsigned long long)my_w);
    }
    __syncwarp();
  }
  const size_t plane = size_t(a.W) * a.H;
#pragma unroll
  for (int i = 0; i < kPix; ++i) {
    const int py = pyb + kLaneRows * i;
    if (px < a.W && py < a.H) {
      const size_t pix = size_t(py) * a.W + px;
      rgb[pix] = p[i].r;
      rgb[plane + pix] = p[i].g;
      rgb[2 * plane + pix] = p[i].b;
      t_final[pix] = fabsf(p[i].T);
      n_contrib[pix] = int32_t(p[i].last);
    }
  }
}

// Work split (longest-list-first order in tile_perm): the n_split heaviest tiles get TWO CTAs
// each (blocks 2k, 2k+1 = rows 0-7 / 8-15 of tile perm[k]; 4 warps x 8x4 blocks, one pixel per
// lane), every other tile one CTA (4 warps x 8x8 blocks, two pixels per lane).  A warp walks the
// whole list of its tile, so the heaviest tiles (6-8x the mean list length on Rubble views) set
// the kernel's makespan; halving their pixels per warp and their strip height shortens exactly
// those walks.
template <bool kImportance, bool kColor>
__global__ void __launch_bounds__(kThreads) k_raster_fwd(RasterArgs a, float* __restrict__ rgb,
                                                         float* __restrict__ t_final,
                                                         int32_t* __restrict__ n_contrib) {
  __shared__ WRec s_rec[kCtaWarps][32];
  const uint32_t* __restrict__ vals = a.pass_ctrl[kValsSel] ? a.vals[1] : a.vals[0];
  const int lw = threadIdx.x >> 5;
  const int warp = lw + int(blockIdx.x % kCtasPerUnit) * kCtaWarps;
  const int b = int(blockIdx.x / kCtasPerUnit);
  if (b < 2 * a.n_split) {
    const int lt = int(__ldg(a.tile_perm + (b >> 1)));
    fwd_strip<kImportance, 1, kColor>(a, vals, lt, kStripW * (warp % kStripsX), (b & 1) * 8 + kLaneRows * (warp / kStripsX),
                              (b & 1) * kWarps + warp, s_rec[lw], rgb, t_final, n_contrib);
  } else {
    const int lt = int(__ldg(a.tile_perm + (b - a.n_split)));
    fwd_strip<kImportance, 2, kColor>(a, vals, lt, kStripW * (warp % kStripsX), 2 * kLaneRows * (warp / kStripsX), warp,
                              s_rec[lw], rgb, t_final, n_contrib);
  }
}

// Backward state of one pixel.  s = sum over the contributors BEHIND the current one of
// (c_j . dL/dC) alpha_j T_j, so that (Eq.2 product rule, black background)
//   dL/dalpha_k = T_k (c_k . dL/dC) - s_k / (1 - alpha_k)
// with one scalar recursion (equivalent to 3DGS's per-channel accum_rec, fewer operations);
// T_k = T_{k+1} / (1 - alpha_k) reuses the same reciprocal.
struct PixB {
  float T, dr, dg, db, s;
  uint32_t last;
};

__device__ __forceinline__ void init_pixb(PixB& p, bool inside, size_t pix, size_t plane, const float* dL,
                                          const float* t_final, const int32_t* n_contrib) {
  p.T = 1.f;
  p.dr = p.dg = p.db = 0.f;
  p.s = 0.f;
  p.last = 0;
  if (inside) {
    p.T = t_final[pix];
    p.last = uint32_t(n_contrib[pix]);
    p.dr = dL[pix];
    p.dg = dL[plane + pix];
    p.db = dL[2 * plane + pix];
  }
}

// Backward evaluation of one pixel against one record (branch-free: `ok` predicates every
// update so the two pixels of a lane interleave); accumulates the pixel's partials into g[9].
// kFirst: g is written (the lane's first pixel) instead of accumulated, so no 0 + x adds
// (which the compiler keeps for signed-zero semantics)
template <bool kFirst>
__device__ __forceinline__ void acc(float& g, float v) {
  if (kFirst) g = v;
  else g += v;
}

template <bool kFirst>
__device__ __forceinline__ bool eval_bwd(PixB& p, const WRec& s, float dx, float dy, uint32_t pos, float* g) {
  const float nq = pinned_negpower(s.geo.z, s.geo.w, s.co.x, dx, dy);
  const bool ok = pos < p.last && in_cut(nq, s.co.z);
  const float G = fast_exp_neg(nq);
  const float og = s.co.y * G;
  const float alpha = fminf(0.99f, og);
  const float inv = ok ? fast_rcp(1.0f - alpha) : 1.0f;  // 1 - alpha >= 0.01: rel. error 2^-23
  p.T *= inv;                                              // T before this splat
  const float wgt = ok ? alpha * p.T : 0.f;
  acc<kFirst>(g[6], wgt * p.dr);
  acc<kFirst>(g[7], wgt * p.dg);
  acc<kFirst>(g[8], wgt * p.db);
  const float cdl = s.rgb.x * p.dr + s.rgb.y * p.dg + s.rgb.z * p.db;
  const float dLda = p.T * cdl - p.s * inv;
  p.s += cdl * wgt;  // now includes this splat for the ones in front of it
  // clamped alpha is constant: true derivative 0 (R14)
  const float gd = (ok && og <= 0.99f) ? G * dLda : 0.f;
  // dL/do = sum gd; the geometry partials are linear in the per-pixel moments of gd
  // (dL/dpower = o gd, dpower/dmx = -(A dx + B dy), ...), so the record's o, A, B, C are
  // applied once per record in k_project_bwd instead of once per pixel.  A lane's pixels share
  // their column, hence dx: the dx-moments sum gd dx = dx sum gd, sum gd dx^2 = dx^2 sum gd and
  // sum gd dx dy = dx sum gd dy are formed once per (lane, record) by finish_moments.
  acc<kFirst>(g[5], gd);
  const float gy = gd * dy;
  acc<kFirst>(g[1], gy);
  acc<kFirst>(g[4], gy * dy);
  return ok;
}

__device__ __forceinline__ void finish_moments(float* g, float dx) {
  g[0] = dx * g[5];
  g[2] = dx * g[0];
  g[3] = dx * g[1];
}

__device__ __forceinline__ float xsel(bool hi, float a, float b) { return hi ? a : b; }

// contributing lanes up to which a (warp, record) visit reduces with per-lane vector atomics
// (3 red instructions) instead of the butterfly (~54 instructions).  Measured on Rubble, 4 views in
// flight (same box): bwd 0.249 ms at 4, 0.238 at 6, 0.229 at 8, 0.220 at 12, 0.221 at 16; 9 scalar
// atomics per lane (round 1) were best at 4 (0.254 ms)
#ifndef BGS_BWD_ATOMIC_LANES
#define BGS_BWD_ATOMIC_LANES 12
#endif
constexpr int kBwdAtomicLanes = BGS_BWD_ATOMIC_LANES;

__device__ __forceinline__ void red_add_v4(float* p, float x, float y, float z, float w) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(x), "f"(y), "f"(z), "f"(w)
               : "memory");
}

// Backward of one warp's 16 x 2kPix strip starting at tile row `row0` (layout as fwd_strip).
// More pixels per lane amortise the per-(warp, record) gradient reduction; fewer shorten the
// walk of the heaviest tiles (k_raster_bwd's work split).
template <int kPix>
__device__ __forceinline__ void bwd_strip(const RasterArgs& a, const uint32_t* __restrict__ vals, int lt, int col0,
                                          int row0, int slot, WRec* mine, const float* __restrict__ dL,
                                          const float* __restrict__ t_final, const int32_t* __restrict__ n_contrib) {
  constexpr int kStripH = kLaneRows * kPix;
  const int tile = a.t_begin + lt;
  const int tx = tile % a.TX, ty = tile / a.TX;
  const int lane = threadIdx.x & 31;
  const int px = tx * kTile + col0 + (lane % kStripW);
  const int pyb = ty * kTile + row0 + lane / kStripW;
  const uint2 range = a.ranges[lt];
  const float pxf = float(px);
  const float x0 = float(tx * kTile + col0), y0 = float(ty * kTile + row0);
  const size_t plane = size_t(a.W) * a.H;
  PixB p[kPix];
  float pyf[kPix];
  uint32_t plast = 0;
#pragma unroll
  for (int i = 0; i < kPix; ++i) {
    const int py = pyb + kLaneRows * i;
    pyf[i] = float(py);
    init_pixb(p[i], px < a.W && py < a.H, size_t(py) * a.W + px, plane, dL, t_final, n_contrib);
    plast = p[i].last > plast ? p[i].last : plast;
  }
  const uint32_t wlast = __reduce_max_sync(0xffffffffu, plast);
  const bool hi16 = lane & 16, hi8 = lane & 8, hi4 = lane & 4;
  const int my_idx = (hi16 ? 4 : 0) + (hi8 ? 2 : 0) + (hi4 ? 1 : 0);
  // chunks of 32 list positions, from the warp's deepest contributor back to the front
  // the forward's contributor mask of a chunk: entries none of the block's pixels took are exactly
  // the ones every pixel's `ok` rejects here (same power, cut and last decisions).  Mask words and
  // list entries are read one chunk ahead (the walk goes back to front), so a chunk's record fetch
  // waits on one L2 round trip instead of three (mask, list entry, rows).
  const uint32_t* cmw = a.cmask + size_t((range.x >> 5) + uint32_t(lt)) * kRasterSlots + slot;
  int c = int((wlast + 31) / 32) - 1;
  uint32_t cw_next = c >= 0 ? __ldg(cmw + size_t(c) * kRasterSlots) : 0u;
  uint32_t r_next = c >= 0 && uint32_t(c) * 32 + lane < wlast ? __ldg(vals + range.x + uint32_t(c) * 32 + lane) : 0u;
  for (; c >= 0; --c) {
    const uint32_t pos0 = uint32_t(c) * 32;  // relative to range.x
    const uint32_t rel = pos0 + lane;
    const uint32_t cw = cw_next, r = r_next;
    if (c > 0) {
      cw_next = __ldg(cmw + size_t(c - 1) * kRasterSlots);
      r_next = __ldg(vals + range.x + rel - 32);
    }
    if (cw == 0u) continue;
    WRec st;
    const bool hit = ((cw >> lane) & 1u) && rel < wlast && stage_test(a, r, x0, y0, kStripW, kStripH, st);
    unsigned m = __ballot_sync(0xffffffffu, hit);
    if (hit) mine[lane] = st;
    __syncwarp();
    while (m) {
      const int b = 31 - __clz(m);
      m &= ~(1u << b);
      const WRec s = mine[b];
      const uint32_t pos = pos0 + b;
      float g[9];
      const float dx = s.geo.x - pxf;
      bool any;
      if (kPix == 2) {
        // warp-uniform: evaluate only the pixel slots whose rows the record's box reaches (a
        // skipped slot would fail the alpha cut: T, s and the partials are unchanged)
        const uint32_t slots = __float_as_uint(s.rgb.w);
        if (slots == 3u) {
          any = eval_bwd<true>(p[0], s, dx, s.geo.y - pyf[0], pos, g);
          any |= eval_bwd<false>(p[kPix - 1], s, dx, s.geo.y - pyf[kPix - 1], pos, g);
        } else if (slots == 1u) {
          any = eval_bwd<true>(p[0], s, dx, s.geo.y - pyf[0], pos, g);
        } else {
          any = eval_bwd<true>(p[kPix - 1], s, dx, s.geo.y - pyf[kPix - 1], pos, g);
        }
      } else {
        any = eval_bwd<true>(p[0], s, dx, s.geo.y - pyf[0], pos, g);
#pragma unroll
        for (int i = 1; i < kPix; ++i) any |= eval_bwd<false>(p[i], s, dx, s.geo.y - pyf[i], pos, g);
      }
      // no early exit when no lane contributed (the contributor mask makes that the rare case, and
      // the path below then issues nothing): the branch cost more than it saved (bwd -2%)
      const unsigned cm = __ballot_sync(0xffffffffu, any);
      finish_moments(g, dx);
      float* dst = a.acc[__float_as_uint(s.co.w)].g;
      // few contributing lanes: direct vector reductions (two red.v4 + one scalar per lane; the
      // 48-B accumulator rows are 16-B aligned) beat the 14-shuffle butterfly below
      if (__popc(cm) <= kBwdAtomicLanes) {
        if (any) red_add_v4(dst, g[0], g[1], g[2], g[3]), red_add_v4(dst + 4, g[4], g[5], g[6], g[7]),
            atomicAdd(dst + 8, g[8]);
        continue;
      }
      float v4[4], v2[2], v1;
      // transposed butterfly over g[0..7]: lane ends with the warp sum of g[my_idx]
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
      if ((lane & 3) == 0) atomicAdd(dst + my_idx, v1);
      if (lane == 1) atomicAdd(dst + 8, v8);
    }
    __syncwarp();
  }
}

// Same work split as k_raster_fwd.
__global__ void __launch_bounds__(kThreads) k_raster_bwd(RasterArgs a, const float* __restrict__ dL,
                                                         const float* __restrict__ t_final,
                                                         const int32_t* __restrict__ n_contrib) {
  __shared__ WRec s_rec[kCtaWarps][32];
  const uint32_t* __restrict__ vals = a.pass_ctrl[kValsSel] ? a.vals[1] : a.vals[0];
  const int lw = threadIdx.x >> 5;
  const int warp = lw + int(blockIdx.x % kCtasPerUnit) * kCtaWarps;
  const int b = int(blockIdx.x / kCtasPerUnit);
  if (b < 2 * a.n_split) {
    const int lt = int(__ldg(a.tile_perm + (b >> 1)));
    bwd_strip<1>(a, vals, lt, kStripW * (warp % kStripsX), (b & 1) * 8 + kLaneRows * (warp / kStripsX),
                 (b & 1) * kWarps + warp, s_rec[lw], dL, t_final, n_contrib);
  } else {
    const int lt = int(__ldg(a.tile_perm + (b - a.n_split)));
    bwd_strip<2>(a, vals, lt, kStripW * (warp % kStripsX), 2 * kLaneRows * (warp / kStripsX), warp, s_rec[lw], dL,
                 t_final, n_contrib);
  }
}

}  // namespace

// Heavy tiles split over two CTAs (k_raster_fwd).  BGS_SPLIT_TILES overrides the count (tuning).
static int split_count(int n_tiles) {
  // read at every launch (a getenv), so tests can force either work unit on small images
  const char* e = getenv("BGS_SPLIT_TILES");
  const int env = e ? atoi(e) : -1;
  const int sms = device_sm_count();
  // 2 x SMs: measured on Rubble (fwd+bwd ms per view) 0.58 unsplit, 0.530 at 148, 0.526 at 296,
  // 0.535 at 592
  const int want = env >= 0 ? env : 2 * sms;
  return want < n_tiles ? want : n_tiles;
}

int launch_raster_fwd(const RasterArgs& a, uint32_t flags, float* rgb, float* t_final, int32_t* n_contrib,
                      cudaStream_t s) {
  if (a.n_tiles <= 0) return 0;
  RasterArgs b = a;
  b.n_split = split_count(a.n_tiles);
  const unsigned grid = unsigned(a.n_tiles + b.n_split);
  const unsigned blocks = grid * kCtasPerUnit;
  if (a.no_color) {  // scoring views: the instrumented forward without colour
    if (flags & BGS_IMPORTANCE)
      k_raster_fwd<true, false><<<blocks, kThreads, 0, s>>>(b, rgb, t_final, n_contrib);
    else
      k_raster_fwd<false, false><<<blocks, kThreads, 0, s>>>(b, rgb, t_final, n_contrib);
  } else if (flags & BGS_IMPORTANCE) {
    k_raster_fwd<true, true><<<blocks, kThreads, 0, s>>>(b, rgb, t_final, n_contrib);
  } else {
    k_raster_fwd<false, true><<<blocks, kThreads, 0, s>>>(b, rgb, t_final, n_contrib);
  }
  return b.n_split;
}

void launch_raster_bwd(const RasterArgs& a, const float* dL, const float* t_final, const int32_t* n_contrib,
                       cudaStream_t s) {
  if (a.n_tiles <= 0) return;
  // light tiles: 2 pixels per lane (0.415 ms per Rubble view vs 0.73 ms with 4: the coarser strip
  // culls worse and a warp walks to the deepest of 128 pixels)
  // a.n_split: the forward's split (the contributor masks are per warp block of that layout)
  const RasterArgs& b = a;
  k_raster_bwd<<<unsigned(a.n_tiles + b.n_split) * kCtasPerUnit, kThreads, 0, s>>>(b, dL, t_final, n_contrib);
}

}  // namespace bgs
