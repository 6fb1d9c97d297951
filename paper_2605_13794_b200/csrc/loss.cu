// NEXT-4 supervision: the photometric loss of Eq.7 on the
// owned tiles, fused with its gradient, and the scale regulariser of Eq.8.
//
// Eq.7 per view: l_v = (1 - lambda) ||I^ - I||_1 + lambda (1 - SSIM(I^, I)), both terms means over
// the 3 H W elements; L_photo = (1/B) sum_b l_b.  SSIM (reading R34): the 3DGS form, per channel,
// 11x11 Gaussian window sigma = 1.5 (normalised), zero padding ("same" size), C1 = 0.01^2,
// C2 = 0.03^2, mean of the SSIM map over all pixels and channels.
//
// Gradient of the SSIM mean (derivation in DESIGN.md §10): with S(p) the map at p and
// f_mu = dS/dmu_x, f_s = dS/dsigma_x^2, f_c = dS/dsigma_xy at p,
//   dS_total/dx(q) = sum_p g(p - q) [a(p) + 2 x(q) b(p) + y(q) c(p)]
//   a = f_mu - 2 mu_x f_s - mu_y f_c,  b = f_s,  c = f_c   (a, b, c = 0 outside the image)
// so one CTA computes, for a 32x32 output tile of one channel, the window statistics and a, b, c
// on the tile + 5 px halo (from x, y on the tile + 10 px halo) entirely in shared memory
// (separable 11-tap passes) and convolves a, b, c back: no intermediate map touches HBM.
// Partial sums of |x - y| and S over the owned pixels go to one double2 per CTA, summed in a
// fixed order by k_loss_sums (deterministic).
//
// Eq.8: L_scale = (1/|V|) sum_{i in V} min_j sigma_ij over the visible set V (radius > 0, this
// view, all ranks); dL/dsigma_{i, argmin} = beta / |V| (first index among equal minima, R35).
// V on a rank = the records bgs_project emitted (radius > 0), so both passes read F records
// (index + scale row) instead of the whole shard.
#include "bgs_internal.cuh"

namespace bgs {
namespace {

constexpr int kLT = 32;             // output tile side
constexpr int kLH = 5;              // window half width
constexpr int kLS = kLT + 2 * kLH;  // statistics region side (42)
constexpr int kLX = kLT + 4 * kLH;  // input region side (52)
constexpr int kLThreads = 256;
constexpr float kC1 = 0.01f * 0.01f;
constexpr float kC2 = 0.03f * 0.03f;

// 65 KB (3 CTAs per SM): a, b, c reuse the inputs' space (x, y are dead after the horizontal
// statistics pass; step 5 re-reads its own output pixels from L2), and the horizontal sums of
// a, b, c reuse the statistics' space
struct LossSmem {
  union {
    struct {
      float x[kLX][kLX], y[kLX][kLX];  // inputs, zero outside the image (steps 1-2)
    } in;
    float abc[3][kLS][kLS];  // a, b, c on the statistics region (steps 3-4)
  } A;
  union {
    float h[5][kLX][kLS];     // horizontal window sums of x, y, xx, yy, xy (steps 2-3)
    float habc[3][kLS][kLT];  // horizontal window sums of a, b, c (steps 4-5)
  } B;
};

__device__ __forceinline__ bool owned_px(int px, int py, const LossArgs& a) {
  const int t = (py / kTile) * a.TX + px / kTile;
  return t >= a.t_begin && t < a.t_end;
}

__global__ void __launch_bounds__(kLThreads) k_loss_photo(LossArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LossSmem& S = *reinterpret_cast<LossSmem*>(smem_raw);
  const int c = blockIdx.z;
  const int X0 = blockIdx.x * kLT, Y0 = blockIdx.y * kLT;
  const int tid = threadIdx.x;
  const size_t plane = size_t(a.W) * a.H;
  const float* __restrict__ xp = a.x + c * plane;
  const float* __restrict__ yp = a.y + c * plane;
  const int bid = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  // any owned pixel in this output tile?  (16-px tiles: the 2x2 covered by a 32-px tile)
  bool any = false;
  for (int k = 0; k < 4; ++k) {
    const int px = X0 + (k & 1) * kTile, py = Y0 + (k >> 1) * kTile;
    any |= px < a.W && py < a.H && owned_px(px, py, a);
  }
  if (!any) {
    if (tid == 0) a.partials[bid] = make_double2(0.0, 0.0);
    return;
  }
  // 1. inputs on the tile + 10 px halo
  // (all of a thread's loads issued before its first shared store: 22 loads in flight)
  constexpr int kN1 = (kLX * kLX + kLThreads - 1) / kLThreads;
  float vx[kN1], vy[kN1];
#pragma unroll
  for (int t = 0; t < kN1; ++t) {
    const int i = tid + t * kLThreads;
    const int r = i / kLX, j = i % kLX;
    const int px = X0 - 2 * kLH + j, py = Y0 - 2 * kLH + r;
    const bool in = i < kLX * kLX && px >= 0 && px < a.W && py >= 0 && py < a.H;
    vx[t] = in ? __ldg(xp + size_t(py) * a.W + px) : 0.f;
    vy[t] = in ? __ldg(yp + size_t(py) * a.W + px) : 0.f;
  }
#pragma unroll
  for (int t = 0; t < kN1; ++t) {
    const int i = tid + t * kLThreads;
    if (i < kLX * kLX) {
      S.A.in.x[i / kLX][i % kLX] = vx[t];
      S.A.in.y[i / kLX][i % kLX] = vy[t];
    }
  }
  __syncthreads();
  // 2. horizontal window sums for the statistics columns: each item is a run of kR2 outputs of
  // one row, its kR2 + 10 inputs held in registers (2 shared loads per input instead of 11 per
  // tap)
  constexpr int kR2 = 6;
  for (int i = tid; i < kLX * (kLS / kR2); i += kLThreads) {
    const int r = i / (kLS / kR2), j0 = (i % (kLS / kR2)) * kR2;
    float u[kR2 + 2 * kLH], v[kR2 + 2 * kLH], uu[kR2 + 2 * kLH], vv[kR2 + 2 * kLH], uv[kR2 + 2 * kLH];
#pragma unroll
    for (int k = 0; k < kR2 + 2 * kLH; ++k) {
      u[k] = S.A.in.x[r][j0 + k];
      v[k] = S.A.in.y[r][j0 + k];
      uu[k] = u[k] * u[k];
      vv[k] = v[k] * v[k];
      uv[k] = u[k] * v[k];
    }
#pragma unroll
    for (int o = 0; o < kR2; ++o) {
      float mx = 0.f, my = 0.f, sxx = 0.f, syy = 0.f, sxy = 0.f;
#pragma unroll
      for (int k = 0; k < 2 * kLH + 1; ++k) {
        const float g = a.g[k];
        mx += g * u[o + k];
        my += g * v[o + k];
        sxx += g * uu[o + k];
        syy += g * vv[o + k];
        sxy += g * uv[o + k];
      }
      S.B.h[0][r][j0 + o] = mx;
      S.B.h[1][r][j0 + o] = my;
      S.B.h[2][r][j0 + o] = sxx;
      S.B.h[3][r][j0 + o] = syy;
      S.B.h[4][r][j0 + o] = sxy;
    }
  }
  __syncthreads();
  // 3. vertical sums -> statistics, SSIM map, a, b, c; partial sums over the owned output pixels
  // (runs of kR3 rows of one column, one map at a time through registers)
  constexpr int kR3 = 7;  // 42 columns x 6 runs = 252 items: one round of 256 threads
  double s_l1 = 0.0, s_ssim = 0.0;
  for (int i = tid; i < kLS * (kLS / kR3); i += kLThreads) {
    const int j = i % kLS, r0 = (i / kLS) * kR3;
    float m[5][kR3];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      float col[kR3 + 2 * kLH];
#pragma unroll
      for (int k = 0; k < kR3 + 2 * kLH; ++k) col[k] = S.B.h[q][r0 + k][j];
#pragma unroll
      for (int o = 0; o < kR3; ++o) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 2 * kLH + 1; ++k) acc += a.g[k] * col[o + k];
        m[q][o] = acc;
      }
    }
#pragma unroll
    for (int o = 0; o < kR3; ++o) {
      const int r = r0 + o;
      const int px = X0 - kLH + j, py = Y0 - kLH + r;
      float fa = 0.f, fb = 0.f, fc = 0.f;
      if (px >= 0 && px < a.W && py >= 0 && py < a.H) {
        const float mux = m[0][o], muy = m[1][o];
        const float sx2 = m[2][o] - mux * mux, sy2 = m[3][o] - muy * muy, sxy = m[4][o] - mux * muy;
        const float ln = 2.f * mux * muy + kC1, cn = 2.f * sxy + kC2;
        const float ld = mux * mux + muy * muy + kC1, cd = sx2 + sy2 + kC2;
        // one IEEE reciprocal: 1/ld = cd inv and 1/cd = ld inv (the products round once more than
        // the quotients would; fp32 tolerance of the parity tests)
        const float inv = 1.f / (ld * cd);
        const float ssim = ln * cn * inv;
        const float f_mu = 2.f * muy * cn * inv - ssim * 2.f * mux * (cd * inv);
        const float f_s = -ssim * (ld * inv);
        const float f_c = 2.f * ln * inv;
        fa = f_mu - 2.f * mux * f_s - muy * f_c;
        fb = f_s;
        fc = f_c;
        if (r >= kLH && r < kLH + kLT && j >= kLH && j < kLH + kLT && owned_px(px, py, a)) s_ssim += double(ssim);
      }
      S.A.abc[0][r][j] = fa;
      S.A.abc[1][r][j] = fb;
      S.A.abc[2][r][j] = fc;
    }
  }
  __syncthreads();
  // 4. horizontal window sums of a, b, c for the output columns (runs of kR4 outputs)
  constexpr int kR4 = 8;
  for (int i = tid; i < kLS * (kLT / kR4); i += kLThreads) {
    const int r = i / (kLT / kR4), j0 = (i % (kLT / kR4)) * kR4;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float row[kR4 + 2 * kLH];
#pragma unroll
      for (int k = 0; k < kR4 + 2 * kLH; ++k) row[k] = S.A.abc[q][r][j0 + k];
#pragma unroll
      for (int o = 0; o < kR4; ++o) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 2 * kLH + 1; ++k) acc += a.g[k] * row[o + k];
        S.B.habc[q][r][j0 + o] = acc;
      }
    }
  }
  __syncthreads();
  // 5. vertical sums -> dl/dx on the owned output pixels (runs of kR5 rows of one column)
  constexpr int kR5 = 4;
  float* __restrict__ dl = a.dL + c * plane;
  for (int i = tid; i < kLT * (kLT / kR5); i += kLThreads) {
    const int j = i % kLT, r0 = (i / kLT) * kR5;
    // this run's own pixels from L2, issued before the window sums
    float xs[kR5], ys[kR5];
#pragma unroll
    for (int o = 0; o < kR5; ++o) {
      const int px = X0 + j, py = Y0 + r0 + o;
      const bool in = px < a.W && py < a.H;
      xs[o] = in ? __ldg(xp + size_t(py) * a.W + px) : 0.f;
      ys[o] = in ? __ldg(yp + size_t(py) * a.W + px) : 0.f;
    }
    float u[3][kR5];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float col[kR5 + 2 * kLH];
#pragma unroll
      for (int k = 0; k < kR5 + 2 * kLH; ++k) col[k] = S.B.habc[q][r0 + k][j];
#pragma unroll
      for (int o = 0; o < kR5; ++o) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 2 * kLH + 1; ++k) acc += a.g[k] * col[o + k];
        u[q][o] = acc;
      }
    }
#pragma unroll
    for (int o = 0; o < kR5; ++o) {
      const int r = r0 + o;
      const int px = X0 + j, py = Y0 + r;
      if (px >= a.W || py >= a.H || !owned_px(px, py, a)) continue;
      const float xv = xs[o], yv = ys[o];
      const float dS = u[0][o] + 2.f * xv * u[1][o] + yv * u[2][o];
      const float sgn = xv > yv ? 1.f : (xv < yv ? -1.f : 0.f);
      s_l1 += double(fabsf(xv - yv));
      dl[size_t(py) * a.W + px] = a.k_l1 * sgn - a.k_ssim * dS;
    }
  }
  // block sums of the two partials (fixed order: deterministic)
  __shared__ double red[2][kLThreads / 32];
  for (int o = 16; o >= 1; o >>= 1) {
    s_l1 += __shfl_xor_sync(0xffffffffu, s_l1, o);
    s_ssim += __shfl_xor_sync(0xffffffffu, s_ssim, o);
  }
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = s_l1;
    red[1][tid >> 5] = s_ssim;
  }
  __syncthreads();
  if (tid == 0) {
    double u = 0.0, v = 0.0;
    for (int w = 0; w < kLThreads / 32; ++w) {
      u += red[0][w];
      v += red[1][w];
    }
    a.partials[bid] = make_double2(u, v);
  }
}

// one block: sums[0..1] = sum of the per-CTA partials in index order
__global__ void k_loss_sums(const double2* __restrict__ partials, int n, double* sums) {
  __shared__ double red[2][32];
  double u = 0.0, v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    u += partials[i].x;
    v += partials[i].y;
  }
  for (int o = 16; o >= 1; o >>= 1) {
    u += __shfl_xor_sync(0xffffffffu, u, o);
    v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = u;
    red[1][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double uu = 0.0, vv = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) {
      uu += red[0][w];
      vv += red[1][w];
    }
    sums[0] = uu;
    sums[1] = vv;
  }
}

// out = {l_v, L1_v, SSIM_v} from the (all-reduced) sums over the 3 H W elements
__global__ void k_loss_finish(const double* sums, double n_elem, double lambda, double* out) {
  const double l1 = sums[0] / n_elem, ssim = sums[1] / n_elem;
  out[0] = (1.0 - lambda) * l1 + lambda * (1.0 - ssim);
  out[1] = l1;
  out[2] = ssim;
}

// world > 1: the owned pixels of rgb into a zeroed full image (the all-reduce of that image gives
// every rank the halo pixels its windows need)
__global__ void k_owned_copy(const float* __restrict__ rgb, int W, int H, int TX, int t_begin, int t_end,
                             float* __restrict__ full) {
  const size_t plane = size_t(W) * H;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(plane)) return;
  const int px = int(i % W), py = int(i / W);
  const int t = (py / kTile) * TX + px / kTile;
  if (t < t_begin || t >= t_end) return;
  for (int c = 0; c < 3; ++c) full[c * plane + i] = rgb[c * plane + i];
}

// Eq.8, pass 1: per-block (sum of min sigma, count) over this view's projected records (the
// Gaussians with radius > 0: exactly the ones bgs_project emitted, rec_lidx = their local index)
constexpr int kScaleThreads = 256;
__global__ void __launch_bounds__(kScaleThreads) k_scale_sum(const float4* __restrict__ scale,
                                                              const uint32_t* __restrict__ lidx, int64_t n,
                                                              double2* __restrict__ partials) {
  double s = 0.0, cnt = 0.0;
  for (int64_t r = int64_t(blockIdx.x) * kScaleThreads + threadIdx.x; r < n; r += int64_t(gridDim.x) * kScaleThreads) {
    const float4 v = __ldg(scale + __ldg(lidx + r));
    s += double(fminf(v.x, fminf(v.y, v.z)));
    cnt += 1.0;
  }
  __shared__ double red[2][kScaleThreads / 32];
  for (int o = 16; o >= 1; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = s;
    red[1][threadIdx.x >> 5] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double u = 0.0, v = 0.0;
    for (int w = 0; w < kScaleThreads / 32; ++w) {
      u += red[0][w];
      v += red[1][w];
    }
    partials[blockIdx.x] = make_double2(u, v);
  }
}

__global__ void k_scale_finish(const double* sums, double* out) {
  out[0] = sums[1] > 0.0 ? sums[0] / sums[1] : 0.0;
  out[1] = sums[1];
}

// Eq.8, pass 2: g_scale[i][argmin] += beta / |V| for this view's records
__global__ void __launch_bounds__(kScaleThreads) k_scale_grad(const float4* __restrict__ scale,
                                                               const uint32_t* __restrict__ lidx, int64_t n,
                                                               const double* __restrict__ sums, float beta,
                                                               float* __restrict__ g_scale) {
  const double cnt = sums[1];
  if (cnt <= 0.0) return;
  const float k = float(double(beta) / cnt);
  for (int64_t r = int64_t(blockIdx.x) * kScaleThreads + threadIdx.x; r < n; r += int64_t(gridDim.x) * kScaleThreads) {
    const uint32_t i = __ldg(lidx + r);
    const float4 v = __ldg(scale + i);
    const int j = (v.x <= v.y && v.x <= v.z) ? 0 : (v.y <= v.z ? 1 : 2);
    atomicAdd(g_scale + 4 * size_t(i) + j, k);  // rows shared by views in flight: a reduction
  }
}

}  // namespace

size_t loss_smem_bytes() { return sizeof(LossSmem); }

int64_t loss_n_blocks(int W, int H) {
  return int64_t((W + kLT - 1) / kLT) * ((H + kLT - 1) / kLT) * 3;
}

void launch_loss_photo(const LossArgs& a, cudaStream_t s) {
  static std::atomic<int> attr[kMaxDevices];
  per_device(attr, [] {
    cudaFuncSetAttribute(k_loss_photo, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(LossSmem)));
    return 1;
  });
  const dim3 grid(unsigned((a.W + kLT - 1) / kLT), unsigned((a.H + kLT - 1) / kLT), 3u);
  k_loss_photo<<<grid, kLThreads, sizeof(LossSmem), s>>>(a);
}

void launch_loss_sums(const double2* partials, int n, double* sums, cudaStream_t s) {
  k_loss_sums<<<1, 1024, 0, s>>>(partials, n, sums);
}

void launch_loss_finish(const double* sums, double n_elem, double lambda, double* out, cudaStream_t s) {
  k_loss_finish<<<1, 1, 0, s>>>(sums, n_elem, lambda, out);
}

void launch_owned_copy(const float* rgb, int W, int H, int TX, int t_begin, int t_end, float* full, cudaStream_t s) {
  const int64_t n = int64_t(W) * H;
  if (n > 0) k_owned_copy<<<unsigned((n + 255) / 256), 256, 0, s>>>(rgb, W, H, TX, t_begin, t_end, full);
}

int scale_n_blocks(int64_t n) {
  const int64_t b = (n + kScaleThreads - 1) / kScaleThreads;
  return int(b < 4 * 148 ? (b > 0 ? b : 1) : 4 * 148);
}

void launch_scale_sum(const float4* scale, const uint32_t* lidx, int64_t n, double2* partials, cudaStream_t s) {
  k_scale_sum<<<unsigned(scale_n_blocks(n)), kScaleThreads, 0, s>>>(scale, lidx, n, partials);
}

void launch_scale_finish(const double* sums, double* out, cudaStream_t s) { k_scale_finish<<<1, 1, 0, s>>>(sums, out); }

void launch_scale_grad(const float4* scale, const uint32_t* lidx, int64_t n, const double* sums, float beta,
                       float* g_scale, cudaStream_t s) {
  if (n > 0)
    k_scale_grad<<<unsigned(scale_n_blocks(n)), kScaleThreads, 0, s>>>(scale, lidx, n, sums, beta, g_scale);
}

}  // namespace bgs
