// NEXT-3: adaptive density control with the phi-reweighted statistic and the LOD
// heritage rule, on the owned shard.
//
// bgs_densify_accumulate (per view, after bgs_route_reverse): for every local record of the view
// (= every Gaussian with radius > 0) stat_i += phi_i * |dL/dmean2d|_ndc and count_i += 1
// ("the gradient-magnitude statistic that drives clone-and-split is reweighted by this
// factor"; phi = 1 when no report exists).  dL/d(mx, my) come from the owner-summed pixel moments
// of the compositing backward: dL/dmx = -o (A g0 + B g1), dL/dmy = -o (B g0 + C g1);
// the norm is taken in NDC units (x W/2, y H/2: the 3DGS view-space statistic, reading R37).
//
// bgs_densify_apply ("periodically clones, splits, and prunes"; heritage P:194): with
// avg_i = stat_i / max(1, count_i) and the RAW parameters: clone if avg >= tau and
// max_j s_ij <= dense_extent, split if avg >= tau and max_j s_ij > dense_extent, and prune every
// row (parents and children alike) whose opacity < min_opacity.  Output order (3DGS, R39):
// surviving originals that were not split (input order), clones (parent order), first children of
// the split parents, second children.  Clone = exact copy, level kept; split child = parent with
// mu + R(q) (s * z), z ~ N(0, I) from a counter-based generator of (seed, parent gid, child, axis)
// (R40), log s - log 1.6, level + 1.  Adam moments: kept for originals, zero for new rows.
// Two passes: k_dc_count (per-block category counts) -> host-visible totals (HOST-SYNC, capacity
// check) -> k_dc_emit (block-local warp-ballot scans place every row).
#include "bgs_internal.cuh"

namespace bgs {
namespace {

constexpr int kDcThreads = 256;

__device__ __forceinline__ unsigned long long dc_mix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// u in (0, 1): top 53 bits of splitmix64(seed ^ splitmix64(k)) + half a quantum (as R30)
__device__ __forceinline__ double dc_uniform(unsigned long long seed, unsigned long long k) {
  const unsigned long long x = dc_mix64(seed ^ dc_mix64(k));
  return (double(x >> 11) + 0.5) * 1.1102230246251565e-16;
}

// standard normal of (seed, gid, child c, axis a): Box-Muller on the uniforms of counters 2k, 2k+1,
// k = gid * 8 + 3 c + a
__device__ __forceinline__ double dc_normal(unsigned long long seed, unsigned long long gid, int c, int ax) {
  const unsigned long long k = gid * 8ull + unsigned(3 * c + ax);
  const double u1 = dc_uniform(seed, 2 * k), u2 = dc_uniform(seed, 2 * k + 1);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

__global__ void __launch_bounds__(kDcThreads) k_dc_accumulate(DensifyAccArgs a) {
  const int64_t r = int64_t(blockIdx.x) * kDcThreads + threadIdx.x;
  if (r >= a.F) return;
  const uint32_t i = __ldg(a.lidx + r);
  const float4 q0 = __ldg(reinterpret_cast<const float4*>(a.recs + r));      // mx, my, A, B
  const float4 q1 = __ldg(reinterpret_cast<const float4*>(a.recs + r) + 1);  // C, o, ...
  const Acc& ac = a.acc[r];
  const float g0 = ac.g[0], g1 = ac.g[1];
  const float dmx = -q1.y * (q0.z * g0 + q0.w * g1);
  const float dmy = -q1.y * (q0.w * g0 + q1.x * g1);
  const float nx = dmx * a.half_w, ny = dmy * a.half_h;
  const float phi = a.phi ? float(__ldg(a.phi + i)) : 1.f;
  atomicAdd(a.stat + i, phi * sqrtf(nx * nx + ny * ny));  // views in flight share the statistic
  atomicAdd(a.count + i, 1u);
}

struct DcRow {
  bool keep, clone, split;  // original kept / one clone / two children (after pruning)
};

__device__ __forceinline__ DcRow dc_decide(const DensifyArgs& a, int64_t i) {
  // decisions in fp32 on exact monotone images of the thresholds (R39): sigmoid(l) < m <=>
  // l < logit(m), max s > e <=> max log s > log e (both thresholds rounded once on the host), and
  // avg = stat / max(1, count) with one IEEE division, as the oracle takes them
  const float4 ml = a.p_in[0][i];
  const float4 ls = a.p_in[2][i];
  const bool alive = !(ml.w < a.logit_min);  // children copy the parent's opacity
  const uint32_t c = a.count[i];
  const float avg = __fdiv_rn(a.stat[i], float(c > 0 ? c : 1u));
  const bool dens = avg >= a.tau;
  const bool big = fmaxf(ls.x, fmaxf(ls.y, ls.z)) > a.log_extent;
  DcRow d;
  d.split = alive && dens && big;
  d.clone = alive && dens && !big;
  d.keep = alive && !(dens && big);
  return d;
}

// per block: (kept originals, clones, split parents)
__global__ void __launch_bounds__(kDcThreads) k_dc_count(DensifyArgs a) {
  const int64_t i = int64_t(blockIdx.x) * kDcThreads + threadIdx.x;
  DcRow d{false, false, false};
  if (i < a.n) d = dc_decide(a, i);
  __shared__ uint32_t red[3][kDcThreads / 32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint32_t k = __popc(__ballot_sync(0xffffffffu, d.keep));
  const uint32_t c = __popc(__ballot_sync(0xffffffffu, d.clone));
  const uint32_t s = __popc(__ballot_sync(0xffffffffu, d.split));
  if (l == 0) {
    red[0][w] = k;
    red[1][w] = c;
    red[2][w] = s;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    uint32_t t = 0;
    for (int j = 0; j < kDcThreads / 32; ++j) t += red[threadIdx.x][j];
    a.block_counts[3 * int64_t(blockIdx.x) + threadIdx.x] = t;
  }
}

// exclusive scan of the per-block counts (one block; n_blocks <= a few 10^5), totals at the end
__global__ void k_dc_scan(uint32_t* counts, int64_t nb, unsigned long long* totals) {
  __shared__ unsigned long long carry[3];
  __shared__ unsigned long long wsum[3][32];
  if (threadIdx.x < 3) carry[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    const int64_t b = base + threadIdx.x;
    for (int c = 0; c < 3; ++c) {
      const unsigned long long v = b < nb ? counts[3 * b + c] : 0ull;
      // inclusive warp scan
      unsigned long long x = v;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) >= o) x += y;
      }
      if ((threadIdx.x & 31) == 31) wsum[c][threadIdx.x >> 5] = x;
      __syncthreads();
      if (threadIdx.x < 32) {
        unsigned long long t = threadIdx.x < (blockDim.x >> 5) ? wsum[c][threadIdx.x] : 0ull;
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
          if (threadIdx.x >= o) t += y;
        }
        wsum[c][threadIdx.x] = t;  // inclusive over warps
      }
      __syncthreads();
      const unsigned long long before = (threadIdx.x >> 5) ? wsum[c][(threadIdx.x >> 5) - 1] : 0ull;
      if (b < nb) counts[3 * b + c] = uint32_t(carry[c] + before + x - v);
      __syncthreads();
      if (threadIdx.x == 0) carry[c] += wsum[c][(blockDim.x >> 5) - 1];
      __syncthreads();
    }
  }
  if (threadIdx.x < 3) totals[threadIdx.x] = carry[threadIdx.x];
}

// 16-byte planes, level and activated 16-byte planes of one output row (one thread per row: the
// rows of a warp land in one or two contiguous runs)
__device__ __forceinline__ void put_row(const DensifyArgs& a, int64_t src, int64_t dst, bool fresh, float4 ml,
                                        float4 q, float4 ls, int lod) {
  a.p_out[0][dst] = ml;
  a.p_out[1][dst] = q;
  a.p_out[2][dst] = ls;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k = 0; k < 3; ++k) {
    a.m_out[k][dst] = fresh ? z4 : a.m_in[k][src];
    a.v_out[k][dst] = fresh ? z4 : a.v_in[k][src];
  }
  a.lod_out[dst] = uint8_t(lod);
  if (a.act[0]) {  // activated planes for the next render
    a.act[0][dst] = make_float4(ml.x, ml.y, ml.z, 1.f / (1.f + expf(-ml.w)));
    const float in = 1.f / sqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
    a.act[1][dst] = make_float4(q.x * in, q.y * in, q.z * in, q.w * in);
    a.act[2][dst] = make_float4(expf(ls.x), expf(ls.y), expf(ls.z), 0.f);
  }
}

// The 192-B SH rows (parameter, m, v and the activated copy) of the warp's output rows, copied by
// the whole warp one row at a time: lane e moves float4 e of the row set (12 per plane), so every
// load and store is a contiguous 192-B run instead of 16 B per lane at a 192-B stride.
__device__ __forceinline__ void copy_sh_rows(const DensifyArgs& a, int64_t src, int64_t d0, int64_t d1, bool f0,
                                             bool f1) {
  const int l = threadIdx.x & 31;
  const bool act = a.act[0] && a.sh_act && a.sh_act != a.sh_out;
  const int ne = act ? 48 : 36;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j = 0; j < 32; ++j) {
    const int64_t sj = __shfl_sync(0xffffffffu, src, j);
    for (int t = 0; t < 2; ++t) {
      const int64_t dj = __shfl_sync(0xffffffffu, t ? d1 : d0, j);
      const bool fj = __shfl_sync(0xffffffffu, t ? f1 : f0, j);
      if (dj < 0) continue;  // warp-uniform
      for (int e = l; e < ne; e += 32) {
        const int plane = e / 12, k = e % 12;
        float4 v;
        float* dstp;
        if (plane == 0) {
          v = reinterpret_cast<const float4*>(a.sh_in)[sj * 12 + k];
          dstp = a.sh_out;
        } else if (plane == 1) {
          v = fj ? z4 : reinterpret_cast<const float4*>(a.sh_m_in)[sj * 12 + k];
          dstp = a.sh_m_out;
        } else if (plane == 2) {
          v = fj ? z4 : reinterpret_cast<const float4*>(a.sh_v_in)[sj * 12 + k];
          dstp = a.sh_v_out;
        } else {
          v = reinterpret_cast<const float4*>(a.sh_in)[sj * 12 + k];
          dstp = a.sh_act;
        }
        reinterpret_cast<float4*>(dstp)[dj * 12 + k] = v;
      }
    }
  }
}

__global__ void __launch_bounds__(kDcThreads) k_dc_emit(DensifyArgs a) {
  const int64_t i = int64_t(blockIdx.x) * kDcThreads + threadIdx.x;
  DcRow d{false, false, false};
  if (i < a.n) d = dc_decide(a, i);
  // block-local exclusive ranks of the three categories
  __shared__ uint32_t wpre[3][kDcThreads / 32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const unsigned lt = (1u << l) - 1u;
  const unsigned bk = __ballot_sync(0xffffffffu, d.keep), bc = __ballot_sync(0xffffffffu, d.clone),
                 bs = __ballot_sync(0xffffffffu, d.split);
  if (l == 0) {
    wpre[0][w] = __popc(bk);
    wpre[1][w] = __popc(bc);
    wpre[2][w] = __popc(bs);
  }
  __syncthreads();
  uint32_t off[3] = {0, 0, 0};
  for (int j = 0; j < w; ++j)
    for (int c = 0; c < 3; ++c) off[c] += wpre[c][j];
  // every lane of a live warp stays for the cooperative SH copy (rows past n have no destination)
  const uint32_t* base = a.block_counts + 3 * int64_t(blockIdx.x);
  const int64_t K = int64_t(a.totals[0]), Cn = int64_t(a.totals[1]), Sn = int64_t(a.totals[2]);
  const int64_t ii = i < a.n ? i : 0;
  const float4 ml = a.p_in[0][ii], q = a.p_in[1][ii], ls = a.p_in[2][ii];
  const int lod = int(a.lod_in[ii]);
  int64_t d0 = -1, d1 = -1;
  bool f0 = false, f1 = true;
  if (d.keep) {
    d0 = int64_t(base[0]) + off[0] + __popc(bk & lt);
    put_row(a, i, d0, false, ml, q, ls, lod);
  }
  if (d.clone) {
    d1 = K + int64_t(base[1]) + off[1] + __popc(bc & lt);
    put_row(a, i, d1, true, ml, q, ls, lod);
  }
  if (d.split) {
    const int64_t r = int64_t(base[2]) + off[2] + __popc(bs & lt);
    d0 = K + Cn + r;
    d1 = K + Cn + Sn + r;
    f0 = true;
    const unsigned long long gid = (unsigned long long)i * unsigned(a.world) + unsigned(a.rank);
    // R(q) of the normalised quaternion (w, x, y, z), rows
    const float in = 1.f / sqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
    const float qw = q.x * in, qx = q.y * in, qy = q.z * in, qz = q.w * in;
    const float R[9] = {1.f - 2.f * (qy * qy + qz * qz), 2.f * (qx * qy - qw * qz), 2.f * (qx * qz + qw * qy),
                        2.f * (qx * qy + qw * qz), 1.f - 2.f * (qx * qx + qz * qz), 2.f * (qy * qz - qw * qx),
                        2.f * (qx * qz - qw * qy), 2.f * (qy * qz + qw * qx), 1.f - 2.f * (qx * qx + qy * qy)};
    const float s[3] = {expf(ls.x), expf(ls.y), expf(ls.z)};
    const float4 lsc = make_float4(ls.x - a.log_div, ls.y - a.log_div, ls.z - a.log_div, ls.w);
    for (int c = 0; c < 2; ++c) {
      float v[3];
      for (int ax = 0; ax < 3; ++ax) v[ax] = s[ax] * float(dc_normal(a.seed, gid, c, ax));
      const float4 mc = make_float4(ml.x + (R[0] * v[0] + R[1] * v[1] + R[2] * v[2]),
                                    ml.y + (R[3] * v[0] + R[4] * v[1] + R[5] * v[2]),
                                    ml.z + (R[6] * v[0] + R[7] * v[1] + R[8] * v[2]), ml.w);
      put_row(a, i, K + Cn + int64_t(c) * Sn + r, true, mc, q, lsc, lod + 1 < a.max_level ? lod + 1 : a.max_level);
    }
  }
  copy_sh_rows(a, ii, d0, d1, f0, f1);
}

}  // namespace

void launch_densify_accumulate(const DensifyAccArgs& a, cudaStream_t s) {
  if (a.F > 0) k_dc_accumulate<<<unsigned((a.F + kDcThreads - 1) / kDcThreads), kDcThreads, 0, s>>>(a);
}

int64_t densify_n_blocks(int64_t n) { return (n + kDcThreads - 1) / kDcThreads; }

void launch_densify_count(const DensifyArgs& a, cudaStream_t s) {
  const int64_t nb = densify_n_blocks(a.n);
  if (nb > 0) k_dc_count<<<unsigned(nb), kDcThreads, 0, s>>>(a);
  k_dc_scan<<<1, 1024, 0, s>>>(a.block_counts, nb, a.totals);
}

void launch_densify_emit(const DensifyArgs& a, cudaStream_t s) {
  const int64_t nb = densify_n_blocks(a.n);
  if (nb > 0) k_dc_emit<<<unsigned(nb), kDcThreads, 0, s>>>(a);
}

}  // namespace bgs
