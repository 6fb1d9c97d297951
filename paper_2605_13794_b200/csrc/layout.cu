// Shard layout (bgs_spatial_order): a Morton (Z-order) permutation of a shard's Gaussians.
//
// Not a step of the paper's method: a one-time data-layout utility.  The global id of a Gaussian
// is only a label (PAPER.md P:166-168 shards by index parity; P:170 / S:248 renumber on
// redistribution).  Storing each shard in Z-order makes the Gaussians that fall in one view
// lie close together in memory, so the per-view gathers and read-modify-writes of 16-B rows
// (projection, colour, projection backward, importance) touch whole DRAM granules instead of
// one 16-B row per 64-B granule.  Index parity over Z-ordered ids also gives every rank a
// spatially uniform subsample.
//
// Codes: 16 bits per axis over the shard's bounding box, interleaved into 48 bits, sorted with
// the library's onesweep passes (sort.cu) as (code, index) pairs; ties keep index order.
#include "bgs_internal.cuh"

namespace bgs {
namespace {

__device__ __forceinline__ unsigned int f2ord(float f) {
  const unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned int o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

__global__ void __launch_bounds__(256) k_bbox(const float4* mo, int64_t n, unsigned int* box /*min xyz, max xyz*/) {
  unsigned int mn[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, mx[3] = {0u, 0u, 0u};
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 p = __ldg(mo + i);
    const unsigned int o[3] = {f2ord(p.x), f2ord(p.y), f2ord(p.z)};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      mn[k] = min(mn[k], o[k]);
      mx[k] = max(mx[k], o[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    mn[k] = __reduce_min_sync(0xffffffffu, mn[k]);
    mx[k] = __reduce_max_sync(0xffffffffu, mx[k]);
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      atomicMin(box + k, mn[k]);
      atomicMax(box + 3 + k, mx[k]);
    }
  }
}

__device__ __forceinline__ unsigned long long spread3(unsigned int v) {  // 16 bits -> every 3rd bit
  unsigned long long x = v & 0xffffull;
  x = (x | (x << 16)) & 0x0000ff0000ffull;
  x = (x | (x << 8)) & 0x00f00f00f00full;
  x = (x | (x << 4)) & 0x0c30c30c30c3ull;
  x = (x | (x << 2)) & 0x249249249249ull;
  return x;
}

__global__ void __launch_bounds__(256) k_morton(const float4* mo, int64_t n, const unsigned int* box, SortArgs a) {
  __shared__ uint32_t s_hist[kMaxSortPasses][256];
  for (int j = threadIdx.x; j < kMaxSortPasses * 256; j += blockDim.x) (&s_hist[0][0])[j] = 0;
  __syncthreads();
  float lo[3], sc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    lo[k] = ord2f(box[k]);
    const float ext = ord2f(box[3 + k]) - lo[k];
    sc[k] = ext > 0.f ? 65535.f / ext : 0.f;
  }
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 p = __ldg(mo + i);
    const float v[3] = {p.x, p.y, p.z};
    unsigned int q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) q[k] = (unsigned int)fminf(65535.f, fmaxf(0.f, (v[k] - lo[k]) * sc[k]));
    const unsigned long long key = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
    a.keys[0][i] = key;
    a.vals[0][i] = uint32_t(i);
    for (int pz = 0; pz < a.n_passes; ++pz) atomicAdd(&s_hist[pz][(key >> (8 * pz)) & 255u], 1u);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < a.n_passes * 256; j += blockDim.x) {
    const uint32_t c = (&s_hist[0][0])[j];
    if (c) atomicAdd(a.digit_hist + j, c);
  }
}

__global__ void k_copy_perm(const SortArgs a, int64_t n, uint32_t* perm) {
  const uint32_t* v = a.pass_ctrl[kFinalSel] ? a.vals[1] : a.vals[0];
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    perm[i] = v[i];
}

unsigned grid_of(int64_t n) {
  int64_t b = (n + 255) / 256;
  return unsigned(b > 148 * 16 ? 148 * 16 : (b < 1 ? 1 : b));
}

}  // namespace

void launch_spatial_order(const float4* mean_opac, int64_t n, unsigned int* box, const SortArgs& a, uint32_t* perm,
                          cudaStream_t s, int64_t* launches) {
  k_bbox<<<grid_of(n), 256, 0, s>>>(mean_opac, n, box);
  k_morton<<<grid_of(n), 256, 0, s>>>(mean_opac, n, box, a);
  *launches += 2;
  launch_sort_passes(a, n, s, launches, 8);
  k_copy_perm<<<grid_of(n), 256, 0, s>>>(a, n, perm);
  *launches += 1;
}

}  // namespace bgs
