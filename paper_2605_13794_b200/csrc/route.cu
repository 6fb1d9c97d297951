// a3 cost-aware tile ownership, a4 forward routing pack, a10 reverse gather-sum (bgs_route,
// bgs_route_reverse) for world > 1.  At world == 1 routing is the identity and none of these
// kernels runs.
//
// PAPER.md §3.2: "The image being rendered is partitioned into tiles, each assigned to one
// GPU. After projection, every GPU exchanges its projected Gaussians with every other GPU in a
// single all-to-all step. Each Gaussian is routed to whichever GPUs own the tiles it lands
// on"; "a cost-aware tile partition keeps rasterization load balanced" (no algorithm
// given: reading R24 / D6, integer midpoint-quantile split of c_t = pairs_t + 1 into
// contiguous runs).  Reverse: "gradients propagate through ... the screen-space routing".
//
// Slot assignment is deterministic: a record's position inside the segment for destination d
// is (block offset of its CTA for d) + (records of earlier warps of the CTA for d) + (earlier
// lanes of its warp for d), recomputed identically by the pack and by the reverse gather, so no
// per-(record, destination) index is stored.
#include "bgs_internal.cuh"

namespace bgs {
namespace {

__global__ void __launch_bounds__(1024) k_tile_costs(const int32_t* diff, int TX, int TY, int32_t* pairs) {
  // 2D inclusive prefix of the (TY+1)x(TX+1) difference array, restricted to TY x TX.
  extern __shared__ int32_t s_d[];
  const int W1 = TX + 1, n = (TY + 1) * W1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_d[i] = diff[i];
  __syncthreads();
  for (int y = threadIdx.x; y <= TY; y += blockDim.x) {
    int run = 0;
    for (int x = 0; x <= TX; ++x) {
      run += s_d[y * W1 + x];
      s_d[y * W1 + x] = run;
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x <= TX; x += blockDim.x) {
    int run = 0;
    for (int y = 0; y <= TY; ++y) {
      run += s_d[y * W1 + x];
      s_d[y * W1 + x] = run;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < TX * TY; t += blockDim.x) pairs[t] = s_d[(t / TX) * W1 + (t % TX)];
}

// given != nullptr: the caller's owner map (bgs_route's tile_owner_in) replaces the a3 split; it
// must be contiguous non-decreasing runs in [0, world) (checked: pown[world] = 1 when it is not)
__global__ void __launch_bounds__(1024) k_owner_map(const int32_t* pairs, int T, int world, int32_t* owner,
                                                    int32_t* run /*[2*world]: begin, end*/,
                                                    long long* pown /*[world + 1]*/, const int32_t* given) {
  extern __shared__ long long s_c[];  // T inclusive prefix of c_t
  // serial-per-chunk scan: T <= 65025, chunks per thread
  const int nt = blockDim.x;
  const int per = (T + nt - 1) / nt;
  const int b = threadIdx.x * per, e = min(T, b + per);
  long long loc = 0;
  for (int t = b; t < e; ++t) loc += (long long)pairs[t] + 1;
  __shared__ long long s_part[1024];
  s_part[threadIdx.x] = loc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run_ = 0;
    for (int i = 0; i < nt; ++i) {
      const long long v = s_part[i];
      s_part[i] = run_;
      run_ += v;
    }
    s_part[nt - 1] += 0;
    s_c[T] = run_;  // C
  }
  __syncthreads();
  long long P = s_part[threadIdx.x];
  for (int t = b; t < e; ++t) {
    s_c[t] = P;  // exclusive prefix P_t
    P += (long long)pairs[t] + 1;
  }
  __syncthreads();
  const long long C = s_c[T];
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += nt) {
    if (given) {
      const int32_t o = given[t];
      const bool bad = o < 0 || o >= world || (t > 0 && given[t - 1] > o);
      if (bad) s_bad = 1;
      owner[t] = o < 0 ? 0 : (o >= world ? world - 1 : o);
    } else {
      const long long ct = (long long)pairs[t] + 1;
      long long o = ((2 * s_c[t] + ct) * world) / (2 * C);
      owner[t] = int32_t(o < world - 1 ? o : world - 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) pown[world] = s_bad;
  if (threadIdx.x < world) {
    const int r = threadIdx.x;
    int lo = 0, hi = T;  // first t with owner >= r
    while (lo < hi) {
      const int m = (lo + hi) / 2;
      if (owner[m] >= r) hi = m; else lo = m + 1;
    }
    const int beg = lo;
    lo = 0;
    hi = T;
    while (lo < hi) {
      const int m = (lo + hi) / 2;
      if (owner[m] >= r + 1) hi = m; else lo = m + 1;
    }
    run[2 * r] = beg;
    run[2 * r + 1] = lo;
    long long p = 0;
    for (int t = beg; t < lo; ++t) p += pairs[t];
    pown[r] = p;
  }
}

// Record count: the host's F, or (batched steps, F_dev != nullptr) the projection counter on the
// device, bounded by the launch capacity F (the grid covers the capacity; CTAs past the count exit).
__device__ __forceinline__ int64_t rec_count(int64_t F, const unsigned long long* F_dev) {
  if (!F_dev) return F;
  const int64_t d = int64_t(*F_dev);
  return d < F ? d : F;
}

__device__ __forceinline__ uint32_t dest_mask_of(uint32_t rect, const int32_t* owner, int TX) {
  const int x0 = rect & 255, y0 = (rect >> 8) & 255, x1 = (rect >> 16) & 255, y1 = rect >> 24;
  uint32_t m = 0;
  for (int y = y0; y < y1; ++y) {
    const int lo = __ldg(owner + y * TX + x0), hi = __ldg(owner + y * TX + x1 - 1);
    m |= ((2u << hi) - 1u) & ~((1u << lo) - 1u);  // bits lo..hi (runs are contiguous)
  }
  return m;
}

// position of this lane's record among the CTA's records bound for d (block-local order)
__device__ __forceinline__ void block_positions(uint32_t mask, int world, uint32_t* pos_out,
                                                uint32_t (*s_w)[kMaxWorld]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t inwarp[kMaxWorld];
  for (int d = 0; d < world; ++d) {
    const unsigned b = __ballot_sync(0xffffffffu, (mask >> d) & 1u);
    inwarp[d] = __popc(b & lt);
    if (lane == 0) s_w[w][d] = __popc(b);
  }
  __syncthreads();
  for (int d = 0; d < world; ++d) {
    uint32_t off = 0;
    for (int ww = 0; ww < w; ++ww) off += s_w[ww][d];
    pos_out[d] = off + inwarp[d];
  }
}

__global__ void __launch_bounds__(kRouteBlock) k_dest_count(const Rec* recs, int64_t F_cap,
                                                            const unsigned long long* F_dev, const int32_t* owner,
                                                            int TX, int world, uint8_t* dest_mask,
                                                            uint32_t* block_counts) {
  __shared__ uint32_t s_w[kRouteBlock / 32][kMaxWorld];
  const int64_t F = rec_count(F_cap, F_dev);
  if (int64_t(blockIdx.x) * blockDim.x >= F && blockIdx.x > 0) return;  // past the count (block 0 always writes)
  const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t mask = 0;
  if (f < F) {
    mask = dest_mask_of(recs[f].rect, owner, TX);
    dest_mask[f] = uint8_t(mask);
  }
  uint32_t pos[kMaxWorld];
  block_positions(mask, world, pos, s_w);
  if (threadIdx.x < world) {
    uint32_t tot = 0;
    for (int ww = 0; ww < kRouteBlock / 32; ++ww) tot += s_w[ww][threadIdx.x];
    block_counts[int64_t(blockIdx.x) * world + threadIdx.x] = tot;
  }
}

__global__ void __launch_bounds__(kMaxWorld * 32) k_block_scan(uint32_t* counts, int64_t F_cap,
                                                               const unsigned long long* F_dev, int world,
                                                               unsigned long long* totals) {
  // one warp per destination: exclusive scan over blocks
  const int64_t F = rec_count(F_cap, F_dev);
  const int64_t n_blocks = F > 0 ? (F + kRouteBlock - 1) / kRouteBlock : 1;
  const int d = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (d >= world) return;
  unsigned long long run = 0;
  for (int64_t base = 0; base < n_blocks; base += 32) {
    const int64_t b = base + lane;
    const uint32_t v = b < n_blocks ? counts[b * world + d] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (b < n_blocks) counts[b * world + d] = uint32_t(run + incl - v);
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) totals[d] = run;
}

__global__ void __launch_bounds__(kRouteBlock) k_pack(const Rec* recs, int64_t F_cap,
                                                      const unsigned long long* F_dev, const uint8_t* dest_mask,
                                                      const uint32_t* block_offs, int world,
                                                      const int64_t* send_base, Rec* send) {
  __shared__ uint32_t s_w[kRouteBlock / 32][kMaxWorld];
  const int64_t F = rec_count(F_cap, F_dev);
  if (int64_t(blockIdx.x) * blockDim.x >= F) return;
  const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t mask = f < F ? dest_mask[f] : 0u;
  uint32_t pos[kMaxWorld];
  block_positions(mask, world, pos, s_w);
  if (f >= F) return;
  const float4* src = reinterpret_cast<const float4*>(recs + f);
  const float4 q0 = src[0], q1 = src[1], q2 = src[2];
  for (int d = 0; d < world; ++d) {
    if (!((mask >> d) & 1u)) continue;
    const int64_t o = send_base[d] + block_offs[int64_t(blockIdx.x) * world + d] + pos[d];
    float4* dst = reinterpret_cast<float4*>(send + o);
    dst[0] = q0;
    dst[1] = q1;
    dst[2] = q2;
  }
}

__global__ void __launch_bounds__(kRouteBlock) k_gather_sum(const Acc* rev, int64_t F_cap,
                                                            const unsigned long long* F_dev, const uint8_t* dest_mask,
                                                            const uint32_t* block_offs, int world,
                                                            const int64_t* send_base, Acc* out) {
  __shared__ uint32_t s_w[kRouteBlock / 32][kMaxWorld];
  const int64_t F = rec_count(F_cap, F_dev);
  if (int64_t(blockIdx.x) * blockDim.x >= F) return;
  const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t mask = f < F ? dest_mask[f] : 0u;
  uint32_t pos[kMaxWorld];
  block_positions(mask, world, pos, s_w);
  if (f >= F) return;
  Acc s;
#pragma unroll
  for (int k = 0; k < 9; ++k) s.g[k] = 0.f;
  s.a = 0;
  s.w = 0;
  for (int d = 0; d < world; ++d) {  // destination-rank ascending: deterministic order
    if (!((mask >> d) & 1u)) continue;
    const Acc& p = rev[send_base[d] + block_offs[int64_t(blockIdx.x) * world + d] + pos[d]];
#pragma unroll
    for (int k = 0; k < 9; ++k) s.g[k] += p.g[k];
    s.a += p.a;
    s.w += p.w;
  }
  out[f] = s;
}

// BGS_IMPORTANCE_ONLY reverse (scoring sweeps, no backward): per received record only (w, a),
// 12 B = uint3 {w lo, w hi, a} instead of the 48-B accumulator
__global__ void __launch_bounds__(256) k_pack_imp(const Acc* __restrict__ acc, int64_t R, uint3* __restrict__ out) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const unsigned long long w = acc[r].w;
  out[r] = make_uint3(uint32_t(w), uint32_t(w >> 32), acc[r].a);
}

__global__ void __launch_bounds__(kRouteBlock) k_gather_imp(const uint3* rev, int64_t F, const uint8_t* dest_mask,
                                                            const uint32_t* block_offs, int world,
                                                            const int64_t* send_base, Acc* out) {
  __shared__ uint32_t s_w[kRouteBlock / 32][kMaxWorld];
  const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t mask = f < F ? dest_mask[f] : 0u;
  uint32_t pos[kMaxWorld];
  block_positions(mask, world, pos, s_w);
  if (f >= F) return;
  Acc s;
#pragma unroll
  for (int k = 0; k < 9; ++k) s.g[k] = 0.f;
  s.a = 0;
  s.w = 0;
  for (int d = 0; d < world; ++d) {  // destination-rank ascending (integer sums: order-free anyway)
    if (!((mask >> d) & 1u)) continue;
    const uint3 p = rev[send_base[d] + block_offs[int64_t(blockIdx.x) * world + d] + pos[d]];
    s.w += (unsigned long long)p.x | ((unsigned long long)p.y << 32);
    s.a += p.z;
  }
  out[f] = s;
}

__global__ void k_reduce_i32(PtrList src, int32_t* dst, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t v = 0;
  for (int k = 0; k < src.n; ++k) v += static_cast<const int32_t*>(src.p[k])[i];
  dst[i] = v;
}

__global__ void k_reduce_u64(PtrList src, unsigned long long* dst, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long v = 0;
  for (int k = 0; k < src.n; ++k) v += static_cast<const unsigned long long*>(src.p[k])[i];
  dst[i] = v;
}

template <class T>
__global__ void k_reduce_sum(PtrList src, T* dst, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T v = static_cast<const T*>(src.p[0])[i];
  for (int k = 1; k < src.n; ++k) v += static_cast<const T*>(src.p[k])[i];  // rank order
  dst[i] = v;
}

}  // namespace

void launch_tile_costs(const int32_t* diff, int TX, int TY, int32_t* pairs_t, cudaStream_t s) {
  const size_t smem = size_t(TX + 1) * (TY + 1) * sizeof(int32_t);
  static std::atomic<int> attr[kMaxDevices];
  per_device(attr, [] {
    cudaFuncSetAttribute(k_tile_costs, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return 1;
  });
  k_tile_costs<<<1, 1024, smem, s>>>(diff, TX, TY, pairs_t);
}

void launch_owner_map(const int32_t* pairs_t, int T, int world, int32_t* owner, int32_t* run, long long* pown,
                      const int32_t* given, cudaStream_t s) {
  const size_t smem = size_t(T + 1) * sizeof(long long);
  static std::atomic<int> attr[kMaxDevices];
  per_device(attr, [] {
    cudaFuncSetAttribute(k_owner_map, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return 1;
  });
  k_owner_map<<<1, 1024, smem, s>>>(pairs_t, T, world, owner, run, pown, given);
}

// F: the record count, or with F_dev the capacity the grid covers (the count is read on the device)
void launch_dest_count(const Rec* recs, int64_t F, const unsigned long long* F_dev, const int32_t* owner, int TX,
                       int world, uint8_t* dest_mask, uint32_t* block_counts, cudaStream_t s) {
  const int64_t nb = (F + kRouteBlock - 1) / kRouteBlock;
  if (nb > 0)
    k_dest_count<<<unsigned(nb), kRouteBlock, 0, s>>>(recs, F, F_dev, owner, TX, world, dest_mask, block_counts);
}

void launch_block_scan(uint32_t* block_counts, int64_t F, const unsigned long long* F_dev, int world,
                       unsigned long long* totals, cudaStream_t s) {
  k_block_scan<<<1, kMaxWorld * 32, 0, s>>>(block_counts, F, F_dev, world, totals);
}

void launch_pack(const Rec* recs, int64_t F, const unsigned long long* F_dev, const uint8_t* dest_mask,
                 const uint32_t* block_offs, int world, const int64_t* send_base, Rec* send, cudaStream_t s) {
  const int64_t nb = (F + kRouteBlock - 1) / kRouteBlock;
  if (nb > 0)
    k_pack<<<unsigned(nb), kRouteBlock, 0, s>>>(recs, F, F_dev, dest_mask, block_offs, world, send_base, send);
}

void launch_gather_sum(const Acc* rev, int64_t F, const unsigned long long* F_dev, const uint8_t* dest_mask,
                       const uint32_t* block_offs, int world, const int64_t* send_base, Acc* out, cudaStream_t s) {
  const int64_t nb = (F + kRouteBlock - 1) / kRouteBlock;
  if (nb > 0)
    k_gather_sum<<<unsigned(nb), kRouteBlock, 0, s>>>(rev, F, F_dev, dest_mask, block_offs, world, send_base, out);
}

void launch_pack_imp(const Acc* acc, int64_t R, void* out, cudaStream_t s) {
  if (R > 0) k_pack_imp<<<unsigned((R + 255) / 256), 256, 0, s>>>(acc, R, static_cast<uint3*>(out));
}

void launch_gather_imp(const void* rev, int64_t F, const uint8_t* dest_mask, const uint32_t* block_offs, int world,
                       const int64_t* send_base, Acc* out, cudaStream_t s) {
  const int64_t nb = (F + kRouteBlock - 1) / kRouteBlock;
  if (nb > 0)
    k_gather_imp<<<unsigned(nb), kRouteBlock, 0, s>>>(static_cast<const uint3*>(rev), F, dest_mask, block_offs, world,
                                                      send_base, out);
}

void launch_reduce_sum_i32(PtrList src, int32_t* dst, int64_t n, cudaStream_t s) {
  if (n > 0) k_reduce_i32<<<unsigned((n + 255) / 256), 256, 0, s>>>(src, dst, n);
}

void launch_reduce_sum_f32(PtrList src, float* dst, int64_t n, cudaStream_t s) {
  if (n > 0) k_reduce_sum<float><<<unsigned((n + 255) / 256), 256, 0, s>>>(src, dst, n);
}

void launch_reduce_sum_f64(PtrList src, double* dst, int64_t n, cudaStream_t s) {
  if (n > 0) k_reduce_sum<double><<<unsigned((n + 255) / 256), 256, 0, s>>>(src, dst, n);
}

void launch_reduce_sum_u64(PtrList src, unsigned long long* dst, int64_t n, cudaStream_t s) {
  if (n > 0) k_reduce_u64<<<unsigned((n + 255) / 256), 256, 0, s>>>(src, dst, n);
}

}  // namespace bgs
