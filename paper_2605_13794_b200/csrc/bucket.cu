// a5 pair emission, a6 sort, a7 ranges as a PER-TILE BUCKET SORT (bgs_sort_tiles, default path).
//
// PAPER.md P:152 ("tile-based front-to-back alpha compositing"), Eq.2 P:156-160 (N(p) depth
// ordered), SPEC S:116 / S:172 (ties by global id, reading R12): the pairs of every owned tile
// must end up ordered by (depth, gid).  The per-tile pair counts are known before any pair is
// written (world 1: the projection's 2D difference array of the rects, prefix-summed; world > 1:
// the all-reduced counts of a3, which are exactly what the owner receives), so
//   k_bucket_ranges  exclusive scan of the owned tiles' counts -> ranges [start, end) (a7, final)
//                    and one write cursor per tile;
//   k_bucket_emit    one warp expands the rects of 32 received records cooperatively (as k_emit)
//                    and places every (record, owned tile) pair in its tile's bucket at a cursor
//                    position (one atomic per group of lanes with the same tile: __match_any_sync),
//                    key = f32 bits(depth) - lo (depths are positive floats: the bit patterns order
//                    like the values and the subtraction is exact), value = record index; also the
//                    per-record raster constants (aux);
//   k_bucket_radix   one warp per owned tile: stable LSD radix sort of its bucket by the key,
//                    ceil(nb / 8) 8-bit passes (nb = bit width of the view's depth-bit span, ~22-24
//                    on Rubble views: 3 passes instead of 4 over (tile, depth) keys), ping-ponging
//                    between the two key / value buffers in global memory (a bucket is a few KB and
//                    stays in L2); then runs of exactly equal depth are ordered by global id.
// Per-tile work replaces the global passes and their decoupled look-back; the result is the unique
// order (tile, depth, gid), bit-identical to the onesweep path (BGS_SORT=onesweep).
#include <algorithm>

#include "bgs_internal.cuh"

namespace bgs {
namespace {

constexpr int kSortWarps = 8;     // warps per CTA of the per-tile radix sort (blockDim 256 = one digit per thread)
constexpr int kSmemKeys = 2048;   // large buckets up to this size are sorted in shared memory (32 KB)
constexpr int kWarpKeys = 512;    // buckets up to this size are sorted by one warp (8 KB per warp)

__global__ void __launch_bounds__(1024) k_bucket_ranges(const int32_t* __restrict__ counts, int t_begin, int n,
                                                        uint2* __restrict__ ranges, uint32_t* __restrict__ cursor,
                                                        uint32_t* __restrict__ work /*[3 + n]*/) {
  // one CTA: chunked exclusive scan (each thread a contiguous run of tiles).  work = {n_large, next
  // large, next small, large tiles...}: buckets above kWarpKeys are sorted by a whole CTA
  __shared__ uint32_t s_part[1024];
  __shared__ uint32_t s_nl;
  if (threadIdx.x == 0) s_nl = 0;
  const int nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int b = threadIdx.x * per, e = min(n, b + per);
  uint32_t loc = 0;
  for (int t = b; t < e; ++t) loc += uint32_t(counts[t_begin + t]);
  s_part[threadIdx.x] = loc;
  __syncthreads();
  for (int o = 1; o < nt; o <<= 1) {  // Hillis-Steele inclusive scan of the per-thread sums
    const uint32_t v = threadIdx.x >= o ? s_part[threadIdx.x - o] : 0u;
    __syncthreads();
    s_part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = s_part[threadIdx.x] - loc;
  for (int t = b; t < e; ++t) {
    const uint32_t c = uint32_t(counts[t_begin + t]);
    ranges[t] = c ? make_uint2(run, run + c) : make_uint2(0u, 0u);  // empty tiles [0, 0) as in O7
    cursor[t] = run;
    if (c > uint32_t(kWarpKeys)) work[3 + atomicAdd(&s_nl, 1u)] = uint32_t(t);
    run += c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    work[0] = s_nl;
    work[1] = 0;
    work[2] = 0;
  }
}

// Per-tile pair counts of a record set (rect coverage, the owned run [t_lo, t_hi)): one shared-
// memory histogram per CTA of a persistent grid, flushed with one global atomic per nonzero bin
// (4 global atomics per record into a (TX+1)(TY+1) difference array contend on a few thousand
// addresses and cost ~0.1 ms per Rubble view).  n_dev (nullable): record count on the device.
__global__ void __launch_bounds__(256) k_tile_count(const Rec* __restrict__ recs, int64_t n_cap,
                                                    const unsigned long long* __restrict__ n_dev, int TX, int t_lo,
                                                    int t_hi, int32_t* __restrict__ counts) {
  extern __shared__ int32_t s_cnt[];
  const int nt = t_hi - t_lo;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  int64_t n = n_cap;
  if (n_dev) n = min(n, int64_t(*n_dev));
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t rect = __ldg(&recs[r].rect);
    const int x0 = rect & 255, y0 = (rect >> 8) & 255, x1 = (rect >> 16) & 255, y1 = rect >> 24;
    for (int y = y0; y < y1; ++y) {
      const int lo = max(y * TX + x0, t_lo), hi = min(y * TX + x1, t_hi);
      for (int t = lo; t < hi; ++t) atomicAdd(&s_cnt[t - t_lo], 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    const int32_t c = s_cnt[i];
    if (c) atomicAdd(counts + i, c);
  }
}

// Persistent like k_emit: each CTA walks chunks of 256 received records.
__global__ void __launch_bounds__(256) k_bucket_emit(SortArgs a, uint32_t* __restrict__ cursor) {
  const int lane = threadIdx.x & 31;
  uint32_t* __restrict__ keys_out = reinterpret_cast<uint32_t*>(a.keys[0]);
  // depth bits of the received records span [lo, hi] (counters C_DLO / C_DHI)
  const uint32_t dlo = 0xffffffffu - uint32_t(a.counters[C_DLO]);
  const int64_t n_chunks = (a.n_recv + 255) / 256;
  for (int64_t ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
    const int64_t r = ch * 256 + threadIdx.x;
    uint32_t rect = 0, area = 0, dbits = 0;
    if (r < a.n_recv) {
      const uint4 q2 = __ldg(reinterpret_cast<const uint4*>(a.recv + r) + 2);  // (b, depth, gid, rect)
      rect = q2.w;
      dbits = q2.y;
      if (a.aux) {
        // per-record raster constants (see k_emit): thr = -ln(255 o) (D3, pinned fp64 ln) and the
        // conservative half extents of the alpha >= 1/255 ellipse
        const float4 q0 = __ldg(reinterpret_cast<const float4*>(a.recv + r));
        const float4 q1 = __ldg(reinterpret_cast<const float4*>(a.recv + r) + 1);
        const float thr = alpha_cut_thr(q1.y);
        const float k = -2.0f * thr;
        const float det = q0.z * q1.x - q0.w * q0.w;
        float hx = -1e30f, hy = -1e30f;  // empty box: never contributes
        if (k > 0.f && det > 0.f) {
          hx = sqrtf(k * q1.x / det) * 1.001f + 0.01f;
          hy = sqrtf(k * q0.z / det) * 1.001f + 0.01f;
        }
        a.aux[r] = make_float4(thr, hx, hy, 0.f);
      }
      const int x0 = rect & 255, y0 = (rect >> 8) & 255, x1 = (rect >> 16) & 255, y1 = rect >> 24;
      area = uint32_t((x1 - x0) * (y1 - y0));
    }
    uint32_t incl = area;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const uint32_t total_area = __shfl_sync(0xffffffffu, incl, 31);
    for (uint32_t chunk = 0; chunk < total_area; chunk += 32) {
      const uint32_t slot = chunk + lane;
      int j = 0;  // smallest lane j with incl[j] > slot
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, incl, j + step - 1);
        if (v <= slot) j += step;
      }
      j = min(j, 31);
      const uint32_t rj = __shfl_sync(0xffffffffu, rect, j);
      const uint32_t dj = __shfl_sync(0xffffffffu, dbits, j);
      const uint32_t ij = __shfl_sync(0xffffffffu, incl, j);
      const uint32_t aj = __shfl_sync(0xffffffffu, area, j);
      int lt = -1;
      if (slot < total_area) {
        const uint32_t k = slot - (ij - aj);
        const int x0 = rj & 255, y0 = (rj >> 8) & 255, x1 = (rj >> 16) & 255;
        const int w = x1 - x0;
        const int t = (y0 + int(k) / w) * a.TX + x0 + int(k) % w;
        if (t >= a.t_begin && t < a.t_end) lt = t - a.t_begin;
      }
      // one cursor atomic per group of lanes that place into the same tile
      const unsigned peers = __match_any_sync(0xffffffffu, lt);
      if (lt >= 0) {
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(cursor + lt, uint32_t(__popc(peers)));
        base = __shfl_sync(peers, base, leader);
        const uint32_t pos = base + __popc(peers & ((1u << lane) - 1u));
        if (int64_t(pos) < a.cap) {
          keys_out[pos] = dj - dlo;  // exact: depths are positive floats, bits - lo preserves order
          a.vals[0][pos] = uint32_t(ch * 256 + (threadIdx.x & ~31) + j);
        }
      }
    }
  }
}

// One CTA (8 warps) per owned tile sorts its bucket [r.x, r.y) by the u32 key with a stable LSD
// radix sort, ceil(nb / 8) 8-bit passes (nb = bit width of the view's depth-bit span: 3 passes on
// Rubble views).  Warp w owns the contiguous segment w of the bucket; per pass: per-warp digit
// counts (lanes with equal digits ranked by __match_any_sync, the group's lowest lane adds the
// count), offsets in (digit, warp) order by one block scan, then the stable scatter.  Buckets up to
// kSmemKeys entries are sorted in shared memory, larger ones between the two key / value buffers in
// global memory (L2-resident).  Runs of exactly equal depth are then ordered by global id (R12).
template <bool kShared>
__device__ void cta_radix(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, uint32_t n, int passes,
                          uint32_t (*s_cnt)[256], uint32_t* s_tot) {
  const int w = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint32_t seg = (n + kSortWarps - 1) / kSortWarps;
  const uint32_t sb = min(n, w * seg), se = min(n, sb + seg);
  for (int p = 0; p < passes; ++p) {
    const uint32_t* sk = (p & 1) ? k1 : k0;
    const uint32_t* sv = (p & 1) ? v1 : v0;
    uint32_t* dk = (p & 1) ? k0 : k1;
    uint32_t* dv = (p & 1) ? v0 : v1;
    const int sh = 8 * p;
#pragma unroll
    for (int k = 0; k < 8; ++k) s_cnt[w][lane * 8 + k] = 0;
    __syncwarp();
    for (uint32_t base = sb; base < se; base += 32) {
      const uint32_t i = base + lane;
      const uint32_t d = i < se ? (sk[i] >> sh) & 255u : 256u + lane;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      if (i < se && (peers & lt_mask) == 0) s_cnt[w][d] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // digit totals, exclusive scan over digits (thread d), then per-warp offsets in warp order
    const int d = threadIdx.x;  // blockDim == 256
    uint32_t tot = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) tot += s_cnt[ww][d];
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= uint32_t(o)) incl += t;
    }
    if (lane == 31) s_tot[w] = incl;
    __syncthreads();
    uint32_t run = incl - tot;
    for (int ww = 0; ww < w; ++ww) run += s_tot[ww];
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) {
      const uint32_t c = s_cnt[ww][d];
      s_cnt[ww][d] = run;
      run += c;
    }
    __syncthreads();
    for (uint32_t base = sb; base < se; base += 32) {
      const uint32_t i = base + lane;
      uint32_t key = 0, val = 0;
      if (i < se) {
        key = sk[i];
        val = sv[i];
      }
      const uint32_t dg = i < se ? (key >> sh) & 255u : 256u + lane;
      const unsigned peers = __match_any_sync(0xffffffffu, dg);
      uint32_t pos = 0;
      if (i < se) pos = s_cnt[w][dg] + __popc(peers & lt_mask);
      __syncwarp();
      if (i < se) {
        if ((peers & lt_mask) == 0) s_cnt[w][dg] += __popc(peers);
        dk[pos] = key;
        dv[pos] = val;
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

// Exact depth ties: each run of equal keys ordered by global id (insertion sort; runs are tiny).
// Threads tid, tid + nthr, ... own the run starts.
__device__ void fix_ties(const SortArgs& a, const uint32_t* k, uint32_t* v, uint32_t n, uint32_t tid, uint32_t nthr) {
  for (uint32_t i = tid; i + 1 < n; i += nthr) {
    const uint32_t key = k[i];
    if (k[i + 1] != key || (i > 0 && k[i - 1] == key)) continue;
    uint32_t e = i + 1;
    while (e + 1 < n && k[e + 1] == key) ++e;
    for (uint32_t x = i + 1; x <= e; ++x) {
      const uint32_t vx = v[x];
      const uint32_t gx = a.recv[vx].gid;
      uint32_t y = x;
      while (y > i && a.recv[v[y - 1]].gid > gx) {
        v[y] = v[y - 1];
        --y;
      }
      v[y] = vx;
    }
  }
}

// One warp: stable LSD radix sort of n <= kWarpKeys keys in shared memory (the same per-digit
// ranking as cta_radix with one segment), result back in (gk, gv).
__device__ void warp_radix(const SortArgs& a, uint32_t* gk, uint32_t* gv, uint32_t n, int passes, uint32_t* buf,
                           uint32_t* hist) {
  const uint32_t lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  uint32_t *k0 = buf, *v0 = buf + kWarpKeys, *k1 = buf + 2 * kWarpKeys, *v1 = buf + 3 * kWarpKeys;
  for (uint32_t i = lane; i < n; i += 32) {
    k0[i] = gk[i];
    v0[i] = gv[i];
  }
  __syncwarp();
  for (int p = 0; p < passes; ++p) {
    const uint32_t* sk = (p & 1) ? k1 : k0;
    const uint32_t* sv = (p & 1) ? v1 : v0;
    uint32_t* dk = (p & 1) ? k0 : k1;
    uint32_t* dv = (p & 1) ? v0 : v1;
    const int sh = 8 * p;
#pragma unroll
    for (int k = 0; k < 8; ++k) hist[lane * 8 + k] = 0;
    __syncwarp();
    for (uint32_t base = 0; base < n; base += 32) {
      const uint32_t i = base + lane;
      const uint32_t d = i < n ? (sk[i] >> sh) & 255u : 256u + lane;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      if (i < n && (peers & lt_mask) == 0) hist[d] += __popc(peers);
      __syncwarp();
    }
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = hist[lane * 8 + k];
      sum += v[k];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= uint32_t(o)) incl += t;
    }
    uint32_t run = incl - sum;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      hist[lane * 8 + k] = run;
      run += v[k];
    }
    __syncwarp();
    for (uint32_t base = 0; base < n; base += 32) {
      const uint32_t i = base + lane;
      uint32_t key = 0, val = 0;
      if (i < n) {
        key = sk[i];
        val = sv[i];
      }
      const uint32_t d = i < n ? (key >> sh) & 255u : 256u + lane;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      uint32_t pos = 0;
      if (i < n) pos = hist[d] + __popc(peers & lt_mask);
      __syncwarp();
      if (i < n) {
        if ((peers & lt_mask) == 0) hist[d] += __popc(peers);
        dk[pos] = key;
        dv[pos] = val;
      }
      __syncwarp();
    }
  }
  const uint32_t* fk = (passes & 1) ? k1 : k0;
  const uint32_t* fv = (passes & 1) ? v1 : v0;
  for (uint32_t i = lane; i < n; i += 32) {
    gk[i] = fk[i];
    gv[i] = fv[i];
  }
  __syncwarp();
  fix_ties(a, gk, gv, n, lane, 32);
}

// Persistent work-stealing sort of every owned tile's bucket: each CTA first takes whole large
// buckets (> kWarpKeys, listed by k_bucket_ranges) one at a time, then its warps take the small
// ones one per warp.
__global__ void __launch_bounds__(32 * kSortWarps) k_bucket_radix(SortArgs a, int n_tiles, uint32_t* work) {
  __shared__ uint32_t s_cnt[kSortWarps][256];
  __shared__ uint32_t s_tot[kSortWarps];
  __shared__ uint32_t s_item;
  extern __shared__ uint32_t s_buf[];  // large: [4][kSmemKeys]; small: per warp [4][kWarpKeys]
  const uint32_t lo = 0xffffffffu - uint32_t(a.counters[C_DLO]);
  const uint32_t hi = uint32_t(a.counters[C_DHI]);
  const uint32_t span = hi > lo ? hi - lo : 0u;
  const int nb = span ? 32 - __clz(span) : 0;
  const int passes = (nb + 7) / 8;
  const uint32_t n_large = work[0];
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(work + 1, 1u);
    __syncthreads();
    const uint32_t item = s_item;
    __syncthreads();
    if (item >= n_large) break;
    const uint2 r = a.ranges[work[3 + item]];
    const uint32_t n = r.y - r.x;
    uint32_t* gk0 = reinterpret_cast<uint32_t*>(a.keys[0]) + r.x;
    uint32_t* gv0 = a.vals[0] + r.x;
    if (passes > 0) {
      if (n <= uint32_t(kSmemKeys)) {
        uint32_t *k0 = s_buf, *v0 = s_buf + kSmemKeys, *k1 = s_buf + 2 * kSmemKeys, *v1 = s_buf + 3 * kSmemKeys;
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
          k0[i] = gk0[i];
          v0[i] = gv0[i];
        }
        __syncthreads();
        cta_radix<true>(k0, v0, k1, v1, n, passes, s_cnt, s_tot);
        const uint32_t* fk = (passes & 1) ? k1 : k0;
        const uint32_t* fv = (passes & 1) ? v1 : v0;
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
          gk0[i] = fk[i];
          gv0[i] = fv[i];
        }
      } else {
        uint32_t* gk1 = reinterpret_cast<uint32_t*>(a.keys[1]) + r.x;
        uint32_t* gv1 = a.vals[1] + r.x;
        cta_radix<false>(gk0, gv0, gk1, gv1, n, passes, s_cnt, s_tot);
        if (passes & 1) {  // every bucket ends in buffer 0
          for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            gk0[i] = gk1[i];
            gv0[i] = gv1[i];
          }
        }
      }
      __syncthreads();
    }
    fix_ties(a, gk0, gv0, n, threadIdx.x, blockDim.x);
    __syncthreads();
  }
  // small buckets: one warp each
  const int w = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t* buf = s_buf + size_t(w) * 4 * kWarpKeys;
  for (;;) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(work + 2, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= uint32_t(n_tiles)) break;
    const uint2 r = a.ranges[t];
    const uint32_t n = r.y - r.x;
    if (n <= 1 || n > uint32_t(kWarpKeys)) continue;
    uint32_t* gk0 = reinterpret_cast<uint32_t*>(a.keys[0]) + r.x;
    uint32_t* gv0 = a.vals[0] + r.x;
    warp_radix(a, gk0, gv0, n, passes, buf, s_cnt[w]);
  }
}

}  // namespace

void launch_tile_count(const Rec* recs, int64_t n_cap, const unsigned long long* n_dev, int TX, int t_lo, int t_hi,
                       int32_t* counts, cudaStream_t s) {
  const int nt = t_hi - t_lo;
  if (nt <= 0 || n_cap <= 0) return;
  const size_t smem = size_t(nt) * 4;
  static std::atomic<int> attr[kMaxDevices];
  per_device(attr, [] {
    cudaFuncSetAttribute(k_tile_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    return 1;
  });
  const int64_t blocks = std::min<int64_t>((n_cap + 255) / 256, int64_t(device_sm_count()) * 2);
  k_tile_count<<<unsigned(blocks), 256, smem, s>>>(recs, n_cap, n_dev, TX, t_lo, t_hi, counts);
}

void launch_bucket_sort(const SortArgs& a, const int32_t* tile_counts, uint32_t* cursor, uint32_t* order,
                        cudaStream_t s, int64_t* launches) {
  const int nt = a.t_end - a.t_begin;
  if (nt <= 0) return;
  k_bucket_ranges<<<1, 1024, 0, s>>>(tile_counts, a.t_begin, nt, a.ranges, cursor, cursor + nt);
  ++*launches;
  if (a.n_recv > 0) {
    const int64_t chunks = (a.n_recv + 255) / 256;
    static std::atomic<int> slots[kMaxDevices];
    const int max_blocks = per_device(slots, [] {
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bucket_emit, 256, 0);
      return device_sm_count() * (occ < 8 ? (occ > 0 ? occ : 1) : 8);
    });
    const int64_t blocks = chunks < max_blocks ? chunks : max_blocks;
    k_bucket_emit<<<unsigned(blocks), 256, 0, s>>>(a, cursor);
    ++*launches;
  }
  // the raster's longest-first tile order
  launch_tile_order(a.ranges, nt, order, s);
  ++*launches;
  const size_t smem = size_t(4) * kSmemKeys * 4 > size_t(kSortWarps) * 4 * kWarpKeys * 4
                          ? size_t(4) * kSmemKeys * 4
                          : size_t(kSortWarps) * 4 * kWarpKeys * 4;
  static std::atomic<int> attr[kMaxDevices];
  static std::atomic<int> grid[kMaxDevices];
  per_device(attr, [smem] {
    cudaFuncSetAttribute(k_bucket_radix, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    return 1;
  });
  const int g = per_device(grid, [smem] {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bucket_radix, 32 * kSortWarps, smem);
    return device_sm_count() * (occ > 0 ? occ : 1);
  });
  k_bucket_radix<<<unsigned(g), 32 * kSortWarps, smem, s>>>(a, nt, cursor + nt);
  ++*launches;
}

}  // namespace bgs
