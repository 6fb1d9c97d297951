// a5 pair emission, a6 onesweep LSD radix sort, a7 tile ranges (bgs_sort_tiles).
//
// PAPER.md P:152 ("rasterized by tile-based front-to-back alpha compositing"), Eq.2
// (N(p) depth-ordered), SPEC S:116 / S:172 (ties by global id, reading R12).
//
// Key (32 bits) = (local tile << kd) | ((f32 bits(depth) - lo) >> sd) (KeyLayout,
// bgs_internal.cuh).  depth > near_clip > 0, so the unsigned order of the bits is the numeric
// order of the depths and subtracting the minimum maps them exactly onto [0, 2^nb); the lowest
// sd = nb - kd of those bits are dropped when nb + tile bits > 32 and k_ranges_fixup orders the
// resulting runs of equal keys by (full depth bits, gid), so the final order is exact.  Rubble
// views: nb = 22..24 and 12 tile bits -> 4 passes over 4-byte keys (vs 6 over 8-byte keys for
// tile << 31 | bits).  The digit histograms of the passes that see depth bits only are added
// once per record (weighted by its owned pair count); only tile-bearing digits count per pair.
//
// a5: one warp expands the rects of 32 received records cooperatively (slot = position in a
//     rect, warp-scan + 5-step shuffle search for the owning lane), keeps the slots whose tile
//     is owned, compacts them with a ballot and writes them coalesced after ONE atomicAdd per
//     warp (warp-aggregated atomics, north_star).  The same kernel builds the 8-bit digit
//     histograms of every pass (the "upfront" histogram of onesweep) in shared memory.
// a6: per pass, a CTA takes the next partition of 4096 keys (dynamic partition id so the
//     look-back always waits on CTAs that already run), ranks keys inside each warp with
//     __match_any_sync, publishes its per-digit counts with decoupled look-back (flag in
//     bits 31:30 of one 32-bit word: 1 = aggregate, 2 = inclusive prefix), reorders the
//     partition in shared memory and writes each digit run contiguously.  Passes whose digit
//     is the same for every key are skipped on the device (no host round trip): a tiny scan
//     kernel writes per-pass active flags and ping-pong selectors.
// a7: one pass over the sorted keys writes [start, end) per tile and re-orders runs of
//     identical (tile, depth) keys by global id (insertion sort; runs are tiny).
#include "bgs_internal.cuh"

namespace bgs {
namespace {

constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1u;
// pass_ctrl layout
constexpr int kCtrlActive = 0;   // [8]
constexpr int kCtrlSel = 8;      // [7] input buffer of pass p
constexpr int kCtrlPart = 16;    // [8] partition counters

__device__ __forceinline__ uint32_t make_key(uint32_t lt, uint32_t dbits, KeyLayout kl) {
  return uint32_t((static_cast<unsigned long long>(lt) << kl.kd) | ((dbits - kl.lo) >> kl.sd));
}

// Exclusive scan of one value per thread over a 256-thread CTA (warp shuffles + 8 warp totals).
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t* s_w /*[8]*/) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  uint32_t wb = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) wb += k < w ? s_w[k] : 0u;
  __syncthreads();  // s_w reusable by the caller
  return wb + inc - v;
}

__global__ void __launch_bounds__(256) k_depth_range(const Rec* __restrict__ recv, int64_t n,
                                                     unsigned long long* counters) {
  uint32_t dhi = 0, dlo = 0;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t db = __float_as_uint(__ldg(&recv[r].depth));
    dhi = db > dhi ? db : dhi;
    dlo = (0xffffffffu - db) > dlo ? (0xffffffffu - db) : dlo;
  }
  dhi = __reduce_max_sync(0xffffffffu, dhi);
  dlo = __reduce_max_sync(0xffffffffu, dlo);
  if ((threadIdx.x & 31) == 0 && dhi) {
    atomicMax(counters + C_DHI, (unsigned long long)dhi);
    atomicMax(counters + C_DLO, (unsigned long long)dlo);
  }
}

// Persistent: each CTA walks chunks of 256 received records and keeps its digit histograms in
// shared memory across them, so the global histogram atomics scale with the grid, not with R.
__global__ void __launch_bounds__(256) k_emit(SortArgs a) {
  __shared__ uint32_t s_hist[kMaxSortPasses][256];
  __shared__ uint32_t s_wown[8];
  __shared__ unsigned long long s_bbase;
  for (int j = threadIdx.x; j < kMaxSortPasses * 256; j += blockDim.x) (&s_hist[0][0])[j] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const KeyLayout kl = key_layout(a.counters[C_DLO], a.counters[C_DHI], a.tbits);
  const int p_pair = kl.kd / 8;  // passes below this one see depth bits only
  uint32_t* __restrict__ keys_out = reinterpret_cast<uint32_t*>(a.keys[0]);
  const int64_t n_chunks = (a.n_recv + 255) / 256;
  for (int64_t ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
  const int64_t r = ch * 256 + threadIdx.x;
  uint32_t rect = 0, area = 0, own = 0, dbits = 0;
  if (r < a.n_recv) {
    const uint4 q2 = __ldg(reinterpret_cast<const uint4*>(a.recv + r) + 2);  // (b, depth, gid, rect)
    rect = q2.w;
    dbits = q2.y;
    if (a.aux) {
      // per-record raster constants, computed once here instead of once per (tile, warp):
      // thr = -ln(255 o) (alpha >= 1/255 <=> power >= thr, D3; pinned fp64 ln, bgs_internal.cuh) and the half extents of the
      // ellipse {d : d^T Q d <= -2 thr} (sqrt(-2 thr (Q^-1)_xx), sqrt(-2 thr (Q^-1)_yy)) widened
      // by 1e-3 relative + 0.01 px so that box culling is conservative under fp32 rounding
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
    // owned count: rows of the rect intersected with the contiguous run [t_begin, t_end)
    for (int y = y0; y < y1; ++y) {
      const int lo = max(y * a.TX + x0, a.t_begin), hi = min(y * a.TX + x1, a.t_end);
      own += hi > lo ? uint32_t(hi - lo) : 0u;
    }
    // digits made of depth bits only are the same for every pair of this record: one weighted
    // add per record instead of one per pair
    if (own) {
      const uint32_t dk = (dbits - kl.lo) >> kl.sd;
      for (int p = 0; p < p_pair && p < a.n_passes; ++p) atomicAdd(&s_hist[p][(dk >> (8 * p)) & 255u], own);
    }
  }
  // warp inclusive scans of area and own
  uint32_t incl = area, oincl = own;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    const uint32_t w = __shfl_up_sync(0xffffffffu, oincl, o);
    if (lane >= o) {
      incl += v;
      oincl += w;
    }
  }
  const uint32_t total_area = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t total_own = __shfl_sync(0xffffffffu, oincl, 31);
  // one global atomic per chunk (warp totals scanned in shared memory)
  const int warp = threadIdx.x >> 5;
  if (lane == 0) s_wown[warp] = total_own;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int w = 0; w < 8; ++w) {
      const uint32_t c = s_wown[w];
      s_wown[w] = run;
      run += c;
    }
    s_bbase = run ? atomicAdd(a.counters + C_P, (unsigned long long)run) : 0ull;
  }
  __syncthreads();
  const unsigned long long base = s_bbase + s_wown[warp];
  const int npass = a.n_passes;
  uint32_t run = 0;
  for (uint32_t chunk = 0; chunk < total_area; chunk += 32) {
    const uint32_t slot = chunk + lane;
    bool ok = false;
    uint32_t key = 0;
    uint32_t val = 0;
    // smallest lane j with incl[j] > slot
    int j = 0;
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
    if (slot < total_area) {
      const uint32_t k = slot - (ij - aj);
      const int x0 = rj & 255, y0 = (rj >> 8) & 255, x1 = (rj >> 16) & 255;
      const int w = x1 - x0;
      const int t = (y0 + int(k) / w) * a.TX + x0 + int(k) % w;
      if (t >= a.t_begin && t < a.t_end) {
        ok = true;
        key = make_key(uint32_t(t - a.t_begin), dj, kl);
        val = uint32_t(ch * 256 + (threadIdx.x & ~31) + j);
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      const unsigned long long pos = base + run + __popc(m & ((1u << lane) - 1u));
      if ((int64_t)pos < a.cap) {
        keys_out[pos] = key;
        a.vals[0][pos] = val;
      }
      for (int p = p_pair; p < npass; ++p) atomicAdd(&s_hist[p][(key >> (8 * p)) & 255u], 1u);
    }
    run += __popc(m);
  }
  __syncthreads();  // s_wown / s_bbase reused by the next chunk
  }
  for (int j = threadIdx.x; j < a.n_passes * 256; j += blockDim.x) {
    const uint32_t c = (&s_hist[0][0])[j];
    if (c) atomicAdd(a.digit_hist + j, c);
  }
}

// One CTA: per pass, detect constant digits (inactive pass), exclusive-scan the digit
// histogram in place, and assign ping-pong input selectors.
__global__ void __launch_bounds__(256) k_digit_scan(SortArgs a) {
  __shared__ uint32_t s_w[8];
  const unsigned long long P = a.counters[C_P];
  uint32_t sel = 0;
  for (int p = 0; p < a.n_passes; ++p) {
    const uint32_t c = a.digit_hist[p * 256 + threadIdx.x];
    // all keys share this digit (also P == 0): the pass is skipped
    const int active = !__syncthreads_or((unsigned long long)c == P);
    a.digit_hist[p * 256 + threadIdx.x] = block_excl_scan256(c, s_w);
    if (threadIdx.x == 0) {
      a.pass_ctrl[kCtrlActive + p] = uint32_t(active);
      a.pass_ctrl[kCtrlSel + p] = sel;
    }
    if (active) sel ^= 1u;
  }
  if (threadIdx.x == 0) a.pass_ctrl[kFinalSel] = sel;
}

template <int NW, typename K, int ITEMS>
__global__ void __launch_bounds__(NW * 32, sizeof(K) == 4 ? (ITEMS <= 8 ? 5 : 3) : 2) k_onesweep(SortArgs a, int64_t P, int pass,
                                                                            int n_parts) {
  constexpr int NT = NW * 32;
  constexpr int PART = NT * ITEMS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* s_keys = reinterpret_cast<K*>(smem_raw);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + PART);
  __shared__ uint32_t s_whist[NW][256];
  __shared__ uint32_t s_bstart[256];
  __shared__ uint32_t s_gstart[256];
  __shared__ int s_part;

  if (a.pass_ctrl[kCtrlActive + pass] == 0) return;
  const uint32_t sel = a.pass_ctrl[kCtrlSel + pass];
  const K* __restrict__ kin = reinterpret_cast<const K*>(sel ? a.keys[1] : a.keys[0]);
  const uint32_t* __restrict__ vin = sel ? a.vals[1] : a.vals[0];
  K* __restrict__ kout = reinterpret_cast<K*>(sel ? a.keys[0] : a.keys[1]);
  uint32_t* __restrict__ vout = sel ? a.vals[0] : a.vals[1];
  const int shift = 8 * pass;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

  if (tid == 0) s_part = int(atomicAdd(a.pass_ctrl + kCtrlPart + pass, 1u));
  for (int j = tid; j < NW * 256; j += NT) (&s_whist[0][0])[j] = 0;
  __syncthreads();
  const int part = s_part;
  const int64_t base = int64_t(part) * PART;
  const int64_t wbase = base + int64_t(w) * (32 * ITEMS);

  K key[ITEMS];
  uint32_t val[ITEMS];
  uint32_t rank[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    if (idx < P) {
      key[i] = kin[idx];
      val[i] = vin[idx];
    } else {
      key[i] = K(~K(0));
      val[i] = 0;
    }
  }
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    const bool valid = idx < P;
    const uint32_t d = valid ? uint32_t((key[i] >> shift) & 255u) : 256u + lane;  // invalid: unique
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    uint32_t prev = 0;
    if (valid) prev = s_whist[w][d];
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) s_whist[w][d] = prev + __popc(peers);
    __syncwarp();
    rank[i] = prev + __popc(peers & lt);
  }
  __syncthreads();
  // per digit: exclusive offsets across warps, block count
  const int d = tid;  // NT == 256
  uint32_t cnt = 0;
#pragma unroll
  for (int ww = 0; ww < NW; ++ww) {
    const uint32_t c = s_whist[ww][d];
    s_whist[ww][d] = cnt;
    cnt += c;
  }
  // decoupled look-back over partitions for digit d
  uint32_t* st = a.status + (size_t(pass) * n_parts) * 256;
  volatile uint32_t* my = st + size_t(part) * 256 + d;
  uint32_t excl = 0;
  if (part == 0) {
    *my = kFlagInc | cnt;
  } else {
    *my = kFlagAgg | cnt;
    // look back 4 predecessors per round trip: consume them nearest first until an inclusive
    // prefix; stop at a not-yet-published one and re-read from there (partition 0 is always
    // inclusive, so the walk never passes it)
    int j = part - 1;
    bool found = false;
    while (!found) {
      uint32_t sv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        sv[k] = j - k >= 0 ? uint32_t(*(volatile uint32_t*)(st + size_t(j - k) * 256 + d)) : uint32_t(2u << 30);
      int used = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t f = sv[k] & ~kValMask;
        if (f == 0) break;
        excl += sv[k] & kValMask;
        if (f == kFlagInc) {
          found = true;
          break;
        }
        used = k + 1;
      }
      j -= used;
    }
    *my = kFlagInc | (excl + cnt);
  }
  // block-local exclusive scan of cnt over digits (256 threads)
  __shared__ uint32_t s_w8[8];
  s_bstart[d] = block_excl_scan256(cnt, s_w8);
  s_gstart[d] = a.digit_hist[pass * 256 + d] + excl;
  __syncthreads();
  // local reorder in shared memory (stable: warp-major, then item, then lane == input order)
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    if (idx < P) {
      const uint32_t dd = uint32_t((key[i] >> shift) & 255u);
      const uint32_t pos = s_bstart[dd] + s_whist[w][dd] + rank[i];
      s_keys[pos] = key[i];
      s_vals[pos] = val[i];
    }
  }
  __syncthreads();
  const int nvalid = int(P - base < int64_t(PART) ? P - base : int64_t(PART));
  for (int j = tid; j < nvalid; j += NT) {
    const K k = s_keys[j];
    const uint32_t dd = uint32_t((k >> shift) & 255u);
    const uint32_t o = s_gstart[dd] + (uint32_t(j) - s_bstart[dd]);
    kout[o] = k;
    vout[o] = s_vals[j];
  }
}

__global__ void __launch_bounds__(256) k_ranges_fixup(SortArgs a, int64_t P) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const uint32_t sel = a.pass_ctrl[kFinalSel];
  const uint32_t* keys = reinterpret_cast<const uint32_t*>(sel ? a.keys[1] : a.keys[0]);
  const uint32_t* vin = sel ? a.vals[1] : a.vals[0];
  uint32_t* vout = sel ? a.vals[0] : a.vals[1];
  if (i == 0) a.pass_ctrl[kValsSel] = sel ^ 1u;
  const int kd = key_layout(a.counters[C_DLO], a.counters[C_DHI], a.tbits).kd;
  const uint32_t k = keys[i];
  const uint32_t t = uint32_t((unsigned long long)k >> kd);
  const bool eq_prev = i > 0 && keys[i - 1] == k;
  const bool eq_next = i + 1 < P && keys[i + 1] == k;
  if ((i == 0 || uint32_t((unsigned long long)keys[i - 1] >> kd) != t)) a.ranges[t].x = uint32_t(i);
  if ((i + 1 == P || uint32_t((unsigned long long)keys[i + 1] >> kd) != t)) a.ranges[t].y = uint32_t(i + 1);
  const uint32_t v = vin[i];
  if (!eq_prev && !eq_next) {
    vout[i] = v;
    return;
  }
  // member of a run of identical keys (same tile, same kept depth bits; short -- KeyLayout
  // drops only the lowest sd depth bits): its final slot is the run start plus its rank by
  // (full f32 depth bits, global id) (R12).  Every member ranks itself; no dependent chains.
  int64_t s = i, e = i;
  while (s > 0 && keys[s - 1] == k) --s;
  while (e + 1 < P && keys[e + 1] == k) ++e;
  const unsigned long long mine = ((unsigned long long)__float_as_uint(a.recv[v].depth) << 32) | a.recv[v].gid;
  int64_t rank = 0;
  for (int64_t j = s; j <= e; ++j) {
    if (j == i) continue;
    const Rec& rj = a.recv[vin[j]];
    const unsigned long long o = ((unsigned long long)__float_as_uint(rj.depth) << 32) | rj.gid;
    rank += (o < mine || (o == mine && j < i)) ? 1 : 0;
  }
  vout[s + rank] = v;
}

}  // namespace

void launch_emit(const SortArgs& a, cudaStream_t s) {
  if (a.n_recv <= 0) return;
  const int64_t chunks = (a.n_recv + 255) / 256;
  static std::atomic<int> slots[kMaxDevices];
  const int max_blocks = per_device(slots, [] {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_emit, 256, 0);
    return device_sm_count() * (occ < 4 ? (occ > 0 ? occ : 1) : 4);
  });
  const int64_t blocks = chunks < max_blocks ? chunks : max_blocks;
  k_emit<<<unsigned(blocks), 256, 0, s>>>(a);
}

void launch_depth_range(const Rec* recv, int64_t n, unsigned long long* counters, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t nb = (n + 255) / 256;
  const int64_t blocks = nb < 148 * 8 ? nb : 148 * 8;
  k_depth_range<<<unsigned(blocks), 256, 0, s>>>(recv, n, counters);
}

template <typename K, int ITEMS>
static void sort_passes(const SortArgs& a, int64_t P, cudaStream_t s, int64_t* launches) {
  constexpr int PART = kSortBlock * ITEMS;
  const int n_parts = int((P + PART - 1) / PART);
  const size_t smem = size_t(PART) * (sizeof(K) + sizeof(uint32_t));
  static std::atomic<int> attr[kMaxDevices];
  per_device(attr, [smem] {
    cudaFuncSetAttribute(k_onesweep<8, K, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    return 1;
  });
  for (int p = 0; p < a.n_passes; ++p) {
    k_onesweep<8, K, ITEMS><<<n_parts, 256, smem, s>>>(a, P, p, n_parts);
    ++*launches;
  }
}

void launch_sort_passes(const SortArgs& a, int64_t P, cudaStream_t s, int64_t* launches, int key_bytes) {
  k_digit_scan<<<1, 256, 0, s>>>(a);
  ++*launches;
  if (P <= 0) return;
  if (key_bytes == 4)
    sort_passes<uint32_t, kViewSortItems>(a, P, s, launches);
  else
    sort_passes<unsigned long long, kSortItems>(a, P, s, launches);
}

void launch_ranges_fixup(const SortArgs& a, int64_t P, cudaStream_t s) {
  if (P <= 0) return;
  k_ranges_fixup<<<unsigned((P + 255) / 256), 256, 0, s>>>(a, P);
}

namespace {
// Longest-list-first launch order for the raster kernels (LPT scheduling): a one-CTA counting
// sort of the owned tiles by list length into 256 descending buckets.  The heaviest tiles
// start in the first wave instead of extending the tail.
__global__ void __launch_bounds__(1024) k_tile_order(const uint2* ranges, int n, uint32_t* perm) {
  __shared__ uint32_t s_cnt[256];
  __shared__ uint32_t s_w[8];
  __shared__ uint32_t s_max;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 256) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_max = 1;
  __syncthreads();
  uint32_t mx = 0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) mx = max(mx, ranges[t].y - ranges[t].x);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) atomicMax(&s_max, mx);
  __syncthreads();
  const uint32_t width = (s_max + 255) / 256;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const uint32_t b = min(255u, (ranges[t].y - ranges[t].x) / width);
    atomicAdd(&s_cnt[255 - b], 1u);
  }
  __syncthreads();
  // exclusive scan of the 256 bucket counts by warps 0..7 (shuffles + 8 warp totals)
  uint32_t c = 0, inc = 0;
  if (warp < 8) {
    c = s_cnt[threadIdx.x];
    inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) s_w[warp] = inc;
  }
  __syncthreads();
  if (warp < 8) {
    uint32_t wb = 0;
    for (int k = 0; k < warp; ++k) wb += s_w[k];
    s_cnt[threadIdx.x] = wb + inc - c;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const uint32_t b = min(255u, (ranges[t].y - ranges[t].x) / width);
    perm[atomicAdd(&s_cnt[255 - b], 1u)] = uint32_t(t);
  }
}
}  // namespace

void launch_tile_order(const uint2* ranges, int n_tiles, uint32_t* perm, cudaStream_t s) {
  if (n_tiles > 0) k_tile_order<<<1, 1024, 0, s>>>(ranges, n_tiles, perm);
}

}  // namespace bgs
