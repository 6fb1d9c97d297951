// NEXT-1: the scoring report's phi, the two scheduled pruning passes and the
// index-parity redistribution of the survivors (bgs_score_phi, bgs_prune_stochastic,
// bgs_prune_mass_cut, bgs_redistribute).  PAPER.md P:185; SPEC S:291-317;
// readings R30-R33 in DESIGN.md.
//
// Selection ("keep the top of (key desc, global id asc)") is one exact distributed radix select
// used by both passes: 8 rounds of 8-bit digits over a u64 key with per-round (count, mass)
// histograms summed over ranks, then (when the threshold key is shared by more items than are
// needed) 4 count-only rounds over the global ids of the ties.  Pass 1 counts items (keep k);
// pass 2 accumulates mass (smallest prefix reaching num/den of the total).  Every decision is an
// integer comparison, so the kept set is bit-identical to the oracle's and independent of M.
//
// Pass-1 keys: u = splitmix64-based uniform of (seed, global id), key = ln(u)/s with a pinned
// fp64 ln (exact exponent split + fixed atanh series, one IEEE op per step, no contraction),
// mapped to an order-preserving u64.  Pass-2 keys: q = floor(s 2^24).
#include "bgs_internal.cuh"

namespace bgs {

namespace {

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double uniform_open(unsigned long long seed, unsigned long long gid) {
  const unsigned long long x = mix64(seed ^ mix64(gid));
  return __dmul_rn(__dadd_rn(double(x >> 11), 0.5), 1.1102230246251565e-16);  // 2^-53
}

// order-preserving map of a double onto u64 (larger double -> larger u64)
__device__ __forceinline__ unsigned long long ord64(double x) {
  const unsigned long long b = __double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_phi(int64_t n, const uint32_t* __restrict__ c_rad, const uint32_t* __restrict__ c_vis,
                      double* __restrict__ phi) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) phi[i] = __ddiv_rn(double(c_vis[i]), __dadd_rn(double(c_rad[i]), 1e-8));
}

__global__ void k_keys_race(int64_t n, const double* __restrict__ s, unsigned long long seed, int rank, int world,
                            unsigned long long* __restrict__ key) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double si = s[i];
  const unsigned long long gid = (unsigned long long)i * unsigned(world) + unsigned(rank);
  const double k = si > 0.0 ? __ddiv_rn(ln_pinned(uniform_open(seed, gid)), si) : -__longlong_as_double(0x7ff0000000000000ll);
  key[i] = ord64(k);
}

__global__ void k_keys_mass(int64_t n, const double* __restrict__ s, unsigned long long* __restrict__ key) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double si = s[i];
  key[i] = si > 0.0 ? (unsigned long long)floor(__dmul_rn(si, 16777216.0)) : 0ull;
}

// ---- the distributed top selection ------------------------------------------------------------

struct alignas(16) SelState {
  unsigned long long total;   // mass (or count) over all ranks
  unsigned long long above;   // mass (or count) strictly above the selected prefix
  unsigned long long prefix;  // selected high digits of the threshold key
  unsigned long long tau;
  unsigned long long kt;      // ties to keep
  unsigned long long ntie;
  unsigned long long below;   // ties with gid below the selected gid prefix
  uint32_t gprefix, gid_thr, need_gid, pad;
};

constexpr int kSelRounds = 8;
constexpr int kSelGRounds = 4;

__global__ void k_sel_total(int64_t n, const unsigned long long* __restrict__ key, int mass,
                            unsigned long long* __restrict__ total) {
  unsigned long long v = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    v += mass ? key[i] : 1ull;
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(total, v);
}

__global__ void __launch_bounds__(256) k_sel_hist(int64_t n, const unsigned long long* __restrict__ key,
                                                  const SelState* st, int round,
                                                  unsigned long long* __restrict__ hist /*[256] cnt, [256] mass*/) {
  __shared__ unsigned long long s_cnt[256], s_mass[256];
  s_cnt[threadIdx.x] = 0;
  s_mass[threadIdx.x] = 0;
  __syncthreads();
  const int shift = 8 * (kSelRounds - 1 - round);
  const unsigned long long prefix = st->prefix;
  const int lane = threadIdx.x & 31;
  // warp-uniform trip count; lanes sharing a digit are reduced in-warp first (early rounds put
  // almost every item in one bin, which serialised per-lane shared atomics)
  for (int64_t b = int64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31); b < n; b += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = b + lane;
    const unsigned long long k = i < n ? key[i] : 0ull;
    const bool cand = i < n && !(shift + 8 < 64 && (k >> (shift + 8)) != prefix);
    const uint32_t d = cand ? uint32_t((k >> shift) & 255u) : 256u + lane;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t lo = uint32_t(k & 0xffffffu), mid = uint32_t((k >> 24) & 0xffffffu), hi = uint32_t(k >> 48);
    const uint32_t slo = __reduce_add_sync(peers, lo), smid = __reduce_add_sync(peers, mid),
                   shi = __reduce_add_sync(peers, hi);
    if (cand && lane == __ffs(peers) - 1) {
      atomicAdd(&s_cnt[d], (unsigned long long)__popc(peers));
      atomicAdd(&s_mass[d], (unsigned long long)slo + ((unsigned long long)smid << 24) + ((unsigned long long)shi << 48));
    }
  }
  __syncthreads();
  if (s_cnt[threadIdx.x]) {
    atomicAdd(hist + threadIdx.x, s_cnt[threadIdx.x]);
    atomicAdd(hist + 256 + threadIdx.x, s_mass[threadIdx.x]);
  }
}

// one CTA of 256: pick the digit where the cumulative (from the top) weight crosses the target.
// mass: den (above + incl) >= num total; count: above + incl >= k.
__global__ void __launch_bounds__(256) k_sel_decide(SelState* st, int round, const unsigned long long* hist,
                                                    int mass, long long num, long long den, unsigned long long k) {
  __shared__ unsigned long long s_suf[256];
  __shared__ int s_pick;
  const int d = threadIdx.x;
  if (round == 0 && d == 0) {
    st->above = 0;
    st->prefix = 0;
  }
  __syncthreads();
  // inclusive suffix sums of the weight over digits >= 255 - j (Hillis-Steele; once per round)
  s_suf[255 - d] = mass ? hist[256 + d] : hist[d];
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const unsigned long long v = d >= o ? s_suf[d - o] : 0ull;
    __syncthreads();
    s_suf[d] += v;
    __syncthreads();
  }
  if (d == 0) s_pick = -1;
  __syncthreads();
  const unsigned long long above = st->above;
  const unsigned long long incl = s_suf[255 - d], excl = d < 255 ? s_suf[254 - d] : 0ull;
  bool cross;
  if (mass) {
    const unsigned __int128 tgt = (unsigned __int128)num * st->total;
    cross = (unsigned __int128)den * (above + incl) >= tgt && (unsigned __int128)den * (above + excl) < tgt;
  } else {
    cross = above + incl >= k && above + excl < k;
  }
  if (cross && hist[d] > 0) s_pick = d;
  __syncthreads();
  if (d == 0 && s_pick >= 0) {
    const int pick = s_pick;
    st->above = above + (pick < 255 ? s_suf[254 - pick] : 0ull);
    st->prefix = (st->prefix << 8) | unsigned(pick);
    if (round == kSelRounds - 1) {
      const unsigned long long tau = st->prefix, ntie = hist[pick];
      unsigned long long kt;
      if (mass) {
        const unsigned __int128 need = (unsigned __int128)num * st->total - (unsigned __int128)den * st->above;
        const unsigned __int128 per = (unsigned __int128)den * tau;  // > 0: a zero-mass bin never crosses
        kt = (unsigned long long)((need + per - 1) / per);
      } else {
        kt = k - st->above;
      }
      st->tau = tau;
      st->ntie = ntie;
      st->kt = kt < ntie ? kt : ntie;
      st->need_gid = st->kt < ntie ? 1u : 0u;
      st->gprefix = 0;
      st->below = 0;
      st->gid_thr = 0xffffffffu;
    }
  }
}

__global__ void __launch_bounds__(256) k_sel_gid_hist(int64_t n, const unsigned long long* __restrict__ key,
                                                      const SelState* st, int round, int rank, int world,
                                                      unsigned long long* __restrict__ hist) {
  __shared__ unsigned long long s_cnt[256];
  s_cnt[threadIdx.x] = 0;
  __syncthreads();
  if (st->need_gid) {
    const int shift = 8 * (kSelGRounds - 1 - round);
    const unsigned long long tau = st->tau;
    const uint32_t gp = st->gprefix;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
      if (key[i] != tau) continue;
      const uint32_t g = uint32_t(i) * uint32_t(world) + uint32_t(rank);
      if (shift + 8 < 32 && (g >> (shift + 8)) != gp) continue;
      atomicAdd(&s_cnt[(g >> shift) & 255u], 1ull);
    }
  }
  __syncthreads();
  if (s_cnt[threadIdx.x]) atomicAdd(hist + threadIdx.x, s_cnt[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_sel_gid_decide(SelState* st, int round, const unsigned long long* hist) {
  __shared__ unsigned long long s_pre[256];
  __shared__ int s_pick;
  if (!st->need_gid) return;
  const int d = threadIdx.x;
  s_pre[d] = hist[d];
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const unsigned long long v = d >= o ? s_pre[d - o] : 0ull;
    __syncthreads();
    s_pre[d] += v;
    __syncthreads();
  }
  if (d == 0) s_pick = -1;
  __syncthreads();
  const unsigned long long below = st->below, kt = st->kt;
  const unsigned long long incl = s_pre[d], excl = d > 0 ? s_pre[d - 1] : 0ull;
  if (below + incl >= kt && below + excl < kt) s_pick = d;
  __syncthreads();
  if (d == 0 && s_pick >= 0) {
    st->below = below + (s_pick > 0 ? s_pre[s_pick - 1] : 0ull);
    st->gprefix = (st->gprefix << 8) | uint32_t(s_pick);
    if (round == kSelGRounds - 1) st->gid_thr = st->gprefix;
  }
}

__global__ void k_sel_mark(int64_t n, const unsigned long long* __restrict__ key, const SelState* st, int rank,
                           int world, uint8_t* __restrict__ keep) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = key[i], tau = st->tau;
  bool sel = k > tau;
  if (k == tau) sel = !st->need_gid || uint32_t(i) * uint32_t(world) + uint32_t(rank) <= st->gid_thr;
  keep[i] = sel ? 1 : 0;
}

__global__ void k_keep_positive(int64_t n, const double* __restrict__ s, uint8_t* __restrict__ keep,
                                unsigned long long* __restrict__ count) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool k = i < n && s[i] > 0.0;
  if (i < n) keep[i] = k ? 1 : 0;
  const unsigned m = __ballot_sync(0xffffffffu, k);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(count, (unsigned long long)__popc(m));
}

__global__ void k_fill_u8(int64_t n, uint8_t* p, uint8_t v) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

unsigned blocks_for(int64_t n) { return unsigned((n + 255) / 256); }

}  // namespace

void launch_phi(int64_t n, const uint32_t* c_rad, const uint32_t* c_vis, double* phi, cudaStream_t s) {
  if (n > 0) k_phi<<<blocks_for(n), 256, 0, s>>>(n, c_rad, c_vis, phi);
}

void launch_keys_race(int64_t n, const double* sc, unsigned long long seed, int rank, int world,
                      unsigned long long* key, cudaStream_t s) {
  if (n > 0) k_keys_race<<<blocks_for(n), 256, 0, s>>>(n, sc, seed, rank, world, key);
}

void launch_keys_mass(int64_t n, const double* sc, unsigned long long* key, cudaStream_t s) {
  if (n > 0) k_keys_mass<<<blocks_for(n), 256, 0, s>>>(n, sc, key);
}

size_t sel_state_bytes() { return sizeof(SelState); }
int sel_rounds() { return kSelRounds; }
int sel_gid_rounds() { return kSelGRounds; }

void launch_sel_total(int64_t n, const unsigned long long* key, int mass, unsigned long long* total, cudaStream_t s) {
  if (n > 0) k_sel_total<<<blocks_for(n) < 1184u ? blocks_for(n) : 1184u, 256, 0, s>>>(n, key, mass, total);
}

void launch_sel_hist(int64_t n, const unsigned long long* key, const void* st, int round, unsigned long long* hist,
                     cudaStream_t s) {
  if (n > 0)
    k_sel_hist<<<blocks_for(n) < 1184u ? blocks_for(n) : 1184u, 256, 0, s>>>(n, key, static_cast<const SelState*>(st),
                                                                          round, hist);
}

void launch_sel_decide(void* st, const unsigned long long* total, int round, const unsigned long long* hist, int mass,
                       long long num, long long den, unsigned long long k, cudaStream_t s) {
  if (round == 0)
    cudaMemcpyAsync(&static_cast<SelState*>(st)->total, total, 8, cudaMemcpyDeviceToDevice, s);
  k_sel_decide<<<1, 256, 0, s>>>(static_cast<SelState*>(st), round, hist, mass, num, den, k);
}

void launch_sel_gid_hist(int64_t n, const unsigned long long* key, const void* st, int round, int rank, int world,
                         unsigned long long* hist, cudaStream_t s) {
  if (n > 0)
    k_sel_gid_hist<<<blocks_for(n) < 1184u ? blocks_for(n) : 1184u, 256, 0, s>>>(
        n, key, static_cast<const SelState*>(st), round, rank, world, hist);
}

void launch_sel_gid_decide(void* st, int round, const unsigned long long* hist, cudaStream_t s) {
  k_sel_gid_decide<<<1, 256, 0, s>>>(static_cast<SelState*>(st), round, hist);
}

void launch_sel_mark(int64_t n, const unsigned long long* key, const void* st, int rank, int world, uint8_t* keep,
                     cudaStream_t s) {
  if (n > 0) k_sel_mark<<<blocks_for(n), 256, 0, s>>>(n, key, static_cast<const SelState*>(st), rank, world, keep);
}

void launch_keep_positive(int64_t n, const double* sc, uint8_t* keep, unsigned long long* count, cudaStream_t s) {
  if (n > 0) k_keep_positive<<<blocks_for(n), 256, 0, s>>>(n, sc, keep, count);
}

void launch_fill_u8(int64_t n, uint8_t* p, uint8_t v, cudaStream_t s) {
  if (n > 0) k_fill_u8<<<blocks_for(n), 256, 0, s>>>(n, p, v);
}

// ---- index-parity redistribution (R33) --------------------------------------------------------

namespace {

// 256-B parameter row moved between shards: mean_opac, quat, scale, sh[48], lod, new local index
struct __align__(16) ParamRow {
  float4 mo, q, sc;
  float sh[48];
  uint32_t lod;
  uint32_t new_local;
  uint32_t pad[2];
};
static_assert(sizeof(ParamRow) == 256, "row is 256 B");

__global__ void k_pack_bits(int64_t n, const uint8_t* __restrict__ keep, uint32_t* __restrict__ bits) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const unsigned m = __ballot_sync(0xffffffffu, i < n && keep[i]);
  if ((threadIdx.x & 31) == 0 && i < n) bits[i >> 5] = m;
}

// keep bit of global id g from the gathered per-rank masks (rank s holds gids s, s+M, ...)
__device__ __forceinline__ bool gkeep(const uint32_t* masks, int64_t words_per_rank, int world, int64_t g) {
  const int64_t s = g % world, l = g / world;
  return (masks[s * words_per_rank + (l >> 5)] >> (l & 31)) & 1u;
}

__global__ void k_gid_block_counts(int64_t N, const uint32_t* __restrict__ masks, int64_t wpr, int world,
                                   uint32_t* __restrict__ bc) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool k = g < N && gkeep(masks, wpr, world, g);
  const uint32_t c = __syncthreads_count(k);
  if (threadIdx.x == 0) bc[blockIdx.x] = c;
}

// exclusive scan of the block counts in place; total in *out_total (one CTA)
__global__ void __launch_bounds__(1024) k_scan_blocks(uint32_t* bc, int64_t nb, unsigned long long* out_total) {
  __shared__ unsigned long long s_run;
  __shared__ unsigned long long s_w[32];
  if (threadIdx.x == 0) s_run = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const unsigned long long v = i < nb ? bc[i] : 0u;
    unsigned long long inc = v;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    unsigned long long wb = 0;
    for (int k = 0; k < w; ++k) wb += s_w[k];
    const unsigned long long run = s_run;
    if (i < nb) bc[i] = uint32_t(run + wb + inc - v);
    __syncthreads();
    if (threadIdx.x == 1023) s_run = run + wb + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) *out_total = s_run;
}

// new gid of every kept item of THIS rank -> destination rank and new local index
__global__ void k_new_ids(int64_t N, const uint32_t* __restrict__ masks, int64_t wpr, int world, int rank,
                          const uint32_t* __restrict__ bc, int64_t n_local, uint32_t* __restrict__ new_gid) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool k = g < N && gkeep(masks, wpr, world, g);
  // rank of g among the kept inside its block: prefix count over the block (warp ballots)
  __shared__ uint32_t s_w[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, k);
  if (lane == 0) s_w[w] = __popc(m);
  __syncthreads();
  uint32_t off = 0;
  for (int j = 0; j < w; ++j) off += s_w[j];
  if (g < N && g % world == rank) {
    const int64_t l = g / world;
    if (l < n_local) new_gid[l] = k ? bc[blockIdx.x] + off + __popc(m & ((1u << lane) - 1u)) : 0xffffffffu;
  }
}

__global__ void k_dest_hist(int64_t n, const uint32_t* __restrict__ new_gid, int world, unsigned long long* cnt) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && new_gid[i] != 0xffffffffu) atomicAdd(cnt + (new_gid[i] % uint32_t(world)), 1ull);
}

// rows grouped by destination rank (slot inside a group from a warp-aggregated cursor; the row
// carries its new local index, so the receiver does not depend on the packing order)
__global__ void k_pack_rows(int64_t n, const uint32_t* __restrict__ new_gid, int world,
                            const int64_t* __restrict__ dest_base, unsigned long long* __restrict__ cursor,
                            const float4* __restrict__ mo, const float4* __restrict__ q, const float4* __restrict__ sc,
                            const float* __restrict__ sh, const uint8_t* __restrict__ lod, ParamRow* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t ng = i < n ? new_gid[i] : 0xffffffffu;
  const bool kept = ng != 0xffffffffu;
  const uint32_t d = kept ? ng % uint32_t(world) : 0x80000000u | (threadIdx.x & 31);
  const unsigned peers = __match_any_sync(0xffffffffu, d);
  const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
  unsigned long long base = 0;
  if (kept && lane == leader) base = atomicAdd(cursor + d, (unsigned long long)__popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (!kept) return;
  ParamRow r;
  r.mo = mo[i];
  r.q = q[i];
  r.sc = sc[i];
#pragma unroll
  for (int k = 0; k < 48; ++k) r.sh[k] = sh[size_t(48) * i + k];
  r.lod = lod ? lod[i] : 0u;
  r.new_local = ng / uint32_t(world);
  r.pad[0] = r.pad[1] = 0;
  out[dest_base[d] + base + __popc(peers & ((1u << lane) - 1u))] = r;
}

// world 1: survivors written straight to their new index
__global__ void k_scatter_direct(int64_t n, const uint32_t* __restrict__ new_gid, const float4* __restrict__ mo,
                                 const float4* __restrict__ q, const float4* __restrict__ sc,
                                 const float* __restrict__ sh, const uint8_t* __restrict__ lod, float4* __restrict__ omo,
                                 float4* __restrict__ oq, float4* __restrict__ osc, float* __restrict__ osh,
                                 uint8_t* __restrict__ olod, int64_t cap) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t ng = new_gid[i];
  if (ng == 0xffffffffu || int64_t(ng) >= cap) return;
  omo[ng] = mo[i];
  oq[ng] = q[i];
  osc[ng] = sc[i];
  const float4* src = reinterpret_cast<const float4*>(sh + size_t(48) * i);
  float4* dst = reinterpret_cast<float4*>(osh + size_t(48) * ng);
#pragma unroll
  for (int k = 0; k < 12; ++k) dst[k] = src[k];
  if (olod) olod[ng] = lod ? lod[i] : 0;
}

__global__ void k_unpack_rows(int64_t n, const ParamRow* __restrict__ in, float4* __restrict__ mo,
                              float4* __restrict__ q, float4* __restrict__ sc, float* __restrict__ sh,
                              uint8_t* __restrict__ lod, int64_t cap) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const ParamRow& r = in[i];
  const int64_t l = r.new_local;
  if (l >= cap) return;
  mo[l] = r.mo;
  q[l] = r.q;
  sc[l] = r.sc;
#pragma unroll
  for (int k = 0; k < 48; ++k) sh[size_t(48) * l + k] = r.sh[k];
  if (lod) lod[l] = uint8_t(r.lod);
}

}  // namespace

size_t param_row_bytes() { return sizeof(ParamRow); }

void launch_pack_bits(int64_t n, const uint8_t* keep, uint32_t* bits, cudaStream_t s) {
  if (n > 0) k_pack_bits<<<blocks_for(n), 256, 0, s>>>(n, keep, bits);
}

void launch_new_ids(int64_t N, const uint32_t* masks, int64_t wpr, int world, int rank, uint32_t* bc,
                    unsigned long long* total, int64_t n_local, uint32_t* new_gid, cudaStream_t s) {
  if (N <= 0) return;
  const int64_t nb = (N + 255) / 256;
  k_gid_block_counts<<<unsigned(nb), 256, 0, s>>>(N, masks, wpr, world, bc);
  k_scan_blocks<<<1, 1024, 0, s>>>(bc, nb, total);
  k_new_ids<<<unsigned(nb), 256, 0, s>>>(N, masks, wpr, world, rank, bc, n_local, new_gid);
}

void launch_dest_hist(int64_t n, const uint32_t* new_gid, int world, unsigned long long* cnt, cudaStream_t s) {
  if (n > 0) k_dest_hist<<<blocks_for(n), 256, 0, s>>>(n, new_gid, world, cnt);
}

void launch_pack_rows(int64_t n, const uint32_t* new_gid, int world, const int64_t* dest_base,
                      unsigned long long* cursor, const bgs_gaussians& g, void* out, cudaStream_t s) {
  if (n > 0)
    k_pack_rows<<<blocks_for(n), 256, 0, s>>>(n, new_gid, world, dest_base, cursor,
                                              reinterpret_cast<const float4*>(g.mean_opac),
                                              reinterpret_cast<const float4*>(g.quat),
                                              reinterpret_cast<const float4*>(g.scale), g.sh, g.lod,
                                              static_cast<ParamRow*>(out));
}

void launch_scatter_direct(int64_t n, const uint32_t* new_gid, const bgs_gaussians& g, const bgs_gaussians_out& o,
                           int64_t cap, cudaStream_t s) {
  if (n > 0)
    k_scatter_direct<<<blocks_for(n), 256, 0, s>>>(
        n, new_gid, reinterpret_cast<const float4*>(g.mean_opac), reinterpret_cast<const float4*>(g.quat),
        reinterpret_cast<const float4*>(g.scale), g.sh, g.lod, reinterpret_cast<float4*>(o.mean_opac),
        reinterpret_cast<float4*>(o.quat), reinterpret_cast<float4*>(o.scale), o.sh, o.lod, cap);
}

void launch_unpack_rows(int64_t n, const void* in, const bgs_gaussians_out& o, int64_t cap, cudaStream_t s) {
  if (n > 0)
    k_unpack_rows<<<blocks_for(n), 256, 0, s>>>(n, static_cast<const ParamRow*>(in),
                                                reinterpret_cast<float4*>(o.mean_opac),
                                                reinterpret_cast<float4*>(o.quat), reinterpret_cast<float4*>(o.scale),
                                                o.sh, o.lod, cap);
}

}  // namespace bgs
