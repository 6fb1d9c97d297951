// a12 importance bookkeeping for one view (bgs_importance).
//
// Eq.3: s_i = sum_{v: a_{i,v} > 0} w_{i,v} / (a_{i,v} + eps), eps = 1e-8 (R17);
// c^rad_{i,v} = [radius > 0], c^vis_{i,v} = [w_{i,v} in the per-view top-99% mass] and
// Cull_{i,v} = 1 - c^vis_{i,v}.  The top set is the smallest prefix of the
// view's Gaussians ordered by (w desc, global id asc) whose mass reaches 99% of the total
// (R16), over ALL ranks (the view is global).
//
// Selection = exact distributed radix select on the u64 fixed-point w (D5): 7 rounds of
// 8-bit digits from bit 55 down; per round every rank builds a 256-bin (count, mass)
// histogram of the candidates that still match the selected high digits, the histograms are
// summed over ranks (all-reduce), and the digit where the cumulative mass from the top
// crosses the target is picked.  After the last round the threshold value tau is exact; the
// number k of ties (w == tau) to include is closed form, and when 0 < k < #ties a count-only
// radix select over global ids (4 rounds) finds the k smallest ids.  Every decision is
// integer, so the result is bit-exact and independent of M.
//
// world > 1: one kernel per histogram / decision (the all-reduce sits between them, stream
// ordered, no host round trip).  world == 1: ONE cooperative kernel runs every round with
// grid-wide barriers; each CTA recomputes the (identical) decision from the global histogram
// so a round costs one grid barrier.  Histograms are warp-aggregated (__match_any_sync +
// __reduce_add_sync on three 24-bit limbs of w) before the shared-memory atomics.
#include <cooperative_groups.h>
#include <cstdlib>

#include "bgs_internal.cuh"

namespace cg = cooperative_groups;

namespace bgs {

struct alignas(16) ImpState {
  unsigned long long total;      // sum of w over all ranks
  unsigned long long above;      // mass strictly above the selected prefix
  unsigned long long prefix;     // selected high digits of tau
  unsigned long long tau;        // threshold value (valid after the w rounds)
  unsigned long long k;          // ties to include
  unsigned long long below;      // ties with gid below the selected gid prefix
  unsigned long long ntie;       // number of ties (w == tau)
  uint32_t gprefix;              // selected high digits of the gid threshold
  uint32_t gid_thr;              // include ties with gid <= gid_thr
  uint32_t need_gid;             // 0 < k < ntie
  uint32_t empty;                // total == 0
  uint32_t r0;                   // first w round with a non-zero digit (from the MSB histogram)
  unsigned long long next_cnt;   // items in the crossing bin of the last round (next round's candidates)
  uint32_t tshift;               // selection: (w >> tshift) >= prefix (0 after all rounds)
  uint32_t final_;               // threshold resolved (crossing bin holds one item): no more rounds
  uint32_t bstar;                // world > 1 coarse path: the crossing coarse bin
  unsigned long long ncand;      // world > 1 coarse path: items (all ranks) in the crossing bin
};
static_assert(sizeof(ImpState) <= kImpStateBytes, "ImpState fits its arena slot");

namespace {

constexpr int kWRounds = 7;   // bits [0, 56)
constexpr int kGRounds = 4;   // gid bits [0, 32)

struct Item {
  unsigned long long w;
  uint32_t a;
  uint32_t lidx;
  bool rad;
};

__device__ __forceinline__ Item load_item(const ImportanceArgs& a, int64_t t) {
  Item it;
  if (a.item_lidx) {
    const Acc& ac = a.acc[t];
    it.w = ac.w;
    it.a = ac.a;
    it.lidx = a.item_lidx[t];
    it.rad = true;  // every record had radius > 0
  } else {
    it.w = a.w_dense[t];
    it.a = a.a_dense[t];
    it.lidx = uint32_t(t);
    it.rad = a.radius[t] > 0;
  }
  return it;
}

__device__ __forceinline__ unsigned long long load_w(const ImportanceArgs& a, int64_t t) {
  return a.wbuf ? a.wbuf[t] : (a.item_lidx ? a.acc[t].w : a.w_dense[t]);
}

__device__ __forceinline__ uint32_t gid_of(const ImportanceArgs& a, uint32_t lidx) {
  return lidx * uint32_t(a.world) + uint32_t(a.rank);
}

// Inclusive scan of one u64 per thread over a 256-thread CTA (shuffles + 8 warp totals).
__device__ __forceinline__ unsigned long long block_incl_scan256(unsigned long long v) {
  __shared__ unsigned long long s_w[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) s_w[w] = v;
  __syncthreads();
  unsigned long long wb = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) wb += k < w ? s_w[k] : 0ull;
  __syncthreads();
  return wb + v;
}

// ---- bodies shared by the per-round kernels and the cooperative kernel -----------------

// s, c_rad, the (rank-local) total mass total[0] and the histogram of the most significant
// bit of w in total[1..64] (so the rounds above the global maximum can be skipped); one
// atomic per CTA for the total
__device__ void stats_body(const ImportanceArgs& a, unsigned long long* total) {
  __shared__ unsigned long long s_w[8];
  __shared__ uint32_t s_msb[64];
  if (threadIdx.x < 64) s_msb[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long wsum = 0;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < a.n_items;
       t += int64_t(gridDim.x) * blockDim.x) {
    const Item it = load_item(a, t);
    wsum += it.w;
    if (a.wbuf) a.wbuf[t] = it.w;  // dense copy for the radix rounds (8 B instead of a 48-B row)
    if (it.w) atomicAdd(&s_msb[63 - __clzll((long long)it.w)], 1u);
    // reductions, not read-modify-writes: several views may be in flight on one shard (their
    // contexts share the caller's s / c_rad / c_vis)
    if (it.a > 0) atomicAdd(a.s + it.lidx, (double(it.w) * (1.0 / 16777216.0)) / (double(it.a) + 1e-8));
    if (it.rad) atomicAdd(a.c_rad + it.lidx, 1u);
  }
  __syncthreads();
  if (threadIdx.x < 64 && s_msb[threadIdx.x]) atomicAdd(total + 1 + threadIdx.x, (unsigned long long)s_msb[threadIdx.x]);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long sum = 0;
    for (int i = 0; i < 8; ++i) sum += s_w[i];
    if (sum) atomicAdd(total, sum);
  }
  __syncthreads();
}

// Per-warp candidate segments (world-1 cooperative kernel): warp gw (global warp id) owns
// cand[gw * cap, gw * cap + cnt[gw]), filled by one full scan and rescanned by later rounds, so
// no atomics and no cross-warp order are involved.
struct Seg {
  uint32_t* cand;
  uint32_t* cnt;
  int64_t cap;
};

// one warp's candidates into the CTA histogram (warp-aggregated shared-memory atomics: the early
// rounds put almost every candidate in one bin, which serialised per-lane 64-bit atomics)
__device__ __forceinline__ void hist_add(bool cand, uint32_t d, unsigned long long w, int lane,
                                         unsigned long long* s_cnt, unsigned long long* s_mass) {
  const unsigned peers = __match_any_sync(0xffffffffu, d);
  const bool single = peers == (1u << lane);
  if (cand && single) {
    atomicAdd(&s_cnt[d], 1ull);
    atomicAdd(&s_mass[d], w);
  }
  // groups of lanes sharing a digit: reduce in-warp first (redux.sync runs once per group)
  const bool multi = cand && !single;
  if (__any_sync(0xffffffffu, multi) && multi) {
    const uint32_t lo = uint32_t(w & 0xffffffu), mid = uint32_t((w >> 24) & 0xffffffu), hi = uint32_t(w >> 48);
    const uint32_t slo = __reduce_add_sync(peers, lo);
    const uint32_t smid = __reduce_add_sync(peers, mid);
    const uint32_t shi = __reduce_add_sync(peers, hi);
    if (lane == __ffs(peers) - 1) {
      atomicAdd(&s_cnt[d], (unsigned long long)__popc(peers));
      atomicAdd(&s_mass[d], (unsigned long long)slo + ((unsigned long long)smid << 24) + ((unsigned long long)shi << 48));
    }
  }
}

// candidates of round r: w > 0 and w >> (shift + 8) == prefix.  seg_mode 0: scan every item;
// 1: scan every item and append the candidates to this warp's segment; 2: scan the segment only
// (a superset of this round's candidates: they matched every earlier prefix).
__device__ void hist_body(const ImportanceArgs& a, unsigned long long prefix, int round,
                          unsigned long long* hist /*[256] count, [256] mass*/, int seg_mode = 0, Seg seg = {}) {
  __shared__ unsigned long long s_cnt[256], s_mass[256];
  s_cnt[threadIdx.x] = 0;
  s_mass[threadIdx.x] = 0;
  __syncthreads();
  const int64_t n = a.n_items;
  const int shift = 8 * (kWRounds - 1 - round);
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  auto is_cand = [&](unsigned long long w) { return w != 0 && !(shift + 8 < 64 && (w >> (shift + 8)) != prefix); };
  if (seg_mode == 2) {
    const uint32_t cnt = seg.cnt[gw];
    const uint32_t* L = seg.cand + gw * seg.cap;
    for (uint32_t b = 0; b < cnt; b += 32) {
      const uint32_t j = b + lane;
      const unsigned long long w = j < cnt ? load_w(a, L[j]) : 0ull;
      const bool cand = j < cnt && is_cand(w);
      hist_add(cand, cand ? uint32_t((w >> shift) & 255u) : 256u + lane, w, lane, s_cnt, s_mass);
    }
  } else {
    uint32_t appended = 0;
    uint32_t* L = seg_mode == 1 ? seg.cand + gw * seg.cap : nullptr;
    // warp-uniform trip count so every lane reaches the warp collectives
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31); base < n; base += stride) {
      const int64_t t = base + lane;
      const unsigned long long w = t < n ? load_w(a, t) : 0ull;
      const bool cand = t < n && is_cand(w);
      if (seg_mode == 1) {
        const unsigned cm = __ballot_sync(0xffffffffu, cand);
        if (cand) L[appended + __popc(cm & ((1u << lane) - 1u))] = uint32_t(t);
        appended += __popc(cm);
      }
      hist_add(cand, cand ? uint32_t((w >> shift) & 255u) : 256u + lane, w, lane, s_cnt, s_mass);
    }
    if (seg_mode == 1 && lane == 0) seg.cnt[gw] = appended;
  }
  __syncthreads();
  if (s_cnt[threadIdx.x]) {
    atomicAdd(hist + threadIdx.x, s_cnt[threadIdx.x]);
    atomicAdd(hist + 256 + threadIdx.x, s_mass[threadIdx.x]);
  }
  __syncthreads();
}

// thread 0: state before the first round (total and MSB histogram already summed over ranks)
__device__ void init_state(ImpState* st, const unsigned long long* total) {
  st->total = total[0];
  st->empty = total[0] == 0;
  st->above = 0;
  st->prefix = 0;
  st->need_gid = 0;
  st->tau = 0;
  st->tshift = 0;
  st->final_ = 0;
  int maxbit = 0;
  for (int b = 63; b >= 0; --b)
    if (total[1 + b]) {
      maxbit = b;
      break;
    }
  // rounds whose 8-bit digit lies above the maximum are all-zero digits: skipped
  const int r0 = (kWRounds - 1) - maxbit / 8;
  st->r0 = uint32_t(r0 < 0 ? 0 : r0);
}

// whole CTA: pick the digit where the cumulative mass (from the top) crosses num/den of total.
// `st` may be global (one-CTA kernel) or shared (cooperative kernel); thread 0 writes it.
__device__ void decide_body(ImpState* st, int round, const unsigned long long* hist, int num, int den) {
  __shared__ unsigned long long s_suf[256];
  __shared__ int s_pick;
  const int d = threadIdx.x;
  if (st->empty || st->final_ || round < int(st->r0)) return;
  const unsigned long long target = (unsigned long long)num * st->total;  // need den*prefix >= target
  // s_suf[j] = mass of digits >= 255 - j; the crossing digit is the largest d with
  // den*(above + mass(>= d)) >= target
  s_suf[d] = block_incl_scan256(hist[256 + 255 - d]);
  if (d == 0) s_pick = -1;
  __syncthreads();
  const unsigned long long above = st->above;
  const unsigned long long incl = s_suf[255 - d];
  const unsigned long long excl = d < 255 ? s_suf[254 - d] : 0ull;
  const bool cross = (unsigned long long)den * (above + incl) >= target &&
                     (unsigned long long)den * (above + excl) < target;
  if (cross && hist[d] > 0) s_pick = d;
  __syncthreads();
  if (d == 0) {
    const int pick = s_pick;
    if (pick >= 0) {
      st->above = above + (pick < 255 ? s_suf[254 - pick] : 0ull);
      st->prefix = (st->prefix << 8) | unsigned(pick);
      st->tshift = uint32_t(8 * (kWRounds - 1 - round));
      st->next_cnt = hist[pick];
      if (round < kWRounds - 1 && hist[pick] == 1) {
        // the crossing bin holds one item: it is the threshold item (k = ntie = 1) and the
        // selection is exactly {w : (w >> tshift) >= prefix}; the remaining rounds are skipped
        st->final_ = 1u;
        st->k = 1;
        st->ntie = 1;
        st->need_gid = 0;
        st->gid_thr = 0xffffffffu;
      }
      if (round == kWRounds - 1) {
        const unsigned long long tau = st->prefix;
        st->tau = tau;
        const unsigned long long ntie = hist[pick];
        const unsigned long long need = target - (unsigned long long)den * st->above;  // > 0
        const unsigned long long k = (need + (unsigned long long)den * tau - 1) / ((unsigned long long)den * tau);
        st->k = k < ntie ? k : ntie;
        st->ntie = ntie;
        st->need_gid = (st->k < ntie) ? 1u : 0u;
        st->gprefix = 0;
        st->below = 0;
        st->gid_thr = 0xffffffffu;
      }
    }
  }
  __syncthreads();
}

// seg != null: scan this warp's candidate segment only (every tie w == tau is in it)
__device__ void gid_hist_body(const ImportanceArgs& a, unsigned long long tau, uint32_t gp, int round,
                              unsigned long long* hist /*[256] counts*/, const Seg* seg = nullptr) {
  __shared__ unsigned long long s_cnt[256];
  s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int shift = 8 * (kGRounds - 1 - round);
  auto visit = [&](int64_t t) {
    if (load_w(a, t) != tau) return;
    const uint32_t g = gid_of(a, a.item_lidx ? a.item_lidx[t] : uint32_t(t));
    if (shift + 8 < 32 && (g >> (shift + 8)) != gp) return;
    atomicAdd(&s_cnt[(g >> shift) & 255u], 1ull);
  };
  if (seg) {
    const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t cnt = seg->cnt[gw];
    const uint32_t* L = seg->cand + gw * seg->cap;
    for (uint32_t j = threadIdx.x & 31; j < cnt; j += 32) visit(L[j]);
  } else {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n_items;
         i += int64_t(gridDim.x) * blockDim.x)
      visit(i);
  }
  __syncthreads();
  if (s_cnt[threadIdx.x]) atomicAdd(hist + threadIdx.x, s_cnt[threadIdx.x]);
  __syncthreads();
}

__device__ void gid_decide_body(ImpState* st, int round, const unsigned long long* hist) {
  __shared__ unsigned long long s_pre[256];
  __shared__ int s_pick;
  if (st->empty || !st->need_gid) return;
  const int d = threadIdx.x;
  s_pre[d] = block_incl_scan256(hist[d]);
  if (d == 0) s_pick = -1;
  __syncthreads();
  const unsigned long long below = st->below, k = st->k;
  const unsigned long long incl = s_pre[d], excl = d > 0 ? s_pre[d - 1] : 0ull;
  if (below + incl >= k && below + excl < k) s_pick = d;
  __syncthreads();
  if (d == 0 && s_pick >= 0) {
    st->below = below + (s_pick > 0 ? s_pre[s_pick - 1] : 0ull);
    st->gprefix = (st->gprefix << 8) | uint32_t(s_pick);
    if (round == kGRounds - 1) st->gid_thr = st->gprefix;
  }
  __syncthreads();
}

__device__ void mark_body(const ImportanceArgs& a, const ImpState& st) {
  if (st.empty) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31); base < a.n_items; base += stride) {
    const int64_t t = base + lane;
    bool sel = false;
    uint32_t lidx = 0;
    if (t < a.n_items) {
      const unsigned long long w = load_w(a, t);
      // (w >> tshift) >= prefix; after all rounds tshift = 0 and prefix = tau
      sel = w != 0 && (w >> st.tshift) >= st.prefix;
      lidx = a.item_lidx ? a.item_lidx[t] : uint32_t(t);
      if (sel && w == st.tau && st.need_gid && gid_of(a, lidx) > st.gid_thr) sel = false;
    }
    if (sel) atomicAdd(a.c_vis + lidx, 1u);
    // one atomicAnd per (warp, cull word): records come in local-index order, so a warp's
    // selected items share a few words
    const uint32_t word = sel ? (lidx >> 5) : (0x80000000u | uint32_t(lane));
    const unsigned peers = __match_any_sync(0xffffffffu, word);
    const uint32_t bits = __reduce_or_sync(peers, sel ? (1u << (lidx & 31)) : 0u);
    if (sel && lane == __ffs(peers) - 1) atomicAnd(a.cull + word, ~bits);
  }
}

// all bits [0, n_bits) set, bits past n_bits in the last word clear (grid-stride)
__device__ __forceinline__ void fill_bits_body(uint32_t* words, int64_t n_bits) {
  const int64_t nw = (n_bits + 31) / 32;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < nw; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t rem = n_bits - 32 * t;
    words[t] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
  }
}

// ---- per-round kernels (world > 1) -----------------------------------------------------

__global__ void __launch_bounds__(256) k_imp_stats(ImportanceArgs a, unsigned long long* total) {
  stats_body(a, total);
}

__global__ void __launch_bounds__(256) k_imp_hist(ImportanceArgs a, const ImpState* st, int round,
                                                  unsigned long long* hist) {
  if (st->empty || st->final_ || round < int(st->r0)) return;
  hist_body(a, st->prefix, round, hist);
}

__global__ void __launch_bounds__(256) k_imp_decide(ImpState* st, const unsigned long long* total_in, int round,
                                                    const unsigned long long* hist, int num, int den) {
  if (round == 0) {
    if (threadIdx.x == 0) init_state(st, total_in);
    __syncthreads();
  }
  decide_body(st, round, hist, num, den);
}

__global__ void __launch_bounds__(256) k_imp_gid_hist(ImportanceArgs a, const ImpState* st, int round,
                                                      unsigned long long* hist) {
  if (st->empty || !st->need_gid) return;
  gid_hist_body(a, st->tau, st->gprefix, round, hist);
}

__global__ void __launch_bounds__(256) k_imp_gid_decide(ImpState* st, int round, const unsigned long long* hist) {
  gid_decide_body(st, round, hist);
}

__global__ void __launch_bounds__(256) k_imp_mark(ImportanceArgs a, const ImpState* st) {
  const ImpState s = *st;
  mark_body(a, s);
}

// ---- world == 1: everything in one cooperative launch ------------------------------------

// set = [total + MSB histogram (65)] [w rounds 7 x 512] [gid rounds 4 x 256] [candidate count 1]
constexpr int64_t kImpSetWords = 65 + kWRounds * 512 + kGRounds * 256 + 1;

// `set` was zeroed by the previous call (or at allocation); `next` is zeroed here for the next
// call, so the launch needs no memsets.  The cull words are filled here too.
__global__ void __launch_bounds__(256) k_imp_coop(ImportanceArgs a, ImpState* st_out, unsigned long long* set,
                                                  unsigned long long* next, uint32_t* cand, int num, int den) {
  cg::grid_group grid = cg::this_grid();
  __shared__ ImpState st;
  unsigned long long* total = set;
  unsigned long long* hist = set + 65;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < kImpSetWords;
       t += int64_t(gridDim.x) * blockDim.x)
    next[t] = 0;
  fill_bits_body(a.cull, a.n_local);
  stats_body(a, total);
  grid.sync();
  if (threadIdx.x == 0) init_state(&st, total);
  __syncthreads();
  // The first round whose candidates (the previous crossing bin) are at most half of the items
  // scans everything once more and leaves each warp its candidates in a private segment; the
  // later rounds and the gid rounds rescan only the segments.  Every CTA holds the same state,
  // so the choice is grid-uniform.
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  Seg seg{cand, cand + ((a.n_items + stride - 1) / stride) * stride, (a.n_items + stride - 1) / stride * 32};
  bool listed = false;
  for (int r = int(st.r0); r < kWRounds && !st.empty && !st.final_; ++r) {
    int mode = 0;
    if (listed) mode = 2;
    else if (r > int(st.r0) && 2 * st.next_cnt <= (unsigned long long)a.n_items) mode = 1;
    hist_body(a, st.prefix, r, hist + r * 512, mode, seg);
    listed = listed || mode == 1;
    grid.sync();
    decide_body(&st, r, hist + r * 512, num, den);
  }
  if (!st.empty && st.need_gid) {
    // every tie (w == tau) matched the prefix of every round, so it is in the segments
    for (int r = 0; r < kGRounds; ++r) {
      gid_hist_body(a, st.tau, st.gprefix, r, hist + kWRounds * 512 + r * 256, listed ? &seg : nullptr);
      grid.sync();
      gid_decide_body(&st, r, hist + kWRounds * 512 + r * 256);
    }
  }
  mark_body(a, st);
  if (blockIdx.x == 0 && threadIdx.x == 0) *st_out = st;
}

// all bits [0, n_bits) set, bits past n_bits in the last word clear
__global__ void k_fill_bits(uint32_t* words, int64_t n_bits) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nw = (n_bits + 31) / 32;
  if (t >= nw) return;
  const int64_t rem = n_bits - 32 * t;
  words[t] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
}

// ---- world > 1, two collectives per view ---------------------------------------------------
// (1) every rank: s, c_rad and a coarse histogram of w over 4096 log-linear bins (count, mass):
//     bin(w) = 64 e + (6 bits below the leading one), e = msb(w); monotone in w.  ONE all-reduce.
// (2) every rank decides the same crossing bin b* (mass above b* short of num/den of the total, with
//     b* reaching it) and reads the global count of b* (one host read), packs its items of b* as
//     (w, gid) and ONE all-gather gives every rank all of them.
// (3) one CTA per rank selects exactly among the gathered candidates (radix rounds on w from the
//     leading bit, then on gid among ties), so tau and the gid cut are bit-identical on every rank
//     and equal to the round path's (same integer definition).
constexpr int kCoarseBins = 4096;

__device__ __forceinline__ uint32_t coarse_bin(unsigned long long w) {
  const int e = 63 - __clzll((long long)w);
  const uint32_t m = e >= 6 ? uint32_t(w >> (e - 6)) & 63u : uint32_t(w << (6 - e)) & 63u;
  return uint32_t(e) * 64u + m;
}

__global__ void __launch_bounds__(256) k_imp_stats_coarse(ImportanceArgs a, unsigned long long* hist /*[2][4096]*/) {
  extern __shared__ unsigned long long s_h[];  // [2][4096]
  for (int i = threadIdx.x; i < 2 * kCoarseBins; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31); base < a.n_items; base += stride) {
    const int64_t t = base + lane;
    unsigned long long w = 0;
    if (t < a.n_items) {
      const Item it = load_item(a, t);
      w = it.w;
      if (a.wbuf) a.wbuf[t] = it.w;
      if (it.a > 0) atomicAdd(a.s + it.lidx, (double(it.w) * (1.0 / 16777216.0)) / (double(it.a) + 1e-8));
      if (it.rad) atomicAdd(a.c_rad + it.lidx, 1u);
    }
    const bool cand = w != 0;
    hist_add(cand, cand ? coarse_bin(w) : (1u << 20) + lane, w, lane, s_h, s_h + kCoarseBins);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kCoarseBins; i += blockDim.x)
    if (s_h[i]) {
      atomicAdd(hist + i, s_h[i]);
      atomicAdd(hist + kCoarseBins + i, s_h[kCoarseBins + i]);
    }
}

// one CTA of 1024: the crossing coarse bin from the top
__global__ void __launch_bounds__(1024) k_imp_coarse_decide(ImpState* st, const unsigned long long* hist, int num,
                                                            int den) {
  __shared__ unsigned long long s_part[1024];
  __shared__ unsigned long long s_total;
  // thread j owns bins [4 j, 4 j + 4); suffix sums of the mass from the top
  const int j = threadIdx.x;
  unsigned long long m[4], loc = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    m[k] = hist[kCoarseBins + 4 * j + k];
    loc += m[k];
  }
  s_part[j] = loc;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // inclusive suffix scan: s_part[j] = mass of bins >= 4 j
    const unsigned long long v = j + o < 1024 ? s_part[j + o] : 0ull;
    __syncthreads();
    s_part[j] += v;
    __syncthreads();
  }
  if (j == 0) s_total = s_part[0];
  __syncthreads();
  const unsigned long long total = s_total;
  const unsigned long long target = (unsigned long long)num * total;
  unsigned long long above = j + 1 < 1024 ? s_part[j + 1] : 0ull;  // bins >= 4 j + 4
  if (j == 0) {  // every field written (the selection copies the whole state)
    ImpState z{};
    z.total = total;
    z.empty = total == 0;
    z.gid_thr = 0xffffffffu;
    *st = z;
  }
  __syncthreads();
  if (total == 0) return;
  for (int k = 3; k >= 0; --k) {
    const int b = 4 * j + k;
    const bool cross = (unsigned long long)den * (above + m[k]) >= target && (unsigned long long)den * above < target;
    if (cross && hist[b] > 0) {
      st->bstar = uint32_t(b);
      st->above = above;
      st->ncand = hist[b];
    }
    above += m[k];
  }
}

__global__ void __launch_bounds__(256) k_imp_gather_cand(ImportanceArgs a, const ImpState* st,
                                                         unsigned long long* buf /*[0] count, then (w, gid, -)*/) {
  if (st->empty) return;
  const uint32_t b = st->bstar;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < a.n_items; t += int64_t(gridDim.x) * blockDim.x) {
    const unsigned long long w = load_w(a, t);
    if (w == 0 || coarse_bin(w) != b) continue;
    const unsigned long long pos = atomicAdd(buf, 1ull);
    const uint32_t lidx = a.item_lidx ? a.item_lidx[t] : uint32_t(t);
    buf[2 + 2 * pos] = w;
    buf[3 + 2 * pos] = gid_of(a, lidx);
  }
}

// One CTA (256 threads): exact selection among the gathered candidates of every rank.  Rank r's
// block starts at gath + r * stride (u64 words): [count][pad][(w, gid) x count].
__global__ void __launch_bounds__(256) k_imp_select_cand(ImpState* st, const unsigned long long* gath, int world,
                                                         int64_t stride, int num, int den) {
  __shared__ unsigned long long s_hist[512];  // [256] counts, [256] masses (decide_body's layout)
  unsigned long long* s_cnt = s_hist;
  unsigned long long* s_mass = s_hist + 256;
  __shared__ ImpState S;
  if (st->empty) return;
  if (threadIdx.x == 0) {
    S = *st;
    S.prefix = 0;
    S.k = 0;
    S.below = 0;
    S.gprefix = 0;
    S.need_gid = 0;
    S.final_ = 0;
    const int e = int(S.bstar / 64);
    const int r0 = (kWRounds - 1) - e / 8;
    S.r0 = uint32_t(r0 < 0 ? 0 : r0);
    // digits above the leading bit are 0 for every candidate: the prefix starts from them
  }
  __syncthreads();
  auto for_each = [&](auto fn) {
    for (int r = 0; r < world; ++r) {
      const unsigned long long* blk = gath + r * stride;
      const int64_t n = int64_t(blk[0]);
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) fn(blk[2 + 2 * i], uint32_t(blk[3 + 2 * i]));
    }
  };
  const int lane = threadIdx.x & 31;
  for (int r = int(S.r0); r < kWRounds && !S.final_; ++r) {
    s_cnt[threadIdx.x] = 0;
    s_mass[threadIdx.x] = 0;
    __syncthreads();
    const int shift = 8 * (kWRounds - 1 - r);
    const unsigned long long prefix = S.prefix;
    // warp-uniform trip counts so the warp-aggregated histogram (most candidates share a digit in
    // the first rounds: per-lane 64-bit shared atomics would serialise) can use warp collectives
    for (int rr = 0; rr < world; ++rr) {
      const unsigned long long* blk = gath + rr * stride;
      const int64_t n = int64_t(blk[0]);
      for (int64_t base = threadIdx.x & ~31; base < n; base += blockDim.x) {
        const int64_t i = base + lane;
        const unsigned long long w = i < n ? blk[2 + 2 * i] : 0ull;
        const bool cand = i < n && !(shift + 8 < 64 && (w >> (shift + 8)) != prefix);
        hist_add(cand, cand ? uint32_t((w >> shift) & 255u) : 256u + lane, w, lane, s_cnt, s_mass);
      }
    }
    __syncthreads();
    decide_body(&S, r, s_cnt, num, den);  // reads hist[d] counts, hist[256 + d] masses
  }
  __syncthreads();
  if (S.final_) {
    // the crossing bin of an earlier round held exactly one candidate: its w is tau
    const unsigned long long pre = S.prefix;
    const uint32_t tsh = S.tshift;
    for_each([&](unsigned long long w, uint32_t) {
      if ((w >> tsh) == pre) S.tau = w;
    });
    __syncthreads();
    if (threadIdx.x == 0) {
      S.prefix = S.tau;
      S.tshift = 0;
    }
    __syncthreads();
  }
  if (S.need_gid) {
    for (int r = 0; r < kGRounds; ++r) {
      s_cnt[threadIdx.x] = 0;
      __syncthreads();
      const int shift = 8 * (kGRounds - 1 - r);
      const unsigned long long tau = S.tau;
      const uint32_t gp = S.gprefix;
      for_each([&](unsigned long long w, uint32_t g) {
        if (w != tau) return;
        if (shift + 8 < 32 && (g >> (shift + 8)) != gp) return;
        atomicAdd(&s_cnt[(g >> shift) & 255u], 1ull);
      });
      __syncthreads();
      gid_decide_body(&S, r, s_cnt);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    S.tshift = 0;
    S.prefix = S.tau;
    *st = S;
  }
}

unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  return unsigned(b < 1 ? 1 : b);
}

}  // namespace

static_assert(sizeof(ImpState) <= kImpStateBytes, "state fits its arena slot");
int imp_w_rounds() { return kWRounds; }
int imp_g_rounds() { return kGRounds; }

void launch_fill_bits(uint32_t* words, int64_t n_bits, cudaStream_t s) {
  const int64_t nw = (n_bits + 31) / 32;
  if (nw > 0) k_fill_bits<<<unsigned((nw + 255) / 256), 256, 0, s>>>(words, n_bits);
}

void launch_imp_stats(const ImportanceArgs& a, unsigned long long* total, cudaStream_t s) {
  if (a.n_items > 0) k_imp_stats<<<grid_for(a.n_items), 256, 0, s>>>(a, total);
}

void launch_imp_hist(const ImportanceArgs& a, const ImpState* st, int round, unsigned long long* hist,
                     cudaStream_t s) {
  k_imp_hist<<<grid_for(a.n_items), 256, 0, s>>>(a, st, round, hist);
}

void launch_imp_decide(ImpState* st, const unsigned long long* total, int round, const unsigned long long* hist,
                       int num, int den, cudaStream_t s) {
  k_imp_decide<<<1, 256, 0, s>>>(st, total, round, hist, num, den);
}

void launch_imp_gid_hist(const ImportanceArgs& a, const ImpState* st, int round, unsigned long long* hist,
                         cudaStream_t s) {
  k_imp_gid_hist<<<grid_for(a.n_items), 256, 0, s>>>(a, st, round, hist);
}

void launch_imp_gid_decide(ImpState* st, int round, const unsigned long long* hist, cudaStream_t s) {
  k_imp_gid_decide<<<1, 256, 0, s>>>(st, round, hist);
}

void launch_imp_mark(const ImportanceArgs& a, const ImpState* st, cudaStream_t s) {
  if (a.n_items > 0) k_imp_mark<<<grid_for(a.n_items), 256, 0, s>>>(a, st);
}

int64_t imp_set_words() { return kImpSetWords; }

void launch_imp_stats_coarse(const ImportanceArgs& a, unsigned long long* hist, cudaStream_t s) {
  static std::atomic<int> attr[kMaxDevices];
  per_device(attr, [] {
    cudaFuncSetAttribute(k_imp_stats_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(2 * kCoarseBins * sizeof(unsigned long long)));
    return 1;
  });
  if (a.n_items > 0)
    k_imp_stats_coarse<<<grid_for(a.n_items) < 296u ? grid_for(a.n_items) : 296u, 256,
                         2 * kCoarseBins * sizeof(unsigned long long), s>>>(a, hist);
}

void launch_imp_coarse_decide(ImpState* st, const unsigned long long* hist, int num, int den, cudaStream_t s) {
  k_imp_coarse_decide<<<1, 1024, 0, s>>>(st, hist, num, den);
}

void launch_imp_gather_cand(const ImportanceArgs& a, const ImpState* st, unsigned long long* buf, cudaStream_t s) {
  if (a.n_items > 0) k_imp_gather_cand<<<grid_for(a.n_items), 256, 0, s>>>(a, st, buf);
}

void launch_imp_select_cand(ImpState* st, const unsigned long long* gathered, int world, int64_t stride_words,
                            int num, int den, cudaStream_t s) {
  k_imp_select_cand<<<1, 256, 0, s>>>(st, gathered, world, stride_words, num, den);
}

int64_t imp_coarse_words() { return 2 * kCoarseBins; }
size_t imp_state_ncand_offset() { return offsetof(ImpState, ncand); }

static int coop_blocks() {
  static std::atomic<int> slots[kMaxDevices];
  return per_device(slots, [] {
    int per_sm = 0, blocks = 0;
    const int sms = device_sm_count();
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_imp_coop, 256, 0);
    // 2 CTAs per SM: a cooperative grid holds its SM slots while it waits at grid syncs, which
    // starves the other views in flight; measured on Rubble (4 in flight / one view's importance
    // stage): 4/SM 1273-1294 views/s / 0.091 ms, 2/SM 1336-1343 / 0.105 ms, 1/SM 1342 / 0.155 ms
    const char* e = getenv("BGS_IMP_COOP_PER_SM");  // tuning only
    const int cap = e && atoi(e) > 0 ? atoi(e) : 2;
    blocks = sms * (per_sm < cap ? per_sm : cap);
    return blocks < 1 ? 1 : blocks;
  });
}

int64_t imp_cand_words(int64_t n_items) {
  const int64_t stride = int64_t(coop_blocks()) * 256;
  return (n_items + stride - 1) / stride * stride + stride / 32 + 1;
}

cudaError_t launch_imp_coop(const ImportanceArgs& a, ImpState* st, unsigned long long* set,
                            unsigned long long* next, uint32_t* cand, int num, int den, cudaStream_t s) {
  const int blocks = coop_blocks();
  ImportanceArgs aa = a;
  int nn = num, dd = den;
  void* args[] = {&aa, &st, &set, &next, &cand, &nn, &dd};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_imp_coop), dim3(blocks), dim3(256), args, 0, s);
}

}  // namespace bgs
