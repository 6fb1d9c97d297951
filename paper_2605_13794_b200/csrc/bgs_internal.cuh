// Internal declarations shared by the libbgs translation units (NOT part of the ABI).
// Layouts here are documented in DESIGN.md §6 ("Data layout in HBM").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/bgs.h"

namespace bgs {

constexpr int kTile = 16;           // 16x16 pixel tiles (vanilla 3DGS)
constexpr int kMaxWorld = 8;        // dest mask is one byte
constexpr int kSortBlock = 256;     // onesweep CTA
constexpr int kSortItems = 16;      // keys per thread per onesweep partition
constexpr int kSortPart = kSortBlock * kSortItems;  // 4096 keys per partition (Morton layout sort)
constexpr int kViewSortItems = 16;  // per-view pair sort (u32 keys); 8 measured slower (longer look-back chains)
constexpr int kViewSortPart = kSortBlock * kViewSortItems;
constexpr int kMaxSortPasses = 6;   // 8-bit digits over <= 48 key bits

// ProjectedSplat record, 48 B, three 16-B rows.
struct __align__(16) Rec {
  float mx, my, A, B;        // mean2d (px), conic A, B
  float C, opac, r, g;       // conic C, opacity, colour
  float b, depth;            // colour, camera z
  uint32_t gid;              // global id = local*world + rank
  uint32_t rect;             // x0 | y0<<8 | x1<<16 | y1<<24  (tiles, exclusive max)
};
static_assert(sizeof(Rec) == 48, "record is 48 B");

// Per-splat accumulators: 9 gradients + a + w_fixed (48 B), the unit of the reverse exchange.
struct __align__(16) Acc {
  float g[9];                // dL/d(mx, my, A, B, C, o, r, g, b)
  uint32_t a;                // qualifying pixel count a_{i,v}
  unsigned long long w;      // sum of rint(alpha*T*2^24)
};
static_assert(sizeof(Acc) == 48, "accumulator is 48 B");

// Device counters (u64 each) in the ctx arena.
enum Counter : int {
  C_F = 0,        // records produced by project
  C_PALL = 1,     // sum of rect areas (pairs over all tiles) of this rank's records
  C_NLOD = 2,     // |L^(m)|
  C_NACT = 3,     // |A^(m)|
  C_P = 4,        // pairs emitted for owned tiles
  C_CAND = 5,     // candidates passing the conservative off-screen bound
  C_DLO = 6,      // 0xffffffff - min f32 bits(depth) over the records the pairs come from (atomicMax)
  C_DHI = 7,      // max f32 bits(depth) over the same records
  C_NCOUNTERS = 8
};

// Sort key of a pair (a5/a6), 32 bits: (local tile << kd) | ((bits(depth) - lo) >> sd).
// lo = min depth bits, nb = bit width of (max - min) depth bits.  Depths are positive floats, so
// their bit patterns order like the values and bits - lo is an exact order-preserving map onto
// [0, 2^nb).  kd = min(nb, 32 - tbits) of those bits are kept (sd = nb - kd dropped from the
// bottom, 0 unless nb + tbits > 32); the key then orders pairs by (tile, depth) up to runs of
// equal keys, which k_ranges_fixup orders by (full depth bits, global id) -- so the final order
// is exactly (tile, depth, gid) (R12).  Rubble views: nb = 22..24, tbits = 12, sd = 2..4.
struct KeyLayout {
  uint32_t lo;
  int nb, kd, sd;
};
__host__ __device__ inline KeyLayout key_layout(unsigned long long c_dlo, unsigned long long c_dhi, int tbits) {
  KeyLayout k;
  k.lo = 0xffffffffu - uint32_t(c_dlo);
  const uint32_t hi = uint32_t(c_dhi);
  const uint32_t span = hi > k.lo ? hi - k.lo : 0u;
#ifdef __CUDA_ARCH__
  k.nb = 32 - __clz(span);
#else
  int nb = 0;
  while (nb < 32 && (span >> nb) != 0u) ++nb;
  k.nb = nb;
#endif
  k.kd = k.nb < 32 - tbits ? k.nb : 32 - tbits;
  k.sd = k.nb - k.kd;
  return k;
}

struct CameraK {
  float fx, fy, cx, cy;
  int W, H, TX, TY;
  float R[9], t[3], campos[3], near_clip;
};

struct ProjectArgs {
  const float4* mean_opac;
  const float4* quat;
  const float4* scale;
  const float* sh;
  const uint8_t* lod;
  const uint32_t* cull;      // nullable
  const float4* bounds;      // nullable: per BGS_BOUNDS_BLOCK rows {min mu, max s}, {max mu, -} (hierarchical cull)
  int64_t n;
  CameraK cam;
  int gate_enabled, l_max, fb_num, fb_den;
  float D2[32];
  int no_color;
  int rank, world;
  float lim[4];              // Jacobian clamp limits x+, x-, y+, y- (same float expressions as the oracle)
  float cull_K;              // fx^2 (1 + Lx^2) + fy^2 (1 + Ly^2) for the conservative radius bound
  // outputs
  int32_t* radius;
  Rec* recs;
  uint32_t* rec_lidx;
  unsigned long long* counters;
  int32_t* tile_diff;        // nullable: (TY+1)*(TX+1) 2D difference array of rect coverage
  uint32_t* cand;            // [n] candidate list written by k_cull
  float4* jdir;              // [3 F] per local record: colour Jacobian wrt the view direction + clamp bits (k_color)
  int64_t rec_cap;
};

void launch_gate_count(const ProjectArgs& a, cudaStream_t s);
void launch_project(const ProjectArgs& a, cudaStream_t s);
void launch_color(const ProjectArgs& a, cudaStream_t s);  // after launch_project; F read on device
void launch_shard_bounds(const float4* mean_opac, const float4* scale, int64_t n, float4* bounds, cudaStream_t s);

// sort (a5-a7)
struct SortArgs {
  const Rec* recv;
  int64_t n_recv;
  int TX, t_begin, t_end;
  unsigned long long* keys[2];
  uint32_t* vals[2];
  int64_t cap;               // capacity of key/val buffers
  unsigned long long* counters;
  uint32_t* digit_hist;      // [kMaxSortPasses][256]
  uint32_t* pass_ctrl;       // [16]: active flags, src selectors, partition counters
  uint32_t* status;          // look-back status [n_parts][256] per pass
  int n_passes;
  int tbits;                 // bits of the local tile index (per-view sort: 32-bit keys, KeyLayout)
  uint2* ranges;             // [t_end - t_begin]
  float4* aux;               // [n_recv] per-record raster constants (thr, half extent x, half extent y, -)
};
// emits pairs and digit histograms; returns nothing (P stays on device, counters[C_P])
void launch_emit(const SortArgs& a, cudaStream_t s);
// world > 1: depth range of the received records into counters C_DLO / C_DHI (zeroed by the caller)
void launch_depth_range(const Rec* recv, int64_t n, unsigned long long* counters, cudaStream_t s);
// key_bytes: 4 (per-view pairs, keys[] hold uint32_t) or 8 (Morton layout, unsigned long long)
void launch_sort_passes(const SortArgs& a, int64_t P, cudaStream_t s, int64_t* launches, int key_bytes);
void launch_ranges_fixup(const SortArgs& a, int64_t P, cudaStream_t s);
void launch_tile_order(const uint2* ranges, int n_tiles, uint32_t* perm, cudaStream_t s);
// bucket.cu: a5-a7 as a per-tile bucket sort.  tile_counts: pairs per tile (indexed by global tile,
// the owned run [t_begin, t_end) is used); cursor: [t_end - t_begin] scratch.  Writes ranges, the
// sorted 64-bit keys (f32 bits(depth) << 32 | gid) to keys[0] and the record indices to vals[0].
// order: [t_end - t_begin] longest-first tile order (also the raster's tile_perm)
void launch_bucket_sort(const SortArgs& a, const int32_t* tile_counts, uint32_t* cursor, uint32_t* order,
                        cudaStream_t s, int64_t* launches);
// Pairs per tile of a record set (rect coverage) for the tiles [t_lo, t_hi) (t_hi - t_lo <= 16384),
// accumulated into counts[t - t_lo] (zeroed by the caller); n_dev (nullable): count on the device.
void launch_tile_count(const Rec* recs, int64_t n_cap, const unsigned long long* n_dev, int TX, int t_lo, int t_hi,
                       int32_t* counts, cudaStream_t s);
// layout.cu: Morton permutation of a shard (keys/vals/digit_hist/pass_ctrl/status of `a` used as scratch)
void launch_spatial_order(const float4* mean_opac, int64_t n, unsigned int* box, const SortArgs& a, uint32_t* perm,
                          cudaStream_t s, int64_t* launches);
// which buffer (0/1) holds the sorted data after the passes: read from pass_ctrl on device
// by the consumers below.

// raster (a8, a9)
struct RasterArgs {
  const Rec* recv;
  const uint2* ranges;
  const unsigned long long* keys[2];
  const uint32_t* vals[2];
  const uint32_t* pass_ctrl;  // value buffer selector at pass_ctrl[kValsSel]
  int t_begin, n_tiles, TX, W, H;
  Acc* acc;
  const float4* aux;          // per received record: thr, box half extents (from k_emit)
  const uint32_t* tile_perm;  // launch order of the owned tiles (longest list first)
  int n_split;                // the first n_split tiles of tile_perm run as two half-tile CTAs
  uint32_t* cmask;            // contributor masks: written by the forward, read by the backward
  int no_color;               // the view was projected with BGS_NO_COLOR: no colour compositing
};
constexpr int kRasterSlots = 8;  // warp blocks per tile (8 in a split tile, 4 otherwise)
constexpr int kFinalSel = 15;  // buffer holding the sorted keys after the passes
constexpr int kValsSel = 24;   // buffer holding the final (tie-fixed) values, written by k_ranges_fixup
// returns the number of split tiles used (the backward must be launched with the same split)
int launch_raster_fwd(const RasterArgs& a, uint32_t flags, float* rgb, float* t_final, int32_t* n_contrib,
                      cudaStream_t s);
void launch_raster_bwd(const RasterArgs& a, const float* dL, const float* t_final, const int32_t* n_contrib,
                       cudaStream_t s);

// projection backward (a11)
struct ProjectBwdArgs {
  const float4* mean_opac;
  const float4* quat;
  const float4* scale;
  const float* sh;
  const uint32_t* rec_lidx;
  const Acc* acc;            // per local record, owner-summed
  const float4* jdir;        // [3 F] k_color's colour Jacobian wrt the view direction + clamp bits
  int64_t F;
  CameraK cam;
  float4* g_mean_opac;
  float4* g_quat;
  float4* g_scale;
  float* g_sh;
};
void launch_project_bwd(const ProjectBwdArgs& a, cudaStream_t s);

// routing (a3, a4, a10) for world > 1
void launch_tile_costs(const int32_t* diff, int TX, int TY, int32_t* pairs_t, cudaStream_t s);
void launch_owner_map(const int32_t* pairs_t, int T, int world, int32_t* owner, int32_t* run, long long* pown,
                      const int32_t* given, cudaStream_t s);
// F_dev (nullable): the record count on the device (batched steps); F is then the grid's capacity
void launch_dest_count(const Rec* recs, int64_t F, const unsigned long long* F_dev, const int32_t* owner, int TX,
                       int world, uint8_t* dest_mask, uint32_t* block_counts, cudaStream_t s);
void launch_block_scan(uint32_t* block_counts, int64_t F, const unsigned long long* F_dev, int world,
                       unsigned long long* totals, cudaStream_t s);
void launch_pack(const Rec* recs, int64_t F, const unsigned long long* F_dev, const uint8_t* dest_mask,
                 const uint32_t* block_offs, int world, const int64_t* send_base, Rec* send, cudaStream_t s);
void launch_gather_sum(const Acc* rev, int64_t F, const unsigned long long* F_dev, const uint8_t* dest_mask,
                       const uint32_t* block_offs, int world, const int64_t* send_base, Acc* out, cudaStream_t s);
// BGS_IMPORTANCE_ONLY reverse: (w, a) of the received records as 12-B units, and their gather-sum
void launch_pack_imp(const Acc* acc, int64_t R, void* out, cudaStream_t s);
void launch_gather_imp(const void* rev, int64_t F, const uint8_t* dest_mask, const uint32_t* block_offs, int world,
                       const int64_t* send_base, Acc* out, cudaStream_t s);
struct PtrList {
  const void* p[kMaxWorld];
  int n;
};
void launch_reduce_sum_i32(PtrList src, int32_t* dst, int64_t n, cudaStream_t s);
void launch_reduce_sum_u64(PtrList src, unsigned long long* dst, int64_t n, cudaStream_t s);
void launch_reduce_sum_f32(PtrList src, float* dst, int64_t n, cudaStream_t s);
void launch_reduce_sum_f64(PtrList src, double* dst, int64_t n, cudaStream_t s);
constexpr int kRouteBlock = 256;

// importance (a12)
struct ImportanceArgs {
  int64_t n_items;           // n_local (dense) or F (per record)
  const uint32_t* item_lidx; // nullable: dense when null
  const int32_t* radius;     // dense only
  const unsigned long long* w_dense;
  const uint32_t* a_dense;
  const Acc* acc;            // per record when dense arrays are null
  int64_t n_local;
  int rank, world;
  double* s;
  uint32_t* c_rad;
  uint32_t* c_vis;
  uint32_t* cull;
  unsigned long long* wbuf;  // [n_items] scratch: w copied densely by the stats pass
};
struct ImpState;
constexpr size_t kImpStateBytes = 128;
int imp_w_rounds();
int imp_g_rounds();
void launch_imp_stats(const ImportanceArgs& a, unsigned long long* total, cudaStream_t s);
void launch_imp_hist(const ImportanceArgs& a, const ImpState* st, int round, unsigned long long* hist,
                     cudaStream_t s);
void launch_imp_decide(ImpState* st, const unsigned long long* total, int round, const unsigned long long* hist,
                       int num, int den, cudaStream_t s);
void launch_imp_gid_hist(const ImportanceArgs& a, const ImpState* st, int round, unsigned long long* hist,
                         cudaStream_t s);
void launch_imp_gid_decide(ImpState* st, int round, const unsigned long long* hist, cudaStream_t s);
void launch_imp_mark(const ImportanceArgs& a, const ImpState* st, cudaStream_t s);
void launch_fill_bits(uint32_t* words, int64_t n_bits, cudaStream_t s);
// world == 1: cull fill + stats + every round + mark in one cooperative launch.  `set` (total,
// histograms, candidate count; imp_set_words() u64) must be zero on entry; the kernel zeroes
// `next` (same size) for the following call.  cand: u32 scratch [n_items].
int64_t imp_set_words();
int64_t imp_cand_words(int64_t n_items);  // u32 scratch the cooperative kernel's candidate segments need
// world > 1, two collectives: coarse (count, mass) histogram over 4096 log-linear bins of w (zeroed
// by the caller, all-reduced between the calls), the crossing bin, its candidates packed as
// [count, pad, (w, gid) x count] u64 words, and the exact selection among every rank's candidates
void launch_imp_stats_coarse(const ImportanceArgs& a, unsigned long long* hist, cudaStream_t s);
void launch_imp_coarse_decide(ImpState* st, const unsigned long long* hist, int num, int den, cudaStream_t s);
void launch_imp_gather_cand(const ImportanceArgs& a, const ImpState* st, unsigned long long* buf, cudaStream_t s);
void launch_imp_select_cand(ImpState* st, const unsigned long long* gathered, int world, int64_t stride_words,
                            int num, int den, cudaStream_t s);
int64_t imp_coarse_words();
size_t imp_state_ncand_offset();
cudaError_t launch_imp_coop(const ImportanceArgs& a, ImpState* st, unsigned long long* set,
                            unsigned long long* next, uint32_t* cand, int num, int den, cudaStream_t s);

// NEXT-1 simplification (simplify.cu)
void launch_phi(int64_t n, const uint32_t* c_rad, const uint32_t* c_vis, double* phi, cudaStream_t s);
void launch_keys_race(int64_t n, const double* sc, unsigned long long seed, int rank, int world,
                      unsigned long long* key, cudaStream_t s);
void launch_keys_mass(int64_t n, const double* sc, unsigned long long* key, cudaStream_t s);
size_t sel_state_bytes();
int sel_rounds();
int sel_gid_rounds();
void launch_sel_total(int64_t n, const unsigned long long* key, int mass, unsigned long long* total, cudaStream_t s);
void launch_sel_hist(int64_t n, const unsigned long long* key, const void* st, int round, unsigned long long* hist,
                     cudaStream_t s);
void launch_sel_decide(void* st, const unsigned long long* total, int round, const unsigned long long* hist, int mass,
                       long long num, long long den, unsigned long long k, cudaStream_t s);
void launch_sel_gid_hist(int64_t n, const unsigned long long* key, const void* st, int round, int rank, int world,
                         unsigned long long* hist, cudaStream_t s);
void launch_sel_gid_decide(void* st, int round, const unsigned long long* hist, cudaStream_t s);
void launch_sel_mark(int64_t n, const unsigned long long* key, const void* st, int rank, int world, uint8_t* keep,
                     cudaStream_t s);
void launch_keep_positive(int64_t n, const double* sc, uint8_t* keep, unsigned long long* count, cudaStream_t s);
void launch_fill_u8(int64_t n, uint8_t* p, uint8_t v, cudaStream_t s);
size_t param_row_bytes();
void launch_pack_bits(int64_t n, const uint8_t* keep, uint32_t* bits, cudaStream_t s);
void launch_new_ids(int64_t N, const uint32_t* masks, int64_t wpr, int world, int rank, uint32_t* bc,
                    unsigned long long* total, int64_t n_local, uint32_t* new_gid, cudaStream_t s);
void launch_dest_hist(int64_t n, const uint32_t* new_gid, int world, unsigned long long* cnt, cudaStream_t s);
void launch_pack_rows(int64_t n, const uint32_t* new_gid, int world, const int64_t* dest_base,
                      unsigned long long* cursor, const bgs_gaussians& g, void* out, cudaStream_t s);
void launch_scatter_direct(int64_t n, const uint32_t* new_gid, const bgs_gaussians& g, const bgs_gaussians_out& o,
                           int64_t cap, cudaStream_t s);
void launch_unpack_rows(int64_t n, const void* in, const bgs_gaussians_out& o, int64_t cap, cudaStream_t s);

// NEXT-4 supervision: Eq.7 photometric loss on the owned tiles (fused with its gradient) and the
// Eq.8 scale regulariser (loss.cu)
struct LossArgs {
  const float* x;      // rendered image [3][H][W] (full image at world > 1: all-reduced)
  const float* y;      // target image [3][H][W]
  float* dL;           // dl/dx on the owned pixels, [3][H][W]
  double2* partials;   // per CTA: (sum |x - y|, sum SSIM) over its owned pixels
  int W, H, TX, t_begin, t_end;
  float k_l1, k_ssim;  // batch_inv (1 - lambda) / (3 H W), batch_inv lambda / (3 H W)
  float g[11];         // normalised 1-D Gaussian window, sigma 1.5
};
size_t loss_smem_bytes();
int64_t loss_n_blocks(int W, int H);
void launch_loss_photo(const LossArgs& a, cudaStream_t s);
void launch_loss_sums(const double2* partials, int n, double* sums, cudaStream_t s);
void launch_loss_finish(const double* sums, double n_elem, double lambda, double* out, cudaStream_t s);
void launch_owned_copy(const float* rgb, int W, int H, int TX, int t_begin, int t_end, float* full, cudaStream_t s);
int scale_n_blocks(int64_t n);
void launch_scale_sum(const float4* scale, const uint32_t* lidx, int64_t n, double2* partials, cudaStream_t s);
void launch_scale_finish(const double* sums, double* out, cudaStream_t s);
void launch_scale_grad(const float4* scale, const uint32_t* lidx, int64_t n, const double* sums, float beta,
                       float* g_scale, cudaStream_t s);

// NEXT-3 fused Adam on the owned shard (adam.cu)
struct AdamArgs {
  int64_t n;
  float4* p[3];        // raw: (mu, opacity logit), q_raw, (log s, 0)
  float4* m[3];
  float4* v[3];
  float4* g[3];        // gradients w.r.t. the ACTIVATED parameters; zeroed after the step
  float4* act[3];      // activated planes written: (mu, sigmoid), q / |q|, (exp(log s), 0)
  float *sh_p, *sh_m, *sh_v, *sh_g, *sh_act;  // [n][48]; sh_act may equal sh_p (then not written)
  const uint32_t* visible;  // nullable bit mask: rows with bit 0 are not touched
  float lr_mean, lr_opacity, lr_quat, lr_scale, lr_sh_dc, lr_sh_rest;
  float b1, b2, om1, om2, eps, c1, c2;  // om = 1 - b (double on the host), c1 = 1/(1 - b1^t), c2 = 1/(1 - b2^t)
};
void launch_adam(const AdamArgs& a, cudaStream_t s);
void launch_visibility_or(const int32_t* radius, int64_t n, uint32_t* mask, cudaStream_t s);

// NEXT-3 density control (densify.cu)
struct DensifyAccArgs {
  int64_t F;
  const uint32_t* lidx;  // local index of each record
  const Rec* recs;       // the view's local records (mx, my, A, B | C, o, ...)
  const Acc* acc;        // owner-summed moments per local record
  const double* phi;     // nullable: phi = 1
  float half_w, half_h;  // NDC scaling of dL/dmean2d (R37)
  float* stat;
  uint32_t* count;
};
void launch_densify_accumulate(const DensifyAccArgs& a, cudaStream_t s);

struct DensifyArgs {
  int64_t n;
  int rank, world;
  const float4* p_in[3];
  const float4* m_in[3];
  const float4* v_in[3];
  const float *sh_in, *sh_m_in, *sh_v_in;
  const uint8_t* lod_in;
  const float* stat;
  const uint32_t* count;
  float tau, log_extent, logit_min, log_div;
  unsigned long long seed;
  int max_level;  // K - 1: split children's level is min(l + 1, K - 1) (heritage rule)
  uint32_t* block_counts;        // 3 per block, scanned in place
  unsigned long long* totals;    // kept, clones, split parents
  float4* p_out[3];
  float4* m_out[3];
  float4* v_out[3];
  float *sh_out, *sh_m_out, *sh_v_out;
  uint8_t* lod_out;
  float4* act[3];                // nullable: activated planes of the output
  float* sh_act;
};
int64_t densify_n_blocks(int64_t n);
void launch_densify_count(const DensifyArgs& a, cudaStream_t s);
void launch_densify_emit(const DensifyArgs& a, cudaStream_t s);

// Pinned fp64 natural logarithm (reading R30; also the alpha-cut threshold thr = -ln(255 o), D3):
// u = m 2^e with m in [sqrt(2)/2, sqrt(2)) (exact split), ln(m) = 2 atanh(f), f = (m - 1)/(m + 1),
// the 12-term odd series in Horner form, every step one correctly rounded IEEE op (explicit _rn
// intrinsics: no contraction in any TU), so the oracle's plain-C++ / numpy versions of the same
// steps give the same bits.  u > 0, normal, finite.
__device__ __forceinline__ double ln_pinned(double u) {
  // 1/(2k+1) as correctly rounded doubles (compile-time IEEE division)
  constexpr double kInvOdd[12] = {1.0 / 1,  1.0 / 3,  1.0 / 5,  1.0 / 7,  1.0 / 9,  1.0 / 11,
                                  1.0 / 13, 1.0 / 15, 1.0 / 17, 1.0 / 19, 1.0 / 21, 1.0 / 23};
  const unsigned long long b = __double_as_longlong(u);
  int e = int((b >> 52) & 0x7ff) - 1023;
  double m = __longlong_as_double((long long)((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull));  // [1, 2)
  if (m > 1.4142135623730951) {
    m = __dmul_rn(m, 0.5);
    e += 1;
  }
  const double f = __ddiv_rn(__dadd_rn(m, -1.0), __dadd_rn(m, 1.0));
  const double f2 = __dmul_rn(f, f);
  double p = kInvOdd[11];
#pragma unroll
  for (int k = 10; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, f2), kInvOdd[k]);
  const double lm = __dmul_rn(__dadd_rn(f, f), p);
  return __dadd_rn(__dmul_rn(double(e), 0.6931471805599453), lm);
}

// thr = -ln(255 o) rounded to float: alpha = o G >= 1/255 <=> power >= thr (D3), pinned (above)
__device__ __forceinline__ float alpha_cut_thr(float o) { return float(-ln_pinned(__dmul_rn(255.0, double(o)))); }

// Per-device cache of a host-side launch parameter (SM count, occupancy-derived grid size, a
// dynamic shared-memory opt-in done once per device).  `slots` is a function-local static array;
// the value is computed on first use on each device ordinal of the calling thread's current device
// (compute() must return > 0 and be idempotent: two threads racing on a first use both store the
// same value).
constexpr int kMaxDevices = 64;
template <class F>
inline int per_device(std::atomic<int> (&slots)[kMaxDevices], F compute) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return compute();
  int v = slots[dev].load(std::memory_order_acquire);
  if (v <= 0) {
    v = compute();
    slots[dev].store(v, std::memory_order_release);
  }
  return v;
}

inline int device_sm_count() {
  static std::atomic<int> slots[kMaxDevices];
  return per_device(slots, [] {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
  });
}

}  // namespace bgs
