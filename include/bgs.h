/* =========================================================================================
 * bgs.h — C ABI of libbgs: the BlitzGS per-view distributed splatting step on B200 (sm_100a).
 *
 * Paper: "BlitzGS" (arXiv 2605.13794).  Citations: P:n = PAPER.md line n, S:n = SPEC.md line n
 * (the paper text and the spec written from it).  Readings R1..R28 / decisions D1..D7 are
 * listed in DESIGN.md §2.
 *
 * One view of the method, in call order per rank:
 *   bgs_project        a1 gate (Eq.4-6) + a2 EWA projection / SH colour
 *   bgs_route          a3 cost-aware tile ownership + a4 single all-to-all
 *   bgs_sort_tiles     a5 (tile,depth) pair emission + a6 onesweep radix sort + a7 tile ranges
 *   bgs_raster_fwd     a8 front-to-back compositing, Eq.2, + w_{i,v}, a_{i,v}
 *   bgs_raster_bwd     a9 backward of Eq.2
 *   bgs_route_reverse  a10 reverse exchange of per-splat gradients to the owning shard
 *   bgs_project_bwd    a11 backward of the projection
 *   bgs_importance     a12 Eq.3 score, c^rad, c^vis top-99% mass, Cull column
 *   bgs_loss_photo     NEXT-4 Eq.7 L1 + SSIM on the owned tiles with its gradient
 *   bgs_loss_scale     NEXT-4 Eq.8 scale regulariser over the visible set
 *   bgs_adam_step      NEXT-3 fused activation-chain-rule + Adam step on the owned shard
 *   bgs_densify_*      NEXT-3 phi-reweighted density statistic, clone / split / prune with heritage
 * bgs_view_step / bgs_view_step_host run a1..a11 (+a12 when requested) in one call.
 *
 * Conventions (all entry points):
 *  - Status codes only; nothing throws across the ABI.  On a non-OK status the message is
 *    available from bgs_last_error(ctx) until the next call on that ctx.
 *  - Pointers documented "device" must be device-accessible memory on the ctx's device
 *    (e.g. torch CUDA tensors); "host" pointers are ordinary (optionally pinned) memory.
 *  - All inputs and fixed-size outputs are CALLER-owned.  Variable-size intermediates
 *    (records, exchange buffers, pairs, per-splat gradients) live in the ctx arena and stay
 *    valid until the next call of the same stage on that ctx.
 *  - Every call enqueues on `stream` (a cudaStream_t passed as void*; NULL selects the calling
 *    thread's per-thread default stream cudaStreamPerThread, never the legacy default stream).
 *    Successive calls on one ctx must use one stream (or be ordered by the caller).  Calls marked
 *    HOST-SYNC block the host on that stream once (to size variable buffers).
 *  - One ctx per rank and per host thread.  world > 1 uses NCCL (ncclCommInitRank from a
 *    unique id) or, for single-GPU testing, an in-process group sharing one device.
 *  - Layouts: Gaussian parameters are structure-of-arrays of 16-byte rows so kernels issue
 *    128-bit loads; the global id of local Gaussian j on rank m is j*world + m (index
 *    parity sharding).
 * ========================================================================================= */
#ifndef BGS_H_
#define BGS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BGS_OK = 0,
  BGS_ERR_INVALID_ARGUMENT = 1, /* null pointer, n<0, W/H<=0, fx/fy<=0, world mismatch, world>8 */
  BGS_ERR_CAPACITY = 2,         /* arena could not grow; bytes requested in bgs_last_error */
  BGS_ERR_CUDA = 3,             /* a CUDA runtime error (message has cudaGetErrorString) */
  BGS_ERR_NCCL = 4,             /* an NCCL error */
  BGS_ERR_CONTRACT = 5,         /* stage called out of order / shapes inconsistent */
  BGS_ERR_INTERNAL = 6
} bgs_status;

typedef struct bgs_ctx bgs_ctx;

/* flags */
#define BGS_NO_COLOR 1u   /* a2 skips SH colour (instrumented scoring pass "bypasses color shading") */
#define BGS_IMPORTANCE 2u /* a8 accumulates w_fixed (sum of alpha*T in 2^-24 units) and a per splat */
#define BGS_IMPORTANCE_ONLY 8u /* a10 sends only (w_fixed, a), 12 B per record (scoring sweeps: no backward) */

/* Pinhole camera.  R row-major world->camera, x right, y down, camera looks +z;
 * campos = -R^T t is the camera centre c_v of Eq.5 (caller-computed); pixels are centred at
 * integer coordinates (R6); near_clip in world units (R7). */
typedef struct {
  float fx, fy, cx, cy;
  int32_t width, height;
  float R[9];
  float t[3];
  float campos[3];
  float near_clip;
} bgs_camera;

/* The local shard G^(m), ACTIVATED parameters (R13: exp/sigmoid/normalise live in the
 * caller).  All device pointers, n_local rows each:
 *   mean_opac float4 (mu_x, mu_y, mu_z, opacity in (0,1))
 *   quat      float4 (w, x, y, z), unit norm
 *   scale     float4 (s_x, s_y, s_z, unused) per-axis standard deviation > 0
 *   sh        float  [n_local][16][3] degree-3 SH, coefficient-major, RGB inner (R1)
 *   lod       uint8  [n_local] LOD label l_i
 *   bounds    nullable: per block of BGS_BOUNDS_BLOCK rows, 8 floats {min mu_x, min mu_y, min mu_z,
 *             max_j s_j, max mu_x, max mu_y, max mu_z, 0} written by bgs_shard_bounds for THESE
 *             parameters (stale bounds are a contract violation: refresh after every update).  With
 *             bounds, a1 skips every block whose box cannot reach the image (hierarchical culling;
 *             ungated steps only), reading 32 B per block instead of 32 B per Gaussian. */
#define BGS_BOUNDS_BLOCK 1024
typedef struct {
  int64_t n_local;
  const float* mean_opac;
  const float* quat;
  const float* scale;
  const float* sh;
  const uint8_t* lod;
  const float* bounds;
} bgs_gaussians;

/* Gradients w.r.t. the activated parameters, same layouts as bgs_gaussians (device,
 * caller-owned, ACCUMULATED into with +=: the caller zeroes them once per optimizer step).
 * mean_opac row = (dL/dmu_x, dL/dmu_y, dL/dmu_z, dL/do); quat row = dL/d(w,x,y,z);
 * scale row = (dL/ds_x, dL/ds_y, dL/ds_z, 0); sh [n][16][3]. */
typedef struct {
  float* mean_opac;
  float* quat;
  float* scale;
  float* sh;
} bgs_gaussian_grads;

/* Distance-based LOD gate, Eq.4-5 with fallback.
 * keep_lod(i) = l_i <= clamp(round_half_up(log2(d0/|mu_i - c_v|)), 0, l_max)
 * evaluated as l_i == 0 || (l_i <= l_max && d^2 <= D2[l_i]), D2[l] = (d0*2^(1/2-l))^2
 * (reading R18).  When enabled == 0 or fallback_den*|L| > fallback_num*|G^(m)| (R20; 19/20)
 * the whole shard passes.  d0 > 0 world units (R19). */
typedef struct {
  int32_t enabled;
  int32_t l_max;
  double d0;
  int32_t fallback_num;
  int32_t fallback_den;
} bgs_lod_gate;

/* ---------------------------------------------------------------------------------------
 * Context
 * --------------------------------------------------------------------------------------- */
/* 128-byte NCCL unique id for world > 1 (rank 0 creates, caller broadcasts). */
bgs_status bgs_get_unique_id(void* out_128_bytes);
/* One rank of a world-size group.  world == 1: nccl_unique_id may be NULL (no NCCL).
 * world > 1: ncclCommInitRank; must be called concurrently by all ranks.  world <= 8. */
bgs_status bgs_ctx_create(int32_t rank, int32_t world, const void* nccl_unique_id, int32_t device,
                          bgs_ctx** out);
/* An in-process group of `world` contexts on ONE device whose collectives are device-to-device
 * copies (test transport: the M>1 kernels and routing on a single GPU).  Each ctx must then
 * be driven by its own host thread, concurrently.  out: array of `world` ctx pointers. */
bgs_status bgs_ctx_create_local_group(int32_t world, int32_t device, bgs_ctx** out);
bgs_status bgs_ctx_destroy(bgs_ctx* ctx);
const char* bgs_last_error(const bgs_ctx* ctx);
/* Kernels this ctx has launched since creation (the bench's gpu_launches evidence). */
int64_t bgs_launch_count(const bgs_ctx* ctx);
/* Times a call on this ctx blocked the host on the device (stream / event synchronisations inside
 * HOST-SYNC calls) since creation (the bench's host_syncs_per_view evidence). */
int64_t bgs_host_sync_count(const bgs_ctx* ctx);

/* Per-view counters (valid after the producing stage; host-visible after a HOST-SYNC call):
 *   0 N_local  1 n_lod (|L^(m)|)  2 n_active (|A^(m)|)  3 F (in-frustum records)  4 D (records
 *   sent, sum of destination multiplicity)  5 R (records received)  6 P (pairs of owned tiles)
 *   7 tile_begin  8 tile_end (owned run)  9 fallback (0/1)  10 sort passes run  11 P_all
 *   (pairs over all tiles of this rank's splats)  12 width 13 height */
#define BGS_Q_COUNT 14
bgs_status bgs_query(bgs_ctx* ctx, int64_t* out /*[BGS_Q_COUNT] host*/);

/* Borrowed device views of arena intermediates for parity tests (valid until the next call of
 * the producing stage):
 *   0 records [F]x48 B {mx,my,A,B, C,o,r,g, b,depth,gid,rect(x0|y0<<8|x1<<16|y1<<24)}
 *   1 record local index [F] u32       2 received records [R]x48 B (== 0 when world == 1)
 *   3 sorted keys [P] u32 ((tile-tile_begin) << kd | (f32 bits(depth) - lo) >> (nb - kd)), lo =
 *     0xffffffff - counters[6], hi = counters[7] (min / max depth bits of the received records),
 *     nb = bit width of hi - lo, kd = min(nb, 32 - tile bits), tile bits = bit width of
 *     (tile_end - tile_begin - 1); equal keys are ordered by (depth, global id)
 *                                                                     4 sorted values [P] u32
 *     (index into received records)    5 tile ranges [tile_end-tile_begin] uint2 [start,end)
 *   6 per-received-splat accumulators [R]x48 B {m_x, m_y, m_xx, m_xy, m_yy, dL/do, dL/d(r,g,b) f32,
 *     a u32, w_fixed u64}; m_* = sums over pixels of gd*dx, gd*dy, gd*dx^2, gd*dx*dy, gd*dy^2 with
 *     gd = G dL/dalpha, (dx,dy) = mean2d - pixel, so dL/dmx = -o(A m_x + B m_y), dL/dmy =
 *     -o(B m_x + C m_y), dL/dA = -o m_xx/2, dL/dB = -o m_xy, dL/dC = -o m_yy/2 (Eq.2 chain rule)
 *   7 per-local-record owner-summed accumulators [F]x48 B (same layout; == 6 when world == 1)
 *   8 tile owner map [T] i32    9 dest mask [F] u8    10 per-tile pair counts (all ranks) [T] i32
 *   11 device counters [8] u64 (0 F, 1 P_all, 2 n_lod, 3 n_active, 4 P, 5 candidates, 6 and 7 the
 *      depth range of buffer 3) */
/* (synchronizes the ctx's device before answering: a test-only accessor) */
bgs_status bgs_debug_buffer(bgs_ctx* ctx, int32_t which, void** dev_ptr, int64_t* bytes);

/* ---------------------------------------------------------------------------------------
 * Steps
 * --------------------------------------------------------------------------------------- */
/* a1+a2.  cull_column: nullable device u32[ceil(n_local/32)], bit j = Cull_{j,v} (Eq.6).
 * radius_out: device int32[n_local]; 0 when gated, culled, behind near_clip or off-screen
 * (c^rad_{i,v} = radius > 0).  flags: BGS_NO_COLOR.  HOST-SYNC (reads F and P). */
bgs_status bgs_project(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam, const bgs_lod_gate* gate,
                       const uint32_t* cull_column, uint32_t flags, int32_t* radius_out, void* stream);

/* Block bounds for hierarchical culling (a1): for each block of BGS_BOUNDS_BLOCK consecutive rows of
 * the shard, the box of the means and the largest per-axis standard deviation (8 floats, layout in
 * bgs_gaussians.bounds).  bounds_out: device f32 [ceil(n_local / BGS_BOUNDS_BLOCK)][8].  One pass
 * over the means and scales (32 B per row); call after every parameter update (the Z-ordered shard
 * layout of bgs_spatial_order makes the boxes tight). */
bgs_status bgs_shard_bounds(bgs_ctx* ctx, const bgs_gaussians* g, float* bounds_out, void* stream);

/* a3+a4.  Per-tile pair counts are all-reduced, tiles split into contiguous cost-balanced
 * runs (owner(t) = min(M-1, floor((2 P_t + c_t) M / (2 C))), c_t = pairs_t + 1, D6), and
 * every record is sent to each rank owning a tile of its rect in ONE all-to-all.
 * tile_owner_in: nullable device int32[T]; when given it replaces that split (it must be
 * contiguous non-decreasing runs in [0, world), identical on every rank, else
 * BGS_ERR_INVALID_ARGUMENT; the pair counts are still all-reduced for the owners' P).
 * tile_owner_out: nullable device int32[T], the map used.  n_recv_out: nullable host int64, R (the
 * records this rank receives).  World 1: the identity (owner 0 everywhere, R = F).
 * HOST-SYNC (exchange sizes). */
bgs_status bgs_route(bgs_ctx* ctx, const int32_t* tile_owner_in, int32_t* tile_owner_out, int64_t* n_recv_out,
                     void* stream);

/* a5+a6+a7.  Pairs (owned tile, received record) keyed (tile, depth); onesweep LSD radix sort;
 * runs of equal keys ordered by global id (R12); per-tile [start,end) ranges. */
bgs_status bgs_sort_tiles(bgs_ctx* ctx, void* stream);

/* a8.  Writes the OWNED tiles of rgb (device f32 [3][H][W], black background), t_final
 * (device f32 [H][W]) and n_contrib (device i32 [H][W] = 1 + position in the tile list of the
 * last contributor).  flags: BGS_IMPORTANCE (accumulate w_fixed, a per received splat). */
bgs_status bgs_raster_fwd(bgs_ctx* ctx, uint32_t flags, float* rgb, float* t_final, int32_t* n_contrib,
                          void* stream);

/* a9.  dL_drgb: device f32 [3][H][W] (read on owned tiles only).  t_final / n_contrib: the
 * buffers written by the preceding bgs_raster_fwd on this ctx (same view); the backward also
 * reads the per-(8x8 block, 32-entry chunk) contributor masks that forward left in the arena
 * and evaluates only the list entries some pixel of the block composited. */
bgs_status bgs_raster_bwd(bgs_ctx* ctx, const float* dL_drgb, const float* t_final, const int32_t* n_contrib,
                          void* stream);

/* a10.  Returns per-received-splat partials (9 grads + w_fixed + a, 48 B) to the source ranks along
 * the transposed counts of a4 and sums them per local record in destination-rank order.
 * flags: BGS_IMPORTANCE_ONLY sends (w_fixed, a) only, 12 B per record (the instrumented scoring
 * pass "bypasses color shading" and has no backward); the gradients are then zero. */
bgs_status bgs_route_reverse(bgs_ctx* ctx, uint32_t flags, void* stream);

/* a11.  grads += d(loss)/d(activated params) for every projected local Gaussian.  Reads the colour
 * Jacobian along the view direction that a2 left in the arena, so the projection of this view must
 * not have used BGS_NO_COLOR (BGS_ERR_CONTRACT otherwise). */
bgs_status bgs_project_bwd(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam,
                           const bgs_gaussian_grads* grads, void* stream);

/* a12.  Eq.3 score and visibility bits for this view, selection GLOBAL over ranks.
 * radius: device i32[n_local] from bgs_project.  w_fixed / a: nullable device u64 / u32
 * [n_local]; when NULL the ctx's reverse-routed per-record values of this view are used.
 * s (f64), c_rad, c_vis (u32): device [n_local], accumulated.  cull_out: device
 * u32[ceil(n_local/32)], overwritten: bit j = 1 - c^vis_{j,v}.  Top set: smallest
 * prefix of (w desc, global id asc) with mass_den*prefix >= mass_num*total (99/100, R16). */
bgs_status bgs_importance(bgs_ctx* ctx, int64_t n_local, const int32_t* radius, const uint64_t* w_fixed,
                          const uint32_t* a, int32_t mass_num, int32_t mass_den, double* s, uint32_t* c_rad,
                          uint32_t* c_vis, uint32_t* cull_out, void* stream);

/* a1..a11 in one call (a12 too when importance != NULL).  The per-view image gradient comes
 * from the caller (the loss of Eq.7 is outside the hot path). */
typedef struct {
  double* s;
  uint32_t* c_rad;
  uint32_t* c_vis;
  uint32_t* cull_out;
  int32_t mass_num, mass_den;
} bgs_importance_out;

bgs_status bgs_view_step(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam, const bgs_lod_gate* gate,
                         const uint32_t* cull_column, uint32_t flags, int32_t* radius_out, float* rgb,
                         float* t_final, int32_t* n_contrib, const float* dL_drgb, const bgs_gaussian_grads* grads,
                         const bgs_importance_out* importance, void* stream);

/* Same with the per-view I/O in HOST memory (end-to-end path): dL_drgb_host (f32 [3][H][W])
 * is copied to the device and rgb_host (f32 [3][H][W], owned tiles) back, inside the call.
 * Scratch device images live in the arena.  Host buffers should be pinned. */
bgs_status bgs_view_step_host(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam,
                              const bgs_lod_gate* gate, const uint32_t* cull_column, uint32_t flags,
                              int32_t* radius_out, const float* dL_drgb_host, float* rgb_host,
                              const bgs_gaussian_grads* grads, const bgs_importance_out* importance, void* stream);
/* Non-blocking form: returns once everything is enqueued.  The upload runs on a ctx-owned copy
 * stream and only the compositing backward waits for it; the image is downloaded on a second copy
 * stream as soon as the forward is done (overlapping the backward).  rgb_host is valid, and
 * dL_drgb_host may be reused, after `stream` is synchronised (the call makes `stream` wait for
 * both copies).  Several ctxs on several streams keep several views (and their copies) in flight. */
bgs_status bgs_view_step_host_async(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam,
                                    const bgs_lod_gate* gate, const uint32_t* cull_column, uint32_t flags,
                                    int32_t* radius_out, const float* dL_drgb_host, float* rgb_host,
                                    const bgs_gaussian_grads* grads, const bgs_importance_out* importance,
                                    void* stream);

/* Per-stage device timing of bgs_view_step / bgs_train_view_step: when enabled, CUDA events are
 * recorded on the working stream between its stages; bgs_stage_times waits for the last one and
 * writes the elapsed ms of the most recent step: [project, route, sort, raster_fwd, loss,
 * raster_bwd, route_reverse, project_bwd, importance] (ms_out host f32 [9]; loss is ~0 without
 * supervision). */
bgs_status bgs_set_stage_timing(bgs_ctx* ctx, int32_t enable);
bgs_status bgs_stage_times(bgs_ctx* ctx, float* ms_out);

/* ---------------------------------------------------------------------------------------
 * Shard layout (not a step of the method; a one-time data-layout utility)
 * --------------------------------------------------------------------------------------- */
/* Z-order (Morton) permutation of a shard: perm_out[new] = old local index, from 16-bit-per-axis
 * codes of mu over the shard's bounding box, sorted with the library's onesweep (ties keep index
 * order).  The caller applies it to every per-Gaussian array (parameters, optimizer state) and
 * relabels: after reordering, local j of rank m is global id j*world + m again (ids are labels;
 * the paper renumbers on redistribution).  Spatially coherent shards make the
 * per-view gathers of 16-B rows touch whole DRAM granules.  mean_opac: device float4[n];
 * perm_out: device u32[n].  Invalidates the ctx's current view.  HOST-SYNC. */
bgs_status bgs_spatial_order(bgs_ctx* ctx, const float* mean_opac, int64_t n, uint32_t* perm_out, void* stream);

/* ---------------------------------------------------------------------------------------
 * NEXT-1: the scoring report's phi and the scheduled simplification
 * (readings R30-R33).  s / c_rad / c_vis are the
 * per-Gaussian outputs accumulated by bgs_importance over a V-view sweep.  Every selection is
 * GLOBAL over the ranks of the ctx and bit-identical for any M.
 * --------------------------------------------------------------------------------------- */

/* Output shard of bgs_redistribute: device arrays with room for `capacity` rows each, layouts
 * as bgs_gaussians (lod nullable). */
typedef struct {
  int64_t capacity;
  float* mean_opac;
  float* quat;
  float* scale;
  float* sh;
  uint8_t* lod;
} bgs_gaussians_out;

/* phi_i = c_vis_i / (c_rad_i + 1e-8) (fp64).  c_rad, c_vis: device u32 [n_local];
 * phi: device f64 [n_local]. */
bgs_status bgs_score_phi(bgs_ctx* ctx, int64_t n_local, const uint32_t* c_rad, const uint32_t* c_vis, double* phi,
                         void* stream);

/* Pass 1, stochastic importance-weighted sampling without replacement:
 * keep_out[i] = 1 for the keep_count Gaussians (counted over ALL ranks) with the largest
 * exponential-race keys ln(u)/s (u from (seed, global id); s = 0 -> -inf; ties by global id;
 * R30).  keep_count <= 0 keeps nothing, >= the global population keeps all.  s: device f64
 * [n_local]; keep_out: device u8 [n_local].  HOST-SYNC. */
bgs_status bgs_prune_stochastic(bgs_ctx* ctx, int64_t n_local, const double* s, int64_t keep_count, uint64_t seed,
                                uint8_t* keep_out, void* stream);

/* Pass 2, deterministic cumulative-mass cut: keep the smallest prefix of
 * (floor(s 2^24) desc, global id asc) whose mass reaches num/den of the global total (R31);
 * num == den keeps exactly the s > 0 set.  All-zero scores keep only global id 0 and set
 * *all_zero_out (host, nullable) to 1.  0 < num <= den.  HOST-SYNC. */
bgs_status bgs_prune_mass_cut(bgs_ctx* ctx, int64_t n_local, const double* s, int32_t num, int32_t den,
                              uint8_t* keep_out, int32_t* all_zero_out, void* stream);

/* Every rank's shard size (sizes_out: host int64 [world]) for a skew policy ("an
 * index-parity redistribution rebalances shard sizes across GPUs once the per-GPU skew exceeds a
 * fixed threshold"; the threshold is the caller's).  HOST-SYNC. */
bgs_status bgs_shard_sizes(bgs_ctx* ctx, int64_t n_local, int64_t* sizes_out);

/* Index-parity redistribution of the survivors (R33): rows with keep[i] != 0 are
 * renumbered densely in global-id order (new gid), sent to rank new_gid mod M and stored at
 * local index new_gid div M of `out` (exact copies).  Shards may be unequal (after density
 * control): the global order is gid = j M + m over slices padded to the largest shard.  To
 * carry Adam moments, call again with the moment planes in place of the parameter planes and
 * the same keep mask (the renumbering is deterministic).  *n_out (host) = this rank's new shard
 * size; BGS_ERR_CAPACITY when it exceeds out->capacity.  out must not alias in.  HOST-SYNC. */
bgs_status bgs_redistribute(bgs_ctx* ctx, const bgs_gaussians* in, const uint8_t* keep, const bgs_gaussians_out* out,
                            int64_t* n_out, void* stream);

/* ---------------------------------------------------------------------------------------
 * NEXT-4 supervision: the loss of Eq.7-8 on the owned tiles
 * --------------------------------------------------------------------------------------- */
/* Eq.7 photometric term of one view, fused with its gradient.  Call after
 * bgs_raster_fwd of the view on this ctx (ownership and camera of that view).
 * l_v = (1 - lambda) mean|rgb - target| + lambda (1 - SSIM(rgb, target)), means over the 3 H W
 * elements; SSIM per channel with the 11x11 Gaussian window (sigma 1.5, normalised), zero
 * padding, C1 = 0.01^2, C2 = 0.03^2 (reading R34).  rgb: device f32 [3][H][W] as written by
 * bgs_raster_fwd (owned tiles valid; at world > 1 the owned pixels of every rank are summed
 * into one full image first so that windows straddling ownership boundaries see the same
 * pixels as on one GPU).  target: device f32 [3][H][W] (read on the owned tiles + 10 px).
 * dL_drgb: device f32 [3][H][W], OVERWRITTEN on the owned tiles with
 * batch_inv * dl_v/drgb (batch_inv = 1/B of Eq.7; sign(0) = 0 for the L1 term).
 * out: device f64 [3], overwritten with {l_v, L1_v, SSIM_v} (global over ranks; not scaled by
 * batch_inv).  0 <= lambda <= 1. */
bgs_status bgs_loss_photo(bgs_ctx* ctx, const float* rgb, const float* target, float lambda, float batch_inv,
                          float* dL_drgb, double* out, void* stream);

/* Eq.8 scale regulariser of one view: L_scale = (1/|V|) sum_{i in V} min_j s_ij,
 * V = the Gaussians with radius > 0 in the view last projected on this ctx (bgs_project's
 * records), over ALL ranks; grads->scale[i][argmin_j s_ij] += beta / |V| for the visible local
 * Gaussians (first axis among equal minima, R35; beta includes the caller's 1/B).  g: the shard
 * that view was projected from.  out: device f64 [2], overwritten with {L_scale, |V|}; |V| = 0
 * gives L_scale = 0 and no gradient. */
bgs_status bgs_loss_scale(bgs_ctx* ctx, const bgs_gaussians* g, float beta, const bgs_gaussian_grads* grads,
                          double* out, void* stream);

/* a1..a12 with supervision (NEXT-4): after the forward, Eq.7 on the owned tiles writes
 * this view's dL/dC into dL_scratch (device f32 [3][H][W]) and Eq.8 adds to grads->scale
 * (beta != 0; needs grads); the backward then runs on that dL/dC. */
typedef struct {
  const float* target;  /* device f32 [3][H][W], the view's ground-truth image I_b */
  float lambda;         /* Eq.7 blend, [0, 1] */
  float batch_inv;      /* 1/B of Eq.7 */
  float beta;           /* Eq.8 weight including the caller's 1/B; 0 skips Eq.8 */
  double* loss_out;     /* device f64 [5], overwritten: {l_v, L1_v, SSIM_v, L_scale, |V|} */
} bgs_supervision;

bgs_status bgs_train_view_step(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam, const bgs_lod_gate* gate,
                               const uint32_t* cull_column, uint32_t flags, int32_t* radius_out,
                               const bgs_supervision* sup, float* rgb, float* t_final, int32_t* n_contrib,
                               float* dL_scratch, const bgs_gaussian_grads* grads, const bgs_importance_out* importance,
                               void* stream);

/* The same step from host buffers, asynchronous like bgs_view_step_host_async: target_host
 * (f32 [3][H][W], pinned for overlap) is uploaded on a ctx-owned copy stream that the loss waits
 * for; the five loss values (as loss_out above) are downloaded to loss_host (f64 [5], pinned)
 * as soon as the loss is final, overlapping the backward.  A later sync of `stream` covers
 * loss_host. */
bgs_status bgs_train_view_step_host_async(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam,
                                          const bgs_lod_gate* gate, const uint32_t* cull_column, uint32_t flags,
                                          int32_t* radius_out, const float* target_host, float lambda,
                                          float batch_inv, float beta, double* loss_host,
                                          const bgs_gaussian_grads* grads, const bgs_importance_out* importance,
                                          void* stream);

/* ---- NEXT-2: the batched step ("a mini-batch of B cameras") ----
 * One view of a batch: the camera by value and the caller's per-view device buffers (as for
 * bgs_view_step).  cull_column and dL_drgb are nullable (no Cull column / forward only). */
typedef struct {
  bgs_camera cam;
  const uint32_t* cull_column;
  int32_t* radius_out;  /* device i32 [n_local] */
  float* rgb;           /* device f32 [3][H][W] (owned tiles written) */
  float* t_final;       /* device f32 [H][W] */
  int32_t* n_contrib;   /* device i32 [H][W] */
  const float* dL_drgb; /* device f32 [3][H][W] or NULL */
  uint32_t* cull_out;   /* device u32 [ceil(n_local/32)]: this view's Cull column (a12), or NULL (not kept) */
  const bgs_supervision* sup; /* host struct or NULL: supervised view (Eq.7-8 as bgs_train_view_step;
                                 dL_drgb is then ignored and dL_scratch receives this view's dL/dC) */
  float* dL_scratch;          /* device f32 [3][H][W], required with sup */
} bgs_batch_view;

#define BGS_GRAPH 4u /* bgs_batch_step: record the post-sizing part of the batch as one CUDA graph */

/* a1..a11 (+ a12 when importance != NULL) for n_views (1..16) views in ONE call.  Each view runs on
 * an internal view slot (own arena and stream, forked from / joined back into `stream`), so the
 * views of the batch overlap.  The host reads sizes ONCE per batch (HOST-SYNC once: every view's
 * projection counters and, at world > 1, the exchanged per-destination counts); at world > 1 the
 * batch issues ONE all-reduce of the B x T tile pair counts, ONE exchange of the B x M counts, ONE
 * grouped all-to-all of all views' records and ONE reverse all-to-all (+ a12's rounds per view)
 * instead of four collectives per view.  Views must share the image size, and each view needs its own
 * radius / rgb / t_final / n_contrib (/ cull_out, dL_scratch) buffers: the views run concurrently.  Results equal B
 * bgs_view_step calls (pixels, n_contrib, w, a, routing bit-identical; gradients up to fp32 atomic
 * order).  grads and importance's s, c_rad, c_vis are accumulated by every view (reductions); each
 * view's Cull column goes to its own cull_out (importance->cull_out is not used).  flags:
 * BGS_NO_COLOR, BGS_GRAPH (world 1; ignored at world > 1: everything after the host read is
 * captured into a CUDA graph, its executable updated in place each batch and launched once; when an
 * arena must grow the batch runs eagerly instead and the next one is captured).  The views' intermediates stay in
 * the slots until the next batch (bgs_batch_view_ctx). */
bgs_status bgs_batch_step(bgs_ctx* ctx, int32_t n_views, const bgs_gaussians* g, const bgs_lod_gate* gate,
                          uint32_t flags, const bgs_batch_view* views, const bgs_gaussian_grads* grads,
                          const bgs_importance_out* importance, void* stream);
/* Borrowed handle of view slot b of the last batch: bgs_query / bgs_debug_buffer on that view, and
 * bgs_densify_accumulate of that view (on the batch's stream, before the next batch); valid until
 * ctx is destroyed; must not be passed to any other call (nor destroyed). */
bgs_status bgs_batch_view_ctx(bgs_ctx* ctx, int32_t b, bgs_ctx** out);
/* out (host i64 [6]): host syncs, collectives issued, batches, graph launches, graph
 * instantiations, graph captures abandoned (eager fallback), all since ctx creation. */
bgs_status bgs_batch_stats(bgs_ctx* ctx, int64_t* out);


/* ---------------------------------------------------------------------------------------
 * NEXT-3: optimizer step on the owned shard ("each GPU stores only its
 * local shard and its optimizer state")
 * --------------------------------------------------------------------------------------- */
/* RAW (pre-activation) parameters of the local shard and their Adam moments, device, n_local
 * rows each, layouts as bgs_gaussians: mean_logit float4 (mu_x, mu_y, mu_z, opacity logit),
 * quat_raw float4 (w, x, y, z, any non-zero norm), log_scale float4 (log s_x, log s_y, log s_z, 0),
 * sh [n][48].  m[k] / v[k]: first / second moments of plane k (0 mean_logit, 1 quat_raw,
 * 2 log_scale, 3 sh), same layouts. */
typedef struct {
  int64_t n_local;
  float* mean_logit;
  float* quat_raw;
  float* log_scale;
  float* sh;
  float* m[4];
  float* v[4];
} bgs_train_params;

/* Adam hyper-parameters (reading R38: the 3DGS parameter groups; values are the caller's).
 * step = t >= 1 (bias corrections 1 - beta^t). */
typedef struct {
  float lr_mean, lr_opacity, lr_quat, lr_scale, lr_sh_dc, lr_sh_rest;
  double beta1, beta2, eps;  /* double: 1 - beta and the bias corrections are formed on the host */
  int32_t step;
} bgs_adam_hparams;

/* One fused optimizer step over the shard: grads (w.r.t. the ACTIVATED parameters, as the view
 * steps accumulate them) -> chain rule through opacity = sigmoid(logit), s = exp(log s),
 * q = q_raw/|q_raw| (mean and SH identity) -> Adam m, v, bias-corrected update of the raw
 * parameters -> activated planes written to act (mean_opac, quat, scale; act->sh may equal
 * p->sh, else the SH rows are copied; act->lod untouched) -> grads ZEROED for the next step.
 * visible: nullable device u32[ceil(n/32)] bit mask; rows with bit 0 are not read or written
 * (selective Adam); NULL updates every row (standard Adam). */
bgs_status bgs_adam_step(bgs_ctx* ctx, const bgs_train_params* p, const bgs_gaussian_grads* grads,
                         const bgs_gaussians_out* act, const uint32_t* visible, const bgs_adam_hparams* h,
                         void* stream);

/* Selective-Adam visibility mask of a batch (3DGS "visibility filter"; P:342 B views per step):
 * mask[i/32] |= bit (i%32) for every local Gaussian with radius[i] > 0 (bgs_project's radius_out of
 * one view of the batch).  radius: device i32 [n_local]; mask: device u32 [ceil(n_local/32)],
 * caller-zeroed once per batch, ORed with atomics (views in flight may share it). */
bgs_status bgs_visibility_mask(bgs_ctx* ctx, int64_t n_local, const int32_t* radius, uint32_t* mask, void* stream);

/* Density-control statistic of one view (R37): after bgs_route_reverse of the view on
 * this ctx, for every local Gaussian the view projected (radius > 0):
 *   stat[i] += phi_i * |(dL/dmx * W/2, dL/dmy * H/2)|,  count[i] += 1
 * (dL/dmean2d from the owner-summed compositing partials, in NDC units as the 3DGS view-space
 * statistic).  phi: nullable device f64 [n_local] (bgs_score_phi; NULL = 1).  stat: device f32,
 * count: device u32 [n_local], accumulated with reductions (views in flight may share them). */
bgs_status bgs_densify_accumulate(bgs_ctx* ctx, int64_t n_local, const double* phi, float* stat, uint32_t* count,
                                  void* stream);

/* Density-control thresholds (R39, R40; values are the caller's).  The decisions
 * are taken in fp32 as l < logit(min_opacity), max_j log s_ij > log(dense_extent) (thresholds
 * rounded once from double) and stat / max(1, count) >= grad_threshold. */
typedef struct {
  float grad_threshold;  /* tau on stat / max(1, count) (3DGS: 2e-4) */
  float dense_extent;    /* percent_dense * scene extent: clone if max_j s_ij <= this, else split */
  float min_opacity;     /* prune rows with opacity below this (3DGS: 0.005) */
  float split_div;       /* split children scale = s / split_div (3DGS: 1.6) */
  uint64_t seed;         /* split samples: z = N(0, I) of (seed, parent global id, child, axis) */
  int32_t k_levels;      /* K, the number of LOD levels (1..256): a split child's level is
                            min(parent level + 1, K - 1) (heritage rule; S:374, S:379 keep l in [0, K-1]) */
} bgs_densify_params;

/* Clone / split / prune the local shard ("clones, splits, and prunes"; heritage rule P:194:
 * clone keeps the level, split increments it).  in: the shard's raw parameters and Adam moments
 * (bgs_train_params), lod_in u8 [n]; stat / count from bgs_densify_accumulate.  out: raw planes
 * and moments of the new shard, out->n_local = CAPACITY in rows; lod_out u8 [capacity]; act_out
 * (nullable): activated planes of the new shard (act_out->sh may equal out->sh).  Order: kept
 * originals (input order), clones (parent order), first then second children of split parents;
 * moments copied for originals, zero for new rows; clones keep the parent's level, split children get
 * min(level + 1, K - 1).  *n_out (host) = new row count;
 * BGS_ERR_CAPACITY (nothing written) when it exceeds the capacity.  out must not alias in.  The
 * caller re-zeros stat / count for the new shard.  Global ids are j*M + rank as before; a
 * skew-triggered bgs_redistribute can follow.  HOST-SYNC. */
bgs_status bgs_densify_apply(bgs_ctx* ctx, const bgs_train_params* in, const uint8_t* lod_in, const float* stat,
                             const uint32_t* count, const bgs_densify_params* dp, const bgs_train_params* out,
                             uint8_t* lod_out, const bgs_gaussians_out* act_out, int64_t* n_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BGS_H_ */
