/* include/tabi.h -- C ABI of the B200-native TABI atlas packer.
 *
 * TABI = "Tight And Balanced Interactive" atlas packing, arxiv 2602.07782
 * (/root/reference/PAPER.md, cited "P:<line>").  One call packs N charts into a
 * fixed W x H atlas with minimal downscaling, following the paper's problem
 * statement: "Our input consists of a set of 2D charts ... provided
 * as polygonal meshes with coordinates defined in texel space ... Our
 * algorithm outputs per-chart scales and rigid transformations (translation,
 * rotation, and/or reflection) that arrange the charts inside the atlas with
 * no overlaps between the charts or their gutters."
 *
 * Every stage (proxies, sort, profiles, compaction, balanced fold-and-push,
 * scale search) runs as hand-written sm_100a CUDA kernels on one GPU; there is
 * no CPU fallback.  No C++ or torch types cross this boundary.
 */
#ifndef TABI_H
#define TABI_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TABI_ABI_VERSION 1
#define TABI_MAX_LOCAL_AABBS 64   /* k upper bound (quality knob) */
#define TABI_MAX_SCALES 256       /* M upper bound (paper: 64)    */
#define TABI_MAX_ATLAS_SIDE 16384

typedef enum {
  TABI_OK = 0,
  TABI_EINVAL = 1,      /* bad spec or chart (info->bad_chart names the chart) */
  TABI_NO_FIT = 2,      /* no candidate scale packs: out untouched     */
  TABI_ECUDA = 3,       /* CUDA runtime failure; see tabi_last_error()         */
  TABI_ECAPACITY = 4,   /* input larger than the context was created for      */
  TABI_PENDING = 5      /* tabi_pack_query: the asynchronous pack is still running */
} tabi_status;

enum {
  TABI_F_NO_HC = 1u,                 /* ablation: never compact horizontally */
  TABI_F_NO_BALANCE = 2u,            /* ablation: no knees, static L/R alternation    */
  TABI_F_ADJACENT_LOCKS_ONLY = 4u,   /* paper-literal Alg. 1 (adjacent pairs only)    */
  TABI_F_PREROTATE = 8u,             /* UV pre-rotation to the OBB angle (for UV
                                        charts, not TSS -- rotation by non-90-degree angles
                                        resamples the texture); see tabi_placement step 0 */
  TABI_F_NO_OBB = 16u,               /* ablation: no OBB bound on the footprints (D6/D11);
                                        with local_aabb_count = 1 the proxy is the plain AABB
                                        (Chameleon / balanced-only) */
  TABI_F_EXACT_TAIL = 32u            /* hybrid tail variant (DESIGN R6): the tail is
                                        folded exactly by Alg. 3 with compaction at m/M -- no
                                        intermediate downscale; tail charts keep scale m/M */
};

typedef struct tabi_ctx tabi_ctx;    /* opaque: device workspace + stream, one per host thread */

/* Atlas + knobs (SPEC AtlasSpec S:33-36).  Invariants, else TABI_EINVAL:
 *   1 <= atlas_w, atlas_h <= 16384;  0 <= gutter <= 64;  1 <= scale_count <= 256;
 *   1 <= local_aabb_count <= 64;  -1 <= t_opt_bp <= 10000;  flags in TABI_F_* (0..63). */
typedef struct {
  int32_t atlas_w, atlas_h;   /* texels */
  int32_t gutter;             /* texels around every chart, none at atlas edges; paper 1 */
  int32_t scale_count;        /* M: candidates s = m/M, m = 1..M; paper 64 */
  int32_t local_aabb_count;   /* k local AABBs per axis; paper 10 */
  int32_t t_opt_bp;           /* prefix-tail threshold, basis points of atlas_h;
                                 -1 = paper policy (0 if N <= 10000 else 100).
                                 > 0: hybrid mode -- a candidate switches to
                                 prefix (FastAtlas) rows once no knee is pending and the
                                 tallest chart of the next row is below t_opt * H; the
                                 tail's scale is re-solved for sigma <= 1 (R3). */
  uint32_t flags;             /* TABI_F_* */
} tabi_spec;

/* Per-chart output, 32 bytes, indexed by INPUT chart order.
 * Transform of an input vertex p = (x, y) * (res_x, res_y) (texels), exact in
 * 1/256-texel units (q = round_half_even(256 * p)):
 *   0. if prerot = j > 0 (TABI_F_PREROTATE): q <- (round_half_even((qx C + qy S) / 2^30),
 *      round_half_even((-qx S + qy C) / 2^30)) with (C, S) the Q30 cos / sin of j pi / 16
 *      (the chart's minimum-area OBB angle, D6) -- its OBB becomes axis-aligned
 *   1. u = qx - min_qx, v = qy - min_qy           (chart AABB to the origin)
 *   2. if rot90:  (u, v) <- (h' - v, u)           (h' = the original AABB height;
 *                                                   the chart becomes taller than wide)
 *   3. if flip_x: u <- w - u ; if flip_y: v <- h - v   (orientation; w, h posed extents)
 *   4. (u, v) <- (u, v) * scale_num / (scale_den * 256)                 (texels)
 *   5. if mirror_x: u <- box_w - u   (right-to-left row, "Reflect charts")
 *   6. atlas position = (tx + u, ty + v)
 * box_w = ceil(w * scale), box_h = ceil(h * scale) in texels (the integer box
 * the mirror of step 5 is taken about). */
typedef struct {
  int32_t tx, ty;
  int32_t scale_num, scale_den;   /* scale = scale_num / scale_den = m / M */
  int32_t box_w, box_h;
  uint8_t rot90, flip_x, flip_y, mirror_x;
  uint8_t mode;                   /* 0 = sequential row, 1 = hybrid-tail row: prefix rows
                                     at scale p / 2^20, or exact rows at m / M
                                     under TABI_F_EXACT_TAIL (R6) */
  uint8_t prerot;                 /* pre-rotation angle index j (step 0), 0 = none */
  uint8_t pad[2];
} tabi_placement;

typedef struct {
  int32_t scale_index;            /* winning m (0 on NO_FIT) */
  int32_t fused;                  /* 1: waves ran as one fused persistent kernel (stages
                                     [3] and [4] are then inside [5]); 0: split kernels */
  double l2_stretch;             /* Sander L2 stretch of the packed->input map; M/m */
  int32_t rows, knees_found, knee_rows, prefix_rows;   /* winner's statistics */
  int32_t bad_chart;              /* first offending chart on EINVAL, else -1 */
  int32_t gpu_launches;           /* kernels launched by this call */
  float stage_ms[8];              /* per-stage device time if TABI_TIMING=1, else 0:
                                     [0] H2D [1] proxies [2] sort [3] profiles
                                     [4] offsets+locks [5] fold&push [6] select [7] D2H */
  int64_t work_pack;              /* fold&push: frontline column visits, all candidates
                                     (push + score per evaluated configuration, + commit) */
  int64_t work_profile;           /* footprint entries evaluated, sum over m, s of Wd + Hd */
  float device_ms;                /* device time of this call on its stream (CUDA events):
                                     from the first enqueued operation to the last copy of
                                     the last wave, host-side call overhead excluded */
  int32_t reserved;
} tabi_info;

/* Create a context on `cuda_device`.  max_charts / max_vertices bound every
 * later call (TABI_ECAPACITY beyond them); device workspace is linear in
 * max_charts ("memory consumption ... linear in the number of charts")
 * and grows on demand for the per-candidate footprint buffers.
 * Returns TABI_ECUDA if the device cannot be initialised. */
tabi_status tabi_ctx_create(tabi_ctx** out, int cuda_device, int32_t max_charts,
                            int64_t max_vertices, int32_t max_atlas_side);
void tabi_ctx_destroy(tabi_ctx* ctx);

/* Pack n_charts charts.
 *   xy          2*V floats x0,y0,x1,y1,... ; chart c owns vertices
 *               [chart_start[c], chart_start[c+1]); one closed outline per chart,
 *               either winding, >= 3 vertices, non-zero area after snapping,
 *               |coordinate * res| * 256 <= 2^24.
 *   chart_start n_charts + 1 int32, chart_start[0] = 0, non-decreasing.
 *   res_x/res_y multiply x/y (texel resolution of UV input; 1 if already texels).
 *   on_device   0: xy, chart_start, out are host pointers; the call copies in, runs,
 *               copies out and returns when `out`/`info` are final.
 *               1: xy, chart_start, out are device pointers; the call still returns
 *               after completion (info needs the winner) but does no bulk copies
 *               (tabi_pack_async returns after enqueueing).
 * The whole scale search (every candidate wave) is one CUDA-graph launch with a
 * device-side wave loop and a single host synchronisation.
 *   stream      cudaStream_t to run on, or NULL for the context's own (non-blocking)
 *               stream; cudaStreamLegacy orders the call with the legacy default stream.
 * Ownership: the caller owns every pointer; nothing is retained after return.
 * Deterministic: identical inputs give bit-identical outputs. */
tabi_status tabi_pack(tabi_ctx* ctx, const float* xy, const int32_t* chart_start,
                      int32_t n_charts, float res_x, float res_y, const tabi_spec* spec,
                      tabi_placement* out, tabi_info* info, int on_device, void* stream);

/* Asynchronous pack (SURVEY §8(b) "returns after enqueueing, completion is
 * stream-ordered"): the same pack as tabi_pack with on_device = 1, enqueued on
 * `stream` as ONE CUDA graph launch -- the proxies, the sort, every candidate
 * wave of the scale search (a WHILE node whose body ends in a device-side
 * decision, so no host round trip between waves) and the result copy --
 * and returns without waiting.  xy, chart_start and out are device pointers;
 * the caller keeps them valid and unmodified until tabi_pack_wait returns.
 * `out` is final once the stream passes the pack (when the pack succeeds);
 * status and statistics come from tabi_pack_wait.  One pack per context may be
 * in flight; use several contexts to overlap packs.  Errors found before
 * enqueueing (bad spec, capacity, CUDA) are returned at once and nothing is
 * pending; TABI_EINVAL also if TABI_GRAPH=0 or TABI_TIMING=1 is set. */
tabi_status tabi_pack_async(tabi_ctx* ctx, const float* xy, const int32_t* chart_start,
                            int32_t n_charts, float res_x, float res_y, const tabi_spec* spec,
                            tabi_placement* out, void* stream);
/* Wait for the context's pending asynchronous pack and return its status
 * (TABI_OK, TABI_NO_FIT, TABI_EINVAL with info->bad_chart, ...) with `info` as
 * tabi_pack fills it.  If the device-side capacity check failed (footprint
 * slots or lock-pair lists larger than the context's buffers), the buffers grow
 * and the pack re-runs synchronously from the same arguments.  TABI_EINVAL if
 * nothing is pending. */
tabi_status tabi_pack_wait(tabi_ctx* ctx, tabi_info* info);
/* Non-blocking completion check of the pending asynchronous pack: TABI_PENDING
 * while its device work runs, TABI_OK once tabi_pack_wait would not block,
 * TABI_EINVAL if nothing is pending, TABI_ECUDA on a device error. */
tabi_status tabi_pack_query(tabi_ctx* ctx);

const char* tabi_status_str(tabi_status s);
const char* tabi_last_error(tabi_ctx* ctx);   /* last CUDA error text, or "" */

/* ---- many independent atlases on ONE GPU as one device pipeline ----
 * SURVEY §3(iii) / §8(e); "one work group per scale factor" is the unit
 * of work.  The atlases' charts are stored back to back:
 *   xy           all outlines, 2*V floats;
 *   chart_start  N + 1 int32 GLOBAL vertex offsets into xy (chart_start[0] = 0),
 *                N = atlas_start[n_atlases]; chart c owns [chart_start[c], chart_start[c+1]);
 *   atlas_start  n_atlases + 1 int32 chart offsets (HOST pointer always): atlas a owns the
 *                global charts [atlas_start[a], atlas_start[a+1]); chart indices in
 *                infos[a].bad_chart are atlas-local;
 *   res_xy       2 * n_atlases floats (host) or NULL (1, 1 for every atlas);
 *   spec         one spec for every atlas;
 *   out          N placements, global chart order (host or device, as on_device);
 *                entries of an atlas whose status is not TABI_OK are unspecified;
 *   infos        n_atlases entries or NULL (scale_index, l2_stretch, rows, knees,
 *                bad_chart as for tabi_pack; stage_ms / device_ms are 0);
 *   atlas_status n_atlases tabi_status or NULL;
 *   binfo        batch totals or NULL.
 * Pipeline (one stream, 4 kernels, one sync): batched proxies over every chart
 * -> one CTA per atlas for its sort + slot layout -> a persistent kernel whose
 * CTAs take (atlas, candidate) items from a device work queue: each item
 * rasterizes the atlas's footprints at that scale, computes its pair offsets
 * and runs Alg. 4 in the CTA's own buffers; a failed candidate queues the next
 * lower scale, a success writes the atlas's placements.  The candidates of one
 * atlas are evaluated top-down from its area bound, so the result of every
 * atlas is bit-identical to tabi_pack's.  Atlases with more than 2048 charts,
 * with a hybrid tail (t_opt resolving to > 0), or that overflow the batch's
 * per-CTA buffers are packed afterwards by tabi_pack on the same context
 * (binfo->solo_atlases counts them; the context's max_charts / max_vertices
 * must cover them).  Workspace grows to the largest batch seen.
 * Returns TABI_OK if every atlas is OK or NO_FIT, else the first other error
 * (per-atlas detail in atlas_status). */
typedef struct {
  float device_ms;                /* batch device span on the stream (CUDA events): first
                                     enqueued copy .. last result copy */
  float stage_ms[4];              /* TABI_TIMING=1 only (else 0): [0] input copies + reset,
                                     [1] proxies, [2] sort + slot layout, [3] pack kernel */
  int32_t gpu_launches;           /* kernels launched (batch + solo packs) */
  int32_t candidates_evaluated;   /* (atlas, candidate) items run by the batch kernel */
  int32_t batched_atlases;        /* atlases packed by the device batch */
  int32_t solo_atlases;           /* atlases packed by tabi_pack afterwards */
  int64_t work_pack;              /* batch kernel: frontline column visits (as tabi_info) */
  int64_t work_profile;           /* batch kernel: footprint entries rasterized (Wd + Hd) */
  int64_t cycles[3];              /* batch kernel: SM cycles summed over its items, in
                                     footprint rasterization, pair offsets + locks, Alg. 4 */
  float tail_ms;                  /* batch kernel load balance: time from the median CTA's
                                     last item end to the last CTA's */
  float busy_frac;                /* mean over CTAs of (last item end - start) / kernel span */
  int32_t ranks_in_flight;        /* candidate ranks of one atlas evaluated at once (K >= 1:
                                     more when the batch has few atlases for the GPU) */
  int32_t reserved;
} tabi_batch_info;

tabi_status tabi_pack_many(tabi_ctx* ctx, int32_t n_atlases, const float* xy,
                           const int32_t* chart_start, const int32_t* atlas_start,
                           const float* res_xy, const tabi_spec* spec, tabi_placement* out,
                           tabi_info* infos, int32_t* atlas_status, tabi_batch_info* binfo,
                           int on_device, void* stream);

/* ---- batches of independent atlases over several GPUs ----
 * A single pack never shards; a batch shards by atlas.  tabi_shard_plan
 * assigns atlas i to GPU assignment[i] by LPT (longest processing time first):
 * atlases sorted by estimated cost n*(1 + log2 n) descending (ties by index),
 * each to the currently least-loaded GPU (ties to the lowest GPU index).
 * Deterministic; pure host code.  Returns TABI_EINVAL on bad arguments. */
tabi_status tabi_shard_plan(int32_t n_atlases, const int32_t* n_charts, int32_t n_gpus,
                            int32_t* assignment);
/* Pack n_atlases atlases (host pointers) on n_gpus contexts, one host thread
 * per context, atlases assigned by tabi_shard_plan.  out[i] / infos[i] receive
 * atlas i's placements / info.  Returns TABI_OK if every atlas packed or hit
 * NO_FIT (see infos[i].scale_index == 0), else the first other error.  There is
 * no inter-GPU communication: results land in the caller's host buffers. */
tabi_status tabi_pack_batch(tabi_ctx* const* ctxs, int32_t n_gpus, int32_t n_atlases,
                            const float* const* xy, const int32_t* const* chart_start,
                            const int32_t* n_charts, const float* res_xy, const tabi_spec* specs,
                            tabi_placement* const* out, tabi_info* infos);

/* ---- validation and metrics on the GPU ----
 * P:85 / P:353: "texels covered by two or more charts ... with 1 pixel gutter
 * dilation"; S:545-553 fix the conservative raster rule: texel (i, r) is
 * covered by chart c iff the OPEN square (i, i+1) x (r, r+1) meets the closed
 * outline of c mapped by placements[c] (tabi_placement steps 0-6, exact
 * integer arithmetic).  Counts:
 *   overlap  atlas texels covered by >= 2 charts;
 *   gutter   atlas texels covered by >= 2 charts after a Chebyshev dilation of
 *            each chart's in-atlas coverage by `gutter` texels (atlas edges
 *            exempt);
 *   oob      covered texels outside [0, atlas_w) x [0, atlas_h);
 *   covered  atlas texels covered by >= 1 chart; occupancy = covered / (W H).
 * l2_stretch: every chart map is a similarity of scale
 * s_c = scale_num / scale_den, so per-triangle stretch is 1/s_c and the
 * area-weighted RMS is sqrt(sum_c A_c / s_c^2 / sum_c A_c), A_c the area of the
 * snapped outline (before step 0).  Deterministic. */
typedef struct {
  int64_t overlap, gutter, oob, covered;
  double occupancy, l2_stretch;
  int32_t bad_chart;     /* on TABI_EINVAL: first chart whose outline does not snap
                            (|coord * res| * 256 > 2^24, non-finite, < 3 vertices) or
                            whose placement is malformed (scale <= 0, prerot > 7); else -1 */
  int32_t gpu_launches;  /* kernels launched by this call */
} tabi_validation;

/* Validate n_charts placements (e.g. the `out` of a tabi_pack) against their
 * outlines.  xy / chart_start / res as for tabi_pack; placements n_charts
 * entries.  on_device 0: host pointers (copied in); 1: device pointers.
 * Device scratch is one byte per texel of every chart's g-dilated texel box
 * plus 2 bits per atlas texel; it grows on demand and is kept on ctx.  Returns
 * TABI_EINVAL on bad arguments (atlas side outside [1, 65536], gutter outside
 * [0, 64], n_charts < 1 or above the context's max_charts), TABI_ECUDA on a
 * CUDA error.  Independent of the last tabi_pack (its introspection state is
 * untouched). */
tabi_status tabi_validate(tabi_ctx* ctx, const float* xy, const int32_t* chart_start,
                          int32_t n_charts, float res_x, float res_y, int32_t atlas_w,
                          int32_t atlas_h, int32_t gutter, const tabi_placement* placements,
                          tabi_validation* out, int on_device, void* stream);

/* ---- introspection of the last tabi_pack on ctx (parity tests; host outputs) ---- */

/* Final-pose proxy of one chart, 1088 bytes (D3-D8 of SURVEY.md §8(c)). */
typedef struct {
  int32_t w, h;                   /* posed extents, 1/256 texel */
  int64_t area2;                  /* 2 x |polygon area| */
  int32_t xmin, ymin;             /* snapped input AABB min */
  int32_t rot90, fx, fy, k;
  int32_t top[64], bot[64], left[64], right[64];   /* merged local AABBs */
  int32_t obb_j, prerot;          /* prerot: pre-rotation angle index (TABI_F_PREROTATE) */
  int64_t umin, umax, vmin, vmax; /* OBB in the Q30-rotated frame, theta = obb_j * pi/16 */
} tabi_proxy_dbg;

typedef struct {
  int32_t success, score, rows, knees_found, knee_rows, prefix_rows;
  int32_t p;                      /* prefix tail: final scale numerator over 2^20, else 0 */
  int32_t evaluated;              /* 0: skipped (above the area bound or below the winning wave) */
  int32_t switched_at;            /* first prefix-folded sorted position, -1 if none */
  int32_t reserved;
  uint64_t apre_lo, apre_hi;      /* 2 x area of the prefix-folded charts (int128) */
} tabi_cand_dbg;

tabi_status tabi_debug_proxies(tabi_ctx* ctx, tabi_proxy_dbg* out);   /* n_charts entries */
tabi_status tabi_debug_perm(tabi_ctx* ctx, int32_t* perm);             /* sorted pos -> chart */
tabi_status tabi_debug_candidates(tabi_ctx* ctx, tabi_cand_dbg* out);  /* scale_count entries */
/* Footprint of the chart at sorted position s for candidate m (1..M):
 * wd_hd[0..1] = (Wd, Hd); columns/rows receive Wd / Hd int32 values each. */
tabi_status tabi_debug_profile(tabi_ctx* ctx, int32_t m, int32_t s, int32_t* wd_hd,
                               int32_t* dtop, int32_t* dbot, int32_t* dleft, int32_t* dright);
/* Adjacent compacting advance off(s, s+1) and lock bits (bit0: s cannot move
 * above s+1, bit1: s+1 cannot move above s) for candidate m, n_charts entries. */
tabi_status tabi_debug_offsets(tabi_ctx* ctx, int32_t m, int32_t* off, uint8_t* lockbits);
/* Device timeline of the last wave (%globaltimer ns), 16 entries:
 * [0] last raster group end and [1] last packer end, both from the fused
 * kernel's first CTA start (0 if split); [2] packer ns waiting for tiles (sum
 * over packers); [3] raster ns waiting for a left neighbour tile (sum);
 * [4] tiles rasterized; [5] fused (0/1); [6..13] K4 row-phase SM cycles
 * summed over packers (knee update, fold, HC choice + lock pairs, push,
 * Alg. 1, score, select + commit, FindKnee); [14] of which push staging, [15]
 * of which commit staging.  [6..15] are 0 unless the library was built with
 * -DTABI_PHASE_TRACE. */
tabi_status tabi_debug_trace(tabi_ctx* ctx, int64_t* out16);
/* Fused rasterizer per-item phase SM cycles of the last wave, summed over
 * raster groups, 16 entries (0 unless built with -DTABI_PHASE_TRACE): [0..6]
 * queue fetch, cells, large charts + accounting, boundary arrivals, pair
 * offsets, publish, setup; [7] 0; [8..11] wave slot 0's first-row timeline in
 * ns from the kernel start: tile 0 footprints done, tile 0 published, packer
 * 0's first fold unblocked, packer 0's first row done; [12..15] 0. */
tabi_status tabi_debug_trace_raster(tabi_ctx* ctx, int64_t* out16);
/* Latency floor of the packer's per-row building blocks: one
 * 512-thread CTA times dependent chains on `cuda_device`; out8 receives ns per
 * operation: [0] barrier, [1] barrier + shared-memory exchange (two barriers),
 * [2] block max-reduce (two barriers), [3] shared atomicMax + barrier,
 * [4] dependent L2 load, [5] the SM clock in MHz it measured.  Diagnostic;
 * independent of any context. */
tabi_status tabi_debug_latency_floor(int cuda_device, double* out8);

#ifdef __cplusplus
}
#endif
#endif
