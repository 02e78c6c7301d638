/*
 * csplat.h -- C ABI of the B200 (sm_100a) hot path of "Compact 3D Gaussian
 * Splatting for Dense Visual SLAM" (arXiv 2403.11247).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; readings R1..R26 and
 * the decision arithmetic (DA) are defined in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Ownership: every data pointer is a caller-owned CUDA DEVICE pointer
 *    (e.g. from torch.empty(device="cuda")), unless the comment says "host".
 *    Struct arguments themselves live in HOST memory and are read during the
 *    call only.  The library never allocates, frees or retains device
 *    memory beyond the call; scratch comes from a caller buffer sized by
 *    csplat_workspace_bytes().
 *  - Asynchrony: all work is enqueued on `stream` (a cudaStream_t; NULL = the
 *    legacy default stream).  Results are valid once the stream reaches the
 *    end of the enqueued work.  Only csplat_bin_tiles with CSPLAT_SYNC (and
 *    argument validation) synchronises with the host.
 *  - Layouts: Gaussian attributes are planar SoA [k][n] float32; images are
 *    planar [c][H][W] float32; codebooks [L][P][d] float32; indices [L][n]
 *    uint8 (P <= 256) or uint16; the 64-byte projected record is described in
 *    DESIGN.md §4.
 *  - Alignment: every float plane and record buffer must be 16-byte aligned
 *    (CSPLAT_ERR_ALIGNMENT otherwise).
 *  - Errors: every function returns a csplat_status; it never aborts and
 *    never throws across the ABI.  CSPLAT_ERR_CUDA carries the CUDA error text
 *    in csplat_last_error() (thread-local).  Device faults surface as
 *    CSPLAT_ERR_CUDA on a later call or at the caller's next synchronisation.
 *    Non-finite attribute values are culled (never propagated).  n = 0 is
 *    valid (black images, zero gradients).
 *  - Device: compute capability 10.0 (B200) only; otherwise
 *    CSPLAT_ERR_UNSUPPORTED.
 */
#ifndef CSPLAT_H
#define CSPLAT_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum csplat_status {
    CSPLAT_OK = 0,
    CSPLAT_ERR_INVALID_ARG = 1,  /* null required pointer, n < 0, W/H <= 0, fx/fy <= 0, !(0<near<far), L/P/d out of range */
    CSPLAT_ERR_ALIGNMENT = 2,    /* a plane or record buffer is not 16-byte aligned */
    CSPLAT_ERR_CAPACITY = 3,     /* more (tile, Gaussian) pairs than pair_capacity (CSPLAT_SYNC only) */
    CSPLAT_ERR_WORKSPACE = 4,    /* ws_bytes < csplat_workspace_bytes(...) */
    CSPLAT_ERR_CUDA = 5,         /* launch / runtime error; text in csplat_last_error */
    CSPLAT_ERR_UNSUPPORTED = 6   /* device is not compute capability 10.x */
};

#define CSPLAT_TILE 16           /* screen tile edge in pixels (R4) */
#define CSPLAT_RECORD_BYTES 64   /* projected record size */

/* Device status bits.  A status word is a caller-owned device uint32 that
 * library kernels OR these bits into and NEVER clear (the caller zeroes it,
 * e.g. once per window iteration, and reads it whenever it likes -- one word
 * can collect the status of many asynchronous calls, CUDA-graph replays
 * included).  SURVEY §8(b): "overflow is written to a device status word and
 * downstream kernels early-out"; "out-of-range codebook indices are culled
 * and set a device status bit". */
#define CSPLAT_STATUS_CAPACITY 1u    /* a tile's (tile, Gaussian) pairs did not fit the pair
                                        capacity: that tile's range is left EMPTY, so the
                                        renderers treat it as background (early-out) */
#define CSPLAT_STATUS_CODE_INDEX 2u  /* a codebook index >= P: that Gaussian is culled */

/* Flags */
#define CSPLAT_SYNC 1u           /* bin_tiles: read n_pairs back, return CAPACITY if it exceeds the capacity */
#define CSPLAT_POSE_ONLY 2u      /* render_bwd: only the pose gradient (tracking) */
#define CSPLAT_ACCUMULATE 4u     /* render_bwd: add into the outputs instead of overwriting */
#define CSPLAT_WS_ZEROED 16u     /* render_bwd: the caller guarantees ws's accumulator is all
                                    zero (no memset); csplat_chain_views: clear every
                                    accumulator entry it consumed, so it stays zero */
#define CSPLAT_SKIP_CHAIN 8u     /* render_bwd: stop after the compositing backward (a7): the
                                    per-Gaussian screen-space gradient is left in ws as
                                    [n][12] float32 (raw moments Sx, Sy, Sxx, Sxy, Syy of
                                    alpha dL/dalpha, dL/do_hat, dL/dz, dL/drgb, 2 pad;
                                    DESIGN.md §7) followed (256-byte aligned) by a
                                    ceil(n/32)-word bitmap of the Gaussians that got a
                                    partial; `out` is not touched */

/* Pinhole intrinsics K ("known camera intrinsic K"), image size
 * (1..32767 pixels per side), clip (R21). */
typedef struct {
    float fx, fy, cx, cy;
    int32_t width, height;
    float near_z, far_z;
} csplat_camera;

/* World->camera [R|t], row-major 3x4, HOST memory ("{R_i|t_i}"). */
typedef struct { float m[12]; } csplat_view;

/* Renderer constants: mask threshold eps (Eq 6; R12, default 0.01),
 * alpha cap (R1, 0.99), transmittance cutoff (R3, 1e-4), 2D dilation (R5, 0.3). */
typedef struct { float mask_eps, alpha_max, t_min, dilation; } csplat_params;

/* Gaussian map (Eq 6; parameterisation R15), device SoA planes.
 * n_dev (optional, device int64): if non-NULL, only the first *n_dev <= n
 * Gaussians exist (e.g. the survivor count written by csplat_mask_prune);
 * the rest are treated as culled. */
typedef struct {
    int64_t n;
    const int64_t *n_dev;
    const float *mean;       /* [3][n] world position                  */
    const float *opacity;    /* [n]    opacity logit, o = sigmoid(.)    */
    const float *rgb;        /* [3][n] colour c_i of Eq 3              */
    const float *log_scale;  /* [3][n] log of the scale S (Eq 1)       */
    const float *quat;       /* [4][n] rotation R as wxyz quaternion   */
    const float *mask;       /* [n]    mask logit m (Eq 6)             */
} csplat_gaussians;

/* Mutable Gaussian planes (output of csplat_mask_prune), capacity >= n. */
typedef struct {
    int64_t capacity;
    float *mean, *opacity, *rgb, *log_scale, *quat, *mask;
} csplat_gaussians_out;

/* R-VQ geometry codebooks (Eq 10; R16-R18): log-scale (d=3) and
 * quaternion (d=4) codes, and per-Gaussian indices [L][n]. */
typedef struct {
    int32_t stages, size, idx_bytes, reserved;  /* L, P, 1 or 2 */
    const float *scale_codes;  /* [L][P][3] */
    const float *rot_codes;    /* [L][P][4] */
    const void *scale_idx;     /* [L][n] uint8/uint16 */
    const void *rot_idx;       /* [L][n] uint8/uint16 */
    uint32_t *status;          /* optional device status word (NULL = not reported):
                                  CSPLAT_STATUS_CODE_INDEX is OR-ed in when a decoded
                                  Gaussian has an index >= P (that Gaussian is culled) */
} csplat_codebook;

/* Gradients: planes [k][n] like csplat_gaussians (any may be NULL to skip),
 * pose[6] = dL/d(omega, v) for the left perturbation V' = Exp(xi) V (R22). */
typedef struct {
    float *mean, *opacity, *rgb, *log_scale, *quat, *mask;
    float *pose;
} csplat_grads;

/* a1 + a2(decode) + a3: projection (Eq 1-2) with the binary mask
 * (Eq 6-7) and R-VQ decode (Eq 10; cb may be NULL for raw
 * geometry).  Writes the 64-byte record rec[n] and the touched-tile count
 * count[n] (0 = culled), bit-exactly as DESIGN.md §3 (DA). */
int csplat_project(const csplat_gaussians *g, const csplat_codebook *cb, const csplat_camera *cam,
                   const csplat_view *view, const csplat_params *prm, void *rec, int32_t *count,
                   void *stream);

/* csplat_project with the world->camera view read from DEVICE memory
 * (view_dev: 12 floats, row-major [R|t]) when the kernel runs, so a pose
 * updated on the device by csplat_pose_step is picked up inside a captured
 * CUDA graph (NEXT-1 tracking).  Otherwise identical to csplat_project. */
int csplat_project_dv(const csplat_gaussians *g, const csplat_codebook *cb,
                      const csplat_camera *cam, const float *view_dev, const csplat_params *prm,
                      void *rec, int32_t *count, void *stream);

/* a1 + a2-decode + a3 over n_views views at once (SURVEY §8(b) n_views, §8(e)
 * "multi-view projection that reads each Gaussian once"): each Gaussian is
 * read, decoded and its Sigma (Eq 1) formed once, then projected into every
 * view.  views: host array [n_views]; rec [n_views][n] records, count
 * [n_views][n]: view v's outputs are bit-identical to csplat_project(views[v]). */
int csplat_project_views(const csplat_gaussians *g, const csplat_codebook *cb,
                         const csplat_camera *cam, const csplat_view *views, int32_t n_views,
                         const csplat_params *prm, void *rec, int32_t *count, void *stream);

/* csplat_project_bin over n_views views at once: the multi-view projection
 * above with the bucket pass fused in per view, then one batched per-tile
 * sort of every view.  Per view v (same capacity for every view): rec + v n,
 * count + v n, pair_gid + v pair_capacity, tile_range + v (T+1) (entry T = the
 * view's status slot, see csplat_bin_tiles), n_pairs_dev + v, its binning
 * workspace at ws + v ws_bytes_per_view (>= csplat_workspace_bytes(
 * CSPLAT_OP_BIN_TILES, n, pair_capacity, cam), a multiple of 256; ws 256-byte
 * aligned), tile_active (optional) + v ceil(T/32) words.  Outputs bit-identical
 * to csplat_project_bin per view.  No host synchronisation (overflow: the
 * status slots).  tile_lists (optional, NEXT-4's sparse views; needs
 * tile_active): per view v at tile_lists + v list_stride a device int32 list
 * {count, tile_0 < tile_1 < ...} of exactly the tiles set in its tile_active
 * words, count <= max_list (host): only those tiles are sorted and get
 * ranges, every other tile's range is empty (the same output as without the
 * list, at max_list instead of T CTAs per view). */
int csplat_project_bin_views(const csplat_gaussians *g, const csplat_codebook *cb,
                             const csplat_camera *cam, const csplat_view *views, int32_t n_views,
                             const csplat_params *prm, const uint32_t *tile_active,
                             const int32_t *tile_lists, int64_t list_stride, int32_t max_list,
                             void *rec, int32_t *count, int64_t pair_capacity, uint32_t *pair_gid,
                             uint32_t *tile_range, int64_t *n_pairs_dev, void *ws,
                             size_t ws_bytes_per_view, void *stream);

/* a8 summed over n_views views (the window's ACCUMULATE of csplat_render_bwd's
 * chain, in one pass): ws = n_views consecutive csplat_render_bwd workspaces
 * (each csplat_workspace_bytes(CSPLAT_OP_RENDER_BWD, n, 0, cam) bytes, 256-byte
 * aligned), each left by csplat_render_bwd with CSPLAT_SKIP_CHAIN (the
 * screen-space accumulator and the bitmap of the Gaussians it reached);
 * rec [n_views][n] the views' records.  The Gaussian is read and decoded once; the view-dependent
 * chain (mean, J, Sigma', pose) runs per view that reached it and the rest
 * (Sigma -> rotation / scale, opacity, STE mask) once on the per-view sum.
 * out: the 15 gradient planes (overwritten, or added with CSPLAT_ACCUMULATE);
 * out->pose (optional) = [n_views][6] per-view pose gradients.  With
 * CSPLAT_WS_ZEROED every consumed accumulator entry is cleared (so csplat_render_bwd
 * may skip its memset next time).  POSE_ONLY is not supported. */
int csplat_chain_views(const csplat_gaussians *g, const csplat_codebook *cb,
                       const csplat_camera *cam, const csplat_view *views, int32_t n_views,
                       const csplat_params *prm, const void *rec, void *ws, uint32_t flags,
                       const csplat_grads *out, void *stream);

/* a4 + a5: tile binning and (tile, depth) ordering (R4, R11).
 * Outputs, for n_pairs = sum(count) pairs:
 *   pair_gid[pair_capacity]   one entry per pair, ordered by (tile, bits(z_c), index):
 *                             bits 0-27 the Gaussian index (n < 2^28), bits 28-31
 *                             the pair's 8x8-block cull mask: bit w (x half w & 1,
 *                             y half w >> 1 of the tile) set unless alpha < 1/255
 *                             provably holds over that whole block.
 *                             The renderers gather each listed record from rec
 *                             (the forward by TMA gather4, the backward by
 *                             cp.async into shared memory).
 *   tile_range[T+1][2]        [start, end) of every tile, T = ceil(W/16)*ceil(H/16);
 *                             entry T is the view's STATUS slot {status word, max
 *                             n_pairs}: the library ORs CSPLAT_STATUS_CAPACITY into
 *                             tile_range[2T] and atomically maxes the total pair
 *                             count (clamped to 2^32-1) into tile_range[2T+1]; it
 *                             never clears them (the caller zeroes the slot once,
 *                             then reads it after any number of calls)
 *   n_pairs_dev               device int64: the total (may exceed the capacity)
 * Capacity overflow: a tile whose pairs do not all fit (its prefix + count
 * exceeds pair_capacity, or its bucket spill was lost) gets an EMPTY range and
 * sets CSPLAT_STATUS_CAPACITY, so every downstream kernel treats it as
 * background (early-out) instead of rendering a truncated list; tiles that fit
 * are exact.  With CSPLAT_SYNC the call also synchronises and returns
 * CSPLAT_ERR_CAPACITY.
 * ws: csplat_workspace_bytes(CSPLAT_OP_BIN_TILES, n, pair_capacity, cam). */
int csplat_bin_tiles(const void *rec, const int32_t *count, int64_t n, const csplat_camera *cam,
                     int64_t pair_capacity, uint32_t *pair_gid,
                     uint32_t *tile_range, int64_t *n_pairs_dev, uint32_t flags, void *ws,
                     size_t ws_bytes, void *stream);

/* a1 + a2-decode + a3 + a4 + a5 in one call: csplat_project followed by
 * csplat_bin_tiles_active, with the bucket pass of the binning (the
 * warp-cooperative expansion of each Gaussian's tile rectangle into the tile
 * buckets) fused into the projection kernel while the records are still in
 * registers.  Outputs are bit-identical to the two calls: rec and count as
 * csplat_project (same layout, ownership and alignment), pair_gid,
 * tile_range and n_pairs_dev as csplat_bin_tiles_active (tile_active may be
 * NULL = every tile).  n = g->n; ws: csplat_workspace_bytes(CSPLAT_OP_BIN_TILES,
 * g->n, pair_capacity, cam).  flags: CSPLAT_SYNC as csplat_bin_tiles.
 * Errors as the two calls. */
int csplat_project_bin(const csplat_gaussians *g, const csplat_codebook *cb,
                       const csplat_camera *cam, const csplat_view *view,
                       const csplat_params *prm, void *rec, int32_t *count,
                       const uint32_t *tile_active, int64_t pair_capacity, uint32_t *pair_gid, uint32_t *tile_range, int64_t *n_pairs_dev,
                       uint32_t flags, void *ws, size_t ws_bytes, void *stream);

/* csplat_project_bin with the view in DEVICE memory (see csplat_project_dv). */
int csplat_project_bin_dv(const csplat_gaussians *g, const csplat_codebook *cb,
                          const csplat_camera *cam, const float *view_dev,
                          const csplat_params *prm, void *rec, int32_t *count,
                          const uint32_t *tile_active, int64_t pair_capacity, uint32_t *pair_gid, uint32_t *tile_range, int64_t *n_pairs_dev,
                          uint32_t flags, void *ws, size_t ws_bytes, void *stream);

/* a1 + a2-decode + a3 + a4 + a5 + a6 in one call: csplat_project_bin (every
 * tile active) followed by csplat_render_fwd, with the per-tile sort and the
 * forward split into tile chunks that run as a pipeline on two library-owned
 * streams forked from and joined back into `stream` (capturable in a CUDA
 * graph): the latency-bound sort of chunk c+1 overlaps the issue-bound forward
 * of chunk c.  Outputs are bit-identical to those calls (tested): rec, count,
 * pair_gid, tile_range, n_pairs_dev as csplat_project_bin; color
 * [3][H][W], depth, silhouette, t_final [H][W] and n_contrib [H][W] as
 * csplat_render_fwd.  Pairs beyond pair_capacity are dropped (ranges clamped;
 * no CSPLAT_SYNC check here: read n_pairs_dev).  ws: csplat_workspace_bytes(
 * CSPLAT_OP_BIN_TILES, g->n, pair_capacity, cam).  Errors as those calls.
 * The library's fork streams and events are per device and shared by
 * csplat_project_bin_render, csplat_render_step and csplat_tracking_step:
 * calls from several host threads onto one device must be serialised by the
 * caller (enqueueing order defines the fork/join order). */
int csplat_project_bin_render(const csplat_gaussians *g, const csplat_codebook *cb,
                              const csplat_camera *cam, const csplat_view *view,
                              const csplat_params *prm, void *rec, int32_t *count,
                              int64_t pair_capacity, uint32_t *pair_gid,
                              uint32_t *tile_range, int64_t *n_pairs_dev, void *ws,
                              size_t ws_bytes, float *color, float *depth, float *silhouette,
                              float *t_final, int32_t *n_contrib, void *stream);

/* csplat_project_bin_render with the view in DEVICE memory (csplat_project_dv). */
int csplat_project_bin_render_dv(const csplat_gaussians *g, const csplat_codebook *cb,
                                 const csplat_camera *cam, const float *view_dev,
                                 const csplat_params *prm, void *rec, int32_t *count,
                                 int64_t pair_capacity, uint32_t *pair_gid,
                                 uint32_t *tile_range, int64_t *n_pairs_dev, void *ws,
                                 size_t ws_bytes, float *color, float *depth, float *silhouette,
                                 float *t_final, int32_t *n_contrib, void *stream);

/* a1 + a2-decode + a3 .. a8 for one view in one call (the C2 step after the
 * prune and the R-VQ assignment): csplat_project_bin_render followed by
 * csplat_render_bwd, with the backward kernel joining each tile chunk's
 * pipeline (sort -> forward -> backward on one library stream per chunk,
 * forked from / joined into `stream`), then the per-Gaussian chain on
 * `stream`.  Arguments as those calls (ws_bin: CSPLAT_OP_BIN_TILES
 * workspace; ws_bwd: CSPLAT_OP_RENDER_BWD workspace; flags: CSPLAT_ACCUMULATE,
 * CSPLAT_POSE_ONLY is rejected).  Outputs equal the separate calls: the
 * discrete ones and the images bit for bit, the gradients up to the order of
 * the backward's float atomics. */
int csplat_render_step(const csplat_gaussians *g, const csplat_codebook *cb,
                       const csplat_camera *cam, const csplat_view *view,
                       const csplat_params *prm, void *rec, int32_t *count,
                       int64_t pair_capacity, uint32_t *pair_gid,
                       uint32_t *tile_range, int64_t *n_pairs_dev, void *ws_bin,
                       size_t ws_bin_bytes, float *color, float *depth, float *silhouette,
                       float *t_final, int32_t *n_contrib, const float *d_color,
                       const float *d_depth, const float *d_silhouette, uint32_t flags,
                       const csplat_grads *out, void *ws_bwd, size_t ws_bwd_bytes,
                       void *stream);

/* NEXT-1: one tracking iteration's render in one call -- csplat_render_step
 * with the loss-fused backward of csplat_tracking_bwd (Eq 12 + Eq 14 formed
 * per pixel from the images this call renders and obs_color / obs_depth;
 * |R| = *n_valid_dev from csplat_count_valid_depth) in each tile chunk, then
 * the chain.  Exactly one of view / view_dev (device, as csplat_project_dv).
 * flags: CSPLAT_POSE_ONLY for tracking.  loss3_dev (L_t, L_c, L_d) is
 * overwritten.  Other arguments, outputs and errors as csplat_render_step and
 * csplat_tracking_bwd. */
int csplat_tracking_step(const csplat_gaussians *g, const csplat_codebook *cb,
                         const csplat_camera *cam, const csplat_view *view,
                         const float *view_dev, const csplat_params *prm, void *rec,
                         int32_t *count, int64_t pair_capacity, uint32_t *pair_gid, uint32_t *tile_range, int64_t *n_pairs_dev,
                         void *ws_bin, size_t ws_bin_bytes, float *color, float *depth,
                         float *silhouette, float *t_final, int32_t *n_contrib,
                         const float *obs_color, const float *obs_depth,
                         const uint64_t *n_valid_dev, float lambda_depth, float sil_gate,
                         uint32_t flags, const csplat_grads *out, float *loss3_dev,
                         void *ws_bwd, size_t ws_bwd_bytes, void *stream);

/* csplat_bin_tiles restricted to the tiles whose bit is set in tile_active
 * (device uint32[ceil(T/32)], bit t & 31 of word t >> 5; NULL = every tile):
 * the pairs of the other tiles are not emitted and their ranges are empty, so
 * the output is csplat_bin_tiles' with those tiles' lists removed.  NEXT-4 uses
 * it to bin only the tiles that hold sampled rays (csplat_ba_patches). */
int csplat_bin_tiles_active(const void *rec, const int32_t *count, int64_t n,
                            const csplat_camera *cam, const uint32_t *tile_active,
                            int64_t pair_capacity, uint32_t *pair_gid,
                            uint32_t *tile_range, int64_t *n_pairs_dev, uint32_t flags, void *ws,
                            size_t ws_bytes, void *stream);

/* a6: front-to-back compositing of colour, depth and silhouette (Eq 3-5,
 * P:98-109; R1-R3, R7-R10).  Outputs color [3][H][W], depth, silhouette,
 * t_final [H][W] float32 and n_contrib [H][W] int32 (local index + 1 of the
 * last composited entry of the pixel's tile list; the backward's replay bound).
 * Inputs: rec (csplat_project) and the pair lists pair_gid / tile_range
 * (csplat_bin_tiles). */
int csplat_render_fwd(const void *rec, const uint32_t *pair_gid, const uint32_t *tile_range,
                      const csplat_camera *cam, const csplat_params *prm, float *color,
                      float *depth, float *silhouette, float *t_final, int32_t *n_contrib,
                      void *stream);

/* csplat_render_fwd / csplat_render_bwd over the tiles of a device list only
 * (NEXT-4's sparse views: a few active tiles per keyframe): tile_list =
 * {count, tile_0, tile_1, ...} (device int32, count <= max_tiles, the host's
 * bound for the grid).  Pixels of other tiles are not written (forward) and
 * not replayed (backward); everything else as the full calls. */
int csplat_render_fwd_list(const void *rec, const uint32_t *pair_gid, const uint32_t *tile_range,
                           const int32_t *tile_list, int32_t max_tiles, const csplat_camera *cam,
                           const csplat_params *prm, float *color, float *depth, float *silhouette,
                           float *t_final, int32_t *n_contrib, void *stream);
int csplat_render_bwd_list(const csplat_gaussians *g, const csplat_codebook *cb,
                           const csplat_camera *cam, const csplat_view *view,
                           const csplat_params *prm, const void *rec, const uint32_t *pair_gid,
                           const uint32_t *tile_range, const int32_t *tile_list,
                           int32_t max_tiles, const float *t_final, const int32_t *n_contrib,
                           const float *d_color, const float *d_depth, const float *d_silhouette,
                           uint32_t flags, const csplat_grads *out, void *ws, size_t ws_bytes,
                           void *stream);

/* a7 + a8: backward of a6 through a3, a2-decode and the STE mask (Eq 6), with
 * the pose gradient (R14, R20, R22, R23).  d_color [3][H][W], d_depth,
 * d_silhouette [H][W] are dL/d(outputs).  The forward-state arguments (rec,
 * pair_gid, tile_range, t_final, n_contrib) must come from csplat_project /
 * csplat_bin_tiles / csplat_render_fwd on the same inputs (not verified).
 * Gradients are w.r.t. mean, opacity logit, rgb, (decoded) log-scale, (decoded)
 * quaternion, mask logit and pose.  flags: CSPLAT_POSE_ONLY, CSPLAT_ACCUMULATE.
 * ws: csplat_workspace_bytes(CSPLAT_OP_RENDER_BWD, n, 0, cam). */
int csplat_render_bwd(const csplat_gaussians *g, const csplat_codebook *cb,
                      const csplat_camera *cam, const csplat_view *view, const csplat_params *prm,
                      const void *rec, const uint32_t *pair_gid, const uint32_t *tile_range,
                      const float *t_final, const int32_t *n_contrib, const float *d_color,
                      const float *d_depth, const float *d_silhouette, uint32_t flags,
                      const csplat_grads *out, void *ws, size_t ws_bytes, void *stream);

/* csplat_render_bwd with the view in DEVICE memory (see csplat_project_dv). */
int csplat_render_bwd_dv(const csplat_gaussians *g, const csplat_codebook *cb,
                         const csplat_camera *cam, const float *view_dev,
                         const csplat_params *prm, const void *rec, const uint32_t *pair_gid,
                         const uint32_t *tile_range, const float *t_final,
                         const int32_t *n_contrib, const float *d_color, const float *d_depth,
                         const float *d_silhouette, uint32_t flags, const csplat_grads *out,
                         void *ws, size_t ws_bytes, void *stream);

/* NEXT-1 loss-fused backward: csplat_render_bwd whose
 * upstream gradients are those of the tracking objective, formed per pixel in
 * the backward's prologue instead of read: Eq 12 gated by Eq 14
 * (P:207-210), reading R27 -- g = 1[S > sil_gate], v = 1[D_obs > 0],
 * dL/dC = 2 g (C - C_obs)/(W H), dL/dD = 2 lambda_depth g v (D - D_obs)/|R|,
 * dL/dS = 0, with |R| = *n_valid_dev (csplat_count_valid_depth of the same
 * obs_depth).  Pixels whose upstream is zero (gated out, or no valid depth and
 * no colour residual) are not replayed; a warp or tile with none left is
 * skipped.  color/depth/silhouette: csplat_render_fwd's outputs; obs_*: the
 * observed frame (device).  loss3_dev (device float[3], may be NULL) receives
 * (L_t, L_c, L_d), zeroed by the call.  Exactly one of view (host)
 * / view_dev (device, see csplat_project_dv) is non-NULL.  Other arguments,
 * flags (CSPLAT_POSE_ONLY for tracking) and ws as csplat_render_bwd. */
int csplat_tracking_bwd(const csplat_gaussians *g, const csplat_codebook *cb,
                        const csplat_camera *cam, const csplat_view *view, const float *view_dev,
                        const csplat_params *prm, const void *rec, const uint32_t *pair_gid,
                        const uint32_t *tile_range, const float *t_final,
                        const int32_t *n_contrib, const float *color, const float *depth,
                        const float *silhouette, const float *obs_color, const float *obs_depth,
                        const uint64_t *n_valid_dev, float lambda_depth, float sil_gate,
                        uint32_t flags, const csplat_grads *out, float *loss3_dev, void *ws,
                        size_t ws_bytes, void *stream);

/* |R| of Eq 12 for a frame: *n_valid_dev (device uint64) = the number of
 * pixels of obs_depth [H][W] (device) with a valid depth (> 0). */
int csplat_count_valid_depth(const float *obs_depth, int32_t width, int32_t height,
                             uint64_t *n_valid_dev, void *stream);

/* NEXT-1: the pose step of a tracking iteration on the device (Sec 3.4,
 * the pose is optimised by minimising the tracking objective):
 * view_dev (12 floats, world->camera [R|t]) <- Exp(xi) view_dev with
 * xi = -(lr_rot * g[0..2], lr_trans * g[3..5]), g = pose_grad_dev (the 6-float
 * pose gradient of csplat_render_bwd, left perturbation (omega, v), R22);
 * Exp applied as p' = Rod(omega) p + v, evaluated in float64. */
int csplat_pose_step(float *view_dev, const float *pose_grad_dev, float lr_rot, float lr_trans,
                     void *stream);

/* a2: greedy residual VQ assignment (Eq 10; R17): for each of the n
 * d-dimensional vectors x [d][n] and each stage l, idx[l][i] = argmin_k
 * ||C^l[k] - (x_i - S_hat^{l-1}_i)||^2 (DA distances, ties to the lowest k).
 * codes [L][P][d]; idx_out [L][n] with idx_bytes 1 (P <= 256) or 2;
 * recon_out [d][n] (optional) = S_hat^L.  n_dev optional (see csplat_gaussians).
 * Limits: 1 <= d <= 8, 1 <= L <= 16, 1 <= P <= 65536. */
int csplat_rvq_assign(const float *x, int64_t n, const int64_t *n_dev, int32_t d,
                      const float *codes, int32_t L, int32_t P, void *idx_out, int32_t idx_bytes,
                      float *recon_out, void *stream);

/* a9: mask prune (Fig 3): keep Gaussian i iff
 * m_i > tau (Eq 6 / R12), compact all planes of `in` (and, if in_idx is not
 * NULL, its scale/rot index planes into out_scale_idx / out_rot_idx [L][cap])
 * preserving order.  reset_mask_logit: if not NaN, survivors' mask is set to
 * it (sliding-window reset).  keep_map [n] (optional) = new index or -1.
 * n_kept_dev: device int64 survivor count.
 * ws: csplat_workspace_bytes(CSPLAT_OP_MASK_PRUNE, n, 0, NULL). */
int csplat_mask_prune(const csplat_gaussians *in, const csplat_codebook *in_idx, float mask_eps,
                      float reset_mask_logit, const csplat_gaussians_out *out,
                      void *out_scale_idx, void *out_rot_idx, int32_t *keep_map,
                      int64_t *n_kept_dev, void *ws, size_t ws_bytes, void *stream);

/* NEXT-1: the tracking objective of Sec 3.4 -- Eq 12 gated by the
 * rendered silhouette as in Eq 14; the SIFT reprojection term is
 * out of scope (reading R27 in DESIGN.md).  Per pixel p: g = 1[S_p > sil_gate],
 * v = 1[obs_depth_p > 0];  L_c = (1/HW) sum g |C - C_obs|^2,
 * L_d = (1/|R|) sum g v (D - D_obs)^2 with |R| = #valid-depth pixels (>= 1),
 * L_t = L_c + lambda_depth L_d.  Writes the upstream gradients of
 * csplat_render_bwd: d_color = 2 g (C - C_obs)/HW, d_depth = 2 lambda g v
 * (D - D_obs)/|R|, d_silhouette = 0 (the gate is not differentiated), and
 * loss3_dev (optional, device float[3]) = (L_t, L_c, L_d).  Inputs planar
 * [3][H][W] / [H][W] float32 (device).  ws: csplat_workspace_bytes(
 * CSPLAT_OP_TRACKING_LOSS, 0, 0, NULL). */
int csplat_tracking_loss(const float *color, const float *depth, const float *silhouette,
                         const float *obs_color, const float *obs_depth, int32_t width,
                         int32_t height, float lambda_depth, float sil_gate, float *d_color,
                         float *d_depth, float *d_silhouette, float *loss3_dev, void *ws,
                         size_t ws_bytes, void *stream);

/* NEXT-2: the straight-through gradient of the R-VQ decode (Eq 10 first
 * line: S_hat = sum_l C^l[i^l]; reading R31).  d_shat [d][n] (device) =
 * dL/dS_hat, the decoded-geometry gradient csplat_render_bwd writes into
 * grads.log_scale (d = 3) or grads.quat (d = 4).  d_codes [L][P][d] (device,
 * 16-byte aligned for d = 4) gets, for every stage l and code k, the sum of
 * dL/dS_hat_n over the vectors with idx[l][n] = k (S_hat is linear in every
 * code: each stage's chosen code receives the full gradient); overwritten
 * unless flags has CSPLAT_ACCUMULATE.  The STE gradient of the raw vector S
 * itself is d_shat (no call needed).  Indices >= P are skipped.  Sums use
 * float32 vector reductions (order-dependent rounding).  n_dev as in
 * csplat_gaussians. */
int csplat_rvq_code_grad(const float *d_shat, int64_t n, const int64_t *n_dev, int32_t d,
                         const void *idx, int32_t idx_bytes, int32_t L, int32_t P,
                         float *d_codes, uint32_t flags, void *stream);

/* NEXT-2: Fig 4 codebook initialisation of one stage ("randomly select
 * codebook initialization with the closest code"; reading R32).  codes
 * [L][P][d] (device): stage `stage` is overwritten with C[k] = the stage
 * residual x_s - S_hat_s^{stage-1} of the sampled vector s = sample[k]
 * (device int64[P], each in [0, n); the random draw is the caller's), S_hat
 * the decision-arithmetic stage-order sum of the codes of the earlier stages
 * at idx [L][n] (from csplat_rvq_assign over those stages; unused for stage
 * 0).  The closest-code assignment that follows is csplat_rvq_assign.  Calls
 * for stages 0..L-1 in order, each followed by an assignment over stages
 * 0..stage, initialise the whole codebook (paper_2403_11247_b200.rvq_init). */
int csplat_rvq_init_stage(const float *x, int64_t n, int32_t d, float *codes, int32_t L,
                          int32_t P, int32_t stage, const void *idx, int32_t idx_bytes,
                          const int64_t *sample, void *stream);

/* NEXT-2: R-VQ codebook update (Eq 11; reading R28): one k-means
 * M-step for the assignment idx [L][n] (from csplat_rvq_assign): with the
 * residual r_n^l = x_n - S_hat_n^{l-1} (the DA stage-order sums of
 * csplat_rvq_assign), codes_out[l][k] = mean of the r_n^l with idx[l][n] = k
 * (codes with no member are copied), counts_out [L][P] (optional) = members,
 * loss_out [L+1] (optional, device float) = per-stage sum ||r - C^l[i]||^2 and
 * L_r = sum / (n P).  codes_out may alias codes.  Sums use float32 atomics
 * (order-dependent rounding).  ws: csplat_workspace_bytes(CSPLAT_OP_RVQ_UPDATE,
 * L * P, d, NULL). */
int csplat_rvq_update(const float *x, int64_t n, const int64_t *n_dev, int32_t d,
                      const float *codes, int32_t L, int32_t P, const void *idx, int32_t idx_bytes,
                      float *codes_out, int32_t *counts_out, float *loss_out, void *ws,
                      size_t ws_bytes, void *stream);

/* NEXT-3 (sliding-window mask schedule):
 * csplat_mask_loss: the mask sparsity loss of Eq 8, L_m = (1/N_a)
 * sum Sig(m_n) over the Gaussians in the current frustum, taken as those the
 * projection kept (count[n] > 0, from csplat_project; reading R29):
 * d_mask[n] += lambda Sig'(m_n) / N_a for them (accumulates into the render
 * gradient), loss_dev (optional, device float[1]) = L_m.
 * ws: csplat_workspace_bytes(CSPLAT_OP_MASK_LOSS, 0, 0, NULL). */
int csplat_mask_loss(const csplat_gaussians *g, const int32_t *count, float lambda,
                     float *d_mask, float *loss_dev, void *ws, size_t ws_bytes, void *stream);

/* csplat_keyframe_overlap: "tallying points within the frustum of each
 * keyframe": every valid pixel (depth > 0) of the current depth map
 * [H][W] (device) is back-projected with the current world->camera view `cur`
 * and counted for keyframe k (views: HOST array of K <= 256 views, same
 * camera) when its depth in k lies in (near, far) and it projects inside
 * [0, W-1] x [0, H-1]; float32 decision arithmetic (reading R29), so the
 * counts are exact.  counts_dev: device int64[K].
 * ws: csplat_workspace_bytes(CSPLAT_OP_KEYFRAME_OVERLAP, K, 0, NULL). */
int csplat_keyframe_overlap(const float *depth, const csplat_camera *cam, const csplat_view *cur,
                            const csplat_view *views, int32_t K, int64_t *counts_dev, void *ws,
                            size_t ws_bytes, void *stream);

/* NEXT-4: random-ray global bundle adjustment (Sec 3.4; reading
 * R30).  The N rays sampled from the keyframe database are N/64 random 8x8
 * pixel patches aligned to the 8-pixel grid; patches[b] = by * (W/8) + bx
 * names the block with origin (8 bx, 8 by) of one keyframe (device int32;
 * ids outside the image's whole blocks are ignored).  Precondition: the ids of
 * one keyframe are DISTINCT (a sample without replacement, as the reading
 * states): a repeated id would count its rays twice in the loss and |R| but
 * write its upstream gradient once.  Not checked on the device.
 *
 * csplat_ba_patches: for the patches of one keyframe, clears and sets its
 * active-tile mask (device uint32[ceil(T/32)], for csplat_bin_tiles_active)
 * and ADDS the patch pixels with a valid observed depth (obs_depth > 0, the
 * set R of Eq 12) to *n_valid_dev (device uint64; the caller zeroes it once
 * per sample and sums it over the keyframes, and over ranks). */
int csplat_ba_patches(const float *obs_depth, const csplat_camera *cam, const int32_t *patches,
                      int64_t n_patches, uint32_t *tile_active, uint64_t *n_valid_dev,
                      void *stream);

/* csplat_ba_patch_loss: one keyframe's share of the BA objective over the
 * whole sample (N = n_rays > 0 rays over all keyframes, |R| = *n_valid_dev,
 * P = N/64 patches):
 *   L_c  = (1/N) sum_rays sum_c (C - C_obs)^2,  L_d = (1/|R|) sum_R (D - D_obs)^2  (Eq 12)
 *   SSIM = mean over patches and channels of the 8x8-window SSIM
 *          (2 mx my + C1)(2 sxy + C2) / ((mx^2 + my^2 + C1)(sx^2 + sy^2 + C2)),
 *          population moments, C1 = 0.01^2, C2 = 0.03^2
 *   L_ba = L_c + lambda_depth L_d + lambda_ssim (1 - SSIM)      (no silhouette gate)
 * Writes the upstream gradients of csplat_render_bwd on the whole image
 * (d_color [3][H][W], d_depth, d_silhouette [H][W]; zero off the patches)
 * and ADDS its shares of (L_c, L_d, SSIM) to loss3_dev[0..2] (device float;
 * the caller zeroes it per sample).  Inputs: the rendered color / depth of
 * csplat_render_fwd and the observed images, all device float32. */
int csplat_ba_patch_loss(const float *color, const float *depth, const float *obs_color,
                         const float *obs_depth, const csplat_camera *cam, const int32_t *patches,
                         int64_t n_patches, int64_t n_rays, const uint64_t *n_valid_dev,
                         float lambda_depth, float lambda_ssim, float *d_color, float *d_depth,
                         float *d_silhouette, float *loss3_dev, void *stream);

enum csplat_op {
  CSPLAT_OP_BIN_TILES = 1,
  CSPLAT_OP_RENDER_BWD = 2,
  CSPLAT_OP_MASK_PRUNE = 3,
  CSPLAT_OP_TRACKING_LOSS = 4,
  CSPLAT_OP_RVQ_UPDATE = 5,  /* n = L * P codes, pairs = d */
  CSPLAT_OP_MASK_LOSS = 6,
  CSPLAT_OP_KEYFRAME_OVERLAP = 7  /* n = K */
};

/* Scratch bytes needed by `op` for n Gaussians / pair_capacity pairs. */
size_t csplat_workspace_bytes(int op, int64_t n, int64_t pair_capacity, const csplat_camera *cam);

/* Copies the calling thread's last error text into buf (host); returns its length. */
int csplat_last_error(char *buf, size_t len);
const char *csplat_status_string(int status);
/* ABI version (major << 16 | minor). */
int csplat_version(void);

/* The composed entry points (csplat_project_bin_render, csplat_render_step,
 * csplat_tracking_step) fork their tile chunks onto library streams: one set
 * of streams and events per (calling host thread, device), created on that
 * thread's first composed call and destroyed at thread exit or by this call.
 * Per-thread sets mean concurrent callers never share a fork/join event.
 * These are the only resources the library keeps between calls (it never
 * retains caller memory).  Call only when the thread has no composed call in
 * flight (e.g. after synchronising its streams).  Returns CSPLAT_OK. */
int csplat_release_thread_resources(void);

#ifdef __cplusplus
}
#endif
#endif
