/*
 * lidarsplat_cuda.h -- C ABI of the B200 (sm_100a) per-frame rendering path.
 *
 * Replaces the reference's operator boundary, the `_kernels` backend protocol
 * (/root/reference/pkg/src/lidarsplat/_kernels/__init__.py:15-50) whose
 * implementations are _native.pyx:19-297 / _numpy.py:20-183, plus the fused
 * per-frame fast path that render.py / filtering.py / bridge.py drive.
 *
 * Conventions (all entry points):
 *   - every pointer argument named d_* is DEVICE memory owned by the caller;
 *     h_* / fixed-size arrays are HOST memory read during the call only;
 *   - every call is asynchronous on `stream` (a cudaStream_t, NULL = legacy);
 *   - return 0 on success, LS_EINVAL for bad arguments (nothing launched),
 *     otherwise the cudaError_t of the failing launch;
 *   - the library never allocates or frees caller memory and holds no global
 *     mutable state: calls are re-entrant per stream (the reference kernels
 *     are called concurrently from a ThreadPoolExecutor, render.py:121-141).
 */
#ifndef LIDARSPLAT_CUDA_H
#define LIDARSPLAT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LS_EINVAL (-22)
#define LS_TILE_POINTS 128          /* points per warp tile of the frame passes */
#define LS_PACKED_COUNT_LIMIT 65793u /* 255*count < 2^24 => f32 accumulator sums exact */

/* Pinhole camera + pose, values exactly as CameraModel holds them
 * (geometry.py:62-108): rot row-major world->camera, p_c = R p + t. */
typedef struct ls_camera {
    double rot[9];
    double t[3];
    double fx, fy, cx, cy;
    int64_t width, height;
    double z_near, z_far;
} ls_camera;

/* Device-resident scan: the grid's cell-major arrays (grid.py:25-41) plus the
 * per-scan tile index that lets the frame passes skip culled cells. */
typedef struct ls_scene {
    const float *d_positions;    /* (n_points,3) f32, cell-major, 16 B aligned       */
    const uint8_t *d_colors;     /* (n_points,3) u8, cell-major, 4 B aligned         */
    int64_t n_points;
    const int64_t *d_occ_cells;  /* (n_occ,) ascending occupied cell ids             */
    const int64_t *d_occ_offsets;/* (n_occ+1,) point offset of each occupied cell    */
    int64_t n_occ;
    const int32_t *d_tile_c0;    /* (n_tiles,) first occupied cell touching tile t   */
    const int32_t *d_tile_c1;    /* (n_tiles,) last occupied cell touching tile t    */
    int64_t n_tiles;             /* ceil(n_points / LS_TILE_POINTS)                  */
    double origin[3];
    double cell_size;
    int64_t dims[3];
} ls_scene;

/* Depth-filter knobs (filtering.py:25-46 FilterParams). */
typedef struct ls_filter_params {
    int32_t levels_n;
    double filter_strength;
    double edge_threshold;
} ls_filter_params;

int ls_version(void);
const char *ls_status_string(int status);

/* ------------------------------------------------------------------------
 * (i) Device-pointer twins of the 8 `_kernels` functions.
 * ---------------------------------------------------------------------- */

/* _native.pyx:19-44 assign_cells: ids[k] = (ix*dy+iy)*dz+iz, clamp(floor((p-o)/cell)) */
int ls_assign_cells(const float *d_positions, int64_t n, const double origin[3],
                    double cell_size, const int64_t dims[3], int64_t *d_ids, void *stream);

/* _native.pyx:47-68 counting_sort: stable; offsets (n_cells+1), order (n). */
size_t ls_counting_sort_workspace(int64_t n, int64_t n_cells);
int ls_counting_sort(const int64_t *d_ids, int64_t n, int64_t n_cells, int64_t *d_offsets,
                     int64_t *d_order, void *d_workspace, size_t workspace_bytes, void *stream);

/* Candidate ranges [starts_r, ends_r) enumerate k = 0..n-1 in range order
 * (render.py:84-143).  Both projection twins need n_ranges+1 int64 of
 * workspace for the range prefix. */
size_t ls_ranges_workspace(int64_t n_ranges);

/* _native.pyx:71-121 project_min_depth: minz (f64, H*W) inout, pix_cache (i64,
 * -1 = rejected) and z_cache (f64) out, indexed by candidate order k. */
int ls_project_min_depth(const float *d_positions, const int64_t *d_starts,
                         const int64_t *d_ends, int64_t n_ranges, const ls_camera *cam,
                         double *d_minz, int64_t *d_pix_cache, double *d_z_cache,
                         void *d_workspace, size_t workspace_bytes, void *stream);

/* _native.pyx:124-148 project_accumulate: accum (u64, H*W x 4) inout. */
int ls_project_accumulate(const uint8_t *d_colors, const int64_t *d_starts,
                          const int64_t *d_ends, int64_t n_ranges, const int64_t *d_pix_cache,
                          const double *d_z_cache, double eps_rel, const double *d_minz,
                          uint64_t *d_accum, void *d_workspace, size_t workspace_bytes,
                          void *stream);

/* _native.pyx:151-170 min_pool_2x2: out is ceil(h/2) x ceil(w/2). */
int ls_min_pool_2x2(const float *d_img, int64_t h, int64_t w, float *d_out, void *stream);

/* _native.pyx:173-196 laplacian_edges: out u8 (h,w). */
int ls_laplacian_edges(const float *d_img, int64_t h, int64_t w, double threshold,
                       uint8_t *d_out, void *stream);

/* _native.pyx:199-237 filter_keep: out f32 (fh,fw), +inf where dropped. */
int ls_filter_keep(const float *d_coarse, int64_t ch, int64_t cw, const uint8_t *d_edges,
                   const float *d_fine, int64_t fh, int64_t fw, double filter_strength,
                   float *d_out, void *stream);

/* _native.pyx:240-297 bilinear_fill: out f32 (fh,fw). */
int ls_bilinear_fill(const float *d_coarse, int64_t ch, int64_t cw, const float *d_fine,
                     int64_t fh, int64_t fw, float *d_out, void *stream);

/* render.py:146-161 assemble_frame from the exact (u64 x 4) accumulators. */
int ls_assemble(const double *d_minz, const uint64_t *d_accum, int64_t n_pixels, float *d_rgb,
                float *d_depth, uint8_t *d_alpha, void *stream);

/* ------------------------------------------------------------------------
 * (ii) Fused per-frame fast path (what project_points / depth_filter /
 *      the render service run on a device-resident scan).
 * ---------------------------------------------------------------------- */

/* Device-scan order (internal to the fast path; the public grid fields keep
 * the reference's stable order): d_order receives the permutation that sorts
 * points by (cell id, 30-bit Morton code of the in-cell position).  Applied
 * to cell-major points it keeps every cell's range and makes each warp tile
 * spatially compact.  Workspace: ls_morton_order_workspace(n, n_cells). */
size_t ls_morton_order_workspace(int64_t n, int64_t n_cells);
int ls_morton_order(const float *d_positions, int64_t n, const double origin[3],
                    double cell_size, const int64_t dims[3], int64_t *d_order, void *d_workspace,
                    size_t workspace_bytes, void *stream);

/* Gather the cloud into cell-major order (grid.py:126-127). */
int ls_gather_points(const float *d_positions, const uint8_t *d_colors, const int64_t *d_order,
                     int64_t n, float *d_sorted_positions, uint8_t *d_sorted_colors,
                     void *stream);

/* Occupied cells of a grid from its cell_offsets (grid.py:47-48):
 * writes ids ascending + their point offsets; *d_n_occ receives the count.
 * Workspace: ls_occupied_workspace(n_cells). */
size_t ls_occupied_workspace(int64_t n_cells);
int ls_occupied_cells(const int64_t *d_cell_offsets, int64_t n_cells, int64_t *d_occ_cells,
                      int64_t *d_occ_offsets, int64_t *d_n_occ, void *d_workspace,
                      size_t workspace_bytes, void *stream);

/* Per-scan tile index: d_tile_c0/c1 for tiles of LS_TILE_POINTS points. */
int ls_scene_tile_index(const int64_t *d_occ_offsets, int64_t n_occ, int64_t n_points,
                        int32_t *d_tile_c0, int32_t *d_tile_c1, void *stream);

/* grid.py:131-151 cull_cells: CULL_SLACK-inflated p-vertex test of every
 * occupied cell against the six frustum planes (h_planes (6,4) f64 row-major,
 * geometry.py:134-158).  Warp ballots pack the verdicts into d_keep_bits
 * (ceil(n_occ/32) u32 words, bit j = cell j kept). */
int ls_cull(const ls_scene *scene, const double h_planes[24], double slack,
            uint32_t *d_keep_bits, void *stream);

/* Ordered (ascending) compaction of the kept cell ids, identical to the
 * reference's cull_cells return value.  *d_count receives the count.
 * Workspace: ls_compact_workspace(n_occ). */
size_t ls_compact_workspace(int64_t n_occ);
int ls_cull_compact(const uint32_t *d_keep_bits, const int64_t *d_occ_cells, int64_t n_occ,
                    int64_t *d_out_cells, int64_t *d_count, void *d_workspace,
                    size_t workspace_bytes, void *stream);

/* Per-frame work list of the non-culled warp tiles (after ls_cull): d_list
 * receives one u32 per tile that keeps any point (bit 31 = tile straddles a
 * culled cell), d_count (1 u32, reset by this call) their number.  d_list
 * must hold n_tiles entries. */
int ls_tile_worklist(const ls_scene *scene, const uint32_t *d_keep_bits, uint32_t *d_list,
                     uint32_t *d_count, void *stream);

/* Both projection passes over the culled scan.  d_keep_bits NULL = no cull
 * (every point is a candidate; d_list/d_count are then ignored), else the
 * work list is built first (ls_tile_worklist).
 * d_minz_bits: (H*W) u64, the f64 bit pattern of the running minimum,
 *   must hold +inf (0x7FF0000000000000) on entry.
 * d_cache: NULL (pass 2 re-projects every candidate), or
 *   ls_frame_cache_bytes(scene) bytes of 16 B aligned scratch: pass 1 then
 *   records each candidate's pixel and f16-rounded-down depth and pass 2
 *   decides from them (a candidate within one f16 ulp of the soft z-buffer
 *   threshold re-derives its exact f64 depth).  Same frame either way.
 *   Requires W*H < 2^32 - 1.
 * d_accum4: (H*W x 4) f32 accumulators {sum r, sum g, sum b, count}, zero on
 *   entry, one 16 B vector atomic per kept point.  Integer-valued f32 adds
 *   are exact and order-free while every field stays < 2^24 (guaranteed while
 *   no pixel keeps > LS_PACKED_COUNT_LIMIT points); ls_frame_finish flags a
 *   frame where a field reached 2^24. */
int ls_frame_project(const ls_scene *scene, const uint32_t *d_keep_bits, uint32_t *d_list,
                     uint32_t *d_count, const ls_camera *cam, double eps_rel,
                     uint64_t *d_minz_bits, uint32_t *d_cache, float *d_accum4, void *stream);

/* Bytes of the optional pass-1 -> pass-2 cache: 768 B per warp tile
 * ([128 x u32 pixel][128 x f16 depth]). */
size_t ls_frame_cache_bytes(const ls_scene *scene);

/* Pass 1 only / pass 2 only of ls_frame_project over an existing work list
 * (d_list NULL = all tiles); with a cache both passes must see the same list.
 * Multi-GPU: an all-reduce MIN of d_minz_bits runs between them, a reduce SUM
 * of d_accum4 after. */
int ls_frame_pass1(const ls_scene *scene, const uint32_t *d_keep_bits, const uint32_t *d_list,
                   const uint32_t *d_count, const ls_camera *cam, uint64_t *d_minz_bits,
                   uint32_t *d_cache, void *stream);
int ls_frame_pass2(const ls_scene *scene, const uint32_t *d_keep_bits, const uint32_t *d_list,
                   const uint32_t *d_count, const ls_camera *cam, double eps_rel,
                   const uint64_t *d_minz_bits, const uint32_t *d_cache, float *d_accum4,
                   void *stream);

/* Multi-view batched projection (render.py:84-143 project_candidates, run
 * once per view): ONE read of the culled scan's tiles feeds
 * n_views <= LS_MAX_VIEWS cameras of the same width/height.  Every view's
 * frame is bit-identical to ls_frame_project of that view alone (same f64
 * arithmetic, same per-view culling, order-free reductions).
 * d_keep_bits: NULL = no cull, else n_views blocks of bits_stride u32 words,
 *   block v = ls_cull of view v (bits_stride >= ceil(n_occ/32)); the work
 *   list is built over their union: d_list n_tiles entries, d_status n_tiles
 *   u32 (per entry: bit 2v = view v keeps a cell of the tile, bit 2v+1 = view
 *   v also culls one), d_count 1 u32 (reset by the call).
 * d_minz_bits: n_views x (W*H) u64, +inf on entry (view v at v*W*H).
 * d_cache: NULL (pass 2 re-projects), or ls_frame_views_cache_bytes(scene,
 *   n_views) bytes, 16 B aligned: pass 1 records each (candidate, view)'s
 *   pixel and f32-rounded-down depth, pass 2 decides from them (the
 *   ls_frame_project cache rule, per view).  Same frames either way.
 * d_accum4: n_views x (W*H*4) f32, zero on entry; one ls_frame_finish per view
 *   (at the view's offsets) folds them into frames. */
#define LS_MAX_VIEWS 8
/* Re-target a captured frame graph to another camera.  graph / graph_exec
 * are the cudaGraph_t / cudaGraphExec_t of a stream capture of one fused
 * frame (ls_cull, ls_tile_worklist, ls_frame_pass1, ls_frame_pass2, the
 * assembly / filter and U-Net launches); the cull nodes take the new frustum
 * planes (24 doubles, as ls_cull) and the projection-pass nodes the new
 * camera.  Returns 0, LS_EINVAL when the graph holds no such node, or a CUDA
 * error. */
int ls_frame_graph_set_camera(void *graph, void *graph_exec, const ls_camera *cam,
                              const double h_planes[24]);

int ls_tile_worklist_views(const ls_scene *scene, const uint32_t *d_keep_bits,
                           int64_t bits_stride, int32_t n_views, uint32_t *d_list,
                           uint32_t *d_status, uint32_t *d_count, void *stream);
int ls_frame_project_views(const ls_scene *scene, const uint32_t *d_keep_bits,
                           int64_t bits_stride, uint32_t *d_list, uint32_t *d_status,
                           uint32_t *d_count, const ls_camera *cams, int32_t n_views,
                           double eps_rel, uint64_t *d_minz_bits, uint32_t *d_cache,
                           float *d_accum4, void *stream);
size_t ls_frame_views_cache_bytes(const ls_scene *scene, int32_t n_views);

/* Level sizes of the min pyramid (filtering.py:67-83); returns the float
 * count of the workspace ls_frame_finish needs for levels 0..L-1. */
int64_t ls_pyramid_floats(int64_t height, int64_t width, int32_t levels_n);

/* Assemble (render.py:146-161) + depth filter (filtering.py:60-147) + U-Net
 * input prep (weights.ts:90-95 normalizeDepth, bridge.ts:37-44 packing).
 *   in:  d_minz_bits, d_accum4 (consumed and reset to +inf / 0 for the next frame)
 *   out: raw frame d_rgb (H,W,3) f32, d_depth (H,W) f32, d_alpha (H,W) u8
 *        filtered frame d_frgb/d_fdepth/d_falpha (any may be NULL),
 *        d_keep (H,W) u8 mask (may be NULL),
 *        d_unet_in (may be NULL): bf16 NHWC, unet_h rows x W x unet_c channels
 *          [r,g,b,zNear/max(d,zNear),alpha, 0...] of the FILTERED frame,
 *          rows >= H left untouched (caller zero-fills once).
 *   U-Net-only frames: with a filter and d_unet_in, d_rgb / d_alpha may be
 *     NULL when no filtered output is requested either -- the assembly then
 *     writes every pixel's U-Net input and the final filter step clears the
 *     rejected ones (same input, no f32 rgb round trip); d_depth stays required.
 *   d_pyramid: ls_pyramid_floats(H,W,L) floats of scratch.
 *   d_flags: 1 int32; bit0 set if a pixel's accumulator may have lost exactness.
 * filter==NULL skips the filter (raw frame only). */
int ls_frame_finish(uint64_t *d_minz_bits, float *d_accum4, int64_t width, int64_t height,
                    const ls_filter_params *filter, float *d_rgb, float *d_depth,
                    uint8_t *d_alpha, float *d_frgb, float *d_fdepth, uint8_t *d_falpha,
                    uint8_t *d_keep, uint16_t *d_unet_in, int64_t unet_h, int32_t unet_c,
                    double unet_znear, float *d_pyramid, int32_t *d_flags, void *stream);

/* Bridge input (FE:bridge.ts:31-53 UNetBridgeModel.reconstruct + FE:model/
 * weights.ts:90-95 normalizeDepth): d_planes is an RGDA tensor's (5,H,W) f32
 * planes [r, g, b, depth, alpha]; writes the first H*W pixels of the U-Net's
 * bf16 NHWC input, unet_c channels [r, g, b, zNear/max(d,zNear) (0 if d <= 0),
 * alpha, 0...] (unet_c even, >= 6; 16 B aligned when a multiple of 8). */
int ls_unet_pack_rgbda(const float *d_planes, int64_t height, int64_t width, int32_t unet_c,
                       double unet_znear, uint16_t *d_unet_in, void *stream);

/* Depth filter of an arbitrary (H,W) depth image (0 = empty): the keep mask
 * of filtering.py:124-131 filter_depth_image. */
int ls_filter_depth_image(const float *d_depth, int64_t height, int64_t width,
                          const ls_filter_params *filter, uint8_t *d_keep, float *d_pyramid,
                          void *stream);

/* filtering.py:134-147 depth_filter on a device frame: filtered rgb/depth/
 * alpha (multiply-by-mask) and the keep mask; d_pyramid as above. */
int ls_depth_filter_frame(const float *d_rgb, const float *d_depth, const uint8_t *d_alpha,
                          int64_t height, int64_t width, const ls_filter_params *filter,
                          float *d_frgb, float *d_fdepth, uint8_t *d_falpha, uint8_t *d_keep,
                          float *d_pyramid, void *stream);

/* A filter_strength sweep over one device frame (BASELINE configs[3]; the
 * reference runs filtering.py:134-147 once per strength): the strength-
 * independent min-pool pyramid is built once, then every strength's
 * non-final steps run in one launch and every strength's final step in
 * another.  Strength k's keep mask / filtered frame land at plane k of
 * d_keep (K,H,W) / d_frgb (K,H,W,3) / d_fdepth (K,H,W) / d_falpha (K,H,W)
 * (any may be NULL; rgb/alpha inputs are needed only for the filtered
 * frame), each bit-identical to ls_depth_filter_frame at that strength.
 * 1 <= n_strengths <= 16, 1 <= levels_n <= 5; d_work holds
 * ls_filter_sweep_floats(height, width, levels_n, n_strengths) floats. */
int64_t ls_filter_sweep_floats(int64_t height, int64_t width, int32_t levels_n,
                               int32_t n_strengths);
int ls_depth_filter_sweep(const float *d_rgb, const float *d_depth, const uint8_t *d_alpha,
                          int64_t height, int64_t width, int32_t levels_n,
                          double edge_threshold, const double *h_strengths, int32_t n_strengths,
                          float *d_frgb, float *d_fdepth, uint8_t *d_falpha, uint8_t *d_keep,
                          float *d_work, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LIDARSPLAT_CUDA_H */
