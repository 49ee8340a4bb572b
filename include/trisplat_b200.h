/*
 * trisplat_b200.h -- C ABI of the B200-native triangle-splat rasterizer.
 *
 * Drop-in boundary for the reference package's Python operator API (the
 * reference has no FFI; these entry points are what its Python surface
 * binds):
 *
 *   ts_forward    replaces render()                     render.py:364-432
 *                 (project_scene render.py:253-312, build_tile_lists
 *                  render.py:349-361, rasterize_forward _kernels.py:59-132,
 *                  stats reduction render.py:411-418)
 *   ts_backward   replaces render_backward()            backward.py:93-211
 *                 (rasterize_backward _kernels.py:181-318, _phis_q_grad
 *                  backward.py:59-90, chain backward.py:158-210)
 *   ts_debug_copy exposes project_scene / build_tile_lists internals for
 *                 parity dumps (render.py:134-156, 349-361)
 *
 * Conventions: plain pointers and sizes, no framework types.  All array
 * arguments are DEVICE pointers (CUDA), outputs are caller-allocated, every
 * call is ordered on the given stream.  Functions return 0 on success or a
 * negative TS_ERR_* code; ts_error_string() names it.  A context owns its
 * scratch memory and the state of its last forward pass; it is safe to use
 * one context per host thread / stream.  Input validation mirrors the
 * reference: non-finite parameters are reported per group (vertices,
 * opacity, sigma, sh) as the first offending triangle index
 * (soup.py:67-77) through ts_forward_result.err_index.
 */
#ifndef TRISPLAT_B200_H
#define TRISPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_OK 0
#define TS_ERR_INVALID_ARG -1
#define TS_ERR_CUDA -2
#define TS_ERR_OOM -3
#define TS_ERR_NO_FORWARD -4
#define TS_ERR_NONFINITE -5
#define TS_ERR_TILE_SIZE -6
#define TS_ERR_FRAGMENTS -7
#define TS_ERR_NO_BWD_STATE -8
#define TS_ERR_CAPACITY -9

/* geometry.py:32-74: intrinsics + world->camera pose x_cam = R x + t */
typedef struct ts_camera {
    double fx, fy, cx, cy, z_near;
    double R[9]; /* row-major */
    double t[3];
    int32_t width, height;
} ts_camera;

typedef struct ts_options {
    int32_t mode;       /* 0 = NORMALIZED, 1 = SIGMOID (geometry.py:25-29) */
    int32_t sh_degree;  /* active SH degree 0..3 (render.py:300) */
    int32_t tile_size;  /* must be 16 */
    int32_t solid;      /* soup.solid: opacity treated as 1 (render.py:262) */
    double tau_cutoff;  /* bbox cutoff, default 1/255 (geometry.py:22) */
    double tau_contrib; /* pixel-count floor, default 1/255 (render.py:27) */
    double background[3];
    int32_t precision;   /* 0 = fast fp32 path with fp64 guard-band fix-up, 1 = exact fp64 */
    int32_t param_dtype; /* 0 = float32 parameters, 1 = float64 parameters */
    int32_t validate;    /* 1 = non-finite check (soup.py:67-77), 0 = skip */
    int32_t keep_backward; /* 1 = also store the per-triangle state ts_backward needs */
} ts_options;

/* Triangle soup parameters (soup.py:17-30), device pointers, SoA blocks:
 * vertices (N,3,3), opacity (N), sigma (N), sh (N,16,3) band-major. */
typedef struct ts_soup {
    const void* vertices;
    const void* opacity;
    const void* sigma;
    const void* sh;
    int64_t n;
} ts_soup;

/* RenderOutput (render.py:84-91).  Any pointer may be NULL to skip it. */
typedef struct ts_forward_out {
    float* image;        /* (H,W,3) clipped to [0,1] */
    float* alpha_map;    /* (H,W) */
    float* max_weight;   /* (N) per_triangle_max_weight */
    int32_t* pixel_count;/* (N) per_triangle_pixel_count */
    float* area;         /* (N) per_triangle_area (0 if culled) */
    int32_t* last_src;   /* (H,W) source id of the last composited fragment, -1 if none */
    int32_t* n_frag;     /* (H,W) composited fragments per pixel */
} ts_forward_out;

/* Host-side summary of a forward pass, filled by ts_forward. */
typedef struct ts_forward_result {
    int64_t n_visible;    /* M: accepted triangles */
    int64_t n_entries;    /* E: tile entries */
    int64_t n_flagged;    /* pixels re-resolved by the fp64 guard-band fix-up */
    int64_t err_index[4]; /* first non-finite triangle per group, -1 if none */
} ts_forward_result;

/* GradientSet (backward.py:24-56), device pointers, float32. */
typedef struct ts_grads {
    float* d_vertices; /* (N,3,3) */
    float* d_opacity;  /* (N) */
    float* d_sigma;    /* (N) */
    float* d_sh;       /* (N,16,3) */
} ts_grads;

typedef struct ts_context ts_context;

int ts_context_create(ts_context** out, int device);
int ts_context_destroy(ts_context* ctx);
const char* ts_error_string(int code);
const char* ts_version(void);

/* render(): project, cull, depth-sort, bin, composite.  Every stage is sized
 * from host capacities and the device counters of the projection, so the
 * whole frame is enqueued without a host round trip; the call then
 * synchronizes the stream once to fill *result and report non-finite input
 * (and, if the tile entries outgrew their buffer, redoes binning + blend). */
int ts_forward(ts_context* ctx, const ts_camera* cam, const ts_options* opt, const ts_soup* soup,
               const ts_forward_out* out, ts_forward_result* result, void* stream);

/* Asynchronous forwards: with ts_set_async(ctx, 1), ts_forward returns after
 * enqueueing the frame (result fields set to -1, no error report).
 * ts_forward_status synchronizes the stream, fills *result for the last
 * forward and returns its status: TS_ERR_NONFINITE (validate=1),
 * TS_ERR_CAPACITY if its tile entries outgrew the context's buffer (the frame
 * must be repeated; the next forward allocates enough), else TS_OK.  An
 * overflow is also reported without polling: the overflow flag lives in
 * mapped page-locked memory and the next asynchronous ts_forward returns
 * TS_ERR_CAPACITY (enqueuing nothing) once the device has raised it; the
 * caller then calls ts_forward_status and repeats the affected frames. */
int ts_set_async(ts_context* ctx, int enable);
int ts_forward_status(ts_context* ctx, ts_forward_result* result, void* stream);

/* Cross-check paths (tests): the defaults are the product path.
 *   TS_OPT_LEGACY_BINNING  1: global depth radix sort + tile duplication + stable
 *                          tile sort (render.py:275-277, 315-361 literally)
 *                          instead of tile-first binning with per-tile sorts.
 *   TS_OPT_TILE_BACKWARD   1: the tile backward (per-pixel back-to-front
 *                          recursion, _kernels.py:245-318) instead of the
 *                          streaming backward over the training forward's
 *                          fragment records (it is also the automatic fallback
 *                          when the record buffer overflows). */
enum { TS_OPT_LEGACY_BINNING = 1, TS_OPT_TILE_BACKWARD = 2 };
int ts_set_option(ts_context* ctx, int option, int64_t value);

/* render_backward(): gradients of sum(d_image * image_unclipped) w.r.t. all
 * 59 parameters of every triangle, for the scene of the context's last
 * ts_forward (same soup/camera/options).  The soup parameter buffers passed
 * to that ts_forward are read again here: they must stay allocated and
 * unmodified until ts_backward returns.  d_image is (H,W,3) float32.
 * accumulate=1 adds into the gradient buffers, 0 overwrites them. */
int ts_backward(ts_context* ctx, const float* d_image, const ts_grads* grads, int accumulate,
                void* stream);

/* ts_backward with the final chain to the 59 parameter gradients split into
 * n_chunks triangle ranges [bounds[k], bounds[k+1]) (host int64[n_chunks+1]:
 * bounds[0] = 0, bounds[n_chunks] = N, every bounds[k < n_chunks] a multiple
 * of 64), recording the caller's CUDA event events[k] (cudaEvent_t) on the
 * stream once range k's gradients are final.  A view-parallel trainer makes
 * its collective stream wait on events[k] and all-reduces that bucket while
 * the next range computes. */
int ts_backward_chunked(ts_context* ctx, const float* d_image, const ts_grads* grads, int accumulate, int n_chunks,
                        const int64_t* bounds, void* const* events, void* stream);

/* Deferred chain for training steps over several views of one soup (SURVEY
 * 8e: the batch gradient is the sum of the views' render_backward results).
 * ts_backward_screen runs the blend backward of the last ts_forward (a
 * training forward, fast path, fp32 parameters) into the next of up to
 * TS_MAX_CHAIN_VIEWS (8) pending-view slots, keeping the view's camera and
 * cull flags; ts_chain_views then chains every pending view to the 59
 * parameter gradients in one pass (one read of the parameters and one
 * read-add-write of grads for all of them, instead of one per view) and empties
 * the slots.  Equivalent to ts_backward on each view in turn with accumulate=1
 * after the first (the per-view fp64 vertex / opacity / sigma terms are summed
 * before their single fp32 rounding).  The soup buffers must stay unmodified
 * until ts_chain_views returns; n_chunks / bounds / events as in
 * ts_backward_chunked (0 / NULL / NULL for one pass).  ts_pending_views returns
 * the number of filled slots.  TS_ERR_INVALID_ARG: slots full, a different soup
 * or mode than the pending views, exact precision or fp64 parameters;
 * TS_ERR_NO_BWD_STATE from ts_chain_views: no pending view. */
int ts_backward_screen(ts_context* ctx, const float* d_image, void* stream);
int ts_chain_views(ts_context* ctx, const ts_grads* grads, int accumulate, int n_chunks, const int64_t* bounds,
                   void* const* events, void* stream);
int ts_pending_views(ts_context* ctx);

/* Two-phase allocation: size every per-frame buffer of the context for scenes of
 * up to n triangles at width x height (entries: expected tile entries, <= 0:
 * 4 per triangle; keep_backward: also the training forward's records, the
 * fragment-record buffer for 8 fragments per entry and the backward's
 * screen-space rows), so later ts_forward / ts_backward calls of that size
 * allocate nothing.  ts_workspace_bytes: device bytes the context holds. */
int ts_reserve(ts_context* ctx, int64_t n, int width, int height, int64_t entries, int keep_backward);
int64_t ts_workspace_bytes(ts_context* ctx);

/* Host helper of the drop-in upload: dst[i] = (float)src[i] for i < n on a
 * persistent pool of up to `threads` host threads (<= 0: all, at most 16).
 * Returns 1 if every value converted exactly (the fp64 array holds fp32 values,
 * e.g. the reference's synthetic soups, which round every parameter to fp32),
 * 0 if not (dst then holds the rounded values), TS_ERR_INVALID_ARG for bad
 * arguments.  render() uploads such soups as fp32 -- half the PCIe bytes, the
 * same values -- and fp64 otherwise. */
int ts_pack_f32(const double* src, float* dst, int64_t n, int threads);

/* The whole lossless upload in one call: src (host fp64, n values) -> dst
 * (device fp32) on `stream`, chunk by chunk through a small ring of page-locked
 * slots (nslot slots of chunk_bytes; <= 0: 4 x 4 MB) on the current device; the
 * conversion of a chunk (ts_pack_f32's thread pool) overlaps the DMA of the
 * previous one.  flags bit 0: streaming (non-temporal) stores into the slots.
 * Returns 1 when every value was an fp32 value (dst is complete once `stream`
 * reaches the copies), 0 when one was not (the copies issued so far have
 * finished, dst is incomplete: upload fp64 instead), < 0 on error. */
int ts_upload_f32(const double* src, int64_t n, float* dst, void* stream, int64_t chunk_bytes, int nslot,
                  int flags);

/* Fragment lists of the last ts_forward: render(collect_fragments=True)
 * (render.py:383-399, 420-425; count_fragments _kernels.py:135-178,
 * collect branch _kernels.py:107-116).
 *  ts_fragment_offsets   CSR offsets (int64, H*W+1; pixel p owns
 *                        offsets[p]:offsets[p+1]) into `offsets` (device,
 *                        may be NULL) and the fragment total F into
 *                        *n_fragments (host).  Synchronizes the stream.
 *  ts_collect_fragments  fills triangle (int32 source ids), weight (float64
 *                        T*alpha) and depth (float64 camera-space z) of the F
 *                        fragments in compositing order (device arrays of F
 *                        elements, offsets as returned above).  Fast path
 *                        (precision 0) only. */
int ts_fragment_offsets(ts_context* ctx, int64_t* offsets, int64_t* n_fragments, void* stream);
int ts_collect_fragments(ts_context* ctx, const int64_t* offsets, int32_t* triangle, double* weight,
                         double* depth, void* stream);

/* render_backward(frag_grads=(offsets, d_weight, d_depth)) (backward.py:122-142,
 * _kernels.py:262-272): ts_backward plus upstream gradients on the blend
 * weight and depth of every fragment of the last forward, in the CSR layout
 * of ts_fragment_offsets (device arrays).  A layout that differs from this
 * scene/camera returns TS_ERR_FRAGMENTS.  Needs a keep_backward forward on
 * the fast path.  weight (nullable): the fragments' blend weights of this
 * forward (ts_collect_fragments' weight array); with it the gradient streams
 * over the forward's fragment records (per-pixel suffix sums of d_weight *
 * weight from the CSR), without it the tile backward replays every pixel. */
int ts_backward_fragments(ts_context* ctx, const float* d_image, const int64_t* offsets, const double* weight,
                          const double* d_weight, const double* d_depth, const ts_grads* grads,
                          int accumulate, void* stream);

/* Photometric loss (losses.py:122-142): (1-lambda) L1 + lambda (1-SSIM)/2 of
 * two H x W x 3 fp32 images on the device (11x11 Gaussian window, sigma 1.5;
 * the SSIM term is 0 below the window size, skipped for lambda == 0).
 * out: device double[2] = {loss, mean SSIM}; d_image (nullable): device
 * float[H*W*3], the gradient of the loss w.r.t. rendered.  Ordered on the
 * stream; the context supplies the scratch. */
int ts_photometric_loss(ts_context* ctx, const float* rendered, const float* target, int height, int width,
                        double lambda_dssim, double* out, float* d_image, void* stream);
/* Mean SSIM over channels (losses.py:110-119) into out[1] (device double[2]). */
int ts_ssim(ts_context* ctx, const float* x, const float* y, int height, int width, double* out, void* stream);

/* Distortion loss (losses.py:169-203) over fragment lists in the CSR layout of
 * ts_fragment_offsets / ts_collect_fragments (device arrays; n_pixels + 1
 * offsets, fp64 weight / depth): out (device double[1]) = value averaged over
 * image_size pixels (n_pixels if <= 0); d_weight / d_depth (nullable, device
 * double[F]).  Sorted runs use the prefix-sum form, unsorted ones the pairwise
 * form. */
int ts_distortion_loss(ts_context* ctx, const int64_t* offsets, const double* weight, const double* depth,
                       int64_t n_pixels, int64_t image_size, double* out, double* d_weight, double* d_depth,
                       void* stream);
/* Normal loss (losses.py:219-292) of fp32 device vertices (N,3,3) against the
 * normals of a device fp64 depth map (H x W = cam->height x cam->width) for the
 * fragment lists (offsets of H*W+1, triangle ids int32, weights fp64, F
 * fragments): out (device double[1]) = mean over fragments of w (1 - n.N);
 * d_vertices (nullable, device double[N*9]); d_weight (nullable, device
 * double[F]).  Depth normals are held fixed (as in the reference). */
int ts_normal_loss(ts_context* ctx, const float* vertices, int64_t n, const int64_t* offsets,
                   const int32_t* triangle, const double* weight, int64_t n_fragments, const double* depth,
                   const ts_camera* cam, double* out, double* d_vertices, double* d_weight, void* stream);
/* depth_from_fragments (losses.py:206-216): device double[n_pixels]. */
int ts_fragment_depth(ts_context* ctx, const int64_t* offsets, const double* weight, const double* depth,
                      int64_t n_pixels, double* out_depth, void* stream);

/* Adam step (training.py:81-110) in place on fp32 device parameters
 * (vertices (N,3,3), opacity (N), sigma (N), sh (N,16,3)) with the gradients
 * of ts_backward; m, v: device fp32 moments of 59 N elements in the flat
 * gradient layout [vertices | opacity | sigma | sh], zero-initialised by the
 * caller; t: device int64[1], the steps taken so far (AdamState.t): this
 * step uses t + 1 for the bias correction and t is incremented only if the
 * update ran (no non-finite gradient); lrs: host
 * double[4] per-group rates; bad: device int64[4] receiving, per group, the
 * first triangle with a non-finite gradient (-1 if none) -- if any
 * group has one, nothing is updated (the reference raises ValueError). */
int ts_adam_step(ts_context* ctx, float* vertices, float* opacity, float* sigma, float* sh, int64_t n,
                 const ts_grads* grads, float* m, float* v, int64_t* t, const double* lrs, int64_t* bad,
                 void* stream);

/* ---------------- adaptive density control (density.py:27-263) ----------------
 * The array work of ViewStats / prune / sample_candidates / midpoint_subdivide /
 * clone_with_noise on device-resident triangles; the sequential pick loop of
 * densify_step (a prefix sum over the picks' costs) and the numpy random draws
 * stay with the caller.  dtype: 0 = float32 parameters, 1 = float64.  Index
 * arrays are device int64.  pool / kept may be NULL (identity). */
#define TS_SAMPLE_INVERSE_SIGMA 0
#define TS_SAMPLE_OPACITY 1
/* ViewStats.update + aggregation (density.py:42-71): fold one view's forward
 * statistics (ts_forward_out max_weight / pixel_count / area) into acc_*
 * (device double[N] max weight, int32[N] views with pixel_count >= min_pixels,
 * double[N] area sum); first != 0 initialises them.  Call per view in the
 * order the views were first recorded. */
int ts_view_stats_accumulate(ts_context* ctx, int64_t n, const float* max_weight, const int32_t* pixel_count,
                             const float* area, int min_pixels, int first, double* acc_max_weight,
                             int32_t* acc_views, double* acc_area, void* stream);
/* prune (density.py:74-94): flags (device uint8[N]) bit 0 max weight < tau_prune,
 * bit 1 views < min_views, bit 2 opacity < opacity_dead; kept (device int64[N])
 * receives the unflagged indices in order, n_kept (device int64[1]) their count. */
int ts_prune_mark(ts_context* ctx, int64_t n, const double* acc_max_weight, const int32_t* acc_views,
                  const void* opacity, int dtype, double tau_prune, int min_views, double opacity_dead,
                  uint8_t* flags, int64_t* kept, int64_t* n_kept, void* stream);
/* sample_candidates (density.py:103-120): weights of the pool members
 * (member k is triangle kept[pool[k]]) from param (sigma for
 * TS_SAMPLE_INVERSE_SIGMA, opacity for TS_SAMPLE_OPACITY), keys =
 * exponential[k] / max(w, 1e-300) (device double[n_pool], the caller's
 * rng.exponential(size=n_pool)), picked (device int64[count]) = the first count
 * positions of the stable ascending order of the keys (pool-local indices). */
int ts_sample_candidates(ts_context* ctx, int64_t n_pool, const int64_t* pool, const int64_t* kept,
                         const void* param, int dtype, int criterion, const double* exponential, int64_t count,
                         int64_t* picked, void* stream);
/* Per pick (device int64[count] pool-local): source triangle kept[pool[picked]],
 * its mean area acc_area / max(n_views, 1) and whether |(v1-v0) x (v2-v0)| < 1e-12
 * (density.py:130-131, 154-157). */
int ts_pick_info(ts_context* ctx, int64_t count, const int64_t* picked, const int64_t* pool, const int64_t* kept,
                 const double* acc_area, int64_t n_views, const void* vertices, int dtype, int64_t* source,
                 double* mean_area, uint8_t* degenerate, void* stream);
/* dst[r, :] = src[origin[r], :] (zeros where origin[r] < 0) for rows of width
 * elements of elem_bytes (4 or 8): TriangleSoup.select / AdamState.remap
 * (soup.py select, training.py:64-78). */
int ts_gather_rows(ts_context* ctx, int64_t n_out, const int64_t* origin, const void* src, void* dst, int width,
                   int elem_bytes, void* stream);
/* Children vertices (density.py:123-171): code[k] in 0..3 -> subdivision corner
 * of parent[k]; code[k] = 4 + r -> clone jittered in the parent's plane with
 * uniforms[6r..6r+5] (angle / 2 pi, radius / (max_noise_factor * mean edge) per
 * vertex, the caller's rng.uniform draws in order); code < 0 -> left as is. */
int ts_child_vertices(ts_context* ctx, int64_t n_child, const int64_t* parent, const int32_t* code,
                      const double* uniforms, double max_noise_factor, const void* src_vertices, void* dst_vertices,
                      int dtype, void* stream);

/* ---------------- model I/O: binary PLY body (scene_io.py:365-455) ----------------
 * ts_ply_pack: the body of export_mesh(..., "ply") for N triangles (vertices
 * (N,3,3), sh (N,16,3), dtype 0 f32 / 1 f64): vertex_bytes (device, 45 N bytes,
 * 16-byte aligned) = 3 N records {float x,y,z; uchar r,g,b} with the quantised
 * degree-0 colour, face_bytes (device, 16 N bytes, 16-byte aligned) = N records
 * {int 3; int 3i,3i+1,3i+2}.  The header is the caller's (ASCII, scene_io.py:384-396).
 * ts_ply_unpack: import_ply's body decode for n_face faces over n_vertex vertex
 * records: vertices from the face indices, SH DC from the first vertex's colour,
 * opacity 1, sigma given, other SH 0.  bad (device uint64[1]) = all ones if the
 * body is valid, else (1 << 62 | face) for the first face whose count is not 3,
 * or (2 << 62 | face) for the first out-of-range index when every count is 3. */
int ts_ply_pack(ts_context* ctx, const void* vertices, const void* sh, int dtype, int64_t n, uint8_t* vertex_bytes,
                void* face_bytes, void* stream);
int ts_ply_unpack(ts_context* ctx, const uint8_t* vertex_bytes, int64_t n_vertex, const void* face_bytes,
                  int64_t n_face, double sigma, int dtype, void* vertices, void* opacity, void* sigma_out, void* sh,
                  uint64_t* bad, void* stream);

/* Debug/parity dumps of the last forward pass (device destination):
 *  TS_DUMP_SORTED_IDX  int32[M]       depth-sorted source ids (render.py:275-277)
 *  TS_DUMP_TILE_START  int32[T+1]     CSR tile offsets (render.py:355-357)
 *  TS_DUMP_ENTRY_RANK  int32[E]       tile entries as depth ranks (render.py:358-360)
 *  TS_DUMP_BBOX        int32[N*4]     x0,x1,y0,y1 per source (0s if culled) (render.py:243-250)
 *  TS_DUMP_DEPTH       float64[N]     camera-space centroid depth per accepted source (0 if culled)
 *  TS_DUMP_SGRAD       float64[N*16]  screen-space gradients of the last ts_backward
 *                                     (gq[6], go, gsig, grgb[3], gphis, gz, pad) per source */
#define TS_DUMP_SORTED_IDX 1
#define TS_DUMP_TILE_START 2
#define TS_DUMP_ENTRY_RANK 3
#define TS_DUMP_BBOX 4
#define TS_DUMP_DEPTH 5
#define TS_DUMP_SGRAD 6
/*  TS_DUMP_FRAGREC uint64 count, then count x 48-byte fragment records of the
 *                  last training forward (T, C[3] fp64; pixel, source, ordinal u32) */
#define TS_DUMP_FRAGREC 7
/*  TS_DUMP_PROJECTION float64[M*64 + N]: project_scene (render.py:253-312) of the
 *                  last forward, one row of 64 per depth-sorted accepted triangle:
 *                  xc[9] q[6] z area phis nrm[6] doff[3] esign[3] sig opa rgb[3]
 *                  raw_rgb[3] basis[16] viewdir[3] u_norm bbox[4] (2 pad), in the
 *                  reference's fp64 operation order; then area_full[N] */
#define TS_DUMP_PROJECTION 8
int ts_debug_copy(ts_context* ctx, int what, void* dst, size_t bytes, void* stream);

/* build_tile_lists (render.py:315-361) for any tile size >= 1: bbox is the
 * device int64 (M x 4) x0,x1,y0,y1 of M triangles in depth-rank order; writes
 * the device CSR tile_start (int64[ntx*nty+1]) and entry_tri (int64[E], ranks;
 * each tile's list in rank order) and *n_entries = E.  With tile_start or
 * entry_tri null it only returns E (size query).  Synchronises the stream. */
int ts_tile_lists(ts_context* ctx, const int64_t* bbox, int64_t m, int tile_size, int width, int height,
                  int64_t* tile_start, int64_t* entry_tri, int64_t* n_entries, void* stream);

/* Per-stage device timing with CUDA events recorded on the call's stream.
 * ts_profile(ctx, 1) enables it; ts_stage_times fills ms[TS_NUM_STAGES] with
 * the durations of the last ts_forward / ts_backward stages (0 if not run). */
#define TS_STAGE_PREPROCESS 0
#define TS_STAGE_DEPTH_SORT 1
#define TS_STAGE_BINNING 2
#define TS_STAGE_BLEND 3
#define TS_STAGE_FIXUP 4
#define TS_STAGE_BLEND_BWD 5
#define TS_STAGE_CHAIN_BWD 6
#define TS_NUM_STAGES 7
int ts_profile(ts_context* ctx, int enable);
int ts_stage_times(ts_context* ctx, float* ms, int n);

/* Pixels of the last fast-path ts_forward whose guard band required the
 * exact fix-up (valid once the forward's stream has been synchronized). */
int ts_flagged_pixels(ts_context* ctx, int64_t* n_flagged);

/* Kernel launches issued by this library since load (for launch counting). */
int64_t ts_launch_count(ts_context* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TRISPLAT_B200_H */
