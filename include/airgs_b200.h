/*
 * airgs_b200 -- C-ABI of the B200-native AirGS per-frame evaluation path.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * (passed as void*), returns 0 on success or a negative status whose value
 * maps 1:1 onto the reference exception taxonomy
 * (/root/reference/pkg/src/splatstream/errors.py:8-67), and never lets a C++
 * exception cross the boundary.  Output buffers are caller-owned; scratch
 * lives in an opaque per-device context that only grows (no allocation in
 * steady-state hot calls).  Calls are reentrant per context; use one context
 * per host thread / stream.
 *
 * Layouts (HBM):
 *   params    plane-major float64 [width][ld]   (one plane per attribute, the
 *             GSAI layout; row-major (n,width) of the reference is transposed
 *             once at upload)
 *   images    float64 (height, width, 3) row-major, the reference layout
 *   usage     int64 [n] per-primitive counts
 *
 * See INTEGRATION.md for the reference-side bindings.
 */
#ifndef AIRGS_B200_H
#define AIRGS_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define AIRGS_API __attribute__((visibility("default")))
#else
#define AIRGS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:8-67) ------------------------------------ */
#define AIRGS_OK 0
#define AIRGS_E_STRUCTURAL -1   /* StructuralError  */
#define AIRGS_E_VALIDATION -2   /* ValidationError  */
#define AIRGS_E_CAPACITY -3     /* CapacityError    */
#define AIRGS_E_DECODE -5       /* DecodeError      */
#define AIRGS_E_CUDA -100       /* CUDA runtime failure (RuntimeError) */
#define AIRGS_E_INTERNAL -101

typedef struct airgs_ctx airgs_ctx;

/* Pinhole camera (ss/camera.py:16-65).  rot/trans are pose[:3,:3] and
 * pose[:3,3]; center is -rot^T @ trans computed by the caller exactly as the
 * reference's Camera.center property does (host numpy). */
typedef struct airgs_camera {
    double rot[9];
    double trans[3];
    double center[3];
    double focal;
    double near_clip;
    int32_t width;
    int32_t height;
} airgs_camera;

/* One primitive set (ss/model.py:125-185 GaussianFrame) resident in HBM. */
typedef struct airgs_frame {
    const double *params; /* plane-major [width][ld] */
    int64_t count;        /* primitives n */
    int64_t ld;           /* plane stride in elements, >= count */
    int32_t width;        /* 17 (SH degree 0) or 26 (SH degree 1) */
    int32_t reserved;
} airgs_frame;

/* One evaluated view = (frame, camera) pair.  Any output may be NULL. */
typedef struct airgs_view_item {
    int32_t frame;          /* index into frames[] */
    int32_t camera;         /* index into cams[]   */
    const double *target;   /* (h,w,3) float64 reference image for SSE, or NULL */
    double *image;          /* (h,w,3) float64 clipped render out, or NULL */
    int64_t *usage;         /* int64[count], counts are ADDED (+=), or NULL */
    const int64_t *frozen_pos; /* int64[count] or NULL: frozen compositing order
                                * (ss/rasterizer.py:128-142): position of each primitive
                                * in the frozen order, -1 if absent (kept primitives
                                * absent from it are appended in depth order) */
    const int32_t *tile_minrank; /* int32[tiles] or NULL: clean-tile skip of the
                                * pruning-level sweep (SSE-only items: target set,
                                * image and usage NULL).  16x16 tile g (row-major)
                                * with tile_minrank[g] >= tile_keep_min is known to
                                * render identically to the target, so its SSE
                                * contribution is exactly 0 and it is not composited
                                * (airgs_tile_footprint builds the array) */
    int32_t tile_keep_min;
    int32_t reserved;
} airgs_view_item;

/* ---- context ------------------------------------------------------------ */
AIRGS_API int airgs_ctx_create(airgs_ctx **out, int32_t device);
AIRGS_API int airgs_ctx_destroy(airgs_ctx *ctx);
/* Human-readable message of the last failing call on this context. */
AIRGS_API const char *airgs_last_error(const airgs_ctx *ctx);
/* Number of kernel launches issued by this context since creation. */
AIRGS_API int64_t airgs_launch_count(const airgs_ctx *ctx);

/* Per-kernel device timing with CUDA events on the launching stream around
 * the compositing and projection kernels (for roofline reporting).  Reads
 * the accumulated totals, then if enable >= 0 arms (1) or disarms (0) timing
 * and resets the counters; enable < 0 only reads. */
AIRGS_API int airgs_timing(airgs_ctx *ctx, int32_t enable, double *composite_ms,
                           int64_t *composite_launches, double *project_ms,
                           int64_t *project_launches);
/* Per-stage device timing, the generalisation of airgs_timing: ms[k] /
 * launches[k] for stage k in 0..nstages-1 = 0 compositing, 1 projection,
 * 2 tile binning, 3 tile-list sort, 4 GSDP decode, 5 delta apply,
 * 6 SSE reduction, 7 quantisation (payload sizes) -- CUDA events on the
 * launching stream around each stage's kernels.  enable as for airgs_timing. */
AIRGS_API int airgs_timing_stages(airgs_ctx *ctx, int32_t enable, double *ms, int64_t *launches,
                                  int32_t nstages);

/* Diagnostic evaluation counters (no reference equivalent; used by bench.py
 * for the algorithmic-work roofline).  While armed, renders
 * use a counting variant of the compositing kernel that also accumulates, over
 * all (pixel, primitive) pairs of the reference's Gaussian-major loop
 * (ss/_composite.pyx:42-73): counts[0] = pairs inside the clipped bbox,
 * counts[1] = those evaluated before the pixel terminated (0.999*T <= 1/255),
 * counts[2] = contributing pairs (= summed usage), counts[3] = (tile,
 * primitive) entries of the binned tile lists, counts[4] = projected records
 * written (primitives reaching a tile, summed over views); counts holds 5
 * int64.  Returns the counts since
 * the last (re)arm; enable = 1 arms, 0 disarms, -1 only reads.  Synchronises. */
AIRGS_API int airgs_eval_stats(airgs_ctx *ctx, int32_t enable, int64_t *counts);

/* Decision margins of the renders since the counters were armed (SURVEY.md
 * s8(a) numerics contract: "the harness must report decision margins"):
 * margins[0] = min |w - 1/255| / (1/255) over the exactly evaluated weight
 *              tests (pairs the fp32 pass rejects have margin >= ~4e-5 by
 *              its guard band), ss/_composite.pyx:62;
 * margins[1] = min |0.999 T - 1/255| / (1/255) after any contribution
 *              (early-termination test);
 * margins[2] = min gap in ulps between adjacent distinct depth keys of a
 *              tile list (ss/rasterizer.py:127 stable argsort);
 * margins[3] = number of adjacent exact depth ties (ordered by index);
 * margins[4] = min distance of a bbox floor/ceil argument to an integer (px),
 *              ss/rasterizer.py:177-180;
 * margins[5] = min |z - near_clip| (cull), ss/rasterizer.py:124;
 * margins[6] = min |alpha - 1/255| / (1/255) (opacity cull), ss/rasterizer.py:124.
 * Synchronises. */
AIRGS_API int airgs_eval_margins(airgs_ctx *ctx, double *margins);

/* Backward pass of one view (training; ss/rasterizer.py:248-369 render_forward
 * + render_backward with the compiled _composite.backward, ss/_composite.pyx:
 * 77-152): recomputes the forward with its contribution record, back-
 * propagates d_image (device float64 (h, w, 3), dLoss/dpixel of the
 * unclipped forward image) through compositing and projection, and writes
 * the pre-activation parameter gradients grads (device float64 row-major
 * [count][width], every row written).  Depth order is the forward's,
 * frozen through frozen_pos as in airgs_view_item (or NULL). */
AIRGS_API int airgs_render_backward(airgs_ctx *ctx, const airgs_frame *frame, const airgs_camera *cam,
                                    const int64_t *frozen_pos, const double *d_image, double *grads,
                                    void *stream);

/* Compositing order of one view (ss/rasterizer.py:243-246 compositing_orders,
 * _prepare's stable depth sort of the kept primitives, or the frozen order
 * rule when frozen_pos != NULL): order_out (device int64[count]) receives the
 * kept primitives' indices, *kept_out their number.  Synchronises. */
AIRGS_API int airgs_compositing_order(airgs_ctx *ctx, const airgs_frame *frame, const airgs_camera *cam,
                                      const int64_t *frozen_pos, int64_t *order_out, int64_t *kept_out,
                                      void *stream);

/* ---- image metrics of the trainer's loss ---------------------------------- */

/* Mean windowed SSIM of the luminance of a vs b (device float64, (h, w) when
 * channels == 1 or (h, w, 3)), ss/metrics.py:77-86, and optionally its
 * gradient w.r.t. a (same shape as a), ss/metrics.py:89-113.  window = the
 * reference's 11-tap Gaussian g (sigma 1.5) normalised to sum 1 (host
 * float64[11]).  ssim_out: device float64[1].  grad may be NULL.  Fails with
 * AIRGS_E_STRUCTURAL when the image is smaller than the window. */
AIRGS_API int airgs_ssim(airgs_ctx *ctx, const double *a, const double *b, int32_t height, int32_t width,
                         int32_t channels, const double *window, double *ssim_out, double *grad, void *stream);

/* mean |a - b| over n values (ss/metrics.py:116-118) into l1_out (device
 * float64[1]) and optionally its gradient sign(a - b) / n (ss/metrics.py:121). */
AIRGS_API int airgs_l1(airgs_ctx *ctx, const double *a, const double *b, int64_t n, double *l1_out, double *grad,
                       void *stream);

/* ---- parameter transfer / on-disk formats -------------------------------- */

/* Row-major little-endian float64 rows (n x width) starting at
 * bytes + byte_offset (device memory, any alignment) -> plane-major
 * planes[c * ld + i].  The device side of GaussianFrame uploads and of the
 * GSSC scene loader (ss/model.py:318-350, rows at byte 15 + ...). */
AIRGS_API int airgs_rows_to_planes(airgs_ctx *ctx, const uint8_t *bytes, int64_t byte_offset, int64_t n,
                                   int32_t width, double *planes, int64_t ld, void *stream);

/* Deferred checking for pipelined batches: with enable = 1, airgs_gsdp_decode
 * and airgs_render skip their host synchronisations (validity, bucket
 * overflow) and fold the error flags into a device word; enable = 0
 * synchronises and returns the accumulated flags in *flags_out (0: every call
 * was valid; otherwise the caller re-runs the batch in checked mode, which
 * raises the reference's exact errors and handles bucket overflow). */
AIRGS_API int airgs_defer(airgs_ctx *ctx, int32_t enable, uint32_t *flags_out);

/* ---- rasterizer --------------------------------------------------------- */

/* Batched render: replaces ss/rasterizer.py:113-240 (_activate, _prepare,
 * render, render_with_usage) for every item at once.  sse (device float64
 * [nitems], may be NULL) receives sum((clip(render) - target)^2) over all
 * h*w*3 values for items with a target (ss/metrics.py:37-43 numerator).
 * Fails with AIRGS_E_VALIDATION on a zero quaternion or non-finite parameter
 * (ss/rasterizer.py:105-106) and AIRGS_E_STRUCTURAL on an empty frame
 * (ss/rasterizer.py:114-115). */
AIRGS_API int airgs_render(airgs_ctx *ctx, const airgs_frame *frames, int32_t nframes,
                 const airgs_camera *cams, int32_t ncams,
                 const airgs_view_item *items, int32_t nitems,
                 double *sse, void *stream);

/* Tile footprint for the pruning-level sweep's clean-tile skip
 * (ss/pruning.py:122-131 re-renders every level; only the tiles a pruned
 * primitive reaches can differ from the unpruned reference render).  For
 * every camera v and primitive i with rank[i] < rank_cap, the 16x16 tiles of
 * its clipped bbox (widened by one pixel; the binning's tile set is a subset)
 * receive minrank[v * tile_stride + g] = min(., rank[i]).  Run it over the
 * unpruned frame and over the frame with every ranked entry pruned: a level
 * that prunes ranks < k changes no primitive reaching tile g when
 * minrank[g] >= k, so that tile's pixels equal the reference's bit for bit.
 * Primitives that the renderer would refuse (zero quaternion, non-finite)
 * are skipped: the render of that frame fails anyway.  The caller fills
 * minrank with INT32_MAX first; device buffers, asynchronous. */
AIRGS_API int airgs_tile_footprint(airgs_ctx *ctx, const airgs_frame *frame, const airgs_camera *cams,
                                   int32_t ncams, const int32_t *rank, int32_t rank_cap, int32_t *minrank,
                                   int64_t tile_stride, void *stream);

/* Debug capture of one view's depth-ordered tile lists (the binning + sort
 * stage that precedes compositing; SURVEY.md s8(c) tile keys): for every
 * 16x16 tile g (row-major, tiles_x = ceil(w/16)), counts[g] = list length and
 * ids[g*max_per_tile + k] = the k-th primitive index of its list in
 * compositing order (entries beyond max_per_tile are not written).  A
 * primitive is listed in tile g iff its clipped bbox overlaps g and so does
 * the padded AABB of its weight-threshold ellipse; within a
 * list the order is the reference's stable depth order
 * (ss/rasterizer.py:126-127).  Device buffers; synchronises. */
AIRGS_API int airgs_debug_tile_lists(airgs_ctx *ctx, const airgs_frame *frame, const airgs_camera *cam,
                                     int64_t max_per_tile, int32_t *counts, int32_t *ids, void *stream);

/* The reference's pluggable compositing seam, ss/_composite.pyx:18-74
 * forward(means2d, conics, alphas, colors, bboxes, height, width):
 * primitives already in depth order with clipped int64 bboxes.  Writes the
 * UNclipped image (h,w,3), final transmittance (h,w) and usage int64[k]
 * (all device, caller-owned).  record=True (training masks) is not
 * supported by this path. */
AIRGS_API int airgs_composite_forward(airgs_ctx *ctx, int64_t k, const double *means2d,
                            const double *conics, const double *alphas,
                            const double *colors, const int64_t *bboxes,
                            int32_t height, int32_t width, double *image,
                            double *t_final, int64_t *usage, void *stream);

/* forward(..., record=True) of the kernel seam (ss/_composite.pyx:18-74):
 * airgs_composite_forward plus the reference's contribution masks, uint8
 * [total bbox area], primitive i's clipped bbox row-major at mask_offsets[i]
 * (device int64 [k], the prefix of the non-empty bbox areas). */
AIRGS_API int airgs_composite_forward_record(airgs_ctx *ctx, int64_t k, const double *means2d,
                                             const double *conics, const double *alphas, const double *colors,
                                             const int64_t *bboxes, int32_t height, int32_t width, double *image,
                                             double *t_final, int64_t *usage, const int64_t *mask_offsets,
                                             uint8_t *masks, void *stream);

/* backward(...) of the kernel seam (ss/_composite.pyx:77-152): masks and
 * t_final as returned by the recorded forward, d_image (h, w, 3); grads9
 * (device float64 [k][9]) receives d_means2d (2), d_conics (3), d_alphas,
 * d_colors (3) per primitive. */
AIRGS_API int airgs_composite_backward(airgs_ctx *ctx, int64_t k, const double *means2d, const double *conics,
                                       const double *alphas, const double *colors, const int64_t *bboxes,
                                       int32_t height, int32_t width, const int64_t *mask_offsets,
                                       const uint8_t *masks, const double *t_final, const double *d_image,
                                       double *grads9, void *stream);

/* Sum of squared differences of two device float64 arrays of n values
 * (ss/metrics.py:40 numerator), deterministic order.  out: device double. */
AIRGS_API int airgs_sse(airgs_ctx *ctx, const double *a, const double *b, int64_t n,
              double *out, void *stream);

/* ---- codec (ss/codec.py) ------------------------------------------------ */

/* GSAI attribute planes -> plane-major params (ss/codec.py:95-121,161-169).
 * blob: device copy of the container bytes.  The caller parses and validates
 * the 25-byte header on the host (magic, version, depth, truncation) and
 * passes n (count), m (planes), plane_pixels = w*h.  Each plane j starts at
 * byte 25 + j*(16 + 2*plane_pixels): (scale, offset) f64 LE then u16 LE.
 * out[j*ld + i] = (double)q * scale_j + offset_j (separate mul, add). */
AIRGS_API int airgs_gsai_decode(airgs_ctx *ctx, const uint8_t *blob, int64_t nbytes,
                      int64_t n, int32_t m, int64_t plane_pixels,
                      double *out, int64_t ld, void *stream);

/* GSDP payload -> dense delta overlay (ss/codec.py:217-248).
 * payload: device bytes; entry_count / quant_step from the host-parsed
 * 24-byte header; width = param_width.  Decodes the gap varints in parallel,
 * prefix-sums them to indices, and scatters rows[c*ld + idx] =
 * (double)q * quant_step and present[idx] = 1 (later duplicates win).
 * Writes the number of distinct entries to *entries_out (device int64) and
 * the strictly increasing entry indices to idx_out (device int64[entry_count]).
 * rows == NULL decodes the indices only (no range check, no scatter).
 * Errors: AIRGS_E_DECODE (truncated varint / varint too long / truncated
 * payload), AIRGS_E_STRUCTURAL (index >= base_count). */
AIRGS_API int airgs_gsdp_decode(airgs_ctx *ctx, const uint8_t *payload, int64_t nbytes,
                      int64_t entry_count, double quant_step, int32_t width,
                      int64_t base_count, double *rows, int64_t ld,
                      uint8_t *present, int64_t *idx_out, int64_t *entries_out,
                      void *stream);

/* Fused decode_delta + apply_delta for the keyframe probe (ss/codec.py:217-248
 * then ss/model.py:269-284): params_out (plane-major, width x ld, device) =
 * canonical with rows[idx] += (double)q * quant_step for every entry of the
 * GSDP payload, without materialising the dense overlay.  Varint scan (per-
 * block counts, then each block numbers its varints and tags a row map with
 * entry numbers), then one streaming pass over the canonical planes (128-bit,
 * every parameter written once).  Bit-identical to airgs_gsdp_decode followed
 * by airgs_delta_apply; malformed payloads take the exact decoder's path and
 * return its status (AIRGS_E_DECODE / AIRGS_E_STRUCTURAL, same messages).
 * Under airgs_defer the checks fold into the deferred word instead. */
AIRGS_API int airgs_gsdp_decode_apply(airgs_ctx *ctx, const uint8_t *payload, int64_t nbytes, int64_t entry_count,
                                      double quant_step, int32_t width, const double *canonical, int64_t count,
                                      int64_t ld, double *params_out, void *stream);

/* airgs_gsdp_decode_apply for a pipelined sequence of frames: under
 * airgs_defer, the varint scan of next_payload (the frame the caller decodes
 * next; NULL: none) is enqueued ahead on the context's side stream, so it
 * overlaps this frame's render, and the next call finds it done (matched by
 * payload pointer, sizes and layout; otherwise it scans in line).  Two row-map
 * slots alternate.  Outside airgs_defer it is airgs_gsdp_decode_apply.  Same
 * results and statuses. */
AIRGS_API int airgs_gsdp_decode_apply_ahead(airgs_ctx *ctx, const uint8_t *payload, int64_t nbytes,
                                            int64_t entry_count, const uint8_t *next_payload, int64_t next_nbytes,
                                            int64_t next_entry_count, double quant_step, int32_t width,
                                            const double *canonical, int64_t count, int64_t ld, double *params_out,
                                            void *stream);

/* Position after the entry_count gap varints (sequential walk, reference
 * order); *err_out: 0 ok, 1 truncated varint, 2 varint too long.  Used to
 * infer param_width when the caller does not pin it (ss/codec.py:235-240). */
AIRGS_API int airgs_gsdp_varint_end(airgs_ctx *ctx, const uint8_t *payload, int64_t nbytes,
                          int64_t entry_count, int64_t *pos_out, int32_t *err_out,
                          void *stream);

/* Server-side encoders (ss/codec.py:124-158,187-214).
 * airgs_plane_minmax: per plane (min, max) of params -> lohi_out (host
 * double[2*m], interleaved).  The caller derives scale_j = (hi-lo)/65535 (0
 * for a constant plane) exactly as encode_frame does, then
 * airgs_gsai_encode writes u16 planes [m][plane_pixels] (device) with
 * clip(rint((v - lo)/scale), 0, 65535), zero padding beyond n. */
AIRGS_API int airgs_plane_minmax(airgs_ctx *ctx, const double *params, int64_t n, int32_t m,
                                 int64_t ld, double *lohi_out, void *stream);
AIRGS_API int airgs_gsai_encode(airgs_ctx *ctx, const double *params, int64_t n, int32_t m,
                                int64_t ld, const double *lo, const double *scale,
                                int64_t plane_pixels, uint16_t *planes, void *stream);
/* GSDP body for the entries with nz[i] != 0 (use airgs_quantize first):
 * gap varints then i32 rows, written to out[24 ..] (device); the caller
 * writes the 24-byte header.  capacity >= 24 + E*(10 + 4*width). */
AIRGS_API int airgs_gsdp_encode(airgs_ctx *ctx, const double *rows, const uint8_t *nz, int64_t n,
                                int32_t width, int64_t ld, double step, uint8_t *out,
                                int64_t capacity, int64_t *nbytes_out, int64_t *entries_out,
                                void *stream);

/* ---- delta algebra (ss/model.py:241-311) -------------------------------- */
/* Layout contract of the plane-major kernels below (compose, apply,
 * quantize): planes start 16-byte aligned, ld is even, and every per-primitive
 * array (present, sel, rank, nz) holds ld entries -- the kernels move two
 * primitives per thread as 128-bit double2 (the padding lane i + 1 >= n is
 * written as 0).  paper_2512_20943_b200.device allocates ld = ceil8(n). */

/* n-way compose of dense overlays in list order with one |.|max > eps filter
 * at the end (ss/model.py:294-311); sign[d] = -1 negates overlay d
 * (DeltaTensor.negate, ss/model.py:241-246).  apply_eps = 0 skips the filter
 * (the base-is-empty shortcut of ss/pruning.py:111). */
AIRGS_API int airgs_delta_compose(airgs_ctx *ctx, int32_t ndeltas, const double *const *rows,
                        const uint8_t *const *present, const double *signs,
                        int64_t n, int32_t width, int64_t ld, double eps,
                        int32_t apply_eps, double *out_rows, uint8_t *out_present,
                        void *stream);

/* params_out = canonical + selected overlay row (ss/model.py:269-284).
 * Overlay A (rows_a/present_a) is used for primitive i when
 *   (sel_a == NULL || sel_a[i]) && (keep_rank == NULL || keep_rank[i] >= keep_min)
 * -- the pruning-level mask of ss/pruning.py:79-90 -- and overlay B
 * (rows_b/present_b, may be NULL) otherwise.  A selected overlay whose
 * present flag is 0 leaves the canonical row untouched. */
AIRGS_API int airgs_delta_apply(airgs_ctx *ctx, const double *canonical, const double *rows_a,
                      const uint8_t *present_a, const uint8_t *sel_a, const int32_t *keep_rank,
                      int32_t keep_min, const double *rows_b, const uint8_t *present_b,
                      int64_t n, int32_t width, int64_t ld, double *params_out, void *stream);

/* ---- pruning (ss/pruning.py, ss/codec.py:187-214) ------------------------ */

/* Quantisation rule of encode_delta: q = rint(v/step) per component; an
 * entry survives iff any q != 0.  nz_out[i] = survives (u8, 0 for absent).
 * Fails with AIRGS_E_STRUCTURAL if a surviving |q| > 2^31-1 (first offending
 * index in *bad_index_out, host int64).  deq_out (optional, plane-major like
 * rows) receives the decoded values q*step of surviving entries: exactly what
 * decode_delta(encode_delta(.)) yields (ss/codec.py:195,247). */
AIRGS_API int airgs_quantize(airgs_ctx *ctx, const double *rows, const uint8_t *present,
                   int64_t n, int32_t width, int64_t ld, double step,
                   uint8_t *nz_out, double *deq_out, int64_t *bad_index_out, void *stream);

/* Usage-ordered prune ranks (ss/pruning.py:72-76): among present entries,
 * order by (usage ascending, index descending); rank_out[i] = position in
 * that order (INT32_MAX for absent).  *count_out (host) = entry count. */
AIRGS_API int airgs_prune_rank(airgs_ctx *ctx, const uint8_t *present, const int64_t *usage,
                     int64_t n, int32_t *rank_out, int64_t *count_out, void *stream);

/* Exact GSDP sizes for L pruning levels (ss/codec.py:200-207): level l keeps
 * entries with rank >= kmin[l] that also survive quantisation (nz).  size =
 * 24 + sum varint_len(gap) + 4*width*kept.  sizes_out: host int64[L]. */
AIRGS_API int airgs_level_sizes(airgs_ctx *ctx, const uint8_t *nz, const int32_t *rank,
                      int64_t n, int32_t width, const int64_t *kmin, int32_t nlevels,
                      int64_t *sizes_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* AIRGS_B200_H */
