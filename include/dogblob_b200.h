/*
 * dogblob_b200.h -- C ABI of the B200-native DoG blob-detector hot path.
 *
 * The reference (`pkg/src/dogblob`, pure Python) has no FFI; its boundary is
 * the Python detector API and the seam is the `backend` string
 * (convolve.py:34,206-207).  A `backend="cuda"` implementation binds exactly
 * the entry points below (ctypes stub: paper_2010_08486_b200/_lib.py, and
 * INTEGRATION.md shows the reference-side patch).  Each entry point names the
 * reference function it replaces.
 *
 * Conventions
 *   - plain pointers and sizes only; `stream` is a cudaStream_t passed as void*;
 *   - every function returns 0 on success, a DOGBLOB_E* code otherwise;
 *     `dogblob_last_error()` returns the thread-local message;
 *   - nothing allocates device memory after plan creation: the caller owns the
 *     workspace / result buffers (sizes come from the *_bytes queries);
 *   - a plan is immutable and may be shared by concurrent callers as long as
 *     each caller brings its own workspace, result buffer and stream
 *     (mirrors the shared, immutable `Detector`, detector.py:309-331);
 *   - all launches are asynchronous on `stream`; no host synchronisation
 *     happens inside any entry point except the *_sync helpers;
 *   - candidate-capacity overflow is reported in the result header
 *     (`n_* > capacity`, DOGBLOB_FLAG_OVERFLOW), never silently truncated.
 */
#ifndef DOGBLOB_B200_H
#define DOGBLOB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DOGBLOB_ABI_VERSION 1
#define DOGBLOB_N_EVENTS 5

enum {
    DOGBLOB_OK = 0,
    DOGBLOB_EINVAL = 1,   /* bad argument  -> Python ValueError   */
    DOGBLOB_ECUDA = 2,    /* CUDA failure  -> Python RuntimeError */
    DOGBLOB_ENOMEM = 3,   /* buffer too small */
};

/* One detected circle -- field-for-field `Blob` (detector.py:67-76) plus the
 * DoG slice index it came from (-1 once pruning has merged it). */
typedef struct dogblob_blob {
    double x, y;          /* integer-valued in the pipeline; doubles so that the
                             prune stage accepts the reference's float centres */
    double sigma;
    double radius;        /* sqrt(2) * sigma */
    double response;      /* float32 DoG value widened */
    int32_t slice;
    uint32_t flags;       /* DOGBLOB_BLOB_* */
} dogblob_blob;

#define DOGBLOB_BLOB_SCALE_EDGE 1u   /* at_scale_boundary */
#define DOGBLOB_BLOB_MERGED     2u   /* radius/sigma rewritten by pruning */

/* Header at the start of every result buffer; blobs follow at offset 64. */
typedef struct dogblob_result_header {
    int32_t n_blobs;        /* records that follow (after pruning if requested) */
    int32_t n_candidates;   /* blobs before pruning */
    int32_t n_flagged;      /* voxels that passed the 3-D maximum + threshold test */
    int32_t n_plateau;      /* of those, members of multi-voxel plateaus */
    int32_t n_merges;       /* merges performed by pruning */
    uint32_t flags;         /* DOGBLOB_FLAG_* */
    int32_t capacity;       /* max blobs this buffer can hold */
    /* device-side stage times in ns (globaltimer): scale space + DoG | extrema | ordering +
     * pruning + packing -- the convolve_ms / extrema_ms / prune_ms of Detector.run
     * (detector.py:336-357) without any host-side event call */
    int32_t conv_ns, extrema_ns, prune_ns;
    /* phase profile of the whole-GPU pruning kernel (0 when the single-CTA path ran):
     * [0..2] six 16-bit marks in us since its first ticket (grid build, first sweep, part
     * labelling, merge loops, packing, end; saturating), [3] sweeps << 24 | parts */
    int32_t prune_profile[4];
    int32_t n_seeds;        /* tensor-core engine: voxels the column pass handed to the extrema kernel (diagnostic) */
    int32_t reserved;
} dogblob_result_header;

#define DOGBLOB_FLAG_OVERFLOW 1u     /* a capacity was exceeded: result incomplete */
#define DOGBLOB_RESULT_HEADER_BYTES 64

typedef struct dogblob_plan dogblob_plan;

int dogblob_abi_version(void);
const char *dogblob_last_error(void);

/* ---- plan: ladder + separable tap tables for one image shape -------------
 * replaces Detector.__init__ / build_kernel_bank / Detector.plan_for
 * (detector.py:316-331, scale_space.py:84-119).
 *   sigmas[n_levels]     ladder (float64)
 *   radii[n_levels]      ceil(truncate * sigma_i)
 *   taps                 concatenated 1-D unit-sum taps w_i[-r_i..r_i] (float32)
 *   tap_offsets[n_levels] start of level i inside `taps`
 *   max_blobs            capacity for flagged voxels / candidates / blobs
 */
int dogblob_plan_create(int device, int height, int width, int n_levels,
                        const double *sigmas, const int32_t *radii,
                        const float *taps, const int64_t *tap_offsets,
                        int max_blobs, dogblob_plan **out);
void dogblob_plan_destroy(dogblob_plan *plan);
size_t dogblob_workspace_bytes(const dogblob_plan *plan);
size_t dogblob_result_bytes(const dogblob_plan *plan);
/* row pitch (in floats) of the device image the plan expects, >= width */
int64_t dogblob_image_pitch(const dogblob_plan *plan);
/* convolution engine this plan's frames run on (same results within float32 rounding):
 * 0 = FP32 sliding-window kernels, 2 = tcgen05 tensor-core Toeplitz GEMM with an fp16 hi/lo operand
 * split (default build; one max reduction per frame), 1 = the same with tf32 operands (build option).
 * Chosen at plan time from the ladder and the frame size; DOGBLOB_CONV=fma|umma overrides. */
int dogblob_plan_conv_engine(const dogblob_plan *plan);
/* level groups of the fused column + DoG pass on this plan's engine (diagnostics / flop accounting):
 * writes min(n_groups + 1, cap) boundaries to `begin` and returns n_groups; group g sweeps levels
 * begin[g] .. begin[g+1]-1 and, on the tensor engine, also level begin[g+1] (computed twice). */
int dogblob_plan_conv_groups(const dogblob_plan *plan, int32_t *begin, int cap);

/* ---- the hot path ---------------------------------------------------------
 * replaces Detector.run minus preprocessing (detector.py:343-359):
 * convolve_bank -> dog_stack -> find_extrema -> prune_overlaps.
 *   d_image     device float32, `height` rows of dogblob_image_pitch() floats
 *   d_result    device buffer of dogblob_result_bytes(): header + blobs, sorted
 *               by (-response, y, x, sigma)
 *   events      NULL or DOGBLOB_N_EVENTS cudaEvent_t recorded at: start, after
 *               the row pass, after the fused column+DoG pass, after extrema,
 *               after pruning/packing
 */
int dogblob_detect(const dogblob_plan *plan, const float *d_image,
                   float threshold, int neighborhood, double overlap, int prune,
                   void *d_workspace, void *d_result, void *stream,
                   void *const *events);

/* Same call with HOST buffers: pitched H2D copy of the frame, dogblob_detect,
 * D2H of header + the first `h_result_blobs` records into pinned `h_result`.
 * The caller synchronises the stream, reads the header, and fetches any
 * remaining records with dogblob_fetch_blobs. */
int dogblob_detect_host(const dogblob_plan *plan, const float *h_image,
                        float threshold, int neighborhood, double overlap, int prune,
                        void *d_image, void *d_workspace, void *d_result,
                        void *h_result, int h_result_blobs, void *stream,
                        void *const *events);
/* dogblob_detect_host with the upload overlapped: the frame goes up in row chunks on
 * `copy_stream`, each followed by a 4-byte copy of a gate word, while the row pass already runs
 * on `stream` and every tile waits only for the image rows it reads (a 1024^2 frame starts
 * computing after the first quarter has arrived).
 *   h_image      PINNED host frame (stays untouched until the stream has been synchronised)
 *   copy_stream  a second stream of the caller, different from `stream`
 *   h_gate       pinned int32[DOGBLOB_GATE_INTS], zeroed once; belongs to this buffer set
 *   frame_done   event (dogblob_event_create) of this buffer set: recorded here behind the
 *                frame's last operation; the next call waits on it before it overwrites d_image
 * One buffer set (d_image, d_workspace, d_result, h_result, h_gate, frame_done) = one frame in
 * flight: synchronise `stream` before the set is used again.
 * FP32 engine only (dogblob_plan_conv_engine() == 0): the tensor engine scales its fp16 operands
 * by the frame's maximum and needs the whole frame first; it returns DOGBLOB_EINVAL here. */
#define DOGBLOB_GATE_CHUNKS 4
#define DOGBLOB_GATE_INTS 16
int dogblob_detect_host_streamed(const dogblob_plan *plan, const float *h_image,
                                 float threshold, int neighborhood, double overlap, int prune,
                                 void *d_image, void *d_workspace, void *d_result,
                                 void *h_result, int h_result_blobs, void *stream,
                                 void *copy_stream, int32_t *h_gate, void *frame_done,
                                 void *const *events);
int dogblob_upload_image(const dogblob_plan *plan, const float *h_image,
                         void *d_image, void *stream);
int dogblob_fetch_blobs(const void *d_result, int first, int count,
                        dogblob_blob *h_out, void *stream);
/* header + the first n_blobs records, as dogblob_detect_host copies them */
int dogblob_fetch_result(const void *d_result, int n_blobs, void *h_result, void *stream);

/* ---- stage entry points (the reference's stage functions) -----------------
 * convolve_bank(..., backend="cuda") (convolve.py:189-218): levels in image
 * orientation, dense float32 [n_levels][height][width]. */
int dogblob_scale_space(const dogblob_plan *plan, const float *d_image,
                        void *d_workspace, float *d_levels, void *stream);
/* the fused scale-space + DoG kernels, result transposed back to
 * [n_levels-1][height][width] (what dog_stack(convolve_bank(..)) returns). */
int dogblob_dog(const dogblob_plan *plan, const float *d_image,
                void *d_workspace, float *d_slices, void *stream);
/* dog_stack (detector.py:117-126) on an existing dense level stack. */
int dogblob_dog_from_levels(int n_levels, int height, int width,
                            const float *d_levels, const double *sigmas,
                            float *d_slices, void *stream);
/* find_extrema (detector.py:149-188) on a dense [n_slices][height][width]
 * stack. slice_sigmas is a HOST array; workspace from dogblob_blobspace_bytes. */
size_t dogblob_blobspace_bytes(int max_blobs);
size_t dogblob_result_bytes_for(int max_blobs);
int dogblob_extrema(int n_slices, int height, int width, const float *d_slices,
                    const double *slice_sigmas, float threshold, int neighborhood,
                    int max_blobs, void *d_blobspace, void *d_result, void *stream);
/* prune_overlaps (detector.py:250-280): d_blobs_in holds n records in any
 * order; result buffer receives the survivors, sorted. */
int dogblob_prune(int n, const dogblob_blob *d_blobs_in, double overlap,
                  int max_blobs, void *d_blobspace, void *d_result, void *stream);

/* ---- pre-processing --------------------------------------
 * images.preprocess (images.py:112-157): Gaussian smoothing with scipy's
 * float64 line filter, then the nearest-rank contrast stretch to [0, 1].
 *   d_src/d_dst   device float32 images with row pitches in floats (may alias
 *                 the pitched image buffer dogblob_detect reads)
 *   radius        int(truncate * smooth_sigma + 0.5), 0 disables smoothing
 *   weights       HOST array of radius + 1 float64 taps, centre first
 *   rank_lo/hi    0-based ranks of the two order statistics in the sorted image:
 *                 min(max(ceil(q * n) - 1, 0), n - 1), q = sat/2 and 1 - sat/2
 *   d_scratch     dogblob_preprocess_bytes(height, width)
 * dogblob_preprocess_status copies the status word (bit 0: the input held a
 * NaN/Inf pixel, images.py:40-41) into pinned host memory. */
size_t dogblob_preprocess_bytes(int height, int width);
int dogblob_preprocess(int height, int width, const float *d_src, int64_t src_pitch,
                       int radius, const double *weights, int64_t rank_lo, int64_t rank_hi,
                       void *d_scratch, float *d_dst, int64_t dst_pitch, void *stream);
int dogblob_preprocess_status(const void *d_scratch, uint32_t *h_status, void *stream);

/* ---- small helpers so that a non-CUDA host language can drive the ABI ----- */
int dogblob_event_create(void **event);
int dogblob_event_destroy(void *event);
int dogblob_event_record(void *event, void *stream);
int dogblob_event_elapsed_ms(void *start, void *stop, float *ms);
/* out_ms[k] = time from events[k] to events[k + 1], k < n_events - 1: the stage times of
 * dogblob_detect's DOGBLOB_N_EVENTS events (timings_ms of Detector.run, detector.py:336-357)
 * in one call */
int dogblob_event_intervals_ms(void *const *events, int n_events, float *out_ms);
int dogblob_stream_sync(void *stream);
int dogblob_device_count(int *count);
/* ---- float64 tier ------------------------------------------------------------------------------
 * Detector.run(img, dtype=np.float64) / convolve_bank(dtype=np.float64) of the reference
 * (detector.py:333, convolve.py:76-77,189-218): the whole path in float64 on the FP64 pipe, separable,
 * slow and simple - the oracle-grade "truth" tier.  No plan: taps arrive as float64 (host arrays
 * `sigmas`, `radii`, `taps`, `tap_offsets` as in dogblob_plan_create, but double taps); images and
 * stacks are DENSE device arrays (pitch = width).
 *   dogblob_scale_space_f64   d_levels[L][H][W] = k_i * img; d_tmp: one plane of scratch
 *   dogblob_dog_inplace_f64   d_levels[i] <- (levels[i] - levels[i+1]) * sigma_i, i < L - 1
 *   dogblob_extrema_f64       find_extrema on a float64 stack (same result layout as dogblob_extrema)
 *   dogblob_detect_f64        all of it + pruning; d_workspace of dogblob_f64_workspace_bytes() */
size_t dogblob_f64_workspace_bytes(int height, int width, int n_levels, int max_blobs);
int dogblob_scale_space_f64(int height, int width, int n_levels, const int32_t *radii, const double *taps,
                            const int64_t *tap_offsets, const double *d_image, double *d_tmp,
                            double *d_levels, void *stream);
int dogblob_dog_inplace_f64(int n_levels, int height, int width, double *d_levels, const double *sigmas,
                            void *stream);
int dogblob_extrema_f64(int n_slices, int height, int width, const double *d_slices,
                        const double *slice_sigmas, double threshold, int neighborhood, int max_blobs,
                        void *d_blobspace, void *d_result, void *stream);
int dogblob_detect_f64(int height, int width, int n_levels, const double *sigmas, const int32_t *radii,
                       const double *taps, const int64_t *tap_offsets, const double *d_image,
                       double threshold, int neighborhood, double overlap, int prune, int max_blobs,
                       void *d_workspace, void *d_result, void *stream);

/* ---- evaluation and scene generation on the device (sweeps over thousands of frames) -------------
 * dogblob_match_voc: evaluate.py:48-109 (match_voc) for n_jobs independent frames, one CTA each.
 *   d_pred        (x, y, radius) float64 triples of all jobs, each job's predictions in visiting
 *                 order (descending response, ties by y, x); job j owns [pred_begin[j], pred_begin[j+1])
 *   d_truth       (x, y, r) float64 triples; job j owns [truth_begin[j], truth_begin[j+1])
 *   d_taken       scratch, one byte per truth
 *   d_match       per prediction: index of the matched truth inside its job, -1 = false positive
 *   d_match_iou   per prediction: IoU of the match (0 if none);  d_tp: per job true positives
 * Identical to the host loop (float64, same operation order, first truth among equal maxima).
 * dogblob_synth_frames: PLIF-like frames + their truth circles generated on the device (the scene
 * model of synth.py:50-162 with allow_overlap=True).  PERF ONLY: counter-based random streams, not
 * numpy's - statistically like the reference's frames, never bit-identical; parity always uses host
 * frames.  d_frames[n_frames][height][pitch] float32, d_truth[n_frames][n_droplets][3] float64. */
int dogblob_match_voc(int n_jobs, const double *d_pred, const int32_t *d_pred_begin, const double *d_truth,
                      const int32_t *d_truth_begin, double iou_threshold, void *d_taken, int32_t *d_match,
                      double *d_match_iou, int32_t *d_tp, void *stream);
int dogblob_synth_frames(int n_frames, int height, int width, int64_t pitch, int n_droplets, double r_min,
                         double r_max, uint64_t seed, double poisson_scale, double gaussian_sigma,
                         float *d_frames, double *d_truth, void *stream);

/* Raw buffers for hosts without CUDA bindings (the reference-side stub):
 * zero-filled device memory on `device`, page-locked host memory. */
int dogblob_device_alloc(int device, size_t bytes, void **out);
int dogblob_device_free(int device, void *ptr);
int dogblob_pinned_alloc(size_t bytes, void **out);
int dogblob_pinned_free(void *ptr);

#ifdef __cplusplus
}
#endif
#endif /* DOGBLOB_B200_H */
