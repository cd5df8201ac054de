// Shared declarations of the dogblob_b200 CUDA library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <vector>

#include "../../include/dogblob_b200.h"

namespace dogblob {

// ---- error plumbing --------------------------------------------------------
void set_error(const std::string &msg);

#define DB_CUDA(expr)                                                              \
    do {                                                                           \
        cudaError_t _e = (expr);                                                   \
        if (_e != cudaSuccess) {                                                   \
            ::dogblob::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
            return DOGBLOB_ECUDA;                                                  \
        }                                                                          \
    } while (0)

#define DB_REQUIRE(cond, msg)                  \
    do {                                       \
        if (!(cond)) {                         \
            ::dogblob::set_error(msg);         \
            return DOGBLOB_EINVAL;             \
        }                                      \
    } while (0)

// ---- tiling constants of the separable convolution ---------------------------
constexpr int kTY = 16;                 // outputs per thread along the convolved axis
constexpr int kWarps = 8;               // warps per CTA, stacked along the convolved axis
constexpr int kTileRows = kTY * kWarps; // 128
constexpr int kTileCols = 128;          // contiguous floats per CTA (4 per lane)
constexpr int kPad = 128;               // plane dimensions are padded to this
constexpr int kPrefetch = 4;            // input rows in flight per thread
constexpr int kConvThreads = 32 * kWarps;

struct LevelDesc {
    int rpad;         // r_i = ceil(truncate * sigma_i) rounded up to a multiple of 8 (zero taps)
    int n_mid;        // full chunks between the first and the last: (2 rpad + 16) / 16 - 2
    int tap_ofs;      // start (in float2) of this level's duplicated tap table: 2 rpad + 1 taps
                      // followed by 15 zeros (2 rpad + 16 entries = a whole number of chunks)
    float sigma_f32;  // float32(sigma_i), the DoG scale factor
};

// Per-plan level table, passed to the convolution kernels BY VALUE as a __grid_constant__
// parameter (constant bank): a CTA reads its level descriptor without a global round trip.
constexpr int kMaxLevels = 320;
struct LevelTable {
    LevelDesc lv[kMaxLevels];
    int order[kMaxLevels];            // row pass: launch order (longest first)
    int group_begin[kMaxLevels + 1];  // column pass: level groups
    int n_levels, n_groups;
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---- blob bookkeeping shared by extrema / prune ------------------------------
struct Counters {            // one per result, lives in the blob space
    int n_flagged;           // voxels passing the NMS + threshold test
    int n_plateau;           // plateau members appended to `plateau`
    int n_candidates;        // blobs before pruning (singles + plateau components)
    int n_blobs;             // final
    int n_merges;
    unsigned flags;
    int small_done;          // 1 once finalize_small_kernel has sorted / pruned / packed the frame
    unsigned plateau_ticket; // CTA ticket of plateau_kernel
    // device-side stage stamps (globaltimer, ns): start of the frame, start of extrema, start of
    // ordering/pruning; the kernel that finishes the frame turns them into the header's stage times
    unsigned long long t_start, t_extrema, t_prune;
    int n_seeds;             // tensor engine: seeds appended by the column pass (HitFlags::seeds), may exceed the capacity
    int pad;
};

struct Voxel { int s, row, col; int pad; double val; };     // val: the slice's value (float32 values are exact in it)

// Device-side control block of prune_large_kernel (prune.cu): ticket dispenser, completion
// counter and the log of published phases.
constexpr int kMaxPhases = 128;
struct PhaseRec { int type, first_item, n_items, pad; unsigned long long t_ns, pad2; };
struct PruneCtl {
    unsigned ticket, done;       // next work item / completed work items
    int n_phases;                // published entries of phase[]
    int changed, sweeps;         // radius-bound fixed point
    int n_roots, merges, kept;
    double ext[5];               // xmin, xmax, ymin, ymax, rmax of the candidates
    double pad;
    PhaseRec phase[kMaxPhases];
};

// Layout of the blob space (device), all arrays sized by `cap`.
struct BlobSpace {
    Counters *ctr;
    Voxel *plateau;              // plateau members
    int *parent;                 // union-find over plateau members
    int *pl_count;               // per-root member count
    unsigned long long *pl_sum_row, *pl_sum_col;
    unsigned long long *pl_first;   // min over members of (y << 44 | x << 24 | member): raster-first voxel
    dogblob_blob *unsorted;      // candidates in emission order
    dogblob_blob *sorted;        // candidates in (-response, y, x, sigma) order
    int *first;                  // prune: smallest offending partner j > i, or -1
    int *alive;
    int *comp;                   // prune: interaction component (root index) of every blob
    int *cmin;                   // prune: per-root smallest row with an offending partner
    unsigned long long *bound;   // prune: per-root largest radius (bits of a positive double)
    int *cell_of;                // prune grid
    int *cell_start;             // kMaxCells + 1
    int *cell_fill;              // kMaxCells
    int *cell_items;
    double *grid_params;         // [0]=x0 [1]=y0 [2]=cell size [3]=gx [4]=gy
    PruneCtl *ctl;
    int cap;
};

constexpr int kMaxCellsPerAxis = 256;
constexpr int kMaxCells = kMaxCellsPerAxis * kMaxCellsPerAxis;

size_t blobspace_bytes(int cap);
BlobSpace carve_blobspace(void *base, int cap);

// ---- launchers (defined in the .cu files) ------------------------------------
struct ConvGeometry {
    int H, W;            // image
    int Hp, Wp;          // padded to kPad
    int L;               // levels
    int G;               // level groups of the fused column+DoG pass
    int max_table;       // float2 entries of the longest tap table (2 max_rpad + 16)
    int max_group_table; // float2 entries of the longest level group's concatenated tables
    int max_rpad;        // largest padded radius
};

// streamed row pass: `word` (device int) holds base + k once row chunks 0..k-1 of the frame are
// resident; chunk c = image rows [c * rows_per_chunk, (c + 1) * rows_per_chunk)
struct RowGate { const int *word; int base; int rows_per_chunk; unsigned long long *t_start; };
cudaError_t launch_row_pass(const ConvGeometry &g, const float *d_img, float *d_rows_t,
                            const LevelTable &tbl, const float2 *d_taps, cudaStream_t st,
                            const RowGate *gate = nullptr);
cudaError_t launch_col_dog_pass(const ConvGeometry &g, const float *d_rows_t, float *d_dog_t,
                                float *d_edge, const LevelTable &tbl, const float2 *d_taps,
                                cudaStream_t st);
cudaError_t launch_col_levels_pass(const ConvGeometry &g, const float *d_rows_t, float *d_lev_t,
                                   const LevelTable &unit_tbl, const float2 *d_taps,
                                   cudaStream_t st);
cudaError_t launch_edge_dog(const ConvGeometry &g, const float *d_edge, float *d_dog_t,
                            const LevelTable &tbl, cudaStream_t st);
// which blocks of 8 rows x 32 columns of the (x-major) DoG slices hold a value above the detection threshold;
// the tensor-core column pass only STORES the 32 x 32 boxes that contain such a block, so the flags
// are also the validity map of the slice memory (everything else reads as -inf in the extrema kernel)
struct HitFlags {
    unsigned char *data = nullptr;       // [slice][col_blocks][row_blocks] (row blocks contiguous)
    int row_blocks = 0, col_blocks = 0;
    // Seeds (optional): the column pass also tests every value above the threshold against the in-slice
    // neighbours it has in registers (same row: the thread's own columns; rows above / below: the
    // neighbouring lanes) and appends the survivors - a superset of the in-slice local maxima, some ten
    // thousand voxels per frame - to this list as slice << 48 | row << 24 | column of the x-major slice
    // (row = x, column = y).  The extrema kernel
    // then only visits the seeds (nms_seed_kernel) instead of walking the slices.  *n_seeds counts past
    // the capacity: more seeds than seed_cap = the list is incomplete and the strip kernel runs instead.
    unsigned long long *seeds = nullptr;
    int *n_seeds = nullptr;
    int seed_cap = 0;
};
constexpr int kFlagColShift = 5, kFlagRowShift = 3;      // 32 columns x 8 rows
inline size_t hit_flag_bytes(int planes, int Hp, int Wp) {
    return (size_t)planes * (Hp >> kFlagRowShift) * (Wp >> kFlagColShift);
}
// tensor-core (tcgen05) versions of the passes, scale_space_umma.cu
struct ToeplitzTable {               // per level: float offset, rows, log2 of the tap scale
    int ofs[kMaxLevels];
    int rows[kMaxLevels];
    int tscale[kMaxLevels];
};
// Buffers of the tensor-core engine (all fp16, frame-scaled units):
//   X planes [hi | lo][H + 2 Py][Wp]      the frame with its reflected halo rows
//   R planes [hi | lo][L][Hp][Wq]         pass-1 output rows, interior at column Ppad, reflected
//                                         halo columns on both sides (Wq = Wp + 2 Ppad)
struct UmmaLayout { int Py, Ppad, Wq; size_t x_bytes, r_bytes; };
UmmaLayout umma_layout(const ConvGeometry &g);
bool umma_supported(const ConvGeometry &g);
void build_toeplitz(const LevelDesc *lv, int n_levels, const float2 *taps, std::vector<float> &out,
                    ToeplitzTable &tab);
cudaError_t configure_umma_kernels(int device);
cudaError_t launch_prep_umma(const ConvGeometry &g, const float *d_img, void *d_x, uint32_t *d_max_bits,
                             cudaStream_t st, const BlobSpace *bs = nullptr);
int umma_max_words();      // uint32 words behind d_max_bits: the frame's max + the partial maxima
cudaError_t launch_row_pass_umma(const ConvGeometry &g, const void *d_x, void *d_r, const LevelTable &tbl,
                                 const ToeplitzTable &ttab, const float *d_toep, cudaStream_t st,
                                 const uint32_t *d_max_bits, int max_ctas = 0);
// x-major DoG slices D^T [L - 1][Wp][Hp], like the FP32 engine's (levels = true: the L levels themselves)
cudaError_t launch_col_pass_umma(const ConvGeometry &g, const void *d_r, float *d_out, const LevelTable &tbl,
                                 const ToeplitzTable &ttab, const float *d_toep, cudaStream_t st,
                                 const uint32_t *d_max_bits, bool levels, const int *d_sched, int sched_slots,
                                 int sched_ctas, float threshold = 0.f, HitFlags flags = HitFlags{});
cudaError_t launch_untranspose(const float *d_src_t, int planes, int Hp, int Wp, int H, int W,
                               float *d_dst, cudaStream_t st);
cudaError_t launch_dog_from_levels(int L, int64_t plane_elems, const float *d_levels,
                                   const float *d_sigma_f32, float *d_out, cudaStream_t st);
cudaError_t configure_conv_kernels(int device);
size_t col_pass_smem(int group_table, int max_rpad, bool dog);

// extrema: NMS + compaction + plateau coalescing + ordering.  `flags` (optional): one byte per
// 8-row x 32-column block of every slice, non-zero if the block holds a value above the threshold
// (written by the tensor-core column pass, which does not store blocks without one); strips without
// a hit are skipped unread, inside a strip only the rows next to a hit block are loaded, and every
// block without a hit reads as -inf.
cudaError_t launch_extrema(const float *d_slices, int S, int rows, int cols, int64_t pitch,
                           int64_t plane, bool transposed, const double *d_slice_sigma,
                           float threshold, int half, const BlobSpace &bs, cudaStream_t st,
                           HitFlags flags = HitFlags{});
// float64 tier (fp64.cu, extrema.cu): dense [L][H][W] double planes, slow and simple
cudaError_t launch_extrema_f64(const double *d_slices, int S, int rows, int cols, const double *d_slice_sigma,
                               double threshold, int half, const BlobSpace &bs, cudaStream_t st);
cudaError_t launch_scale_space_f64(int H, int W, int L, const int *h_radii, const double *d_taps,
                                   const int64_t *h_tap_offsets, const double *d_image, double *d_tmp,
                                   double *d_levels, cudaStream_t st);
cudaError_t launch_dog_inplace_f64(int L, int64_t plane_elems, double *d_levels, const double *d_sigmas,
                                   cudaStream_t st);
// evaluation on the device (evaluate.cu): greedy VOC matching, one CTA per job (frame)
cudaError_t launch_match_voc(int n_jobs, const double *d_pred, const int *d_pred_begin, const double *d_truth,
                             const int *d_truth_begin, double thr, unsigned char *d_taken, int *d_match,
                             double *d_match_iou, int *d_tp, cudaStream_t st);
// perf-only scene generator on the device (synth_device.cu)
cudaError_t launch_synth_frames(int n_frames, int H, int W, int64_t pitch, int n_droplets, double r_min,
                                double r_max, unsigned long long seed, double poisson_scale, double gaussian_sigma,
                                float *d_frames, double *d_truth, cudaStream_t st);
// pruning + final packing into the result buffer
cudaError_t launch_prune_and_pack(const BlobSpace &bs, double overlap, bool prune,
                                  void *d_result, int result_cap, cudaStream_t st);
cudaError_t launch_load_blobs(const BlobSpace &bs, const dogblob_blob *d_in, int n,
                              cudaStream_t st);
cudaError_t configure_finalize_kernels();   // per device, before the first launch_prune_and_pack
constexpr int kSmallMax = 1024;   // threads (and shared-memory slots) of the single-CTA finalize kernel
int small_limit();                // frames with at most this many candidates finish in that one CTA
cudaError_t launch_reset_counters(const BlobSpace &bs, cudaStream_t st);

}  // namespace dogblob
