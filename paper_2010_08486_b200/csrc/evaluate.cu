// PASCAL-VOC style greedy matching of detections to ground-truth circles on the device
// (reference: evaluate.py:48-109): predictions in descending-response order, each claims the
// still unmatched truth with the highest bounding-box IoU (inclusive pixel extents, side 2 r + 1;
// the first truth among equal maxima) if that IoU reaches the threshold.  float64 arithmetic in
// the reference's operation order, so the matches are identical to the host loop.
//
// The loop over predictions is sequential by definition; one CTA walks it and spreads every
// prediction's scan over the truths across its threads (large sweeps: thousands of frames are
// matched concurrently, one CTA each, see dogblob_match_voc_batch).
#include <climits>

#include "common.cuh"

namespace dogblob {

namespace {

constexpr int kMatchThreads = 512;

__device__ __forceinline__ double box_iou_dev(double x1, double y1, double r1, double x2, double y2, double r2) {
    const double iw = __dadd_rn(__dsub_rn(fmin(__dadd_rn(x1, r1), __dadd_rn(x2, r2)), fmax(__dsub_rn(x1, r1), __dsub_rn(x2, r2))), 1.0);
    const double ih = __dadd_rn(__dsub_rn(fmin(__dadd_rn(y1, r1), __dadd_rn(y2, r2)), fmax(__dsub_rn(y1, r1), __dsub_rn(y2, r2))), 1.0);
    if (iw <= 0.0 || ih <= 0.0) return 0.0;
    const double inter = __dmul_rn(iw, ih);
    const double s1 = __dadd_rn(__dmul_rn(2.0, r1), 1.0), s2 = __dadd_rn(__dmul_rn(2.0, r2), 1.0);
    const double a1 = __dmul_rn(s1, s1), a2 = __dmul_rn(s2, s2);
    return __ddiv_rn(inter, __dsub_rn(__dadd_rn(a1, a2), inter));
}

// job j: predictions pred[pred_begin[j] .. pred_begin[j+1]) as (x, y, radius) triples in visiting
// order, truths truth[truth_begin[j] .. truth_begin[j+1]); outputs per prediction the matched truth
// (index inside the job, -1 = false positive) and its IoU, per job tp.
__global__ void __launch_bounds__(kMatchThreads)
match_voc_kernel(const double *__restrict__ pred, const int *__restrict__ pred_begin,
                 const double *__restrict__ truth, const int *__restrict__ truth_begin, double thr,
                 unsigned char *__restrict__ taken, int *__restrict__ match, double *__restrict__ match_iou,
                 int *__restrict__ tp_out) {
    __shared__ double s_iou[kMatchThreads / 32];
    __shared__ int s_idx[kMatchThreads / 32];
    __shared__ int s_best;
    const int job = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int p0 = pred_begin[job], p1 = pred_begin[job + 1];
    const int t0 = truth_begin[job], nt = truth_begin[job + 1] - t0;
    const double *tr = truth + 3 * (int64_t)t0;
    unsigned char *tk = taken + t0;
    for (int t = tid; t < nt; t += kMatchThreads) tk[t] = 0;
    __syncthreads();
    int tp = 0;
    for (int p = p0; p < p1; ++p) {
        const double px = pred[3 * (int64_t)p], py = pred[3 * (int64_t)p + 1], pr = pred[3 * (int64_t)p + 2];
        double best = 0.0;
        int best_t = INT_MAX;
        for (int t = tid; t < nt; t += kMatchThreads) {       // ascending t per thread: strict > keeps the first
            if (tk[t]) continue;
            const double iou = box_iou_dev(px, py, pr, tr[3 * t], tr[3 * t + 1], tr[3 * t + 2]);
            if (iou > best) { best = iou; best_t = t; }
        }
        // (max iou, then smallest index): the scan order of the host loop
        for (int o = 16; o > 0; o >>= 1) {
            const double oi = __shfl_xor_sync(0xffffffffu, best, o);
            const int ot = __shfl_xor_sync(0xffffffffu, best_t, o);
            if (oi > best || (oi == best && ot < best_t)) { best = oi; best_t = ot; }
        }
        if (lane == 0) { s_iou[warp] = best; s_idx[warp] = best_t; }
        __syncthreads();
        if (warp == 0) {
            best = lane < kMatchThreads / 32 ? s_iou[lane] : 0.0;
            best_t = lane < kMatchThreads / 32 ? s_idx[lane] : INT_MAX;
            for (int o = 16; o > 0; o >>= 1) {
                const double oi = __shfl_xor_sync(0xffffffffu, best, o);
                const int ot = __shfl_xor_sync(0xffffffffu, best_t, o);
                if (oi > best || (oi == best && ot < best_t)) { best = oi; best_t = ot; }
            }
            if (lane == 0) {
                const bool hit = best_t != INT_MAX && best > 0.0 && best >= thr;
                match[p] = hit ? best_t : -1;
                match_iou[p] = hit ? best : 0.0;
                if (hit) tk[best_t] = 1;
                s_best = hit ? 1 : 0;
            }
        }
        __syncthreads();
        tp += s_best;
    }
    if (tid == 0) tp_out[job] = tp;
}

}  // namespace

cudaError_t launch_match_voc(int n_jobs, const double *d_pred, const int *d_pred_begin, const double *d_truth,
                             const int *d_truth_begin, double thr, unsigned char *d_taken, int *d_match,
                             double *d_match_iou, int *d_tp, cudaStream_t st) {
    if (n_jobs <= 0) return cudaSuccess;
    match_voc_kernel<<<n_jobs, kMatchThreads, 0, st>>>(d_pred, d_pred_begin, d_truth, d_truth_begin, thr, d_taken,
                                                      d_match, d_match_iou, d_tp);
    return cudaGetLastError();
}

}  // namespace dogblob
