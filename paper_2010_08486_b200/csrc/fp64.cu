// float64 tier of the scale space (reference: Detector.run(img, dtype=np.float64), convolve.py:63-86,
// 189-218; dog_stack detector.py:117-126): two separable 1-D correlations with the reflect boundary
// (...cba|abc..., period 2 N) on the FP64 pipe, one thread per output element, and the DoG in place.
// Oracle-grade and deliberately simple: this is the T1 "truth" of the near-tie classifier on the
// device, not a production path (C2: ~50 ms per frame against 0.5 ms in float32).
#include "common.cuh"

namespace dogblob {

namespace {

__device__ __forceinline__ int fold_f64(int i, int n) {
    if ((unsigned)i < (unsigned)n) return i;
    const int period = 2 * n;
    int t = i % period;
    if (t < 0) t += period;
    return t < n ? t : period - 1 - t;
}

// AXIS 0: along rows (y), AXIS 1: along columns (x); one level, dense [H][W] planes.
// Taps are accumulated from the outermost pair inwards (small -> large magnitudes), each product
// rounded and added separately (no FMA contraction), like the float32 kernels.
template <int AXIS>
__global__ void __launch_bounds__(256)
conv_axis_f64_kernel(const double *__restrict__ in, double *__restrict__ out, int H, int W,
                     const double *__restrict__ taps, int r) {
    const int x = blockIdx.x * 256 + threadIdx.x, y = blockIdx.y;
    if (x >= W) return;
    const int n = AXIS == 0 ? H : W, pos = AXIS == 0 ? y : x;
    double acc = 0.0;
    for (int k = r; k >= 1; --k) {
        const int a = fold_f64(pos - k, n), b = fold_f64(pos + k, n);
        const double va = AXIS == 0 ? in[(int64_t)a * W + x] : in[(int64_t)y * W + a];
        const double vb = AXIS == 0 ? in[(int64_t)b * W + x] : in[(int64_t)y * W + b];
        acc = __dadd_rn(acc, __dmul_rn(taps[r - k], va));
        acc = __dadd_rn(acc, __dmul_rn(taps[r + k], vb));
    }
    acc = __dadd_rn(acc, __dmul_rn(taps[r], in[(int64_t)y * W + x]));
    out[(int64_t)y * W + x] = acc;
}

// levels[i] <- (levels[i] - levels[i + 1]) * sigma_i for i = 0 .. L - 2 (numpy: diffs, then scale)
__global__ void __launch_bounds__(256)
dog_inplace_f64_kernel(double *__restrict__ levels, int L, int64_t plane, const double *__restrict__ sigmas) {
    const int64_t p = blockIdx.x * (int64_t)256 + threadIdx.x;
    if (p >= plane) return;
    double cur = levels[p];
    for (int i = 0; i + 1 < L; ++i) {
        const double nxt = levels[(int64_t)(i + 1) * plane + p];
        levels[(int64_t)i * plane + p] = __dmul_rn(__dsub_rn(cur, nxt), sigmas[i]);
        cur = nxt;
    }
}

}  // namespace

cudaError_t launch_scale_space_f64(int H, int W, int L, const int *h_radii, const double *d_taps,
                                   const int64_t *h_tap_offsets, const double *d_image, double *d_tmp,
                                   double *d_levels, cudaStream_t st) {
    const dim3 grid((W + 255) / 256, H);
    for (int i = 0; i < L; ++i) {
        const double *w = d_taps + h_tap_offsets[i];
        conv_axis_f64_kernel<0><<<grid, 256, 0, st>>>(d_image, d_tmp, H, W, w, h_radii[i]);
        conv_axis_f64_kernel<1><<<grid, 256, 0, st>>>(d_tmp, d_levels + (int64_t)i * H * W, H, W, w, h_radii[i]);
    }
    return cudaGetLastError();
}

cudaError_t launch_dog_inplace_f64(int L, int64_t plane_elems, double *d_levels, const double *d_sigmas,
                                   cudaStream_t st) {
    dog_inplace_f64_kernel<<<(unsigned)((plane_elems + 255) / 256), 256, 0, st>>>(d_levels, L, plane_elems, d_sigmas);
    return cudaGetLastError();
}

}  // namespace dogblob
