// Pre-processing on the GPU: Gaussian smoothing + saturation-bounded contrast stretch.
//
// Replaces images.preprocess (pkg/src/dogblob/images.py:112-157), which Detector.run
// applies when params.preprocess is set (detector.py:339-340):
//   smooth           = scipy.ndimage.gaussian_filter(img, sigma, mode="reflect", truncate=5)
//                      on float32: axis 0 then axis 1, each line filtered in float64 by the
//                      symmetric branch of NI_Correlate1D
//                          tmp = x[l] * w[0];  for k = R..1: tmp += (x[l-k] + x[l+k]) * w[k]
//                      (separate multiply and add) and rounded to float32 on store;
//   contrast_stretch = lo/hi are the nearest-rank quantiles of the sorted image,
//                      out = clip((v - f32(lo)) / f32(hi - lo), 0, 1), all zeros if hi <= lo.
// The order statistics are found exactly with a 4-pass 8-bit radix select over the
// order-preserving integer image of the float32 values (no sort).  The library is
// compiled with -fmad=false, so the float64 accumulation below is not contracted.
#include "common.cuh"

namespace dogblob {

namespace {

constexpr int kMaxSmoothRadius = 255;     // smooth_sigma <= 50 (the service's bound): radius int(5 sigma + 0.5) <= 250

struct SmoothWeights {
    double w[kMaxSmoothRadius + 1];   // w[0] centre ... w[radius]
    int radius;
};

struct SelectState {                  // lives at the start of the scratch buffer
    unsigned int hist[2][256];
    unsigned int prefix[2];
    unsigned long long rank[2];
    unsigned int done;                // CTA ticket of the current pass
    unsigned int status;              // bit 0: non-finite input pixel
    unsigned int pad[2];
};

constexpr size_t kStateBytes = 4096;
static_assert(sizeof(SelectState) <= kStateBytes, "SelectState outgrew its slot");

__device__ __forceinline__ int fold(int i, int n) {
    const int period = 2 * n;
    int t = i % period;
    if (t < 0) t += period;
    return t < n ? t : period - 1 - t;
}

// AXIS 0: filter along y (lines are columns); AXIS 1: along x.
template <int AXIS>
__global__ void __launch_bounds__(256)
smooth_axis_kernel(const float *__restrict__ src, int64_t src_pitch, float *__restrict__ dst,
                   int64_t dst_pitch, int H, int W, SmoothWeights sw, SelectState *state) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= W) return;
    const float centre = src[(int64_t)y * src_pitch + x];
    if (AXIS == 0 && !isfinite(centre)) atomicOr(&state->status, 1u);
    double tmp = (double)centre * sw.w[0];
    for (int k = sw.radius; k >= 1; --k) {
        double a, b;
        if (AXIS == 0) {
            a = (double)src[(int64_t)fold(y - k, H) * src_pitch + x];
            b = (double)src[(int64_t)fold(y + k, H) * src_pitch + x];
        } else {
            a = (double)src[(int64_t)y * src_pitch + fold(x - k, W)];
            b = (double)src[(int64_t)y * src_pitch + fold(x + k, W)];
        }
        tmp = tmp + (a + b) * sw.w[k];
    }
    dst[(int64_t)y * dst_pitch + x] = (float)tmp;
}

__device__ __forceinline__ unsigned int ordered_key(float v) {
    const unsigned int u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_to_float(unsigned int k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__global__ void select_init_kernel(SelectState *state, unsigned long long rank_lo,
                                   unsigned long long rank_hi) {
    const int t = threadIdx.x;
    state->hist[0][t] = 0;
    state->hist[1][t] = 0;
    if (t == 0) {
        state->prefix[0] = state->prefix[1] = 0;
        state->rank[0] = rank_lo;
        state->rank[1] = rank_hi;
        state->done = 0;
        state->status = 0;
    }
}

// One radix pass (digit `pass`, most significant first) for both order statistics;
// the last CTA to finish narrows prefix/rank and clears the histograms.
__global__ void __launch_bounds__(256)
select_pass_kernel(const float *__restrict__ img, int64_t pitch, int H, int W, int pass,
                   SelectState *state) {
    __shared__ unsigned int h[2][256];
    __shared__ bool last;
    h[0][threadIdx.x] = 0;
    h[1][threadIdx.x] = 0;
    __syncthreads();
    const int shift = 24 - 8 * pass;
    const unsigned int p0 = state->prefix[0], p1 = state->prefix[1];
    const int64_t total = (int64_t)H * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / W), x = (int)(i - (int64_t)y * W);
        const unsigned int key = ordered_key(img[(int64_t)y * pitch + x]);
        const unsigned int hi_bits = pass == 0 ? 0u : (key >> (shift + 8));
        const unsigned int digit = (key >> shift) & 255u;
        if (pass == 0 || hi_bits == p0) atomicAdd(&h[0][digit], 1u);
        if (pass == 0 || hi_bits == p1) atomicAdd(&h[1][digit], 1u);
    }
    __syncthreads();
    if (h[0][threadIdx.x]) atomicAdd(&state->hist[0][threadIdx.x], h[0][threadIdx.x]);
    if (h[1][threadIdx.x]) atomicAdd(&state->hist[1][threadIdx.x], h[1][threadIdx.x]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(&state->done, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x < 2) {
        const int t = threadIdx.x;
        unsigned long long rank = state->rank[t], cum = 0;
        unsigned int digit = 255;
        for (unsigned int b = 0; b < 256; ++b) {
            const unsigned long long c = ((volatile unsigned int *)state->hist[t])[b];
            if (rank < cum + c) { digit = b; break; }
            cum += c;
        }
        state->rank[t] = rank - cum;
        state->prefix[t] = (state->prefix[t] << 8) | digit;
    }
    __syncthreads();
    state->hist[0][threadIdx.x] = 0;
    state->hist[1][threadIdx.x] = 0;
    if (threadIdx.x == 0) state->done = 0;
}

__global__ void __launch_bounds__(256)
stretch_kernel(const float *__restrict__ src, int64_t src_pitch, float *__restrict__ dst,
               int64_t dst_pitch, int H, int W, const SelectState *__restrict__ state) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= W) return;
    const float lo = key_to_float(state->prefix[0]);
    const float hi = key_to_float(state->prefix[1]);
    float out = 0.f;
    if (hi > lo) {
        const float scale = (float)((double)hi - (double)lo);   // np.float32(hi - lo), hi/lo Python floats
        out = __fdiv_rn(__fsub_rn(src[(int64_t)y * src_pitch + x], lo), scale);
        out = fminf(fmaxf(out, 0.f), 1.f);
    }
    dst[(int64_t)y * dst_pitch + x] = out;
}

}  // namespace

size_t preprocess_bytes(int H, int W) {
    const size_t pitch = ((size_t)W + 127) / 128 * 128;
    return kStateBytes + 2 * (size_t)H * pitch * sizeof(float);
}

cudaError_t launch_preprocess(int H, int W, const float *d_src, int64_t src_pitch, int radius,
                              const double *weights, int64_t rank_lo, int64_t rank_hi,
                              void *d_scratch, float *d_dst, int64_t dst_pitch, cudaStream_t st) {
    SmoothWeights sw;
    sw.radius = radius;
    for (int k = 0; k <= kMaxSmoothRadius; ++k) sw.w[k] = (k <= radius) ? weights[k] : 0.0;
    auto *state = reinterpret_cast<SelectState *>(d_scratch);
    const int64_t pitch = ((int64_t)W + 127) / 128 * 128;
    float *tmp0 = reinterpret_cast<float *>(reinterpret_cast<char *>(d_scratch) + kStateBytes);
    float *tmp1 = tmp0 + (size_t)H * pitch;
    const dim3 grid((W + 255) / 256, H);
    select_init_kernel<<<1, 256, 0, st>>>(state, (unsigned long long)rank_lo,
                                         (unsigned long long)rank_hi);
    smooth_axis_kernel<0><<<grid, 256, 0, st>>>(d_src, src_pitch, tmp0, pitch, H, W, sw, state);
    smooth_axis_kernel<1><<<grid, 256, 0, st>>>(tmp0, pitch, tmp1, pitch, H, W, sw, state);
    const int64_t total = (int64_t)H * W;
    int blocks = (int)((total + 256 * 8 - 1) / (256 * 8));
    if (blocks > 148 * 4) blocks = 148 * 4;
    if (blocks < 1) blocks = 1;
    for (int pass = 0; pass < 4; ++pass)
        select_pass_kernel<<<blocks, 256, 0, st>>>(tmp1, pitch, H, W, pass, state);
    stretch_kernel<<<grid, 256, 0, st>>>(tmp1, pitch, d_dst, dst_pitch, H, W, state);
    return cudaGetLastError();
}

}  // namespace dogblob

using namespace dogblob;

extern "C" {

size_t dogblob_preprocess_bytes(int height, int width) {
    return (height >= 1 && width >= 1) ? preprocess_bytes(height, width) : 0;
}

int dogblob_preprocess(int height, int width, const float *d_src, int64_t src_pitch, int radius,
                       const double *weights, int64_t rank_lo, int64_t rank_hi, void *d_scratch,
                       float *d_dst, int64_t dst_pitch, void *stream) {
    DB_REQUIRE(height >= 1 && width >= 1, "expected a non-empty 2-D image");
    DB_REQUIRE(d_src && weights && d_scratch && d_dst, "NULL argument");
    DB_REQUIRE(radius >= 0 && radius <= kMaxSmoothRadius,
               "smoothing radius above 255 (smooth_sigma > 51) is not supported");
    DB_REQUIRE(src_pitch >= width && dst_pitch >= width, "pitch smaller than the image width");
    const int64_t n = (int64_t)height * width;
    DB_REQUIRE(rank_lo >= 0 && rank_lo < n && rank_hi >= 0 && rank_hi < n, "rank out of range");
    DB_CUDA(launch_preprocess(height, width, d_src, src_pitch, radius, weights, rank_lo, rank_hi,
                              d_scratch, d_dst, dst_pitch, reinterpret_cast<cudaStream_t>(stream)));
    return DOGBLOB_OK;
}

int dogblob_preprocess_status(const void *d_scratch, uint32_t *h_status, void *stream) {
    DB_REQUIRE(d_scratch && h_status, "NULL argument");
    const char *p = reinterpret_cast<const char *>(d_scratch) + offsetof(SelectState, status);
    DB_CUDA(cudaMemcpyAsync(h_status, p, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                            reinterpret_cast<cudaStream_t>(stream)));
    return DOGBLOB_OK;
}

int dogblob_event_record(void *event, void *stream) {
    DB_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(event),
                            reinterpret_cast<cudaStream_t>(stream)));
    return DOGBLOB_OK;
}

}  // extern "C"
