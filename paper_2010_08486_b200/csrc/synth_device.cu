// PLIF-like synthetic frames generated ON the device, for throughput / precision-recall sweeps
// over thousands of frames (the scene model of synth.py:50-162: bright sphere-cap
// droplets v(d) = sqrt(1 - (d/r)^2) on black, rim antialiased by 4 x 4 sub-pixel coverage, maximum
// composition, then Poisson(scale v) / scale shot noise + N(0, sigma) read noise, clamped at 0).
//
// PERF ONLY: the random streams are a counter-based hash, not numpy's PCG64 / ziggurat, so these
// frames are statistically like the reference's but not bit-identical to them.  Parity is always
// judged on frames of the host generator (synth.py, sha256-pinned against the reference).
#include "common.cuh"

namespace dogblob {

namespace {

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {      // splitmix64 finaliser
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned long long rng_u64(unsigned long long seed, unsigned long long stream,
                                                      unsigned long long counter) {
    return mix64(mix64(seed + 0x9e3779b97f4a7c15ull * (stream + 1)) ^ (counter * 0xd1342543de82ef95ull + 1));
}
__device__ __forceinline__ double u01(unsigned long long x) { return (double)(x >> 11) * (1.0 / 9007199254740992.0); }

// truth[f][i] = (x, y, r): r uniform in [r_min, r_max], centre uniform with the whole antialiased
// footprint inside the frame (synth.py:127-131 with allow_overlap=True)
__global__ void place_kernel(int n_frames, int n_droplets, int H, int W, double r_min, double r_max,
                             unsigned long long seed, double *__restrict__ truth) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_frames * n_droplets) return;
    const unsigned long long f = i / n_droplets, d = i % n_droplets;
    const double r = r_min + (r_max - r_min) * u01(rng_u64(seed, 3 * f, 3 * d));
    const double lo = r + 1.0;
    const double x = lo + (W - 1.0 - r - 1.0 - lo) * u01(rng_u64(seed, 3 * f, 3 * d + 1));
    const double y = lo + (H - 1.0 - r - 1.0 - lo) * u01(rng_u64(seed, 3 * f, 3 * d + 2));
    truth[3 * (int64_t)i] = x;
    truth[3 * (int64_t)i + 1] = y;
    truth[3 * (int64_t)i + 2] = r;
}

// one CTA per (frame, droplet): 4 x 4 supersampled sphere cap over the footprint, maximum composition
// (non-negative floats order like their bit patterns: atomicMax on int)
__global__ void __launch_bounds__(256)
paint_kernel(int n_droplets, int H, int W, int64_t pitch, const double *__restrict__ truth, float *__restrict__ frames) {
    const int f = blockIdx.y, d = blockIdx.x;
    const double *t = truth + 3 * ((int64_t)f * n_droplets + d);
    const double cx = t[0], cy = t[1], r = t[2];
    const int y0 = max((int)floor(cy - r - 1.0), 0), y1 = min((int)ceil(cy + r + 1.0) + 1, H);
    const int x0 = max((int)floor(cx - r - 1.0), 0), x1 = min((int)ceil(cx + r + 1.0) + 1, W);
    const int nx = x1 - x0, n = nx * (y1 - y0);
    float *img = frames + (int64_t)f * H * pitch;
    const double inv_r2 = 1.0 / (r * r);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const int y = y0 + k / nx, x = x0 + k % nx;
        double acc = 0.0;
#pragma unroll
        for (int sy = 0; sy < 4; ++sy)
#pragma unroll
            for (int sx = 0; sx < 4; ++sx) {
                const double dy = y + (sy + 0.5) * 0.25 - 0.5 - cy, dx = x + (sx + 0.5) * 0.25 - 0.5 - cx;
                acc += sqrt(fmax(1.0 - (dy * dy + dx * dx) * inv_r2, 0.0));
            }
        const float v = (float)(acc * (1.0 / 16.0));
        if (v > 0.f) atomicMax(reinterpret_cast<int *>(img + (int64_t)y * pitch + x), __float_as_int(v));
    }
}

// shot noise + read noise, in place.  Poisson: exact inversion below lambda = 12, the rounded
// normal approximation above (relative error of the variance < 1 %: fine for a perf generator).
__global__ void __launch_bounds__(256)
noise_kernel(int n_frames, int H, int W, int64_t pitch, unsigned long long seed, double scale, double sigma,
             float *__restrict__ frames) {
    const int64_t total = (int64_t)n_frames * H * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = i / ((int64_t)H * W), rem = i - f * (int64_t)H * W;
        const int y = (int)(rem / W), x = (int)(rem % W);
        float *p = frames + (f * H + y) * pitch + x;
        const double lam = fmax((double)*p, 0.0) * scale;
        const unsigned long long a = rng_u64(seed, 3 * f + 1, 2 * (unsigned long long)rem);
        const unsigned long long b = rng_u64(seed, 3 * f + 1, 2 * (unsigned long long)rem + 1);
        // two independent normals (Box-Muller)
        const double u1 = fmax(u01(a), 1e-300), u2 = u01(b);
        const double rad = sqrt(-2.0 * log(u1));
        double s, c;
        sincospi(2.0 * u2, &s, &c);
        double count;
        if (lam < 12.0) {
            double prod = u01(rng_u64(seed, 3 * f + 2, (unsigned long long)rem * 64)), limit = exp(-lam);
            int k = 0;
            while (prod > limit && k < 63) {
                ++k;
                prod *= u01(rng_u64(seed, 3 * f + 2, (unsigned long long)rem * 64 + k));
            }
            count = (double)k;
        } else {
            count = fmax(rint(lam + sqrt(lam) * rad * c), 0.0);
        }
        const double v = count / scale + sigma * rad * s;
        *p = (float)fmax(v, 0.0);
    }
}

}  // namespace

cudaError_t launch_synth_frames(int n_frames, int H, int W, int64_t pitch, int n_droplets, double r_min,
                                double r_max, unsigned long long seed, double poisson_scale, double gaussian_sigma,
                                float *d_frames, double *d_truth, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(d_frames, 0, (size_t)n_frames * H * pitch * sizeof(float), st);
    if (e != cudaSuccess) return e;
    if (n_droplets > 0) {
        const int n = n_frames * n_droplets;
        place_kernel<<<(n + 255) / 256, 256, 0, st>>>(n_frames, n_droplets, H, W, r_min, r_max, seed, d_truth);
        paint_kernel<<<dim3(n_droplets, n_frames), 256, 0, st>>>(n_droplets, H, W, pitch, d_truth, d_frames);
    }
    if (poisson_scale > 0.0)
        noise_kernel<<<148 * 8, 256, 0, st>>>(n_frames, H, W, pitch, seed, poisson_scale, gaussian_sigma, d_frames);
    return cudaGetLastError();
}

}  // namespace dogblob
