// Sliding-window inner loop WITH the global-load path of the real kernels:
// variants of addressing / prefetch depth, to find what costs FMA-pipe utilisation.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

constexpr int TY = 16;

// MODE 0: rows from smem (reference, no LDG)
// MODE 1: LDG.128, int32 element-offset table in smem (current kernel)
// MODE 2: LDG.128, int64 byte-offset table in smem
// MODE 3: LDG.128, running pointer p += pitch (no table, no boundary logic)
template <int MODE, int PF>
__global__ void __launch_bounds__(256, 2) sweep_kernel(const float *__restrict__ img, int64_t pitch,
                                                      float *out, int chunks, int n_rows) {
    extern __shared__ __align__(16) unsigned char smem[];
    float2 *taps = reinterpret_cast<float2 *>(smem);             // 1024
    float4 *srows = reinterpret_cast<float4 *>(taps + 1024);     // 1024
    int *tbl32 = reinterpret_cast<int *>(srows + 1024);          // 4096
    long long *tbl64 = reinterpret_cast<long long *>(tbl32 + 4096);   // 4096
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        taps[i] = make_float2(1.0f / (i + 1), 1.0f / (i + 1));
        srows[i] = make_float4(i, i + 1, i + 2, i + 3);
    }
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
        int r = (blockIdx.x * 7 + i) % n_rows;
        tbl32[i] = r * (int)pitch;
        tbl64[i] = (long long)r * pitch * 4;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float *base = img + (blockIdx.x % 8) * 128;
    const char *bbase = reinterpret_cast<const char *>(base) + lane * 16;
    const int *r32 = tbl32 + warp * 16;
    const long long *r64 = tbl64 + warp * 16;
    const float *p = base + (int64_t)((blockIdx.x * 7 + warp * 16) % n_rows) * pitch;
    float4 v[PF];
    auto load = [&](int idx) -> float4 {
        if (MODE == 1) return __ldg(reinterpret_cast<const float4 *>(base + r32[idx]) + lane);
        if (MODE == 2) return __ldg(reinterpret_cast<const float4 *>(bbase + r64[idx]));
        if (MODE == 3) { float4 q = __ldg(reinterpret_cast<const float4 *>(p) + lane); p += pitch; return q; }
        return srows[(idx * 32 + lane) & 1023];
    };
    int idx = 0;
#pragma unroll
    for (int k = 0; k < PF; ++k) v[k] = load(idx++);
    float2 acc[TY][2], ring[TY];
#pragma unroll
    for (int j = 0; j < TY; ++j) { ring[j] = make_float2(0, 0); acc[j][0] = acc[j][1] = make_float2(0, 0); }
    const float2 *tp = taps;
    for (int c = 0; c < chunks; ++c) {
#pragma unroll
        for (int u = 0; u < TY; ++u) {
            ring[u] = tp[u];
            const float4 q = v[u % PF];
            const float2 a = make_float2(q.x, q.y), b = make_float2(q.z, q.w);
            v[u % PF] = load(idx + u);
#pragma unroll
            for (int j = 0; j < TY; ++j) {
                const float2 t = ring[(u - j + TY) % TY];
                acc[j][0] = __ffma2_rn(t, a, acc[j][0]);
                acc[j][1] = __ffma2_rn(t, b, acc[j][1]);
            }
        }
        tp = taps + ((c * TY) & 511);
        idx = (idx + TY) & 2047;
        if (MODE == 3 && (c & 15) == 15) p = base + (int64_t)((blockIdx.x * 7 + warp * 16) % n_rows) * pitch;
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < TY; ++j) s += acc[j][0].x + acc[j][0].y + acc[j][1].x + acc[j][1].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int PF>
void run(const char *name, const float *img, int64_t pitch, int n_rows, int chunks = 40, int waves = 4) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int blocks = sms * 2 * waves;
    float *out; cudaMalloc(&out, (size_t)blocks * 256 * 4);
    size_t smem = 1024 * 8 + 1024 * 16 + 4096 * 4 + 4096 * 8;
    cudaFuncSetAttribute(sweep_kernel<MODE, PF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    sweep_kernel<MODE, PF><<<blocks, 256, smem>>>(img, pitch, out, chunks, n_rows);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) sweep_kernel<MODE, PF><<<blocks, 256, smem>>>(img, pitch, out, chunks, n_rows);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    double flops = (double)blocks * 256 * chunks * TY * TY * 2 * 2 * 2;
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, sweep_kernel<MODE, PF>);
    printf("%-40s regs=%3d spill=%4zu  %.1f TFLOP/s (%.3f ms) err=%s\n", name, fa.numRegs, fa.localSizeBytes,
           flops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    const int n_rows = 1024; const int64_t pitch = 1024;
    float *img; cudaMalloc(&img, n_rows * pitch * 4 * 8); cudaMemset(img, 0, n_rows * pitch * 4 * 8);
    run<0, 4>("smem rows (no LDG)", img, pitch, n_rows);
    run<1, 4>("LDG int32 table PF=4 (current)", img, pitch, n_rows);
    run<2, 4>("LDG int64 byte table PF=4", img, pitch, n_rows);
    run<3, 4>("LDG running pointer PF=4", img, pitch, n_rows);
    run<1, 2>("LDG int32 table PF=2", img, pitch, n_rows);
    run<2, 2>("LDG int64 byte table PF=2", img, pitch, n_rows);
    run<2, 6>("LDG int64 byte table PF=6", img, pitch, n_rows);
    run<1, 8>("LDG int32 table PF=8", img, pitch, n_rows);
    run<1, 4>("current, 160 chunks x 1 wave", img, pitch, n_rows, 160, 1);
    run<1, 4>("current, 20 chunks x 8 waves", img, pitch, n_rows, 20, 8);
    run<1, 4>("current, 11 chunks x 13 waves", img, pitch, n_rows, 11, 13);
    run<1, 4>("current, 5 chunks x 32 waves", img, pitch, n_rows, 5, 32);
    run<1, 4>("current, 2 chunks x 80 waves", img, pitch, n_rows, 2, 80);
    return 0;
}
