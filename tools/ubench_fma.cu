// Microbenchmark: FP32 FMA issue rate on sm_100a, scalar FFMA vs packed FFMA2,
// with register and with shared-memory/uniform operands. Prints TFLOP/s.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

template <int MODE>
__global__ void __launch_bounds__(256) fma_kernel(float *out, int iters, float a0, float b0) {
    float2 acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    float2 a = make_float2(a0, a0 * 1.0001f), b = make_float2(b0, b0 * 0.9999f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if (MODE == 0) {            // scalar FFMA x2
                    acc[i].x = fmaf(acc[i].x, a.x, b.x);
                    acc[i].y = fmaf(acc[i].y, a.y, b.y);
                } else {                    // packed
                    acc[i] = __ffma2_rn(acc[i], a, b);
                }
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i].x + acc[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
double run(int blocks, int iters) {
    float *out;
    cudaMalloc(&out, (size_t)blocks * 256 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    fma_kernel<MODE><<<blocks, 256>>>(out, iters, 0.999f, 0.001f);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    fma_kernel<MODE><<<blocks, 256>>>(out, iters, 0.999f, 0.001f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)blocks * 256 * iters * 8.0 * 16 * 2 * 2;
    cudaFree(out);
    return flops / (ms * 1e-3) / 1e12;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SMs=%d clock=%d kHz\n", sms, clk);
    for (int occ : {1, 2, 4, 8}) {
        int blocks = sms * occ;
        printf("blocks/SM=%d  FFMA: %.1f TFLOP/s   FFMA2: %.1f TFLOP/s\n", occ,
               run<0>(blocks, 4000), run<1>(blocks, 4000));
    }
    return 0;
}
