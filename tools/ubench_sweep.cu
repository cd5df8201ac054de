// Microbenchmark of the sliding-window inner loop (no global loads): how close to the
// FFMA2 peak does the 32-FFMA2-per-step pattern get with the tap ring in uniform vs
// vector registers, at different occupancies?
#include <cuda_runtime.h>
#include <cstdio>

constexpr int TY = 16;

template <bool FORCE_VEC, int MINB>
__global__ void __launch_bounds__(256, MINB) sweep_kernel(float *out, int chunks, int zero) {
    __shared__ float2 taps[1024];
    __shared__ float4 rows[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        taps[i] = make_float2(1.0f / (i + 1), 1.0f / (i + 1));
        rows[i] = make_float4(i, i + 1, i + 2, i + 3);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int off = FORCE_VEC ? zero * lane : 0;   // not provably uniform -> ring stays in vector regs
    float2 acc[TY][2], ring[TY];
#pragma unroll
    for (int j = 0; j < TY; ++j) { ring[j] = make_float2(0, 0); acc[j][0] = acc[j][1] = make_float2(0, 0); }
    const float2 *tp = taps;
    const float4 *rp = rows + lane;
    for (int c = 0; c < chunks; ++c) {
#pragma unroll
        for (int u = 0; u < TY; ++u) {
            ring[u] = tp[u + off];
            const float4 v = rp[u * 32 & 1023];
            const float2 a = make_float2(v.x, v.y), b = make_float2(v.z, v.w);
#pragma unroll
            for (int j = 0; j < TY; ++j) {
                const float2 t = ring[(u - j + TY) % TY];
                acc[j][0] = __ffma2_rn(t, a, acc[j][0]);
                acc[j][1] = __ffma2_rn(t, b, acc[j][1]);
            }
        }
        tp = taps + ((c * TY) & 511);
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < TY; ++j) s += acc[j][0].x + acc[j][0].y + acc[j][1].x + acc[j][1].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <bool FORCE_VEC, int MINB>
void run(const char *name, int blocks_per_sm) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int blocks = sms * blocks_per_sm, chunks = 2000;
    float *out; cudaMalloc(&out, (size_t)blocks * 256 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    sweep_kernel<FORCE_VEC, MINB><<<blocks, 256>>>(out, chunks, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    sweep_kernel<FORCE_VEC, MINB><<<blocks, 256>>>(out, chunks, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)blocks * 256 * chunks * TY * TY * 2 * 2 * 2;
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, sweep_kernel<FORCE_VEC, MINB>);
    printf("%-32s blocks/SM=%d regs=%d  %.1f TFLOP/s (%.3f ms)\n", name, blocks_per_sm, fa.numRegs,
           flops / (ms * 1e-3) / 1e12, ms);
    cudaFree(out);
}

int main() {
    run<false, 2>("ring uniform, 2 CTA/SM", 2);
    run<false, 2>("ring uniform, lb2 (1 resident)", 1);
    run<false, 1>("ring uniform, 1 CTA/SM", 1);
    run<true, 2>("ring vector, 2 CTA/SM", 2);
    run<true, 1>("ring vector, 1 CTA/SM", 1);
    run<false, 3>("ring uniform, 3 CTA/SM", 3);
    return 0;
}
