// Does a shared-memory matrix descriptor accept a NEGATIVE leading byte offset (two's complement in
// its 14-bit field, i.e. address arithmetic modulo 2^18)?  If so a Toeplitz operand T[n][k] =
// v[k - n + c] needs only ONE 16-byte chunk per row (the K half 1 of row n is the K half 0 of row
// n - 8): half the shared memory and half the copy of the prebuilt arrays.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ubench_toeplitz_wrap tools/ubench_toeplitz_wrap.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

extern __shared__ __align__(1024) unsigned char smem[];

// A = Toeplitz (compact, M = 128 rows), B = data [N = 128][16] K-major no swizzle; D = A * B^T
__global__ void __launch_bounds__(128, 1) wrap_kernel(const __half *g_compact, const __half *g_b, float *out, int variant) {
    __shared__ __align__(8) unsigned long long bar;
    __shared__ uint32_t tmem_slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)), "r"(128u) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // compact array: (128 + 8) chunks of 16 B at smem + 0; B at smem + 4096 (4 KB)
    for (int i = threadIdx.x; i < 136 * 8; i += 128) reinterpret_cast<__half *>(smem)[i] = g_compact[i];
    for (int i = threadIdx.x; i < 128 * 16; i += 128) reinterpret_cast<__half *>(smem + 4096)[i] = g_b[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        // row n, K half 0 at base + 16 (n + 8); K half 1 = 128 bytes BELOW
        const uint32_t a_addr = smem_u32(smem) + 128;
        uint64_t adesc;
        if (variant == 0)       // LBO = -128 as a 14-bit two's complement field
            adesc = (uint64_t)((a_addr & 0x3ffffu) >> 4) | ((uint64_t)0x3ff8u << 16) | ((uint64_t)(128u >> 4) << 32) | (1ull << 46);
        else                    // control: LBO = +128 (wrong operand, must mismatch)
            adesc = (uint64_t)((a_addr & 0x3ffffu) >> 4) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(128u >> 4) << 32) | (1ull << 46);
        const uint64_t bdesc = (uint64_t)(((smem_u32(smem) + 4096) & 0x3ffffu) >> 4) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(256u >> 4) << 32) | (1ull << 46);
        const uint32_t idesc = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(adesc), "l"(bdesc), "r"(idesc) : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    }
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c = 0; c < 128; c += 8) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n\ttcgen05.wait::ld.sync.aligned;"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(tmem + ((uint32_t)(32 * warp) << 16) + c) : "memory");
        for (int j = 0; j < 8; ++j) out[(32 * warp + lane) * 128 + c + j] = __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u) : "memory");
}

int main() {
    // v[i], A[n][k] = v[k - n + 127], n < 128, k < 16 -> i in [0, 142]
    std::vector<float> v(160);
    for (auto &x : v) x = (float)(rand() % 64 - 32) / 8.f;
    std::vector<float> B(128 * 16);
    for (auto &x : B) x = (float)(rand() % 64 - 32) / 8.f;
    // compact: chunk for row n (n = -8 .. 127), element e: v[e - n + 127]
    std::vector<__half> compact(136 * 8), hb(128 * 16);
    for (int n = -8; n < 128; ++n)
        for (int e = 0; e < 8; ++e) {
            const int i = e - n + 127;
            compact[(n + 8) * 8 + e] = __float2half(i >= 0 && i < 160 ? v[i] : 0.f);
        }
    // B K-major no swizzle: 8-row groups of 256 B = [K half 0: 8 rows x 16 B][K half 1]
    for (int n = 0; n < 128; ++n)
        for (int k = 0; k < 16; ++k) hb[(n >> 3) * 128 + (k >> 3) * 64 + (n & 7) * 8 + (k & 7)] = __float2half(B[n * 16 + k]);
    __half *d_c, *d_b;
    float *d_out;
    CK(cudaMalloc(&d_c, compact.size() * 2)); CK(cudaMalloc(&d_b, hb.size() * 2)); CK(cudaMalloc(&d_out, 128 * 128 * 4));
    CK(cudaMemcpy(d_c, compact.data(), compact.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_b, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice));
    for (int variant = 0; variant < 2; ++variant) {
        CK(cudaMemset(d_out, 0, 128 * 128 * 4));
        wrap_kernel<<<1, 128, 8192>>>(d_c, d_b, d_out, variant);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("variant %d: %s\n", variant, cudaGetErrorString(e)); return 1; }
        std::vector<float> out(128 * 128);
        CK(cudaMemcpy(out.data(), d_out, out.size() * 4, cudaMemcpyDeviceToHost));
        double worst = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 128; ++n) {
                double ref = 0;
                for (int k = 0; k < 16; ++k) ref += (double)v[k - m + 127] * B[n * 16 + k];
                worst = fmax(worst, fabs(ref - out[m * 128 + n]));
            }
        printf("variant %d (%s): max |err| = %g %s\n", variant, variant == 0 ? "LBO = -128 (wrapped)" : "LBO = +128 (control, must differ)", worst,
               worst < 1e-3 ? "MATCH" : "mismatch");
    }
    return 0;
}
