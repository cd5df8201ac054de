// Where does an M = 64 tcgen05.mma (cta_group::1, kind::f16) put its accumulator rows in TMEM, may the
// accumulator address carry a lane offset, and what does it cost next to M = 128?  (Question behind it: the
// first / last four k-steps of every level only reach one half of the 128 Toeplitz rows.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ubench_umma_m64 tools/ubench_umma_m64.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    long long t0 = clock64();
    while (!mbar_try_wait(bar, parity))
        if (clock64() - t0 > 2000000000ll) { printf("timeout\n"); __trap(); }
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void umma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__host__ __device__ constexpr uint32_t instr_desc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// K-major, no swizzle: [K half 2][row group][8 rows][8 halfs]; LBO = bytes between the K halves, SBO = 128
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t addr, uint32_t lbo) {
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(128u >> 4) << 32) | (1ull << 46);
}

constexpr int kRowsA = 128, kRowsB = 256;

__global__ void __launch_bounds__(128) layout_kernel(float *out, int m, int lane_off, int a_row_off) {
    __shared__ __align__(1024) __half sa[2 * kRowsA * 8];
    __shared__ __align__(1024) __half sb[2 * kRowsB * 8];
    __shared__ unsigned long long bar;
    __shared__ uint32_t tmem_slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 2 * kRowsA * 8; i += 128) {
        const int kh = i / (kRowsA * 8), r = (i / 8) % kRowsA, e = i % 8;
        sa[i] = __float2half((kh == 0 && e == 0) ? (float)(r + 1) : 0.f);     // A[r][0] = r + 1
    }
    for (int i = tid; i < 2 * kRowsB * 8; i += 128) {
        const int kh = i / (kRowsB * 8), e = i % 8;
        sb[i] = __float2half((kh == 0 && e == 0) ? 1.f : 0.f);                // B[n][0] = 1
    }
    if (tid == 0) { mbar_init(smem_u32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    fence_proxy_async();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)), "r"(32u) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    // sentinel in all 128 lanes x 16 columns
    {
        const uint32_t s = __float_as_uint(-1.f);
        const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};"
                     ::"r"(ta), "r"(s) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint64_t ad = desc_kmajor(smem_u32(sa) + (uint32_t)a_row_off * 16u, kRowsA * 16);
        const uint64_t bd = desc_kmajor(smem_u32(sb), kRowsB * 16);
        umma_ss(tmem + ((uint32_t)lane_off << 16), ad, bd, instr_desc_f16(m, 16), 0u);
        umma_commit(smem_u32(&bar));
    }
    mbar_wait(smem_u32(&bar), 0);
    tc_fence_after();
    uint32_t r[16];
    const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n\t"
                 "tcgen05.wait::ld.sync.aligned;"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(ta) : "memory");
    for (int j = 0; j < 16; ++j) out[tid * 16 + j] = __uint_as_float(r[j]);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32u) : "memory");
}

// cost: `reps` back-to-back MMAs of (m, n), one commit
__global__ void __launch_bounds__(128) cost_kernel(long long *cycles, int m, int n, int reps) {
    __shared__ __align__(1024) __half sa[2 * kRowsA * 8];
    __shared__ __align__(1024) __half sb[2 * kRowsB * 8];
    __shared__ unsigned long long bar;
    __shared__ uint32_t tmem_slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 2 * kRowsA * 8; i += 128) sa[i] = __float2half(0.5f);
    for (int i = tid; i < 2 * kRowsB * 8; i += 128) sb[i] = __float2half(0.25f);
    if (tid == 0) { mbar_init(smem_u32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    fence_proxy_async();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)), "r"(256u) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (tid == 0) {
        const uint64_t ad = desc_kmajor(smem_u32(sa), kRowsA * 16);
        const uint64_t bd = desc_kmajor(smem_u32(sb), kRowsB * 16);
        const uint32_t id = instr_desc_f16(m, n);
        const long long t0 = clock64();
        for (int i = 0; i < reps; ++i) umma_ss(tmem, ad, bd, id, i > 0);
        umma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        cycles[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u) : "memory");
}

int main() {
    float *d_out;
    CK(cudaMalloc(&d_out, 128 * 16 * sizeof(float)));
    std::vector<float> h(128 * 16);
    const int cases[][3] = {{128, 0, 0}, {64, 0, 0}, {64, 64, 0}, {64, 0, 64}, {64, 64, 64}, {64, 32, 0}, {64, 16, 0}};
    for (auto &c : cases) {
        layout_kernel<<<1, 128>>>(d_out, c[0], c[1], c[2]);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("M = %d, D lane offset %d, A row offset %d: %s\n", c[0], c[1], c[2], cudaGetErrorString(e)); return 1; }
        CK(cudaMemcpy(h.data(), d_out, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
        printf("M = %3d, D lane offset %2d, A row offset %2d: lane -> A row (column 0; '.' = untouched):\n  ", c[0], c[1], c[2]);
        for (int l = 0; l < 128; ++l) {
            if (h[l * 16] == -1.f) printf(" .");
            else printf(" %d", (int)h[l * 16] - 1);
            if (l % 32 == 31) printf("\n  ");
        }
        bool cols_same = true;
        for (int l = 0; l < 128; ++l)
            for (int j = 1; j < 16; ++j) cols_same = cols_same && h[l * 16 + j] == h[l * 16];
        printf("all 16 columns equal: %s\n", cols_same ? "yes" : "NO");
    }
    long long *d_c, hc[148];
    CK(cudaMalloc(&d_c, 148 * sizeof(long long)));
    for (int ctas : {1, 148})
        for (int m : {128, 64})
            for (int n : {128, 256}) {
                cost_kernel<<<ctas, 128>>>(d_c, m, n, 256);
                CK(cudaDeviceSynchronize());
                cost_kernel<<<ctas, 128>>>(d_c, m, n, 256);
                CK(cudaDeviceSynchronize());
                CK(cudaMemcpy(hc, d_c, ctas * sizeof(long long), cudaMemcpyDeviceToHost));
                long long mx = 0;
                for (int i = 0; i < ctas; ++i) mx = hc[i] > mx ? hc[i] : mx;
                printf("%3d CTAs, M = %3d, N = %3d: %.1f cycles per MMA (256 back to back + commit)\n", ctas, m, n, mx / 256.0);
            }
    return 0;
}
