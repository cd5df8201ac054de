// Micro-benchmark: what does tcgen05.commit cost the issuing thread, alone and between MMAs?
// (round 2: the scale-space passes spent ~420 cycles per commit in their issuer warp.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ubench_umma_commit tools/ubench_umma_commit.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

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
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void umma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return (uint64_t)((addr & 0x3ffffu) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           (1ull << 46) | ((uint64_t)layout << 61);
}

// the scale-space kernel's issue statements (whole warp executes, one elected lane issues)
__device__ __forceinline__ void umma_f16_triple_ss(uint32_t d_main, uint32_t d_small, uint32_t a_hi, uint32_t a_lo,
                                                   uint32_t b_hi, uint32_t b_lo, uint32_t a_upper, uint32_t b_upper,
                                                   uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, q, e;\n\t.reg .b64 a0, a1, b0, b1;\n\t"
        "setp.ne.b32 p, %9, 0;\n\t"
        "setp.eq.b32 q, 0, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "mov.b64 a0, {%2, %6};\n\t"
        "mov.b64 a1, {%3, %6};\n\t"
        "mov.b64 b0, {%4, %7};\n\t"
        "mov.b64 b1, {%5, %7};\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a0, b0, %8, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%1], a0, b1, %8, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%1], a1, b0, %8, q;\n\t}"
        ::"r"(d_main), "r"(d_small), "r"(a_hi), "r"(a_lo), "r"(b_hi), "r"(b_lo), "r"(a_upper),
          "r"(b_upper), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
        ::"r"(bar) : "memory");
}

struct Args {
    int iters;          // groups
    int mmas;           // MMAs per group (0: none)
    int commits;        // commits per group (each to its own barrier of a ring of 8)
    int waiter;         // 1: a second warp waits on every barrier phase (like a TMA loader would)
    long long *cycles;
};

extern __shared__ __align__(1024) unsigned char smem[];

__global__ void __launch_bounds__(128, 1) commit_kernel(const Args a) {
    __shared__ __align__(8) unsigned long long bar[9];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) unsigned long long seq[2];
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 9; ++i) mbar_init(smem_u32(&bar[i]), (i == 8 && a.waiter >= 4) ? 2 : 1);
        mbar_init(smem_u32(&seq[0]), 1); mbar_init(smem_u32(&seq[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)), "r"(512u) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (uint32_t i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3c003c00u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_slot;
    const uint32_t idesc = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    if (threadIdx.x == 0 && a.waiter < 2) {
        const uint64_t ad = make_desc(smem_u32(smem), 128, 256, 0);
        const uint64_t bd = make_desc(smem_u32(smem + 16384), 128, 256, 0);
        const long long t0 = clock64();
        uint32_t c = 0;
        for (int it = 0; it < a.iters; ++it) {
            for (int m = 0; m < a.mmas; ++m) umma_ss(tmem + (m & 1) * 128, ad, bd, idesc, 1);
            for (int k = 0; k < a.commits; ++k, ++c) umma_commit(smem_u32(&bar[c & 7]));
        }
        const long long t1 = clock64();
        umma_commit(smem_u32(&bar[8]));
        while (!mbar_try_wait(smem_u32(&bar[8]), 0)) {}
        const long long t2 = clock64();
        if (blockIdx.x == 0) { a.cycles[0] = t1 - t0; a.cycles[1] = t2 - t0; }
    } else if (warp == 2 && a.waiter >= 2) {
        // kernel-style issue: the whole warp runs the loop, descriptors depend on the k-step
        const uint32_t a_lo = ((smem_u32(smem) & 0x3ffffu) >> 4) | ((128u >> 4) << 16);
        const uint32_t b_lo = ((smem_u32(smem + 32768) & 0x3ffffu) >> 4) | ((128u >> 4) << 16);
        const uint32_t upper = (256u >> 4) | (1u << 14);
        const long long t0 = clock64();
        uint32_t c = 0;
        for (int it = 0; it < a.iters; ++it) {
            if (a.waiter == 2) {
                for (int m = 0; m < a.mmas; ++m) {
                    const uint32_t w = a_lo + 32u * (uint32_t)(m & 7);
                    umma_f16_triple_ss(tmem, tmem + 128, w, w + 1024, b_lo + 16u * (uint32_t)(m & 3), b_lo + 512, upper, upper, idesc, m > 0);
                }
            } else {
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    if (m < a.mmas) {
                    const uint32_t w = a_lo + 32u * (uint32_t)(m & 7);
                    umma_f16_triple_ss(tmem, tmem + 128, w, w + 1024, b_lo + 16u * (uint32_t)(m & 3), b_lo + 512, upper, upper, idesc, m > 0);
                    }
                }
            }
            for (int k = 0; k < a.commits; ++k, ++c) umma_commit_elect(smem_u32(&bar[c & 7]));
        }
        const long long t1 = clock64();
        umma_commit_elect(smem_u32(&bar[8]));
        while (!mbar_try_wait(smem_u32(&bar[8]), 0)) {}
        const long long t2 = clock64();
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) { a.cycles[0] = t1 - t0; a.cycles[1] = t2 - t0; }
    } else if (threadIdx.x == 32 && a.waiter == 1) {
        const uint32_t total = (uint32_t)a.iters * a.commits;
        for (uint32_t c = 0; c < total; ++c)
            while (!mbar_try_wait(smem_u32(&bar[c & 7]), (c >> 3) & 1)) {}
    } else if ((warp == 0 || warp == 1) && a.waiter == 4) {
        // two issuer warps alternate groups; `seq` hands the issue order over (plain arrive after the
        // group's MMAs have been issued), each warp commits its own groups
        const uint32_t a_lo = ((smem_u32(smem) & 0x3ffffu) >> 4) | ((128u >> 4) << 16);
        const uint32_t b_lo = ((smem_u32(smem + 32768) & 0x3ffffu) >> 4) | ((128u >> 4) << 16);
        const uint32_t upper = (256u >> 4) | (1u << 14);
        const long long t0 = clock64();
        for (int it = warp; it < a.iters; it += 2) {
            if (it > 0) while (!mbar_try_wait(smem_u32(&seq[(it - 1) & 1]), ((it - 1) >> 1) & 1)) {}
            for (int m = 0; m < a.mmas; ++m) {
                const uint32_t w = a_lo + 32u * (uint32_t)(m & 7);
                umma_f16_triple_ss(tmem, tmem + 128, w, w + 1024, b_lo + 16u * (uint32_t)(m & 3), b_lo + 512, upper, upper, idesc, 1);
            }
            if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&seq[it & 1])) : "memory");
            __syncwarp();
            for (int k = 0; k < a.commits; ++k) umma_commit_elect(smem_u32(&bar[(it & 3) * 2 + (k & 1)]));
        }
        const long long t1 = clock64();
        umma_commit_elect(smem_u32(&bar[8]));     // count 2 in this mode
        while (!mbar_try_wait(smem_u32(&bar[8]), 0)) {}
        const long long t2 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) { a.cycles[0] = t1 - t0; a.cycles[1] = t2 - t0; }
    } else if ((warp == 0 || warp == 1) && a.waiter == 5) {
        // two INDEPENDENT issuer warps: each owns an accumulator pair and its own barriers, no hand-over
        const uint32_t a_lo = ((smem_u32(smem) & 0x3ffffu) >> 4) | ((128u >> 4) << 16);
        const uint32_t b_lo = ((smem_u32(smem + 32768) & 0x3ffffu) >> 4) | ((128u >> 4) << 16);
        const uint32_t upper = (256u >> 4) | (1u << 14);
        const uint32_t acc = tmem + 256u * (uint32_t)warp;
        const long long t0 = clock64();
        for (int it = warp; it < a.iters; it += 2) {
            for (int m = 0; m < a.mmas; ++m) {
                const uint32_t w = a_lo + 32u * (uint32_t)(m & 7);
                umma_f16_triple_ss(acc, acc + 128, w, w + 1024, b_lo + 16u * (uint32_t)(m & 3), b_lo + 512, upper, upper, idesc, 1);
            }
            for (int k = 0; k < a.commits; ++k) umma_commit_elect(smem_u32(&bar[(it & 3) * 2 + (k & 1)]));
        }
        const long long t1 = clock64();
        umma_commit_elect(smem_u32(&bar[8]));     // count 2 in this mode
        while (!mbar_try_wait(smem_u32(&bar[8]), 0)) {}
        const long long t2 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) { a.cycles[0] = t1 - t0; a.cycles[1] = t2 - t0; }
    } else if (threadIdx.x == 9999) {
        const uint32_t total = (uint32_t)a.iters * a.commits;
        for (uint32_t c = 0; c < total; ++c)
            while (!mbar_try_wait(smem_u32(&bar[c & 7]), (c >> 3) & 1)) {}
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

int main() {
    long long *d_cyc;
    CK(cudaMalloc(&d_cyc, 16));
    CK(cudaFuncSetAttribute(commit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    const int cfg[][3] = {{0, 1, 0}, {0, 1, 1}, {6, 0, 0}, {6, 1, 0}, {6, 1, 1}, {12, 1, 0}, {24, 1, 0}, {48, 1, 0},
                          {3, 1, 0}, {6, 2, 0}, {6, 3, 0}, {1, 1, 0}};
    for (auto &c : cfg) {
        Args a{1000, c[0], c[1], c[2], d_cyc};
        for (int rep = 0; rep < 2; ++rep) {
            commit_kernel<<<1, 128, 64 * 1024>>>(a);
            CK(cudaDeviceSynchronize());
        }
        long long h[2];
        CK(cudaMemcpy(h, d_cyc, 16, cudaMemcpyDeviceToHost));
        printf("group = %2d MMAs (128x128x16, 64 cyc each) + %d commits, waiter %d: issue %.1f cyc/group, complete %.1f cyc/group (MMA floor %d)\n",
               c[0], c[1], c[2], h[0] / 1000.0, h[1] / 1000.0, c[0] * 64);
    }
    // kernel-style: k-steps of 3 MMAs (192 cycles of tensor pipe each)
    const int cfg2[][3] = {{0, 1, 2}, {1, 0, 2}, {2, 0, 2}, {4, 0, 2}, {1, 1, 2}, {2, 1, 2}, {4, 1, 2}, {8, 1, 2}, {16, 1, 2},
                           {2, 1, 3}, {4, 1, 3}, {4, 0, 3}, {2, 2, 2}, {4, 3, 2},
                           {1, 1, 4}, {2, 1, 4}, {4, 1, 4}, {2, 0, 4}, {2, 2, 4},
                           {2, 0, 5}, {2, 1, 5}, {4, 1, 5}, {4, 0, 5}, {8, 1, 5}};
    for (auto &c : cfg2) {
        Args a{1000, c[0], c[1], c[2], d_cyc};
        for (int rep = 0; rep < 2; ++rep) {
            commit_kernel<<<1, 128, 64 * 1024>>>(a);
            CK(cudaDeviceSynchronize());
        }
        long long h[2];
        CK(cudaMemcpy(h, d_cyc, 16, cudaMemcpyDeviceToHost));
        printf("warp issue (%s): %2d k-steps (3 MMAs each) + %d commits: issue %.1f cyc/group, complete %.1f cyc/group (MMA floor %d)\n",
               c[2] == 2 ? "rolled" : c[2] == 4 ? "two issuers" : c[2] == 5 ? "two independent issuers" : "unrolled", c[0], c[1], h[0] / 1000.0, h[1] / 1000.0, c[0] * 192);
    }
    return 0;
}
