// Micro-benchmark + layout check for tcgen05.mma with BOTH operands in shared memory (SS form),
// the building block of the round-2 scale-space passes (csrc/scale_space_umma.cu):
//
//   P1 (convolve along the strided axis):   A = Toeplitz, K-major, no swizzle (128 x 16 fp16)
//                                           B = data rows, MN-major, SWIZZLE_128B (TMA box [k][64 n])
//   P2 (convolve along the contiguous axis): A = data, K-major, SWIZZLE_128B (TMA box [128 m][64 k])
//                                           B = Toeplitz, K-major, no swizzle (N x 16 fp16)
//
// 1. correctness: the operand layouts / descriptors above against a host GEMM (manual fill and
//    TMA fill), 2. issue + execution cost of back-to-back MMAs for several N, 1 and 148 CTAs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ubench_umma_ss tools/ubench_umma_ss.cu
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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
        if (clock64() - t0 > 4000000000ll) { printf("timeout\n"); __trap(); }
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1, uint32_t bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, uint32_t bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
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
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// smem descriptor: start>>4 | LBO>>4 << 16 | SBO>>4 << 32 | version 1 << 46 | layout << 61
__host__ __device__ inline uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
// kind::f16, F16 operands, F32 accumulate
__host__ __device__ inline uint32_t make_idesc(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

struct Args {
    const unsigned char *g_a, *g_b;     // prefilled operand images (bytes as they must sit in smem)
    uint32_t a_bytes, b_bytes;
    uint32_t a_off, b_off;              // smem offsets of the operands (from the 1024-aligned base)
    uint32_t a_lbo, a_sbo, a_layout, b_lbo, b_sbo, b_layout;
    uint32_t a_kstep, b_kstep;          // descriptor start advance per k-step (bytes)
    int ksteps;                         // correctness: k-steps accumulated
    uint32_t idesc;
    int N;
    float *out;                         // [128][N]
    int use_tma;                        // 1: P1 (B by TMA 3-D map), 2: P2 (A by TMA 2-D map)
    // throughput
    int iters, mode, ring, nacc;        // mode 0 SS, 1 TS
    uint32_t a_ring_stride, b_ring_stride;
    long long *cycles;
};

extern __shared__ __align__(1024) unsigned char smem[];

__global__ void __launch_bounds__(128, 1) check_kernel(const Args a, const __grid_constant__ CUtensorMap tmap) {
    __shared__ __align__(8) unsigned long long bar[2];
    __shared__ uint32_t tmem_slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *base = smem;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar[0]), 1);
        mbar_init(smem_u32(&bar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)), "r"(512u) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // manual fill (generic proxy), then make it visible to the async proxy
    if (a.use_tma != 2) for (uint32_t i = threadIdx.x; i < a.a_bytes; i += blockDim.x) base[a.a_off + i] = a.g_a[i];
    if (a.use_tma != 1) for (uint32_t i = threadIdx.x; i < a.b_bytes; i += blockDim.x) base[a.b_off + i] = a.g_b[i];
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        if (a.use_tma == 1) {          // B: [K rows][N] fp16 global, 3-D map {64, K, N/64}, box {64, 16*ksteps, N/64}
            mbar_expect_tx(smem_u32(&bar[1]), (uint32_t)(a.ksteps * 16 * a.N * 2));
            tma_load_3d(smem_u32(base + a.b_off), &tmap, 0, 0, 0, smem_u32(&bar[1]));
            mbar_wait(smem_u32(&bar[1]), 0);
        } else if (a.use_tma == 2) {   // A: [128 rows][64 k] fp16 global, box {64, 128}
            mbar_expect_tx(smem_u32(&bar[1]), 128u * 128u);
            tma_load_2d(smem_u32(base + a.a_off), &tmap, 0, 0, smem_u32(&bar[1]));
            mbar_wait(smem_u32(&bar[1]), 0);
        }
        tc_fence_after();
        for (int k = 0; k < a.ksteps; ++k) {
            const uint64_t ad = make_desc(smem_u32(base + a.a_off) + k * a.a_kstep, a.a_lbo, a.a_sbo, a.a_layout);
            const uint64_t bd = make_desc(smem_u32(base + a.b_off) + k * a.b_kstep, a.b_lbo, a.b_sbo, a.b_layout);
            umma_ss(tmem, ad, bd, a.idesc, k > 0);
        }
        umma_commit(smem_u32(&bar[0]));
    }
    mbar_wait(smem_u32(&bar[0]), 0);
    tc_fence_after();
    const int m = 32 * warp + lane;
    for (int c = 0; c < a.N; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + c, r);
        for (int j = 0; j < 32; ++j) a.out[m * a.N + c + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

// Throughput: one thread issues `iters` k-steps of 3 MMAs (hi*hi -> acc0, hi*lo and lo*hi -> acc1),
// operands cycling over a ring of stages; cycles from the first issue to the last completion.
__global__ void __launch_bounds__(128, 1) rate_kernel(const Args a) {
    __shared__ __align__(8) unsigned long long bar[1];
    __shared__ uint32_t tmem_slot;
    const int warp = threadIdx.x >> 5;
    unsigned char *base = smem;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar[0]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)), "r"(512u) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (uint32_t i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(base)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x03ff03ffu);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        const uint32_t a0 = smem_u32(base + a.a_off), b0 = smem_u32(base + a.b_off);
        const uint64_t ad0 = make_desc(a0, a.a_lbo, a.a_sbo, a.a_layout);
        const uint64_t bd0 = make_desc(b0, a.b_lbo, a.b_sbo, a.b_layout);
        const uint32_t acc_main = tmem, acc_small = tmem + (a.nacc > 1 ? 256 : 0);
        const long long t0 = clock64();
        int s = 0;
#pragma unroll 4
        for (int it = 0; it < a.iters; ++it) {
            const uint64_t ad = ad0 + (uint64_t)((s * a.a_ring_stride) >> 4);
            const uint64_t bd = bd0 + (uint64_t)((s * a.b_ring_stride) >> 4);
            const uint64_t ad2 = ad + (uint64_t)(a.a_kstep >> 4), bd2 = bd + (uint64_t)(a.b_kstep >> 4);
            if (a.mode == 0) {
                umma_ss(acc_main, ad, bd, a.idesc, 1);
                umma_ss(acc_small, ad, bd2, a.idesc, 1);
                umma_ss(acc_small, ad2, bd, a.idesc, 1);
            } else {
                const uint32_t at = tmem + 480 + (s & 1) * 16;
                umma_ts(acc_main, at, bd, a.idesc, 1);
                umma_ts(acc_small, at, bd2, a.idesc, 1);
                umma_ts(acc_small, at + 8, bd, a.idesc, 1);
            }
            s = s + 1 == a.ring ? 0 : s + 1;
        }
        const long long t1 = clock64();
        umma_commit(smem_u32(&bar[0]));
        mbar_wait(smem_u32(&bar[0]), 0);
        const long long t2 = clock64();
        if (blockIdx.x == 0) { a.cycles[0] = t1 - t0; a.cycles[1] = t2 - t0; }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encoder() {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    return reinterpret_cast<EncodeTiledFn>(p);
}

static float frand() { return (float)((rand() % 17) - 8) / 4.0f; }   // exactly representable in fp16

// ---- layouts (byte offsets inside the operand image) -------------------------------
static size_t off_kmajor_nosw(int row, int k) {      // 8-row groups of 256 B = [k half 0][k half 1]
    return (size_t)(row >> 3) * 256 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2;
}
static size_t off_mn_sw128(int n, int k, size_t lbo, size_t sbo) {     // B operand, N contiguous
    const int nb = n >> 6, ni = n & 63, chunk = ni >> 3, within = ni & 7, kr = k & 7;
    return (size_t)nb * lbo + (size_t)(k >> 3) * sbo + (size_t)kr * 128 + (size_t)((chunk ^ kr) * 16) + within * 2;
}
static size_t off_k_sw128(int row, int k) {           // A operand, K contiguous, 64-k atom
    const int chunk = k >> 3, within = k & 7, rr = row & 7;
    return (size_t)(row >> 3) * 1024 + (size_t)rr * 128 + (size_t)((chunk ^ rr) * 16) + within * 2;
}

static int run_check(const char *name, int which, int N, int ksteps, int use_tma) {
    const int M = 128, K = 16 * ksteps;
    std::vector<float> A((size_t)M * K), B((size_t)K * N);
    for (auto &v : A) v = frand();
    for (auto &v : B) v = frand();
    Args a{};
    std::vector<unsigned char> ia, ib;
    std::vector<__half> gsrc;          // TMA source
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof(tmap));
    void *d_src = nullptr;
    if (which == 1) {
        // A Toeplitz-like: K-major no swizzle, one 128 x 16 block per k-step (4 KB apart)
        ia.assign((size_t)ksteps * 4096, 0);
        for (int ks = 0; ks < ksteps; ++ks)
            for (int m = 0; m < M; ++m)
                for (int k = 0; k < 16; ++k)
                    *reinterpret_cast<__half *>(&ia[(size_t)ks * 4096 + off_kmajor_nosw(m, k)]) = __float2half(A[(size_t)m * K + ks * 16 + k]);
        a.a_lbo = 128; a.a_sbo = 256; a.a_layout = 0; a.a_kstep = 4096;
        // B data: MN-major SW128, rows k (128 B each), N blocks of 64 at lbo
        const size_t sbo = 1024, lbo = (size_t)K * 128;
        ib.assign((size_t)(N / 64) * lbo, 0);
        for (int k = 0; k < K; ++k)
            for (int n = 0; n < N; ++n)
                *reinterpret_cast<__half *>(&ib[off_mn_sw128(n, k, lbo, sbo)]) = __float2half(B[(size_t)k * N + n]);
        a.b_lbo = (uint32_t)lbo; a.b_sbo = (uint32_t)sbo; a.b_layout = 2; a.b_kstep = 2048;
        a.idesc = make_idesc(128, N, 0, 1);
        if (use_tma) {
            gsrc.resize((size_t)K * N);
            for (size_t i = 0; i < gsrc.size(); ++i) gsrc[i] = __float2half(B[i]);
            CK(cudaMalloc(&d_src, gsrc.size() * 2));
            CK(cudaMemcpy(d_src, gsrc.data(), gsrc.size() * 2, cudaMemcpyHostToDevice));
            const cuuint64_t dims[3] = {64, (cuuint64_t)K, (cuuint64_t)(N / 64)};
            const cuuint64_t strides[2] = {(cuuint64_t)N * 2, 128};
            const cuuint32_t box[3] = {64, (cuuint32_t)K, (cuuint32_t)(N / 64)};
            const cuuint32_t es[3] = {1, 1, 1};
            CUresult r = encoder()(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, d_src, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) { printf("%s: tensor map encode failed (%d)\n", name, (int)r); return 1; }
        }
    } else {
        // A data: K-major SW128, one box [128][64 k]; ksteps <= 4
        ia.assign(16384, 0);
        for (int m = 0; m < M; ++m)
            for (int k = 0; k < K; ++k)
                *reinterpret_cast<__half *>(&ia[off_k_sw128(m, k)]) = __float2half(A[(size_t)m * K + k]);
        a.a_lbo = 16; a.a_sbo = 1024; a.a_layout = 2; a.a_kstep = 32;
        // B Toeplitz-like: K-major no swizzle, N x 16 per k-step
        const size_t blk = (size_t)N * 32;
        ib.assign((size_t)ksteps * blk, 0);
        for (int ks = 0; ks < ksteps; ++ks)
            for (int n = 0; n < N; ++n)
                for (int k = 0; k < 16; ++k)
                    *reinterpret_cast<__half *>(&ib[(size_t)ks * blk + off_kmajor_nosw(n, k)]) = __float2half(B[(size_t)(ks * 16 + k) * N + n]);
        a.b_lbo = 128; a.b_sbo = 256; a.b_layout = 0; a.b_kstep = (uint32_t)blk;
        a.idesc = make_idesc(128, N, 0, 0);
        if (use_tma) {
            gsrc.resize((size_t)M * 64, __float2half(0.f));
            for (int m = 0; m < M; ++m)
                for (int k = 0; k < K; ++k) gsrc[(size_t)m * 64 + k] = __float2half(A[(size_t)m * K + k]);
            CK(cudaMalloc(&d_src, gsrc.size() * 2));
            CK(cudaMemcpy(d_src, gsrc.data(), gsrc.size() * 2, cudaMemcpyHostToDevice));
            const cuuint64_t dims[2] = {64, (cuuint64_t)M};
            const cuuint64_t strides[1] = {128};
            const cuuint32_t box[2] = {64, 128};
            const cuuint32_t es[2] = {1, 1};
            CUresult r = encoder()(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d_src, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) { printf("%s: tensor map encode failed (%d)\n", name, (int)r); return 1; }
        }
    }
    a.a_bytes = (uint32_t)ia.size(); a.b_bytes = (uint32_t)ib.size();
    a.a_off = 0; a.b_off = (uint32_t)((ia.size() + 1023) / 1024 * 1024);
    a.ksteps = ksteps; a.N = N; a.use_tma = use_tma ? which : 0;
    unsigned char *d_a, *d_b;
    float *d_out;
    CK(cudaMalloc(&d_a, ia.size())); CK(cudaMalloc(&d_b, ib.size())); CK(cudaMalloc(&d_out, (size_t)M * N * 4));
    CK(cudaMemcpy(d_a, ia.data(), ia.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_b, ib.data(), ib.size(), cudaMemcpyHostToDevice));
    a.g_a = d_a; a.g_b = d_b; a.out = d_out;
    const size_t smem_bytes = a.b_off + ib.size() + 1024;
    CK(cudaFuncSetAttribute(check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    check_kernel<<<1, 128, smem_bytes>>>(a, tmap);
    CK(cudaDeviceSynchronize());
    std::vector<float> out((size_t)M * N);
    CK(cudaMemcpy(out.data(), d_out, out.size() * 4, cudaMemcpyDeviceToHost));
    double worst = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double ref = 0;
            for (int k = 0; k < K; ++k) ref += (double)A[(size_t)m * K + k] * B[(size_t)k * N + n];
            worst = std::max(worst, std::abs(ref - out[(size_t)m * N + n]));
        }
    printf("check %-44s N=%3d ksteps=%d tma=%d: max |err| = %g  %s\n", name, N, ksteps, use_tma, worst, worst == 0 ? "OK" : "MISMATCH");
    cudaFree(d_a); cudaFree(d_b); cudaFree(d_out); if (d_src) cudaFree(d_src);
    return worst == 0 ? 0 : 1;
}

static void run_rate(const char *name, int which, int mode, int N, int nacc, int ctas, int iters) {
    Args a{};
    a.mode = mode; a.N = N; a.nacc = nacc; a.iters = iters; a.ring = 4;
    if (which == 1) {          // P1: A Toeplitz nosw (sliding window), B data MN SW128 stages of 32 rows
        a.a_off = 0; a.a_lbo = 128; a.a_sbo = 256; a.a_layout = 0; a.a_kstep = 32 * 1024; a.a_ring_stride = 512;   // lo array 32 KB further
        a.b_off = 64 * 1024; a.b_lbo = 4096; a.b_sbo = 1024; a.b_layout = 2; a.b_kstep = (uint32_t)(N / 64) * 4096;  // lo plane behind hi
        a.b_ring_stride = 2048;
        a.idesc = make_idesc(128, N, 0, 1);
    } else {                   // P2: A data K SW128 (box 16 KB hi, lo behind), B Toeplitz nosw window
        a.a_off = 64 * 1024; a.a_lbo = 16; a.a_sbo = 1024; a.a_layout = 2; a.a_kstep = 16384; a.a_ring_stride = 32;
        a.b_off = 0; a.b_lbo = 128; a.b_sbo = 256; a.b_layout = 0; a.b_kstep = 32 * 1024; a.b_ring_stride = 512;
        a.idesc = make_idesc(128, N, 0, 0);
    }
    long long *d_cyc;
    CK(cudaMalloc(&d_cyc, 16));
    a.cycles = d_cyc;
    CK(cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int rep = 0; rep < 2; ++rep) {
        rate_kernel<<<ctas, 128, 160 * 1024>>>(a);
        CK(cudaDeviceSynchronize());
    }
    long long h[2];
    CK(cudaMemcpy(h, d_cyc, 16, cudaMemcpyDeviceToHost));
    printf("rate  %-34s %s N=%3d acc=%d ctas=%3d: issue %.1f cyc/MMA, complete %.1f cyc/MMA (floor %d)\n", name,
           mode ? "TS" : "SS", N, nacc, ctas, (double)h[0] / (3.0 * iters), (double)h[1] / (3.0 * iters), N / 2);
    cudaFree(d_cyc);
}

int main() {
    srand(1);
    int bad = 0;
    for (int tma = 0; tma <= 1; ++tma) {
        bad += run_check("P1: A K-major nosw, B MN-major SW128", 1, 128, 2, tma);
        bad += run_check("P1: A K-major nosw, B MN-major SW128", 1, 256, 2, tma);
        bad += run_check("P1: A K-major nosw, B MN-major SW128", 1, 64, 1, tma);
        bad += run_check("P2: A K-major SW128, B K-major nosw", 2, 128, 4, tma);
        bad += run_check("P2: A K-major SW128, B K-major nosw", 2, 256, 3, tma);
        bad += run_check("P2: A K-major SW128, B K-major nosw", 2, 48, 1, tma);
    }
    for (int ctas : {1, 148}) {
        for (int N : {32, 64, 128, 256}) run_rate("P1 (Toeplitz A, data B MN-major)", 1, 0, N >= 64 ? N : 64, 2, ctas, 2000);
        for (int N : {16, 32, 64, 128, 256}) run_rate("P2 (data A K-major, Toeplitz B)", 2, 0, N, 2, ctas, 2000);
        for (int N : {16, 64, 128, 256}) run_rate("TS (A in TMEM, Toeplitz B)", 2, 1, N, N > 128 ? 1 : 2, ctas, 2000);
        run_rate("P2 one accumulator", 2, 0, 128, 1, ctas, 2000);
    }
    printf(bad ? "SOME CHECKS FAILED\n" : "all checks OK\n");
    return 0;
}
