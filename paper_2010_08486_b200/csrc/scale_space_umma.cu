// Separable Gaussian scale space + fused DoG on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Same two passes, same buffers and the same results (within float32 rounding) as
// scale_space.cu (reference: convolve.py:63-218, detector.py:117-126), but the banded
// correlation along the strided axis is issued as a Toeplitz GEMM:
//
//     D[m][n] = sum_k  X[k][m] * T[k][n],      T[k][n] = w[k - n]  (0 <= k - n <= 2 rpad)
//
//   m : 128 positions along the CONTIGUOUS axis of the input plane (one TMEM lane each)
//   n : 128 outputs along the convolved (strided) axis
//   k : the 128 + 2 rpad input rows the 128 outputs read, 8 per tcgen05.mma (kind::tf32)
//
// float32 accuracy from tf32 tensor cores: both operands are split x = hi + lo with
// hi = rna_tf32(x), lo = rna_tf32(x - hi) (22 significant bits) and every k-step issues the three
// products hi*lo + lo*hi + hi*hi into one float32 accumulator (the lo*lo term is below 2^-22).
//
// Data flow of one CTA (persistent, one per SM, 512 threads):
//   warps 8..15 "loaders"   global rows -> registers (coalesced along m) -> hi/lo split ->
//                           tcgen05.st into the A staging columns of TMEM (A never touches
//                           shared memory; 8 stages of 2 k-steps)
//   warps 1..3  "builders"  the level's Toeplitz operand in shared memory, K-major, no swizzle.
//                           T only depends on k - n, so ONE array G[p][kk] = w[kk - p + Kp - 8]
//                           serves every k-step: step m0 reads the 128-row window that starts
//                           at row Kp - 8 - m0 (the descriptor's start address slides, nothing
//                           is copied).  Double buffered across levels.
//   warp 0      "issuer"    one thread: 3 tcgen05.mma per k-step, tcgen05.commit releases the
//                           A stage / the Toeplitz buffer / publishes the accumulator
//   warps 4..7  "drain"     tcgen05.ld of the finished accumulator (lane = m, so a warp's
//                           store of one n is 128 contiguous bytes), DoG against the previous
//                           level kept in thread-private shared-memory slots, global stores.
//                           Two accumulators: the drain of level i overlaps the MMAs of i+1.
// TMEM columns: [0,256) two 128 x 128 float32 accumulators, [256,512) A staging.
#include <cstdlib>

#include "common.cuh"

namespace dogblob {

namespace {

constexpr int kUT = 128;              // tile edge on both axes
constexpr int kUThreads = 512;
constexpr int kStages = 8;            // A staging stages
constexpr int kStageRows = 16;        // input rows per stage = 2 k-steps of 8
constexpr int kStageCols = 32;        // TMEM columns per stage: (hi 8 + lo 8) per k-step
constexpr int kAccCols = 128;
constexpr int kStageCol0 = 2 * kAccCols;
constexpr int kLoaderGroups = 2;      // groups of 4 warps; group g fills stages with index % 2 == g
constexpr int kBuilderWarps = 3;
constexpr uint32_t kSpinLimit = 1u << 27;

enum UmmaMode { kModeRows = 0, kModeDog = 1, kModeLevels = 2 };

struct UmmaArgs {
    const float *in;        // rows: the image; columns: the row-filtered planes
    int64_t in_pitch;       // elements between rows of `in`
    int64_t in_plane;       // elements between level planes of `in` (0: every level reads plane 0)
    int n_rows;             // valid rows of `in` along the convolved axis (reflect period)
    float *out;
    int64_t out_pitch, out_plane;
    float *edge;            // DoG mode: parked boundary levels
    const float2 *taps;     // duplicated (w, w) tap tables, see api.cu
    int tiles_c, tiles_r;   // tiles along the contiguous / the convolved axis
    int n_units;            // tiles_c * tiles_r * n_groups
    int toep_floats;        // floats of one Toeplitz array (hi or lo) of the widest level
    unsigned long long *prof;   // DOGBLOB_UMMA_PROF: per-role cycle counters (see launch_umma)
    int debug;              // DOGBLOB_UMMA_DEBUG: 1 loaders skip global loads, 2 builders build once,
                            // 4 drain skips stores, 8 issuer skips the MMAs (timing experiments only)
};

// ---- PTX wrappers -------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}
// A deadlock here would hang the GPU; trap instead (the launch then reports an error).
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, int tag) {
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++spins > kSpinLimit) {
            if ((threadIdx.x & 31) == 0)
                printf("umma: barrier timeout tag=%d block=%d warp=%d parity=%u\n", tag, blockIdx.x,
                       threadIdx.x >> 5, parity);
            __trap();
        }
    }
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t slot_smem, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot_smem),
                 "r"(cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
                 : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem descriptor], kind::tf32, M = 128
__device__ __forceinline__ void umma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t u;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
    return u;
}
__device__ __forceinline__ void split_tf32(float x, uint32_t &hi, uint32_t &lo) {
    hi = tf32_rna(x);
    lo = tf32_rna(__fsub_rn(x, __uint_as_float(hi)));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
          "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),
          "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
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
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor (cute::UMMA::SmemDescriptor): K-major, no swizzle.
//   bits [0,14)  start address >> 4        bits [16,30) leading byte offset >> 4 (between the
//   bits [32,46) stride byte offset >> 4                two 16-byte K halves of a k-step)
//   bits [46,48) version = 1 (Blackwell)   bits [61,64) layout type = 0 (SWIZZLE_NONE)
// Toeplitz array: 8-row group g at g * 256 bytes: [K half 0: 8 rows x 16 B][K half 1: 8 rows x 16 B]
constexpr uint32_t kToepGroupBytes = 256, kToepHalfBytes = 128;
__device__ __forceinline__ uint64_t toeplitz_desc(uint32_t smem_addr) {
    return (uint64_t)((smem_addr >> 4) & 0x3FFFu) | ((uint64_t)(kToepHalfBytes >> 4) << 16) |
           ((uint64_t)(kToepGroupBytes >> 4) << 32) | (1ull << 46);
}
// Instruction descriptor (cute::UMMA::InstrDescriptor): D = F32, A = B = TF32, both K-major,
// dense, N at bits [17,23) as N >> 3, M at bits [24,29) as M >> 4.
__host__ __device__ constexpr uint32_t instr_desc(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ int fold_row_u(int i, int n) {
    if ((unsigned)i < (unsigned)n) return i;
    const int period = 2 * n;
    int t = i % period;
    if (t < 0) t += period;
    return t < n ? t : period - 1 - t;
}

// Optional per-role cycle accounting (prof != nullptr): lane 0 of one warp per role accumulates
// clock64 deltas per category and adds them to prof[] when the CTA ends.
struct RoleClock {
    unsigned long long acc[4] = {0, 0, 0, 0};
    long long t = 0;
    bool on;
    __device__ __forceinline__ explicit RoleClock(bool enabled) : on(enabled) { if (on) t = clock64(); }
    __device__ __forceinline__ void lap(int cat) {
        if (on) { const long long n = clock64(); acc[cat] += (unsigned long long)(n - t); t = n; }
    }
    __device__ __forceinline__ void flush(unsigned long long *prof, int base) {
        if (on)
            for (int i = 0; i < 4; ++i) atomicAdd(prof + base + i, acc[i]);
    }
};

struct Unit { int g, r0, c0; };
__device__ __forceinline__ Unit decode_unit(int u, const UmmaArgs &a) {
    Unit x;
    x.c0 = (u % a.tiles_c) * kUT;
    const int t = u / a.tiles_c;
    x.r0 = (t % a.tiles_r) * kUT;
    x.g = t / a.tiles_r;
    return x;
}

struct SharedCtl {
    unsigned long long data_full[kStages], data_empty[kStages];
    unsigned long long toep_full[2], toep_empty[2];
    unsigned long long acc_full[2], acc_empty[2];
    uint32_t tmem_base;
    uint32_t pad[3];
};

template <int MODE>
__global__ void __launch_bounds__(kUThreads, 1)
umma_pass_kernel(const UmmaArgs a, const __grid_constant__ LevelTable tbl) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    SharedCtl *ctl = reinterpret_cast<SharedCtl *>(smem_raw);
    float *toep = reinterpret_cast<float *>(smem_raw + 1024);     // [buffer 2][hi, lo][toep_floats]
    float *s_prev = toep + 4 * (size_t)a.toep_floats;              // DoG: [n 128][m 128]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(smem_u32(&ctl->data_full[s]), 4);
            mbar_init(smem_u32(&ctl->data_empty[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&ctl->toep_full[b]), kBuilderWarps);
            mbar_init(smem_u32(&ctl->toep_empty[b]), 1);
            mbar_init(smem_u32(&ctl->acc_full[b]), 1);
            mbar_init(smem_u32(&ctl->acc_empty[b]), 4);
        }
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(smem_u32(&ctl->tmem_base), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(&ctl->tmem_base);

    if (warp == 0) {
        // ================= issuer =================
        uint32_t stage_it = 0, lvl_it = 0;
        constexpr uint32_t idesc = instr_desc(kUT, kUT);
        RoleClock rc(a.prof != nullptr && lane == 0);
        for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
            const Unit un = decode_unit(u, a);
            const int lb = tbl.group_begin[un.g], le = tbl.group_begin[un.g + 1];
            for (int level = lb; level < le; ++level, ++lvl_it) {
                const int Kp = kUT + 2 * tbl.lv[level].rpad;
                const int n_stage = Kp / kStageRows;
                const uint32_t b = lvl_it & 1, par = (lvl_it >> 1) & 1;
                rc.lap(3);
                mbar_wait(smem_u32(&ctl->toep_full[b]), par, 1);
                rc.lap(0);
                mbar_wait(smem_u32(&ctl->acc_empty[b]), par ^ 1, 2);
                rc.lap(1);
                tc_fence_after();
                const uint32_t t_hi = smem_u32(toep + (size_t)(2 * b) * a.toep_floats);
                const uint32_t t_lo = smem_u32(toep + (size_t)(2 * b + 1) * a.toep_floats);
                const uint32_t acc = tmem + b * kAccCols;
                for (int st = 0; st < n_stage; ++st, ++stage_it) {
                    const uint32_t s = stage_it % kStages, sp = (stage_it / kStages) & 1;
                    rc.lap(3);
                    mbar_wait(smem_u32(&ctl->data_full[s]), sp, 3);
                    rc.lap(2);
                    tc_fence_after();
                    if (lane == 0) {
#pragma unroll
                        for (int ks = 0; ks < 2; ++ks) {
                            if (a.debug & 8) break;
                            if (a.debug & 48) {     // timing experiments: independent chains / fewer MMAs
                                const int m0x = st * kStageRows + ks * 8;
                                const uint32_t winx = (uint32_t)((Kp - 8 - m0x) >> 3) * kToepGroupBytes;
                                const uint32_t ax = tmem + kStageCol0 + s * kStageCols + ks * 16;
                                const uint32_t other = tmem + (b ^ 1) * kAccCols;
                                if (a.debug & 16) {
                                    umma_tf32_ts(other, ax, toeplitz_desc(t_lo + winx), idesc, 1);
                                    umma_tf32_ts(acc, ax, toeplitz_desc(t_hi + winx), idesc, (st | ks) != 0);
                                    umma_tf32_ts(other, ax + 8, toeplitz_desc(t_hi + winx), idesc, 1);
                                } else {
                                    umma_tf32_ts(acc, ax, toeplitz_desc(t_hi + winx), idesc, (st | ks) != 0);
                                }
                                continue;
                            }
                            const int m0 = st * kStageRows + ks * 8;
                            const uint32_t win = (uint32_t)((Kp - 8 - m0) >> 3) * kToepGroupBytes;
                            const uint64_t d_hi = toeplitz_desc(t_hi + win);
                            const uint64_t d_lo = toeplitz_desc(t_lo + win);
                            const uint32_t a_hi = tmem + kStageCol0 + s * kStageCols + ks * 16;
                            const uint32_t a_lo = a_hi + 8;
                            umma_tf32_ts(acc, a_hi, d_lo, idesc, (st | ks) != 0);
                            umma_tf32_ts(acc, a_lo, d_hi, idesc, 1);
                            umma_tf32_ts(acc, a_hi, d_hi, idesc, 1);
                        }
                        umma_commit(smem_u32(&ctl->data_empty[s]));
                    }
                    __syncwarp();
                }
                if (lane == 0) {
                    umma_commit(smem_u32(&ctl->toep_empty[b]));
                    umma_commit(smem_u32(&ctl->acc_full[b]));
                }
                __syncwarp();
            }
        }
        rc.lap(3);
        rc.flush(a.prof, 0);
    } else if (warp <= kBuilderWarps) {
        // ================= Toeplitz builders =================
        const int tid = threadIdx.x - 32;
        uint32_t lvl_it = 0;
        RoleClock rc(a.prof != nullptr && tid == 0);
        for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
            const Unit un = decode_unit(u, a);
            const int lb = tbl.group_begin[un.g], le = tbl.group_begin[un.g + 1];
            for (int level = lb; level < le; ++level, ++lvl_it) {
                const LevelDesc lv = tbl.lv[level];
                const int Kp = kUT + 2 * lv.rpad;
                const uint32_t b = lvl_it & 1, par = (lvl_it >> 1) & 1;
                rc.lap(1);
                mbar_wait(smem_u32(&ctl->toep_empty[b]), par ^ 1, 4);
                rc.lap(0);
                float *g_hi = toep + (size_t)(2 * b) * a.toep_floats;
                float *g_lo = g_hi + a.toep_floats;
                const float2 *w = a.taps + lv.tap_ofs;
                int n4 = (Kp - 8 + kUT) * 2;            // 16-byte pieces: rows x 2 K halves
                if ((a.debug & 2) && lvl_it >= 2) n4 = 0;
                for (int i = tid; i < n4; i += 32 * kBuilderWarps) {
                    const int p = i >> 1, half = i & 1;
                    // G[p][kk] = w[kk - (p - (Kp - 8))], kk = 4 half .. 4 half + 3
                    const int t0 = 4 * half - p + (Kp - 8);
                    uint32_t hi[4], lo[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int t = t0 + e;
                        const float v = (t >= 0 && t <= 2 * lv.rpad) ? __ldg(&w[t].x) : 0.f;
                        split_tf32(v, hi[e], lo[e]);
                    }
                    const int ofs = (p >> 3) * 64 + half * 32 + (p & 7) * 4;     // floats
                    *reinterpret_cast<uint4 *>(g_hi + ofs) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                    *reinterpret_cast<uint4 *>(g_lo + ofs) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&ctl->toep_full[b]));
            }
        }
        rc.lap(1);
        rc.flush(a.prof, 4);
    } else if (warp < 8) {
        // ================= drain (accumulator -> DoG -> global) =================
        const int q = warp & 3;
        const int m = 32 * q + lane;
        uint32_t lvl_it = 0;
        RoleClock rc(a.prof != nullptr && warp == 4 && lane == 0);
        for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
            const Unit un = decode_unit(u, a);
            const int lb = tbl.group_begin[un.g], le = tbl.group_begin[un.g + 1];
            for (int level = lb; level < le; ++level, ++lvl_it) {
                const uint32_t b = lvl_it & 1, par = (lvl_it >> 1) & 1;
                rc.lap(1);
                mbar_wait(smem_u32(&ctl->acc_full[b]), par, 5);
                rc.lap(0);
                tc_fence_after();
                const uint32_t acc = tmem + b * kAccCols + ((uint32_t)(32 * q) << 16);
                const bool park_first = MODE == kModeDog && level == lb && un.g > 0;
                const bool park_last = MODE == kModeDog && level == le - 1 && un.g < tbl.n_groups - 1;
                const float sig = MODE == kModeDog && level > lb ? tbl.lv[level - 1].sigma_f32 : 0.f;
#pragma unroll 1
                for (int c = 0; c < kUT / 32; ++c) {
                    uint32_t r[32];
                    tmem_ld32(acc + c * 32, r);
                    tmem_wait_ld();
                    if (a.debug & 4) continue;
                    if (MODE == kModeRows) {
                        // lane = x (contiguous input axis), registers = 32 consecutive y of T[x][y]
                        float *dst = a.out + (int64_t)level * a.out_plane +
                                     (int64_t)(un.c0 + m) * a.out_pitch + un.r0 + c * 32;
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            *reinterpret_cast<uint4 *>(dst + j) = make_uint4(r[j], r[j + 1], r[j + 2], r[j + 3]);
                    } else {
                        // lane = y (contiguous), registers = 32 consecutive output rows x
                        const int64_t tile_ofs = (int64_t)(un.r0 + c * 32) * a.out_pitch + un.c0 + m;
                        if (MODE == kModeLevels) {
                            float *dst = a.out + (int64_t)level * a.out_plane + tile_ofs;
#pragma unroll
                            for (int j = 0; j < 32; ++j) dst[(int64_t)j * a.out_pitch] = __uint_as_float(r[j]);
                        } else {
                            if (park_first || park_last) {
                                float *dst = a.edge + (int64_t)(2 * un.g + (park_first ? 0 : 1)) * a.out_plane + tile_ofs;
#pragma unroll
                                for (int j = 0; j < 32; ++j) dst[(int64_t)j * a.out_pitch] = __uint_as_float(r[j]);
                                if (park_first && park_last) {      // single-level group
                                    dst = a.edge + (int64_t)(2 * un.g + 1) * a.out_plane + tile_ofs;
#pragma unroll
                                    for (int j = 0; j < 32; ++j) dst[(int64_t)j * a.out_pitch] = __uint_as_float(r[j]);
                                }
                            }
                            float *slot = s_prev + (c * 32) * kUT + m;
                            if (level > lb) {
                                float *dst = a.out + (int64_t)(level - 1) * a.out_plane + tile_ofs;
#pragma unroll
                                for (int j = 0; j < 32; ++j) {
                                    const float prev = slot[j * kUT];
                                    dst[(int64_t)j * a.out_pitch] =
                                        __fmul_rn(__fsub_rn(prev, __uint_as_float(r[j])), sig);
                                }
                            }
                            if (level < le - 1) {
#pragma unroll
                                for (int j = 0; j < 32; ++j) slot[j * kUT] = __uint_as_float(r[j]);
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&ctl->acc_empty[b]));
            }
        }
        rc.lap(1);
        rc.flush(a.prof, 8);
    } else {
        // ================= loaders (global -> hi/lo -> TMEM A staging) =================
        const int q = warp & 3;
        const int grp = (warp - 8) >> 2;
        const int m = 32 * q + lane;
        uint32_t stage_it = 0;
        RoleClock rc(a.prof != nullptr && warp == 8 && lane == 0);
        for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
            const Unit un = decode_unit(u, a);
            const int lb = tbl.group_begin[un.g], le = tbl.group_begin[un.g + 1];
            for (int level = lb; level < le; ++level) {
                const int rpad = tbl.lv[level].rpad;
                const int n_stage = (kUT + 2 * rpad) / kStageRows;
                const float *src = a.in + (int64_t)level * a.in_plane + un.c0 + m;
                const int row_base = un.r0 - rpad;
                for (int st = 0; st < n_stage; ++st, ++stage_it) {
                    if ((int)(stage_it % kLoaderGroups) != grp) continue;
                    const uint32_t s = stage_it % kStages, sp = (stage_it / kStages) & 1;
                    float v[kStageRows];
#pragma unroll
                    for (int k = 0; k < kStageRows; ++k)
                        v[k] = (a.debug & 1) ? 1.f : __ldg(src + (int64_t)fold_row_u(row_base + st * kStageRows + k, a.n_rows) * a.in_pitch);
                    rc.lap(3);
                    mbar_wait(smem_u32(&ctl->data_empty[s]), sp ^ 1, 6);
                    rc.lap(0);
                    tc_fence_after();
                    const uint32_t dst = tmem + kStageCol0 + s * kStageCols + ((uint32_t)(32 * q) << 16);
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks) {
                        uint32_t r[16];
#pragma unroll
                        for (int k = 0; k < 8; ++k) split_tf32(v[ks * 8 + k], r[k], r[8 + k]);
                        tmem_st16(dst + ks * 16, r);
                    }
                    rc.lap(1);
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(&ctl->data_full[s]));
                    rc.lap(2);
                }
            }
        }
        rc.lap(3);
        rc.flush(a.prof, 12);
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int toeplitz_floats(int max_rpad) { return (kUT + 2 * max_rpad - 8 + kUT) * 8; }

size_t umma_smem(int max_rpad, bool dog) {
    return 1024 + 4 * (size_t)toeplitz_floats(max_rpad) * sizeof(float) +
           (dog ? (size_t)kUT * kUT * sizeof(float) : 0);
}

int persistent_ctas(int n_units) {
    static const int sms = [] {
        int dev = 0, n = 148;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (const char *e = std::getenv("DOGBLOB_UMMA_CTAS")) n = std::max(1, std::atoi(e));
        return n;
    }();
    return std::min(n_units, sms);
}

template <int MODE>
cudaError_t launch_umma(const UmmaArgs &a, const LevelTable &tbl, int max_rpad, cudaStream_t st) {
    const size_t smem = umma_smem(max_rpad, MODE == kModeDog);
    UmmaArgs b = a;
    if (const char *e = std::getenv("DOGBLOB_UMMA_DEBUG")) b.debug = std::atoi(e);
    static unsigned long long *d_prof = nullptr;
    const bool prof = std::getenv("DOGBLOB_UMMA_PROF") != nullptr;
    if (prof) {
        if (!d_prof) cudaMalloc(&d_prof, 16 * sizeof(unsigned long long));
        cudaMemsetAsync(d_prof, 0, 16 * sizeof(unsigned long long), st);
        b.prof = d_prof;
    }
    const int ctas = persistent_ctas(b.n_units);
    umma_pass_kernel<MODE><<<ctas, kUThreads, smem, st>>>(b, tbl);
    if (prof) {
        unsigned long long h[16];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, d_prof, sizeof(h), cudaMemcpyDeviceToHost);
        static const char *names[16] = {
            "issuer  wait toeplitz", "issuer  wait acc free", "issuer  wait data", "issuer  issue+other",
            "builder wait buffer", "builder build", "-", "-",
            "drain   wait acc", "drain   ld+store", "-", "-",
            "loader  wait stage free", "loader  split+st (load latency)", "loader  wait::st+arrive", "loader  loads issue+other"};
        fprintf(stderr, "umma mode %d, %d CTAs, kilo-cycles per CTA:", MODE, ctas);
        for (int i = 0; i < 16; ++i)
            if (names[i][0] != '-') fprintf(stderr, "\n   %-34s %8.1f", names[i], h[i] / 1e3 / ctas);
        fprintf(stderr, "\n");
    }
    return cudaGetLastError();
}

}  // namespace

bool umma_supported(const ConvGeometry &g) {
    return umma_smem(g.max_rpad, true) <= 227 * 1024;
}

cudaError_t configure_umma_kernels(int device) {
    int optin = 0;
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(umma_pass_kernel<kModeRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(umma_pass_kernel<kModeDog>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(umma_pass_kernel<kModeLevels>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
}

// img[y][x] -> T_i[x][y]: contiguous axis x, convolved axis y, stored transposed
cudaError_t launch_row_pass_umma(const ConvGeometry &g, const float *d_img, float *d_rows_t,
                                 const LevelTable &tbl, const float2 *d_taps, cudaStream_t st) {
    UmmaArgs a{};
    a.in = d_img; a.in_pitch = g.Wp; a.in_plane = 0; a.n_rows = g.H;
    a.out = d_rows_t; a.out_pitch = g.Hp; a.out_plane = (int64_t)g.Hp * g.Wp;
    a.edge = nullptr; a.taps = d_taps;
    a.tiles_c = g.Wp / kUT; a.tiles_r = g.Hp / kUT;
    a.n_units = a.tiles_c * a.tiles_r * tbl.n_groups;
    a.toep_floats = toeplitz_floats(g.max_rpad);
    return launch_umma<kModeRows>(a, tbl, g.max_rpad, st);
}

// T_i[x][y] -> D_i^T[x][y]: contiguous axis y, convolved axis x
cudaError_t launch_col_dog_pass_umma(const ConvGeometry &g, const float *d_rows_t, float *d_dog_t,
                                     float *d_edge, const LevelTable &tbl, const float2 *d_taps,
                                     cudaStream_t st) {
    UmmaArgs a{};
    a.in = d_rows_t; a.in_pitch = g.Hp; a.in_plane = (int64_t)g.Hp * g.Wp; a.n_rows = g.W;
    a.out = d_dog_t; a.out_pitch = g.Hp; a.out_plane = a.in_plane;
    a.edge = d_edge; a.taps = d_taps;
    a.tiles_c = g.Hp / kUT; a.tiles_r = g.Wp / kUT;
    a.n_units = a.tiles_c * a.tiles_r * tbl.n_groups;
    a.toep_floats = toeplitz_floats(g.max_rpad);
    return launch_umma<kModeDog>(a, tbl, g.max_rpad, st);
}

cudaError_t launch_col_levels_pass_umma(const ConvGeometry &g, const float *d_rows_t, float *d_lev_t,
                                        const LevelTable &unit_tbl, const float2 *d_taps,
                                        cudaStream_t st) {
    UmmaArgs a{};
    a.in = d_rows_t; a.in_pitch = g.Hp; a.in_plane = (int64_t)g.Hp * g.Wp; a.n_rows = g.W;
    a.out = d_lev_t; a.out_pitch = g.Hp; a.out_plane = a.in_plane;
    a.edge = nullptr; a.taps = d_taps;
    a.tiles_c = g.Hp / kUT; a.tiles_r = g.Wp / kUT;
    a.n_units = a.tiles_c * a.tiles_r * unit_tbl.n_groups;
    a.toep_floats = toeplitz_floats(g.max_rpad);
    return launch_umma<kModeLevels>(a, unit_tbl, g.max_rpad, st);
}

}  // namespace dogblob
