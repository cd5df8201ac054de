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
//   k : the 128 + 2 rpad input rows the 128 outputs read, 16 per tcgen05.mma (kind::f16)
//
// float32 accuracy from fp16 tensor-core operands: both operands are split x = hi + lo with
// hi = fp16(x), lo = fp16(x - hi) (11 + 11 significand bits; exact power-of-two scales keep them in
// fp16's range, see DOGBLOB_UMMA_F16 below) and every step issues the three products hi*hi, hi*lo
// and lo*hi (the lo*lo term is below 2^-22).  The tensor core truncates its float32 accumulator
// after every MMA, so each issuing warp owns one accumulator (half the chain) and the drain adds
// them in float32.  Build option: tf32 operands (K = 8, no scales).
//
// Data flow of one CTA (persistent, one per SM, 544 threads):
//   warps 2..3  "loaders"    32 input rows x 512 B per stage into shared memory: one TMA box
//                            (interior) or 16-byte cp.async with folded rows (image border)
//   warps 8..15 "converters" read the rows back with lane = m, split hi/lo, tcgen05.st into the A
//                            staging columns of TMEM (A is an MMA operand from TMEM only)
//   warp 1      "Toeplitz"   the level's Toeplitz operand, prebuilt on the host, one bulk copy per
//                            level into shared memory (K-major, no swizzle).  T only depends on
//                            k - n, so ONE array G[p][kk] = w[kk - p + Kp - 8] serves every k-step:
//                            step m0 reads the 128-row window that starts at row Kp - 8 - m0 (the
//                            descriptor's start address slides).  Double buffered across levels.
//   warps 0, 16 "issuers"    stages alternate between the two warps; one elected lane issues
//                            3 tcgen05.mma per k-step, tcgen05.commit releases the A stage / the
//                            Toeplitz buffer / publishes the accumulator halves
//   warps 4..7  "drain"      tcgen05.ld of a finished accumulator half (lane = m, so a warp's store
//                            of one n is 128 contiguous bytes), sum of the three accumulators, DoG
//                            against the previous level kept in thread-private shared-memory
//                            slots, global stores; hands the half back zeroed
// TMEM columns: [0,384) three 128 x 128 float32 accumulators, [384,512) two A stages.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda.h>
#include <cuda_fp16.h>      // CUtensorMap (types only: the encoder is fetched through the runtime)

#include "common.cuh"

namespace dogblob {

namespace {

constexpr int kUT = 128;              // tile edge on both axes
// DOGBLOB_UMMA_F16 = 1 (default): fp16 hi/lo operands (kind::f16, K = 16 rows per MMA: half as many
// MMAs as the tf32 split, 11 + 11 significand bits all the same).  fp16's range is covered by exact
// power-of-two scales: the frame by 2^e (max |x| * 2^e in [2^12, 2^13), e from frame_max_kernel in
// front of the row pass), every level's taps by 2^t (largest tap in [512, 1024)); the drain undoes
// both.  Values far below the frame's maximum lose relative, not absolute, precision.
// DOGBLOB_UMMA_F16 = 0: tf32 hi/lo operands (K = 8), no frame scale, so the row pass can start
// under a streamed upload; 10 % slower.
#ifndef DOGBLOB_UMMA_F16
#define DOGBLOB_UMMA_F16 1
#endif
#ifndef DOGBLOB_UMMA_ISSUERS
#define DOGBLOB_UMMA_ISSUERS 2       // fp16: 0.181 + 0.184 ms at C2 (one issuer: 0.189 + 0.188)
#endif
// accumulators: one per issuing warp; a single issuer alternates between two (even / odd steps)
#define DOGBLOB_UMMA_ACCS (DOGBLOB_UMMA_ISSUERS > 1 ? DOGBLOB_UMMA_ISSUERS : 2)
constexpr int kIssuers = DOGBLOB_UMMA_ISSUERS;      // issuing warps: warp 0 and warps 16 ..
#ifndef DOGBLOB_UMMA_DRAIN_GROUPS
#define DOGBLOB_UMMA_DRAIN_GROUPS 1      // 2: column pass -3 %, row pass +6 % (672 threads cap the registers at 80)
#endif
constexpr int kDrainGroups = DOGBLOB_UMMA_DRAIN_GROUPS;   // 4 warps each; group 0 = warps 4..7, group 1 = the last 4 warps
constexpr int kDrainB = 16 + kIssuers - 1;                 // first warp of the second drain group
constexpr int kUThreads = 32 * (kDrainB + 4 * (kDrainGroups - 1));
constexpr int kIssuerB = 16;          // warp index of the second issuer
#ifndef DOGBLOB_UMMA_STAGEK
#define DOGBLOB_UMMA_STAGEK 4
#endif
constexpr int kStageK = DOGBLOB_UMMA_STAGEK;          // k-steps (8 input rows each) per stage
constexpr int kAccs = DOGBLOB_UMMA_ACCS;
constexpr int kStages = (512 - 128 * DOGBLOB_UMMA_ACCS) / (16 * kStageK);   // A staging stages (the TMEM columns the accumulators leave)
constexpr int kStageRows = 8 * kStageK;   // input rows per stage
constexpr int kStageCols = 16 * kStageK;  // TMEM columns per stage: (hi 8 + lo 8) per k-step
constexpr int kAccCols = 128;
// TMEM columns: one 128 x 128 float32 accumulator per issuing warp, then the A staging
constexpr int kStageCol0 = kAccs * kAccCols;
constexpr int kHalf = kUT / 2;        // accumulators are handed to the drain in two column halves
constexpr int kLoaderGroups = 2;      // groups of 4 warps; group g fills stages with index % 2 == g
constexpr int kMaxRawStages = 8;      // raw input-row stages in shared memory (16 KB each)
constexpr unsigned long long kWaitLimitNs = 20ull * 1000 * 1000 * 1000;   // deadlock trap (20 s)

enum UmmaMode { kModeRows = 0, kModeDog = 1, kModeLevels = 2 };

struct UmmaArgs {
    const float *in;        // rows: the image; columns: the row-filtered planes
    int64_t in_pitch;       // elements between rows of `in`
    int64_t in_plane;       // elements between level planes of `in` (0: every level reads plane 0)
    int n_rows;             // valid rows of `in` along the convolved axis (reflect period)
    float *out;
    int64_t out_pitch, out_plane;
    float *edge;            // DoG mode: parked boundary levels
    const uint32_t *frame_max_bits;   // F16 mode: float bits of the frame's max |x| (device word)
    const float *toep;      // prebuilt Toeplitz arrays of every level (hi | lo), see build_toeplitz
    int raw_stages;         // raw input-row stages that fit in shared memory
    int by_order;           // units are single levels in tbl.order[] (longest first): row pass
    int n_order;            // by_order: number of levels
    // streamed upload (row pass only, see RowGate in common.cuh): the frame arrives in row chunks
    // while the kernel runs; *gate_word - gate_base = chunks resident.  Tile rows are then the
    // slowest unit index, so early units only need early chunks.
    const int *gate_word;
    int gate_base, gate_rows_per_chunk;
    unsigned long long *gate_t_start;
    int use_tma;            // interior stages arrive as one TMA box (tensor map valid)
    int tma_plane_rows;     // rows between level planes in the tensor map (0: one plane)
    int tiles_c, tiles_r;   // tiles along the contiguous / the convolved axis
    int n_units;            // tiles_c * tiles_r * n_groups
    const int *sched;       // optional: position i of a CTA's round-robin walk -> unit (cost-balanced order)
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
// A deadlock here would hang the GPU; trap instead (the launch then reports an error).  The limit
// is wall time, not spins: under a profiler's replay a wait can legitimately be very long.
__device__ __noinline__ void mbar_timeout(int tag, uint32_t parity) {
    if ((threadIdx.x & 31) == 0)
        printf("umma: barrier timeout tag=%d block=%d warp=%d parity=%u\n", tag, blockIdx.x, threadIdx.x >> 5,
               parity);
    __trap();
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, int tag) {
    if (mbar_try_wait(bar, parity)) return;
    const unsigned long long t0 = globaltimer_ns();
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity))
        if ((++spins & 0xfffu) == 0 && globaltimer_ns() - t0 > kWaitLimitNs) mbar_timeout(tag, parity);
}
// long waits (drain, copiers): back off so that the spinning warp leaves its issue slots to
// the converters that share the SM sub-partition
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity, int tag) {
    if (mbar_try_wait(bar, parity)) return;
    const unsigned long long t0 = globaltimer_ns();
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        __nanosleep(64);
        if ((++spins & 0xfffu) == 0 && globaltimer_ns() - t0 > kWaitLimitNs) mbar_timeout(tag, parity);
    }
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
// global -> shared bulk copy (no tensor map), completion counted in bytes on `bar`
__device__ __forceinline__ void bulk_copy_g2s(uint32_t dst_smem, const void *src, uint32_t bytes,
                                              uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dst_smem), "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_only(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
// one TMA box (tensor map: rows of the input planes, 128 floats x 16 rows, no swizzle)
__device__ __forceinline__ void tma_load_2d(uint32_t dst_smem, const CUtensorMap *map, int col, int row,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(dst_smem), "l"(map), "r"(col), "r"(row), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst_smem, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_smem), "l"(src) : "memory");
}
// the barrier gets one (pre-counted) arrival once all earlier cp.async of this thread landed
__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ uint64_t make_desc(uint32_t lo, uint32_t hi) {
    uint64_t d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "r"(lo), "r"(hi));
    return d;
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
// Warp-uniform variants: the whole warp executes them, one elected lane issues.  Keeping the
// issuer's control flow and operands warp uniform lets ptxas hold descriptors in uniform
// registers instead of wrapping every tcgen05.mma in a per-lane (ELECT / R2UR) loop.
__device__ __forceinline__ void umma_tf32_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                                   uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// The three MMAs of one k-step (hi*lo, lo*hi, hi*hi into one accumulator) in ONE statement: the
// operands are moved to uniform registers once per k-step instead of once per MMA.
__device__ __forceinline__ void umma_tf32_triple_elect(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo,
                                                       uint32_t desc_b_lo, uint32_t desc_b_hi,
                                                       uint32_t desc_upper, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 dl, dh;\n\t"
        "setp.eq.b32 p, 0, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "mov.b64 dl, {%3, %5};\n\t"
        "mov.b64 dh, {%4, %5};\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], dl, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], dh, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], dh, %6, p;\n\t}"
        ::"r"(d_tmem), "r"(a_hi), "r"(a_lo), "r"(desc_b_lo), "r"(desc_b_hi), "r"(desc_upper), "r"(idesc)
        : "memory");
}
__device__ __forceinline__ void umma_f16_triple_elect(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo,
                                                      uint32_t desc_b_lo, uint32_t desc_b_hi,
                                                      uint32_t desc_upper, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 dl, dh;\n\t"
        "setp.eq.b32 p, 0, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "mov.b64 dl, {%3, %5};\n\t"
        "mov.b64 dh, {%4, %5};\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], dl, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], dh, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], dh, %6, p;\n\t}"
        ::"r"(d_tmem), "r"(a_hi), "r"(a_lo), "r"(desc_b_lo), "r"(desc_b_hi), "r"(desc_upper), "r"(idesc)
        : "memory");
}
// F16 mode: exponent e with max|x| * 2^e in [2^12, 2^13) (0 for an all-zero, NaN or Inf frame)
__device__ __forceinline__ int frame_scale_exp(const uint32_t *max_bits) {
    const uint32_t b = __ldcg(max_bits);
    const int ex = (int)((b >> 23) & 0xffu);
    if (ex == 0 || ex == 255) return 0;
    return max(-100, min(100, 12 - (ex - 127)));       // the scale itself must stay a normal float
}
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((uint32_t)(127 + e) << 23); }
// two floats -> packed f16x2 (first argument in the LOW half: K element 2c, second in the high half)
__device__ __forceinline__ uint32_t pack_f16x2(float lo_elem, float hi_elem) {
    uint32_t d;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi_elem), "f"(lo_elem));
    return d;
}
__device__ __forceinline__ void umma_commit_elect(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
        ::"r"(bar) : "memory");
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
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
// tcgen05.ld is asynchronous: its destination registers are only valid after tcgen05.wait::ld.
// The wait therefore names them as read-write operands, so the compiler cannot place any use (or
// any register-to-register copy) of them between the load and the wait.
__device__ __forceinline__ void tmem_wait_ld16(uint32_t (&r)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15])
                 :: "memory");
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
// Instruction descriptor (cute::UMMA::InstrDescriptor): D = F32, A = B = TF32, both K-major,
// dense, N at bits [17,23) as N >> 3, M at bits [24,29) as M >> 4.
// kind::f16 with F16 operands: format fields 0, D = F32
__host__ __device__ constexpr uint32_t instr_desc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__host__ __device__ constexpr uint32_t instr_desc(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ int fold_row_u(int i, int n) {
    if ((unsigned)i < (unsigned)n) return i;
    const int once = i < 0 ? -i - 1 : 2 * n - 1 - i;      // one reflection covers radius <= n
    if ((unsigned)once < (unsigned)n) return once;
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
__device__ __forceinline__ Unit decode_unit(int i, const UmmaArgs &a) {
    const int u = a.sched ? __ldg(a.sched + i) : i;
    Unit x;
    x.c0 = (u % a.tiles_c) * kUT;
    const int t = u / a.tiles_c;
    if (a.gate_word) {                  // streamed: tile row slowest, levels (longest first) inside
        x.g = t % a.n_order;
        x.r0 = (t / a.n_order) * kUT;
    } else {
        x.r0 = (t % a.tiles_r) * kUT;
        x.g = t / a.tiles_r;
    }
    return x;
}

// this warp's 32 lanes x 64 columns of the three accumulators <- 0
__device__ __forceinline__ void zero_acc_half(uint32_t lane_base, int half, int dgroup) {
    const uint32_t z[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int c = dgroup; c < kHalf / 16; c += kDrainGroups) {
        const uint32_t col = (uint32_t)(half * kHalf + c * 16);
#pragma unroll
        for (int i = 0; i < kAccs; ++i) tmem_st16(lane_base + i * kAccCols + col, z);
    }
    tmem_wait_st();
}

struct SharedCtl {
    unsigned long long raw_full[kMaxRawStages], raw_empty[kMaxRawStages];
    unsigned long long data_full[kStages], data_empty[kStages];
    unsigned long long toep_full[2], toep_empty[2];
    unsigned long long acc_full[2], acc_empty[2];
    uint32_t tmem_base;
    uint32_t pad[3];
};
static_assert(sizeof(SharedCtl) <= 1024, "control block");

template <int MODE>
__global__ void __launch_bounds__(kUThreads, 1)
umma_pass_kernel(const UmmaArgs a, const __grid_constant__ LevelTable tbl,
                 const __grid_constant__ ToeplitzTable ttab, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    SharedCtl *ctl = reinterpret_cast<SharedCtl *>(smem_raw);
    float *toep = reinterpret_cast<float *>(smem_raw + 1024);     // [buffer 2][hi | lo][toep_floats]
    float *s_prev = toep + 4 * (size_t)a.toep_floats;              // DoG: [n 128][m 128]
    float *raw = s_prev + (MODE == kModeDog ? kUT * kUT : 0);      // [raw stage][16 rows][128]
    const int R = a.raw_stages;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < R; ++s) {
            mbar_init(smem_u32(&ctl->raw_full[s]), 64);
            mbar_init(smem_u32(&ctl->raw_empty[s]), 4);
        }
        for (int s = 0; s < kStages; ++s) {
            mbar_init(smem_u32(&ctl->data_full[s]), 4);
            mbar_init(smem_u32(&ctl->data_empty[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&ctl->toep_full[b]), 1);
            mbar_init(smem_u32(&ctl->toep_empty[b]), kIssuers);
            mbar_init(smem_u32(&ctl->acc_full[b]), kIssuers);
            mbar_init(smem_u32(&ctl->acc_empty[b]), 4 * kDrainGroups);
        }
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(smem_u32(&ctl->tmem_base), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // The CTA owns all 512 columns, so the allocation starts at TMEM address 0; using the literal
    // keeps every TMEM address and descriptor of the issuer in uniform registers.
    if (*reinterpret_cast<volatile uint32_t *>(&ctl->tmem_base) != 0u) __trap();
    constexpr uint32_t tmem = 0u;

    // the accumulators start zeroed: the issuers only ever accumulate
    const bool is_drain = (warp >= 4 && warp < 8) || (kDrainGroups > 1 && warp >= kDrainB);
    const int dgroup = warp >= kDrainB ? 1 : 0;
    if (is_drain) {
        const uint32_t lane_base0 = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
        zero_acc_half(lane_base0, 0, dgroup);
        zero_acc_half(lane_base0, 1, dgroup);
        tc_fence_before();
    }
    __syncthreads();
    tc_fence_after();

    if (warp == 0 || (warp >= kIssuerB && warp < kDrainB)) {
        // ================= issuers (whole warps, one elected lane issues) =================
        // Band structure: k-step m0 only feeds outputs n in [m0 - 2 rpad, m0 + 7], so its MMAs are
        // issued for that column range only (rounded to 16; the Toeplitz window and the
        // accumulator address move with it).
        // Accuracy: the tensor core truncates the float32 accumulator after every MMA, a bias of
        // half an ulp of the running sum per MMA.  Every issuing warp owns one accumulator (half
        // the chain length, about half the magnitude each); the drain adds them in float32.
        // The accumulators are single buffered and handed over in two column halves: outputs
        // n < 64 are complete after k-step (63 + 2 rpad) / 8 and the next level's first 8 k-steps
        // only touch n < 64, so the drain of one half overlaps the MMAs of the other.
        // Issue rate: preparing and issuing one tcgen05.mma costs the issuing warp about 120 cycles
        // (operands travel vector -> uniform registers), three times what the tensor pipe needs
        // for it (ncu: pipe 27 % busy with one issuer).  Stages therefore alternate between two
        // issuing warps.  Each warp accumulates into its OWN accumulator, so the summation order
        // of every output is fixed (results are bit-reproducible from run to run) however the
        // tensor pipe interleaves the two instruction streams; the drain hands the accumulator
        // halves back zeroed, so no MMA has to be "the first"; each warp commits what it issued.
        const uint32_t me = warp == 0 ? 0u : (uint32_t)(warp - kIssuerB + 1);
        uint32_t stage_it = 0, lvl_it = 0;
        constexpr uint32_t idesc0 = instr_desc(kUT, 0);
        constexpr uint32_t desc_hi = (kToepGroupBytes >> 4) | (1u << 14);        // SBO, version 1
        RoleClock rc(a.prof != nullptr && lane == 0 && warp == 0);
        for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
            const Unit un = decode_unit(u, a);
            const int lb = a.by_order ? tbl.order[un.g] : tbl.group_begin[un.g];
            const int le = a.by_order ? lb + 1 : tbl.group_begin[un.g + 1];
            for (int level = lb; level < le; ++level, ++lvl_it) {
                const int rpad2 = 2 * tbl.lv[level].rpad;
                const int Kp = kUT + rpad2;
#if DOGBLOB_UMMA_F16
                constexpr int kStepRows = 16, kSteps = kStageRows / 16;      // MMA steps of 16 rows
#else
                constexpr int kStepRows = 8, kSteps = kStageK;
#endif
                const int n_k = Kp / kStepRows;
                const int n_stage = (n_k + kSteps - 1) / kSteps;
                // my last stage with a step that feeds n < 64 (rows up to 63 + 2 rpad)
                int st_low = ((kHalf - 1 + rpad2) / kStepRows) / kSteps;
                st_low -= (int)((stage_it + (uint32_t)st_low + kIssuers - me) % kIssuers);
                const uint32_t b = lvl_it & 1, par = (lvl_it >> 1) & 1, lpar = lvl_it & 1;
                rc.lap(3);
                mbar_wait(smem_u32(&ctl->toep_full[b]), par, 1);
                rc.lap(0);
                mbar_wait(smem_u32(&ctl->acc_empty[0]), lpar ^ 1, 2);
                rc.lap(1);
                tc_fence_after();
                // low descriptor word of the window of k-step 0 (row Kp - 8); every k-step moves the
                // window up by 8 rows = one 256-byte group = 16 descriptor units
                const uint32_t t_hi = smem_u32(toep + (size_t)(2 * b) * a.toep_floats);
                const uint32_t lo_off = (uint32_t)ttab.rows[level] * 2u;            // hi -> lo array
                const uint32_t win0 = ((t_hi + (uint32_t)((Kp - kStepRows) >> 3) * kToepGroupBytes) >> 4) |
                                      ((kToepHalfBytes >> 4) << 16);
                bool high_ok = false;
                for (int st = (int)((me + kIssuers - stage_it % kIssuers) % kIssuers); st < n_stage; st += kIssuers) {
                    if (!high_ok && st >= 64 / kStageRows) {      // rows from 64 on reach n >= 64
                        mbar_wait(smem_u32(&ctl->acc_empty[1]), lpar ^ 1, 9);
                        high_ok = true;
                    }
                    const uint32_t g = stage_it + (uint32_t)st, sl = g % kStages;
                    const uint32_t a0 = tmem + kStageCol0 + sl * kStageCols;
                    rc.lap(3);
                    mbar_wait(smem_u32(&ctl->data_full[sl]), (g / kStages) & 1, 3);
                    rc.lap(2);
                    tc_fence_after();
#pragma unroll
                    for (int ks = 0; ks < kSteps; ++ks) {
                        const int kidx = st * kSteps + ks;
                        if (kidx < n_k && !(a.debug & 8)) {
                            const int m0 = kStepRows * kidx;
                            int ns = max(0, m0 - rpad2) & ~15;
                            int ne = min(kUT, (m0 + kStepRows + 15) & ~15);
                            if (a.debug & 32) {          // experiment: untrimmed half / full width
                                ns = m0 - rpad2 >= kHalf ? kHalf : 0;
                                ne = m0 + kStepRows <= kHalf ? kHalf : kUT;
                            }
                            // the window moves up by kStepRows rows = kStepRows / 8 groups of 16 units
                            const uint32_t dh = win0 - (uint32_t)(2 * kStepRows) * (uint32_t)kidx + 2u * (uint32_t)ns;
                            const uint32_t acc = tmem + (kIssuers > 1 ? me : (uint32_t)(kidx & 1)) * kAccCols + ns;   // this warp's accumulator(s)
#if DOGBLOB_UMMA_F16
                            const uint32_t a_hi = a0 + ks * 32, a_lo = a_hi + 8;
                            const uint32_t idesc = instr_desc_f16(kUT, 0) | ((uint32_t)((ne - ns) >> 3) << 17);
                            umma_f16_triple_elect(acc, a_hi, a_lo, dh + lo_off, dh, desc_hi, idesc);
#else
                            const uint32_t a_hi = a0 + ks * 16, a_lo = a_hi + 8;
                            const uint32_t idesc = idesc0 | ((uint32_t)((ne - ns) >> 3) << 17);
                            umma_tf32_triple_elect(acc, a_hi, a_lo, dh + lo_off, dh, desc_hi, idesc);
#endif
                        }
                    }
                    umma_commit_elect(smem_u32(&ctl->data_empty[sl]));
                    if (st == st_low) umma_commit_elect(smem_u32(&ctl->acc_full[0]));
                }
                stage_it += (uint32_t)n_stage;
                umma_commit_elect(smem_u32(&ctl->toep_empty[b]));
                umma_commit_elect(smem_u32(&ctl->acc_full[1]));
            }
        }
        rc.lap(3);
        rc.flush(a.prof, 0);
        if (rc.on) {        // slowest / fastest CTA (issuer's whole life)
            const unsigned long long tot = rc.acc[0] + rc.acc[1] + rc.acc[2] + rc.acc[3];
            atomicMax(a.prof + 10, tot);
            atomicMin(a.prof + 11, tot);
        }
    } else if (warp == 1) {
        // ================= Toeplitz copier: prebuilt hi|lo arrays, one bulk copy per level ========
        uint32_t lvl_it = 0;
        RoleClock rc(a.prof != nullptr && lane == 0);
        for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
            const Unit un = decode_unit(u, a);
            const int lb = a.by_order ? tbl.order[un.g] : tbl.group_begin[un.g];
            const int le = a.by_order ? lb + 1 : tbl.group_begin[un.g + 1];
            for (int level = lb; level < le; ++level, ++lvl_it) {
                const uint32_t b = lvl_it & 1, par = (lvl_it >> 1) & 1;
                rc.lap(1);
                mbar_wait_sleep(smem_u32(&ctl->toep_empty[b]), par ^ 1, 4);
                rc.lap(0);
                if (lane == 0) {
                    const uint32_t bytes = (uint32_t)ttab.rows[level] * 64u;     // hi + lo
                    const uint32_t bar = smem_u32(&ctl->toep_full[b]);
                    mbar_expect_tx(bar, bytes);
                    bulk_copy_g2s(smem_u32(toep + (size_t)(2 * b) * a.toep_floats),
                                  a.toep + ttab.ofs[level], bytes, bar);
                }
                __syncwarp();
            }
        }
        rc.lap(1);
        rc.flush(a.prof, 4);
    } else if (warp < 4) {
        // ================= row loaders: 32 input rows x 512 B per raw stage =====================
        // interior stages: one TMA box; stages that cross the image border: 64 threads x 16
        // LDGSTS of 16 bytes with folded rows (thread t: column group t & 31 of rows (t >> 5) + 2 i).
        const int t = threadIdx.x - 64;
        const int cg = t & 31, rsub = t >> 5;
        uint32_t rs = 0, rp = 0;                          // raw stage and its phase parity
        int gate_have = 0;
        bool gate_stamped = false;
        RoleClock rc(a.prof != nullptr && t == 0);
        for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
            const Unit un = decode_unit(u, a);
            const int lb = a.by_order ? tbl.order[un.g] : tbl.group_begin[un.g];
            const int le = a.by_order ? lb + 1 : tbl.group_begin[un.g + 1];
            for (int level = lb; level < le; ++level) {
                const int rpad = tbl.lv[level].rpad;
                const int n_stage = (kUT + 2 * rpad + kStageRows - 1) / kStageRows;
                const float *src = a.in + (int64_t)level * a.in_plane + un.c0 + 4 * cg;
                int row0 = un.r0 - rpad;
                for (int st = 0; st < n_stage; ++st, row0 += kStageRows, rp ^= (rs + 1 == (uint32_t)R),
                         rs = (rs + 1 == (uint32_t)R) ? 0 : rs + 1) {
                    rc.lap(1);
                    mbar_wait(smem_u32(&ctl->raw_empty[rs]), rp ^ 1, 7);
                    rc.lap(0);
                    if (a.gate_word) {
                        // last image row this stage reads (rows above 0 / below n_rows fold inwards)
                        int need_row = row0 + kStageRows - 1;
                        if (row0 < 0) need_row = max(need_row, -row0 - 1);
                        need_row = min(need_row, a.n_rows - 1);
                        if (a.n_rows < kStageRows + tbl.lv[level].rpad) need_row = a.n_rows - 1;
                        const int need = need_row / a.gate_rows_per_chunk + 1;
                        if (need > gate_have) {
                            while ((gate_have = *(const volatile int *)a.gate_word - a.gate_base) < need)
                                __nanosleep(200);
                            __threadfence();
                        }
                        if (!gate_stamped) {
                            gate_stamped = true;
                            if (blockIdx.x == 0 && t == 0 && a.gate_t_start) *a.gate_t_start = globaltimer_ns();
                        }
                    }
                    const uint32_t bar = smem_u32(&ctl->raw_full[rs]);
                    if (a.use_tma && row0 >= 0 && row0 + kStageRows <= a.n_rows) {
                        if (t == 0) {
                            mbar_expect_tx_only(bar, kStageRows * kUT * 4);
                            tma_load_2d(smem_u32(raw + (size_t)rs * kStageRows * kUT), &tmap, un.c0,
                                        level * a.tma_plane_rows + row0, bar);
                        }
                        mbar_arrive(bar);
                        continue;
                    }
                    const uint32_t dst = smem_u32(raw + ((size_t)rs * kStageRows + rsub) * kUT + 4 * cg);
#pragma unroll 4
                    for (int i = 0; i < kStageRows / 2; ++i)
                        cp_async16(dst + i * 2 * kUT * 4,
                                   src + (int64_t)fold_row_u(row0 + rsub + 2 * i, a.n_rows) * a.in_pitch);
                    cp_async_arrive_noinc(bar);
                }
            }
        }
        rc.lap(1);
        rc.flush(a.prof, 6);
    } else if (is_drain) {
        // ================= drain (accumulators -> DoG -> global), one column half at a time ======
        const int q = warp & 3;
        const int m = 32 * q + lane;
        uint32_t lvl_it = 0;
        RoleClock rc(a.prof != nullptr && warp == 4 && lane == 0);
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
#if DOGBLOB_UMMA_F16
        const int frame_exp = frame_scale_exp(a.frame_max_bits);
#endif
        for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
            const Unit un = decode_unit(u, a);
            const int lb = a.by_order ? tbl.order[un.g] : tbl.group_begin[un.g];
            const int le = a.by_order ? lb + 1 : tbl.group_begin[un.g + 1];
            for (int level = lb; level < le; ++level, ++lvl_it) {
                const uint32_t lpar = lvl_it & 1;
                const bool park_first = MODE == kModeDog && level == lb && un.g > 0;
                const bool park_last = MODE == kModeDog && level == le - 1 && un.g < tbl.n_groups - 1;
                const float sig = MODE == kModeDog && level > lb ? tbl.lv[level - 1].sigma_f32 : 0.f;
#if DOGBLOB_UMMA_F16
                // exact (powers of two), applied one after the other so neither factor underflows
                const float unscale_t = pow2f(-ttab.tscale[level]), unscale_x = pow2f(-frame_exp);
#endif
#pragma unroll 1
                for (int half = 0; half < 2; ++half) {
                    rc.lap(1);
                    mbar_wait_sleep(smem_u32(&ctl->acc_full[half]), lpar, 5);
                    rc.lap(0);
                    tc_fence_after();
#pragma unroll 1
                    for (int c = dgroup; c < kHalf / 16; c += kDrainGroups) {   // the groups share a half
                        const int n0 = half * kHalf + c * 16;
                        uint32_t ra[kAccs][16];
#pragma unroll
                        for (int i = 0; i < kAccs; ++i) tmem_ld16(lane_base + i * kAccCols + n0, ra[i]);
#pragma unroll
                        for (int i = 0; i < kAccs; ++i) tmem_wait_ld16(ra[i]);
                        if (a.debug & 4) continue;
                        float r[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            r[j] = __uint_as_float(ra[0][j]);
#pragma unroll
                            for (int i = 1; i < kAccs; ++i) r[j] = __fadd_rn(r[j], __uint_as_float(ra[i][j]));
#if DOGBLOB_UMMA_F16
                            r[j] = __fmul_rn(__fmul_rn(r[j], unscale_t), unscale_x);
#endif
                        }
                        if (MODE == kModeRows) {
                            // lane = x (contiguous input axis), registers = 16 consecutive y of T[x][y]
                            float *dst = a.out + (int64_t)level * a.out_plane +
                                         (int64_t)(un.c0 + m) * a.out_pitch + un.r0 + n0;
#pragma unroll
                            for (int j = 0; j < 16; j += 4)
                                *reinterpret_cast<float4 *>(dst + j) = make_float4(r[j], r[j + 1], r[j + 2], r[j + 3]);
                        } else {
                            // lane = y (contiguous), registers = 16 consecutive output rows x
                            const int64_t tile_ofs = (int64_t)(un.r0 + n0) * a.out_pitch + un.c0 + m;
                            if (MODE == kModeLevels) {
                                float *dst = a.out + (int64_t)level * a.out_plane + tile_ofs;
#pragma unroll
                                for (int j = 0; j < 16; ++j) dst[(int64_t)j * a.out_pitch] = r[j];
                            } else {
                                if (park_first || park_last) {
                                    float *dst = a.edge + (int64_t)(2 * un.g + (park_first ? 0 : 1)) * a.out_plane + tile_ofs;
#pragma unroll
                                    for (int j = 0; j < 16; ++j) dst[(int64_t)j * a.out_pitch] = r[j];
                                    if (park_first && park_last) {      // single-level group
                                        dst = a.edge + (int64_t)(2 * un.g + 1) * a.out_plane + tile_ofs;
#pragma unroll
                                        for (int j = 0; j < 16; ++j) dst[(int64_t)j * a.out_pitch] = r[j];
                                    }
                                }
                                float *slot = s_prev + n0 * kUT + m;
                                if (level > lb) {
                                    float *dst = a.out + (int64_t)(level - 1) * a.out_plane + tile_ofs;
#pragma unroll
                                    for (int j = 0; j < 16; ++j)
                                        dst[(int64_t)j * a.out_pitch] = __fmul_rn(__fsub_rn(slot[j * kUT], r[j]), sig);
                                }
                                if (level < le - 1) {
#pragma unroll
                                    for (int j = 0; j < 16; ++j) slot[j * kUT] = r[j];
                                }
                            }
                        }
                    }
                    zero_acc_half(lane_base, half, dgroup);  // every MMA accumulates (none is "first")
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(&ctl->acc_empty[half]));
                }
            }
        }
        rc.lap(1);
        rc.flush(a.prof, 8);
    } else {
        // ================= converters (raw rows -> hi/lo -> TMEM A staging) =================
        const int q = warp & 3;
        const int grp = (warp - 8) >> 2;
        const int m = 32 * q + lane;
        RoleClock rc(a.prof != nullptr && warp == 8 && lane == 0);
#if DOGBLOB_UMMA_F16
        const float xscale = pow2f(frame_scale_exp(a.frame_max_bits));
#endif
        int total = 0;                                   // stages this CTA processes
        for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
            const Unit un = decode_unit(u, a);
            const int lb = a.by_order ? tbl.order[un.g] : tbl.group_begin[un.g];
            const int le = a.by_order ? lb + 1 : tbl.group_begin[un.g + 1];
            for (int level = lb; level < le; ++level)
                total += (kUT + 2 * tbl.lv[level].rpad + kStageRows - 1) / kStageRows;
        }
        uint32_t rs = grp % R, rp = (grp / R) & 1;
        for (uint32_t stage_it = grp; stage_it < (uint32_t)total; stage_it += kLoaderGroups,
                      rs += kLoaderGroups, rp ^= (rs >= (uint32_t)R), rs -= (rs >= (uint32_t)R) ? R : 0) {
            const uint32_t s = stage_it % kStages, sp = (stage_it / kStages) & 1;
            rc.lap(3);
            mbar_wait(smem_u32(&ctl->raw_full[rs]), rp, 8);
            rc.lap(0);
            const float *src = raw + (size_t)rs * kStageRows * kUT + m;
            const uint32_t dst = tmem + kStageCol0 + s * kStageCols + ((uint32_t)(32 * q) << 16);
#pragma unroll
            for (int h = 0; h < kStageK / 2; ++h) {       // 16 rows = 2 k-steps at a time
                float v[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) v[k] = src[(16 * h + k) * kUT];
                uint32_t r0[16], r1[16];
#if DOGBLOB_UMMA_F16
                // 16 rows = one MMA step: columns 0..7 hi (2 rows per column), 8..15 lo
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float s0 = __fmul_rn(v[2 * k], xscale), s1 = __fmul_rn(v[2 * k + 1], xscale);
                    const uint32_t hp = pack_f16x2(s0, s1);
                    const float2 hf = __half22float2(*reinterpret_cast<const __half2 *>(&hp));
                    r0[k] = hp;
                    r0[8 + k] = pack_f16x2(__fsub_rn(s0, hf.x), __fsub_rn(s1, hf.y));
                    r1[k] = 0; r1[8 + k] = 0;
                }
#else
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    split_tf32(v[k], r0[k], r0[8 + k]);
                    split_tf32(v[8 + k], r1[k], r1[8 + k]);
                }
#endif
                if (h == kStageK / 2 - 1) {               // all rows of the raw stage are in registers
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(&ctl->raw_empty[rs]));
                }
                if (h == 0) {
                    rc.lap(1);
                    mbar_wait(smem_u32(&ctl->data_empty[s]), sp ^ 1, 6);
                    rc.lap(2);
                    tc_fence_after();
                }
                tmem_st16(dst + 32 * h, r0);
#if !DOGBLOB_UMMA_F16
                tmem_st16(dst + 32 * h + 16, r1);
#endif
                // tcgen05.st reads its source registers asynchronously: they must not be reused
                // (the next half's values land in the same physical registers) before wait::st.
                // Found the hard way: without this wait some builds returned a few corrupted
                // stages per frame, different from run to run (tools/umma_repro.py).
                tmem_wait_st();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&ctl->data_full[s]));
        }
        rc.lap(3);
        rc.flush(a.prof, 12);
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

#if DOGBLOB_UMMA_F16
int toeplitz_rows(int rpad) { return kUT + 2 * rpad - 16 + kUT; }
#else
int toeplitz_rows(int rpad) { return kUT + 2 * rpad - 8 + kUT; }
#endif
int toeplitz_floats(int max_rpad) { return toeplitz_rows(max_rpad) * 8; }

constexpr size_t kSmemLimit = 227 * 1024;
size_t umma_fixed_smem(int max_rpad, bool dog) {
    return 1024 + 4 * (size_t)toeplitz_floats(max_rpad) * sizeof(float) +
           (dog ? (size_t)kUT * kUT * sizeof(float) : 0);
}
int raw_stages_for(int max_rpad, bool dog) {
    const size_t fixed = umma_fixed_smem(max_rpad, dog);
    if (fixed + 2 * kStageRows * kUT * 4 > kSmemLimit) return 0;
    // a multiple of the number of converter groups: a raw stage is then always converted by the
    // same group, so no waiter is ever two phases behind its barrier (a parity wait cannot tell
    // phase n from phase n + 2)
    const size_t r = std::min<size_t>(kMaxRawStages, (kSmemLimit - fixed) / (kStageRows * kUT * 4));
    return (int)(r / kLoaderGroups * kLoaderGroups);
}

// 2-D tensor map over the input rows: inner dimension = the pitch (contiguous axis), outer = all
// rows of all level planes; box = 128 floats x 16 rows, no swizzle, no interleave.
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);
bool encode_rows_map(CUtensorMap *map, const float *base, uint64_t pitch, uint64_t rows) {
    static EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    if (!fn) return false;
    const cuuint64_t dims[2] = {pitch, rows};
    const cuuint64_t strides[1] = {pitch * sizeof(float)};
    const cuuint32_t box[2] = {(cuuint32_t)kUT, (cuuint32_t)kStageRows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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
cudaError_t launch_umma(const UmmaArgs &a, const LevelTable &tbl, const ToeplitzTable &ttab,
                        int max_rpad, cudaStream_t st) {
    UmmaArgs b = a;
    b.toep_floats = toeplitz_floats(max_rpad);
    b.raw_stages = raw_stages_for(max_rpad, MODE == kModeDog);
    if (const char *e = std::getenv("DOGBLOB_UMMA_RAW")) b.raw_stages = std::max(2, std::min(b.raw_stages, std::atoi(e))) / kLoaderGroups * kLoaderGroups;
    const size_t smem = umma_fixed_smem(max_rpad, MODE == kModeDog) +
                        (size_t)b.raw_stages * kStageRows * kUT * 4;
    if (const char *e = std::getenv("DOGBLOB_UMMA_DEBUG")) b.debug = std::atoi(e);
    static unsigned long long *d_prof = nullptr;
    const bool prof = std::getenv("DOGBLOB_UMMA_PROF") != nullptr;
    if (prof) {
        if (!d_prof) cudaMalloc(&d_prof, 16 * sizeof(unsigned long long));
        cudaMemsetAsync(d_prof, 0, 16 * sizeof(unsigned long long), st);
        cudaMemsetAsync(d_prof + 11, 0xff, sizeof(unsigned long long), st);
        b.prof = d_prof;
    }
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof(tmap));
    b.use_tma = 0;
    if (!std::getenv("DOGBLOB_UMMA_NO_TMA")) {
        const int planes = b.in_plane ? tbl.n_levels : 1;
        const int plane_rows = b.in_plane ? (int)(b.in_plane / b.in_pitch) : b.n_rows;
        b.tma_plane_rows = b.in_plane ? plane_rows : 0;
        if (encode_rows_map(&tmap, b.in, (uint64_t)b.in_pitch, (uint64_t)planes * plane_rows)) b.use_tma = 1;
    }
    const int ctas = persistent_ctas(b.n_units);
    umma_pass_kernel<MODE><<<ctas, kUThreads, smem, st>>>(b, tbl, ttab, tmap);
    if (prof) {
        unsigned long long h[16];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, d_prof, sizeof(h), cudaMemcpyDeviceToHost);
        static const char *names[16] = {
            "issuer    wait toeplitz", "issuer    wait acc free", "issuer    wait data", "issuer    issue+other",
            "toeplitz  wait buffer", "toeplitz  issue", "rows      wait raw stage free", "rows      cp.async issue",
            "drain     wait acc", "drain     ld+store", "-", "-",
            "converter wait raw rows", "converter lds+split", "converter wait stage free", "converter st+arrive"};
        fprintf(stderr, "umma mode %d, %d CTAs, %d raw stages, kilo-cycles per CTA:", MODE, ctas, b.raw_stages);
        for (int i = 0; i < 16; ++i)
            if (names[i][0] != '-') fprintf(stderr, "\n   %-34s %8.1f", names[i], h[i] / 1e3 / ctas);
        fprintf(stderr, "\n   issuer total: slowest CTA %.1f, fastest %.1f\n", h[10] / 1e3, h[11] / 1e3);
    }
    return cudaGetLastError();
}

}  // namespace

bool umma_supported(const ConvGeometry &g) { return raw_stages_for(g.max_rpad, true) >= 2; }

// Toeplitz operand of every level, as the kernel wants it in shared memory (see the header of
// this file): per level `rows` = Kp - 8 + 128 rows of 8 taps, hi array then lo array, 8-row groups
// of 256 bytes = [K half 0: 8 rows x 16 B][K half 1: 8 rows x 16 B].
// G[p][kk] = w[kk - p + Kp - 8]; taps: the plan's duplicated table (entry t = offset t - rpad).
static uint32_t host_tf32_rna(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;        // round to nearest, ties away (finite inputs)
    return u;
}
void build_toeplitz(const LevelDesc *lv, int n_levels, const float2 *taps, std::vector<float> &out,
                    ToeplitzTable &tab) {
    out.clear();
    for (int i = 0; i < n_levels; ++i) {
        const int rpad = lv[i].rpad, Kp = kUT + 2 * rpad, rows = toeplitz_rows(rpad);
        tab.ofs[i] = (int)out.size();
        tab.rows[i] = rows;
        tab.tscale[i] = 0;
        out.resize(out.size() + (size_t)rows * 16, 0.f);
        const float2 *w = taps + lv[i].tap_ofs;
#if DOGBLOB_UMMA_F16
        // fp16 hi | lo arrays: rows of 16 taps (32 bytes), 8-row groups of 256 bytes =
        // [K half 0: 8 rows x 8 taps][K half 1]; taps scaled by 2^t so that the largest is in [512, 1024)
        float wmax = 0.f;
        for (int t = 0; t <= 2 * rpad; ++t) wmax = std::max(wmax, w[t].x);
        int tsc = 0;
        if (wmax > 0.f) { int ex; std::frexp(wmax, &ex); tsc = 10 - ex; }      // wmax * 2^tsc in [512, 1024)
        tab.tscale[i] = tsc;
        __half *hi = reinterpret_cast<__half *>(out.data() + tab.ofs[i]);
        __half *lo = hi + (size_t)rows * 16;
        for (int p = 0; p < rows; ++p)
            for (int kk = 0; kk < 16; ++kk) {
                const int t = kk - p + (Kp - 16);
                const float v = (t >= 0 && t <= 2 * rpad) ? std::ldexp(w[t].x, tsc) : 0.f;
                const __half h = __float2half_rn(v);
                const __half l = __float2half_rn(v - __half2float(h));
                const size_t o = (size_t)(p >> 3) * 128 + (kk >> 3) * 64 + (p & 7) * 8 + (kk & 7);
                hi[o] = h;
                lo[o] = l;
            }
#else
        float *hi = out.data() + tab.ofs[i], *lo = hi + (size_t)rows * 8;
        for (int p = 0; p < rows; ++p)
            for (int kk = 0; kk < 8; ++kk) {
                const int t = kk - p + (Kp - 8);
                const float v = (t >= 0 && t <= 2 * rpad) ? w[t].x : 0.f;
                const uint32_t h = host_tf32_rna(v);
                float hf;
                std::memcpy(&hf, &h, 4);
                const uint32_t l = host_tf32_rna(v - hf);
                float lf;
                std::memcpy(&lf, &l, 4);
                const size_t o = (size_t)(p >> 3) * 64 + (kk >> 2) * 32 + (p & 7) * 4 + (kk & 3);
                hi[o] = hf;
                lo[o] = lf;
            }
#endif
    }
}

// F16 mode: max |x| of the frame as float bits (non-negative floats order like unsigned integers)
__global__ void frame_max_kernel(const float *__restrict__ img, int64_t n4, uint32_t *__restrict__ max_bits) {
    float m = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(img) + i);
        m = fmaxf(fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))), m);
    }
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(max_bits, __float_as_uint(m));
}
bool umma_needs_frame_max() { return DOGBLOB_UMMA_F16 != 0; }
cudaError_t launch_frame_max(const float *d_img, int64_t n_floats, uint32_t *d_max_bits, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(d_max_bits, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    frame_max_kernel<<<148, 256, 0, st>>>(d_img, n_floats / 4, d_max_bits);
    return cudaGetLastError();
}

// Cost-balanced static schedule.  CTA b walks positions b, b + n_ctas, ... ; the units are sorted
// by modelled cost (stages, +1.5 per stage that crosses the image border and goes through the
// folded cp.async path, +1 per level) and dealt to the CTAs in boustrophedon order, so every CTA
// gets a similar sum.  rows_axis = valid rows along the convolved axis (H for the row pass, W for
// the column pass).
std::vector<int> build_umma_schedule(const ConvGeometry &g, const LevelTable &tbl, bool rows_pass) {
    const int tiles_c = (rows_pass ? g.Wp : g.Hp) / kUT, tiles_r = (rows_pass ? g.Hp : g.Wp) / kUT;
    const int n_rows = rows_pass ? g.H : g.W;
    const int n_g = rows_pass ? tbl.n_levels : tbl.n_groups;
    const int n_units = tiles_c * tiles_r * n_g;
    std::vector<std::pair<double, int>> cost(n_units);
    for (int u = 0; u < n_units; ++u) {
        const int t = u / tiles_c, tr = t % tiles_r, gi = t / tiles_r;
        const int lb = rows_pass ? tbl.order[gi] : tbl.group_begin[gi];
        const int le = rows_pass ? lb + 1 : tbl.group_begin[gi + 1];
        double c = 0.0;
        for (int level = lb; level < le; ++level) {
            const int rpad = tbl.lv[level].rpad;
            const int n_stage = (kUT + 2 * rpad + kStageRows - 1) / kStageRows;
            int row0 = tr * kUT - rpad;
            for (int st = 0; st < n_stage; ++st, row0 += kStageRows)
                c += (row0 >= 0 && row0 + kStageRows <= n_rows) ? 1.0 : 2.5;
            c += 1.0;
        }
        cost[u] = {c, u};
    }
    std::stable_sort(cost.begin(), cost.end(), [](const std::pair<double, int> &x, const std::pair<double, int> &y) {
        return x.first > y.first;
    });
    const int ctas = persistent_ctas(n_units);
    std::vector<int> sched(n_units);
    for (int r = 0; r < n_units; ++r) {
        const int round = r / ctas, k = r % ctas;
        const int last = std::min(ctas, n_units - round * ctas);        // units in this round
        const int pos = (round & 1) ? last - 1 - k : k;
        sched[round * ctas + pos] = cost[r].second;
    }
    return sched;
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
                                 const LevelTable &tbl, const ToeplitzTable &ttab,
                                 const float *d_toep, cudaStream_t st, const RowGate *gate,
                                 const uint32_t *d_max_bits, const int *d_sched) {
    UmmaArgs a{};
    a.frame_max_bits = d_max_bits;
    a.in = d_img; a.in_pitch = g.Wp; a.in_plane = 0; a.n_rows = g.H;
    a.out = d_rows_t; a.out_pitch = g.Hp; a.out_plane = (int64_t)g.Hp * g.Wp;
    a.edge = nullptr; a.toep = d_toep;
    a.tiles_c = g.Wp / kUT; a.tiles_r = g.Hp / kUT;
    a.by_order = 1;                       // independent levels: finest units, longest first
    a.n_order = tbl.n_levels;
    a.n_units = a.tiles_c * a.tiles_r * tbl.n_levels;
    a.sched = gate ? nullptr : d_sched;       // streamed uploads need the tile-row-major order
    if (gate) {
        a.gate_word = gate->word; a.gate_base = gate->base;
        a.gate_rows_per_chunk = gate->rows_per_chunk; a.gate_t_start = gate->t_start;
    }
    return launch_umma<kModeRows>(a, tbl, ttab, g.max_rpad, st);
}

// T_i[x][y] -> D_i^T[x][y]: contiguous axis y, convolved axis x
cudaError_t launch_col_dog_pass_umma(const ConvGeometry &g, const float *d_rows_t, float *d_dog_t,
                                     float *d_edge, const LevelTable &tbl, const ToeplitzTable &ttab,
                                     const float *d_toep, cudaStream_t st, const uint32_t *d_max_bits,
                                     const int *d_sched) {
    UmmaArgs a{};
    a.frame_max_bits = d_max_bits;
    a.sched = d_sched;
    a.in = d_rows_t; a.in_pitch = g.Hp; a.in_plane = (int64_t)g.Hp * g.Wp; a.n_rows = g.W;
    a.out = d_dog_t; a.out_pitch = g.Hp; a.out_plane = a.in_plane;
    a.edge = d_edge; a.toep = d_toep;
    a.tiles_c = g.Hp / kUT; a.tiles_r = g.Wp / kUT;
    a.n_units = a.tiles_c * a.tiles_r * tbl.n_groups;
    return launch_umma<kModeDog>(a, tbl, ttab, g.max_rpad, st);
}

cudaError_t launch_col_levels_pass_umma(const ConvGeometry &g, const float *d_rows_t, float *d_lev_t,
                                        const LevelTable &unit_tbl, const ToeplitzTable &ttab,
                                        const float *d_toep, cudaStream_t st, const uint32_t *d_max_bits) {
    UmmaArgs a{};
    a.frame_max_bits = d_max_bits;
    a.in = d_rows_t; a.in_pitch = g.Hp; a.in_plane = (int64_t)g.Hp * g.Wp; a.n_rows = g.W;
    a.out = d_lev_t; a.out_pitch = g.Hp; a.out_plane = a.in_plane;
    a.edge = nullptr; a.toep = d_toep;
    a.tiles_c = g.Hp / kUT; a.tiles_r = g.Wp / kUT;
    a.n_units = a.tiles_c * a.tiles_r * unit_tbl.n_groups;
    return launch_umma<kModeLevels>(a, unit_tbl, ttab, g.max_rpad, st);
}

}  // namespace dogblob
