// Separable Gaussian scale space + fused DoG on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Same results (within float32 rounding) as scale_space.cu (reference: convolve.py:63-218,
// detector.py:117-126), but each banded 1-D correlation is issued as a Toeplitz GEMM with BOTH
// operands in shared memory, brought there by TMA, and no operand is transposed anywhere:
//
//   pass 1 (along y, the strided axis)      D1[y_out][x] = sum_k  T[y_out][k] * X[k][x]
//       A = Toeplitz window (K-major, no swizzle)     B = image rows, MN-major, SWIZZLE_128B
//   pass 2 (along x, the contiguous axis)   D2^T[x_out][y] = sum_k  T[x_out][k] * R[y][k]
//       A = Toeplitz window (K-major, no swizzle)     B = pass-1 rows, K-major, SWIZZLE_128B
//   Both passes issue the SAME two instructions per k-step (the stage's hi and lo planes are the two N halves
//   of one B operand, the small accumulator sits right behind the main one in TMEM):
//       [main | small] += T_hi * [X_hi | X_lo]   (N = 256)        small += T_lo * X_hi   (N = 128)
//   Pass 2's accumulator therefore holds the TRANSPOSED tile (TMEM lane = output column x, accumulator
//   column = row y) and the slices are written transposed, D^T[slice][x][y] - the orientation the FP32
//   engine writes too, which the extrema kernels take as a flag.
//
//   T[n][k] = w[k - n] (0 <= k - n <= 2 rpad), tiles of 128 x 128 outputs, K = 128 + 2 rpad inputs
//   along the convolved axis, 16 per tcgen05.mma.kind::f16 (M = 128).
//
// float32 accuracy from fp16 operands: data and taps are split x = hi + lo, hi = fp16(x),
// lo = fp16(x - hi) (11 + 11 significand bits; exact power-of-two scales keep both in range: the
// frame by 2^e with max|x| 2^e in [2^12, 2^13), every level's taps by 2^t with the largest tap in
// [512, 1024)) and every k-step issues hi*hi, hi*lo and lo*hi.  The tensor core truncates its
// float32 accumulator after every MMA (-1/2 ulp of the running sum each), so the large products
// (hi*hi) and the small ones (2^-11 of them) go to SEPARATE accumulators: the chain that carries the
// magnitude is a third as long, the other one's truncation is negligible; the drain adds the two.
//
// The operands are pre-split in memory: the frame once (prep_split_kernel: fp16 hi | lo planes with
// the reflected halo rows materialised), the pass-1 output by pass 1's drain (hi | lo planes with
// the reflected halo columns written next to the interior) - the same 4 bytes per element as a
// float32 plane, and every stage of both passes is one TMA box straight into MMA operand layout.
//
// Toeplitz operand, compact: the operand rows are indexed by the REVERSED output n' = 127 - n, so
// T'[n'][k] = w[k + n' - 127] depends on k + n' only: the second K half of row n' is the first K
// half of row n' + 8 and ONE 16-byte chunk per row, C[r][e] = w[r + e - 127], serves every k-step
// (LBO = SBO = 128: overlapping core matrices; step j reads the window that starts at row 16 j).
// Half the shared memory and half the copy of a [row][16 taps] array.  The drains undo the
// reversal for free (TMEM lane m' is output row 127 - m' of the tile in pass 1, output column
// 127 - m' = row of the transposed tile in pass 2: an address).
//
// One persistent CTA per SM, 384 threads:
//   warp 0      issuer     ONE elected thread runs the whole loop (its descriptor arithmetic lives
//                          in uniform registers): 2 MMAs per k-step, tcgen05.commit frees the data
//                          stage / the Toeplitz buffer / publishes the accumulator pair.  A commit
//                          costs the issuing thread ~250 cycles during which the tensor pipe runs
//                          dry (tools/ubench_umma_commit.cu), hence stages of 4 k-steps
//   warp 1      loader     one TMA box per stage (pass 1: 64 input rows x 128 x, hi | lo = 32 KB;
//                          pass 2: 128 rows x 64 k, hi | lo = 32 KB)
//   warp 2      Toeplitz   the level's prebuilt compact arrays (hi | lo), bulk copies into a ring
//                          of 2 buffers
//   warps 4..11 drain      tcgen05.ld of the accumulator pair (lane = output row, 64 columns per
//                          thread), scales, pass 1: hi/lo split -> swizzled staging (two boxes per
//                          column half, alternating: one barrier per round) -> TMA store, and for
//                          tiles at the frame border the same rows with their columns reversed ->
//                          TMA store into the halo columns (no negative store coordinates: a
//                          partly outside box is illegal on stores; the half tile under the right
//                          edge shifts its reversed row instead; widths that are not a multiple of
//                          8 get their right halo from edge_halo_kernel); pass 2: DoG against the
//                          previous level kept in
//                          REGISTERS, per-warp staging box -> TMA store into the transposed float32
//                          slice (boxes without a value above the threshold are not stored), seed test
// TMEM: two buffers of {main, small} 128 x 128 float32 accumulators (512 columns), so the drain of
// one level overlaps the MMAs of the next.
// Units: pass 1 = (tile, level), longest level first, round robin; pass 2 = (tile, level group) on
// a static longest-processing-time schedule made at plan time (api.cu: plan_umma_schedule).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda.h>           // CUtensorMap (types only: the encoder is fetched through the runtime)
#include <cuda_fp16.h>

#include "common.cuh"

namespace dogblob {

namespace {

constexpr int kUT = 128;                  // tile edge on both axes
// 12 warps = 3 per scheduler: 168 registers per thread (dropping the idle fourth role warp would not raise
// the limit: one scheduler would still hold three warps)
constexpr int kThreads = 384;
constexpr int kDrainWarp0 = 4;            // warps 4..11 drain
constexpr int kDrainWarps = 8;
constexpr int kAccCols = 128;
#ifndef DOGBLOB_UMMA_ROWS1
#define DOGBLOB_UMMA_ROWS1 64
#endif
constexpr int kRowsPerStage1 = DOGBLOB_UMMA_ROWS1;             // pass 1: input rows per data stage (16 per k-step)
constexpr int kStageBytes1 = 512 * kRowsPerStage1;             // pass 1: [hi | lo][2 x-blocks][rows][128 B]
constexpr int kStageBytes2 = 32768;       // pass 2: [hi | lo][128 rows][128 B]
#ifndef DOGBLOB_UMMA_STAGING1
#define DOGBLOB_UMMA_STAGING1 0
#endif
// pass 1 drain staging: 16 KB boxes per column half, two per half (one being stored while the next is filled)
// unless that costs the fourth data stage (wide ladders: large Toeplitz buffers); 0 = choose, 1 / 2 = force
constexpr int kStagingForce1 = DOGBLOB_UMMA_STAGING1;
__host__ __device__ constexpr int staging_bytes1(int bufs) { return 32768 * bufs; }
constexpr int kStagingBytes2 = 32768;     // pass 2 drain staging: one 4 KB box (32 rows x 32 floats) per drain warp
constexpr int kMaxStages = 8;
#ifndef DOGBLOB_UMMA_BACKOFF
#define DOGBLOB_UMMA_BACKOFF 0
#endif
#ifndef DOGBLOB_UMMA_TOEP1
#define DOGBLOB_UMMA_TOEP1 2
#endif
#ifndef DOGBLOB_UMMA_TOEP2
#define DOGBLOB_UMMA_TOEP2 2
#endif
constexpr int kToepBuffers1 = DOGBLOB_UMMA_TOEP1, kToepBuffers2 = DOGBLOB_UMMA_TOEP2;   // Toeplitz ring depth per pass
constexpr int kMaxToepBuffers = 4;
constexpr unsigned long long kWaitLimitNs = 20ull * 1000 * 1000 * 1000;   // deadlock trap (20 s)

enum UmmaMode { kModeRows = 0, kModeDog = 1, kModeLevels = 2 };

struct UmmaArgs {
    int tiles_x, tiles_y;   // tiles along x (contiguous) and y
    int n_units;            // tiles * (levels | level groups)
    const int *sched;       // static schedule: unit of (slot, CTA) or -1; nullptr = round robin over n_units
    int n_sched;            // slots * CTAs (round robin: n_units)
    int n_ctas;             // CTAs the schedule was made for (0: one per SM, at most n_units)
    int by_order;           // units are single levels in tbl.order[] (pass 1) or groups (pass 2)
    int H, W, Hp, Wp;
    int Py;                 // halo rows above / below the frame in the X planes
    int Ppad;               // halo columns left / right of the interior in the R planes
    int64_t r_pitch;        // elements per row of the R planes (Wq)
    int64_t r_plane;        // elements between the hi and the lo plane set (L * Hp * Wq)
    __half *r_base;         // pass 1: R planes, for the mirrored halo columns
    const uint32_t *frame_max_bits;   // float bits of the frame's max |x| (device word)
    const float *toep;      // prebuilt Toeplitz arrays of every level (hi | lo), see build_toeplitz
    int toep_bytes;         // bytes of one Toeplitz buffer in shared memory (widest level, hi + lo)
    int staging_off;        // byte offset of the drain staging (1 KB aligned; the data stages follow it)
    int stages;             // data stages that fit in shared memory
    unsigned long long *prof;   // DOGBLOB_UMMA_PROF: per-role cycle counters (see launch_umma)
    HitFlags flags;         // pass 2 (DoG): blocks with a value above `thr` (nullptr: not wanted)
    float thr;
    int debug;              // DOGBLOB_UMMA_DEBUG: timing experiments (results are garbage), see launch_umma
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
// kBackoff: the waiter is not on the critical path (drain, loader, Toeplitz copier) and sleeps between
// polls, which leaves issue slots - and power, the bench runs at the 1 kW cap - to the warps that work
template <int kBackoff = 0>
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, int tag) {
    if (mbar_try_wait(bar, parity)) return;
    const unsigned long long t0 = globaltimer_ns();
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (kBackoff > 0) __nanosleep(kBackoff);
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
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            int c3, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
        ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, int c0, int c1, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                 ::"l"(map), "r"(c0), "r"(c1), "r"(src) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, int c0, int c1, int c2, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                 ::"l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(src) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
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
// one MMA: D (+)= A * B; the descriptors arrive as their low words plus the constant upper words
// (single-thread form: the caller is the one elected thread of the issuer warp)
__device__ __forceinline__ void umma_f16_ss_1t(uint32_t d, uint32_t a_lo32, uint32_t b_lo32, uint32_t a_upper,
                                               uint32_t b_upper, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 a0, b0;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "mov.b64 a0, {%1, %3};\n\t"
        "mov.b64 b0, {%2, %4};\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a0, b0, %5, p;\n\t}"
        ::"r"(d), "r"(a_lo32), "r"(b_lo32), "r"(a_upper), "r"(b_upper), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit_1t(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(ok));
    return ok != 0;
}
__device__ __forceinline__ void umma_commit_elect(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
        ::"r"(bar) : "memory");
}
// exponent e with max|x| * 2^e in [2^12, 2^13) (0 for an all-zero, NaN or Inf frame)
__device__ __forceinline__ int frame_scale_exp_bits(uint32_t b) {
    const int ex = (int)((b >> 23) & 0xffu);
    if (ex == 0 || ex == 255) return 0;
    return max(-100, min(100, 12 - (ex - 127)));       // the scale itself must stay a normal float
}
__device__ __forceinline__ int frame_scale_exp(const uint32_t *max_bits) { return frame_scale_exp_bits(__ldcg(max_bits)); }
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((uint32_t)(127 + e) << 23); }
// two floats -> packed f16x2 (first argument in the LOW half)
__device__ __forceinline__ uint32_t pack_f16x2(float lo_elem, float hi_elem) {
    uint32_t d;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi_elem), "f"(lo_elem));
    return d;
}
// x0, x1 -> packed fp16 hi parts and packed fp16 residuals
__device__ __forceinline__ void split_pair(float x0, float x1, uint32_t &hi, uint32_t &lo) {
    hi = pack_f16x2(x0, x1);
    const float2 hf = __half22float2(*reinterpret_cast<const __half2 *>(&hi));
    lo = pack_f16x2(__fsub_rn(x0, hf.x), __fsub_rn(x1, hf.y));
}
// tcgen05.ld is asynchronous: its destination registers are only valid after tcgen05.wait::ld.
// Load and wait are one statement, so the compiler cannot place any use in between.
__device__ __forceinline__ void tmem_ld32_pair(uint32_t taddr_a, uint32_t taddr_b, uint32_t (&r)[32],
                                               uint32_t (&s)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%64];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, "
        "%48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%65];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
          "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "=r"(s[4]), "=r"(s[5]), "=r"(s[6]),
          "=r"(s[7]), "=r"(s[8]), "=r"(s[9]), "=r"(s[10]), "=r"(s[11]), "=r"(s[12]), "=r"(s[13]),
          "=r"(s[14]), "=r"(s[15]), "=r"(s[16]), "=r"(s[17]), "=r"(s[18]), "=r"(s[19]),
          "=r"(s[20]), "=r"(s[21]), "=r"(s[22]), "=r"(s[23]), "=r"(s[24]), "=r"(s[25]),
          "=r"(s[26]), "=r"(s[27]), "=r"(s[28]), "=r"(s[29]), "=r"(s[30]), "=r"(s[31])
        : "r"(taddr_a), "r"(taddr_b)
        : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

__device__ __forceinline__ void st_shared_b32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Shared-memory matrix descriptors (cute::UMMA::SmemDescriptor):
//   bits [0,14) start address >> 4    [16,30) leading byte offset >> 4    [32,46) stride byte
//   offset >> 4    [46,48) version = 1    [61,64) layout type (0 none, 2 SWIZZLE_128B)
// Toeplitz array (K-major, no swizzle), COMPACT: the operand rows are indexed by the REVERSED output
// n' = 127 - n, so T'[n'][k] = w[k + n' - 127] depends on k + n' only and the K half 1 of row n' is
// the K half 0 of row n' + 8: one 16-byte chunk per row, C[r][e] = w[r + e - 127], 8-row groups at
// SBO = 128 and the second K half at LBO = 128 (the core matrices overlap in memory).
constexpr uint32_t kToepLowLbo = (128u >> 4) << 16;
constexpr uint32_t kToepUpper = (128u >> 4) | (1u << 14);
// pass-1 data (MN-major, SWIZZLE_128B): x-block of 64 at LBO = 4096 (32 rows x 128 B), 8-row
// k group at SBO = 1024
constexpr uint32_t kData1LowLbo = ((128u * kRowsPerStage1) >> 4) << 16;
constexpr uint32_t kData1Upper = (1024u >> 4) | (1u << 14) | (2u << 29);
// pass-2 data (K-major, SWIZZLE_128B): 8-row group at SBO = 1024, LBO unused
constexpr uint32_t kData2LowLbo = 1u << 16;
constexpr uint32_t kData2Upper = (1024u >> 4) | (1u << 14) | (2u << 29);
// Instruction descriptor (cute::UMMA::InstrDescriptor), kind::f16: F16 operands (format 0),
// D = F32 (bit 4), B MN-major (bit 16), N >> 3 at bits [17,23), M >> 4 at bits [24,29)
__host__ __device__ constexpr uint32_t instr_desc_f16(int M, int N, int b_mn) {
    return (1u << 4) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__host__ __device__ __forceinline__ int fold_row_u(int i, int n) {
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

// unit -> (x0, y0, first level, end level).  Pass 1: single levels, longest first.  Pass 2 (DoG):
// level groups that OVERLAP by one level (the first level of group g + 1 is computed by group g
// too), so every DoG slice has both its levels inside one unit and nothing is parked in memory.
struct Unit { int x0, y0, lb, le; };
__device__ __forceinline__ Unit unit_of(int tx, int ty, int g, const UmmaArgs &a, const LevelTable &tbl, int mode) {
    Unit r;
    r.x0 = tx * kUT;
    r.y0 = ty * kUT;
    if (a.by_order) {
        r.lb = tbl.order[g];
        r.le = r.lb + 1;
    } else {
        r.lb = tbl.group_begin[g];
        r.le = tbl.group_begin[g + 1] + ((mode == kModeDog && g + 1 < tbl.n_groups) ? 1 : 0);
    }
    return r;
}
__device__ __forceinline__ Unit decode_unit(int u, const UmmaArgs &a, const LevelTable &tbl, int mode) {
    const int t = u / a.tiles_x;
    return unit_of(u % a.tiles_x, t % a.tiles_y, t / a.tiles_y, a, tbl, mode);
}
// Round robin without a schedule (pass 1: a unit per level): unit blockIdx.x + i * gridDim.x as (tile x, tile y,
// group), advanced by carries instead of three integer divisions per unit on the issuing thread's critical path
struct UnitWalk {
    int tx, ty, g, dx, dy, dg;
    __device__ __forceinline__ explicit UnitWalk(const UmmaArgs &a) {
        int u = blockIdx.x;
        tx = u % a.tiles_x; u /= a.tiles_x; ty = u % a.tiles_y; g = u / a.tiles_y;
        u = gridDim.x;
        dx = u % a.tiles_x; u /= a.tiles_x; dy = u % a.tiles_y; dg = u / a.tiles_y;
    }
    __device__ __forceinline__ void advance(const UmmaArgs &a) {
        tx += dx; ty += dy; g += dg;
        if (tx >= a.tiles_x) { tx -= a.tiles_x; ++ty; }
        if (ty >= a.tiles_y) { ty -= a.tiles_y; ++g; }      // ty < 2 tiles_y: one carry
    }
};

struct SharedCtl {
    unsigned long long data_full[kMaxStages], data_empty[kMaxStages];
    unsigned long long toep_full[kMaxToepBuffers], toep_empty[kMaxToepBuffers];
    unsigned long long acc_full[2], acc_empty[2];
    uint32_t tmem_base;
    uint32_t pad[3];
    uint32_t box_hit[2][2][4];      // pass 2: [store round parity][column half][drain warp] ballots "above the threshold"
};
constexpr int kCtlBytes = 512;
static_assert(sizeof(SharedCtl) <= kCtlBytes, "control block");

template <int MODE, int kStagingBufs1>
__global__ void __launch_bounds__(kThreads, 1)
umma_pass_kernel(const UmmaArgs a, const __grid_constant__ LevelTable tbl,
                 const __grid_constant__ ToeplitzTable ttab, const __grid_constant__ CUtensorMap map_in,
                 const __grid_constant__ CUtensorMap map_out, const __grid_constant__ CUtensorMap map_aux,
                 const __grid_constant__ CUtensorMap map_cut) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    SharedCtl *ctl = reinterpret_cast<SharedCtl *>(smem_raw);
    unsigned char *toep = smem_raw + kCtlBytes;                               // [buffer 2][hi | lo]
    unsigned char *staging = smem_raw + a.staging_off;                   // [column half 2][16 KB box (x 2 in pass 1)]
    constexpr bool kRows = MODE == kModeRows;
    constexpr int NT = kRows ? kToepBuffers1 : kToepBuffers2;
    unsigned char *data = staging + (kRows ? staging_bytes1(kStagingBufs1) : kStagingBytes2);     // [stage][...]
    constexpr int kStageBytes = kRows ? kStageBytes1 : kStageBytes2;
    constexpr int kStepsPerStage = kRows ? kRowsPerStage1 / 16 : 4;                         // k-steps of 16 per data stage
    const int S = a.stages;

    // the shuffle makes the warp index provably warp-uniform: the role branches below are then uniform
    // control flow and the issuer's descriptor arithmetic can live in uniform registers
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;

    if (a.prof != nullptr && threadIdx.x == 0) atomicMin(a.prof + 16, globaltimer_ns());      // first CTA in
    if (threadIdx.x == 0) {
        if (smem_u32(smem_raw) & 1023u) __trap();                         // swizzled boxes need 1 KB alignment
        for (int s = 0; s < S; ++s) {
            mbar_init(smem_u32(&ctl->data_full[s]), 1);
            mbar_init(smem_u32(&ctl->data_empty[s]), 1);
        }
        for (int b = 0; b < NT; ++b) {
            mbar_init(smem_u32(&ctl->toep_full[b]), 1);
            mbar_init(smem_u32(&ctl->toep_empty[b]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&ctl->acc_full[b]), 1);
            mbar_init(smem_u32(&ctl->acc_empty[b]), kDrainWarps);
        }
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(smem_u32(&ctl->tmem_base), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // The CTA owns all 512 columns, so the allocation starts at TMEM address 0; using the literal
    // keeps every TMEM address of the issuer in uniform registers.
    if (*reinterpret_cast<volatile uint32_t *>(&ctl->tmem_base) != 0u) __trap();
    constexpr uint32_t tmem = 0u;

    if (warp == 0) {
        // ================= issuer (ONE elected thread runs the whole loop) =================
        // Every MMA is M = 128 x K = 16; the tensor pipe spends 64 cycles on it per 128 columns of N
        // (measured, tools/ubench_umma_ss.cu).
        uint32_t lvl_it = 0, sl = 0, sl_par = 0;            // data stage slot and its phase parity
        uint32_t tb = 0, tb_par = 0;                        // Toeplitz buffer and its phase parity
        RoleClock rc(a.prof != nullptr);
        if (a.prof != nullptr && lane == 0) {
            atomicMax(a.prof + 17, globaltimer_ns());      // last CTA reaches its issuer loop
            atomicMin(a.prof + 20, globaltimer_ns());      // first CTA reaches it
        }
        UnitWalk walk(a);
        if (elect_one())
        for (int ui = blockIdx.x; ui < a.n_sched; ui += gridDim.x, walk.advance(a)) {
            const int u = a.sched ? __ldg(a.sched + ui) : ui;
            if (u < 0) continue;
            const Unit un = a.sched ? decode_unit(u, a, tbl, MODE) : unit_of(walk.tx, walk.ty, walk.g, a, tbl, MODE);
            for (int level = un.lb; level < un.le; ++level, ++lvl_it) {
                const int rpad2 = 2 * tbl.lv[level].rpad;
                const int Kp = kUT + rpad2;
                const int n_k = Kp / 16;
                const int n_stage = (n_k + kStepsPerStage - 1) / kStepsPerStage;
                const uint32_t b = lvl_it & 1, par = (lvl_it >> 1) & 1;
                rc.lap(3);
                mbar_wait(smem_u32(&ctl->toep_full[tb]), tb_par, 1);
                rc.lap(0);
                mbar_wait(smem_u32(&ctl->acc_empty[b]), par ^ 1, 2);
                rc.lap(1);
                tc_fence_after();
                // low descriptor word of the Toeplitz window of k-step 0 (row 0); every k-step moves
                // the window down by 16 rows of 16 bytes = 16 descriptor units
                const uint32_t t_hi = smem_u32(toep + (size_t)tb * a.toep_bytes);
                // hi -> lo array (16 B per row)
                const uint32_t lo_off = (uint32_t)ttab.rows[level];
                const uint32_t win0 = (t_hi >> 4) | kToepLowLbo;
                const uint32_t d_main = tmem + b * 2 * kAccCols, d_small = d_main + kAccCols;
                for (int st = 0; st < n_stage; ++st) {
                    rc.lap(3);
                    mbar_wait(smem_u32(&ctl->data_full[sl]), sl_par, 3);
                    rc.lap(2);
                    tc_fence_after();
                    const uint32_t sbase = smem_u32(data + (size_t)sl * kStageBytes);
                    // pass 2: the last stage is shifted left so that it ends exactly at Kp (no read
                    // beyond the halo); k-step j then sits (16 j - first_k) columns into the box
                    const int first_k = kRows ? kRowsPerStage1 * st : (st == n_stage - 1 ? Kp - 64 : 64 * st);
                    const int j0 = kStepsPerStage * st;
                    const int j1 = min(n_k, j0 + kStepsPerStage);
                    if (!(a.debug & 8)) {
                        // Both passes: A = Toeplitz window (M = 128 outputs of the convolved axis), B = 16 inputs of
                        // the stage with the hi and the lo plane as ONE operand of N = 256 (pass 1: MN-major image
                        // rows, N = x; pass 2: K-major rows of R, N = y - the lo box sits 128 rows = 16 KB behind the
                        // hi box, exactly where rows 128..255 of a 256-row operand belong).  Per k-step
                        //     [main | small] += T_hi * [X_hi | X_lo]   (N = 256)      small += T_lo * X_hi   (N = 128)
                        // The narrow MMAs of a stage go first and the wide ones last: a commit holds the issuing
                        // thread ~250 cycles, and only what is queued behind it keeps the tensor pipe busy meanwhile
                        // (two N = 256 MMAs = 256 cycles).  The level's very first MMA must be the wide one that
                        // initialises both accumulators.
                        constexpr int b_mn = kRows ? 1 : 0;
                        const uint32_t i256 = instr_desc_f16(kUT, 2 * kUT, b_mn), i128 = instr_desc_f16(kUT, kUT, b_mn);
                        constexpr uint32_t b_upper = kRows ? kData1Upper : kData2Upper;
                        // byte offset of k-step j inside the stage: pass 1: 16 rows of 128 B; pass 2: 32 B along the row
                        auto b_desc = [&](int j) {
                            return kRows ? ((sbase + (uint32_t)(16 * j - first_k) * 128u) >> 4) | kData1LowLbo
                                         : ((sbase + (uint32_t)(16 * j - first_k) * 2u) >> 4) | kData2LowLbo;
                        };
                        if (j0 == 0) umma_f16_ss_1t(d_main, win0, b_desc(0), kToepUpper, b_upper, i256, 0u);
#pragma unroll
                        for (int q = 0; q < kStepsPerStage; ++q) {
                            const int j = j0 + q;
                            if (j < j1)
                                umma_f16_ss_1t(d_small, win0 + 16u * (uint32_t)j + lo_off, b_desc(j), kToepUpper, b_upper, i128, 1u);
                        }
#pragma unroll
                        for (int q = 0; q < kStepsPerStage; ++q) {
                            const int j = j0 + q;
                            if (j < j1 && j > 0)
                                umma_f16_ss_1t(d_main, win0 + 16u * (uint32_t)j, b_desc(j), kToepUpper, b_upper, i256, 1u);
                        }
                    }
                    // A commit stalls the issuing thread (~250 cycles, the tensor pipe runs dry behind
                    // it: tools/ubench_umma_commit.cu), hence stages of 4 k-steps in both passes.
                    // (Releasing stages in pairs - one commit per 8 k-steps - is slower in both passes: the
                    // later release costs more than the saved bubble.)
                    umma_commit_1t(smem_u32(&ctl->data_empty[sl]));
                    if (++sl == (uint32_t)S) { sl = 0; sl_par ^= 1u; }
                }
                umma_commit_1t(smem_u32(&ctl->toep_empty[tb]));
                umma_commit_1t(smem_u32(&ctl->acc_full[b]));
                if (++tb == (uint32_t)NT) { tb = 0; tb_par ^= 1u; }
            }
        }
        __syncwarp();
        if (lane != 0) rc.on = false;      // lane 0 is the elected thread in practice; only it reports
        rc.lap(3);
        rc.flush(a.prof, 0);
        if (rc.on) {
            atomicMax(a.prof + 18, globaltimer_ns());      // last issuer loop ends
            atomicMin(a.prof + 21, globaltimer_ns());      // first one ends
        }
        if (rc.on) {        // slowest / fastest CTA (issuer's whole life)
            const unsigned long long tot = rc.acc[0] + rc.acc[1] + rc.acc[2] + rc.acc[3];
            a.prof[32 + blockIdx.x] = tot;
            atomicMax(a.prof + 14, tot);
            atomicMin(a.prof + 15, tot);
        }
    } else if (warp == 1) {
        // ================= loader: one TMA box per data stage =================
        uint32_t sl = 0, sl_par = 1;                       // waits on `empty` start one phase ahead
        RoleClock rc(a.prof != nullptr);
        if (elect_one()) {
            for (int ui = blockIdx.x; ui < a.n_sched; ui += gridDim.x) {
            const int u = a.sched ? __ldg(a.sched + ui) : ui;
            if (u < 0) continue;
                const Unit un = decode_unit(u, a, tbl, MODE);
                for (int level = un.lb; level < un.le; ++level) {
                    const int rpad = tbl.lv[level].rpad;
                    const int Kp = kUT + 2 * rpad;
                    const int n_stage = (Kp / 16 + kStepsPerStage - 1) / kStepsPerStage;
                    for (int st = 0; st < n_stage; ++st, sl = (sl + 1 == (uint32_t)S ? 0 : sl + 1), sl_par ^= (sl == 0)) {
                        rc.lap(1);
                        mbar_wait<DOGBLOB_UMMA_BACKOFF>(smem_u32(&ctl->data_empty[sl]), sl_par, 7);
                        rc.lap(0);
                        const uint32_t bar = smem_u32(&ctl->data_full[sl]);
                        const uint32_t dst = smem_u32(data + (size_t)sl * kStageBytes);
                        if (a.debug & 1) { mbar_arrive(bar); continue; }
                        mbar_expect_tx(bar, kStageBytes);
                        if (kRows)      // X planes: {64 x, rows, x-block, hi | lo}; rows beyond the planes read as 0
                            tma_load_4d(dst, &map_in, 0, a.Py + un.y0 - rpad + kRowsPerStage1 * st, un.x0 / 64, 0, bar);
                        else            // R planes: {columns, rows of all levels, hi | lo}
                            tma_load_3d(dst, &map_in,
                                        a.Ppad + un.x0 - rpad + (st == n_stage - 1 ? Kp - 64 : 64 * st),
                                        level * a.Hp + un.y0, 0, bar);
                    }
                }
            }
        }
        __syncwarp();
        if (lane != 0) rc.on = false;
        rc.lap(1);
        rc.flush(a.prof, 4);
    } else if (warp == 2) {
        // ================= Toeplitz copier: prebuilt hi | lo arrays, bulk copies per level ========
        uint32_t tb = 0, tb_par = 1;                       // waits on `empty` start one phase ahead
        if (elect_one()) {
            for (int ui = blockIdx.x; ui < a.n_sched; ui += gridDim.x) {
            const int u = a.sched ? __ldg(a.sched + ui) : ui;
            if (u < 0) continue;
                const Unit un = decode_unit(u, a, tbl, MODE);
                for (int level = un.lb; level < un.le; ++level) {
                    mbar_wait<DOGBLOB_UMMA_BACKOFF>(smem_u32(&ctl->toep_empty[tb]), tb_par, 4);
                    const uint32_t bar = smem_u32(&ctl->toep_full[tb]);
                    const uint32_t dst = smem_u32(toep + (size_t)tb * a.toep_bytes);
                    if (++tb == (uint32_t)NT) { tb = 0; tb_par ^= 1u; }
                    if (a.debug & 16) { mbar_arrive(bar); continue; }
                    const uint32_t rows = (uint32_t)ttab.rows[level];
                    mbar_expect_tx(bar, rows * 32u);                              // hi + lo
                    bulk_copy_g2s(dst, a.toep + ttab.ofs[level], rows * 32u, bar);
                }
            }
        }
        __syncwarp();
    } else if (warp >= kDrainWarp0) {
        // ================= drain: accumulators -> (hi | lo rows) or (DoG slice) -> TMA store ========
        // warp = lane quarter q (TMEM lanes 32 q .. 32 q + 31 = output rows) x column half h
        const int dw = warp - kDrainWarp0;
        const int q = dw & 3, h = dw >> 2;
        // TMEM lane 32 q + lane; the Toeplitz operand's rows are reversed: lane m' = output row (pass 1) /
        // output column (pass 2) 127 - m'
        const int row = kUT - 1 - (32 * q + lane);                             // pass 1: output row inside the tile
        const bool store_leader = q == 0 && lane == 0;       // issues this half's TMA stores
        const int bar_a = 1 + 2 * h, bar_b = 2 + 2 * h;      // named barriers of this half (128 threads)
        uint32_t lvl_it = 0, round_it = 0;
        RoleClock rc(a.prof != nullptr && dw == 0 && lane == 0);
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(64 * h);
        const uint32_t stg = smem_u32(staging + (size_t)h * 16384 * kStagingBufs1);      // pass 1
        const uint32_t stg_row = stg + (uint32_t)row * 128u;
        const uint32_t swz = (uint32_t)(row & 7);
        // pass 2: one 32-row x 128-byte box per drain warp
        const uint32_t wbox = smem_u32(staging + (size_t)dw * 4096);
        const int frame_exp = frame_scale_exp(a.frame_max_bits);
        const float unscale_x = pow2f(-frame_exp);
        float prev[64];                                      // pass 2: previous level of this thread's outputs
        // pass 2: seeds of the previous chunk waiting for their list index (column bits, first index, key of column 0)
        uint32_t p_mask = 0u;
        int p_at = 0;
        unsigned long long p_key = 0ull;
        auto flush_seeds = [&]() {
            for (; p_mask != 0u; p_mask &= p_mask - 1u, ++p_at)
                if (p_at < a.flags.seed_cap)
                    a.flags.seeds[p_at] = p_key + (unsigned long long)(__ffs(p_mask) - 1);
        };
#pragma unroll
        for (int j = 0; j < 64; ++j) prev[j] = 0.f;
        for (int ui = blockIdx.x; ui < a.n_sched; ui += gridDim.x) {
            const int u = a.sched ? __ldg(a.sched + ui) : ui;
            if (u < 0) continue;
            const Unit un = decode_unit(u, a, tbl, MODE);
            for (int level = un.lb; level < un.le; ++level, ++lvl_it) {
                const uint32_t b = lvl_it & 1, par = (lvl_it >> 1) & 1;
                // exact (powers of two), applied one after the other so neither factor underflows
                const float unscale_t = pow2f(-ttab.tscale[level]);
                const uint32_t acc = lane_base + b * 2 * kAccCols;
                rc.lap(1);
                mbar_wait<DOGBLOB_UMMA_BACKOFF>(smem_u32(&ctl->acc_full[b]), par, 5);
                rc.lap(0);
                tc_fence_after();
                if (kRows) {
                    // ---- pass 1: v = level value in frame-scaled units -> fp16 hi | lo words ----
                    uint32_t hw[32], lw[32];                 // 64 columns: 32 packed pairs each
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t ra[32], rb[32];
                        tmem_ld32_pair(acc + 32 * c, acc + kAccCols + 32 * c, ra, rb);
#pragma unroll
                        for (int j = 0; j < 32; j += 2) {
                            const float v0 = __fmul_rn(__fadd_rn(__uint_as_float(ra[j]), __uint_as_float(rb[j])), unscale_t);
                            const float v1 = __fmul_rn(__fadd_rn(__uint_as_float(ra[j + 1]), __uint_as_float(rb[j + 1])), unscale_t);
                            split_pair(v0, v1, hw[16 * c + j / 2], lw[16 * c + j / 2]);
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(&ctl->acc_empty[b]));
                    rc.lap(2);
                    // Rounds through this half's two 16 KB staging boxes (alternating): hi plane, lo
                    // plane, and for tiles next to the left / right frame border the same rows with
                    // their columns REVERSED: the reflected halo columns of pass 2's input, stored next
                    // to the interior (column -1 - x <- x, column 2 W - 1 - x <- x).  One barrier per
                    // round: before it the leader waits until the PREVIOUS round's store has read its
                    // box, which frees that box for the next round.
                    const int rpad = tbl.lv[level].rpad;
                    const int xs0 = un.x0 + 64 * h;
                    const int right_w = rpad + (a.Wp - a.W);
                    const bool left = xs0 < rpad, right = xs0 + 64 > a.W - right_w && xs0 < a.W;
                    const bool right_tma = right && (a.W & 7) == 0 && xs0 + 64 <= a.W;    // no negative store coordinates
                    // the half that the frame's right edge cuts (W a multiple of 8, not of 64): its W - xs0 valid columns,
                    // reversed, are the FIRST halo columns - the reversed row is staged (xs0 + 64 - W) / 8 chunks further
                    // left and stored through a map that starts at column W and ends after W - xs0 columns
                    const bool right_cut = right && (a.W & 7) == 0 && xs0 + 64 > a.W && !left;
                    const int cut_chunks = right_cut ? (xs0 + 64 - a.W) >> 3 : 0;
                    const int n_rounds = (a.debug & 2) ? 0 : ((left || right_tma || right_cut) && !(a.debug & 64)) ? 4 : 2;
                    for (int rd = 0; rd < n_rounds; ++rd, ++round_it) {      // uniform per half
                        const uint32_t buf = kStagingBufs1 == 2 ? (round_it & 1u) : 0u;
                        const uint32_t dst = stg_row + buf * 16384u;
                        const bool lo_plane = rd & 1;
                        if (kStagingBufs1 == 1) {          // single box: the previous store must have read it
                            if (store_leader) bulk_wait_read();
                            named_bar(bar_b, 128);
                        }
                        if (rd < 2) {
#pragma unroll
                            for (int c = 0; c < 8; ++c) {
                                const uint32_t *w = lo_plane ? lw : hw;
                                st_shared_v4(dst + (((uint32_t)c ^ swz) << 4), w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
                            }
                        } else {
#pragma unroll
                            for (int c = 0; c < 8; ++c) {            // chunk c of the reversed row = chunk 7 - c, elements reversed
                                const uint32_t *w = lo_plane ? lw : hw;
                                const int at = c - cut_chunks;      // uniform; a cut half drops its first chunks (columns >= W)
                                if (at >= 0)
                                    st_shared_v4(dst + (((uint32_t)at ^ swz) << 4),
                                                 __byte_perm(w[4 * (7 - c) + 3], 0, 0x1032), __byte_perm(w[4 * (7 - c) + 2], 0, 0x1032),
                                                 __byte_perm(w[4 * (7 - c) + 1], 0, 0x1032), __byte_perm(w[4 * (7 - c)], 0, 0x1032));
                            }
                        }
                        fence_proxy_async_smem();
                        if (kStagingBufs1 == 2 && store_leader) bulk_wait_read();
                        named_bar(bar_a, 128);
                        if (store_leader && !(a.debug & 32)) {
                            const uint32_t src = stg + buf * 16384u;
                            const int yrow = level * a.Hp + un.y0;
                            if (rd < 2) {
                                tma_store_3d(&map_out, a.Ppad + xs0, yrow, lo_plane, src);
                            } else {
                                // map_aux starts at the first column right of the frame (column W)
                                if (left) tma_store_3d(&map_out, a.Ppad - xs0 - 64, yrow, lo_plane, src);
                                if (right_tma) tma_store_3d(&map_aux, a.W - xs0 - 64, yrow, lo_plane, src);
                                if (right_cut) tma_store_3d(&map_cut, 0, yrow, lo_plane, src);
                            }
                            bulk_commit();
                        }
                    }
                    if (right && (a.W & 7) == 0 && !right_tma && !right_cut && !(a.debug & (2 | 64))) {
                        // a frame narrower than a kernel radius, cut half that also feeds the left halo: element by
                        // element (widths that are not a multiple of 8: edge_halo_kernel mirrors the right halo)
                        __half *rrow = a.r_base + ((int64_t)level * a.Hp + un.y0 + row) * a.r_pitch + a.Ppad;
#pragma unroll
                        for (int pl = 0; pl < 2; ++pl) {
                            unsigned short *prow = reinterpret_cast<unsigned short *>(rrow + (int64_t)pl * a.r_plane);
                            const uint32_t *w = pl == 0 ? hw : lw;
#pragma unroll
                            for (int e = 0; e < 64; ++e) {
                                const int x = xs0 + e;
                                const unsigned short v = (unsigned short)((e & 1) ? (w[e >> 1] >> 16) : (w[e >> 1] & 0xffffu));
                                if (x >= a.W - right_w && x < a.W) prow[2 * a.W - 1 - x] = v;
                            }
                        }
                    }
                    rc.lap(3);
                } else {
                    // ---- pass 2: level value -> DoG slice against the previous level (registers) ----
                    // TMEM lane = output COLUMN x (reversed: lane m' is column 127 - m'), accumulator column = row y.
                    // The slices are written TRANSPOSED, D^T[slice][x][y] (like the FP32 engine's): a thread's 32
                    // accumulator columns are 128 contiguous bytes of row x of D^T, staged with 16-byte stores.
                    const bool emit = MODE == kModeLevels || level > un.lb;
                    const float sig = MODE == kModeDog && level > un.lb ? tbl.lv[level - 1].sigma_f32 : 0.f;
                    const int out_plane = MODE == kModeLevels ? level : level - 1;
                    // With a threshold (detection), a 32 x 32 box of the slice in which nothing exceeds it is
                    // not even stored: the extrema kernel reads blocks without a hit as -inf (HitFlags double
                    // as the validity map), so whatever that memory holds is never looked at.
                    const bool want_flags = MODE == kModeDog && a.flags.data != nullptr;
                    const bool may_skip = want_flags && !(a.debug & 512);
                    // the float after the threshold: e > thr  <=>  e >= thr_next (thr is not NaN; +inf never gets here)
                    const float thr_next = __uint_as_float(a.thr == 0.f ? 1u : a.thr > 0.f ? __float_as_uint(a.thr) + 1u : __float_as_uint(a.thr) - 1u);
                    const int xbox = un.x0 + 96 - 32 * q;        // first row of D^T in this warp's boxes
                    const int br = 31 - lane;                    // this thread's row inside the box
                    const bool row_in = xbox + br < a.W;
                    const uint32_t wbox_row = wbox + (uint32_t)br * 128u, bswz = (uint32_t)(br & 7);
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int ybase = un.y0 + 64 * h + 32 * c;      // first column of D^T in this box
                        bool hit = false;
                        uint32_t ra[32], rb[32];
                        tmem_ld32_pair(acc + 32 * c, acc + kAccCols + 32 * c, ra, rb);
                        if (c == 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(smem_u32(&ctl->acc_empty[b]));
                        }
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float v = __fmul_rn(__fmul_rn(__fadd_rn(__uint_as_float(ra[j]), __uint_as_float(rb[j])), unscale_t), unscale_x);
                            if (MODE == kModeDog) {
                                const float d = __fmul_rn(__fsub_rn(prev[32 * c + j], v), sig);
                                ra[j] = __float_as_uint(d);
                                prev[32 * c + j] = v;
                                hit = hit || d > a.thr;
                            } else {
                                ra[j] = __float_as_uint(v);
                            }
                        }
                        rc.lap(2);
                        if (MODE == kModeDog) flush_seeds();
                        if (emit && !(a.debug & 2)) {            // uniform per level
                            bool store = true;
                            uint32_t hit_rows = 0u;          // bit r: row r of the box has a value above the threshold
                            if (want_flags) {
                                // this warp's 32 rows x 32 columns of D^T: which of its four 8-row blocks hold a value
                                // above the threshold (rows right of the frame do not count)?
                                const uint32_t m = hit_rows = __brev(__ballot_sync(0xffffffffu, hit && row_in));
                                if (lane == 0) {
                                    const uint32_t word = ((m & 0xffu) ? 1u : 0u) | ((m & 0xff00u) ? 0x100u : 0u) |
                                                          ((m & 0xff0000u) ? 0x10000u : 0u) | ((m & 0xff000000u) ? 0x1000000u : 0u);
                                    *reinterpret_cast<uint32_t *>(a.flags.data +
                                        ((int64_t)out_plane * a.flags.col_blocks + ((un.y0 >> 5) + 2 * h + c)) * a.flags.row_blocks +
                                        (xbox >> 3)) = word;
                                }
                                if (may_skip) store = m != 0u;
                            }
                            if (store) {
                                // This warp's own 32 x 32 box (4 KB, swizzled like a 128-row box): no barrier with
                                // the other drain warps anywhere in this pass - a warp that stores or tests seeds
                                // does not hold up one that has nothing above the threshold.
                                if (lane == 0) bulk_wait_read();     // the warp's previous store has read the box
                                __syncwarp();
#pragma unroll
                                for (int k = 0; k < 8; ++k)
                                    st_shared_v4(wbox_row + (((uint32_t)k ^ bswz) << 4), ra[4 * k], ra[4 * k + 1], ra[4 * k + 2], ra[4 * k + 3]);
                                fence_proxy_async_smem();
                                __syncwarp();
                                if (lane == 0 && !(a.debug & (32 | 4096))) {
                                    tma_store_2d(&map_out, ybase, out_plane * a.Wp + xbox, wbox);
                                    bulk_commit();
                                }
                            }
                            if (a.flags.seeds != nullptr && hit_rows != 0u && !(a.debug & 1024)) {      // uniform per warp; after the store: the box is read meanwhile
                                // Seeds: values above the threshold that no in-slice neighbour KNOWN HERE exceeds
                                // (same row of D^T: this thread's other columns of the chunk; rows above / below: the
                                // adjacent lanes; everything else, and everything outside the frame, counts as
                                // -inf).  A lane without a neighbour lane gets its own row maximum back from the
                                // shuffle, which a row maximum passes by construction.
                                const int nvalid = row_in ? a.H - ybase : 0;         // elements j < nvalid are inside
                                if (nvalid < 32) {                                    // frame edge: rare
#pragma unroll
                                    for (int j = 0; j < 32; ++j)
                                        if (j >= nvalid) ra[j] = 0xff800000u;        // -inf
                                }
                                // e > thr and e >= its neighbours  <=>  e >= max(neighbours, the float after thr):
                                // three 3-input maxima, two shuffles and one comparison per element
                                uint32_t seedmask = 0u;
#pragma unroll
                                for (int j = 0; j < 32; ++j) {
                                    const float e = __uint_as_float(ra[j]);
                                    const float l = j > 0 ? __uint_as_float(ra[j - 1]) : -INFINITY;
                                    const float r = j < 31 ? __uint_as_float(ra[j + 1]) : -INFINITY;
                                    const float mm = fmaxf(fmaxf(l, r), e);
                                    const float up = __shfl_up_sync(0xffffffffu, mm, 1);
                                    const float dn = __shfl_down_sync(0xffffffffu, mm, 1);
                                    const float t = fmaxf(fmaxf(up, dn), fmaxf(fmaxf(l, r), thr_next));
                                    if (e >= t) seedmask |= 1u << j;
                                }
                                if (seedmask != 0u && !(a.debug & 2048)) {
                                    // the list index comes back from L2 ~1 us later: the entries are written after the
                                    // next chunk's accumulator load and arithmetic (flush_seeds above)
                                    p_at = atomicAdd(a.flags.n_seeds, __popc(seedmask));
                                    p_mask = seedmask;
                                    p_key = ((unsigned long long)out_plane << 48) | ((unsigned long long)(xbox + br) << 24) |
                                            (unsigned long long)ybase;
                                }
                            }
                        }
                        rc.lap(3);
                    }
                }
            }
        }
        if (MODE == kModeDog) flush_seeds();
        if (kRows ? store_leader : lane == 0) bulk_wait_all();
        rc.lap(1);
        rc.flush(a.prof, 8);
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
    if (a.prof != nullptr && threadIdx.x == 0) atomicMax(a.prof + 19, globaltimer_ns());      // last CTA out
}

constexpr int kMaxParts = 256;          // partial maxima of frame_max_kernel (one per CTA)

// max |x| over the partial maxima of frame_max_kernel, as float bits (non-negative floats order like
// unsigned integers); every CTA of the consumer reduces the <= 256 words itself: no atomics, no memset
__device__ __forceinline__ uint32_t reduce_parts(const uint32_t *__restrict__ parts, int n_parts) {
    __shared__ uint32_t s_m[8];
    __shared__ uint32_t s_all;
    uint32_t m = (int)threadIdx.x < n_parts ? __ldcg(parts + threadIdx.x) : 0u;
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t a = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) a = max(a, s_m[i]);
        s_all = a;
    }
    __syncthreads();
    return s_all;
}

// Frame -> fp16 hi | lo planes [2][H + 2 Py][Wp] in frame-scaled units, reflected halo rows
// materialised (row r of the planes = frame row fold(r - Py)), pad columns x >= W zero.  Also
// publishes the frame's max |x| word for the passes that follow.
__global__ void __launch_bounds__(256)
prep_split_kernel(const float *__restrict__ img, int64_t pitch, int H, int W, int Wp, int Py,
                  const uint32_t *__restrict__ parts, int n_parts, uint32_t *__restrict__ max_bits,
                  __half *__restrict__ xp) {
    const uint32_t mbits = reduce_parts(parts, n_parts);
    if (blockIdx.x == 0 && threadIdx.x == 0) *max_bits = mbits;
    const float xscale = pow2f(frame_scale_exp_bits(mbits));
    const int rows = H + 2 * Py, groups = Wp / 8;
    const int64_t plane = (int64_t)rows * Wp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)rows * groups;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / groups), x = (int)(i % groups) * 8;
        const float *src = img + (int64_t)fold_row_u(r - Py, H) * pitch + x;
        float v[8];
        if (x + 8 <= W) {
            const float4 p = __ldg(reinterpret_cast<const float4 *>(src));
            const float4 s = __ldg(reinterpret_cast<const float4 *>(src) + 1);
            v[0] = p.x; v[1] = p.y; v[2] = p.z; v[3] = p.w; v[4] = s.x; v[5] = s.y; v[6] = s.z; v[7] = s.w;
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = x + k < W ? __ldg(src + k) : 0.f;
        }
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            split_pair(__fmul_rn(v[2 * k], xscale), __fmul_rn(v[2 * k + 1], xscale), hi[k], lo[k]);
        *reinterpret_cast<uint4 *>(xp + (int64_t)r * Wp + x) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4 *>(xp + plane + (int64_t)r * Wp + x) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
}

// per-CTA max |x| of the frame -> parts[blockIdx.x]; CTA 0 also resets the frame's counters
// (reset_counters_kernel folded in: one launch less in front of every frame)
__global__ void __launch_bounds__(256)
frame_max_kernel(const float *__restrict__ img, int64_t n4, uint32_t *__restrict__ parts, Counters *ctr, int *ctl) {
    __shared__ float s_m[8];
    if (blockIdx.x == 0 && ctr != nullptr) {
        if (threadIdx.x == 0) {
            Counters z = {};
            z.t_start = globaltimer_ns();
            *ctr = z;
        }
        if (threadIdx.x < 8) ctl[threadIdx.x] = 0;      // ticket, done, n_phases, ... of the pruning control block
    }
    float m = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(img) + i);
        m = fmaxf(fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))), m);
    }
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < 8; ++i) m = fmaxf(m, s_m[i]);
        // NaN compares false everywhere above: a NaN frame yields the max of its other pixels (scale only)
        parts[blockIdx.x] = m > 0.f ? __float_as_uint(m) : 0u;
    }
}

int toeplitz_rows(int rpad) { return kUT + 2 * rpad - 16 + kUT + 8; }
// one Toeplitz buffer in shared memory (hi + lo arrays of the widest level)
int toeplitz_buffer_bytes(int max_rpad, bool rows_pass) {
    (void)rows_pass;
    return (toeplitz_rows(max_rpad) * 32 + 127) / 128 * 128;
}
// control block + Toeplitz ring, rounded up to the 1 KB alignment of the swizzled boxes behind it
size_t staging_offset(int max_rpad, bool rows_pass) {
    const size_t ring = (size_t)(rows_pass ? kToepBuffers1 : kToepBuffers2) * toeplitz_buffer_bytes(max_rpad, rows_pass);
    return (kCtlBytes + ring + 1023) / 1024 * 1024;
}

constexpr size_t kSmemLimit = 227 * 1024;
int data_stages_for(int max_rpad, bool rows_pass, int staging_bufs) {
    const size_t fixed = staging_offset(max_rpad, rows_pass) + (rows_pass ? staging_bytes1(staging_bufs) : kStagingBytes2);
    const size_t per = rows_pass ? kStageBytes1 : kStageBytes2;
    if (fixed + 2 * per > kSmemLimit) return 0;
    return (int)std::min<size_t>(kMaxStages, (kSmemLimit - fixed) / per);
}

// pass 1: the second staging box per half is worth less than a fourth data stage (C2: 4 stages either way,
// 0.109 vs 0.116 ms with one box; C4: 0.526 ms with one box and 4 stages, 0.559 with two boxes and 3)
int staging_bufs_for(int max_rpad) {
    if (kStagingForce1 == 1 || kStagingForce1 == 2) return kStagingForce1;
    return data_stages_for(max_rpad, true, 2) >= 4 || data_stages_for(max_rpad, true, 1) < 4 ? 2 : 1;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);
EncodeTiledFn tensor_map_encoder() {
    static EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}
// SWIZZLE_128B tensor map; dims / strides (bytes, dims 1..) / box in elements
bool encode_map(CUtensorMap *map, CUtensorMapDataType type, int rank, const void *base, const cuuint64_t *dims,
                const cuuint64_t *strides, const cuuint32_t *box) {
    EncodeTiledFn fn = tensor_map_encoder();
    if (!fn) return false;
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return fn(map, type, (cuuint32_t)rank, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int persistent_ctas(int n_units) {
    static const int sms = [] {
        int dev = 0, n = 148;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n;
    }();
    return std::min(n_units, sms);
}

// DOGBLOB_UMMA_PROF (read once): per-role cycle counters of every launch, printed to stderr
bool umma_prof_enabled() {
    static const bool on = std::getenv("DOGBLOB_UMMA_PROF") != nullptr;
    return on;
}

// test tooling (tools/umma_masks.py sets it before every timed batch): re-read only while the
// variable exists when the library is first used, so production launches never call getenv
int umma_debug_mask() {
    static const bool present = std::getenv("DOGBLOB_UMMA_DEBUG") != nullptr;
    if (!present) return 0;
    const char *e = std::getenv("DOGBLOB_UMMA_DEBUG");
    return e ? std::atoi(e) : 0;
}

// Frame widths that are not a multiple of 8: the reflected halo right of the frame cannot be written with 16-byte
// chunks (the reflection shifts the columns by an odd distance), so the row pass leaves it out and this kernel
// mirrors it afterwards: column W + i <- column W - 1 - i for i < rpad(level) + Wp - W, one warp per row of both
// planes (rows = [hi | lo][level][Hp]).  It also overwrites the columns [W, w8) that the interior stores, clipped at
// the next 16-byte chunk, filled with pad-region outputs.
__global__ void __launch_bounds__(256)
edge_halo_kernel(__half *r, int64_t n_rows, int64_t pitch, int edge, int pad_w, int Hp, int L,
                 const __grid_constant__ LevelTable tbl) {
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (row >= n_rows) return;
    const int n = tbl.lv[(int)((row / Hp) % L)].rpad + pad_w;
    __half *p = r + row * pitch + edge;
    for (int i = threadIdx.x & 31; i < n; i += 32) p[i] = p[-1 - i];
}

template <int MODE>
cudaError_t launch_umma(UmmaArgs b, const LevelTable &tbl, const ToeplitzTable &ttab, int max_rpad,
                        const CUtensorMap &map_in, const CUtensorMap &map_out, const CUtensorMap &map_aux, const CUtensorMap &map_cut,
                        cudaStream_t st) {
    constexpr bool rows_pass = MODE == kModeRows;
    b.toep_bytes = toeplitz_buffer_bytes(max_rpad, rows_pass);
    b.staging_off = (int)staging_offset(max_rpad, rows_pass);
    const int staging_bufs = rows_pass ? staging_bufs_for(max_rpad) : 1;
    b.stages = data_stages_for(max_rpad, rows_pass, staging_bufs);
    if (b.stages < 2) return cudaErrorInvalidConfiguration;
    const size_t smem = (size_t)b.staging_off + (rows_pass ? staging_bytes1(staging_bufs) : kStagingBytes2) +
                        (size_t)b.stages * (rows_pass ? kStageBytes1 : kStageBytes2);
    static unsigned long long *d_prof = nullptr;
    const bool prof = umma_prof_enabled();
    // DOGBLOB_UMMA_DEBUG (timing experiments, results are garbage): 1 no data TMA, 2 drain without
    // staging / stores, 8 no MMAs, 16 no Toeplitz copies, 32 no TMA stores, 64 no halo column stores,
    // 512 every box stored (no skipping), 1024 no seed test, 2048 seed test without the list appends,
    // 4096 column pass stages its boxes but does not issue their TMA stores
    b.debug = umma_debug_mask();
    if (prof) {
        if (!d_prof) cudaMalloc(&d_prof, 256 * sizeof(unsigned long long));
        cudaMemsetAsync(d_prof, 0, 24 * sizeof(unsigned long long), st);
        cudaMemsetAsync(d_prof + 15, 0xff, 2 * sizeof(unsigned long long), st);
        cudaMemsetAsync(d_prof + 20, 0xff, 2 * sizeof(unsigned long long), st);
        b.prof = d_prof;
    }
    const int ctas = b.n_ctas > 0 ? b.n_ctas : persistent_ctas(b.n_units);
    if (staging_bufs == 2)
        umma_pass_kernel<MODE, rows_pass ? 2 : 1><<<ctas, kThreads, smem, st>>>(b, tbl, ttab, map_in, map_out, map_aux, map_cut);
    else
        umma_pass_kernel<MODE, 1><<<ctas, kThreads, smem, st>>>(b, tbl, ttab, map_in, map_out, map_aux, map_cut);
    if (prof) {
        unsigned long long h[256];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, d_prof, sizeof(h), cudaMemcpyDeviceToHost);
        static const char *names[16] = {
            "issuer  wait toeplitz", "issuer  wait acc free", "issuer  wait data", "issuer  issue+other",
            "loader  issue", "loader  wait stage free", "-", "-",
            "drain   wait+tmem ld", "drain   wait acc", "drain   math", "drain   staging+store",
            "-", "-", "-", "-"};
        fprintf(stderr, "umma mode %d, %d CTAs, %d stages, kilo-cycles per CTA:", MODE, ctas, b.stages);
        for (int i = 0; i < 16; ++i)
            if (names[i][0] != '-') fprintf(stderr, "\n   %-34s %8.1f", names[i], h[i] / 1e3 / ctas);
        fprintf(stderr, "\n   issuer total: slowest CTA %.1f, fastest %.1f\n", h[14] / 1e3, h[15] / 1e3);
        if (std::getenv("DOGBLOB_UMMA_PROF_CTAS")) {
            fprintf(stderr, "   issuer kilo-cycles per CTA:");
            for (int i = 0; i < ctas && i < 224; ++i) fprintf(stderr, " %.0f", h[32 + i] / 1e3);
            fprintf(stderr, "\n");
        }
        fprintf(stderr, "   timeline (us after the first CTA starts): issuer loops begin %.2f .. %.2f, end %.2f .. %.2f, last CTA exits %.2f\n",
                (h[20] - h[16]) / 1e3, (h[17] - h[16]) / 1e3, (h[21] - h[16]) / 1e3, (h[18] - h[16]) / 1e3, (h[19] - h[16]) / 1e3);
    }
    return cudaGetLastError();
}

}  // namespace

// The tensor-core passes need: both Toeplitz buffers, the drain staging and >= 2 data stages in
// shared memory; every halo column mirrored from inside the frame (one reflection).
bool umma_supported(const ConvGeometry &g) {
    return data_stages_for(g.max_rpad, true, 1) >= 2 && data_stages_for(g.max_rpad, false, 1) >= 2 &&
           g.W >= g.max_rpad + (g.Wp - g.W) && tensor_map_encoder() != nullptr;
}

UmmaLayout umma_layout(const ConvGeometry &g) {
    UmmaLayout l;
    l.Py = g.max_rpad;
    l.Ppad = (g.max_rpad + 63) / 64 * 64;
    l.Wq = g.Wp + 2 * l.Ppad;
    l.x_bytes = 2 * (size_t)(g.H + 2 * l.Py) * g.Wp * sizeof(__half);
    l.r_bytes = 2 * (size_t)g.L * g.Hp * l.Wq * sizeof(__half);
    return l;
}

// Toeplitz operand of every level, as the kernels want it in shared memory (compact form, see
// kToepUpper): per level `rows` = Kp - 16 + 128 + 8 rows of 8 taps, fp16 hi array then lo array,
// C[r][e] = w[r + e - 127]; taps scaled by 2^t so that the largest is in [512, 1024).  The window of
// k-step j (inputs 16 j .. 16 j + 15) starts at row 16 j; its row n' holds the taps of output
// n = 127 - n'.  taps: the plan's duplicated table (entry t = offset t - rpad).
void build_toeplitz(const LevelDesc *lv, int n_levels, const float2 *taps, std::vector<float> &out,
                    ToeplitzTable &tab) {
    out.clear();
    for (int i = 0; i < n_levels; ++i) {
        const int rpad = lv[i].rpad, rows = toeplitz_rows(rpad);
        tab.ofs[i] = (int)out.size();
        tab.rows[i] = rows;
        out.resize(out.size() + (size_t)rows * 8, 0.f);          // rows x (8 hi + 8 lo) halfs = rows x 8 floats
        const float2 *w = taps + lv[i].tap_ofs;
        float wmax = 0.f;
        for (int t = 0; t <= 2 * rpad; ++t) wmax = std::max(wmax, w[t].x);
        int tsc = 0;
        if (wmax > 0.f) { int ex; std::frexp(wmax, &ex); tsc = 10 - ex; }      // wmax * 2^tsc in [512, 1024)
        tab.tscale[i] = tsc;
        __half *hi = reinterpret_cast<__half *>(out.data() + tab.ofs[i]);
        __half *lo = hi + (size_t)rows * 8;
        for (int r = 0; r < rows; ++r)
            for (int e = 0; e < 8; ++e) {
                const int t = r + e - (kUT - 1);
                const float v = (t >= 0 && t <= 2 * rpad) ? std::ldexp(w[t].x, tsc) : 0.f;
                const __half h = __float2half_rn(v);
                hi[(size_t)r * 8 + e] = h;
                lo[(size_t)r * 8 + e] = __float2half_rn(v - __half2float(h));
            }
    }
}

cudaError_t configure_umma_kernels(int device) {
    int optin = 0;
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(umma_pass_kernel<kModeRows, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(umma_pass_kernel<kModeRows, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(umma_pass_kernel<kModeDog, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(umma_pass_kernel<kModeLevels, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
}

// frame -> max |x| -> fp16 hi | lo planes with reflected halo rows (d_x: umma_layout().x_bytes)
// d_max_bits: the frame's max word followed by kMaxParts partial words (umma_max_words() uint32 in all);
// bs (optional): the frame's counters are reset by the first kernel
cudaError_t launch_prep_umma(const ConvGeometry &g, const float *d_img, void *d_x, uint32_t *d_max_bits,
                             cudaStream_t st, const BlobSpace *bs) {
    const UmmaLayout l = umma_layout(g);
    const int64_t n4 = (int64_t)g.H * g.Wp / 4;
    const int parts = (int)std::min<int64_t>(kMaxParts, std::max<int64_t>(1, n4 / 1024));
    uint32_t *d_parts = d_max_bits + 1;
    frame_max_kernel<<<parts, 256, 0, st>>>(d_img, n4, d_parts, bs ? bs->ctr : nullptr,
                                            bs ? reinterpret_cast<int *>(bs->ctl) : nullptr);
    const int64_t items = (int64_t)(g.H + 2 * l.Py) * (g.Wp / 8);
    const int blocks = (int)std::min<int64_t>((items + 255) / 256, 148 * 8);
    prep_split_kernel<<<blocks, 256, 0, st>>>(d_img, g.Wp, g.H, g.W, g.Wp, l.Py, d_parts, parts, d_max_bits,
                                              reinterpret_cast<__half *>(d_x));
    return cudaGetLastError();
}
int umma_max_words() { return 1 + kMaxParts; }

// pass 1: X planes -> R planes (level rows in frame-scaled fp16 hi | lo, halo columns mirrored)
cudaError_t launch_row_pass_umma(const ConvGeometry &g, const void *d_x, void *d_r, const LevelTable &tbl,
                                 const ToeplitzTable &ttab, const float *d_toep, cudaStream_t st,
                                 const uint32_t *d_max_bits, int max_ctas) {
    const UmmaLayout l = umma_layout(g);
    UmmaArgs a{};
    a.tiles_x = g.Wp / kUT; a.tiles_y = g.Hp / kUT;
    a.by_order = 1;                       // independent levels: finest units, longest first
    a.n_units = a.tiles_x * a.tiles_y * tbl.n_levels;
    a.n_sched = a.n_units;
    a.n_ctas = max_ctas > 0 ? std::min(max_ctas, a.n_units) : 0;
    a.H = g.H; a.W = g.W; a.Hp = g.Hp; a.Wp = g.Wp; a.Py = l.Py; a.Ppad = l.Ppad;
    a.r_pitch = l.Wq; a.r_plane = (int64_t)g.L * g.Hp * l.Wq;
    a.r_base = reinterpret_cast<__half *>(d_r);
    a.frame_max_bits = d_max_bits; a.toep = d_toep;
    CUtensorMap map_in, map_out, map_aux, map_cut;
    const int xrows = g.H + 2 * l.Py;
    {   // X planes as {64 x, rows, x-block, hi | lo}; box = 32 rows of one 128-column tile, both planes
        const cuuint64_t dims[4] = {64, (cuuint64_t)xrows, (cuuint64_t)(g.Wp / 64), 2};
        const cuuint64_t strides[3] = {(cuuint64_t)g.Wp * 2, 128, (cuuint64_t)xrows * g.Wp * 2};
        const cuuint32_t box[4] = {64, kRowsPerStage1, 2, 2};
        if (!encode_map(&map_in, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, d_x, dims, strides, box))
            return cudaErrorInvalidValue;
    }
    const int w8 = (g.W + 7) & ~7;
    {   // R planes as {columns up to the end of the last valid 16-byte chunk, rows of all levels, hi | lo}: stores
        // beyond are clipped.  The clip must not fall INSIDE a chunk: other CTAs write the halo columns next to
        // the frame at the same time, and a partially clipped chunk proved not to be a byte-exact write under
        // that race (tools/stress_engines.py, 725 x 898).  The up to 7 halo columns [W, w8) this leaves wrong
        // are rewritten by edge_halo_kernel below, together with the rest of the right halo.
        const cuuint64_t dims[3] = {(cuuint64_t)(l.Ppad + w8), (cuuint64_t)g.L * g.Hp, 2};
        const cuuint64_t strides[2] = {(cuuint64_t)l.Wq * 2, (cuuint64_t)a.r_plane * 2};
        const cuuint32_t box[3] = {64, 128, 1};
        if (!encode_map(&map_out, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, d_r, dims, strides, box))
            return cudaErrorInvalidValue;
    }
    map_aux = map_out;
    if ((g.W & 7) == 0) {   // right halo view: starts at the first column behind the frame (16-byte aligned)
        const cuuint64_t dims[3] = {(cuuint64_t)(l.Wq - l.Ppad - g.W), (cuuint64_t)g.L * g.Hp, 2};
        const cuuint64_t strides[2] = {(cuuint64_t)l.Wq * 2, (cuuint64_t)a.r_plane * 2};
        const cuuint32_t box[3] = {64, 128, 1};
        if (!encode_map(&map_aux, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
                        reinterpret_cast<__half *>(d_r) + l.Ppad + g.W, dims, strides, box))
            return cudaErrorInvalidValue;
    }
    map_cut = map_out;
    if ((g.W & 7) == 0 && (g.W & 63) != 0) {   // the half tile that the right edge cuts: its W % 64 mirrored columns behind the frame
        const cuuint64_t dims[3] = {(cuuint64_t)(g.W & 63), (cuuint64_t)g.L * g.Hp, 2};
        const cuuint64_t strides[2] = {(cuuint64_t)l.Wq * 2, (cuuint64_t)a.r_plane * 2};
        const cuuint32_t box[3] = {64, 128, 1};
        if (!encode_map(&map_cut, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
                        reinterpret_cast<__half *>(d_r) + l.Ppad + g.W, dims, strides, box))
            return cudaErrorInvalidValue;
    }
    const cudaError_t err = launch_umma<kModeRows>(a, tbl, ttab, g.max_rpad, map_in, map_out, map_aux, map_cut, st);
    if (err != cudaSuccess || w8 == g.W) return err;
    const int64_t n_rows = 2 * (int64_t)g.L * g.Hp;
    edge_halo_kernel<<<(unsigned)((n_rows + 7) / 8), 256, 0, st>>>(a.r_base, n_rows, a.r_pitch, l.Ppad + g.W, g.Wp - g.W, g.Hp, g.L, tbl);
    return cudaGetLastError();
}

// pass 2: R planes -> transposed DoG slices D^T [L - 1][Wp][Hp] (levels = true: the levels themselves, [L][Wp][Hp])
cudaError_t launch_col_pass_umma(const ConvGeometry &g, const void *d_r, float *d_out, const LevelTable &tbl,
                                 const ToeplitzTable &ttab, const float *d_toep, cudaStream_t st,
                                 const uint32_t *d_max_bits, bool levels, const int *d_sched, int sched_slots,
                                 int sched_ctas, float threshold, HitFlags flags) {
    const UmmaLayout l = umma_layout(g);
    UmmaArgs a{};
    a.tiles_x = g.Wp / kUT; a.tiles_y = g.Hp / kUT;
    a.by_order = 0;
    a.n_units = a.tiles_x * a.tiles_y * tbl.n_groups;
    a.sched = d_sched; a.n_sched = d_sched ? sched_slots * sched_ctas : a.n_units;
    a.n_ctas = d_sched ? sched_ctas : 0;
    a.flags = levels ? HitFlags{} : flags;
    a.thr = threshold;
    a.H = g.H; a.W = g.W; a.Hp = g.Hp; a.Wp = g.Wp; a.Py = l.Py; a.Ppad = l.Ppad;
    a.r_pitch = l.Wq; a.r_plane = (int64_t)g.L * g.Hp * l.Wq;
    a.frame_max_bits = d_max_bits; a.toep = d_toep;
    CUtensorMap map_in, map_out;
    {   // R planes as {columns, rows of all levels, hi | lo}; box = 128 rows x 64 columns of both planes
        const cuuint64_t dims[3] = {(cuuint64_t)l.Wq, (cuuint64_t)g.L * g.Hp, 2};
        const cuuint64_t strides[2] = {(cuuint64_t)l.Wq * 2, (cuuint64_t)a.r_plane * 2};
        const cuuint32_t box[3] = {64, 128, 2};
        if (!encode_map(&map_in, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, d_r, dims, strides, box))
            return cudaErrorInvalidValue;
    }
    {   // transposed output planes D^T {H valid columns (y), rows x of all planes}; box = 32 rows x 32 floats (one per drain warp)
        const cuuint64_t dims[2] = {(cuuint64_t)g.H, (cuuint64_t)g.L * g.Wp};
        const cuuint64_t strides[1] = {(cuuint64_t)g.Hp * 4};
        const cuuint32_t box[2] = {32, 32};
        if (!encode_map(&map_out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d_out, dims, strides, box))
            return cudaErrorInvalidValue;
    }
    if (levels) return launch_umma<kModeLevels>(a, tbl, ttab, g.max_rpad, map_in, map_out, map_out, map_out, st);
    return launch_umma<kModeDog>(a, tbl, ttab, g.max_rpad, map_in, map_out, map_out, map_out, st);
}

}  // namespace dogblob
