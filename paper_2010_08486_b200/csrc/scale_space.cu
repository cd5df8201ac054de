// Separable Gaussian scale space + fused DoG for sm_100a.
//
// Replaces convolve_bank (pkg/src/dogblob/convolve.py:63-218) and dog_stack
// (pkg/src/dogblob/detector.py:117-126).  The reference kernels are exactly
// separable (k_i = w_i (x) w_i, scale_space.py:76-81), so each level is two 1-D
// correlations with the reflect ("edge sample repeated", period 2N) boundary of
// convolve.py:4,94.
//
// Both passes are the same register-tiled sliding-window correlation along the
// STRIDED axis of a row-major plane, so every global access is coalesced along
// the contiguous axis:
//   pass 1 (row_pass):      img[y][x]      -> T_i[x][y] = sum_k w_i[k] img[fold(y+k)][x]
//                           (written transposed through a shared-memory tile)
//   pass 2 (col_dog_pass):  T_i[x][y]      -> L_i^T[x][y] = sum_k w_i[k] T_i[fold(x+k)][y]
//                           D_i^T = f32(sigma_i) * (L_i^T - L_{i+1}^T)   (only D is stored)
// A thread owns 4 columns x kTY outputs (64 accumulators as 32 float2) and walks
// the kTY + 2r input rows once; the tap window slides through a register ring
// that is statically indexed by full unrolling.  FMAs are issued as packed
// fma.rn.f32x2 (FFMA2) so that loads and address arithmetic issue in the shadow
// of the FMA pipe.
#include <cstdlib>

#include "common.cuh"

namespace dogblob {

namespace {

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// Reflect boundary ("edge sample repeated", period 2n): folded row index of any integer.
__device__ __forceinline__ int fold_row(int i, int n) {
    const int period = 2 * n;
    int t = i % period;
    if (t < 0) t += period;
    return t < n ? t : period - 1 - t;
}

// Per-CTA table of folded row offsets (in elements) for input rows
// first_row .. first_row + count - 1; replaces per-step boundary arithmetic by one
// broadcast LDS.
__device__ __forceinline__ void stage_row_offsets(int *s_rows, int first_row, int count, int n_rows,
                                                  int pitch) {
    for (int i = threadIdx.x; i < count; i += blockDim.x)
        s_rows[i] = fold_row(first_row + i, n_rows) * pitch;
}

template <bool ADJACENT, bool NC = true>
__device__ __forceinline__ void load_row(const float *__restrict__ row, int lane, float (&v)[4]) {
    if (ADJACENT) {
        // NC = false: the frame may still be arriving while the kernel runs (streamed row
        // pass), so the read-only (non-coherent) path is not allowed
        float4 q;
        if (NC) q = __ldg(reinterpret_cast<const float4 *>(row) + lane);
        else q = __ldcg(reinterpret_cast<const float4 *>(row) + lane);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = __ldg(row + lane + 32 * c);
    }
}

// One sweep: acc[j][p] = sum_k w[k] * in[fold(out_row0 + j + k - R)][cols(p)], R = lv.rpad.
//
// The tap radius is padded with zeros to a multiple of 8 (R), so the sweep is exactly
// (2R + 16) / 16 chunks of 16 input rows and both ends are chunk aligned:
//   step s (input row out_row0 - R + s) feeds output j with tap[s - j], 0 <= s - j <= 2R
//   first chunk  : sub-step u feeds outputs j <= u          (136 FMA groups)
//   middle chunks: every sub-step feeds all 16 outputs      (256 each)
//   last chunk   : sub-step u feeds outputs j >= u          (136)
// so no FMA is spent on the triangular head and tail of the sliding window.  The tap
// window lives in a 16-entry ring that is statically indexed by full unrolling.
__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// `frontier`: this warp is the first of its CTA to touch new input rows (the warp with
// the highest row range); it pulls rows kL2Ahead steps ahead into L2 so that its
// register prefetch (kPrefetch rows) only has to cover L2 latency, not HBM latency.
constexpr int kL2Ahead = 16;

// one full chunk: 16 sub-steps, each feeds all 16 outputs
template <bool NC>
__device__ __forceinline__ void full_chunk(const float *__restrict__ in,
                                           const int *__restrict__ rows,
                                           const float2 *__restrict__ taps, int lane,
                                           float (&v)[kPrefetch][4], float2 (&ring)[kTY],
                                           float2 (&acc)[kTY][2], bool frontier) {
#pragma unroll
    for (int u = 0; u < kTY; ++u) {
        ring[u] = taps[u];
        const float2 a = make_float2(v[u % kPrefetch][0], v[u % kPrefetch][1]);
        const float2 b = make_float2(v[u % kPrefetch][2], v[u % kPrefetch][3]);
        load_row<true, NC>(in + rows[u], lane, v[u % kPrefetch]);
        if (frontier && (u & 3) == 0)     // 4 rows x 4 lines per request group
            prefetch_l2(in + rows[u + kL2Ahead + (lane >> 3)] + (lane & 7) * 16);
#pragma unroll
        for (int j = 0; j < kTY; ++j) {
            const float2 t = ring[(u - j + kTY) % kTY];
            acc[j][0] = ffma2(t, a, acc[j][0]);
            acc[j][1] = ffma2(t, b, acc[j][1]);
        }
    }
}

// v[] holds input rows 0 .. kPrefetch-1 of this sweep, loaded by the caller.
// Measured alternatives that did NOT help (identical results, tools/sweep_modes.py history):
// running the head and/or tail through the full-chunk code on zero taps (smaller code, no
// cold straight-line blocks, but 256 instead of 136 FMA groups: row pass +3..10 %), and
// 8 instead of 4 rows in flight during the head (+0 %): the FMA pipe, not the head's load
// latency or instruction fetch, sets the pace.
template <bool NC = true>
__device__ __forceinline__ void sweep(const float *__restrict__ in, const int *__restrict__ rows,
                                      int n_mid, const float2 *__restrict__ taps, int lane,
                                      float (&v)[kPrefetch][4], float2 (&acc)[kTY][2],
                                      bool frontier = false) {
    rows += kPrefetch;
    float2 ring[kTY];
    // ---- first chunk: sub-step u feeds outputs j <= u ----
#pragma unroll
    for (int u = 0; u < kTY; ++u) {
        ring[u] = taps[u];
        const float2 a = make_float2(v[u % kPrefetch][0], v[u % kPrefetch][1]);
        const float2 b = make_float2(v[u % kPrefetch][2], v[u % kPrefetch][3]);
        load_row<true, NC>(in + rows[u], lane, v[u % kPrefetch]);
#pragma unroll
        for (int j = 0; j <= u; ++j) {
            const float2 t = ring[u - j];
            if (j == u) {          // first contribution to output j: multiply, no accumulate
                acc[j][0] = make_float2(__fmul_rn(t.x, a.x), __fmul_rn(t.y, a.y));
                acc[j][1] = make_float2(__fmul_rn(t.x, b.x), __fmul_rn(t.y, b.y));
            } else {
                acc[j][0] = ffma2(t, a, acc[j][0]);
                acc[j][1] = ffma2(t, b, acc[j][1]);
            }
        }
    }
    taps += kTY;
    rows += kTY;
    // ---- middle chunks ----
    for (int chunk = 0; chunk < n_mid; ++chunk) {
        full_chunk<NC>(in, rows, taps, lane, v, ring, acc, frontier);
        taps += kTY;
        rows += kTY;
    }
    // ---- last chunk: sub-step u feeds outputs j >= u ----
    ring[0] = taps[0];
#pragma unroll
    for (int u = 0; u < kTY; ++u) {
        const float2 a = make_float2(v[u % kPrefetch][0], v[u % kPrefetch][1]);
        const float2 b = make_float2(v[u % kPrefetch][2], v[u % kPrefetch][3]);
        if (u + kPrefetch < kTY) load_row<true, NC>(in + rows[u], lane, v[u % kPrefetch]);
#pragma unroll
        for (int j = u; j < kTY; ++j) {
            const float2 t = ring[(u - j + kTY) % kTY];
            acc[j][0] = ffma2(t, a, acc[j][0]);
            acc[j][1] = ffma2(t, b, acc[j][1]);
        }
    }
}

// n float2 entries global -> shared without register staging (LDGSTS, 16 bytes each; n is
// even and both sides are 16-byte aligned); completion via cp_async_wait_all
__device__ __forceinline__ void stage_taps_async(float2 *s_taps, const float2 *__restrict__ g_taps,
                                                 int n) {
    for (int i = 2 * threadIdx.x; i < n; i += 2 * blockDim.x) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(s_taps + i);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(g_taps + i));
    }
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ int table_len(const LevelDesc &lv) { return 2 * lv.rpad + kTY; }

// ---- pass 1: correlate along y, store transposed ------------------------------
// The 128 x 128 output tile is transposed through shared memory with 16-byte accesses on
// both sides: element (x, y) lives at x * 128 + (((y >> 2) ^ (x >> 2)) & 31) * 4 + (y & 3).
// A thread owns 4 adjacent columns x = 4 lane + c and 16 consecutive y, so it writes
// STS.128 whose 16-byte bank group is (const ^ lane) -> conflict free per quarter warp;
// rows are read back as permuted 16-byte groups (conflict free) and stored with
// fully coalesced STG.128.
__device__ __forceinline__ int tile_index(int x, int y4) {        // y4 = y / 4
    return x * kTileRows + (((y4 ^ (x >> 2)) & 31) << 2);
}

// STREAMED: the frame is still being copied in (row chunks on another stream, each followed by
// a copy of the gate word: gate.base + k once chunks 0..k-1 are resident).  Tile rows are the
// slowest grid index, so early CTAs need early chunks only; a CTA waits for the last image row
// it reads.  The kernel must not be launched unless the copies WILL be issued (it spins).
template <bool STREAMED>
__global__ void __launch_bounds__(kConvThreads, 2)
row_pass_kernel(const float *__restrict__ img, int64_t img_pitch, int H,
                float *__restrict__ out_t, int64_t out_pitch, int64_t out_plane,
                const __grid_constant__ LevelTable tbl, const float2 *__restrict__ g_taps,
                int max_table, RowGate gate) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *tile = reinterpret_cast<float *>(smem_raw);                       // [128 x][128 y]
    float2 *s_taps = reinterpret_cast<float2 *>(tile + kTileCols * kTileRows);
    int *s_rows = reinterpret_cast<int *>(s_taps + max_table);

    const int level = tbl.order[STREAMED ? blockIdx.y : blockIdx.z];
    const LevelDesc lv = tbl.lv[level];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int col0 = blockIdx.x * kTileCols;            // x
    const int row0 = (STREAMED ? blockIdx.z : blockIdx.y) * kTileRows;   // y
    if (STREAMED) {
        // last image row this tile touches (reflection folds rows below 0 upwards)
        const int need_row = lv.rpad >= H ? H - 1
                                          : min(H - 1, max(row0 + kTileRows - 1 + lv.rpad, lv.rpad - row0 - 1));
        const int need = need_row / gate.rows_per_chunk + 1;
        if (threadIdx.x == 0) {
            while (*(const volatile int *)gate.word - gate.base < need) __nanosleep(200);
            __threadfence();
            // the frame's compute clock starts when its first tile has its rows
            if ((blockIdx.x | blockIdx.y | blockIdx.z) == 0 && gate.t_start) *gate.t_start = globaltimer_ns();
        }
        __syncthreads();
    }
    // everything with memory latency is issued before the barrier: taps (async copy) and
    // the first input rows of this warp (offsets folded directly, the table is not ready yet)
    stage_taps_async(s_taps, g_taps + lv.tap_ofs, table_len(lv));
    float v[kPrefetch][4];
#pragma unroll
    for (int p = 0; p < kPrefetch; ++p)
        load_row<true, !STREAMED>(img + col0 + (int64_t)fold_row(row0 + warp * kTY - lv.rpad + p, H) * img_pitch,
                                  lane, v[p]);
    stage_row_offsets(s_rows, row0 - lv.rpad, kTileRows + 2 * lv.rpad + kPrefetch, H, (int)img_pitch);
    cp_async_wait_all();
    __syncthreads();

    float2 acc[kTY][2];
    sweep<!STREAMED>(img + col0, s_rows + warp * kTY, lv.n_mid, s_taps, lane, v, acc);

#pragma unroll
    for (int q = 0; q < kTY / 4; ++q) {                 // four consecutive y per store
        const int y4 = warp * (kTY / 4) + q;
        const int j = 4 * q;
        *reinterpret_cast<float4 *>(&tile[tile_index(4 * lane + 0, y4)]) =
            make_float4(acc[j][0].x, acc[j + 1][0].x, acc[j + 2][0].x, acc[j + 3][0].x);
        *reinterpret_cast<float4 *>(&tile[tile_index(4 * lane + 1, y4)]) =
            make_float4(acc[j][0].y, acc[j + 1][0].y, acc[j + 2][0].y, acc[j + 3][0].y);
        *reinterpret_cast<float4 *>(&tile[tile_index(4 * lane + 2, y4)]) =
            make_float4(acc[j][1].x, acc[j + 1][1].x, acc[j + 2][1].x, acc[j + 3][1].x);
        *reinterpret_cast<float4 *>(&tile[tile_index(4 * lane + 3, y4)]) =
            make_float4(acc[j][1].y, acc[j + 1][1].y, acc[j + 2][1].y, acc[j + 3][1].y);
    }
    __syncthreads();
    float *dst = out_t + (int64_t)level * out_plane + (int64_t)col0 * out_pitch + row0;
#pragma unroll 4
    for (int i = threadIdx.x; i < kTileCols * (kTileRows / 4); i += kConvThreads) {
        const int xl = i >> 5, y4 = i & 31;             // one warp = one x row, 512 B
        const float4 q = *reinterpret_cast<const float4 *>(&tile[tile_index(xl, y4)]);
        reinterpret_cast<float4 *>(dst + (int64_t)xl * out_pitch)[y4] = q;
    }
}

// ---- pass 2: correlate along x (rows of the transposed planes), fused DoG ------
// grid.z = level group g; the CTA walks levels [group_begin[g], group_begin[g+1])
// keeping the previous level's outputs in shared memory (thread private slots) and emits
// D_i = f32(sigma_i) (L_i - L_{i+1}) for every pair inside the group, so no level of
// the group reaches memory.  Only the two levels at a group boundary are parked in
// `edge` planes (first level of group g -> edge[2g], last level -> edge[2g+1]);
// edge_dog_kernel turns each boundary pair into the one missing slice.
// The tap tables of the whole group and the folded row offsets are staged once, so the
// level loop has no barrier: the 8 warps of a CTA drift apart and their epilogues
// (DoG, stores) overlap the FMA work of the others.
template <bool DOG>
__global__ void __launch_bounds__(kConvThreads, 2)
col_pass_kernel(const float *__restrict__ rows_t, int64_t pitch, int64_t plane, int n_rows,
                float *__restrict__ out, float *__restrict__ edge,
                const __grid_constant__ LevelTable tbl, const float2 *__restrict__ g_taps,
                int max_rpad, unsigned frontier_warps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2 *s_prev = reinterpret_cast<float2 *>(smem_raw);                    // [kTY*2][256]
    float2 *s_taps0 = s_prev + (DOG ? kTY * 2 * kConvThreads : 0);            // whole group
    const int n_groups = tbl.n_groups;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int col0 = blockIdx.x * kTileCols;
    const int row0 = blockIdx.y * kTileRows + warp * kTY;
    const int g = blockIdx.z;
    const int lev_begin = tbl.group_begin[g];
    const int lev_end = tbl.group_begin[g + 1];
    const int tap_base = tbl.lv[lev_begin].tap_ofs;
    const int tap_count = tbl.lv[lev_end - 1].tap_ofs + table_len(tbl.lv[lev_end - 1]) - tap_base;
    int *s_rows = reinterpret_cast<int *>(s_taps0 + tap_count);
    const int64_t tile_ofs = (int64_t)row0 * pitch + col0;
    stage_taps_async(s_taps0, g_taps + tap_base, tap_count);
    // folded offsets of every input row any level of this CTA can touch
    stage_row_offsets(s_rows, (int)blockIdx.y * kTileRows - max_rpad,
                      kTileRows + 2 * max_rpad + kPrefetch + kL2Ahead + 4, n_rows, (int)pitch);
    cp_async_wait_all();
    __syncthreads();                                         // row table + taps visible

    float v[kPrefetch][4];
    {
        const LevelDesc lv0 = tbl.lv[lev_begin];
        const float *in = rows_t + (int64_t)lev_begin * plane + col0;
        const int *rows = s_rows + warp * kTY + (max_rpad - lv0.rpad);
#pragma unroll
        for (int p = 0; p < kPrefetch; ++p) load_row<true>(in + rows[p], lane, v[p]);
    }
    for (int level = lev_begin; level < lev_end; ++level) {
        const LevelDesc lv = tbl.lv[level];
        const float2 *s_taps = s_taps0 + (lv.tap_ofs - tap_base);
        const float *in = rows_t + (int64_t)level * plane + col0;
        const int *rows = s_rows + warp * kTY + (max_rpad - lv.rpad);
        float2 acc[kTY][2];
        sweep(in, rows, lv.n_mid, s_taps, lane, v, acc, (frontier_warps >> warp) & 1u);
        if (!DOG) {
            float *dst = out + (int64_t)level * plane + tile_ofs;
#pragma unroll
            for (int j = 0; j < kTY; ++j)
                reinterpret_cast<float4 *>(dst + (int64_t)j * pitch)[lane] =
                    make_float4(acc[j][0].x, acc[j][0].y, acc[j][1].x, acc[j][1].y);
        } else {
            const bool park_first = (level == lev_begin) && g > 0;
            const bool park_last = (level == lev_end - 1) && g < n_groups - 1;
#pragma unroll 1
            for (int e = 0; e < 2; ++e) {        // rare path: kept rolled to save registers
                if (e == 0 ? !park_first : !park_last) continue;
                float *dst = edge + (int64_t)(2 * g + e) * plane + tile_ofs;
#pragma unroll
                for (int j = 0; j < kTY; ++j) {
                    reinterpret_cast<float4 *>(dst)[lane] =
                        make_float4(acc[j][0].x, acc[j][0].y, acc[j][1].x, acc[j][1].y);
                    dst += pitch;
                }
            }
            if (level > lev_begin) {
                const float s = tbl.lv[level - 1].sigma_f32;
                float *dst = out + (int64_t)(level - 1) * plane + tile_ofs;
#pragma unroll
                for (int j = 0; j < kTY; ++j) {
                    const float2 p0 = s_prev[(2 * j + 0) * kConvThreads + threadIdx.x];
                    const float2 p1 = s_prev[(2 * j + 1) * kConvThreads + threadIdx.x];
                    float4 d;   // sigma * (narrow - wide): subtract, then scale (two roundings)
                    d.x = __fmul_rn(__fsub_rn(p0.x, acc[j][0].x), s);
                    d.y = __fmul_rn(__fsub_rn(p0.y, acc[j][0].y), s);
                    d.z = __fmul_rn(__fsub_rn(p1.x, acc[j][1].x), s);
                    d.w = __fmul_rn(__fsub_rn(p1.y, acc[j][1].y), s);
                    reinterpret_cast<float4 *>(dst + (int64_t)j * pitch)[lane] = d;
                }
            }
            if (level < lev_end - 1) {
#pragma unroll
                for (int j = 0; j < kTY; ++j) {
                    s_prev[(2 * j + 0) * kConvThreads + threadIdx.x] = acc[j][0];
                    s_prev[(2 * j + 1) * kConvThreads + threadIdx.x] = acc[j][1];
                }
            }
        }
        if (level + 1 < lev_end) {             // first rows of the next level
            const float *in2 = in + plane;
            const int *rows2 = s_rows + warp * kTY + (max_rpad - tbl.lv[level + 1].rpad);
#pragma unroll
            for (int p = 0; p < kPrefetch; ++p) load_row<true>(in2 + rows2[p], lane, v[p]);
        }
    }
}

// the slice that straddles groups g and g+1: D = f32(sigma) * (last(g) - first(g+1))
__global__ void __launch_bounds__(256)
edge_dog_kernel(const float *__restrict__ edge, int64_t plane, float *__restrict__ out,
                const __grid_constant__ LevelTable tbl) {
    const int g = blockIdx.y;
    const int slice = tbl.group_begin[g + 1] - 1;
    const float s = tbl.lv[slice].sigma_f32;
    const float4 *a = reinterpret_cast<const float4 *>(edge + (int64_t)(2 * g + 1) * plane);
    const float4 *b = reinterpret_cast<const float4 *>(edge + (int64_t)(2 * (g + 1)) * plane);
    float4 *d = reinterpret_cast<float4 *>(out + (int64_t)slice * plane);
    const int64_t n4 = plane / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float4 x = __ldg(a + i), y = __ldg(b + i);
        d[i] = make_float4(__fmul_rn(__fsub_rn(x.x, y.x), s), __fmul_rn(__fsub_rn(x.y, y.y), s),
                           __fmul_rn(__fsub_rn(x.z, y.z), s), __fmul_rn(__fsub_rn(x.w, y.w), s));
    }
}

// ---- layout helpers -------------------------------------------------------------
// src_t: [planes][Wp][Hp] (x-major)  ->  dst: dense [planes][H][W]
__global__ void untranspose_kernel(const float *__restrict__ src_t, int Hp, int Wp, int H, int W,
                                   float *__restrict__ dst) {
    __shared__ float tile[32][33];
    const int64_t plane_in = (int64_t)Hp * Wp, plane_out = (int64_t)H * W;
    const float *src = src_t + blockIdx.z * plane_in;
    float *d = dst + blockIdx.z * plane_out;
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int x = x0 + i, y = y0 + threadIdx.x;
        tile[i][threadIdx.x] = (x < W && y < H) ? src[(int64_t)x * Hp + y] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int y = y0 + i, x = x0 + threadIdx.x;
        if (x < W && y < H) d[(int64_t)y * W + x] = tile[threadIdx.x][i];
    }
}

__global__ void dog_from_levels_kernel(int n_slices, int64_t plane, const float *__restrict__ lv,
                                       const float *__restrict__ sigma_f32,
                                       float *__restrict__ out) {
    const int64_t total = (int64_t)n_slices * plane;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(i / plane);
        out[i] = __fmul_rn(__fsub_rn(lv[i], lv[i + plane]), sigma_f32[s]);
    }
}

size_t row_table_bytes(int max_rpad) {
    return (size_t)(kTileRows + 2 * max_rpad + kPrefetch + kL2Ahead + 4) * sizeof(int);
}
size_t row_pass_smem(int max_table, int max_rpad) {
    return (size_t)kTileCols * kTileRows * sizeof(float) + (size_t)max_table * sizeof(float2) +
           row_table_bytes(max_rpad);
}
size_t col_pass_smem_impl(int group_table, int max_rpad, bool dog) {
    return (dog ? (size_t)kTY * 2 * kConvThreads * sizeof(float2) : 0) +
           (size_t)group_table * sizeof(float2) + row_table_bytes(max_rpad);
}

// Which warps of a column-pass CTA pull rows kL2Ahead steps ahead into L2 (bit w = warp w).
// Default: the warp with the highest row range, the first to touch new rows.
unsigned frontier_warps() {
    static const unsigned mask = [] {
        const char *e = std::getenv("DOGBLOB_FRONTIER");
        return e ? (unsigned)std::strtoul(e, nullptr, 0) : (1u << (kWarps - 1));
    }();
    return mask;
}

}  // namespace

size_t col_pass_smem(int group_table, int max_rpad, bool dog) {
    return col_pass_smem_impl(group_table, max_rpad, dog);
}

// Opt every convolution kernel in to the device's full shared-memory carve-out once; the
// per-launch size is what the plan's geometry asks for.
cudaError_t configure_conv_kernels(int device) {
    int optin = 0;
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(row_pass_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(row_pass_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(col_pass_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(col_pass_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin);
}

cudaError_t launch_row_pass(const ConvGeometry &g, const float *d_img, float *d_rows_t,
                            const LevelTable &tbl, const float2 *d_taps, cudaStream_t st,
                            const RowGate *gate) {
    const size_t smem = row_pass_smem(g.max_table, g.max_rpad);
    if (gate) {
        dim3 grid(g.Wp / kTileCols, g.L, g.Hp / kTileRows);
        row_pass_kernel<true><<<grid, kConvThreads, smem, st>>>(d_img, g.Wp, g.H, d_rows_t, g.Hp,
                                                                (int64_t)g.Hp * g.Wp, tbl, d_taps,
                                                                g.max_table, *gate);
    } else {
        dim3 grid(g.Wp / kTileCols, g.Hp / kTileRows, g.L);
        row_pass_kernel<false><<<grid, kConvThreads, smem, st>>>(d_img, g.Wp, g.H, d_rows_t, g.Hp,
                                                                 (int64_t)g.Hp * g.Wp, tbl, d_taps,
                                                                 g.max_table, RowGate{nullptr, 0, 1, nullptr});
    }
    return cudaGetLastError();
}

cudaError_t launch_col_dog_pass(const ConvGeometry &g, const float *d_rows_t, float *d_dog_t,
                                float *d_edge, const LevelTable &tbl, const float2 *d_taps,
                                cudaStream_t st) {
    dim3 grid(g.Hp / kTileCols, g.Wp / kTileRows, g.G);
    const int64_t plane = (int64_t)g.Hp * g.Wp;
    const size_t smem = col_pass_smem_impl(g.max_group_table, g.max_rpad, true);
    col_pass_kernel<true><<<grid, kConvThreads, smem, st>>>(d_rows_t, g.Hp, plane, g.W, d_dog_t, d_edge,
                                                            tbl, d_taps, g.max_rpad, frontier_warps());
    return launch_edge_dog(g, d_edge, d_dog_t, tbl, st);
}

// the slices that straddle two level groups, from the parked boundary levels
cudaError_t launch_edge_dog(const ConvGeometry &g, const float *d_edge, float *d_dog_t,
                            const LevelTable &tbl, cudaStream_t st) {
    const int64_t plane = (int64_t)g.Hp * g.Wp;
    if (tbl.n_groups > 1) {
        int bx = (int)((plane / 4 + 255) / 256);
        if (bx > 148 * 2) bx = 148 * 2;
        edge_dog_kernel<<<dim3(bx, tbl.n_groups - 1), 256, 0, st>>>(d_edge, plane, d_dog_t, tbl);
    }
    return cudaGetLastError();
}

cudaError_t launch_col_levels_pass(const ConvGeometry &g, const float *d_rows_t, float *d_lev_t,
                                   const LevelTable &unit_tbl, const float2 *d_taps,
                                   cudaStream_t st) {
    dim3 grid(g.Hp / kTileCols, g.Wp / kTileRows, g.L);
    col_pass_kernel<false><<<grid, kConvThreads, col_pass_smem_impl(g.max_table, g.max_rpad, false), st>>>(
        d_rows_t, g.Hp, (int64_t)g.Hp * g.Wp, g.W, d_lev_t, nullptr, unit_tbl, d_taps, g.max_rpad, frontier_warps());
    return cudaGetLastError();
}

cudaError_t launch_untranspose(const float *d_src_t, int planes, int Hp, int Wp, int H, int W,
                               float *d_dst, cudaStream_t st) {
    dim3 grid((W + 31) / 32, (H + 31) / 32, planes);
    untranspose_kernel<<<grid, dim3(32, 8), 0, st>>>(d_src_t, Hp, Wp, H, W, d_dst);
    return cudaGetLastError();
}

cudaError_t launch_dog_from_levels(int L, int64_t plane_elems, const float *d_levels,
                                   const float *d_sigma_f32, float *d_out, cudaStream_t st) {
    const int64_t total = (int64_t)(L - 1) * plane_elems;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    dog_from_levels_kernel<<<blocks, 256, 0, st>>>(L - 1, plane_elems, d_levels, d_sigma_f32, d_out);
    return cudaGetLastError();
}

}  // namespace dogblob
