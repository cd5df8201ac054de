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
#include "common.cuh"

namespace dogblob {

namespace {

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// Reflect boundary as a bouncing cursor: ... 2 1 0 | 0 1 2 ... N-1 | N-1 N-2 ...
// The row pointer is advanced incrementally (no per-step multiply): on a bounce
// the edge row is repeated once and the direction flips.
struct FoldCursor {
    int m, dir, n;
    const float *p;      // -> row m
    int64_t dp;          // dir * pitch (elements)
    __device__ __forceinline__ FoldCursor(const float *base, int64_t pitch, int start, int n_)
        : n(n_) {
        int period = 2 * n_;
        int t = start % period;
        if (t < 0) t += period;
        if (t < n_) { m = t; dir = 1; } else { m = period - 1 - t; dir = -1; }
        p = base + (int64_t)m * pitch;
        dp = dir > 0 ? pitch : -pitch;
    }
    __device__ __forceinline__ void step() {
        const int nm = m + dir;
        const bool bounce = (nm == n) | (nm < 0);
        if (bounce) { dir = -dir; dp = -dp; }
        else { m = nm; p += dp; }
    }
};

template <bool ADJACENT>
__device__ __forceinline__ void load_row(const float *__restrict__ row, int lane, float (&v)[4]) {
    if (ADJACENT) {
        float4 q = __ldg(reinterpret_cast<const float4 *>(row) + lane);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = __ldg(row + lane + 32 * c);
    }
}

// One sweep: acc[j][p] = sum_k w[k] * in[fold(out_row0 + j + k)][cols(p)]
// `taps` is the zero-padded, duplicated table P of this level in shared memory:
// P[m] = w[m - (kTY-1)] for kTY-1 <= m <= 2r + kTY-1, else 0, so that the tap of
// (input step s, output j) is P[s - j + kTY - 1] and no bounds test is needed.
template <bool ADJACENT>
__device__ __forceinline__ void sweep(const float *__restrict__ in, int64_t pitch, int n_rows,
                                      int first_in_row, int n_chunks,
                                      const float2 *__restrict__ taps, int lane,
                                      float2 (&acc)[kTY][2]) {
    FoldCursor cur(in, pitch, first_in_row, n_rows);
    float v[kPrefetch][4];
#pragma unroll
    for (int p = 0; p < kPrefetch; ++p) {
        load_row<ADJACENT>(cur.p, lane, v[p]);
        cur.step();
    }
    float2 ring[kTY];
#pragma unroll
    for (int j = 0; j < kTY; ++j) {
        ring[j] = make_float2(0.f, 0.f);
        acc[j][0] = make_float2(0.f, 0.f);
        acc[j][1] = make_float2(0.f, 0.f);
    }
    const float2 *tp = taps + (kTY - 1);
    for (int chunk = 0; chunk < n_chunks; ++chunk) {
#pragma unroll
        for (int u = 0; u < kTY; ++u) {
            ring[u] = tp[u];
            const float2 a = make_float2(v[u % kPrefetch][0], v[u % kPrefetch][1]);
            const float2 b = make_float2(v[u % kPrefetch][2], v[u % kPrefetch][3]);
            load_row<ADJACENT>(cur.p, lane, v[u % kPrefetch]);
            cur.step();
#pragma unroll
            for (int j = 0; j < kTY; ++j) {
                const float2 t = ring[(u - j + kTY) % kTY];
                acc[j][0] = ffma2(t, a, acc[j][0]);
                acc[j][1] = ffma2(t, b, acc[j][1]);
            }
        }
        tp += kTY;
    }
}

__device__ __forceinline__ void stage_taps(float2 *s_taps, const float2 *__restrict__ g_taps,
                                           const LevelDesc &lv) {
    const int n = lv.n_chunks * kTY + kTY - 1;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_taps[i] = g_taps[lv.tap_ofs + i];
}

constexpr int kTilePitch = kTileRows + 1;  // 129: conflict-free transposed writes

// ---- pass 1: correlate along y, store transposed ------------------------------
__global__ void __launch_bounds__(kConvThreads, 2)
row_pass_kernel(const float *__restrict__ img, int64_t img_pitch, int H,
                float *__restrict__ out_t, int64_t out_pitch, int64_t out_plane,
                const LevelDesc *__restrict__ levels, const float2 *__restrict__ g_taps,
                const int *__restrict__ level_order) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *tile = reinterpret_cast<float *>(smem_raw);                       // [128][129]
    float2 *s_taps = reinterpret_cast<float2 *>(tile + kTileCols * kTilePitch);

    const int level = level_order[blockIdx.z];
    const LevelDesc lv = levels[level];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int col0 = blockIdx.x * kTileCols;            // x
    const int row0 = blockIdx.y * kTileRows;            // y
    stage_taps(s_taps, g_taps, lv);
    __syncthreads();

    float2 acc[kTY][2];
    sweep<false>(img + col0, img_pitch, H, row0 + warp * kTY - lv.radius, lv.n_chunks, s_taps,
                 lane, acc);

    // tile[x_local][y_local]; lane stride 1 in x -> bank = lane + const: conflict free
#pragma unroll
    for (int j = 0; j < kTY; ++j) {
        const int yl = warp * kTY + j;
        tile[(lane + 0) * kTilePitch + yl] = acc[j][0].x;
        tile[(lane + 32) * kTilePitch + yl] = acc[j][0].y;
        tile[(lane + 64) * kTilePitch + yl] = acc[j][1].x;
        tile[(lane + 96) * kTilePitch + yl] = acc[j][1].y;
    }
    __syncthreads();
    float *dst = out_t + (int64_t)level * out_plane + (int64_t)col0 * out_pitch + row0;
    for (int i = threadIdx.x; i < kTileCols * kTileRows; i += kConvThreads) {
        const int xl = i >> 7, yl = i & 127;
        dst[(int64_t)xl * out_pitch + yl] = tile[xl * kTilePitch + yl];
    }
}

// ---- pass 2: correlate along x (rows of the transposed planes), fused DoG ------
// grid.z = level group g; the CTA walks levels group_begin[g] .. group_begin[g+1]
// (inclusive: the first level of the next group is recomputed here so that no
// level is ever written to memory) and emits D_i for i in [begin, end).
template <bool DOG>
__global__ void __launch_bounds__(kConvThreads, 2)
col_pass_kernel(const float *__restrict__ rows_t, int64_t pitch, int64_t plane, int n_rows,
                float *__restrict__ out, const LevelDesc *__restrict__ levels,
                const float2 *__restrict__ g_taps, const int *__restrict__ group_begin,
                int n_levels) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2 *s_prev = reinterpret_cast<float2 *>(smem_raw);                    // [kTY*2][256]
    float2 *s_taps = s_prev + (DOG ? kTY * 2 * kConvThreads : 0);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int col0 = blockIdx.x * kTileCols;
    const int row0 = blockIdx.y * kTileRows + warp * kTY;
    const int lev_begin = group_begin[blockIdx.z];
    int lev_end = group_begin[blockIdx.z + 1];               // exclusive for outputs
    const int lev_last = DOG ? min(lev_end, n_levels - 1) : lev_end - 1;

    for (int level = lev_begin; level <= lev_last; ++level) {
        const LevelDesc lv = levels[level];
        __syncthreads();                                     // previous taps no longer in use
        stage_taps(s_taps, g_taps, lv);
        __syncthreads();
        float2 acc[kTY][2];
        sweep<true>(rows_t + (int64_t)level * plane + col0, pitch, n_rows, row0 - lv.radius,
                    lv.n_chunks, s_taps, lane, acc);
        if (!DOG) {
            float *dst = out + (int64_t)level * plane + (int64_t)row0 * pitch + col0;
#pragma unroll
            for (int j = 0; j < kTY; ++j)
                reinterpret_cast<float4 *>(dst + (int64_t)j * pitch)[lane] =
                    make_float4(acc[j][0].x, acc[j][0].y, acc[j][1].x, acc[j][1].y);
        } else {
            if (level > lev_begin) {
                const float s = levels[level - 1].sigma_f32;
                float *dst = out + (int64_t)(level - 1) * plane + (int64_t)row0 * pitch + col0;
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
            if (level < lev_last) {
#pragma unroll
                for (int j = 0; j < kTY; ++j) {
                    s_prev[(2 * j + 0) * kConvThreads + threadIdx.x] = acc[j][0];
                    s_prev[(2 * j + 1) * kConvThreads + threadIdx.x] = acc[j][1];
                }
            }
        }
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

size_t row_pass_smem(int max_table) {
    return (size_t)kTileCols * kTilePitch * sizeof(float) + (size_t)max_table * sizeof(float2);
}
size_t col_pass_smem(int max_table, bool dog) {
    return (dog ? (size_t)kTY * 2 * kConvThreads * sizeof(float2) : 0) +
           (size_t)max_table * sizeof(float2);
}

}  // namespace

cudaError_t configure_conv_kernels(int max_table) {
    cudaError_t e;
    e = cudaFuncSetAttribute(row_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)row_pass_smem(max_table));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(col_pass_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)col_pass_smem(max_table, true));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(col_pass_kernel<false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)col_pass_smem(max_table, false));
}

cudaError_t launch_row_pass(const ConvGeometry &g, const float *d_img, float *d_rows_t,
                            const LevelDesc *d_levels, const float2 *d_taps,
                            const int *d_level_order, cudaStream_t st) {
    dim3 grid(g.Wp / kTileCols, g.Hp / kTileRows, g.L);
    row_pass_kernel<<<grid, kConvThreads, row_pass_smem(g.max_table), st>>>(
        d_img, g.Wp, g.H, d_rows_t, g.Hp, (int64_t)g.Hp * g.Wp, d_levels, d_taps, d_level_order);
    return cudaGetLastError();
}

cudaError_t launch_col_dog_pass(const ConvGeometry &g, const float *d_rows_t, float *d_dog_t,
                                const LevelDesc *d_levels, const float2 *d_taps,
                                const int *d_group_begin, cudaStream_t st) {
    dim3 grid(g.Hp / kTileCols, g.Wp / kTileRows, g.G);
    col_pass_kernel<true><<<grid, kConvThreads, col_pass_smem(g.max_table, true), st>>>(
        d_rows_t, g.Hp, (int64_t)g.Hp * g.Wp, g.W, d_dog_t, d_levels, d_taps, d_group_begin, g.L);
    return cudaGetLastError();
}

cudaError_t launch_col_levels_pass(const ConvGeometry &g, const float *d_rows_t, float *d_lev_t,
                                   const LevelDesc *d_levels, const float2 *d_taps,
                                   const int *d_unit_groups, cudaStream_t st) {
    dim3 grid(g.Hp / kTileCols, g.Wp / kTileRows, g.L);
    col_pass_kernel<false><<<grid, kConvThreads, col_pass_smem(g.max_table, false), st>>>(
        d_rows_t, g.Hp, (int64_t)g.Hp * g.Wp, g.W, d_lev_t, d_levels, d_taps, d_unit_groups, g.L);
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
