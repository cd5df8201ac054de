// Scale-space extrema for sm_100a: 3-D non-maximum suppression with threshold,
// warp-ballot/popc stream compaction, plateau coalescing and ordering.
//
// Replaces find_extrema / _coalesce_plateaus / _sort_blobs
// (pkg/src/dogblob/detector.py:129-193):
//   flagged(v)  <=>  D[v] == max over the n^3 block (missing neighbours = -inf)
//                    and D[v] > float32(threshold)
//               <=>  D[v] > thr and no neighbour is strictly greater;
//   8-connected flagged voxels of one slice form one blob at the half-even
//   rounded centroid (adjacent flagged voxels necessarily share one value);
//   blobs are ordered by (-response, y, x, sigma).
//
// The volume is read exactly once, as float4 along the contiguous axis; only
// voxels above the threshold (a few per million) touch their neighbours.
#include "common.cuh"

namespace dogblob {

namespace {

struct Volume {
    const float *__restrict__ data;
    int S, rows, cols;           // valid extents
    int64_t pitch, plane;
    __device__ __forceinline__ float at(int s, int r, int c) const {
        return __ldg(data + (int64_t)s * plane + (int64_t)r * pitch + c);
    }
};

// no neighbour in the (2h+1)^3 block is strictly greater than v
__device__ bool is_block_max(const Volume &vol, int s, int r, int c, float v, int h) {
    const int s0 = max(s - h, 0), s1 = min(s + h, vol.S - 1);
    const int r0 = max(r - h, 0), r1 = min(r + h, vol.rows - 1);
    const int c0 = max(c - h, 0), c1 = min(c + h, vol.cols - 1);
    for (int ss = s0; ss <= s1; ++ss)
        for (int rr = r0; rr <= r1; ++rr)
            for (int cc = c0; cc <= c1; ++cc)
                if (vol.at(ss, rr, cc) > v) return false;
    return true;
}

// does a flagged voxel share an in-slice 8-neighbour that is flagged too?  For
// n >= 3 such a neighbour necessarily has the same value (each is >= the other);
// for n == 1 every voxel above the threshold is flagged.
__device__ bool has_flagged_neighbour(const Volume &vol, int s, int r, int c, float v, int h,
                                      float thr) {
    for (int dr = -1; dr <= 1; ++dr)
        for (int dc = -1; dc <= 1; ++dc) {
            if (dr == 0 && dc == 0) continue;
            const int rr = r + dr, cc = c + dc;
            if (rr < 0 || rr >= vol.rows || cc < 0 || cc >= vol.cols) continue;
            const float nv = vol.at(s, rr, cc);
            if (h >= 1 ? (nv == v && is_block_max(vol, s, rr, cc, nv, h)) : (nv > thr)) return true;
        }
    return false;
}

__device__ __forceinline__ dogblob_blob make_blob(int s, double x, double y, float val, int S,
                                                  const double *__restrict__ slice_sigma) {
    dogblob_blob b;
    b.x = x;
    b.y = y;
    b.sigma = slice_sigma[s];
    b.radius = 1.4142135623730951 * b.sigma;   // math.sqrt(2.0) * sigma, one rounding
    b.response = (double)val;
    b.slice = s;
    b.flags = (s == 0 || s == S - 1) ? DOGBLOB_BLOB_SCALE_EDGE : 0u;
    return b;
}

// ---- NMS + compaction -----------------------------------------------------------
// A CTA stages a (kNmsRows + 2) x (1024 + 2) tile of one DoG slice in shared memory
// (every load issued up front: 10 independent 16-byte loads per thread), so the
// threshold test and the 8 in-slice neighbours of the 3x3x3 block cost no global
// traffic.  Only 2-D local maxima above the threshold (a few thousand per frame)
// read their 18 cross-slice neighbours, in two batches of 9 independent loads.
constexpr int kNmsRows = 8;
constexpr int kNmsCols = 1024;                 // 256 threads x 4
constexpr int kNmsPitch = kNmsCols + 8;        // halo column at index 3 and kNmsCols + 4

template <int VEC>
__global__ void __launch_bounds__(256)
nms_kernel(Volume vol, float thr, int h, bool transposed, const double *__restrict__ slice_sigma,
           BlobSpace bs) {
    __shared__ __align__(16) float tile[(kNmsRows + 2) * kNmsPitch];
    const int s = blockIdx.z;
    const int r0 = blockIdx.y * kNmsRows;
    const int c0 = blockIdx.x * kNmsCols;
    const int t = threadIdx.x;
    const unsigned lane = t & 31;
    const float *plane = vol.data + (int64_t)s * vol.plane;
    const int c = c0 + 4 * t;
    // ---- stage the tile (+1 halo on every side, -inf outside the plane) ----
#pragma unroll
    for (int rr = 0; rr < kNmsRows + 2; ++rr) {
        const int r = r0 - 1 + rr;
        float4 q = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        if (r >= 0 && r < vol.rows && c < vol.cols) {
            const float *p = plane + (int64_t)r * vol.pitch + c;
            if (VEC == 4) {
                q = __ldg(reinterpret_cast<const float4 *>(p));   // pitch-padded: in bounds
                if (c + 1 >= vol.cols) q.y = -INFINITY;
                if (c + 2 >= vol.cols) q.z = -INFINITY;
                if (c + 3 >= vol.cols) q.w = -INFINITY;
            } else {
                q.x = __ldg(p);
                if (c + 1 < vol.cols) q.y = __ldg(p + 1);
                if (c + 2 < vol.cols) q.z = __ldg(p + 2);
                if (c + 3 < vol.cols) q.w = __ldg(p + 3);
            }
        }
        *reinterpret_cast<float4 *>(&tile[rr * kNmsPitch + 4 + 4 * t]) = q;
    }
    if (t < 2 * (kNmsRows + 2)) {
        const int rr = t >> 1, side = t & 1;
        const int r = r0 - 1 + rr;
        const int cc = side ? c0 + kNmsCols : c0 - 1;
        float x = -INFINITY;
        if (r >= 0 && r < vol.rows && cc >= 0 && cc < vol.cols)
            x = __ldg(plane + (int64_t)r * vol.pitch + cc);
        tile[rr * kNmsPitch + (side ? kNmsCols + 4 : 3)] = x;
    }
    __syncthreads();
    // ---- test ----
#pragma unroll 1
    for (int q = 1; q <= kNmsRows; ++q) {
        const int r = r0 - 1 + q;
        const float *row = &tile[q * kNmsPitch + 4 + 4 * t];
        const float4 mid = *reinterpret_cast<const float4 *>(row);
        const bool any = (mid.x > thr) | (mid.y > thr) | (mid.z > thr) | (mid.w > thr);
        if (!__any_sync(0xffffffffu, any)) continue;
        // 3 x 6 window [left | 4 own columns | right] of rows q-1, q, q+1: three 16-byte and
        // six 4-byte shared loads feed all 8 in-slice neighbours of the 4 voxels
        float w[3][6];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const float *rp = row + (d - 1) * kNmsPitch;
            const float4 c4 = *reinterpret_cast<const float4 *>(rp);
            w[d][0] = rp[-1];
            w[d][1] = c4.x; w[d][2] = c4.y; w[d][3] = c4.z; w[d][4] = c4.w;
            w[d][5] = rp[4];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float val = w[1][k + 1];
            bool cand = val > thr;            // out-of-plane voxels hold -inf
            if (h >= 1)                       // the 8 in-slice neighbours are in every n >= 3 block
                cand = cand && !(w[0][k] > val) && !(w[0][k + 1] > val) && !(w[0][k + 2] > val) &&
                       !(w[1][k] > val) && !(w[1][k + 2] > val) &&
                       !(w[2][k] > val) && !(w[2][k + 1] > val) && !(w[2][k + 2] > val);
            if (!__any_sync(0xffffffffu, cand)) continue;
            bool flagged = false, plateau = false;
            if (cand) {
                if (h == 1) {                 // 3x3x3: in-slice part done, two batches of 9 loads
                    flagged = true;
#pragma unroll
                    for (int ds = -1; ds <= 1; ds += 2) {
                        const int ss = s + ds;
                        if (ss < 0 || ss >= vol.S) continue;
                        float nb[9];
#pragma unroll
                        for (int j = 0; j < 9; ++j) {
                            const int rr = r + j / 3 - 1, cc = c + k + j % 3 - 1;
                            nb[j] = (rr >= 0 && rr < vol.rows && cc >= 0 && cc < vol.cols)
                                        ? vol.at(ss, rr, cc) : -INFINITY;
                        }
#pragma unroll
                        for (int j = 0; j < 9; ++j) flagged = flagged && !(nb[j] > val);
                    }
                } else {
                    flagged = is_block_max(vol, s, r, c + k, val, h);
                }
                if (flagged) plateau = has_flagged_neighbour(vol, s, r, c + k, val, h, thr);
            }
            // warp-aggregated append: one atomic per warp and list
            const unsigned m_single = __ballot_sync(0xffffffffu, flagged && !plateau);
            const unsigned m_plat = __ballot_sync(0xffffffffu, flagged && plateau);
            if (!(m_single | m_plat)) continue;
            const unsigned lt = (1u << lane) - 1u;
            int base_s = 0, base_p = 0;
            if (lane == 0) {
                atomicAdd(&bs.ctr->n_flagged, __popc(m_single) + __popc(m_plat));
                if (m_single) base_s = atomicAdd(&bs.ctr->n_candidates, __popc(m_single));
                if (m_plat) base_p = atomicAdd(&bs.ctr->n_plateau, __popc(m_plat));
            }
            base_s = __shfl_sync(0xffffffffu, base_s, 0);
            base_p = __shfl_sync(0xffffffffu, base_p, 0);
            if (flagged && !plateau) {
                const int idx = base_s + __popc(m_single & lt);
                if (idx < bs.cap) {
                    const int cc = c + k;
                    bs.unsorted[idx] = make_blob(s, transposed ? r : cc, transposed ? cc : r, val,
                                                 vol.S, slice_sigma);
                } else {
                    atomicOr(&bs.ctr->flags, DOGBLOB_FLAG_OVERFLOW);
                }
            } else if (flagged) {
                const int idx = base_p + __popc(m_plat & lt);
                if (idx < bs.cap) {
                    bs.plateau[idx] = Voxel{s, r, c + k, val};
                    bs.parent[idx] = idx;
                    bs.pl_count[idx] = 0;
                    bs.pl_sum_row[idx] = 0ull;
                    bs.pl_sum_col[idx] = 0ull;
                    bs.pl_first[idx] = ~0ull;
                } else {
                    atomicOr(&bs.ctr->flags, DOGBLOB_FLAG_OVERFLOW);
                }
            }
        }
    }
}

// ---- plateau coalescing: lock-free union-find over the (rare) plateau members ----
__device__ __forceinline__ int uf_find(int *parent, int x) {
    int p = ((volatile int *)parent)[x];
    while (p != x) { x = p; p = ((volatile int *)parent)[x]; }
    return x;
}
__device__ void uf_union(int *parent, int a, int b) {
    while (true) {
        a = uf_find(parent, a);
        b = uf_find(parent, b);
        if (a == b) return;
        if (a > b) { int t = a; a = b; b = t; }
        if (atomicCAS(&parent[b], b, a) == b) return;   // larger root hooks under smaller
    }
}

// One launch: every CTA links its share of member pairs; the last CTA to finish reduces the
// components and emits one blob per root.  With no plateau member (the usual case on noisy
// frames) the kernel returns at once.
__global__ void __launch_bounds__(256)
plateau_kernel(BlobSpace bs, int S, bool transposed, const double *__restrict__ slice_sigma) {
    const int n = min(bs.ctr->n_plateau, bs.cap);
    if (n == 0) return;
    __shared__ Voxel tile[256];
    __shared__ bool last;
    for (int a0 = blockIdx.x * blockDim.x; a0 < n; a0 += gridDim.x * blockDim.x) {
        const int a = a0 + threadIdx.x;
        Voxel va = (a < n) ? bs.plateau[a] : Voxel{-9, -9, -9, 0.f};
        for (int b0 = 0; b0 < a0 + (int)blockDim.x && b0 < n; b0 += blockDim.x) {
            __syncthreads();
            if (b0 + (int)threadIdx.x < n) tile[threadIdx.x] = bs.plateau[b0 + threadIdx.x];
            __syncthreads();
            const int lim = min((int)blockDim.x, n - b0);
            if (a < n)
                for (int k = 0; k < lim; ++k) {
                    const int b = b0 + k;
                    if (b >= a) break;
                    const Voxel vb = tile[k];
                    if (vb.s == va.s && abs(vb.row - va.row) <= 1 && abs(vb.col - va.col) <= 1)
                        uf_union(bs.parent, a, b);
                }
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(&bs.ctr->plateau_ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int a = threadIdx.x; a < n; a += blockDim.x) {
        const int root = uf_find(bs.parent, a);
        const Voxel v = bs.plateau[a];
        atomicAdd(&bs.pl_count[root], 1);
        atomicAdd(&bs.pl_sum_row[root], (unsigned long long)v.row);
        atomicAdd(&bs.pl_sum_col[root], (unsigned long long)v.col);
        // the component's response is the value at its raster-first (y, then x) voxel
        const unsigned long long y = transposed ? v.col : v.row, x = transposed ? v.row : v.col;
        atomicMin(&bs.pl_first[root], (y << 44) | (x << 24) | (unsigned long long)a);
    }
    __threadfence();
    __syncthreads();
    for (int a = threadIdx.x; a < n; a += blockDim.x) {
        if (((volatile int *)bs.parent)[a] != a) continue;
        const Voxel v = bs.plateau[(int)(((volatile unsigned long long *)bs.pl_first)[a] & 0xFFFFFFull)];
        const double cnt = (double)((volatile int *)bs.pl_count)[a];
        // ndimage.center_of_mass: float64 sum / count, then Python round() = half-even
        const double cr = rint((double)((volatile unsigned long long *)bs.pl_sum_row)[a] / cnt);
        const double cc = rint((double)((volatile unsigned long long *)bs.pl_sum_col)[a] / cnt);
        const int idx = atomicAdd(&bs.ctr->n_candidates, 1);
        if (idx < bs.cap)
            bs.unsorted[idx] = make_blob(v.s, transposed ? cr : cc, transposed ? cc : cr, v.val, S,
                                         slice_sigma);
        else
            atomicOr(&bs.ctr->flags, DOGBLOB_FLAG_OVERFLOW);
    }
}

// ---- ordering: rank sort on the full key (stable on the input index) ----------------
__global__ void reset_counters_kernel(BlobSpace bs) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        Counters z = {};
        *bs.ctr = z;
    }
    // ticket, done, n_phases, changed, sweeps, n_roots, merges, kept of the pruning control block
    if (blockIdx.x == 0 && threadIdx.x < 8) reinterpret_cast<int *>(bs.ctl)[threadIdx.x] = 0;
}

__global__ void load_blobs_kernel(BlobSpace bs, const dogblob_blob *__restrict__ in, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        bs.unsorted[i] = in[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) bs.ctr->n_candidates = n;
}

}  // namespace

cudaError_t launch_reset_counters(const BlobSpace &bs, cudaStream_t st) {
    reset_counters_kernel<<<1, 32, 0, st>>>(bs);
    return cudaGetLastError();
}

cudaError_t launch_load_blobs(const BlobSpace &bs, const dogblob_blob *d_in, int n,
                              cudaStream_t st) {
    int blocks = (n + 255) / 256;
    if (blocks < 1) blocks = 1;
    if (blocks > 296) blocks = 296;
    load_blobs_kernel<<<blocks, 256, 0, st>>>(bs, d_in, n);
    return cudaGetLastError();
}

cudaError_t launch_extrema(const float *d_slices, int S, int rows, int cols, int64_t pitch,
                           int64_t plane, bool transposed, const double *d_slice_sigma,
                           float threshold, int half, const BlobSpace &bs, cudaStream_t st) {
    Volume vol{d_slices, S, rows, cols, pitch, plane};
    const bool vec4 = (pitch % 4 == 0) && (plane % 4 == 0) &&
                      ((reinterpret_cast<uintptr_t>(d_slices) & 15u) == 0);
    const dim3 grid((cols + kNmsCols - 1) / kNmsCols, (rows + kNmsRows - 1) / kNmsRows, S);
    if (vec4)
        nms_kernel<4><<<grid, 256, 0, st>>>(vol, threshold, half, transposed, d_slice_sigma, bs);
    else
        nms_kernel<1><<<grid, 256, 0, st>>>(vol, threshold, half, transposed, d_slice_sigma, bs);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    plateau_kernel<<<148, 256, 0, st>>>(bs, S, transposed, d_slice_sigma);
    return cudaGetLastError();
}

}  // namespace dogblob
