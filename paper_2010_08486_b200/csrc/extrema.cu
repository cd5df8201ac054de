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
#include <cstdlib>

#include <algorithm>

#include "common.cuh"

namespace dogblob {

namespace {

template <typename T>
struct VolumeT {
    const T *__restrict__ data;
    int S, rows, cols;           // valid extents
    int64_t pitch, plane;
    // Optional validity map (tensor engine): one byte per 8-row x 32-column block of every slice, as
    // HitFlags.  The producer does not even STORE blocks without a value above the threshold, so
    // whatever the memory of such a block holds (an older frame) must read as -inf: it can never beat
    // a candidate, which is above the threshold by definition.
    const unsigned char *__restrict__ valid = nullptr;
    int v_row_blocks = 0, v_col_blocks = 0;
    __device__ __forceinline__ bool block_valid(int s, int r, int c) const {
        return valid == nullptr || valid[((int64_t)s * v_col_blocks + (c >> kFlagColShift)) * v_row_blocks + (r >> kFlagRowShift)] != 0;
    }
    __device__ __forceinline__ T at(int s, int r, int c) const {
        if (!block_valid(s, r, c)) return (T)-INFINITY;      // (loading first and selecting afterwards measured 10-20 % slower)
        return __ldg(data + (int64_t)s * plane + (int64_t)r * pitch + c);
    }
};
using Volume = VolumeT<float>;     // production path; VolumeT<double>: the float64 tier (fp64.cu)

// no neighbour in the (2h+1)^3 block is strictly greater than v
template <typename T>
__device__ bool is_block_max(const VolumeT<T> &vol, int s, int r, int c, T v, int h) {
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
template <typename T>
__device__ bool has_flagged_neighbour(const VolumeT<T> &vol, int s, int r, int c, T v, int h, T thr) {
    for (int dr = -1; dr <= 1; ++dr)
        for (int dc = -1; dc <= 1; ++dc) {
            if (dr == 0 && dc == 0) continue;
            const int rr = r + dr, cc = c + dc;
            if (rr < 0 || rr >= vol.rows || cc < 0 || cc >= vol.cols) continue;
            const T nv = vol.at(s, rr, cc);
            if (h >= 1 ? (nv == v && is_block_max(vol, s, rr, cc, nv, h)) : (nv > thr)) return true;
        }
    return false;
}

__device__ __forceinline__ dogblob_blob make_blob(int s, double x, double y, double val, int S,
                                                  const double *__restrict__ slice_sigma) {
    dogblob_blob b;
    b.x = x;
    b.y = y;
    b.sigma = slice_sigma[s];
    b.radius = 1.4142135623730951 * b.sigma;   // math.sqrt(2.0) * sigma, one rounding
    b.response = val;
    b.slice = s;
    b.flags = (s == 0 || s == S - 1) ? DOGBLOB_BLOB_SCALE_EDGE : 0u;
    return b;
}

// A voxel that passed the in-slice test (`cand`): finish the (2h+1)^3 test against the
// neighbouring slices, classify single / plateau member, and append with one atomic per warp
// and list (ballot + popc).  Called by all 32 lanes (convergent), cand may be false.
template <typename T>
__device__ __forceinline__ void resolve_and_append(const VolumeT<T> &vol, int s, int r, int cc, T val,
                                                   bool cand, int h, T thr, bool transposed,
                                                   const double *__restrict__ slice_sigma,
                                                   const BlobSpace &bs, unsigned lane) {
    bool flagged = false, plateau = false;
    if (cand) {
        if (h == 1) {                 // 3x3x3: in-slice part done, two batches of 9 loads
            flagged = true;
#pragma unroll
            for (int ds = -1; ds <= 1; ds += 2) {
                const int ss = s + ds;
                if (ss < 0 || ss >= vol.S) continue;
                T nb[9];
#pragma unroll
                for (int j = 0; j < 9; ++j) {
                    const int rr = r + j / 3 - 1, c2 = cc + j % 3 - 1;
                    nb[j] = (rr >= 0 && rr < vol.rows && c2 >= 0 && c2 < vol.cols)
                                ? vol.at(ss, rr, c2) : (T)-INFINITY;
                }
#pragma unroll
                for (int j = 0; j < 9; ++j) flagged = flagged && !(nb[j] > val);
            }
        } else {
            flagged = is_block_max(vol, s, r, cc, val, h);
        }
        if (flagged) plateau = has_flagged_neighbour(vol, s, r, cc, val, h, thr);
    }
    // warp-aggregated append: one atomic per warp and list
    const unsigned m_single = __ballot_sync(0xffffffffu, flagged && !plateau);
    const unsigned m_plat = __ballot_sync(0xffffffffu, flagged && plateau);
    if (!(m_single | m_plat)) return;
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
            bs.unsorted[idx] = make_blob(s, transposed ? r : cc, transposed ? cc : r, (double)val,
                                         vol.S, slice_sigma);
        } else {
            atomicOr(&bs.ctr->flags, DOGBLOB_FLAG_OVERFLOW);
        }
    } else if (flagged) {
        const int idx = base_p + __popc(m_plat & lt);
        if (idx < bs.cap) {
            bs.plateau[idx] = Voxel{s, r, cc, 0, (double)val};
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

// ---- NMS for the 3x3x3 block on 16-byte aligned planes: register sliding window --------
// One warp owns a strip of 128 columns (4 per lane) and kBandRows rows of one slice and walks
// down the rows keeping three of them in registers; the left / right neighbours of a lane's
// four columns come from the adjacent lanes (two shuffles per row; lanes 0 and 31 read the
// strip's halo column).  A row's ring slot is reloaded, with a running pointer, as soon as the
// row has moved into the window; the 8 in-slice neighbours are reduced with 3-input maxima
// shared between the four voxels of a lane.  The shared-memory kernel below (kept for other
// neighbourhood sizes and unaligned planes) spent its time on index arithmetic (IMAD 26 %,
// ISETP 10 %, LEA 9 % of its instructions): C2 80 -> 65 us, C4 0.34 -> 0.22 ms.
// template parameters: kGroup rows in flight per lane, kBandRows tested rows per warp
// (kBandRows + 2 must be a multiple of kGroup)
constexpr int kQueueCap = 1024;             // queued maxima per warp before a flush

struct RowRegs { float4 q; float halo; };      // halo: column c-1 (lane 0) or c+4 (lane 31)

// one warp, one strip of 128 columns x kBandRows rows of slice s (tile = 8 strips side by side)
template <int kGroup, int kBandRows, int kWarps>
__device__ __forceinline__ void nms_strip(const Volume &vol, float thr, bool transposed,
                                          const double *__restrict__ slice_sigma, const BlobSpace &bs,
                                          const HitFlags &flags, int s, int tile_y, int tile_x,
                                          unsigned short *queue) {
    const unsigned lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // the 8 warps of a CTA sit side by side on the same rows: together they read 4 KB runs
    const int r_first = tile_y * kBandRows;                // first tested row
    const int c = (tile_x * kWarps + warp) * 128 + 4 * (int)lane;
    if (c - 4 * (int)lane >= vol.cols) return;
    // The producing kernel recorded which 8-row x 64-column blocks of the slice hold a value above
    // the threshold at all.  A strip without one cannot emit anything and is not even read; in the
    // others only the rows of hit blocks and their two neighbours are loaded (`need`, bit = local
    // row with r_first - 1 as bit 0): a row further away is neither tested nor anybody's neighbour.
    unsigned long long need = ~0ull;                       // rows to load (local row bits)
    unsigned long long valid_q = ~0ull, valid_h = ~0ull;   // rows whose own columns / halo column hold stored data
    if (flags.data != nullptr) {
        static_assert(kBandRows + 2 <= 64, "row mask");
        const int cb = (c - 4 * (int)lane) >> kFlagColShift;
        const int r_last = min(r_first + kBandRows - 1, vol.rows - 1);
        // row masks of the six 32-column blocks the strip can touch (halo left, its four quarters, halo
        // right) over the <= 5 row blocks of its 33 rows: ONE flag load per lane (lane = 5 k + j: column
        // block k, row block j), a ballot, and the masks are rebuilt from the ballot bits
        unsigned long long v[6] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
        const int rb_lo = max(r_first - 1, 0) >> 3, rb_hi = min(r_last + 1, vol.rows - 1) >> 3;
        const int nrb = rb_hi - rb_lo + 1;
        unsigned char f = 0;
        {
            const int k = (int)lane / 5, j = (int)lane % 5, cbk = cb - 1 + k;
            if (lane < 30 && j < nrb && cbk >= 0 && cbk < flags.col_blocks)
                f = __ldg(flags.data + ((int64_t)s * flags.col_blocks + cbk) * flags.row_blocks + rb_lo + j);
        }
        const unsigned ball = __ballot_sync(0xffffffffu, f != 0);
        if ((ball & 0x01ffffe0u) == 0u) return;              // no hit block in the strip's own four quarters
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            if (j >= nrb) break;
            const int rb = rb_lo + j;
            const int lo = max(8 * rb, r_first - 1) - (r_first - 1), hi = min(8 * rb + 7, r_last + 1) - (r_first - 1);   // local rows
            const unsigned long long bits = ((hi + 1 >= 64 ? ~0ull : (1ull << (hi + 1)) - 1ull)) & ~((1ull << lo) - 1ull);
#pragma unroll
            for (int k = 0; k < 6; ++k)
                if ((ball >> (5 * k + j)) & 1u) v[k] |= bits;
        }
        // tested rows are local rows 1 .. r_last - r_first + 1; a strip without a hit cannot emit anything
        const int n_tested = r_last - r_first + 1;
        const unsigned long long test = (v[1] | v[2] | v[3] | v[4]) & (((1ull << (n_tested + 1)) - 1ull) & ~1ull);
        if (test == 0ull) return;
        need = test | (test << 1) | (test >> 1);
        const unsigned quarter = lane >> 3;
        valid_q = quarter == 0 ? v[1] : quarter == 1 ? v[2] : quarter == 2 ? v[3] : v[4];
        valid_h = lane == 0 ? v[0] : v[5];
    }
    const int nvalid = min(max(vol.cols - c, 0), 4);       // valid columns of this lane
    const bool edge_lane = (lane == 0) || (lane == 31);
    const int halo_col = lane == 0 ? c - 1 : c + 4;
    const bool halo_ok = edge_lane && halo_col >= 0 && halo_col < vol.cols;
    const int halo_off = lane == 0 ? -1 : 4;
    const float ninf = -INFINITY;
    // rows outside the plane are never loaded either: fold the bounds into the row mask once
    // (local row l is plane row r_first - 1 + l), so that the streaming loop tests one mask bit per row
    {
        const int first_ok = r_first == 0 ? 1 : 0;                             // local row 0 is row -1 of the plane
        const int n_ok = min(kBandRows + 2, vol.rows - (r_first - 1));         // local rows below this are inside
        unsigned long long inside = (n_ok >= 64 ? ~0ull : (1ull << n_ok) - 1ull);
        if (first_ok) inside &= ~1ull;
        need &= inside;
    }
    // three running row pointers (one per ring slot), advanced by kGroup rows per group
    const int64_t step = (int64_t)kGroup * vol.pitch;
    const float *pr[kGroup];
#pragma unroll
    for (int k = 0; k < kGroup; ++k)
        pr[k] = vol.data + (int64_t)s * vol.plane + (int64_t)(r_first - 1 + k) * vol.pitch + c;

    const bool strip_ragged = (c - 4 * (int)lane) + 128 > vol.cols;             // warp uniform: the plane's last strip
    // needq / needh: rows this lane loads its four columns / its halo column from (wanted by the strip AND
    // stored by the producer: blocks without a hit were never written and read as -inf)
    const unsigned long long needq = need & valid_q, needh = need & valid_h;
    auto load_row = [&](bool want_q, bool want_h, const float *ptr) -> RowRegs {
        RowRegs o;
        o.q = make_float4(ninf, ninf, ninf, ninf);
        o.halo = ninf;
        if (want_q && nvalid > 0) o.q = __ldg(reinterpret_cast<const float4 *>(ptr));   // pitch-padded: in bounds
        if (want_h && halo_ok) o.halo = __ldg(ptr + halo_off);
        return o;
    };
    // window rows as [left, x, y, z, w, right]; the three rows rotate through w[0..2]
    // (kGroup is a multiple of 3, so the roles are static inside the unrolled group)
    static_assert(kGroup % 3 == 0, "the window rotates with period 3");
    float w[3][6];
    auto widen = [&](const RowRegs &g, float (&o)[6]) {
        float4 q = g.q;
        if (strip_ragged) {
            if (nvalid < 1) q.x = ninf;
            if (nvalid < 2) q.y = ninf;
            if (nvalid < 3) q.z = ninf;
            if (nvalid < 4) q.w = ninf;
        }
        const float l = __shfl_up_sync(0xffffffffu, q.w, 1);
        const float rgt = __shfl_down_sync(0xffffffffu, q.x, 1);
        o[0] = lane == 0 ? g.halo : l;
        o[1] = q.x; o[2] = q.y; o[3] = q.z; o[4] = q.w;
        o[5] = lane == 31 ? g.halo : rgt;
    };

    // 2-D local maxima above the threshold are queued (16 bits: local row, local column) and
    // resolved against the neighbouring slices outside the streaming loop, so that the rare,
    // register-hungry part stays out of it
    int qcount = 0;                                         // warp uniform

    // ring of kGroup rows in flight: a row's slot is reloaded (kGroup rows ahead) as soon as
    // it has moved into the window
    RowRegs ring[kGroup];
#pragma unroll
    for (int k = 0; k < kGroup; ++k) {
        ring[k] = load_row((needq >> k) & 1ull, (needh >> k) & 1ull, pr[k]);
        pr[k] += step;
    }
    unsigned long long ahead_q = needq >> kGroup, ahead_h = needh >> kGroup;      // bit k: the row that ring[k] loads next
#pragma unroll
    for (int k = 0; k < 6; ++k) { w[0][k] = ninf; w[1][k] = ninf; w[2][k] = ninf; }

    constexpr int n_groups = (kBandRows + 2) / kGroup;
    static_assert((kBandRows + 2) % kGroup == 0, "band + halo rows must be whole groups");
    const unsigned lt = (1u << lane) - 1u;
    const int rows_here = min(kBandRows, vol.rows - r_first);    // tested local rows are 1 .. rows_here
    // bit k + 1: is the row tested at step k of the current group (local row rg + k - 1) inside 1 .. rows_here?
    unsigned long long live_bits = ((rows_here >= 63 ? ~0ull : (1ull << (rows_here + 1)) - 1ull) & ~1ull) << 2;
    int g = 0;
    while (true) {
#pragma unroll 1
        for (; g < n_groups && qcount <= kQueueCap - kGroup * 128; ++g) {
            const int rg = g * kGroup;                      // local index of the row in ring[0]
#pragma unroll
            for (int k = 0; k < kGroup; ++k) {
                // local row rg + k enters slot (k + 2) % 3; the tested row rg + k - 1 sits in
                // slot (k + 1) % 3, the row above it in slot k % 3
                float (&up)[6] = w[k % 3];
                float (&mid)[6] = w[(k + 1) % 3];
                float (&dn)[6] = w[(k + 2) % 3];
                // (skipping the widening / the test of rows outside the hit blocks with uniform branches
                // on the row masks was measured: 30 % SLOWER, the branches break the unrolled rotation)
                widen(ring[k], dn);
                if (g + 1 < n_groups) {
                    ring[k] = load_row((ahead_q >> k) & 1ull, (ahead_h >> k) & 1ull, pr[k]);
                    pr[k] += step;
                }
                const int rl = rg + k - 1;
                const float top = fmaxf(fmaxf(mid[1], mid[2]), fmaxf(mid[3], mid[4]));
                const bool live = (live_bits >> (k + 1)) & 1ull;
                if (!__any_sync(0xffffffffu, live && top > thr)) continue;
                // max over the 8 in-slice neighbours of voxel v: columns v and v+2 whole, column
                // v+1 without the centre
                float colmax[6], pair[4];
#pragma unroll
                for (int j = 0; j < 6; ++j) colmax[j] = fmaxf(fmaxf(up[j], mid[j]), dn[j]);
#pragma unroll
                for (int v = 0; v < 4; ++v) pair[v] = fmaxf(up[v + 1], dn[v + 1]);
                unsigned mine = 0;
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const float val = mid[v + 1];
                    const float nb = fmaxf(fmaxf(colmax[v], colmax[v + 2]), pair[v]);
                    if (live && val > thr && !(nb > val)) mine |= 1u << v;
                }
                if (!__any_sync(0xffffffffu, mine != 0)) continue;
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const bool cand = (mine >> v) & 1u;
                    const unsigned m = __ballot_sync(0xffffffffu, cand);
                    if (cand) queue[qcount + __popc(m & lt)] = (unsigned short)((rl << 7) | (4 * lane + v));
                    qcount += __popc(m);
                }
            }
            ahead_q >>= kGroup;
            ahead_h >>= kGroup;
            live_bits >>= kGroup;
        }
        // ---- resolve the queued maxima (cross-slice test, plateau test, append) ----
        __syncwarp();
        for (int q0 = 0; q0 < qcount; q0 += 32) {
            const int q = q0 + (int)lane;
            const bool have = q < qcount;
            const unsigned e = have ? queue[q] : 0u;
            const int r = r_first - 1 + (int)(e >> 7);
            const int cc = c - 4 * (int)lane + (int)(e & 127u);
            const float val = have ? vol.at(s, r, cc) : 0.f;
            resolve_and_append(vol, s, r, cc, val, have, 1, thr, transposed, slice_sigma, bs, lane);
        }
        __syncwarp();
        qcount = 0;
        if (g >= n_groups) break;
    }
}

// kWarps strips side by side per CTA.  With hit flags most strips return at once: one warp per CTA
// then frees its slot immediately instead of idling next to a busy neighbour.
template <int kGroup, int kBandRows, int kWarps, int kMinCtas>
__global__ void __launch_bounds__(32 * kWarps, kMinCtas)
nms_window_kernel(Volume vol, float thr, bool transposed, const double *__restrict__ slice_sigma,
                  BlobSpace bs, HitFlags flags) {
    __shared__ unsigned short s_queue[kWarps][kQueueCap];
    if ((blockIdx.x | blockIdx.y | blockIdx.z | threadIdx.x) == 0) bs.ctr->t_extrema = globaltimer_ns();
    nms_strip<kGroup, kBandRows, kWarps>(vol, thr, transposed, slice_sigma, bs, flags, blockIdx.z, blockIdx.y, blockIdx.x,
                                         s_queue[threadIdx.x >> 5]);
}

// ---- seeds of the tensor-core column pass (HitFlags::seeds) ------------------------------
// The column pass has already tested every value above the threshold against the in-slice neighbours
// it holds in registers; what it could not see (neighbours owned by another thread-chunk, warp or CTA)
// is finished here, one seed per lane: the 8 in-slice neighbours, then the two neighbouring slices.
// A few thousand seeds per frame instead of a walk over every block with a hit.
__global__ void __launch_bounds__(256)
nms_seed_kernel(Volume vol, float thr, int h, bool transposed, const double *__restrict__ slice_sigma, BlobSpace bs,
                HitFlags flags, int strips_x, int bands_y) {
    __shared__ unsigned short s_queue[8][kQueueCap];
    if ((blockIdx.x | threadIdx.x) == 0) bs.ctr->t_extrema = globaltimer_ns();
    const int n = *flags.n_seeds;
    const unsigned lane = threadIdx.x & 31;
    if (n > flags.seed_cap) {
        // More seeds than the list holds (flat noise above the threshold): the list is incomplete, the strip
        // kernel's walk over the slices runs instead, on this grid (8 strips side by side per CTA).
        const int total = strips_x * bands_y * vol.S;
        for (int idx = blockIdx.x; idx < total; idx += gridDim.x) {
            const int x = idx % strips_x, t = idx / strips_x;
            nms_strip<3, 31, 8>(vol, thr, transposed, slice_sigma, bs, flags, t / bands_y, t % bands_y, x,
                                s_queue[threadIdx.x >> 5]);
            __syncwarp();
        }
        return;
    }
    for (int base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; base < n; base += gridDim.x * blockDim.x) {
        const int i = base + (int)lane;             // whole warps stay convergent
        bool cand = i < n;
        int s = 0, r = 0, c = 0;
        float val = 0.f;
        if (cand) {
            const unsigned long long key = flags.seeds[i];
            s = (int)(key >> 48); r = (int)((key >> 24) & 0xffffffull); c = (int)(key & 0xffffffull);
            val = __ldg(vol.data + (int64_t)s * vol.plane + (int64_t)r * vol.pitch + c);      // its block has a hit: stored
            float nb[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = j < 4 ? j : j + 1;
                const int rr = r + k / 3 - 1, cc = c + k % 3 - 1;
                nb[j] = (rr >= 0 && rr < vol.rows && cc >= 0 && cc < vol.cols) ? vol.at(s, rr, cc) : -INFINITY;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) cand = cand && !(nb[j] > val);
        }
        if (!__any_sync(0xffffffffu, cand)) continue;
        resolve_and_append(vol, s, r, c, val, cand, h, thr, transposed, slice_sigma, bs, lane);
    }
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
    if ((blockIdx.x | blockIdx.y | blockIdx.z | threadIdx.x) == 0) bs.ctr->t_extrema = globaltimer_ns();
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
            resolve_and_append(vol, s, r, c + k, val, cand, h, thr, transposed, slice_sigma, bs, lane);
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
        Voxel va = (a < n) ? bs.plateau[a] : Voxel{-9, -9, -9, 0, 0.0};
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
        z.t_start = globaltimer_ns();
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

// ---- float64 tier (Detector.run(img, dtype=np.float64), convolve.py:76-77): the simple form ----
// One thread per voxel; a voxel above the threshold walks its whole (2h+1)^3 block.  Slow is fine:
// this is the oracle-grade path (T1 of the near-tie classifier), not the production one.
__global__ void __launch_bounds__(256)
nms_point_f64_kernel(VolumeT<double> vol, double thr, int h, const double *__restrict__ slice_sigma, BlobSpace bs) {
    if ((blockIdx.x | blockIdx.y | blockIdx.z | threadIdx.x) == 0) bs.ctr->t_extrema = globaltimer_ns();
    const int s = blockIdx.z, r = blockIdx.y;
    const unsigned lane = threadIdx.x & 31;
    for (int c0 = blockIdx.x * 256; c0 < vol.cols; c0 += gridDim.x * 256) {      // whole warps stay convergent
        const int c = c0 + (int)threadIdx.x;
        const bool in = c < vol.cols;
        const double val = in ? vol.at(s, r, c) : 0.0;
        bool cand = in && val > thr;
        if (!__any_sync(0xffffffffu, cand)) continue;
        if (cand && h == 1) {       // the in-slice part of the 3x3x3 test (resolve_and_append does the rest)
            for (int j = 0; j < 9 && cand; ++j) {
                const int rr = r + j / 3 - 1, cc = c + j % 3 - 1;
                if (j != 4 && rr >= 0 && rr < vol.rows && cc >= 0 && cc < vol.cols && vol.at(s, rr, cc) > val) cand = false;
            }
        }
        resolve_and_append<double>(vol, s, r, c, val, cand, h, thr, false, slice_sigma, bs, lane);
    }
}

cudaError_t launch_extrema_f64(const double *d_slices, int S, int rows, int cols, const double *d_slice_sigma,
                               double threshold, int half, const BlobSpace &bs, cudaStream_t st) {
    VolumeT<double> vol{d_slices, S, rows, cols, cols, (int64_t)rows * cols};
    nms_point_f64_kernel<<<dim3((cols + 255) / 256, rows, S), 256, 0, st>>>(vol, threshold, half, d_slice_sigma, bs);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    plateau_kernel<<<148, 256, 0, st>>>(bs, S, false, d_slice_sigma);
    return cudaGetLastError();
}

static int sm_count() {
    static const int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

cudaError_t launch_extrema(const float *d_slices, int S, int rows, int cols, int64_t pitch,
                           int64_t plane, bool transposed, const double *d_slice_sigma,
                           float threshold, int half, const BlobSpace &bs, cudaStream_t st, HitFlags flags) {
    Volume vol{d_slices, S, rows, cols, pitch, plane};
    if (flags.data != nullptr) {
        vol.valid = flags.data;
        vol.v_row_blocks = flags.row_blocks;
        vol.v_col_blocks = flags.col_blocks;
    }
    const bool vec4 = (pitch % 4 == 0) && (plane % 4 == 0) &&
                      ((reinterpret_cast<uintptr_t>(d_slices) & 15u) == 0);
    const dim3 grid((cols + kNmsCols - 1) / kNmsCols, (rows + kNmsRows - 1) / kNmsRows, S);
    if (vec4 && half == 1) {
        // 3 rows in flight per lane, 31 tested rows per warp, 4 CTAs per SM: the best of the
        // measured variants ((6,34,3) ties; (6,34,2), (3,61,4), (3,31,3) are 5..10 % slower)
        constexpr int kBand = 31;
        const int tiles_y = (rows + kBand - 1) / kBand;
        if (flags.data != nullptr && flags.seeds != nullptr) {
            nms_seed_kernel<<<sm_count(), 256, 0, st>>>(vol, threshold, half, transposed, d_slice_sigma, bs, flags,
                                                        (cols + 1023) / 1024, tiles_y);
        } else if (flags.data != nullptr)
            nms_window_kernel<3, kBand, 1, 32><<<dim3((cols + 127) / 128, tiles_y, S), 32, 0, st>>>(
                vol, threshold, transposed, d_slice_sigma, bs, flags);
        else
            nms_window_kernel<3, kBand, 8, 4><<<dim3((cols + 1023) / 1024, tiles_y, S), 256, 0, st>>>(
                vol, threshold, transposed, d_slice_sigma, bs, flags);
    } else if (vec4)
        nms_kernel<4><<<grid, 256, 0, st>>>(vol, threshold, half, transposed, d_slice_sigma, bs);
    else
        nms_kernel<1><<<grid, 256, 0, st>>>(vol, threshold, half, transposed, d_slice_sigma, bs);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    plateau_kernel<<<148, 256, 0, st>>>(bs, S, transposed, d_slice_sigma);
    return cudaGetLastError();
}

}  // namespace dogblob
