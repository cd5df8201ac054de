// Overlap pruning on the GPU with the reference's exact sequential semantics.
//
// Replaces prune_overlaps / _overlap_matrix (pkg/src/dogblob/detector.py:221-280),
// which the paper left on the CPU.  The reference repeats
//   { dense N x N overlap matrix; take the row-major-first pair (i < j) of the
//     response-sorted list with overlap > thr; blob i keeps centre/response,
//     radius <- mean, sigma <- radius / sqrt 2, OR the boundary flags; delete j }
// until no pair offends.  Here the blobs are bucketed on a uniform grid whose
// cell is >= 2 r_max (an offending pair needs d < r_i + r_j, and merged radii
// never exceed r_max), `first[i]` caches the smallest offending partner j > i,
// and one persistent CTA replays the merge order, touching only the 3x3 cell
// neighbourhoods a merge can change.  All overlap arithmetic is float64 with
// the operation order of the reference (compiled with -fmad=false).
#include <float.h>
#include <cstdlib>

#include "common.cuh"

namespace dogblob {

namespace {

constexpr double kPi = 3.141592653589793;
constexpr double kSqrt2 = 1.4142135623730951;

// hypot for the centre distance: exact sqrt for integer offsets (the pipeline
// case), one Newton correction otherwise; both agree with a correctly rounded
// hypot except on rare half-ulp cases.
__device__ __forceinline__ double centre_distance(double dx, double dy) {
    const double s = dx * dx + dy * dy;
    if (dx == rint(dx) && dy == rint(dy) && fabs(dx) < 33554432.0 && fabs(dy) < 33554432.0)
        return sqrt(s);
    return hypot(dx, dy);
}

// normalised overlap of matrix entry [i][j] (detector.py:221-247)
__device__ double overlap_ij(double xi, double yi, double ri, double xj, double yj, double rj) {
    const double d = centre_distance(xi - xj, yi - yj);
    const double rmin = fmin(ri, rj), rmax = fmax(ri, rj);
    if (d <= rmax - rmin) return 1.0;
    if (!(d < ri + rj) || !(d > 0.0)) return 0.0;
    double c1 = (d * d + ri * ri - rj * rj) / (2.0 * d * ri);
    double c2 = (d * d + rj * rj - ri * ri) / (2.0 * d * rj);
    c1 = fmin(fmax(c1, -1.0), 1.0);
    c2 = fmin(fmax(c2, -1.0), 1.0);
    const double a1 = ri * ri * acos(c1);
    const double a2 = rj * rj * acos(c2);
    double q = (-d + ri + rj) * (d + ri - rj) * (d - ri + rj) * (d + ri + rj);
    q = fmax(q, 0.0);
    const double s = 0.5 * sqrt(q);
    return (a1 + a2 - s) / (kPi * rmin * rmin);
}

struct Grid {
    double x0, y0, cell;
    int gx, gy;
    __device__ __forceinline__ int cx(double x) const {
        int c = (int)floor((x - x0) / cell);
        return min(max(c, 0), gx - 1);
    }
    __device__ __forceinline__ int cy(double y) const {
        int c = (int)floor((y - y0) / cell);
        return min(max(c, 0), gy - 1);
    }
};

template <typename T, typename Op>
__device__ T block_reduce(T v, Op op, T *scratch /* >= 33 */, int nw = 0 /* live warps, 0 = all */) {
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (nw == 0) nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (lane == 0) scratch[w] = v;
    __syncthreads();
    if (w == 0) {
        T r = scratch[lane < nw ? lane : 0];
        for (int o = 16; o > 0; o >>= 1) r = op(r, __shfl_xor_sync(0xffffffffu, r, o));
        if (lane == 0) scratch[32] = r;
    }
    __syncthreads();
    return scratch[32];
}

// =========================================================================================
// Frames above the single-CTA limit: ONE whole-GPU kernel, phases chained on the device.
//
// The work is a sequence of phases (order the candidates, bucket them, first partners,
// radius bounds, parts, per-part merge loops, packing); how many bound sweeps are needed and
// how many parts exist is only known on the device.  Work items of all phases are numbered
// in one global order and handed out by an atomic ticket; phase k+1 is *published* (type,
// first item, item count) by the CTA that completes the last item of phase k, so the
// publication doubles as a grid-wide barrier.  A CTA only ever waits for items with smaller
// tickets, and every ticket is held by a CTA that is already running: no co-residency
// assumption, no cooperative launch, no host round trip, and a frame that finished in
// finalize_small_kernel costs one immediate return.
//
// Everything that another SM may have written earlier in this kernel is read through L2
// (ld.global.cg): L1 is not coherent across SMs and several arrays are re-used between phases.

enum PhaseType : int {
    PH_RANK = 0, PH_SCATTER, PH_COUNT, PH_SCAN, PH_FILL, PH_FIRST, PH_SWEEP, PH_SATURATE, PH_UNION,
    PH_LINK, PH_MERGE, PH_PACK_COUNT, PH_PACK_WRITE, PH_END
};

constexpr int kLargeThreads = 256;
constexpr int kItemBlobs = 256;       // thread-per-blob phases
constexpr int kRankParts = 8;         // a candidate's rank is the sum of <= 8 partial ranks
constexpr int kWarpBlobs = 32;        // warp-per-blob phases: 4 blobs per warp
constexpr int kPackBlobs = 1024;      // 4 per thread
constexpr int kMaxSweeps = 96;

__device__ __forceinline__ int ldcg_i(const int *p) { return __ldcg(p); }
__device__ __forceinline__ dogblob_blob ldcg_blob(const dogblob_blob *p) {
    union { int4 q[3]; dogblob_blob b; } u;
    const int4 *s = reinterpret_cast<const int4 *>(p);
    u.q[0] = __ldcg(s); u.q[1] = __ldcg(s + 1); u.q[2] = __ldcg(s + 2);
    return u.b;
}
__device__ __forceinline__ double ldcg_d(const double *p) { return __ldcg(p); }
__device__ __forceinline__ double ldcg_bound(const BlobSpace &bs, int i) {
    return __longlong_as_double((long long)__ldcg(bs.bound + i));
}
__device__ __forceinline__ unsigned long long now_ns() { return globaltimer_ns(); }

__device__ __forceinline__ int clamp_ns(unsigned long long a, unsigned long long b) {
    return b > a ? (int)min(b - a, 2000000000ull) : 0;
}
// the kernel that finishes a frame fills the header's device-side stage times
__device__ void write_stage_times(const Counters &c, dogblob_result_header *hdr) {
    const unsigned long long t_end = globaltimer_ns();
    hdr->conv_ns = c.t_extrema ? clamp_ns(c.t_start, c.t_extrema) : 0;
    hdr->extrema_ns = c.t_extrema ? clamp_ns(c.t_extrema, c.t_prune) : 0;
    hdr->prune_ns = clamp_ns(c.t_prune, t_end);
}
__device__ void atomic_min_double(double *addr, double v) {
    unsigned long long *a = reinterpret_cast<unsigned long long *>(addr);
    unsigned long long old = *a;
    while (v < __longlong_as_double((long long)old)) {
        const unsigned long long seen = atomicCAS(a, old, (unsigned long long)__double_as_longlong(v));
        if (seen == old) break;
        old = seen;
    }
}
__device__ void atomic_max_double(double *addr, double v) {
    unsigned long long *a = reinterpret_cast<unsigned long long *>(addr);
    unsigned long long old = *a;
    while (v > __longlong_as_double((long long)old)) {
        const unsigned long long seen = atomicCAS(a, old, (unsigned long long)__double_as_longlong(v));
        if (seen == old) break;
        old = seen;
    }
}

__device__ __forceinline__ Grid load_grid_cg(const BlobSpace &bs) {
    Grid g;
    g.x0 = ldcg_d(bs.grid_params + 0);
    g.y0 = ldcg_d(bs.grid_params + 1);
    g.cell = ldcg_d(bs.grid_params + 2);
    g.gx = (int)ldcg_d(bs.grid_params + 3);
    g.gy = (int)ldcg_d(bs.grid_params + 4);
    return g;
}

struct SortKey { double resp, y, x, sigma; };
__device__ __forceinline__ bool key_before(const SortKey &a, int ia, const SortKey &b, int ib) {
    // sorted(key=(-response, y, x, sigma)); ties keep input order
    if (a.resp != b.resp) return a.resp > b.resp;
    if (a.y != b.y) return a.y < b.y;
    if (a.x != b.x) return a.x < b.x;
    if (a.sigma != b.sigma) return a.sigma < b.sigma;
    return ia < ib;
}

// the geometric part of a record: x, y (first 16 bytes) and sigma, radius (next 16)
struct XYR { double x, y, r; };
__device__ __forceinline__ XYR ldcg_xyr(const dogblob_blob *p) {
    const int4 *s = reinterpret_cast<const int4 *>(p);
    const int4 a = __ldcg(s), b = __ldcg(s + 1);
    XYR o;
    o.x = __longlong_as_double(((long long)(unsigned)a.y << 32) | (unsigned)a.x);
    o.y = __longlong_as_double(((long long)(unsigned)a.w << 32) | (unsigned)a.z);
    o.r = __longlong_as_double(((long long)(unsigned)b.w << 32) | (unsigned)b.z);
    return o;
}
__device__ __forceinline__ double2 ldcg_xy(const dogblob_blob *p) {
    const int4 a = __ldcg(reinterpret_cast<const int4 *>(p));
    return make_double2(__longlong_as_double(((long long)(unsigned)a.y << 32) | (unsigned)a.x),
                        __longlong_as_double(((long long)(unsigned)a.w << 32) | (unsigned)a.z));
}

// Visit every blob bucketed in the 3 x 3 cells around (cx, cy).  The three cells of one grid
// row are adjacent in cell order, so their items are ONE contiguous range of cell_items: the
// warp splits into three lane groups (lane % 3 = row), each striding its row's range, and a
// typical neighbourhood is covered in a single step.  f(k) is called with a blob index.
template <typename F>
__device__ __forceinline__ void for_neighbours_warp(const BlobSpace &bs, const Grid &g, int cx, int cy,
                                                    int lane, F f) {
    const int row = lane % 3, t = lane / 3, nt = row < 2 ? 11 : 10;
    const int yy = cy - 1 + row;
    if (yy < 0 || yy >= g.gy) return;
    const int c0 = yy * g.gx + max(cx - 1, 0), c1 = yy * g.gx + min(cx + 1, g.gx - 1);
    const int e = ldcg_i(bs.cell_start + c1 + 1);
    for (int p = ldcg_i(bs.cell_start + c0) + t; p < e; p += nt) f(ldcg_i(bs.cell_items + p));
}

// smallest alive j > i offending with i (whole warp)
__device__ int scan_first_partner(const BlobSpace &bs, const Grid &g, int i, double thr, int lane) {
    const XYR bi = ldcg_xyr(bs.sorted + i);
    int best = INT_MAX;
    for_neighbours_warp(bs, g, g.cx(bi.x), g.cy(bi.y), lane, [&](int j) {
        if (j <= i || j >= best || !(ldcg_i(bs.alive + j) & 1)) return;
        const XYR bj = ldcg_xyr(bs.sorted + j);
        if (overlap_ij(bi.x, bi.y, bi.r, bj.x, bj.y, bj.r) > thr) best = j;
    });
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    return best;
}

// The reference's loop is sequential, but merges only interact through blobs that can
// overlap.  ub(a) bounds every radius blob a can ever take: a's radius only changes when a
// (the lower index) absorbs some b > a and becomes the mean, so
//     ub(a) = max(r_a, max{ ub(b) : b > a, dist(a, b) < ub(a) + ub(b) }),
// taken as the least fixed point from below (monotone in-place sweeps until one full sweep
// changes nothing; any pre-fixed point, e.g. the global r_max everywhere, is a valid
// fallback).  By induction no merge ever joins blobs that are not linked by
// "dist < ub(a) + ub(b)", so the connected parts of that graph evolve independently and the
// global row-major-first order restricted to a part is that part's own sequential order:
// one warp replays each part's merge loop on its own, all parts at once.
__device__ __forceinline__ int comp_find(int *comp, int x) {
    int p = __ldcg(comp + x);
    while (p != x) { x = p; p = __ldcg(comp + x); }
    return x;
}
__device__ void comp_union(int *comp, int a, int b) {
    while (true) {
        a = comp_find(comp, a);
        b = comp_find(comp, b);
        if (a == b) return;
        if (a > b) { int t = a; a = b; b = t; }
        if (atomicCAS(&comp[b], b, a) == b) return;
    }
}

// offending rows of a part live in a linked list: head in cmin[root], links in cell_of[]
// (free after the grid is built); bit 1 of alive[] = "listed"
__device__ __forceinline__ void list_push(const BlobSpace &bs, int root, int k) {
    if (!(atomicOr(&bs.alive[k], 2) & 2)) bs.cell_of[k] = atomicExch(&bs.cmin[root], k);
}

// one warp merges row i with its first partner and repairs the cached partners around it
__device__ void merge_row(const BlobSpace &bs, const Grid &g, int root, int i, double thr, int lane) {
    const int j = ldcg_i(bs.first + i);
    if (lane == 0) {
        dogblob_blob a = ldcg_blob(bs.sorted + i);
        const dogblob_blob w = ldcg_blob(bs.sorted + j);
        const double nr = 0.5 * (a.radius + w.radius);
        a.radius = nr;
        a.sigma = nr / kSqrt2;
        a.flags |= (w.flags & DOGBLOB_BLOB_SCALE_EDGE) | DOGBLOB_BLOB_MERGED;
        a.slice = -1;
        bs.sorted[i] = a;
        bs.alive[j] = 0;
        __threadfence();
    }
    __syncwarp();
    const XYR bi = ldcg_xyr(bs.sorted + i);
    const double2 bj = ldcg_xy(bs.sorted + j);
    // (a) first[i] again; (b) rows k < i of this part had no partner and can only gain i
    int best = INT_MAX;
    for_neighbours_warp(bs, g, g.cx(bi.x), g.cy(bi.y), lane, [&](int k) {
        if (k == i || !(ldcg_i(bs.alive + k) & 1)) return;
        const XYR bk = ldcg_xyr(bs.sorted + k);
        if (k > i) {
            if (k < best && overlap_ij(bi.x, bi.y, bi.r, bk.x, bk.y, bk.r) > thr) best = k;
        } else if (overlap_ij(bk.x, bk.y, bk.r, bi.x, bi.y, bi.r) > thr) {
            bs.first[k] = i;
            list_push(bs, root, k);
        }
    });
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) bs.first[i] = (best == INT_MAX) ? -1 : best;
    // (c) rows that pointed at the deleted blob need a new partner: collect them (ballot per
    // grid row of the neighbourhood), then the whole warp rescans each
    {
        const int cx = g.cx(bj.x), cy = g.cy(bj.y);
        for (int yy = max(cy - 1, 0); yy <= min(cy + 1, g.gy - 1); ++yy) {
            const int s0 = ldcg_i(bs.cell_start + yy * g.gx + max(cx - 1, 0));
            const int e = ldcg_i(bs.cell_start + yy * g.gx + min(cx + 1, g.gx - 1) + 1);
            for (int p0 = s0; p0 < e; p0 += 32) {
                const int p = p0 + lane;
                const int k = p < e ? ldcg_i(bs.cell_items + p) : -1;
                const bool hit = k >= 0 && k != i && (ldcg_i(bs.alive + k) & 1) &&
                                 ldcg_i(bs.first + k) == j;
                unsigned m = __ballot_sync(0xffffffffu, hit);
                while (m) {
                    const int src = __ffs(m) - 1;
                    m &= m - 1;
                    const int kk = __shfl_sync(0xffffffffu, k, src);
                    const int b2 = scan_first_partner(bs, g, kk, thr, lane);
                    if (lane == 0) bs.first[kk] = (b2 == INT_MAX) ? -1 : b2;   // kk stays listed
                }
            }
        }
    }
    __threadfence();
    __syncwarp();
}

// the whole merge loop of one part, by one warp: repeatedly the smallest listed row that is
// alive and still has a partner; rows that lost their partner are unlinked on the way
__device__ int merge_part(const BlobSpace &bs, const Grid &g, int root, double thr, int lane) {
    int merges = 0;
    while (true) {
        int best = INT_MAX;
        if (lane == 0) {
            int prev = -1;
            int e = ldcg_i(bs.cmin + root);
            while (e >= 0) {
                const int nxt = ldcg_i(bs.cell_of + e);
                if ((ldcg_i(bs.alive + e) & 1) && ldcg_i(bs.first + e) >= 0) {
                    best = min(best, e);
                    prev = e;
                } else {                               // unlink; it may be pushed again later
                    if (prev < 0) bs.cmin[root] = nxt; else bs.cell_of[prev] = nxt;
                    atomicAnd(&bs.alive[e], ~2);
                }
                e = nxt;
            }
            __threadfence();
        }
        best = __shfl_sync(0xffffffffu, best, 0);
        if (best == INT_MAX) break;
        merge_row(bs, g, root, best, thr, lane);
        ++merges;
    }
    return merges;
}

// ranking: the j range is cut into nj <= kRankParts chunks (multiples of 256)
__device__ __forceinline__ int rank_chunk(int n) {
    const int per = (n + kRankParts - 1) / kRankParts;
    return max(kItemBlobs, (per + kItemBlobs - 1) / kItemBlobs * kItemBlobs);
}
__device__ int phase_items(int type, int n, int n_roots) {
    switch (type) {
        case PH_RANK: {
            const int cj = rank_chunk(n);
            return ((n + kItemBlobs - 1) / kItemBlobs) * ((n + cj - 1) / cj);
        }
        case PH_SCAN: return 1;
        case PH_FIRST: case PH_SWEEP: case PH_UNION: return (n + kWarpBlobs - 1) / kWarpBlobs;
        case PH_MERGE: return (n_roots + 7) / 8;
        case PH_PACK_COUNT: case PH_PACK_WRITE: return (n + kPackBlobs - 1) / kPackBlobs;
        default: return (n + kItemBlobs - 1) / kItemBlobs;
    }
}

__global__ void __launch_bounds__(kLargeThreads)
prune_large_kernel(BlobSpace bs, double thr, int do_prune, dogblob_result_header *hdr,
                   dogblob_blob *out, int out_cap) {
    if (bs.ctr->small_done) return;
    PruneCtl *ctl = bs.ctl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = min(bs.ctr->n_candidates, bs.cap);
    __shared__ int s_type, s_item, s_count, s_last;
    __shared__ double sd[33];
    __shared__ int si[33];
    __shared__ SortKey s_keys[kItemBlobs];
    const bool pruning = do_prune && n >= 2;
    int cur = 0;                                   // phase this CTA looks at (thread 0)
    int ph_first = 0, ph_count = 0, ph_type = PH_RANK;

    while (true) {
        // ---- take a ticket, find its phase (waiting for the publication = grid barrier) ----
        if (tid == 0) {
            const int t = (int)atomicAdd(&ctl->ticket, 1u);
            if (t == 0) {                          // the first ticket publishes phase 0
                ctl->phase[0].type = n > 0 ? PH_RANK : PH_PACK_WRITE;
                ctl->phase[0].first_item = 0;
                ctl->phase[0].n_items = n > 0 ? phase_items(PH_RANK, n, 0) : 1;
                ctl->ext[0] = DBL_MAX; ctl->ext[1] = -DBL_MAX;
                ctl->ext[2] = DBL_MAX; ctl->ext[3] = -DBL_MAX; ctl->ext[4] = 0.0;
                ctl->phase[0].t_ns = now_ns();
                __threadfence();
                *(volatile int *)&ctl->n_phases = 1;
            }
            int type;
            while (true) {
                while (*(volatile int *)&ctl->n_phases <= cur) __nanosleep(40);
                __threadfence();
                type = __ldcg(&ctl->phase[cur].type);
                ph_first = __ldcg(&ctl->phase[cur].first_item);
                ph_count = __ldcg(&ctl->phase[cur].n_items);
                if (type == PH_END || t < ph_first + ph_count) break;
                ++cur;
            }
            ph_type = type;
            s_type = type;
            s_item = t - ph_first;
            s_count = ph_count;
        }
        __syncthreads();
        const int type = s_type, item = s_item, ph_count_all = s_count;
        if (type == PH_END) return;

        // ---- the item ----
        switch (type) {
        case PH_RANK: {
            // partial rank of candidate i against j chunk jb; the partials live in eight arrays
            // that are free at this point.  The cell counters are cleared on the side.
            int *const part[kRankParts] = {bs.first, bs.alive, bs.comp, bs.cmin,
                                           bs.cell_of, bs.cell_items, bs.pl_count, bs.parent};
            const int cj = rank_chunk(n);
            const int nj = (n + cj - 1) / cj;
            const int ib = item / nj, jb = item % nj;
            const int i = ib * kItemBlobs + tid;
            SortKey mk = {0, 0, 0, 0};
            if (i < n) {
                const dogblob_blob me = ldcg_blob(bs.unsorted + i);
                mk = SortKey{me.response, me.y, me.x, me.sigma};
            }
            int rank = 0;
            const int jend = min(n, (jb + 1) * cj);
            for (int j0 = jb * cj; j0 < jend; j0 += kItemBlobs) {
                __syncthreads();
                if (j0 + tid < jend) {
                    const dogblob_blob o = ldcg_blob(bs.unsorted + j0 + tid);
                    s_keys[tid] = SortKey{o.response, o.y, o.x, o.sigma};
                }
                __syncthreads();
                const int lim = min(kItemBlobs, jend - j0);
                if (i < n)
                    for (int k = 0; k < lim; ++k) rank += key_before(s_keys[k], j0 + k, mk, i) ? 1 : 0;
            }
            if (i < n) part[jb][i] = rank;
            if (pruning)
                for (int c = item * kLargeThreads + tid; c <= kMaxCells; c += ph_count_all * kLargeThreads) {
                    bs.cell_start[c] = 0;
                    if (c < kMaxCells) bs.cell_fill[c] = 0;
                }
            break;
        }
        case PH_SCATTER: {
            int *const part[kRankParts] = {bs.first, bs.alive, bs.comp, bs.cmin,
                                           bs.cell_of, bs.cell_items, bs.pl_count, bs.parent};
            const int cj = rank_chunk(n);
            const int nj = (n + cj - 1) / cj;
            const int i = item * kItemBlobs + tid;
            double xmin = DBL_MAX, xmax = -DBL_MAX, ymin = DBL_MAX, ymax = -DBL_MAX, rmax = 0.0;
            if (i < n) {
                const dogblob_blob b = ldcg_blob(bs.unsorted + i);
                int rank = 0;
                for (int q = 0; q < nj; ++q) rank += ldcg_i(part[q] + i);
                bs.sorted[rank] = b;
                xmin = xmax = b.x; ymin = ymax = b.y; rmax = b.radius;
            }
            auto fmn = [](double a, double b) { return fmin(a, b); };
            auto fmx = [](double a, double b) { return fmax(a, b); };
            xmin = block_reduce(xmin, fmn, sd); xmax = block_reduce(xmax, fmx, sd);
            ymin = block_reduce(ymin, fmn, sd); ymax = block_reduce(ymax, fmx, sd);
            rmax = block_reduce(rmax, fmx, sd);
            if (tid == 0) {
                atomic_min_double(&ctl->ext[0], xmin); atomic_max_double(&ctl->ext[1], xmax);
                atomic_min_double(&ctl->ext[2], ymin); atomic_max_double(&ctl->ext[3], ymax);
                atomic_max_double(&ctl->ext[4], rmax);
            }
            break;
        }
        case PH_COUNT: {
            const Grid g = load_grid_cg(bs);
            const int i = item * kItemBlobs + tid;
            if (i < n) {
                const double2 b = ldcg_xy(bs.sorted + i);
                const int c = g.cy(b.y) * g.gx + g.cx(b.x);
                bs.cell_of[i] = c;
                bs.alive[i] = 1;
                atomicAdd(&bs.cell_start[c + 1], 1);
            }
            break;
        }
        case PH_SCAN: {                            // one CTA: cell_start[c] = blobs in cells < c
            const Grid g = load_grid_cg(bs);
            const int ncell = g.gx * g.gy;
            const int per = (ncell + kLargeThreads - 1) / kLargeThreads;
            const int c0 = 1 + tid * per, c1 = min(c0 + per, ncell + 1);
            int sum = 0;
            for (int c = c0; c < c1; ++c) sum += ldcg_i(bs.cell_start + c);
            int v = sum;
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += t;
            }
            if (lane == 31) si[warp] = v;
            __syncthreads();
            if (warp == 0) {
                int t = lane < kLargeThreads / 32 ? si[lane] : 0;
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, t, o);
                    if (lane >= o) t += u;
                }
                si[lane] = t;
            }
            __syncthreads();
            int run = (warp > 0 ? si[warp - 1] : 0) + v - sum;      // exclusive prefix of this thread
            for (int c = c0; c < c1; ++c) {
                run += ldcg_i(bs.cell_start + c);
                bs.cell_start[c] = run;
            }
            break;
        }
        case PH_FILL: {
            const int i = item * kItemBlobs + tid;
            if (i < n) {
                const int c = ldcg_i(bs.cell_of + i);
                const int slot = ldcg_i(bs.cell_start + c) + atomicAdd(&bs.cell_fill[c], 1);
                bs.cell_items[slot] = i;
            }
            break;
        }
        case PH_FIRST: {
            const Grid g = load_grid_cg(bs);
            for (int q = 0; q < kWarpBlobs / 8; ++q) {
                const int i = item * kWarpBlobs + warp * (kWarpBlobs / 8) + q;
                if (i >= n) break;
                const int best = scan_first_partner(bs, g, i, thr, lane);
                if (lane == 0) {
                    bs.first[i] = (best == INT_MAX) ? -1 : best;
                    bs.comp[i] = i;
                    bs.cmin[i] = -1;
                    bs.bound[i] = (unsigned long long)__double_as_longlong(ldcg_xyr(bs.sorted + i).r);
                }
            }
            break;
        }
        case PH_SWEEP: {
            const Grid g = load_grid_cg(bs);
            for (int q = 0; q < kWarpBlobs / 8; ++q) {
                const int i = item * kWarpBlobs + warp * (kWarpBlobs / 8) + q;
                if (i >= n) break;
                const double2 bi = ldcg_xy(bs.sorted + i);
                const double u0 = ldcg_bound(bs, i);
                double ui = u0;
                for_neighbours_warp(bs, g, g.cx(bi.x), g.cy(bi.y), lane, [&](int j) {
                    if (j <= i) return;
                    const double uj = ldcg_bound(bs, j);
                    if (uj <= ui) return;
                    const double2 bj = ldcg_xy(bs.sorted + j);
                    const double dx = bi.x - bj.x, dy = bi.y - bj.y, reach = ui + uj;
                    if (dx * dx + dy * dy < reach * reach * 1.0000001 + 1e-9) ui = uj;
                });
                for (int o = 16; o > 0; o >>= 1) ui = fmax(ui, __shfl_xor_sync(0xffffffffu, ui, o));
                if (lane == 0 && ui > u0) {
                    bs.bound[i] = (unsigned long long)__double_as_longlong(ui);
                    *(volatile int *)&ctl->changed = 1;
                }
            }
            break;
        }
        case PH_SATURATE: {                        // too many sweeps: r_max everywhere is a valid bound
            const int i = item * kItemBlobs + tid;
            if (i < n) bs.bound[i] = (unsigned long long)__double_as_longlong(ldcg_d(&ctl->ext[4]));
            break;
        }
        case PH_UNION: {
            const Grid g = load_grid_cg(bs);
            for (int q = 0; q < kWarpBlobs / 8; ++q) {
                const int i = item * kWarpBlobs + warp * (kWarpBlobs / 8) + q;
                if (i >= n) break;
                const double2 bi = ldcg_xy(bs.sorted + i);
                const double ui = ldcg_bound(bs, i);
                for_neighbours_warp(bs, g, g.cx(bi.x), g.cy(bi.y), lane, [&](int j) {
                    if (j <= i) return;
                    const double2 bj = ldcg_xy(bs.sorted + j);
                    const double dx = bi.x - bj.x, dy = bi.y - bj.y;
                    const double reach = ui + ldcg_bound(bs, j);
                    if (dx * dx + dy * dy < reach * reach * 1.0000001 + 1e-9) comp_union(bs.comp, i, j);
                });
            }
            break;
        }
        case PH_LINK: {
            const int i = item * kItemBlobs + tid;
            if (i < n) {
                const int root = comp_find(bs.comp, i);
                bs.comp[i] = root;
                if (ldcg_i(bs.first + i) >= 0) {
                    atomicOr(&bs.alive[i], 2);
                    const int old = atomicExch(&bs.cmin[root], i);
                    bs.cell_of[i] = old;
                    if (old < 0) bs.pl_count[atomicAdd(&ctl->n_roots, 1)] = root;   // list of active parts
                }
            }
            break;
        }
        case PH_MERGE: {
            const Grid g = load_grid_cg(bs);
            const int q = item * 8 + warp;
            if (q < __ldcg(&ctl->n_roots)) {
                const int m = merge_part(bs, g, ldcg_i(bs.pl_count + q), thr, lane);
                if (lane == 0 && m) atomicAdd(&ctl->merges, m);
            }
            break;
        }
        case PH_PACK_COUNT: {
            int keep = 0;
            for (int k = 0; k < kPackBlobs / kLargeThreads; ++k) {
                const int i = item * kPackBlobs + tid * (kPackBlobs / kLargeThreads) + k;
                keep += __syncthreads_count((i < n) && (!pruning || (ldcg_i(bs.alive + i) & 1)));
            }
            if (tid == 0) bs.cell_fill[item] = keep;
            break;
        }
        case PH_PACK_WRITE: {
            if (n == 0) break;
            constexpr int kPer = kPackBlobs / kLargeThreads;
            const int i0 = item * kPackBlobs + tid * kPer;
            int flag[kPer], mine = 0;
            for (int k = 0; k < kPer; ++k) {
                flag[k] = (i0 + k < n) && (!pruning || (ldcg_i(bs.alive + i0 + k) & 1));
                mine += flag[k];
            }
            int v = mine;
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += t;
            }
            if (lane == 31) si[warp] = v;
            __syncthreads();
            if (warp == 0) {
                int t = lane < kLargeThreads / 32 ? si[lane] : 0;
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, t, o);
                    if (lane >= o) t += u;
                }
                si[lane] = t;
            }
            __syncthreads();
            int pos = ldcg_i(bs.cell_start + item) + (warp > 0 ? si[warp - 1] : 0) + v - mine;
            for (int k = 0; k < kPer; ++k)
                if (flag[k]) {
                    if (pos < out_cap) out[pos] = ldcg_blob(bs.sorted + i0 + k);
                    ++pos;
                }
            break;
        }
        default: break;
        }

        // ---- completion; the CTA that completes a phase publishes the next one ----
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const int done = (int)atomicAdd(&ctl->done, 1u) + 1;
            s_last = (done == ph_first + ph_count);
            if (s_last) {
                __threadfence();
                int next = PH_END;
                switch (ph_type) {
                    case PH_RANK: next = PH_SCATTER; break;
                    case PH_SCATTER: {
                        if (!pruning) { next = PH_PACK_COUNT; break; }
                        next = PH_COUNT;
                        const double xmin = ldcg_d(&ctl->ext[0]), xmax = ldcg_d(&ctl->ext[1]);
                        const double ymin = ldcg_d(&ctl->ext[2]), ymax = ldcg_d(&ctl->ext[3]);
                        const double rmax = ldcg_d(&ctl->ext[4]);
                        double cell = fmax(2.0 * rmax, 1e-9) * 1.0000001;   // strictly covers d < r_i + r_j
                        cell = fmax(cell, fmax(xmax - xmin, ymax - ymin) / (double)(kMaxCellsPerAxis - 1));
                        const int gx = min(kMaxCellsPerAxis, (int)floor((xmax - xmin) / cell) + 1);
                        const int gy = min(kMaxCellsPerAxis, (int)floor((ymax - ymin) / cell) + 1);
                        bs.grid_params[0] = xmin; bs.grid_params[1] = ymin; bs.grid_params[2] = cell;
                        bs.grid_params[3] = (double)gx; bs.grid_params[4] = (double)gy;
                        break;
                    }
                    case PH_COUNT: next = PH_SCAN; break;
                    case PH_SCAN: next = PH_FILL; break;
                    case PH_FILL: next = PH_FIRST; break;
                    case PH_FIRST: next = PH_SWEEP; ctl->changed = 0; ctl->sweeps = 1; break;
                    case PH_SWEEP:
                        if (__ldcg(&ctl->changed)) {
                            ctl->changed = 0;
                            if (ctl->sweeps < kMaxSweeps) { next = PH_SWEEP; ctl->sweeps += 1; }
                            else next = PH_SATURATE;
                        } else {
                            next = PH_UNION;
                        }
                        break;
                    case PH_SATURATE: next = PH_UNION; break;
                    case PH_UNION: next = PH_LINK; break;
                    case PH_LINK: next = __ldcg(&ctl->n_roots) > 0 ? PH_MERGE : PH_PACK_COUNT; break;
                    case PH_MERGE: next = PH_PACK_COUNT; break;
                    case PH_PACK_COUNT: {
                        next = PH_PACK_WRITE;
                        int run = 0;                                  // chunk offsets
                        for (int c = 0; c < ph_count; ++c) {
                            const int k = ldcg_i(bs.cell_fill + c);
                            bs.cell_start[c] = run;
                            run += k;
                        }
                        ctl->kept = run;
                        break;
                    }
                    case PH_PACK_WRITE: {
                        next = PH_END;
                        const Counters c = *bs.ctr;
                        const int kept = n > 0 ? ctl->kept : 0;
                        hdr->n_blobs = min(kept, out_cap);
                        hdr->n_candidates = c.n_candidates;
                        hdr->n_flagged = c.n_flagged;
                        hdr->n_plateau = c.n_plateau;
                        hdr->n_merges = __ldcg(&ctl->merges);
                        unsigned f = c.flags;
                        if (c.n_candidates > bs.cap || c.n_plateau > bs.cap || kept > out_cap)
                            f |= DOGBLOB_FLAG_OVERFLOW;
                        hdr->flags = f;
                        hdr->capacity = out_cap;
                        // phase profile: us from the first ticket to the publication of ...
                        const unsigned long long t0 = __ldcg(&ctl->phase[0].t_ns);
                        // us from the first ticket to: grid build, first sweep, part labelling,
                        // merge loops, packing (phases that did not run keep the next mark)
                        int mark[5] = {-1, -1, -1, -1, -1};
                        for (int k = 1; k <= cur; ++k) {
                            const int ty = __ldcg(&ctl->phase[k].type);
                            const int us = (int)((__ldcg(&ctl->phase[k].t_ns) - t0) / 1000);
                            const int slot = ty == PH_COUNT ? 0 : ty == PH_SWEEP ? 1 : ty == PH_UNION ? 2
                                           : ty == PH_MERGE ? 3 : ty == PH_PACK_COUNT ? 4 : -1;
                            if (slot >= 0 && mark[slot] < 0) mark[slot] = us;
                        }
                        for (int q = 3; q >= 0; --q) if (mark[q] < 0) mark[q] = mark[q + 1];
                        const int total = (int)((now_ns() - t0) / 1000);
                        auto u16 = [](int v) { return (unsigned)min(max(v, 0), 65535); };
                        hdr->prune_profile[0] = (int)(u16(mark[0]) | (u16(mark[1]) << 16));
                        hdr->prune_profile[1] = (int)(u16(mark[2]) | (u16(mark[3]) << 16));
                        hdr->prune_profile[2] = (int)(u16(mark[4]) | (u16(total) << 16));
                        hdr->prune_profile[3] = (ctl->sweeps << 24) | (__ldcg(&ctl->n_roots) & 0xFFFFFF);
                        hdr->n_seeds = c.n_seeds; hdr->reserved = 0;
                        write_stage_times(c, hdr);
                        break;
                    }
                    default: break;
                }
                const int k = cur + 1;
                {
                    ctl->phase[k].type = next;
                    ctl->phase[k].first_item = ph_first + ph_count;
                    ctl->phase[k].n_items = next == PH_END ? 0 : phase_items(next, n, __ldcg(&ctl->n_roots));
                    ctl->phase[k].t_ns = now_ns();
                    __threadfence();
                    *(volatile int *)&ctl->n_phases = k + 1;
                }
            }
        }
        __syncthreads();
    }
}

// ---- frames with <= kSmallMax candidates: order, prune and pack in ONE CTA ---------------
// Same semantics as rank_sort + prune_build/first/loop, without the grid: every pair
// is tested directly (n^2 / 2 cheap rejections), all state lives in shared memory.
struct SmallBlob { double x, y, r, resp, sigma; int slice; unsigned flags; };

__global__ void __launch_bounds__(kSmallMax)
finalize_small_kernel(BlobSpace bs, double thr, int do_prune, dogblob_result_header *hdr,
                      dogblob_blob *out, int out_cap, int limit) {
    extern __shared__ __align__(16) unsigned char small_raw[];
    SmallBlob *sb = reinterpret_cast<SmallBlob *>(small_raw);                 // sorted blobs
    SmallBlob *raw = sb + kSmallMax;                                          // emission order
    int *first = reinterpret_cast<int *>(raw + kSmallMax);
    int *alive = first + kSmallMax;
    __shared__ int s_red[33];
    __shared__ int s_pos, s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_raw = bs.ctr->n_candidates;
    if (tid == 0) bs.ctr->t_prune = globaltimer_ns();
    if (n_raw > limit || n_raw > bs.cap) {
        if (tid == 0) bs.ctr->small_done = 0;
        return;
    }
    const int n = n_raw;
    auto imin = [](int a, int b) { return min(a, b); };

    // ---- order: rank on (-response, y, x, sigma), ties by input index ----
    if (tid < n) {
        const dogblob_blob b = bs.unsorted[tid];
        raw[tid] = SmallBlob{b.x, b.y, b.radius, b.response, b.sigma, b.slice, b.flags};
    }
    __syncthreads();
    const int n_warps = blockDim.x >> 5;
    for (int i = warp; i < n; i += n_warps) {            // one warp per blob, lanes over j
        const SmallBlob me = raw[i];
        int cnt = 0;
        for (int j = lane; j < n; j += 32) {
            const SmallBlob o = raw[j];
            bool before;
            if (o.resp != me.resp) before = o.resp > me.resp;
            else if (o.y != me.y) before = o.y < me.y;
            else if (o.x != me.x) before = o.x < me.x;
            else if (o.sigma != me.sigma) before = o.sigma < me.sigma;
            else before = j < i;
            cnt += before ? 1 : 0;
        }
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) {
            sb[cnt] = me;
            alive[cnt] = 1;
        }
    }
    __syncthreads();
    int merges = 0;
    if (do_prune && n >= 2) {
        // ---- first[i]: smallest j > i with overlap > thr ----
        for (int i = warp; i < n; i += n_warps) {        // one warp per row, lanes over j
            const SmallBlob a = sb[i];
            int best = INT_MAX;
            for (int j0 = i + 1; j0 < n && best == INT_MAX; j0 += 32) {
                const int j = j0 + lane;
                bool hit = false;
                if (j < n) {
                    const SmallBlob b = sb[j];
                    const double dx = a.x - b.x, dy = a.y - b.y, rr = a.r + b.r;
                    if (dx * dx + dy * dy < rr * rr * 1.0000001 + 1e-9)   // else disjoint for sure
                        hit = overlap_ij(a.x, a.y, a.r, b.x, b.y, b.r) > thr;
                }
                const unsigned m = __ballot_sync(0xffffffffu, hit);
                if (m) best = j0 + __ffs(m) - 1;
            }
            if (lane == 0) first[i] = (best == INT_MAX) ? -1 : best;
        }
        if (tid == 0) s_pos = 0;
    }
    // Only the warps that hold a blob stay for the sequential part: every barrier of the merge
    // loop then spans ceil(n / 32) warps instead of 32 (exited warps leave the barrier count).
    __syncthreads();
    const int nw = max(1, (n + 31) >> 5);
    if (warp >= nw) return;
    if (do_prune && n >= 2) {
        while (true) {
            int mine = (tid >= s_pos && tid < n && alive[tid] && first[tid] >= 0) ? tid : INT_MAX;
            const int istar = block_reduce(mine, imin, s_red, nw);
            if (istar == INT_MAX) break;
            const int j = first[istar];
            __syncthreads();
            if (tid == 0) {
                SmallBlob a = sb[istar];
                const SmallBlob w = sb[j];
                const double nr = 0.5 * (a.r + w.r);
                a.r = nr;
                a.sigma = nr / kSqrt2;
                a.flags |= (w.flags & DOGBLOB_BLOB_SCALE_EDGE) | DOGBLOB_BLOB_MERGED;
                a.slice = -1;
                sb[istar] = a;
                alive[j] = 0;
                s_pos = istar;
            }
            ++merges;
            __syncthreads();
            const SmallBlob bi = sb[istar];
            // (a) new first partner of istar: block-wide min over j > istar
            int cand = INT_MAX;
            if (tid > istar && tid < n && alive[tid]) {
                const SmallBlob b = sb[tid];
                if (overlap_ij(bi.x, bi.y, bi.r, b.x, b.y, b.r) > thr) cand = tid;
            }
            // (b) rows k < istar can only gain istar; (c) rows that pointed at j rescan
            if (tid < istar && alive[tid]) {
                const SmallBlob b = sb[tid];
                if (overlap_ij(b.x, b.y, b.r, bi.x, bi.y, bi.r) > thr) {
                    first[tid] = istar;
                    atomicMin(&s_pos, tid);
                }
            } else if (tid > istar && tid < n && alive[tid] && first[tid] == j) {
                const SmallBlob a = sb[tid];
                int best = -1;
                for (int q = tid + 1; q < n; ++q) {
                    if (!alive[q]) continue;
                    const SmallBlob b = sb[q];
                    if (overlap_ij(a.x, a.y, a.r, b.x, b.y, b.r) > thr) { best = q; break; }
                }
                first[tid] = best;
            }
            cand = block_reduce(cand, imin, s_red, nw);
            if (tid == 0) first[istar] = (cand == INT_MAX) ? -1 : cand;
            __syncthreads();
        }
    }
    // ---- pack survivors in order ----
    __syncthreads();
    const int keep = (tid < n) && (!do_prune || n < 2 || alive[tid]);
    int v = keep;
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) s_red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        int t = lane < nw ? s_red[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += u;
        }
        s_red[lane] = t;
    }
    __syncthreads();
    const int pos = (warp > 0 ? s_red[warp - 1] : 0) + v - keep;
    if (tid == 0) s_carry = s_red[nw - 1];
    if (keep && pos < out_cap) {
        const SmallBlob b = sb[tid];
        dogblob_blob o;
        o.x = b.x; o.y = b.y; o.sigma = b.sigma; o.radius = b.r; o.response = b.resp;
        o.slice = b.slice; o.flags = b.flags;
        out[pos] = o;
    }
    if (tid == 0) {
        const Counters c = *bs.ctr;
        hdr->n_blobs = min(s_carry, out_cap);
        hdr->n_candidates = c.n_candidates;
        hdr->n_flagged = c.n_flagged;
        hdr->n_plateau = c.n_plateau;
        hdr->n_merges = merges;
        unsigned f = c.flags;
        if (c.n_plateau > bs.cap || s_carry > out_cap) f |= DOGBLOB_FLAG_OVERFLOW;
        hdr->flags = f;
        hdr->capacity = out_cap;
        for (int q = 0; q < 4; ++q) hdr->prune_profile[q] = 0;
        hdr->n_seeds = c.n_seeds; hdr->reserved = 0;
        write_stage_times(c, hdr);
        bs.ctr->small_done = 1;
    }
}

constexpr size_t kSmallSmem = (size_t)kSmallMax * (2 * sizeof(SmallBlob) + 2 * sizeof(int));

}  // namespace

// One SM is faster than the multi-kernel grid path only for a few hundred candidates.
int small_limit() {
    static const int v = [] {
        const char *e = std::getenv("DOGBLOB_SMALL_LIMIT");
        const int x = e ? std::atoi(e) : 320;
        return x < 0 ? 0 : (x > kSmallMax ? kSmallMax : x);
    }();
    return v;
}

cudaError_t configure_finalize_kernels() {
    return cudaFuncSetAttribute(finalize_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kSmallSmem);
}

cudaError_t launch_prune_and_pack(const BlobSpace &bs, double overlap, bool prune,
                                  void *d_result, int result_cap, cudaStream_t st) {
    auto *hdr = reinterpret_cast<dogblob_result_header *>(d_result);
    auto *out = reinterpret_cast<dogblob_blob *>(reinterpret_cast<char *>(d_result) +
                                                 DOGBLOB_RESULT_HEADER_BYTES);
    // <= kSmallMax candidates: everything in one CTA; the general kernels then return at once
    finalize_small_kernel<<<1, kSmallMax, kSmallSmem, st>>>(bs, overlap, prune ? 1 : 0, hdr, out,
                                                            result_cap, small_limit());
    // larger frames: one whole-GPU kernel whose phases chain on the device
    prune_large_kernel<<<148 * 2, kLargeThreads, 0, st>>>(bs, overlap, prune ? 1 : 0, hdr, out,
                                                          result_cap);
    return cudaGetLastError();
}

}  // namespace dogblob
