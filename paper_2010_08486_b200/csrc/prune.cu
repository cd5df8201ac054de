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

constexpr int kLoopThreads = 1024;
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

__device__ __forceinline__ Grid load_grid(const BlobSpace &bs) {
    Grid g;
    g.x0 = bs.grid_params[0];
    g.y0 = bs.grid_params[1];
    g.cell = bs.grid_params[2];
    g.gx = (int)bs.grid_params[3];
    g.gy = (int)bs.grid_params[4];
    return g;
}

template <typename T, typename Op>
__device__ T block_reduce(T v, Op op, T *scratch /* >= 33 */) {
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
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

// ---- build the grid (single CTA): extents, cell size, counting sort -------------------
__global__ void __launch_bounds__(kLoopThreads) prune_build_kernel(BlobSpace bs) {
    if (bs.ctr->small_done) return;
    __shared__ double sd[33];
    __shared__ int si[33];
    const int n = min(bs.ctr->n_candidates, bs.cap);
    const int tid = threadIdx.x;
    double xmin = DBL_MAX, xmax = -DBL_MAX, ymin = DBL_MAX, ymax = -DBL_MAX, rmax = 0.0;
    for (int i = tid; i < n; i += blockDim.x) {
        const dogblob_blob b = bs.sorted[i];
        xmin = fmin(xmin, b.x); xmax = fmax(xmax, b.x);
        ymin = fmin(ymin, b.y); ymax = fmax(ymax, b.y);
        rmax = fmax(rmax, b.radius);
        bs.alive[i] = 1;
        bs.first[i] = -1;
    }
    auto fmn = [](double a, double b) { return fmin(a, b); };
    auto fmx = [](double a, double b) { return fmax(a, b); };
    xmin = block_reduce(xmin, fmn, sd); xmax = block_reduce(xmax, fmx, sd);
    ymin = block_reduce(ymin, fmn, sd); ymax = block_reduce(ymax, fmx, sd);
    rmax = block_reduce(rmax, fmx, sd);
    if (n == 0) { xmin = ymin = 0.0; xmax = ymax = 1.0; }
    double cell = fmax(2.0 * rmax, 1e-9) * 1.0000001;   // strictly covers d < r_i + r_j
    cell = fmax(cell, fmax(xmax - xmin, ymax - ymin) / (double)(kMaxCellsPerAxis - 1));
    const int gx = min(kMaxCellsPerAxis, (int)floor((xmax - xmin) / cell) + 1);
    const int gy = min(kMaxCellsPerAxis, (int)floor((ymax - ymin) / cell) + 1);
    if (tid == 0) {
        bs.grid_params[0] = xmin; bs.grid_params[1] = ymin; bs.grid_params[2] = cell;
        bs.grid_params[3] = (double)gx; bs.grid_params[4] = (double)gy;
    }
    Grid g{xmin, ymin, cell, gx, gy};
    const int ncell = gx * gy;
    for (int c = tid; c <= ncell; c += blockDim.x) bs.cell_start[c] = 0;
    for (int c = tid; c < ncell; c += blockDim.x) bs.cell_fill[c] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) {
        const dogblob_blob b = bs.sorted[i];
        const int c = g.cy(b.y) * gx + g.cx(b.x);
        bs.cell_of[i] = c;
        atomicAdd(&bs.cell_start[c + 1], 1);
    }
    __syncthreads();
    // inclusive scan of cell_start[1..ncell] in chunks of blockDim.x
    __shared__ int carry;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int c0 = 1; c0 <= ncell; c0 += blockDim.x) {
        const int c = c0 + tid;
        int v = (c <= ncell) ? bs.cell_start[c] : 0;
        const int lane = tid & 31, w = tid >> 5;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (lane == 31) si[w] = v;
        __syncthreads();
        if (w == 0) {
            int t = si[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += u;
            }
            si[lane] = t;
        }
        __syncthreads();
        const int prefix = carry + (w > 0 ? si[w - 1] : 0);
        if (c <= ncell) bs.cell_start[c] = v + prefix;
        __syncthreads();
        if (tid == blockDim.x - 1) carry = v + prefix;
        __syncthreads();
    }
    for (int i = tid; i < n; i += blockDim.x) {
        const int c = bs.cell_of[i];
        const int slot = bs.cell_start[c] + atomicAdd(&bs.cell_fill[c], 1);
        bs.cell_items[slot] = i;
    }
}

// smallest alive j > i (or, with below=true, test only partner `only`) offending with i
__device__ int scan_first_partner(const BlobSpace &bs, const Grid &g, int i, double thr,
                                  int t, int nt) {
    const dogblob_blob bi = bs.sorted[i];
    const int cx = g.cx(bi.x), cy = g.cy(bi.y);
    int best = INT_MAX;
    for (int yy = max(cy - 1, 0); yy <= min(cy + 1, g.gy - 1); ++yy)
        for (int xx = max(cx - 1, 0); xx <= min(cx + 1, g.gx - 1); ++xx) {
            const int c = yy * g.gx + xx;
            const int e = bs.cell_start[c + 1];
            for (int p = bs.cell_start[c] + t; p < e; p += nt) {
                const int j = bs.cell_items[p];
                if (j <= i || j >= best || !(bs.alive[j] & 1)) continue;
                const dogblob_blob bj = bs.sorted[j];
                if (overlap_ij(bi.x, bi.y, bi.radius, bj.x, bj.y, bj.radius) > thr) best = j;
            }
        }
    return best;
}

// ---- first[i] for every blob: one warp per blob, whole GPU ---------------------------
__global__ void __launch_bounds__(256) prune_first_kernel(BlobSpace bs, double thr) {
    if (bs.ctr->small_done) return;
    const int n = min(bs.ctr->n_candidates, bs.cap);
    if (n < 2) return;
    const Grid g = load_grid(bs);
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        int best = scan_first_partner(bs, g, i, thr, lane, 32);
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) bs.first[i] = (best == INT_MAX) ? -1 : best;
    }
}

// ---- merge loop + final packing (single persistent CTA) -----------------------------------
// The reference's loop is sequential, but merges only interact through blobs that can
// overlap.  ub(a) bounds every radius blob a can ever take: a's radius only changes when a
// (the lower index) absorbs some b > a and becomes the mean, so
//     ub(a) = max(r_a, max{ ub(b) : b > a, dist(a, b) < ub(a) + ub(b) }),
// taken as the least fixed point from below.  By induction no merge ever joins blobs that
// are not linked by "dist < ub(a) + ub(b)", so the connected parts of that graph evolve
// independently and the global row-major-first order restricted to a part is that part's
// own sequential order: each round merges the smallest offending row of EVERY part at once
// (one warp per row).  Rounds = longest merge chain of a part, not the number of merges.
__device__ __forceinline__ int comp_find(int *comp, int x) {
    int p = ((volatile int *)comp)[x];
    while (p != x) { x = p; p = ((volatile int *)comp)[x]; }
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

__device__ __forceinline__ double ub_of(const BlobSpace &bs, int i) {
    return __longlong_as_double((long long)((volatile unsigned long long *)bs.bound)[i]);
}

// rows with an offending partner live in a compact list (bit 1 of alive[] = "listed")
__device__ __forceinline__ void list_row(const BlobSpace &bs, int k, int *s_len) {
    if (!(atomicOr(&bs.alive[k], 2) & 2)) bs.cell_of[atomicAdd(s_len, 1)] = k;
}

// one warp merges row i with its first partner and repairs the cached partners around it
__device__ void merge_row(const BlobSpace &bs, const Grid &g, int i, double thr, int lane,
                          int *s_len) {
    const int j = bs.first[i];
    if (lane == 0) {
        dogblob_blob a = bs.sorted[i];
        const dogblob_blob w = bs.sorted[j];
        const double nr = 0.5 * (a.radius + w.radius);
        a.radius = nr;
        a.sigma = nr / kSqrt2;
        a.flags |= (w.flags & DOGBLOB_BLOB_SCALE_EDGE) | DOGBLOB_BLOB_MERGED;
        a.slice = -1;
        bs.sorted[i] = a;
        bs.alive[j] = 0;
    }
    __syncwarp();
    const dogblob_blob bi = bs.sorted[i];
    const dogblob_blob bj = bs.sorted[j];
    // (a) first[i] again; (b) rows k < i of this part had no partner and can only gain i
    int best = INT_MAX;
    {
        const int cx = g.cx(bi.x), cy = g.cy(bi.y);
        for (int yy = max(cy - 1, 0); yy <= min(cy + 1, g.gy - 1); ++yy)
            for (int xx = max(cx - 1, 0); xx <= min(cx + 1, g.gx - 1); ++xx) {
                const int c = yy * g.gx + xx;
                const int e = bs.cell_start[c + 1];
                for (int p = bs.cell_start[c] + lane; p < e; p += 32) {
                    const int k = bs.cell_items[p];
                    if (k == i || !(bs.alive[k] & 1)) continue;
                    const dogblob_blob bk = bs.sorted[k];
                    if (k > i) {
                        if (k < best && overlap_ij(bi.x, bi.y, bi.radius, bk.x, bk.y, bk.radius) > thr)
                            best = k;
                    } else if (overlap_ij(bk.x, bk.y, bk.radius, bi.x, bi.y, bi.radius) > thr) {
                        bs.first[k] = i;
                        list_row(bs, k, s_len);
                    }
                }
            }
    }
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) bs.first[i] = (best == INT_MAX) ? -1 : best;
    // (c) rows that pointed at the deleted blob need a new partner
    {
        const int cx = g.cx(bj.x), cy = g.cy(bj.y);
        for (int yy = max(cy - 1, 0); yy <= min(cy + 1, g.gy - 1); ++yy)
            for (int xx = max(cx - 1, 0); xx <= min(cx + 1, g.gx - 1); ++xx) {
                const int c = yy * g.gx + xx;
                const int s0 = bs.cell_start[c], e = bs.cell_start[c + 1];
                for (int p0 = s0; p0 < e; p0 += 32) {
                    const int p = p0 + lane;
                    const int k = p < e ? bs.cell_items[p] : -1;
                    const bool hit = k >= 0 && k != i && (bs.alive[k] & 1) && bs.first[k] == j;
                    unsigned m = __ballot_sync(0xffffffffu, hit);
                    while (m) {
                        const int src = __ffs(m) - 1;
                        m &= m - 1;
                        const int kk = __shfl_sync(0xffffffffu, k, src);
                        int b2 = scan_first_partner(bs, g, kk, thr, lane, 32);
                        for (int o = 16; o > 0; o >>= 1)
                            b2 = min(b2, __shfl_xor_sync(0xffffffffu, b2, o));
                        if (lane == 0) bs.first[kk] = (b2 == INT_MAX) ? -1 : b2;   // kk stays listed
                    }
                }
            }
    }
}

__global__ void __launch_bounds__(kLoopThreads)
prune_loop_kernel(BlobSpace bs, double thr, int do_prune, dogblob_result_header *hdr,
                  dogblob_blob *out, int out_cap) {
    if (bs.ctr->small_done) return;
    __shared__ int s_red[33];
    __shared__ int s_flag, s_nact, s_len, s_carry;
    __shared__ int s_act[kLoopThreads];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = min(bs.ctr->n_candidates, bs.cap);
    int merges = 0;

    if (do_prune && n >= 2) {
        const Grid g = load_grid(bs);
        // ---- ub(): least fixed point from below (Jacobi sweeps over the grid neighbourhoods) ----
        if (tid == 0) s_len = 0;
        for (int i = tid; i < n; i += blockDim.x) {
            bs.comp[i] = i;
            bs.cmin[i] = INT_MAX;
            bs.bound[i] = (unsigned long long)__double_as_longlong(bs.sorted[i].radius);
        }
        __syncthreads();
        while (true) {
            if (tid == 0) s_flag = 0;
            __syncthreads();
            for (int i = tid; i < n; i += blockDim.x) {
                const dogblob_blob bi = bs.sorted[i];
                double ui = ub_of(bs, i);
                const int cx = g.cx(bi.x), cy = g.cy(bi.y);
                bool grew = false;
                for (int yy = max(cy - 1, 0); yy <= min(cy + 1, g.gy - 1); ++yy)
                    for (int xx = max(cx - 1, 0); xx <= min(cx + 1, g.gx - 1); ++xx) {
                        const int c = yy * g.gx + xx;
                        const int e = bs.cell_start[c + 1];
                        for (int p = bs.cell_start[c]; p < e; ++p) {
                            const int j = bs.cell_items[p];
                            if (j <= i) continue;
                            const double uj = ub_of(bs, j);
                            if (uj <= ui) continue;
                            const dogblob_blob bj = bs.sorted[j];
                            const double dx = bi.x - bj.x, dy = bi.y - bj.y, reach = ui + uj;
                            if (dx * dx + dy * dy < reach * reach * 1.0000001 + 1e-9) {
                                ui = uj;
                                grew = true;
                            }
                        }
                    }
                if (grew) {
                    bs.bound[i] = (unsigned long long)__double_as_longlong(ui);
                    s_flag = 1;
                }
            }
            __syncthreads();
            const int changed = s_flag;
            __syncthreads();
            if (!changed) break;
        }
        // ---- parts: connected components of dist < ub(a) + ub(b) ----
        for (int i = tid; i < n; i += blockDim.x) {
            const dogblob_blob bi = bs.sorted[i];
            const double ui = ub_of(bs, i);
            const int cx = g.cx(bi.x), cy = g.cy(bi.y);
            for (int yy = max(cy - 1, 0); yy <= min(cy + 1, g.gy - 1); ++yy)
                for (int xx = max(cx - 1, 0); xx <= min(cx + 1, g.gx - 1); ++xx) {
                    const int c = yy * g.gx + xx;
                    const int e = bs.cell_start[c + 1];
                    for (int p = bs.cell_start[c]; p < e; ++p) {
                        const int j = bs.cell_items[p];
                        if (j <= i) continue;
                        const dogblob_blob bj = bs.sorted[j];
                        const double dx = bi.x - bj.x, dy = bi.y - bj.y, reach = ui + ub_of(bs, j);
                        if (dx * dx + dy * dy < reach * reach * 1.0000001 + 1e-9)
                            comp_union(bs.comp, i, j);
                    }
                }
        }
        __syncthreads();
        for (int i = tid; i < n; i += blockDim.x) bs.comp[i] = comp_find(bs.comp, i);
        __syncthreads();
        for (int i = tid; i < n; i += blockDim.x)
            if (bs.first[i] >= 0) list_row(bs, i, &s_len);
        __syncthreads();

        // ---- rounds: the smallest offending row of every part, all parts at once ----
        while (true) {
            if (tid == 0) s_nact = 0;
            __syncthreads();
            const int len = s_len;
            for (int q = tid; q < len; q += blockDim.x) {
                const int i = bs.cell_of[q];
                if ((bs.alive[i] & 1) && bs.first[i] >= 0) atomicMin(&bs.cmin[bs.comp[i]], i);
            }
            __syncthreads();
            for (int q = tid; q < len; q += blockDim.x) {
                const int i = bs.cell_of[q];
                if ((bs.alive[i] & 1) && bs.first[i] >= 0 && bs.cmin[bs.comp[i]] == i) {
                    bs.cmin[bs.comp[i]] = INT_MAX;
                    const int slot = atomicAdd(&s_nact, 1);
                    if (slot < kLoopThreads) s_act[slot] = i;   // the rest wait for the next round
                }
            }
            __syncthreads();
            const int nact = min(s_nact, kLoopThreads);
            if (nact == 0) break;
            for (int q = warp; q < nact; q += (blockDim.x >> 5))
                merge_row(bs, g, s_act[q], thr, lane, &s_len);
            merges += nact;
            __syncthreads();
        }
    }

    // ---- pack survivors in order ------------------------------------------------------
    __syncthreads();
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += blockDim.x) {
        const int i = base + tid;
        const int keep = (i < n) && (!do_prune || n < 2 || (bs.alive[i] & 1));
        int v = keep;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (lane == 31) s_red[warp] = v;
        __syncthreads();
        if (warp == 0) {
            int t = s_red[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += u;
            }
            s_red[lane] = t;
        }
        __syncthreads();
        const int pos = s_carry + (warp > 0 ? s_red[warp - 1] : 0) + v - keep;
        if (keep && pos < out_cap) out[pos] = bs.sorted[i];
        __syncthreads();
        if (tid == blockDim.x - 1) s_carry = pos + keep;
        __syncthreads();
    }
    if (tid == 0) {
        const Counters c = *bs.ctr;
        hdr->n_blobs = min(s_carry, out_cap);
        hdr->n_candidates = c.n_candidates;
        hdr->n_flagged = c.n_flagged;
        hdr->n_plateau = c.n_plateau;
        hdr->n_merges = merges;
        unsigned f = c.flags;
        if (c.n_candidates > bs.cap || c.n_plateau > bs.cap || s_carry > out_cap)
            f |= DOGBLOB_FLAG_OVERFLOW;
        hdr->flags = f;
        hdr->capacity = out_cap;
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
        __syncthreads();
        while (true) {
            int mine = (tid >= s_pos && tid < n && alive[tid] && first[tid] >= 0) ? tid : INT_MAX;
            const int istar = block_reduce(mine, imin, s_red);
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
            cand = block_reduce(cand, imin, s_red);
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
        int t = s_red[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += u;
        }
        s_red[lane] = t;
    }
    __syncthreads();
    const int pos = (warp > 0 ? s_red[warp - 1] : 0) + v - keep;
    if (keep && pos < out_cap) {
        const SmallBlob b = sb[tid];
        dogblob_blob o;
        o.x = b.x; o.y = b.y; o.sigma = b.sigma; o.radius = b.r; o.response = b.resp;
        o.slice = b.slice; o.flags = b.flags;
        out[pos] = o;
    }
    if (tid == blockDim.x - 1) s_carry = pos + keep;
    __syncthreads();
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
    cudaError_t e = launch_rank_sort(bs, st);
    if (e != cudaSuccess) return e;
    if (prune) {
        prune_build_kernel<<<1, kLoopThreads, 0, st>>>(bs);
        prune_first_kernel<<<148 * 2, 256, 0, st>>>(bs, overlap);
    }
    prune_loop_kernel<<<1, kLoopThreads, 0, st>>>(bs, overlap, prune ? 1 : 0, hdr, out, result_cap);
    return cudaGetLastError();
}

}  // namespace dogblob
