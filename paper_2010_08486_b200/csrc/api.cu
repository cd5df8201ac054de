// C ABI of libdogblob_b200 (see include/dogblob_b200.h).
#include <algorithm>
#include <functional>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace dogblob {

static thread_local std::string g_error;
void set_error(const std::string &msg) { g_error = msg; }

static inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

size_t blobspace_bytes(int cap) {
    size_t b = 0;
    const size_t c = (size_t)cap;
    b += align_up(sizeof(Counters), 256);
    b += align_up(c * sizeof(Voxel), 256);
    b += align_up(c * sizeof(int), 256) * 2;                  // parent, pl_count
    b += align_up(c * sizeof(unsigned long long), 256) * 3;   // pl_sum_row/col, pl_first
    b += align_up(c * sizeof(dogblob_blob), 256) * 2;         // unsorted, sorted
    b += align_up(c * sizeof(int), 256) * 6;                  // first, alive, cell_of, cell_items, comp, cmin
    b += align_up(c * sizeof(unsigned long long), 256);       // bound
    b += align_up((size_t)(kMaxCells + 1) * sizeof(int), 256);
    b += align_up((size_t)kMaxCells * sizeof(int), 256);
    b += align_up(8 * sizeof(double), 256);
    b += align_up(sizeof(PruneCtl), 256);
    return b;
}

BlobSpace carve_blobspace(void *base, int cap) {
    char *p = reinterpret_cast<char *>(base);
    const size_t c = (size_t)cap;
    auto take = [&](size_t bytes) { char *q = p; p += align_up(bytes, 256); return q; };
    BlobSpace bs;
    bs.ctr = reinterpret_cast<Counters *>(take(sizeof(Counters)));
    bs.plateau = reinterpret_cast<Voxel *>(take(c * sizeof(Voxel)));
    bs.parent = reinterpret_cast<int *>(take(c * sizeof(int)));
    bs.pl_count = reinterpret_cast<int *>(take(c * sizeof(int)));
    bs.pl_sum_row = reinterpret_cast<unsigned long long *>(take(c * sizeof(unsigned long long)));
    bs.pl_sum_col = reinterpret_cast<unsigned long long *>(take(c * sizeof(unsigned long long)));
    bs.pl_first = reinterpret_cast<unsigned long long *>(take(c * sizeof(unsigned long long)));
    bs.unsorted = reinterpret_cast<dogblob_blob *>(take(c * sizeof(dogblob_blob)));
    bs.sorted = reinterpret_cast<dogblob_blob *>(take(c * sizeof(dogblob_blob)));
    bs.first = reinterpret_cast<int *>(take(c * sizeof(int)));
    bs.alive = reinterpret_cast<int *>(take(c * sizeof(int)));
    bs.comp = reinterpret_cast<int *>(take(c * sizeof(int)));
    bs.cmin = reinterpret_cast<int *>(take(c * sizeof(int)));
    bs.bound = reinterpret_cast<unsigned long long *>(take(c * sizeof(unsigned long long)));
    bs.cell_of = reinterpret_cast<int *>(take(c * sizeof(int)));
    bs.cell_items = reinterpret_cast<int *>(take(c * sizeof(int)));
    bs.cell_start = reinterpret_cast<int *>(take((size_t)(kMaxCells + 1) * sizeof(int)));
    bs.cell_fill = reinterpret_cast<int *>(take((size_t)kMaxCells * sizeof(int)));
    bs.grid_params = reinterpret_cast<double *>(take(8 * sizeof(double)));
    bs.ctl = reinterpret_cast<PruneCtl *>(take(sizeof(PruneCtl)));
    bs.cap = cap;
    return bs;
}

}  // namespace dogblob

using namespace dogblob;

struct dogblob_plan {
    int device;
    ConvGeometry geo;
    int max_blobs;
    std::vector<LevelDesc> levels;
    std::vector<double> sigmas;
    // device constants
    LevelTable table;        // fused pass: launch order + level groups
    LevelTable unit_table;   // stage API: one level per group
    LevelTable umma_table;   // tensor-core column pass: groups balanced for persistent CTAs
    float2 *d_taps = nullptr;
    bool use_umma = false;   // plan-time choice of the convolution engine (see dogblob_plan_create)
    ToeplitzTable toeplitz;  // tensor-core passes: prebuilt Toeplitz operands of every level
    float *d_toeplitz = nullptr;
    int *d_umma_sched = nullptr;   // tensor-core column pass: unit of (slot, CTA), -1 = none (see plan_umma_schedule)
    int umma_sched_slots = 0, umma_sched_ctas = 0;
    int umma_ctas = 0;             // persistent CTAs of the tensor-core passes (SMs minus the spare ones)
    double *d_slice_sigma = nullptr;
    float *d_sigma_f32 = nullptr;
    // workspace layout (bytes from the workspace base)
    // FP32 engine: rows_t = row-filtered planes (x-major), dog_t = DoG^T planes, edge = parked levels;
    // tensor engine: rows_t = R planes (fp16 hi | lo), x = X planes, dog_t = DoG^T planes too (x-major),
    // no edge planes
    size_t off_rows_t = 0, off_x = 0, off_dog_t = 0, off_edge = 0, off_blobspace = 0, off_gate = 0, off_flags = 0, off_seeds = 0, total = 0;
    int seed_cap = 0;               // tensor engine: capacity of the column pass's seed list (0 = no seeds, strip kernel)
};

namespace {

int round_up(int v, int a) { return (v + a - 1) / a * a; }

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) { ok = false; return; }
        if (prev != dev && cudaSetDevice(dev) != cudaSuccess) ok = false;
    }
    ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

// Partition the L levels into G contiguous groups of similar tap count for the fused
// column+DoG pass; group g sweeps levels [begin[g], begin[g+1]).
std::vector<int> balance_groups(const std::vector<LevelDesc> &lv, int G, double fixed_cost = -1.0) {
    const int L = (int)lv.size();
    G = std::max(1, std::min(G, L));
    std::vector<double> pre(L + 1, 0.0);
    // cost of a level in full-chunk units: middle chunks + head/tail (136/128 of a full one)
    // + its fixed part (DoG epilogue, pipeline refill)
    static const double fixed_fma = [] {
        const char *e = std::getenv("DOGBLOB_LEVEL_COST");
        return e ? std::atof(e) : 1.07;
    }();
    const double fixed = fixed_cost >= 0.0 ? fixed_cost : fixed_fma;
    for (int i = 0; i < L; ++i) pre[i + 1] = pre[i] + lv[i].n_mid + fixed;
    std::vector<int> begin(G + 1, 0);
    begin[G] = L;
    for (int g = 1; g < G; ++g) {
        const double target = pre[L] * g / G;
        int b = (int)(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
        b = std::max(b, begin[g - 1] + 1);
        b = std::min(b, L - (G - g));
        begin[g] = b;
    }
    return begin;
}

// Number of level groups: fill whole waves of CTAs (2 resident per SM) as exactly as
// possible; every extra group costs one boundary slice through the edge planes.
int choose_groups(int tiles, int L, double slots = 2.0 * 148.0) {
    int best = 1;
    double best_score = -1.0;
    for (int G = 1; G <= std::min(L, 24); ++G) {
        const double waves = tiles * G / slots;
        const double eff = waves / std::ceil(waves);
        const double score = eff - 0.004 * G;
        if (score > best_score) { best_score = score; best = G; }
    }
    return best;
}

// Tensor-core column pass: level groups and a static schedule for `ctas` persistent CTAs.
// A unit = (tile, group); group g also computes the first level of group g + 1 (the DoG slice
// between them needs both), so every boundary costs one duplicated level.  With equal groups the
// 64 G units of a 1024^2 frame deal out as 4 / 4 / 4 / 3 per CTA: the kernel ends with its slowest
// CTA, 4 equal units.  Unequal groups pack better: a few SMALL groups at the fine end of the ladder
// (cheap levels: cheap duplicates) give the longest-processing-time-first assignment small units to
// level the CTAs with.  Cost of a level = its k-steps + a fixed part (commits, drain hand-over).
struct UmmaSchedule {
    std::vector<int> begin;      // group boundaries
    std::vector<int> flat;       // [slot][cta] -> unit (group * tiles + tile) or -1
    int slots = 0;
    double makespan = 0.0, mean = 0.0;
};
UmmaSchedule plan_umma_schedule(const std::vector<LevelDesc> &lv, int tiles, int ctas, double level_fixed,
                                int force_groups) {
    const int L = (int)lv.size();
    std::vector<double> c(L), pre(L + 1, 0.0);
    for (int i = 0; i < L; ++i) {
        c[i] = (128 + 2 * lv[i].rpad) / 16 + level_fixed;
        pre[i + 1] = pre[i] + c[i];
    }
    // cost of group q of a partition: its levels plus the first level of the next group
    auto group_costs = [&](const std::vector<int> &begin, std::vector<double> &gc) {
        const int G = (int)begin.size() - 1;
        gc.resize(G);
        for (int q = 0; q < G; ++q) gc[q] = pre[std::min(begin[q + 1] + (q + 1 < G ? 1 : 0), L)] - pre[begin[q]];
    };
    // makespan of the longest-processing-time-first assignment (units of a group are equal: deal
    // them out group by group, largest first, always to the least loaded CTA)
    std::vector<double> heap;
    auto lpt = [&](const std::vector<double> &gc) {
        std::vector<double> sorted(gc);
        std::sort(sorted.begin(), sorted.end(), std::greater<double>());
        heap.assign(ctas, 0.0);          // min-heap on the load
        auto cmp = std::greater<double>();
        for (double v : sorted)
            for (int t = 0; t < tiles; ++t) {
                std::pop_heap(heap.begin(), heap.end(), cmp);
                heap.back() += v;
                std::push_heap(heap.begin(), heap.end(), cmp);
            }
        return *std::max_element(heap.begin(), heap.end());
    };
    UmmaSchedule best;
    best.makespan = 1e300;
    uint32_t rng = 12345u;
    std::vector<double> gc;
    const int g_hi = std::min(L - 1, std::max(2, std::min(14, 4 * ctas / std::max(1, tiles) + 2)));
    for (int G = 1; G <= g_hi; ++G) {
        if (force_groups > 0 && G != std::min(force_groups, g_hi)) continue;
        std::vector<int> begin(G + 1, 0);
        begin[G] = L;
        for (int g = 1; g < G; ++g) {             // start from groups of equal cost
            int b = (int)(std::lower_bound(pre.begin(), pre.end(), pre[L] * g / G) - pre.begin());
            begin[g] = std::min(std::max(b, begin[g - 1] + 1), L - (G - g));
        }
        group_costs(begin, gc);
        double cur = lpt(gc);
        for (int it = 0; G > 1 && it < 400; ++it) {       // hill climbing on the boundaries
            rng = rng * 1664525u + 1013904223u;
            const int g = 1 + (int)((rng >> 8) % (uint32_t)(G - 1));
            const int d = ((rng >> 4) & 1) ? 1 : -1;
            std::vector<int> nb(begin);
            nb[g] += d * (1 + (int)((rng >> 5) & 1));
            if (!(nb[g - 1] < nb[g] && nb[g] < nb[g + 1])) continue;
            group_costs(nb, gc);
            const double v = lpt(gc);
            if (v <= cur) { cur = v; begin.swap(nb); }
        }
        if (cur < best.makespan * (1.0 - 1e-9)) {
            best.makespan = cur;
            best.begin = begin;
        }
    }
    // the assignment itself, CTA by CTA
    const int G = (int)best.begin.size() - 1;
    group_costs(best.begin, gc);
    std::vector<int> order(G);
    for (int q = 0; q < G; ++q) order[q] = q;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return gc[a] > gc[b]; });
    std::vector<double> load(ctas, 0.0);
    std::vector<std::vector<int>> mine(ctas);
    for (int q : order)
        for (int t = 0; t < tiles; ++t) {
            const int b = (int)(std::min_element(load.begin(), load.end()) - load.begin());
            load[b] += gc[q];
            mine[b].push_back(q * tiles + t);
        }
    best.slots = 0;
    for (auto &v : mine) best.slots = std::max(best.slots, (int)v.size());
    best.flat.assign((size_t)best.slots * ctas, -1);
    double sum = 0.0;
    for (int b = 0; b < ctas; ++b) {
        sum += load[b];
        for (size_t k = 0; k < mine[b].size(); ++k) best.flat[k * ctas + b] = mine[b][k];
    }
    best.mean = sum / ctas;
    return best;
}

// float64 tier helpers
static size_t f64_taps_count(int n_levels, const int32_t *radii, const int64_t *tap_offsets) {
    size_t n = 0;
    for (int i = 0; i < n_levels; ++i) n = std::max(n, (size_t)tap_offsets[i] + 2 * (size_t)radii[i] + 1);
    return n;
}
// device copy of a small host array, freed behind the stream's work
template <typename T>
static cudaError_t upload_async(const T *h, size_t n, T **d, cudaStream_t st) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(d), n * sizeof(T), st);
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(*d, h, n * sizeof(T), cudaMemcpyHostToDevice, st);
}

}  // namespace

extern "C" {

int dogblob_abi_version(void) { return DOGBLOB_ABI_VERSION; }
const char *dogblob_last_error(void) { return g_error.c_str(); }

int dogblob_plan_create(int device, int height, int width, int n_levels, const double *sigmas,
                        const int32_t *radii, const float *taps, const int64_t *tap_offsets,
                        int max_blobs, dogblob_plan **out) {
    DB_REQUIRE(out != nullptr, "out must not be NULL");
    *out = nullptr;
    DB_REQUIRE(height >= 1 && width >= 1, "expected a non-empty 2-D image");
    DB_REQUIRE(n_levels >= 2, "a ladder needs at least two levels");
    DB_REQUIRE(n_levels <= kMaxLevels, "more than 320 ladder levels are not supported");
    DB_REQUIRE(sigmas && radii && taps && tap_offsets, "NULL table");
    DB_REQUIRE(max_blobs >= 1 && max_blobs < (1 << 24), "max_blobs must be in [1, 2^24)");
    DB_REQUIRE(height <= 32768 && width <= 32768, "image dimension above 32768");
    for (int i = 0; i < n_levels; ++i) {
        DB_REQUIRE(sigmas[i] > 0.0, "sigma must be > 0");
        DB_REQUIRE(radii[i] >= 0 && 2 * radii[i] + 1 <= 4097, "kernel width exceeds cap 4097");
    }
    DeviceGuard guard(device);
    DB_REQUIRE(guard.ok, "cannot select CUDA device");

    auto *plan = new dogblob_plan();
    plan->device = device;
    plan->max_blobs = max_blobs;
    plan->sigmas.assign(sigmas, sigmas + n_levels);
    ConvGeometry &g = plan->geo;
    g.H = height; g.W = width; g.L = n_levels;
    g.Hp = round_up(height, kPad);
    g.Wp = round_up(width, kPad);

    // duplicated tap tables (w, w), radius zero-padded to a multiple of 8 so that the
    // sliding-window sweep is a whole number of 16-row chunks (see sweep())
    std::vector<float2> table;
    plan->levels.resize(n_levels);
    int max_table = 0, max_rpad = 0;
    for (int i = 0; i < n_levels; ++i) {
        const int r = radii[i];
        const int rpad = std::max(8, (r + 7) / 8 * 8);
        LevelDesc &lv = plan->levels[i];
        lv.rpad = rpad;
        lv.n_mid = (2 * rpad + kTY) / kTY - 2;
        lv.tap_ofs = (int)table.size();
        lv.sigma_f32 = (float)sigmas[i];
        const int len = 2 * rpad + kTY;      // 2 rpad + 1 taps, then 15 zeros
        max_table = std::max(max_table, len);
        max_rpad = std::max(max_rpad, rpad);
        const float *w = taps + tap_offsets[i];
        for (int m = 0; m < len; ++m) {
            const int k = m - (rpad - r);
            const float v = (k >= 0 && k <= 2 * r) ? w[k] : 0.f;
            table.push_back(make_float2(v, v));
        }
    }
    g.max_table = max_table;
    g.max_rpad = max_rpad;

    // level groups of the fused pass: about two waves of CTAs at 2 CTAs / SM
    const int tiles = (g.Hp / kTileCols) * (g.Wp / kTileRows);
    int G = choose_groups(tiles, n_levels);
    if (const char *env = std::getenv("DOGBLOB_GROUPS")) G = std::max(1, std::atoi(env));
    std::vector<int> group_begin = balance_groups(plan->levels, G);
    // the fused pass stages the tap tables of a whole group in shared memory: split further
    // until two CTAs fit on an SM (one level per group always fits one CTA)
    auto group_table = [&](const std::vector<int> &begin) {
        int worst = 0;
        for (size_t q = 0; q + 1 < begin.size(); ++q) {
            int len = 0;
            for (int i = begin[q]; i < begin[q + 1]; ++i) len += 2 * plan->levels[i].rpad + kTY;
            worst = std::max(worst, len);
        }
        return worst;
    };
    const size_t smem_budget = 113 * 1024;
    while ((int)group_begin.size() - 1 < n_levels &&
           col_pass_smem(group_table(group_begin), max_rpad, true) > smem_budget) {
        ++G;
        group_begin = balance_groups(plan->levels, G);
    }
    g.G = (int)group_begin.size() - 1;
    g.max_group_table = group_table(group_begin);

    // Row-pass launch order: longest levels first (short tail).  Interleaving long and short
    // levels to de-phase co-resident CTAs was measured and does not help.
    std::vector<int> order(n_levels);
    for (int i = 0; i < n_levels; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        return plan->levels[a].n_mid > plan->levels[b].n_mid;
    });
    std::vector<int> unit(n_levels + 1);
    for (int i = 0; i <= n_levels; ++i) unit[i] = i;
    std::vector<float> sig32(n_levels);
    for (int i = 0; i < n_levels; ++i) sig32[i] = (float)sigmas[i];

#define PLAN_CUDA(expr)                                                                \
    do {                                                                               \
        cudaError_t _e = (expr);                                                       \
        if (_e != cudaSuccess) {                                                       \
            set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));             \
            dogblob_plan_destroy(plan);                                                \
            return DOGBLOB_ECUDA;                                                      \
        }                                                                              \
    } while (0)
    std::memset(&plan->table, 0, sizeof(LevelTable));
    for (int i = 0; i < n_levels; ++i) {
        plan->table.lv[i] = plan->levels[i];
        plan->table.order[i] = order[i];
    }
    plan->table.n_levels = n_levels;
    plan->unit_table = plan->table;
    plan->table.n_groups = g.G;
    for (int i = 0; i <= g.G; ++i) plan->table.group_begin[i] = group_begin[i];
    plan->unit_table.n_groups = n_levels;
    for (int i = 0; i <= n_levels; ++i) plan->unit_table.group_begin[i] = unit[i];
    // tensor-core column pass: one persistent CTA per SM, (tile, group) units on a static schedule
    UmmaSchedule usched;
    {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        // The persistent passes leave `spare` SMs free: their CTAs fill an SM's shared memory, so the small
        // kernels of OTHER frames (other streams: single-CTA finalize, plateau, counters) could otherwise only
        // run in the gaps between two passes.  DOGBLOB_UMMA_SPARE_SMS overrides (plan time only).
        int spare = 1;
        if (const char *es = std::getenv("DOGBLOB_UMMA_SPARE_SMS")) spare = std::max(0, std::atoi(es));
        sms = std::max(1, sms - spare);
        plan->umma_ctas = sms;
        const char *ec = std::getenv("DOGBLOB_UMMA_LEVEL_COST");       // plan time only
        const char *eg = std::getenv("DOGBLOB_UMMA_GROUPS");
        usched = plan_umma_schedule(plan->levels, tiles, std::min(sms, tiles * std::max(1, n_levels - 1)),
                                    ec ? std::atof(ec) : 6.0, eg ? std::atoi(eg) : 0);
        const int G_umma = (int)usched.begin.size() - 1;
        plan->umma_table = plan->table;
        plan->umma_table.n_groups = G_umma;
        for (int i = 0; i <= G_umma; ++i) plan->umma_table.group_begin[i] = usched.begin[i];
        plan->umma_sched_slots = usched.slots;
        plan->umma_sched_ctas = (int)(usched.flat.size() / std::max(1, usched.slots));
        if (std::getenv("DOGBLOB_UMMA_PROF"))
            fprintf(stderr, "umma schedule: %d groups, %d slots, makespan %.1f vs mean %.1f k-step units\n", G_umma,
                    usched.slots, usched.makespan, usched.mean);
        if (std::getenv("DOGBLOB_UMMA_PROF_CTAS")) {
            fprintf(stderr, "   groups:");
            for (int i = 0; i <= G_umma; ++i) fprintf(stderr, " %d", usched.begin[i]);
            fprintf(stderr, "\n   units per CTA (group ids):");
            for (int b = 0; b < plan->umma_sched_ctas; ++b) {
                fprintf(stderr, " [");
                for (int k = 0; k < usched.slots; ++k)
                    if (usched.flat[(size_t)k * plan->umma_sched_ctas + b] >= 0)
                        fprintf(stderr, "%d", usched.flat[(size_t)k * plan->umma_sched_ctas + b] / tiles);
                fprintf(stderr, "]");
            }
            fprintf(stderr, "\n");
        }
    }
    PLAN_CUDA(cudaMalloc(&plan->d_taps, table.size() * sizeof(float2)));
    PLAN_CUDA(cudaMalloc(&plan->d_slice_sigma, n_levels * sizeof(double)));
    PLAN_CUDA(cudaMalloc(&plan->d_sigma_f32, n_levels * sizeof(float)));
    PLAN_CUDA(cudaMemcpy(plan->d_taps, table.data(), table.size() * sizeof(float2),
                         cudaMemcpyHostToDevice));
    PLAN_CUDA(cudaMemcpy(plan->d_slice_sigma, sigmas, n_levels * sizeof(double),
                         cudaMemcpyHostToDevice));
    PLAN_CUDA(cudaMemcpy(plan->d_sigma_f32, sig32.data(), n_levels * sizeof(float),
                         cudaMemcpyHostToDevice));
    // Engine choice (plan time).  The Toeplitz GEMM spends 128 + 2 rpad input rows per 128 outputs
    // and level, the sliding window 2 rpad + 33, but on the tensor cores: measured over frame sizes and
    // ladders (tools/engine_crossover.py, profiles/r02_engine_crossover.md) the tensor-core passes win
    // from a mean padded radius of ~28 on (sigma <= 10 at truncate 5: C1) as soon as the frame has six
    // tiles (four from ~40 on), from ~20 on (sigma <= 6: C5) with 36 tiles (1.25 .. 1.7 x on sparse frames; on the dense C5
    // frame, where the column pass stores and seed-tests nearly every box, the two engines are equal),
    // and for any ladder on frames that exceed what the FP32 engine keeps in L2 (>= 128 tiles).  The
    // wider choice is limited to the radii it was measured and validated with (sigma <= 30 at truncate
    // 5); beyond them round 1's rule stands (C4).
    // DOGBLOB_CONV=fma|umma (read here, once per plan) overrides.
    {
        double sum_rpad = 0.0;
        for (int i = 0; i < n_levels; ++i) sum_rpad += plan->levels[i].rpad;
        const double mean_rpad = sum_rpad / n_levels;
        const bool wins = (mean_rpad >= 48.0 && tiles >= 48) ||
                          (g.max_rpad <= 152 && (tiles >= 128 || (mean_rpad >= 40.0 && tiles >= 4) || (mean_rpad >= 28.0 && tiles >= 6) ||
                                                 (mean_rpad >= 20.0 && tiles >= 36)));
        plan->use_umma = umma_supported(g) && wins;
        if (const char *e = std::getenv("DOGBLOB_CONV")) {
            if (e[0] == 'f') plan->use_umma = false;
            if (e[0] == 'u') plan->use_umma = umma_supported(g);
        }
    }
    if (plan->use_umma) {
        std::vector<float> toep;
        std::memset(&plan->toeplitz, 0, sizeof(ToeplitzTable));
        build_toeplitz(plan->levels.data(), n_levels, table.data(), toep, plan->toeplitz);
        PLAN_CUDA(cudaMalloc(&plan->d_toeplitz, toep.size() * sizeof(float)));
        PLAN_CUDA(cudaMemcpy(plan->d_toeplitz, toep.data(), toep.size() * sizeof(float),
                             cudaMemcpyHostToDevice));
        PLAN_CUDA(cudaMalloc(&plan->d_umma_sched, usched.flat.size() * sizeof(int)));
        PLAN_CUDA(cudaMemcpy(plan->d_umma_sched, usched.flat.data(), usched.flat.size() * sizeof(int),
                             cudaMemcpyHostToDevice));
    }
    PLAN_CUDA(configure_conv_kernels(device));
    PLAN_CUDA(configure_umma_kernels(device));
    PLAN_CUDA(configure_finalize_kernels());
#undef PLAN_CUDA

    const size_t plane = (size_t)g.Hp * g.Wp * sizeof(float);
    size_t off = 0;
    if (plan->use_umma) {
        const UmmaLayout ul = umma_layout(g);
        plan->off_rows_t = off; off += align_up(ul.r_bytes, 1024);
        plan->off_x = off;      off += align_up(ul.x_bytes, 1024);
        plan->off_dog_t = off;  off += align_up(plane * n_levels, 1024);   // L planes: also holds levels
        plan->off_edge = off;
    } else {
        plan->off_rows_t = off; off += align_up(plane * n_levels, 256);
        plan->off_x = off;
        plan->off_dog_t = off;  off += align_up(plane * n_levels, 256);   // L planes: also holds levels
        plan->off_edge = off;   off += align_up(plane * 2 * g.G, 256);    // boundary levels
    }
    plan->off_blobspace = off; off += blobspace_bytes(max_blobs);
    plan->off_gate = off;   off += 4096;                                  // streamed upload: gate word; +64: frame max word + partial maxima
    plan->off_flags = off;  off += align_up(hit_flag_bytes(n_levels, g.Hp, g.Wp), 256);   // tensor engine: hit blocks
    if (plan->use_umma) {
        // seeds: a few thousand per frame; one per 64 voxels is far beyond any frame with distinct blobs, and a
        // frame beyond that (flat noise above the threshold) falls back to the strip kernel
        const int64_t voxels = (int64_t)(n_levels - 1) * g.H * g.W;
        plan->seed_cap = (int)std::min<int64_t>(1 << 20, std::max<int64_t>(1 << 16, voxels / 64));
        if (const char *e = std::getenv("DOGBLOB_SEED_CAP")) plan->seed_cap = std::max(0, std::atoi(e));   // tests: force the fallback
        plan->off_seeds = off;  off += align_up((size_t)plan->seed_cap * sizeof(unsigned long long), 256);
    }
    plan->total = off;
    *out = plan;
    return DOGBLOB_OK;
}

void dogblob_plan_destroy(dogblob_plan *plan) {
    if (!plan) return;
    DeviceGuard guard(plan->device);
    cudaFree(plan->d_taps);
    cudaFree(plan->d_toeplitz);
    cudaFree(plan->d_umma_sched);
    cudaFree(plan->d_slice_sigma);
    cudaFree(plan->d_sigma_f32);
    delete plan;
}

size_t dogblob_workspace_bytes(const dogblob_plan *plan) { return plan ? plan->total : 0; }
size_t dogblob_result_bytes_for(int max_blobs) {
    return DOGBLOB_RESULT_HEADER_BYTES + (size_t)std::max(max_blobs, 0) * sizeof(dogblob_blob);
}
size_t dogblob_result_bytes(const dogblob_plan *plan) {
    return plan ? dogblob_result_bytes_for(plan->max_blobs) : 0;
}
int64_t dogblob_image_pitch(const dogblob_plan *plan) { return plan ? plan->geo.Wp : 0; }
int dogblob_plan_conv_engine(const dogblob_plan *plan) { return plan && plan->use_umma ? 2 : 0; }
int dogblob_plan_conv_groups(const dogblob_plan *plan, int32_t *begin, int cap) {
    if (!plan) return 0;
    const LevelTable &t = plan->use_umma ? plan->umma_table : plan->table;
    for (int i = 0; begin && i <= t.n_groups && i < cap; ++i) begin[i] = t.group_begin[i];
    return t.n_groups;
}
size_t dogblob_blobspace_bytes(int max_blobs) { return blobspace_bytes(std::max(max_blobs, 1)); }

static int check_threshold_args(int neighborhood, double overlap) {
    DB_REQUIRE(neighborhood >= 1 && neighborhood % 2 == 1, "neighborhood must be odd and >= 1");
    DB_REQUIRE(overlap >= 0.0 && overlap <= 1.0, "overlap threshold must be in [0, 1]");
    return DOGBLOB_OK;
}

// tensor engine: float bits of the frame's max |x| (scale of the fp16 operand split)
static uint32_t *frame_max_word(const dogblob_plan *plan, void *d_workspace) {
    return reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(d_workspace) + plan->off_gate + 64);
}
// Scale-space pass 1 on the plan's engine: the tensor-core Toeplitz GEMM (scale_space_umma.cu:
// frame -> fp16 hi | lo planes -> level rows) or the FP32 sliding-window kernel (scale_space.cu).
// `reset` (tensor engine only): the frame's counters are cleared by the first kernel of the pass
static cudaError_t row_pass_any(const dogblob_plan *plan, const float *d_image, void *d_workspace,
                                cudaStream_t st, const RowGate *gate, const BlobSpace *reset = nullptr) {
    char *ws = reinterpret_cast<char *>(d_workspace);
    if (plan->use_umma) {
        uint32_t *mx = frame_max_word(plan, d_workspace);
        cudaError_t e = launch_prep_umma(plan->geo, d_image, ws + plan->off_x, mx, st, reset);
        if (e != cudaSuccess) return e;
        return launch_row_pass_umma(plan->geo, ws + plan->off_x, ws + plan->off_rows_t, plan->table,
                                    plan->toeplitz, plan->d_toeplitz, st, mx, plan->umma_ctas);
    }
    return launch_row_pass(plan->geo, d_image, reinterpret_cast<float *>(ws + plan->off_rows_t), plan->table,
                           plan->d_taps, st, gate);
}
static HitFlags hit_flags_of(const dogblob_plan *plan, void *d_workspace) {
    HitFlags f;
    f.data = reinterpret_cast<unsigned char *>(d_workspace) + plan->off_flags;
    f.row_blocks = plan->geo.Wp >> kFlagRowShift;      // blocks of the transposed slices: rows = x, columns = y
    f.col_blocks = plan->geo.Hp >> kFlagColShift;
    if (plan->seed_cap > 0) {
        char *ws = reinterpret_cast<char *>(d_workspace);
        f.seeds = reinterpret_cast<unsigned long long *>(ws + plan->off_seeds);
        f.n_seeds = &carve_blobspace(ws + plan->off_blobspace, plan->max_blobs).ctr->n_seeds;
        f.seed_cap = plan->seed_cap;
    }
    return f;
}
// pass 2 fused with the DoG: both engines write the slices transposed (D^T[slice][x][y]).
// `threshold`: the tensor engine also records which blocks of the slices exceed it (for the extrema
// kernel); NaN = not wanted (stage entry points).
static cudaError_t col_dog_pass_any(const dogblob_plan *plan, void *d_workspace, cudaStream_t st,
                                    float threshold = NAN) {
    char *ws = reinterpret_cast<char *>(d_workspace);
    float *dog = reinterpret_cast<float *>(ws + plan->off_dog_t);
    if (plan->use_umma)
        return launch_col_pass_umma(plan->geo, ws + plan->off_rows_t, dog, plan->umma_table, plan->toeplitz,
                                    plan->d_toeplitz, st, frame_max_word(plan, d_workspace), false,
                                    plan->d_umma_sched, plan->umma_sched_slots, plan->umma_sched_ctas,
                                    threshold, std::isnan(threshold) ? HitFlags{} : hit_flags_of(plan, d_workspace));
    return launch_col_dog_pass(plan->geo, reinterpret_cast<const float *>(ws + plan->off_rows_t), dog,
                               reinterpret_cast<float *>(ws + plan->off_edge), plan->table, plan->d_taps, st);
}
// dense [planes][H][W] copy of the engine's transposed plane stack
static cudaError_t planes_to_dense(const dogblob_plan *plan, const float *d_planes, int planes, float *d_dst,
                                   cudaStream_t st) {
    const ConvGeometry &g = plan->geo;
    return launch_untranspose(d_planes, planes, g.Hp, g.Wp, g.H, g.W, d_dst, st);
}

// reset + row pass (optionally gated on a streamed upload), then the rest of the frame
static int launch_frame_head(const dogblob_plan *plan, const float *d_image, void *d_workspace,
                             cudaStream_t st, void *const *events, const RowGate *gate) {
    char *ws = reinterpret_cast<char *>(d_workspace);
    BlobSpace bs = carve_blobspace(ws + plan->off_blobspace, plan->max_blobs);
    if (events) DB_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(events[0]), st));
    if (!plan->use_umma) DB_CUDA(launch_reset_counters(bs, st));     // tensor engine: folded into its first kernel
    DB_CUDA(row_pass_any(plan, d_image, d_workspace, st, gate, plan->use_umma ? &bs : nullptr));
    if (events) DB_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(events[1]), st));
    return DOGBLOB_OK;
}

static int launch_frame_tail(const dogblob_plan *plan, float threshold, int neighborhood,
                             double overlap, int prune, void *d_workspace, void *d_result,
                             cudaStream_t st, void *const *events) {
    char *ws = reinterpret_cast<char *>(d_workspace);
    float *dog = reinterpret_cast<float *>(ws + plan->off_dog_t);
    BlobSpace bs = carve_blobspace(ws + plan->off_blobspace, plan->max_blobs);
    const ConvGeometry &g = plan->geo;
    auto ev = [&](int k) -> cudaError_t {
        return events ? cudaEventRecord(reinterpret_cast<cudaEvent_t>(events[k]), st)
                      : cudaSuccess;
    };
    const bool use_flags = plan->use_umma && neighborhood == 3 && !std::isnan(threshold);
    DB_CUDA(col_dog_pass_any(plan, d_workspace, st, use_flags ? threshold : NAN));
    DB_CUDA(ev(2));
    // both engines: D^T planes, rows = x (W valid), cols = y (H valid)
    DB_CUDA(launch_extrema(dog, g.L - 1, g.W, g.H, g.Hp, (int64_t)g.Hp * g.Wp, true,
                           plan->d_slice_sigma, threshold, neighborhood / 2, bs, st,
                           use_flags ? hit_flags_of(plan, d_workspace) : HitFlags{}));
    DB_CUDA(ev(3));
    DB_CUDA(launch_prune_and_pack(bs, overlap, prune != 0, d_result, plan->max_blobs, st));
    DB_CUDA(ev(4));
    return DOGBLOB_OK;
}

int dogblob_detect(const dogblob_plan *plan, const float *d_image, float threshold,
                   int neighborhood, double overlap, int prune, void *d_workspace,
                   void *d_result, void *stream, void *const *events) {
    DB_REQUIRE(plan && d_image && d_workspace && d_result, "NULL argument");
    if (int rc = check_threshold_args(neighborhood, overlap)) return rc;
    DeviceGuard guard(plan->device);
    DB_REQUIRE(guard.ok, "cannot select CUDA device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (int rc = launch_frame_head(plan, d_image, d_workspace, st, events, nullptr)) return rc;
    return launch_frame_tail(plan, threshold, neighborhood, overlap, prune, d_workspace, d_result, st,
                             events);
}

int dogblob_upload_image(const dogblob_plan *plan, const float *h_image, void *d_image,
                         void *stream) {
    DB_REQUIRE(plan && h_image && d_image, "NULL argument");
    DeviceGuard guard(plan->device);
    DB_REQUIRE(guard.ok, "cannot select CUDA device");
    const ConvGeometry &g = plan->geo;
    DB_CUDA(cudaMemcpy2DAsync(d_image, (size_t)g.Wp * sizeof(float), h_image,
                              (size_t)g.W * sizeof(float), (size_t)g.W * sizeof(float), g.H,
                              cudaMemcpyHostToDevice, reinterpret_cast<cudaStream_t>(stream)));
    return DOGBLOB_OK;
}

int dogblob_detect_host(const dogblob_plan *plan, const float *h_image, float threshold,
                        int neighborhood, double overlap, int prune, void *d_image,
                        void *d_workspace, void *d_result, void *h_result, int h_result_blobs,
                        void *stream, void *const *events) {
    DB_REQUIRE(h_result != nullptr && h_result_blobs >= 0, "bad host result buffer");
    if (int rc = dogblob_upload_image(plan, h_image, d_image, stream)) return rc;
    if (int rc = dogblob_detect(plan, reinterpret_cast<const float *>(d_image), threshold,
                                neighborhood, overlap, prune, d_workspace, d_result, stream,
                                events))
        return rc;
    const int nb = std::min(h_result_blobs, plan->max_blobs);
    DB_CUDA(cudaMemcpyAsync(h_result, d_result,
                            DOGBLOB_RESULT_HEADER_BYTES + (size_t)nb * sizeof(dogblob_blob),
                            cudaMemcpyDeviceToHost, reinterpret_cast<cudaStream_t>(stream)));
    return DOGBLOB_OK;
}

int dogblob_detect_host_streamed(const dogblob_plan *plan, const float *h_image, float threshold,
                                 int neighborhood, double overlap, int prune, void *d_image,
                                 void *d_workspace, void *d_result, void *h_result,
                                 int h_result_blobs, void *stream, void *copy_stream,
                                 int32_t *h_gate, void *frame_done, void *const *events) {
    DB_REQUIRE(plan && h_image && d_image && d_workspace && d_result, "NULL argument");
    DB_REQUIRE(h_result != nullptr && h_result_blobs >= 0, "bad host result buffer");
    DB_REQUIRE(copy_stream && h_gate && frame_done && copy_stream != stream,
               "streamed upload needs its own copy stream, a pinned gate array and an event");
    if (int rc = check_threshold_args(neighborhood, overlap)) return rc;
    // the tensor engine's fp16 operand split needs the whole frame's maximum before its first MMA
    DB_REQUIRE(!plan->use_umma, "streamed upload is only available on the FP32 engine "
                                "(dogblob_plan_conv_engine() == 0); use dogblob_detect_host");
    DeviceGuard guard(plan->device);
    DB_REQUIRE(guard.ok, "cannot select CUDA device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(copy_stream);
    cudaEvent_t done = reinterpret_cast<cudaEvent_t>(frame_done);
    const ConvGeometry &g = plan->geo;
    int *d_word = reinterpret_cast<int *>(reinterpret_cast<char *>(d_workspace) + plan->off_gate);

    // row chunks: at most DOGBLOB_GATE_CHUNKS, whole multiples of 64 rows
    int rows_per_chunk = ((g.H + DOGBLOB_GATE_CHUNKS - 1) / DOGBLOB_GATE_CHUNKS + 63) / 64 * 64;
    const int n_chunks = (g.H + rows_per_chunk - 1) / rows_per_chunk;
    // h_gate[0]: gate value before this frame (0 = first use: initialise the device word);
    // h_gate[1 + c]: value copied behind chunk c.  The previous frame of these buffers has been
    // collected by the caller, so its copies are complete and the array can be rewritten.
    if (h_gate[0] == 0) {
        h_gate[0] = 1;
        DB_CUDA(cudaMemcpy(d_word, h_gate, sizeof(int), cudaMemcpyHostToDevice));
    }
    const int base = h_gate[0];
    for (int c = 0; c < n_chunks; ++c) h_gate[1 + c] = base + c + 1;
    h_gate[0] = base + n_chunks;
    if (h_gate[0] > 0x3fffffff) h_gate[0] = 0;   // re-initialise long before the counter wraps

    DB_CUDA(cudaStreamWaitEvent(cs, done, 0));    // the buffers' previous frame is off the device
    BlobSpace bs0 = carve_blobspace(reinterpret_cast<char *>(d_workspace) + plan->off_blobspace,
                                    plan->max_blobs);
    const RowGate gate{d_word, base, rows_per_chunk, &bs0.ctr->t_start};
    if (int rc = launch_frame_head(plan, reinterpret_cast<const float *>(d_image), d_workspace, st,
                                   events, &gate))
        return rc;
    // from here on the row pass is spinning on the gate: every path must deliver the last value
    cudaError_t err = cudaSuccess;
    for (int c = 0; c < n_chunks && err == cudaSuccess; ++c) {
        const int r0 = c * rows_per_chunk, nr = std::min(rows_per_chunk, g.H - r0);
        err = cudaMemcpy2DAsync(reinterpret_cast<float *>(d_image) + (size_t)r0 * g.Wp,
                                (size_t)g.Wp * sizeof(float), h_image + (size_t)r0 * g.W,
                                (size_t)g.W * sizeof(float), (size_t)g.W * sizeof(float), nr,
                                cudaMemcpyHostToDevice, cs);
        if (err == cudaSuccess)
            err = cudaMemcpyAsync(d_word, h_gate + 1 + c, sizeof(int), cudaMemcpyHostToDevice, cs);
    }
    if (err != cudaSuccess) {
        cudaMemcpy(d_word, h_gate + n_chunks, sizeof(int), cudaMemcpyHostToDevice);   // release the kernel
        set_error(std::string("streamed upload: ") + cudaGetErrorString(err));
        return DOGBLOB_ECUDA;
    }
    if (int rc = launch_frame_tail(plan, threshold, neighborhood, overlap, prune, d_workspace,
                                   d_result, st, events))
        return rc;
    const int nb = std::min(h_result_blobs, plan->max_blobs);
    DB_CUDA(cudaMemcpyAsync(h_result, d_result,
                            DOGBLOB_RESULT_HEADER_BYTES + (size_t)nb * sizeof(dogblob_blob),
                            cudaMemcpyDeviceToHost, st));
    DB_CUDA(cudaEventRecord(done, st));
    return DOGBLOB_OK;
}

int dogblob_fetch_blobs(const void *d_result, int first, int count, dogblob_blob *h_out,
                        void *stream) {
    DB_REQUIRE(d_result && h_out && first >= 0 && count >= 0, "bad argument");
    if (count == 0) return DOGBLOB_OK;
    const char *src = reinterpret_cast<const char *>(d_result) + DOGBLOB_RESULT_HEADER_BYTES +
                      (size_t)first * sizeof(dogblob_blob);
    DB_CUDA(cudaMemcpyAsync(h_out, src, (size_t)count * sizeof(dogblob_blob),
                            cudaMemcpyDeviceToHost, reinterpret_cast<cudaStream_t>(stream)));
    return DOGBLOB_OK;
}

int dogblob_fetch_result(const void *d_result, int n_blobs, void *h_result, void *stream) {
    DB_REQUIRE(d_result && h_result && n_blobs >= 0, "bad argument");
    DB_CUDA(cudaMemcpyAsync(h_result, d_result,
                            DOGBLOB_RESULT_HEADER_BYTES + (size_t)n_blobs * sizeof(dogblob_blob),
                            cudaMemcpyDeviceToHost, reinterpret_cast<cudaStream_t>(stream)));
    return DOGBLOB_OK;
}

int dogblob_scale_space(const dogblob_plan *plan, const float *d_image, void *d_workspace,
                        float *d_levels, void *stream) {
    DB_REQUIRE(plan && d_image && d_workspace && d_levels, "NULL argument");
    DeviceGuard guard(plan->device);
    DB_REQUIRE(guard.ok, "cannot select CUDA device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    char *ws = reinterpret_cast<char *>(d_workspace);
    float *lev = reinterpret_cast<float *>(ws + plan->off_dog_t);
    const ConvGeometry &g = plan->geo;
    DB_CUDA(row_pass_any(plan, d_image, d_workspace, st, nullptr));
    if (plan->use_umma)
        DB_CUDA(launch_col_pass_umma(g, ws + plan->off_rows_t, lev, plan->unit_table, plan->toeplitz,
                                     plan->d_toeplitz, st, frame_max_word(plan, d_workspace), true, nullptr, 0, 0));
    else
        DB_CUDA(launch_col_levels_pass(g, reinterpret_cast<const float *>(ws + plan->off_rows_t), lev,
                                       plan->unit_table, plan->d_taps, st));
    DB_CUDA(planes_to_dense(plan, lev, g.L, d_levels, st));
    return DOGBLOB_OK;
}

int dogblob_dog(const dogblob_plan *plan, const float *d_image, void *d_workspace,
                float *d_slices, void *stream) {
    DB_REQUIRE(plan && d_image && d_workspace && d_slices, "NULL argument");
    DeviceGuard guard(plan->device);
    DB_REQUIRE(guard.ok, "cannot select CUDA device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    char *ws = reinterpret_cast<char *>(d_workspace);
    float *dog = reinterpret_cast<float *>(ws + plan->off_dog_t);
    DB_CUDA(row_pass_any(plan, d_image, d_workspace, st, nullptr));
    DB_CUDA(col_dog_pass_any(plan, d_workspace, st));
    DB_CUDA(planes_to_dense(plan, dog, plan->geo.L - 1, d_slices, st));
    return DOGBLOB_OK;
}

int dogblob_dog_from_levels(int n_levels, int height, int width, const float *d_levels,
                            const double *sigmas, float *d_slices, void *stream) {
    DB_REQUIRE(n_levels >= 2 && height >= 1 && width >= 1, "bad stack shape");
    DB_REQUIRE(d_levels && sigmas && d_slices, "NULL argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    std::vector<float> s32(n_levels);
    for (int i = 0; i < n_levels; ++i) s32[i] = (float)sigmas[i];
    float *d_s = nullptr;
    DB_CUDA(cudaMallocAsync(&d_s, n_levels * sizeof(float), st));
    DB_CUDA(cudaMemcpyAsync(d_s, s32.data(), n_levels * sizeof(float), cudaMemcpyHostToDevice, st));
    DB_CUDA(cudaStreamSynchronize(st));   // s32 is a stack-lifetime host buffer
    DB_CUDA(launch_dog_from_levels(n_levels, (int64_t)height * width, d_levels, d_s, d_slices, st));
    DB_CUDA(cudaFreeAsync(d_s, st));
    return DOGBLOB_OK;
}

int dogblob_extrema(int n_slices, int height, int width, const float *d_slices,
                    const double *slice_sigmas, float threshold, int neighborhood, int max_blobs,
                    void *d_blobspace, void *d_result, void *stream) {
    DB_REQUIRE(n_slices >= 1 && height >= 1 && width >= 1, "bad stack shape");
    DB_REQUIRE(d_slices && slice_sigmas && d_blobspace && d_result && max_blobs >= 1,
               "bad argument");
    if (int rc = check_threshold_args(neighborhood, 0.0)) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    BlobSpace bs = carve_blobspace(d_blobspace, max_blobs);
    double *d_sig = nullptr;
    DB_CUDA(cudaMallocAsync(&d_sig, n_slices * sizeof(double), st));
    DB_CUDA(cudaMemcpyAsync(d_sig, slice_sigmas, n_slices * sizeof(double),
                            cudaMemcpyHostToDevice, st));
    DB_CUDA(cudaStreamSynchronize(st));
    DB_CUDA(configure_finalize_kernels());
    DB_CUDA(launch_reset_counters(bs, st));
    DB_CUDA(launch_extrema(d_slices, n_slices, height, width, width, (int64_t)height * width,
                           false, d_sig, threshold, neighborhood / 2, bs, st));
    DB_CUDA(launch_prune_and_pack(bs, 0.0, false, d_result, max_blobs, st));
    DB_CUDA(cudaFreeAsync(d_sig, st));
    return DOGBLOB_OK;
}

// ---- float64 tier -------------------------------------------------------------------------------
size_t dogblob_f64_workspace_bytes(int height, int width, int n_levels, int max_blobs) {
    const size_t plane = align_up((size_t)std::max(height, 1) * std::max(width, 1) * sizeof(double), 256);
    return plane * ((size_t)std::max(n_levels, 1) + 1) + blobspace_bytes(std::max(max_blobs, 1));
}

int dogblob_scale_space_f64(int height, int width, int n_levels, const int32_t *radii, const double *taps,
                            const int64_t *tap_offsets, const double *d_image, double *d_tmp,
                            double *d_levels, void *stream) {
    DB_REQUIRE(height >= 1 && width >= 1, "expected a non-empty 2-D image");
    DB_REQUIRE(n_levels >= 1 && radii && taps && tap_offsets && d_image && d_tmp && d_levels, "bad argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    double *d_taps = nullptr;
    DB_CUDA(upload_async(taps, f64_taps_count(n_levels, radii, tap_offsets), &d_taps, st));
    DB_CUDA(cudaStreamSynchronize(st));          // the host array may be released by the caller
    DB_CUDA(launch_scale_space_f64(height, width, n_levels, radii, d_taps, tap_offsets, d_image, d_tmp, d_levels, st));
    DB_CUDA(cudaFreeAsync(d_taps, st));
    return DOGBLOB_OK;
}

int dogblob_dog_inplace_f64(int n_levels, int height, int width, double *d_levels, const double *sigmas,
                            void *stream) {
    DB_REQUIRE(n_levels >= 2 && height >= 1 && width >= 1 && d_levels && sigmas, "bad argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    double *d_sig = nullptr;
    DB_CUDA(upload_async(sigmas, (size_t)n_levels, &d_sig, st));
    DB_CUDA(cudaStreamSynchronize(st));
    DB_CUDA(launch_dog_inplace_f64(n_levels, (int64_t)height * width, d_levels, d_sig, st));
    DB_CUDA(cudaFreeAsync(d_sig, st));
    return DOGBLOB_OK;
}

int dogblob_extrema_f64(int n_slices, int height, int width, const double *d_slices,
                        const double *slice_sigmas, double threshold, int neighborhood, int max_blobs,
                        void *d_blobspace, void *d_result, void *stream) {
    DB_REQUIRE(n_slices >= 1 && height >= 1 && width >= 1, "bad stack shape");
    DB_REQUIRE(d_slices && slice_sigmas && d_blobspace && d_result && max_blobs >= 1, "bad argument");
    if (int rc = check_threshold_args(neighborhood, 0.0)) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    BlobSpace bs = carve_blobspace(d_blobspace, max_blobs);
    double *d_sig = nullptr;
    DB_CUDA(upload_async(slice_sigmas, (size_t)n_slices, &d_sig, st));
    DB_CUDA(cudaStreamSynchronize(st));
    DB_CUDA(configure_finalize_kernels());
    DB_CUDA(launch_reset_counters(bs, st));
    DB_CUDA(launch_extrema_f64(d_slices, n_slices, height, width, d_sig, threshold, neighborhood / 2, bs, st));
    DB_CUDA(launch_prune_and_pack(bs, 0.0, false, d_result, max_blobs, st));
    DB_CUDA(cudaFreeAsync(d_sig, st));
    return DOGBLOB_OK;
}

int dogblob_detect_f64(int height, int width, int n_levels, const double *sigmas, const int32_t *radii,
                       const double *taps, const int64_t *tap_offsets, const double *d_image,
                       double threshold, int neighborhood, double overlap, int prune, int max_blobs,
                       void *d_workspace, void *d_result, void *stream) {
    DB_REQUIRE(height >= 1 && width >= 1, "expected a non-empty 2-D image");
    DB_REQUIRE(n_levels >= 2, "a ladder needs at least two levels");
    DB_REQUIRE(sigmas && radii && taps && tap_offsets && d_image && d_workspace && d_result && max_blobs >= 1,
               "bad argument");
    if (int rc = check_threshold_args(neighborhood, overlap)) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t plane = align_up((size_t)height * width * sizeof(double), 256);
    char *ws = reinterpret_cast<char *>(d_workspace);
    double *d_tmp = reinterpret_cast<double *>(ws);
    double *d_levels = reinterpret_cast<double *>(ws + plane);
    BlobSpace bs = carve_blobspace(ws + plane * ((size_t)n_levels + 1), max_blobs);
    double *d_taps = nullptr, *d_sig = nullptr;
    DB_CUDA(upload_async(taps, f64_taps_count(n_levels, radii, tap_offsets), &d_taps, st));
    DB_CUDA(upload_async(sigmas, (size_t)n_levels, &d_sig, st));
    DB_CUDA(cudaStreamSynchronize(st));
    DB_CUDA(configure_finalize_kernels());
    DB_CUDA(launch_reset_counters(bs, st));
    // dense planes of exactly H * W doubles: the level stack starts one (aligned) plane into the workspace
    DB_CUDA(launch_scale_space_f64(height, width, n_levels, radii, d_taps, tap_offsets, d_image, d_tmp, d_levels, st));
    DB_CUDA(launch_dog_inplace_f64(n_levels, (int64_t)height * width, d_levels, d_sig, st));
    DB_CUDA(launch_extrema_f64(d_levels, n_levels - 1, height, width, d_sig, threshold, neighborhood / 2, bs, st));
    DB_CUDA(launch_prune_and_pack(bs, overlap, prune != 0, d_result, max_blobs, st));
    DB_CUDA(cudaFreeAsync(d_taps, st));
    DB_CUDA(cudaFreeAsync(d_sig, st));
    return DOGBLOB_OK;
}

int dogblob_match_voc(int n_jobs, const double *d_pred, const int32_t *d_pred_begin, const double *d_truth,
                      const int32_t *d_truth_begin, double iou_threshold, void *d_taken, int32_t *d_match,
                      double *d_match_iou, int32_t *d_tp, void *stream) {
    DB_REQUIRE(n_jobs >= 0, "bad job count");
    DB_REQUIRE(iou_threshold > 0.0 && iou_threshold <= 1.0, "iou_threshold must be in (0, 1]");
    if (n_jobs == 0) return DOGBLOB_OK;
    DB_REQUIRE(d_pred_begin && d_truth_begin && d_tp, "NULL argument");
    DB_CUDA(launch_match_voc(n_jobs, d_pred, d_pred_begin, d_truth, d_truth_begin, iou_threshold,
                             reinterpret_cast<unsigned char *>(d_taken), d_match, d_match_iou, d_tp,
                             reinterpret_cast<cudaStream_t>(stream)));
    return DOGBLOB_OK;
}

int dogblob_synth_frames(int n_frames, int height, int width, int64_t pitch, int n_droplets, double r_min,
                         double r_max, uint64_t seed, double poisson_scale, double gaussian_sigma,
                         float *d_frames, double *d_truth, void *stream) {
    DB_REQUIRE(n_frames >= 1 && height >= 1 && width >= 1 && pitch >= width, "bad frame geometry");
    DB_REQUIRE(n_droplets >= 0, "n_spheres must be >= 0");
    DB_REQUIRE(r_min > 0.0 && r_max >= r_min, "bad radius range");
    DB_REQUIRE(std::min(width, height) >= 2.0 * r_max + 3.0, "radius cannot fit inside the frame");
    DB_REQUIRE(poisson_scale >= 0.0 && gaussian_sigma >= 0.0, "bad noise parameters");
    DB_REQUIRE(d_frames && (n_droplets == 0 || d_truth), "NULL argument");
    DB_CUDA(launch_synth_frames(n_frames, height, width, pitch, n_droplets, r_min, r_max, seed, poisson_scale,
                                gaussian_sigma, d_frames, d_truth, reinterpret_cast<cudaStream_t>(stream)));
    return DOGBLOB_OK;
}

int dogblob_prune(int n, const dogblob_blob *d_blobs_in, double overlap, int max_blobs,
                  void *d_blobspace, void *d_result, void *stream) {
    DB_REQUIRE(n >= 0 && max_blobs >= 1 && n <= max_blobs, "blob count exceeds max_blobs");
    DB_REQUIRE(d_blobspace && d_result && (n == 0 || d_blobs_in), "NULL argument");
    if (int rc = check_threshold_args(3, overlap)) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    BlobSpace bs = carve_blobspace(d_blobspace, max_blobs);
    DB_CUDA(configure_finalize_kernels());
    DB_CUDA(launch_reset_counters(bs, st));
    DB_CUDA(launch_load_blobs(bs, d_blobs_in, n, st));
    DB_CUDA(launch_prune_and_pack(bs, overlap, true, d_result, max_blobs, st));
    return DOGBLOB_OK;
}

int dogblob_event_create(void **event) {
    DB_REQUIRE(event != nullptr, "NULL argument");
    cudaEvent_t e;
    DB_CUDA(cudaEventCreate(&e));
    *event = e;
    return DOGBLOB_OK;
}
int dogblob_event_destroy(void *event) {
    DB_CUDA(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(event)));
    return DOGBLOB_OK;
}
int dogblob_event_elapsed_ms(void *start, void *stop, float *ms) {
    DB_REQUIRE(ms != nullptr, "NULL argument");
    DB_CUDA(cudaEventElapsedTime(ms, reinterpret_cast<cudaEvent_t>(start),
                                 reinterpret_cast<cudaEvent_t>(stop)));
    return DOGBLOB_OK;
}
int dogblob_event_intervals_ms(void *const *events, int n_events, float *out_ms) {
    DB_REQUIRE(events != nullptr && out_ms != nullptr && n_events >= 2, "bad argument");
    for (int k = 0; k + 1 < n_events; ++k)
        DB_CUDA(cudaEventElapsedTime(out_ms + k, reinterpret_cast<cudaEvent_t>(events[k]),
                                     reinterpret_cast<cudaEvent_t>(events[k + 1])));
    return DOGBLOB_OK;
}
int dogblob_stream_sync(void *stream) {
    DB_CUDA(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)));
    return DOGBLOB_OK;
}
int dogblob_device_count(int *count) {
    DB_REQUIRE(count != nullptr, "NULL argument");
    DB_CUDA(cudaGetDeviceCount(count));
    return DOGBLOB_OK;
}
int dogblob_device_alloc(int device, size_t bytes, void **out) {
    DB_REQUIRE(out != nullptr && bytes > 0, "bad argument");
    *out = nullptr;
    DeviceGuard guard(device);
    DB_REQUIRE(guard.ok, "cannot select CUDA device");
    DB_CUDA(cudaMalloc(out, bytes));
    DB_CUDA(cudaMemset(*out, 0, bytes));
    return DOGBLOB_OK;
}
int dogblob_device_free(int device, void *ptr) {
    if (!ptr) return DOGBLOB_OK;
    DeviceGuard guard(device);
    DB_REQUIRE(guard.ok, "cannot select CUDA device");
    DB_CUDA(cudaFree(ptr));
    return DOGBLOB_OK;
}
int dogblob_pinned_alloc(size_t bytes, void **out) {
    DB_REQUIRE(out != nullptr && bytes > 0, "bad argument");
    *out = nullptr;
    DB_CUDA(cudaMallocHost(out, bytes));
    std::memset(*out, 0, bytes);
    return DOGBLOB_OK;
}
int dogblob_pinned_free(void *ptr) {
    if (ptr) DB_CUDA(cudaFreeHost(ptr));
    return DOGBLOB_OK;
}

}  // extern "C"
