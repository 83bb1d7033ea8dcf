// tc_internal.h -- host-side internal interfaces between the library's translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdlib.h>
#include <stdint.h>

#include <string>

namespace tc {

// ------------------------------------------------------------------ errors ---
void set_error(const std::string &msg);
const char *last_error();

#define TC_CUDA(expr)                                                                    \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess) {                                                         \
            ::tc::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" + \
                            __FILE__ + ":" + std::to_string(__LINE__) + ")");            \
            return -2;                                                                   \
        }                                                                                \
    } while (0)

// Every kernel launch site ends with TC_LAUNCHED(): counts the launch (tc_launch_count)
// and surfaces launch errors.
void note_launch();
#define TC_LAUNCHED()                          \
    do {                                       \
        ::tc::note_launch();                   \
        TC_CUDA(cudaGetLastError());           \
    } while (0)

#define TC_CHECK(expr)             \
    do {                           \
        int _rc = (expr);          \
        if (_rc != 0) return _rc;  \
    } while (0)

// ---------------------------------------------------------- schedule options ---
// Count/preprocess schedule parameters.  The defaults are the measured-best schedule; they
// change only through tc_set_option() (an explicit ABI call used by the schedule-coverage
// tests and the development probes) -- never through the environment, so a stray variable
// cannot change what the product runs.  Every schedule computes the same exact count.
struct Options {
    int64_t vmajor = -1;         // v-major in-edge schedule: -1 auto, 0 off, 1 on
    int64_t vzone_log2 = 23;     // v-major zone = top 2^vzone_log2 ranks (clamped to [18, 31]; 22: +1 ms)
    int64_t vlow_all = 1;        // heads below the hub zone may run v-major
    int64_t vm_bias = 3;         // per-edge choice bias: v-major iff bias/4 * vcost < ucost (4: +1.5 ms)
    int64_t dense_factor = 3;    // AND a dense head's bitmap when words < factor * items
    int64_t hub_unroll = 4;      // k_count_hub sweep unroll (2..4)
    int64_t l2_persist_mb = 32;  // u-major-only schedule: persisting-L2 window size
    int64_t l2_target = 0;       // 0: tail of dense bitmaps, 1: tail of edge_dst
    int64_t concurrent = 0;      // v-major kernels on a second stream
    int64_t share = 1;           // SM share per concurrent kernel
    int64_t midwarp = 1;         // warp-per-task kernel for the mid class (0 off, 2 also class 1)
    int64_t light = -1;          // light kernel: -1 auto, 0 CTA windows, 1 thread/edge, 2 warp windows
    int64_t skew = 32;           // warp-window light kernel: binary-search ratio
    int64_t light_vec = 0;       // thread/edge light kernel: vector loads of the suffix
    int64_t shard_model = 0;     // tc_work_bounds model (0: capped work, 1: rank model)
    int64_t shard_ovh = 128;     // per-edge constant of the rank-space shard model
    int64_t shard_ucap = 1024;   // cap on d+(u) in the rank-space shard model
    int64_t shard_ovh2 = 256;    // per-edge byte-equivalent overhead of shard model 2
    int64_t copy_threads = 0;    // host threads of the staged pageable H2D copy (0: auto)
    int64_t seg_fork = 1;        // rank-space preprocess: size-class sorts on concurrent streams
    int64_t vin_overlap = 1;     // v-major in-edge index on a side stream beside the u-major kernels
    int64_t vin_grid = 4;        // CTAs per SM of the in-edge fill when it overlaps
    int64_t vhub_unroll = 2;     // k_count_vhub: 16-byte chunks per lane per pipelined round (1, 2, 4)
    int64_t vhub_blocks = 1;     // k_count_vhub: source blocks of the top-band tasks (<= 1: unblocked)
    int64_t vhub_b16w = 4;       // per-edge choice: bytes charged per 16-bit suffix item (4 = as 32-bit)
    int64_t hub_cap_div = 8;     // k_count_hub: cuckoo table of the non-hub part sized max / div
    int64_t vix = 1;             // rank-space preprocess fills the v-major in-edge index in the sorts
    int64_t vhub = 1;            // hub heads of the v-major schedule on k_count_vhub (lean sweep, 16-bit top band)
    int64_t seg_w2k = 0;         // rank-space preprocess: 1025..2048-element lists on a warp register sort
    int64_t seg_k16 = 1;         // rank-space preprocess: 257..512-element lists on a 512-wide sort
    int64_t dense_ranks = 1 << 17;  // dense-hub bitmaps for the top ranks
    int64_t bucket = 1;          // rank-space preprocess: bucket scatter + segmented sort
    int64_t count_stats = 0;     // tc_count_with_timings fills the per-kernel-class fields
    int64_t hubpack = 0;         // 1: hub-head suffixes read from an 18-bit packed copy (slower)
    int64_t rank_primary = 1;    // tc_preprocess builds the rank-space CSR, reference ids lazily
    // shard plan class weights (1/1000 ps per byte; per edge / in-edge), fitted -- tc_count.cu
    int64_t shard_w_dense = 118, shard_w_sparse = 273, shard_w_light = 5500, shard_w_stage = 18000;
    int64_t shard_w_edge = 0, shard_w_hub = 153, shard_w_vlow = 300, shard_w_vedge = 62000;
};
Options &opts();

// ------------------------------------------------------------------ memory ---
// Stream-ordered allocations.  Per-call scratch comes from a dedicated pool (release
// threshold "keep everything"), so the same-sized temporaries of repeated calls are
// reused without remapping; graphs handed to the caller (persistent) come from the
// device's default pool, so they never fragment the scratch pool.
int dalloc(void **p, size_t bytes, cudaStream_t s, bool persistent = false);
void dfree(void *p, cudaStream_t s);
cudaMemPool_t scratch_pool();

template <typename T>
int dalloc_t(T **p, size_t count, cudaStream_t s, bool persistent = false) {
    return dalloc(reinterpret_cast<void **>(p), count * sizeof(T), s, persistent);
}

// ------------------------------------------------------------- radix sort ---
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
#ifndef TC_SORT_THREADS
#define TC_SORT_THREADS 256
#endif
#ifndef TC_SORT_KPT
#define TC_SORT_KPT 16
#endif
constexpr int kSortThreads = TC_SORT_THREADS;
constexpr int kSortKPT = TC_SORT_KPT;
constexpr int kSortTile = kSortThreads * kSortKPT;  // 4096 keys per tile
constexpr int kMaxPasses = 8;

struct RadixPlan {
    int npass = 0;
    int shift[kMaxPasses] = {0};
    int bits[kMaxPasses] = {0};
};
RadixPlan make_radix_plan(int key_bits);

enum SortOut { kOutKeys = 0, kOutSoA = 1, kOutAoS = 2 };

// Device histogram of every pass's digit over `keys` (adds into hist[npass][kRadix]).
int radix_histogram(const uint64_t *keys, uint64_t n, const RadixPlan &plan, uint32_t *hist,
                    cudaStream_t s);

// LSD radix sort of n 64-bit keys (optionally carrying a 32-bit payload) over the plan's
// bits.  `hist` is the per-pass digit histogram (from radix_histogram or fused into a
// producer kernel).  keys/alt (and vals/valt) are ping-pong buffers.  With out_mode
// kOutSoA / kOutAoS the last pass writes (key >> split, key & mask) to out_a/out_b
// (SoA) or out_a as uint2 pairs (AoS); otherwise *sorted_keys (*sorted_vals) points at
// whichever ping-pong buffer holds the result.
int radix_sort(uint64_t *keys, uint64_t *alt, uint32_t *vals, uint32_t *valt, uint64_t n,
               const RadixPlan &plan, const uint32_t *hist, int out_mode, uint32_t *out_a,
               uint32_t *out_b, int split_bits, uint64_t **sorted_keys, uint32_t **sorted_vals,
               cudaStream_t s);

inline int bits_for(uint64_t maxval) {
    int b = 0;
    while (b < 64 && (maxval >> b) != 0) ++b;
    return b;
}

// The per-edge v-major choice parameters (tc_vsplit.cuh: vmajor_edge).
struct VSplit {
    uint32_t z0, hz, vt, hwp, factor, nhcap;  // v-major zone [z0, n); z0 = ~0: v-major off
    uint32_t bias;                            // v-major iff bias/4 * vcost < ucost
    uint32_t lowall;                          // below hz: 0 = short suffixes only, 1 = by bytes
    const uint32_t *hubstart;
    uint32_t packed = 0;                      // hub-head suffixes read from the 18-bit copy
    uint32_t packed_cost = 0;                 // the per-edge choice charges packed bytes
    uint32_t t16 = 0xffffffffu;               // heads >= t16 read 16-bit suffixes (k_count_vhub)
    uint32_t b16w = 4;                        // ... charged b16w bytes per suffix item
};

// ------------------------------------------------------------ device graph ---
struct DeviceGraph {
    uint64_t m = 0, n = 0;
    uint32_t *src = nullptr;   // edge_src  u32[m]
    uint32_t *dst = nullptr;   // edge_dst  u32[m] (+ padding)
    int64_t *off = nullptr;    // node_offsets i64[n+1]
    uint32_t *off32 = nullptr; // u32 copy of node_offsets when m < 2^32 (count kernels)
    uint32_t max_out = 0;      // max out-degree
    int device = 0;
    // Rank space: vertices relabelled by their (degree, id) rank, so orientation is
    // "low rank -> high rank" and the hub zone [hz, n) holds the top kHubRanks ranks.
    // hubstart[v] = first position of adj(v) whose rank is >= hz (lists are sorted).
    bool rank_space = false;
    uint32_t hz = 0;
    uint32_t *hubstart = nullptr;
    bool hubstart_ready = false;  // hubstart filled by the rank-space segmented sort
    // Dense hubs: every vertex v of rank >= vt (the top kDenseRanks) also has adj(v) as a
    // bitmap over hub-zone words [ws4(v), hwp) at dense_bits + dense_off[v - vt], where
    // ws4(v) = ((v + 1 - hz) / 32) rounded down to a multiple of 4 and hwp = hub-zone
    // words rounded up to a multiple of 4.
    uint32_t vt = 0, hwp = 0, dense_words = 0;
    uint32_t *dense_off = nullptr;   // [n - vt + 1] word offsets (multiples of 4)
    uint32_t *dense_bits = nullptr;
    bool persistent = false;  // arrays from the default pool (outlive the call)
    // v-major in-edge capacity layout (rank-space preprocessing only): vin_cap[i] = in-degree
    // prefix over the v-major zone [vin_z0, n) (exclusive scan, n - vin_z0 + 1 entries)
    uint32_t *vin_cap = nullptr;
    uint32_t vin_z0 = 0;
    uint64_t vin_total = 0;  // vin_cap[n - vin_z0]
    // v-major in-edge index filled by the rank-space segmented sorts (full-range counts whose
    // split equals vix_vp use it instead of k_vin_pass): fill counts and (edge, end) entries
    uint32_t *vix_cnt = nullptr;
    uint2 *vix_in_e = nullptr;
    VSplit vix_vp{};
    bool vix_ready = false;
};

// First vertex of the v-major zone: the top 2^vzone_log2 ranks (default 2^22), never
// above the hub zone start hz.
inline uint32_t vzone_start_of(uint64_t n, uint32_t hz) {
    const int64_t lg = opts().vzone_log2;
    const uint64_t Z = 1ull << (lg < 18 ? 18 : lg > 31 ? 31 : lg);
    const uint64_t z0 = n > Z ? n - Z : 0;
    return (uint32_t)(z0 < hz ? z0 : hz);
}
// vin_cap for a rank-space graph from its degrees in rank order (tc_count.cu).
int vin_capacity_dev(DeviceGraph *g, const uint32_t *deg_by_rank, cudaStream_t s);

#ifndef TC_HUB_LOG2
#define TC_HUB_LOG2 18
#endif
constexpr uint32_t kHubRanks = 1u << TC_HUB_LOG2;  // hub zone size: 32 KB shared-memory bitmap
constexpr uint32_t kDenseRanks = 1u << 17;  // dense-hub bitmaps: 1 GB at R-MAT s26

int graph_alloc(DeviceGraph *g, uint64_t m, uint64_t n, cudaStream_t s);
void graph_release(DeviceGraph *g, cudaStream_t s);
// node_offsets (and off32, max_out) from a grouped edge_src (reference preprocess.py:36-46).
int build_node_array_dev(const uint32_t *firsts, uint64_t k, uint64_t n, int64_t *off,
                         uint32_t *off32, uint32_t *max_out, cudaStream_t s);
// The scan half of it from per-vertex counts; `sums` holds ceil(n / kScanTile) u64.
int node_array_from_counts(const uint32_t *cnt, uint64_t n, uint64_t k, int64_t *off, uint32_t *off32,
                           uint32_t *max_out, unsigned long long *sums, cudaStream_t s);
// off[i] = sum of cnt[0..i) for i < n (exclusive scan, u32 -> i64).
int exclusive_scan_dev(const uint32_t *cnt, uint64_t n, int64_t *off, cudaStream_t s);
// Rebuild edge_src, off32 and max_out from node_offsets (after a broadcast of dst + off).
int finalize_graph_dev(DeviceGraph *g, cudaStream_t s);
// Full reference preprocess on device-resident pairs (reference preprocess.py:74-84).
int preprocess_dev(const uint32_t *pairs, uint64_t npairs, uint64_t n, DeviceGraph *out,
                   cudaStream_t s);
// The same pipeline producing the rank-space oriented CSR (+ hubstart) directly; with
// id_of_rank (u32[n], caller-allocated) also the inverse relabelling.
// pre: degrees (u32[n], zero-initialised then accumulated by degree_hist_dev over every
// chunk of the pairs, e.g. while they were copied in) and its invalid-id flag; the
// preprocess takes ownership of pre->deg (scratch pool, stream s).
struct PreDegrees {
    uint32_t *deg = nullptr, *bad = nullptr;
};
int preprocess_rank_dev(const uint32_t *pairs, uint64_t npairs, uint64_t n, DeviceGraph *out,
                        cudaStream_t s, uint32_t *id_of_rank = nullptr, const PreDegrees *pre = nullptr);
// First-column histogram of pairs (u32 pairs) into deg; *bad |= 1 on an id >= n.
int degree_hist_dev(const uint32_t *pairs, uint64_t npairs, uint64_t n, uint32_t *deg, uint32_t *bad,
                    cudaStream_t s);
// Reference-id CSR of a preprocess_rank_dev graph (exact inverse relabelling + sort).
int derank_dev(const DeviceGraph &r, const uint32_t *id_of_rank, DeviceGraph *out, cudaStream_t s);
// Distributed preprocessing steps (tc_preprocess.cu).
int dist_degrees_dev(const uint32_t *pairs, uint64_t npairs, uint64_t n, uint32_t *deg, cudaStream_t s);
int dist_orient_dev(const uint32_t *pairs, uint64_t npairs, uint64_t n, const uint32_t *deg,
                    uint64_t **keys_out, uint64_t *nkeys, uint32_t *outdeg, cudaStream_t s);
int dist_layout_dev(DeviceGraph *g, const uint32_t *outdeg, int parts, int64_t *cuts,
                    int64_t *ecuts, cudaStream_t s);
int dist_split_dev(const uint64_t *keys, uint64_t nkeys, uint64_t n, const int64_t *cuts, int parts,
                   int64_t *counts, cudaStream_t s);
int dist_place_dev(DeviceGraph *g, uint64_t *keys, uint64_t nkeys, uint64_t pos, cudaStream_t s);
// Rank-space copy of an oriented graph given in original ids (same triangles).  Returns
// kNotRankOrientable (nothing allocated in *out) when some edge does not point to a higher
// (out + in degree, id) rank -- a hand-built OrientedGraph or the preprocess of a
// non-symmetric edge array; such graphs are counted by the original-id kernels.
constexpr int kNotRankOrientable = 1;
int relabel_dev(const DeviceGraph &g, DeviceGraph *out, cudaStream_t s);
// hubstart[] and hz of a rank-space graph (after dst/off are in place).
int build_hubstart_dev(DeviceGraph *g, cudaStream_t s);
// Sort 2m pairs lexicographically (reference preprocess.py:23-33) into out_pairs.
int sort_pairs_dev(const uint32_t *pairs, uint64_t npairs, uint64_t n, uint32_t *out_pairs,
                   cudaStream_t s);
// Order-preserving orientation filter (reference preprocess.py:49-62).
int orient_compact_dev(const uint32_t *pairs, uint64_t npairs, const int64_t *deg, uint64_t n,
                       uint32_t *out_pairs, uint64_t *kept, cudaStream_t s);

// ---------------------------------------------------------------- counting ---
enum CountAlgo { kAlgoAuto = 0, kAlgoMergeThread = 1 };

struct CountStats {
    float classify_ms = 0, light_ms = 0, heavy_ms = 0, vmajor_ms = 0;
    uint64_t light_vertices = 0, heavy_tasks = 0;
};

// Triangles over oriented edges [lo, hi).  Result written to *d_total (device u64,
// accumulated, caller zeroes).  No host synchronisation inside.
int count_range_dev(const DeviceGraph &g, uint64_t lo, uint64_t hi, int algo,
                    unsigned long long *d_total, cudaStream_t s, CountStats *stats);
int intersect_dev(const DeviceGraph &g, uint32_t u, uint32_t v, uint64_t *out, cudaStream_t s);
// Estimated-work partition of [0, m) into npools ranges (bounds[npools+1], host out).
int work_bounds_dev(const DeviceGraph &g, int npools, int64_t *bounds, cudaStream_t s);
// Multi-GPU shard plan (tc_shard_plan): edge bounds balancing the non-v-major work and head
// bounds balancing the v-major work; count_shard_dev counts one shard of it.
int shard_plan_dev(const DeviceGraph &g, int parts, int64_t *ebounds, int64_t *hbounds, cudaStream_t s);
void shard_cost_sizes(const DeviceGraph &g, int parts, uint64_t *nt, uint64_t *tile, uint64_t *nz, uint32_t *z0);
int shard_costs_dev(const DeviceGraph &g, int parts, unsigned long long *edge_tiles, unsigned long long *head_costs,
                    cudaStream_t s);
int shard_stats_dev(const DeviceGraph &g, uint64_t lo, uint64_t hi, uint32_t hlo, uint32_t hhi, uint64_t out[9],
                    cudaStream_t s);
int count_shard_dev(const DeviceGraph &g, uint64_t lo, uint64_t hi, uint32_t hlo, uint32_t hhi,
                    unsigned long long *d_total, cudaStream_t s, CountStats *stats);
// Σ over edges of d+(u)+d+(v) (the merge-model work W), host out.
int merge_work_dev(const DeviceGraph &g, uint64_t *out, cudaStream_t s);
// Compulsory bytes of the full-count schedule of a rank-space graph, by kernel class
// (v-major, u-major heavy, light, per-edge, heavy staging); see tc_count.cu.
int schedule_bytes_dev(const DeviceGraph &g, uint64_t lo, uint64_t hi, uint64_t out[5], cudaStream_t s);

// ---------------------------------------------------------------- generators ---
int rmat_dev(int scale, int edge_factor, const double probs[4], const uint64_t state[2],
             const uint64_t inc[2], uint32_t **pairs_out, uint64_t *npairs_out,
             uint64_t *nverts_out, cudaStream_t s);
// 2-D random geometric graph: n points from PCG64 random((n, 2)); edge iff squared
// distance < radius^2 (IEEE double, no contraction).  Sorted pairs, both directions.
int rgg_dev(uint64_t n, double radius, const uint64_t state[2], const uint64_t inc[2],
            uint32_t **pairs_out, uint64_t *npairs_out, uint64_t *nverts_out, cudaStream_t s);
// ingest (tc_ingest.cu)
int validate_pairs_dev(const uint32_t *pairs, uint64_t np, uint64_t n, int *code, uint64_t *index,
                       cudaStream_t s);
int wedges_dev(const uint32_t *pairs, uint64_t np, uint64_t n, uint64_t *out, double *outd,
               cudaStream_t s);
int read_tri1(const char *path, uint32_t **pinned, uint64_t *npairs);
int parse_edge_list(const char *path, uint32_t **pinned, uint64_t *npairs, uint64_t *err_line,
                    int *err_kind);
int ba_dev(uint64_t n, uint32_t m_attach, const uint64_t state[2], const uint64_t inc[2],
           uint32_t **pairs_out, uint64_t *npairs_out, uint64_t *nverts_out, cudaStream_t s);

}  // namespace tc
