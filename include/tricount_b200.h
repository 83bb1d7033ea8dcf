/*
 * tricount_b200.h -- C ABI of the B200 (sm_100a) exact triangle counter.
 *
 * Drop-in boundary for the reference `tricount` hot path (reference files under
 * /root/reference/pkg/src/tricount).  The reference exposes a Python function API over
 * numpy arrays (no FFI); each entry point below replaces one of those functions and is
 * bound from Python with ctypes.  All functions return 0 on
 * success and a negative status on failure (-1 argument/contract error, -2 CUDA error,
 * -3 out of memory); tc_last_error() returns the thread-local message.  Host buffers are
 * borrowed for the duration of the call; device graphs are owned by the library until
 * tc_graph_free().  Every call is synchronous with respect to its results.
 *
 * Threading: every entry point may be called from any thread, concurrently on different
 * graphs (reference SPEC.md:294).  Calls that touch the device are serialised by one
 * library lock (each already saturates the GPU) and every count accumulates into its own
 * device counter.
 *
 * Arrays: pairs are uint32 (u, v) pairs, row-major [npairs][2] (reference EdgeArray.edges,
 * graph.py:101-129); an oriented graph is edge_src u32[m], edge_dst u32[m],
 * node_offsets i64[n+1] (reference OrientedGraph, graph.py:146-193).
 */
#ifndef TRICOUNT_B200_H
#define TRICOUNT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TC_ABI_VERSION 3  /* 2: tc_times gained vmajor_ms; 3: tc_set_option, thread-safe calls */

typedef struct tc_graph tc_graph; /* device-resident OrientedGraph */

/* Phase timings in milliseconds, measured with CUDA events on the library stream. */
typedef struct tc_times {
    double h2d_ms;        /* host->device copy of the input pairs               */
    double preprocess_ms; /* preprocessing kernels (degree .. node array)        */
    double count_ms;      /* counting kernels + 8-byte result copy               */
    double total_ms;      /* whole call                                          */
    double classify_ms;   /* count detail: source classification                 */
    double heavy_ms;      /* count detail: u-major heavy-source kernels          */
    double light_ms;      /* count detail: light-source kernel                   */
    uint64_t heavy_tasks; /* count detail: CTA tasks issued                      */
    double vmajor_ms;     /* count detail: v-major hub-head kernel (in classify) */
} tc_times;

/* count algorithm selector */
#define TC_ALGO_AUTO 0         /* light/heavy source-centric kernels (default)        */
#define TC_ALGO_MERGE_THREAD 1 /* paper's thread-per-edge merge (A/B baseline)        */

/* ---- lifecycle: replaces count.py:143-150 warm_kernel (JIT warm-up -> CUDA init) ---- */
int tc_init(int device);
int tc_shutdown(void);
const char *tc_last_error(void);
int tc_abi_version(void);

/* ---- preprocess.py:74-84 preprocess(g) -> OrientedGraph ----------------------------
 * pairs: host (pairs_on_device = 0) or device pointer; nverts = EdgeArray.num_vertices. */
int tc_preprocess(const uint32_t *pairs, uint64_t npairs, uint64_t nverts, int pairs_on_device,
                  tc_graph **out, tc_times *t);
/* flags: TC_PREPROCESS_RANK_SPACE builds the count-ready rank-space CSR instead (vertices
 * relabelled by (degree, id) rank -- same orientation, same triangles, different ids);
 * count_with_timings uses it internally.  Downloads of such a graph are in rank ids. */
#define TC_PREPROCESS_RANK_SPACE 1
int tc_preprocess_ex(const uint32_t *pairs, uint64_t npairs, uint64_t nverts, int pairs_on_device,
                     int flags, tc_graph **out, tc_times *t);

/* ---- OrientedGraph transfer (graph.py:146-193) -------------------------------------- */
int tc_graph_upload(const uint32_t *edge_src, const uint32_t *edge_dst,
                    const int64_t *node_offsets, uint64_t m, uint64_t n, tc_graph **out);
/* Replication (multi-GPU): allocate an empty device graph, fill edge_dst and node_offsets
 * through tc_graph_device_ptrs (e.g. an NCCL broadcast), then tc_graph_finalize rebuilds
 * edge_src, the u32 offsets and the max out-degree on the device. */
int tc_graph_create(uint64_t m, uint64_t n, int flags, tc_graph **out);
int tc_graph_finalize(tc_graph *g);
int tc_graph_download(const tc_graph *g, uint32_t *edge_src, uint32_t *edge_dst,
                      int64_t *node_offsets);
int tc_graph_info(const tc_graph *g, uint64_t *m, uint64_t *n, uint32_t *max_out_degree);
int tc_graph_flags(const tc_graph *g, int *flags);
int tc_graph_device_ptrs(const tc_graph *g, uint32_t **edge_src, uint32_t **edge_dst,
                         int64_t **node_offsets);
int tc_graph_free(tc_graph *g);

/* ---- count.py:162-178 count_triangles / count.py:63-99 _count_strided over [lo, hi) --- */
int tc_count(const tc_graph *g, int64_t lo, int64_t hi, int algo, uint64_t *out, tc_times *t);
/* ---- count.py:181-204 count_partitioned: bounds[npools+1] must cover [0, m) ---------- */
int tc_count_partitioned(const tc_graph *g, const int64_t *bounds, int npools, int algo,
                         uint64_t *out, tc_times *t);
/* ---- count.py:102-136 intersect_count ------------------------------------------------ */
int tc_intersect_count(const tc_graph *g, uint32_t u, uint32_t v, uint64_t *out);
/* ---- count.py:207-229 count_with_timings: preprocess + count, phase timings ---------- */
int tc_count_with_timings(const uint32_t *pairs, uint64_t npairs, uint64_t nverts,
                          int pairs_on_device, int algo, uint64_t *out, tc_times *t);

/* ---- multi-GPU sharding: estimated-work bounds[npools+1] ---------- */
int tc_work_bounds(const tc_graph *g, int npools, int64_t *bounds);
/* Multi-GPU shard plan of a full count (rank-space copy of g): shard r
 * counts the edges [edge_bounds[r], edge_bounds[r+1]) that are not v-major plus the v-major
 * edges of the whole graph whose head lies in [head_bounds[r], head_bounds[r+1]).  Edge
 * bounds balance the u-major + light bytes, head bounds the v-major bytes, so every shard
 * gets 1/parts of both, and each head's bitmap is built by one shard only.  Both arrays
 * hold parts + 1 entries; the shard counts sum to the full count. */
int tc_shard_plan(const tc_graph *g, int parts, int64_t *edge_bounds, int64_t *head_bounds);
/* The plan's model costs, for measurement-guided refinement (distributed.ShardPlanner):
 * per-tile edge-side costs (ntiles tiles of `tile` edges) and per-head head-side costs
 * (nheads heads from head0), in the plan's time units. */
int tc_shard_cost_sizes(const tc_graph *g, int parts, uint64_t *ntiles, uint64_t *tile, uint64_t *nheads,
                        uint32_t *head0);
int tc_shard_costs(const tc_graph *g, int parts, uint64_t *edge_tiles, uint64_t *head_costs);
/* Cost features of one shard (calibration of the plan's weights; see csrc/tc_count.cu). */
int tc_shard_stats(const tc_graph *g, int64_t lo, int64_t hi, int64_t head_lo, int64_t head_hi,
                   uint64_t out[9]);
int tc_count_shard(const tc_graph *g, int64_t lo, int64_t hi, int64_t head_lo, int64_t head_hi,
                   uint64_t *out, tc_times *t);
/* merge-model work W = sum over oriented edges of d+(u) + d+(v) (roofline numerator) */
int tc_merge_work(const tc_graph *g, uint64_t *out);

/* ---- preprocess.py sub-steps (host buffers in and out) ------------------------------- */
/* preprocess.py:23-33 sort_edges: lexicographic (first, second) order */
int tc_sort_edges(const uint32_t *pairs, uint64_t npairs, uint64_t nverts, uint32_t *out_pairs);
/* preprocess.py:36-46 build_node_array from a grouped first column */
int tc_build_node_array(const uint32_t *firsts, uint64_t k, uint64_t n, int64_t *offsets);
/* preprocess.py:49-62 orient_and_compact (order preserving); degrees i64[n] */
int tc_orient_and_compact(const uint32_t *pairs, uint64_t npairs, const int64_t *degrees,
                          uint64_t n, uint32_t *out_pairs, uint64_t *kept);

/* ---- generators.py:203-284 rmat on the device (input production, bit-identical) ------ *
 * state/inc: numpy default_rng(seed).bit_generator.state (hi, lo words).  Returns a
 * device buffer of npairs (u, v) pairs (free with tc_device_free) and num_vertices.    */
int tc_gen_rmat(int scale, int edge_factor, const double probs[4], const uint64_t state[2],
                const uint64_t inc[2], uint32_t **dev_pairs, uint64_t *npairs, uint64_t *nverts);

/* ---- generators.py:287-322 barabasi_albert (bit-identical; host sampling loop, device
 * symmetrisation).  Device pairs (free with tc_device_free) and num_vertices.          */
int tc_gen_ba(uint64_t n, uint32_t m_attach, const uint64_t state[2], const uint64_t inc[2],
              uint32_t **dev_pairs, uint64_t *npairs, uint64_t *nverts);

/* ---- distributed preprocessing -----------------
 * One process per GPU, each holding a shard of the edge array.  The caller moves data
 * between the steps with its collectives (torch.distributed / NCCL):
 *   1. tc_dist_degrees: deg_dev[n] = first-column histogram of the shard  -> all-reduce SUM
 *   2. tc_dist_orient: ranks from the global degrees, the shard's kept pairs as sorted
 *      rank-space keys (*keys_dev, free with tc_device_free) + outdeg_dev[n] by source rank
 *                                                                        -> all-reduce SUM
 *   3. tc_graph_create(m, n, TC_PREPROCESS_RANK_SPACE) + tc_dist_layout: node_offsets
 *      from the global out-degrees; cuts[parts+1] = source-rank boundaries balanced by
 *      edges, edge_cuts[parts+1] = their edge positions
 *   4. tc_dist_split: counts[parts] of the shard's keys per destination range -> all-to-all
 *   5. tc_dist_place: sort the received keys (in place) into edge_dst[edge_pos ...]
 *                                                     -> all-gather the edge_dst slices
 *   6. tc_graph_finalize.                                                                  */
int tc_dist_degrees(const uint32_t *pairs, uint64_t npairs, int pairs_on_device, uint64_t nverts,
                    uint32_t *deg_dev);
int tc_dist_orient(const uint32_t *pairs, uint64_t npairs, int pairs_on_device, uint64_t nverts,
                   const uint32_t *deg_dev, uint64_t **keys_dev, uint64_t *nkeys, uint32_t *outdeg_dev);
int tc_dist_layout(tc_graph *g, const uint32_t *outdeg_dev, int parts, int64_t *cuts,
                   int64_t *edge_cuts);
int tc_dist_split(const uint64_t *keys_dev, uint64_t nkeys, uint64_t nverts, const int64_t *cuts,
                  int parts, int64_t *counts);
int tc_dist_place(tc_graph *g, uint64_t *keys_dev, uint64_t nkeys, uint64_t edge_pos);

/* ---- random geometric graph, BASELINE config 5 (the reference has no generator, SURVEY.md
 * §8(c)): points = numpy default_rng(seed).random((n, 2)) (x = draw 2i, y = draw 2i+1);
 * edge {i, j} iff (xi-xj)^2 + (yi-yj)^2 < radius^2 in IEEE double (no FMA contraction).
 * Sorted pairs, both directions (as edge_array_from_undirected); num_vertices = 1 + the
 * largest id with an edge.                                                              */
int tc_gen_rgg(uint64_t n, double radius, const uint64_t state[2], const uint64_t inc[2],
               uint32_t **dev_pairs, uint64_t *npairs, uint64_t *nverts);

/* ---- ingest ----------------------------------------------------- */
/* io.py:127-152 read_binary: TRI1 file -> pinned host pairs (free with tc_host_free).
 * Status -4 I/O error, -5 truncated (TruncatedFileError), -6 bad magic (BadMagicError). */
int tc_read_tri1(const char *path, uint32_t **host_pairs, uint64_t *npairs);
/* io.py:51-99 read_edge_list's parser (multi-threaded): text "u v" lines -> pinned host
 * pairs in file order (free with tc_host_free).  Status -7 = parse error: *err_line is the
 * 1-based line, *err_kind 1 wrong field count, 2 not an integer pair, 3 id out of u32
 * range (ParseError).  Mode handling (strict/symmetrize/normalize) is the caller's. */
int tc_parse_edge_list(const char *path, uint32_t **host_pairs, uint64_t *npairs,
                       uint64_t *err_line, int *err_kind);
/* graph.py:196-242 validate_edge_array on the device.  *code: 0 valid, 1 self-loop,
 * 2 duplicate, 3 missing reverse, 4 vertex id >= nverts; *index: the offending input index
 * the reference reports (first self-loop / earliest second occurrence / first pair
 * without reverse / first out-of-range pair). */
int tc_validate_edge_array(const uint32_t *pairs, uint64_t npairs, uint64_t nverts,
                           int pairs_on_device, int *code, uint64_t *index);
/* metrics.py:17-24 wedge_count: sum_v C(deg v, 2) (exact u64; approx = same in double,
 * for the reference's 64-bit overflow check). */
int tc_wedge_count(const uint32_t *pairs, uint64_t npairs, uint64_t nverts, int pairs_on_device,
                   uint64_t *out, double *approx);

/* ---- memory helpers (bench / host integration) --------------------------------------- */
int tc_device_alloc(uint64_t bytes, void **p);
int tc_device_free(void *p);
int tc_memcpy(void *dst, const void *src, uint64_t bytes, int kind); /* 0 h2d, 1 d2h, 2 d2d */
int tc_host_alloc(uint64_t bytes, void **p); /* pinned */
int tc_host_free(void *p);
int tc_host_register(void *p, uint64_t bytes);
int tc_host_unregister(void *p);
int tc_synchronize(void);
int tc_l2_flush(void); /* write a buffer larger than L2 (timing hygiene) */
/* CUDA events on the library stream (8 slots) and the number of kernels launched */
int tc_timer_record(int slot);
int tc_timer_elapsed(int slot_a, int slot_b, double *ms);
int tc_launch_count(uint64_t *out);
/* keep >= bytes reserved in the library's device memory pool (called automatically by
 * tc_preprocess* / tc_count_with_timings with an estimate of their scratch) */
int tc_reserve(uint64_t bytes);

/* Schedule options (no reference counterpart; the reference's numba kernel has none).  The
 * defaults are the measured-best schedule and are what every product call runs; the count is
 * exact under every setting.  Only the schedule-coverage tests and the development probes set
 * them -- the library never reads the environment.  Names: vmajor, vzone_log2, vlow_all,
 * vm_bias, dense_factor, hub_unroll, l2_persist_mb, l2_target, concurrent, share, midwarp,
 * light, skew, light_vec, shard_model, shard_ovh, shard_ucap, dense_ranks, bucket,
 * count_stats, hubpack, rank_primary, seg_fork, vin_overlap, vin_grid, seg_k16, seg_w2k,
 * vhub, vhub_unroll, vhub_blocks, vhub_b16w, hub_cap_div, vix, shard_w_* (see
 * csrc/tc_internal.h Options).  Unknown names return -1. */
/* Compulsory HBM bytes of the full-count schedule (rank-space copy of g): out[0] v-major
 * suffix streams + index entries, [1] u-major heavy-source reads of heads, [2] light-source
 * reads, [3] 16 B per edge (src, dst, two offsets), [4] heavy-source staging.  The roofline
 * numerator of bench.py; no reference counterpart. */
int tc_schedule_bytes(const tc_graph *g, uint64_t out[5]);
/* The same over oriented edges [lo, hi) of a rank-space graph (shard cost calibration). */
int tc_schedule_bytes_range(const tc_graph *g, int64_t lo, int64_t hi, uint64_t out[5]);

int tc_set_option(const char *name, int64_t value);
int tc_get_option(const char *name, int64_t *value);
int tc_reset_options(void);

#ifdef __cplusplus
}
#endif
#endif /* TRICOUNT_B200_H */
