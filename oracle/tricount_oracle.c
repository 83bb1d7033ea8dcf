/*
 * tricount_oracle.c -- CPU restatement of the reference `tricount` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the sm_100a
 * product path in paper_1503_00576_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / `--impl reference` arm may load it.  The product
 * never links or calls it (there is no CPU fallback).
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/pkg/src/tricount):
 *
 *   or_sort_keys          preprocess.py:23-33 sort_edges + graph.py:84-98 pack_edge_keys
 *                         (np.sort of (u<<32)|v keys; here an LSD radix sort, same order)
 *   or_build_node_array   preprocess.py:36-46 build_node_array
 *                         (np.searchsorted(firsts, arange(n+1), side="left"))
 *   or_preprocess         preprocess.py:74-84 preprocess: sort -> node array -> degrees
 *                         (np.diff, preprocess.py:79-80) -> orient_and_compact
 *                         (preprocess.py:49-62) -> unzip (preprocess.py:65-71) -> node array
 *   or_count_strided      count.py:63-99 _count_strided (two-pointer merge, bounds
 *                         checked before every read)
 *   or_intersect_count    count.py:102-136 intersect_count
 *   or_count_triangles    count.py:162-178 count_triangles (W strided workers + sum)
 *   or_count_partitioned  count.py:181-204 count_partitioned (P pools x W workers)
 *   or_rmat_*             generators.py:203-284 rmat (PCG64 stream restated, see below)
 *   or_ba_pairs           generators.py:287-322 barabasi_albert (numpy integers() restated)
 *   or_rgg_*              random geometric graph (BASELINE config 5).  The reference has
 *                         NO generator for it; the definition is ours
 *                         (points = numpy random((n, 2)), edge iff squared distance <
 *                         r^2) and parity is pinned by counting its output with the
 *                         reference counter (tests/golden/make_golden.py --rgg).
 *
 * Parity of this restatement is pinned by tests/test_oracle.py against golden vectors
 * produced by the reference package itself (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

static int clamp_threads(int t) {
    if (t <= 0) t = omp_get_max_threads();
    return t < 1 ? 1 : t;
}

/* ---------------------------------------------------------------- sort ---- */

/* LSD radix sort of 64-bit keys over bits [0, key_bits), 8-bit digits.
 * Produces the same ascending order as np.sort (keys compare as integers). */
static void radix_sort_u64(uint64_t *keys, uint64_t *tmp, uint64_t k, int key_bits,
                           int threads) {
    if (k < 2) return;
    int nthr = clamp_threads(threads);
    size_t *hist = (size_t *)calloc((size_t)nthr * 256, sizeof(size_t));
    uint64_t *src = keys, *dst = tmp;
    int passes = (key_bits + 7) / 8;
    for (int p = 0; p < passes; ++p) {
        int shift = 8 * p;
        memset(hist, 0, (size_t)nthr * 256 * sizeof(size_t));
#pragma omp parallel num_threads(nthr)
        {
            int t = omp_get_thread_num();
            uint64_t lo = k * (uint64_t)t / nthr, hi = k * (uint64_t)(t + 1) / nthr;
            size_t *h = hist + (size_t)t * 256;
            for (uint64_t i = lo; i < hi; ++i) h[(src[i] >> shift) & 255]++;
#pragma omp barrier
#pragma omp single
            {
                size_t run = 0;
                for (int d = 0; d < 256; ++d)
                    for (int tt = 0; tt < nthr; ++tt) {
                        size_t c = hist[(size_t)tt * 256 + d];
                        hist[(size_t)tt * 256 + d] = run;
                        run += c;
                    }
            }
            for (uint64_t i = lo; i < hi; ++i) {
                uint64_t x = src[i];
                dst[h[(x >> shift) & 255]++] = x;
            }
        }
        uint64_t *s = src; src = dst; dst = s;
    }
    if (src != keys) memcpy(keys, src, k * sizeof(uint64_t));
    free(hist);
}

static int bits_for(uint64_t maxval) {
    int b = 0;
    while (b < 64 && (maxval >> b) != 0) ++b;
    return b;
}

/* preprocess.py:23-33 + graph.py:84-98: pack (first<<32)|second and sort. */
int or_sort_keys(const uint32_t *pairs, uint64_t npairs, uint64_t *keys_out, int threads) {
    int nthr = clamp_threads(threads);
    uint32_t maxfirst = 0;
#pragma omp parallel for num_threads(nthr) reduction(max : maxfirst)
    for (uint64_t i = 0; i < npairs; ++i) {
        keys_out[i] = ((uint64_t)pairs[2 * i] << 32) | pairs[2 * i + 1];
        if (pairs[2 * i] > maxfirst) maxfirst = pairs[2 * i];
    }
    uint64_t *tmp = (uint64_t *)malloc((npairs ? npairs : 1) * sizeof(uint64_t));
    if (!tmp) return -1;
    radix_sort_u64(keys_out, tmp, npairs, 32 + bits_for(maxfirst), nthr);
    free(tmp);
    return 0;
}

/* preprocess.py:36-46: offsets[i] = first index j with firsts[j] >= i, i in [0, n]. */
void or_build_node_array(const uint32_t *firsts, uint64_t k, uint64_t n, int64_t *offsets) {
    uint64_t j = 0;
    for (uint64_t i = 0; i <= n; ++i) {
        while (j < k && (uint64_t)firsts[j] < i) ++j;
        offsets[i] = (int64_t)j;
    }
}

/* Node array from sorted packed keys (first vertex in the high word): offs[i] = number of
 * keys whose first vertex is < i, built in parallel from run boundaries. */
static void node_array_from_keys(const uint64_t *keys, uint64_t k, uint64_t n, int64_t *offsets,
                                 int nthr) {
    if (k == 0) {
        for (uint64_t i = 0; i <= n; ++i) offsets[i] = 0;
        return;
    }
    /* vertices before the first key and after the last one */
#pragma omp parallel for num_threads(nthr)
    for (uint64_t i = 0; i <= (keys[0] >> 32); ++i) offsets[i] = 0;
#pragma omp parallel for num_threads(nthr)
    for (uint64_t i = (keys[k - 1] >> 32) + 1; i <= n; ++i) offsets[i] = (int64_t)k;
    /* a run boundary at j (first of j-1 < i <= first of j) sets offsets[i] = j */
#pragma omp parallel for num_threads(nthr) schedule(static)
    for (uint64_t j = 1; j < k; ++j) {
        uint64_t a = keys[j - 1] >> 32, b = keys[j] >> 32;
        for (uint64_t i = a + 1; i <= b; ++i) offsets[i] = (int64_t)j;
    }
}

/* preprocess.py:74-84.  Outputs must hold npairs entries (src/dst) and n+1 (off).
 * Returns the oriented edge count through m_out.  The reference runs this phase
 * single-threaded in numpy; the port uses all threads (order-preserving compaction by
 * per-thread counts + prefix, so the output is identical). */
int or_preprocess(const uint32_t *pairs, uint64_t npairs, uint64_t n, uint32_t *src,
                  uint32_t *dst, int64_t *off, uint64_t *m_out, int threads) {
    int nthr = clamp_threads(threads);
    if (npairs == 0) {
        for (uint64_t i = 0; i <= n; ++i) off[i] = 0;
        *m_out = 0;
        return 0;
    }
    uint64_t *keys = (uint64_t *)malloc(npairs * sizeof(uint64_t));
    int64_t *offs_all = (int64_t *)malloc((n + 1) * sizeof(int64_t));
    uint64_t *cnt = (uint64_t *)calloc((size_t)nthr + 1, sizeof(uint64_t));
    if (!keys || !offs_all || !cnt) { free(keys); free(offs_all); free(cnt); return -1; }
    if (or_sort_keys(pairs, npairs, keys, nthr) != 0) { free(keys); free(offs_all); free(cnt); return -1; }
    node_array_from_keys(keys, npairs, n, offs_all, nthr);
    /* degrees = np.diff(offsets_all); orient keeps (deg u, u) < (deg v, v) in sorted
     * order (preprocess.py:49-62), then unzip (preprocess.py:65-71). */
#pragma omp parallel num_threads(nthr)
    {
        int t = omp_get_thread_num();
        uint64_t lo = npairs * (uint64_t)t / nthr, hi = npairs * (uint64_t)(t + 1) / nthr, c = 0;
        for (uint64_t i = lo; i < hi; ++i) {
            uint32_t u = (uint32_t)(keys[i] >> 32), v = (uint32_t)keys[i];
            int64_t du = offs_all[u + 1] - offs_all[u];
            int64_t dv = (uint64_t)v < n ? offs_all[v + 1] - offs_all[v] : 0;
            c += (du < dv || (du == dv && u < v));
        }
        cnt[t + 1] = c;
#pragma omp barrier
#pragma omp single
        for (int q = 0; q < nthr; ++q) cnt[q + 1] += cnt[q];
        uint64_t o = cnt[t];
        for (uint64_t i = lo; i < hi; ++i) {
            uint32_t u = (uint32_t)(keys[i] >> 32), v = (uint32_t)keys[i];
            int64_t du = offs_all[u + 1] - offs_all[u];
            int64_t dv = (uint64_t)v < n ? offs_all[v + 1] - offs_all[v] : 0;
            if (du < dv || (du == dv && u < v)) {
                src[o] = u;
                dst[o] = v;
                ++o;
            }
        }
    }
    uint64_t m = cnt[nthr];
    /* node array over the compacted sources (packed as keys for the shared helper) */
#pragma omp parallel for num_threads(nthr)
    for (uint64_t i = 0; i < m; ++i) keys[i] = (uint64_t)src[i] << 32;
    node_array_from_keys(keys, m, n, off, nthr);
    *m_out = m;
    free(keys);
    free(offs_all);
    free(cnt);
    return 0;
}

/* --------------------------------------------------------------- count ---- */

/* count.py:63-99, statement for statement. */
uint64_t or_count_strided(const uint32_t *edge_src, const uint32_t *edge_dst,
                          const int64_t *node_offsets, int64_t lo, int64_t hi,
                          int64_t offset, int64_t stride) {
    uint64_t total = 0;
    for (int64_t i = lo + offset; i < hi; i += stride) {
        uint32_t u = edge_src[i], v = edge_dst[i];
        int64_t u_it = node_offsets[u], u_end = node_offsets[u + 1];
        int64_t v_it = node_offsets[v], v_end = node_offsets[v + 1];
        if (u_it == u_end || v_it == v_end) continue;
        uint32_t a = edge_dst[u_it], b = edge_dst[v_it];
        for (;;) {
            if (a < b) {
                if (++u_it == u_end) break;
                a = edge_dst[u_it];
            } else if (b < a) {
                if (++v_it == v_end) break;
                b = edge_dst[v_it];
            } else {
                ++total;
                ++u_it;
                ++v_it;
                if (u_it == u_end || v_it == v_end) break;
                a = edge_dst[u_it];
                b = edge_dst[v_it];
            }
        }
    }
    return total;
}

/* count.py:102-136. */
uint64_t or_intersect_count(const uint32_t *edge_dst, const int64_t *node_offsets,
                            uint32_t u, uint32_t v) {
    int64_t u_it = node_offsets[u], u_end = node_offsets[u + 1];
    int64_t v_it = node_offsets[v], v_end = node_offsets[v + 1];
    uint64_t c = 0;
    while (u_it < u_end && v_it < v_end) {
        uint32_t a = edge_dst[u_it], b = edge_dst[v_it];
        if (a < b) ++u_it;
        else if (b < a) ++v_it;
        else { ++c; ++u_it; ++v_it; }
    }
    return c;
}

/* count.py:181-204: P contiguous pools, each strided over W workers; sum. */
uint64_t or_count_partitioned(const uint32_t *edge_src, const uint32_t *edge_dst,
                              const int64_t *node_offsets, const int64_t *bounds, int npools,
                              int workers) {
    uint64_t total = 0;
    int tasks = npools * workers;
#pragma omp parallel for num_threads(clamp_threads(tasks)) schedule(dynamic, 1) reduction(+ : total)
    for (int t = 0; t < tasks; ++t) {
        int p = t / workers, w = t % workers;
        total += or_count_strided(edge_src, edge_dst, node_offsets, bounds[p], bounds[p + 1], w,
                                  workers);
    }
    return total;
}

/* count.py:162-178: W strided workers over [0, m). */
uint64_t or_count_triangles(const uint32_t *edge_src, const uint32_t *edge_dst,
                            const int64_t *node_offsets, int64_t m, int workers) {
    int64_t b[2] = {0, m};
    if (m == 0) return 0;
    return or_count_partitioned(edge_src, edge_dst, node_offsets, b, 1, workers);
}

/* Bounded sample for the CPU baseline: only edges i with i % stride == phase,
 * spread over `threads` threads (the reference's own strided assignment, count.py:69). */
uint64_t or_count_sampled(const uint32_t *edge_src, const uint32_t *edge_dst,
                          const int64_t *node_offsets, int64_t m, int64_t stride, int threads) {
    uint64_t total = 0;
    int nthr = clamp_threads(threads);
#pragma omp parallel for num_threads(nthr) schedule(dynamic, 1) reduction(+ : total)
    for (int t = 0; t < nthr; ++t)
        total += or_count_strided(edge_src, edge_dst, node_offsets, 0, m, (int64_t)t * stride,
                                  (int64_t)nthr * stride);
    return total;
}

/* Σ over oriented edges of d+(u)+d+(v): the merge-model work W. */
uint64_t or_merge_work(const uint32_t *edge_src, const uint32_t *edge_dst,
                       const int64_t *node_offsets, int64_t m) {
    uint64_t w = 0;
#pragma omp parallel for reduction(+ : w)
    for (int64_t i = 0; i < m; ++i) {
        uint32_t u = edge_src[i], v = edge_dst[i];
        w += (uint64_t)(node_offsets[u + 1] - node_offsets[u]) +
             (uint64_t)(node_offsets[v + 1] - node_offsets[v]);
    }
    return w;
}

/* ---------------------------------------------------------------- rmat ---- */
/*
 * generators.py:241-279 draws `scale` arrays of doubles per batch from numpy's
 * default_rng(seed) = PCG64 (XSL-RR 128/64; state = state*M + inc, then output),
 * random() = (next64 >> 11) * 2^-53.  numpy itself is not bundled with this oracle, so
 * the initial (state, inc) pair is passed in by the caller (numpy's SeedSequence
 * seeding, read from Generator.bit_generator.state).  or_rmat_levels fills src/dst
 * for one batch exactly as the reference's level loop does.
 */
typedef unsigned __int128 u128;
static const u128 PCG_MULT = (((u128)0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;

static inline uint64_t pcg_output(u128 s) {
    uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    unsigned rot = (unsigned)(s >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
}

/* state after `delta` steps: s*M^delta + inc*(M^delta-1)/(M-1), by squaring. */
static u128 pcg_advance(u128 s, u128 inc, uint64_t delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = PCG_MULT, cur_plus = inc;
    while (delta) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * s + acc_plus;
}

/* One batch of the reference level loop (generators.py:249-256).  The stream starts
 * at (state_hi, state_lo) advanced by `skip` draws.  Writes src/dst (< 2^scale). */
void or_rmat_levels(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                    uint64_t skip, uint64_t batch, int scale, double a, double t_ab,
                    double t_abc, int64_t *src, int64_t *dst, int threads) {
    u128 s0 = ((u128)state_hi << 64) | state_lo, inc = ((u128)inc_hi << 64) | inc_lo;
    memset(src, 0, batch * sizeof(int64_t));
    memset(dst, 0, batch * sizeof(int64_t));
    int nthr = clamp_threads(threads);
    for (int l = 0; l < scale; ++l) {
#pragma omp parallel num_threads(nthr)
        {
            int t = omp_get_thread_num();
            uint64_t lo = batch * (uint64_t)t / nthr, hi = batch * (uint64_t)(t + 1) / nthr;
            u128 s = pcg_advance(s0, inc, skip + (uint64_t)l * batch + lo);
            for (uint64_t j = lo; j < hi; ++j) {
                s = s * PCG_MULT + inc;
                double r = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
                int sb = r >= t_ab;
                int db = (r >= a && r < t_ab) || r >= t_abc;
                src[j] = (src[j] << 1) | sb;
                dst[j] = (dst[j] << 1) | db;
            }
        }
    }
}

/* ------------------------------------------------------------------ BA ---- */
/*
 * generators.py:287-322 barabasi_albert(n, m_attach, seed): preferential attachment from
 * K_{m_attach}.  Draws use numpy Generator.integers(0, len(repeated), size=k), i.e.
 * Lemire's bounded method on PCG64's buffered 32-bit outputs (low half of a 64-bit draw
 * first, the high half on the next call).  Writes the canonical (t, new) pairs in the
 * reference's append order; returns the pair count or -1 on allocation failure.
 */
typedef struct {
    u128 s, inc;
    int has;
    uint32_t buf;
} or_pcg;

static uint32_t or_next32(or_pcg *g) {
    if (g->has) { g->has = 0; return g->buf; }
    g->s = g->s * PCG_MULT + g->inc;
    uint64_t v = pcg_output(g->s);
    g->has = 1;
    g->buf = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

static uint32_t or_bounded(or_pcg *g, uint32_t high) {  /* integers(0, high), high >= 1 */
    uint32_t rng = high - 1;
    if (rng == 0) return 0;
    uint32_t excl = rng + 1;
    uint64_t m = (uint64_t)or_next32(g) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        uint32_t thr = (0xFFFFFFFFu - rng) % excl;
        while (left < thr) {
            m = (uint64_t)or_next32(g) * excl;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

int64_t or_ba_pairs(uint64_t n, uint32_t m_attach, uint64_t state_hi, uint64_t state_lo,
                    uint64_t inc_hi, uint64_t inc_lo, uint32_t *pairs_out) {
    or_pcg g = {((u128)state_hi << 64) | state_lo, ((u128)inc_hi << 64) | inc_lo, 0, 0};
    uint64_t np = 0;
    uint64_t cap_rep = 2 * ((uint64_t)m_attach * m_attach + (n - m_attach) * (uint64_t)m_attach) + 2;
    uint32_t *rep = (uint32_t *)malloc(cap_rep * sizeof(uint32_t));
    if (!rep) return -1;
    uint64_t nrep = 0;
    for (uint32_t i = 0; i < m_attach; ++i)
        for (uint32_t j = i + 1; j < m_attach; ++j) {
            pairs_out[2 * np] = i; pairs_out[2 * np + 1] = j; ++np;
            rep[nrep++] = i; rep[nrep++] = j;
        }
    uint32_t tg[64];
    for (uint64_t v = m_attach; v < n; ++v) {
        uint32_t nt = 0;
        if (nrep == 0) tg[nt++] = or_bounded(&g, (uint32_t)v);
        while (nt < m_attach) {
            uint32_t k = m_attach - nt, draws[64];
            for (uint32_t d = 0; d < k; ++d) draws[d] = or_bounded(&g, (uint32_t)nrep);
            for (uint32_t d = 0; d < k; ++d) {
                uint32_t t = rep[draws[d]], seen = 0;
                for (uint32_t q = 0; q < nt; ++q) seen |= tg[q] == t;
                if (!seen) tg[nt++] = t;
            }
        }
        for (uint32_t a = 1; a < nt; ++a)  /* sorted(targets) */
            for (uint32_t b = a; b > 0 && tg[b - 1] > tg[b]; --b) { uint32_t x = tg[b]; tg[b] = tg[b - 1]; tg[b - 1] = x; }
        for (uint32_t q = 0; q < nt; ++q) {
            pairs_out[2 * np] = tg[q]; pairs_out[2 * np + 1] = (uint32_t)v; ++np;
            rep[nrep++] = tg[q]; rep[nrep++] = (uint32_t)v;
        }
    }
    free(rep);
    return (int64_t)np;
}

/* ----------------------------------------------------------------- RGG ---- */
/* Points: numpy default_rng(seed).random((n, 2)) -> x_i = draw 2i, y_i = draw 2i+1. */
void or_rgg_points(uint64_t n, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                   uint64_t inc_lo, double *xs, double *ys, int threads) {
    u128 s0 = ((u128)state_hi << 64) | state_lo, inc = ((u128)inc_hi << 64) | inc_lo;
    int nthr = clamp_threads(threads);
#pragma omp parallel num_threads(nthr)
    {
        int t = omp_get_thread_num();
        uint64_t lo = n * (uint64_t)t / nthr, hi = n * (uint64_t)(t + 1) / nthr;
        u128 s = pcg_advance(s0, inc, 2 * lo);
        for (uint64_t i = lo; i < hi; ++i) {
            s = s * PCG_MULT + inc;
            xs[i] = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
            s = s * PCG_MULT + inc;
            ys[i] = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
        }
    }
}

typedef struct {
    uint32_t grid;
    uint32_t *start; /* [grid*grid + 1] */
    uint32_t *ids;   /* point ids bucketed by cell, ascending within a cell */
} or_cells;

static uint32_t rgg_cell(double v, uint32_t grid) {
    uint32_t c = (uint32_t)(v * grid);
    return c < grid ? c : grid - 1;
}

static int rgg_cells(const double *xs, const double *ys, uint64_t n, double r, or_cells *c) {
    double fg = (double)(int64_t)(1.0 / r) - 2.0;  /* cell side > r (a different grid from the GPU's) */
    c->grid = fg < 1 ? 1u : (fg > 65535 ? 65535u : (uint32_t)fg);
    uint64_t cells = (uint64_t)c->grid * c->grid;
    c->start = (uint32_t *)calloc(cells + 1, sizeof(uint32_t));
    c->ids = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
    if (!c->start || !c->ids) return -1;
    for (uint64_t i = 0; i < n; ++i)
        c->start[(uint64_t)rgg_cell(ys[i], c->grid) * c->grid + rgg_cell(xs[i], c->grid) + 1]++;
    for (uint64_t k = 0; k < cells; ++k) c->start[k + 1] += c->start[k];
    uint32_t *fill = (uint32_t *)malloc(cells * sizeof(uint32_t));
    if (!fill) return -1;
    memcpy(fill, c->start, cells * sizeof(uint32_t));
    for (uint64_t i = 0; i < n; ++i)
        c->ids[fill[(uint64_t)rgg_cell(ys[i], c->grid) * c->grid + rgg_cell(xs[i], c->grid)]++] = (uint32_t)i;
    free(fill);
    return 0;
}

static int cmp_u32(const void *a, const void *b) {
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return (x > y) - (x < y);
}

/* Neighbours of i (ascending) into out (may be NULL: count only). */
static uint32_t rgg_neighbours(const double *xs, const double *ys, const or_cells *c, double r2,
                               uint64_t i, uint32_t *out) {
    uint32_t g = c->grid, cx = rgg_cell(xs[i], g), cy = rgg_cell(ys[i], g), k = 0;
    uint32_t x0 = cx ? cx - 1 : 0, x1 = cx + 1 < g ? cx + 1 : g - 1;
    uint32_t y0 = cy ? cy - 1 : 0, y1 = cy + 1 < g ? cy + 1 : g - 1;
    for (uint32_t yy = y0; yy <= y1; ++yy)
        for (uint32_t q = c->start[(uint64_t)yy * g + x0]; q < c->start[(uint64_t)yy * g + x1 + 1]; ++q) {
            uint32_t j = c->ids[q];
            if (j == i) continue;
            volatile double dx = xs[i] - xs[j], dy = ys[i] - ys[j];
            volatile double dx2 = dx * dx, dy2 = dy * dy;
            if (dx2 + dy2 < r2) {
                if (out) out[k] = j;
                ++k;
            }
        }
    if (out) qsort(out, k, sizeof(uint32_t), cmp_u32);
    return k;
}

/* Pair count of the graph (both directions); deg[i] filled when non-NULL. */
int64_t or_rgg_count(const double *xs, const double *ys, uint64_t n, double r, uint32_t *deg,
                     int threads) {
    or_cells c;
    if (rgg_cells(xs, ys, n, r, &c)) return -1;
    double r2 = r * r;
    int64_t total = 0;
#pragma omp parallel for num_threads(clamp_threads(threads)) schedule(dynamic, 4096) reduction(+ : total)
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t k = rgg_neighbours(xs, ys, &c, r2, i, NULL);
        if (deg) deg[i] = k;
        total += k;
    }
    free(c.start);
    free(c.ids);
    return total;
}

/* All pairs (i, j), i ascending then j ascending; offsets[i] = first pair of i (n+1). */
int or_rgg_fill(const double *xs, const double *ys, uint64_t n, double r,
                const int64_t *offsets, uint32_t *pairs_out, int threads) {
    or_cells c;
    if (rgg_cells(xs, ys, n, r, &c)) return -1;
    double r2 = r * r;
    int bad = 0;
#pragma omp parallel num_threads(clamp_threads(threads))
    {
        uint32_t cap = 1024, *buf = (uint32_t *)malloc(cap * sizeof(uint32_t));
#pragma omp for schedule(dynamic, 4096)
        for (uint64_t i = 0; i < n; ++i) {
            uint64_t k = (uint64_t)(offsets[i + 1] - offsets[i]);
            if (k > cap) {
                cap = (uint32_t)k;
                buf = (uint32_t *)realloc(buf, cap * sizeof(uint32_t));
            }
            if (rgg_neighbours(xs, ys, &c, r2, i, buf) != k) bad = 1;
            for (uint64_t q = 0; q < k; ++q) {
                pairs_out[2 * (offsets[i] + q)] = (uint32_t)i;
                pairs_out[2 * (offsets[i] + q) + 1] = buf[q];
            }
        }
        free(buf);
    }
    free(c.start);
    free(c.ids);
    return bad ? -1 : 0;
}

/* ------------------------------------------------------ rmat, whole loop ---- */
/*
 * generators.py:241-284 in one call (the numpy version of the dedupe loop needs ~100 GB
 * and tens of minutes at scale 26; this one sorts in parallel).  Per round, exactly as the
 * reference: batch = max(4096, int(need * 1.3)) draws per level; keep src != dst; keys =
 * (min << 32) | max in draw order; order-preserving de-dup (first occurrence wins); drop
 * keys already in `have`; the first `need` survivors in draw order join `have`.  Because
 * `have` is re-sorted every round, the survivors are collected in key order from a STABLE
 * key sort of (key, draw position): the first element of each equal-key run is the first
 * occurrence, and "the first `need` survivors in draw order" = the survivors whose draw
 * position is <= the position of the need-th survivor.
 * Writes the sorted canonical keys to have (target entries).  Returns 0, -1 (allocation)
 * or -2 (sampling saturated: 25 rounds without a new edge, generators.py:268-274).
 */
static void radix_sort_kv(uint64_t *k, uint64_t *kt, uint32_t *v, uint32_t *vt, uint64_t n,
                          int key_bits, int nthr, uint64_t **ko, uint32_t **vo) {
    size_t *hist = (size_t *)calloc((size_t)nthr * 256, sizeof(size_t));
    uint64_t *sk = k, *dk = kt;
    uint32_t *sv = v, *dv = vt;
    int passes = (key_bits + 7) / 8;
    for (int p = 0; p < passes; ++p) {
        int shift = 8 * p;
        memset(hist, 0, (size_t)nthr * 256 * sizeof(size_t));
#pragma omp parallel num_threads(nthr)
        {
            int t = omp_get_thread_num();
            uint64_t lo = n * (uint64_t)t / nthr, hi = n * (uint64_t)(t + 1) / nthr;
            size_t *h = hist + (size_t)t * 256;
            for (uint64_t i = lo; i < hi; ++i) h[(sk[i] >> shift) & 255]++;
#pragma omp barrier
#pragma omp single
            {
                size_t run = 0;
                for (int d = 0; d < 256; ++d)
                    for (int tt = 0; tt < nthr; ++tt) {
                        size_t c = hist[(size_t)tt * 256 + d];
                        hist[(size_t)tt * 256 + d] = run;
                        run += c;
                    }
            }
            for (uint64_t i = lo; i < hi; ++i) {
                size_t o = h[(sk[i] >> shift) & 255]++;
                dk[o] = sk[i];
                dv[o] = sv[i];
            }
        }
        uint64_t *a = sk; sk = dk; dk = a;
        uint32_t *b = sv; sv = dv; dv = b;
    }
    free(hist);
    *ko = sk;
    *vo = sv;
}

int or_rmat_canonical(int scale, uint64_t target, double a, double t_ab, double t_abc,
                      uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                      uint64_t *have, int threads) {
    const int nthr = clamp_threads(threads);
    const u128 s0 = ((u128)state_hi << 64) | state_lo, inc = ((u128)inc_hi << 64) | inc_lo;
    uint64_t have_n = 0, drawn = 0;
    int stalled = 0;
    uint64_t *cnt = (uint64_t *)calloc((size_t)nthr + 1, sizeof(uint64_t));
    if (!cnt) return -1;
    while (have_n < target) {
        const uint64_t need = target - have_n;
        uint64_t batch = (uint64_t)((double)need * 1.3);
        if (batch < 4096) batch = 4096;
        uint32_t *sd = (uint32_t *)malloc(batch * 2 * sizeof(uint32_t));
        uint64_t *keys = (uint64_t *)malloc(batch * sizeof(uint64_t));
        uint32_t *pos = (uint32_t *)malloc(batch * sizeof(uint32_t));
        if (!sd || !keys || !pos) { free(sd); free(keys); free(pos); free(cnt); return -1; }
        /* level loop (generators.py:249-256): level l of item j is draw drawn + l*batch + j */
#pragma omp parallel num_threads(nthr)
        {
            int t = omp_get_thread_num();
            uint64_t lo = batch * (uint64_t)t / nthr, hi = batch * (uint64_t)(t + 1) / nthr;
            for (uint64_t j = lo; j < hi; ++j) sd[2 * j] = sd[2 * j + 1] = 0;
            for (int l = 0; l < scale; ++l) {
                u128 s = pcg_advance(s0, inc, drawn + (uint64_t)l * batch + lo);
                for (uint64_t j = lo; j < hi; ++j) {
                    s = s * PCG_MULT + inc;
                    double r = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
                    uint32_t sb = r >= t_ab;
                    uint32_t db = (r >= a && r < t_ab) || r >= t_abc;
                    sd[2 * j] = (sd[2 * j] << 1) | sb;
                    sd[2 * j + 1] = (sd[2 * j + 1] << 1) | db;
                }
            }
            /* keep = src != dst, order-preserving (per-thread count + prefix) */
            uint64_t c = 0;
            for (uint64_t j = lo; j < hi; ++j) c += sd[2 * j] != sd[2 * j + 1];
            cnt[t + 1] = c;
#pragma omp barrier
#pragma omp single
            {
                cnt[0] = 0;
                for (int q = 0; q < nthr; ++q) cnt[q + 1] += cnt[q];
            }
            uint64_t o = cnt[t];
            for (uint64_t j = lo; j < hi; ++j) {
                uint32_t x = sd[2 * j], y = sd[2 * j + 1];
                if (x == y) continue;
                uint32_t mn = x < y ? x : y, mx = x < y ? y : x;
                keys[o] = ((uint64_t)mn << 32) | mx;
                pos[o] = (uint32_t)o;
                ++o;
            }
        }
        drawn += batch * (uint64_t)scale;
        const uint64_t nk = cnt[nthr];
        /* reuse sd as the ping-pong buffers: it holds 8*batch bytes = keys' size; pos needs
         * its own (4*batch) */
        uint64_t *kt = (uint64_t *)sd;
        uint32_t *pt = (uint32_t *)malloc((nk ? nk : 1) * sizeof(uint32_t));
        if (!pt) { free(sd); free(keys); free(pos); free(cnt); return -1; }
        uint64_t *sk;
        uint32_t *sp;
        /* key bits: min/max ids < 2^scale in the two 32-bit halves */
        radix_sort_kv(keys, kt, pos, pt, nk, 32 + scale, nthr, &sk, &sp);
        /* survivors: first of an equal-key run and absent from `have` (merge join) */
        uint8_t *flag = (uint8_t *)calloc(nk ? nk : 1, 1);
        if (!flag) { free(sd); free(keys); free(pos); free(pt); free(cnt); return -1; }
#pragma omp parallel num_threads(nthr)
        {
            int t = omp_get_thread_num();
            uint64_t lo = nk * (uint64_t)t / nthr, hi = nk * (uint64_t)(t + 1) / nthr;
            if (lo < hi) {
                /* first have entry >= sk[lo] */
                uint64_t L = 0, R = have_n;
                while (L < R) {
                    uint64_t mid = (L + R) / 2;
                    if (have[mid] < sk[lo]) L = mid + 1; else R = mid;
                }
                uint64_t h = L;
                for (uint64_t i = lo; i < hi; ++i) {
                    if (i > 0 && sk[i - 1] == sk[i]) continue;  /* not the first occurrence */
                    while (h < have_n && have[h] < sk[i]) ++h;
                    if (h < have_n && have[h] == sk[i]) continue;
                    flag[sp[i]] = 1;
                }
            }
        }
        /* draw position of the need-th survivor (or keep all) */
        uint64_t cut = nk;  /* positions < cut are taken */
        {
            uint64_t *sc = (uint64_t *)calloc((size_t)nthr + 1, sizeof(uint64_t));
#pragma omp parallel num_threads(nthr)
            {
                int t = omp_get_thread_num();
                uint64_t lo = nk * (uint64_t)t / nthr, hi = nk * (uint64_t)(t + 1) / nthr, c = 0;
                for (uint64_t i = lo; i < hi; ++i) c += flag[i];
                sc[t + 1] = c;
            }
            uint64_t run = 0;
            for (int q = 0; q < nthr && cut == nk; ++q) {
                uint64_t lo = nk * (uint64_t)q / nthr, hi = nk * (uint64_t)(q + 1) / nthr;
                if (run + sc[q + 1] >= need) {
                    for (uint64_t i = lo; i < hi; ++i)
                        if (flag[i] && ++run == need) { cut = i + 1; break; }
                } else {
                    run += sc[q + 1];
                }
            }
            free(sc);
        }
        /* the taken survivors in key order: compact sk (in place; sequential, ~1 ns each) */
        uint64_t nnew = 0;
        for (uint64_t i = 0; i < nk; ++i)
            if (sp[i] < cut && flag[sp[i]]) sk[nnew++] = sk[i];
        free(flag);
        if (nnew == 0) {
            if (++stalled >= 25) { free(sd); free(keys); free(pos); free(pt); free(cnt); return -2; }
        } else {
            stalled = 0;
            /* have = sort(have ∪ new): backward merge in place */
            uint64_t i = have_n, j = nnew, o = have_n + nnew;
            while (j > 0) {
                if (i > 0 && have[i - 1] > sk[j - 1]) have[--o] = have[--i];
                else have[--o] = sk[--j];
            }
            have_n += nnew;
        }
        free(sd);
        free(keys);
        free(pos);
        free(pt);
    }
    free(cnt);
    return 0;
}

/* graph.py:265-276 edge_array_from_undirected on sorted canonical keys (lo < hi): both
 * directions, lexicographically sorted, as u32 pairs [2k][2]. */
int or_symmetrize_canonical(const uint64_t *keys, uint64_t k, uint32_t *pairs, int threads) {
    const int nthr = clamp_threads(threads);
    uint64_t *rev = (uint64_t *)malloc((k ? k : 1) * sizeof(uint64_t));
    uint64_t *tmp = (uint64_t *)malloc((k ? k : 1) * sizeof(uint64_t));
    if (!rev || !tmp) { free(rev); free(tmp); return -1; }
    uint64_t mx = 0;
#pragma omp parallel for num_threads(nthr) reduction(max : mx)
    for (uint64_t i = 0; i < k; ++i) {
        rev[i] = (keys[i] << 32) | (keys[i] >> 32);
        if ((keys[i] & 0xffffffffu) > mx) mx = keys[i] & 0xffffffffu;
    }
    radix_sort_u64(rev, tmp, k, 32 + bits_for(mx), nthr);
    free(tmp);
    /* merge the two sorted lists (keys are distinct across them: lo<hi vs hi>lo) */
    uint64_t i = 0, j = 0, o = 0;
    while (i < k || j < k) {
        uint64_t x;
        if (j >= k || (i < k && keys[i] < rev[j])) x = keys[i++];
        else x = rev[j++];
        pairs[2 * o] = (uint32_t)(x >> 32);
        pairs[2 * o + 1] = (uint32_t)x;
        ++o;
    }
    free(rev);
    return 0;
}
