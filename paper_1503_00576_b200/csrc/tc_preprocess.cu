// tc_preprocess.cu -- the reference preprocessing pipeline (reference preprocess.py:74-84)
// as sm_100a kernels.  The reference sorts all 2m pairs, derives degrees from the node
// array, orients, unzips and rebuilds the node array.  Here the order is
//   degree histogram -> orient + compact (fused digit histograms) -> LSD radix sort of
//   the m oriented keys (last pass writes SoA edge_src/edge_dst) -> node array,
// which yields the bit-identical OrientedGraph: orientation is a per-pair predicate, so
// filtering before sorting selects the same set, and sorting the survivors gives the
// order the reference's order-preserving compaction of a sorted list gives.
#include <stdlib.h>

#include "tc_common.cuh"
#include "tc_internal.h"
#include "tc_vsplit.cuh"

namespace tc {

int dalloc(void **p, size_t bytes, cudaStream_t s, bool persistent) {
    *p = nullptr;
    if (bytes == 0) bytes = 16;
    cudaMemPool_t pool = persistent ? nullptr : scratch_pool();
    cudaError_t e = pool ? cudaMallocFromPoolAsync(p, bytes, pool, s) : cudaMallocAsync(p, bytes, s);
    if (e != cudaSuccess) {
        set_error(std::string("device allocation of ") + std::to_string(bytes) +
                  " bytes failed: " + cudaGetErrorString(e));
        return -3;
    }
    return 0;
}

void dfree(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

namespace {

constexpr int kPP = 8;  // pairs per thread per iteration (warp-striped)

// deg[u] += 1 for every pair (u, .): reference degrees = np.diff(node array of the sorted
// pairs) (preprocess.py:79-80), i.e. the first-column histogram (graph.py:279-281).
// Runs of equal u inside a warp (the common, sorted-input case) become one atomic.
#ifndef TC_DEG_PP
#define TC_DEG_PP 8  // 4 / 8 / 16 pairs per lane: 4.9 / 4.7 / 4.9 ms at s26
#endif
constexpr int kDegPP = TC_DEG_PP;  // pairs per lane per iteration of the degree histogram

__global__ void __launch_bounds__(256) k_degree_hist(const uint2 *__restrict__ pairs,
                                                     uint64_t npairs, uint32_t *__restrict__ deg,
                                                     uint64_t n, unsigned *__restrict__ bad) {
    constexpr int kPP = kDegPP;
    const unsigned lane = lane_id();
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = gw * 32 * kPP; base < npairs; base += nw * 32 * kPP) {
        uint2 p[kPP];
#pragma unroll
        for (int i = 0; i < kPP; ++i) {
            uint64_t idx = base + i * 32 + lane;
            p[i] = idx < npairs ? ld_stream_u2(pairs + idx) : make_uint2(0, 0);
        }
#pragma unroll
        for (int i = 0; i < kPP; ++i) {
            uint64_t idx = base + i * 32 + lane;
            bool ok = idx < npairs;
            uint32_t u = p[i].x;
            uint32_t prev = __shfl_up_sync(TC_FULL_MASK, u, 1);
            bool prev_ok = lane > 0 && (idx - 1) < npairs;
            bool head = !ok || lane == 0 || !prev_ok || prev != u;
            unsigned heads = __ballot_sync(TC_FULL_MASK, head);
            if (ok && head) {
                unsigned above = heads & ~((2u << lane) - 1u);
                if (lane == 31) above = 0;
                unsigned next = above ? (unsigned)(__ffs(above) - 1) : 32u;
                if ((uint64_t)u >= n || (uint64_t)p[i].y >= n) atomicOr(bad, 1u);
                else atomicAdd(deg + u, next - lane);
            } else if (ok && (uint64_t)p[i].y >= n) {
                atomicOr(bad, 1u);
            }
        }
    }
}

// Keep (u, v) iff (deg u, u) < (deg v, v) (reference preprocess.py:49-62); write the
// packed key (u << vb) | v for the radix sort, and fold every kept key into the
// per-pass digit histograms (saves a separate histogram read of the keys).
// One atomicAdd on the output cursor per block iteration (2048 pairs).
// RANK: `deg` holds ranks; keep (u, v) iff rank u < rank v (the same order as (deg, id))
// and emit the relabelled key (rank u << vb) | rank v.
template <bool RANK>
__global__ void __launch_bounds__(256) k_orient(const uint2 *__restrict__ pairs, uint64_t npairs,
                                                const uint32_t *__restrict__ deg, uint64_t n, int vb,
                                                uint64_t *__restrict__ keys, uint64_t capacity,
                                                unsigned long long *__restrict__ cursor,
                                                RadixPlan plan, uint32_t *__restrict__ ghist,
                                                uint32_t *__restrict__ outdeg = nullptr) {
    __shared__ uint32_t sh[kMaxPasses * kRadix];
    __shared__ uint32_t s_wcnt[2][32];
    __shared__ unsigned long long s_base[2];
    for (int i = threadIdx.x; i < plan.npass * kRadix; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    unsigned iter = 0;
    const uint64_t per_block = (uint64_t)blockDim.x * kPP;
    for (uint64_t base = (uint64_t)blockIdx.x * per_block; base < npairs;
         base += (uint64_t)gridDim.x * per_block) {
        // all pair loads first, then all degree/rank gathers: 2 kPP independent
        // gathers in flight per thread (the kernel is gather-latency bound)
        uint2 pr[kPP];
#pragma unroll
        for (int i = 0; i < kPP; ++i) {
            const uint64_t idx = base + warp * 32 * kPP + i * 32 + lane;
            pr[i] = idx < npairs ? ld_stream_u2(pairs + idx) : make_uint2(0xffffffffu, 0xffffffffu);
        }
        uint32_t du[kPP], dv[kPP];
#pragma unroll
        for (int i = 0; i < kPP; ++i) {
            const bool ok = (uint64_t)pr[i].x < n && (uint64_t)pr[i].y < n;  // else flagged upstream
            du[i] = __ldg(deg + (ok ? pr[i].x : 0u));
            dv[i] = __ldg(deg + (ok ? pr[i].y : 0u));
            if (!ok) { du[i] = 0xffffffffu; dv[i] = 0u; }  // never kept (du > dv)
        }
        uint64_t key[kPP];
        unsigned keepmask = 0;
#pragma unroll
        for (int i = 0; i < kPP; ++i) {
            bool fwd;
            if (RANK) {
                fwd = du[i] < dv[i];
                key[i] = ((uint64_t)du[i] << vb) | dv[i];
            } else {
                fwd = du[i] < dv[i] || (du[i] == dv[i] && pr[i].x < pr[i].y);
                key[i] = ((uint64_t)pr[i].x << vb) | pr[i].y;
            }
            if (fwd) keepmask |= 1u << i;
        }
        if (RANK && outdeg) {
            // out-degree by source rank; consecutive lanes mostly share the source (inputs
            // grouped by first id): one atomic per run of equal sources in the warp
#pragma unroll
            for (int i = 0; i < kPP; ++i) {
                const bool k = (keepmask >> i) & 1u;
                const unsigned src = k ? du[i] : 0xffffffffu;
                const unsigned peers = __match_any_sync(TC_FULL_MASK, src);
                if (k && lane == (unsigned)(__ffs(peers) - 1)) atomicAdd(outdeg + src, (unsigned)__popc(peers));
            }
        }
        // block compaction: warp scan, then warp 0 scans the warp totals and reserves the
        // block's output range with one cursor atomic -- two barriers per iteration (the
        // warp-base array alternates between two buffers, so no trailing barrier)
        const uint32_t mine = __popc(keepmask);
        const uint32_t incl = warp_inclusive_scan(mine);
        uint32_t *wc = s_wcnt[iter & 1];
        if (lane == 31) wc[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const unsigned nw = blockDim.x >> 5;
            const uint32_t w = lane < nw ? wc[lane] : 0u;
            const uint32_t wi = warp_inclusive_scan(w);
            const uint32_t tot = __shfl_sync(TC_FULL_MASK, wi, nw - 1);
            if (lane < nw) wc[lane] = wi - w;
            if (lane == 0) s_base[iter & 1] = tot ? atomicAdd(cursor, (unsigned long long)tot) : 0ull;
        }
        __syncthreads();
        uint64_t out = s_base[iter & 1] + wc[warp] + incl - mine;
        ++iter;
#pragma unroll
        for (int i = 0; i < kPP; ++i) {
            if (keepmask & (1u << i)) {
                // streaming store: the keys must not evict the rank table the gathers hit
                if (out < capacity) __stcs(reinterpret_cast<unsigned long long *>(keys) + out, key[i]);
                ++out;
#pragma unroll
                for (int p = 0; p < kMaxPasses; ++p)
                    if (p < plan.npass)
                        atomicAdd(&sh[p * kRadix + ((key[i] >> plan.shift[p]) & ((1u << plan.bits[p]) - 1))], 1u);
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < plan.npass * kRadix; i += blockDim.x)
        if (sh[i]) atomicAdd(&ghist[i], sh[i]);
}

// Node array from a grouped first column (reference preprocess.py:36-46, paper steps 4
// and 8): out-degree histogram of the column (runs of equal ids inside a warp become one
// atomic), then an exclusive scan into node_offsets.  Gaps of empty vertices -- huge in
// rank space, where every isolated vertex ranks first -- cost nothing extra.
__global__ void __launch_bounds__(256) k_run_hist(const uint32_t *__restrict__ col, uint64_t k,
                                                  uint32_t *__restrict__ cnt) {
    const unsigned lane = lane_id();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < k;
         base += stride) {
        const uint64_t i = base + lane;
        const bool ok = i < k;
        const uint32_t u = ok ? col[i] : 0xffffffffu;
        const uint32_t prev = __shfl_up_sync(TC_FULL_MASK, u, 1);
        const bool head = ok && (lane == 0 || prev != u);
        const unsigned heads = __ballot_sync(TC_FULL_MASK, head || !ok);
        if (head) {
            unsigned above = lane == 31 ? 0u : heads & ~((2u << lane) - 1u);
            const unsigned next = above ? (unsigned)(__ffs(above) - 1) : 32u;
            atomicAdd(cnt + u, next - lane);
        }
    }
}

constexpr int kScanTile = 4096;

__global__ void __launch_bounds__(256) k_tile_sum(const uint32_t *__restrict__ cnt, uint64_t n,
                                                  unsigned long long *__restrict__ sums) {
    const uint64_t b = (uint64_t)blockIdx.x * kScanTile;
    unsigned long long acc = 0;
    for (uint64_t i = b + threadIdx.x; i < b + kScanTile && i < n; i += 256) acc += cnt[i];
    __shared__ unsigned long long s_red[8];
    acc = warp_sum(acc);
    if (lane_id() == 0) s_red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < 8; ++w) t += s_red[w];
        sums[blockIdx.x] = t;
    }
}

__global__ void k_scan_sums(unsigned long long *__restrict__ sums, uint64_t nt) {
    __shared__ unsigned long long s_w[32];
    unsigned long long carry = 0;
    for (uint64_t b = 0; b < nt; b += blockDim.x) {
        const uint64_t i = b + threadIdx.x;
        const unsigned long long x = i < nt ? sums[i] : 0;
        unsigned long long t;
        const unsigned long long e = block_exclusive_scan<unsigned long long>(x, s_w, &t);
        if (i < nt) sums[i] = carry + e;
        carry += t;
    }
}

__global__ void __launch_bounds__(256) k_scan_apply(const uint32_t *__restrict__ cnt, uint64_t n,
                                                    const unsigned long long *__restrict__ base,
                                                    int64_t *__restrict__ off,
                                                    uint32_t *__restrict__ off32) {
    __shared__ unsigned long long s_w[32];
    const uint64_t b = (uint64_t)blockIdx.x * kScanTile;
    unsigned long long carry = base[blockIdx.x];
    for (uint64_t c = b; c < b + kScanTile && c < n; c += 256) {
        const uint64_t i = c + threadIdx.x;
        const unsigned long long x = i < n ? cnt[i] : 0;
        unsigned long long t;
        const unsigned long long e = block_exclusive_scan<unsigned long long>(x, s_w, &t);
        if (i < n) {
            off[i] = (int64_t)(carry + e);
            if (off32) off32[i] = (uint32_t)(carry + e);
        }
        carry += t;
    }
}

// Max out-degree over the node array.
__global__ void __launch_bounds__(256) k_max_degree(const int64_t *__restrict__ off, uint64_t n,
                                                    uint32_t *__restrict__ max_out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t best = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint32_t d = (uint32_t)(off[i + 1] - off[i]);
        best = d > best ? d : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint32_t y = __shfl_xor_sync(TC_FULL_MASK, best, o);
        best = y > best ? y : best;
    }
    if (lane_id() == 0 && best) atomicMax(max_out, best);
}

// edge_src from node_offsets (rebuilding a replicated graph without shipping edge_src):
// one warp per vertex writes its run of source ids.
__global__ void __launch_bounds__(256) k_expand_src(const int64_t *__restrict__ off, uint64_t n,
                                                    uint32_t *__restrict__ src,
                                                    uint32_t *__restrict__ off32) {
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    for (uint64_t u = gw; u < n; u += nw) {
        const int64_t b = off[u], e = off[u + 1];
        for (int64_t i = b + lane; i < e; i += 32) src[i] = (uint32_t)u;
        if (lane == 0 && off32) {
            off32[u] = (uint32_t)b;
            if (u + 1 == n) off32[n] = (uint32_t)e;
        }
    }
}

// Pack any (u, v) pairs into (u << vb) | v keys (for sorting the unoriented pairs).
__global__ void k_pack(const uint2 *__restrict__ pairs, uint64_t npairs, int vb,
                       uint64_t *__restrict__ keys) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += stride) {
        uint2 p = ld_stream_u2(pairs + i);
        keys[i] = ((uint64_t)p.x << vb) | p.y;
    }
}

// Order-preserving orientation filter for sorted pairs (standalone API step).
__global__ void __launch_bounds__(256) k_orient_flags(const uint2 *__restrict__ pairs, uint64_t npairs,
                                                      const int64_t *__restrict__ deg,
                                                      uint32_t *__restrict__ tile_counts) {
    __shared__ uint32_t s_scan[32];
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t keep = 0;
    if (i < npairs) {
        uint2 p = pairs[i];
        int64_t du = deg[p.x], dv = deg[p.y];
        keep = du < dv || (du == dv && p.x < p.y);
    }
    uint32_t tot;
    block_exclusive_scan<uint32_t>(keep, s_scan, &tot);
    if (threadIdx.x == 0) tile_counts[blockIdx.x] = tot;
}

__global__ void k_scan_small(uint32_t *__restrict__ counts, uint64_t nblocks,
                             unsigned long long *__restrict__ excl, unsigned long long *__restrict__ total) {
    // single block, sequential chunks of 1024
    __shared__ unsigned long long s_w[32];
    unsigned long long carry = 0;
    for (uint64_t b = 0; b < nblocks; b += blockDim.x) {
        uint64_t i = b + threadIdx.x;
        unsigned long long x = i < nblocks ? counts[i] : 0;
        unsigned long long t;
        unsigned long long e = block_exclusive_scan<unsigned long long>(x, s_w, &t);
        if (i < nblocks) excl[i] = carry + e;
        carry += t;
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(256) k_orient_scatter(const uint2 *__restrict__ pairs, uint64_t npairs,
                                                        const int64_t *__restrict__ deg,
                                                        const unsigned long long *__restrict__ excl,
                                                        uint2 *__restrict__ out) {
    __shared__ uint32_t s_scan[32];
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t keep = 0;
    uint2 p = make_uint2(0, 0);
    if (i < npairs) {
        p = pairs[i];
        int64_t du = deg[p.x], dv = deg[p.y];
        keep = du < dv || (du == dv && p.x < p.y);
    }
    uint32_t tot;
    uint32_t pos = block_exclusive_scan<uint32_t>(keep, s_scan, &tot);
    if (keep) out[excl[blockIdx.x] + pos] = p;
}

// ------------------------------------------------------------- rank space ---
// rank = position of the vertex in (degree, id) order: a stable sort of the ids (already
// in id order) by degree.
__global__ void k_deg_keys(const uint32_t *__restrict__ deg, uint64_t n, uint64_t *__restrict__ keys,
                           uint32_t *__restrict__ ids) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        keys[i] = deg[i];
        ids[i] = (uint32_t)i;
    }
}

__global__ void k_scatter_rank(const uint32_t *__restrict__ ids, uint64_t n,
                               uint32_t *__restrict__ rank, const uint64_t *__restrict__ skeys,
                               uint32_t *__restrict__ deg_by_rank) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        rank[ids[i]] = (uint32_t)i;
        if (deg_by_rank) deg_by_rank[i] = (uint32_t)skeys[i];
    }
}

__global__ void k_max_u32(const uint32_t *__restrict__ a, uint64_t n, uint32_t *__restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t best = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        best = a[i] > best ? a[i] : best;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint32_t y = __shfl_xor_sync(TC_FULL_MASK, best, o);
        best = y > best ? y : best;
    }
    if (lane_id() == 0 && best) atomicMax(out, best);
}

// Undirected degree of an oriented graph: out-degree + in-degree.
__global__ void k_outdeg(const int64_t *__restrict__ off, uint64_t n, uint32_t *__restrict__ deg) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        deg[i] = (uint32_t)(off[i + 1] - off[i]);
}

__global__ void __launch_bounds__(256) k_indeg(const uint32_t *__restrict__ dst, uint64_t m,
                                               uint32_t *__restrict__ deg) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i - threadIdx.x < m; i += stride) {
        const bool ok = i < m;
        const uint32_t w = ok ? dst[i] : 0xffffffffu;
        const unsigned peers = __match_any_sync(TC_FULL_MASK, w);
        if (ok && (int)lane_id() == __ffs(peers) - 1) atomicAdd(deg + w, __popc(peers));
    }
}

__global__ void k_invert_perm(const uint32_t *__restrict__ perm, uint64_t n, uint32_t *__restrict__ inv) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) inv[perm[i]] = (uint32_t)i;
}

__global__ void k_relabel_keys(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                               uint64_t m, const uint32_t *__restrict__ rank, int vb,
                               uint64_t *__restrict__ keys, uint32_t *__restrict__ bad) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    bool ok = true;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        const uint32_t ru = __ldg(rank + src[i]), rv = __ldg(rank + dst[i]);
        ok &= ru < rv;
        keys[i] = ((uint64_t)ru << vb) | rv;
    }
    // the rank-space kernels need every edge to point to a higher rank
    if (__any_sync(TC_FULL_MASK, !ok) && lane_id() == 0) atomicOr(bad, 1u);
}

// hubstart[v] = first position of adj(v) with rank >= hz, or the list end.
__global__ void k_hub_init(const uint32_t *__restrict__ off32, uint64_t n, uint32_t *__restrict__ hs) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        hs[i] = off32[i + 1];
}

__global__ void k_hub_boundary(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                               const uint32_t *__restrict__ off32, uint64_t m, uint32_t hz,
                               uint32_t *__restrict__ hs) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += stride) {
        if (dst[p] < hz) continue;
        const uint32_t v = src[p];
        if (p == off32[v] || dst[p - 1] < hz) hs[v] = (uint32_t)p;
    }
}

// Dense-hub bitmaps (see DeviceGraph): word offsets of every dense vertex, then one bit
// per adjacency entry of a dense vertex.
__global__ void k_dense_len(uint32_t T, uint32_t vt, uint32_t hz, uint32_t hwp,
                            uint32_t *__restrict__ len) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < T; i += gridDim.x * blockDim.x) {
        const uint32_t v = vt + i;
        const uint32_t ws4 = ((v + 1 - hz) >> 5) & ~3u;
        len[i] = hwp > ws4 ? hwp - ws4 : 0u;
    }
}

__global__ void k_excl_scan_u32(uint32_t *__restrict__ a, uint32_t n1) {
    // in place exclusive scan of a[0..n1) (n1 <= a few 10^5), one block
    __shared__ uint32_t s_w[32];
    uint32_t carry = 0;
    for (uint32_t b = 0; b < n1; b += blockDim.x) {
        const uint32_t i = b + threadIdx.x;
        const uint32_t x = i < n1 ? a[i] : 0u;
        uint32_t t;
        const uint32_t e = block_exclusive_scan<uint32_t>(x, s_w, &t);
        if (i < n1) a[i] = carry + e;
        carry += t;
    }
}

__global__ void __launch_bounds__(256) k_dense_fill(const uint32_t *__restrict__ src,
                                                    const uint32_t *__restrict__ dst, uint64_t p0,
                                                    uint64_t m, uint32_t vt, uint32_t hz,
                                                    const uint32_t *__restrict__ dense_off,
                                                    uint32_t *__restrict__ bits) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t p = p0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += stride) {
        const uint32_t v = src[p], r = dst[p] - hz;
        const uint32_t ws4 = ((v + 1 - hz) >> 5) & ~3u;
        atomicOr(bits + dense_off[v - vt] + (r >> 5) - ws4, 1u << (r & 31));
    }
}

}  // namespace

int graph_alloc(DeviceGraph *g, uint64_t m, uint64_t n, cudaStream_t s) {
    g->m = m;
    g->n = n;
    const bool ps = g->persistent;
    TC_CHECK(dalloc_t(&g->src, m + 8, s, ps));
    TC_CHECK(dalloc_t(&g->dst, m + 8, s, ps));  // +32 B so 32-byte chunk loads stay in bounds
    TC_CHECK(dalloc_t(&g->off, n + 1, s, ps));
    g->off32 = nullptr;
    if (m < (1ull << 32)) TC_CHECK(dalloc_t(&g->off32, n + 1, s, ps));
    TC_CUDA(cudaGetDevice(&g->device));
    return 0;
}

void graph_release(DeviceGraph *g, cudaStream_t s) {
    dfree(g->src, s);
    dfree(g->dst, s);
    dfree(g->off, s);
    dfree(g->off32, s);
    dfree(g->hubstart, s);
    dfree(g->dense_off, s);
    dfree(g->dense_bits, s);
    dfree(g->vin_cap, s);
    dfree(g->vix_cnt, s);
    dfree(g->vix_in_e, s);
    g->vix_cnt = nullptr;
    g->vix_in_e = nullptr;
    g->vix_ready = false;
    g->vin_cap = nullptr;
    g->dense_off = g->dense_bits = nullptr;
    g->src = g->dst = nullptr;
    g->off = nullptr;
    g->off32 = nullptr;
    g->hubstart = nullptr;
}

int finalize_graph_dev(DeviceGraph *g, cudaStream_t s) {
    uint32_t *dmax = nullptr;
    TC_CHECK(dalloc_t(&dmax, 1, s));
    if (g->n) {
        k_expand_src<<<grid_for(g->n * 32, 256, kSMs * 16), 256, 0, s>>>(g->off, g->n, g->src, g->off32);
        TC_LAUNCHED();
    } else if (g->off32) {
        TC_CUDA(cudaMemsetAsync(g->off32, 0, sizeof(uint32_t), s));
    }
    TC_CUDA(cudaMemsetAsync(g->dst + g->m, 0, 8 * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(dmax, 0, sizeof(uint32_t), s));
    if (g->n) {
        k_max_degree<<<grid_for(g->n, 256, kSMs * 8), 256, 0, s>>>(g->off, g->n, dmax);
        TC_LAUNCHED();
    }
    TC_CUDA(cudaMemcpyAsync(&g->max_out, dmax, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(dmax, s);
    if (g->rank_space) TC_CHECK(build_hubstart_dev(g, s));
    return 0;
}

int exclusive_scan_dev(const uint32_t *cnt, uint64_t n, int64_t *off, cudaStream_t s) {
    if (n == 0) return 0;
    const uint64_t nt = (n + kScanTile - 1) / kScanTile;
    unsigned long long *sums = nullptr;
    TC_CHECK(dalloc_t(&sums, nt, s));
    k_tile_sum<<<(unsigned)nt, 256, 0, s>>>(cnt, n, sums);
    TC_LAUNCHED();
    k_scan_sums<<<1, 512, 0, s>>>(sums, nt);
    TC_LAUNCHED();
    k_scan_apply<<<(unsigned)nt, 256, 0, s>>>(cnt, n, sums, off, nullptr);
    TC_LAUNCHED();
    dfree(sums, s);
    return 0;
}

int build_node_array_dev(const uint32_t *firsts, uint64_t k, uint64_t n, int64_t *off,
                         uint32_t *off32, uint32_t *max_out, cudaStream_t s) {
    uint32_t *cnt = nullptr;
    unsigned long long *sums = nullptr;
    const uint64_t nt = (n + kScanTile - 1) / kScanTile;
    TC_CHECK(dalloc_t(&cnt, n ? n : 1, s));
    TC_CHECK(dalloc_t(&sums, nt ? nt : 1, s));
    if (n) TC_CUDA(cudaMemsetAsync(cnt, 0, n * sizeof(uint32_t), s));
    if (k) {
        k_run_hist<<<grid_for(k, 256, kSMs * 16), 256, 0, s>>>(firsts, k, cnt);
        TC_LAUNCHED();
    }
    TC_CHECK(node_array_from_counts(cnt, n, k, off, off32, max_out, sums, s));
    dfree(cnt, s);
    dfree(sums, s);
    return 0;
}

// off / off32 = exclusive scan of per-vertex counts (k = total), max_out = max count.
int node_array_from_counts(const uint32_t *cnt, uint64_t n, uint64_t k, int64_t *off, uint32_t *off32,
                           uint32_t *max_out, unsigned long long *sums, cudaStream_t s) {
    const uint64_t nt = (n + kScanTile - 1) / kScanTile;
    if (n) {
        k_tile_sum<<<(unsigned)nt, 256, 0, s>>>(cnt, n, sums);
        TC_LAUNCHED();
        k_scan_sums<<<1, 512, 0, s>>>(sums, nt);
        TC_LAUNCHED();
        k_scan_apply<<<(unsigned)nt, 256, 0, s>>>(cnt, n, sums, off, off32);
        TC_LAUNCHED();
    }
    // off[n] = k (every pair lies in some vertex's run for a valid grouped column)
    const int64_t kk = (int64_t)k;
    TC_CUDA(cudaMemcpyAsync(off + n, &kk, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    if (off32) {
        const uint32_t k32 = (uint32_t)k;
        TC_CUDA(cudaMemcpyAsync(off32 + n, &k32, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    }
    if (max_out) {
        TC_CUDA(cudaMemsetAsync(max_out, 0, sizeof(uint32_t), s));
        if (n) {
            k_max_u32<<<grid_for(n, 256, kSMs * 8), 256, 0, s>>>(cnt, n, max_out);
            TC_LAUNCHED();
        }
    }
    TC_CUDA(cudaStreamSynchronize(s));  // host-side k/k32 sources of the async copies
    return 0;
}

int preprocess_dev(const uint32_t *pairs_u32, uint64_t npairs, uint64_t n, DeviceGraph *out,
                   cudaStream_t s) {
    const uint2 *pairs = reinterpret_cast<const uint2 *>(pairs_u32);
    if (n >= (1ull << 32)) {
        set_error("num_vertices must be < 2^32 on the device path");
        return -1;
    }
    const int vb = n > 1 ? bits_for(n - 1) : 1;
    const RadixPlan plan = make_radix_plan(2 * vb);

    uint32_t *deg = nullptr, *hist = nullptr, *scratch = nullptr;
    unsigned long long *cursor = nullptr;
    TC_CHECK(dalloc_t(&deg, n ? n : 1, s));
    TC_CHECK(dalloc_t(&scratch, 4, s));  // [0] bad-id flag, [1] max out-degree
    TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
    TC_CHECK(dalloc_t(&cursor, 1, s));
    TC_CUDA(cudaMemsetAsync(deg, 0, (n ? n : 1) * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(scratch, 0, 4 * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), s));

    if (npairs) {
        k_degree_hist<<<grid_for(npairs, 256 * kDegPP, kSMs * 8), 256, 0, s>>>(pairs, npairs, deg, n,
                                                                            scratch);
        TC_LAUNCHED();
    }
    // Valid (symmetric) input keeps exactly npairs/2; anything else is sized on a rerun.
    uint64_t capacity = npairs / 2 + 1;
    uint64_t *keys = nullptr, *alt = nullptr;
    TC_CHECK(dalloc_t(&keys, capacity, s));
    if (npairs) {
        k_orient<false><<<grid_for(npairs, 256 * kPP, kSMs * 8), 256, 0, s>>>(pairs, npairs, deg, n, vb, keys,
                                                                       capacity, cursor, plan, hist);
        TC_LAUNCHED();
    }
    uint32_t flags[2];
    unsigned long long kept = 0;
    TC_CUDA(cudaMemcpyAsync(flags, scratch, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaMemcpyAsync(&kept, cursor, sizeof(kept), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    if (flags[0]) {
        dfree(deg, s); dfree(scratch, s); dfree(hist, s); dfree(cursor, s); dfree(keys, s);
        set_error("edge array holds a vertex id >= num_vertices");
        return -1;
    }
    if (kept > capacity) {  // not a symmetric edge array: redo with room for every survivor
        dfree(keys, s);
        capacity = kept;
        TC_CHECK(dalloc_t(&keys, capacity, s));
        TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
        TC_CUDA(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), s));
        k_orient<false><<<grid_for(npairs, 256 * kPP, kSMs * 8), 256, 0, s>>>(pairs, npairs, deg, n, vb, keys,
                                                                       capacity, cursor, plan, hist);
        TC_LAUNCHED();
    }
    const uint64_t m = kept;
    TC_CHECK(graph_alloc(out, m, n, s));
    TC_CHECK(dalloc_t(&alt, m ? m : 1, s));
    TC_CHECK(radix_sort(keys, alt, nullptr, nullptr, m, plan, hist, kOutSoA, out->src, out->dst, vb,
                        nullptr, nullptr, s));
    TC_CUDA(cudaMemsetAsync(out->dst + m, 0, 8 * sizeof(uint32_t), s));
    TC_CHECK(build_node_array_dev(out->src, m, n, out->off, out->off32, scratch + 1, s));
    TC_CUDA(cudaMemcpyAsync(&out->max_out, scratch + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    dfree(deg, s);
    dfree(hist, s);
    dfree(cursor, s);
    dfree(keys, s);
    dfree(alt, s);
    dfree(scratch, s);
    TC_CUDA(cudaStreamSynchronize(s));
    return 0;
}

int sort_pairs_dev(const uint32_t *pairs_u32, uint64_t npairs, uint64_t n, uint32_t *out_pairs,
                   cudaStream_t s) {
    if (npairs == 0) return 0;
    const uint2 *pairs = reinterpret_cast<const uint2 *>(pairs_u32);
    const int vb = n > 1 ? bits_for(n - 1) : 1;
    const RadixPlan plan = make_radix_plan(2 * vb);
    uint64_t *keys = nullptr, *alt = nullptr;
    uint32_t *hist = nullptr;
    TC_CHECK(dalloc_t(&keys, npairs, s));
    TC_CHECK(dalloc_t(&alt, npairs, s));
    TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
    TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
    k_pack<<<grid_for(npairs, 256, kSMs * 16), 256, 0, s>>>(pairs, npairs, vb, keys);
    TC_LAUNCHED();
    TC_CHECK(radix_histogram(keys, npairs, plan, hist, s));
    TC_CHECK(radix_sort(keys, alt, nullptr, nullptr, npairs, plan, hist, kOutAoS, out_pairs, nullptr,
                        vb, nullptr, nullptr, s));
    dfree(keys, s);
    dfree(alt, s);
    dfree(hist, s);
    return 0;
}

int orient_compact_dev(const uint32_t *pairs_u32, uint64_t npairs, const int64_t *deg, uint64_t n,
                       uint32_t *out_pairs, uint64_t *kept, cudaStream_t s) {
    *kept = 0;
    if (npairs == 0) return 0;
    const uint2 *pairs = reinterpret_cast<const uint2 *>(pairs_u32);
    uint64_t nb = (npairs + 255) / 256;
    uint32_t *counts = nullptr;
    unsigned long long *excl = nullptr, *total = nullptr;
    TC_CHECK(dalloc_t(&counts, nb, s));
    TC_CHECK(dalloc_t(&excl, nb, s));
    TC_CHECK(dalloc_t(&total, 1, s));
    k_orient_flags<<<(unsigned)nb, 256, 0, s>>>(pairs, npairs, deg, counts);
    TC_LAUNCHED();
    k_scan_small<<<1, 512, 0, s>>>(counts, nb, excl, total);
    TC_LAUNCHED();
    k_orient_scatter<<<(unsigned)nb, 256, 0, s>>>(pairs, npairs, deg, excl,
                                                  reinterpret_cast<uint2 *>(out_pairs));
    TC_LAUNCHED();
    unsigned long long t = 0;
    TC_CUDA(cudaMemcpyAsync(&t, total, sizeof(t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    *kept = t;
    dfree(counts, s);
    dfree(excl, s);
    dfree(total, s);
    return 0;
}

namespace {

// rank[] of every vertex from its degree (stable sort of ids by degree).
int compute_ranks(const uint32_t *deg, uint64_t n, uint32_t *rank, cudaStream_t s,
                  uint32_t *deg_by_rank = nullptr) {
    if (n == 0) return 0;
    uint32_t *dmax = nullptr, *hist = nullptr, *ids = nullptr, *ialt = nullptr, *sids = nullptr;
    uint64_t *keys = nullptr, *kalt = nullptr;
    TC_CHECK(dalloc_t(&dmax, 1, s));
    TC_CUDA(cudaMemsetAsync(dmax, 0, sizeof(uint32_t), s));
    k_max_u32<<<grid_for(n, 256, kSMs * 8), 256, 0, s>>>(deg, n, dmax);
    TC_LAUNCHED();
    uint32_t maxdeg = 0;
    TC_CUDA(cudaMemcpyAsync(&maxdeg, dmax, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    const RadixPlan plan = make_radix_plan(bits_for(maxdeg));
    TC_CHECK(dalloc_t(&keys, n, s));
    TC_CHECK(dalloc_t(&kalt, n, s));
    TC_CHECK(dalloc_t(&ids, n, s));
    TC_CHECK(dalloc_t(&ialt, n, s));
    TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
    TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
    k_deg_keys<<<grid_for(n, 256, kSMs * 16), 256, 0, s>>>(deg, n, keys, ids);
    TC_LAUNCHED();
    TC_CHECK(radix_histogram(keys, n, plan, hist, s));
    uint64_t *skeys = nullptr;
    TC_CHECK(radix_sort(keys, kalt, ids, ialt, n, plan, hist, kOutKeys, nullptr, nullptr, 0, &skeys,
                        &sids, s));
    k_scatter_rank<<<grid_for(n, 256, kSMs * 16), 256, 0, s>>>(sids, n, rank, skeys, deg_by_rank);
    TC_LAUNCHED();
    dfree(dmax, s);
    dfree(hist, s);
    dfree(keys, s);
    dfree(kalt, s);
    dfree(ids, s);
    dfree(ialt, s);
    return 0;
}

}  // namespace

// Hub zone [hz, n), dense-hub threshold vt, hub words hwp of a rank-space graph.
static void set_hub_params(DeviceGraph *g) {
    g->hz = g->n > kHubRanks ? (uint32_t)(g->n - kHubRanks) : 0u;
    g->rank_space = true;
    const uint32_t hub_n = (uint32_t)(g->n - g->hz);
    g->hwp = ((hub_n + 31) / 32 + 3) & ~3u;
    const uint32_t dense_ranks = (uint32_t)opts().dense_ranks;
    const uint32_t T = hub_n < dense_ranks ? hub_n : dense_ranks;
    g->vt = (uint32_t)g->n - T;
}

int build_hubstart_dev(DeviceGraph *g, cudaStream_t s) {
    if (!g->off32) {
        set_error("rank space needs m < 2^32");
        return -1;
    }
    g->hz = g->n > kHubRanks ? (uint32_t)(g->n - kHubRanks) : 0u;
    if (!g->hubstart) TC_CHECK(dalloc_t(&g->hubstart, g->n ? g->n : 1, s, g->persistent));
    if (g->n && !g->hubstart_ready) {
        k_hub_init<<<grid_for(g->n, 256, kSMs * 16), 256, 0, s>>>(g->off32, g->n, g->hubstart);
        TC_LAUNCHED();
    }
    if (g->m && !g->hubstart_ready) {
        k_hub_boundary<<<grid_for(g->m, 256, kSMs * 16), 256, 0, s>>>(g->src, g->dst, g->off32, g->m,
                                                                      g->hz, g->hubstart);
        TC_LAUNCHED();
    }
    set_hub_params(g);
    const uint32_t T = (uint32_t)g->n - g->vt;
    dfree(g->dense_off, s);
    dfree(g->dense_bits, s);
    if (!g->vix_ready) {  // the prebuilt v-major index was laid out on this capacity layout
        dfree(g->vin_cap, s);
        g->vin_cap = nullptr;
    }
    g->dense_off = g->dense_bits = nullptr;
    TC_CHECK(dalloc_t(&g->dense_off, (size_t)T + 1, s, g->persistent));
    uint32_t words = 0;
    if (T) {
        k_dense_len<<<grid_for(T, 256, kSMs * 4), 256, 0, s>>>(T, g->vt, g->hz, g->hwp, g->dense_off);
        TC_LAUNCHED();
        TC_CUDA(cudaMemsetAsync(g->dense_off + T, 0, sizeof(uint32_t), s));
        k_excl_scan_u32<<<1, 1024 - 32, 0, s>>>(g->dense_off, T + 1);
        TC_LAUNCHED();
        TC_CUDA(cudaMemcpyAsync(&words, g->dense_off + T, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        uint32_t p0 = 0;
        TC_CUDA(cudaMemcpyAsync(&p0, g->off32 + g->vt, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
        TC_CHECK(dalloc_t(&g->dense_bits, (size_t)words + 4, s, g->persistent));
        g->dense_words = words + 4;
        TC_CUDA(cudaMemsetAsync(g->dense_bits, 0, ((size_t)words + 4) * sizeof(uint32_t), s));
        if (g->m > p0) {
            k_dense_fill<<<grid_for(g->m - p0, 256, kSMs * 16), 256, 0, s>>>(
                g->src, g->dst, p0, g->m, g->vt, g->hz, g->dense_off, g->dense_bits);
            TC_LAUNCHED();
        }
    }
    return 0;
}

// ------------------------------------------------------- bucket CSR build ---
// Rank-space CSR without the global key sort: the out-degree histogram (fused into
// k_orient) gives node_offsets directly; every oriented key is scattered into its source's
// bucket (warp-aggregated cursor atomics -- sources repeat along the key stream), then
// each adjacency list is sorted in place by a size-class segmented sort:
//   d <= 16      thread per list, bitonic network in registers;
//   17..64       warp per list, 2 elements per lane, shuffle bitonic;
//   65..4096     CTA per list, shared-memory bitonic;
//   > 4096       (few lists) composite (list, v) keys through the global LSD radix sort.
// The result is byte-identical to the sorted-key build (adjacency lists hold distinct
// ranks, so their sorted order is unique).
namespace {

__global__ void __launch_bounds__(256)
    k_bucket_scatter(const uint64_t *__restrict__ keys, uint64_t m, int vb,
                     const uint32_t *__restrict__ off32, uint32_t *__restrict__ cursor,
                     uint32_t *__restrict__ dst) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t mask = (1ull << vb) - 1;
    const unsigned lane = lane_id();
    // uniform trip count per warp so the warp-aggregated atomics see full warps
    const uint64_t wbase = ((uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u));
    for (uint64_t b = wbase; b < m; b += stride) {
        const uint64_t i = b + lane;
        const bool ok = i < m;
        const uint64_t key = ok ? __ldcs(keys + i) : 0ull;
        const uint32_t u = ok ? (uint32_t)(key >> vb) : 0xffffffffu;
        const unsigned peers = __match_any_sync(TC_FULL_MASK, u);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (ok && (int)lane == leader) base = atomicAdd(cursor + u, (unsigned)__popc(peers));
        base = __shfl_sync(TC_FULL_MASK, base, leader);
        if (ok) dst[__ldg(off32 + u) + base + __popc(peers & lanemask_lt())] = (uint32_t)(key & mask);
    }
}

// Lists by size class (append order is irrelevant: lists are disjoint).
// w512 == nullptr: 257..1024 all go to w1k (one 1024-wide network); w2k == nullptr:
// 1025..2048 go to the CTA shared-memory sort with 2049..4096.
__global__ void k_seg_classify(const uint32_t *__restrict__ off32, uint64_t n,
                               uint32_t *__restrict__ mid, uint32_t *__restrict__ big,
                               uint32_t *__restrict__ warpl, uint32_t *__restrict__ w256,
                               uint32_t *__restrict__ w512, uint32_t *__restrict__ w1k,
                               uint32_t *__restrict__ w2k, unsigned *__restrict__ counts) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride) {
        const uint32_t d = off32[u + 1] - off32[u];
        if (d <= 16) continue;
        if (d <= 64) warpl[atomicAdd(counts + 0, 1u)] = (uint32_t)u;
        else if (d <= 256) w256[atomicAdd(counts + 3, 1u)] = (uint32_t)u;
        else if (d <= 512 && w512) w512[atomicAdd(counts + 5, 1u)] = (uint32_t)u;
        else if (d <= 1024) w1k[atomicAdd(counts + 4, 1u)] = (uint32_t)u;
        else if (d <= 2048 && w2k) w2k[atomicAdd(counts + 6, 1u)] = (uint32_t)u;
        else if (d <= 4096) mid[atomicAdd(counts + 1, 1u)] = (uint32_t)u;
        else big[atomicAdd(counts + 2, 1u)] = (uint32_t)u;
    }
}

__device__ __forceinline__ void cswap(uint32_t &a, uint32_t &b) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

// d <= 16: thread per list, 16-wide bitonic network in registers (pad = ~0).
__global__ void __launch_bounds__(256)
    k_seg_sort16(const uint32_t *__restrict__ off32, uint64_t n, uint32_t *__restrict__ dst, uint32_t hz,
                 uint32_t *__restrict__ hs, const VFill vf) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride) {
        const uint32_t s = off32[u], d = off32[u + 1] - s;
        if (d > 16) continue;
        if (d < 2) {
            if (hs) hs[u] = s + (d == 1 && dst[s] < hz ? 1u : 0u);
            continue;
        }
        uint32_t x[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = (uint32_t)i < d ? dst[s + i] : 0xffffffffu;
#pragma unroll
        for (int k = 2; k <= 16; k <<= 1)
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int l = i ^ j;
                    if (l > i) {
                        if ((i & k) == 0) cswap(x[i], x[l]);
                        else cswap(x[l], x[i]);
                    }
                }
        uint32_t below = 0;  // non-hub prefix length (elements < hz; pads are ~0)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if ((uint32_t)i < d) dst[s + i] = x[i];
            below += x[i] < hz ? 1u : 0u;
        }
#pragma unroll
        for (int i0 = 0; i0 < 16; i0 += 4) {  // the index fill, 4 elements at a time
            const uint32_t eg[4] = {s + i0, s + i0 + 1, s + i0 + 2, s + i0 + 3};
            const uint32_t vg[4] = {x[i0], x[i0 + 1], x[i0 + 2], x[i0 + 3]};
            const bool okg[4] = {(uint32_t)i0 < d, (uint32_t)i0 + 1 < d, (uint32_t)i0 + 2 < d, (uint32_t)i0 + 3 < d};
            vfill_batch<4>(vf, eg, s + d, vg, okg);
        }
        if (hs) hs[u] = s + below;
    }
}

// 17..64: warp per list, element 2*lane+h in register h; bitonic over 64 with shuffles.
__global__ void __launch_bounds__(256)
    k_seg_sort64(const uint32_t *__restrict__ off32, const uint32_t *__restrict__ list,
                 const unsigned *__restrict__ count, uint32_t *__restrict__ dst, uint32_t hz,
                 uint32_t *__restrict__ hs, const VFill vf) {
    const unsigned lane = lane_id();
    const unsigned nl = *count;
    const unsigned gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nw = (gridDim.x * blockDim.x) >> 5;
    for (unsigned w = gw; w < nl; w += nw) {
        const uint32_t u = list[w];
        const uint32_t s = off32[u], d = off32[u + 1] - s;
        uint32_t x[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t i = 2 * lane + h;
            x[h] = i < d ? dst[s + i] : 0xffffffffu;
        }
        for (int k = 2; k <= 64; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                if (j == 1) {  // partner inside the lane
                    const uint32_t i = 2 * lane;
                    if ((i & k) == 0) cswap(x[0], x[1]);
                    else cswap(x[1], x[0]);
                } else {  // partner lane = lane ^ (j / 2), same register
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t i = 2 * lane + h;
                        const uint32_t y = __shfl_xor_sync(TC_FULL_MASK, x[h], j >> 1);
                        const bool lower = (i & j) == 0;  // i < partner
                        const bool asc = (i & k) == 0;
                        x[h] = (lower == asc) ? min(x[h], y) : max(x[h], y);
                    }
                }
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t i = 2 * lane + h;
            if (i < d) dst[s + i] = x[h];
        }
        {
            const uint32_t e2[2] = {s + 2 * lane, s + 2 * lane + 1};
            const bool ok2[2] = {2 * lane < d, 2 * lane + 1 < d};
            vfill_batch<2>(vf, e2, s + d, x, ok2);
        }
        if (hs) {
            const uint32_t below = __popc(__ballot_sync(TC_FULL_MASK, x[0] < hz)) +
                                   __popc(__ballot_sync(TC_FULL_MASK, x[1] < hz));
            if (lane == 0) hs[u] = s + below;
        }
    }
}

// 65..32K lists: warp per list, K registers per lane, element i = 32 r + lane; partners at
// distance j >= 32 are in the same lane (register r ^ j/32), closer ones in lane ^ j.
template <int K>
__global__ void __launch_bounds__(256)
    k_seg_sort_warp(const uint32_t *__restrict__ off32, const uint32_t *__restrict__ list,
                    const unsigned *__restrict__ count, uint32_t *__restrict__ dst, uint32_t hz,
                    uint32_t *__restrict__ hs, const VFill vf) {
    constexpr int N = 32 * K;
    const unsigned lane = lane_id();
    const unsigned nl = *count;
    const unsigned gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nw = (gridDim.x * blockDim.x) >> 5;
    for (unsigned w = gw; w < nl; w += nw) {
        const uint32_t u = list[w];
        const uint32_t s = off32[u], d = off32[u + 1] - s;
        uint32_t x[K];
#pragma unroll
        for (int r = 0; r < K; ++r) {
            const uint32_t i = 32 * r + lane;
            x[r] = i < d ? dst[s + i] : 0xffffffffu;
        }
#pragma unroll
        for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                if (j >= 32) {
#pragma unroll
                    for (int r = 0; r < K; ++r) {
                        const int q = r ^ (j >> 5);
                        if (q > r) {
                            // i & k for i = 32 r + lane, k >= 64: depends on r only
                            if (((32 * r) & k) == 0) cswap(x[r], x[q]);
                            else cswap(x[q], x[r]);
                        }
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < K; ++r) {
                        const uint32_t i = 32 * r + lane;
                        const uint32_t y = __shfl_xor_sync(TC_FULL_MASK, x[r], j);
                        const bool lower = (i & j) == 0;
                        const bool asc = (i & k) == 0;
                        x[r] = (lower == asc) ? min(x[r], y) : max(x[r], y);
                    }
                }
            }
        }
        uint32_t below = 0;
#pragma unroll
        for (int r = 0; r < K; ++r) {
            const uint32_t i = 32 * r + lane;
            if (i < d) dst[s + i] = x[r];
            below += __popc(__ballot_sync(TC_FULL_MASK, x[r] < hz));
        }
        // the index fill in groups of G registers (all loads / atomics of a group together)
        constexpr int G = K < 8 ? K : 8;
#pragma unroll
        for (int r0 = 0; r0 < K; r0 += G) {
            uint32_t eg[G], vg[G];
            bool okg[G];
#pragma unroll
            for (int j = 0; j < G; ++j) {
                eg[j] = s + 32 * (r0 + j) + lane;
                vg[j] = x[r0 + j];
                okg[j] = 32 * (r0 + j) + lane < d;
            }
            vfill_batch<G>(vf, eg, s + d, vg, okg);
        }
        if (hs && lane == 0) hs[u] = s + below;
    }
}

// 257..4096: CTA per list, shared-memory bitonic over the next power of two.
#ifndef TC_SORT4K_NT
#define TC_SORT4K_NT 256
#endif
__global__ void __launch_bounds__(TC_SORT4K_NT)
    k_seg_sort4k(const uint32_t *__restrict__ off32, const uint32_t *__restrict__ list,
                 const unsigned *__restrict__ count, uint32_t *__restrict__ dst, uint32_t hz,
                 uint32_t *__restrict__ hs, const VFill vf) {
    __shared__ uint32_t sh[4096];
    const unsigned nl = *count;
    for (unsigned w = blockIdx.x; w < nl; w += gridDim.x) {
        const uint32_t u = list[w];
        const uint32_t s = off32[u], d = off32[u + 1] - s;
        uint32_t N = 2048;
        while (N < d) N <<= 1;
        for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) sh[i] = i < d ? dst[s + i] : 0xffffffffu;
        __syncthreads();
        for (uint32_t k = 2; k <= N; k <<= 1) {
            for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                for (uint32_t t = threadIdx.x; t < N / 2; t += blockDim.x) {
                    const uint32_t i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), l = i + j;
                    const uint32_t a = sh[i], b = sh[l];
                    if ((a > b) == ((i & k) == 0)) {
                        sh[i] = b;
                        sh[l] = a;
                    }
                }
                __syncthreads();
            }
        }
        for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) {
            dst[s + i] = sh[i];
            vfill(vf, s + i, s + d, sh[i]);
        }
        if (hs && threadIdx.x == 0) {  // lower bound of hz in the sorted list
            uint32_t a = 0, n2 = d;
            while (n2 > 0) {
                const uint32_t h2 = n2 >> 1;
                if (sh[a + h2] < hz) { a += h2 + 1; n2 -= h2 + 1; } else n2 = h2;
            }
            hs[u] = s + a;
        }
        __syncthreads();
    }
}

// > 4096: composite keys (big-list index << vb | v) in list order.
__global__ void k_big_keys(const uint32_t *__restrict__ off32, const uint32_t *__restrict__ big,
                           const uint32_t *__restrict__ cstart, uint32_t nbig, int vb,
                           const uint32_t *__restrict__ dst, uint64_t *__restrict__ keys) {
    for (uint32_t b = blockIdx.x; b < nbig; b += gridDim.x) {
        const uint32_t u = big[b], s = off32[u], d = off32[u + 1] - s, c = cstart[b];
        for (uint32_t i = threadIdx.x; i < d; i += blockDim.x)
            keys[c + i] = ((uint64_t)b << vb) | dst[s + i];
    }
}

__global__ void k_big_back(const uint32_t *__restrict__ off32, const uint32_t *__restrict__ big,
                           const uint32_t *__restrict__ cstart, uint32_t nbig, int vb,
                           const uint64_t *__restrict__ keys, uint32_t *__restrict__ dst, const VFill vf) {
    const uint64_t mask = (1ull << vb) - 1;
    for (uint32_t b = blockIdx.x; b < nbig; b += gridDim.x) {
        const uint32_t u = big[b], s = off32[u], d = off32[u + 1] - s, c = cstart[b];
        for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) {
            const uint32_t x = (uint32_t)(keys[c + i] & mask);
            dst[s + i] = x;
            vfill(vf, s + i, s + d, x);
        }
    }
}

// hubstart of the long lists below the hub zone before their sort (the v-major test reads
// it for heads in [z0, hz) with |adj(v)| > nhcap): elements < hz of the unsorted list, one
// warp per list.
__global__ void __launch_bounds__(256)
    k_hub_count_long(const uint32_t *__restrict__ off32, const uint32_t *__restrict__ dst, uint32_t z0,
                     uint32_t hz, uint32_t nhcap, uint32_t *__restrict__ hs) {
    const unsigned lane = lane_id();
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t b = z0 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; b < hz; b += nw * 32) {
        const uint32_t v = b + lane;
        const uint32_t d = v < hz ? off32[v + 1] - off32[v] : 0u;
        unsigned lm = __ballot_sync(TC_FULL_MASK, d > nhcap);
        while (lm) {
            const int l = __ffs(lm) - 1;
            lm &= lm - 1;
            const uint32_t w = b + l, s = off32[w], e = off32[w + 1];
            uint32_t c = 0;
            for (uint32_t i = s + lane; i < e; i += 32) c += dst[i] < hz ? 1u : 0u;
            c = warp_sum(c);
            if (lane == 0) hs[w] = s + c;
        }
    }
}

__global__ void k_big_hubstart(const uint32_t *__restrict__ off32, const uint32_t *__restrict__ big,
                               uint32_t nbig, const uint32_t *__restrict__ dst, uint32_t hz,
                               uint32_t *__restrict__ hs) {
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nbig; b += gridDim.x * blockDim.x) {
        const uint32_t u = big[b], s = off32[u];
        uint32_t a = 0, n2 = off32[u + 1] - s;
        while (n2 > 0) {
            const uint32_t h2 = n2 >> 1;
            if (dst[s + a + h2] < hz) { a += h2 + 1; n2 -= h2 + 1; } else n2 = h2;
        }
        hs[u] = s + a;
    }
}

__global__ void k_big_sizes(const uint32_t *__restrict__ off32, const uint32_t *__restrict__ big,
                            uint32_t nbig, uint32_t *__restrict__ sz) {
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nbig; b += gridDim.x * blockDim.x)
        sz[b] = off32[big[b] + 1] - off32[big[b]];
}

// edge_src from node_offsets: thread per vertex (long lists are rare and short-lived).
__global__ void __launch_bounds__(256)
    k_fill_src(const uint32_t *__restrict__ off32, uint64_t n, uint32_t *__restrict__ src) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const unsigned lane = lane_id();
    // thread per vertex for short lists; lists longer than 32 are written by the whole warp
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); b < n; b += stride) {
        const uint64_t u = b + lane;
        uint32_t s = 0, e = 0;
        if (u < n) {
            s = off32[u];
            e = off32[u + 1];
        }
        const bool longl = e - s > 32;
        if (!longl)
            for (uint32_t p = s; p < e; ++p) src[p] = (uint32_t)u;
        unsigned lm = __ballot_sync(TC_FULL_MASK, longl);
        while (lm) {
            const int l = __ffs(lm) - 1;
            lm &= lm - 1;
            const uint32_t ls = __shfl_sync(TC_FULL_MASK, s, l), le = __shfl_sync(TC_FULL_MASK, e, l);
            for (uint32_t p = ls + lane; p < le; p += 32) src[p] = (uint32_t)(b + l);
        }
    }
}

}  // namespace

// keys: m oriented rank keys (u << vb | v), outdeg: per-source counts (consumed as cursors).
// Side streams for independent kernels of one call (created once; callers hold the API lock).
static cudaStream_t fork_stream(int i) {
    static cudaStream_t ss[4] = {nullptr, nullptr, nullptr, nullptr};
    if (!ss[i]) cudaStreamCreateWithFlags(&ss[i], cudaStreamNonBlocking);
    return ss[i];
}

// Prepares the v-major in-edge index that the segmented sorts fill (VFill) when full counts
// of this graph will run the v-major schedule: hub parameters, the capacity layout from the
// degrees, hubstart of the long low-zone lists, zeroed fill counts.  Returns vf.vp.z0 = ~0
// (fill off) otherwise.
static int prepare_vfill(DeviceGraph *g, const uint32_t *deg_by_rank, const uint32_t *max_out_dev, VFill *vf,
                         cudaStream_t s) {
    vf->vp.z0 = 0xffffffffu;
    if (!deg_by_rank || !opts().vix || !g->off32 || !g->hubstart || g->n == 0) return 0;
    set_hub_params(g);
    TC_CUDA(cudaMemcpyAsync(&g->max_out, max_out_dev, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    if (!vmajor_schedule(*g)) return 0;
    TC_CHECK(vin_capacity_dev(g, deg_by_rank, s));
    const VSplit vp = make_vsplit(*g, true);
    const uint32_t nz = (uint32_t)(g->n - vp.z0);
    TC_CHECK(dalloc_t(&g->vix_cnt, (size_t)nz + 1, s, g->persistent));  // [nz]: overflow flag
    TC_CHECK(dalloc_t(&g->vix_in_e, g->vin_total ? g->vin_total : 1, s, g->persistent));
    TC_CUDA(cudaMemsetAsync(g->vix_cnt, 0, ((size_t)nz + 1) * sizeof(uint32_t), s));
    if (vp.z0 < g->hz) {
        k_hub_count_long<<<kSMs * 8, 256, 0, s>>>(g->off32, g->dst, vp.z0, g->hz, vp.nhcap, g->hubstart);
        TC_LAUNCHED();
    }
    vf->vp = vp;
    vf->off32 = g->off32;
    vf->start = g->vin_cap;
    vf->cnt = g->vix_cnt;
    vf->flag = g->vix_cnt + nz;
    vf->in_e = g->vix_in_e;
    g->vix_vp = vp;
    return 0;
}

static int bucket_csr_dev(const uint64_t *keys, uint64_t m, uint64_t n, int vb, uint32_t *outdeg,
                          DeviceGraph *out, uint32_t *max_out_dev, cudaStream_t s,
                          const uint32_t *deg_by_rank) {
    unsigned long long *sums = nullptr;
    const uint64_t nt = (n + kScanTile - 1) / kScanTile;
    TC_CHECK(dalloc_t(&sums, nt ? nt : 1, s));
    TC_CHECK(node_array_from_counts(outdeg, n, m, out->off, out->off32, max_out_dev, sums, s));
    dfree(sums, s);
    if (n) TC_CUDA(cudaMemsetAsync(outdeg, 0, n * sizeof(uint32_t), s));
    if (m) {
        k_bucket_scatter<<<grid_for(m, 256, kSMs * 16), 256, 0, s>>>(keys, m, vb, out->off32, outdeg, out->dst);
        TC_LAUNCHED();
    }
    if (!n) return 0;
    uint32_t *warpl = nullptr, *w256 = nullptr, *w512 = nullptr, *w1k = nullptr, *mid = nullptr, *big = nullptr;
    unsigned *counts = nullptr;
    // 257..512 on a 512-wide network (half the comparators of the 1024-wide one)
    const bool k16 = opts().seg_k16 != 0;
    TC_CHECK(dalloc_t(&counts, 8, s));
    TC_CHECK(dalloc_t(&warpl, n, s));
    TC_CHECK(dalloc_t(&w256, n, s));
    if (k16) TC_CHECK(dalloc_t(&w512, n, s));
    // 1025..2048 as a warp network in registers (64 per lane) instead of shared memory
    const bool w2 = opts().seg_w2k != 0;
    uint32_t *w2k = nullptr;
    if (w2) TC_CHECK(dalloc_t(&w2k, n, s));
    TC_CHECK(dalloc_t(&w1k, n, s));
    TC_CHECK(dalloc_t(&mid, n, s));
    TC_CHECK(dalloc_t(&big, n, s));
    TC_CUDA(cudaMemsetAsync(counts, 0, 8 * sizeof(unsigned), s));
    k_seg_classify<<<grid_for(n, 256, kSMs * 8), 256, 0, s>>>(out->off32, n, mid, big, warpl, w256,
                                                              w512, w1k, w2k, counts);
    TC_LAUNCHED();
    // hubstart (first element >= hz of every list) falls out of the sorts for free
    const uint32_t hz = n > kHubRanks ? (uint32_t)(n - kHubRanks) : 0u;
    if (!out->hubstart) TC_CHECK(dalloc_t(&out->hubstart, n, s, out->persistent));
    uint32_t *hs = out->hubstart;
    // the v-major in-edge index is filled as the sorts place every element
    VFill vf;
    TC_CHECK(prepare_vfill(out, deg_by_rank, max_out_dev, &vf, s));
    // The size classes sort disjoint lists: the five latency-bound sorts run concurrently
    // (forked off s, joined back before the long-list radix pass reads `counts`).
    const bool fork = opts().seg_fork != 0;
    cudaEvent_t ev_fork = nullptr, ev_join[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaStream_t ss[4] = {s, s, s, s};
    if (fork) {
        TC_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        TC_CUDA(cudaEventRecord(ev_fork, s));
        for (int i = 0; i < 4; ++i) {
            ss[i] = fork_stream(i);
            TC_CUDA(cudaEventCreateWithFlags(&ev_join[i], cudaEventDisableTiming));
            TC_CUDA(cudaStreamWaitEvent(ss[i], ev_fork, 0));
        }
    }
    k_seg_sort4k<<<kSMs * 8 * 256 / TC_SORT4K_NT, TC_SORT4K_NT, 0, ss[0]>>>(out->off32, mid, counts + 1, out->dst, hz, hs, vf);
    TC_LAUNCHED();
    k_seg_sort_warp<32><<<kSMs * 8, 256, 0, ss[1]>>>(out->off32, w1k, counts + 4, out->dst, hz, hs, vf);
    TC_LAUNCHED();
    if (k16) {
        k_seg_sort_warp<16><<<kSMs * 8, 256, 0, ss[2]>>>(out->off32, w512, counts + 5, out->dst, hz, hs, vf);
        TC_LAUNCHED();
    }
    if (w2) {
        k_seg_sort_warp<64><<<kSMs * 4, 256, 0, ss[0]>>>(out->off32, w2k, counts + 6, out->dst, hz, hs, vf);
        TC_LAUNCHED();
    }
    k_seg_sort_warp<8><<<kSMs * 8, 256, 0, ss[2]>>>(out->off32, w256, counts + 3, out->dst, hz, hs, vf);
    TC_LAUNCHED();
    k_seg_sort64<<<kSMs * 8, 256, 0, ss[3]>>>(out->off32, warpl, counts + 0, out->dst, hz, hs, vf);
    TC_LAUNCHED();
    k_seg_sort16<<<grid_for(n, 256, kSMs * 16), 256, 0, s>>>(out->off32, n, out->dst, hz, hs, vf);
    TC_LAUNCHED();
    if (fork) {
        for (int i = 0; i < 4; ++i) {
            TC_CUDA(cudaEventRecord(ev_join[i], ss[i]));
            TC_CUDA(cudaStreamWaitEvent(s, ev_join[i], 0));
            cudaEventDestroy(ev_join[i]);
        }
        cudaEventDestroy(ev_fork);
    }
    unsigned nbig = 0;
    TC_CUDA(cudaMemcpyAsync(&nbig, counts + 2, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    if (nbig) {
        uint32_t *cstart = nullptr;
        TC_CHECK(dalloc_t(&cstart, (size_t)nbig + 1, s));
        k_big_sizes<<<grid_for(nbig, 256, kSMs), 256, 0, s>>>(out->off32, big, nbig, cstart);
        TC_LAUNCHED();
        TC_CUDA(cudaMemsetAsync(cstart + nbig, 0, sizeof(uint32_t), s));
        k_excl_scan_u32<<<1, 1024 - 32, 0, s>>>(cstart, nbig + 1);
        TC_LAUNCHED();
        uint32_t tot = 0;
        TC_CUDA(cudaMemcpyAsync(&tot, cstart + nbig, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
        uint64_t *bk = nullptr, *balt = nullptr, *sorted = nullptr;
        uint32_t *hist = nullptr;
        TC_CHECK(dalloc_t(&bk, tot, s));
        TC_CHECK(dalloc_t(&balt, tot, s));
        TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
        TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
        k_big_keys<<<nbig < kSMs * 8 ? nbig : kSMs * 8, 256, 0, s>>>(out->off32, big, cstart, nbig, vb,
                                                                    out->dst, bk);
        TC_LAUNCHED();
        const int bb = nbig > 1 ? bits_for(nbig - 1) : 1;
        const RadixPlan plan = make_radix_plan(bb + vb);
        TC_CHECK(radix_histogram(bk, tot, plan, hist, s));
        TC_CHECK(radix_sort(bk, balt, nullptr, nullptr, tot, plan, hist, kOutKeys, nullptr, nullptr, 0,
                            &sorted, nullptr, s));
        k_big_back<<<nbig < kSMs * 8 ? nbig : kSMs * 8, 256, 0, s>>>(out->off32, big, cstart, nbig, vb,
                                                                    sorted, out->dst, vf);
        TC_LAUNCHED();
        k_big_hubstart<<<grid_for(nbig, 256, kSMs), 256, 0, s>>>(out->off32, big, nbig, out->dst, hz, hs);
        TC_LAUNCHED();
        dfree(bk, s);
        dfree(balt, s);
        dfree(hist, s);
        dfree(cstart, s);
    }
    k_fill_src<<<grid_for(n, 256, kSMs * 16), 256, 0, s>>>(out->off32, n, out->src);
    TC_LAUNCHED();
    out->hubstart_ready = true;
    if (vf.vp.z0 != 0xffffffffu) {
        // a non-symmetric input overflows the capacity layout: no prebuilt index then (the
        // count builds an exact one)
        uint32_t flag = 0;
        TC_CUDA(cudaMemcpyAsync(&flag, vf.flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
        out->vix_ready = flag == 0;
        if (!out->vix_ready) {
            dfree(out->vix_cnt, s);
            dfree(out->vix_in_e, s);
            out->vix_cnt = nullptr;
            out->vix_in_e = nullptr;
        }
    }
    dfree(counts, s);
    dfree(warpl, s);
    dfree(w256, s);
    dfree(w512, s);
    dfree(w2k, s);
    dfree(w1k, s);
    dfree(mid, s);
    dfree(big, s);
    return 0;
}

int degree_hist_dev(const uint32_t *pairs_u32, uint64_t npairs, uint64_t n, uint32_t *deg, uint32_t *bad,
                    cudaStream_t s) {
    if (!npairs) return 0;
    k_degree_hist<<<grid_for(npairs, 256 * kDegPP, kSMs * 8), 256, 0, s>>>(
        reinterpret_cast<const uint2 *>(pairs_u32), npairs, deg, n, bad);
    TC_LAUNCHED();
    return 0;
}

int preprocess_rank_dev(const uint32_t *pairs_u32, uint64_t npairs, uint64_t n, DeviceGraph *out,
                        cudaStream_t s, uint32_t *id_of_rank, const PreDegrees *pre) {
    const uint2 *pairs = reinterpret_cast<const uint2 *>(pairs_u32);
    if (n >= (1ull << 32) || npairs / 2 >= (1ull << 32)) {
        set_error("rank-space preprocessing needs num_vertices < 2^32 and m < 2^32");
        return -1;
    }
    const int vb = n > 1 ? bits_for(n - 1) : 1;
    const RadixPlan plan = make_radix_plan(2 * vb);
    uint32_t *deg = nullptr, *rank = nullptr, *hist = nullptr, *scratch = nullptr;
    unsigned long long *cursor = nullptr;
    if (pre) {
        deg = pre->deg;  // histogram already taken chunk by chunk during the H2D copy (owned now)
    } else {
        TC_CHECK(dalloc_t(&deg, n ? n : 1, s));
    }
    TC_CHECK(dalloc_t(&rank, n ? n : 1, s));
    TC_CHECK(dalloc_t(&scratch, 4, s));
    TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
    TC_CHECK(dalloc_t(&cursor, 1, s));
    if (!pre) TC_CUDA(cudaMemsetAsync(deg, 0, (n ? n : 1) * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(scratch, 0, 4 * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), s));
    if (npairs && !pre) {
        k_degree_hist<<<grid_for(npairs, 256 * kDegPP, kSMs * 8), 256, 0, s>>>(pairs, npairs, deg, n,
                                                                            scratch);
        TC_LAUNCHED();
    }
    uint32_t bad = 0;
    TC_CUDA(cudaMemcpyAsync(&bad, pre ? pre->bad : scratch, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    if (bad) {
        set_error("edge array holds a vertex id >= num_vertices");
        return -1;
    }
    const int64_t bucket_env = opts().bucket;
    const bool bucket = bucket_env != 0 && n > 0;
    uint32_t *deg_by_rank = nullptr;  // degrees in rank order (v-major capacity layout)
    if (bucket) TC_CHECK(dalloc_t(&deg_by_rank, n, s));
    TC_CHECK(compute_ranks(deg, n, rank, s, deg_by_rank));
    uint64_t capacity = npairs / 2 + 1;
    uint64_t *keys = nullptr, *alt = nullptr;
    TC_CHECK(dalloc_t(&keys, capacity, s));
    uint32_t *outdeg = bucket ? deg : nullptr;  // degrees are consumed by compute_ranks
    const RadixPlan oplan = bucket ? RadixPlan{} : plan;
    if (bucket) TC_CUDA(cudaMemsetAsync(outdeg, 0, n * sizeof(uint32_t), s));
    if (npairs) {
        k_orient<true><<<grid_for(npairs, 256 * kPP, kSMs * 8), 256, 0, s>>>(
            pairs, npairs, rank, n, vb, keys, capacity, cursor, oplan, hist, outdeg);
        TC_LAUNCHED();
    }
    unsigned long long kept = 0;
    TC_CUDA(cudaMemcpyAsync(&kept, cursor, sizeof(kept), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    if (kept > capacity) {  // not a symmetric edge array: redo with room for every survivor
        dfree(keys, s);
        capacity = kept;
        TC_CHECK(dalloc_t(&keys, capacity, s));
        TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
        TC_CUDA(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), s));
        if (bucket) TC_CUDA(cudaMemsetAsync(outdeg, 0, n * sizeof(uint32_t), s));
        k_orient<true><<<grid_for(npairs, 256 * kPP, kSMs * 8), 256, 0, s>>>(
            pairs, npairs, rank, n, vb, keys, capacity, cursor, oplan, hist, outdeg);
        TC_LAUNCHED();
    }
    const uint64_t m = kept;
    TC_CHECK(graph_alloc(out, m, n, s));
    if (bucket) {
        TC_CHECK(bucket_csr_dev(keys, m, n, vb, outdeg, out, scratch + 1, s, deg_by_rank));
        TC_CUDA(cudaMemsetAsync(out->dst + m, 0, 8 * sizeof(uint32_t), s));
    } else {
        TC_CHECK(dalloc_t(&alt, m ? m : 1, s));
        TC_CHECK(radix_sort(keys, alt, nullptr, nullptr, m, plan, hist, kOutSoA, out->src, out->dst, vb,
                            nullptr, nullptr, s));
        TC_CUDA(cudaMemsetAsync(out->dst + m, 0, 8 * sizeof(uint32_t), s));
        TC_CHECK(build_node_array_dev(out->src, m, n, out->off, out->off32, scratch + 1, s));
    }
    TC_CHECK(build_hubstart_dev(out, s));
    if (deg_by_rank) {
        if (!out->vix_ready) TC_CHECK(vin_capacity_dev(out, deg_by_rank, s));
        dfree(deg_by_rank, s);
    }
    TC_CUDA(cudaMemcpyAsync(&out->max_out, scratch + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    if (id_of_rank && n) {  // the inverse of the relabelling (lazy reference-id CSR)
        k_invert_perm<<<grid_for(n, 256, kSMs * 8), 256, 0, s>>>(rank, n, id_of_rank);
        TC_LAUNCHED();
    }
    dfree(deg, s);
    dfree(rank, s);
    dfree(hist, s);
    dfree(cursor, s);
    dfree(keys, s);
    dfree(alt, s);
    dfree(scratch, s);
    TC_CUDA(cudaStreamSynchronize(s));
    return 0;
}

// The reference-id CSR of a rank-space graph from preprocess_rank_dev (its exact relabelling:
// same orientation, ranks replaced by ids): keys (id(u) << vb) | id(v), radix sorted, node
// array -- the arrays reference preprocess.py:74-84 returns, built only when asked for.
int derank_dev(const DeviceGraph &r, const uint32_t *id_of_rank, DeviceGraph *out, cudaStream_t s) {
    const uint64_t n = r.n, m = r.m;
    const int vb = n > 1 ? bits_for(n - 1) : 1;
    const RadixPlan plan = make_radix_plan(2 * vb);
    uint32_t *hist = nullptr, *scratch = nullptr;
    uint64_t *keys = nullptr, *alt = nullptr;
    TC_CHECK(dalloc_t(&scratch, 4, s));
    TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
    TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(scratch, 0, 4 * sizeof(uint32_t), s));
    TC_CHECK(dalloc_t(&keys, m ? m : 1, s));
    TC_CHECK(dalloc_t(&alt, m ? m : 1, s));
    if (m) {
        // scratch[2]: the ordering flag of k_relabel_keys, meaningless here (ids are unordered)
        k_relabel_keys<<<grid_for(m, 256, kSMs * 16), 256, 0, s>>>(r.src, r.dst, m, id_of_rank, vb, keys,
                                                                     scratch + 2);
        TC_LAUNCHED();
    }
    TC_CHECK(radix_histogram(keys, m, plan, hist, s));
    TC_CHECK(graph_alloc(out, m, n, s));
    TC_CHECK(radix_sort(keys, alt, nullptr, nullptr, m, plan, hist, kOutSoA, out->src, out->dst, vb,
                        nullptr, nullptr, s));
    TC_CUDA(cudaMemsetAsync(out->dst + m, 0, 8 * sizeof(uint32_t), s));
    TC_CHECK(build_node_array_dev(out->src, m, n, out->off, out->off32, scratch + 1, s));
    TC_CUDA(cudaMemcpyAsync(&out->max_out, scratch + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(hist, s);
    dfree(scratch, s);
    dfree(keys, s);
    dfree(alt, s);
    return 0;
}

int relabel_dev(const DeviceGraph &g, DeviceGraph *out, cudaStream_t s) {
    if (g.n >= (1ull << 32) || g.m >= (1ull << 32)) {
        set_error("rank-space relabelling needs num_vertices < 2^32 and m < 2^32");
        return -1;
    }
    const uint64_t n = g.n, m = g.m;
    const int vb = n > 1 ? bits_for(n - 1) : 1;
    const RadixPlan plan = make_radix_plan(2 * vb);
    uint32_t *deg = nullptr, *rank = nullptr, *hist = nullptr, *scratch = nullptr;
    TC_CHECK(dalloc_t(&deg, n ? n : 1, s));
    TC_CHECK(dalloc_t(&rank, n ? n : 1, s));
    TC_CHECK(dalloc_t(&scratch, 4, s));
    TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
    TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(scratch, 0, 4 * sizeof(uint32_t), s));
    if (n) {
        k_outdeg<<<grid_for(n, 256, kSMs * 16), 256, 0, s>>>(g.off, n, deg);
        TC_LAUNCHED();
    }
    if (m) {
        k_indeg<<<grid_for(m, 256, kSMs * 16), 256, 0, s>>>(g.dst, m, deg);
        TC_LAUNCHED();
    }
    TC_CHECK(compute_ranks(deg, n, rank, s));
    uint64_t *keys = nullptr, *alt = nullptr;
    TC_CHECK(dalloc_t(&keys, m ? m : 1, s));
    TC_CHECK(dalloc_t(&alt, m ? m : 1, s));
    if (m) {
        k_relabel_keys<<<grid_for(m, 256, kSMs * 16), 256, 0, s>>>(g.src, g.dst, m, rank, vb, keys,
                                                                     scratch + 2);
        TC_LAUNCHED();
        uint32_t bad = 0;
        TC_CUDA(cudaMemcpyAsync(&bad, scratch + 2, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
        if (bad) {  // not oriented by (out + in degree, id): the caller counts in original ids
            dfree(deg, s);
            dfree(rank, s);
            dfree(hist, s);
            dfree(scratch, s);
            dfree(keys, s);
            dfree(alt, s);
            return kNotRankOrientable;
        }
    }
    TC_CHECK(radix_histogram(keys, m, plan, hist, s));
    TC_CHECK(graph_alloc(out, m, n, s));
    TC_CHECK(radix_sort(keys, alt, nullptr, nullptr, m, plan, hist, kOutSoA, out->src, out->dst, vb,
                        nullptr, nullptr, s));
    TC_CUDA(cudaMemsetAsync(out->dst + m, 0, 8 * sizeof(uint32_t), s));
    TC_CHECK(build_node_array_dev(out->src, m, n, out->off, out->off32, scratch + 1, s));
    TC_CHECK(build_hubstart_dev(out, s));
    TC_CUDA(cudaMemcpyAsync(&out->max_out, scratch + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(deg, s);
    dfree(rank, s);
    dfree(hist, s);
    dfree(scratch, s);
    dfree(keys, s);
    dfree(alt, s);
    return 0;
}

// ---- distributed preprocessing -----------------------------------
// Each rank holds a shard of the pairs.  Global degrees = sum of the shards' first-column
// histograms (all-reduce); ranks follow identically on every rank; each rank orients and
// relabels its shard, sorts it, and ships every key to the rank owning its source range
// (all-to-all); the owner sorts what it received into its slice of edge_dst; slices are
// then all-gathered and every rank finalises the same count-ready CSR.
namespace {

__global__ void __launch_bounds__(256) k_key_src_hist(const uint64_t *__restrict__ keys, uint64_t k,
                                                      int vb, uint32_t *__restrict__ cnt) {
    const unsigned lane = lane_id();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < k;
         base += stride) {
        const uint64_t i = base + lane;
        const bool ok = i < k;
        const uint32_t u = ok ? (uint32_t)(keys[i] >> vb) : 0xffffffffu;
        const unsigned peers = __match_any_sync(TC_FULL_MASK, u);
        if (ok && (int)lane == __ffs(peers) - 1) atomicAdd(cnt + u, __popc(peers));
    }
}

// cuts[r] = first rank u with off[u] >= r * m / parts (r = 0..parts; cuts[parts] = n)
__global__ void k_edge_cuts(const int64_t *__restrict__ off, uint64_t n, int parts,
                            int64_t *__restrict__ cuts, int64_t *__restrict__ ecuts) {
    const int r = threadIdx.x;
    if (r > parts) return;
    const int64_t m = off[n];
    if (r == parts) {
        cuts[r] = (int64_t)n;
        ecuts[r] = m;
        return;
    }
    const int64_t want = (int64_t)((__int128)m * r / parts);
    uint64_t a = 0, len = n;  // first u in [0, n) with off[u] >= want
    while (len > 0) {
        const uint64_t h = len >> 1;
        if (off[a + h] < want) { a += h + 1; len -= h + 1; }
        else len = h;
    }
    cuts[r] = (int64_t)a;
    ecuts[r] = off[a];
}

// counts[r] = #keys with source rank in [cuts[r], cuts[r+1]) (keys sorted)
__global__ void k_key_split(const uint64_t *__restrict__ keys, uint64_t k, int vb,
                            const int64_t *__restrict__ cuts, int parts, int64_t *__restrict__ counts) {
    __shared__ uint64_t pos[65];
    const int r = threadIdx.x;
    if (r <= parts) {
        const uint64_t want = (uint64_t)cuts[r] << vb;
        uint64_t a = 0, len = k;
        while (len > 0) {
            const uint64_t h = len >> 1;
            if (keys[a + h] < want) { a += h + 1; len -= h + 1; }
            else len = h;
        }
        pos[r] = r == parts ? k : a;
    }
    __syncthreads();
    if (r < parts) counts[r] = (int64_t)(pos[r + 1] - pos[r]);
}

}  // namespace

int dist_degrees_dev(const uint32_t *pairs_u32, uint64_t npairs, uint64_t n, uint32_t *deg,
                     cudaStream_t s) {
    const uint2 *pairs = reinterpret_cast<const uint2 *>(pairs_u32);
    uint32_t *bad_d = nullptr;
    TC_CHECK(dalloc_t(&bad_d, 1, s));
    TC_CUDA(cudaMemsetAsync(bad_d, 0, sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(deg, 0, (n ? n : 1) * sizeof(uint32_t), s));
    if (npairs) {
        k_degree_hist<<<grid_for(npairs, 256 * kDegPP, kSMs * 8), 256, 0, s>>>(pairs, npairs, deg, n, bad_d);
        TC_LAUNCHED();
    }
    uint32_t bad = 0;
    TC_CUDA(cudaMemcpyAsync(&bad, bad_d, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(bad_d, s);
    if (bad) {
        set_error("edge array holds a vertex id >= num_vertices");
        return -1;
    }
    return 0;
}

int dist_orient_dev(const uint32_t *pairs_u32, uint64_t npairs, uint64_t n, const uint32_t *deg,
                    uint64_t **keys_out, uint64_t *nkeys, uint32_t *outdeg, cudaStream_t s) {
    const uint2 *pairs = reinterpret_cast<const uint2 *>(pairs_u32);
    *keys_out = nullptr;
    *nkeys = 0;
    if (n >= (1ull << 32)) {
        set_error("num_vertices must be < 2^32 on the device path");
        return -1;
    }
    const int vb = n > 1 ? bits_for(n - 1) : 1;
    const RadixPlan plan = make_radix_plan(2 * vb);
    uint32_t *rank = nullptr, *hist = nullptr;
    unsigned long long *cursor = nullptr;
    TC_CHECK(dalloc_t(&rank, n ? n : 1, s));
    TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
    TC_CHECK(dalloc_t(&cursor, 1, s));
    TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), s));
    TC_CUDA(cudaMemsetAsync(outdeg, 0, (n ? n : 1) * sizeof(uint32_t), s));
    TC_CHECK(compute_ranks(deg, n, rank, s));
    // a shard of a symmetric array keeps about half its pairs, but not exactly: size for all
    uint64_t capacity = npairs ? npairs : 1;
    uint64_t *keys = nullptr, *alt = nullptr;
    TC_CHECK(dalloc_t(&keys, capacity, s, true));
    if (npairs) {
        k_orient<true><<<grid_for(npairs, 256 * kPP, kSMs * 8), 256, 0, s>>>(
            pairs, npairs, rank, n, vb, keys, capacity, cursor, plan, hist);
        TC_LAUNCHED();
    }
    unsigned long long kept = 0;
    TC_CUDA(cudaMemcpyAsync(&kept, cursor, sizeof(kept), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    TC_CHECK(dalloc_t(&alt, kept ? kept : 1, s, true));
    uint64_t *sorted = keys;
    TC_CHECK(radix_sort(keys, alt, nullptr, nullptr, kept, plan, hist, kOutKeys, nullptr, nullptr, 0,
                        &sorted, nullptr, s));
    if (kept) {
        k_key_src_hist<<<grid_for(kept, 256, kSMs * 16), 256, 0, s>>>(sorted, kept, vb, outdeg);
        TC_LAUNCHED();
    }
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(sorted == keys ? alt : keys, s);
    dfree(rank, s);
    dfree(hist, s);
    dfree(cursor, s);
    *keys_out = sorted;
    *nkeys = kept;
    return 0;
}

int dist_layout_dev(DeviceGraph *g, const uint32_t *outdeg, int parts, int64_t *cuts,
                    int64_t *ecuts, cudaStream_t s) {
    if (parts < 1 || parts > 64) {
        set_error("parts must be in 1..64");
        return -1;
    }
    TC_CHECK(exclusive_scan_dev(outdeg, g->n, g->off, s));
    const int64_t mm = (int64_t)g->m;
    TC_CUDA(cudaMemcpyAsync(g->off + g->n, &mm, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    int64_t *d = nullptr;
    TC_CHECK(dalloc_t(&d, 2 * (parts + 1), s));
    k_edge_cuts<<<1, 96, 0, s>>>(g->off, g->n, parts, d, d + parts + 1);
    TC_LAUNCHED();
    TC_CUDA(cudaMemcpyAsync(cuts, d, (parts + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaMemcpyAsync(ecuts, d + parts + 1, (parts + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(d, s);
    if (ecuts[parts] != mm) {
        set_error("out-degrees do not sum to the graph's edge count");
        return -1;
    }
    return 0;
}

int dist_split_dev(const uint64_t *keys, uint64_t nkeys, uint64_t n, const int64_t *cuts, int parts,
                   int64_t *counts, cudaStream_t s) {
    if (parts < 1 || parts > 64) {
        set_error("parts must be in 1..64");
        return -1;
    }
    const int vb = n > 1 ? bits_for(n - 1) : 1;
    int64_t *d = nullptr;
    TC_CHECK(dalloc_t(&d, 2 * (parts + 1), s));
    TC_CUDA(cudaMemcpyAsync(d, cuts, (parts + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    k_key_split<<<1, 96, 0, s>>>(keys, nkeys, vb, d, parts, d + parts + 1);
    TC_LAUNCHED();
    TC_CUDA(cudaMemcpyAsync(counts, d + parts + 1, parts * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(d, s);
    return 0;
}

int dist_place_dev(DeviceGraph *g, uint64_t *keys, uint64_t nkeys, uint64_t pos, cudaStream_t s) {
    if (pos + nkeys > g->m) {
        set_error("placed slice exceeds the graph's edge count");
        return -1;
    }
    if (nkeys == 0) return 0;
    const int vb = g->n > 1 ? bits_for(g->n - 1) : 1;
    const RadixPlan plan = make_radix_plan(2 * vb);
    uint64_t *alt = nullptr;
    uint32_t *hist = nullptr;
    TC_CHECK(dalloc_t(&alt, nkeys, s));
    TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
    TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
    TC_CHECK(radix_histogram(keys, nkeys, plan, hist, s));
    // src lands in the graph's own edge_src (rebuilt by finalize anyway)
    TC_CHECK(radix_sort(keys, alt, nullptr, nullptr, nkeys, plan, hist, kOutSoA, g->src + pos,
                        g->dst + pos, vb, nullptr, nullptr, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(alt, s);
    dfree(hist, s);
    return 0;
}

}  // namespace tc
