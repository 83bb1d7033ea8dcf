// tc_count.cu -- exact triangle counting over the oriented CSR (the hot path).
//
// Reference: count.py:63-99 (_count_strided, a per-edge two-pointer merge of adj(u)
// and adj(v)), count.py:162-204 (edge-range / pool drivers).  The result is
//     sum over oriented edges (u, v) in [lo, hi) of |adj(u) ∩ adj(v)|,
// which is what this file computes, organised around the SOURCE vertex u so that
// adj(u) is loaded once and reused by all of u's out-edges:
//
//  * light sources (1 <= d+(u) <= 32): one CTA per window of 512 consecutive edges.
//    The source lists of the window are staged in shared memory; all items of all
//    edges (u, v) -- every element w of every adj(v) -- are flattened across the CTA
//    (load-balanced, each lane keeps 8 independent coalesced loads in flight) and w is
//    tested against adj(u) by a <= 5-step binary search in shared memory.
//  * heavy sources (d+(u) > 32): one CTA per (u, chunk of <= 1024 edges).  adj(u) is
//    staged into a shared-memory open-addressing hash table (load <= 1/2), the items of
//    a 512-edge window are split evenly across the 16 warps, and each w costs one
//    coalesced load plus ~1.5 shared-memory probes.  For d+(u) > 16384 the table would
//    not fit and adj(u) is staged as a sorted array probed by binary search.
//  * k_count_merge_thread: the paper's thread-per-edge merge kept
//    as an A/B baseline and as an independent device-side check.
//
// Counts are u32 per lane per item batch, u64 per thread, one u64 atomic per CTA.
#include "tc_common.cuh"
#include "tc_internal.h"

namespace tc {

namespace {

constexpr uint32_t kEmpty = 0xffffffffu;
constexpr int kLightMax = 32;
constexpr int kHeavyThreads = 512;
constexpr int kHeavyWarps = kHeavyThreads / 32;
constexpr int kWin = 512;       // edges staged per window (== kHeavyThreads)
constexpr int kChunk = 1024;    // edges per heavy task
constexpr int kClasses = 4;
// Heavy classes by d+(u): hash-table capacity (entries) per class; 0 = sorted-array mode.
// Tables are sized 8 d (load <= 1/8) up to the class capacity.
constexpr uint32_t kClassMax[kClasses] = {512, 2048, 16384, 0xffffffffu};
constexpr uint32_t kClassCap[kClasses] = {4096, 16384, 49152, 0};

struct RangeDev {
    uint64_t lo, hi, m;
    uint32_t u_lo, u_hi;
};

constexpr int kUnroll = 8;  // independent item loads in flight per lane

// Fibonacci hash, range-reduced to [0, T) with a multiply-high (any T, not only 2^k).
__device__ __forceinline__ uint32_t hash_slot(uint32_t w, uint32_t T) {
    return __umulhi(w * 0x9E3779B1u, T);
}

template <typename T>
__device__ __forceinline__ void block_add_total(T acc, unsigned long long *total) {
    __shared__ unsigned long long s_red[32];
    unsigned long long x = warp_sum<unsigned long long>((unsigned long long)acc);
    if (lane_id() == 0) s_red[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned long long y = threadIdx.x < (blockDim.x >> 5) ? s_red[threadIdx.x] : 0ull;
        y = warp_sum(y);
        if (threadIdx.x == 0 && y) atomicAdd(total, y);
    }
}

__global__ void k_range_init(const uint32_t *__restrict__ src, uint64_t lo, uint64_t hi,
                             uint64_t m, RangeDev *__restrict__ rg) {
    rg->lo = lo;
    rg->hi = hi;
    rg->m = m;
    rg->u_lo = hi > lo ? src[lo] : 0u;
    rg->u_hi = hi > lo ? src[hi - 1] + 1u : 0u;
}

// ----------------------------------------------------------------- window ---
// Edges whose source is light (d+(u) <= 32), in windows of kWin consecutive edges.
// Every light source list that owns an edge of the window lies inside
// dst[ws-31, we+31), so the window stages that slice in shared memory once; each item
// w of each adj(v) is then tested against its source list by a <= 5-step binary
// search in shared memory.  Items of the window are split evenly over the warps and
// each lane keeps kUnroll independent loads in flight.
constexpr int kStage = kWin + 2 * kLightMax;

template <typename OffT>
__global__ void __launch_bounds__(kHeavyThreads)
    k_count_window(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                   const OffT *__restrict__ off, const RangeDev *__restrict__ rg,
                   unsigned *__restrict__ next, unsigned long long *__restrict__ total) {
    __shared__ uint32_t s_stage[kStage];
    __shared__ OffT s_eb[kWin];
    __shared__ uint32_t s_st[kWin + 4];
    __shared__ uint32_t s_ua[kWin];  // (list start in s_stage) | (d+(u) << 16)
    __shared__ uint32_t s_scan[32];
    __shared__ unsigned s_win;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const uint64_t lo = rg->lo, hi = rg->hi, m = rg->m;
    const uint64_t nwin = (hi - lo + kWin - 1) / kWin;
    unsigned long long acc = 0;
    for (;;) {
        if (threadIdx.x == 0) s_win = atomicAdd(next, 1u);
        __syncthreads();
        const uint64_t wi = s_win;
        if (wi >= nwin) break;
        const uint64_t ws = lo + wi * kWin;
        const uint64_t we = ws + kWin < hi ? ws + kWin : hi;
        const uint64_t sb = ws >= (uint64_t)(kLightMax - 1) ? ws - (kLightMax - 1) : 0;
        const uint64_t se = we + (kLightMax - 1) < m ? we + (kLightMax - 1) : m;
        for (uint32_t i = threadIdx.x; i < (uint32_t)(se - sb); i += kHeavyThreads)
            s_stage[i] = __ldg(dst + sb + i);
        uint32_t len = 0, ua = 0;
        OffT vs = 0;
        if (threadIdx.x < (uint32_t)(we - ws)) {
            const uint64_t e = ws + threadIdx.x;
            const uint32_t u = __ldg(src + e);
            const OffT su = __ldg(off + u);
            const uint32_t du = (uint32_t)(__ldg(off + u + 1) - su);
            if (du <= (uint32_t)kLightMax) {
                const uint32_t v = __ldg(dst + e);
                vs = __ldg(off + v);
                len = (uint32_t)(__ldg(off + v + 1) - vs);
                ua = (uint32_t)((uint64_t)su - sb) | (du << 16);
            }
        }
        uint32_t tot;
        const uint32_t st = block_exclusive_scan<uint32_t>(len, s_scan, &tot);
        if (threadIdx.x < kWin) {
            s_eb[threadIdx.x] = vs - (OffT)st;
            s_st[threadIdx.x] = st;
            s_ua[threadIdx.x] = ua;
        }
        if (threadIdx.x == 0) s_st[kWin] = tot;
        __syncthreads();
        const uint32_t i0 = (uint32_t)((uint64_t)tot * warp / kHeavyWarps);
        const uint32_t i1 = (uint32_t)((uint64_t)tot * (warp + 1) / kHeavyWarps);
        if (i0 < i1) {
            uint32_t k = 0;
            {
                const uint32_t item = i0 + lane;
                uint32_t a = 0, b = kWin;  // largest k with s_st[k] <= item
                while (b - a > 1) {
                    const uint32_t mid = (a + b) >> 1;
                    if (s_st[mid] <= item) a = mid; else b = mid;
                }
                k = a;
            }
            uint32_t nextb = s_st[k + 1];
            OffT eb = s_eb[k];
            uint32_t ua = s_ua[k];
            uint32_t found = 0;
            for (uint32_t base = i0; base < i1; base += 32 * kUnroll) {
                uint32_t w[kUnroll], la[kUnroll];
#pragma unroll
                for (int j = 0; j < kUnroll; ++j) {
                    const uint32_t item = base + j * 32 + lane;
                    w[j] = 0;
                    la[j] = 0;  // empty list: never matches
                    if (item < i1) {
                        if (item >= nextb) {
                            do { nextb = s_st[++k + 1]; } while (item >= nextb);
                            eb = s_eb[k];
                            ua = s_ua[k];
                        }
                        w[j] = __ldg(dst + (OffT)(eb + (OffT)item));
                        la[j] = ua;
                    }
                }
#pragma unroll
                for (int j = 0; j < kUnroll; ++j) {
                    uint32_t a = la[j] & 0xffffu, n = la[j] >> 16;
                    const uint32_t end = a + n;
                    while (n > 0) {
                        const uint32_t half = n >> 1;
                        if (s_stage[a + half] < w[j]) { a += half + 1; n -= half + 1; }
                        else n = half;
                    }
                    found += (a < end && s_stage[a] == w[j]) ? 1u : 0u;
                }
            }
            acc += found;
        }
        __syncthreads();
    }
    block_add_total(acc, total);
}

// ------------------------------------------------------------------ heavy ---
template <typename OffT>
__global__ void k_classify(const OffT *__restrict__ off, const RangeDev *__restrict__ rg,
                           uint2 *__restrict__ t0, uint2 *__restrict__ t1, uint2 *__restrict__ t2,
                           uint2 *__restrict__ t3, unsigned *__restrict__ ntasks) {
    const uint64_t lo = rg->lo, hi = rg->hi;
    const uint32_t u_lo = rg->u_lo, u_hi = rg->u_hi;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t u = u_lo + blockIdx.x * blockDim.x + threadIdx.x; u < u_hi; u += stride) {
        const OffT s = off[u], e = off[u + 1];
        const uint32_t d = (uint32_t)(e - s);
        if (d <= (uint32_t)kLightMax) continue;
        const uint64_t es = (uint64_t)s > lo ? (uint64_t)s : lo;
        const uint64_t ee = (uint64_t)e < hi ? (uint64_t)e : hi;
        if (es >= ee) continue;
        const int cls = d <= kClassMax[0] ? 0 : d <= kClassMax[1] ? 1 : d <= kClassMax[2] ? 2 : 3;
        const uint32_t chunks = (uint32_t)((ee - es + kChunk - 1) / kChunk);
        const unsigned slot = atomicAdd(ntasks + cls, chunks);
        uint2 *t = cls == 0 ? t0 : cls == 1 ? t1 : cls == 2 ? t2 : t3;
        for (uint32_t c = 0; c < chunks; ++c) t[slot + c] = make_uint2(u, c);
    }
}

// MODE 0: adj(u) in a shared-memory hash table; MODE 1: adj(u) as a sorted smem array.
// Lane state caches the current edge: its item range end (nextb) and the dst index
// base (eb = start of adj(v) - first item of v), so an item costs a compare, an add
// and a load unless it crosses into the next edge.
template <typename OffT, int MODE>
__global__ void __launch_bounds__(kHeavyThreads)
    k_count_heavy(const uint32_t *__restrict__ dst, const OffT *__restrict__ off,
                  const RangeDev *__restrict__ rg, const uint2 *__restrict__ tasks,
                  const unsigned *__restrict__ ntasks, unsigned *__restrict__ next, uint32_t tcap,
                  unsigned long long *__restrict__ total) {
    extern __shared__ __align__(16) unsigned char smem[];
    OffT *s_eb = reinterpret_cast<OffT *>(smem);
    uint32_t *s_st = reinterpret_cast<uint32_t *>(s_eb + kWin);
    uint32_t *table = s_st + kWin + 4;
    __shared__ uint32_t s_scan[32];
    __shared__ unsigned s_task;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const uint64_t lo = rg->lo, hi = rg->hi;
    const unsigned nt = *ntasks;
    unsigned long long acc = 0;
    for (;;) {
        if (threadIdx.x == 0) s_task = atomicAdd(next, 1u);
        __syncthreads();
        const unsigned t = s_task;
        if (t >= nt) break;
        const uint2 task = tasks[t];
        const uint32_t u = task.x;
        const OffT s = off[u], e = off[u + 1];
        const uint32_t d = (uint32_t)(e - s);
        uint64_t es = (uint64_t)s > lo ? (uint64_t)s : lo;
        uint64_t ee = (uint64_t)e < hi ? (uint64_t)e : hi;
        es += (uint64_t)task.y * kChunk;
        ee = ee < es + kChunk ? ee : es + kChunk;

        uint32_t T = 0;
        if (MODE == 0) {
            T = 8 * d < tcap ? 8 * d : tcap;
            for (uint32_t i = threadIdx.x; i < T; i += kHeavyThreads) table[i] = kEmpty;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < d; i += kHeavyThreads) {
                const uint32_t w = __ldg(dst + s + i);
                uint32_t h = hash_slot(w, T);
                for (;;) {
                    const uint32_t prev = atomicCAS(table + h, kEmpty, w);
                    if (prev == kEmpty || prev == w) break;
                    h = h + 1 == T ? 0 : h + 1;
                }
            }
        } else {
            for (uint32_t i = threadIdx.x; i < d; i += kHeavyThreads) table[i] = __ldg(dst + s + i);
        }
        __syncthreads();

        for (uint64_t ws = es; ws < ee; ws += kWin) {
            const uint32_t nwin = (uint32_t)(ee - ws < (uint64_t)kWin ? ee - ws : (uint64_t)kWin);
            uint32_t len = 0;
            OffT vs = 0;
            if (threadIdx.x < nwin) {
                const uint32_t v = __ldg(dst + ws + threadIdx.x);
                vs = __ldg(off + v);
                len = (uint32_t)(__ldg(off + v + 1) - vs);
            }
            uint32_t tot;
            const uint32_t st = block_exclusive_scan<uint32_t>(len, s_scan, &tot);
            if (threadIdx.x < nwin) {
                s_eb[threadIdx.x] = vs - (OffT)st;
                s_st[threadIdx.x] = st;
            }
            if (threadIdx.x == 0) s_st[nwin] = tot;
            __syncthreads();
            const uint32_t i0 = (uint32_t)((uint64_t)tot * warp / kHeavyWarps);
            const uint32_t i1 = (uint32_t)((uint64_t)tot * (warp + 1) / kHeavyWarps);
            if (i0 < i1) {
                uint32_t k = 0;
                {
                    const uint32_t item = i0 + lane;
                    uint32_t a = 0, b = nwin;  // largest k < nwin with s_st[k] <= item
                    while (b - a > 1) {
                        const uint32_t mid = (a + b) >> 1;
                        if (s_st[mid] <= item) a = mid; else b = mid;
                    }
                    k = a;
                }
                uint32_t nextb = s_st[k + 1];
                OffT eb = s_eb[k];
                uint32_t found = 0;
                for (uint32_t base = i0; base < i1; base += 32 * kUnroll) {
                    uint32_t w[kUnroll];
#pragma unroll
                    for (int j = 0; j < kUnroll; ++j) {
                        const uint32_t it = base + j * 32 + lane;
                        w[j] = kEmpty;
                        if (it < i1) {
                            if (it >= nextb) {
                                do { nextb = s_st[++k + 1]; } while (it >= nextb);
                                eb = s_eb[k];
                            }
                            w[j] = __ldg(dst + (OffT)(eb + (OffT)it));
                        }
                    }
#pragma unroll
                    for (int j = 0; j < kUnroll; ++j) {
                        if (MODE == 0) {
                            uint32_t h = hash_slot(w[j], T);
                            uint32_t x = table[h];
                            if (x != w[j] && x != kEmpty) {
                                do {
                                    h = h + 1 == T ? 0 : h + 1;
                                    x = table[h];
                                } while (x != w[j] && x != kEmpty);
                            }
                            found += (x == w[j] && w[j] != kEmpty) ? 1u : 0u;
                        } else {
                            if (w[j] == kEmpty) continue;
                            uint32_t a = 0, n = d;
                            while (n > 0) {
                                const uint32_t half = n >> 1;
                                if (table[a + half] < w[j]) { a += half + 1; n -= half + 1; }
                                else n = half;
                            }
                            found += (a < d && table[a] == w[j]) ? 1u : 0u;
                        }
                    }
                }
                acc += found;
            }
            __syncthreads();
        }
    }
    block_add_total(acc, total);
}

// ------------------------------------------------------- paper baseline ---
// Thread per oriented edge, grid-stride, bounds checked like the
// reference (count.py:69-98).
template <typename OffT>
__global__ void __launch_bounds__(256) k_count_merge_thread(const uint32_t *__restrict__ src,
                                                            const uint32_t *__restrict__ dst,
                                                            const OffT *__restrict__ off,
                                                            uint64_t lo, uint64_t hi,
                                                            unsigned long long *__restrict__ total) {
    unsigned long long acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += stride) {
        const uint32_t u = src[i], v = dst[i];
        OffT ui = off[u], ue = off[u + 1], vi = off[v], ve = off[v + 1];
        if (ui == ue || vi == ve) continue;
        uint32_t a = dst[ui], b = dst[vi];
        for (;;) {
            if (a < b) {
                if (++ui == ue) break;
                a = dst[ui];
            } else if (b < a) {
                if (++vi == ve) break;
                b = dst[vi];
            } else {
                ++acc;
                ++ui;
                ++vi;
                if (ui == ue || vi == ve) break;
                a = dst[ui];
                b = dst[vi];
            }
        }
    }
    block_add_total(acc, total);
}

__global__ void k_intersect(const uint32_t *__restrict__ dst, const int64_t *__restrict__ off,
                            uint32_t u, uint32_t v, unsigned long long *__restrict__ out) {
    int64_t ui = off[u], ue = off[u + 1], vi = off[v], ve = off[v + 1];
    unsigned long long c = 0;
    while (ui < ue && vi < ve) {
        const uint32_t a = dst[ui], b = dst[vi];
        if (a < b) ++ui;
        else if (b < a) ++vi;
        else { ++c; ++ui; ++vi; }
    }
    *out = c;
}

// Per-tile sum of the merge work d+(src_i) + d+(dst_i) + overhead (for shard bounds).
template <typename OffT>
__global__ void __launch_bounds__(256) k_tile_work(const uint32_t *__restrict__ src,
                                                   const uint32_t *__restrict__ dst,
                                                   const OffT *__restrict__ off, uint64_t m,
                                                   uint64_t tile, uint32_t overhead,
                                                   unsigned long long *__restrict__ sums) {
    const uint64_t b = (uint64_t)blockIdx.x * tile;
    const uint64_t e = b + tile < m ? b + tile : m;
    unsigned long long acc = 0;
    for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        const uint32_t u = src[i], v = dst[i];
        acc += (unsigned long long)(off[u + 1] - off[u]) + (unsigned long long)(off[v + 1] - off[v]) +
               overhead;
    }
    __shared__ unsigned long long s_red[32];
    acc = warp_sum(acc);
    if (lane_id() == 0) s_red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned long long y = threadIdx.x < (blockDim.x >> 5) ? s_red[threadIdx.x] : 0ull;
        y = warp_sum(y);
        if (threadIdx.x == 0) sums[blockIdx.x] = y;
    }
}

size_t heavy_smem(int cls, uint32_t max_out, bool off64) {
    size_t b = (size_t)kWin * (off64 ? 8 : 4) + (kWin + 4) * 4;
    if (kClassCap[cls] > 0) b += (size_t)4 * kClassCap[cls];
    else b += (size_t)4 * max_out;
    return b;
}

template <typename OffT>
int count_impl(const DeviceGraph &g, const OffT *off, uint64_t lo, uint64_t hi,
               unsigned long long *d_total, cudaStream_t s, CountStats *stats) {
    const bool off64 = sizeof(OffT) == 8;
    RangeDev *rg = nullptr;
    unsigned *counters = nullptr;  // [0..3] ntasks per class, [4..7] queue heads, [8] windows
    TC_CHECK(dalloc_t(&rg, 1, s));
    TC_CHECK(dalloc_t(&counters, 2 * kClasses + 1, s));
    TC_CUDA(cudaMemsetAsync(counters, 0, (2 * kClasses + 1) * sizeof(unsigned), s));
    k_range_init<<<1, 1, 0, s>>>(g.src, lo, hi, g.m, rg);
    TC_LAUNCHED();

    // Task capacity per class: every vertex in class c has > lower_c edges.
    const uint32_t lower[kClasses] = {(uint32_t)kLightMax, kClassMax[0], kClassMax[1], kClassMax[2]};
    const uint64_t span = hi - lo;
    uint2 *tasks[kClasses];
    for (int c = 0; c < kClasses; ++c) {
        uint64_t cap = 0;
        if (g.max_out > lower[c]) cap = span / (lower[c] + 1) + span / kChunk + 2;
        TC_CHECK(dalloc_t(&tasks[c], cap ? cap : 1, s));
    }
    cudaEvent_t ev[4];
    for (auto &e : ev) TC_CUDA(cudaEventCreate(&e));
    TC_CUDA(cudaEventRecord(ev[0], s));
    const uint32_t nverts = (uint32_t)(g.n < 0xffffffffull ? g.n : 0xffffffffull);
    if (g.max_out > (uint32_t)kLightMax) {
        k_classify<OffT><<<grid_for(nverts, 256, kSMs * 8), 256, 0, s>>>(off, rg, tasks[0], tasks[1],
                                                                         tasks[2], tasks[3], counters);
        TC_LAUNCHED();
    }
    TC_CUDA(cudaEventRecord(ev[1], s));
    // Heavy classes first (largest tasks first), then the light sweep.
    for (int c = kClasses - 1; c >= 0; --c) {
        if (g.max_out <= lower[c]) continue;
        const size_t sm = heavy_smem(c, g.max_out, off64);
        if (sm > 227 * 1024) {
            set_error("max out-degree too large for the shared-memory staging path");
            return -1;
        }
        int blocks_per_sm = 1;
        if (kClassCap[c] > 0) {
            auto kern = k_count_heavy<OffT, 0>;
            TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, kHeavyThreads, sm));
            if (blocks_per_sm < 1) blocks_per_sm = 1;
            kern<<<kSMs * blocks_per_sm, kHeavyThreads, sm, s>>>(g.dst, off, rg, tasks[c], counters + c,
                                                                counters + kClasses + c, kClassCap[c],
                                                                d_total);
        } else {
            auto kern = k_count_heavy<OffT, 1>;
            TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, kHeavyThreads, sm));
            if (blocks_per_sm < 1) blocks_per_sm = 1;
            kern<<<kSMs * blocks_per_sm, kHeavyThreads, sm, s>>>(g.dst, off, rg, tasks[c], counters + c,
                                                                counters + kClasses + c, 0, d_total);
        }
        TC_LAUNCHED();
    }
    TC_CUDA(cudaEventRecord(ev[2], s));
    k_count_window<OffT><<<kSMs * 4, kHeavyThreads, 0, s>>>(g.src, g.dst, off, rg,
                                                            counters + 2 * kClasses, d_total);
    TC_LAUNCHED();
    TC_CUDA(cudaEventRecord(ev[3], s));
    if (stats) {
        TC_CUDA(cudaEventSynchronize(ev[3]));
        cudaEventElapsedTime(&stats->classify_ms, ev[0], ev[1]);
        cudaEventElapsedTime(&stats->heavy_ms, ev[1], ev[2]);
        cudaEventElapsedTime(&stats->light_ms, ev[2], ev[3]);
        unsigned h[kClasses];
        TC_CUDA(cudaMemcpy(h, counters, sizeof(h), cudaMemcpyDeviceToHost));
        stats->heavy_tasks = (uint64_t)h[0] + h[1] + h[2] + h[3];
    }
    for (auto &e : ev) cudaEventDestroy(e);
    for (int c = 0; c < kClasses; ++c) dfree(tasks[c], s);
    dfree(rg, s);
    dfree(counters, s);
    return 0;
}

}  // namespace

int count_range_dev(const DeviceGraph &g, uint64_t lo, uint64_t hi, int algo,
                    unsigned long long *d_total, cudaStream_t s, CountStats *stats) {
    if (hi > g.m) hi = g.m;
    if (lo >= hi) return 0;
    if (algo == kAlgoMergeThread) {
        const uint64_t span = hi - lo;
        if (g.off32)
            k_count_merge_thread<uint32_t><<<grid_for(span, 256, kSMs * 16), 256, 0, s>>>(
                g.src, g.dst, g.off32, lo, hi, d_total);
        else
            k_count_merge_thread<int64_t><<<grid_for(span, 256, kSMs * 16), 256, 0, s>>>(
                g.src, g.dst, g.off, lo, hi, d_total);
        TC_LAUNCHED();
        return 0;
    }
    if (g.off32) return count_impl<uint32_t>(g, g.off32, lo, hi, d_total, s, stats);
    return count_impl<int64_t>(g, g.off, lo, hi, d_total, s, stats);
}

int intersect_dev(const DeviceGraph &g, uint32_t u, uint32_t v, uint64_t *out, cudaStream_t s) {
    unsigned long long *d = nullptr, h = 0;
    TC_CHECK(dalloc_t(&d, 1, s));
    k_intersect<<<1, 1, 0, s>>>(g.dst, g.off, u, v, d);
    TC_LAUNCHED();
    TC_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(d, s);
    *out = h;
    return 0;
}

namespace {
int tile_sums(const DeviceGraph &g, uint64_t tile, uint32_t overhead, unsigned long long **sums_out,
              uint64_t *ntiles_out, cudaStream_t s) {
    const uint64_t nt = (g.m + tile - 1) / tile;
    unsigned long long *sums = nullptr;
    TC_CHECK(dalloc_t(&sums, nt ? nt : 1, s));
    if (nt) {
        if (g.off32)
            k_tile_work<uint32_t><<<(unsigned)nt, 256, 0, s>>>(g.src, g.dst, g.off32, g.m, tile, overhead, sums);
        else
            k_tile_work<int64_t><<<(unsigned)nt, 256, 0, s>>>(g.src, g.dst, g.off, g.m, tile, overhead, sums);
        TC_LAUNCHED();
    }
    *sums_out = sums;
    *ntiles_out = nt;
    return 0;
}
}  // namespace

int work_bounds_dev(const DeviceGraph &g, int npools, int64_t *bounds, cudaStream_t s) {
    // Per-edge estimated work d+(u) + d+(v) + c; cuts at k*W/P with a
    // tile granularity fine enough that rounding is negligible against m/P.
    uint64_t tile = g.m / ((uint64_t)npools * 1024);
    if (tile < 1) tile = 1;
    if (tile > 4096) tile = 4096;
    unsigned long long *sums = nullptr;
    uint64_t nt = 0;
    TC_CHECK(tile_sums(g, tile, 8, &sums, &nt, s));
    std::string err;
    unsigned long long *h = (unsigned long long *)malloc((nt ? nt : 1) * sizeof(unsigned long long));
    if (!h) { set_error("host allocation failed"); return -3; }
    TC_CUDA(cudaMemcpyAsync(h, sums, nt * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(sums, s);
    unsigned long long W = 0;
    for (uint64_t i = 0; i < nt; ++i) W += h[i];
    bounds[0] = 0;
    unsigned long long run = 0;
    uint64_t t = 0;
    for (int p = 1; p < npools; ++p) {
        const long double target = (long double)W * p / npools;
        while (t < nt && (long double)(run + h[t]) <= target) run += h[t++];
        // cut at the tile edge closest to the target
        uint64_t cut = t;
        if (t < nt && (long double)(run + h[t]) - target < target - (long double)run) cut = t + 1;
        uint64_t b = cut * tile;
        if (b > g.m) b = g.m;
        if ((int64_t)b < bounds[p - 1]) b = (uint64_t)bounds[p - 1];
        bounds[p] = (int64_t)b;
    }
    bounds[npools] = (int64_t)g.m;
    free(h);
    return 0;
}

int merge_work_dev(const DeviceGraph &g, uint64_t *out, cudaStream_t s) {
    unsigned long long *sums = nullptr;
    uint64_t nt = 0;
    const uint64_t tile = 1 << 16;
    TC_CHECK(tile_sums(g, tile, 0, &sums, &nt, s));
    unsigned long long *h = (unsigned long long *)malloc((nt ? nt : 1) * sizeof(unsigned long long));
    if (!h) { set_error("host allocation failed"); return -3; }
    TC_CUDA(cudaMemcpyAsync(h, sums, nt * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(sums, s);
    unsigned long long W = 0;
    for (uint64_t i = 0; i < nt; ++i) W += h[i];
    free(h);
    *out = W;
    return 0;
}

}  // namespace tc
