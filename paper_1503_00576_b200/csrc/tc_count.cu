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
#include <stdlib.h>

#include "tc_common.cuh"
#include "tc_internal.h"
#include "tc_vsplit.cuh"

namespace tc {

namespace {

constexpr uint32_t kEmpty = 0xffffffffu;
constexpr int kLightMax = 32;
constexpr int kWinThreads = 256;  // window (light-source) CTA size == edges per window
constexpr int kChunk = 1024;    // edges per heavy task
constexpr int kClasses = 4;
// Heavy classes by d+(u): cuckoo tables of 4 d slots (load <= 1/4) up to the class
// capacity (in slots; class 2 reaches load 1/3 at d = 16384); 0 = sorted-array mode.  Small CTAs for the
// small classes so that many independent tasks overlap their setup phases on an SM.
constexpr uint32_t kClassMax[kClasses] = {512, 2048, 16384, 0xffffffffu};
constexpr uint32_t kClassCap[kClasses] = {2048, 8192, 49152, 0};
constexpr int kClassThreads[kClasses] = {128, 256, 512, 512};
constexpr uint32_t kWinSlots = 4 * kWinThreads + 256;  // window (source, w) cuckoo slots

struct RangeDev {
    uint64_t lo, hi, m;
    uint32_t u_lo, u_hi;
};

constexpr int kUnroll = 2;  // 16-byte chunks (4 items) in flight per lane per step

// ---------------------------------------------------------------- cuckoo ---
// Both count kernels probe a shared-memory cuckoo table: every key lives in one of two
// slots h1(key), h2(key), so a lookup is exactly two shared loads and two compares --
// no probe loop, no divergence.  Tables are built cooperatively with atomicExch
// (evict-and-reinsert, Alcantara et al. style); a build that exceeds the eviction bound
// is retried with the next hash seed.  Load factor <= 1/4 makes retries rare.
constexpr int kCuckooMaxKicks = 64;

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ unsigned long long lds64(uint32_t addr) {
    unsigned long long v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint32_t seed_mult(uint32_t seed, int which) {
    // odd multipliers derived from the seed (Fibonacci / murmur constants)
    return (which ? 0x85EBCA77u : 0x9E3779B1u) + 0x632BE5A6u * seed * 2u;
}

struct Cuckoo32 {
    uint32_t base;  // shared address of slot 0
    uint32_t T;     // slots
    uint32_t c1, c2;
    __device__ __forceinline__ uint32_t h1(uint32_t k) const { return __umulhi(k * c1, T); }
    __device__ __forceinline__ uint32_t h2(uint32_t k) const { return __umulhi(k * c2, T); }
    __device__ __forceinline__ bool contains(uint32_t w) const {
        const uint32_t x = lds32(base + 4 * h1(w));
        const uint32_t y = lds32(base + 4 * h2(w));
        return (x == w) | (y == w);
    }
};

// Membership in a sorted list (global memory): the fallback probe when a cuckoo table
// cannot be built within kCuckooSeeds seeds (pathological key sets) -- slower, never wrong,
// never a trap.
constexpr uint32_t kCuckooSeeds = 16;

__device__ __forceinline__ bool sorted_contains(const uint32_t *__restrict__ a, uint32_t n, uint32_t w) {
    uint32_t lo = 0, len = n;
    while (len > 0) {
        const uint32_t h = len >> 1;
        if (__ldg(a + lo + h) < w) { lo += h + 1; len -= h + 1; } else len = h;
    }
    return lo < n && __ldg(a + lo) == w;
}

// Insert `key` into a 32-bit cuckoo table; returns false after too many evictions.
__device__ __forceinline__ bool cuckoo_insert32(uint32_t *tab, const Cuckoo32 &c, uint32_t key) {
    uint32_t h = c.h1(key);
    for (int i = 0; i < kCuckooMaxKicks; ++i) {
        const uint32_t old = atomicExch(tab + h, key);
        if (old == kEmpty || old == key) return true;
        key = old;
        const uint32_t a = c.h1(key);
        h = (h == a) ? c.h2(key) : a;
    }
    return false;  // a key is left out: the caller rebuilds with another seed
}

// (source id, w) pairs for the window kernel: 64-bit keys.
struct Cuckoo64 {
    uint32_t base, T, c1, c2;
    __device__ __forceinline__ uint32_t mix(unsigned long long k, uint32_t c) const {
        return ((uint32_t)k * c) ^ ((uint32_t)(k >> 32) * 0xC2B2AE35u);
    }
    __device__ __forceinline__ uint32_t h1(unsigned long long k) const { return __umulhi(mix(k, c1), T); }
    __device__ __forceinline__ uint32_t h2(unsigned long long k) const { return __umulhi(mix(k, c2), T); }
    __device__ __forceinline__ bool contains(unsigned long long key) const {
        const unsigned long long x = lds64(base + 8 * h1(key));
        const unsigned long long y = lds64(base + 8 * h2(key));
        return (x == key) | (y == key);
    }
};

__device__ __forceinline__ bool cuckoo_insert64(unsigned long long *tab, const Cuckoo64 &c,
                                                unsigned long long key) {
    uint32_t h = c.h1(key);
    for (int i = 0; i < kCuckooMaxKicks; ++i) {
        const unsigned long long old = atomicExch(tab + h, key);
        if (old == ~0ull || old == key) return true;
        key = old;
        const uint32_t a = c.h1(key);
        h = (h == a) ? c.h2(key) : a;
    }
    return false;
}

// Per-window edge table in shared memory: edge k's list adj(v) = dst[vs_k, ve_k) is read
// as 16-byte chunks starting at the aligned a_k = vs_k & ~3; chunk j of the window
// (cst_k <= j < cst_{k+1}) is at dst + cb_k + 4 j with cb_k = a_k - 4 cst_k.
template <typename OffT>
struct EdgeTable {
    OffT *cb, *vs, *ve;
    uint32_t *cst;  // window + 1
    uint32_t *aux;  // per-edge probe argument (window: source id)
};

// Sweep chunks [c0, c1) of the window: every lane loads U 16-byte chunks, then tests
// each valid item with probe(w, aux).  Returns the number of hits.  Lanes past c1 reload
// the last chunk with an empty valid span, so the loop body has no divergent branches
// apart from the (rare) cursor advance.
template <typename OffT, bool HAS_AUX, int U = kUnroll, typename Probe>
__device__ __forceinline__ uint32_t sweep(const uint32_t *__restrict__ dst, const EdgeTable<OffT> &et,
                                          uint32_t nwin, uint32_t c0, uint32_t c1, Probe probe) {
    const unsigned lane = lane_id();
    uint32_t k = 0;
    {
        const uint32_t c = c0 + lane < c1 ? c0 + lane : c1 - 1;
        uint32_t a = 0, b = nwin;  // largest k < nwin with cst[k] <= c
        while (b - a > 1) {
            const uint32_t mid = (a + b) >> 1;
            if (et.cst[mid] <= c) a = mid; else b = mid;
        }
        k = a;
    }
    uint32_t nextb = et.cst[k + 1];
    OffT cb = et.cb[k], lo = et.vs[k];
    uint32_t span = (uint32_t)(et.ve[k] - lo);
    uint32_t aux = HAS_AUX ? et.aux[k] : 0u;
    uint32_t found = 0;
    for (uint32_t base = c0; base < c1; base += 32 * U) {
        uint4 q[U];
        uint32_t rel[U], sp[U], x[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            uint32_t c = base + j * 32 + lane;
            const bool live = c < c1;
            c = live ? c : c1 - 1;
            if (c >= nextb) {
                do { nextb = et.cst[++k + 1]; } while (c >= nextb);
                cb = et.cb[k];
                lo = et.vs[k];
                span = (uint32_t)(et.ve[k] - lo);
                if (HAS_AUX) aux = et.aux[k];
            }
            const OffT p = (OffT)(cb + (OffT)(4 * c));
            q[j] = __ldg(reinterpret_cast<const uint4 *>(dst + p));
            rel[j] = (uint32_t)(p - lo);
            sp[j] = live ? span : 0u;
            x[j] = aux;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t w4[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
            // item i is valid iff lo <= p + i < hi, i.e. (p + i - lo) < span unsigned
#pragma unroll
            for (int i = 0; i < 4; ++i)
                found += ((rel[j] + i < sp[j]) & probe(w4[i], x[j])) ? 1u : 0u;
        }
    }
    return found;
}

// sweep() over a window table addressed by 32-bit shared addresses held in registers
// (uint32_t offsets, no aux): the generic version's table reads make the compiler rebuild
// the shared-window base (S2R SR_CgaCtaId) at every cursor advance.
struct EdgeTableSA {
    uint32_t cb, vs, ve, cst;  // shared addresses of the per-edge arrays
};
template <int U, typename Probe>
__device__ __forceinline__ uint32_t sweep_sa(const uint32_t *__restrict__ dst, const EdgeTableSA et, uint32_t nwin,
                                             uint32_t c0, uint32_t c1, Probe probe) {
    const unsigned lane = lane_id();
    uint32_t k = 0;
    {
        const uint32_t c = c0 + lane < c1 ? c0 + lane : c1 - 1;
        uint32_t a = 0, b = nwin;
        while (b - a > 1) {
            const uint32_t mid = (a + b) >> 1;
            if (lds32(et.cst + 4 * mid) <= c) a = mid; else b = mid;
        }
        k = a;
    }
    uint32_t nextb = lds32(et.cst + 4 * (k + 1));
    uint32_t cb = lds32(et.cb + 4 * k), lo = lds32(et.vs + 4 * k);
    uint32_t span = lds32(et.ve + 4 * k) - lo;
    uint32_t found = 0;
    for (uint32_t base = c0; base < c1; base += 32 * U) {
        uint4 q[U];
        uint32_t rel[U], sp[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            uint32_t c = base + j * 32 + lane;
            const bool live = c < c1;
            c = live ? c : c1 - 1;
            if (c >= nextb) {
                do {
                    ++k;
                    nextb = lds32(et.cst + 4 * (k + 1));
                } while (c >= nextb);
                cb = lds32(et.cb + 4 * k);
                lo = lds32(et.vs + 4 * k);
                span = lds32(et.ve + 4 * k) - lo;
            }
            const uint32_t p = cb + 4 * c;
            q[j] = __ldg(reinterpret_cast<const uint4 *>(dst + p));
            rel[j] = p - lo;
            sp[j] = live ? span : 0u;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t w4[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) found += ((rel[j] + i < sp[j]) & probe(w4[i])) ? 1u : 0u;
        }
    }
    return found;
}

// sweep() specialised to a shared-memory bitmap probe over the hub zone: item w hits iff
// bit (w - hz) of `bitmap` is set.  Branch-free and lean: an invalid item (outside its
// list in a boundary chunk) is replaced by hz before the probe (bit 0 of word 0 -- always
// in range) and its hit is masked; valid items are >= hz by construction of the callers.
template <int U>
__device__ __forceinline__ uint32_t sweep_bits(const uint32_t *__restrict__ dst, const EdgeTable<uint32_t> &et,
                                               uint32_t nwin, uint32_t c0, uint32_t c1,
                                               const uint32_t *bitmap, uint32_t hz) {
    const unsigned lane = lane_id();
    uint32_t k = 0;
    {
        const uint32_t c = c0 + lane < c1 ? c0 + lane : c1 - 1;
        uint32_t a = 0, b = nwin;
        while (b - a > 1) {
            const uint32_t mid = (a + b) >> 1;
            if (et.cst[mid] <= c) a = mid; else b = mid;
        }
        k = a;
    }
    uint32_t nextb = et.cst[k + 1];
    uint32_t cb = et.cb[k], lo = et.vs[k];
    uint32_t span = et.ve[k] - lo;
    uint32_t found = 0;
    for (uint32_t base = c0; base < c1; base += 32 * U) {
        uint4 q[U];
        uint32_t rel[U], sp[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            uint32_t c = base + j * 32 + lane;
            const bool live = c < c1;
            c = live ? c : c1 - 1;
            if (c >= nextb) {
                do { nextb = et.cst[++k + 1]; } while (c >= nextb);
                cb = et.cb[k];
                lo = et.vs[k];
                span = et.ve[k] - lo;
            }
            const uint32_t p = cb + 4 * c;
            q[j] = __ldg(reinterpret_cast<const uint4 *>(dst + p));
            rel[j] = p - lo;
            sp[j] = live ? span : 0u;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t w4[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t ok = (rel[j] + i < sp[j]) ? 1u : 0u;
                const uint32_t r = (ok ? w4[i] : hz) - hz;
                found += (bitmap[r >> 5] >> (r & 31)) & ok;
            }
        }
    }
    return found;
}

// Hub items packed to 18 bits (2.25 B per item instead of 4): position p of edge_dst holds
// r = dst[p] - hz as lo16[p] (u16) plus 2 high bits in hi2[p / 4] (bits 2i..2i+1 for the i-th
// item of the aligned group of 4).  A 16-byte chunk of 4 items becomes one 8-byte + one
// 1-byte load.  Only positions holding hub items (>= hz) are meaningful; the sweeps read
// lists whose valid items are all hub items (suffixes after a hub head).
#ifndef TC_PACK_U
#define TC_PACK_U 8  // chunks in flight per lane in the packed sweep (9 B each: keep bytes in flight)
#endif
struct HubPack {
    const uint16_t *lo16;
    const uint8_t *hi2;
};

template <int U>
__device__ __forceinline__ uint32_t sweep_bits18(const HubPack hp, const EdgeTable<uint32_t> &et,
                                                 uint32_t nwin, uint32_t c0, uint32_t c1,
                                                 const uint32_t *bitmap) {
    const unsigned lane = lane_id();
    uint32_t k = 0;
    {
        const uint32_t c = c0 + lane < c1 ? c0 + lane : c1 - 1;
        uint32_t a = 0, b = nwin;
        while (b - a > 1) {
            const uint32_t mid = (a + b) >> 1;
            if (et.cst[mid] <= c) a = mid; else b = mid;
        }
        k = a;
    }
    uint32_t nextb = et.cst[k + 1];
    uint32_t cb = et.cb[k], lo = et.vs[k];
    uint32_t span = et.ve[k] - lo;
    uint32_t found = 0;
    for (uint32_t base = c0; base < c1; base += 32 * U) {
        uint2 q[U];
        uint32_t hb[U], rel[U], sp[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            uint32_t c = base + j * 32 + lane;
            const bool live = c < c1;
            c = live ? c : c1 - 1;
            if (c >= nextb) {
                do { nextb = et.cst[++k + 1]; } while (c >= nextb);
                cb = et.cb[k];
                lo = et.vs[k];
                span = et.ve[k] - lo;
            }
            const uint32_t p = cb + 4 * c;
            q[j] = __ldg(reinterpret_cast<const uint2 *>(hp.lo16 + p));
            hb[j] = __ldg(hp.hi2 + (p >> 2));
            rel[j] = p - lo;
            sp[j] = live ? span : 0u;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t r4[4] = {(q[j].x & 0xffffu) | ((hb[j] & 3u) << 16),
                                    (q[j].x >> 16) | (((hb[j] >> 2) & 3u) << 16),
                                    (q[j].y & 0xffffu) | (((hb[j] >> 4) & 3u) << 16),
                                    (q[j].y >> 16) | (((hb[j] >> 6) & 3u) << 16)};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t ok = (rel[j] + i < sp[j]) ? 1u : 0u;
                const uint32_t r = ok ? r4[i] : 0u;
                found += (bitmap[r >> 5] >> (r & 31)) & ok;
            }
        }
    }
    return found;
}

// Builds the packed hub representation of edge_dst: one thread per aligned group of 4.
__global__ void __launch_bounds__(256) k_pack_hub(const uint32_t *__restrict__ dst, uint64_t m, uint32_t hz,
                                                  uint16_t *__restrict__ lo16, uint8_t *__restrict__ hi2) {
    const uint64_t ng = (m + 3) / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += stride) {
        const uint4 w = __ldg(reinterpret_cast<const uint4 *>(dst) + g);  // dst is padded
        const uint32_t r0 = w.x >= hz ? w.x - hz : 0u, r1 = w.y >= hz ? w.y - hz : 0u;
        const uint32_t r2 = w.z >= hz ? w.z - hz : 0u, r3 = w.w >= hz ? w.w - hz : 0u;
        reinterpret_cast<uint2 *>(lo16)[g] =
            make_uint2((r0 & 0xffffu) | (r1 << 16), (r2 & 0xffffu) | (r3 << 16));
        hi2[g] = (uint8_t)(((r0 >> 16) & 3u) | (((r1 >> 16) & 3u) << 2) | (((r2 >> 16) & 3u) << 4) |
                           (((r3 >> 16) & 3u) << 6));
    }
}

// Dense edges of a heavy source: |adj(u) ∩ adj(v)| = popcount(B_u & B_v) over the hub
// words v can reach.  Chunk c of edge k reads 4 words of B_v at global word cb_k + 4c and
// 4 words of the shared-memory B_u at word vs_k + 4c (both 16-byte aligned).
template <int U>
__device__ __forceinline__ uint32_t sweep_and(const uint32_t *__restrict__ bits,
                                              const EdgeTable<uint32_t> &et, uint32_t nwin,
                                              uint32_t c0, uint32_t c1, uint32_t bm) {
    const unsigned lane = lane_id();
    uint32_t k = 0;
    {
        const uint32_t c = c0 + lane < c1 ? c0 + lane : c1 - 1;
        uint32_t a = 0, b = nwin;
        while (b - a > 1) {
            const uint32_t mid = (a + b) >> 1;
            if (et.cst[mid] <= c) a = mid; else b = mid;
        }
        k = a;
    }
    uint32_t nextb = et.cst[k + 1], gb = et.cb[k], sb = et.vs[k];
    uint32_t found = 0;
    for (uint32_t base = c0; base < c1; base += 32 * U) {
        uint4 q[U];
        uint32_t sw[U], live[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            uint32_t c = base + j * 32 + lane;
            live[j] = c < c1 ? 0xffffffffu : 0u;
            c = c < c1 ? c : c1 - 1;
            if (c >= nextb) {
                do { nextb = et.cst[++k + 1]; } while (c >= nextb);
                gb = et.cb[k];
                sb = et.vs[k];
            }
            q[j] = __ldg(reinterpret_cast<const uint4 *>(bits + gb + 4 * c));
            sw[j] = sb + 4 * c;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint4 b = lds128(bm + 4 * sw[j]);
            found += __popc(q[j].x & b.x & live[j]) + __popc(q[j].y & b.y & live[j]) +
                     __popc(q[j].z & b.z & live[j]) + __popc(q[j].w & b.w & live[j]);
        }
    }
    return found;
}

// sweep_and with the edge table read through 32-bit shared addresses (a_cst / a_cb / a_vs:
// cst, cb, vs) computed once per pass, whole rounds without liveness masks (only the last
// round of a warp's range is masked), and a 32-bit word index into B_v: the per-chunk
// address, owner-advance and mask work was most of k_count_hub's instructions (ncu).
#ifndef TC_AND2
#define TC_AND2 1
#endif
template <int U>
__device__ __forceinline__ uint32_t sweep_and2(const uint32_t *__restrict__ bits, uint32_t a_cst, uint32_t a_cb,
                                               uint32_t a_vs, uint32_t nwin, uint32_t c0, uint32_t c1,
                                               uint32_t bm) {
    const unsigned lane = lane_id();
    uint32_t k = 0;
    {
        const uint32_t c = c0 + lane < c1 ? c0 + lane : c1 - 1;
        uint32_t a = 0, b = nwin;
        while (b - a > 1) {
            const uint32_t mid = (a + b) >> 1;
            if (lds32(a_cst + 4 * mid) <= c) a = mid; else b = mid;
        }
        k = a;
    }
    uint32_t nextb = lds32(a_cst + 4 * (k + 1)), gb = lds32(a_cb + 4 * k), sa = bm + 4 * lds32(a_vs + 4 * k);
    uint32_t found = 0;
    uint32_t base = c0;
    for (; base + 32 * U <= c1; base += 32 * U) {
        uint4 q[U];
        uint32_t sw[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t c = base + j * 32 + lane;
            if (c >= nextb) {
                do {
                    ++k;
                    nextb = lds32(a_cst + 4 * (k + 1));
                } while (c >= nextb);
                gb = lds32(a_cb + 4 * k);
                sa = bm + 4 * lds32(a_vs + 4 * k);
            }
            q[j] = __ldg(reinterpret_cast<const uint4 *>(bits + (gb + 4 * c)));
            sw[j] = sa + 16 * c;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint4 b = lds128(sw[j]);
            found += __popc(q[j].x & b.x) + __popc(q[j].y & b.y) + __popc(q[j].z & b.z) + __popc(q[j].w & b.w);
        }
    }
    if (base < c1) {  // last, partial round: lanes past c1 reload the last chunk, masked
        uint4 q[U];
        uint32_t sw[U], live[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            uint32_t c = base + j * 32 + lane;
            live[j] = c < c1 ? 0xffffffffu : 0u;
            c = c < c1 ? c : c1 - 1;
            if (c >= nextb) {
                do {
                    ++k;
                    nextb = lds32(a_cst + 4 * (k + 1));
                } while (c >= nextb);
                gb = lds32(a_cb + 4 * k);
                sa = bm + 4 * lds32(a_vs + 4 * k);
            }
            q[j] = __ldg(reinterpret_cast<const uint4 *>(bits + (gb + 4 * c)));
            sw[j] = sa + 16 * c;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint4 b = lds128(sw[j]);
            found += __popc(q[j].x & b.x & live[j]) + __popc(q[j].y & b.y & live[j]) +
                     __popc(q[j].z & b.z & live[j]) + __popc(q[j].w & b.w & live[j]);
        }
    }
    return found;
}

// sweep_bits with the edge table (a_cst / a_cb / a_vs / a_ve) and the bitmap (bm) read
// through 32-bit shared addresses held in registers (see sweep_and2).
template <int U>
__device__ __forceinline__ uint32_t sweep_bits_sa(const uint32_t *__restrict__ dst, uint32_t a_cst, uint32_t a_cb,
                                                  uint32_t a_vs, uint32_t a_ve, uint32_t nwin, uint32_t c0,
                                                  uint32_t c1, uint32_t bm, uint32_t hz) {
    const unsigned lane = lane_id();
    uint32_t k = 0;
    {
        const uint32_t c = c0 + lane < c1 ? c0 + lane : c1 - 1;
        uint32_t a = 0, b = nwin;
        while (b - a > 1) {
            const uint32_t mid = (a + b) >> 1;
            if (lds32(a_cst + 4 * mid) <= c) a = mid; else b = mid;
        }
        k = a;
    }
    uint32_t nextb = lds32(a_cst + 4 * (k + 1));
    uint32_t cb = lds32(a_cb + 4 * k), lo = lds32(a_vs + 4 * k);
    uint32_t span = lds32(a_ve + 4 * k) - lo;
    uint32_t found = 0;
    for (uint32_t base = c0; base < c1; base += 32 * U) {
        uint4 q[U];
        uint32_t rel[U], sp[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            uint32_t c = base + j * 32 + lane;
            const bool live = c < c1;
            c = live ? c : c1 - 1;
            if (c >= nextb) {
                do {
                    ++k;
                    nextb = lds32(a_cst + 4 * (k + 1));
                } while (c >= nextb);
                cb = lds32(a_cb + 4 * k);
                lo = lds32(a_vs + 4 * k);
                span = lds32(a_ve + 4 * k) - lo;
            }
            const uint32_t p = cb + 4 * c;
            q[j] = __ldg(reinterpret_cast<const uint4 *>(dst + p));
            rel[j] = p - lo;
            sp[j] = live ? span : 0u;
        }
        uint32_t wd[4 * U], sh[4 * U], okm[4 * U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t w4[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t ok = (rel[j] + i < sp[j]) ? 1u : 0u;
                const uint32_t r = (ok ? w4[i] : hz) - hz;
                okm[4 * j + i] = ok;
                sh[4 * j + i] = r;
                wd[4 * j + i] = lds32(bm + 4 * (r >> 5));
            }
        }
#pragma unroll
        for (int t = 0; t < 4 * U; ++t) found += __funnelshift_r(wd[t], wd[t], sh[t]) & okm[t];
    }
    return found;
}

// Block-wide exclusive scan of two values per thread with one set of barriers.
// smem: 2 * 32 entries.  Returns the block totals in *ta, *tb.
__device__ __forceinline__ void block_exclusive_scan2(unsigned long long a, uint32_t b, unsigned long long *s_a,
                                                      uint32_t *s_b, unsigned long long *xa, uint32_t *xb,
                                                      unsigned long long *ta, uint32_t *tb) {
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned long long ia = warp_inclusive_scan(a);
    uint32_t ib = warp_inclusive_scan(b);
    if (lane == 31) {
        s_a[warp] = ia;
        s_b[warp] = ib;
    }
    __syncthreads();
    if (warp == 0) {
        const unsigned long long wa = lane < nw ? s_a[lane] : 0ull;
        const uint32_t wb = lane < nw ? s_b[lane] : 0u;
        const unsigned long long wia = warp_inclusive_scan(wa);
        const uint32_t wib = warp_inclusive_scan(wb);
        if (lane < nw) {
            s_a[lane] = wia - wa;
            s_b[lane] = wib - wb;
        }
        if (lane == nw - 1) {
            s_a[31] = wia;
            s_b[31] = wib;
        }
    }
    __syncthreads();
    *xa = s_a[warp] + ia - a;
    *xb = s_b[warp] + ib - b;
    *ta = s_a[31];
    *tb = s_b[31];
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
// Edges whose source is light (d+(u) <= 32), in windows of NT consecutive edges.
// Every light source list that owns an edge of the window lies inside dst[ws-31, we+31);
// those lists are inserted once per window into a shared-memory hash of (source, w)
// pairs.  The items of the window -- every element w of every adj(v) -- are then read as
// 16-byte chunks, split evenly over the warps, and tested with one 16-byte bucket load.
// HUB (rank space): a bitmap of the hub zone [hz, hz + 32 hwords) marks every hub
// neighbour of any light source of the window; a clear bit rejects an item with one
// shared load, and only candidates (set bit, or a non-hub w) pay the exact cuckoo test.
// HUB also enables the dense-hub shortcut: for an edge (u, v) with v among the top ranks,
// only the elements of adj(u) after v can close a triangle (ranks increase along a list),
// so those <= 31 candidates are tested against v's global bitmap instead of streaming
// all of adj(v).
template <typename OffT, int NT, bool HUB>
__global__ void __launch_bounds__(NT)
    k_count_window(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                   const OffT *__restrict__ off, const RangeDev *__restrict__ rg,
                   unsigned *__restrict__ next, uint32_t hz, uint32_t hwords, uint32_t vt,
                   const uint32_t *__restrict__ dense_off, const uint32_t *__restrict__ dense_bits,
                   uint32_t dense_words, unsigned long long *__restrict__ total) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long *s_tab = reinterpret_cast<unsigned long long *>(smem);  // kWinSlots
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(s_tab + kWinSlots);       // hwords (HUB)
    __shared__ OffT s_cb[NT], s_vs[NT], s_ve[NT];
    __shared__ uint32_t s_cst[NT + 4];
    __shared__ uint32_t s_aux[NT];
    __shared__ uint32_t s_scan[32];
    __shared__ unsigned s_win, s_fail;
    constexpr int NW = NT / 32;
    const unsigned warp = threadIdx.x >> 5;
    const uint64_t lo = rg->lo, hi = rg->hi, m = rg->m;
    const uint64_t nwin_total = (hi - lo + NT - 1) / NT;
    const EdgeTable<OffT> et{s_cb, s_vs, s_ve, s_cst, s_aux};
    const uint32_t bm = smem_addr(bitmap), hbits = 32 * hwords;
    if (HUB)
        for (uint32_t i = threadIdx.x; i < hwords; i += NT) bitmap[i] = 0;
    unsigned long long acc = 0;
    for (;;) {
        if (threadIdx.x == 0) s_win = atomicAdd(next, 1u);
        __syncthreads();
        const uint64_t wi = s_win;
        if (wi >= nwin_total) break;
        const uint64_t ws = lo + wi * NT;
        const uint64_t we = ws + NT < hi ? ws + NT : hi;
        const uint32_t nwin = (uint32_t)(we - ws);
        // the window's light source lists -> cuckoo table of (source, w) keys
        const uint64_t sb = ws >= (uint64_t)(kLightMax - 1) ? ws - (kLightMax - 1) : 0;
        const uint64_t se = we + (kLightMax - 1) < m ? we + (kLightMax - 1) : m;
        Cuckoo64 ck{smem_addr(s_tab), kWinSlots, 0, 0};
        for (uint32_t seed = 0;; ++seed) {
            if (seed == 32) __trap();  // cannot happen at load <= 1/4; never miscount
            ck.c1 = seed_mult(seed, 0);
            ck.c2 = seed_mult(seed, 1);
            for (uint32_t i = threadIdx.x; i < kWinSlots; i += NT) s_tab[i] = ~0ull;
            if (threadIdx.x == 0) s_fail = 0;
            __syncthreads();
            for (uint64_t P = sb + threadIdx.x; P < se; P += NT) {
                const uint32_t su_u = __ldg(src + P);
                const OffT su = __ldg(off + su_u), eu = __ldg(off + su_u + 1);
                if (eu - su <= (OffT)kLightMax && (uint64_t)su < we && (uint64_t)eu > ws) {
                    const uint32_t w = __ldg(dst + P);
                    const unsigned long long key = ((unsigned long long)su_u << 32) | w;
                    if (!cuckoo_insert64(s_tab, ck, key)) s_fail = 1;
                    if (HUB && seed == 0 && w - hz < hbits) atomicOr(bitmap + ((w - hz) >> 5), 1u << ((w - hz) & 31));
                }
            }
            __syncthreads();
            const bool failed = s_fail != 0;
            __syncthreads();
            if (!failed) break;
        }
        OffT vs = 0, ve = 0, ua = 0, ub = 0;
        uint32_t u = 0, bias = 0;
        bool dense = false;
        if (threadIdx.x < nwin) {
            const uint64_t e = ws + threadIdx.x;
            u = __ldg(src + e);
            const OffT su = __ldg(off + u), eu = __ldg(off + u + 1);
            if (eu - su <= (OffT)kLightMax) {
                const uint32_t v = __ldg(dst + e);
                vs = __ldg(off + v);
                ve = __ldg(off + v + 1);
                // u-side test when fewer candidates of adj(u) follow v than adj(v) has items
                dense = HUB && v >= vt && (OffT)(eu - (OffT)e - 1) < ve - vs;
                if (dense) {
                    ua = (OffT)e + 1;  // adj(u) after v
                    ub = eu;
                    bias = __ldg(dense_off + (v - vt)) - (((v + 1 - hz) >> 5) & ~3u);
                    vs = ve = 0;
                }
            }
        }
        // pass 0: v-side items of sparse edges against the window's (source, w) table;
        // pass 1: u-side candidates of dense edges against v's global bitmap.
        for (int pass = 0; pass < (HUB ? 2 : 1); ++pass) {
            const OffT a = pass == 0 ? vs : ua, bnd = pass == 0 ? ve : ub;
            const OffT a4 = a & ~(OffT)3;
            const uint32_t chunks = bnd > a ? (uint32_t)((bnd - a4 + 3) >> 2) : 0u;
            uint32_t tot;
            const uint32_t cst = block_exclusive_scan<uint32_t>(chunks, s_scan, &tot);
            if (tot == 0) continue;  // block-uniform
            s_cb[threadIdx.x] = a4 - (OffT)(4 * cst);
            s_vs[threadIdx.x] = a;
            s_ve[threadIdx.x] = bnd;
            s_cst[threadIdx.x] = cst;
            s_aux[threadIdx.x] = pass == 0 ? u : bias;
            if (threadIdx.x == 0) s_cst[NT] = tot;
            __syncthreads();
            const uint32_t c0 = (uint32_t)((uint64_t)tot * warp / NW);
            const uint32_t c1 = (uint32_t)((uint64_t)tot * (warp + 1) / NW);
            if (c0 < c1) {
                if (pass == 1) {
                    // masked-out chunk items are probed too: clamp them into the array
                    acc += sweep<OffT, true, 4>(dst, et, NT, c0, c1, [&](uint32_t w, uint32_t bw) {
                        const uint32_t r = w - hz;
                        const uint32_t i = min(bw + (r >> 5), dense_words - 1);
                        return ((__ldg(dense_bits + i) >> (r & 31)) & 1u) != 0u;
                    });
                } else if (HUB) {
                    acc += sweep<OffT, true, 4>(dst, et, NT, c0, c1, [&](uint32_t w, uint32_t sid) {
                        const uint32_t r = w - hz;
                        const uint32_t word = lds32(bm + 4 * min(r >> 5, hwords - 1));
                        bool hit = false;
                        if (r >= hbits || ((word >> (r & 31)) & 1u))
                            hit = ck.contains(((unsigned long long)sid << 32) | w);
                        return hit;
                    });
                } else {
                    acc += sweep<OffT, true>(dst, et, NT, c0, c1, [&](uint32_t w, uint32_t sid) {
                        return ck.contains(((unsigned long long)sid << 32) | w);
                    });
                }
            }
            __syncthreads();
        }
        if (HUB) {  // clear the bits this window set
            for (uint64_t P = sb + threadIdx.x; P < se; P += NT) {
                const uint32_t w = __ldg(dst + P);
                if (w - hz < hbits) bitmap[(w - hz) >> 5] = 0;
            }
            __syncthreads();
        }
    }
    block_add_total(acc, total);
}

// ------------------------------------------------------------ light, TPE ---
// Thread per oriented edge (u, v) with a light source (d+(u) <= 32).  In rank space
// (RANKED) ranks increase along a list and every element of adj(v) exceeds v, so only the
// suffix A = adj(u) after v -- dst[e+1, eu), <= 31 elements -- can close a triangle;
// otherwise A is all of adj(u).  B = adj(v).  The intersection |A ∩ B| is taken by one of
//  * bitmap test (HUB, v a dense hub, |A| < |B|): each element of A is one bit of v's
//    global bitmap (independent loads);
//  * binary search (skewed lengths, |A| log|B| < |A| + |B|): each element of A is
//    searched in B, the lower bound moving forward monotonically;
//  * merge: VEC = 4-wide block merge over aligned 16-byte chunks of A and B (16 compares
//    per step, the block with the smaller maximum advances, ~(|A|+|B|)/4 dependent
//    steps); otherwise the scalar branch-free two-pointer merge.
// VEC needs sentinels outside the id range: rank space, n <= 2^32 - 2, elements >= 1.
__device__ __forceinline__ uint32_t eq4(uint32_t x, const uint4 &b) {
    return (x == b.x) | (x == b.y) | (x == b.z) | (x == b.w);
}

template <typename OffT, bool RANKED, bool HUB, bool VEC>
__global__ void __launch_bounds__(256)
    k_count_light_tpe(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                      const OffT *__restrict__ off, const RangeDev *__restrict__ rg, uint32_t hz,
                      uint32_t vt, const uint32_t *__restrict__ dense_off,
                      const uint32_t *__restrict__ dense_bits, uint32_t dense_words,
                      VSplit vp, unsigned long long *__restrict__ total) {
    const uint64_t lo = rg->lo, hi = rg->hi;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (uint64_t e = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < hi; e += stride) {
        const uint32_t u = __ldg(src + e);
        const OffT su = __ldg(off + u), eu = __ldg(off + u + 1);
        OffT i = RANKED ? (OffT)e + 1 : su;
        if (eu - su > (OffT)kLightMax || i >= eu) continue;
        const uint32_t v = __ldg(dst + e);
        OffT j = __ldg(off + v);
        const OffT je = __ldg(off + v + 1);
        if (j >= je) continue;
        if (RANKED && vmajor_edge(vp, (uint32_t)e, (uint32_t)eu, v, (uint32_t)j, (uint32_t)je)) continue;
        const uint32_t la = (uint32_t)(eu - i), lb = (uint32_t)(je - j);
        if (HUB && v >= vt && la < lb) {
            const uint32_t bias = __ldg(dense_off + (v - vt)) - (((v + 1 - hz) >> 5) & ~3u);
            for (; i < eu; ++i) {
                const uint32_t r = __ldg(dst + i) - hz;
                const uint32_t wi = min(bias + (r >> 5), dense_words - 1);
                acc += (__ldg(dense_bits + wi) >> (r & 31)) & 1u;
            }
            continue;
        }
        if (la * (32u - __clz(lb)) < la + lb) {
            for (; i < eu && j < je; ++i) {
                const uint32_t a = __ldg(dst + i);
                OffT n = je - j;  // lower_bound(a) in [j, je)
                while (n > 0) {
                    const OffT h = n >> 1;
                    if (__ldg(dst + j + h) < a) { j += h + 1; n -= h + 1; }
                    else n = h;
                }
                if (j < je && __ldg(dst + j) == a) { ++acc; ++j; }
            }
            continue;
        }
        if (VEC) {
            OffT pa = i & ~(OffT)3, pb = j & ~(OffT)3;
            for (;;) {
                const uint4 qa = __ldg(reinterpret_cast<const uint4 *>(dst + pa));
                const uint4 qb = __ldg(reinterpret_cast<const uint4 *>(dst + pb));
                // invalid A lanes -> 0, invalid B lanes -> ~0: neither is a valid element
                const uint32_t a0 = pa + 0 >= i && pa + 0 < eu ? qa.x : 0u;
                const uint32_t a1 = pa + 1 >= i && pa + 1 < eu ? qa.y : 0u;
                const uint32_t a2 = pa + 2 >= i && pa + 2 < eu ? qa.z : 0u;
                const uint32_t a3 = pa + 3 < eu ? qa.w : 0u;
                uint4 bb;
                bb.x = pb + 0 >= j && pb + 0 < je ? qb.x : ~0u;
                bb.y = pb + 1 >= j && pb + 1 < je ? qb.y : ~0u;
                bb.z = pb + 2 >= j && pb + 2 < je ? qb.z : ~0u;
                bb.w = pb + 3 < je ? qb.w : ~0u;
                acc += eq4(a0, bb) + eq4(a1, bb) + eq4(a2, bb) + eq4(a3, bb);
                // block maxima; a block that ends its list counts as +inf
                const uint32_t amax = pa + 4 <= eu ? qa.w : ~0u;
                const uint32_t bmax = pb + 4 <= je ? qb.w : ~0u;
                if (amax <= bmax) pa += 4;
                if (bmax <= amax) pb += 4;
                if (pa >= eu || pb >= je) break;
            }
            continue;
        }
        uint32_t a = __ldg(dst + i), b = __ldg(dst + j);
        for (;;) {
            acc += a == b;
            const bool sa = a <= b, sb = b <= a;
            i += sa;
            j += sb;
            if (i >= eu || j >= je) break;
            if (sa) a = __ldg(dst + i);
            if (sb) b = __ldg(dst + j);
        }
    }
    block_add_total(acc, total);
}

// ----------------------------------------------------------- light, warp ---
// Rank space, light sources.  One warp per window of 32 consecutive oriented edges, no
// block-level synchronisation.  For lane e = (u, v) only the suffix A_e = dst[e+1, eu)
// of adj(u) can close a triangle (ranks increase along a list, every element of adj(v)
// exceeds v), and eu <= e + 32 for a light u, so every A_e of the window lies in
// dst[ws+1, ws+64): the warp stages that slice in shared memory once.  Per edge:
//  * dense-hub v with |A| < |B| (HUB): the lane tests its <= 31 suffix elements in v's
//    global bitmap (independent loads);
//  * strongly skewed |B| > kSkew |A|: the lane binary-searches each suffix element in
//    adj(v) (moving lower bound);
//  * otherwise the items of all B = adj(v) of the window are flattened over the 32 lanes
//    as 16-byte chunks (warp scan of chunk counts) and every item w is looked up in its
//    edge's A by a fixed 5-step binary search in shared memory.
constexpr int kLwWarps = 8;  // warps per CTA

template <typename OffT, bool HUB>
__global__ void __launch_bounds__(32 * kLwWarps)
    k_count_light_warp(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                       const OffT *__restrict__ off, const RangeDev *__restrict__ rg, uint32_t hz,
                       uint32_t vt, const uint32_t *__restrict__ dense_off,
                       const uint32_t *__restrict__ dense_bits, uint32_t dense_words,
                       uint32_t skew, unsigned long long *__restrict__ total) {
    __shared__ uint32_t s_list[kLwWarps][64];
    __shared__ OffT s_cb[kLwWarps][32], s_vs[kLwWarps][32], s_ve[kLwWarps][32];
    __shared__ uint32_t s_a[kLwWarps][32], s_cst[kLwWarps][33];
    const unsigned lane = lane_id(), wp = threadIdx.x >> 5;
    const uint64_t lo = rg->lo, hi = rg->hi, m = rg->m;
    const uint64_t nwin = (hi - lo + 31) / 32;
    const uint64_t wstride = (uint64_t)gridDim.x * kLwWarps;
    uint32_t *list = s_list[wp];
    const uint32_t lbase = smem_addr(list);
    uint32_t acc = 0;
    for (uint64_t wi = (uint64_t)blockIdx.x * kLwWarps + wp; wi < nwin; wi += wstride) {
        const uint64_t ws = lo + wi * 32;
        const uint64_t e = ws + lane;
        // stage dst[ws+1, ws+65) (positions past m read as 0; never inside a suffix)
        list[lane] = ws + 1 + lane < m ? __ldg(dst + ws + 1 + lane) : 0u;
        list[32 + lane] = ws + 33 + lane < m ? __ldg(dst + ws + 33 + lane) : 0u;
        __syncwarp();
        uint32_t chunks = 0, a0 = 0, a1 = 0;
        OffT vs = 0, ve = 0;
        if (e < hi) {
            const uint32_t u = __ldg(src + e);
            const OffT su = __ldg(off + u), eu = __ldg(off + u + 1);
            if (eu - su <= (OffT)kLightMax && (OffT)e + 1 < eu) {
                const uint32_t v = __ldg(dst + e);
                vs = __ldg(off + v);
                ve = __ldg(off + v + 1);
                const uint32_t la = (uint32_t)(eu - (OffT)e - 1), lb = (uint32_t)(ve - vs);
                a0 = lane;  // A_e = list[a0, a1)
                a1 = lane + la;
                if (lb == 0) {
                } else if (HUB && v >= vt && la < lb) {
                    const uint32_t bias = __ldg(dense_off + (v - vt)) - (((v + 1 - hz) >> 5) & ~3u);
                    for (uint32_t k = a0; k < a1; ++k) {
                        const uint32_t r = list[k] - hz;
                        const uint32_t wi2 = min(bias + (r >> 5), dense_words - 1);
                        acc += (__ldg(dense_bits + wi2) >> (r & 31)) & 1u;
                    }
                } else if (lb > skew * la) {
                    OffT j = vs;
                    for (uint32_t k = a0; k < a1 && j < ve; ++k) {
                        const uint32_t a = list[k];
                        OffT n = ve - j;
                        while (n > 0) {
                            const OffT h = n >> 1;
                            if (__ldg(dst + j + h) < a) { j += h + 1; n -= h + 1; }
                            else n = h;
                        }
                        if (j < ve && __ldg(dst + j) == a) { ++acc; ++j; }
                    }
                } else {
                    chunks = (uint32_t)((ve - (vs & ~(OffT)3) + 3) >> 2);
                }
            }
        }
        const uint32_t incl = warp_inclusive_scan(chunks);
        const uint32_t tot = __shfl_sync(TC_FULL_MASK, incl, 31);
        const uint32_t cst = incl - chunks;
        s_cb[wp][lane] = (vs & ~(OffT)3) - (OffT)(4 * cst);
        s_vs[wp][lane] = vs;
        s_ve[wp][lane] = ve;
        s_a[wp][lane] = a0 | (a1 << 8);
        s_cst[wp][lane] = cst;
        if (lane == 0) s_cst[wp][32] = tot;
        __syncwarp();
        if (tot) {
            // owner k of chunk c: largest k with cst[k] <= c (edges without chunks have
            // cst[k] == cst[k+1] and are skipped by the forward advance)
            uint32_t c = lane < tot ? lane : tot - 1;
            uint32_t k = 0;
            {
                uint32_t a = 0, b = 32;
                while (b - a > 1) {
                    const uint32_t mid = (a + b) >> 1;
                    if (s_cst[wp][mid] <= c) a = mid; else b = mid;
                }
                k = a;
            }
            uint32_t nextb = s_cst[wp][k + 1];
            OffT cb = s_cb[wp][k], lo_k = s_vs[wp][k];
            uint32_t span = (uint32_t)(s_ve[wp][k] - lo_k), ab = s_a[wp][k];
            for (uint32_t base = 0; base < tot; base += 32) {
                c = base + lane;
                const bool live = c < tot;
                c = live ? c : tot - 1;
                if (c >= nextb) {
                    do { nextb = s_cst[wp][++k + 1]; } while (c >= nextb);
                    cb = s_cb[wp][k];
                    lo_k = s_vs[wp][k];
                    span = (uint32_t)(s_ve[wp][k] - lo_k);
                    ab = s_a[wp][k];
                }
                const OffT p = cb + (OffT)(4 * c);
                const uint4 q = __ldg(reinterpret_cast<const uint4 *>(dst + p));
                const uint32_t rel = (uint32_t)(p - lo_k), sp = live ? span : 0u;
                const uint32_t ka = ab & 0xff, kb = ab >> 8;
                const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const uint32_t w = w4[t];
                    // lower bound of w in list[ka, kb) in 5 fixed steps
                    uint32_t pos = ka;
#pragma unroll
                    for (uint32_t step = 16; step; step >>= 1) {
                        const uint32_t qq = pos + step - 1;
                        const uint32_t x = lds32(lbase + 4 * min(qq, 63u));
                        pos = (qq < kb && x < w) ? pos + step : pos;
                    }
                    const uint32_t y = lds32(lbase + 4 * min(pos, 63u));
                    acc += ((rel + t < sp) & (pos < kb) & (y == w)) ? 1u : 0u;
                }
            }
        }
        __syncwarp();
    }
    block_add_total(acc, total);
}

// ------------------------------------------------------------------ heavy ---
template <typename OffT>
__global__ void k_classify(const OffT *__restrict__ off, const RangeDev *__restrict__ rg,
                           const uint32_t *__restrict__ hend, uint2 *__restrict__ t0,
                           uint2 *__restrict__ t1, uint2 *__restrict__ t2, uint2 *__restrict__ t3,
                           unsigned *__restrict__ ntasks) {
    const uint64_t lo = rg->lo, hi = rg->hi;
    const uint32_t u_lo = rg->u_lo, u_hi = rg->u_hi;
    const uint32_t stride = gridDim.x * blockDim.x;
    const unsigned lane = lane_id();
    // warp-uniform trip count; one task-cursor atomic per (warp, class) instead of per source
    for (uint32_t b = u_lo + blockIdx.x * blockDim.x + (threadIdx.x & ~31u); b < u_hi; b += stride) {
        const uint32_t u = b + lane;
        int cls = -1;
        uint32_t chunks = 0;
        if (u < u_hi) {
            const OffT s = off[u], e = off[u + 1];
            const uint32_t d = (uint32_t)(e - s);
            const uint64_t es = (uint64_t)s > lo ? (uint64_t)s : lo;
            uint64_t ee = (uint64_t)e < hi ? (uint64_t)e : hi;
            if (hend && (uint64_t)hend[u] < ee) ee = hend[u];  // v-major: hub heads excluded
            if (d > (uint32_t)kLightMax && es < ee) {
                constexpr uint32_t m0 = kClassMax[0], m1 = kClassMax[1], m2 = kClassMax[2];
                cls = d <= m0 ? 0 : d <= m1 ? 1 : d <= m2 ? 2 : 3;
                chunks = (uint32_t)((ee - es + kChunk - 1) / kChunk);
            }
        }
#pragma unroll
        for (int c = 0; c < kClasses; ++c) {
            const uint32_t x = cls == c ? chunks : 0u;
            if (!__any_sync(TC_FULL_MASK, x != 0)) continue;
            const uint32_t incl = warp_inclusive_scan(x);
            const uint32_t tot = __shfl_sync(TC_FULL_MASK, incl, 31);
            unsigned base = 0;
            if (lane == 31) base = atomicAdd(ntasks + c, tot);
            base = __shfl_sync(TC_FULL_MASK, base, 31);
            if (x) {
                uint2 *t = c == 0 ? t0 : c == 1 ? t1 : c == 2 ? t2 : t3;
                const unsigned slot = base + incl - x;
                for (uint32_t k = 0; k < x; ++k) t[slot + k] = make_uint2(u, k);
            }
        }
    }
}

// MODE 0: adj(u) in a linear-probing hash table; MODE 1: adj(u) as a sorted smem array.
// NT threads per CTA; windows of NT edges.
template <typename OffT, int MODE, int NT>
__global__ void __launch_bounds__(NT)
    k_count_heavy(const uint32_t *__restrict__ dst, const OffT *__restrict__ off,
                  const RangeDev *__restrict__ rg, const uint2 *__restrict__ tasks,
                  const unsigned *__restrict__ ntasks, unsigned *__restrict__ next, uint32_t cap,
                  unsigned long long *__restrict__ total) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *table = reinterpret_cast<uint32_t *>(smem);  // cap slots (MODE 0) / d (MODE 1)
    __shared__ OffT s_cb[NT], s_vs[NT], s_ve[NT];
    __shared__ uint32_t s_cst[NT + 4];
    __shared__ uint32_t s_scan[32];
    __shared__ unsigned s_task, s_fail;
    constexpr int NW = NT / 32;
    const unsigned warp = threadIdx.x >> 5;
    const uint64_t lo = rg->lo, hi = rg->hi;
    const unsigned nt = *ntasks;
    const EdgeTable<OffT> et{s_cb, s_vs, s_ve, s_cst, nullptr};
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

        Cuckoo32 ck{smem_addr(table), 4 * d < cap ? 4 * d : cap, 0, 0};
        bool tab_ok = true;
        if (MODE == 0) {
            tab_ok = false;
            for (uint32_t seed = 0; seed < kCuckooSeeds && !tab_ok; ++seed) {
                ck.c1 = seed_mult(seed, 0);
                ck.c2 = seed_mult(seed, 1);
                for (uint32_t i = threadIdx.x; i < ck.T; i += NT) table[i] = kEmpty;
                if (threadIdx.x == 0) s_fail = 0;
                __syncthreads();
                for (uint32_t i = threadIdx.x; i < d; i += NT)
                    if (!cuckoo_insert32(table, ck, __ldg(dst + s + i))) s_fail = 1;
                __syncthreads();
                tab_ok = s_fail == 0;
                __syncthreads();
            }
        } else {
            for (uint32_t i = threadIdx.x; i < d; i += NT) table[i] = __ldg(dst + s + i);
        }

        for (uint64_t ws = es; ws < ee; ws += NT) {
            const uint32_t nwin = (uint32_t)(ee - ws < (uint64_t)NT ? ee - ws : (uint64_t)NT);
            uint32_t chunks = 0;
            OffT vs = 0, ve = 0, a4 = 0;
            if (threadIdx.x < nwin) {
                const uint32_t v = __ldg(dst + ws + threadIdx.x);
                vs = __ldg(off + v);
                ve = __ldg(off + v + 1);
                a4 = vs & ~(OffT)3;
                chunks = ve > vs ? (uint32_t)((ve - a4 + 3) >> 2) : 0u;
            }
            uint32_t tot;
            const uint32_t cst = block_exclusive_scan<uint32_t>(chunks, s_scan, &tot);
            if (threadIdx.x < nwin) {
                s_cb[threadIdx.x] = a4 - (OffT)(4 * cst);
                s_vs[threadIdx.x] = vs;
                s_ve[threadIdx.x] = ve;
                s_cst[threadIdx.x] = cst;
            }
            if (threadIdx.x == 0) s_cst[nwin] = tot;
            __syncthreads();
            const uint32_t c0 = (uint32_t)((uint64_t)tot * warp / NW);
            const uint32_t c1 = (uint32_t)((uint64_t)tot * (warp + 1) / NW);
            if (c0 < c1) {
                if (MODE == 0 && tab_ok) {
                    acc += sweep<OffT, false>(dst, et, nwin, c0, c1,
                                              [&](uint32_t w, uint32_t) { return ck.contains(w); });
                } else if (MODE == 0) {
                    acc += sweep<OffT, false>(dst, et, nwin, c0, c1,
                                              [&](uint32_t w, uint32_t) { return sorted_contains(dst + s, d, w); });
                } else {
                    acc += sweep<OffT, false>(dst, et, nwin, c0, c1, [&](uint32_t w, uint32_t) {
                        uint32_t a = 0, n = d;
                        while (n > 0) {
                            const uint32_t half = n >> 1;
                            if (table[a + half] < w) { a += half + 1; n -= half + 1; }
                            else n = half;
                        }
                        return a < d && table[a] == w;
                    });
                }
            }
            __syncthreads();
        }
    }
    block_add_total(acc, total);
}

// -------------------------------------------------------------------- hub ---
// Rank-space heavy sources.  Ranks put the hub vertices in [hz, n); ~99 % of all items w
// (R-MAT s26) fall there.  adj(u) ∩ hub zone is staged as a kHubRanks-bit bitmap (one
// shared load per item, and sorted items of a list hit neighbouring words, so warps
// see few bank conflicts); the few non-hub elements of adj(u) go into a small cuckoo
// table.  hubstart[v] splits every adj(v) into a non-hub prefix and a hub suffix, which
// are swept separately so each probe path is branch-free.
#ifndef TC_HUB_FUSED
#define TC_HUB_FUSED 1  // the three per-window passes scanned together (one barrier pair)
#endif
#ifdef TC_HUB_MINB
#define TC_HUB_BOUNDS(nt) __launch_bounds__(nt, TC_HUB_MINB)
#else
#define TC_HUB_BOUNDS(nt) __launch_bounds__(nt)
#endif
template <int NT, int U>
__global__ void TC_HUB_BOUNDS(NT)
    k_count_hub(const uint32_t *__restrict__ dst, const uint32_t *__restrict__ off,
                const uint32_t *__restrict__ hubstart, uint32_t hz, uint32_t hwords,
                uint32_t vt, const uint32_t *__restrict__ dense_off,
                const uint32_t *__restrict__ dense_bits, uint32_t dense_factor, VSplit vp,
                const RangeDev *__restrict__ rg, const uint2 *__restrict__ tasks,
                const unsigned *__restrict__ ntasks, unsigned *__restrict__ next, uint32_t cap,
                const HubPack hp, unsigned long long *__restrict__ total) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(smem);  // hwords
    uint32_t *ctab = bitmap + hwords;                        // cap slots
#if TC_HUB_FUSED
    // one table per pass (0: hub suffixes, 1: non-hub prefixes, 2: dense ANDs), all three
    // scanned at once: one barrier pair per window instead of one per pass
    __shared__ uint32_t s_cb3[3][NT], s_vs3[3][NT], s_ve3[2][NT];
    __shared__ uint32_t s_cst3[3][NT + 4];
    __shared__ unsigned long long s_sa[32];
    __shared__ uint32_t s_sb[32];
#else
    __shared__ uint32_t s_cb[NT], s_vs[NT], s_ve[NT];
    __shared__ uint32_t s_cst[NT + 4];
    __shared__ uint32_t s_scan[32];
#endif
    __shared__ unsigned s_task, s_fail;
    constexpr int NW = NT / 32;
    const unsigned warp = threadIdx.x >> 5;
    const uint64_t lo = rg->lo, hi = rg->hi;
    const unsigned nt = *ntasks;
#if !TC_HUB_FUSED
    const EdgeTable<uint32_t> et{s_cb, s_vs, s_ve, s_cst, nullptr};
#endif
    // shared addresses in registers (opaque moves: no SR_CgaCtaId rebuild at every use)
    uint32_t bm;
    asm volatile("mov.b32 %0, %1;" : "=r"(bm) : "r"(smem_addr(bitmap)));
#if TC_HUB_FUSED
    uint32_t t3;
    asm volatile("mov.b32 %0, %1;" : "=r"(t3) : "r"(smem_addr(&s_cb3[0][0])));
    const uint32_t a_cst2 = t3 + (smem_addr(&s_cst3[2][0]) - smem_addr(&s_cb3[0][0]));
    const uint32_t a_cb2 = t3 + (smem_addr(&s_cb3[2][0]) - smem_addr(&s_cb3[0][0]));
    const uint32_t a_vs2 = t3 + (smem_addr(&s_vs3[2][0]) - smem_addr(&s_cb3[0][0]));
    const uint32_t a_cst0 = t3 + (smem_addr(&s_cst3[0][0]) - smem_addr(&s_cb3[0][0]));
    const uint32_t a_cb0 = t3;
    const uint32_t a_vs0 = t3 + (smem_addr(&s_vs3[0][0]) - smem_addr(&s_cb3[0][0]));
    const uint32_t a_ve0 = t3 + (smem_addr(&s_ve3[0][0]) - smem_addr(&s_cb3[0][0]));
#endif
    for (uint32_t i = threadIdx.x; i < hwords; i += NT) bitmap[i] = 0;
    unsigned long long acc = 0;
    for (;;) {
        if (threadIdx.x == 0) s_task = atomicAdd(next, 1u);
        __syncthreads();
        const unsigned t = s_task;
        if (t >= nt) break;
        const uint2 task = tasks[t];
        const uint32_t u = task.x;
        const uint32_t s = off[u], e = off[u + 1], hsu = hubstart[u];
        const uint32_t nh = hsu - s;  // non-hub prefix of adj(u)
        uint64_t es = (uint64_t)s > lo ? (uint64_t)s : lo;
        uint64_t ee = (uint64_t)e < hi ? (uint64_t)e : hi;
        es += (uint64_t)task.y * kChunk;
        ee = ee < es + kChunk ? ee : es + kChunk;

        Cuckoo32 ck{smem_addr(ctab), 3 * nh < cap ? 3 * nh : cap, 0, 0};
        bool tab_ok = true;
        if (nh) {
            tab_ok = false;
            // a non-hub part beyond the table's 1/3 load goes straight to binary search
            for (uint32_t seed = 0; seed < kCuckooSeeds && !tab_ok && 3 * nh <= cap; ++seed) {
                ck.c1 = seed_mult(seed, 0);
                ck.c2 = seed_mult(seed, 1);
                for (uint32_t i = threadIdx.x; i < ck.T; i += NT) ctab[i] = kEmpty;
                if (threadIdx.x == 0) s_fail = 0;
                __syncthreads();
                for (uint32_t i = threadIdx.x; i < nh; i += NT)
                    if (!cuckoo_insert32(ctab, ck, __ldg(dst + s + i))) s_fail = 1;
                __syncthreads();
                tab_ok = s_fail == 0;
                __syncthreads();
            }
        }
        for (uint32_t i = nh + threadIdx.x; i < e - s; i += NT) {
            const uint32_t r = __ldg(dst + s + i) - hz;
            atomicOr(bitmap + (r >> 5), 1u << (r & 31));
        }
        __syncthreads();

        // Window metadata is software-pipelined: the head v of window k+2 and the offsets /
        // hubstart / dense offset of window k+1 are loaded while window k is swept, so the
        // dependent chain edge -> v -> off[v] is off the critical path.
        auto load_v = [&](uint64_t w) -> uint32_t {
            return w + threadIdx.x < ee ? __ldg(dst + w + threadIdx.x) : 0xffffffffu;
        };
        auto load_meta = [&](uint32_t x, uint32_t &a0, uint32_t &a1, uint32_t &a2, uint32_t &a3) {
            if (x != 0xffffffffu) {
                a0 = __ldg(off + x);
                a1 = __ldg(off + x + 1);
                a2 = __ldg(hubstart + x);
                a3 = x >= vt ? __ldg(dense_off + (x - vt)) : 0u;
            }
        };
        uint32_t v_n = load_v(es), v_nn = load_v(es + NT);
        uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
        load_meta(v_n, m0, m1, m2, m3);
        for (uint64_t ws = es; ws < ee; ws += NT) {
            const uint32_t nwin = (uint32_t)(ee - ws < (uint64_t)NT ? ee - ws : (uint64_t)NT);
            uint32_t v = v_n, vs = m0, ve = m1, hv = 0, dgo = 0, dws = 0;
            const uint32_t hv_l = m2, dgo_l = m3;
            bool dense = false;
            // next window's metadata (its head arrived one window ago), head of the one after
            v_n = v_nn;
            m0 = m1 = m2 = m3 = 0;
            load_meta(v_n, m0, m1, m2, m3);
            v_nn = load_v(ws + 2 * (uint64_t)NT);
            if (threadIdx.x < nwin) {
                if (vmajor_edge(vp, (uint32_t)(ws + threadIdx.x), e, v, vs, ve)) {
                    vs = ve = 0;  // counted by k_count_vmajor
                } else {
                    // v's adjacency is also a bitmap: AND with B_u when its words cost less
                    // than probing its items (~3.5 vs ~12 instructions per unit)
                    if (v >= vt) {
                        dws = ((v + 1 - hz) >> 5) & ~3u;
                        dense = (hwords - dws) < dense_factor * (ve - vs);
                        if (dense) dgo = dgo_l;
                    }
                    if (dense) vs = ve = 0;
                    else hv = hv_l;
                }
            } else {
                v = vs = ve = 0;
            }
            // pass 0: hub suffixes [hv, ve) of sparse edges against the bitmap;
            // pass 1: non-hub prefixes [vs, hv) against the cuckoo table (only if adj(u)
            //         has non-hub elements -- otherwise they cannot match);
            // pass 2: dense edges, popcount(B_u & B_v) over v's hub words.
#if TC_HUB_FUSED
            {
                const uint32_t h4 = hv & ~3u, v4 = vs & ~3u;
                const uint32_t ch0 = ve > hv ? (ve - h4 + 3) >> 2 : 0u;
                const uint32_t ch1 = nh && hv > vs ? (hv - v4 + 3) >> 2 : 0u;
                const uint32_t ch2 = dense ? (hwords - dws) >> 2 : 0u;
                unsigned long long x01, t01;
                uint32_t x2, t2;
                block_exclusive_scan2((unsigned long long)ch0 | ((unsigned long long)ch1 << 32), ch2, s_sa, s_sb,
                                      &x01, &x2, &t01, &t2);
                const uint32_t x0 = (uint32_t)x01, x1 = (uint32_t)(x01 >> 32);
                const uint32_t tt[3] = {(uint32_t)t01, (uint32_t)(t01 >> 32), t2};
                if (tt[0] | tt[1] | tt[2]) {  // block-uniform
                    const uint32_t t = threadIdx.x;
                    s_cb3[0][t] = h4 - 4 * x0;
                    s_vs3[0][t] = hv;
                    s_ve3[0][t] = ve;
                    s_cst3[0][t] = x0;
                    s_cb3[1][t] = v4 - 4 * x1;
                    s_vs3[1][t] = vs;
                    s_ve3[1][t] = hv;
                    s_cst3[1][t] = x1;
                    s_cb3[2][t] = dgo - 4 * x2;
                    s_vs3[2][t] = dws - 4 * x2;
                    s_cst3[2][t] = x2;
                    if (t < 3) s_cst3[t][NT] = tt[t];
                    __syncthreads();
#pragma unroll
                    for (int pass = 0; pass < 3; ++pass) {
                        const uint32_t tot = tt[pass];
                        const uint32_t c0 = (uint32_t)((uint64_t)tot * warp / NW);
                        const uint32_t c1 = (uint32_t)((uint64_t)tot * (warp + 1) / NW);
                        if (c0 >= c1) continue;
                        const EdgeTable<uint32_t> et{s_cb3[pass], s_vs3[pass], pass < 2 ? s_ve3[pass] : nullptr,
                                                     s_cst3[pass], nullptr};
                        if (pass == 2) {
#if TC_AND2
                            acc += sweep_and2<U>(dense_bits, a_cst2, a_cb2, a_vs2, NT, c0, c1, bm);
#else
                            acc += sweep_and<U>(dense_bits, et, NT, c0, c1, bm);
#endif
                        } else if (pass == 0) {
                            if (hp.lo16) acc += sweep_bits18<U>(hp, et, NT, c0, c1, bitmap);
#if TC_AND2
                            else acc += sweep_bits_sa<U>(dst, a_cst0, a_cb0, a_vs0, a_ve0, NT, c0, c1, bm, hz);
#else
                            else acc += sweep_bits<U>(dst, et, NT, c0, c1, bitmap, hz);
#endif
                        } else if (tab_ok) {
                            acc += sweep<uint32_t, false>(dst, et, NT, c0, c1,
                                                          [&](uint32_t w, uint32_t) { return ck.contains(w); });
                        } else {
                            acc += sweep<uint32_t, false>(dst, et, NT, c0, c1, [&](uint32_t w, uint32_t) {
                                return sorted_contains(dst + s, nh, w);
                            });
                        }
                    }
                    __syncthreads();
                }
            }
#else
            for (int pass = 0; pass < 3; ++pass) {
                if (pass == 1 && !nh) continue;
                uint32_t chunks, cb, vsb;
                if (pass < 2) {
                    const uint32_t a = pass == 0 ? hv : vs, b = pass == 0 ? ve : hv;
                    const uint32_t a4 = a & ~3u;
                    chunks = b > a ? (b - a4 + 3) >> 2 : 0u;
                    cb = a4;
                    vsb = a;
                    s_ve[threadIdx.x] = b;
                } else {
                    chunks = dense ? (hwords - dws) >> 2 : 0u;
                    cb = dgo;
                    vsb = dws;
                }
                uint32_t tot;
                const uint32_t cst = block_exclusive_scan<uint32_t>(chunks, s_scan, &tot);
                if (tot == 0) continue;  // block-uniform
                s_cb[threadIdx.x] = cb - 4 * cst;
                s_vs[threadIdx.x] = pass < 2 ? vsb : vsb - 4 * cst;
                s_cst[threadIdx.x] = cst;
                if (threadIdx.x == 0) s_cst[NT] = tot;
                __syncthreads();
                const uint32_t c0 = (uint32_t)((uint64_t)tot * warp / NW);
                const uint32_t c1 = (uint32_t)((uint64_t)tot * (warp + 1) / NW);
                if (c0 < c1) {
                    if (pass == 2) {
                        acc += sweep_and<U>(dense_bits, et, NT, c0, c1, bm);
                    } else if (pass == 0) {
                        // hub suffixes [hubstart[v], ve): every valid item is >= hz
                        if (hp.lo16) acc += sweep_bits18<U>(hp, et, NT, c0, c1, bitmap);
                        else acc += sweep_bits<U>(dst, et, NT, c0, c1, bitmap, hz);
                    } else if (tab_ok) {
                        acc += sweep<uint32_t, false>(dst, et, NT, c0, c1,
                                                      [&](uint32_t w, uint32_t) { return ck.contains(w); });
                    } else {
                        acc += sweep<uint32_t, false>(dst, et, NT, c0, c1, [&](uint32_t w, uint32_t) {
                            return sorted_contains(dst + s, nh, w);
                        });
                    }
                }
                __syncthreads();
            }
#endif
        }
        // clear the bits this task set (O(d), not O(bitmap))
        for (uint32_t i = nh + threadIdx.x; i < e - s; i += NT)
            bitmap[(__ldg(dst + s + i) - hz) >> 5] = 0;
        __syncthreads();
    }
    block_add_total(acc, total);
}

// --------------------------------------------------------- mid, warp/task ---
// Heavy sources of the smallest class (33 <= d+(u) <= 512), rank space: ONE WARP per task
// instead of a CTA.  adj(u) goes into a per-warp shared-memory cuckoo table (load <= 1/4,
// 8 KB), the task's u-major edges (v-major heads and empty intersections dropped) are taken
// 32 at a time, and all items of their adj(v) are flattened over the warp's lanes as
// 16-byte chunks and probed in the table.  No block barriers: 8 independent tasks per CTA
// keep their dependent load chains (task -> offsets -> lists) in flight together, which
// the CTA-per-task hub kernel (one 32 KB bitmap per task) cannot.
constexpr int kMidWarps = 8;
#ifndef TC_MID_LOADINV
#define TC_MID_LOADINV 2  // 2: 4 KB per warp, 6 CTAs per SM (3: 6 KB, 4 CTAs; s26 mid 14.6 -> 13.6 ms)
#endif
constexpr uint32_t kMidLoadInv = TC_MID_LOADINV;  // per-warp cuckoo table load <= 1/kMidLoadInv
constexpr uint32_t kMidSlots = kMidLoadInv * 512;

#ifndef TC_MID_MINB
#define TC_MID_MINB 6  // 6 CTAs per SM: 40 registers, no spills (ptxas picked 32 + spills: mid 9.7 -> 9.2 ms)
#endif
template <int WARPS, uint32_t SLOTS, uint32_t LOADINV>
__global__ void __launch_bounds__(32 * WARPS, TC_MID_MINB)
    k_count_mid_warp(const uint32_t *__restrict__ dst, const uint32_t *__restrict__ off, VSplit vp,
                     const RangeDev *__restrict__ rg, const uint2 *__restrict__ tasks,
                     const unsigned *__restrict__ ntasks, unsigned *__restrict__ next,
                     unsigned long long *__restrict__ total) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_cb[WARPS][32], s_vs[WARPS][32], s_ve[WARPS][32];
    __shared__ uint32_t s_cst[WARPS][36];
    const unsigned lane = lane_id(), wp = threadIdx.x >> 5;
    uint32_t *tab = reinterpret_cast<uint32_t *>(smem) + wp * SLOTS;
    const EdgeTable<uint32_t> et{s_cb[wp], s_vs[wp], s_ve[wp], s_cst[wp], nullptr};
    const uint64_t lo = rg->lo, hi = rg->hi;
    const unsigned nt = *ntasks;
    uint32_t acc = 0;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(next, 1u);
        t = __shfl_sync(TC_FULL_MASK, t, 0);
        if (t >= nt) break;
        const uint2 task = tasks[t];
        const uint32_t u = task.x;
        const uint32_t s = __ldg(off + u), e = __ldg(off + u + 1), d = e - s;
        uint64_t es = (uint64_t)s > lo ? (uint64_t)s : lo;
        uint64_t ee = (uint64_t)e < hi ? (uint64_t)e : hi;
        es += (uint64_t)task.y * kChunk;
        ee = ee < es + kChunk ? ee : es + kChunk;
        Cuckoo32 ck{smem_addr(tab), LOADINV * d < SLOTS ? LOADINV * d : SLOTS, 0, 0};
        bool tab_ok = false;
        for (uint32_t seed = 0; seed < kCuckooSeeds && !tab_ok; ++seed) {
            ck.c1 = seed_mult(seed, 0);
            ck.c2 = seed_mult(seed, 1);
            for (uint32_t i = lane; i < ck.T; i += 32) tab[i] = kEmpty;
            __syncwarp();
            bool fail = false;
            for (uint32_t i = lane; i < d; i += 32)
                if (!cuckoo_insert32(tab, ck, __ldg(dst + s + i))) fail = true;
            __syncwarp();
            tab_ok = !__any_sync(TC_FULL_MASK, fail);
        }
        // window metadata software-pipelined: heads two windows ahead, their offsets one
        // window ahead (the chain edge -> v -> off[v] is off the critical path)
        auto load_v = [&](uint64_t w) -> uint32_t { return w + lane < ee ? __ldg(dst + w + lane) : 0xffffffffu; };
        uint32_t v_n = load_v(es), v_nn = load_v(es + 32), m0 = 0, m1 = 0;
        if (v_n != 0xffffffffu) {
            m0 = __ldg(off + v_n);
            m1 = __ldg(off + v_n + 1);
        }
        for (uint64_t ws = es; ws < ee; ws += 32) {
            const uint32_t v = v_n;
            uint32_t vs = m0, ve = m1, chunks = 0;
            v_n = v_nn;
            m0 = m1 = 0;
            if (v_n != 0xffffffffu) {
                m0 = __ldg(off + v_n);
                m1 = __ldg(off + v_n + 1);
            }
            v_nn = load_v(ws + 64);
            if (v != 0xffffffffu) {
                const uint32_t p = (uint32_t)(ws + lane);
                if (p + 1 < e && vs < ve && !vmajor_edge(vp, p, e, v, vs, ve))
                    chunks = (ve - (vs & ~3u) + 3) >> 2;
                else
                    vs = ve = 0;
            } else {
                vs = ve = 0;
            }
            const uint32_t incl = warp_inclusive_scan(chunks);
            const uint32_t tot = __shfl_sync(TC_FULL_MASK, incl, 31);
            if (tot == 0) continue;  // warp-uniform
            const uint32_t cst = incl - chunks;
            s_cb[wp][lane] = (vs & ~3u) - 4 * cst;
            s_vs[wp][lane] = vs;
            s_ve[wp][lane] = ve;
            s_cst[wp][lane] = cst;
            if (lane == 0) s_cst[wp][32] = tot;
            __syncwarp();
            if (tab_ok)
                acc += sweep<uint32_t, false, 2>(dst, et, 32, 0, tot,
                                                [&](uint32_t w, uint32_t) { return ck.contains(w); });
            else
                acc += sweep<uint32_t, false, 2>(dst, et, 32, 0, tot, [&](uint32_t w, uint32_t) {
                    return sorted_contains(dst + s, d, w);
                });
            __syncwarp();
        }
    }
    block_add_total(acc, total);
}

// ---------------------------------------------------------------- v-major ---
// Rank space, edges e = (u, v) whose head v is in the hub zone [hz, n) (R-MAT s26: 77 % of
// all edges, ~90 % of the u-major kernels' bytes).  adj(v) lies in (v, n), inside the hub
// zone, and only the suffix of adj(u) after v -- dst[e+1, off[u+1]) -- can close a
// triangle.  Grouping these edges by v lets a CTA stage adj(v) ONCE as a shared-memory
// bitmap over hub words [ws(v), hwp) and stream the suffixes of all of v's in-edges
// against it (one LDS bit test per item): the re-read data becomes the suffixes of adj(u)
// (coalesced streams, 4 B per item) instead of adj(v) / v's bitmap per in-edge.
//
// Index: in-edges of each hub head, counting sort by v (only edges whose suffix and adj(v)
// are both non-empty); tasks = (v, chunk of kVChunk in-edges) in v order.
#ifndef TC_VCHUNK
#define TC_VCHUNK 2048
#endif
constexpr uint32_t kVChunk = TC_VCHUNK;

// Both index passes evaluate the v-major predicate of every edge; each thread keeps
// kVinPP edges in flight (all loads of a stage issued before any is used): the passes are
// bound by dependent global-load latency (src/dst -> offsets -> atomic), not bandwidth.
constexpr int kVinPP = 8;

template <bool FILL>
__global__ void __launch_bounds__(256)
    k_vin_pass(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
               const uint32_t *__restrict__ off, const RangeDev *__restrict__ rg, VSplit vp,
               const uint32_t *__restrict__ start, uint32_t *__restrict__ cnt,
               uint2 *__restrict__ in_e, uint32_t *__restrict__ capflag, uint32_t hlo, uint32_t hhi) {
    const uint64_t lo = rg->lo, hi = rg->hi;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * kVinPP;
    for (uint64_t b = lo + ((uint64_t)blockIdx.x * blockDim.x) * kVinPP + threadIdx.x; b < hi; b += stride) {
        uint32_t v[kVinPP], u[kVinPP];
#pragma unroll
        for (int i = 0; i < kVinPP; ++i) {
            const uint64_t e = b + (uint64_t)i * blockDim.x;
            v[i] = e < hi ? __ldg(dst + e) : 0u;
            u[i] = e < hi ? __ldg(src + e) : 0u;
        }
        uint32_t eu[kVinPP], vs[kVinPP], ve[kVinPP];
#pragma unroll
        for (int i = 0; i < kVinPP; ++i) {
            const uint64_t e = b + (uint64_t)i * blockDim.x;
            // head filter [hlo, hhi): a shard counts the v-major edges of its own heads
            const bool cand = e < hi && v[i] >= vp.z0 && v[i] >= hlo && v[i] < hhi;
            eu[i] = cand ? __ldg(off + u[i] + 1) : 0u;
            vs[i] = cand ? __ldg(off + v[i]) : 0u;
            ve[i] = cand ? __ldg(off + v[i] + 1) : 0u;
        }
        // all atomics of the batch first (independent, in flight together), then the stores
        uint32_t pos[kVinPP];
#pragma unroll
        for (int i = 0; i < kVinPP; ++i) {
            const uint32_t e = (uint32_t)(b + (uint64_t)i * blockDim.x);
            pos[i] = 0xffffffffu;
            if (v[i] < vp.z0 || v[i] < hlo || v[i] >= hhi) continue;
            if (e + 1 >= eu[i] || vs[i] >= ve[i] || !vmajor_edge(vp, e, eu[i], v[i], vs[i], ve[i])) continue;
            const uint32_t h = v[i] - vp.z0;
            if (FILL) {
                const uint32_t k = atomicAdd(cnt + h, 1u);
                // capacity layout: a slot past v's capacity means the input was not
                // symmetric (in-degree != degree - out-degree); flag it, never write past
                if (capflag && k >= __ldg(start + h + 1) - __ldg(start + h)) *capflag = 1u;
                else pos[i] = __ldg(start + h) + k;
            } else {
                atomicAdd(cnt + h, 1u);
            }
        }
#if defined(TC_VIN_PROBE) && TC_VIN_PROBE == 1  // diagnostic build: atomics only, no index stores
        if (false) {
#else
        if (FILL) {
#endif
#pragma unroll
            for (int i = 0; i < kVinPP; ++i)
                if (pos[i] != 0xffffffffu)
                    in_e[pos[i]] = make_uint2((uint32_t)(b + (uint64_t)i * blockDim.x), eu[i]);
        }
    }
}

// start[i] = exclusive scan of cnt, tstart[i] = exclusive scan of task counts
// ceil(cnt / kVChunk); start[nh], tstart[nh] = totals; cnt is zeroed (fill cursors).
// Three launches: per-tile sums, one-block scan of the tile sums, per-tile apply.
constexpr uint32_t kVinTile = 4096;

// TASKS = false: value = cnt, output start, cnt zeroed (fill cursors);
// TASKS = true:  value = ceil(cnt / kVChunk), output tstart, cnt kept (fill counts).
template <bool TASKS>
__device__ __forceinline__ uint32_t vin_val(uint32_t c) { return TASKS ? (c + kVChunk - 1) / kVChunk : c; }

template <bool TASKS>
__global__ void __launch_bounds__(256) k_vin_tilesum(const uint32_t *__restrict__ cnt, uint32_t nh,
                                                     uint32_t *__restrict__ tsum) {
    const uint32_t b = blockIdx.x * kVinTile;
    uint32_t x = 0;
    for (uint32_t i = b + threadIdx.x; i < b + kVinTile && i < nh; i += 256) x += vin_val<TASKS>(cnt[i]);
    __shared__ uint32_t s_w[32];
    uint32_t tx;
    block_exclusive_scan<uint32_t>(x, s_w, &tx);
    if (threadIdx.x == 0) tsum[blockIdx.x] = tx;
}

__global__ void k_vin_tilescan(uint32_t *__restrict__ tsum, uint32_t ntile, uint32_t *__restrict__ out,
                               uint32_t nh) {
    __shared__ uint32_t s_w[32];
    uint32_t cx = 0;
    for (uint32_t b = 0; b < ntile; b += blockDim.x) {
        const uint32_t i = b + threadIdx.x;
        const uint32_t v = i < ntile ? tsum[i] : 0u;
        uint32_t tx;
        const uint32_t ex = block_exclusive_scan<uint32_t>(v, s_w, &tx);
        if (i < ntile) tsum[i] = cx + ex;
        cx += tx;
    }
    if (threadIdx.x == 0) out[nh] = cx;
}

template <bool TASKS>
__global__ void __launch_bounds__(256) k_vin_apply(uint32_t *__restrict__ cnt, uint32_t nh,
                                                   const uint32_t *__restrict__ tsum,
                                                   uint32_t *__restrict__ out) {
    __shared__ uint32_t s_w[32];
    const uint32_t b = blockIdx.x * kVinTile;
    uint32_t carry = tsum[blockIdx.x];
    for (uint32_t o = 0; o < kVinTile; o += 256) {
        const uint32_t i = b + o + threadIdx.x;
        const uint32_t c = i < nh ? vin_val<TASKS>(cnt[i]) : 0u;
        uint32_t tx;
        const uint32_t ex = block_exclusive_scan<uint32_t>(c, s_w, &tx);
        if (i < nh) {
            out[i] = carry + ex;
            if (!TASKS) cnt[i] = 0;
        }
        carry += tx;
    }
}

// exclusive scan of vin_val<TASKS>(cnt) into out[0..nh] (three launches)
template <bool TASKS>
int vin_scan(uint32_t *cnt, uint32_t nh, uint32_t *out, cudaStream_t s) {
    const uint32_t ntile = (nh + kVinTile - 1) / kVinTile;
    uint32_t *tsum = nullptr;
    TC_CHECK(dalloc_t(&tsum, ntile ? ntile : 1, s));
    k_vin_tilesum<TASKS><<<ntile, 256, 0, s>>>(cnt, nh, tsum);
    TC_LAUNCHED();
    k_vin_tilescan<<<1, 1024 - 32, 0, s>>>(tsum, ntile, out, nh);  // block scan: <= 31 warps
    TC_LAUNCHED();
    k_vin_apply<TASKS><<<ntile, 256, 0, s>>>(cnt, nh, tsum, out);
    TC_LAUNCHED();
    dfree(tsum, s);
    return 0;
}

__global__ void k_vin_capacity(const uint32_t *__restrict__ deg_by_rank, const uint32_t *__restrict__ off,
                               uint32_t z0, uint32_t nz, uint32_t *__restrict__ cap) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nz; i += gridDim.x * blockDim.x) {
        const uint32_t v = z0 + i;
        const uint32_t d = deg_by_rank[v], o = off[v + 1] - off[v];
        cap[i] = d > o ? d - o : 0u;  // in-degree = degree - out-degree (symmetric input)
    }
}

// Tasks in head order; heads below the hub zone (h < hb) whose list exceeds `small` are
// also appended to `big` (they run as CTA tasks, the warp kernel skips them).
__global__ void k_vin_tasks(const uint32_t *__restrict__ start, const uint32_t *__restrict__ tstart,
                            uint32_t nh, uint2 *__restrict__ tasks, const uint32_t *__restrict__ off,
                            uint32_t z0, uint32_t hb, uint32_t small, uint2 *__restrict__ big,
                            unsigned *__restrict__ nbig) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < nh; h += stride) {
        const uint32_t t0 = tstart[h], t1 = tstart[h + 1];
        for (uint32_t t = t0; t < t1; ++t) tasks[t] = make_uint2(h, t - t0);
        if (h < hb && t1 > t0 && off[z0 + h + 1] - off[z0 + h] > small) {
            const unsigned b = atomicAdd(nbig, t1 - t0);
            for (uint32_t t = t0; t < t1; ++t) big[b + t - t0] = make_uint2(h, t - t0);
        }
    }
}

#ifndef TC_VHUB_WPT
#define TC_VHUB_WPT 2  // in-edges per thread per window of k_count_vhub (window = WPT * NT)
#endif
#ifndef TC_VM_MINB
// 5 CTAs per SM (48 registers): with the hub heads in k_count_vhub this kernel only runs the
// long low-zone lists, latency-bound (ncu 10.5 -> 9.8 ms at s26; 4 CTAs: 10.6 ms)
#define TC_VM_MINB 5
#endif
#if TC_VM_MINB > 0
#define TC_VM_BOUNDS(nt) __launch_bounds__(nt, TC_VM_MINB)
#else
#define TC_VM_BOUNDS(nt) __launch_bounds__(nt)
#endif
template <int NT, int U>
__global__ void TC_VM_BOUNDS(NT)
    k_count_vmajor(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                   const uint32_t *__restrict__ off, const uint32_t *__restrict__ hubstart,
                   uint32_t z0, uint32_t hz, uint32_t hwp, uint32_t cap,
                   const uint32_t *__restrict__ start, const uint32_t *__restrict__ fillc,
                   const uint2 *__restrict__ in_e,
                   const uint2 *__restrict__ tasks, const uint32_t *__restrict__ tlo,
                   const uint32_t *__restrict__ ntasks, unsigned *__restrict__ next,
                   const HubPack hp, unsigned long long *__restrict__ total) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(smem);  // hwp words
    uint32_t *ctab = bitmap + hwp;                           // cap slots (v below hz)
    constexpr int VWPT = TC_VHUB_WPT;
    constexpr uint32_t VWIN = (uint32_t)NT * VWPT;
    __shared__ uint32_t s_cb[VWIN], s_vs[VWIN], s_ve[VWIN];
    __shared__ uint32_t s_cst[VWIN + 4];
    __shared__ uint32_t s_scan[32];
    __shared__ unsigned s_task, s_fail;
    constexpr int NW = NT / 32;
    const unsigned warp = threadIdx.x >> 5;
    const unsigned nt = *ntasks, t0 = *tlo;
    const EdgeTable<uint32_t> et{s_cb, s_vs, s_ve, s_cst, nullptr};
    // shared addresses in registers (opaque moves: no SR_CgaCtaId rebuild at every use)
    uint32_t bm, tb;
    asm volatile("mov.b32 %0, %1;" : "=r"(bm) : "r"(smem_addr(bitmap)));
    asm volatile("mov.b32 %0, %1;" : "=r"(tb) : "r"(smem_addr(s_cb)));
    const EdgeTableSA eta{tb, tb + (smem_addr(s_vs) - smem_addr(s_cb)), tb + (smem_addr(s_ve) - smem_addr(s_cb)),
                          tb + (smem_addr(s_cst) - smem_addr(s_cb))};
    unsigned long long acc = 0;
    for (;;) {
        if (threadIdx.x == 0) s_task = t0 + atomicAdd(next, 1u);
        __syncthreads();
        const unsigned t = s_task;
        if (t >= nt) break;
        const uint2 task = tasks[t];
        const uint32_t h = task.x, v = z0 + h;
        const uint32_t vs = __ldg(off + v), ve = __ldg(off + v + 1);
        // hub part of adj(v) -> bitmap over hub words [ws, hwp); below the hub zone the
        // non-hub prefix [vs, hs) goes into a cuckoo table
        const uint32_t hs = v >= hz ? vs : __ldg(hubstart + v);
        const uint32_t nh = hs - vs;
        const uint32_t ws = v >= hz ? ((v + 1 - hz) >> 5) & ~3u : 0u;
        for (uint32_t i = ws + 4 * threadIdx.x; i < hwp; i += 4 * NT)
            *reinterpret_cast<uint4 *>(bitmap + i) = make_uint4(0, 0, 0, 0);
        Cuckoo32 ck{bm + 4 * hwp, 4 * nh < cap ? 4 * nh : cap, 0, 0};  // ctab = bitmap + hwp
        bool tab_ok = true;
        if (nh) {
            tab_ok = false;
            for (uint32_t seed = 0; seed < kCuckooSeeds && !tab_ok; ++seed) {
                ck.c1 = seed_mult(seed, 0);
                ck.c2 = seed_mult(seed, 1);
                for (uint32_t i = threadIdx.x; i < ck.T; i += NT) ctab[i] = kEmpty;
                if (threadIdx.x == 0) s_fail = 0;
                __syncthreads();
                for (uint32_t i = vs + threadIdx.x; i < hs; i += NT)
                    if (!cuckoo_insert32(ctab, ck, __ldg(dst + i))) s_fail = 1;
                __syncthreads();
                tab_ok = s_fail == 0;
                __syncthreads();
            }
        }
        __syncthreads();
        for (uint32_t i = hs + threadIdx.x; i < ve; i += NT) {
            const uint32_t r = __ldg(dst + i) - hz;
            atomicOr(bitmap + (r >> 5), 1u << (r & 31));
        }
        __syncthreads();
        const uint32_t p0 = __ldg(start + h) + task.y * kVChunk;
        // fill count, clamped to the slot range (an overflowed capacity layout is recounted)
        const uint32_t p1 = min(p0 + kVChunk, min(__ldg(start + h) + __ldg(fillc + h), __ldg(start + h + 1)));
        // windows of WPT * NT in-edges, WPT consecutive entries per thread (as k_count_vhub)
        uint2 ie_n[VWPT];
#pragma unroll
        for (int i = 0; i < VWPT; ++i) {
            const uint32_t j = p0 + VWPT * threadIdx.x + i;
            ie_n[i] = j < p1 ? __ldg(in_e + j) : make_uint2(0u, 0u);
        }
        for (uint32_t ps = p0; ps < p1; ps += VWIN) {
            const uint32_t nwin = min(VWIN, p1 - ps);
            uint32_t ch[VWPT], av[VWPT], bv[VWPT], csum = 0;
#pragma unroll
            for (int i = 0; i < VWPT; ++i) {
                const uint2 ie = ie_n[i];  // (edge, end of adj(u)); the next window's is loaded now
                const uint32_t jn = ps + VWIN + VWPT * threadIdx.x + i;
                ie_n[i] = jn < p1 ? __ldg(in_e + jn) : make_uint2(0u, 0u);
                const bool ok = VWPT * threadIdx.x + i < nwin;
                av[i] = ok ? ie.x + 1 : 0u;
                bv[i] = ok ? ie.y : 0u;
                ch[i] = ok ? (bv[i] - (av[i] & ~3u) + 3) >> 2 : 0u;  // a < b by construction
                csum += ch[i];
            }
            uint32_t tot;
            uint32_t run = block_exclusive_scan<uint32_t>(csum, s_scan, &tot);
#pragma unroll
            for (int i = 0; i < VWPT; ++i) {
                const uint32_t j = VWPT * threadIdx.x + i;
                s_cb[j] = (av[i] & ~3u) - 4 * run;
                s_vs[j] = av[i];
                s_ve[j] = bv[i];
                s_cst[j] = run;
                run += ch[i];
            }
            if (threadIdx.x == 0) s_cst[VWIN] = tot;
            __syncthreads();
            const uint32_t c0 = (uint32_t)((uint64_t)tot * warp / NW);
            const uint32_t c1 = (uint32_t)((uint64_t)tot * (warp + 1) / NW);
            if (c0 < c1) {
                // suffix items are > v: hub items hit words >= ws (staged); non-hub items
                // (only when v < hz) are looked up in the cuckoo table
                if (v < hz && tab_ok) {  // suffix items below hz exist: bitmap or cuckoo per item
                    acc += sweep_sa<U>(dst, eta, VWIN, c0, c1, [&](uint32_t w) {
                        const uint32_t r = w - hz;
                        const bool b = ((lds32(bm + 4 * min(r >> 5, hwp - 1)) >> (r & 31)) & 1u) != 0u;
                        return w >= hz ? b : (nh != 0 && ck.contains(w));
                    });
                } else if (v < hz) {  // cuckoo build failed: binary search of the non-hub part
                    acc += sweep<uint32_t, false, U>(dst, et, VWIN, c0, c1, [&](uint32_t w, uint32_t) {
                        const uint32_t r = w - hz;
                        const bool b = ((lds32(bm + 4 * min(r >> 5, hwp - 1)) >> (r & 31)) & 1u) != 0u;
                        return w >= hz ? b : sorted_contains(dst + vs, nh, w);
                    });
                } else if (hp.lo16) {
                    // suffix items exceed v >= hz: every valid item is a hub item, read from
                    // the 18-bit packed copy (2.25 B per item)
                    acc += sweep_bits18<TC_PACK_U>(hp, et, VWIN, c0, c1, bitmap);
                } else {
                    acc += sweep_bits<U>(dst, et, VWIN, c0, c1, bitmap, hz);
                }
            }
            __syncthreads();
        }
    }
    block_add_total(acc, total);
}

// ------------------------------------------------------- v-major, hub heads ---
// Hub heads v >= hz: the same per-head schedule as k_count_vmajor, with a leaner item sweep.
//  * No per-item bounds: the flattened sweep covers only the whole aligned chunks of each
//    suffix [a, b) (16 bytes, or 32 bytes of 16-bit items); the < 1 chunk of items before
//    the first and after the last whole chunk are probed one by one by the thread that owns
//    the in-edge.  The hot loop is load, shift, mask, LDS, shift, add.
//  * Heads in the top 2^16 ranks (t16 = n - 2^16): every suffix item after v lies in
//    [t16, n), so the suffixes are read from a 16-bit copy of edge_dst (lo16[p] = dst[p] -
//    t16; 2 B per item, 8 items per 16-byte chunk) against a 2^16-bit bitmap (8 KB).  At
//    R-MAT s26 these heads carry 52 % of the hub-head suffix items (scripts/hub16_stats.py).

__device__ __forceinline__ uint32_t bit16(const unsigned char *bm, uint32_t x) {
    // item x (16-bit): word x >> 5 at byte (x >> 3) & ~3 (x < 2^16), bit x & 31
    return (*reinterpret_cast<const uint32_t *>(bm + ((x >> 3) & 0x1ffcu)) >> (x & 31u)) & 1u;
}

__device__ __forceinline__ uint32_t bit32(const unsigned char *bm, uint32_t w, uint32_t hz, uint32_t amask) {
    const uint32_t r = w - hz;
    return (*reinterpret_cast<const uint32_t *>(bm + ((r >> 3) & amask)) >> (r & 31u)) & 1u;
}

// Chunk c of the window belongs to the in-edge k with cst[k] <= c < cst[k+1]; its items are
// at element cb[k] + E c (E = items per 16-byte chunk).  Lanes past c1 count nothing.
// Software-pipelined: the U chunks of the next round are in flight while this round's items
// are probed, and all shared-memory probes of a round are issued before their results are
// used (the probe chain LDS -> shift -> add is latency-bound otherwise).
// A chunk is CW consecutive 32-bit words: 16-bit items come in 32-byte chunks (16 items, one
// 256-bit load), 32-bit items in 16-byte chunks (4 items).
#ifndef TC_B16W
#define TC_B16W 8  // words per 16-bit chunk: 4 (16 B, 8 items) or 8 (32 B, one 256-bit load)
#endif
template <bool B16>
struct ChunkT {
    static constexpr int CW = B16 ? TC_B16W : 4;               // words per chunk
    static constexpr uint32_t E = B16 ? 2u * TC_B16W : 4u;      // items per chunk
    uint32_t w[CW];
};

template <bool B16>
__device__ __forceinline__ void ldg_chunk(const void *arr, uint32_t p, ChunkT<B16> &q) {
    if (B16 && ChunkT<B16>::CW == 4) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(static_cast<const uint16_t *>(arr) + p));
        q.w[0] = v.x;
        q.w[1] = v.y;
        q.w[2] = v.z;
        q.w[3] = v.w;
    } else if (B16) {
        const uint16_t *a = static_cast<const uint16_t *>(arr) + p;  // 32-byte aligned
        asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(q.w[0]), "=r"(q.w[1]), "=r"(q.w[2]), "=r"(q.w[3]), "=r"(q.w[4]), "=r"(q.w[5]),
                       "=r"(q.w[6]), "=r"(q.w[7])
                     : "l"(a));
    } else {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(static_cast<const uint32_t *>(arr) + p));
        q.w[0] = v.x;
        q.w[1] = v.y;
        q.w[2] = v.z;
        q.w[3] = v.w;
    }
}

// Chunk c of the window belongs to the in-edge k with cst[k] <= c < cst[k+1]; its items are
// at element cb[k] + E c.  Lanes past c1 count nothing.  Software-pipelined: the U chunks
// of the next round are in flight while this round's items are probed, and all
// shared-memory probes of a round are issued before their results are used (the probe
// chain LDS -> shift -> add is latency-bound otherwise).
// TC_VHUB_SA: the bitmap and the window table are addressed through 32-bit shared
// addresses computed once per kernel (bm32, a_cb, a_cst): without them the compiler
// rebuilds the CTA's shared-window base (S2R SR_CgaCtaId) for every cursor advance and
// adds it to every probe address.
#ifndef TC_VHUB_SA
#define TC_VHUB_SA 1
#endif
#ifndef TC_VHUB_ALIGN
#define TC_VHUB_ALIGN 1
#endif
template <int U, bool B16>
__device__ __forceinline__ uint32_t sweep_nomask(const void *__restrict__ arr, const uint32_t *s_cb,
                                                 const uint32_t *s_cst, uint32_t nwin, uint32_t c0, uint32_t c1,
                                                 const unsigned char *bm, uint32_t hz, uint32_t amask,
                                                 uint32_t bm32, uint32_t a_cb, uint32_t a_cst) {
#if TC_VHUB_SA
    auto cst_at = [&](uint32_t i) { return lds32(a_cst + 4 * i); };
    auto cb_at = [&](uint32_t i) { return lds32(a_cb + 4 * i); };
#else
    auto cst_at = [&](uint32_t i) { return s_cst[i]; };
    auto cb_at = [&](uint32_t i) { return s_cb[i]; };
    (void)bm32;
    (void)a_cb;
    (void)a_cst;
#endif
    using Q = ChunkT<B16>;
    constexpr uint32_t E = Q::E;
    constexpr int NIC = (int)E;   // items per chunk
    constexpr int NI = NIC * U;   // items per lane per round
    const unsigned lane = lane_id();
    uint32_t k = 0;
    {
        const uint32_t c = c0 + lane < c1 ? c0 + lane : c1 - 1;
        uint32_t a = 0, b = nwin;
        while (b - a > 1) {
            const uint32_t mid = (a + b) >> 1;
            if (cst_at(mid) <= c) a = mid; else b = mid;
        }
        k = a;
    }
    uint32_t nextb = cst_at(k + 1), cb = cb_at(k);
    auto fetch = [&](uint32_t base, Q (&q)[U], uint32_t &live) {
        live = 0;
#pragma unroll
        for (int j = 0; j < U; ++j) {
            uint32_t c = base + j * 32 + lane;
            live |= (c < c1 ? 1u : 0u) << j;
            c = c < c1 ? c : c1 - 1;
            if (c >= nextb) {
                do { nextb = cst_at(++k + 1); } while (c >= nextb);
                cb = cb_at(k);
            }
#ifdef TC_VHUB_NOLOAD  // diagnostic build: no suffix loads (items synthesised)
#pragma unroll
            for (int i = 0; i < Q::CW; ++i) q[j].w[i] = (cb + E * c) * 2654435761u + i;
#else
            ldg_chunk<B16>(arr, cb + E * c, q[j]);
#endif
        }
    };
    auto probe = [&](const Q (&q)[U], uint32_t live) -> uint32_t {
        uint32_t ad[NI], sh[NI], wd[NI];
#pragma unroll
        for (int j = 0; j < U; ++j) {
#pragma unroll
            for (int i = 0; i < Q::CW; ++i) {
                const uint32_t x = q[j].w[i];
                if (B16) {
#if TC_VHUB_SA && TC_VHUB_ALIGN
                    ad[NIC * j + 2 * i] = ((x >> 3) & 0x1ffcu) | bm32;  // bm32: 8 KB aligned
                    ad[NIC * j + 2 * i + 1] = ((x >> 19) & 0x1ffcu) | bm32;
#else
                    ad[NIC * j + 2 * i] = (x >> 3) & 0x1ffcu;
                    ad[NIC * j + 2 * i + 1] = (x >> 19) & 0x1ffcu;
#endif
                    sh[NIC * j + 2 * i] = x;
                    sh[NIC * j + 2 * i + 1] = x >> 16;
                } else {
                    const uint32_t r = x - hz;
                    ad[NIC * j + i] = (r >> 3) & amask;
                    sh[NIC * j + i] = r;
                }
            }
        }
#pragma unroll
        for (int t = 0; t < NI; ++t)
#ifdef TC_VHUB_NOPROBE  // diagnostic build: no shared-memory probes
            wd[t] = ad[t];
#else
#if TC_VHUB_SA
            wd[t] = lds32(B16 && TC_VHUB_ALIGN ? ad[t] : bm32 + ad[t]);
#else
            wd[t] = *reinterpret_cast<const uint32_t *>(bm + ad[t]);
#endif
#endif
        uint32_t f = 0;
#pragma unroll
        for (int j = 0; j < U; ++j) {
            uint32_t h = 0;
#pragma unroll
            for (int t = 0; t < NIC; ++t) h += (wd[j * NIC + t] >> (sh[j * NIC + t] & 31u)) & 1u;
            f += ((live >> j) & 1u) ? h : 0u;
        }
        return f;
    };
    uint32_t found = 0;
    Q qa[U], qb[U];
    uint32_t la = 0, lb = 0;
    fetch(c0, qa, la);
    for (uint32_t base = c0;;) {
        const uint32_t nb = base + 32 * U;
        if (nb < c1) fetch(nb, qb, lb);  // warp-uniform
        found += probe(qa, la);
        if (nb >= c1) break;
        base = nb + 32 * U;
        if (base < c1) fetch(base, qa, la);
        found += probe(qb, lb);
        if (base >= c1) break;
    }
    return found;
}

// BT: tasks are (head, first, end) index ranges (the source-blocked top-band tasks);
// otherwise (head, chunk) as in k_count_vmajor.
#ifdef TC_VHUB_MINB
#define TC_VHUB_BOUNDS(nt) __launch_bounds__(nt, TC_VHUB_MINB)
#else
#define TC_VHUB_BOUNDS(nt) __launch_bounds__(nt)
#endif
template <int NT, int U, bool BT>
__global__ void TC_VHUB_BOUNDS(NT)
    k_count_vhub(const uint32_t *__restrict__ dst, const uint16_t *__restrict__ lo16,
                 const uint32_t *__restrict__ off, uint32_t z0, uint32_t hz, uint32_t t16, uint32_t hwp,
                 uint32_t amask, const uint32_t *__restrict__ start, const uint32_t *__restrict__ fillc,
                 const uint2 *__restrict__ in_e, const void *__restrict__ tasks,
                 const uint32_t *__restrict__ tlo, const uint32_t *__restrict__ ntasks,
                 unsigned *__restrict__ next, unsigned long long *__restrict__ total) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
#if TC_VHUB_ALIGN
    // the bitmap starts on an 8 KB boundary: a 16-bit item's probe address is one LOP3
    // ((x >> 3) & 0x1ffc | base) instead of mask + add
    unsigned char *smem = smem_raw + ((0u - smem_addr(smem_raw)) & 8191u);
#else
    unsigned char *smem = smem_raw;
#endif
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(smem);  // (amask + 4) / 4 words
    constexpr int WPT = TC_VHUB_WPT;
    constexpr uint32_t WIN = (uint32_t)NT * WPT;
    __shared__ uint32_t s_cb[WIN];
    __shared__ uint32_t s_cst[WIN + 4];
    __shared__ uint32_t s_scan[32];
    __shared__ unsigned s_task;
    constexpr int NW = NT / 32;
    // shared addresses held in registers (opaque moves: otherwise the compiler rebuilds the
    // shared-window base from SR_CgaCtaId at every use)
    uint32_t bm32, a_cb;
    asm volatile("mov.b32 %0, %1;" : "=r"(bm32) : "r"(smem_addr(smem)));
    asm volatile("mov.b32 %0, %1;" : "=r"(a_cb) : "r"(smem_addr(s_cb)));
    const uint32_t a_cst = a_cb + (smem_addr(s_cst) - smem_addr(s_cb));
    const unsigned warp = threadIdx.x >> 5;
    const unsigned nt = *ntasks, t0 = *tlo;
    // the probes of outside items may read any word of the allocation: define them all
    for (uint32_t i = threadIdx.x; i < (amask + 4) / 4 || i < kT16 / 32; i += NT) bitmap[i] = 0;
    unsigned long long acc = 0;
    for (;;) {
        if (threadIdx.x == 0) s_task = t0 + atomicAdd(next, 1u);
        __syncthreads();
        const unsigned t = s_task;
        if (t >= nt) break;
        uint32_t h, p0, p1;
        if (BT) {
            const uint4 task = static_cast<const uint4 *>(tasks)[t];
            h = task.x;
            p0 = task.y;
            p1 = task.z;
        } else {
            const uint2 task = static_cast<const uint2 *>(tasks)[t];
            h = task.x;
            p0 = __ldg(start + h) + task.y * kVChunk;
            // fill count, clamped to the slot range (an overflowed capacity layout is recounted)
            p1 = min(p0 + kVChunk, min(__ldg(start + h) + __ldg(fillc + h), __ldg(start + h + 1)));
        }
        const uint32_t v = z0 + h;
        const uint32_t vs = __ldg(off + v), ve = __ldg(off + v + 1);
        const bool b16 = v >= t16;  // block-uniform
        const uint32_t base = b16 ? t16 : hz;
        const uint32_t wend = b16 ? kT16 / 32 : hwp;
        const uint32_t ws = ((v + 1 - base) >> 5) & ~3u;
        for (uint32_t i = ws + 4 * threadIdx.x; i < wend; i += 4 * NT)
            *reinterpret_cast<uint4 *>(bitmap + i) = make_uint4(0, 0, 0, 0);
        __syncthreads();
        for (uint32_t i = vs + threadIdx.x; i < ve; i += NT) {
            const uint32_t r = __ldg(dst + i) - base;
            atomicOr(bitmap + (r >> 5), 1u << (r & 31));
        }
        __syncthreads();
        // windows of WPT * NT in-edges, WPT consecutive entries per thread (fewer barriers and
        // scans per item); the next window's entries are loaded while this one is swept
        uint2 ie_n[WPT];
#pragma unroll
        for (int i = 0; i < WPT; ++i) {
            const uint32_t j = p0 + WPT * threadIdx.x + i;
            ie_n[i] = j < p1 ? __ldg(in_e + j) : make_uint2(0u, 0u);
        }
        for (uint32_t ps = p0; ps < p1; ps += WIN) {
            const uint32_t nwin = min(WIN, p1 - ps);
            uint32_t ch[WPT], Fv[WPT];
            uint2 ie[WPT];
#pragma unroll
            for (int i = 0; i < WPT; ++i) {
                ie[i] = ie_n[i];
                const uint32_t j = ps + WIN + WPT * threadIdx.x + i;
                ie_n[i] = j < p1 ? __ldg(in_e + j) : make_uint2(0u, 0u);
            }
            uint32_t csum = 0;
#pragma unroll
            for (int i = 0; i < WPT; ++i) {
                ch[i] = 0;
                Fv[i] = 0;
                if (WPT * threadIdx.x + i < nwin) {
                    // whole aligned chunks [A, B) of the suffix [a, b) go to the sweep; the few
                    // items of [a, A) and [B, b) (< one chunk each) are probed here, one by one
                    const uint32_t a = ie[i].x + 1, b = ie[i].y;  // a < b by construction
                    const uint32_t E = b16 ? ChunkT<true>::E : ChunkT<false>::E;
                    const uint32_t A = (a + E - 1) & ~(E - 1), B = b & ~(E - 1);
                    uint32_t lead_end = b, tail_begin = b;  // no whole chunk: every item here
                    if (A < B) {
                        Fv[i] = A;
                        ch[i] = (B - A) / E;
                        lead_end = A;
                        tail_begin = B;
                    }
                    uint32_t x = 0;
                    if (b16) {
                        for (uint32_t p = a; p < lead_end; ++p) x += bit16(smem, __ldg(lo16 + p));
                        for (uint32_t p = tail_begin; p < b; ++p) x += bit16(smem, __ldg(lo16 + p));
                    } else {
                        for (uint32_t p = a; p < lead_end; ++p) x += bit32(smem, __ldg(dst + p), hz, amask);
                        for (uint32_t p = tail_begin; p < b; ++p) x += bit32(smem, __ldg(dst + p), hz, amask);
                    }
                    acc += x;
                }
                csum += ch[i];
            }
            uint32_t tot;
            uint32_t run = block_exclusive_scan<uint32_t>(csum, s_scan, &tot);
#pragma unroll
            for (int i = 0; i < WPT; ++i) {
                const uint32_t j = WPT * threadIdx.x + i;
                s_cb[j] = Fv[i] - (b16 ? ChunkT<true>::E : ChunkT<false>::E) * run;
                s_cst[j] = run;
                run += ch[i];
            }
            if (threadIdx.x == 0) s_cst[WIN] = tot;
            __syncthreads();
            const uint32_t c0 = (uint32_t)((uint64_t)tot * warp / NW);
            const uint32_t c1 = (uint32_t)((uint64_t)tot * (warp + 1) / NW);
            if (c0 < c1) {
                if (b16)
                    acc += sweep_nomask<TC_B16W == 4 ? U : (U + 1) / 2, true>(lo16, s_cb, s_cst, WIN, c0, c1, smem, hz,
                                                                              amask, bm32, a_cb, a_cst);
                else acc += sweep_nomask<U, false>(dst, s_cb, s_cst, WIN, c0, c1, smem, hz, amask, bm32, a_cb, a_cst);
            }
            __syncthreads();
        }
    }
    block_add_total(acc, total);
}

// Source blocks for the top-band heads.  Their suffix streams (2 B per item) re-read each
// source's band items once per head it points to (R-MAT s26: ~140 reads per item).  Tasks
// ordered (source block, head) keep the streams of one block of edge_dst -- ~1/nb of the
// band data -- in L2 while every head's bitmap is staged once per block.  The fill appends
// in-edges roughly in edge order (grid-stride over edges), so a head's list is split at the
// block bounds by binary search on the edge index; splits are made monotone, so the tasks
// partition every list whatever the order (exactness never depends on it).
__global__ void k_band_splits(const uint32_t *__restrict__ start, const uint32_t *__restrict__ fillc,
                              const uint2 *__restrict__ in_e, uint32_t h16, uint32_t nb16, uint32_t nb,
                              uint64_t bsize, uint32_t *__restrict__ spl, uint32_t *__restrict__ cnt) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb16; i += stride) {
        const uint32_t h = h16 + i;
        const uint32_t P0 = start[h], P1 = min(start[h] + fillc[h], start[h + 1]);
        uint32_t prev = P0;
        spl[(size_t)i * (nb + 1)] = P0;
        for (uint32_t S = 1; S <= nb; ++S) {
            uint32_t q = P1;
            if (S < nb) {
                const uint64_t E = (uint64_t)S * bsize;
                uint32_t a = prev, n2 = P1 - prev;  // first position with edge >= E
                while (n2 > 0) {
                    const uint32_t hh = n2 >> 1;
                    if ((uint64_t)in_e[a + hh].x < E) { a += hh + 1; n2 -= hh + 1; } else n2 = hh;
                }
                q = a;
            }
            spl[(size_t)i * (nb + 1) + S] = q;
            cnt[(size_t)(S - 1) * nb16 + i] = (q - prev + kVChunk - 1) / kVChunk;
            prev = q;
        }
    }
}

// tasks (head, first, end, 0) in (block, head) order from the scanned counts
__global__ void k_band_tasks(const uint32_t *__restrict__ spl, const uint32_t *__restrict__ tst,
                             uint32_t h16, uint32_t nb16, uint32_t nb, uint4 *__restrict__ tasks) {
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t N = nb16 * nb;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += stride) {
        const uint32_t S = j / nb16, i = j - S * nb16;
        const uint32_t lo = spl[(size_t)i * (nb + 1) + S], hi = spl[(size_t)i * (nb + 1) + S + 1];
        for (uint32_t t = tst[j]; t < tst[j + 1]; ++t) {
            const uint32_t a = lo + (t - tst[j]) * kVChunk;
            tasks[t] = make_uint4(h16 + i, a, min(a + kVChunk, hi), 0u);
        }
    }
}

// 16-bit copy of edge_dst for the top-2^16 heads: lo16[p] = dst[p] - t16 (mod 2^16; only
// items >= t16 are ever counted).  dst is padded to a multiple of 4 + 4.
__global__ void __launch_bounds__(256) k_pack16(const uint32_t *__restrict__ dst, uint64_t m, uint32_t t16,
                                                uint16_t *__restrict__ lo16) {
    const uint64_t ng = (m + 3) / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += stride) {
        const uint4 w = __ldg(reinterpret_cast<const uint4 *>(dst) + g);
        reinterpret_cast<uint2 *>(lo16)[g] = make_uint2(((w.x - t16) & 0xffffu) | ((w.y - t16) << 16),
                                                       ((w.z - t16) & 0xffffu) | ((w.w - t16) << 16));
    }
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
// RANKED (rank-space count schedule): an edge costs about min(|suffix of adj(u) after v|,
// |adj(v)|) -- the per-edge v-major/u-major choice reads the cheaper side -- plus a
// constant; otherwise the reference merge work d+(u) + d+(v).
template <typename OffT, bool RANKED = false>
__global__ void __launch_bounds__(256) k_tile_work(const uint32_t *__restrict__ src,
                                                   const uint32_t *__restrict__ dst,
                                                   const OffT *__restrict__ off, uint64_t m,
                                                   uint64_t tile, uint32_t overhead,
                                                   unsigned long long *__restrict__ sums,
                                                   uint32_t ucap = 0xffffffffu) {
    const uint64_t b = (uint64_t)blockIdx.x * tile;
    const uint64_t e = b + tile < m ? b + tile : m;
    unsigned long long acc = 0;
    for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        const uint32_t u = src[i], v = dst[i];
        const unsigned long long dv = (unsigned long long)(off[v + 1] - off[v]);
        if (RANKED) {
            const unsigned long long suf = (unsigned long long)(off[u + 1] - (OffT)i - 1);
            acc += (suf < dv ? suf : dv) + overhead;
        } else {
            const unsigned long long du = (unsigned long long)(off[u + 1] - off[u]);
            acc += (du < ucap ? du : ucap) + dv + overhead;
        }
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

// Dynamic shared memory of a heavy class: the table for the largest d+(u) in the class.
size_t heavy_smem(int cls, uint32_t max_out) {
    if (kClassCap[cls] == 0) return (size_t)4 * max_out;
    const uint32_t dmax = max_out < kClassMax[cls] ? max_out : kClassMax[cls];
    const uint64_t slots = 4ull * dmax < kClassCap[cls] ? 4ull * dmax : kClassCap[cls];
    return (size_t)4 * slots;
}

static uint32_t vzone_start(const DeviceGraph &g) { return vzone_start_of(g.n, g.hz); }

static uint32_t dense_factor_env() {
    return (uint32_t)opts().dense_factor;
}

}  // namespace

// The v-major split every kernel of one count evaluates (the same predicate everywhere, so
// each edge is counted exactly once).
VSplit make_vsplit(const DeviceGraph &g, bool vmajor) {
    VSplit vp{vmajor ? vzone_start(g) : 0xffffffffu, g.hz, g.vt, g.hwp, dense_factor_env(), kVNonHubCap,
              (uint32_t)opts().vm_bias, (uint32_t)opts().vlow_all, g.hubstart};
    vp.packed = vmajor && opts().hubpack ? 1u : 0u;
    vp.packed_cost = vmajor && opts().hubpack == 1 ? 1u : 0u;  // 2: packed reads, 4-byte costs
    if (vmajor && !vp.packed && opts().vhub) {
        vp.t16 = g.n - g.hz > kT16 ? (uint32_t)(g.n - kT16) : g.hz;
        vp.b16w = (uint32_t)(opts().vhub_b16w > 0 ? opts().vhub_b16w : 4);
    }
    return vp;
}

bool vsplit_same(const VSplit &a, const VSplit &b) {
    return a.z0 == b.z0 && a.hz == b.hz && a.vt == b.vt && a.hwp == b.hwp && a.factor == b.factor &&
           a.nhcap == b.nhcap && a.bias == b.bias && a.lowall == b.lowall && a.hubstart == b.hubstart &&
           a.packed == b.packed && a.packed_cost == b.packed_cost && a.t16 == b.t16 && a.b16w == b.b16w;
}

bool vmajor_schedule(const DeviceGraph &g) {
    const int64_t vm_env = opts().vmajor;
    bool vmajor = vm_env != 0 && g.off32 && g.rank_space && g.hubstart && g.n > g.hz &&
                  (vm_env == 1 || (g.m >= (1ull << 27) && g.max_out > 256));
    const uint32_t lower[kClasses] = {(uint32_t)kLightMax, kClassMax[0], kClassMax[1], kClassMax[2]};
    for (int c = 0; c < kClasses && vmajor; ++c)
        if (g.max_out > lower[c] &&
            4 * ((size_t)g.hwp + 3 * (g.max_out < kClassMax[c] ? g.max_out : kClassMax[c])) > 200 * 1024)
            vmajor = false;
    return vmajor;
}

namespace {

template <int NT>
int launch_hub(const DeviceGraph &g, const RangeDev *rg, const uint2 *tasks, const unsigned *ntasks,
               unsigned *next, uint32_t cap, bool vmajor, int share, HubPack hp,
               unsigned long long *d_total, cudaStream_t s) {
    const uint32_t hwords = g.hwp;
    const size_t sm = 4 * ((size_t)hwords + cap);
    const int64_t unroll = opts().hub_unroll;
    auto kern = unroll >= 4 ? k_count_hub<NT, 4> : unroll == 3 ? k_count_hub<NT, 3> : k_count_hub<NT, 2>;
    TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int per_sm = 1;
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, sm));
    per_sm = (per_sm + share - 1) / share;
    if (per_sm < 1) per_sm = 1;
    const uint32_t dense_factor = dense_factor_env();
    const VSplit vp = make_vsplit(g, vmajor);
    kern<<<kSMs * per_sm, NT, sm, s>>>(g.dst, g.off32, g.hubstart, g.hz, hwords, g.vt, g.dense_off,
                                       g.dense_bits, dense_factor, vp, rg, tasks, ntasks, next, cap,
                                       vp.packed ? hp : HubPack{nullptr, nullptr}, d_total);
    TC_LAUNCHED();
    return 0;
}

template <typename OffT, int MODE, int NT>
int launch_heavy(const DeviceGraph &g, const OffT *off, const RangeDev *rg, const uint2 *tasks,
                 const unsigned *ntasks, unsigned *next, uint32_t cap, size_t sm,
                 unsigned long long *d_total, cudaStream_t s) {
    auto kern = k_count_heavy<OffT, MODE, NT>;
    TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int per_sm = 1;
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, sm));
    if (per_sm < 1) per_sm = 1;
    kern<<<kSMs * per_sm, NT, sm, s>>>(g.dst, off, rg, tasks, ntasks, next, cap, d_total);
    TC_LAUNCHED();
    return 0;
}

// L2 persisting window over the last l2_persist_mb (default 32; 0 = off) of dense_bits:
// -2 % count time at R-MAT s26 (522 -> 511 ms); larger windows starve the rest of L2.
static size_t l2_window_bytes() {
    const int64_t mb = opts().l2_persist_mb;
    return mb > 0 ? (size_t)mb << 20 : 0;
}

static bool apply_l2_window(const DeviceGraph &g, cudaStream_t s) {
    size_t want = l2_window_bytes();
    // l2_target: 0 = tail of the dense-hub bitmaps, 1 = tail of edge_dst (the adjacency
    // lists of the top-ranked sources, whose suffixes the v-major kernel re-reads most)
    const int64_t target = opts().l2_target;
    const char *base = target == 1 ? reinterpret_cast<const char *>(g.dst)
                                   : reinterpret_cast<const char *>(g.dense_bits);
    const size_t tbytes = target == 1 ? (size_t)g.m * 4 : (size_t)g.dense_words * 4;
    if (!want || !base || !tbytes) return false;
    int dev = 0, maxwin = 0, maxpersist = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    cudaDeviceGetAttribute(&maxpersist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    const size_t total = tbytes;
    if (want > total) want = total;
    if (want > (size_t)maxwin) want = (size_t)maxwin;
    if (want > (size_t)maxpersist) want = (size_t)maxpersist;
    if (!want) return false;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) return false;
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.base_ptr = const_cast<char *>(base) + ((total - want) & ~(size_t)127);
    v.accessPolicyWindow.num_bytes = want;
    v.accessPolicyWindow.hitRatio = 1.0f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    return cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess;
}

static void clear_l2_window(cudaStream_t s) {
    cudaStreamSynchronize(s);  // the count kernels ran under the window
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);  // give the carve-out back
}

// v-major heads below the hub zone (|adj(v)| <= kVNonHubCap): ONE WARP per task (v, chunk
// of in-edges), adj(v) in a per-warp cuckoo table, the suffixes of the in-edges flattened
// over the lanes and probed.  These heads have small in-degrees, so many small independent
// tasks are in flight per SM (no block barriers).
constexpr int kVlWarps = 8;
#ifndef TC_VL_LOADINV
#define TC_VL_LOADINV 2  // 2: 4 KB per warp, 6 CTAs per SM (3: 6 KB, 4 CTAs; s26 vlow 27 -> 23 ms)
#endif
constexpr uint32_t kVlLoadInv = TC_VL_LOADINV;  // per-warp cuckoo table load <= 1/kVlLoadInv
constexpr uint32_t kVlSlots = kVlLoadInv * kVNonHubCap;  // cuckoo load <= 1/3: 4 CTAs per SM

// FB = false: the cuckoo path; a task whose table cannot be built is deferred (its index
// appended to `defer`).  FB = true: the deferred tasks, probed by binary search of the sorted
// adj(v) -- a separate instantiation so the hot kernel carries no fallback code.
template <bool FB>
__global__ void __launch_bounds__(32 * kVlWarps)
    k_count_vlow_warp(const uint32_t *__restrict__ dst, const uint32_t *__restrict__ off, uint32_t z0,
                      const uint32_t *__restrict__ start, const uint32_t *__restrict__ fillc,
                      const uint2 *__restrict__ in_e,
                      const uint2 *__restrict__ tasks, const uint32_t *__restrict__ ntasks,
                      unsigned *__restrict__ next, uint32_t *__restrict__ defer,
                      unsigned *__restrict__ ndefer, unsigned long long *__restrict__ total) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_cb[kVlWarps][32], s_vs[kVlWarps][32], s_ve[kVlWarps][32];
    __shared__ uint32_t s_cst[kVlWarps][36];
    const unsigned lane = lane_id(), wp = threadIdx.x >> 5;
    uint32_t *tab = reinterpret_cast<uint32_t *>(smem) + wp * kVlSlots;
    const EdgeTable<uint32_t> et{s_cb[wp], s_vs[wp], s_ve[wp], s_cst[wp], nullptr};
    const unsigned nt = FB ? *ndefer : *ntasks;
    uint32_t acc = 0;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(next, 1u);
        t = __shfl_sync(TC_FULL_MASK, t, 0);
        if (t >= nt) break;
        if (FB) t = defer[t];
        const uint2 task = tasks[t];
        const uint32_t h = task.x, v = z0 + h;
        const uint32_t vs = __ldg(off + v), ve = __ldg(off + v + 1), d = ve - vs;
        if (d > kVNonHubCap) continue;  // long list: a CTA task (warp-uniform)
        Cuckoo32 ck{smem_addr(tab), kVlLoadInv * d < kVlSlots ? kVlLoadInv * d : kVlSlots, 0, 0};
        if (!FB) {
            bool deferred = false;
            for (uint32_t seed = 0;; ++seed) {
                if (__builtin_expect(seed == kCuckooSeeds, 0)) {  // warp-uniform, practically never
                    if (lane == 0) defer[atomicAdd(ndefer, 1u)] = t;
                    deferred = true;
                    break;
                }
                ck.c1 = seed_mult(seed, 0);
                ck.c2 = seed_mult(seed, 1);
                for (uint32_t i = lane; i < ck.T; i += 32) tab[i] = kEmpty;
                __syncwarp();
                bool fail = false;
                for (uint32_t i = lane; i < d; i += 32)
                    if (!cuckoo_insert32(tab, ck, __ldg(dst + vs + i))) fail = true;
                __syncwarp();
                if (!__any_sync(TC_FULL_MASK, fail)) break;
            }
            if (deferred) continue;
        }
        const uint32_t p0 = __ldg(start + h) + task.y * kVChunk;
        // fill count, clamped to the slot range (an overflowed capacity layout is recounted)
        const uint32_t p1 = min(p0 + kVChunk, min(__ldg(start + h) + __ldg(fillc + h), __ldg(start + h + 1)));
        // the next batch of in-edges is loaded while the current one is swept
        uint2 ie_n = p0 + lane < p1 ? __ldg(in_e + p0 + lane) : make_uint2(0u, 0u);
        for (uint32_t ps = p0; ps < p1; ps += 32) {
            uint32_t a = 0, b = 0, chunks = 0;
            const uint2 ie = ie_n;
            ie_n = ps + 32 + lane < p1 ? __ldg(in_e + ps + 32 + lane) : make_uint2(0u, 0u);
            if (ps + lane < p1) {
                a = ie.x + 1;
                b = ie.y;
                chunks = (b - (a & ~3u) + 3) >> 2;
            }
            const uint32_t incl = warp_inclusive_scan(chunks);
            const uint32_t tot = __shfl_sync(TC_FULL_MASK, incl, 31);
            const uint32_t cst = incl - chunks;
            s_cb[wp][lane] = (a & ~3u) - 4 * cst;
            s_vs[wp][lane] = a;
            s_ve[wp][lane] = b;
            s_cst[wp][lane] = cst;
            if (lane == 0) s_cst[wp][32] = tot;
            __syncwarp();
            if (tot)
                acc += sweep<uint32_t, false, 2>(dst, et, 32, 0, tot, [&](uint32_t w, uint32_t) {
                    return FB ? sorted_contains(dst + vs, d, w) : ck.contains(w);
                });
            __syncwarp();
        }
    }
    block_add_total(acc, total);
}

// v-major phase: index the hub-head in-edges of [lo, hi) (on stream s) and count them
// (k_count_vmajor) on stream s2 -- concurrently with the u-major kernels when s2 != s, each
// kernel then taking a share of every SM (the v-major kernel is DRAM-bound, the u-major
// ones latency/issue-bound, so they overlap well).  vmajor_finish joins and frees.
struct VmajorState {
    uint32_t *cnt = nullptr, *start = nullptr, *tstart = nullptr;
    uint2 *in_e = nullptr;  // (edge, off[u+1]) per indexed in-edge
    uint2 *big = nullptr;   // CTA tasks of long-list heads below hz
    uint32_t *defer = nullptr;  // warp tasks whose cuckoo build failed (binary-search rerun)
    uint16_t *lo16 = nullptr;   // packed hub copy of edge_dst (HubPack)
    uint16_t *lo16t = nullptr;  // 16-bit copy of edge_dst relative to t16 (k_count_vhub)
    bool borrowed = false;      // cnt / in_e are the graph's prebuilt index (not freed here)
    uint4 *btasks = nullptr;    // source-blocked top-band tasks (k_count_vhub<.., true>)
    uint32_t *bspl = nullptr, *bcnt = nullptr, *btst = nullptr;
    uint32_t nbands = 0, nb16 = 0;
    uint8_t *hi2 = nullptr;
    bool capl = false;      // capacity layout used (overflow flag in next[2])
    unsigned *next = nullptr;
    uint2 *tasks = nullptr;
    HubPack hp{nullptr, nullptr};
    cudaEvent_t e0 = nullptr, e1 = nullptr, done = nullptr;
    cudaStream_t s2 = nullptr;
};

// v-major part 1: the in-edge index and the task lists, on s2 (forked from s).  With s2 != s
// it overlaps the u-major kernels: the fill is bound by L2 atomics, the u-major kernels by
// dependent-load latency, and neither depends on the other.
int vmajor_index(const DeviceGraph &g, const RangeDev *rg, uint64_t span, cudaStream_t s, cudaStream_t s2,
                 VmajorState *st, bool full, uint32_t hlo = 0, uint32_t hhi = 0xffffffffu) {
    const uint32_t z0 = vzone_start(g);
    const uint32_t nh = (uint32_t)(g.n - z0);  // v-major zone size
    const VSplit vp = make_vsplit(g, true);
    // full counts reuse the index the rank-space sorts filled when its split is this one
    st->borrowed = full && g.vix_ready && g.vin_cap && vsplit_same(g.vix_vp, vp);
    TC_CHECK(dalloc_t(&st->start, (size_t)nh + 1, s));
    TC_CHECK(dalloc_t(&st->tstart, (size_t)nh + 1, s));
    // capacity layout from preprocessing (in-degree prefix over the zone) when present: the
    // counting pass is skipped and in-edges land at vin_cap[v] + cursor
    const bool capl = g.vin_cap && g.vin_z0 == z0;
    const uint64_t ie = capl ? (g.vin_total > span ? g.vin_total : span) : span;
    if (st->borrowed) {
        st->cnt = g.vix_cnt;
        st->in_e = g.vix_in_e;
    } else {
        TC_CHECK(dalloc_t(&st->cnt, nh, s));
        TC_CHECK(dalloc_t(&st->in_e, ie ? ie : 1, s));
    }
    TC_CHECK(dalloc_t(&st->tasks, (size_t)nh + span / kVChunk + 1, s));
    // [0], [1] task cursors, [2] capacity overflow flag, [3] big-task count, [4] zero,
    // [5] big cursor, [6] deferred-task count, [7] deferred cursor
    TC_CHECK(dalloc_t(&st->next, 10, s));
    TC_CHECK(dalloc_t(&st->big, (size_t)nh + span / kVChunk + 1, s));
    TC_CHECK(dalloc_t(&st->defer, (size_t)nh + span / kVChunk + 1, s));
    if (!st->borrowed) TC_CUDA(cudaMemsetAsync(st->cnt, 0, (size_t)nh * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(st->next, 0, 10 * sizeof(unsigned), s));
    st->capl = capl;
    // everything below runs on s2 (the index build too, so that with s2 != s it overlaps
    // the u-major kernels on s)
    st->s2 = s2;
    TC_CUDA(cudaEventCreateWithFlags(&st->done, cudaEventDisableTiming));
    TC_CUDA(cudaEventCreate(&st->e0));
    TC_CUDA(cudaEventCreate(&st->e1));
    if (s2 != s) {
        TC_CUDA(cudaEventRecord(st->done, s));
        TC_CUDA(cudaStreamWaitEvent(s2, st->done, 0));
    }
    // beside the u-major kernels the fill keeps a small grid (it needs atomics in flight,
    // not SM slots)
    const int64_t vg = opts().vin_grid;
    const unsigned grid = grid_for(span, 256 * kVinPP, kSMs * (unsigned)(s2 != s && vg > 0 ? vg : 8));
    const uint32_t *startp = g.vin_cap;
    if (!capl && !st->borrowed) {
        k_vin_pass<false><<<grid, 256, 0, s2>>>(g.src, g.dst, g.off32, rg, vp, nullptr, st->cnt, nullptr,
                                                nullptr, hlo, hhi);
        TC_LAUNCHED();
        TC_CHECK(vin_scan<false>(st->cnt, nh, st->start, s2));  // exact layout, cursors zeroed
        startp = st->start;
    }
    if (!st->borrowed) {
        k_vin_pass<true><<<grid, 256, 0, s2>>>(g.src, g.dst, g.off32, rg, vp, startp, st->cnt, st->in_e,
                                               capl ? st->next + 2 : nullptr, hlo, hhi);
        TC_LAUNCHED();
    }
    TC_CHECK(vin_scan<true>(st->cnt, nh, st->tstart, s2));  // tasks from the fill counts
    const uint32_t hb = (uint32_t)(g.hz - z0);  // first hub-zone head: tasks [tstart[hb], ...)
    k_vin_tasks<<<grid_for(nh, 256, kSMs * 4), 256, 0, s2>>>(startp, st->tstart, nh, st->tasks, g.off32, z0, hb,
                                                             kVNonHubCap, st->big, st->next + 3);
    TC_LAUNCHED();
    HubPack hp{nullptr, nullptr};
    if (vp.packed) {
        const uint64_t ng = (g.m + 3) / 4;
        TC_CHECK(dalloc_t(&st->lo16, 4 * ng + 16, s2));
        TC_CHECK(dalloc_t(&st->hi2, ng + 16, s2));
        TC_CUDA(cudaMemsetAsync(st->lo16 + 4 * ng, 0, 32, s2));
        TC_CUDA(cudaMemsetAsync(st->hi2 + ng, 0, 16, s2));
        k_pack_hub<<<grid_for(ng, 256, kSMs * 8), 256, 0, s2>>>(g.dst, g.m, g.hz, st->lo16, st->hi2);
        TC_LAUNCHED();
        hp = HubPack{st->lo16, st->hi2};
    }
    st->hp = hp;
    if (!vp.packed && opts().vhub) {
        // 16-bit copy of edge_dst for the top-2^16 heads of k_count_vhub
        const uint64_t ng = (g.m + 3) / 4;
        const uint32_t t16 = g.n - g.hz > kT16 ? (uint32_t)(g.n - kT16) : g.hz;
        TC_CHECK(dalloc_t(&st->lo16t, 4 * ng + 64, s2));  // 32-byte chunks read past m
        TC_CUDA(cudaMemsetAsync(st->lo16t + 4 * ng, 0, 128, s2));
        k_pack16<<<grid_for(ng, 256, kSMs * 8), 256, 0, s2>>>(g.dst, g.m, t16, st->lo16t);
        TC_LAUNCHED();
        const int64_t nbo = opts().vhub_blocks;
        if (nbo > 1) {
            const uint32_t nb = (uint32_t)(nbo < 256 ? nbo : 256);
            const uint32_t h16 = t16 - z0, nb16 = nh - h16;
            const uint64_t bsize = (g.m + nb - 1) / nb;
            const size_t N = (size_t)nb16 * nb;
            TC_CHECK(dalloc_t(&st->bspl, (size_t)nb16 * (nb + 1), s2));
            TC_CHECK(dalloc_t(&st->bcnt, N, s2));
            TC_CHECK(dalloc_t(&st->btst, N + 1, s2));
            TC_CHECK(dalloc_t(&st->btasks, span / kVChunk + N + 1, s2));
            k_band_splits<<<grid_for(nb16, 256, kSMs * 4), 256, 0, s2>>>(startp, st->cnt, st->in_e, h16, nb16, nb,
                                                                        bsize, st->bspl, st->bcnt);
            TC_LAUNCHED();
            TC_CHECK(vin_scan<false>(st->bcnt, (uint32_t)N, st->btst, s2));
            k_band_tasks<<<grid_for(N, 256, kSMs * 8), 256, 0, s2>>>(st->bspl, st->btst, h16, nb16, nb, st->btasks);
            TC_LAUNCHED();
            st->nbands = nb;
            st->nb16 = nb16;
        }
    }
    return 0;
}

// v-major part 2: the count kernels on st->s2, after `gate` (recorded on s once the u-major
// kernels are queued; nullptr = right away).  The v-major phase time is e0 -> e1.
int vmajor_count(const DeviceGraph &g, unsigned long long *d_total, cudaStream_t s, int share, VmajorState *st,
                 cudaEvent_t gate) {
    cudaStream_t s2 = st->s2;
    if (gate && s2 != s) TC_CUDA(cudaStreamWaitEvent(s2, gate, 0));
    TC_CUDA(cudaEventRecord(st->e0, s2));
    const uint32_t z0 = vzone_start(g);
    const uint32_t nh = (uint32_t)(g.n - z0);
    const uint32_t hb = (uint32_t)(g.hz - z0);
    const uint32_t *startp = st->capl ? g.vin_cap : st->start;
    const HubPack hp = st->hp;
    constexpr int NT = 256;
    auto kern = k_count_vmajor<NT, 4>;
    const uint32_t cap = 0;  // heads below hz run in k_count_vlow_warp
    const size_t sm = 4 * ((size_t)g.hwp + cap);
    TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int per_sm = 1;
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, sm));
    per_sm = per_sm / share;
    if (per_sm < 1) per_sm = 1;
    if (hb) {
        const size_t wsm = (size_t)4 * kVlSlots * kVlWarps;
        TC_CUDA(cudaFuncSetAttribute(k_count_vlow_warp<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
        int wper = 1;
        TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wper, k_count_vlow_warp<false>, 32 * kVlWarps, wsm));
        if (wper < 1) wper = 1;
        k_count_vlow_warp<false><<<kSMs * wper, 32 * kVlWarps, wsm, s2>>>(
            g.dst, g.off32, z0, startp, st->cnt, st->in_e, st->tasks, st->tstart + hb, st->next + 1,
            st->defer, st->next + 6, d_total);
        TC_LAUNCHED();
        // deferred tasks (cuckoo build failed; normally none): binary-search probes
        TC_CUDA(cudaFuncSetAttribute(k_count_vlow_warp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
        k_count_vlow_warp<true><<<kSMs, 32 * kVlWarps, wsm, s2>>>(
            g.dst, g.off32, z0, startp, st->cnt, st->in_e, st->tasks, st->tstart + hb, st->next + 7,
            st->defer, st->next + 6, d_total);
        TC_LAUNCHED();
    }
    if (hb) {  // long-list heads below hz: CTA tasks with bitmap + non-hub cuckoo (load <= 1/4)
        const uint32_t bcap = 4 * kVBigNonHub;
        const size_t bsm = 4 * ((size_t)g.hwp + bcap);
        TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
        int bper = 1;
        TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bper, kern, NT, bsm));
        if (bper < 1) bper = 1;
        kern<<<kSMs * bper, NT, bsm, s2>>>(g.src, g.dst, g.off32, g.hubstart, z0, g.hz, g.hwp, bcap, startp,
                                           st->cnt, st->in_e, st->big, st->next + 4, st->next + 3, st->next + 5,
                                           hp, d_total);
        TC_LAUNCHED();
    }
    if (st->lo16t) {
        // hub heads: lean sweep, 16-bit items for the top 2^16 heads
        const uint32_t t16 = g.n - g.hz > kT16 ? (uint32_t)(g.n - kT16) : g.hz;
        uint32_t w32 = 4;
        while (w32 < g.hwp) w32 <<= 1;
        const uint32_t amask = (w32 * 4 - 1) & ~3u;
        const size_t hsm = 4 * (size_t)(w32 > kT16 / 32 ? w32 : kT16 / 32) + (TC_VHUB_ALIGN ? 8192 : 0);
        const int64_t vu = opts().vhub_unroll;
        auto hk = vu == 4 ? k_count_vhub<NT, 4, false> : vu == 1 ? k_count_vhub<NT, 1, false> : k_count_vhub<NT, 2, false>;
        auto hkb = vu == 4 ? k_count_vhub<NT, 4, true> : vu == 1 ? k_count_vhub<NT, 1, true> : k_count_vhub<NT, 2, true>;
        TC_CUDA(cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
        TC_CUDA(cudaFuncSetAttribute(hkb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
        int hper = 1;
        TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hper, hk, NT, hsm));
        hper = hper / share;
        if (hper < 1) hper = 1;
        // without source blocks one launch covers every hub head; with them the heads below
        // the top band first, then the blocked top-band tasks
        const uint32_t hend = st->nbands ? t16 - z0 : nh;
        hk<<<kSMs * hper, NT, hsm, s2>>>(g.dst, st->lo16t, g.off32, z0, g.hz, t16, g.hwp, amask, startp, st->cnt,
                                         st->in_e, st->tasks, st->tstart + hb, st->tstart + hend, st->next, d_total);
        TC_LAUNCHED();
        if (st->nbands) {
            hkb<<<kSMs * hper, NT, hsm, s2>>>(g.dst, st->lo16t, g.off32, z0, g.hz, t16, g.hwp, amask, startp,
                                              st->cnt, st->in_e, st->btasks, st->next + 4,
                                              st->btst + (size_t)st->nb16 * st->nbands, st->next + 8, d_total);
            TC_LAUNCHED();
        }
    } else {
        TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        kern<<<kSMs * per_sm, NT, sm, s2>>>(g.src, g.dst, g.off32, g.hubstart, z0, g.hz, g.hwp, cap,
                                            startp, st->cnt, st->in_e, st->tasks, st->tstart + hb, st->tstart + nh,
                                            st->next, hp, d_total);
        TC_LAUNCHED();
    }
    TC_CUDA(cudaEventRecord(st->e1, s2));
    TC_CUDA(cudaEventRecord(st->done, s2));
    return 0;
}

int vmajor_finish(VmajorState *st, cudaStream_t s, CountStats *stats, bool *overflow) {
    *overflow = false;
    if (!st->done) return 0;
    if (st->s2 != s) TC_CUDA(cudaStreamWaitEvent(s, st->done, 0));
    if (st->capl) {
        unsigned f = 0;
        TC_CUDA(cudaMemcpyAsync(&f, st->next + 2, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
        *overflow = f != 0;
    }
    if (stats) {
        TC_CUDA(cudaEventSynchronize(st->e1));
        cudaEventElapsedTime(&stats->vmajor_ms, st->e0, st->e1);
    }
    cudaEventDestroy(st->e0);
    cudaEventDestroy(st->e1);
    cudaEventDestroy(st->done);
    if (!st->borrowed) {
        dfree(st->cnt, s);
        dfree(st->in_e, s);
    }
    dfree(st->start, s);
    dfree(st->tstart, s);
    dfree(st->tasks, s);
    dfree(st->big, s);
    dfree(st->defer, s);
    dfree(st->next, s);
    dfree(st->lo16, s);
    dfree(st->lo16t, s);
    dfree(st->btasks, s);
    dfree(st->bspl, s);
    dfree(st->bcnt, s);
    dfree(st->btst, s);
    dfree(st->hi2, s);
    *st = VmajorState{};
    return 0;
}

static cudaStream_t side_stream() {
    static cudaStream_t s2 = nullptr;
    if (!s2) cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    return s2;
}

__global__ void k_add_u64(unsigned long long *__restrict__ out, const unsigned long long *__restrict__ x) {
    *out += *x;
}

template <int WARPS, uint32_t SLOTS, uint32_t LOADINV>
int launch_mid(const DeviceGraph &g, const VSplit &vp, const RangeDev *rg, const uint2 *tasks,
               const unsigned *ntasks, unsigned *next, unsigned long long *d_total, cudaStream_t s) {
    auto kern = k_count_mid_warp<WARPS, SLOTS, LOADINV>;
    const size_t msm = (size_t)4 * SLOTS * WARPS;
    TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msm));
    int per_sm = 1;
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * WARPS, msm));
    if (per_sm < 1) per_sm = 1;
    kern<<<kSMs * per_sm, 32 * WARPS, msm, s>>>(g.dst, g.off32, vp, rg, tasks, ntasks, next, d_total);
    TC_LAUNCHED();
    return 0;
}

// The v-major decision of a count (rank-space graphs with u32 offsets).

// Shard of a multi-GPU count: the non-v-major edges of [lo, hi) plus the v-major edges (of
// the whole graph) whose head lies in [hlo, hhi).  Over a covering set of shards every edge
// is counted exactly once, and every head's bitmap is built once in total.
struct ShardSpec {
    uint32_t hlo, hhi;
};

template <typename OffT>
int count_impl(const DeviceGraph &g, const OffT *off, uint64_t lo, uint64_t hi,
               unsigned long long *d_out, cudaStream_t s, CountStats *stats,
               const ShardSpec *shard = nullptr) {
    // Sources with more out-edges than the shared-memory staging can hold (d+(u) > 51,200:
    // only cliques of ~51K+ vertices reach that) are counted by the paper's thread-per-edge
    // merge over the whole range -- slower, same exact sum.
    for (int c = 0; c < kClasses; ++c) {
        const uint32_t lower_c = c == 0 ? (uint32_t)kLightMax : kClassMax[c - 1];
        if (g.max_out > lower_c && heavy_smem(c, g.max_out) > 200 * 1024) {
            k_count_merge_thread<OffT><<<grid_for(hi - lo, 256, kSMs * 16), 256, 0, s>>>(
                g.src, g.dst, off, lo, hi, d_out);
            TC_LAUNCHED();
            return 0;
        }
    }
    // with a capacity layout the v-major index can detect a non-symmetric input only at the
    // end: count into a private total and add it to *d_out unless a recount is needed
    unsigned long long *d_total = d_out;
    if (g.vin_cap) {
        TC_CHECK(dalloc_t(&d_total, 1, s));
        TC_CUDA(cudaMemsetAsync(d_total, 0, sizeof(unsigned long long), s));
    }
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
    // v-major hub heads (rank space): every heavy class must run the hub kernel (which
    // skips the hub-head edges), so it is all or nothing.
    // vmajor: -1 = auto (large skewed graphs: the in-edge index costs a few ms, the
    // hub reuse it unlocks pays from ~10^8 edges with hub-sized out-degrees), 0 off, 1 on.
    const bool vmajor = sizeof(OffT) == 4 && vmajor_schedule(g);
    if (g.max_out > (uint32_t)kLightMax) {
        k_classify<OffT><<<grid_for(nverts, 256, kSMs * 8), 256, 0, s>>>(
            off, rg, nullptr, tasks[0], tasks[1], tasks[2], tasks[3], counters);
        TC_LAUNCHED();
    }
    // u-major only: the hottest data is the tail of the dense-hub bitmaps (top ranks: short
    // bitmaps read by almost every heavy source); keep a window of it L2-resident (-2 % at
    // s26).  With v-major heads those reads are gone and the window only costs L2 capacity.
    const bool l2win = !vmajor && apply_l2_window(g, s);
    const int64_t conc_env = opts().concurrent;
    const bool conc = vmajor && conc_env;
    const int share = conc ? (int)(opts().share > 0 ? opts().share : 1) : 1;  // SM share of each concurrent kernel
    // the in-edge index builds on the side stream while the u-major kernels run (vin_overlap);
    // the v-major count kernels follow them (persistent grids do not share SMs well, §4.4)
    const bool overlap = vmajor && !conc && opts().vin_overlap != 0;
    VmajorState vst;
    RangeDev *rg_all = nullptr;  // shard mode: the v-major index scans every edge for its heads
    if (vmajor && shard) {
        TC_CHECK(dalloc_t(&rg_all, 1, s));
        k_range_init<<<1, 1, 0, s>>>(g.src, 0, g.m, g.m, rg_all);
        TC_LAUNCHED();
        TC_CHECK(vmajor_index(g, rg_all, g.m, s, (conc || overlap) ? side_stream() : s, &vst, false, shard->hlo,
                              shard->hhi));
    } else if (vmajor) {
        TC_CHECK(vmajor_index(g, rg, span, s, (conc || overlap) ? side_stream() : s, &vst, lo == 0 && hi >= g.m));
    }
    if (vmajor && !overlap) TC_CHECK(vmajor_count(g, d_total, s, share, &vst, nullptr));
    TC_CUDA(cudaEventRecord(ev[1], s));
    // Heavy classes first (largest tasks first), then the light sweep.
    for (int c = kClasses - 1; c >= 0; --c) {
        if (g.max_out <= lower[c]) continue;
        const size_t sm = heavy_smem(c, g.max_out);  // <= 200 KB (checked on entry)
        const unsigned *nt_c = counters + c;
        unsigned *next_c = counters + kClasses + c;
        int rc = 0;
        // non-hub part of adj(u) in a cuckoo table at load <= 1/3 (smem: bitmap + table)
        // cuckoo slots for the non-hub part of adj(u) (load <= 1/3); heavy sources keep most
        // items in the hub zone, so the table is sized for 1/hub_cap_div of the class maximum
        // (a longer non-hub part is binary-searched) -- the smem it saves buys resident CTAs
        const int64_t hcd = opts().hub_cap_div > 0 ? opts().hub_cap_div : 1;
        const uint32_t hub_cap = (uint32_t)(3 * (g.max_out < kClassMax[c] ? g.max_out : kClassMax[c]) / hcd);
        const size_t hub_sm = 4 * ((size_t)g.hwp + hub_cap);
        const int64_t midwarp = opts().midwarp;
        // with v-major on, the hub heads' dense edges are gone and the class-0 tasks are
        // latency-bound: one warp per task (without it the CTA bitmap kernel wins)
        if (c <= (midwarp >= 2 ? 1 : 0) && midwarp && vmajor && sizeof(OffT) == 4 && g.rank_space &&
            g.hubstart) {
            const VSplit vp = make_vsplit(g, vmajor);
            // cuckoo load <= 1/3: 6 KB per warp, 4 CTAs (32 warps) per SM (load 1/4: 3 CTAs, +12 %)
            if (c == 0) TC_CHECK((launch_mid<kMidWarps, kMidSlots, kMidLoadInv>(g, vp, rg, tasks[c], nt_c, next_c, d_total, s)));
            else TC_CHECK((launch_mid<4, 3 * 2048, 3>(g, vp, rg, tasks[c], nt_c, next_c, d_total, s)));
            continue;
        }
        if (sizeof(OffT) == 4 && g.rank_space && g.hubstart && hub_sm <= 200 * 1024) {
            const int ntc = c == 2 ? 512 : 256;
            // the packed copy is built on the v-major stream: usable once that phase is joined
            const HubPack hp = (conc || overlap) ? HubPack{nullptr, nullptr} : HubPack{vst.lo16, vst.hi2};
            rc = ntc == 512 ? launch_hub<512>(g, rg, tasks[c], nt_c, next_c, hub_cap, vmajor, share, hp, d_total, s)
                            : launch_hub<256>(g, rg, tasks[c], nt_c, next_c, hub_cap, vmajor, share, hp, d_total, s);
            if (rc) return rc;
            continue;
        }
        if (c == 0) rc = launch_heavy<OffT, 0, 128>(g, off, rg, tasks[c], nt_c, next_c, kClassCap[c], sm, d_total, s);
        else if (c == 1) rc = launch_heavy<OffT, 0, 256>(g, off, rg, tasks[c], nt_c, next_c, kClassCap[c], sm, d_total, s);
        else if (c == 2) rc = launch_heavy<OffT, 0, 512>(g, off, rg, tasks[c], nt_c, next_c, kClassCap[c], sm, d_total, s);
        else rc = launch_heavy<OffT, 1, 512>(g, off, rg, tasks[c], nt_c, next_c, 0, sm, d_total, s);
        if (rc) return rc;
    }
    TC_CUDA(cudaEventRecord(ev[2], s));
    // Light sources: 1 = thread per edge, 2 = warp windows, 0 = CTA windows; -1 (default) =
    // warp windows for hub-free graphs with long light lists (RGG-like: max out-degree <= 64,
    // m >= 12 n; RGG 2e7 21.5 -> 19.8 ms), thread per edge otherwise (BA: 3.2 vs 4.8 ms;
    // R-MAT: hub heads make the per-edge choices matter).
    const int64_t light_env = opts().light;
    const int light_algo = light_env >= 0 ? light_env
                           : (g.rank_space && g.max_out <= 64 && g.m >= 12 * g.n) ? 2 : 1;
    if (light_algo == 2 && g.rank_space && !vmajor) {
        const bool hub = g.hubstart && g.dense_bits;
        const uint32_t skew = (uint32_t)opts().skew;
        auto kern = hub ? k_count_light_warp<OffT, true> : k_count_light_warp<OffT, false>;
        kern<<<kSMs * 8, 32 * kLwWarps, 0, s>>>(g.src, g.dst, off, rg, g.hz, hub ? g.vt : 0xffffffffu,
                                                g.dense_off, g.dense_bits, g.dense_words, skew, d_total);
    } else if (light_algo == 1 || vmajor) {
        const bool hub = g.rank_space && g.hubstart && g.dense_bits;
        const bool vec = g.rank_space && g.n <= 0xfffffffeull && opts().light_vec;
        auto kern = hub ? (vec ? k_count_light_tpe<OffT, true, true, true> : k_count_light_tpe<OffT, true, true, false>)
                    : g.rank_space ? (vec ? k_count_light_tpe<OffT, true, false, true> : k_count_light_tpe<OffT, true, false, false>)
                                   : k_count_light_tpe<OffT, false, false, false>;
        kern<<<kSMs * 8, 256, 0, s>>>(g.src, g.dst, off, rg, g.hz, hub ? g.vt : 0xffffffffu,
                                      g.dense_off, g.dense_bits, g.dense_words,
                                      make_vsplit(g, vmajor), d_total);
    } else {
        const bool hub = g.rank_space && g.hubstart;
        const uint32_t hwords = hub ? (uint32_t)((g.n - g.hz + 31) / 32) + 1 : 0u;
        auto kern = hub ? k_count_window<OffT, kWinThreads, true> : k_count_window<OffT, kWinThreads, false>;
        const int sm = kWinSlots * 8 + 4 * hwords;
        TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        int per_sm = 1;
        TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWinThreads, sm));
        kern<<<kSMs * (per_sm > 0 ? per_sm : 1), kWinThreads, sm, s>>>(
            g.src, g.dst, off, rg, counters + 2 * kClasses, g.hz, hwords, hub ? g.vt : 0u,
            g.dense_off, g.dense_bits, g.dense_words, d_total);
    }
    TC_LAUNCHED();
    TC_CUDA(cudaEventRecord(ev[3], s));
    if (overlap) TC_CHECK(vmajor_count(g, d_total, s, 1, &vst, ev[3]));
    bool overflow = false;
    TC_CHECK(vmajor_finish(&vst, s, stats, &overflow));
    if (overflow) {
        // not a symmetric edge array: redo the whole range without the capacity layout
        DeviceGraph g2 = g;
        g2.vin_cap = nullptr;
        g2.vix_ready = false;
        for (auto &e : ev) cudaEventDestroy(e);
        for (int c = 0; c < kClasses; ++c) dfree(tasks[c], s);
        dfree(rg_all, s);
        dfree(rg, s);
        dfree(counters, s);
        dfree(d_total, s);
        return count_impl<OffT>(g2, off, lo, hi, d_out, s, stats, shard);
    }
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
    if (l2win) clear_l2_window(s);
    for (int c = 0; c < kClasses; ++c) dfree(tasks[c], s);
    dfree(rg_all, s);
    dfree(rg, s);
    dfree(counters, s);
    if (d_total != d_out) {
        k_add_u64<<<1, 1, 0, s>>>(d_out, d_total);
        TC_LAUNCHED();
        dfree(d_total, s);
    }
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

int count_shard_dev(const DeviceGraph &g, uint64_t lo, uint64_t hi, uint32_t hlo, uint32_t hhi,
                    unsigned long long *d_total, cudaStream_t s, CountStats *stats) {
    if (hi > g.m) hi = g.m;
    if (!g.off32 || !vmajor_schedule(g)) return count_range_dev(g, lo, hi, kAlgoAuto, d_total, s, stats);
    const ShardSpec sh{hlo, hhi};
    // an empty edge range may still own heads: run the v-major part over them
    return count_impl<uint32_t>(g, g.off32, lo, hi > lo ? hi : lo, d_total, s, stats, &sh);
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
              uint64_t *ntiles_out, cudaStream_t s, bool ranked = false, uint32_t ucap = 0xffffffffu) {
    const uint64_t nt = (g.m + tile - 1) / tile;
    unsigned long long *sums = nullptr;
    TC_CHECK(dalloc_t(&sums, nt ? nt : 1, s));
    if (nt) {
        if (g.off32 && ranked)
            k_tile_work<uint32_t, true><<<(unsigned)nt, 256, 0, s>>>(g.src, g.dst, g.off32, g.m, tile, overhead, sums);
        else if (g.off32)
            k_tile_work<uint32_t><<<(unsigned)nt, 256, 0, s>>>(g.src, g.dst, g.off32, g.m, tile, overhead, sums,
                                                               ucap);
        else
            k_tile_work<int64_t><<<(unsigned)nt, 256, 0, s>>>(g.src, g.dst, g.off, g.m, tile, overhead, sums);
        TC_LAUNCHED();
    }
    *sums_out = sums;
    *ntiles_out = nt;
    return 0;
}
}  // namespace

__global__ void k_tile_sched(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                             const uint32_t *__restrict__ off, uint64_t m, uint64_t tile, uint32_t overhead,
                             VSplit vp, bool hub, unsigned long long *__restrict__ sums);

int work_bounds_dev(const DeviceGraph &g, int npools, int64_t *bounds, cudaStream_t s) {
    // Per-edge estimated work d+(u) + d+(v) + c; cuts at k*W/P with a
    // tile granularity fine enough that rounding is negligible against m/P.
    uint64_t tile = g.m / ((uint64_t)npools * 1024);
    if (tile < 1) tile = 1;
    if (tile > 4096) tile = 4096;
    unsigned long long *sums = nullptr;
    uint64_t nt = 0;
    // Rank-space graphs (the count schedule with hub structures / v-major heads): per-edge
    // work d+(v) + min(d+(u), 1024) + 128 -- heavy sources are cheap per edge there, every
    // edge pays a latency-bound constant.  Measured per-shard count times at R-MAT s26,
    // P = 8 (scripts/shard_balance.py): max/mean 1.29 -> 1.19 against d+(u) + d+(v) + 8.
    // Reference-id graphs keep the merge-work model of SURVEY.md §8(e).
    const int64_t model = opts().shard_model;
    const uint32_t ovh_env = (uint32_t)opts().shard_ovh;
    const uint32_t ucap_env = (uint32_t)opts().shard_ucap;
    const bool ranked = model == 1 && g.rank_space;
    const uint32_t ovh = g.rank_space ? ovh_env : 8u, ucap = g.rank_space ? ucap_env : 0xffffffffu;
    if (model == 2 && g.rank_space && g.off32 && g.hubstart) {
        // compulsory bytes of the schedule the ranged count will run, per edge, + overhead
        const uint64_t ntl = (g.m + tile - 1) / tile;
        TC_CHECK(dalloc_t(&sums, ntl ? ntl : 1, s));
        if (ntl) {
            k_tile_sched<<<(unsigned)ntl, 256, 0, s>>>(g.src, g.dst, g.off32, g.m, tile, (uint32_t)opts().shard_ovh2,
                                                      make_vsplit(g, vmajor_schedule(g)), g.dense_bits != nullptr,
                                                      sums);
            TC_LAUNCHED();
        }
        nt = ntl;
    } else {
        TC_CHECK(tile_sums(g, tile, ovh, &sums, &nt, s, ranked, ucap));
    }
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

// ---------------------------------------------------------- schedule byte model ---
// Compulsory HBM bytes of the schedule a full count of a rank-space graph runs (the roofline
// numerator): every edge's data read once, at 4 B per item, along the path
// the count kernels choose for it (same vmajor_edge predicate, same light-kernel variants):
//   [0] v-major edges      4 * |suffix of adj(u) after v| + 8 (its in-edge index entry)
//   [1] u-major heavy      dense head: 4 * bitmap words; otherwise 4 * |adj(v)|
//   [2] light sources      4 * (|suffix| + |adj(v)|) merge; 4 * |suffix| dense-bitmap test;
//                          4 * |suffix| * ceil(log2 |adj(v)|) binary search
//   [3] every edge         16 (src, dst, off[v], off[v+1])
//   [4] heavy staging      4 * d+(u) per heavy source (adj(u) into shared memory once)
// Bytes of edge e under the schedule; *cls = 0..3 (v-major, u-major heavy, light, none).
__device__ __forceinline__ uint64_t edge_bytes(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                                               const uint32_t *__restrict__ off, uint64_t e, const VSplit &vp,
                                               bool hub, int *cls, uint32_t *stage, bool *dense_out = nullptr) {
    const uint32_t u = __ldg(src + e), su = __ldg(off + u), eu = __ldg(off + u + 1), du = eu - su;
    const uint32_t v = __ldg(dst + e), vs = __ldg(off + v), ve = __ldg(off + v + 1), dv = ve - vs;
    *stage = e == su && du > (uint32_t)kLightMax ? 4u * du : 0u;
    *cls = 3;
    if (e + 1 >= eu || vs >= ve) return 0;  // no triangle can close: every kernel skips it
    const uint32_t sfx = eu - (uint32_t)e - 1;
    if (vmajor_edge(vp, (uint32_t)e, eu, v, vs, ve)) {
        *cls = 0;
        // 16-bit suffix copy for heads >= t16 (k_count_vhub): 2 B per item
        return (vp.packed && v >= vp.hz ? 9ull * ((sfx + 3) / 4) : v >= vp.t16 ? 2ull * sfx : 4ull * sfx) + 8;
    }
    if (du > (uint32_t)kLightMax) {
        *cls = 1;
        uint64_t x = 4ull * dv;
        if (hub && v >= vp.hz) {
            const uint32_t ws = ((v + 1 - vp.hz) >> 5) & ~3u;
            if (v >= vp.vt && (vp.hwp - ws) < vp.factor * dv) {
                x = 4ull * (vp.hwp - ws);
                if (dense_out) *dense_out = true;
            } else if (vp.packed) {
                x = 9ull * ((dv + 3) / 4);
            }
        }
        return x;
    }
    *cls = 2;
    uint64_t x = 4ull * (sfx + dv);
    if (hub && v >= vp.vt && sfx < dv) x = 4ull * sfx;
    else if (sfx * (32u - __clz(dv)) < sfx + dv) x = 4ull * sfx * (32u - __clz(dv));
    return x;
}

__global__ void __launch_bounds__(256)
    k_schedule_bytes(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                     const uint32_t *__restrict__ off, uint64_t lo, uint64_t m, VSplit vp, bool hub,
                     unsigned long long *__restrict__ out) {
    unsigned long long b[5] = {0, 0, 0, 0, 0};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        int cls;
        uint32_t stage;
        const uint64_t x = edge_bytes(src, dst, off, e, vp, hub, &cls, &stage);
        b[3] += 16;
        b[4] += stage;
        if (cls < 3) b[cls] += x;
    }
    for (int k = 0; k < 5; ++k) {
        unsigned long long x = b[k];
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(TC_FULL_MASK, x, o);
        if (lane_id() == 0 && x) atomicAdd(out + k, x);
    }
}

// Per-tile sums of the schedule's bytes + `overhead` per edge (the rank-space shard model).
__global__ void __launch_bounds__(256)
    k_tile_sched(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                 const uint32_t *__restrict__ off, uint64_t m, uint64_t tile, uint32_t overhead, VSplit vp,
                 bool hub, unsigned long long *__restrict__ sums) {
    const uint64_t b = (uint64_t)blockIdx.x * tile;
    const uint64_t e1 = b + tile < m ? b + tile : m;
    unsigned long long acc = 0;
    for (uint64_t e = b + threadIdx.x; e < e1; e += blockDim.x) {
        int cls;
        uint32_t stage;
        acc += edge_bytes(src, dst, off, e, vp, hub, &cls, &stage) + stage + overhead;
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

int schedule_bytes_dev(const DeviceGraph &g, uint64_t lo, uint64_t hi, uint64_t out[5], cudaStream_t s) {
    if (!g.rank_space || !g.off32 || !g.hubstart) {
        set_error("the schedule byte model needs a rank-space graph with m < 2^32");
        return -1;
    }
    unsigned long long *d = nullptr;
    TC_CHECK(dalloc_t(&d, 5, s));
    TC_CUDA(cudaMemsetAsync(d, 0, 5 * sizeof(unsigned long long), s));
    const bool vm = vmajor_schedule(g);
    const VSplit vp = make_vsplit(g, vm);
    if (hi > g.m) hi = g.m;
    if (lo < hi) {
        k_schedule_bytes<<<grid_for(hi - lo, 256, kSMs * 16), 256, 0, s>>>(g.src, g.dst, g.off32, lo, hi, vp,
                                                                          g.dense_bits != nullptr, d);
        TC_LAUNCHED();
    }
    unsigned long long h[5];
    TC_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(d, s);
    for (int k = 0; k < 5; ++k) out[k] = h[k];
    return 0;
}

// ---------------------------------------------------------------- shard plan ---
// Time per byte of each class, in 1/1000 ps, fitted to per-shard phase times of R-MAT s26
// shards on one B200 (scripts/shard_calib.py, profiles/r02_shard_calib_s26.jsonl; nnls,
// max rel. error 0.27 edge side / 0.21 head side): dense-head ANDs stream L2-resident
// bitmaps (0.118 ps/B), sparse heavy items 0.273, light sources pay random 32-byte sectors
// (5.5), a heavy source's staging ~18 per staged byte (task setup); v-major suffix bytes
// of hub heads 0.153, of heads below the hub zone (warp tasks) 0.30, plus 62 ps per in-edge
// (index fill).  Each side is balanced separately, so every shard gets 1/P of both.
struct ShardWeights {
    uint64_t dense, sparse, light, stage, edge, hub, vlow, vedge;
};
// Edge side: per-tile bytes of the NON-v-major edges (u-major heavy, light, per-edge, staging).
__global__ void __launch_bounds__(256)
    k_tile_edge_side(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                     const uint32_t *__restrict__ off, uint64_t m, uint64_t tile, VSplit vp, bool hub,
                     ShardWeights w, unsigned long long *__restrict__ sums) {
    const uint64_t b = (uint64_t)blockIdx.x * tile;
    const uint64_t e1 = b + tile < m ? b + tile : m;
    unsigned long long acc = 0;
    for (uint64_t e = b + threadIdx.x; e < e1; e += blockDim.x) {
        int cls;
        uint32_t stage;
        bool dense = false;
        const uint64_t x = edge_bytes(src, dst, off, e, vp, hub, &cls, &stage, &dense);
        acc += (cls == 1 ? x * (dense ? w.dense : w.sparse) : cls == 2 ? x * w.light : 0ull) +
               (uint64_t)stage * w.stage + w.edge;
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

// Head side: v-major bytes per head of the zone [z0, n) (suffix streams + index entries).
__global__ void __launch_bounds__(256)
    k_head_side(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                const uint32_t *__restrict__ off, uint64_t m, VSplit vp, bool hub, ShardWeights w,
                unsigned long long *__restrict__ hb) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        const uint32_t v = __ldg(dst + e);
        if (v < vp.z0) continue;
        int cls;
        uint32_t stage;
        const uint64_t x = edge_bytes(src, dst, off, e, vp, hub, &cls, &stage);
        // heads below the hub zone run in the warp-task kernel (slower per byte)
        // + w.vedge per in-edge: the index fill's atomic + entry
        if (cls == 0) atomicAdd(hb + (v - vp.z0), x * (v < vp.hz ? w.vlow : w.hub) + w.vedge);
    }
}

// + the per-task cost of a head that has v-major in-edges: zeroing its bitmap words and
// staging adj(v).
__global__ void k_head_fixed(const uint32_t *__restrict__ off, uint32_t z0, uint32_t nz, VSplit vp,
                             ShardWeights w, unsigned long long *__restrict__ hb) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < nz; h += stride) {
        if (!hb[h]) continue;
        const uint32_t v = z0 + h;
        const uint32_t ws = v >= vp.hz ? ((v + 1 - vp.hz) >> 5) & ~3u : 0u;
        hb[h] += (4ull * (vp.hwp - ws) + 4ull * (off[v + 1] - off[v])) * w.hub;
    }
}

// Per-shard cost features (calibration of the shard plan's weights, scripts/shard_calib.py):
// edge side over [lo, hi) non-v-major edges: [0] dense AND bytes, [1] sparse heavy item
// bytes, [2] light bytes, [3] edges, [4] heavy staging bytes; head side over heads in
// [hlo, hhi): [5] hub-head v-major bytes, [6] below-hub v-major bytes, [7] v-major edges;
// [8] v-major bytes of the edges in [lo, hi) (by source position: suffix locality probes).
__global__ void __launch_bounds__(256)
    k_shard_stats(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                  const uint32_t *__restrict__ off, uint64_t m, uint64_t lo, uint64_t hi, uint32_t hlo,
                  uint32_t hhi, VSplit vp, bool hub, unsigned long long *__restrict__ out) {
    unsigned long long b[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        int cls;
        uint32_t stage;
        const uint64_t x = edge_bytes(src, dst, off, e, vp, hub, &cls, &stage);
        const uint32_t v = __ldg(dst + e);
        if (cls == 0 && e >= lo && e < hi) b[8] += x;
        if (cls == 0) {
            if (v >= hlo && v < hhi) {
                b[v >= vp.hz ? 5 : 6] += x;
                b[7] += 1;
            }
        } else if (e >= lo && e < hi) {
            b[3] += 1;
            b[4] += stage;
            if (cls == 2) b[2] += x;
            else if (cls == 1) {
                const uint32_t vs = __ldg(off + v), ve = __ldg(off + v + 1);
                const uint32_t ws = ((v + 1 - vp.hz) >> 5) & ~3u;
                const bool dense = hub && v >= vp.hz && v >= vp.vt && (vp.hwp - ws) < vp.factor * (ve - vs);
                b[dense ? 0 : 1] += x;
            }
        }
    }
    for (int k = 0; k < 9; ++k) {
        unsigned long long x = b[k];
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(TC_FULL_MASK, x, o);
        if (lane_id() == 0 && x) atomicAdd(out + k, x);
    }
}

int shard_stats_dev(const DeviceGraph &g, uint64_t lo, uint64_t hi, uint32_t hlo, uint32_t hhi, uint64_t out[9],
                    cudaStream_t s) {
    if (!g.off32 || !g.rank_space || !g.hubstart) {
        set_error("shard stats need a rank-space graph with m < 2^32");
        return -1;
    }
    unsigned long long *d = nullptr;
    TC_CHECK(dalloc_t(&d, 9, s));
    TC_CUDA(cudaMemsetAsync(d, 0, 9 * sizeof(unsigned long long), s));
    if (g.m) {
        k_shard_stats<<<grid_for(g.m, 256, kSMs * 16), 256, 0, s>>>(g.src, g.dst, g.off32, g.m, lo, hi, hlo, hhi,
                                                                   make_vsplit(g, vmajor_schedule(g)),
                                                                   g.dense_bits != nullptr, d);
        TC_LAUNCHED();
    }
    unsigned long long h[9];
    TC_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(d, s);
    for (int k = 0; k < 9; ++k) out[k] = h[k];
    return 0;
}

static void cut_prefix(const unsigned long long *h, uint64_t nt, int parts, uint64_t unit, uint64_t cap,
                       int64_t *bounds, int64_t base) {
    unsigned long long W = 0;
    for (uint64_t i = 0; i < nt; ++i) W += h[i];
    bounds[0] = base;
    unsigned long long run = 0;
    uint64_t t = 0;
    for (int p = 1; p < parts; ++p) {
        const long double target = (long double)W * p / parts;
        while (t < nt && (long double)(run + h[t]) <= target) run += h[t++];
        uint64_t cut = t;
        if (t < nt && (long double)(run + h[t]) - target < target - (long double)run) cut = t + 1;
        uint64_t b = cut * unit;
        if (b > cap) b = cap;
        int64_t bb = base + (int64_t)b;
        if (bb < bounds[p - 1]) bb = bounds[p - 1];
        bounds[p] = bb;
    }
}

// Model costs of the plan: per-tile edge-side costs (nt tiles of `tile` edges) and per-head
// head-side costs (nz heads from z0).  Host arrays; sizes from shard_cost_sizes.
void shard_cost_sizes(const DeviceGraph &g, int parts, uint64_t *nt, uint64_t *tile, uint64_t *nz, uint32_t *z0) {
    uint64_t t = g.m / ((uint64_t)(parts > 0 ? parts : 1) * 1024);
    if (t < 1) t = 1;
    if (t > 4096) t = 4096;
    *tile = t;
    *nt = (g.m + t - 1) / t;
    const bool vm = g.off32 && vmajor_schedule(g);
    *z0 = vm ? vzone_start(g) : (uint32_t)g.n;
    *nz = g.n - *z0;
}

int shard_costs_dev(const DeviceGraph &g, int parts, unsigned long long *edge_tiles, unsigned long long *head_costs,
                    cudaStream_t s) {
    uint64_t nt, tile, nz;
    uint32_t z0;
    shard_cost_sizes(g, parts, &nt, &tile, &nz, &z0);
    const bool vm = g.off32 && vmajor_schedule(g);
    if (!vm) {
        set_error("shard costs need a v-major (rank-space, m >= 2^27 or forced) schedule");
        return -1;
    }
    const VSplit vp = make_vsplit(g, true);
    const bool hub = g.dense_bits != nullptr;
    const Options &o = opts();
    const ShardWeights w{(uint64_t)o.shard_w_dense, (uint64_t)o.shard_w_sparse, (uint64_t)o.shard_w_light,
                         (uint64_t)o.shard_w_stage, (uint64_t)o.shard_w_edge, (uint64_t)o.shard_w_hub,
                         (uint64_t)o.shard_w_vlow, (uint64_t)o.shard_w_vedge};
    unsigned long long *sums = nullptr, *hb = nullptr;
    TC_CHECK(dalloc_t(&sums, nt ? nt : 1, s));
    TC_CHECK(dalloc_t(&hb, nz ? nz : 1, s));
    TC_CUDA(cudaMemsetAsync(hb, 0, (nz ? nz : 1) * sizeof(unsigned long long), s));
    if (nt) {
        k_tile_edge_side<<<(unsigned)nt, 256, 0, s>>>(g.src, g.dst, g.off32, g.m, tile, vp, hub, w, sums);
        TC_LAUNCHED();
        k_head_side<<<grid_for(g.m, 256, kSMs * 16), 256, 0, s>>>(g.src, g.dst, g.off32, g.m, vp, hub, w, hb);
        TC_LAUNCHED();
    }
    if (nz) {
        k_head_fixed<<<grid_for(nz, 256, kSMs * 4), 256, 0, s>>>(g.off32, z0, (uint32_t)nz, vp, w, hb);
        TC_LAUNCHED();
    }
    if (nt) TC_CUDA(cudaMemcpyAsync(edge_tiles, sums, nt * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    if (nz) TC_CUDA(cudaMemcpyAsync(head_costs, hb, nz * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(sums, s);
    dfree(hb, s);
    return 0;
}

int shard_plan_dev(const DeviceGraph &g, int parts, int64_t *ebounds, int64_t *hbounds, cudaStream_t s) {
    const bool vm = g.off32 && vmajor_schedule(g);
    for (int p = 0; p <= parts; ++p) hbounds[p] = p == 0 ? 0 : (int64_t)g.n;
    if (!vm) return work_bounds_dev(g, parts, ebounds, s);
    uint64_t nt, tile, nz;
    uint32_t z0;
    shard_cost_sizes(g, parts, &nt, &tile, &nz, &z0);
    unsigned long long *e = (unsigned long long *)malloc((nt + 1) * sizeof(unsigned long long));
    unsigned long long *h = (unsigned long long *)malloc((nz + 1) * sizeof(unsigned long long));
    if (!e || !h) {
        free(e);
        free(h);
        set_error("host allocation failed");
        return -3;
    }
    const int rc = shard_costs_dev(g, parts, e, h, s);
    if (!rc) {
        cut_prefix(e, nt, parts, tile, g.m, ebounds, 0);
        ebounds[parts] = (int64_t)g.m;
        cut_prefix(h, nz, parts, 1, nz, hbounds, (int64_t)z0);
        hbounds[0] = 0;  // heads below the zone never run v-major: shard 0 owns them (no work)
        hbounds[parts] = (int64_t)g.n;
    }
    free(e);
    free(h);
    return rc;
}

int vin_capacity_dev(DeviceGraph *g, const uint32_t *deg_by_rank, cudaStream_t s) {
    if (!g->off32 || g->n == 0) return 0;
    const uint32_t z0 = vzone_start_of(g->n, g->hz);
    const uint32_t nz = (uint32_t)(g->n - z0);
    uint32_t *tmp = nullptr;
    dfree(g->vin_cap, s);
    g->vin_cap = nullptr;
    TC_CHECK(dalloc_t(&g->vin_cap, (size_t)nz + 1, s, g->persistent));
    TC_CHECK(dalloc_t(&tmp, nz, s));
    k_vin_capacity<<<grid_for(nz, 256, kSMs * 4), 256, 0, s>>>(deg_by_rank, g->off32, z0, nz, tmp);
    TC_LAUNCHED();
    TC_CHECK(vin_scan<false>(tmp, nz, g->vin_cap, s));
    dfree(tmp, s);
    uint32_t total = 0;
    TC_CUDA(cudaMemcpyAsync(&total, g->vin_cap + nz, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    g->vin_total = total;
    g->vin_z0 = z0;
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
