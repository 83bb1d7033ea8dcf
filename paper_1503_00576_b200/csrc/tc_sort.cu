// tc_sort.cu -- hand-written LSD radix sort for sm_100a (one read + one write of the keys
// per digit pass; Onesweep-style chained scan with decoupled look-back).
//
// Replaces the reference's np.sort of packed (first<<32)|second keys
// (reference preprocess.py:23-33, graph.py:84-98).  Keys here are packed more tightly,
// (first << vb) | second with vb = bits(n-1), so the passes cover only 2*vb bits.
//
// Per pass, a CTA owns one 4096-key tile:
//   1. loads 16 keys/thread, warp-striped (coalesced 256 B per warp load);
//   2. ranks keys inside each warp with __match_any_sync (stable: slot-major, lane-minor);
//   3. publishes its per-digit tile counts and looks back over earlier tiles (decoupled
//      look-back) to get its global per-digit base;
//   4. stages the tile in shared memory in digit order and writes it out so consecutive
//      threads write consecutive addresses inside each digit run.
#include "tc_common.cuh"
#include "tc_internal.h"

namespace tc {

namespace {

constexpr uint64_t kFlagA = 1ull << 62;  // aggregate of this tile only
constexpr uint64_t kFlagP = 2ull << 62;  // inclusive prefix through this tile
constexpr uint64_t kValMask = (1ull << 62) - 1;
constexpr int kSortWarps = kSortThreads / 32;

struct PassParams {
    int shift, bits;
};

__global__ void __launch_bounds__(256) k_digit_hist(const uint64_t *__restrict__ keys, uint64_t n,
                                                    RadixPlan plan, uint32_t *__restrict__ ghist) {
    __shared__ uint32_t sh[kMaxPasses * kRadix];
    for (int i = threadIdx.x; i < plan.npass * kRadix; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint64_t k = __ldcs(keys + i);
#pragma unroll
        for (int p = 0; p < kMaxPasses; ++p)
            if (p < plan.npass)
                atomicAdd(&sh[p * kRadix + ((k >> plan.shift[p]) & ((1u << plan.bits[p]) - 1))], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < plan.npass * kRadix; i += blockDim.x)
        if (sh[i]) atomicAdd(&ghist[i], sh[i]);
}

// Exclusive scan of each pass's histogram -> global digit base (one block, kRadix threads).
__global__ void k_digit_base(const uint32_t *__restrict__ ghist, int npass,
                             uint64_t *__restrict__ base) {
    __shared__ uint64_t warp_tot[32];
    for (int p = 0; p < npass; ++p) {
        uint64_t x = ghist[p * kRadix + threadIdx.x];
        uint64_t tot;
        uint64_t ex = block_exclusive_scan<uint64_t>(x, warp_tot, &tot);
        base[p * kRadix + threadIdx.x] = ex;
    }
}

#ifndef TC_SORT_MINB
#define TC_SORT_MINB 4
#endif
template <int MODE, bool HAS_VAL>
__global__ void __launch_bounds__(kSortThreads, TC_SORT_MINB)
    k_radix_pass(const uint64_t *__restrict__ kin, uint64_t *__restrict__ kout,
                 const uint32_t *__restrict__ vin, uint32_t *__restrict__ vout,
                 uint32_t *__restrict__ out_a, uint32_t *__restrict__ out_b, int split_bits,
                 uint64_t n, PassParams pp, const uint64_t *__restrict__ digit_base,
                 uint64_t *__restrict__ status, unsigned *__restrict__ tile_counter) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t *s_keys = reinterpret_cast<uint64_t *>(smem);                       // kSortTile
    uint64_t *s_gbase = s_keys + kSortTile;                                        // kRadix
    uint32_t *s_whist = reinterpret_cast<uint32_t *>(s_gbase + kRadix);           // warps*radix
    uint32_t *s_tstart = s_whist + kSortWarps * kRadix;                           // kRadix
    uint32_t *s_scan = s_tstart + kRadix;                                          // 32
    uint32_t *s_misc = s_scan + 32;                                                // 4
    uint32_t *s_vals = s_misc + 4;                                                 // kSortTile

    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_misc[0] = atomicAdd(tile_counter, 1u);
    for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) s_whist[i] = 0;
    __syncthreads();
    const uint64_t tile = s_misc[0];
    const uint64_t tile_base = tile * kSortTile;
    const unsigned dmask = (1u << pp.bits) - 1;

    uint64_t k[kSortKPT];
    uint32_t v[kSortKPT];
    uint32_t rank[kSortKPT];
#pragma unroll
    for (int i = 0; i < kSortKPT; ++i) {
        uint64_t idx = tile_base + warp * (32 * kSortKPT) + i * 32 + lane;
        bool ok = idx < n;
        k[i] = ok ? __ldcs(kin + idx) : 0;
        if (HAS_VAL) v[i] = ok ? __ldcs(vin + idx) : 0;
    }
#pragma unroll
    for (int i = 0; i < kSortKPT; ++i) {
        uint64_t idx = tile_base + warp * (32 * kSortKPT) + i * 32 + lane;
        unsigned d = idx < n ? (unsigned)(k[i] >> pp.shift) & dmask : (unsigned)kRadix;
#if TC_SORT_BALLOT
        // warp multi-split: lanes with the same digit agree on every digit bit
        unsigned peers = __ballot_sync(TC_FULL_MASK, idx < n);
        if (idx >= n) peers = ~peers;
#pragma unroll
        for (int b = 0; b < kRadixBits; ++b) {
            const unsigned bit = (d >> b) & 1u;
            const unsigned bal = __ballot_sync(TC_FULL_MASK, bit);
            peers &= b < pp.bits ? (bit ? bal : ~bal) : 0xffffffffu;
        }
#else
        unsigned peers = __match_any_sync(TC_FULL_MASK, d);
#endif
        int leader = __ffs(peers) - 1;
        unsigned old = 0;
        if ((int)lane == leader && d < (unsigned)kRadix) {
            old = s_whist[warp * kRadix + d];
            s_whist[warp * kRadix + d] = old + __popc(peers);
        }
        old = __shfl_sync(TC_FULL_MASK, old, leader);
        rank[i] = old + __popc(peers & lanemask_lt());
        __syncwarp();
    }
    __syncthreads();

    // Per digit (one per thread): exclusive prefix over warps, tile total, look-back.
    const unsigned d = threadIdx.x;
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
        uint32_t c = s_whist[w * kRadix + d];
        s_whist[w * kRadix + d] = total;
        total += c;
    }
    uint64_t *my = status + tile * kRadix + d;
    uint64_t excl = 0;
    if (tile == 0) {
        st_volatile_u64(my, kFlagP | total);
    } else {
        st_volatile_u64(my, kFlagA | total);
        // Look back in batches of kLook predecessors (independent loads, one round trip),
        // consuming them newest-first until an inclusive prefix; a tile that has not
        // published yet is re-polled alone.
        constexpr int kLook = 8;
        int64_t j = (int64_t)tile - 1;
        bool done = false;
        while (!done) {
            uint64_t st[kLook];
#pragma unroll
            for (int q = 0; q < kLook; ++q)
                st[q] = j - q >= 0 ? ld_volatile_u64(status + (uint64_t)(j - q) * kRadix + d) : kFlagP;
            int q = 0;
            for (; q < kLook; ++q) {
                const uint64_t flag = st[q] & ~kValMask;
                if (flag == 0) {  // not published yet: re-poll from here
#if TC_SORT_SLEEP
                    __nanosleep(TC_SORT_SLEEP);
#endif
                    break;
                }
                excl += st[q] & kValMask;
                if (flag == kFlagP) { done = true; break; }
            }
            j -= q;
        }
        st_volatile_u64(my, kFlagP | (excl + total));
    }
    s_gbase[d] = digit_base[d] + excl;
    uint32_t tvalid;
    uint32_t tstart = block_exclusive_scan<uint32_t>(total, s_scan, &tvalid);
    s_tstart[d] = tstart;
    __syncthreads();

#pragma unroll
    for (int i = 0; i < kSortKPT; ++i) {
        uint64_t idx = tile_base + warp * (32 * kSortKPT) + i * 32 + lane;
        if (idx < n) {
            unsigned dd = (unsigned)(k[i] >> pp.shift) & dmask;
            uint32_t pos = s_tstart[dd] + s_whist[warp * kRadix + dd] + rank[i];
            s_keys[pos] = k[i];
            if (HAS_VAL) s_vals[pos] = v[i];
        }
    }
    __syncthreads();

    const uint64_t split_mask = split_bits >= 64 ? ~0ull : ((1ull << split_bits) - 1);
    for (uint32_t p = threadIdx.x; p < tvalid; p += kSortThreads) {
        uint64_t key = s_keys[p];
        unsigned dd = (unsigned)(key >> pp.shift) & dmask;
        uint64_t g = s_gbase[dd] + (p - s_tstart[dd]);
        if (MODE == kOutKeys) {
            __stcs(kout + g, key);
            if (HAS_VAL) __stcs(vout + g, s_vals[p]);
        } else if (MODE == kOutSoA) {
            __stcs(out_a + g, (uint32_t)(key >> split_bits));
            __stcs(out_b + g, (uint32_t)(key & split_mask));
        } else {
            __stcs(reinterpret_cast<uint2 *>(out_a) + g,
                   make_uint2((uint32_t)(key >> split_bits), (uint32_t)(key & split_mask)));
        }
    }
}

// No-pass "sort" (all keys equal in the plan's bit range): split/copy only.
__global__ void k_split_copy(const uint64_t *__restrict__ k, uint64_t n, int mode,
                             uint32_t *__restrict__ a, uint32_t *__restrict__ b, int split) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t mask = split >= 64 ? ~0ull : ((1ull << split) - 1);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint64_t key = k[i];
        if (mode == kOutSoA) {
            a[i] = (uint32_t)(key >> split);
            b[i] = (uint32_t)(key & mask);
        } else {
            reinterpret_cast<uint2 *>(a)[i] = make_uint2((uint32_t)(key >> split), (uint32_t)(key & mask));
        }
    }
}

size_t pass_smem(bool has_val) {
    size_t b = kSortTile * 8 + kRadix * 8 + kSortWarps * kRadix * 4 + kRadix * 4 + 32 * 4 + 16;
    if (has_val) b += kSortTile * 4;
    return b;
}

template <int MODE, bool HAS_VAL>
int launch_pass(const uint64_t *kin, uint64_t *kout, const uint32_t *vin, uint32_t *vout,
                uint32_t *a, uint32_t *b, int split, uint64_t n, PassParams pp,
                const uint64_t *base, uint64_t *status, unsigned *counter, cudaStream_t s) {
    auto kern = k_radix_pass<MODE, HAS_VAL>;
    size_t sm = pass_smem(HAS_VAL);
    static bool configured = false;  // per template instance
    if (!configured) {
        TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        configured = true;
    }
    uint64_t tiles = (n + kSortTile - 1) / kSortTile;
    kern<<<(unsigned)tiles, kSortThreads, sm, s>>>(kin, kout, vin, vout, a, b, split, n, pp, base,
                                                   status, counter);
    TC_LAUNCHED();
    return 0;
}

}  // namespace

RadixPlan make_radix_plan(int key_bits) {
    RadixPlan p;
    if (key_bits <= 0) return p;
    p.npass = (key_bits + kRadixBits - 1) / kRadixBits;
    int base = key_bits / p.npass, extra = key_bits % p.npass, sh = 0;
    for (int i = 0; i < p.npass; ++i) {
        p.bits[i] = base + (i < extra ? 1 : 0);
        p.shift[i] = sh;
        sh += p.bits[i];
    }
    return p;
}

int radix_histogram(const uint64_t *keys, uint64_t n, const RadixPlan &plan, uint32_t *hist,
                    cudaStream_t s) {
    if (plan.npass == 0 || n == 0) return 0;
    unsigned grid = grid_for(n, 256 * 16, kSMs * 8);
    k_digit_hist<<<grid, 256, 0, s>>>(keys, n, plan, hist);
    TC_LAUNCHED();
    return 0;
}

int radix_sort(uint64_t *keys, uint64_t *alt, uint32_t *vals, uint32_t *valt, uint64_t n,
               const RadixPlan &plan, const uint32_t *hist, int out_mode, uint32_t *out_a,
               uint32_t *out_b, int split_bits, uint64_t **sorted_keys, uint32_t **sorted_vals,
               cudaStream_t s) {
    if (sorted_keys) *sorted_keys = keys;
    if (sorted_vals) *sorted_vals = vals;
    if (n == 0) return 0;
    if (plan.npass == 0) {
        if (out_mode != kOutKeys) {
            k_split_copy<<<grid_for(n, 256, kSMs * 16), 256, 0, s>>>(keys, n, out_mode, out_a, out_b,
                                                                  split_bits);
            TC_LAUNCHED();
        }
        return 0;
    }
    const uint64_t tiles = (n + kSortTile - 1) / kSortTile;
    uint64_t *base = nullptr, *status = nullptr;
    unsigned *counters = nullptr;
    TC_CHECK(dalloc_t(&base, (size_t)plan.npass * kRadix, s));
    TC_CHECK(dalloc_t(&status, (size_t)tiles * kRadix, s));
    TC_CHECK(dalloc_t(&counters, kMaxPasses, s));
    TC_CUDA(cudaMemsetAsync(counters, 0, kMaxPasses * sizeof(unsigned), s));
    k_digit_base<<<1, kRadix, 0, s>>>(hist, plan.npass, base);
    TC_LAUNCHED();

    const bool hv = vals != nullptr;
    uint64_t *kin = keys, *kout = alt;
    uint32_t *vin = vals, *vout = valt;
    for (int p = 0; p < plan.npass; ++p) {
        TC_CUDA(cudaMemsetAsync(status, 0, (size_t)tiles * kRadix * sizeof(uint64_t), s));
        PassParams pp{plan.shift[p], plan.bits[p]};
        const bool last = p == plan.npass - 1;
        const uint64_t *pb = base + (size_t)p * kRadix;
        int rc;
        if (last && out_mode == kOutSoA) {
            rc = launch_pass<kOutSoA, false>(kin, nullptr, nullptr, nullptr, out_a, out_b,
                                             split_bits, n, pp, pb, status, counters + p, s);
        } else if (last && out_mode == kOutAoS) {
            rc = launch_pass<kOutAoS, false>(kin, nullptr, nullptr, nullptr, out_a, nullptr,
                                             split_bits, n, pp, pb, status, counters + p, s);
        } else if (hv) {
            rc = launch_pass<kOutKeys, true>(kin, kout, vin, vout, nullptr, nullptr, 0, n, pp, pb,
                                             status, counters + p, s);
        } else {
            rc = launch_pass<kOutKeys, false>(kin, kout, nullptr, nullptr, nullptr, nullptr, 0, n,
                                              pp, pb, status, counters + p, s);
        }
        if (rc) return rc;
        if (!(last && out_mode != kOutKeys)) {
            uint64_t *t = kin; kin = kout; kout = t;
            uint32_t *tv = vin; vin = vout; vout = tv;
        }
    }
    if (sorted_keys) *sorted_keys = kin;
    if (sorted_vals) *sorted_vals = vin;
    dfree(base, s);
    dfree(status, s);
    dfree(counters, s);
    return 0;
}

}  // namespace tc
