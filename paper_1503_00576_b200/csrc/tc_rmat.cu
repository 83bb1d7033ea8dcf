// tc_rmat.cu -- device R-MAT generator, bit-identical to the reference
// tricount.generators.rmat (reference generators.py:203-284) for the same seed.
//
// The reference draws, per batch, `scale` arrays of float64 from numpy's
// default_rng(seed) (PCG64 XSL-RR: state = state*M + inc, then output; random() =
// (next64 >> 11) * 2^-53), descends the 2x2 quadrant split, drops self-loops, keeps the
// first occurrence of every canonical key (lo << 32 | hi) in draw order, drops keys it
// already has, takes the first `need` survivors and merges them into the sorted set.
// Here every draw is computed independently by jumping the 128-bit LCG to its stream
// position, and "first occurrence in draw order" is recovered with a stable key/value
// radix sort (value = draw index) plus a scan over draw positions.  Input production for
// parity tests and the bench only; not on the timed path.
#include <algorithm>
#include <vector>

#include "tc_common.cuh"
#include "tc_internal.h"

namespace tc {

namespace {

typedef unsigned __int128 u128;
constexpr int kJumpBits = 40;
constexpr int kMaxScale = 30;
constexpr int kRmatJ = 16;  // consecutive draws per thread per level

struct JumpTable {
    unsigned long long a_lo[kJumpBits], a_hi[kJumpBits], c_lo[kJumpBits], c_hi[kJumpBits];
};
__constant__ JumpTable c_jump;

struct LevelStates {
    unsigned long long lo[kMaxScale], hi[kMaxScale];
};

const u128 kPcgMult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;

__device__ __forceinline__ u128 mk128(unsigned long long hi, unsigned long long lo) {
    return ((u128)hi << 64) | lo;
}

__device__ __forceinline__ uint64_t pcg_out(u128 s) {
    const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    const unsigned rot = (unsigned)(s >> 122);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
}

// Draw-position-parallel level loop (reference generators.py:249-256).  Key layout:
// (lo << scale) | hi for a proper edge, 1 << (2*scale) for a self-loop (sorts last).
__global__ void __launch_bounds__(256) k_rmat_draw(uint64_t batch, int scale, double a, double t_ab,
                                                   double t_abc, LevelStates ls,
                                                   unsigned long long inc_hi,
                                                   unsigned long long inc_lo,
                                                   uint64_t *__restrict__ keys,
                                                   uint32_t *__restrict__ idx) {
    const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
    const u128 inc = mk128(inc_hi, inc_lo);
    const uint64_t j0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRmatJ;
    if (j0 >= batch) return;
    uint32_t src[kRmatJ], dst[kRmatJ];
#pragma unroll
    for (int j = 0; j < kRmatJ; ++j) src[j] = dst[j] = 0;
    for (int l = 0; l < scale; ++l) {
        u128 s = mk128(ls.hi[l], ls.lo[l]);
        uint64_t d = j0;
        for (int k = 0; d; ++k, d >>= 1)
            if (d & 1) s = mk128(c_jump.a_hi[k], c_jump.a_lo[k]) * s + mk128(c_jump.c_hi[k], c_jump.c_lo[k]);
#pragma unroll
        for (int j = 0; j < kRmatJ; ++j) {
            s = s * mult + inc;
            const double r = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
            const uint32_t sb = r >= t_ab;
            const uint32_t db = (r >= a && r < t_ab) || r >= t_abc;
            src[j] = (src[j] << 1) | sb;
            dst[j] = (dst[j] << 1) | db;
        }
    }
#pragma unroll
    for (int j = 0; j < kRmatJ; ++j) {
        const uint64_t p = j0 + j;
        if (p < batch) {
            const uint32_t lo = src[j] < dst[j] ? src[j] : dst[j];
            const uint32_t hi = src[j] < dst[j] ? dst[j] : src[j];
            keys[p] = src[j] == dst[j] ? (1ull << (2 * scale)) : (((uint64_t)lo << scale) | hi);
            idx[p] = (uint32_t)p;
        }
    }
}

// First occurrence of each valid key not already in `have` -> flag[draw index] = 1.
__global__ void k_rmat_heads(const uint64_t *__restrict__ sk, const uint32_t *__restrict__ sv,
                             uint64_t batch, int scale, const uint64_t *__restrict__ have,
                             uint64_t have_n, uint32_t *__restrict__ flag,
                             uint64_t *__restrict__ cand) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t lim = 1ull << (2 * scale);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < batch; i += stride) {
        const uint64_t k = sk[i];
        if (k >= lim) continue;
        if (i > 0 && sk[i - 1] == k) continue;
        if (have_n) {
            uint64_t lo = 0, n = have_n;
            while (n > 0) {
                const uint64_t half = n >> 1;
                if (have[lo + half] < k) { lo += half + 1; n -= half + 1; }
                else n = half;
            }
            if (lo < have_n && have[lo] == k) continue;
        }
        const uint32_t j = sv[i];
        flag[j] = 1;
        cand[j] = k;
    }
}

__global__ void __launch_bounds__(256) k_tile_count(const uint32_t *__restrict__ flag, uint64_t n,
                                                    uint32_t *__restrict__ sums) {
    const uint64_t b = (uint64_t)blockIdx.x * 4096;
    uint32_t acc = 0;
    for (uint64_t i = b + threadIdx.x; i < b + 4096 && i < n; i += 256) acc += flag[i];
    __shared__ uint32_t s_red[8];
    acc = warp_sum(acc);
    if (lane_id() == 0) s_red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < 8; ++w) t += s_red[w];
        sums[blockIdx.x] = t;
    }
}

__global__ void k_scan_tiles(uint32_t *__restrict__ sums, uint64_t nt,
                             unsigned long long *__restrict__ total) {
    __shared__ uint32_t s_w[32];
    uint32_t carry = 0;
    for (uint64_t b = 0; b < nt; b += blockDim.x) {
        const uint64_t i = b + threadIdx.x;
        const uint32_t x = i < nt ? sums[i] : 0;
        uint32_t t;
        const uint32_t e = block_exclusive_scan<uint32_t>(x, s_w, &t);
        if (i < nt) sums[i] = carry + e;
        carry += t;
    }
    if (threadIdx.x == 0) *total = carry;
}

// Selected candidates (the first `need` in draw order) -> out[rank].
__global__ void __launch_bounds__(256) k_rmat_select(const uint32_t *__restrict__ flag,
                                                     const uint64_t *__restrict__ cand, uint64_t n,
                                                     const uint32_t *__restrict__ tile_base,
                                                     uint64_t need, uint64_t *__restrict__ out) {
    __shared__ uint32_t s_w[32];
    const uint64_t b = (uint64_t)blockIdx.x * 4096;
    uint32_t carry = tile_base[blockIdx.x];
    for (uint64_t c = b; c < b + 4096; c += 256) {
        const uint64_t i = c + threadIdx.x;
        const uint32_t f = i < n ? flag[i] : 0;
        uint32_t t;
        const uint32_t e = block_exclusive_scan<uint32_t>(f, s_w, &t);
        if (f && (uint64_t)(carry + e) < need) out[carry + e] = cand[i];
        carry += t;
    }
}

__global__ void k_sym(const uint64_t *__restrict__ have, uint64_t n, int scale,
                      uint64_t *__restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t mask = (1ull << scale) - 1;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t k = have[i];
        const uint64_t lo = k >> scale, hi = k & mask;
        out[2 * i] = k;
        out[2 * i + 1] = (hi << scale) | lo;
    }
}

__global__ void k_max_hi(const uint64_t *__restrict__ have, uint64_t n, int scale,
                         uint32_t *__restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t mask = (1ull << scale) - 1;
    uint32_t best = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t h = (uint32_t)(have[i] & mask);
        best = h > best ? h : best;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const uint32_t y = __shfl_xor_sync(TC_FULL_MASK, best, o);
        best = y > best ? y : best;
    }
    if (lane_id() == 0) atomicMax(out, best);
}

u128 advance_host(u128 s, u128 inc, uint64_t delta) {
    u128 am = 1, ap = 0, cm = kPcgMult, cp = inc;
    while (delta) {
        if (delta & 1) {
            am *= cm;
            ap = ap * cm + cp;
        }
        cp = (cm + 1) * cp;
        cm *= cm;
        delta >>= 1;
    }
    return am * s + ap;
}

// c_jump[k] = the affine map advancing the LCG by 2^k steps (s -> a*s + c).
int upload_jump(u128 inc, cudaStream_t s) {
    static JumpTable jt;  // host source of an async copy: keep it alive
    TC_CUDA(cudaStreamSynchronize(s));
    u128 am = kPcgMult, ap = inc;
    for (int k = 0; k < kJumpBits; ++k) {
        jt.a_lo[k] = (unsigned long long)am;
        jt.a_hi[k] = (unsigned long long)(am >> 64);
        jt.c_lo[k] = (unsigned long long)ap;
        jt.c_hi[k] = (unsigned long long)(ap >> 64);
        ap = ap * (am + 1);
        am = am * am;
    }
    TC_CUDA(cudaMemcpyToSymbolAsync(c_jump, &jt, sizeof(jt), 0, cudaMemcpyHostToDevice, s));
    return 0;
}

}  // namespace

int rmat_dev(int scale, int edge_factor, const double probs[4], const uint64_t state[2],
             const uint64_t inc_in[2], uint32_t **pairs_out, uint64_t *npairs_out,
             uint64_t *nverts_out, cudaStream_t s) {
    if (scale < 1 || scale > kMaxScale || 2 * scale + 1 > 63) {
        set_error("rmat: scale must be in 1..30");
        return -1;
    }
    const double a = probs[0], b = probs[1], c = probs[2];
    const double t_ab = a + b, t_abc = a + b + c;
    const uint64_t n = 1ull << scale;
    const uint64_t target = (uint64_t)edge_factor * n;
    if (target > n * (n - 1) / 2) {
        set_error("rmat: edge_factor too large for a simple graph");
        return -1;
    }
    const u128 s0 = ((u128)state[0] << 64) | state[1];
    const u128 inc = ((u128)inc_in[0] << 64) | inc_in[1];
    TC_CHECK(upload_jump(inc, s));
    const RadixPlan draw_plan = make_radix_plan(2 * scale + 1);
    const RadixPlan have_plan = make_radix_plan(2 * scale);
    uint64_t *have = nullptr;
    uint64_t have_n = 0, drawn = 0;
    int stalled = 0;
    uint32_t *hist = nullptr, *tsum = nullptr;
    unsigned long long *d_total = nullptr;
    TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
    TC_CHECK(dalloc_t(&d_total, 1, s));
    while (have_n < target) {
        const uint64_t need = target - have_n;
        uint64_t batch = (uint64_t)((double)need * 1.3);
        if (batch < 4096) batch = 4096;
        if (batch >= (1ull << 32)) {
            set_error("rmat: batch exceeds 2^32 draws");
            return -1;
        }
        LevelStates ls;
        for (int l = 0; l < scale; ++l) {
            const u128 st = advance_host(s0, inc, drawn + (uint64_t)l * batch);
            ls.lo[l] = (unsigned long long)st;
            ls.hi[l] = (unsigned long long)(st >> 64);
        }
        uint64_t *keys = nullptr, *alt = nullptr, *cand = nullptr, *sk = nullptr;
        uint32_t *idx = nullptr, *valt = nullptr, *flag = nullptr, *sv = nullptr;
        TC_CHECK(dalloc_t(&keys, batch, s));
        TC_CHECK(dalloc_t(&alt, batch, s));
        TC_CHECK(dalloc_t(&idx, batch, s));
        TC_CHECK(dalloc_t(&valt, batch, s));
        const uint64_t threads = (batch + kRmatJ - 1) / kRmatJ;
        k_rmat_draw<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
            batch, scale, a, t_ab, t_abc, ls, (unsigned long long)(inc >> 64),
            (unsigned long long)inc, keys, idx);
        TC_LAUNCHED();
        drawn += batch * (uint64_t)scale;
        TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
        TC_CHECK(radix_histogram(keys, batch, draw_plan, hist, s));
        TC_CHECK(radix_sort(keys, alt, idx, valt, batch, draw_plan, hist, kOutKeys, nullptr, nullptr, 0,
                            &sk, &sv, s));
        // free the non-result ping-pong halves before the next big allocations
        uint64_t *kfree = sk == keys ? alt : keys;
        uint32_t *vfree = sv == idx ? valt : idx;
        dfree(kfree, s);
        dfree(vfree, s);
        TC_CHECK(dalloc_t(&flag, batch, s));
        TC_CHECK(dalloc_t(&cand, batch, s));
        TC_CUDA(cudaMemsetAsync(flag, 0, batch * sizeof(uint32_t), s));
        k_rmat_heads<<<grid_for(batch, 256, kSMs * 16), 256, 0, s>>>(sk, sv, batch, scale, have, have_n,
                                                                     flag, cand);
        TC_LAUNCHED();
        dfree(sk, s);
        dfree(sv, s);
        const uint64_t nt = (batch + 4095) / 4096;
        TC_CHECK(dalloc_t(&tsum, nt, s));
        k_tile_count<<<(unsigned)nt, 256, 0, s>>>(flag, batch, tsum);
        TC_LAUNCHED();
        k_scan_tiles<<<1, 512, 0, s>>>(tsum, nt, d_total);
        TC_LAUNCHED();
        unsigned long long cands = 0;
        TC_CUDA(cudaMemcpyAsync(&cands, d_total, sizeof(cands), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
        const uint64_t take = cands < need ? cands : need;
        uint64_t *merged = nullptr, *malt = nullptr;
        if (take) {
            TC_CHECK(dalloc_t(&merged, have_n + take, s));
            if (have_n)
                TC_CUDA(cudaMemcpyAsync(merged, have, have_n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
            k_rmat_select<<<(unsigned)nt, 256, 0, s>>>(flag, cand, batch, tsum, need, merged + have_n);
            TC_LAUNCHED();
        }
        dfree(flag, s);
        dfree(cand, s);
        dfree(tsum, s);
        if (take == 0) {
            if (++stalled >= 25) {
                set_error("rmat sampling saturated below the target edge count");
                return -1;
            }
            continue;
        }
        stalled = 0;
        dfree(have, s);
        TC_CHECK(dalloc_t(&malt, have_n + take, s));
        TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
        TC_CHECK(radix_histogram(merged, have_n + take, have_plan, hist, s));
        uint64_t *sorted = nullptr;
        TC_CHECK(radix_sort(merged, malt, nullptr, nullptr, have_n + take, have_plan, hist, kOutKeys,
                            nullptr, nullptr, 0, &sorted, nullptr, s));
        dfree(sorted == merged ? malt : merged, s);
        have = sorted;
        have_n += take;
    }
    // edge_array_from_undirected (reference graph.py:265-276): both directions, sorted.
    uint32_t *maxhi = nullptr;
    TC_CHECK(dalloc_t(&maxhi, 1, s));
    TC_CUDA(cudaMemsetAsync(maxhi, 0, sizeof(uint32_t), s));
    k_max_hi<<<grid_for(target, 256, kSMs * 8), 256, 0, s>>>(have, target, scale, maxhi);
    TC_LAUNCHED();
    uint64_t *both = nullptr, *balt = nullptr;
    uint32_t *pairs = nullptr;
    TC_CHECK(dalloc_t(&both, 2 * target, s));
    k_sym<<<grid_for(target, 256, kSMs * 16), 256, 0, s>>>(have, target, scale, both);
    TC_LAUNCHED();
    dfree(have, s);
    TC_CHECK(dalloc_t(&balt, 2 * target, s));
    TC_CHECK(dalloc_t(&pairs, 4 * target + 4, s, true));  // handed to the caller
    TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
    TC_CHECK(radix_histogram(both, 2 * target, have_plan, hist, s));
    TC_CHECK(radix_sort(both, balt, nullptr, nullptr, 2 * target, have_plan, hist, kOutAoS, pairs,
                        nullptr, scale, nullptr, nullptr, s));
    uint32_t mh = 0;
    TC_CUDA(cudaMemcpyAsync(&mh, maxhi, sizeof(mh), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(both, s);
    dfree(balt, s);
    dfree(maxhi, s);
    dfree(hist, s);
    dfree(d_total, s);
    *pairs_out = pairs;
    *npairs_out = 2 * target;
    *nverts_out = (uint64_t)mh + 1;
    return 0;
}

// --------------------------------------------------------------------- BA ---
// Reference generators.py:287-322 barabasi_albert: inherently sequential (each new
// vertex samples targets from the degree-weighted list built so far), so the sampling
// loop runs on the host -- numpy's Generator.integers restated: Lemire's bounded method
// on PCG64's buffered 32-bit outputs -- and only the symmetrisation + sort runs on the
// device.  Input production only.
namespace {

struct HostPcg {
    u128 s, inc;
    bool has = false;
    uint32_t buf = 0;
    uint32_t next32() {
        if (has) {
            has = false;
            return buf;
        }
        s = s * kPcgMult + inc;
        const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
        const unsigned rot = (unsigned)(s >> 122);
        const uint64_t x = hi ^ lo;
        const uint64_t v = (x >> rot) | (x << ((64 - rot) & 63));
        has = true;
        buf = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    uint32_t bounded(uint32_t high) {  // integers(0, high)
        const uint32_t rng = high - 1;
        if (rng == 0) return 0;
        const uint32_t excl = rng + 1;
        uint64_t m = (uint64_t)next32() * excl;
        uint32_t left = (uint32_t)m;
        if (left < excl) {
            const uint32_t thr = (0xFFFFFFFFu - rng) % excl;
            while (left < thr) {
                m = (uint64_t)next32() * excl;
                left = (uint32_t)m;
            }
        }
        return (uint32_t)(m >> 32);
    }
};

__global__ void k_sym_pairs(const uint2 *__restrict__ pairs, uint64_t np, int vb,
                            uint64_t *__restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
        const uint2 p = pairs[i];
        out[2 * i] = ((uint64_t)p.x << vb) | p.y;
        out[2 * i + 1] = ((uint64_t)p.y << vb) | p.x;
    }
}

}  // namespace

int ba_dev(uint64_t n, uint32_t m_attach, const uint64_t state[2], const uint64_t inc[2],
           uint32_t **pairs_out, uint64_t *npairs_out, uint64_t *nverts_out, cudaStream_t s) {
    if (n < 2 || m_attach < 1 || m_attach >= n || m_attach > 1024 || n >= (1ull << 32)) {
        set_error("barabasi_albert: need 2 <= n < 2^32 and 1 <= m_attach < min(n, 1024)");
        return -1;
    }
    HostPcg g;
    g.s = ((u128)state[0] << 64) | state[1];
    g.inc = ((u128)inc[0] << 64) | inc[1];
    const uint64_t count = (uint64_t)m_attach * (m_attach - 1) / 2 + (n - m_attach) * (uint64_t)m_attach;
    uint32_t *hp = nullptr;
    TC_CUDA(cudaHostAlloc(&hp, 8 * (count ? count : 1), cudaHostAllocDefault));
    std::vector<uint32_t> rep;
    rep.reserve(2 * count + 2);
    uint64_t np = 0;
    for (uint32_t i = 0; i < m_attach; ++i)
        for (uint32_t j = i + 1; j < m_attach; ++j) {
            hp[2 * np] = i;
            hp[2 * np + 1] = j;
            ++np;
            rep.push_back(i);
            rep.push_back(j);
        }
    std::vector<uint32_t> tg, draws;
    for (uint64_t v = m_attach; v < n; ++v) {
        tg.clear();
        if (rep.empty()) tg.push_back(g.bounded((uint32_t)v));
        while (tg.size() < m_attach) {
            const uint32_t k = m_attach - (uint32_t)tg.size();
            draws.resize(k);
            for (uint32_t d = 0; d < k; ++d) draws[d] = g.bounded((uint32_t)rep.size());
            for (uint32_t d = 0; d < k; ++d) {
                const uint32_t t = rep[draws[d]];
                if (std::find(tg.begin(), tg.end(), t) == tg.end()) tg.push_back(t);
            }
        }
        std::sort(tg.begin(), tg.end());
        for (uint32_t t : tg) {
            hp[2 * np] = t;
            hp[2 * np + 1] = (uint32_t)v;
            ++np;
            rep.push_back(t);
            rep.push_back((uint32_t)v);
        }
    }
    // edge_array_from_undirected (reference graph.py:265-276): both directions, sorted
    const int vb = bits_for(n - 1);
    const RadixPlan plan = make_radix_plan(2 * vb);
    uint32_t *dcanon = nullptr, *pairs = nullptr, *hist = nullptr;
    uint64_t *keys = nullptr, *alt = nullptr;
    TC_CHECK(dalloc_t(&dcanon, 2 * np, s));
    TC_CHECK(dalloc_t(&keys, 2 * np, s));
    TC_CHECK(dalloc_t(&alt, 2 * np, s));
    TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
    TC_CHECK(dalloc_t(&pairs, 4 * np + 4, s, true));  // handed to the caller
    TC_CUDA(cudaMemcpyAsync(dcanon, hp, 8 * np, cudaMemcpyHostToDevice, s));
    TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
    k_sym_pairs<<<grid_for(np, 256, kSMs * 16), 256, 0, s>>>(reinterpret_cast<const uint2 *>(dcanon),
                                                              np, vb, keys);
    TC_LAUNCHED();
    TC_CHECK(radix_histogram(keys, 2 * np, plan, hist, s));
    TC_CHECK(radix_sort(keys, alt, nullptr, nullptr, 2 * np, plan, hist, kOutAoS, pairs, nullptr, vb,
                        nullptr, nullptr, s));
    TC_CUDA(cudaStreamSynchronize(s));
    cudaFreeHost(hp);
    dfree(dcanon, s);
    dfree(keys, s);
    dfree(alt, s);
    dfree(hist, s);
    *pairs_out = pairs;
    *npairs_out = 2 * np;
    *nverts_out = n;  // every vertex >= 1 edge (BA attaches every new vertex)
    return 0;
}

// ---- random geometric graph (BASELINE config 5; no reference generator exists) --------
// Points: numpy default_rng(seed).random((n, 2)) -- draw 2i is x_i, draw 2i+1 is y_i.
// Edge {i, j}, i != j, iff dx*dx + dy*dy < r*r in IEEE double without contraction (the
// oracle, oracle/tricount_oracle.c or_rgg_pairs, evaluates the same expression).  Cells
// of side 1/G >= r (G = floor(1/r) - 1) so every neighbour lies in the 3x3 block; points
// are bucketed by a stable radix sort of cell ids, counted and emitted warp-per-point
// (ballot compaction), and the emitted (i, j) keys radix-sorted into the reference's
// lexicographic both-directions layout.
namespace {

constexpr int kRggJ = 8;  // points per thread in the draw kernel

__global__ void __launch_bounds__(256) k_rgg_points(uint64_t n, unsigned long long s_hi,
                                                    unsigned long long s_lo,
                                                    unsigned long long inc_hi,
                                                    unsigned long long inc_lo, uint32_t grid,
                                                    double *__restrict__ xs, double *__restrict__ ys,
                                                    uint64_t *__restrict__ cell,
                                                    uint32_t *__restrict__ idx) {
    const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
    const u128 inc = mk128(inc_hi, inc_lo);
    const uint64_t p0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRggJ;
    if (p0 >= n) return;
    u128 s = mk128(s_hi, s_lo);
    uint64_t d = 2 * p0;
    for (int k = 0; d; ++k, d >>= 1)
        if (d & 1) s = mk128(c_jump.a_hi[k], c_jump.a_lo[k]) * s + mk128(c_jump.c_hi[k], c_jump.c_lo[k]);
    for (int j = 0; j < kRggJ && p0 + j < n; ++j) {
        s = s * mult + inc;
        const double x = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
        s = s * mult + inc;
        const double y = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
        const uint64_t p = p0 + j;
        xs[p] = x;
        ys[p] = y;
        uint32_t cx = (uint32_t)(x * grid), cy = (uint32_t)(y * grid);
        cx = cx < grid ? cx : grid - 1;
        cy = cy < grid ? cy : grid - 1;
        cell[p] = (uint64_t)cy * grid + cx;
        idx[p] = (uint32_t)p;
    }
}

__global__ void k_rgg_gather(const uint32_t *__restrict__ sidx, uint64_t n, const double *__restrict__ xs,
                             const double *__restrict__ ys, double2 *__restrict__ sxy) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
        const uint32_t i = sidx[p];
        sxy[p] = make_double2(xs[i], ys[i]);
    }
}

// cstart[c] = first sorted position with cell >= c, c in [0, cells]
__global__ void k_rgg_cell_start(const uint64_t *__restrict__ scell, uint64_t n, uint64_t cells,
                                 uint32_t *__restrict__ cstart) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= cells; c += stride) {
        uint64_t a = 0, len = n;
        while (len > 0) {
            const uint64_t h = len >> 1;
            if (scell[a + h] < c) { a += h + 1; len -= h + 1; }
            else len = h;
        }
        cstart[c] = (uint32_t)a;
    }
}

__device__ __forceinline__ bool rgg_close(double2 a, double2 b, double r2) {
    const double dx = __dsub_rn(a.x, b.x), dy = __dsub_rn(a.y, b.y);
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) < r2;
}

// EMIT = false: deg[i] = neighbours of i.  EMIT = true: keys at off[i] (unsorted).
template <bool EMIT>
__global__ void __launch_bounds__(256) k_rgg_scan(const double2 *__restrict__ sxy,
                                                  const uint32_t *__restrict__ sidx, uint64_t n,
                                                  const uint32_t *__restrict__ cstart, uint32_t grid,
                                                  double r2, int vb, uint32_t *__restrict__ deg,
                                                  const int64_t *__restrict__ off,
                                                  uint64_t *__restrict__ keys) {
    const unsigned lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t p = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); p < n; p += warps) {
        const double2 me = sxy[p];
        const uint32_t i = sidx[p];
        uint32_t cx = (uint32_t)(me.x * grid), cy = (uint32_t)(me.y * grid);
        cx = cx < grid ? cx : grid - 1;
        cy = cy < grid ? cy : grid - 1;
        const uint32_t x0 = cx ? cx - 1 : 0, x1 = cx + 1 < grid ? cx + 1 : grid - 1;
        const uint32_t y0 = cy ? cy - 1 : 0, y1 = cy + 1 < grid ? cy + 1 : grid - 1;
        uint64_t base = EMIT ? (uint64_t)off[i] : 0;
        uint32_t cnt = 0;
        for (uint32_t yy = y0; yy <= y1; ++yy) {
            const uint32_t lo = cstart[(uint64_t)yy * grid + x0];
            const uint32_t hi = cstart[(uint64_t)yy * grid + x1 + 1];
            for (uint32_t q0 = lo; q0 < hi; q0 += 32) {
                const uint32_t q = q0 + lane;
                bool ok = false;
                uint32_t j = 0;
                if (q < hi && q != p) {
                    ok = rgg_close(me, sxy[q], r2);
                    j = sidx[q];
                }
                const unsigned mask = __ballot_sync(TC_FULL_MASK, ok);
                if (EMIT) {
                    if (ok) keys[base + __popc(mask & ((1u << lane) - 1))] = ((uint64_t)i << vb) | j;
                    base += __popc(mask);
                } else {
                    cnt += __popc(mask);
                }
            }
        }
        if (!EMIT && lane == 0) deg[i] = cnt;
    }
}

__global__ void k_last_nonzero(const uint32_t *__restrict__ deg, uint64_t n,
                               unsigned long long *__restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    unsigned long long best = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        if (deg[i]) best = i + 1;
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(TC_FULL_MASK, best, o);
        best = y > best ? y : best;
    }
    if (lane_id() == 0 && best) atomicMax(out, best);
}

}  // namespace

int rgg_dev(uint64_t n, double radius, const uint64_t state[2], const uint64_t inc_in[2],
            uint32_t **pairs_out, uint64_t *npairs_out, uint64_t *nverts_out, cudaStream_t s) {
    *pairs_out = nullptr;
    *npairs_out = *nverts_out = 0;
    if (n < 1 || n >= (1ull << 32) || !(radius > 0) || !(radius < 2)) {
        set_error("random_geometric: need 1 <= n < 2^32 and 0 < radius < 2");
        return -1;
    }
    const double r2 = radius * radius;
    const double fg = floor(1.0 / radius) - 1.0;
    const uint32_t grid = fg < 1 ? 1u : (fg > 65535 ? 65535u : (uint32_t)fg);
    const uint64_t cells = (uint64_t)grid * grid;
    const u128 s0 = ((u128)state[0] << 64) | state[1];
    const u128 inc = ((u128)inc_in[0] << 64) | inc_in[1];
    TC_CHECK(upload_jump(inc, s));
    double *xs = nullptr, *ys = nullptr;
    double2 *sxy = nullptr;
    uint64_t *cell = nullptr, *calt = nullptr, *scell = nullptr;
    uint32_t *idx = nullptr, *ialt = nullptr, *sidx = nullptr, *hist = nullptr, *cstart = nullptr;
    uint32_t *deg = nullptr;
    int64_t *off = nullptr;
    TC_CHECK(dalloc_t(&xs, n, s));
    TC_CHECK(dalloc_t(&ys, n, s));
    TC_CHECK(dalloc_t(&cell, n, s));
    TC_CHECK(dalloc_t(&calt, n, s));
    TC_CHECK(dalloc_t(&idx, n, s));
    TC_CHECK(dalloc_t(&ialt, n, s));
    TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
    TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
    {
        const uint64_t threads = (n + kRggJ - 1) / kRggJ;
        k_rgg_points<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
            n, (unsigned long long)(s0 >> 64), (unsigned long long)s0, (unsigned long long)(inc >> 64),
            (unsigned long long)inc, grid, xs, ys, cell, idx);
        TC_LAUNCHED();
    }
    const RadixPlan cplan = make_radix_plan(bits_for(cells - 1 ? cells - 1 : 1));
    TC_CHECK(radix_histogram(cell, n, cplan, hist, s));
    TC_CHECK(radix_sort(cell, calt, idx, ialt, n, cplan, hist, kOutKeys, nullptr, nullptr, 0, &scell,
                        &sidx, s));
    TC_CHECK(dalloc_t(&sxy, n, s));
    TC_CHECK(dalloc_t(&cstart, cells + 1, s));
    k_rgg_gather<<<grid_for(n, 256, kSMs * 16), 256, 0, s>>>(sidx, n, xs, ys, sxy);
    TC_LAUNCHED();
    k_rgg_cell_start<<<grid_for(cells + 1, 256, kSMs * 16), 256, 0, s>>>(scell, n, cells, cstart);
    TC_LAUNCHED();
    dfree(xs, s);
    dfree(ys, s);
    TC_CHECK(dalloc_t(&deg, n, s));
    TC_CHECK(dalloc_t(&off, n, s));
    const int vb = bits_for(n > 1 ? n - 1 : 1);
    const unsigned wgrid = grid_for(n * 32, 256, kSMs * 16);
    k_rgg_scan<false><<<wgrid, 256, 0, s>>>(sxy, sidx, n, cstart, grid, r2, vb, deg, nullptr, nullptr);
    TC_LAUNCHED();
    TC_CHECK(exclusive_scan_dev(deg, n, off, s));
    int64_t last_off = 0;
    uint32_t last_deg = 0;
    unsigned long long *d_nv = nullptr;
    TC_CHECK(dalloc_t(&d_nv, 1, s));
    TC_CUDA(cudaMemsetAsync(d_nv, 0, sizeof(unsigned long long), s));
    k_last_nonzero<<<grid_for(n, 256, kSMs * 8), 256, 0, s>>>(deg, n, d_nv);
    TC_LAUNCHED();
    unsigned long long nv = 0;
    TC_CUDA(cudaMemcpyAsync(&last_off, off + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaMemcpyAsync(&last_deg, deg + n - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaMemcpyAsync(&nv, d_nv, sizeof(nv), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    const uint64_t np = (uint64_t)last_off + last_deg;
    uint32_t *pairs = nullptr;
    if (np) {
        uint64_t *keys = nullptr, *alt = nullptr;
        TC_CHECK(dalloc_t(&keys, np, s));
        TC_CHECK(dalloc_t(&alt, np, s));
        k_rgg_scan<true><<<wgrid, 256, 0, s>>>(sxy, sidx, n, cstart, grid, r2, vb, nullptr, off, keys);
        TC_LAUNCHED();
        const RadixPlan plan = make_radix_plan(2 * vb);
        TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
        TC_CHECK(radix_histogram(keys, np, plan, hist, s));
        TC_CHECK(dalloc_t(&pairs, 2 * np + 4, s, true));  // handed to the caller
        TC_CHECK(radix_sort(keys, alt, nullptr, nullptr, np, plan, hist, kOutAoS, pairs, nullptr, vb,
                            nullptr, nullptr, s));
        TC_CUDA(cudaStreamSynchronize(s));
        dfree(keys, s);
        dfree(alt, s);
    }
    dfree(cell, s);
    dfree(calt, s);
    dfree(idx, s);
    dfree(ialt, s);
    dfree(hist, s);
    dfree(sxy, s);
    dfree(cstart, s);
    dfree(deg, s);
    dfree(off, s);
    dfree(d_nv, s);
    TC_CUDA(cudaStreamSynchronize(s));
    *pairs_out = pairs;
    *npairs_out = np;
    *nverts_out = nv;
    return 0;
}

}  // namespace tc
