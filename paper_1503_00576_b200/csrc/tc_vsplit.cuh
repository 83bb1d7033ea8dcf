// tc_vsplit.cuh -- the per-edge v-major / u-major choice shared by the count kernels, the
// v-major index builds (k_vin_pass at count time, the fill fused into the rank-space
// segmented sorts) and the shard models.  Every user evaluates the same predicate, so
// each edge is counted exactly once.
#pragma once
#include "tc_common.cuh"
#include "tc_internal.h"

namespace tc {

// Edge e = (u, v) with v in the hub zone runs v-major (k_count_vmajor: re-reads the
// suffix of adj(u) after v, 4 B per item) when that is cheaper than the u-major read of
// v's data (dense bitmap words, or adj(v) as 16-byte chunks).  Every kernel evaluates the
// same predicate, so each edge is counted exactly once.  Edges with an empty suffix or
// an empty adj(v) close no triangle and are skipped by everyone.
#ifndef TC_VBIG
#define TC_VBIG 256  // 256 / 512 / 1K / 2K / 4K / 8K: s26 count 210 / 210 / 213 / 216 / 222 / 236 ms
#endif
constexpr uint32_t kVBigNonHub = TC_VBIG;  // v-major heads below hz with long lists: non-hub cap

#ifndef TC_VLCAP
#define TC_VLCAP 512
#endif
constexpr uint32_t kVNonHubCap = TC_VLCAP;  // v-major below hz: max |adj(v)| of the warp tasks
constexpr uint32_t kT16 = 1u << 16;          // k_count_vhub: the top 2^16 heads read 16-bit suffixes

__device__ __forceinline__ bool vmajor_edge(const VSplit &vp, uint32_t e, uint32_t eu, uint32_t v,
                                            uint32_t vs, uint32_t ve) {
    if (v < vp.z0) return false;
    if (e + 1 >= eu || vs >= ve) return true;  // no work either way
    uint32_t ucost;
    if (v >= vp.hz) {
        const uint32_t ws = ((v + 1 - vp.hz) >> 5) & ~3u;
        const bool dense = v >= vp.vt && (vp.hwp - ws) < vp.factor * (ve - vs);
        ucost = dense ? 4 * (vp.hwp - ws) : (vp.packed_cost ? 9 : 16) * ((ve - (vs & ~3u) + 3) >> 2);
        // the suffix is read from the packed hub copy: 9 bytes per 4 items
        if (vp.packed_cost) return (uint64_t)(9 * ((eu - e - 1 + 3) >> 2) + 8) * vp.bias < (uint64_t)ucost * 4;
        if (v >= vp.t16) return (uint64_t)(vp.b16w * (eu - e - 1) + 8) * vp.bias < (uint64_t)ucost * 4;
    } else {
        // below the hub zone: adj(v) goes into a per-warp cuckoo table (k_count_vlow_warp) when
        // |adj(v)| <= nhcap; longer lists run as CTA tasks (hub part as a bitmap, non-hub part
        // in a cuckoo table of at most kVBigNonHub keys)
        if (!vp.lowall && eu - e - 1 >= 32) return false;
        if (ve - vs > vp.nhcap && __ldg(vp.hubstart + v) - vs > kVBigNonHub) return false;
        ucost = 16 * ((ve - (vs & ~3u) + 3) >> 2) + 16;
    }
    return (uint64_t)(4 * (eu - e - 1) + 8) * vp.bias < (uint64_t)ucost * 4;
}

// The v-major split of one count (tc_count.cu).
VSplit make_vsplit(const DeviceGraph &g, bool vmajor);
bool vsplit_same(const VSplit &a, const VSplit &b);
// Whether full counts of g run the v-major schedule (large skewed rank-space graphs).
bool vmajor_schedule(const DeviceGraph &g);

// v-major in-edge index fill hook: the rank-space segmented sorts place element v at its
// final position e of adj(u) (eu = end of adj(u)) and append (e, eu) to v's in-edge list
// when the edge runs v-major -- the same test and capacity layout as k_vin_pass<true>.
struct VFill {
    VSplit vp;  // vp.z0 = ~0: off
    const uint32_t *off32 = nullptr, *start = nullptr;
    uint32_t *cnt = nullptr, *flag = nullptr;
    uint2 *in_e = nullptr;
};

__device__ __forceinline__ void vfill(const VFill &f, uint32_t e, uint32_t eu, uint32_t v) {
    if (v < f.vp.z0 || e + 1 >= eu) return;
    const uint32_t vs = __ldg(f.off32 + v), ve = __ldg(f.off32 + v + 1);
    if (vs >= ve || !vmajor_edge(f.vp, e, eu, v, vs, ve)) return;
    const uint32_t h = v - f.vp.z0;
    const uint32_t k = atomicAdd(f.cnt + h, 1u);
    const uint32_t b = __ldg(f.start + h);
    if (k >= __ldg(f.start + h + 1) - b) *f.flag = 1u;  // not symmetric: capacity exceeded
#if !defined(TC_VIN_PROBE) || TC_VIN_PROBE != 1  // diagnostic build 1: atomics only
    else f.in_e[b + k] = make_uint2(e, eu);
#endif
}

// vfill over N elements of one list at once: all offset loads first, then all predicates,
// then all cursor atomics, then all stores -- the per-element chains overlap instead of
// running back to back (the sorts are latency-bound).  ok[i]: element i exists.
template <int N>
__device__ __forceinline__ void vfill_batch(const VFill &f, const uint32_t (&e)[N], uint32_t eu,
                                            const uint32_t (&v)[N], const bool (&ok)[N]) {
    if (f.vp.z0 == 0xffffffffu) return;
    uint32_t vs[N], ve[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const bool c = ok[i] && v[i] >= f.vp.z0 && e[i] + 1 < eu;
        vs[i] = c ? __ldg(f.off32 + v[i]) : 1u;
        ve[i] = c ? __ldg(f.off32 + v[i] + 1) : 0u;
    }
    bool take[N];
#pragma unroll
    for (int i = 0; i < N; ++i) take[i] = vs[i] < ve[i] && vmajor_edge(f.vp, e[i], eu, v[i], vs[i], ve[i]);
    uint32_t k[N];
#pragma unroll
    for (int i = 0; i < N; ++i) k[i] = take[i] ? atomicAdd(f.cnt + (v[i] - f.vp.z0), 1u) : 0u;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if (!take[i]) continue;
        const uint32_t h = v[i] - f.vp.z0;
        const uint32_t b = __ldg(f.start + h);
        if (k[i] >= __ldg(f.start + h + 1) - b) *f.flag = 1u;  // not symmetric: capacity exceeded
        else f.in_e[b + k[i]] = make_uint2(e[i], eu);
    }
}

}  // namespace tc
