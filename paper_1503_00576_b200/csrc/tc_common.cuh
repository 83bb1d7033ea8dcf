// tc_common.cuh -- shared device helpers for the sm_100a triangle-counting library.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define TC_FULL_MASK 0xffffffffu

namespace tc {

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs (grids are sized in multiples of this)

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ unsigned lanemask_le() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(r));
    return r;
}

// Inclusive warp scan (Kogge-Stone over shuffles).
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T x) {
    const unsigned lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(TC_FULL_MASK, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    return x;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(TC_FULL_MASK, x, o);
    return x;
}

// Block-wide exclusive scan of one value per thread; returns the block total in *total.
// `smem_warp` needs blockDim.x/32 entries.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T x, T *smem_warp, T *total) {
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T incl = warp_inclusive_scan(x);
    if (lane == 31) smem_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nw ? smem_warp[lane] : T(0);
        T wi = warp_inclusive_scan(w);
        if (lane < nw) smem_warp[lane] = wi - w;
        if (lane == nw - 1) smem_warp[31] = wi;  // nw <= 31 required (blockDim <= 992)
    }
    __syncthreads();
    T res = smem_warp[warp] + incl - x;
    *total = smem_warp[31];
    __syncthreads();
    return res;
}

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_volatile_u64(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Streaming (evict-first) 64-bit load for data read exactly once.
__device__ __forceinline__ uint2 ld_stream_u2(const uint2 *p) { return __ldcs(p); }

inline unsigned grid_for(uint64_t work_items, unsigned per_block, unsigned max_blocks) {
    uint64_t g = (work_items + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (unsigned)g;
}

}  // namespace tc
