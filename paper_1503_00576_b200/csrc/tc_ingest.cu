// tc_ingest.cu -- device-side ingest around the hot path:
//   * TRI1 binary files read straight into pinned host memory (reference io.py:127-152);
//   * validate_edge_array on the device (reference graph.py:196-242): self-loops,
//     duplicate directed pairs, missing reverses -- reporting the same offending pair the
//     reference reports;
//   * wedge count sum_v C(deg v, 2) (reference metrics.py:17-24).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "tc_common.cuh"
#include "tc_internal.h"

namespace tc {

namespace {

// First input index with u == v, and first with an id >= n (atomicMin over indices).
__global__ void k_selfloop(const uint2 *__restrict__ pairs, uint64_t np, uint64_t n,
                           unsigned long long *__restrict__ first,
                           unsigned long long *__restrict__ first_range) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
        const uint2 p = pairs[i];
        if (p.x == p.y) atomicMin(first, (unsigned long long)i);
        if (p.x >= n || p.y >= n) atomicMin(first_range, (unsigned long long)i);
    }
}

__global__ void k_pack_idx(const uint2 *__restrict__ pairs, uint64_t np, int vb, int reverse,
                           uint64_t *__restrict__ keys, uint32_t *__restrict__ idx) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
        const uint2 p = pairs[i];
        keys[i] = reverse ? (((uint64_t)p.y << vb) | p.x) : (((uint64_t)p.x << vb) | p.y);
        if (idx) idx[i] = (uint32_t)i;
    }
}

// Sorted (key, input index) by a stable sort: every element equal to its predecessor is a
// second occurrence; report the smallest such input index (reference graph.py:227-234).
__global__ void k_dups(const uint64_t *__restrict__ sk, const uint32_t *__restrict__ sv, uint64_t np,
                       unsigned long long *__restrict__ first) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = 1 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride)
        if (sk[i] == sk[i - 1]) atomicMin(first, (unsigned long long)sv[i]);
}

// First input index whose reverse key is absent from the sorted keys (graph.py:236-240).
__global__ void k_missing_reverse(const uint2 *__restrict__ pairs, uint64_t np, int vb,
                                  const uint64_t *__restrict__ sk,
                                  unsigned long long *__restrict__ first) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
        const uint2 p = pairs[i];
        const uint64_t want = ((uint64_t)p.y << vb) | p.x;
        uint64_t a = 0, n = np;
        while (n > 0) {
            const uint64_t half = n >> 1;
            if (sk[a + half] < want) { a += half + 1; n -= half + 1; }
            else n = half;
        }
        if (a >= np || sk[a] != want) atomicMin(first, (unsigned long long)i);
    }
}

__global__ void __launch_bounds__(256) k_wedges(const uint32_t *__restrict__ deg, uint64_t n,
                                                unsigned long long *__restrict__ out,
                                                double *__restrict__ outd) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    unsigned long long acc = 0;
    double accd = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const unsigned long long d = deg[i];
        acc += d * (d - (d > 0)) / 2;
        accd += (double)d * (double)(d > 0 ? d - 1 : 0) * 0.5;
    }
    acc = warp_sum(acc);
    for (int o = 16; o > 0; o >>= 1) accd += __shfl_xor_sync(TC_FULL_MASK, accd, o);
    if (lane_id() == 0) {
        atomicAdd(out, acc);
        atomicAdd(outd, accd);
    }
}

__global__ void k_first_col_hist(const uint2 *__restrict__ pairs, uint64_t np, uint32_t *__restrict__ deg) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i - threadIdx.x < np; i += stride) {
        const bool ok = i < np;
        const uint32_t u = ok ? pairs[i].x : 0xffffffffu;
        const unsigned peers = __match_any_sync(TC_FULL_MASK, u);
        if (ok && (int)lane_id() == __ffs(peers) - 1) atomicAdd(deg + u, __popc(peers));
    }
}

}  // namespace

int validate_pairs_dev(const uint32_t *pairs_u32, uint64_t np, uint64_t n, int *code,
                       uint64_t *index, cudaStream_t s) {
    *code = 0;
    *index = 0;
    if (np == 0) return 0;
    if (np >= (1ull << 32)) {
        set_error("validate_edge_array: more than 2^32 pairs");
        return -1;
    }
    const uint2 *pairs = reinterpret_cast<const uint2 *>(pairs_u32);
    unsigned long long *first = nullptr;
    TC_CHECK(dalloc_t(&first, 4, s));
    TC_CUDA(cudaMemsetAsync(first, 0xff, 4 * sizeof(unsigned long long), s));
    k_selfloop<<<grid_for(np, 256, kSMs * 16), 256, 0, s>>>(pairs, np, n, first, first + 3);
    TC_LAUNCHED();
    {
        unsigned long long bad;
        TC_CUDA(cudaMemcpyAsync(&bad, first + 3, sizeof(bad), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
        if (bad != ~0ull) {
            dfree(first, s);
            *code = 4;
            *index = bad;
            return 0;
        }
    }
    const int vb = n > 1 ? bits_for(n - 1) : 1;
    const RadixPlan plan = make_radix_plan(2 * vb);
    uint64_t *keys = nullptr, *alt = nullptr, *sk = nullptr;
    uint32_t *idx = nullptr, *ialt = nullptr, *sv = nullptr, *hist = nullptr;
    TC_CHECK(dalloc_t(&keys, np, s));
    TC_CHECK(dalloc_t(&alt, np, s));
    TC_CHECK(dalloc_t(&idx, np, s));
    TC_CHECK(dalloc_t(&ialt, np, s));
    TC_CHECK(dalloc_t(&hist, kMaxPasses * kRadix, s));
    TC_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
    k_pack_idx<<<grid_for(np, 256, kSMs * 16), 256, 0, s>>>(pairs, np, vb, 0, keys, idx);
    TC_LAUNCHED();
    TC_CHECK(radix_histogram(keys, np, plan, hist, s));
    TC_CHECK(radix_sort(keys, alt, idx, ialt, np, plan, hist, kOutKeys, nullptr, nullptr, 0, &sk, &sv, s));
    k_dups<<<grid_for(np, 256, kSMs * 16), 256, 0, s>>>(sk, sv, np, first + 1);
    TC_LAUNCHED();
    k_missing_reverse<<<grid_for(np, 256, kSMs * 16), 256, 0, s>>>(pairs, np, vb, sk, first + 2);
    TC_LAUNCHED();
    unsigned long long h[3];
    TC_CUDA(cudaMemcpyAsync(h, first, sizeof(h), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(first, s);
    dfree(keys, s);
    dfree(alt, s);
    dfree(idx, s);
    dfree(ialt, s);
    dfree(hist, s);
    // the reference checks in this order: self-loop, duplicate, asymmetry
    for (int c = 0; c < 3; ++c)
        if (h[c] != ~0ull) {
            *code = c + 1;
            *index = h[c];
            return 0;
        }
    return 0;
}

int wedges_dev(const uint32_t *pairs_u32, uint64_t np, uint64_t n, uint64_t *out, double *outd,
               cudaStream_t s) {
    *out = 0;
    *outd = 0;
    if (n == 0) return 0;
    const uint2 *pairs = reinterpret_cast<const uint2 *>(pairs_u32);
    uint32_t *deg = nullptr;
    unsigned long long *acc = nullptr;
    TC_CHECK(dalloc_t(&deg, n, s));
    TC_CHECK(dalloc_t(&acc, 2, s));
    TC_CUDA(cudaMemsetAsync(deg, 0, n * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(acc, 0, 2 * sizeof(unsigned long long), s));
    if (np) {
        k_first_col_hist<<<grid_for(np, 256, kSMs * 16), 256, 0, s>>>(pairs, np, deg);
        TC_LAUNCHED();
    }
    k_wedges<<<grid_for(n, 256, kSMs * 8), 256, 0, s>>>(deg, n, acc, reinterpret_cast<double *>(acc + 1));
    TC_LAUNCHED();
    unsigned long long h[2];
    TC_CUDA(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(deg, s);
    dfree(acc, s);
    *out = h[0];
    memcpy(outd, &h[1], sizeof(double));
    return 0;
}

// TRI1: "TRI1" + u64 pair count + u32 pairs, little endian (reference io.py:18-33,127-152).
// Read with several threads into a pinned buffer so the later H2D runs at PCIe speed.
int read_tri1(const char *path, uint32_t **pinned, uint64_t *npairs) {
    *pinned = nullptr;
    *npairs = 0;
    FILE *f = fopen(path, "rb");
    if (!f) {
        set_error(std::string("cannot open ") + path);
        return -4;
    }
    unsigned char hdr[12];
    const size_t got = fread(hdr, 1, 12, f);
    fseek(f, 0, SEEK_END);
    const long long size = ftell(f);
    fclose(f);
    if (got < 12) {
        set_error("truncated: file shorter than the 12-byte header");
        return -5;
    }
    if (memcmp(hdr, "TRI1", 4) != 0) {
        set_error("bad magic: expected TRI1");
        return -6;
    }
    uint64_t count = 0;
    for (int i = 0; i < 8; ++i) count |= (uint64_t)hdr[4 + i] << (8 * i);
    if ((unsigned long long)size != 12 + 8 * count) {
        set_error("truncated: expected " + std::to_string(12 + 8 * count) + " bytes for " +
                  std::to_string(count) + " pairs, got " + std::to_string(size));
        return -5;
    }
    uint32_t *buf = nullptr;
    TC_CUDA(cudaHostAlloc(&buf, count ? 8 * count : 16, cudaHostAllocDefault));
    const int nthr = count > (1ull << 24) ? 8 : 1;
    std::vector<std::thread> th;
    std::vector<int> ok(nthr, 1);
    for (int t = 0; t < nthr; ++t) {
        th.emplace_back([&, t]() {
            const uint64_t lo = count * t / nthr, hi = count * (t + 1) / nthr;
            FILE *g = fopen(path, "rb");
            if (!g) { ok[t] = 0; return; }
            fseek(g, (long)(12 + 8 * lo), SEEK_SET);
            ok[t] = fread(buf + 2 * lo, 8, hi - lo, g) == hi - lo;
            fclose(g);
        });
    }
    for (auto &x : th) x.join();
    for (int t = 0; t < nthr; ++t)
        if (!ok[t]) {
            cudaFreeHost(buf);
            set_error(std::string("read error on ") + path);
            return -4;
        }
    *pinned = buf;
    *npairs = count;
    return 0;
}

// ---- text edge lists (reference io.py:51-99 read_edge_list) ------------------------------
// Lines split on \n, \r\n or \r (Python text mode); strip; skip empty lines and lines
// starting with '#' or '%'; exactly two fields, each a Python int() literal ([+-]digits with
// single '_' separators) in [0, 2^32).  Errors report the 1-based line and the first failing
// check, in the reference's order: field count, integer syntax, range.
namespace {

inline bool is_ws(unsigned char c) {
    return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}

// 0 ok, 2 syntax error, 3 out of range
int parse_int_token(const char *a, const char *b, uint32_t *out) {
    bool neg = false;
    if (a < b && (*a == '+' || *a == '-')) {
        neg = *a == '-';
        ++a;
    }
    if (a >= b) return 2;
    uint64_t v = 0;
    bool big = false, prev_digit = false;
    for (const char *p = a; p < b; ++p) {
        const char c = *p;
        if (c >= '0' && c <= '9') {
            if (!big) {
                v = v * 10 + (uint64_t)(c - '0');
                if (v > 0xffffffffull) big = true;
            }
            prev_digit = true;
        } else if (c == '_' && prev_digit && p + 1 < b && p[1] >= '0' && p[1] <= '9') {
            prev_digit = false;
        } else {
            return 2;
        }
    }
    if (big || (neg && v != 0)) return 3;
    *out = (uint32_t)v;
    return 0;
}

struct ChunkResult {
    std::vector<uint32_t> pairs;
    uint64_t lines = 0;
    uint64_t err_line = 0;  // 1-based within the chunk, 0 = none
    int err_kind = 0;
};

void parse_chunk(const char *a, const char *b, ChunkResult *r) {
    const char *p = a;
    uint64_t line = 0;
    while (p < b) {
        const char *e = p;
        while (e < b && *e != '\n' && *e != '\r') ++e;
        ++line;
        const char *s = p, *t = e;
        while (s < t && is_ws((unsigned char)*s)) ++s;
        while (t > s && is_ws((unsigned char)t[-1])) --t;
        if (s < t && *s != '#' && *s != '%') {
            const char *tok[3][2];
            int nt = 0;
            const char *q = s;
            while (q < t) {
                while (q < t && is_ws((unsigned char)*q)) ++q;
                if (q >= t) break;
                const char *q0 = q;
                while (q < t && !is_ws((unsigned char)*q)) ++q;
                if (nt < 3) { tok[nt][0] = q0; tok[nt][1] = q; }
                ++nt;
            }
            int kind = 0;
            uint32_t u = 0, v = 0;
            if (nt != 2) {
                kind = 1;
            } else {
                const int ku = parse_int_token(tok[0][0], tok[0][1], &u);
                const int kv = parse_int_token(tok[1][0], tok[1][1], &v);
                kind = (ku == 2 || kv == 2) ? 2 : (ku || kv) ? 3 : 0;
            }
            if (kind) {
                r->err_line = line;
                r->err_kind = kind;
                r->lines = line;
                return;
            }
            r->pairs.push_back(u);
            r->pairs.push_back(v);
        }
        if (e < b && *e == '\r' && e + 1 < b && e[1] == '\n') ++e;
        p = e + 1;
    }
    // a chunk ending in a line break opened no extra line
    r->lines = line;
}

}  // namespace

int parse_edge_list(const char *path, uint32_t **pinned, uint64_t *npairs, uint64_t *err_line,
                    int *err_kind) {
    *pinned = nullptr;
    *npairs = 0;
    *err_line = 0;
    *err_kind = 0;
    FILE *f = fopen(path, "rb");
    if (!f) {
        set_error(std::string("cannot open ") + path);
        return -4;
    }
    fseek(f, 0, SEEK_END);
    const long long size = ftell(f);
    fseek(f, 0, SEEK_SET);
    std::vector<char> data((size_t)size);
    if (size && fread(data.data(), 1, (size_t)size, f) != (size_t)size) {
        fclose(f);
        set_error(std::string("read error on ") + path);
        return -4;
    }
    fclose(f);
    const char *base = data.data(), *end = base + size;
    // chunk starts right after a '\n' (always a line start, even for \r\n files)
    int nthr = (int)std::min<long long>(32, std::max<long long>(1, size >> 22));
    nthr = std::max(1, std::min(nthr, (int)std::thread::hardware_concurrency()));
    std::vector<const char *> cut{base};
    for (int t = 1; t < nthr; ++t) {
        const char *c = base + size * t / nthr;
        if (c < cut.back()) c = cut.back();
        while (c < end && c[-1] != '\n') ++c;
        cut.push_back(c);
    }
    cut.push_back(end);
    std::vector<ChunkResult> res(nthr);
    std::vector<std::thread> th;
    for (int t = 0; t < nthr; ++t) th.emplace_back(parse_chunk, cut[t], cut[t + 1], &res[t]);
    for (auto &x : th) x.join();
    uint64_t lines_before = 0, total = 0;
    for (int t = 0; t < nthr; ++t) {
        if (res[t].err_kind) {
            *err_line = lines_before + res[t].err_line;
            *err_kind = res[t].err_kind;
            set_error("parse error at line " + std::to_string(*err_line));
            return -7;
        }
        // every chunk but the last ends right after a '\n', so its lines are self-contained
        lines_before += res[t].lines;
        total += res[t].pairs.size() / 2;
    }
    uint32_t *buf = nullptr;
    TC_CUDA(cudaHostAlloc(&buf, total ? 8 * total : 16, cudaHostAllocDefault));
    std::vector<std::thread> cp;
    uint64_t at = 0;
    for (int t = 0; t < nthr; ++t) {
        const uint64_t k = res[t].pairs.size();
        cp.emplace_back([=, &res]() { if (k) memcpy(buf + at, res[t].pairs.data(), k * 4); });
        at += k;
    }
    for (auto &x : cp) x.join();
    *pinned = buf;
    *npairs = total;
    return 0;
}

}  // namespace tc
