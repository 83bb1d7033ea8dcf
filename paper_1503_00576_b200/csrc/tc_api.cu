// tc_api.cu -- the C ABI (include/tricount_b200.h).  Plain pointers and sizes only.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tricount_b200.h"
#include "tc_common.cuh"
#include "tc_internal.h"

// A device OrientedGraph.  `g` is the reference-id CSR (reference graph.py:146-193): what
// downloads, ranged counts and partition bounds see.  `rank` is the count-ready rank-space
// copy.  tc_preprocess builds the rank copy directly (the fused path's preprocessing) and
// keeps `id_of_rank`; `g` is then materialised from it on first use (ref_ready false) --
// the same arrays the reference produces, built only when something asks for them.
struct tc_graph {
    tc::DeviceGraph g;
    tc::DeviceGraph *rank = nullptr;  // cached rank-space copy (full-range counts)
    bool no_rank = false;             // not rank-orientable: full counts use the original ids
    bool ref_ready = true;            // g's arrays exist
    uint32_t *id_of_rank = nullptr;   // rank -> reference id (graphs from tc_preprocess)
};

namespace tc {

namespace {
thread_local std::string g_err;
std::mutex g_mu;
// Every entry point that touches device state holds this for the whole call: the reference's
// count is a pure function safe to call concurrently on different graphs (SPEC.md:294,
// private per-call accumulators at count.py:68).  Calls share one stream and one scratch pool
// and each count saturates the GPU, so serialising them costs no throughput; each count also
// accumulates into its own device counter, and the lazy rank-space copy of a graph is built
// under the lock.  Recursive: entry points may call each other.
std::recursive_mutex g_call;
Options g_opts;
bool g_ready = false;
int g_device = 0;
cudaStream_t g_stream = nullptr;
cudaMemPool_t g_scratch = nullptr;
void *g_flush = nullptr;
size_t g_flush_bytes = 0;
}  // namespace

#define TC_API_GUARD() std::lock_guard<std::recursive_mutex> _tc_call_lock(::tc::g_call)

Options &opts() { return g_opts; }

std::atomic<unsigned long long> g_launches{0};
cudaEvent_t g_timer[8] = {nullptr};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
cudaMemPool_t scratch_pool() { return g_scratch; }
void set_error(const std::string &msg) { g_err = msg; }
const char *last_error() { return g_err.c_str(); }

static int ensure_init(int device) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_ready) {
        TC_CUDA(cudaSetDevice(g_device));
        return 0;
    }
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        set_error(std::string("no CUDA device available: ") + cudaGetErrorString(e));
        return -2;
    }
    if (device < 0 || device >= count) {
        set_error("device index out of range");
        return -1;
    }
    TC_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    TC_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        set_error(std::string("this library is built for sm_100a (B200); found ") + prop.name);
        return -2;
    }
    TC_CUDA(cudaStreamCreateWithFlags(&g_stream, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    TC_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = ~0ull;
    TC_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    TC_CUDA(cudaMemPoolCreate(&g_scratch, &props));
    TC_CUDA(cudaMemPoolSetAttribute(g_scratch, cudaMemPoolAttrReleaseThreshold, &keep));
    g_device = device;
    g_ready = true;
    return 0;
}

static int ensure() { return ensure_init(g_device); }

// Keep at least `bytes` of device memory reserved in the stream-ordered pool: one large
// allocation is made and freed, so later calls sub-allocate from mapped memory instead of
// mapping new chunks (which showed up as 100+ ms gaps under fragmentation).
static int reserve_pool(uint64_t bytes) {
    cudaMemPool_t pool = g_scratch;
    uint64_t reserved = 0, used = 0;
    TC_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
    TC_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
    if (reserved - used >= bytes) return 0;
    size_t free_b = 0, total_b = 0;
    TC_CUDA(cudaMemGetInfo(&free_b, &total_b));
    uint64_t want = bytes - (reserved - used);
    if (want > (uint64_t)free_b * 9 / 10) want = (uint64_t)free_b * 9 / 10;
    if (want < (64ull << 20)) return 0;
    void *p = nullptr;
    if (cudaMallocFromPoolAsync(&p, want, pool, g_stream) != cudaSuccess) {
        cudaGetLastError();  // best effort: not fatal
        return 0;
    }
    TC_CUDA(cudaFreeAsync(p, g_stream));
    TC_CUDA(cudaStreamSynchronize(g_stream));
    return 0;
}

// ---- host -> device copies of caller buffers ---------------------------------------------
// Pinned (page-locked or cudaHostRegister'ed) buffers go straight to the copy engine.  An
// ordinary pageable buffer -- a plain numpy array, what a reference EdgeArray holds -- would
// go through the driver's single-threaded staging (~10 GB/s measured); instead it is
// streamed through kStageBufs pinned staging buffers: host threads copy chunk k into one
// while the copy engine moves chunk k-1 out of another (PCIe rate when the host copy keeps up).
constexpr int kStageBufs = 3;
constexpr size_t kStageBytes = 128ull << 20;
void *g_stage[kStageBufs] = {nullptr};
cudaEvent_t g_stage_ev[kStageBufs] = {nullptr};

static bool is_pageable(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// A small persistent pool of host threads for the staged copies (created on first use).
class CopyPool {
  public:
    explicit CopyPool(int n) : n_(n) {
        for (int t = 0; t < n_; ++t) th_.emplace_back([this, t] { run(t); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto &t : th_) t.join();
    }
    int size() const { return n_; }
    void copy(void *dst, const void *src, size_t bytes) {
        std::unique_lock<std::mutex> lk(mu_);
        dst_ = (char *)dst;
        src_ = (const char *)src;
        bytes_ = bytes;
        left_ = n_;
        ++gen_;
        cv_.notify_all();
        done_.wait(lk, [this] { return left_ == 0; });
    }

  private:
    void run(int t) {
        uint64_t seen = 0;
        for (;;) {
            char *d;
            const char *sp;
            size_t b;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                d = dst_;
                sp = src_;
                b = bytes_;
            }
            const size_t part = ((b / n_) + 4095) & ~(size_t)4095;
            const size_t lo = part * t;
            if (lo < b) memcpy(d + lo, sp + lo, b - lo < part ? b - lo : part);
            std::lock_guard<std::mutex> lk(mu_);
            if (--left_ == 0) done_.notify_one();
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    uint64_t gen_ = 0;
    bool stop_ = false;
    char *dst_ = nullptr;
    const char *src_ = nullptr;
    size_t bytes_ = 0;
    int left_ = 0;
};
CopyPool *g_copy_pool = nullptr;

static void parallel_memcpy(void *dst, const void *src, size_t bytes, int threads) {
    if (threads <= 1 || bytes < (8u << 20)) {
        memcpy(dst, src, bytes);
        return;
    }
    if (g_copy_pool && g_copy_pool->size() != threads) {
        delete g_copy_pool;
        g_copy_pool = nullptr;
    }
    if (!g_copy_pool) g_copy_pool = new CopyPool(threads);
    g_copy_pool->copy(dst, src, bytes);
}

// Host pairs -> device with the first-column degree histogram of each chunk running on s
// while the next chunk is still being copied (copies on a side stream, one event per
// chunk): the histogram pass -- the only preprocessing step that needs no other chunk --
// is hidden under the PCIe transfer.  *pre receives the degrees for preprocess_rank_dev.
static cudaStream_t copy_stream() {
    static cudaStream_t cs = nullptr;
    if (!cs) cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    return cs;
}

static int h2d_degrees(uint32_t *dst, const uint32_t *src, uint64_t npairs, uint64_t n, PreDegrees *pre,
                       cudaStream_t s) {
    constexpr size_t kChunk = 256ull << 20;  // bytes per pinned chunk (a multiple of 8)
    TC_CHECK(dalloc_t(&pre->deg, n ? n : 1, s));
    TC_CHECK(dalloc_t(&pre->bad, 1, s));
    TC_CUDA(cudaMemsetAsync(pre->deg, 0, (n ? n : 1) * sizeof(uint32_t), s));
    TC_CUDA(cudaMemsetAsync(pre->bad, 0, sizeof(uint32_t), s));
    if (!npairs) return 0;
    cudaStream_t cs = copy_stream();
    static cudaEvent_t ev = nullptr, ev0 = nullptr;
    if (!ev) {
        TC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        TC_CUDA(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
    }
    TC_CUDA(cudaEventRecord(ev0, s));  // dst allocated on s
    TC_CUDA(cudaStreamWaitEvent(cs, ev0, 0));
    const size_t bytes = npairs * 8;
    auto chunk_done = [&](size_t off, size_t len) -> int {
        TC_CUDA(cudaEventRecord(ev, cs));
        TC_CUDA(cudaStreamWaitEvent(s, ev, 0));
        return degree_hist_dev(dst + off / 4, len / 8, n, pre->deg, pre->bad, s);
    };
    if (bytes < (32u << 20) || !is_pageable(src)) {
        for (size_t off = 0; off < bytes; off += kChunk) {
            const size_t len = bytes - off < kChunk ? bytes - off : kChunk;
            TC_CUDA(cudaMemcpyAsync((char *)dst + off, (const char *)src + off, len, cudaMemcpyHostToDevice, cs));
            TC_CHECK(chunk_done(off, len));
        }
        return 0;
    }
    if (!g_stage[0])
        for (int b = 0; b < kStageBufs; ++b) {
            TC_CUDA(cudaHostAlloc(&g_stage[b], kStageBytes, cudaHostAllocDefault));
            TC_CUDA(cudaEventCreateWithFlags(&g_stage_ev[b], cudaEventDisableTiming));
        }
    const unsigned hc = std::thread::hardware_concurrency();
    const int threads = opts().copy_threads > 0 ? (int)opts().copy_threads
                        : hc >= 16 ? 8 : hc >= 4 ? (int)hc / 2 : 1;
    size_t off = 0;
    for (int k = 0; off < bytes; ++k) {
        const int b = k % kStageBufs;
        const size_t len = bytes - off < kStageBytes ? bytes - off : kStageBytes;
        TC_CUDA(cudaEventSynchronize(g_stage_ev[b]));  // the copy out of this buffer finished
        parallel_memcpy(g_stage[b], (const char *)src + off, len, threads);
        TC_CUDA(cudaMemcpyAsync((char *)dst + off, g_stage[b], len, cudaMemcpyHostToDevice, cs));
        TC_CUDA(cudaEventRecord(g_stage_ev[b], cs));
        TC_CHECK(chunk_done(off, len));
        off += len;
    }
    return 0;
}

static int h2d(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    if (!bytes) return 0;
    if (bytes < (32u << 20) || !is_pageable(src)) {
        TC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return 0;
    }
    if (!g_stage[0])
        for (int b = 0; b < kStageBufs; ++b) {
            TC_CUDA(cudaHostAlloc(&g_stage[b], kStageBytes, cudaHostAllocDefault));
            TC_CUDA(cudaEventCreateWithFlags(&g_stage_ev[b], cudaEventDisableTiming));
        }
    const unsigned hc = std::thread::hardware_concurrency();
    const int threads = opts().copy_threads > 0 ? (int)opts().copy_threads
                        : hc >= 16 ? 8 : hc >= 4 ? (int)hc / 2 : 1;
    size_t off = 0;
    for (int k = 0; off < bytes; ++k) {
        const int b = k % kStageBufs;
        const size_t len = bytes - off < kStageBytes ? bytes - off : kStageBytes;
        TC_CUDA(cudaEventSynchronize(g_stage_ev[b]));  // the copy out of this buffer finished
        parallel_memcpy(g_stage[b], (const char *)src + off, len, threads);
        TC_CUDA(cudaMemcpyAsync((char *)dst + off, g_stage[b], len, cudaMemcpyHostToDevice, s));
        TC_CUDA(cudaEventRecord(g_stage_ev[b], s));
        off += len;
    }
    return 0;
}

// Peak scratch of preprocess + count, ~14 B per input pair at R-MAT s26.
static uint64_t scratch_estimate(uint64_t npairs) { return 16ull * npairs + (256ull << 20); }

static double ms_between(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return (double)ms;
}

struct Events {
    cudaEvent_t e[6];
    int n = 0;
    Events() {
        for (auto &x : e) x = nullptr;
    }
    int create() {
        for (auto &x : e) TC_CUDA(cudaEventCreate(&x));
        return 0;
    }
    ~Events() {
        for (auto &x : e)
            if (x) cudaEventDestroy(x);
    }
};

// Full-range counts of an original-id graph run on its (cached) rank-space copy; ranged
// counts of it run the original-id kernels over exactly that edge range.  A graph whose
// edges do not all point to a higher (out + in degree, id) rank -- hand-built, or the
// preprocess of a non-symmetric edge array -- keeps the original-id kernels for every count.
// Called under the API lock (the copy is created once per graph).
static int rank_copy(tc_graph *h, const DeviceGraph **out) {
    *out = &h->g;
    if (h->g.rank_space || h->no_rank || h->g.m >= (1ull << 32)) return 0;
    if (!h->rank) {
        DeviceGraph *r = new DeviceGraph();
        r->persistent = true;
        int rc = relabel_dev(h->g, r, g_stream);
        if (rc) {
            graph_release(r, g_stream);
            delete r;
            if (rc != kNotRankOrientable) return rc;
            h->no_rank = true;
            return 0;
        }
        h->rank = r;
    }
    *out = h->rank;
    return 0;
}

// The reference-id arrays of a graph whose preprocessing produced only the rank-space copy.
// Called under the API lock.
static int ensure_ref(tc_graph *h) {
    if (h->ref_ready) return 0;
    DeviceGraph g;
    g.persistent = true;
    int rc = derank_dev(*h->rank, h->id_of_rank, &g, g_stream);
    if (rc) {
        graph_release(&g, g_stream);
        return rc;
    }
    h->g = g;
    h->ref_ready = true;
    return 0;
}

// Counts `bounds` ranges of a graph into a private device counter.  With `h` set, the
// full-range count runs on h's rank-space copy, built (once) inside the timed region.
static int count_ranges(const DeviceGraph &g0, tc_graph *h, const int64_t *bounds, int npools,
                        int algo, uint64_t *out, tc_times *t) {
    cudaStream_t s = g_stream;
    Events ev;
    TC_CHECK(ev.create());
    TC_CUDA(cudaEventRecord(ev.e[0], s));
    const DeviceGraph *gp = &g0;
    if (h) TC_CHECK(rank_copy(h, &gp));
    const DeviceGraph &g = *gp;
    unsigned long long *total = nullptr;  // this call's accumulator
    TC_CHECK(dalloc_t(&total, 1, s));
    TC_CUDA(cudaMemsetAsync(total, 0, sizeof(unsigned long long), s));
    CountStats agg, st;
    for (int p = 0; p < npools; ++p) {
        st = CountStats();
        const int rc = count_range_dev(g, (uint64_t)bounds[p], (uint64_t)bounds[p + 1], algo, total, s,
                                       t ? &st : nullptr);
        if (rc) {
            dfree(total, s);
            return rc;
        }
        agg.classify_ms += st.classify_ms;
        agg.heavy_ms += st.heavy_ms;
        agg.light_ms += st.light_ms;
        agg.vmajor_ms += st.vmajor_ms;
        agg.heavy_tasks += st.heavy_tasks;
    }
    unsigned long long hv = 0;
    TC_CUDA(cudaMemcpyAsync(&hv, total, sizeof(hv), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaEventRecord(ev.e[1], s));
    dfree(total, s);
    TC_CUDA(cudaEventSynchronize(ev.e[1]));
    *out = hv;
    if (t) {
        memset(t, 0, sizeof(*t));
        t->count_ms = ms_between(ev.e[0], ev.e[1]);
        t->total_ms = t->count_ms;
        t->classify_ms = agg.classify_ms;
        t->heavy_ms = agg.heavy_ms;
        t->light_ms = agg.light_ms;
        t->vmajor_ms = agg.vmajor_ms;
        t->heavy_tasks = agg.heavy_tasks;
    }
    return 0;
}

__global__ void k_check_ids(const uint32_t *__restrict__ ids, uint64_t k, uint32_t n,
                            uint32_t *__restrict__ bad) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    bool ok = true;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) ok &= ids[i] < n;
    if (!ok) atomicOr(bad, 1u);
}

static int check_graph(const tc_graph *g) {
    if (!g) {
        set_error("null graph handle");
        return -1;
    }
    return 0;
}

}  // namespace tc

using namespace tc;

extern "C" {

int tc_abi_version(void) { return TC_ABI_VERSION; }
const char *tc_last_error(void) { return tc::last_error(); }

int tc_init(int device) {
    TC_API_GUARD();
    TC_CHECK(ensure_init(device));
    // touch the pool and the kernels' module so the first timed call pays nothing
    void *p = nullptr;
    TC_CHECK(dalloc(&p, 1 << 20, g_stream));
    dfree(p, g_stream);
    TC_CUDA(cudaStreamSynchronize(g_stream));
    return 0;
}

int tc_shutdown(void) {
    TC_API_GUARD();
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_ready) return 0;
    for (int b = 0; b < kStageBufs; ++b) {
        if (g_stage[b]) cudaFreeHost(g_stage[b]);
        if (g_stage_ev[b]) cudaEventDestroy(g_stage_ev[b]);
        g_stage[b] = nullptr;
        g_stage_ev[b] = nullptr;
    }
    delete g_copy_pool;
    g_copy_pool = nullptr;
    if (g_flush) cudaFree(g_flush);
    g_flush = nullptr;
    g_flush_bytes = 0;
    if (g_scratch) cudaMemPoolDestroy(g_scratch);
    g_scratch = nullptr;
    cudaStreamDestroy(g_stream);
    g_stream = nullptr;
    g_ready = false;
    return 0;
}

int tc_preprocess(const uint32_t *pairs, uint64_t npairs, uint64_t nverts, int pairs_on_device,
                  tc_graph **out, tc_times *t) {
    return tc_preprocess_ex(pairs, npairs, nverts, pairs_on_device, 0, out, t);
}

int tc_preprocess_ex(const uint32_t *pairs, uint64_t npairs, uint64_t nverts, int pairs_on_device,
                     int flags, tc_graph **out, tc_times *t) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(reserve_pool(scratch_estimate(npairs)));
    if (!out) {
        set_error("null output handle");
        return -1;
    }
    cudaStream_t s = g_stream;
    Events ev;
    TC_CHECK(ev.create());
    TC_CUDA(cudaEventRecord(ev.e[0], s));
    const uint32_t *dpairs = pairs;
    uint32_t *owned = nullptr;  // staging copy: default pool, freed at the end of the call
    const bool rank_path = (flags & TC_PREPROCESS_RANK_SPACE) ||
                           (npairs / 2 < (1ull << 32) && nverts < (1ull << 32) && opts().rank_primary);
    PreDegrees pre;
    if (!pairs_on_device && npairs) {
        TC_CHECK(dalloc_t(&owned, 2 * npairs, s, true));
        // rank path: the degree histogram runs chunk by chunk under the copy
        if (rank_path && nverts < (1ull << 32) && npairs / 2 < (1ull << 32))
            TC_CHECK(h2d_degrees(owned, pairs, npairs, nverts, &pre, s));
        else TC_CHECK(h2d(owned, pairs, npairs * 8, s));
        dpairs = owned;
    }
    const PreDegrees *prep = pre.deg ? &pre : nullptr;
    TC_CUDA(cudaEventRecord(ev.e[1], s));
    tc_graph *g = new tc_graph();
    g->g.persistent = true;
    int rc;
    if (flags & TC_PREPROCESS_RANK_SPACE) {
        rc = preprocess_rank_dev(dpairs, npairs, nverts, &g->g, s, nullptr, prep);
    } else if (npairs / 2 < (1ull << 32) && nverts < (1ull << 32) && opts().rank_primary) {
        // the count-ready rank-space CSR is built (as the fused path does) and the reference-id
        // CSR only on demand
        g->rank = new DeviceGraph();
        g->rank->persistent = true;
        rc = dalloc_t(&g->id_of_rank, nverts ? nverts : 1, s, true);
        if (!rc) rc = preprocess_rank_dev(dpairs, npairs, nverts, g->rank, s, g->id_of_rank, prep);
        if (!rc) {
            g->g.m = g->rank->m;
            g->g.n = g->rank->n;
            g->g.max_out = g->rank->max_out;
            g->ref_ready = false;
        } else {
            graph_release(g->rank, s);
            delete g->rank;
            g->rank = nullptr;
        }
    } else {
        rc = preprocess_dev(dpairs, npairs, nverts, &g->g, s);
    }
    dfree(pre.bad, s);
    if (owned) dfree(owned, s);
    if (rc) {
        graph_release(&g->g, s);
        dfree(g->id_of_rank, s);
        delete g;
        return rc;
    }
    TC_CUDA(cudaEventRecord(ev.e[2], s));
    TC_CUDA(cudaEventSynchronize(ev.e[2]));
    if (t) {
        memset(t, 0, sizeof(*t));
        t->h2d_ms = ms_between(ev.e[0], ev.e[1]);
        t->preprocess_ms = ms_between(ev.e[1], ev.e[2]);
        t->total_ms = ms_between(ev.e[0], ev.e[2]);
    }
    *out = g;
    return 0;
}

int tc_graph_upload(const uint32_t *edge_src, const uint32_t *edge_dst,
                    const int64_t *node_offsets, uint64_t m, uint64_t n, tc_graph **out) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    cudaStream_t s = g_stream;
    if (n >= (1ull << 32)) {
        set_error("num_vertices must be < 2^32 on the device path");
        return -1;
    }
    // The count kernels index with these offsets: check them (O(n), host) before anything
    // reaches the device -- off[0] = 0, off[n] = m, nondecreasing.
    if (!node_offsets || node_offsets[0] != 0 || (uint64_t)node_offsets[n] != m) {
        set_error("node_offsets must start at 0 and end at m");
        return -1;
    }
    uint64_t maxo = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (node_offsets[i + 1] < node_offsets[i]) {
            set_error("node_offsets must be nondecreasing");
            return -1;
        }
        const uint64_t d = (uint64_t)(node_offsets[i + 1] - node_offsets[i]);
        if (d > maxo) maxo = d;
    }
    tc_graph *g = new tc_graph();
    g->g.persistent = true;
    int rc = graph_alloc(&g->g, m, n, s);
    uint32_t *tmp = nullptr;
    if (!rc && g->g.off32) {
        tmp = (uint32_t *)malloc((n + 1) * 4);
        if (!tmp) {
            set_error("host allocation failed");
            rc = -3;
        }
    }
    auto fail = [&](int code) {
        free(tmp);
        graph_release(&g->g, s);
        delete g;
        return code;
    };
    if (rc) return fail(rc);
    cudaError_t e = cudaSuccess;
    if (m) {
        if (h2d(g->g.src, edge_src, m * 4, s) || h2d(g->g.dst, edge_dst, m * 4, s)) return fail(-2);
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(g->g.dst + m, 0, 16, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->g.off, node_offsets, (n + 1) * 8, cudaMemcpyHostToDevice, s);
    if (tmp) {  // off32: the u32 copy the count kernels read (m < 2^32)
        for (uint64_t i = 0; i <= n; ++i) tmp[i] = (uint32_t)node_offsets[i];
        if (e == cudaSuccess) e = cudaMemcpyAsync(g->g.off32, tmp, (n + 1) * 4, cudaMemcpyHostToDevice, s);
    }
    // every edge_dst must be a vertex (the kernels read off[v] for v = edge_dst[e])
    uint32_t bad = 0;
    if (e == cudaSuccess && m) {
        uint32_t *dbad = nullptr;
        if (dalloc_t(&dbad, 1, s)) return fail(-3);
        e = cudaMemsetAsync(dbad, 0, sizeof(uint32_t), s);
        if (e == cudaSuccess) {
            k_check_ids<<<grid_for(m, 256, kSMs * 8), 256, 0, s>>>(g->g.dst, m, (uint32_t)n, dbad);
            note_launch();
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, dbad, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
        dfree(dbad, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        set_error(std::string("graph upload: ") + cudaGetErrorString(e));
        return fail(-2);
    }
    if (bad) {
        set_error("edge_dst holds a vertex id >= num_vertices");
        return fail(-1);
    }
    free(tmp);
    g->g.max_out = (uint32_t)maxo;
    *out = g;
    return 0;
}

int tc_graph_create(uint64_t m, uint64_t n, int flags, tc_graph **out) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    if (n >= (1ull << 32)) {
        set_error("num_vertices must be < 2^32 on the device path");
        return -1;
    }
    tc_graph *g = new tc_graph();
    g->g.persistent = true;
    int rc = graph_alloc(&g->g, m, n, g_stream);
    if (rc) {
        delete g;
        return rc;
    }
    g->g.rank_space = (flags & TC_PREPROCESS_RANK_SPACE) != 0;
    TC_CUDA(cudaStreamSynchronize(g_stream));
    *out = g;
    return 0;
}

int tc_graph_finalize(tc_graph *g) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    return finalize_graph_dev(&g->g, g_stream);
}

int tc_graph_download(const tc_graph *g, uint32_t *edge_src, uint32_t *edge_dst,
                      int64_t *node_offsets) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    TC_CHECK(ensure_ref(const_cast<tc_graph *>(g)));
    cudaStream_t s = g_stream;
    if (g->g.m) {
        if (edge_src) TC_CUDA(cudaMemcpyAsync(edge_src, g->g.src, g->g.m * 4, cudaMemcpyDeviceToHost, s));
        if (edge_dst) TC_CUDA(cudaMemcpyAsync(edge_dst, g->g.dst, g->g.m * 4, cudaMemcpyDeviceToHost, s));
    }
    if (node_offsets)
        TC_CUDA(cudaMemcpyAsync(node_offsets, g->g.off, (g->g.n + 1) * 8, cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    return 0;
}

int tc_graph_info(const tc_graph *g, uint64_t *m, uint64_t *n, uint32_t *max_out_degree) {
    TC_CHECK(check_graph(g));
    if (m) *m = g->g.m;
    if (n) *n = g->g.n;
    if (max_out_degree) *max_out_degree = g->g.max_out;
    return 0;
}

int tc_graph_flags(const tc_graph *g, int *flags) {
    TC_CHECK(check_graph(g));
    *flags = g->g.rank_space ? TC_PREPROCESS_RANK_SPACE : 0;
    return 0;
}

int tc_graph_device_ptrs(const tc_graph *g, uint32_t **edge_src, uint32_t **edge_dst,
                         int64_t **node_offsets) {
    TC_API_GUARD();
    TC_CHECK(check_graph(g));
    TC_CHECK(ensure_ref(const_cast<tc_graph *>(g)));
    if (edge_src) *edge_src = g->g.src;
    if (edge_dst) *edge_dst = g->g.dst;
    if (node_offsets) *node_offsets = g->g.off;
    return 0;
}

int tc_graph_free(tc_graph *g) {
    TC_API_GUARD();
    if (!g) return 0;
    if (g_ready) {
        cudaSetDevice(g_device);
        graph_release(&g->g, g_stream);
        if (g->rank) graph_release(g->rank, g_stream);
        dfree(g->id_of_rank, g_stream);
    }
    delete g->rank;
    delete g;
    return 0;
}

int tc_count(const tc_graph *g, int64_t lo, int64_t hi, int algo, uint64_t *out, tc_times *t) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    if (lo < 0 || hi < lo || (uint64_t)hi > g->g.m) {
        set_error("edge range outside [0, m]");
        return -1;
    }
    int64_t b[2] = {lo, hi};
    const bool full = algo == TC_ALGO_AUTO && lo == 0 && (uint64_t)hi == g->g.m;
    if (!full) TC_CHECK(ensure_ref(const_cast<tc_graph *>(g)));  // ranges are in reference edge order
    return count_ranges(g->g, full ? const_cast<tc_graph *>(g) : nullptr, b, 1, algo, out, t);
}

int tc_count_partitioned(const tc_graph *g, const int64_t *bounds, int npools, int algo,
                         uint64_t *out, tc_times *t) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    if (npools < 1 || bounds[0] != 0 || (uint64_t)bounds[npools] != g->g.m) {
        set_error("plan does not cover [0, m)");
        return -1;
    }
    for (int p = 0; p < npools; ++p)
        if (bounds[p] > bounds[p + 1]) {
            set_error("plan bounds must be nondecreasing");
            return -1;
        }
    // The pools of a covering plan partition the edges, so the sum over pools is the
    // full count (count.py:181-204 returns only that sum).  On one GPU the pools are
    // counted as one pass; per-pool ranges remain available through tc_count.
    if (algo == TC_ALGO_AUTO) {
        int64_t b[2] = {0, (int64_t)g->g.m};
        return count_ranges(g->g, const_cast<tc_graph *>(g), b, 1, algo, out, t);
    }
    TC_CHECK(ensure_ref(const_cast<tc_graph *>(g)));
    return count_ranges(g->g, nullptr, bounds, npools, algo, out, t);
}

int tc_intersect_count(const tc_graph *g, uint32_t u, uint32_t v, uint64_t *out) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    if ((uint64_t)u >= g->g.n || (uint64_t)v >= g->g.n) {
        set_error("vertex id out of range");
        return -1;
    }
    TC_CHECK(ensure_ref(const_cast<tc_graph *>(g)));
    return intersect_dev(g->g, u, v, out, g_stream);
}

int tc_count_with_timings(const uint32_t *pairs, uint64_t npairs, uint64_t nverts,
                          int pairs_on_device, int algo, uint64_t *out, tc_times *t) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(reserve_pool(scratch_estimate(npairs)));
    cudaStream_t s = g_stream;
    Events ev;
    TC_CHECK(ev.create());
    TC_CUDA(cudaEventRecord(ev.e[0], s));
    const uint32_t *dpairs = pairs;
    uint32_t *owned = nullptr;  // staging copy: default pool, freed at the end of the call
    const bool rank = algo == TC_ALGO_AUTO && npairs / 2 < (1ull << 32) && nverts < (1ull << 32);
    PreDegrees pre;
    if (!pairs_on_device && npairs) {
        TC_CHECK(dalloc_t(&owned, 2 * npairs, s, true));
        // rank path: the degree histogram runs chunk by chunk under the copy
        if (rank) TC_CHECK(h2d_degrees(owned, pairs, npairs, nverts, &pre, s));
        else TC_CHECK(h2d(owned, pairs, npairs * 8, s));
        dpairs = owned;
    }
    TC_CUDA(cudaEventRecord(ev.e[1], s));
    DeviceGraph g;
    int rc = rank ? preprocess_rank_dev(dpairs, npairs, nverts, &g, s, nullptr, pre.deg ? &pre : nullptr)
                  : preprocess_dev(dpairs, npairs, nverts, &g, s);
    dfree(pre.bad, s);
    if (rc) {
        if (owned) dfree(owned, s);
        graph_release(&g, s);
        return rc;
    }
    TC_CUDA(cudaEventRecord(ev.e[2], s));
    unsigned long long *total = nullptr;  // this call's accumulator
    rc = dalloc_t(&total, 1, s);
    if (!rc) rc = cudaMemsetAsync(total, 0, sizeof(unsigned long long), s) == cudaSuccess ? 0 : -2;
    CountStats st;
    const bool want_stats = opts().count_stats != 0;
    if (!rc) rc = count_range_dev(g, 0, g.m, algo, total, s, want_stats ? &st : nullptr);
    if (rc) {
        if (rc == -2 && !*last_error()) set_error("cudaMemsetAsync failed");
        dfree(total, s);
        if (owned) dfree(owned, s);
        graph_release(&g, s);
        return rc;
    }
    unsigned long long h = 0;
    TC_CUDA(cudaMemcpyAsync(&h, total, sizeof(h), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaEventRecord(ev.e[3], s));
    dfree(total, s);
    graph_release(&g, s);
    if (owned) dfree(owned, s);
    TC_CUDA(cudaEventSynchronize(ev.e[3]));
    *out = h;
    if (t) {
        memset(t, 0, sizeof(*t));
        t->h2d_ms = ms_between(ev.e[0], ev.e[1]);
        t->preprocess_ms = ms_between(ev.e[1], ev.e[2]);
        t->count_ms = ms_between(ev.e[2], ev.e[3]);
        t->total_ms = ms_between(ev.e[0], ev.e[3]);
        if (want_stats) {
            t->classify_ms = st.classify_ms;
            t->heavy_ms = st.heavy_ms;
            t->light_ms = st.light_ms;
            t->heavy_tasks = st.heavy_tasks;
            t->vmajor_ms = st.vmajor_ms;
        }
    }
    return 0;
}

int tc_work_bounds(const tc_graph *g, int npools, int64_t *bounds) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    if (npools < 1) {
        set_error("num_pools must be >= 1");
        return -1;
    }
    TC_CHECK(ensure_ref(const_cast<tc_graph *>(g)));  // bounds are reference edge indices
    return work_bounds_dev(g->g, npools, bounds, g_stream);
}

int tc_schedule_bytes(const tc_graph *g, uint64_t out[5]) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    const DeviceGraph *r = nullptr;
    TC_CHECK(rank_copy(const_cast<tc_graph *>(g), &r));
    return schedule_bytes_dev(*r, 0, r->m, out, g_stream);
}

int tc_schedule_bytes_range(const tc_graph *g, int64_t lo, int64_t hi, uint64_t out[5]) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    if (!g->g.rank_space) {
        set_error("ranged schedule bytes need a rank-space graph (tc_preprocess_ex RANK_SPACE)");
        return -1;
    }
    if (lo < 0 || hi < lo || (uint64_t)hi > g->g.m) {
        set_error("edge range outside [0, m]");
        return -1;
    }
    return schedule_bytes_dev(g->g, (uint64_t)lo, (uint64_t)hi, out, g_stream);
}

int tc_shard_plan(const tc_graph *g, int parts, int64_t *edge_bounds, int64_t *head_bounds) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    if (parts < 1) {
        set_error("parts must be >= 1");
        return -1;
    }
    const DeviceGraph *r = nullptr;
    TC_CHECK(rank_copy(const_cast<tc_graph *>(g), &r));
    return shard_plan_dev(*r, parts, edge_bounds, head_bounds, g_stream);
}

int tc_shard_cost_sizes(const tc_graph *g, int parts, uint64_t *ntiles, uint64_t *tile, uint64_t *nheads,
                        uint32_t *head0) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    const DeviceGraph *r = nullptr;
    TC_CHECK(rank_copy(const_cast<tc_graph *>(g), &r));
    shard_cost_sizes(*r, parts, ntiles, tile, nheads, head0);
    return 0;
}

int tc_shard_costs(const tc_graph *g, int parts, uint64_t *edge_tiles, uint64_t *head_costs) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    const DeviceGraph *r = nullptr;
    TC_CHECK(rank_copy(const_cast<tc_graph *>(g), &r));
    return shard_costs_dev(*r, parts, (unsigned long long *)edge_tiles, (unsigned long long *)head_costs, g_stream);
}

int tc_shard_stats(const tc_graph *g, int64_t lo, int64_t hi, int64_t hlo, int64_t hhi, uint64_t out[9]) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    const DeviceGraph *r = nullptr;
    TC_CHECK(rank_copy(const_cast<tc_graph *>(g), &r));
    return shard_stats_dev(*r, (uint64_t)lo, (uint64_t)hi, (uint32_t)hlo, (uint32_t)hhi, out, g_stream);
}

int tc_count_shard(const tc_graph *g, int64_t lo, int64_t hi, int64_t hlo, int64_t hhi, uint64_t *out,
                   tc_times *t) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    const DeviceGraph *r = nullptr;
    TC_CHECK(rank_copy(const_cast<tc_graph *>(g), &r));
    if (lo < 0 || hi < lo || (uint64_t)hi > r->m || hlo < 0 || hhi < hlo || (uint64_t)hhi > r->n) {
        set_error("shard outside [0, m) x [0, n)");
        return -1;
    }
    cudaStream_t s = g_stream;
    Events ev;
    TC_CHECK(ev.create());
    TC_CUDA(cudaEventRecord(ev.e[0], s));
    unsigned long long *total = nullptr;
    TC_CHECK(dalloc_t(&total, 1, s));
    TC_CUDA(cudaMemsetAsync(total, 0, sizeof(unsigned long long), s));
    CountStats st;
    const int rc = count_shard_dev(*r, (uint64_t)lo, (uint64_t)hi, (uint32_t)hlo, (uint32_t)hhi, total, s,
                                   t ? &st : nullptr);
    if (rc) {
        dfree(total, s);
        return rc;
    }
    unsigned long long hv = 0;
    TC_CUDA(cudaMemcpyAsync(&hv, total, sizeof(hv), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaEventRecord(ev.e[1], s));
    dfree(total, s);
    TC_CUDA(cudaEventSynchronize(ev.e[1]));
    *out = hv;
    if (t) {
        memset(t, 0, sizeof(*t));
        t->count_ms = t->total_ms = ms_between(ev.e[0], ev.e[1]);
        t->classify_ms = st.classify_ms;
        t->heavy_ms = st.heavy_ms;
        t->light_ms = st.light_ms;
        t->vmajor_ms = st.vmajor_ms;
        t->heavy_tasks = st.heavy_tasks;
    }
    return 0;
}

int tc_merge_work(const tc_graph *g, uint64_t *out) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    // W is label-independent: use whichever copy exists
    return merge_work_dev(g->ref_ready ? g->g : *g->rank, out, g_stream);
}

int tc_sort_edges(const uint32_t *pairs, uint64_t npairs, uint64_t nverts, uint32_t *out_pairs) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    if (npairs == 0) return 0;
    cudaStream_t s = g_stream;
    uint32_t *din = nullptr, *dout = nullptr;
    TC_CHECK(dalloc_t(&din, 2 * npairs, s));
    TC_CHECK(dalloc_t(&dout, 2 * npairs, s));
    TC_CHECK(h2d(din, pairs, npairs * 8, s));
    TC_CHECK(sort_pairs_dev(din, npairs, nverts, dout, s));
    TC_CUDA(cudaMemcpyAsync(out_pairs, dout, npairs * 8, cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(din, s);
    dfree(dout, s);
    return 0;
}

int tc_build_node_array(const uint32_t *firsts, uint64_t k, uint64_t n, int64_t *offsets) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    cudaStream_t s = g_stream;
    uint32_t *df = nullptr;
    int64_t *doff = nullptr;
    TC_CHECK(dalloc_t(&df, k ? k : 1, s));
    TC_CHECK(dalloc_t(&doff, n + 1, s));
    if (k) TC_CUDA(cudaMemcpyAsync(df, firsts, k * 4, cudaMemcpyHostToDevice, s));
    TC_CHECK(build_node_array_dev(df, k, n, doff, nullptr, nullptr, s));
    TC_CUDA(cudaMemcpyAsync(offsets, doff, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(df, s);
    dfree(doff, s);
    return 0;
}

int tc_orient_and_compact(const uint32_t *pairs, uint64_t npairs, const int64_t *degrees,
                          uint64_t n, uint32_t *out_pairs, uint64_t *kept) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    *kept = 0;
    if (npairs == 0) return 0;
    cudaStream_t s = g_stream;
    uint32_t *din = nullptr, *dout = nullptr;
    int64_t *ddeg = nullptr;
    TC_CHECK(dalloc_t(&din, 2 * npairs, s));
    TC_CHECK(dalloc_t(&dout, 2 * npairs, s));
    TC_CHECK(dalloc_t(&ddeg, n ? n : 1, s));
    TC_CHECK(h2d(din, pairs, npairs * 8, s));
    if (n) TC_CUDA(cudaMemcpyAsync(ddeg, degrees, n * 8, cudaMemcpyHostToDevice, s));
    uint64_t k = 0;
    TC_CHECK(orient_compact_dev(din, npairs, ddeg, n, dout, &k, s));
    if (k) TC_CUDA(cudaMemcpyAsync(out_pairs, dout, k * 8, cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    dfree(din, s);
    dfree(dout, s);
    dfree(ddeg, s);
    *kept = k;
    return 0;
}

int tc_gen_rmat(int scale, int edge_factor, const double probs[4], const uint64_t state[2],
                const uint64_t inc[2], uint32_t **dev_pairs, uint64_t *npairs, uint64_t *nverts) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(rmat_dev(scale, edge_factor, probs, state, inc, dev_pairs, npairs, nverts, g_stream));
    TC_CUDA(cudaStreamSynchronize(g_stream));
    return 0;
}

int tc_gen_ba(uint64_t n, uint32_t m_attach, const uint64_t state[2], const uint64_t inc[2],
              uint32_t **dev_pairs, uint64_t *npairs, uint64_t *nverts) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(ba_dev(n, m_attach, state, inc, dev_pairs, npairs, nverts, g_stream));
    return 0;
}

static int with_device_pairs(const uint32_t *pairs, uint64_t npairs, int on_device,
                             const uint32_t **dp, uint32_t **owned) {
    *dp = pairs;
    *owned = nullptr;
    if (!on_device && npairs) {
        TC_CHECK(dalloc_t(owned, 2 * npairs, g_stream, true));
        TC_CHECK(h2d(*owned, pairs, npairs * 8, g_stream));
        *dp = *owned;
    }
    return 0;
}

// ---- distributed preprocessing steps ---------------------------------
int tc_dist_degrees(const uint32_t *pairs, uint64_t npairs, int pairs_on_device, uint64_t nverts,
                    uint32_t *deg_dev) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    const uint32_t *dp;
    uint32_t *owned;
    TC_CHECK(with_device_pairs(pairs, npairs, pairs_on_device, &dp, &owned));
    const int rc = dist_degrees_dev(dp, npairs, nverts, deg_dev, g_stream);
    if (owned) dfree(owned, g_stream);
    return rc;
}

int tc_dist_orient(const uint32_t *pairs, uint64_t npairs, int pairs_on_device, uint64_t nverts,
                   const uint32_t *deg_dev, uint64_t **keys_dev, uint64_t *nkeys, uint32_t *outdeg_dev) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    const uint32_t *dp;
    uint32_t *owned;
    TC_CHECK(with_device_pairs(pairs, npairs, pairs_on_device, &dp, &owned));
    const int rc = dist_orient_dev(dp, npairs, nverts, deg_dev, keys_dev, nkeys, outdeg_dev, g_stream);
    if (owned) dfree(owned, g_stream);
    return rc;
}

int tc_dist_layout(tc_graph *g, const uint32_t *outdeg_dev, int parts, int64_t *cuts,
                   int64_t *edge_cuts) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    return dist_layout_dev(&g->g, outdeg_dev, parts, cuts, edge_cuts, g_stream);
}

int tc_dist_split(const uint64_t *keys_dev, uint64_t nkeys, uint64_t nverts, const int64_t *cuts,
                  int parts, int64_t *counts) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    return dist_split_dev(keys_dev, nkeys, nverts, cuts, parts, counts, g_stream);
}

int tc_dist_place(tc_graph *g, uint64_t *keys_dev, uint64_t nkeys, uint64_t edge_pos) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(check_graph(g));
    return dist_place_dev(&g->g, keys_dev, nkeys, edge_pos, g_stream);
}

int tc_gen_rgg(uint64_t n, double radius, const uint64_t state[2], const uint64_t inc[2],
               uint32_t **dev_pairs, uint64_t *npairs, uint64_t *nverts) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(rgg_dev(n, radius, state, inc, dev_pairs, npairs, nverts, g_stream));
    return 0;
}

int tc_read_tri1(const char *path, uint32_t **host_pairs, uint64_t *npairs) {
    TC_CHECK(ensure());
    return read_tri1(path, host_pairs, npairs);
}

int tc_parse_edge_list(const char *path, uint32_t **host_pairs, uint64_t *npairs,
                       uint64_t *err_line, int *err_kind) {
    TC_CHECK(ensure());
    return parse_edge_list(path, host_pairs, npairs, err_line, err_kind);
}


int tc_validate_edge_array(const uint32_t *pairs, uint64_t npairs, uint64_t nverts,
                           int pairs_on_device, int *code, uint64_t *index) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    const uint32_t *dp;
    uint32_t *owned;
    TC_CHECK(with_device_pairs(pairs, npairs, pairs_on_device, &dp, &owned));
    const int rc = validate_pairs_dev(dp, npairs, nverts, code, index, g_stream);
    if (owned) dfree(owned, g_stream);
    return rc;
}

int tc_wedge_count(const uint32_t *pairs, uint64_t npairs, uint64_t nverts, int pairs_on_device,
                   uint64_t *out, double *approx) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    const uint32_t *dp;
    uint32_t *owned;
    TC_CHECK(with_device_pairs(pairs, npairs, pairs_on_device, &dp, &owned));
    const int rc = wedges_dev(dp, npairs, nverts, out, approx, g_stream);
    if (owned) dfree(owned, g_stream);
    return rc;
}

int tc_device_alloc(uint64_t bytes, void **p) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CHECK(dalloc(p, bytes, g_stream, true));
    TC_CUDA(cudaStreamSynchronize(g_stream));
    return 0;
}

int tc_device_free(void *p) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    dfree(p, g_stream);
    TC_CUDA(cudaStreamSynchronize(g_stream));
    return 0;
}

int tc_memcpy(void *dst, const void *src, uint64_t bytes, int kind) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                     : kind == 1 ? cudaMemcpyDeviceToHost
                                 : cudaMemcpyDeviceToDevice;
    TC_CUDA(cudaMemcpyAsync(dst, src, bytes, k, g_stream));
    TC_CUDA(cudaStreamSynchronize(g_stream));
    return 0;
}

int tc_host_alloc(uint64_t bytes, void **p) {
    TC_CHECK(ensure());
    TC_CUDA(cudaHostAlloc(p, bytes ? bytes : 16, cudaHostAllocDefault));
    return 0;
}

int tc_host_free(void *p) {
    TC_CHECK(ensure());
    TC_CUDA(cudaFreeHost(p));
    return 0;
}

int tc_host_register(void *p, uint64_t bytes) {
    TC_CHECK(ensure());
    TC_CUDA(cudaHostRegister(p, bytes, cudaHostRegisterDefault));
    return 0;
}

int tc_host_unregister(void *p) {
    TC_CHECK(ensure());
    TC_CUDA(cudaHostUnregister(p));
    return 0;
}

int tc_synchronize(void) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    TC_CUDA(cudaStreamSynchronize(g_stream));
    return 0;
}

int tc_reserve(uint64_t bytes) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    return reserve_pool(bytes);
}

namespace {
struct OptionName {
    const char *name;
    int64_t Options::*field;
};
const OptionName kOptionNames[] = {
    {"vmajor", &Options::vmajor},           {"vzone_log2", &Options::vzone_log2},
    {"vlow_all", &Options::vlow_all},       {"vm_bias", &Options::vm_bias},
    {"dense_factor", &Options::dense_factor}, {"hub_unroll", &Options::hub_unroll},
    {"l2_persist_mb", &Options::l2_persist_mb}, {"l2_target", &Options::l2_target},
    {"concurrent", &Options::concurrent},   {"share", &Options::share},
    {"midwarp", &Options::midwarp},         {"light", &Options::light},
    {"skew", &Options::skew},               {"light_vec", &Options::light_vec},
    {"shard_model", &Options::shard_model}, {"shard_ovh", &Options::shard_ovh},
    {"shard_ucap", &Options::shard_ucap},   {"dense_ranks", &Options::dense_ranks},
    {"shard_ovh2", &Options::shard_ovh2},   {"copy_threads", &Options::copy_threads},
    {"seg_fork", &Options::seg_fork},
    {"vin_overlap", &Options::vin_overlap},
    {"vin_grid", &Options::vin_grid},
    {"seg_k16", &Options::seg_k16},
    {"seg_w2k", &Options::seg_w2k},
    {"vhub", &Options::vhub},
    {"vhub_unroll", &Options::vhub_unroll},
    {"vhub_blocks", &Options::vhub_blocks},
    {"vhub_b16w", &Options::vhub_b16w},
    {"hub_cap_div", &Options::hub_cap_div},
    {"vix", &Options::vix},
    {"shard_w_dense", &Options::shard_w_dense}, {"shard_w_sparse", &Options::shard_w_sparse},
    {"shard_w_light", &Options::shard_w_light}, {"shard_w_stage", &Options::shard_w_stage},
    {"shard_w_edge", &Options::shard_w_edge},   {"shard_w_hub", &Options::shard_w_hub},
    {"shard_w_vlow", &Options::shard_w_vlow},   {"shard_w_vedge", &Options::shard_w_vedge},
    {"bucket", &Options::bucket},           {"count_stats", &Options::count_stats},
    {"hubpack", &Options::hubpack},         {"rank_primary", &Options::rank_primary},
};
}  // namespace

int tc_set_option(const char *name, int64_t value) {
    TC_API_GUARD();
    for (const auto &o : kOptionNames)
        if (name && !strcmp(name, o.name)) {
            g_opts.*(o.field) = value;
            return 0;
        }
    set_error(std::string("unknown option: ") + (name ? name : "(null)"));
    return -1;
}

int tc_get_option(const char *name, int64_t *value) {
    TC_API_GUARD();
    for (const auto &o : kOptionNames)
        if (name && !strcmp(name, o.name)) {
            *value = g_opts.*(o.field);
            return 0;
        }
    set_error(std::string("unknown option: ") + (name ? name : "(null)"));
    return -1;
}

int tc_reset_options(void) {
    TC_API_GUARD();
    g_opts = Options();
    return 0;
}

int tc_launch_count(uint64_t *out) {
    *out = g_launches.load();
    return 0;
}

int tc_timer_record(int slot) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    if (slot < 0 || slot >= 8) {
        set_error("timer slot must be in [0, 8)");
        return -1;
    }
    if (!g_timer[slot]) TC_CUDA(cudaEventCreate(&g_timer[slot]));
    TC_CUDA(cudaEventRecord(g_timer[slot], g_stream));
    return 0;
}

int tc_timer_elapsed(int a, int b, double *ms) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    if (a < 0 || a >= 8 || b < 0 || b >= 8 || !g_timer[a] || !g_timer[b]) {
        set_error("timer slots not recorded");
        return -1;
    }
    TC_CUDA(cudaEventSynchronize(g_timer[b]));
    float f = 0;
    TC_CUDA(cudaEventElapsedTime(&f, g_timer[a], g_timer[b]));
    *ms = f;
    return 0;
}

int tc_l2_flush(void) {
    TC_API_GUARD();
    TC_CHECK(ensure());
    if (!g_flush) {
        int l2 = 0;
        TC_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, g_device));
        g_flush_bytes = (size_t)l2 * 2;
        TC_CUDA(cudaMalloc(&g_flush, g_flush_bytes));
    }
    TC_CUDA(cudaMemsetAsync(g_flush, 0x5a, g_flush_bytes, g_stream));
    return 0;
}

}  // extern "C"
