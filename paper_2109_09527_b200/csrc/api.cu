#include <stdlib.h>

#include <chrono>
#include <mutex>
// api.cu -- the extern "C" boundary of libprgpu (include/prgpu.h).
// Validation, host/device pointer handling, graph lifetime.  All compute is
// in ingest.cu / preprocess.cu / iterate.cu.
#include <math.h>
#include <stdarg.h>
#include <vector>
#include <string.h>

#include <new>

#include "internal.h"

namespace prgpu {

static thread_local char g_err[512] = {0};

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

double g_alloc_ms = 0.0;

bool pdl_enabled() {  // PRGPU_PDL=0 turns programmatic dependent launch off (measurement)
    static const bool on = [] {
        const char* e = getenv("PRGPU_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// One private pool per device (created on first use, release threshold
// UINT64_MAX: freed memory is kept for the next graph instead of being
// unmapped at every synchronisation -- re-mapping GBs costs tens of ms per
// pr_graph_create).  The process's default pool is left as the caller set it.
static std::mutex g_pool_mu;
static cudaMemPool_t g_pools[64] = {};

cudaMemPool_t lib_pool() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return nullptr;
    }
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (!g_pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool;
        if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        cudaGetLastError();
        g_pools[dev] = pool;
    }
    return g_pools[dev];
}

static int make_ctx(Ctx& ctx, void* stream) {
    ctx.stream = (cudaStream_t)stream;
    ctx.launches = 0;
    int dev = 0;
    PR_CUDA(cudaGetDevice(&dev));
    PR_CUDA(cudaDeviceGetAttribute(&ctx.num_sms, cudaDevAttrMultiProcessorCount, dev));
    return PR_OK;
}

// Grow the library pool once to `bytes` (allocate + free), so that later
// stream-ordered allocations are carved from memory the pool already holds
// instead of mapping new memory in the middle of a call (measured: up to
// 60 ms per pr_graph_create under allocation churn otherwise).
static void pool_reserve(cudaStream_t s, size_t bytes) {
    const char* e = getenv("PRGPU_POOL_RESERVE");
    if (e && e[0] == '0') return;
    cudaMemPool_t pool = lib_pool();
    if (!pool) return;
    uint64_t have = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &have);
    if (have >= bytes) return;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    if (bytes > have + fr / 2) bytes = have + fr / 2;  // never take more than half of what is free
    void* p = nullptr;
    if (bytes > have && cudaMallocFromPoolAsync(&p, bytes - have, pool, s) == cudaSuccess) cudaFreeAsync(p, s);
    cudaGetLastError();
}

// Every call that enqueues work records the graph's event on its stream at the
// end; pr_destroy waits for it before releasing the buffers (the caller's
// stream may be non-blocking, and pr_run may return with k_unpermute still
// reading them when the ranks are in device memory).
static void mark_done(pr_graph* g, cudaStream_t s) {
    if (!g) return;
    if (!g->fin_ev && cudaEventCreateWithFlags(&g->fin_ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        g->fin_ev = nullptr;
        return;
    }
    if (cudaEventRecord(g->fin_ev, s) != cudaSuccess) cudaGetLastError();
}

// Pinned host copies of the per-graph DevState come from one process-wide
// slab (cudaMallocHost / cudaFreeHost cost milliseconds and synchronise the
// device, once per pr_graph_create / pr_destroy otherwise).
constexpr int kSlabSlots = 256;
static std::mutex g_slab_mu;
static DevState* g_slab = nullptr;
static bool g_slab_used[kSlabSlots] = {false};

static DevState* pinned_state_alloc() {
    {
        std::lock_guard<std::mutex> lk(g_slab_mu);
        if (!g_slab) {
            void* p = nullptr;
            if (cudaMallocHost(&p, sizeof(DevState) * kSlabSlots) == cudaSuccess) g_slab = (DevState*)p;
            cudaGetLastError();
        }
        if (g_slab)
            for (int i = 0; i < kSlabSlots; ++i)
                if (!g_slab_used[i]) {
                    g_slab_used[i] = true;
                    return g_slab + i;
                }
    }
    void* p = nullptr;  // slab exhausted: a private pinned allocation
    if (cudaMallocHost(&p, sizeof(DevState)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return (DevState*)p;
}

static void pinned_state_free(DevState* p) {
    if (!p) return;
    {
        std::lock_guard<std::mutex> lk(g_slab_mu);
        if (g_slab && p >= g_slab && p < g_slab + kSlabSlots) {
            g_slab_used[p - g_slab] = false;
            return;
        }
    }
    cudaFreeHost(p);
}

static bool is_pinned_host_ptr(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

static bool is_device_ptr(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// PRGPU_PROFILE=1: host wall time of each phase (synchronising the stream at
// every mark, so it perturbs the timing it reports); PRGPU_PROFILE=2: CUDA
// events at every mark (no syncs), printed with the host time of each mark
// when the timer is destroyed.  Diagnostics only.
struct PhaseTimer {
    cudaStream_t s;
    const char* what;
    int mode = 0;
    std::chrono::steady_clock::time_point t0, t;
    cudaEvent_t ev[16];
    double host_ms[16];
    const char* names[16];
    int k = 0;
    double alloc0 = g_alloc_ms;
    PhaseTimer(cudaStream_t st, const char* w) : s(st), what(w) {
        const char* e = getenv("PRGPU_PROFILE");
        mode = e ? atoi(e) : 0;
        if (mode == 1) cudaStreamSynchronize(s);
        t0 = t = std::chrono::steady_clock::now();
        if (mode == 2) {
            cudaEventCreate(&ev[0]);
            cudaEventRecord(ev[0], s);
            k = 1;
        }
    }
    void mark(const char* phase) {
        if (mode == 1) {
            cudaStreamSynchronize(s);
            auto now = std::chrono::steady_clock::now();
            fprintf(stderr, "[prgpu] %s.%s %.3f ms\n", what, phase,
                    std::chrono::duration<double, std::milli>(now - t).count());
            t = now;
        } else if (mode == 2 && k < 16) {
            cudaEventCreate(&ev[k]);
            cudaEventRecord(ev[k], s);
            host_ms[k] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            names[k++] = phase;
        }
    }
    ~PhaseTimer() {
        if (mode == 2) fprintf(stderr, "[prgpu] %s host total %.3f ms, of which cudaMallocAsync %.3f ms\n", what,
                               std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
                               g_alloc_ms - alloc0);
        if (mode != 2) return;
        cudaEventSynchronize(ev[k - 1]);
        for (int i = 1; i < k; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            fprintf(stderr, "[prgpu] %s.%s gpu %.3f ms (host mark at %.3f ms)\n", what, names[i], ms, host_ms[i]);
        }
        for (int i = 0; i < k; ++i) cudaEventDestroy(ev[i]);
    }
};

}  // namespace prgpu

using namespace prgpu;

extern "C" {
#pragma GCC visibility push(default)

const char* pr_last_error(void) { return g_err; }

int pr_release_memory(void) {
    g_err[0] = 0;
    cudaMemPool_t pool = lib_pool();
    if (!pool) {
        set_error("pr_release_memory: no library pool on this device");
        return PR_ECUDA;
    }
    PR_CUDA(cudaDeviceSynchronize());  // frees still pending on some stream land first
    PR_CUDA(cudaMemPoolTrimTo(pool, 0));
    return PR_OK;
}

static int create_graph(const char* fn, int64_t n, int64_t m, const int32_t* src, const int32_t* dst, void* stream,
                        pr_graph** out, int rank, int world, pr_allreduce_fn allreduce, void* allreduce_ctx) {
    if (!out) {
        set_error("%s: out is NULL", fn);
        return PR_EINVAL;
    }
    *out = nullptr;
    if (n < 1 || n > 2147483647LL) {
        set_error("%s: n=%lld outside [1, 2^31-1]", fn, (long long)n);
        return PR_EINVAL;
    }
    if (m < 0 || m > 2147483647LL) {
        set_error("%s: m=%lld outside [0, 2^31-1]", fn, (long long)m);
        return PR_EINVAL;
    }
    if (m > 0 && (!src || !dst)) {
        set_error("%s: NULL edge array", fn);
        return PR_EINVAL;
    }
    Ctx ctx;
    PR_TRY(make_ctx(ctx, stream));
    PhaseTimer pt0(ctx.stream, "create");
    // peak of create + preprocess + run: ~ 4 x 8 B per raw edge (sort ping-pong,
    // views) + ~ 80 B per vertex
    pool_reserve(ctx.stream, (size_t)m * (world > 1 ? 24 : 40) + (size_t)n * 96 + ((size_t)64 << 20));
    pr_graph* g = new (std::nothrow) pr_graph();
    if (!g) {
        set_error("%s: host allocation failed", fn);
        return PR_ENOMEM;
    }
    g->n = n;
    g->m_raw = m;
    g->num_sms = ctx.num_sms;
    cudaGetDevice(&g->device);
    int rc = PR_OK;
    int32_t* dsrc = nullptr;
    int32_t* ddst = nullptr;
    do {
        if (!(g->st_host = pinned_state_alloc())) {
            set_error("pinned host allocation failed");
            rc = PR_ENOMEM;
            break;
        }
        if ((rc = dalloc(&g->st, 1, ctx.stream)) != PR_OK) break;
        const int32_t* s = src;
        const int32_t* t = dst;
        // pinned host edge list, one rank: copied in chunks inside the ingest,
        // overlapped with the sorting of the chunks already in
        const bool host_chunked = m > 0 && world == 1 && !allreduce && is_pinned_host_ptr(src) &&
                                  is_pinned_host_ptr(dst) && ingest_chunked_applies(n, m);
        if (m > 0 && !host_chunked && !is_device_ptr(src)) {  // host edge list: copy in (e2e path)
            if ((rc = dalloc(&dsrc, (size_t)m, ctx.stream)) != PR_OK) break;
            if (cudaMemcpyAsync(dsrc, src, sizeof(int32_t) * (size_t)m, cudaMemcpyDefault, ctx.stream) != cudaSuccess) {
                set_error("copy of src failed");
                rc = PR_ECUDA;
                break;
            }
            s = dsrc;
        }
        if (m > 0 && !host_chunked && !is_device_ptr(dst)) {
            if ((rc = dalloc(&ddst, (size_t)m, ctx.stream)) != PR_OK) break;
            if (cudaMemcpyAsync(ddst, dst, sizeof(int32_t) * (size_t)m, cudaMemcpyDefault, ctx.stream) != cudaSuccess) {
                set_error("copy of dst failed");
                rc = PR_ECUDA;
                break;
            }
            t = ddst;
        }
        pt0.mark("setup");
        PhaseTimer pt(ctx.stream, "create");
        if ((rc = ingest(g, s, t, ctx, rank, world, host_chunked)) != PR_OK) break;
        pt.mark("ingest");
        dfree(dsrc, ctx.stream);
        dfree(ddst, ctx.stream);
        if (allreduce) {
            // the rank ingested only the edges into its vertices: its out-degrees
            // are partial; their sum over the ranks is the graph's (every
            // deduplicated edge lives on exactly one rank, the owner of its dst)
            if (cudaStreamSynchronize(ctx.stream) != cudaSuccess ||
                allreduce(allreduce_ctx, g->outdeg, n, world, (void*)ctx.stream) != 0) {
                set_error("%s: the out-degree all-reduce failed", fn);
                rc = PR_ECUDA;
                break;
            }
            pt.mark("allreduce");
        }
        if ((rc = build_relabel(g, ctx, !(world > 1 || allreduce))) != PR_OK) break;
        pt.mark("relabel");
        if (world > 1 || allreduce) {
            g->shard_only = true;
            if ((rc = build_shard(g, rank, world, ctx, true)) != PR_OK) break;
            pt.mark("shard");
        } else {
            if ((rc = build_view_stream(g->plain, ctx, (int32_t)g->n_contrib, g->outdeg, g->cidx)) != PR_OK) break;
            if ((rc = build_view_blocked(g->plain, ctx, g->n_contrib)) != PR_OK) break;
            pt.mark("stream");
        }
        if (cudaStreamSynchronize(ctx.stream) != cudaSuccess) {
            set_error("%s: %s", fn, cudaGetErrorString(cudaGetLastError()));
            rc = PR_ECUDA;
            break;
        }
    } while (0);
    g->launches += ctx.launches;
    if (rc != PR_OK) {
        dfree(dsrc, ctx.stream);
        dfree(ddst, ctx.stream);
        mark_done(g, ctx.stream);
        pr_destroy(g);
        return rc;
    }
    mark_done(g, ctx.stream);
    *out = g;
    return PR_OK;
}

int pr_graph_create(int64_t n, int64_t m, const int32_t* src, const int32_t* dst, void* stream, pr_graph** out) {
    g_err[0] = 0;
    return create_graph("pr_graph_create", n, m, src, dst, stream, out, 0, 1, nullptr, nullptr);
}

int pr_graph_create_sharded(int64_t n, int64_t m, const int32_t* src, const int32_t* dst, int32_t rank,
                            int32_t world, pr_allreduce_fn allreduce, void* allreduce_ctx, void* stream,
                            pr_graph** out) {
    g_err[0] = 0;
    if (out) *out = nullptr;
    if (world < 1 || world > 4096 || rank < 0 || rank >= world || !allreduce) {
        set_error("pr_graph_create_sharded: rank=%d world=%d allreduce=%p (need 0 <= rank < world <= 4096, "
                  "an all-reduce)", rank, world, (void*)allreduce);
        return PR_EINVAL;
    }
    return create_graph("pr_graph_create_sharded", n, m, src, dst, stream, out, rank, world, allreduce,
                        allreduce_ctx);
}

int pr_preprocess(pr_graph* g, uint32_t flags, void* stream) {
    g_err[0] = 0;
    if (!g) {
        set_error("pr_preprocess: NULL graph");
        return PR_EINVAL;
    }
    if (flags & ~(PR_PRE_IDENTICAL | PR_PRE_CHAIN)) {
        set_error("pr_preprocess: unknown flag bits 0x%x", flags);
        return PR_EINVAL;
    }
    if (g->shard_only) {
        set_error("pr_preprocess: a graph from pr_graph_create_sharded holds one rank's rows only");
        return PR_ESTATE;
    }
    Ctx ctx;
    PR_TRY(make_ctx(ctx, stream));
    int rc = preprocess(g, flags, ctx);
    g->launches += ctx.launches;
    mark_done(g, ctx.stream);
    if (rc == PR_OK) PR_CUDA(cudaStreamSynchronize(ctx.stream));
    return rc;
}

int pr_run(pr_graph* g, double d, double threshold, int32_t max_iter, void* stream, uint32_t mode, double* ranks,
           int32_t* iters_out, double* final_delta_out) {
    g_err[0] = 0;
    if (!g || !ranks) {
        set_error("pr_run: NULL graph or ranks");
        return PR_EINVAL;
    }
    if (!(d > 0.0 && d < 1.0)) {
        set_error("pr_run: d=%g outside (0,1)", d);
        return PR_EINVAL;
    }
    if (!(threshold >= 0.0)) {
        set_error("pr_run: threshold must be >= 0 and not NaN");
        return PR_EINVAL;
    }
    if (max_iter < 1) {
        set_error("pr_run: max_iter=%d < 1", max_iter);
        return PR_EINVAL;
    }
    if (mode & ~(PR_MODE_ASYNC | PR_MODE_NOSYNC | PR_NORM_LINF | PR_USE_REDUCTIONS | PR_TIMING | PR_PERFORATE |
                 PR_MODE_PHASED | PR_CHAIN_EAGER)) {
        set_error("pr_run: unknown mode bits 0x%x", mode);
        return PR_EINVAL;
    }
    if ((mode & PR_MODE_ASYNC) && (mode & PR_MODE_NOSYNC)) {
        set_error("pr_run: PR_MODE_ASYNC and PR_MODE_NOSYNC are exclusive");
        return PR_EINVAL;
    }
    if ((mode & PR_MODE_PHASED) && (mode & (PR_MODE_ASYNC | PR_MODE_NOSYNC | PR_PERFORATE))) {
        set_error("pr_run: PR_MODE_PHASED is exclusive with PR_MODE_ASYNC / PR_MODE_NOSYNC / PR_PERFORATE");
        return PR_EINVAL;
    }
    if ((mode & PR_PERFORATE) && (mode & PR_USE_REDUCTIONS)) {
        set_error("pr_run: PR_PERFORATE is defined for the plain view only (not with PR_USE_REDUCTIONS)");
        return PR_EINVAL;
    }
    if ((mode & PR_USE_REDUCTIONS) && !g->pre_done) {
        set_error("pr_run: PR_USE_REDUCTIONS before pr_preprocess");
        return PR_ESTATE;
    }
    if (g->shard_only) {
        set_error("pr_run: a graph from pr_graph_create_sharded holds one rank's rows only (pr_run_sharded)");
        return PR_ESTATE;
    }
    Ctx ctx;
    PR_TRY(make_ctx(ctx, stream));
    int rc = run(g, d, threshold, max_iter, mode, ranks, ctx, iters_out, final_delta_out);
    g->launches += ctx.launches;
    mark_done(g, ctx.stream);
    g->last.total_launches = g->launches;
    return rc;
}

int pr_graph_shard(pr_graph* g, int32_t rank, int32_t world, void* stream) {
    g_err[0] = 0;
    if (!g) {
        set_error("pr_graph_shard: NULL graph");
        return PR_EINVAL;
    }
    if (world < 1 || world > 4096 || rank < 0 || rank >= world) {
        set_error("pr_graph_shard: rank=%d world=%d (need 0 <= rank < world <= 4096)", rank, world);
        return PR_EINVAL;
    }
    if (g->shard_only) {
        set_error("pr_graph_shard: the graph is already one rank's share (pr_graph_create_sharded)");
        return PR_ESTATE;
    }
    Ctx ctx;
    PR_TRY(make_ctx(ctx, stream));
    int rc = build_shard(g, rank, world, ctx);
    g->launches += ctx.launches;
    mark_done(g, ctx.stream);
    if (rc != PR_OK) {
        clear_shard(g, ctx.stream);
        return rc;
    }
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    return PR_OK;
}

int pr_run_sharded(pr_graph* g, double d, double threshold, int32_t max_iter, void* stream, uint32_t mode,
                   double* ranks, pr_exchange_fn exchange, void* exchange_ctx, int32_t* iters_out,
                   double* final_delta_out) {
    g_err[0] = 0;
    if (!g || !ranks || !exchange) {
        set_error("pr_run_sharded: NULL graph, ranks or exchange");
        return PR_EINVAL;
    }
    if (!(d > 0.0 && d < 1.0)) {
        set_error("pr_run_sharded: d=%g outside (0,1)", d);
        return PR_EINVAL;
    }
    if (!(threshold >= 0.0)) {
        set_error("pr_run_sharded: threshold must be >= 0 and not NaN");
        return PR_EINVAL;
    }
    if (max_iter < 1) {
        set_error("pr_run_sharded: max_iter=%d < 1", max_iter);
        return PR_EINVAL;
    }
    if (mode & ~(PR_NORM_LINF | PR_TIMING)) {
        set_error("pr_run_sharded: mode 0x%x (only PR_MODE_SYNC, PR_NORM_LINF, PR_TIMING)", mode);
        return PR_EINVAL;
    }
    cudaPointerAttributes at{};
    const bool dev = cudaPointerGetAttributes(&at, ranks) == cudaSuccess &&
                     (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    if (!dev) {
        set_error("pr_run_sharded: ranks must be device memory");
        return PR_EINVAL;
    }
    if (g->shard_world < 1) {
        set_error("pr_run_sharded: pr_graph_shard has not run");
        return PR_ESTATE;
    }
    Ctx ctx;
    PR_TRY(make_ctx(ctx, stream));
    int rc = run_sharded(g, d, threshold, max_iter, mode, ranks, ctx, exchange, exchange_ctx, iters_out,
                         final_delta_out);
    g->launches += ctx.launches;
    mark_done(g, ctx.stream);
    g->last.total_launches = g->launches;
    return rc;
}

int pr_shard_buffers(const pr_graph* g, void** y0, void** y1, int64_t* len) {
    if (!g || !y0 || !y1 || !len) {
        set_error("pr_shard_buffers: bad arguments");
        return PR_EINVAL;
    }
    if (g->shard_world < 1) {
        set_error("pr_shard_buffers: pr_graph_shard has not run");
        return PR_ESTATE;
    }
    *y0 = g->sy[0];
    *y1 = g->sy[1];
    *len = g->shard_hot + (int64_t)g->shard_world * g->shard_chunk + 1;
    return PR_OK;
}

int pr_shard_set_peers(pr_graph* g, void* const* y0s, void* const* y1s, int32_t world) {
    g_err[0] = 0;
    if (!g) {
        set_error("pr_shard_set_peers: NULL graph");
        return PR_EINVAL;
    }
    if (g->shard_world < 1) {
        set_error("pr_shard_set_peers: pr_graph_shard has not run");
        return PR_ESTATE;
    }
    if (world == 0 || !y0s || !y1s) {  // back to the all-gather exchange
        clear_peers(g);
        return PR_OK;
    }
    if (world != g->shard_world) {
        set_error("pr_shard_set_peers: world %d != the shard's %d", world, g->shard_world);
        return PR_EINVAL;
    }
    if (g->mc) {
        set_error("pr_shard_set_peers: the multicast team is set (exclusive with peer buffers)");
        return PR_ESTATE;
    }
    for (int r = 0; r < world; ++r)
        if (r != g->shard_rank && (!y0s[r] || !y1s[r])) {
            set_error("pr_shard_set_peers: NULL buffer for rank %d", r);
            return PR_EINVAL;
        }
    return set_peers(g, (double* const*)y0s, (double* const*)y1s, world);
}

static int mc_guard(const pr_graph* g, const char* fn) {
    if (!g) {
        set_error("%s: NULL graph", fn);
        return PR_EINVAL;
    }
    if (g->shard_world < 1) {
        set_error("%s: the graph is not sharded", fn);
        return PR_ESTATE;
    }
    return PR_OK;
}

int pr_shard_mc_create(pr_graph* g, void* handle_out) {
    g_err[0] = 0;
    PR_TRY(mc_guard(g, "pr_shard_mc_create"));
    return mc_create(g, handle_out);
}

int pr_shard_mc_attach(pr_graph* g, const void* handle) {
    g_err[0] = 0;
    PR_TRY(mc_guard(g, "pr_shard_mc_attach"));
    return mc_attach(g, handle);
}

int pr_shard_mc_bind(pr_graph* g, void* stream) {
    g_err[0] = 0;
    PR_TRY(mc_guard(g, "pr_shard_mc_bind"));
    Ctx ctx;
    PR_TRY(make_ctx(ctx, stream));
    const int rc = mc_bind(g, ctx);
    if (rc != PR_OK) clear_multicast(g);
    return rc;
}

int pr_shard_device_barrier(pr_graph* g, int32_t on) {
    g_err[0] = 0;
    if (!g) {
        set_error("pr_shard_device_barrier: NULL graph");
        return PR_EINVAL;
    }
    if (on && (g->shard_world < 1 || (g->shard_world > 1 && !g->speer_flags && !(g->mc && g->mc->bound)))) {
        set_error("pr_shard_device_barrier: needs the peer buffers (pr_shard_set_peers / pr_shard_open_ipc) or "
                  "the multicast team (pr_shard_mc_*)");
        return PR_ESTATE;
    }
    if (on && g->shard_world > 65) {
        set_error("pr_shard_device_barrier: world %d > 65", g->shard_world);
        return PR_EINVAL;
    }
    g->sdev_barrier = on != 0;
    return PR_OK;
}

int pr_selftest_peer_barrier(int32_t world, int32_t epochs, void* stream) {
    g_err[0] = 0;
    Ctx ctx;
    PR_TRY(make_ctx(ctx, stream));
    int bad = 0;
    PR_TRY(barrier_selftest(world, epochs, ctx, &bad));
    if (bad != 0) {
        set_error("pr_selftest_peer_barrier: %d mismatches / timeouts (x1e6)", bad);
        return PR_ECUDA;
    }
    return PR_OK;
}

int pr_shard_export_ipc(const pr_graph* g, void* handles) {
    if (!g || !handles) {
        set_error("pr_shard_export_ipc: bad arguments");
        return PR_EINVAL;
    }
    if (g->shard_world < 1) {
        set_error("pr_shard_export_ipc: pr_graph_shard has not run");
        return PR_ESTATE;
    }
    cudaIpcMemHandle_t* h = reinterpret_cast<cudaIpcMemHandle_t*>(handles);
    PR_CUDA(cudaIpcGetMemHandle(&h[0], g->sy[0]));
    PR_CUDA(cudaIpcGetMemHandle(&h[1], g->sy[1]));
    return PR_OK;
}

int pr_shard_open_ipc(pr_graph* g, const void* handles, int32_t world) {
    g_err[0] = 0;
    if (!g || !handles) {
        set_error("pr_shard_open_ipc: bad arguments");
        return PR_EINVAL;
    }
    if (g->shard_world < 1 || world != g->shard_world) {
        set_error("pr_shard_open_ipc: world %d does not match the shard", world);
        return g->shard_world < 1 ? PR_ESTATE : PR_EINVAL;
    }
    clear_peers(g);
    const cudaIpcMemHandle_t* h = reinterpret_cast<const cudaIpcMemHandle_t*>(handles);
    std::vector<void*> y0(world, nullptr), y1(world, nullptr);
    for (int r = 0; r < world; ++r) {
        if (r == g->shard_rank) continue;
        PR_CUDA(cudaIpcOpenMemHandle(&y0[r], h[2 * r], cudaIpcMemLazyEnablePeerAccess));
        g->speer_ipc.push_back(y0[r]);
        PR_CUDA(cudaIpcOpenMemHandle(&y1[r], h[2 * r + 1], cudaIpcMemLazyEnablePeerAccess));
        g->speer_ipc.push_back(y1[r]);
    }
    return set_peers(g, (double* const*)y0.data(), (double* const*)y1.data(), world);
}

int pr_get_phase_plan(const pr_graph* g, int32_t reduced, int64_t* edge_bounds, int64_t* row_bounds, int32_t cap) {
    if (!g || !edge_bounds || !row_bounds) {
        set_error("pr_get_phase_plan: bad arguments");
        return -PR_EINVAL;
    }
    const View& v = reduced ? g->reduced : g->plain;
    if (v.phase_k < 1 || (reduced && !g->pre_done)) {
        set_error("pr_get_phase_plan: no PR_MODE_PHASED run on this view yet");
        return -PR_ESTATE;
    }
    if (cap < v.phase_k + 1) {
        set_error("pr_get_phase_plan: cap %d < %d", cap, v.phase_k + 1);
        return -PR_EINVAL;
    }
    for (int k = 0; k <= v.phase_k; ++k) {
        edge_bounds[k] = v.phase_eb[k];
        row_bounds[k] = v.phase_rb[k];
    }
    return v.phase_k;
}

int pr_get_shard_info(const pr_graph* g, pr_shard_info* out) {
    if (!g || !out) {
        set_error("pr_get_shard_info: bad arguments");
        return PR_EINVAL;
    }
    if (g->shard_world < 1) {
        set_error("pr_get_shard_info: pr_graph_shard has not run");
        return PR_ESTATE;
    }
    out->rank = g->shard_rank;
    out->world = g->shard_world;
    out->owned_vertices = g->shard_owned;
    out->rows = g->shard.nrows;
    out->edges = g->shard.nedges;
    out->chunk = g->shard_chunk;
    return PR_OK;
}

void pr_destroy(pr_graph* g) {
    if (!g) return;
    // the last call's work on its stream must be complete before its buffers
    // return to the pool (they are then freed, stream-ordered, on stream 0)
    if (g->fin_ev) {
        cudaEventSynchronize(g->fin_ev);
        cudaEventDestroy(g->fin_ev);
        g->fin_ev = nullptr;
    }
    cudaGetLastError();
    cudaStream_t s = 0;
    PhaseTimer pt(s, "destroy");
    clear_shard(g, s);
    dfree(g->row_ptr, s);
    dfree(g->col, s);
    dfree(g->outdeg, s);
    dfree(g->cidx, s);
    dfree(g->zlist, s);
    free_view(g->plain, s);
    free_view(g->reduced, s);
    dfree(g->rep, s);
    dfree(g->chain_src, s);
    dfree(g->chain_k, s);
    dfree(g->mem_vid, s);
    dfree(g->mem_src, s);
    dfree(g->mem_k, s);
    dfree(g->mem_srow, s);
    dfree(g->mem_info, s);
    dfree(g->mem_h, s);
    dfree(g->fold_rinfo, s);
    dfree(g->fold_w, s);
    dfree(g->fold_list, s);
    dfree(g->fold_crec, s);
    dfree(g->fold_xc, s);
    dfree(g->fold_rec, s);
    g->fold_n = 0;
    g->fold_nrec = 0;
    g->fold_ready = false;
    dfree(g->xr, s);
    dfree(g->xm, s);
    dfree(g->x, s);
    dfree(g->y[0], s);
    dfree(g->y[1], s);
    dfree(g->cta_partial, s);
    dfree(g->ab, s);
    dfree(g->hist, s);
    dfree(g->delta_log, s);
    dfree(g->st, s);
    pinned_state_free(g->st_host);
    delete g;
    pt.mark("all");
}

int pr_graph_info(const pr_graph* g, int64_t* n, int64_t* E, int64_t* n_members, int32_t* max_chain) {
    if (!g) {
        set_error("pr_graph_info: NULL graph");
        return PR_EINVAL;
    }
    if (n) *n = g->n;
    if (E) *E = g->E;
    if (n_members) *n_members = g->n_members;
    if (max_chain) *max_chain = g->max_chain;
    return PR_OK;
}

int pr_get_csr(const pr_graph* g, int64_t* row_ptr, int32_t* col_idx, int32_t* outdeg, void* stream) {
    if (!g) {
        set_error("pr_get_csr: NULL graph");
        return PR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (row_ptr) PR_CUDA(cudaMemcpyAsync(row_ptr, g->row_ptr, sizeof(int64_t) * (size_t)(g->n + 1), cudaMemcpyDefault, s));
    if (col_idx && g->E > 0)
        PR_CUDA(cudaMemcpyAsync(col_idx, g->col, sizeof(int32_t) * (size_t)g->E, cudaMemcpyDefault, s));
    if (outdeg) PR_CUDA(cudaMemcpyAsync(outdeg, g->outdeg, sizeof(int32_t) * (size_t)g->n, cudaMemcpyDefault, s));
    PR_CUDA(cudaStreamSynchronize(s));
    return PR_OK;
}

int pr_get_reductions(const pr_graph* g, int32_t* rep, int32_t* chain_src, int32_t* chain_k, void* stream) {
    if (!g) {
        set_error("pr_get_reductions: NULL graph");
        return PR_EINVAL;
    }
    if (!g->pre_done) {
        set_error("pr_get_reductions: pr_preprocess has not run");
        return PR_ESTATE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const size_t b = sizeof(int32_t) * (size_t)g->n;
    if (rep) PR_CUDA(cudaMemcpyAsync(rep, g->rep, b, cudaMemcpyDefault, s));
    if (chain_src) PR_CUDA(cudaMemcpyAsync(chain_src, g->chain_src, b, cudaMemcpyDefault, s));
    if (chain_k) PR_CUDA(cudaMemcpyAsync(chain_k, g->chain_k, b, cudaMemcpyDefault, s));
    PR_CUDA(cudaStreamSynchronize(s));
    return PR_OK;
}

int pr_get_delta_log(const pr_graph* g, double* log, int32_t cap) {
    if (!g || !log || cap < 0) {
        set_error("pr_get_delta_log: bad arguments");
        return -PR_EINVAL;
    }
    int32_t k = g->log_len;
    if (k > cap) k = cap;
    if (k > 0) PR_CUDA(cudaMemcpy(log, g->delta_log, sizeof(double) * 2 * (size_t)k, cudaMemcpyDeviceToHost));
    return k;
}

int pr_get_run_stats(const pr_graph* g, pr_run_stats* out) {
    if (!g || !out) {
        set_error("pr_get_run_stats: bad arguments");
        return PR_EINVAL;
    }
    *out = g->last;
    out->total_launches = g->launches;
    return PR_OK;
}

}  // extern "C"
