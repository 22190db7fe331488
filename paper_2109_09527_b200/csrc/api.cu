// api.cu -- the extern "C" boundary of libprgpu (include/prgpu.h).
// Validation, host/device pointer handling, graph lifetime.  All compute is
// in ingest.cu / preprocess.cu / iterate.cu.
#include <math.h>
#include <stdarg.h>
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

static int make_ctx(Ctx& ctx, void* stream) {
    ctx.stream = (cudaStream_t)stream;
    ctx.launches = 0;
    int dev = 0;
    PR_CUDA(cudaGetDevice(&dev));
    PR_CUDA(cudaDeviceGetAttribute(&ctx.num_sms, cudaDevAttrMultiProcessorCount, dev));
    // Keep freed stream-ordered memory in the device pool instead of returning
    // it to the OS at every synchronisation (re-mapping GBs per call otherwise
    // costs tens of ms per pr_graph_create).
    static bool pool_tuned[64] = {false};
    if (dev >= 0 && dev < 64 && !pool_tuned[dev]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
        pool_tuned[dev] = true;
    }
    return PR_OK;
}

static bool is_device_ptr(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace prgpu

using namespace prgpu;

extern "C" {
#pragma GCC visibility push(default)

const char* pr_last_error(void) { return g_err; }

int pr_graph_create(int64_t n, int64_t m, const int32_t* src, const int32_t* dst, void* stream, pr_graph** out) {
    g_err[0] = 0;
    if (!out) {
        set_error("pr_graph_create: out is NULL");
        return PR_EINVAL;
    }
    *out = nullptr;
    if (n < 1 || n > 2147483647LL) {
        set_error("pr_graph_create: n=%lld outside [1, 2^31-1]", (long long)n);
        return PR_EINVAL;
    }
    if (m < 0 || m > 2147483647LL) {
        set_error("pr_graph_create: m=%lld outside [0, 2^31-1]", (long long)m);
        return PR_EINVAL;
    }
    if (m > 0 && (!src || !dst)) {
        set_error("pr_graph_create: NULL edge array");
        return PR_EINVAL;
    }
    Ctx ctx;
    PR_TRY(make_ctx(ctx, stream));
    pr_graph* g = new (std::nothrow) pr_graph();
    if (!g) {
        set_error("pr_graph_create: host allocation failed");
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
        if (cudaMallocHost(&g->st_host, sizeof(DevState)) != cudaSuccess) {
            set_error("cudaMallocHost failed");
            rc = PR_ENOMEM;
            break;
        }
        if ((rc = dalloc(&g->st, 1, ctx.stream)) != PR_OK) break;
        const int32_t* s = src;
        const int32_t* t = dst;
        if (m > 0 && !is_device_ptr(src)) {  // host edge list: copy in (e2e path)
            if ((rc = dalloc(&dsrc, (size_t)m, ctx.stream)) != PR_OK) break;
            if (cudaMemcpyAsync(dsrc, src, sizeof(int32_t) * (size_t)m, cudaMemcpyDefault, ctx.stream) != cudaSuccess) {
                set_error("copy of src failed");
                rc = PR_ECUDA;
                break;
            }
            s = dsrc;
        }
        if (m > 0 && !is_device_ptr(dst)) {
            if ((rc = dalloc(&ddst, (size_t)m, ctx.stream)) != PR_OK) break;
            if (cudaMemcpyAsync(ddst, dst, sizeof(int32_t) * (size_t)m, cudaMemcpyDefault, ctx.stream) != cudaSuccess) {
                set_error("copy of dst failed");
                rc = PR_ECUDA;
                break;
            }
            t = ddst;
        }
        if ((rc = ingest(g, s, t, ctx)) != PR_OK) break;
        dfree(dsrc, ctx.stream);
        dfree(ddst, ctx.stream);
        if ((rc = build_relabel(g, ctx)) != PR_OK) break;
        if ((rc = build_view_tasks(g->plain, ctx)) != PR_OK) break;
        if ((rc = build_view_stream(g->plain, ctx, (int32_t)g->n_contrib, g->outdeg, g->cidx)) != PR_OK) break;
        if (cudaStreamSynchronize(ctx.stream) != cudaSuccess) {
            set_error("pr_graph_create: %s", cudaGetErrorString(cudaGetLastError()));
            rc = PR_ECUDA;
            break;
        }
    } while (0);
    g->launches += ctx.launches;
    if (rc != PR_OK) {
        dfree(dsrc, ctx.stream);
        dfree(ddst, ctx.stream);
        pr_destroy(g);
        return rc;
    }
    *out = g;
    return PR_OK;
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
    Ctx ctx;
    PR_TRY(make_ctx(ctx, stream));
    int rc = preprocess(g, flags, ctx);
    g->launches += ctx.launches;
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
    if (mode & ~(PR_MODE_ASYNC | PR_NORM_LINF | PR_USE_REDUCTIONS | PR_TIMING)) {
        set_error("pr_run: unknown mode bits 0x%x", mode);
        return PR_EINVAL;
    }
    if ((mode & PR_USE_REDUCTIONS) && !g->pre_done) {
        set_error("pr_run: PR_USE_REDUCTIONS before pr_preprocess");
        return PR_ESTATE;
    }
    Ctx ctx;
    PR_TRY(make_ctx(ctx, stream));
    int rc = run(g, d, threshold, max_iter, mode, ranks, ctx, iters_out, final_delta_out);
    g->launches += ctx.launches;
    g->last.total_launches = g->launches;
    return rc;
}

void pr_destroy(pr_graph* g) {
    if (!g) return;
    cudaStream_t s = 0;
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
    dfree(g->xr, s);
    dfree(g->xm, s);
    dfree(g->x, s);
    dfree(g->y[0], s);
    dfree(g->y[1], s);
    dfree(g->cta_partial, s);
    dfree(g->ab, s);
    dfree(g->delta_log, s);
    dfree(g->st, s);
    if (g->st_host) cudaFreeHost(g->st_host);
    delete g;
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
        return PR_EINVAL;
    }
    int32_t k = g->last.iterations;
    if (k > g->log_cap) k = g->log_cap;
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
