// iterate.cu -- the PageRank iteration: K-INIT, K-GATHER (+ fused contrib and
// fused Delta reduction), K-SCATTER (identical / chain members), loop control.
//
//   x_t(v) = (1-d)/n + d * sum_{u in in(v)} y_{t-1}(u),  y(u) = x(u)/outdeg(u)
// (Eq.(1) P:329-332 in the "sum, then times d" form of Alg.2; Q-F).
// Dangling u (outdeg 0) are never gathered (they have no out-edges), so they
// contribute nothing (Alg.2; Q-D).  Delta_t is summed over all n
// vertices (Q-R) and the loop runs "while err > threshold" (Q-S).
#include <math.h>
#include <stdlib.h>
#include <algorithm>
#include <vector>

#include "internal.h"
#include "primitives.cuh"
#include "rowengine.cuh"
#include "streamengine.cuh"

namespace prgpu {

// ----------------------------------------------------------------- policy --
// ASYNC: No-Sync in-place sweep (relaxed loads/stores of one contrib buffer).
// VID:   rows of the view are vid[r] (else row r is vertex r).
template <bool ASYNC, bool VID>
struct PRPolicy {
    using T = double;
    const double* y_in;
    double* y_out;
    double* x;
    const int32_t* od;
    const int32_t* cidx;
    const int32_t* vid;
    double c, d;
    uint64_t pol_last;

    __device__ __forceinline__ void begin() { pol_last = policy_evict_last(); }
    __device__ __forceinline__ double load(int32_t u) const {
        if (ASYNC) return ld_relaxed_f64(y_in + u);
        return ld_gather_tiered_f64(y_in + u, u < GT_L1_TIER, pol_last);
    }
    struct Pre {
        double xo;
        int32_t v, od, ci, pad;
    };
    Pre pre[2];
    // finalize operands, loaded before the row's gathers complete
    __device__ __forceinline__ Pre prefetch(int64_t r) const {
        Pre q;
        q.v = VID ? vid[r] : (int32_t)r;
        q.xo = x[q.v];
        q.od = od[q.v];
        q.ci = cidx[q.v];
        q.pad = 0;
        return q;
    }
    // rows r0 + lane and r0 + lane + 32 of a task with nr rows
    __device__ __forceinline__ void prefetch_rows(int64_t r0, int nr, int lane) {
        if (lane < nr) pre[0] = prefetch(r0 + lane);
        if (lane + 32 < nr) pre[1] = prefetch(r0 + lane + 32);
    }
    __device__ __forceinline__ const Pre& prefetched(int h) const { return pre[h]; }
    // x_t(v) = c + d*S, fused contrib y_t(v) = x_t(v)/outdeg(v), returns |x_t(v) - x_{t-1}(v)|.
    __device__ __forceinline__ double finalize(const Pre& q, double s) const {
        const double xn = __dadd_rn(c, __dmul_rn(d, s));
        x[q.v] = xn;
        if (q.od > 0) {
            const double y = xn / (double)q.od;
            if (ASYNC)
                st_relaxed_f64(y_out + q.ci, y);
            else
                y_out[q.ci] = y;
        }
        return fabs(xn - q.xo);
    }
};

// Reduction scratch: red[0..RED_W) sums, red[RED_W..2*RED_W) maxima, one per warp.
constexpr int RED_W = 32;

// Policy of the edge-stream gather (streamengine.cuh), synchronous sweeps.
// HOT: contribs [0, hot_n) are read from the CTA's shared-memory copy.
template <bool HOT>
struct StreamPolicy {
    using T = double;
    static constexpr bool kHot = HOT;
    const double* y_in;
    double* sums;
    const double* hot;
    int32_t hot_n;
    uint64_t pol_last;

    __device__ __forceinline__ double load(int32_t u) const {
        if (HOT && u < hot_n) return hot[u];
        return ld_gather_tiered_f64(y_in + u, u < SE_L1_TIER, pol_last);
    }
    __device__ __forceinline__ void emit(int64_t r, double s) const { sums[r] = s; }
    __device__ __forceinline__ void prep(int64_t, uint32_t) {}
    __device__ __forceinline__ void emit_at(int, int64_t r, double s) const { sums[r] = s; }
    __device__ __forceinline__ void emit_first(int64_t r, double s) const { sums[r] = s; }
};

// One segment pass of a source-blocked view (blocked.cu): gathers come from
// one L2-resident slice of y; S_seg(r) is added to the parent row's sum.
struct AccumPolicy {
    using T = double;
    static constexpr bool kHot = false;
    const double* y_in;
    double* sums;
    const int32_t* map;  // sub-view row -> parent view row
    const double* hot;
    int32_t hot_n;
    uint64_t pol_last;

    // the slice is re-read ~20x per pass: keep it in L2 against the streams
    // of col, flags, parent ids and the sums updates (evict_first / default)
    __device__ __forceinline__ double load(int32_t u) const {
        double r;
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(y_in + u), "l"(pol_last));
        return r;
    }
    // S(parent) += S_seg as a fire-and-forget red.add: each parent row gets
    // at most one per pass and passes are serial launches, so the additions
    // happen in segment order (deterministic).  The parent ids of a step's
    // closures are prefetched by prep() before the gathers are consumed.
    int32_t m_first;
    int32_t m[SE_V];
    __device__ __forceinline__ static void red_add(double* p, double v) {
#ifdef PRGPU_RED_EVICT_FIRST
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
#else
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
#endif
    }
    __device__ __forceinline__ void prep(int64_t base, uint32_t f) {
        if (f) m_first = __ldg(map + base);
#pragma unroll
        for (int j = 0; j < SE_V; ++j)
            if (f & (1u << j)) m[j] = __ldg(map + base + __popc(f & ((1u << j) - 1)));
    }
    __device__ __forceinline__ void emit(int64_t r, double s) const { red_add(sums + map[r], s); }
    __device__ __forceinline__ void emit_at(int j, int64_t, double s) const { red_add(sums + m[j], s); }
    __device__ __forceinline__ void emit_first(int64_t, double s) const { red_add(sums + m_first, s); }
};

struct IterArgs {
    DevState* st;
    double* cta_partial;        // (L1, Linf) per CTA: gather CTAs, scatter CTAs, zero-in CTAs
    int64_t gather_ctas;
    int64_t scatter_ctas;
    int64_t zero_ctas;          // > 0 only in the first sweep
    const double* hub_delta;    // of the gather view
    int64_t nhubs;
    double* delta_log;
    // sharded run: the last CTA writes this rank's (L1, Linf) here (the tail
    // of its exchanged chunk) instead of taking the stop decision; with peer
    // buffers (pr_shard_set_peers) also at peer_y[q] + shard_off of every peer
    double* shard_out = nullptr;
    double* const* peer_y = nullptr;
    int npeer = 0;
    int64_t shard_off = 0;
};

// The stop test on a sweep's (L1, Linf): iteration count, delta log, done /
// status ("while err > threshold", P:454 / BASELINE L1; max_iter S:176).
__device__ void stop_test(const IterArgs& ia, double l1, double li) {
    DevState* st = ia.st;
    const int it = st->iters + 1;
    st->iters = it;
    st->l1 = l1;
    st->linf = li;
    if (it <= st->log_cap) {
        ia.delta_log[2 * (it - 1)] = l1;
        ia.delta_log[2 * (it - 1) + 1] = li;
    }
    const double dn = st->norm_linf ? li : l1;
    if (dn <= st->tau) {
        st->done = 1;
        st->status = PR_OK;
    } else if (it >= st->max_iter) {
        st->done = 1;
        st->status = PR_NOT_CONVERGED;
    }
}

// Deterministic fixed-order reduction over all CTA partials and hub deltas,
// then the stop test; executed by the last CTA of the iteration.
__device__ void global_finalize(const IterArgs& ia, double* red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __threadfence();
    double s = 0.0, mx = 0.0;
    const int64_t nc = ia.gather_ctas + ia.scatter_ctas + ia.zero_ctas;
    for (int64_t i = tid; i < nc; i += blockDim.x) {
        s += __ldcg(ia.cta_partial + 2 * i);
        mx = fmax(mx, __ldcg(ia.cta_partial + 2 * i + 1));
    }
    for (int64_t i = tid; i < ia.nhubs; i += blockDim.x) {
        double v = __ldcg(ia.hub_delta + i);
        s += v;
        mx = fmax(mx, v);
    }
    s = warp_sum(s);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __syncthreads();
    if (lane == 0) {
        red[warp] = s;
        red[RED_W + warp] = mx;
    }
    __syncthreads();
    if (tid == 0) {
        double l1 = 0.0, li = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            l1 += red[w];
            li = fmax(li, red[RED_W + w]);
        }
        DevState* st = ia.st;
        if (ia.shard_out) {
            ia.shard_out[0] = l1;
            ia.shard_out[1] = li;
            for (int q = 0; q < ia.npeer; ++q) {
                ia.peer_y[q][ia.shard_off] = l1;
                ia.peer_y[q][ia.shard_off + 1] = li;
            }
        } else {
            stop_test(ia, l1, li);
        }
        st->ticket_gather = 0u;
        st->ticket_scatter = 0u;
        __threadfence();
    }
}

__device__ __forceinline__ void block_delta(double l1, double linf, double* red, double* out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    l1 = warp_sum(l1);
#pragma unroll
    for (int o = 16; o; o >>= 1) linf = fmax(linf, __shfl_xor_sync(0xffffffffu, linf, o));
    __syncthreads();
    if (lane == 0) {
        red[warp] = l1;
        red[RED_W + warp] = linf;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += red[w];
            b = fmax(b, red[RED_W + w]);
        }
        out[0] = a;
        out[1] = b;
    }
}

template <bool ASYNC, bool VID>
__global__ void __launch_bounds__(GT_NT, GT_MIN_CTAS)
    k_gather(PRPolicy<ASYNC, VID> p, EngineArgs a, IterArgs ia, int finalize) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    EngineSmem& sm = *reinterpret_cast<EngineSmem*>(smem_raw);
    if (ia.st->done) return;
    p.begin();
    double l1 = 0.0, linf = 0.0;
    engine_run(p, a, sm, l1, linf);
    block_delta(l1, linf, sm.red, ia.cta_partial + 2 * blockIdx.x);
    if (!finalize) return;
    if (threadIdx.x == 0) {
        __threadfence();
        uint32_t t = atomicAdd(&ia.st->ticket_gather, 1u);
        sm.flag = (t == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (sm.flag) global_finalize(ia, sm.red);
}

// K-GATHER, edge-stream form: S(r) of every row of the view into sums[r].
// One CTA of SE_NT threads per SM; no Delta here (K-FINALIZE computes it).
template <class P>
__global__ void __launch_bounds__(SE_NT, 1) k_stream(P p, StreamArgs a, const DevState* st) {
    extern __shared__ __align__(16) double hot_smem[];
    pdl_wait();
    pdl_trigger();
    if (st->done) return;
    p.pol_last = policy_evict_last();
    if (P::kHot) {
        const double2* src = reinterpret_cast<const double2*>(p.y_in);
        double2* dst = reinterpret_cast<double2*>(hot_smem);
        for (int i = threadIdx.x; i < (p.hot_n >> 1); i += blockDim.x) dst[i] = __ldcg(src + i);
        if ((p.hot_n & 1) && threadIdx.x == 0) hot_smem[p.hot_n - 1] = __ldcg(p.y_in + p.hot_n - 1);
        p.hot = hot_smem;
        __syncthreads();
    }
    stream_run(p, a);
}

// K-GATHER with dynamically handed-out spans (PRGPU_DYN_SPAN; a finer span
// layout of the view, DESIGN.md §9 "Tail of the gather").
template <class P>
__global__ void __launch_bounds__(SE_NT, 1) k_stream_dyn(P p, StreamArgs a, const DevState* st) {
    extern __shared__ __align__(16) double hot_smem[];
    pdl_wait();
    pdl_trigger();
    if (st->done) return;
    p.pol_last = policy_evict_last();
    if (P::kHot) {
        const double2* src = reinterpret_cast<const double2*>(p.y_in);
        double2* dst = reinterpret_cast<double2*>(hot_smem);
        for (int i = threadIdx.x; i < (p.hot_n >> 1); i += blockDim.x) dst[i] = __ldcg(src + i);
        if ((p.hot_n & 1) && threadIdx.x == 0) hot_smem[p.hot_n - 1] = __ldcg(p.y_in + p.hot_n - 1);
        p.hot = hot_smem;
        __syncthreads();
    }
    stream_run_dyn(p, a);
}

// K-FINALIZE (sync sweeps): for every row r of the view
//   x_t(v) = c + d*S(r)  (Eq.(1) in the "sum, then times d" form; Q-F),
//   y_t(v) = x_t(v)/outdeg(v) into the next contrib buffer (fused contrib),
// and, in reduced mode, every member m with source row q and distance k:
//   x_t(m) = alpha_k + beta_k * (c + d*S(q))     ((0,1): exact copy; Q-C)
// (c + d*S(q) is bit-identical to x_t of the source).  |x_t - x_{t-1}| of all
// of them feeds the fixed-order Delta reduction and the stop test (a7).
struct FinArgs {
    const double* sums;
    int64_t nrows;
    const int2* rinfo;     // (outdeg, contrib slot) per row
    double* xr;            // x of the rows, row order
    const int32_t* msrow;
    const int32_t* mk;
    const int2* minfo;     // (outdeg, contrib slot) per member
    double* xm;            // x of the members, member order
    int64_t nm;
    const double* ab;
    double* y_out;
    double c, d;
    // loop perforation (PR_PERFORATE, Alg.5): mark rows whose change
    // this sweep is 0 < |delta| < tau_f (fz[r] = 1, else 0) and count them
    uint8_t* fz = nullptr;
    double tau_f = 0.0;
    unsigned long long* nfz = nullptr;
    // PR_MODE_PHASED: rows [row0, nrows) only, Delta partials at CTA index
    // part_off + blockIdx.x, and the stop test only in the sweep's last phase
    int64_t row0 = 0;
    int64_t part_off = 0;
    int last = 1;
    // sharded run with peer buffers: every new contrib is also stored into
    // the same slot of each peer's buffer (the all-gather fused into K-FINALIZE)
    double* const* peer_y = nullptr;
    int npeer = 0;
    uint32_t* dyn_reset = nullptr;  // the gather's span counter, zeroed for the next sweep
};

// Rows are visited grid-stride (all CTAs sweep the row space together, which
// keeps the TLB working set small) in batches of FIN_U rows per thread whose
// loads are all issued before any store.  Every access is coalesced except the
// contrib store y[slot]; x is kept in row / member order (xr, xm) during the
// sweeps and written back to vertex order once, by k_unpermute.
constexpr int FIN_U = 4;

__global__ void __launch_bounds__(GT_NT) k_finalize(FinArgs f, IterArgs ia) {
    __shared__ double red[2 * RED_W];
    __shared__ int flag;
    pdl_wait();
    pdl_trigger();
    if (f.dyn_reset && blockIdx.x == 0 && threadIdx.x == 0) *f.dyn_reset = 0u;  // the gather has completed
    if (ia.st->done) return;
    double l1 = 0.0, linf = 0.0;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const double* __restrict__ sums = f.sums;
    double* __restrict__ xr = f.xr;
    double* __restrict__ y = f.y_out;
    uint32_t nfrozen = 0;
    for (int64_t r0 = f.row0 + t0; r0 < f.nrows; r0 += FIN_U * T) {
        double S[FIN_U], xo[FIN_U];
        int2 inf[FIN_U];
#pragma unroll
        for (int u = 0; u < FIN_U; ++u) {
            const int64_t r = r0 + u * T;
            if (r < f.nrows) {
                S[u] = __ldcs(sums + r);
                xo[u] = xr[r];
                inf[u] = __ldg(f.rinfo + r);
            }
        }
#pragma unroll
        for (int u = 0; u < FIN_U; ++u) {
            const int64_t r = r0 + u * T;
            if (r < f.nrows) {
                const double xn = __dadd_rn(f.c, __dmul_rn(f.d, S[u]));
                xr[r] = xn;
                if (inf[u].x > 0) {
                    const double yv = xn / (double)inf[u].x;
                    y[inf[u].y] = yv;
                    for (int q = 0; q < f.npeer; ++q) f.peer_y[q][inf[u].y] = yv;
                }
                const double dl = fabs(xn - xo[u]);
                l1 += dl;
                linf = fmax(linf, dl);
                if (f.fz) {
                    const bool frz = dl != 0.0 && dl < f.tau_f;
                    f.fz[r] = frz ? 1 : 0;
                    nfrozen += frz;
                }
            }
        }
    }
    if (f.fz) {
        nfrozen = warp_sum(nfrozen);
        if ((threadIdx.x & 31) == 0 && nfrozen) atomicAdd(f.nfz, (unsigned long long)nfrozen);
    }
    double* __restrict__ xm = f.xm;
    for (int64_t i0 = t0; i0 < f.nm; i0 += FIN_U * T) {
        double S[FIN_U], xo[FIN_U];
        int32_t k[FIN_U];
        int2 inf[FIN_U];
#pragma unroll
        for (int u = 0; u < FIN_U; ++u) {
            const int64_t i = i0 + u * T;
            if (i < f.nm) {
                k[u] = __ldg(f.mk + i);
                S[u] = sums[__ldg(f.msrow + i)];
                xo[u] = xm[i];
                inf[u] = __ldg(f.minfo + i);
            }
        }
#pragma unroll
        for (int u = 0; u < FIN_U; ++u) {
            const int64_t i = i0 + u * T;
            if (i < f.nm) {
                const double xs = __dadd_rn(f.c, __dmul_rn(f.d, S[u]));
                const double xn = __dadd_rn(f.ab[2 * k[u]], __dmul_rn(f.ab[2 * k[u] + 1], xs));
                xm[i] = xn;
                if (inf[u].x > 0) y[inf[u].y] = xn / (double)inf[u].x;
                const double dl = fabs(xn - xo[u]);
                l1 += dl;
                linf = fmax(linf, dl);
            }
        }
    }
    block_delta(l1, linf, red, ia.cta_partial + 2 * (f.part_off + blockIdx.x));
    if (!f.last) return;
    if (threadIdx.x == 0) {
        __threadfence();
        uint32_t t = atomicAdd(&ia.st->ticket_gather, 1u);
        flag = (t == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (flag) global_finalize(ia, red);
}

// Sync stream path: x in vertex order from the row / member ordered state.
__global__ void k_unpermute(const double* __restrict__ xr, const int32_t* __restrict__ vid, int64_t nrows,
                            const double* __restrict__ xm, const int32_t* __restrict__ mvid, int64_t nm,
                            double* __restrict__ x) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += T) x[vid ? vid[r] : r] = xr[r];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nm; i += T) x[mvid[i]] = xm[i];
}

__global__ void k_fill_f64(double* __restrict__ a, int64_t cnt, double v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}

// Members (reduced mode): x_t(m) = alpha_k + beta_k * x_t(src), with
// (alpha_0, beta_0) = (0, 1) an exact copy for identical members and
// alpha_{k+1} = c + d alpha_k, beta_{k+1} = d beta_k for chain members at
// distance k from their head (Q-C).  Runs after the gather of the same sweep.
template <bool ASYNC>
__global__ void __launch_bounds__(GT_NT) k_scatter(const int32_t* __restrict__ mvid, const int32_t* __restrict__ msrc,
                                                   const int32_t* __restrict__ mk, int64_t nm, int64_t per_cta,
                                                   const double* __restrict__ ab, double* x, double* y_out,
                                                   const int32_t* __restrict__ od, const int32_t* __restrict__ cidx,
                                                   IterArgs ia) {
    __shared__ double red[2 * RED_W];
    __shared__ int flag;
    if (ia.st->done) return;
    const int64_t b = (int64_t)blockIdx.x * per_cta;
    const int64_t e = min(nm, b + per_cta);
    double l1 = 0.0, linf = 0.0;
    for (int64_t i = b + threadIdx.x; i < e; i += GT_NT) {
        const int32_t v = mvid[i], s = msrc[i], k = mk[i];
        const double xs = x[s];
        const double xn = __dadd_rn(ab[2 * k], __dmul_rn(ab[2 * k + 1], xs));
        const double xo = x[v];
        x[v] = xn;
        const int32_t o = od[v];
        if (o > 0) {
            const double y = xn / (double)o;
            if (ASYNC)
                st_relaxed_f64(y_out + cidx[v], y);
            else
                y_out[cidx[v]] = y;
        }
        const double dl = fabs(xn - xo);
        l1 += dl;
        linf = fmax(linf, dl);
    }
    block_delta(l1, linf, red, ia.cta_partial + 2 * (ia.gather_ctas + blockIdx.x));
    if (threadIdx.x == 0) {
        __threadfence();
        uint32_t t = atomicAdd(&ia.st->ticket_scatter, 1u);
        flag = (t == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (flag) global_finalize(ia, red);
}

// First sweep for the vertices of in-degree 0: Eq.(1) with an empty sum gives
// x_t = (1-d)/n = c for every t >= 1, so they are written here once (x and
// the contrib slot of y_out) and contribute |c - 1/n| to Delta_1 only; from
// sweep 2 on their Delta is exactly 0 and no kernel touches them.
__global__ void __launch_bounds__(GT_NT) k_zero(const int32_t* __restrict__ zl, int64_t nz, int64_t per_cta, double c,
                                                double* x, double* y_out, const int32_t* __restrict__ od,
                                                const int32_t* __restrict__ cidx, double* partial) {
    // grid-stride, 4 vertices per thread with all loads issued first (the
    // old x is read too: it is 1/n from k_init, but Delta_1 must be measured)
    (void)per_cta;
    __shared__ double red[2 * RED_W];
    double l1 = 0.0, linf = 0.0;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nz; i0 += 4 * T) {
        int32_t v[4], o[4], ci[4];
        double xo[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = i0 + u * T < nz ? __ldg(zl + i0 + u * T) : -1;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (v[u] >= 0) {
                xo[u] = x[v[u]];
                o[u] = __ldg(od + v[u]);
                ci[u] = __ldg(cidx + v[u]);
            }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (v[u] >= 0) {
                x[v[u]] = c;
                if (o[u] > 0) y_out[ci[u]] = c / (double)o[u];
                const double dl = fabs(c - xo[u]);
                l1 += dl;
                linf = fmax(linf, dl);
            }
    }
    block_delta(l1, linf, red, partial + 2 * blockIdx.x);
}

// Sync mode: after sweep 1 also store the constant contribs of the in-degree-0
// vertices into the other ping-pong buffer (read by sweep 3, 5, ...).
__global__ void k_zero_y(const int32_t* __restrict__ zl, int64_t nz, double c, double* y,
                         const int32_t* __restrict__ od, const int32_t* __restrict__ cidx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nz; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = zl[i];
        const int32_t o = od[v];
        if (o > 0) y[cidx[v]] = c / (double)o;
    }
}

// Sharded run with peer buffers: the constant contribs of this rank's
// in-degree-0 vertices into every peer's buffer (sweep 1).
__global__ void k_peer_zero(const int32_t* __restrict__ zl, int64_t nz, double c, const int32_t* __restrict__ od,
                            const int32_t* __restrict__ cidx, double* const* peers, int np) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nz; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = zl[i];
        const int32_t o = od[v];
        if (o > 0)
            for (int q = 0; q < np; ++q) peers[q][cidx[v]] = c / (double)o;
    }
}

// x_0 = 1/n (Alg.1), y_0 = x_0/outdeg for sources.
__global__ void k_init(double* __restrict__ x, double* __restrict__ y, const int32_t* __restrict__ od,
                       const int32_t* __restrict__ cidx, int64_t n, double x0) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        x[v] = x0;
        const int32_t o = od[v];
        if (o > 0) y[cidx[v]] = x0 / (double)o;
    }
}

// ------------------------------------------------------ No-Sync --
// Persistent barrier-free kernel (Alg.3 "No-Sync"): every CTA sweeps
// its own static share of the row tasks (and of the members) in place --
// gathers read whatever contribs are visible (relaxed loads), every row's x and
// y are written at once (relaxed stores) -- and after each local sweep publishes
// its (L1, L-inf) delta; it stops when the sum (L1) / max (L-inf) over the
// deltas all CTAs last published is <= tau ("thread-level convergence",
// P:416-418, with the per-iteration reset of Q-E).  No grid barrier: a CTA
// never waits for another one.  Grid = resident CTAs only (a CTA must not wait
// for an unscheduled CTA's first delta, which starts at +big).
struct NoSyncArgs {
    double* err;        // [2 * grid] (L1, Linf) of each CTA's last local sweep
    int32_t* iters;     // [grid] local sweeps of each CTA, over all launches
    int norm_linf;
    double tau;
    int32_t max_local;  // local sweeps allowed in this launch
    const int32_t* mvid;
    const int32_t* msrc;
    const int32_t* mk;
    int64_t nm;
    int64_t mper;
    const double* ab;
    double* x;
    double* y;
    const int32_t* od;
    const int32_t* cidx;
};

template <bool VID>
__global__ void __launch_bounds__(GT_NT, GT_MIN_CTAS) k_nosync(PRPolicy<true, VID> p, EngineArgs a, NoSyncArgs na) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    EngineSmem& sm = *reinterpret_cast<EngineSmem*>(smem_raw);
    __shared__ double res[2];
    p.begin();
    const int64_t mb = (int64_t)blockIdx.x * na.mper;
    const int64_t me = min(na.nm, mb + na.mper);
    uint32_t kbase = 0;  // per-warp mbarrier phase count across local sweeps (lane 0 uses it)
    for (int it = 1;; ++it) {
        double l1 = 0.0, linf = 0.0;
        engine_run(p, a, sm, l1, linf, &kbase);
        for (int64_t i = mb + threadIdx.x; i < me; i += blockDim.x) {  // members (Q-C)
            const int32_t v = na.mvid[i], sv = na.msrc[i], k = na.mk[i];
            const double xs = ld_relaxed_f64(na.x + sv);
            const double xn = __dadd_rn(na.ab[2 * k], __dmul_rn(na.ab[2 * k + 1], xs));
            const double xo = na.x[v];
            st_relaxed_f64(na.x + v, xn);
            const int32_t o = na.od[v];
            if (o > 0) st_relaxed_f64(na.y + na.cidx[v], xn / (double)o);
            const double dl = fabs(xn - xo);
            l1 += dl;
            linf = fmax(linf, dl);
        }
        block_delta(l1, linf, sm.red, res);
        if (threadIdx.x == 0) {
            st_relaxed_f64(na.err + 2 * blockIdx.x, res[0]);
            st_relaxed_f64(na.err + 2 * blockIdx.x + 1, res[1]);
            na.iters[blockIdx.x] += 1;
            double tot = 0.0, mx = 0.0;
            for (unsigned c = 0; c < gridDim.x; ++c) {
                tot += ld_relaxed_f64(na.err + 2 * c);
                mx = fmax(mx, ld_relaxed_f64(na.err + 2 * c + 1));
            }
            const double nv = na.norm_linf ? mx : tot;
            sm.flag = (nv <= na.tau || it >= na.max_local) ? 1 : 0;
        }
        __syncthreads();
        if (sm.flag) break;
    }
}

// Certificate of a No-Sync result: ||F(x) - x|| of the ORIGINAL system, with
// S(r) from one synchronous edge-stream gather of the plain view over the
// current contribs (F(x) = c + d*M*x, Eq.(1)); ||x - x*||_1 <= ||F(x)-x||_1/(1-d).
// (Sum by atomics: not bit-reproducible in its last digits; it is a check.)
template <bool VID>
__global__ void k_residual(const double* __restrict__ sums, int64_t nrows, const int32_t* __restrict__ vid,
                           const double* __restrict__ x, double c, double d, double* out) {
    __shared__ double red[2 * RED_W];
    __shared__ double res[2];
    double l1 = 0.0, linf = 0.0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = VID ? vid[r] : (int32_t)r;
        const double dl = fabs(__dadd_rn(c, __dmul_rn(d, sums[r])) - x[v]);
        l1 += dl;
        linf = fmax(linf, dl);
    }
    block_delta(l1, linf, red, res);
    if (threadIdx.x == 0) {
        atomicAdd(out, res[0]);
        atomicMax(reinterpret_cast<unsigned long long*>(out + 1), (unsigned long long)__double_as_longlong(res[1]));
    }
}

// ------------------------------------------- in-place edge-stream sweeps --
// Async (PR_MODE_ASYNC, one launch per sweep) and No-Sync (PR_MODE_NOSYNC,
// persistent) on the edge-stream engine: the finalize is fused into the
// gather, so a row's new contrib is visible to the gathers that follow in the
// same sweep (Alg.3's in-place pr(u) <- tmp; Q-Y).  Contribs are
// read with relaxed loads, except the hottest slots [0, hot_n), which every
// CTA copies into shared memory at the start of each (local) sweep -- a
// snapshot of values that were visible then, which No-Sync allows.  x is kept
// in row / member order (xr, xm; unpermuted at the end); the finalize operands
// of a step's row closures ((outdeg, slot), x_old) are prefetched right after
// the row-start scan, before the gathers are consumed.
// SYNC = true: the same fused finalize for a SYNCHRONOUS sweep (K-GATHER +
// K-FINALIZE in one launch): contribs are read from y_in (not written in this
// sweep: shared-memory hot tier, L1 tier, .nc loads) and the new contribs go to
// the other ping-pong buffer y.
template <bool SYNC>
struct InPlacePolicyT {
    using T = double;
    static constexpr bool kHot = true;
    const double* y_in;   // async: == y, relaxed loads; sync: the previous sweep's contribs
    double* y;            // async: relaxed stores; sync: plain stores into the next buffer
    const double* hot;
    int32_t hot_n;
    uint64_t pol_last;
    double* xr;
    const int2* rinfo;
    double c, d;
    double l1, linf;
    int2 inf_f;
    double xo_f;
    int2 inf[SE_V];
    double xo[SE_V];

    __device__ __forceinline__ double load(int32_t u) const {
        if (u < hot_n) return hot[u];
        if (SYNC) return ld_gather_tiered_f64(y_in + u, u < SE_L1_TIER, pol_last);
        return ld_relaxed_f64(y_in + u);
    }
    __device__ __forceinline__ void prep(int64_t base, uint32_t f) {
        if (f) {
            inf_f = __ldg(rinfo + base);
            xo_f = ld_relaxed_f64(xr + base);
        }
#pragma unroll
        for (int j = 0; j < SE_V; ++j)
            if (f & (1u << j)) {
                const int64_t r = base + __popc(f & ((1u << j) - 1));
                inf[j] = __ldg(rinfo + r);
                xo[j] = ld_relaxed_f64(xr + r);
            }
    }
    __device__ __forceinline__ void fin(int64_t r, double s, int2 q, double xold) {
        const double xn = __dadd_rn(c, __dmul_rn(d, s));
        st_relaxed_f64(xr + r, xn);
        if (q.x > 0) {
            if (SYNC)
                y[q.y] = xn / (double)q.x;
            else
                st_relaxed_f64(y + q.y, xn / (double)q.x);
        }
        const double dl = fabs(xn - xold);
        l1 += dl;
        linf = fmax(linf, dl);
    }
    __device__ __forceinline__ void emit(int64_t r, double s) { fin(r, s, __ldg(rinfo + r), ld_relaxed_f64(xr + r)); }
    __device__ __forceinline__ void emit_at(int j, int64_t r, double s) { fin(r, s, inf[j], xo[j]); }
    __device__ __forceinline__ void emit_first(int64_t r, double s) { fin(r, s, inf_f, xo_f); }
};

using InPlacePolicy = InPlacePolicyT<false>;

// Members of a reduced view, in place: x(m) = alpha_k + beta_k * x(src) with
// x(src) as currently visible (its row in xr), fused contrib, Delta.
struct MemArgs {
    const int32_t* msrow;
    const int32_t* mk;
    const int2* minfo;
    double* xm;
    int64_t nm;
    int64_t mper;
    const double* ab;
};

__device__ __forceinline__ void members_inplace(InPlacePolicy& p, const MemArgs& ma) {
    const int64_t mb = (int64_t)blockIdx.x * ma.mper;
    const int64_t me = min(ma.nm, mb + ma.mper);
    for (int64_t i = mb + threadIdx.x; i < me; i += blockDim.x) {
        const int32_t k = ma.mk[i];
        const double xs = ld_relaxed_f64(p.xr + ma.msrow[i]);
        const double xn = __dadd_rn(ma.ab[2 * k], __dmul_rn(ma.ab[2 * k + 1], xs));
        const double xo = ma.xm[i];
        ma.xm[i] = xn;
        const int2 q = ma.minfo[i];
        if (q.x > 0) st_relaxed_f64(p.y + q.y, xn / (double)q.x);
        const double dl = fabs(xn - xo);
        p.l1 += dl;
        p.linf = fmax(p.linf, dl);
    }
}

__device__ __forceinline__ void refresh_hot(InPlacePolicy& p, double* hot_smem) {
    for (int i = threadIdx.x; i < p.hot_n; i += blockDim.x) hot_smem[i] = ld_relaxed_f64(p.y_in + i);
    p.hot = hot_smem;
    __syncthreads();
}

// One async sweep (launch level).
__global__ void __launch_bounds__(SE_NT_IP, 1)
    k_stream_async(InPlacePolicy p, StreamArgs a, MemArgs ma, IterArgs ia) {
    extern __shared__ __align__(16) double hot_smem[];
    __shared__ double red[2 * RED_W];
    __shared__ int flag;
    if (ia.st->done) return;
    p.pol_last = 0;
    refresh_hot(p, hot_smem);
    p.l1 = 0.0;
    p.linf = 0.0;
    stream_run(p, a);
    members_inplace(p, ma);
    block_delta(p.l1, p.linf, red, ia.cta_partial + 2 * blockIdx.x);
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t t = atomicAdd(&ia.st->ticket_gather, 1u);
        flag = (t == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (flag) global_finalize(ia, red);
}

// One synchronous sweep with the finalize fused into the gather (rows only;
// in reduced mode k_members_sync follows and runs the global reduction).
__global__ void __launch_bounds__(SE_NT_IP, 1)
    k_stream_fused(InPlacePolicyT<true> p, StreamArgs a, IterArgs ia, int finalize) {
    extern __shared__ __align__(16) double hot_smem[];
    __shared__ double red[2 * RED_W];
    __shared__ int flag;
    if (ia.st->done) return;
    p.pol_last = policy_evict_last();
    {
        const double2* src = reinterpret_cast<const double2*>(p.y_in);
        double2* dst = reinterpret_cast<double2*>(hot_smem);
        for (int i = threadIdx.x; i < (p.hot_n >> 1); i += blockDim.x) dst[i] = __ldcg(src + i);
        if ((p.hot_n & 1) && threadIdx.x == 0) hot_smem[p.hot_n - 1] = __ldcg(p.y_in + p.hot_n - 1);
        p.hot = hot_smem;
        __syncthreads();
    }
    p.l1 = 0.0;
    p.linf = 0.0;
    stream_run(p, a);
    block_delta(p.l1, p.linf, red, ia.cta_partial + 2 * blockIdx.x);
    if (!finalize) return;
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t t = atomicAdd(&ia.st->ticket_gather, 1u);
        flag = (t == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (flag) global_finalize(ia, red);
}

// Members after a fused synchronous sweep: x(m) = alpha_k + beta_k * x_t(src)
// (the source's new value, row order), next contrib, Delta; the last CTA runs
// the global reduction over the gather and member partials.
__global__ void __launch_bounds__(GT_NT) k_members_sync(MemArgs ma, const double* __restrict__ xr, double* y_out,
                                                        IterArgs ia) {
    __shared__ double red[2 * RED_W];
    __shared__ int flag;
    if (ia.st->done) return;
    double l1 = 0.0, linf = 0.0;
    const int64_t mb = (int64_t)blockIdx.x * ma.mper;
    const int64_t me = min(ma.nm, mb + ma.mper);
    for (int64_t i = mb + threadIdx.x; i < me; i += blockDim.x) {
        const int32_t k = ma.mk[i];
        const double xs = __ldcg(xr + ma.msrow[i]);
        const double xn = __dadd_rn(ma.ab[2 * k], __dmul_rn(ma.ab[2 * k + 1], xs));
        const double xo = ma.xm[i];
        ma.xm[i] = xn;
        const int2 q = ma.minfo[i];
        if (q.x > 0) y_out[q.y] = xn / (double)q.x;
        const double dl = fabs(xn - xo);
        l1 += dl;
        linf = fmax(linf, dl);
    }
    block_delta(l1, linf, red, ia.cta_partial + 2 * (ia.gather_ctas + blockIdx.x));
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t t = atomicAdd(&ia.st->ticket_scatter, 1u);
        flag = (t == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (flag) global_finalize(ia, red);
}

// Persistent No-Sync on the edge-stream engine (see k_nosync for the protocol).
__global__ void __launch_bounds__(SE_NT_IP, 1) k_nosync_stream(InPlacePolicy p, StreamArgs a, MemArgs ma, NoSyncArgs na) {
    extern __shared__ __align__(16) double hot_smem[];
    __shared__ double red[2 * RED_W];
    __shared__ double res[2];
    __shared__ int flag;
    p.pol_last = 0;
    for (int it = 1;; ++it) {
        refresh_hot(p, hot_smem);
        p.l1 = 0.0;
        p.linf = 0.0;
        stream_run(p, a);
        members_inplace(p, ma);
        block_delta(p.l1, p.linf, red, res);
        if (threadIdx.x == 0) {
            st_relaxed_f64(na.err + 2 * blockIdx.x, res[0]);
            st_relaxed_f64(na.err + 2 * blockIdx.x + 1, res[1]);
            na.iters[blockIdx.x] += 1;
            double tot = 0.0, mx = 0.0;
            for (unsigned cc = 0; cc < gridDim.x; ++cc) {
                tot += ld_relaxed_f64(na.err + 2 * cc);
                mx = fmax(mx, ld_relaxed_f64(na.err + 2 * cc + 1));
            }
            const double nv = na.norm_linf ? mx : tot;
            flag = (nv <= na.tau || it >= na.max_local) ? 1 : 0;
        }
        __syncthreads();
        if (flag) break;
    }
}

// ------------------------------------------------------------------- host --

struct GatherCfg {
    bool dyn = false;  // sync: spans handed out dynamically (PRGPU_DYN_SPAN)
    bool stream;  // sync: edge-stream gather + K-FINALIZE; async (or PRGPU_ENGINE=tasks): row-task engine
    bool inplace; // async on the edge-stream engine (k_stream_async; PRGPU_ENGINE=tasks: row-task engine)
    bool fused;   // sync stream sweep with the finalize fused into the gather (k_stream_fused)
    bool async, vid;
    int hot_n;
    size_t smem;
    int grid;
    int nt;
};

template <bool ASYNC, bool VID>
static int launch_tasks_t(Ctx& ctx, const View& v, const double* y_in, double* y_out, double* x, pr_graph* g,
                          double c, double d, const IterArgs& ia, const GatherCfg& gc, int finalize) {
    PRPolicy<ASYNC, VID> p{y_in, y_out, x, g->outdeg, g->cidx, v.vid, c, d, 0, {}};
    EngineArgs a{v.tasks, v.ntasks, v.hubs, v.row_ptr, v.col, v.hub_partial, v.hub_delta, v.hub_ticket};
    PR_LAUNCH(ctx, (k_gather<ASYNC, VID>), gc.grid, GT_NT, gc.smem, p, a, ia, finalize);
    return PR_OK;
}

// PRGPU_TRACE=<file>: every edge-stream gather launch records per-warp
// (start, end) globaltimer stamps; run() writes the last launch's to <file>
// (diagnostics of the tail; tools/trace_tail.py).
static unsigned long long* g_trace = nullptr;
static int64_t g_trace_n = 0;
static const char* trace_path() {
    const char* e = getenv("PRGPU_TRACE");
    return (e && *e) ? e : nullptr;
}

static int launch_gather(Ctx& ctx, const View& v, const double* y_in, double* y_out, double* x, pr_graph* g,
                         double c, double d, const IterArgs& ia, const GatherCfg& gc, int finalize,
                         int64_t span_lo = 0, int64_t span_hi = -1) {
    if (gc.stream) {
        auto args = [&](const View& w) {
            StreamArgs a{w.col,  (const uint8_t*)w.sflags, w.step_row, w.nsteps, w.span_steps, w.nspans, w.bin,
                         w.bout, w.b_row, w.b_s0, w.b_s1, w.part_in, w.part_out, w.bticket};
            if (&w == &v) {
                a.span_lo = span_lo;
                a.span_hi = span_hi;
            }
            a.trace = g_trace;
            return a;
        };
        if (v.nseg > 0) {  // source-blocked: S = 0, then one accumulating pass per slot segment
            PR_CUDA(cudaMemsetAsync(v.sums, 0, sizeof(double) * (size_t)v.nrows, ctx.stream));
            for (int q = 0; q < v.nseg; ++q) {
                const View& sv = v.seg[q];
                if (sv.nspans == 0) continue;
                AccumPolicy p{y_in, v.sums, sv.vid, nullptr, 0, 0, 0, {}};
                PR_LAUNCH_PDL(ctx, k_stream<AccumPolicy>, gc.grid, gc.nt, 0, p, args(sv), (const DevState*)g->st);
            }
        } else if (gc.dyn && v.dynv && span_hi < 0 && span_lo == 0) {  // dynamic spans on the finer layout
            StreamArgs a = args(*v.dynv);
            a.dyn_ctr = v.dyn_ctr;
            if (gc.hot_n > 0) {
                StreamPolicy<true> p{y_in, v.sums, nullptr, gc.hot_n, 0};
                PR_LAUNCH_PDL(ctx, k_stream_dyn<StreamPolicy<true>>, gc.grid, gc.nt, gc.smem, p, a,
                              (const DevState*)g->st);
            } else {
                StreamPolicy<false> p{y_in, v.sums, nullptr, 0, 0};
                PR_LAUNCH_PDL(ctx, k_stream_dyn<StreamPolicy<false>>, gc.grid, gc.nt, gc.smem, p, a,
                              (const DevState*)g->st);
            }
        } else if (gc.hot_n > 0) {
            StreamPolicy<true> p{y_in, v.sums, nullptr, gc.hot_n, 0};
            PR_LAUNCH_PDL(ctx, k_stream<StreamPolicy<true>>, gc.grid, gc.nt, gc.smem, p, args(v),
                          (const DevState*)g->st);
        } else {
            StreamPolicy<false> p{y_in, v.sums, nullptr, 0, 0};
            PR_LAUNCH_PDL(ctx, k_stream<StreamPolicy<false>>, gc.grid, gc.nt, gc.smem, p, args(v),
                          (const DevState*)g->st);
        }
        return PR_OK;
    }
    if (gc.async)
        return gc.vid ? launch_tasks_t<true, true>(ctx, v, y_in, y_out, x, g, c, d, ia, gc, finalize)
                      : launch_tasks_t<true, false>(ctx, v, y_in, y_out, x, g, c, d, ia, gc, finalize);
    return gc.vid ? launch_tasks_t<false, true>(ctx, v, y_in, y_out, x, g, c, d, ia, gc, finalize)
                  : launch_tasks_t<false, false>(ctx, v, y_in, y_out, x, g, c, d, ia, gc, finalize);
}

static const void* gather_fn(const GatherCfg& gc) {
    if (gc.stream)
        return gc.hot_n > 0 ? (const void*)k_stream<StreamPolicy<true>> : (const void*)k_stream<StreamPolicy<false>>;
    if (gc.async) return gc.vid ? (const void*)k_gather<true, true> : (const void*)k_gather<true, false>;
    return gc.vid ? (const void*)k_gather<false, true> : (const void*)k_gather<false, false>;
}

static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}

// Kernel variant, dynamic shared memory and persistent grid (all resident CTAs).
static int gather_config(Ctx& ctx, const View& v, pr_graph* g, bool async, GatherCfg* gc, bool force_stream = false) {
    const char* eng = getenv("PRGPU_ENGINE");
    const bool tasks = eng && eng[0] == 't';
    gc->stream = !async && (force_stream || !tasks);
    gc->inplace = async && !tasks;
    gc->fused = gc->stream && !force_stream && v.nseg == 0 && env_int("PRGPU_FUSED", 0) != 0;
    gc->async = async;
    gc->vid = v.vid != nullptr;
    gc->hot_n = 0;
    if (gc->fused) {
        int hot = env_int("PRGPU_HOT", SE_HOT_MAX);
        hot = std::max(0, std::min<int>(std::min(hot, SE_HOT_MAX), (int)g->n_contrib));
        gc->hot_n = hot;
        gc->smem = (size_t)hot * sizeof(double);
        gc->nt = SE_NT_IP;
    } else if (gc->inplace) {
        int hot = env_int("PRGPU_HOT", SE_HOT_IP);
        hot = std::max(0, std::min<int>(std::min(hot, SE_HOT_MAX), (int)g->n_contrib));
        gc->hot_n = hot;
        gc->smem = (size_t)hot * sizeof(double);
        gc->nt = SE_NT_IP;
    } else if (gc->stream) {
        int hot = v.nseg > 0 ? 0 : env_int("PRGPU_HOT", SE_HOT_MAX);
        if (hot > SE_HOT_MAX) hot = SE_HOT_MAX;
        if (hot > g->n_contrib) hot = (int)g->n_contrib;
        if (hot < 0) hot = 0;
        gc->hot_n = hot;
        gc->smem = (size_t)hot * sizeof(double);
        gc->nt = SE_NT;
    } else {
        gc->smem = sizeof(EngineSmem);
        gc->nt = GT_NT;
    }
    const void* fn = gc->fused ? (const void*)k_stream_fused
                               : (gc->inplace ? (const void*)k_stream_async : gather_fn(*gc));
    PR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gc->smem));
    int per_sm = 0;
    PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, gc->nt, gc->smem));
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)ctx.num_sms * per_sm;
    const int wpc = gc->nt / 32;
    int64_t units = (gc->stream || gc->inplace) ? v.nspans : v.ntasks;
    if (gc->stream && v.nseg > 0) {
        units = 0;
        for (int q = 0; q < v.nseg; ++q) units = std::max<int64_t>(units, v.seg[q].nspans);
    }
    int64_t ctas_needed = (units + wpc - 1) / wpc;
    if (grid > ctas_needed) grid = ctas_needed;
    if (grid < 1) grid = 1;
    gc->grid = (int)grid;
    return PR_OK;
}

static int run_nosync(pr_graph* g, double d, double tau, int32_t max_iter, uint32_t mode, double* ranks, Ctx& ctx,
                      int32_t* iters_out, double* delta_out);
static int run_perforated(pr_graph* g, double d, double tau, int32_t max_iter, uint32_t mode, double* ranks,
                          Ctx& ctx, int32_t* iters_out, double* delta_out);

// The row-task engine's tables are built on first use (async / No-Sync with
// PRGPU_ENGINE=tasks); an aliased reduced view shares the plain view's.
static bool tasks_engine_requested() {
    const char* e = getenv("PRGPU_ENGINE");
    return e && e[0] == 't';
}
static int ensure_tasks(pr_graph* g, bool reduced, Ctx& ctx) {
    View& v = reduced ? g->reduced : g->plain;
    if (v.alias) {
        PR_TRY(ensure_tasks(g, false, ctx));
        g->reduced = g->plain;
        g->reduced.alias = true;
        return PR_OK;
    }
    if (!v.tasks && v.nrows > 0) PR_TRY(build_view_tasks(v, ctx));
    return PR_OK;
}

// PR_MODE_PHASED: the phase plan of a view (K contiguous span ranges; the
// rows each phase finalizes are those whose last edge lies in its spans, so a
// row crossing a phase boundary is summed by the later phase's ticket winner).
__global__ void k_phase_rows(const int32_t* __restrict__ step_row, const uint8_t* __restrict__ flags8,
                             int64_t span_steps, int64_t nspans, int K, int64_t nrows, int64_t* __restrict__ rb) {
    const int k = threadIdx.x;
    if (k > K) return;
    if (k == 0) {
        rb[0] = 0;
    } else if (k == K) {
        rb[K] = nrows;
    } else {  // the row containing the phase's first edge (it ends in this phase or later)
        const int64_t st = (int64_t)k * nspans / K * span_steps;
        rb[k] = (int64_t)step_row[st] - ((flags8[st * 32] & 1) ? 0 : 1);
    }
}

static int phase_plan(pr_graph* g, bool reduced, Ctx& ctx, int* K_out) {
    View& v = reduced ? g->reduced : g->plain;
    if (v.alias) {  // an aliased reduced view shares the plain view's plan
        PR_TRY(phase_plan(g, false, ctx, K_out));
        g->reduced = g->plain;
        g->reduced.alias = true;
        return PR_OK;
    }
    // default: 8 phases when every phase still gives each resident warp a span
    // of >= 24 steps (R-MAT-24: 8); fewer on small graphs, where the ~15-20 us
    // a phase costs (two launches, ramp and tail) outweighs the saved sweeps
    const int64_t warps = (int64_t)ctx.num_sms * (SE_NT / 32);
    int K = env_int("PRGPU_PHASES", (int)std::min<int64_t>(8, v.nsteps / (warps * 24)));
    if (K < 1) K = 1;
    if (K > SE_MAX_PHASES) K = SE_MAX_PHASES;
    if (v.nseg > 0 || v.nspans == 0) K = 1;  // source-blocked views run one phase (an in-place Jacobi sweep)
    *K_out = K;
    if (K == 1) {
        if (v.phase_k != 1) {
            v.phase_rb[0] = 0;
            v.phase_rb[1] = v.nrows;
            v.phase_eb[0] = 0;
            v.phase_eb[1] = v.nedges;
            v.phase_k = 1;
        }
        return PR_OK;
    }
    PR_TRY(build_phase_view(v, ctx, K));
    const View& pv = *v.phv;
    if (v.phase_k == K) return PR_OK;
    int64_t* rb = nullptr;
    PR_TRY(dalloc(&rb, (size_t)K + 1, ctx.stream));
    PR_LAUNCH(ctx, k_phase_rows, 1, 128, 0, (const int32_t*)pv.step_row, (const uint8_t*)pv.sflags, pv.span_steps,
              pv.nspans, K, v.nrows, rb);
    PR_CUDA(cudaMemcpyAsync(v.phase_rb, rb, sizeof(int64_t) * (size_t)(K + 1), cudaMemcpyDeviceToHost, ctx.stream));
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    dfree(rb, ctx.stream);
    for (int k = 0; k <= K; ++k)
        v.phase_eb[k] = k == K ? v.nedges
                               : std::min<int64_t>(v.nedges, (int64_t)k * pv.nspans / K * pv.span_steps * SE_STEP);
    v.phase_k = K;
    return PR_OK;
}

// Boundary-row / hub tickets count the pieces of the current sweep.  A
// persistent No-Sync launch stops with CTAs at different sweeps, so tickets can
// be left mid-count; every run starts from zero.
static int reset_tickets(const View& v, cudaStream_t s) {
    if (v.bticket && v.nbound > 0) PR_CUDA(cudaMemsetAsync(v.bticket, 0, sizeof(uint32_t) * (size_t)v.nbound, s));
    if (v.hub_ticket && v.nhubs > 0) PR_CUDA(cudaMemsetAsync(v.hub_ticket, 0, sizeof(uint32_t) * (size_t)v.nhubs, s));
    for (int q = 0; q < v.nseg; ++q) PR_TRY(reset_tickets(v.seg[q], s));
    if (v.phv) PR_TRY(reset_tickets(*v.phv, s));
    if (v.dynv) {
        PR_TRY(reset_tickets(*v.dynv, s));
        PR_CUDA(cudaMemsetAsync(v.dyn_ctr, 0, sizeof(uint32_t), s));
    }
    return PR_OK;
}

// PRGPU_DYN_SPAN=F > 0: the sync gather hands out spans of F steps
// dynamically (built on first use; an aliased reduced view shares the plain
// view's).  0 / unset: static spans.
static int ensure_dyn(pr_graph* g, bool reduced, Ctx& ctx, int64_t F) {
    View& v = reduced ? g->reduced : g->plain;
    if (v.alias) {
        PR_TRY(ensure_dyn(g, false, ctx, F));
        g->reduced = g->plain;
        g->reduced.alias = true;
        return PR_OK;
    }
    if (v.nseg > 0 || v.nspans == 0) return PR_OK;
    return build_dyn_view(v, ctx, F);
}

int run(pr_graph* g, double d, double tau, int32_t max_iter, uint32_t mode, double* ranks, Ctx& ctx,
        int32_t* iters_out, double* delta_out) {
    if (tasks_engine_requested()) PR_TRY(ensure_tasks(g, (mode & PR_USE_REDUCTIONS) != 0, ctx));
    const int dyn_f = env_int("PRGPU_DYN_SPAN", 0);
    const bool dyn = dyn_f > 0 && !(mode & (PR_MODE_ASYNC | PR_MODE_NOSYNC | PR_PERFORATE | PR_MODE_PHASED));
    if (dyn) PR_TRY(ensure_dyn(g, (mode & PR_USE_REDUCTIONS) != 0, ctx, dyn_f));
    PR_TRY(reset_tickets(g->plain, ctx.stream));
    if (g->pre_done) PR_TRY(reset_tickets(g->reduced, ctx.stream));
    if (mode & PR_MODE_NOSYNC) return run_nosync(g, d, tau, max_iter, mode, ranks, ctx, iters_out, delta_out);
    if (mode & PR_PERFORATE) return run_perforated(g, d, tau, max_iter, mode, ranks, ctx, iters_out, delta_out);
    cudaStream_t s = ctx.stream;
    const bool async = (mode & PR_MODE_ASYNC) != 0;
    const bool phased = (mode & PR_MODE_PHASED) != 0;
    const bool reduced = (mode & PR_USE_REDUCTIONS) != 0;
    const bool timing = (mode & PR_TIMING) != 0;
    // PR_TIMING brackets every tstride-th sweep's launches with events (each
    // event pair also blocks the programmatic launch overlap of its sweep)
    const int tstride = std::max(1, env_int("PRGPU_TIMING_STRIDE", 4));
    const int64_t n = g->n;
    const View& v = reduced ? g->reduced : g->plain;
    const int64_t nm = reduced ? g->n_members : 0;
    const int64_t launches0 = ctx.launches;

    // ranks on the device: iterate in place in the caller's buffer
    cudaPointerAttributes at{};
    bool ranks_dev = cudaPointerGetAttributes(&at, ranks) == cudaSuccess &&
                     (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    double* x = ranks;
    if (!ranks_dev) {
        if (!g->x) PR_TRY(dalloc(&g->x, (size_t)n, s));
        x = g->x;
    }
    // contrib slots [0, n_contrib) + slot n_contrib = +0.0, the pad of the stream engine
    const int64_t ny = g->n_contrib + 1;
    for (int b = 0; b < 2; ++b)
        if (!g->y[b]) {
            PR_TRY(dalloc(&g->y[b], (size_t)ny, s));
            PR_CUDA(cudaMemsetAsync(g->y[b] + g->n_contrib, 0, sizeof(double), s));
        }

    // phases of a sweep (PR_MODE_PHASED: K >= 1; else one); K > 1 gathers
    // through the view's finer-span copy
    int K = 1;
    if (phased) PR_TRY(phase_plan(g, reduced, ctx, &K));
    const View& gv = K > 1 ? *v.phv : v;
    GatherCfg gc;
    PR_TRY(gather_config(ctx, gv, g, async, &gc, phased));
    gc.dyn = dyn && v.dynv != nullptr && gc.stream && !gc.fused;
    if (gc.dyn) {
        PR_CUDA(cudaFuncSetAttribute(k_stream_dyn<StreamPolicy<true>>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)gc.smem));
        PR_CUDA(cudaFuncSetAttribute(k_stream_dyn<StreamPolicy<false>>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)gc.smem));
    }
    if (trace_path()) {
        const int64_t nwarps = (int64_t)gc.grid * (gc.nt / 32);
        if (g_trace_n < nwarps) {
            if (g_trace) cudaFree(g_trace);
            PR_CUDA(cudaMalloc(&g_trace, sizeof(unsigned long long) * 2 * (size_t)nwarps));
            g_trace_n = nwarps;
        }
        PR_CUDA(cudaMemsetAsync(g_trace, 0, sizeof(unsigned long long) * 2 * (size_t)g_trace_n, s));
    }
    const int64_t cap4 = (int64_t)ctx.num_sms * 4;
    // K-FINALIZE (stream path): fixed grid per phase, so each CTA's rows and
    // members (and hence its Delta partial) are a fixed set (deterministic)
    int64_t fgrid_k[SE_MAX_PHASES], foff_k[SE_MAX_PHASES];
    int64_t fgrid = 0;
    if (gc.stream) {
        for (int k = 0; k < K; ++k) {
            const int64_t rows = phased ? v.phase_rb[k + 1] - v.phase_rb[k] : v.nrows;
            const int64_t work = rows + (k == K - 1 ? nm : 0);
            fgrid_k[k] =
                std::min<int64_t>(std::max<int64_t>((work + GT_NT * FIN_U - 1) / (GT_NT * FIN_U), 1), cap4 * 2);
            foff_k[k] = fgrid;
            fgrid += fgrid_k[k];
        }
    }
    const int ggrid = (gc.stream && !gc.fused) ? (int)fgrid : gc.grid;  // CTAs writing Delta partials first
    int64_t sgrid = ((gc.fused || (!gc.stream && !gc.inplace)) && nm > 0) ? (nm + GT_NT * 4 - 1) / (GT_NT * 4) : 0;
    if (sgrid > cap4) sgrid = cap4;
    const int64_t sper = sgrid > 0 ? (nm + sgrid - 1) / sgrid : 0;
    const int64_t nz = g->nz;
    int64_t zgrid = nz > 0 ? (nz + GT_NT * 4 - 1) / (GT_NT * 4) : 0;
    if (zgrid > cap4) zgrid = cap4;
    const int64_t zper = zgrid > 0 ? (nz + zgrid - 1) / zgrid : 0;
    const int64_t need = 2 * ((int64_t)ggrid + sgrid + zgrid);
    if (g->partial_cap < need) {
        dfree(g->cta_partial, s);
        PR_TRY(dalloc(&g->cta_partial, (size_t)need, s));
        g->partial_cap = need;
    }
    const int log_cap = max_iter < 4096 ? max_iter : 4096;
    if (g->log_cap < log_cap) {
        dfree(g->delta_log, s);
        PR_TRY(dalloc(&g->delta_log, (size_t)(2 * log_cap), s));
        g->log_cap = log_cap;
    }
    const double c = (1.0 - d) / (double)n;
    if (reduced && nm > 0) {
        std::vector<double> ab(2 * ((size_t)g->max_chain + 1));
        ab[0] = 0.0;
        ab[1] = 1.0;
        for (int k = 1; k <= g->max_chain; ++k) {
            ab[2 * k] = c + d * ab[2 * (k - 1)];
            ab[2 * k + 1] = d * ab[2 * (k - 1) + 1];
        }
        dfree(g->ab, s);
        PR_TRY(dalloc(&g->ab, ab.size(), s));
        PR_CUDA(cudaMemcpyAsync(g->ab, ab.data(), ab.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    DevState* hs = g->st_host;
    *hs = DevState{};
    hs->max_iter = max_iter;
    hs->norm_linf = (mode & PR_NORM_LINF) ? 1 : 0;
    hs->tau = tau;
    hs->log_cap = log_cap;
    PR_CUDA(cudaMemcpyAsync(g->st, hs, sizeof(DevState), cudaMemcpyHostToDevice, s));
    PR_LAUNCH(ctx, k_init, (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx.num_sms * 16), 256, 0, x,
              g->y[0], (const int32_t*)g->outdeg, (const int32_t*)g->cidx, n, 1.0 / (double)n);

    const int64_t sctas = (reduced && (gc.fused || (!gc.stream && !gc.inplace))) ? sgrid : 0;
    IterArgs ia_rest{g->st,
                     g->cta_partial,
                     (int64_t)ggrid,
                     sctas,
                     0,
                     (gc.stream || gc.inplace) ? nullptr : v.hub_delta,
                     (gc.stream || gc.inplace) ? 0 : v.nhubs,
                     g->delta_log};
    IterArgs ia_first = ia_rest;
    ia_first.zero_ctas = zgrid;
    double* zero_partial = g->cta_partial + 2 * ((int64_t)ggrid + sctas);
    const bool gather_finalizes = (gc.fused || !gc.stream) && !(reduced && sgrid > 0);
    const StreamArgs sa{v.col,  (const uint8_t*)v.sflags, v.step_row, v.nsteps, v.span_steps, v.nspans, v.bin,
                        v.bout, v.b_row, v.b_s0, v.b_s1, v.part_in, v.part_out, v.bticket};
    const MemArgs ma{g->mem_srow, g->mem_k, g->mem_info, g->xm, nm, nm > 0 ? (nm + gc.grid - 1) / gc.grid : 0, g->ab};
    if (gc.stream || gc.inplace) {
        const int64_t need_xr = std::max<int64_t>(std::max(g->plain.nrows, g->reduced.nrows), 1);
        if (g->xr_cap < need_xr) {
            dfree(g->xr, s);
            PR_TRY(dalloc(&g->xr, (size_t)need_xr, s));
            g->xr_cap = need_xr;
        }
        if (g->n_members > 0 && !g->xm) PR_TRY(dalloc(&g->xm, (size_t)g->n_members, s));
        const unsigned fg = (unsigned)std::min<int64_t>((v.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
        PR_LAUNCH(ctx, k_fill_f64, fg, 256, 0, g->xr, v.nrows, 1.0 / (double)n);
        if (nm > 0) PR_LAUNCH(ctx, k_fill_f64, fg, 256, 0, g->xm, nm, 1.0 / (double)n);
    }
    FinArgs fa{v.sums, v.nrows, v.rinfo, g->xr, g->mem_srow, g->mem_k, g->mem_info, g->xm, nm, g->ab, nullptr, c, d};

    std::vector<cudaEvent_t> ev;
    double gather_ms = 0.0, scatter_ms = 0.0;
    int timed = 0;
    int host_syncs = 0;
    int64_t launched = 0;
    int batch = 8;
    int32_t prev_it = 0;
    double prev_dn = 0.0;
    while (true) {
        int nb = batch;
        if (launched + nb > max_iter) nb = (int)(max_iter - launched);
        if (timing && (int)ev.size() < 4 * nb) {
            size_t old = ev.size();
            ev.resize(4 * nb);
            for (size_t i = old; i < ev.size(); ++i) PR_CUDA(cudaEventCreate(&ev[i]));
        }
        for (int j = 0; j < nb; ++j) {
            const int64_t it = launched + j;
            const double* y_in = (async || phased) ? g->y[0] : g->y[it & 1];
            double* y_out = (async || phased) ? g->y[0] : g->y[(it + 1) & 1];
            const IterArgs& ia = it == 0 ? ia_first : ia_rest;
            if (it == 0 && zgrid > 0 && !phased)
                PR_LAUNCH(ctx, k_zero, (unsigned)zgrid, GT_NT, 0, (const int32_t*)g->zlist, nz, zper, c, x, y_out,
                          (const int32_t*)g->outdeg, (const int32_t*)g->cidx, zero_partial);
            if (timing && it % tstride == tstride - 1) PR_CUDA(cudaEventRecord(ev[4 * j], s));
            if (phased) {
                // in place, phase by phase: the gather of phase k reads the
                // contribs phases 0..k-1 of this sweep wrote (block Gauss-Seidel)
                for (int k = 0; k < K; ++k) {
                    PR_TRY(launch_gather(ctx, gv, y_in, y_out, x, g, c, d, ia, gc, 0, (int64_t)k * gv.nspans / K,
                                         (int64_t)(k + 1) * gv.nspans / K));
                    FinArgs f = fa;
                    f.y_out = y_out;
                    f.row0 = v.phase_rb[k];
                    f.nrows = v.phase_rb[k + 1];
                    f.nm = k == K - 1 ? nm : 0;
                    f.part_off = foff_k[k];
                    f.last = k == K - 1;
                    // in-degree-0 vertices (sweep 1) once every gather of the
                    // sweep has read their initial contribs, as in sync mode
                    if (it == 0 && zgrid > 0 && k == K - 1)
                        PR_LAUNCH(ctx, k_zero, (unsigned)zgrid, GT_NT, 0, (const int32_t*)g->zlist, nz, zper, c, x,
                                  y_out, (const int32_t*)g->outdeg, (const int32_t*)g->cidx, zero_partial);
                    PR_LAUNCH_PDL(ctx, k_finalize, (unsigned)fgrid_k[k], GT_NT, 0, f, ia);
                }
            } else if (gc.fused) {
                InPlacePolicyT<true> fp{};
                fp.y_in = y_in;
                fp.y = y_out;
                fp.hot_n = gc.hot_n;
                fp.xr = g->xr;
                fp.rinfo = v.rinfo;
                fp.c = c;
                fp.d = d;
                PR_LAUNCH(ctx, k_stream_fused, gc.grid, gc.nt, gc.smem, fp, sa, ia, gather_finalizes ? 1 : 0);
            } else             if (gc.inplace) {
                InPlacePolicy ip{};
                ip.y_in = g->y[0];
                ip.y = g->y[0];
                ip.hot_n = gc.hot_n;
                ip.xr = g->xr;
                ip.rinfo = v.rinfo;
                ip.c = c;
                ip.d = d;
                PR_LAUNCH(ctx, k_stream_async, gc.grid, gc.nt, gc.smem, ip, sa, ma, ia);
            } else {
                PR_TRY(launch_gather(ctx, v, y_in, y_out, x, g, c, d, ia, gc, gather_finalizes));
            }
            if (timing && it % tstride == tstride - 1) PR_CUDA(cudaEventRecord(ev[4 * j + 1], s));
            if (phased) {
                // the whole sweep is timed as gather_ms
            } else if (gc.fused) {
                if (!gather_finalizes) {
                    MemArgs mf{g->mem_srow, g->mem_k, g->mem_info, g->xm, nm, (nm + sgrid - 1) / sgrid, g->ab};
                    PR_LAUNCH(ctx, k_members_sync, (unsigned)sgrid, GT_NT, 0, mf, (const double*)g->xr, y_out, ia);
                }
            } else if (gc.stream) {
                FinArgs f = fa;
                f.y_out = y_out;
                if (gc.dyn) f.dyn_reset = v.dyn_ctr;
                PR_LAUNCH_PDL(ctx, k_finalize, (unsigned)fgrid, GT_NT, 0, f, ia);
            } else if (!gather_finalizes && !gc.inplace) {
                if (async)
                    PR_LAUNCH(ctx, k_scatter<true>, (unsigned)sgrid, GT_NT, 0, (const int32_t*)g->mem_vid,
                              (const int32_t*)g->mem_src, (const int32_t*)g->mem_k, nm, sper, (const double*)g->ab, x,
                              y_out, (const int32_t*)g->outdeg, (const int32_t*)g->cidx, ia);
                else
                    PR_LAUNCH(ctx, k_scatter<false>, (unsigned)sgrid, GT_NT, 0, (const int32_t*)g->mem_vid,
                              (const int32_t*)g->mem_src, (const int32_t*)g->mem_k, nm, sper, (const double*)g->ab, x,
                              y_out, (const int32_t*)g->outdeg, (const int32_t*)g->cidx, ia);
            }
            if (timing && it % tstride == tstride - 1) PR_CUDA(cudaEventRecord(ev[4 * j + 2], s));
            if (it == 0 && nz > 0 && !async && !phased)
                PR_LAUNCH(ctx, k_zero_y, (unsigned)std::min<int64_t>((nz + 255) / 256, (int64_t)ctx.num_sms * 8), 256,
                          0, (const int32_t*)g->zlist, nz, c, (double*)y_in, (const int32_t*)g->outdeg,
                          (const int32_t*)g->cidx);
        }
        PR_CUDA(cudaMemcpyAsync(hs, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        PR_CUDA(cudaStreamSynchronize(s));
        ++host_syncs;
        if (timing) {
            for (int j = 0; j < nb; ++j) {
                if (launched + j >= hs->iters) break;
                if ((launched + j) % tstride != tstride - 1) continue;
                float a = 0.f, b2 = 0.f;
                PR_CUDA(cudaEventElapsedTime(&a, ev[4 * j], ev[4 * j + 1]));
                PR_CUDA(cudaEventElapsedTime(&b2, ev[4 * j + 1], ev[4 * j + 2]));
                gather_ms += a;
                scatter_ms += b2;
                ++timed;
            }
        }
        launched += nb;
        if (hs->done || launched >= max_iter) break;
        // next batch: the sweeps a geometric fit of the last two batch-end
        // deltas predicts until the stop test, + 1 (capped at 64; doubling
        // while there is no fit), so few no-op sweeps are launched past it
        {
            const double dn = hs->norm_linf ? hs->linf : hs->l1;
            int next = batch < 64 ? batch * 2 : 64;
            if (prev_it > 0 && hs->iters > prev_it && prev_dn > 0.0 && dn > 0.0 && dn < prev_dn && tau > 0.0) {
                const double rho = pow(dn / prev_dn, 1.0 / (double)(hs->iters - prev_it));
                const double rem = log(tau / dn) / log(rho);
                if (rem > 0.0 && rem < 64.0) next = (int)ceil(rem) + 1;
            }
            prev_it = hs->iters;
            prev_dn = dn;
            batch = next;
        }
    }
    for (auto e : ev) cudaEventDestroy(e);
    if (const char* tp = trace_path()) {
        std::vector<unsigned long long> ht(2 * (size_t)g_trace_n);
        PR_CUDA(cudaMemcpyAsync(ht.data(), g_trace, sizeof(unsigned long long) * ht.size(), cudaMemcpyDeviceToHost, s));
        PR_CUDA(cudaStreamSynchronize(s));
        if (FILE* f = fopen(tp, "w")) {
            for (int64_t i = 0; i < g_trace_n; ++i) fprintf(f, "%llu %llu\n", ht[2 * i], ht[2 * i + 1]);
            fclose(f);
        }
    }
    if (gc.stream || gc.inplace) {
        const unsigned ug = (unsigned)std::min<int64_t>((v.nrows + nm + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
        PR_LAUNCH(ctx, k_unpermute, ug, 256, 0, (const double*)g->xr, (const int32_t*)v.vid, v.nrows,
                  (const double*)g->xm, (const int32_t*)g->mem_vid, nm, x);
    }
    if (!ranks_dev) {
        PR_CUDA(cudaMemcpyAsync(ranks, x, sizeof(double) * (size_t)n, cudaMemcpyDefault, s));
        PR_CUDA(cudaStreamSynchronize(s));
        ++host_syncs;
    }
    pr_run_stats& rs = g->last;
    g->log_len = std::min<int32_t>(hs->iters, g->log_cap);
    rs.iterations = hs->iters;
    rs.status = hs->status;
    rs.delta_l1 = hs->l1;
    rs.delta_linf = hs->linf;
    rs.run_launches = ctx.launches - launches0;
    rs.host_syncs = host_syncs;
    rs.timed_iterations = timed;
    rs.gather_ms = gather_ms;
    rs.scatter_ms = scatter_ms;
    rs.gather_rows = v.nrows;
    rs.gather_edges = v.nedges;
    rs.scatter_members = nm;
    rs.n_contrib = g->n_contrib;
    rs.n_tasks = v.ntasks;
    rs.edges_gathered = v.nedges * (int64_t)hs->iters;
    rs.phases = K;
    if (iters_out) *iters_out = hs->iters;
    if (delta_out) *delta_out = (mode & PR_NORM_LINF) ? hs->linf : hs->l1;
    return hs->status;
}

// -------------------------------------------------------- sharded (f3) --
// After the exchange: refresh the hot copy y[0, H) from the chunks, and sum
// every rank's (L1, Linf) (the tail of its chunk) in rank order -- identical on
// every rank -- for the stop test.
__global__ void k_shard_combine(IterArgs ia, double* __restrict__ y, const int32_t* __restrict__ hot_src, int64_t H,
                                int world, int64_t chunk, int stop) {
    if (ia.st->done) return;  // (block 0 may set it below; a late hot copy is then unused)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < H; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = y[hot_src[i]];
    if (blockIdx.x != 0 || threadIdx.x != 0 || !stop) return;
    const double* ch = y + H;
    double l1 = 0.0, li = 0.0;
    for (int r = 0; r < world; ++r) {
        l1 += ch[(int64_t)r * chunk + chunk - 2];
        li = fmax(li, ch[(int64_t)r * chunk + chunk - 1]);
    }
    stop_test(ia, l1, li);
}

// ranks[v] = x[v] for the vertices this rank owns, 0.0 elsewhere
__global__ void k_shard_ranks(const double* __restrict__ x, const int32_t* __restrict__ owner, int rank, int64_t n,
                              double* __restrict__ ranks) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        ranks[v] = owner[v] == rank ? x[v] : 0.0;
}

int run_sharded(pr_graph* g, double d, double tau, int32_t max_iter, uint32_t mode, double* ranks, Ctx& ctx,
                pr_exchange_fn exchange, void* exchange_ctx, int32_t* iters_out, double* delta_out) {
    cudaStream_t s = ctx.stream;
    const bool timing = (mode & PR_TIMING) != 0;
    // PR_TIMING brackets every tstride-th sweep's launches with events (each
    // event pair also blocks the programmatic launch overlap of its sweep)
    const int tstride = std::max(1, env_int("PRGPU_TIMING_STRIDE", 4));
    const int64_t n = g->n;
    const View& v = g->shard;
    const int world = g->shard_world, rank = g->shard_rank;
    const int64_t chunk = g->shard_chunk, H = g->shard_hot;
    const bool peers = g->speer_dev != nullptr && world > 1;
    const int64_t launches0 = ctx.launches;
    PR_TRY(reset_tickets(v, s));
    if (!g->x) PR_TRY(dalloc(&g->x, (size_t)n, s));
    double* x = g->x;

    GatherCfg gc;
    PR_TRY(gather_config(ctx, v, g, false, &gc, true));
    if (gc.hot_n > H) {  // the shared-memory tier reads the hot copy only
        gc.hot_n = (int)H;
        gc.smem = (size_t)gc.hot_n * sizeof(double);
    }
    const int64_t cap4 = (int64_t)ctx.num_sms * 4;
    const int64_t fgrid =
        std::min<int64_t>(std::max<int64_t>((v.nrows + GT_NT * FIN_U - 1) / (GT_NT * FIN_U), 1), cap4 * 2);
    const int64_t nz = g->snz;
    int64_t zgrid = nz > 0 ? std::min<int64_t>((nz + GT_NT * 4 - 1) / (GT_NT * 4), cap4) : 0;
    const int64_t zper = zgrid > 0 ? (nz + zgrid - 1) / zgrid : 0;
    const int64_t need = 2 * (fgrid + zgrid);
    if (g->partial_cap < need) {
        dfree(g->cta_partial, s);
        PR_TRY(dalloc(&g->cta_partial, (size_t)need, s));
        g->partial_cap = need;
    }
    const int log_cap = max_iter < 4096 ? max_iter : 4096;
    if (g->log_cap < log_cap) {
        dfree(g->delta_log, s);
        PR_TRY(dalloc(&g->delta_log, (size_t)(2 * log_cap), s));
        g->log_cap = log_cap;
    }
    const int64_t need_xr = std::max<int64_t>(std::max(g->plain.nrows, v.nrows), 1);
    if (g->xr_cap < need_xr) {
        dfree(g->xr, s);
        PR_TRY(dalloc(&g->xr, (size_t)need_xr, s));
        g->xr_cap = need_xr;
    }
    const double c = (1.0 - d) / (double)n;
    DevState* hs = g->st_host;
    *hs = DevState{};
    hs->max_iter = max_iter;
    hs->norm_linf = (mode & PR_NORM_LINF) ? 1 : 0;
    hs->tau = tau;
    hs->log_cap = log_cap;
    PR_CUDA(cudaMemcpyAsync(g->st, hs, sizeof(DevState), cudaMemcpyHostToDevice, s));
    // x0 = 1/n and y0 of EVERY contrib slot (the replica starts complete)
    PR_LAUNCH(ctx, k_init, (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx.num_sms * 16), 256, 0, x,
              g->sy[0], (const int32_t*)g->outdeg, (const int32_t*)g->scidx, n, 1.0 / (double)n);
    IterArgs ia0{g->st, g->cta_partial, 0, 0, 0, nullptr, 0, g->delta_log};
    const unsigned cgrid = (unsigned)std::max<int64_t>(1, (H + 255) / 256);
    PR_LAUNCH(ctx, k_shard_combine, cgrid, 256, 0, ia0, g->sy[0], (const int32_t*)g->shot_src, H, world, chunk, 0);
    // peer buffers: no rank may store into another's buffers before that rank
    // has initialised them (sweep 1's stores would be overwritten)
    if (peers && exchange(exchange_ctx, nullptr, chunk, world, (void*)s) != 0) {
        set_error("pr_run_sharded: the exchange callback failed before sweep 1");
        return PR_ECUDA;
    }
    const unsigned fg = (unsigned)std::min<int64_t>((v.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
    PR_LAUNCH(ctx, k_fill_f64, fg, 256, 0, g->xr, v.nrows, 1.0 / (double)n);
    IterArgs ia_rest{g->st, g->cta_partial, fgrid, 0, 0, nullptr, 0, g->delta_log};
    IterArgs ia_first = ia_rest;
    ia_first.zero_ctas = zgrid;
    double* zero_partial = g->cta_partial + 2 * fgrid;
    FinArgs fa{v.sums, v.nrows, v.rinfo, g->xr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, nullptr, c, d};

    std::vector<cudaEvent_t> ev;
    double gather_ms = 0.0, scatter_ms = 0.0;
    int timed = 0, host_syncs = 0;
    int64_t launched = 0;
    int batch = 8;
    while (true) {
        int nb = batch;
        if (launched + nb > max_iter) nb = (int)(max_iter - launched);
        if (timing && (int)ev.size() < 4 * nb) {
            size_t old = ev.size();
            ev.resize(4 * nb);
            for (size_t i = old; i < ev.size(); ++i) PR_CUDA(cudaEventCreate(&ev[i]));
        }
        for (int j = 0; j < nb; ++j) {
            const int64_t it = launched + j;
            double* y_in = g->sy[it & 1];
            double* y_out = g->sy[(it + 1) & 1];
            IterArgs ia = it == 0 ? ia_first : ia_rest;
            ia.shard_out = y_out + H + (int64_t)rank * chunk + chunk - 2;
            double* const* pout = peers ? g->speer_dev + ((it + 1) & 1) * (world - 1) : nullptr;
            ia.peer_y = pout;
            ia.npeer = peers ? world - 1 : 0;
            ia.shard_off = H + (int64_t)rank * chunk + chunk - 2;
            if (it == 0 && zgrid > 0)
                PR_LAUNCH(ctx, k_zero, (unsigned)zgrid, GT_NT, 0, (const int32_t*)g->szlist, nz, zper, c, x, y_out,
                          (const int32_t*)g->outdeg, (const int32_t*)g->scidx, zero_partial);
            if (timing && it % tstride == tstride - 1) PR_CUDA(cudaEventRecord(ev[4 * j], s));
            if (v.nrows > 0) PR_TRY(launch_gather(ctx, v, y_in, y_out, x, g, c, d, ia, gc, 0));
            if (timing && it % tstride == tstride - 1) PR_CUDA(cudaEventRecord(ev[4 * j + 1], s));
            FinArgs f = fa;
            f.y_out = y_out;
            f.peer_y = pout;
            f.npeer = peers ? world - 1 : 0;
            PR_LAUNCH_PDL(ctx, k_finalize, (unsigned)fgrid, GT_NT, 0, f, ia);
            if (timing && it % tstride == tstride - 1) PR_CUDA(cudaEventRecord(ev[4 * j + 2], s));
            if (it == 0 && nz > 0) {
                const unsigned zg = (unsigned)std::min<int64_t>((nz + 255) / 256, (int64_t)ctx.num_sms * 8);
                PR_LAUNCH(ctx, k_zero_y, zg, 256, 0, (const int32_t*)g->szlist, nz, c, y_in,
                          (const int32_t*)g->outdeg, (const int32_t*)g->scidx);
                if (peers)  // peers' sweep-1 output buffer (their gathers read the other one)
                    PR_LAUNCH(ctx, k_peer_zero, zg, 256, 0, (const int32_t*)g->szlist, nz, c,
                              (const int32_t*)g->outdeg, (const int32_t*)g->scidx, pout, world - 1);
            }
            // ...and their other buffer only in sweep 2 (their sweep-2 output):
            // in sweep 1 it is what they gather from
            if (it == 1 && nz > 0 && peers)
                PR_LAUNCH(ctx, k_peer_zero, (unsigned)std::min<int64_t>((nz + 255) / 256, (int64_t)ctx.num_sms * 8),
                          256, 0, (const int32_t*)g->szlist, nz, c, (const int32_t*)g->outdeg,
                          (const int32_t*)g->scidx, pout, world - 1);
            // all-gather of the chunks (or, with peer buffers, only the
            // cross-rank barrier: every rank's stores landed in every buffer)
            if (exchange(exchange_ctx, peers ? nullptr : y_out + H, chunk, world, (void*)s) != 0) {
                set_error("pr_run_sharded: the exchange callback failed at sweep %lld", (long long)it + 1);
                for (auto e : ev) cudaEventDestroy(e);
                return PR_ECUDA;
            }
            PR_LAUNCH(ctx, k_shard_combine, cgrid, 256, 0, ia, y_out, (const int32_t*)g->shot_src, H, world, chunk, 1);
        }
        PR_CUDA(cudaMemcpyAsync(hs, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        PR_CUDA(cudaStreamSynchronize(s));
        ++host_syncs;
        if (timing) {
            for (int j = 0; j < nb; ++j) {
                if (launched + j >= hs->iters) break;
                if ((launched + j) % tstride != tstride - 1) continue;
                float a = 0.f, b2 = 0.f;
                PR_CUDA(cudaEventElapsedTime(&a, ev[4 * j], ev[4 * j + 1]));
                PR_CUDA(cudaEventElapsedTime(&b2, ev[4 * j + 1], ev[4 * j + 2]));
                gather_ms += a;
                scatter_ms += b2;
                ++timed;
            }
        }
        launched += nb;
        if (hs->done || launched >= max_iter) break;
        if (batch < 64) batch *= 2;
    }
    for (auto e : ev) cudaEventDestroy(e);
    const unsigned ug = (unsigned)std::min<int64_t>((v.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
    PR_LAUNCH(ctx, k_unpermute, ug, 256, 0, (const double*)g->xr, (const int32_t*)v.vid, v.nrows,
              (const double*)nullptr, (const int32_t*)nullptr, (int64_t)0, x);
    PR_LAUNCH(ctx, k_shard_ranks, (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx.num_sms * 16), 256, 0,
              (const double*)x, (const int32_t*)g->sowner, rank, n, ranks);
    PR_CUDA(cudaStreamSynchronize(s));
    pr_run_stats& rs = g->last;
    rs = pr_run_stats{};
    rs.phases = 1;
    g->log_len = std::min<int32_t>(hs->iters, g->log_cap);
    rs.iterations = hs->iters;
    rs.status = hs->status;
    rs.delta_l1 = hs->l1;
    rs.delta_linf = hs->linf;
    rs.run_launches = ctx.launches - launches0;
    rs.host_syncs = host_syncs;
    rs.timed_iterations = timed;
    rs.gather_ms = gather_ms;
    rs.scatter_ms = scatter_ms;
    rs.gather_rows = v.nrows;
    rs.gather_edges = v.nedges;
    rs.n_contrib = g->n_contrib;
    rs.edges_gathered = v.nedges * (int64_t)hs->iters;
    if (iters_out) *iters_out = hs->iters;
    if (delta_out) *delta_out = (mode & PR_NORM_LINF) ? hs->linf : hs->l1;
    return hs->status;
}

// ---------------------------------------------------------------- No-Sync --
static int run_nosync(pr_graph* g, double d, double tau, int32_t max_iter, uint32_t mode, double* ranks, Ctx& ctx,
                      int32_t* iters_out, double* delta_out) {
    cudaStream_t s = ctx.stream;
    const bool reduced = (mode & PR_USE_REDUCTIONS) != 0;
    const int64_t n = g->n;
    const View& v = reduced ? g->reduced : g->plain;
    const int64_t nm = reduced ? g->n_members : 0;
    const int64_t launches0 = ctx.launches;
    cudaPointerAttributes at{};
    const bool ranks_dev = cudaPointerGetAttributes(&at, ranks) == cudaSuccess &&
                           (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    double* x = ranks;
    if (!ranks_dev) {
        if (!g->x) PR_TRY(dalloc(&g->x, (size_t)n, s));
        x = g->x;
    }
    const int64_t ny = g->n_contrib + 1;
    for (int b = 0; b < 2; ++b)
        if (!g->y[b]) {
            PR_TRY(dalloc(&g->y[b], (size_t)ny, s));
            PR_CUDA(cudaMemsetAsync(g->y[b] + g->n_contrib, 0, sizeof(double), s));
        }
    double* y = g->y[0];
    GatherCfg gc;  // row-task engine, persistent grid (all resident CTAs)
    PR_TRY(gather_config(ctx, v, g, true, &gc));
    GatherCfg gp;  // certificate: synchronous edge-stream gather of the plain view
    PR_TRY(gather_config(ctx, g->plain, g, false, &gp, true));
    const int grid = gc.grid;
    const double c = (1.0 - d) / (double)n;
    if (reduced && nm > 0) {
        std::vector<double> ab(2 * ((size_t)g->max_chain + 1));
        ab[0] = 0.0;
        ab[1] = 1.0;
        for (int k = 1; k <= g->max_chain; ++k) {
            ab[2 * k] = c + d * ab[2 * (k - 1)];
            ab[2 * k + 1] = d * ab[2 * (k - 1) + 1];
        }
        dfree(g->ab, s);
        PR_TRY(dalloc(&g->ab, ab.size(), s));
        PR_CUDA(cudaMemcpyAsync(g->ab, ab.data(), ab.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    const int log_cap = max_iter < 4096 ? max_iter : 4096;
    if (g->log_cap < log_cap) {
        dfree(g->delta_log, s);
        PR_TRY(dalloc(&g->delta_log, (size_t)(2 * log_cap), s));
        g->log_cap = log_cap;
    }
    const int64_t cap4 = (int64_t)ctx.num_sms * 4;
    const int64_t nz = g->nz;
    int64_t zgrid = nz > 0 ? std::min<int64_t>((nz + GT_NT * 4 - 1) / (GT_NT * 4), cap4) : 0;
    const int64_t zper = zgrid > 0 ? (nz + zgrid - 1) / zgrid : 0;
    // scratch: err[2*grid] | residual[2] | zero-row partials[2*zgrid]; iters[grid]
    double* scratch = nullptr;
    int32_t* iters = nullptr;
    TmpGuard tg_(ctx.stream);
    tg_.track(scratch);
    tg_.track(iters);
    PR_TRY(dalloc(&scratch, (size_t)(2 * grid + 2 + 2 * zgrid), s));
    PR_TRY(dalloc(&iters, (size_t)grid, s));
    PR_CUDA(cudaMemsetAsync(iters, 0, sizeof(int32_t) * (size_t)grid, s));
    double* err = scratch;
    double* resid = scratch + 2 * grid;
    DevState* hs = g->st_host;
    *hs = DevState{};
    hs->max_iter = max_iter;
    hs->tau = tau;
    PR_CUDA(cudaMemcpyAsync(g->st, hs, sizeof(DevState), cudaMemcpyHostToDevice, s));
    PR_LAUNCH(ctx, k_init, (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx.num_sms * 16), 256, 0, x, y,
              (const int32_t*)g->outdeg, (const int32_t*)g->cidx, n, 1.0 / (double)n);
    // in-degree-0 vertices take their fixed value c (Q-Z) before the first sweep
    if (zgrid > 0)
        PR_LAUNCH(ctx, k_zero, (unsigned)zgrid, GT_NT, 0, (const int32_t*)g->zlist, nz, zper, c, x, y,
                  (const int32_t*)g->outdeg, (const int32_t*)g->cidx, resid + 2);
    if (gc.inplace) {  // edge-stream No-Sync: x in row / member order, unpermuted after each launch
        const int64_t need_xr = std::max<int64_t>(std::max(g->plain.nrows, g->reduced.nrows), 1);
        if (g->xr_cap < need_xr) {
            dfree(g->xr, s);
            PR_TRY(dalloc(&g->xr, (size_t)need_xr, s));
            g->xr_cap = need_xr;
        }
        if (g->n_members > 0 && !g->xm) PR_TRY(dalloc(&g->xm, (size_t)g->n_members, s));
        const unsigned fg = (unsigned)std::min<int64_t>((v.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
        PR_LAUNCH(ctx, k_fill_f64, fg, 256, 0, g->xr, v.nrows, 1.0 / (double)n);
        if (nm > 0) PR_LAUNCH(ctx, k_fill_f64, fg, 256, 0, g->xm, nm, 1.0 / (double)n);
    }
    const int64_t mper = nm > 0 ? (nm + grid - 1) / grid : 0;
    NoSyncArgs na{err, iters, (mode & PR_NORM_LINF) ? 1 : 0, tau, 0, g->mem_vid, g->mem_src, g->mem_k, nm, mper,
                  g->ab, x, y, g->outdeg, g->cidx};
    PRPolicy<true, true> pv{y, y, x, g->outdeg, g->cidx, v.vid, c, d, 0, {}};
    PRPolicy<true, false> pn{y, y, x, g->outdeg, g->cidx, v.vid, c, d, 0, {}};
    EngineArgs ea{v.tasks, v.ntasks, v.hubs, v.row_ptr, v.col, v.hub_partial, v.hub_delta, v.hub_ticket, 1};
    const void* fn = gc.inplace ? (const void*)k_nosync_stream
                                : (gc.vid ? (const void*)k_nosync<true> : (const void*)k_nosync<false>);
    PR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gc.smem));
    int per_sm = 0;
    PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, gc.nt, gc.smem));
    if ((int64_t)grid > (int64_t)ctx.num_sms * std::max(per_sm, 1)) {
        set_error("pr_run(NOSYNC): grid %d exceeds the resident CTAs", grid);
        return PR_ECUDA;
    }
    std::vector<int32_t> hit(grid);
    std::vector<double> hlog;
    int32_t max_it = 0, min_it = 0, med_it = 0, launches = 0, status = PR_NOT_CONVERGED;
    double r_l1 = 0.0, r_linf = 0.0;
    const View& pv_view = g->plain;
    while (true) {
        PR_LAUNCH(ctx, k_fill_f64, 1, 256, 0, err, (int64_t)(2 * grid), 1e300);
        na.max_local = max_iter - max_it;
        if (gc.inplace) {
            InPlacePolicy ip{};
            ip.y_in = y;
            ip.y = y;
            ip.hot_n = gc.hot_n;
            ip.xr = g->xr;
            ip.rinfo = v.rinfo;
            ip.c = c;
            ip.d = d;
            const StreamArgs sa{v.col,  (const uint8_t*)v.sflags, v.step_row, v.nsteps, v.span_steps, v.nspans, v.bin,
                                v.bout, v.b_row, v.b_s0, v.b_s1, v.part_in, v.part_out, v.bticket};
            const MemArgs ma{g->mem_srow, g->mem_k, g->mem_info, g->xm, nm, mper, g->ab};
            PR_LAUNCH(ctx, k_nosync_stream, (unsigned)grid, gc.nt, gc.smem, ip, sa, ma, na);
            const unsigned ug = (unsigned)std::min<int64_t>((v.nrows + nm + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
            PR_LAUNCH(ctx, k_unpermute, ug, 256, 0, (const double*)g->xr, (const int32_t*)v.vid, v.nrows,
                      (const double*)g->xm, (const int32_t*)g->mem_vid, nm, x);
        } else if (gc.vid) {
            PR_LAUNCH(ctx, k_nosync<true>, (unsigned)grid, GT_NT, gc.smem, pv, ea, na);
        } else {
            PR_LAUNCH(ctx, k_nosync<false>, (unsigned)grid, GT_NT, gc.smem, pn, ea, na);
        }
        ++launches;
        // certificate: S over the current contribs, then ||F(x) - x||
        PR_CUDA(cudaMemsetAsync(resid, 0, 2 * sizeof(double), s));
        IterArgs dummy{g->st, nullptr, 0, 0, 0, nullptr, 0, nullptr};
        PR_TRY(launch_gather(ctx, pv_view, y, nullptr, x, g, c, d, dummy, gp, 0));
        const unsigned rg = (unsigned)std::min<int64_t>((pv_view.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 8);
        if (pv_view.nrows > 0) {
            if (pv_view.vid)
                PR_LAUNCH(ctx, k_residual<true>, rg, 256, 0, (const double*)pv_view.sums, pv_view.nrows,
                          (const int32_t*)pv_view.vid, (const double*)x, c, d, resid);
            else
                PR_LAUNCH(ctx, k_residual<false>, rg, 256, 0, (const double*)pv_view.sums, pv_view.nrows,
                          (const int32_t*)nullptr, (const double*)x, c, d, resid);
        }
        double hr[2];
        PR_CUDA(cudaMemcpyAsync(hr, resid, sizeof(hr), cudaMemcpyDeviceToHost, s));
        PR_CUDA(cudaMemcpyAsync(hit.data(), iters, sizeof(int32_t) * (size_t)grid, cudaMemcpyDeviceToHost, s));
        PR_CUDA(cudaStreamSynchronize(s));
        r_l1 = hr[0];
        r_linf = hr[1];
        max_it = *std::max_element(hit.begin(), hit.end());
        min_it = *std::min_element(hit.begin(), hit.end());
        {
            std::vector<int32_t> tmp(hit);
            std::nth_element(tmp.begin(), tmp.begin() + tmp.size() / 2, tmp.end());
            med_it = tmp[tmp.size() / 2];
        }
        if (getenv("PRGPU_NOSYNC_DUMP")) {  // diagnostics: local sweeps of every CTA
            for (int b = 0; b < grid; ++b) fprintf(stderr, "%d%c", hit[b], (b + 1) % 37 ? ' ' : '\n');
            fprintf(stderr, "\n");
        }
        hlog.push_back(r_l1);
        hlog.push_back(r_linf);
        const double rn = (mode & PR_NORM_LINF) ? r_linf : r_l1;
        if (rn <= tau) {
            status = PR_OK;
            break;
        }
        if (max_it >= max_iter) break;
    }
    // delta log: the certified residual after each persistent launch
    const int nlog = std::min<int>((int)hlog.size() / 2, log_cap);
    if (nlog > 0)
        PR_CUDA(cudaMemcpyAsync(g->delta_log, hlog.data(), sizeof(double) * 2 * nlog, cudaMemcpyHostToDevice, s));
    g->log_len = nlog;
    hs->iters = max_it;
    hs->log_cap = log_cap;
    hs->status = status;
    hs->l1 = r_l1;
    hs->linf = r_linf;
    hs->done = 1;
    PR_CUDA(cudaMemcpyAsync(g->st, hs, sizeof(DevState), cudaMemcpyHostToDevice, s));
    if (!ranks_dev) PR_CUDA(cudaMemcpyAsync(ranks, x, sizeof(double) * (size_t)n, cudaMemcpyDefault, s));
    dfree(scratch, s);
    dfree(iters, s);
    PR_CUDA(cudaStreamSynchronize(s));
    pr_run_stats& rs = g->last;
    rs = pr_run_stats{};
    rs.phases = 1;
    rs.iterations = max_it;
    rs.status = status;
    rs.delta_l1 = r_l1;
    rs.delta_linf = r_linf;
    rs.run_launches = ctx.launches - launches0;
    rs.host_syncs = launches + 1;
    rs.gather_rows = v.nrows;
    rs.gather_edges = v.nedges;
    rs.scatter_members = nm;
    rs.n_contrib = g->n_contrib;
    rs.n_tasks = v.ntasks;
    rs.nosync_min_iters = min_it;
    rs.nosync_launches = launches;
    rs.nosync_median_iters = med_it;
    rs.residual = (mode & PR_NORM_LINF) ? r_linf : r_l1;
    if (iters_out) *iters_out = max_it;
    if (delta_out) *delta_out = rs.residual;
    return status;
}

// ------------------------------------------------------------ perforation --
// PR_PERFORATE (Barriers-Opt, Alg.5; reading Q-P in
// DESIGN.md): synchronous plain sweeps in which K-FINALIZE marks every row
// whose change was 0 < |delta| < tau * 1e-5.  At the host sync after each batch
// of sweeps, once enough rows are marked, the gathered view is COMPACTED to the
// unmarked rows: the marked rows keep their value (x, and their contrib in both
// ping-pong buffers) for the rest of the run and are never gathered again, so
// every later sweep streams fewer edges.  Approximate by design.
struct KeepGet {
    const uint8_t* fz;
    __device__ int64_t operator()(int64_t r) const { return fz[r] ? 0 : 1; }
};
struct KeepEmit {
    const uint8_t* fz;
    const int64_t* rp;
    const int32_t* amap;  // active row -> full plain-view row (nullptr: identity)
    const int2* rinfo;
    const double* xr;
    int32_t* src_row;
    int32_t* namap;
    int2* nrinfo;
    double* nxr;
    int64_t* nlen;
    __device__ void operator()(int64_t r, int64_t pos, int64_t f) const {
        if (!f) return;
        src_row[pos] = (int32_t)r;
        namap[pos] = amap ? amap[r] : (int32_t)r;
        nrinfo[pos] = rinfo[r];
        nxr[pos] = xr[r];
        nlen[pos] = rp[r + 1] - rp[r];
    }
};
struct LenGet {
    const int64_t* len;
    int64_t n;
    __device__ int64_t operator()(int64_t i) const { return i < n ? len[i] : 0; }
};
struct RpEmit {
    int64_t* rp;
    __device__ void operator()(int64_t i, int64_t pos, int64_t) const { rp[i] = pos; }
};

// marked rows: contrib into the other ping-pong buffer (frozen from now on)
__global__ void k_pf_freeze_y(const uint8_t* __restrict__ fz, const int2* __restrict__ rinfo, int64_t nr,
                              const double* __restrict__ ycur, double* __restrict__ yoth) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += (int64_t)gridDim.x * blockDim.x)
        if (fz[r] && rinfo[r].x > 0) yoth[rinfo[r].y] = ycur[rinfo[r].y];
}
// active-view x back into the full plain-view row order
__global__ void k_pf_writeback(const double* __restrict__ xa, const int32_t* __restrict__ amap, int64_t nr,
                               double* __restrict__ xfull) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += (int64_t)gridDim.x * blockDim.x)
        xfull[amap[r]] = xa[r];
}
__global__ void k_count_u8(const uint8_t* __restrict__ a, int64_t n, unsigned long long* out) {
    uint32_t c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += a[i] ? 1u : 0u;
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

struct ActiveView {
    View v;                 // gathered rows; v.vid = map to the full plain-view row
    double* xr = nullptr;   // x of its rows
    bool is_full = true;    // the plain view itself (no copies)
};

static void free_active(ActiveView& a, cudaStream_t s) {
    if (a.is_full) return;
    dfree(a.xr, s);
    free_view(a.v, s);  // frees vid (the map), sums, rinfo, col, row_ptr, stream tables
}

static int run_perforated(pr_graph* g, double d, double tau, int32_t max_iter, uint32_t mode, double* ranks,
                          Ctx& ctx, int32_t* iters_out, double* delta_out) {
    cudaStream_t s = ctx.stream;
    const int64_t n = g->n;
    View& V = g->plain;
    const int64_t launches0 = ctx.launches;
    cudaPointerAttributes at{};
    const bool ranks_dev = cudaPointerGetAttributes(&at, ranks) == cudaSuccess &&
                           (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    double* x = ranks;
    if (!ranks_dev) {
        if (!g->x) PR_TRY(dalloc(&g->x, (size_t)n, s));
        x = g->x;
    }
    const int64_t ny = g->n_contrib + 1;
    for (int b = 0; b < 2; ++b)
        if (!g->y[b]) {
            PR_TRY(dalloc(&g->y[b], (size_t)ny, s));
            PR_CUDA(cudaMemsetAsync(g->y[b] + g->n_contrib, 0, sizeof(double), s));
        }
    const int64_t need_xr = std::max<int64_t>(std::max(g->plain.nrows, g->reduced.nrows), 1);
    if (g->xr_cap < need_xr) {
        dfree(g->xr, s);
        PR_TRY(dalloc(&g->xr, (size_t)need_xr, s));
        g->xr_cap = need_xr;
    }
    const double c = (1.0 - d) / (double)n;
    const int64_t cap4 = (int64_t)ctx.num_sms * 4;
    const int64_t fgrid_max = std::min<int64_t>(std::max<int64_t>((V.nrows + GT_NT * FIN_U - 1) / (GT_NT * FIN_U), 1),
                                                cap4 * 2);
    const int64_t nz = g->nz;
    const int64_t zgrid = nz > 0 ? std::min<int64_t>((nz + GT_NT * 4 - 1) / (GT_NT * 4), cap4) : 0;
    const int64_t zper = zgrid > 0 ? (nz + zgrid - 1) / zgrid : 0;
    const int64_t need = 2 * (fgrid_max + zgrid);
    if (g->partial_cap < need) {
        dfree(g->cta_partial, s);
        PR_TRY(dalloc(&g->cta_partial, (size_t)need, s));
        g->partial_cap = need;
    }
    const int log_cap = max_iter < 4096 ? max_iter : 4096;
    if (g->log_cap < log_cap) {
        dfree(g->delta_log, s);
        PR_TRY(dalloc(&g->delta_log, (size_t)(2 * log_cap), s));
        g->log_cap = log_cap;
    }
    uint8_t* fz = nullptr;
    unsigned long long* cnt = nullptr;
    TmpGuard tg_(ctx.stream);
    tg_.track(fz);
    tg_.track(cnt);
    PR_TRY(dalloc(&fz, (size_t)std::max<int64_t>(V.nrows, 1), s));
    PR_TRY(dalloc(&cnt, 2, s));
    PR_CUDA(cudaMemsetAsync(fz, 0, (size_t)std::max<int64_t>(V.nrows, 1), s));
    DevState* hs = g->st_host;
    *hs = DevState{};
    hs->max_iter = max_iter;
    hs->norm_linf = (mode & PR_NORM_LINF) ? 1 : 0;
    hs->tau = tau;
    hs->log_cap = log_cap;
    PR_CUDA(cudaMemcpyAsync(g->st, hs, sizeof(DevState), cudaMemcpyHostToDevice, s));
    PR_LAUNCH(ctx, k_init, (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx.num_sms * 16), 256, 0, x,
              g->y[0], (const int32_t*)g->outdeg, (const int32_t*)g->cidx, n, 1.0 / (double)n);
    const unsigned fg = (unsigned)std::min<int64_t>((V.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
    PR_LAUNCH(ctx, k_fill_f64, fg, 256, 0, g->xr, V.nrows, 1.0 / (double)n);

    ActiveView A;
    A.v = V;  // shallow: the plain view's arrays
    A.xr = g->xr;
    A.is_full = true;
    int64_t edges_gathered = 0;
    int32_t compactions = 0;
    int64_t launched = 0;
    int host_syncs = 0;
    int rc = PR_OK;
    while (true) {
        GatherCfg gc;
        if ((rc = gather_config(ctx, A.v, g, false, &gc, true)) != PR_OK) break;
        const int64_t fgrid =
            std::min<int64_t>(std::max<int64_t>((A.v.nrows + GT_NT * FIN_U - 1) / (GT_NT * FIN_U), 1), cap4 * 2);
        IterArgs ia{g->st, g->cta_partial, fgrid, 0, 0, nullptr, 0, g->delta_log};
        IterArgs ia0 = ia;
        ia0.zero_ctas = zgrid;
        double* zero_partial = g->cta_partial + 2 * fgrid;
        FinArgs fa{A.v.sums, A.v.nrows, A.v.rinfo, A.xr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, nullptr, c, d,
                   fz, tau * 1e-5, cnt};
        const int nb = (int)std::min<int64_t>(8, max_iter - launched);
        for (int j = 0; j < nb; ++j) {
            const int64_t it = launched + j;
            const double* y_in = g->y[it & 1];
            double* y_out = g->y[(it + 1) & 1];
            const IterArgs& iv = it == 0 ? ia0 : ia;
            if (it == 0 && zgrid > 0)
                PR_LAUNCH(ctx, k_zero, (unsigned)zgrid, GT_NT, 0, (const int32_t*)g->zlist, nz, zper, c, x, y_out,
                          (const int32_t*)g->outdeg, (const int32_t*)g->cidx, zero_partial);
            if ((rc = launch_gather(ctx, A.v, y_in, y_out, x, g, c, d, iv, gc, 0)) != PR_OK) break;
            FinArgs f = fa;
            f.y_out = y_out;
            PR_LAUNCH(ctx, k_finalize, (unsigned)fgrid, GT_NT, 0, f, iv);
            if (it == 0 && nz > 0)
                PR_LAUNCH(ctx, k_zero_y, (unsigned)std::min<int64_t>((nz + 255) / 256, (int64_t)ctx.num_sms * 8), 256,
                          0, (const int32_t*)g->zlist, nz, c, (double*)y_in, (const int32_t*)g->outdeg,
                          (const int32_t*)g->cidx);
        }
        if (rc != PR_OK) break;
        PR_CUDA(cudaMemsetAsync(cnt + 1, 0, sizeof(unsigned long long), s));
        if (A.v.nrows > 0)
            PR_LAUNCH(ctx, k_count_u8, (unsigned)std::min<int64_t>((A.v.nrows + 255) / 256 + 1, cap4 * 4), 256, 0,
                      (const uint8_t*)fz, A.v.nrows, cnt + 1);
        unsigned long long marked = 0;
        PR_CUDA(cudaMemcpyAsync(hs, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        PR_CUDA(cudaMemcpyAsync(&marked, cnt + 1, sizeof(marked), cudaMemcpyDeviceToHost, s));
        PR_CUDA(cudaStreamSynchronize(s));
        ++host_syncs;
        const int64_t done_sweeps = std::min<int64_t>(hs->iters, launched + nb) - launched;
        edges_gathered += A.v.nedges * std::max<int64_t>(done_sweeps, 0);
        launched += nb;
        if (hs->done || launched >= max_iter) break;
        if ((int64_t)marked * 20 < A.v.nrows || marked == 0) continue;  // compact once >= 5 % are marked
        // ---- compaction: freeze the marked rows, gather only the others ----
        const double* ycur = g->y[launched & 1];
        double* yoth = g->y[(launched + 1) & 1];
        PR_LAUNCH(ctx, k_pf_freeze_y, fg, 256, 0, (const uint8_t*)fz, (const int2*)A.v.rinfo, A.v.nrows, ycur, yoth);
        if (!A.is_full)
            PR_LAUNCH(ctx, k_pf_writeback, fg, 256, 0, (const double*)A.xr, (const int32_t*)A.v.vid, A.v.nrows, g->xr);
        ActiveView B;
        B.is_full = false;
        const int64_t nr = A.v.nrows - (int64_t)marked;
        int32_t* src_row = nullptr;
        int64_t* nlen = nullptr;
        int64_t* tot = nullptr;
        PR_TRY(dalloc(&src_row, (size_t)std::max<int64_t>(nr, 1), s));
        PR_TRY(dalloc(&nlen, (size_t)std::max<int64_t>(nr, 1), s));
        PR_TRY(dalloc(&tot, 1, s));
        PR_TRY(dalloc(&B.v.vid, (size_t)std::max<int64_t>(nr, 1), s));
        PR_TRY(dalloc(&B.v.rinfo, (size_t)std::max<int64_t>(nr, 1), s));
        PR_TRY(dalloc(&B.xr, (size_t)std::max<int64_t>(nr, 1), s));
        PR_TRY((device_scan<int64_t>(ctx, A.v.nrows, KeepGet{fz},
                                     KeepEmit{fz, A.v.row_ptr, A.is_full ? nullptr : A.v.vid, A.v.rinfo, A.xr, src_row,
                                              B.v.vid, B.v.rinfo, B.xr, nlen},
                                     tot)));
        B.v.nrows = nr;
        PR_TRY(dalloc(&B.v.row_ptr, (size_t)nr + 1, s));
        B.v.owns_row_ptr = true;
        PR_TRY((device_scan<int64_t>(ctx, nr + 1, LenGet{nlen, nr}, RpEmit{B.v.row_ptr}, tot)));
        PR_TRY(read_count(ctx, tot, &B.v.nedges));
        PR_TRY(dalloc(&B.v.col, (size_t)stream_pad(B.v.nedges), s));
        if (nr > 0)
            PR_LAUNCH(ctx, k_copy_rows, (unsigned)std::min<int64_t>((B.v.nedges + 1023) / 1024 / 8 + 1, cap4 * 2), 256,
                      0, (const int32_t*)src_row, nr, (const int64_t*)A.v.row_ptr, (const int32_t*)A.v.col,
                      (const int64_t*)B.v.row_ptr, B.v.col);
        PR_TRY(build_view_stream(B.v, ctx, (int32_t)g->n_contrib, nullptr, nullptr));
        PR_TRY(dalloc(&B.v.sums, (size_t)std::max<int64_t>(nr, 1), s));
        dfree(src_row, s);
        dfree(nlen, s);
        dfree(tot, s);
        free_active(A, s);
        A = B;
        PR_CUDA(cudaMemsetAsync(fz, 0, (size_t)std::max<int64_t>(V.nrows, 1), s));
        ++compactions;
    }
    if (rc == PR_OK) {
        if (!A.is_full)
            PR_LAUNCH(ctx, k_pf_writeback, fg, 256, 0, (const double*)A.xr, (const int32_t*)A.v.vid, A.v.nrows, g->xr);
        const unsigned ug = (unsigned)std::min<int64_t>((V.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
        PR_LAUNCH(ctx, k_unpermute, ug, 256, 0, (const double*)g->xr, (const int32_t*)V.vid, V.nrows,
                  (const double*)nullptr, (const int32_t*)nullptr, (int64_t)0, x);
        if (!ranks_dev) PR_CUDA(cudaMemcpyAsync(ranks, x, sizeof(double) * (size_t)n, cudaMemcpyDefault, s));
    }
    const int64_t frozen = V.nrows - A.v.nrows;
    free_active(A, s);
    dfree(fz, s);
    dfree(cnt, s);
    PR_CUDA(cudaStreamSynchronize(s));
    if (rc != PR_OK) return rc;
    pr_run_stats& rs = g->last;
    rs = pr_run_stats{};
    rs.phases = 1;
    g->log_len = std::min<int32_t>(hs->iters, g->log_cap);
    rs.iterations = hs->iters;
    rs.status = hs->status;
    rs.delta_l1 = hs->l1;
    rs.delta_linf = hs->linf;
    rs.run_launches = ctx.launches - launches0;
    rs.host_syncs = host_syncs;
    rs.gather_rows = V.nrows;
    rs.gather_edges = V.nedges;
    rs.n_contrib = g->n_contrib;
    rs.edges_gathered = edges_gathered;
    rs.frozen_rows = frozen;
    rs.compactions = compactions;
    if (iters_out) *iters_out = hs->iters;
    if (delta_out) *delta_out = (mode & PR_NORM_LINF) ? hs->linf : hs->l1;
    return hs->status;
}

}  // namespace prgpu
