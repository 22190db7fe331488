// rowengine.cuh -- the degree-aware, warp-independent row engine behind
// K-GATHER (and the row-hash step of identical-group detection).
//
// For every row r of a View it computes  S(r) = sum_{e in row r} load(col[e])
// and calls  finalize(r, S(r)).  The rows are cut into warp tasks (built by
// build_view_tasks, ingest.cu); every warp of the grid walks its own static
// list of tasks (task t -> global warp t mod #warps), with no CTA barrier:
//   * row block  (info >= 0): consecutive rows with <= WT_MAXE edges, each of
//     in-degree <= WT_LONG.  The warp issues the block's 128-bit col_idx loads
//     and gathers at once (the edge range is in the descriptor), prefetches
//     the finalize operands of its rows (x, outdeg, contrib slot) in the same
//     wave, stages the gathered values in its private shared-memory slice,
//     then sums rows: lengths <= WT_SHORT serially by the owning lane, longer
//     ones cooperatively (lane-strided partials + xor tree).
//   * long chunk (info < 0): up to WT_HCH edges of one row of in-degree >
//     WT_LONG, reduced in registers (lane-strided, xor tree).  Single-chunk
//     rows finalize directly; multi-chunk ("hub") rows write a partial slot
//     and the warp taking the hub's last ticket sums the partials in chunk
//     order and finalizes the row.
// Every sum is taken in an order that depends only on the row's data, so the
// results are deterministic (not the oracle's order, Q-F).
#pragma once
#include "internal.h"

namespace prgpu {

constexpr int GT_WARPS = GT_NT / 32;

struct EngineArgs {
    const Task* tasks;
    int64_t ntasks;
    const Hub* hubs;
    const int64_t* row_ptr;
    const int32_t* col;
    void* hub_partial;
    double* hub_delta;
    uint32_t* hub_ticket;
};

struct __align__(16) WarpSmem {
    uint64_t vals[WT_VALS];
    int32_t rp[WT_MAXROWS + 3];
};

struct __align__(16) EngineSmem {
    WarpSmem w[GT_WARPS];
    double red[2 * GT_WARPS];
    int flag;
};

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <class P>
__device__ __forceinline__ void engine_rowblock(P& p, const EngineArgs& a, const Task tk, WarpSmem& ws,
                                                double& l1, double& linf) {
    using T = typename P::T;
    T* vals = reinterpret_cast<T*>(ws.vals);
    const int lane = threadIdx.x & 31;
    const int64_t r0 = tk.r0;
    const int nr = (tk.info >> 16) & 0x7fff;
    const int nnz = tk.info & 0xffff;
    const int64_t e0 = tk.e0;
    // finalize operands of rows lane and lane+32 (independent of the gathers)
    typename P::Pre pre0{}, pre1{};
    if (lane < nr) pre0 = p.prefetch(r0 + lane);
    if (lane + 32 < nr) pre1 = p.prefetch(r0 + lane + 32);
    // row offsets relative to e0
    for (int i = lane; i <= nr; i += 32) ws.rp[i] = (int32_t)(a.row_ptr[r0 + i] - e0);
    // stream col_idx (aligned int4) and gather
    const int64_t a0 = e0 & ~(int64_t)3;
    const int lead = (int)(e0 - a0);
    const int n4 = (lead + nnz + 3) >> 2;
    const int4* c4 = reinterpret_cast<const int4*>(a.col + a0);
    for (int q0 = 0; q0 < n4; q0 += 32 * WT_U) {
        int4 cv[WT_U];
#pragma unroll
        for (int u = 0; u < WT_U; ++u) {
            const int q = q0 + u * 32 + lane;
            cv[u] = q < n4 ? p.ld_col(c4 + q) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < WT_U; ++u) {
            const int q = q0 + u * 32 + lane;
            const int base = q * 4 - lead;
            const int cc[4] = {cv[u].x, cv[u].y, cv[u].z, cv[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (q < n4 && base + j >= 0 && base + j < nnz) vals[base + j] = p.load(cc[j]);
        }
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h;
        if (32 * h >= nr) break;
        const bool valid = i < nr;
        const int s = valid ? ws.rp[i] : 0;
        const int len = valid ? ws.rp[i + 1] - s : 0;
        const bool lng = len > WT_SHORT;
        T sum = T(0);
        if (valid && !lng) {
            T s0 = T(0), s1 = T(0);
            int k = 0;
            for (; k + 1 < len; k += 2) {
                s0 += vals[s + k];
                s1 += vals[s + k + 1];
            }
            if (k < len) s0 += vals[s + k];
            sum = s0 + s1;
        }
        uint32_t lmask = __ballot_sync(0xffffffffu, lng);
        while (lmask) {
            const int src = __ffs(lmask) - 1;
            lmask &= lmask - 1;
            const int ls = __shfl_sync(0xffffffffu, s, src);
            const int ll = __shfl_sync(0xffffffffu, len, src);
            T part = T(0);
            for (int k = lane; k < ll; k += 32) part += vals[ls + k];
            part = warp_sum(part);
            if (lane == src) sum = part;
        }
        if (valid) {
            const double dl = p.finalize(h ? pre1 : pre0, sum);
            l1 += dl;
            linf = fmax(linf, dl);
        }
    }
    __syncwarp();
}

template <class P>
__device__ __forceinline__ void engine_longchunk(P& p, const EngineArgs& a, const Task tk, EngineSmem& sm,
                                                 double& l1, double& linf) {
    using T = typename P::T;
    const int lane = threadIdx.x & 31;
    const int64_t row = tk.r0;
    const int nnz = tk.info & 0xffff;
    const int64_t e0 = tk.e0;
    typename P::Pre pre{};
    if (lane == 0 && tk.hub < 0) pre = p.prefetch(row);
    const int64_t a0 = e0 & ~(int64_t)3;
    const int lead = (int)(e0 - a0);
    const int n4 = (lead + nnz + 3) >> 2;
    const int4* c4 = reinterpret_cast<const int4*>(a.col + a0);
    T part = T(0);
    for (int q0 = 0; q0 < n4; q0 += 32 * WT_U) {
        int4 cv[WT_U];
#pragma unroll
        for (int u = 0; u < WT_U; ++u) {
            const int q = q0 + u * 32 + lane;
            cv[u] = q < n4 ? p.ld_col(c4 + q) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < WT_U; ++u) {
            const int q = q0 + u * 32 + lane;
            const int base = q * 4 - lead;
            const int cc[4] = {cv[u].x, cv[u].y, cv[u].z, cv[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (q < n4 && base + j >= 0 && base + j < nnz) part += p.load(cc[j]);
        }
    }
    part = warp_sum(part);
    if (tk.hub < 0) {
        if (lane == 0) {
            const double dl = p.finalize(pre, part);
            l1 += dl;
            linf = fmax(linf, dl);
        }
        return;
    }
    if (lane == 0) {
        const Hub h = a.hubs[tk.hub];
        const int j = (int)((e0 - h.row_e0) / WT_HCH);
        T* hp = reinterpret_cast<T*>(a.hub_partial);
        hp[h.slot + j] = part;
        __threadfence();
        const uint32_t t = atomicAdd(&a.hub_ticket[tk.hub], 1u);
        if (t == (uint32_t)h.nchunks - 1) {
            __threadfence();
            const T* hq = reinterpret_cast<const T*>(a.hub_partial);
            T s = T(0);
            for (int c = 0; c < h.nchunks; ++c) s += __ldcg(hq + h.slot + c);
            const typename P::Pre pr = p.prefetch(row);
            a.hub_delta[tk.hub] = p.finalize(pr, s);
            a.hub_ticket[tk.hub] = 0u;
        }
    }
}

// Runs every task assigned to this warp.  The per-thread (l1, linf)
// accumulators therefore depend only on the static assignment.
template <class P>
__device__ __forceinline__ void engine_run(P& p, const EngineArgs& a, EngineSmem& sm, double& l1, double& linf) {
    const int warp = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * GT_WARPS + warp;
    const int64_t nw = (int64_t)gridDim.x * GT_WARPS;
    WarpSmem& ws = sm.w[warp];
    for (int64_t t = gw; t < a.ntasks; t += nw) {
        const Task tk = a.tasks[t];
        if (tk.info >= 0)
            engine_rowblock(p, a, tk, ws, l1, linf);
        else
            engine_longchunk(p, a, tk, sm, l1, linf);
    }
}

}  // namespace prgpu
