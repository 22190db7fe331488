// rowengine.cuh -- the degree-aware row-block engine behind K-GATHER (and the
// row-hash step of identical-group detection).
//
// For every row r of a View it computes  S(r) = sum_{e in row r} load(col[e])
// and calls  finalize(r, S(r)).  Work is cut into tasks (internal.h):
//   * row block: consecutive rows with < CAP + LONG edges in total.  Phase A
//     streams the block's col_idx range with 128-bit evict-first loads and
//     gathers load(col) for every edge into shared memory (4 independent
//     gathers per int4, U int4 per thread in flight).  Phase B: each lane owns
//     rows (r = warp*32 + lane + k*NT); rows of length <= SHORT are summed
//     serially by their lane, longer rows cooperatively by the owning warp
//     (lane-strided partials + xor-shuffle tree).
//   * hub chunk: HUB_CHUNK edges of one row with in-degree > LONG; each CTA
//     reduces its chunk (fixed tree) into a partial slot; the CTA that takes
//     the last ticket of the hub sums the partials in chunk order and
//     finalizes the row.
// Every sum is taken in an order that depends only on the row's data, so the
// results are deterministic run to run (not equal to the oracle's ascending
// order; DESIGN.md Q-F).
#pragma once
#include "internal.h"

namespace prgpu {

constexpr int GT_WARPS = GT_NT / 32;
constexpr int GT_U = 4;  // int4 col loads in flight per thread in phase A

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

struct __align__(16) EngineSmem {
    uint64_t vals[GT_VALS];
    int32_t rp[GT_MAXROWS + 1];
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
__device__ __forceinline__ void engine_rowblock(P& p, const EngineArgs& a, const Task tk, EngineSmem& sm,
                                                double& l1, double& linf) {
    using T = typename P::T;
    T* vals = reinterpret_cast<T*>(sm.vals);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = tk.r0;
    const int nr = tk.a;
    const int64_t e0 = a.row_ptr[r0];
    for (int i = tid; i <= nr; i += GT_NT) sm.rp[i] = (int32_t)(a.row_ptr[r0 + i] - e0);
    __syncthreads();
    const int nnz = sm.rp[nr];
    // ---- phase A: stream col_idx, gather into shared memory ----
    const int64_t a0 = e0 & ~(int64_t)3;
    const int lead = (int)(e0 - a0);
    const int n4 = (lead + nnz + 3) >> 2;
    const int4* c4 = reinterpret_cast<const int4*>(a.col + a0);
    for (int q0 = 0; q0 < n4; q0 += GT_NT * GT_U) {
        int4 cv[GT_U] = {};
#pragma unroll
        for (int u = 0; u < GT_U; ++u) {
            int q = q0 + u * GT_NT + tid;
            if (q < n4) cv[u] = p.ld_col(c4 + q);
        }
#pragma unroll
        for (int u = 0; u < GT_U; ++u) {
            int q = q0 + u * GT_NT + tid;
            int base = q * 4 - lead;
            int cc[4] = {cv[u].x, cv[u].y, cv[u].z, cv[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (q < n4 && base + j >= 0 && base + j < nnz) vals[base + j] = p.load(cc[j]);
        }
    }
    __syncthreads();
    // ---- phase B: per-row sums, finalize ----
    for (int i0 = warp * 32; i0 < nr; i0 += GT_NT) {
        const int i = i0 + lane;
        const bool valid = i < nr;
        const int s = valid ? sm.rp[i] : 0;
        const int len = valid ? sm.rp[i + 1] - s : 0;
        const bool lng = len > GT_SHORT;
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
            double dl = p.finalize(r0 + i, sum);
            l1 += dl;
            linf = fmax(linf, dl);
        }
    }
    __syncthreads();
}

template <class P>
__device__ __forceinline__ void engine_hubchunk(P& p, const EngineArgs& a, const Task tk, EngineSmem& sm) {
    using T = typename P::T;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Hub h = a.hubs[tk.b];
    const int64_t row = tk.r0;
    const int64_t rs = a.row_ptr[row], re = a.row_ptr[row + 1];
    const int64_t cs = rs + (int64_t)tk.a * GT_HUB_CHUNK;
    const int64_t ce = min(re, cs + (int64_t)GT_HUB_CHUNK);
    const int nnz = (int)(ce - cs);
    const int64_t a0 = cs & ~(int64_t)3;
    const int lead = (int)(cs - a0);
    const int n4 = (lead + nnz + 3) >> 2;
    const int4* c4 = reinterpret_cast<const int4*>(a.col + a0);
    T part = T(0);
    for (int q0 = 0; q0 < n4; q0 += GT_NT * GT_U) {
        int4 cv[GT_U] = {};
#pragma unroll
        for (int u = 0; u < GT_U; ++u) {
            int q = q0 + u * GT_NT + tid;
            if (q < n4) cv[u] = p.ld_col(c4 + q);
        }
#pragma unroll
        for (int u = 0; u < GT_U; ++u) {
            int q = q0 + u * GT_NT + tid;
            int base = q * 4 - lead;
            int cc[4] = {cv[u].x, cv[u].y, cv[u].z, cv[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (q < n4 && base + j >= 0 && base + j < nnz) part += p.load(cc[j]);
        }
    }
    part = warp_sum(part);
    T* red = reinterpret_cast<T*>(sm.red);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (tid == 0) {
        T s = T(0);
#pragma unroll
        for (int w = 0; w < GT_WARPS; ++w) s += red[w];
        T* hp = reinterpret_cast<T*>(a.hub_partial);
        hp[h.slot + tk.a] = s;
        __threadfence();
        uint32_t t = atomicAdd(&a.hub_ticket[tk.b], 1u);
        sm.flag = (t == (uint32_t)h.nchunks - 1) ? 1 : 0;
    }
    __syncthreads();
    if (sm.flag && tid == 0) {
        __threadfence();
        const T* hp = reinterpret_cast<const T*>(a.hub_partial);
        T s = T(0);
        for (int j = 0; j < h.nchunks; ++j) s += __ldcg(hp + h.slot + j);
        a.hub_delta[tk.b] = p.finalize(row, s);
        a.hub_ticket[tk.b] = 0u;
    }
    __syncthreads();
}

// Runs every task assigned to this CTA (static round robin: task i -> CTA
// i mod gridDim.x, so the per-CTA accumulation order is deterministic).
template <class P>
__device__ __forceinline__ void engine_run(P& p, const EngineArgs& a, EngineSmem& sm, double& l1, double& linf) {
    for (int64_t t = blockIdx.x; t < a.ntasks; t += gridDim.x) {
        const Task tk = a.tasks[t];
        if (tk.b < 0)
            engine_rowblock(p, a, tk, sm, l1, linf);
        else
            engine_hubchunk(p, a, tk, sm);
    }
}

}  // namespace prgpu
