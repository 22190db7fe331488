// rowengine.cuh -- the degree-aware, warp-independent row engine behind
// K-GATHER (and the row-hash step of identical-group detection).
//
// For every row r of a View it computes  S(r) = sum_{e in row r} load(col[e])
// and calls  finalize(r, S(r)).  The rows are cut into warp tasks (built by
// build_view_tasks, ingest.cu); every warp of the grid walks its own static
// list of tasks (task t -> global warp t mod #warps), with no CTA barrier.
// A task is consumed as a stream of "pieces" of <= WT_PIECE edges, run as a
// two-stage software pipeline per warp:
//   * the col_idx range of the NEXT piece is fetched into the warp's second
//     shared-memory buffer by one TMA bulk copy (cp.async.bulk + mbarrier),
//     so index loads never occupy the LSU/L1 pipe or registers, and their
//     DRAM latency overlaps the current piece's gathers;
//   * row block (info >= 0, one piece): rows of in-degree <= WT_LONG.  The
//     finalize operands of its rows (x, outdeg, contrib slot) are prefetched,
//     all lanes gather load(col) for the block's edges (indices first, then
//     all gathers, then the stores, so they are in flight together) into the
//     warp's vals buffer, and rows are summed: lengths <= WT_SHORT serially by
//     the owning lane, longer ones cooperatively (lane-strided + xor tree);
//   * chunk (info < 0): <= WT_HCH edges of one row of in-degree > WT_LONG,
//     accumulated per lane over its pieces, then reduced (xor tree).
//     Single-chunk rows finalize directly; multi-chunk ("hub") rows write a
//     partial slot and the warp taking the hub's last ticket sums the
//     partials in chunk order and finalizes the row.
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
    int hub_local = 0;  // also add a hub row's |delta| to the finalizing warp's (l1, linf) (No-Sync kernel)
};

struct __align__(16) WarpSmem {
    int32_t colbuf[2][WT_COLBUF];
    uint64_t vals[WT_VALS];
    uint64_t bar[2];
    int32_t rp[WT_MAXROWS + 3];
};

struct __align__(16) EngineSmem {
    WarpSmem w[GT_WARPS];
    double red[2 * 32];  // block reductions (one sum and one max per warp, up to 32 warps)
    int flag;
};

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ int task_nnz(const Task& tk) { return tk.info & 0xffff; }
__device__ __forceinline__ int task_pieces(const Task& tk) { return (task_nnz(tk) + WT_PIECE - 1) / WT_PIECE; }

// Lane 0: stage col[e - lead .. e + cnt) (16-byte aligned superset) into buf.
__device__ __forceinline__ void stage_cols(const EngineArgs& a, int64_t e, int cnt, int32_t* buf, uint64_t* bar,
                                           uint64_t pol) {
    const int64_t a0 = e & ~(int64_t)3;
    const uint32_t bytes = (uint32_t)(((e - a0) + cnt) * 4 + 15) & ~15u;
    bulk_g2s(buf, a.col + a0, bytes, bar, pol);
}

// Gathers of one staged piece: gv[k] = load(col[e0 + k*32 + lane]) for the
// first cnt edges (indices first, then every gather, so all are in flight).
template <class P>
__device__ __forceinline__ void gather_piece(const P& p, const int32_t* cb, int lead, int cnt,
                                             typename P::T (&gv)[WT_PIECE / 32]) {
    using T = typename P::T;
    const int lane = threadIdx.x & 31;
    constexpr int K = WT_PIECE / 32;
    int ci[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int e = k * 32 + lane;
        ci[k] = e < cnt ? cb[lead + e] : -1;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) gv[k] = ci[k] >= 0 ? p.load(ci[k]) : T(0);
}

template <class P>
__device__ __forceinline__ void engine_rowblock(P& p, const Task& tk, WarpSmem& ws, const int32_t* cb, double& l1,
                                                double& linf) {
    using T = typename P::T;
    constexpr int K = WT_PIECE / 32;
    T* vals = reinterpret_cast<T*>(ws.vals);
    const int lane = threadIdx.x & 31;
    const int nr = (tk.info >> 16) & 0x7fff;
    const int nnz = task_nnz(tk);
    T gv[K];
    gather_piece(p, cb, tk.e0 & 3, nnz, gv);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int e = k * 32 + lane;
        if (e < nnz) vals[e] = gv[k];
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
            const double dl = p.finalize(p.prefetched(h), sum);
            l1 += dl;
            linf = fmax(linf, dl);
        }
    }
}

// End of a chunk task: reduce the lane partials and finalize (or hand the
// partial to the hub protocol).
template <class P>
__device__ __forceinline__ void engine_chunk_end(P& p, const EngineArgs& a, const Task& tk, typename P::T part,
                                                 double& l1, double& linf) {
    using T = typename P::T;
    const int lane = threadIdx.x & 31;
    part = warp_sum(part);
    if (tk.hub < 0) {
        if (lane == 0) {
            const double dl = p.finalize(p.prefetched(0), part);
            l1 += dl;
            linf = fmax(linf, dl);
        }
        return;
    }
    if (lane == 0) {
        const Hub h = a.hubs[tk.hub];
        const int j = (int)(((int64_t)tk.e0 - h.row_e0) / WT_HCH);
        T* hp = reinterpret_cast<T*>(a.hub_partial);
        hp[h.slot + j] = part;
        __threadfence();
        // wrapping ticket (atomicInc: nchunks-1 -> 0): no separate reset, so it
        // also works when chunks of different sweeps interleave (persistent
        // No-Sync kernel: the finalize then reads each chunk's latest partial)
        const uint32_t t = atomicInc(&a.hub_ticket[tk.hub], (uint32_t)h.nchunks - 1);
        if (t == (uint32_t)h.nchunks - 1) {
            __threadfence();
            const T* hq = reinterpret_cast<const T*>(a.hub_partial);
            T s = T(0);
            for (int c = 0; c < h.nchunks; ++c) s += __ldcg(hq + h.slot + c);
            const double dh = p.finalize(p.prefetch((int64_t)tk.r0), s);
            a.hub_delta[tk.hub] = dh;
            if (a.hub_local) {
                l1 += dh;
                linf = fmax(linf, dh);
            }
        }
    }
}

// Runs every task assigned to this warp.  The per-thread (l1, linf)
// accumulators therefore depend only on the static assignment.
// kbase (optional, per warp, persistent kernels): pieces this warp's
// barriers have completed in earlier calls -- the barriers are initialised
// once (kbase == 0) and later calls continue their phase sequence (an
// mbarrier must not be re-initialised while it is in use).
template <class P>
__device__ __forceinline__ void engine_run(P& p, const EngineArgs& a, EngineSmem& sm, double& l1, double& linf,
                                           uint32_t* kbase = nullptr) {
    using T = typename P::T;
    constexpr int K = WT_PIECE / 32;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * GT_WARPS;
    int64_t t = (int64_t)blockIdx.x * GT_WARPS + warp;
    WarpSmem& ws = sm.w[warp];
    if (t >= a.ntasks) return;
    const uint64_t pol = policy_evict_first();
    const uint32_t k0 = kbase ? *kbase : 0u;
    if (lane == 0 && k0 == 0) {
        mbar_init(&ws.bar[0], 1);
        mbar_init(&ws.bar[1], 1);
        fence_mbar_init();
    }
    __syncwarp();
    Task cur = a.tasks[t];
    int j = 0;  // piece of cur
    if (lane == 0) {
        if (k0) fence_proxy_async_smem();  // the buffer was last read by the generic proxy
        stage_cols(a, cur.e0, min(task_nnz(cur), WT_PIECE), ws.colbuf[k0 & 1], &ws.bar[k0 & 1], pol);
    }
    T part = T(0);
    for (uint32_t k = k0;; ++k) {
        const int b = k & 1;
        // next piece: the rest of this chunk, else the first piece of the next task
        Task nt = cur;
        int nj = j + 1;
        int64_t ntn = t;
        if (nj >= task_pieces(cur)) {
            ntn = t + nw;
            nj = 0;
            if (ntn < a.ntasks) nt = a.tasks[ntn];
        }
        const bool has_next = ntn < a.ntasks;
        if (has_next && lane == 0) {
            fence_proxy_async_smem();  // buffer b^1 was last read (generic proxy) by piece k-1
            const int64_t e = (int64_t)nt.e0 + (int64_t)nj * WT_PIECE;
            stage_cols(a, e, min(task_nnz(nt) - nj * WT_PIECE, WT_PIECE), ws.colbuf[b ^ 1], &ws.bar[b ^ 1], pol);
        }
        if (j == 0) {  // task start: finalize operands and row offsets, overlapping the copy
            if (cur.info >= 0) {
                const int nr = (cur.info >> 16) & 0x7fff;
                for (int i = lane; i <= nr; i += 32) ws.rp[i] = (int32_t)(a.row_ptr[cur.r0 + i] - cur.e0);
                p.prefetch_rows((int64_t)cur.r0, nr, lane);
            } else if (cur.hub < 0 && lane == 0) {
                p.prefetch_rows((int64_t)cur.r0, 1, 0);
            }
            part = T(0);
        }
        mbar_wait(&ws.bar[b], (k >> 1) & 1);
        if (cur.info >= 0) {
            engine_rowblock(p, cur, ws, ws.colbuf[b], l1, linf);
        } else {
            const int64_t e = (int64_t)cur.e0 + (int64_t)j * WT_PIECE;
            T gv[K];
            gather_piece(p, ws.colbuf[b], (int)(e & 3), min(task_nnz(cur) - j * WT_PIECE, WT_PIECE), gv);
#pragma unroll
            for (int q = 0; q < K; ++q) part += gv[q];
            if (j + 1 == task_pieces(cur)) engine_chunk_end(p, a, cur, part, l1, linf);
        }
        __syncwarp();
        if (!has_next) {
            if (kbase) *kbase = k + 1;
            break;
        }
        cur = nt;
        j = nj;
        t = ntn;
    }
}

}  // namespace prgpu
