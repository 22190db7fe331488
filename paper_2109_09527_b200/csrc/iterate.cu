// iterate.cu -- the PageRank iteration: K-INIT, K-GATHER (edge stream),
// K-FINALIZE (update + fused contrib + members + fused Delta reduction and stop
// test), the in-place async / No-Sync sweeps, loop perforation, loop control.
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
#include "streamengine.cuh"

namespace prgpu {

// ---------------------------------------------------------------- policies --
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
    __device__ __forceinline__ void st_sum(int64_t r, double s) const { sums[r] = s; }
    __device__ __forceinline__ void emit(int64_t r, double s) const { st_sum(r, s); }
    __device__ __forceinline__ void prep(int64_t, uint32_t) {}
    __device__ __forceinline__ void emit_at(int, int64_t r, double s) const { st_sum(r, s); }
    __device__ __forceinline__ void emit_first(int64_t r, double s) const { st_sum(r, s); }
};

__device__ __forceinline__ void red_add_f64(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// One segment pass of a source-blocked view (blocked.cu): gathers come from
// one L2-resident slice of y; S_seg(r) is added to the parent row's sum.
struct AccumPolicy {
    using T = double;
    static constexpr bool kHot = false;
    const double* y_in;
    double* sums;
    const int32_t* map;  // sub-view row -> parent view row
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
    __device__ __forceinline__ void prep(int64_t base, uint32_t f) {
        if (f) m_first = __ldg(map + base);
#pragma unroll
        for (int j = 0; j < SE_V; ++j)
            if (f & (1u << j)) m[j] = __ldg(map + base + __popc(f & ((1u << j) - 1)));
    }
    __device__ __forceinline__ void emit(int64_t r, double s) const { red_add_f64(sums + map[r], s); }
    __device__ __forceinline__ void emit_at(int j, int64_t, double s) const { red_add_f64(sums + m[j], s); }
    __device__ __forceinline__ void emit_first(int64_t, double s) const { red_add_f64(sums + m_first, s); }
};

// NVLS: one store that lands in the same slot of every team member's buffer
// (p is a multicast address, multicast.cu)
__device__ __forceinline__ void st_mc_f64(double* p, double v) {
    asm volatile("multimem.st.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

struct IterArgs {
    DevState* st;
    double* cta_partial;        // (L1, Linf) per CTA: gather / finalize CTAs, member CTAs, zero-in CTAs
    int64_t gather_ctas;
    int64_t scatter_ctas;
    int64_t zero_ctas;          // > 0 only in the first sweep
    double* delta_log;
    // sharded run: the last CTA writes this rank's (L1, Linf) here (the tail
    // of its exchanged chunk) instead of taking the stop decision; with peer
    // buffers (pr_shard_set_peers) also at peer_y[q] + shard_off of every peer
    double* shard_out = nullptr;
    double* const* peer_y = nullptr;
    int npeer = 0;
    int64_t shard_off = 0;
    double* mc_out = nullptr;   // NVLS: multicast address of the chunk tail (replaces shard_out / peer_y)
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

// Deterministic fixed-order reduction over all CTA partials, then the stop
// test; executed by the last CTA of the sweep.
__device__ void global_finalize(const IterArgs& ia, double* red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __threadfence();
    double s = 0.0, mx = 0.0;
    const int64_t nc = ia.gather_ctas + ia.scatter_ctas + ia.zero_ctas;
    for (int64_t i = tid; i < nc; i += blockDim.x) {
        s += __ldcg(ia.cta_partial + 2 * i);
        mx = fmax(mx, __ldcg(ia.cta_partial + 2 * i + 1));
    }
    s = warp_sum(s);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __syncthreads();
    if (lane == 0) {
        red[warp] = s;
        red[32 + warp] = mx;
    }
    __syncthreads();
    if (tid == 0) {
        double l1 = 0.0, li = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            l1 += red[w];
            li = fmax(li, red[32 + w]);
        }
        DevState* st = ia.st;
        if (ia.mc_out) {
            st_mc_f64(ia.mc_out, l1);
            st_mc_f64(ia.mc_out + 1, li);
        } else if (ia.shard_out) {
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

// (L1, Linf) of the block into out[0..1] (thread 0 writes).  red: 64 doubles.
__device__ __forceinline__ void block_delta(double l1, double linf, double* red, double* out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    l1 = warp_sum(l1);
#pragma unroll
    for (int o = 16; o; o >>= 1) linf = fmax(linf, __shfl_xor_sync(0xffffffffu, linf, o));
    __syncthreads();
    if (lane == 0) {
        red[warp] = l1;
        red[32 + warp] = linf;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += red[w];
            b = fmax(b, red[32 + w]);
        }
        out[0] = a;
        out[1] = b;
    }
}

// Block partial, then the last CTA of the grid (ticket) runs the global
// reduction and the stop test.
__device__ __forceinline__ void partial_and_ticket(const IterArgs& ia, double l1, double linf, double* red,
                                                   int64_t part, uint32_t* ticket, int* flag) {
    block_delta(l1, linf, red, ia.cta_partial + 2 * part);
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t t = atomicAdd(ticket, 1u);
        *flag = (t == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (*flag) global_finalize(ia, red);
}

// ------------------------------------------------------------- K-GATHER --
// Edge-stream form: S(r) of every row of the view into sums[r].  One CTA of
// SE_NT threads per SM; no Delta here (K-FINALIZE computes it).
template <class P>
__global__ void __launch_bounds__(SE_NT, 1) k_stream(P p, StreamArgs a, const DevState* st) {
    extern __shared__ __align__(16) double hot_smem[];
    pdl_wait();
    pdl_trigger();
    if (st->done) return;
    p.pol_last = policy_evict_last();
    if constexpr (P::kHot) {
        const double2* src = reinterpret_cast<const double2*>(p.y_in);
        double2* dst = reinterpret_cast<double2*>(hot_smem);
        for (int i = threadIdx.x; i < (p.hot_n >> 1); i += blockDim.x) dst[i] = __ldcg(src + i);
        if ((p.hot_n & 1) && threadIdx.x == 0) hot_smem[p.hot_n - 1] = __ldcg(p.y_in + p.hot_n - 1);
        p.hot = hot_smem;
        __syncthreads();
    }
    stream_run(p, a);
}

// ----------------------------------------------------------- K-FINALIZE --
// For every row r of the view (sync sweeps)
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
    // loop perforation (PR_PERFORATE, Alg.5): fz[r] is the sticky
    // threshold_check flag of row r.  A flagged row is skipped (keeps x and its
    // contrib, |delta| = 0); an unflagged row whose change this sweep is
    // 0 < |delta| < tau_f is flagged (from the next sweep on) and its contrib
    // is also stored into y_other, the buffer the next sweep writes, so both
    // ping-pong buffers hold its frozen value.
    uint8_t* fz = nullptr;
    double tau_f = 0.0;
    double* y_other = nullptr;
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
    double* mc_y = nullptr;     // NVLS: contribs stored through this multicast address instead
    int vec = 0;                // rows two at a time with 16-byte loads (PRGPU_FIN_VEC)
    // delayed chain resolution (sync reduced mode without PR_CHAIN_EAGER):
    // hist[(t mod L) * nh + h] = x_t of chain source h (L = max_chain + 1
    // sweeps, slot 0 = x_0 = 1/n); chain member m at distance k takes
    // x_t(m) = alpha_j + beta_j * x_{t-j}(h), j = min(k, t)
    double* hist = nullptr;
    const int32_t* mh = nullptr;
    int64_t nh = 0;
    int L = 1;
    // identical members folded into their source row (build_fold): rinfo.x
    // carries FOLD_FLAG on rows with identical members, whose |delta| then
    // counts fold_w[r] = 1 + #members times (x_t(m) = x_t(rep) exactly, so
    // |x_t(m) - x_{t-1}(m)| is the row's own); the member loop visits only
    // fold_list (chain members) and the packed fold_rec records (identical
    // members with outdeg > 0: their contrib and nothing else, one record load
    // then the source row's S); k_unpermute takes their x from the row
    int fold = 0;
    const int32_t* fold_w = nullptr;
    const int32_t* fold_list = nullptr;  // the chain members (nm of them)
    const int4* fold_rec = nullptr;      // identical members with a contrib: (source row, outdeg, slot, -)
    int64_t nrec = 0;
    const int4* fold_crec = nullptr;     // the chain members: (source row, hist index, slot, k), list order
    double* xc = nullptr;                // x of the chain members, list order
};
constexpr int32_t FOLD_FLAG = 1 << 30;
constexpr int32_t FOLD_MASK = FOLD_FLAG - 1;

// Rows are visited grid-stride (all CTAs sweep the row space together, which
// keeps the TLB working set small) in batches of FIN_U rows per thread whose
// loads are all issued before any store.  Every access is coalesced except the
// contrib store y[slot]; x is kept in row / member order (xr, xm) during the
// sweeps and written back to vertex order once, by k_unpermute.
// FIN_U = 2 with 4 CTAs/SM (64 registers, no spills): R-MAT-24 reduced 0.0762
// -> 0.0723 ms against FIN_U = 4 at 73 registers / 3 CTAs/SM (FIN_U = 8: 0.0845;
// 4 pairs / thread: 0.085; profiles/r2/ab_fin.txt)
#ifndef PRGPU_FIN_U
#define PRGPU_FIN_U 2
#endif
#ifndef PRGPU_FIN_MINB
#define PRGPU_FIN_MINB 4
#endif
constexpr int FIN_U = PRGPU_FIN_U;
#ifndef PRGPU_FIN_PAIRS
#define PRGPU_FIN_PAIRS 2
#endif
constexpr int FIN_PAIRS = PRGPU_FIN_PAIRS;
// (the folded rows' Delta weights loaded with the row data, 8 B per row pair,
// instead of after the flag test measured the same: R-MAT-24 reduced 0.0681
// vs 0.0680 ms, profiles/r2/ab_fin_chainrec.jsonl; the thread's first 1 / 2
// folded-member records and their S loaded during the rows loop spill at 64
// registers and measured slower: 0.0717 / 0.0754 vs 0.0679 ms,
// profiles/r2/ab_fin_recpre.jsonl)  // row pairs per thread and iteration of the 16-byte path

// One new contrib: this buffer (and every peer's), or one multicast store.
template <bool REMOTE>
__device__ __forceinline__ void fin_store_y(const FinArgs& f, double* y, int32_t slot, double yv) {
    if (!REMOTE) {
        y[slot] = yv;
    } else if (f.mc_y) {
        st_mc_f64(f.mc_y + slot, yv);
    } else {
        y[slot] = yv;
        for (int q = 0; q < f.npeer; ++q) f.peer_y[q][slot] = yv;
    }
}

// REMOTE: the sharded sweep with peer buffers or a multicast team (every
// contrib also stored remotely); the plain instance keeps fewer registers.
template <bool REMOTE>
__global__ void __launch_bounds__(GT_NT, PRGPU_FIN_MINB) k_finalize(FinArgs f, IterArgs ia) {
    __shared__ double red[64];
    __shared__ int flag;
    pdl_wait();
    pdl_trigger();
    if (ia.st->done) return;
    double l1 = 0.0, linf = 0.0;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const double* __restrict__ sums = f.sums;
    double* __restrict__ xr = f.xr;
    double* __restrict__ y = f.y_out;
    uint32_t nfrozen = 0;
    int64_t rlo = f.row0;  // rows [rlo, nrows) left to the general loop below
    if (f.vec && !f.fz && (f.row0 & 1) == 0) {
        // two consecutive rows per 16-byte load of S, x and (outdeg, slot)
        const double2* __restrict__ S2 = reinterpret_cast<const double2*>(sums);
        double2* __restrict__ X2 = reinterpret_cast<double2*>(xr);
        const int4* __restrict__ I2 = reinterpret_cast<const int4*>(f.rinfo);
        const int64_t p_end = f.nrows >> 1;
        constexpr int FP = FIN_PAIRS;
        for (int64_t p0 = (f.row0 >> 1) + t0; p0 < p_end; p0 += FP * T) {
            double2 sv[FP], xv[FP];
            int4 iv[FP];
#pragma unroll
            for (int u = 0; u < FP; ++u) {
                const int64_t p = p0 + u * T;
                if (p < p_end) {
                    sv[u] = __ldcs(S2 + p);
                    xv[u] = X2[p];
                    iv[u] = __ldg(I2 + p);
                }
            }
#pragma unroll
            for (int u = 0; u < FP; ++u) {
                const int64_t p = p0 + u * T;
                if (p < p_end) {
                    const double xa = __dadd_rn(f.c, __dmul_rn(f.d, sv[u].x));
                    const double xb = __dadd_rn(f.c, __dmul_rn(f.d, sv[u].y));
                    X2[p] = make_double2(xa, xb);
                    const int32_t oa = f.fold ? (iv[u].x & FOLD_MASK) : iv[u].x;
                    const int32_t ob = f.fold ? (iv[u].z & FOLD_MASK) : iv[u].z;
                    if (oa > 0) fin_store_y<REMOTE>(f, y, iv[u].y, xa / (double)oa);
                    if (ob > 0) fin_store_y<REMOTE>(f, y, iv[u].w, xb / (double)ob);
                    const double da = fabs(xa - xv[u].x), db = fabs(xb - xv[u].y);
                    linf = fmax(linf, fmax(da, db));
                    if (f.fold && ((iv[u].x | iv[u].z) & FOLD_FLAG)) {
                        l1 += (iv[u].x & FOLD_FLAG) ? da * (double)__ldg(f.fold_w + 2 * p) : da;
                        l1 += (iv[u].z & FOLD_FLAG) ? db * (double)__ldg(f.fold_w + 2 * p + 1) : db;
                    } else {
                        l1 += da;
                        l1 += db;
                    }
                }
            }
        }
        rlo = p_end << 1;  // the odd last row, if any
    }
    for (int64_t r0 = rlo + t0; r0 < f.nrows; r0 += FIN_U * T) {
        double S[FIN_U], xo[FIN_U];
        int2 inf[FIN_U];
        uint8_t fr[FIN_U];
#pragma unroll
        for (int u = 0; u < FIN_U; ++u) {
            const int64_t r = r0 + u * T;
            fr[u] = 0;
            if (r < f.nrows) {
                S[u] = __ldcs(sums + r);
                xo[u] = xr[r];
                inf[u] = __ldg(f.rinfo + r);
                if (f.fz) fr[u] = f.fz[r];
            }
        }
#pragma unroll
        for (int u = 0; u < FIN_U; ++u) {
            const int64_t r = r0 + u * T;
            if (r < f.nrows && !fr[u]) {
                const double xn = __dadd_rn(f.c, __dmul_rn(f.d, S[u]));
                xr[r] = xn;
                const int32_t od = f.fold ? (inf[u].x & FOLD_MASK) : inf[u].x;
                const double yv = od > 0 ? xn / (double)od : 0.0;
                if (od > 0) fin_store_y<REMOTE>(f, y, inf[u].y, yv);
                const double dl = fabs(xn - xo[u]);
                l1 += (f.fold && (inf[u].x & FOLD_FLAG)) ? dl * (double)__ldg(f.fold_w + r) : dl;
                linf = fmax(linf, dl);
                if (f.fz && dl != 0.0 && dl < f.tau_f) {  // threshold_check <- True (Alg.5)
                    f.fz[r] = 1;
                    ++nfrozen;
                    if (inf[u].x > 0) f.y_other[inf[u].y] = yv;
                }
            }
        }
    }
    if (f.fz) {
        nfrozen = warp_sum(nfrozen);
        if ((threadIdx.x & 31) == 0 && nfrozen) atomicAdd(f.nfz, (unsigned long long)nfrozen);
    }
    if (f.fold) {  // folded identical members with a contrib: y = (c + d*S(source row)) / outdeg
        for (int64_t j0 = t0; j0 < f.nrec; j0 += FIN_U * T) {
            int4 rc[FIN_U];
            double S[FIN_U];
#pragma unroll
            for (int u = 0; u < FIN_U; ++u)
                if (j0 + u * T < f.nrec) rc[u] = __ldg(f.fold_rec + j0 + u * T);
#pragma unroll
            for (int u = 0; u < FIN_U; ++u)
                if (j0 + u * T < f.nrec) S[u] = sums[rc[u].x];
#pragma unroll
            for (int u = 0; u < FIN_U; ++u)
                if (j0 + u * T < f.nrec) y[rc[u].z] = __dadd_rn(f.c, __dmul_rn(f.d, S[u])) / (double)rc[u].y;
        }
    }
    double* __restrict__ xm = f.xm;
    const int t_sw = f.hist ? ia.st->iters + 1 : 0;  // this sweep's number (delayed chains)
    if (f.fold_crec) {
        // folded sweep: the chain members from their packed records (list
        // order, x in xc), every operand one level below the record: delayed,
        // only the distance-1 member (the writer of its source's history)
        // needs S of the source row; the value it resolves from is the
        // history slot of the sweep j = min(k, t) ago (never this sweep's)
        for (int64_t j0 = t0; j0 < f.nm; j0 += FIN_U * T) {
            int4 rc[FIN_U];
            double S[FIN_U], xo[FIN_U], hx[FIN_U];
#pragma unroll
            for (int u = 0; u < FIN_U; ++u) {
                const int64_t j = j0 + u * T;
                if (j < f.nm) {
                    rc[u] = __ldg(f.fold_crec + j);
                    xo[u] = f.xc[j];
                }
            }
#pragma unroll
            for (int u = 0; u < FIN_U; ++u) {
                if (j0 + u * T < f.nm) {
                    if (f.hist) {
                        const int jj = min(rc[u].w, t_sw);
                        hx[u] = f.hist[(int64_t)((t_sw - jj) % f.L) * f.nh + rc[u].y];
                        if (rc[u].w == 1) S[u] = sums[rc[u].x];
                    } else {
                        S[u] = sums[rc[u].x];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < FIN_U; ++u) {
                const int64_t jl = j0 + u * T;
                if (jl < f.nm) {
                    int j = rc[u].w;
                    double xsrc;
                    if (f.hist) {
                        if (j == 1) f.hist[(int64_t)(t_sw % f.L) * f.nh + rc[u].y] = __dadd_rn(f.c, __dmul_rn(f.d, S[u]));
                        j = min(j, t_sw);
                        xsrc = hx[u];
                    } else {
                        xsrc = __dadd_rn(f.c, __dmul_rn(f.d, S[u]));
                    }
                    const double xn = __dadd_rn(f.ab[2 * j], __dmul_rn(f.ab[2 * j + 1], xsrc));
                    f.xc[jl] = xn;
                    y[rc[u].z] = xn;  // out-degree 1: xn / 1
                    const double dl = fabs(xn - xo[u]);
                    l1 += dl;
                    linf = fmax(linf, dl);
                }
            }
        }
    }
    for (int64_t j0 = t0; j0 < (f.fold_crec ? 0 : f.nm); j0 += FIN_U * T) {
        double S[FIN_U], xo[FIN_U];
        int32_t k[FIN_U];
        int2 inf[FIN_U];
        int64_t mi[FIN_U];
#pragma unroll
        for (int u = 0; u < FIN_U; ++u) {
            const int64_t j = j0 + u * T;
            if (j < f.nm) {
                const int64_t i = f.fold ? (int64_t)__ldg(f.fold_list + j) : j;
                mi[u] = i;
                k[u] = __ldg(f.mk + i);
                S[u] = sums[__ldg(f.msrow + i)];
                if (!(f.fold && k[u] == 0)) xo[u] = xm[i];
                inf[u] = __ldg(f.minfo + i);
            }
        }
#pragma unroll
        for (int u = 0; u < FIN_U; ++u) {
            const int64_t i = mi[u];
            if (j0 + u * T < f.nm) {
                const double xs = __dadd_rn(f.c, __dmul_rn(f.d, S[u]));
                if (f.fold && k[u] == 0) {  // folded identical member: its contrib only
                    if (inf[u].x > 0) y[inf[u].y] = xs / (double)inf[u].x;
                    continue;
                }
                int j = k[u];
                double xsrc = xs;
                if (f.hist && j > 0) {  // delayed: the source's value j sweeps ago (Eq.(1) along the chain)
                    const int64_t h = __ldg(f.mh + i);
                    if (j == 1) f.hist[(int64_t)(t_sw % f.L) * f.nh + h] = xs;  // one writer value per source
                    j = min(j, t_sw);
                    xsrc = f.hist[(int64_t)((t_sw - j) % f.L) * f.nh + h];
                }
                const double xn = __dadd_rn(f.ab[2 * j], __dmul_rn(f.ab[2 * j + 1], xsrc));
                xm[i] = xn;
                if (inf[u].x > 0) y[inf[u].y] = xn / (double)inf[u].x;
                const double dl = fabs(xn - xo[u]);
                l1 += dl;
                linf = fmax(linf, dl);
            }
        }
    }
    if (!f.last) {
        block_delta(l1, linf, red, ia.cta_partial + 2 * (f.part_off + blockIdx.x));
        return;
    }
    partial_and_ticket(ia, l1, linf, red, f.part_off + blockIdx.x, &ia.st->ticket_gather, &flag);
}

// x in vertex order from the row / member ordered state.
// (mk, msrow given: the sweeps folded the identical members (k = 0) into their
// source row, whose x they take)
// (clist, xc given: the chain members' x is xc in clist order)
__global__ void k_unpermute(const double* __restrict__ xr, const int32_t* __restrict__ vid, int64_t nrows,
                            const double* __restrict__ xm, const int32_t* __restrict__ mvid, int64_t nm,
                            double* __restrict__ x, const int32_t* __restrict__ mk = nullptr,
                            const int32_t* __restrict__ msrow = nullptr, const int32_t* __restrict__ clist = nullptr,
                            const double* __restrict__ xc = nullptr, int64_t nc = 0) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += T) x[vid ? vid[r] : r] = xr[r];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nm; i += T) {
        if (mk && mk[i] == 0)
            x[mvid[i]] = xr[msrow[i]];
        else if (!xc)
            x[mvid[i]] = xm[i];
    }
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nc; j += T) x[mvid[clist[j]]] = xc[j];
}

// build_fold: multiplicity of every row with identical members, flagged rinfo,
// and the members that keep per-sweep work
__global__ void k_fold_count(const int32_t* __restrict__ mk, const int32_t* __restrict__ msrow, int64_t nm,
                             int32_t* __restrict__ w) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nm; i += (int64_t)gridDim.x * blockDim.x)
        if (mk[i] == 0) atomicAdd(w + msrow[i], 1);
}
__global__ void k_fold_rows(const int2* __restrict__ rinfo, int64_t nrows, int32_t* __restrict__ w,
                            int2* __restrict__ out) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        int2 ri = rinfo[r];
        const int32_t c = w[r];
        if (c > 0) {
            ri.x |= FOLD_FLAG;
            w[r] = c + 1;
        }
        out[r] = ri;
    }
}

// One 16-byte record per chain member in fold_list order, so the member loop
// of K-FINALIZE issues one coalesced load instead of a list load followed by
// five dependent ones.  A chain member has out-degree 1 by definition
// (preprocess.cu: chain(v) <=> indeg 1 and outdeg 1), so its contrib is its x.
__global__ void k_fold_crec(const int32_t* __restrict__ list, int64_t nc, const int32_t* __restrict__ msrow,
                            const int32_t* __restrict__ mh, const int2* __restrict__ minfo,
                            const int32_t* __restrict__ mk, int4* __restrict__ rec) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nc; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = list[j];
        rec[j] = make_int4(msrow[i], mh ? mh[i] : -1, minfo[i].y, mk[i]);
    }
}

__global__ void k_fill_f64(double* __restrict__ a, int64_t cnt, double v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}

// First sweep for the vertices of in-degree 0: Eq.(1) with an empty sum gives
// x_t = (1-d)/n = c for every t >= 1, so they are written here once (x and
// the contrib slot of y_out) and contribute |c - 1/n| to Delta_1 only; from
// sweep 2 on their Delta is exactly 0 and no kernel touches them.
__global__ void __launch_bounds__(GT_NT) k_zero(const int32_t* __restrict__ zl, int64_t nz, double c, double* x,
                                                double* y_out, const int32_t* __restrict__ od,
                                                const int32_t* __restrict__ cidx, double* partial, int mc = 0) {
    // grid-stride, 4 vertices per thread with all loads issued first (the
    // old x is read too: it is 1/n from k_init, but Delta_1 must be measured)
    __shared__ double red[64];
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
                if (o[u] > 0) {
                    if (mc)
                        st_mc_f64(y_out + ci[u], c / (double)o[u]);
                    else
                        y_out[ci[u]] = c / (double)o[u];
                }
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
                         const int32_t* __restrict__ od, const int32_t* __restrict__ cidx, int mc = 0) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nz; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = zl[i];
        const int32_t o = od[v];
        if (o > 0) {
            if (mc)
                st_mc_f64(y + cidx[v], c / (double)o);
            else
                y[cidx[v]] = c / (double)o;
        }
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
struct InPlacePolicy {
    using T = double;
    static constexpr bool kHot = true;
    const double* y_in;   // == y: relaxed loads
    double* y;            // relaxed stores
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
    // loop perforation in place (No-Sync-Opt, Alg.5; reading Q-P):
    // fz[r] = sticky threshold_check flag of row r (nullptr: off)
    uint8_t* fz;
    double tau_f;
    unsigned long long* nfz;  // flags set, counted per thread, added at the end
    uint32_t nfrozen;

    __device__ __forceinline__ double load(int32_t u) const {
        if (u < hot_n) return hot[u];
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
        if (fz && fz[r]) return;  // flagged: keeps x and its contrib, |delta| = 0
        const double xn = __dadd_rn(c, __dmul_rn(d, s));
        st_relaxed_f64(xr + r, xn);
        if (q.x > 0) st_relaxed_f64(y + q.y, xn / (double)q.x);
        const double dl = fabs(xn - xold);
        l1 += dl;
        linf = fmax(linf, dl);
        if (fz && dl != 0.0 && dl < tau_f) {  // threshold_check <- True (Alg.5)
            fz[r] = 1;
            ++nfrozen;
        }
    }
    __device__ __forceinline__ void flush_frozen() const {
        if (nfrozen) atomicAdd(nfz, (unsigned long long)nfrozen);
    }
    __device__ __forceinline__ void emit(int64_t r, double s) { fin(r, s, __ldg(rinfo + r), ld_relaxed_f64(xr + r)); }
    __device__ __forceinline__ void emit_at(int j, int64_t r, double s) { fin(r, s, inf[j], xo[j]); }
    __device__ __forceinline__ void emit_first(int64_t r, double s) { fin(r, s, inf_f, xo_f); }
};

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

__device__ __forceinline__ void members_inplace(const MemArgs& ma, const double* xr, double* y, double& l1,
                                                double& linf) {
    const int64_t mb = (int64_t)blockIdx.x * ma.mper;
    const int64_t me = min(ma.nm, mb + ma.mper);
    for (int64_t i = mb + threadIdx.x; i < me; i += blockDim.x) {
        const int32_t k = ma.mk[i];
        const double xs = ld_relaxed_f64(xr + ma.msrow[i]);
        const double xn = __dadd_rn(ma.ab[2 * k], __dmul_rn(ma.ab[2 * k + 1], xs));
        const double xo = ma.xm[i];
        ma.xm[i] = xn;
        const int2 q = ma.minfo[i];
        if (q.x > 0) st_relaxed_f64(y + q.y, xn / (double)q.x);
        const double dl = fabs(xn - xo);
        l1 += dl;
        linf = fmax(linf, dl);
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
    __shared__ double red[64];
    __shared__ int flag;
    if (ia.st->done) return;
    p.pol_last = 0;
    refresh_hot(p, hot_smem);
    p.l1 = 0.0;
    p.linf = 0.0;
    stream_run(p, a);
    members_inplace(ma, p.xr, p.y, p.l1, p.linf);
    if (p.fz) p.flush_frozen();
    partial_and_ticket(ia, p.l1, p.linf, red, blockIdx.x, &ia.st->ticket_gather, &flag);
}

// ------------------------------------------------------ No-Sync --
// Persistent barrier-free kernel (Alg.3 "No-Sync"): every CTA sweeps
// its own static spans (and member slice) in place -- gathers read whatever
// contribs are visible (relaxed loads), every row's x and y are written at once
// (relaxed stores) -- and after each local sweep publishes its (L1, L-inf)
// delta; it stops when the sum (L1) / max (L-inf) over the deltas all CTAs last
// published is <= tau ("thread-level convergence", with the
// per-iteration reset of Q-E).  No grid barrier: a CTA never waits for another
// one.  Grid = resident CTAs only (a CTA must not wait for an unscheduled
// CTA's first delta, which starts at +big).
struct NoSyncArgs {
    double* err;        // [2 * grid] (L1, Linf) of each CTA's last local sweep
    int32_t* iters;     // [grid] local sweeps of each CTA, over all launches
    int norm_linf;
    double tau;
    int32_t max_local;  // local sweeps allowed in this launch
};

__global__ void __launch_bounds__(SE_NT_IP, 1) k_nosync_stream(InPlacePolicy p, StreamArgs a, MemArgs ma, NoSyncArgs na) {
    extern __shared__ __align__(16) double hot_smem[];
    __shared__ double red[64];
    __shared__ double res[2];
    __shared__ int flag;
    p.pol_last = 0;
    for (int it = 1;; ++it) {
        refresh_hot(p, hot_smem);
        p.l1 = 0.0;
        p.linf = 0.0;
        stream_run(p, a);
        members_inplace(ma, p.xr, p.y, p.l1, p.linf);
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
    if (p.fz) p.flush_frozen();
}

// Certificate of an in-place result: ||F(x) - x|| of the ORIGINAL system, with
// S(r) from one synchronous edge-stream gather of the plain view over the
// current contribs (F(x) = c + d*M*x, Eq.(1)); ||x - x*||_1 <= ||F(x)-x||_1/(1-d).
// (Sum by atomics: not bit-reproducible in its last digits; it is a check.)
__global__ void k_residual(const double* __restrict__ sums, int64_t nrows, const int32_t* __restrict__ vid,
                           const double* __restrict__ x, double c, double d, double* out) {
    __shared__ double red[64];
    __shared__ double res[2];
    double l1 = 0.0, linf = 0.0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = vid ? vid[r] : (int32_t)r;
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

// ------------------------------------------------------------------- host --

struct GatherCfg {
    int hot_n = 0;
    size_t smem = 0;
    int grid = 1;
    int nt = SE_NT;
};

static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}

static StreamArgs stream_args(const View& w) {
    return StreamArgs{w.col,  (const uint8_t*)w.sflags, w.step_row, w.nsteps, w.span_steps, w.nspans, w.bin,
                      w.bout, w.b_row, w.b_s0, w.b_s1, w.part_in, w.part_out, w.bticket};
}

// Kernel, dynamic shared memory and persistent grid (resident CTAs, capped by
// the spans to run) of a gather over v: synchronous (k_stream) or in place
// (k_stream_async / k_nosync_stream).
enum GatherKind { G_SYNC, G_INPLACE };
static int gather_config(Ctx& ctx, const View& v, pr_graph* g, GatherKind kind, GatherCfg* gc) {
    const void* fn = nullptr;
    if (kind == G_SYNC) {
        int hot = v.nseg > 0 ? 0 : env_int("PRGPU_HOT", SE_HOT_MAX);
        gc->hot_n = std::max(0, std::min<int>(std::min(hot, SE_HOT_MAX), (int)g->n_contrib));
        gc->nt = SE_NT;
        fn = gc->hot_n > 0 ? (const void*)k_stream<StreamPolicy<true>> : (const void*)k_stream<StreamPolicy<false>>;
        if (v.nseg > 0) fn = (const void*)k_stream<AccumPolicy>;
    } else {
        int hot = env_int("PRGPU_HOT", SE_HOT_IP);
        gc->hot_n = std::max(0, std::min<int>(std::min(hot, SE_HOT_MAX), (int)g->n_contrib));
        gc->nt = SE_NT_IP;
        fn = (const void*)k_stream_async;
    }
    gc->smem = (size_t)gc->hot_n * sizeof(double);
    PR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gc->smem));
    if (kind == G_INPLACE)
        PR_CUDA(cudaFuncSetAttribute((const void*)k_nosync_stream, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)gc->smem));
    int per_sm = 0;
    PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, gc->nt, gc->smem));
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)ctx.num_sms * per_sm;
    int64_t units = v.nspans;
    if (v.nseg > 0) {
        units = 0;
        for (int q = 0; q < v.nseg; ++q) units = std::max<int64_t>(units, v.seg[q].nspans);
    }
    if (v.phv)
        for (int k = 0; k < v.phv_k; ++k) units = std::max<int64_t>(units, v.phv[k].nspans);
    const int wpc = gc->nt / 32;
    const int64_t ctas_needed = (units + wpc - 1) / wpc;
    gc->grid = (int)std::max<int64_t>(1, std::min(grid, ctas_needed));
    return PR_OK;
}

// Synchronous K-GATHER of view v into sums (the view's own sums unless given):
// one launch, or one accumulating launch per slot segment of a blocked view.
static int launch_gather(Ctx& ctx, pr_graph* g, const View& v, const double* y_in, const GatherCfg& gc,
                         double* sums = nullptr) {
    if (!sums) sums = v.sums;
    if (v.nseg > 0) {  // source-blocked: S = 0, then one accumulating pass per slot segment
        PR_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * (size_t)v.nrows, ctx.stream));
        for (int q = 0; q < v.nseg; ++q) {
            const View& sv = v.seg[q];
            if (sv.nspans == 0) continue;
            AccumPolicy p{y_in, sums, sv.vid, 0, 0, {}};
            PR_LAUNCH_PDL(ctx, k_stream<AccumPolicy>, gc.grid, gc.nt, 0, p, stream_args(sv), (const DevState*)g->st);
        }
    } else if (v.nspans > 0) {
        if (gc.hot_n > 0) {
            StreamPolicy<true> p{y_in, sums, nullptr, gc.hot_n, 0};
            PR_LAUNCH_PDL(ctx, k_stream<StreamPolicy<true>>, gc.grid, gc.nt, gc.smem, p, stream_args(v),
                          (const DevState*)g->st);
        } else {
            StreamPolicy<false> p{y_in, sums, nullptr, 0, 0};
            PR_LAUNCH_PDL(ctx, k_stream<StreamPolicy<false>>, gc.grid, gc.nt, gc.smem, p, stream_args(v),
                          (const DevState*)g->st);
        }
    }
    return PR_OK;
}

// Identical members folded into their source row (FinArgs::fold): tables
// built once per preprocess, on the first sync reduced run that uses them.
struct FoldChainGet {
    const int32_t* mk;
    __device__ int64_t operator()(int64_t i) const { return mk[i] > 0 ? 1 : 0; }
};
struct FoldChainEmit {
    int32_t* list;
    __device__ void operator()(int64_t i, int64_t pos, int64_t f) const {
        if (f) list[pos] = (int32_t)i;
    }
};
struct FoldRecGet {
    const int32_t* mk;
    const int2* minfo;
    __device__ int64_t operator()(int64_t i) const { return (mk[i] == 0 && minfo[i].x > 0) ? 1 : 0; }
};
struct FoldRecEmit {
    const int32_t* msrow;
    const int2* minfo;
    int4* rec;
    __device__ void operator()(int64_t i, int64_t pos, int64_t f) const {
        if (f) rec[pos] = make_int4(msrow[i], minfo[i].x, minfo[i].y, 0);
    }
};
static int build_fold(pr_graph* g, Ctx& ctx, const View& v) {
    if (g->fold_ready) return PR_OK;
    cudaStream_t s = ctx.stream;
    const int64_t nm = g->n_members;
    int64_t* cnt = nullptr;
    TmpGuard tg_(s);
    tg_.track(cnt);
    PR_TRY(dalloc(&g->fold_w, (size_t)v.nrows, s));
    PR_CUDA(cudaMemsetAsync(g->fold_w, 0, sizeof(int32_t) * (size_t)v.nrows, s));
    PR_TRY(dalloc(&g->fold_rinfo, (size_t)v.nrows, s));
    PR_TRY(dalloc(&g->fold_list, (size_t)nm, s));
    PR_TRY(dalloc(&cnt, 2, s));
    const unsigned gm = (unsigned)std::min<int64_t>((nm + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
    const unsigned gr = (unsigned)std::min<int64_t>((v.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
    PR_LAUNCH(ctx, k_fold_count, gm, 256, 0, (const int32_t*)g->mem_k, (const int32_t*)g->mem_srow, nm, g->fold_w);
    PR_LAUNCH(ctx, k_fold_rows, gr, 256, 0, (const int2*)v.rinfo, v.nrows, g->fold_w, g->fold_rinfo);
    PR_TRY(dalloc(&g->fold_rec, (size_t)nm, s));
    PR_TRY((device_scan<int64_t>(ctx, nm, FoldChainGet{g->mem_k}, FoldChainEmit{g->fold_list}, cnt)));
    PR_TRY((device_scan<int64_t>(ctx, nm, FoldRecGet{g->mem_k, g->mem_info},
                                 FoldRecEmit{g->mem_srow, g->mem_info, g->fold_rec}, cnt + 1)));
    int64_t hc[2];
    PR_CUDA(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
    PR_CUDA(cudaStreamSynchronize(s));
    g->fold_n = hc[0];
    g->fold_nrec = hc[1];
    if (g->fold_n > 0) {
        PR_TRY(dalloc(&g->fold_crec, (size_t)g->fold_n, s));
        PR_TRY(dalloc(&g->fold_xc, (size_t)g->fold_n, s));
        const unsigned gc = (unsigned)std::min<int64_t>((g->fold_n + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
        PR_LAUNCH(ctx, k_fold_crec, gc, 256, 0, (const int32_t*)g->fold_list, g->fold_n, (const int32_t*)g->mem_srow,
                  (const int32_t*)g->mem_h, (const int2*)g->mem_info, (const int32_t*)g->mem_k, g->fold_crec);
    }
    g->fold_ready = true;
    return PR_OK;
}

// PR_MODE_PHASED: K row-aligned phases (build_phase_view; reading Q-B).
static int phase_plan(pr_graph* g, bool reduced, Ctx& ctx, int* K_out) {
    View& v = reduced ? g->reduced : g->plain;
    if (v.alias) {  // an aliased reduced view shares the plain view's plan
        PR_TRY(phase_plan(g, false, ctx, K_out));
        g->reduced = g->plain;
        g->reduced.alias = true;
        return PR_OK;
    }
    // default: 8 phases when every phase still gives each resident warp >= 24
    // steps of 256 edges (R-MAT-24: 8); fewer on small graphs, where the
    // ~15-20 us a phase costs (two launches, ramp and tail) outweighs the saved
    // sweeps
    const int64_t warps = (int64_t)ctx.num_sms * (SE_NT / 32);
    int K = env_int("PRGPU_PHASES", (int)std::min<int64_t>(8, v.nsteps / (warps * 24)));
    K = std::max(1, std::min(K, SE_MAX_PHASES));
    if (v.nseg > 0 || v.nspans == 0) K = 1;  // source-blocked views run one phase (an in-place Jacobi sweep)
    *K_out = K;
    if (K == 1) {
        free_phase_view(v, ctx.stream);
        v.phase_rb[0] = 0;
        v.phase_rb[1] = v.nrows;
        v.phase_eb[0] = 0;
        v.phase_eb[1] = v.nedges;
        v.phase_k = 1;
        return PR_OK;
    }
    return build_phase_view(v, ctx, K, (int32_t)g->n_contrib);
}

// Boundary-row tickets count the pieces of the current sweep.  A persistent
// No-Sync launch stops with CTAs at different sweeps, so tickets can be left
// mid-count; every run starts from zero.
static int reset_tickets(const View& v, cudaStream_t s) {
    if (v.bticket && v.nbound > 0) PR_CUDA(cudaMemsetAsync(v.bticket, 0, sizeof(uint32_t) * (size_t)v.nbound, s));
    for (int q = 0; q < v.nseg; ++q) PR_TRY(reset_tickets(v.seg[q], s));
    if (v.phv)
        for (int k = 0; k < v.phv_k; ++k) PR_TRY(reset_tickets(v.phv[k], s));
    return PR_OK;
}

// ---- shared set-up of a run --
struct RunBufs {
    double* x;          // ranks in vertex order (the caller's device buffer, or g->x)
    bool ranks_dev;
};

static int run_buffers(pr_graph* g, Ctx& ctx, double* ranks, int32_t max_iter, RunBufs* rb) {
    cudaStream_t s = ctx.stream;
    cudaPointerAttributes at{};
    rb->ranks_dev = cudaPointerGetAttributes(&at, ranks) == cudaSuccess &&
                    (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    rb->x = ranks;
    if (!rb->ranks_dev) {
        if (!g->x) PR_TRY(dalloc(&g->x, (size_t)g->n, s));
        rb->x = g->x;
    }
    // contrib slots [0, n_contrib) + slot n_contrib = +0.0, the pad of the stream engine
    for (int b = 0; b < 2; ++b)
        if (!g->y[b]) {
            PR_TRY(dalloc(&g->y[b], (size_t)g->n_contrib + 1, s));
            PR_CUDA(cudaMemsetAsync(g->y[b] + g->n_contrib, 0, sizeof(double), s));
        }
    const int64_t need_xr = std::max<int64_t>(std::max(g->plain.nrows, g->reduced.nrows), 1);
    if (g->xr_cap < need_xr) {
        dfree(g->xr, s);
        PR_TRY(dalloc(&g->xr, (size_t)need_xr, s));
        g->xr_cap = need_xr;
    }
    if (g->n_members > 0 && !g->xm) PR_TRY(dalloc(&g->xm, (size_t)g->n_members, s));
    const int log_cap = max_iter < 4096 ? max_iter : 4096;
    if (g->log_cap < log_cap) {
        dfree(g->delta_log, s);
        PR_TRY(dalloc(&g->delta_log, (size_t)(2 * log_cap), s));
        g->log_cap = log_cap;
    }
    return PR_OK;
}

static int ensure_partials(pr_graph* g, Ctx& ctx, int64_t need) {
    if (g->partial_cap < need) {
        dfree(g->cta_partial, ctx.stream);
        PR_TRY(dalloc(&g->cta_partial, (size_t)need, ctx.stream));
        g->partial_cap = need;
    }
    return PR_OK;
}

// chain alpha_k / beta_k (a6): alpha_0 = 0, beta_0 = 1 (identical copy),
// alpha_{k+1} = c + d alpha_k, beta_{k+1} = d beta_k (Q-C)
static int upload_ab(pr_graph* g, Ctx& ctx, double c, double d) {
    std::vector<double> ab(2 * ((size_t)g->max_chain + 1));
    ab[0] = 0.0;
    ab[1] = 1.0;
    for (int k = 1; k <= g->max_chain; ++k) {
        ab[2 * k] = c + d * ab[2 * (k - 1)];
        ab[2 * k + 1] = d * ab[2 * (k - 1) + 1];
    }
    dfree(g->ab, ctx.stream);
    PR_TRY(dalloc(&g->ab, ab.size(), ctx.stream));
    PR_CUDA(cudaMemcpyAsync(g->ab, ab.data(), ab.size() * sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
    return PR_OK;
}

// Device state for a run, x_0 = 1/n, y_0 (k_init) and the row / member x.
static int init_state(pr_graph* g, Ctx& ctx, double tau, int32_t max_iter, uint32_t mode, double* x,
                      const int32_t* cidx, double* y0, const View& v, int64_t nm) {
    cudaStream_t s = ctx.stream;
    const int64_t n = g->n;
    DevState* hs = g->st_host;
    *hs = DevState{};
    hs->max_iter = max_iter;
    hs->norm_linf = (mode & PR_NORM_LINF) ? 1 : 0;
    hs->tau = tau;
    hs->log_cap = max_iter < 4096 ? max_iter : 4096;
    PR_CUDA(cudaMemcpyAsync(g->st, hs, sizeof(DevState), cudaMemcpyHostToDevice, s));
    PR_LAUNCH(ctx, k_init, (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx.num_sms * 16), 256, 0, x, y0,
              (const int32_t*)g->outdeg, cidx, n, 1.0 / (double)n);
    const unsigned fg = (unsigned)std::min<int64_t>((v.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
    PR_LAUNCH(ctx, k_fill_f64, fg, 256, 0, g->xr, v.nrows, 1.0 / (double)n);
    if (nm > 0) PR_LAUNCH(ctx, k_fill_f64, fg, 256, 0, g->xm, nm, 1.0 / (double)n);
    return PR_OK;
}

// Batches of sweeps launched back to back with one host read of the device
// state per batch.  Batches start at 8 and double; once two batch-end deltas
// exist the next batch is the number of sweeps a geometric fit of them
// predicts until the stop test, + 1 (capped at 64), so few no-op sweeps are
// launched past convergence (every kernel returns at once when done is set).
// sweep(it) enqueues sweep `it`; after(it_end) runs after each host sync.
struct LoopStats {
    int host_syncs = 0;
};
template <class F, class A>
static int sweep_loop(pr_graph* g, Ctx& ctx, int32_t max_iter, double tau, F&& sweep, A&& after, LoopStats& ls) {
    cudaStream_t s = ctx.stream;
    DevState* hs = g->st_host;
    int64_t launched = 0;
    int batch = 8;
    int32_t prev_it = 0;
    double prev_dn = 0.0;
    while (true) {
        const int nb = (int)std::min<int64_t>(batch, max_iter - launched);
        for (int j = 0; j < nb; ++j) PR_TRY(sweep(launched + j));
        PR_CUDA(cudaMemcpyAsync(hs, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        PR_CUDA(cudaStreamSynchronize(s));
        ++ls.host_syncs;
        launched += nb;
        PR_TRY(after(launched));
        if (hs->done || launched >= max_iter) break;
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
    return PR_OK;
}

// PR_TIMING: CUDA events around the gather and the finalize of every
// stride-th sweep (each event pair also blocks the programmatic launch overlap
// of its sweep), read after the batch's host sync; sweeps past the stop test
// (no-op launches) are not counted.
struct SweepTimer {
    bool on = false;
    int stride = 4;
    std::vector<cudaEvent_t> ev;
    std::vector<int64_t> rec;  // sweep index of each used event triple
    double gather_ms = 0.0, scatter_ms = 0.0;
    int timed = 0;
    bool wants(int64_t it) const { return on && it % stride == stride - 1; }
    int mark(int64_t it, int which, cudaStream_t s) {
        if (!wants(it)) return PR_OK;
        if (which == 0) {
            rec.push_back(it);
            while (ev.size() < 3 * rec.size()) {
                cudaEvent_t e;
                PR_CUDA(cudaEventCreate(&e));
                ev.push_back(e);
            }
        }
        PR_CUDA(cudaEventRecord(ev[3 * (rec.size() - 1) + which], s));
        return PR_OK;
    }
    int harvest(int32_t iters_done) {
        for (size_t i = 0; i < rec.size(); ++i) {
            if (rec[i] >= iters_done) continue;
            float a = 0.f, b = 0.f;
            PR_CUDA(cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 1]));
            PR_CUDA(cudaEventElapsedTime(&b, ev[3 * i + 1], ev[3 * i + 2]));
            gather_ms += a;
            scatter_ms += b;
            ++timed;
        }
        rec.clear();
        return PR_OK;
    }
    ~SweepTimer() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};

static void fill_stats(pr_graph* g, Ctx& ctx, int64_t launches0, const View& v, int64_t nm, int host_syncs,
                       int K) {
    DevState* hs = g->st_host;
    pr_run_stats& rs = g->last;
    rs = pr_run_stats{};
    g->log_len = std::min<int32_t>(hs->iters, g->log_cap);
    rs.iterations = hs->iters;
    rs.status = hs->status;
    rs.delta_l1 = hs->l1;
    rs.delta_linf = hs->linf;
    rs.run_launches = ctx.launches - launches0;
    rs.host_syncs = host_syncs;
    rs.gather_rows = v.nrows;
    rs.gather_edges = v.nedges;
    rs.scatter_members = nm;
    rs.n_contrib = g->n_contrib;
    rs.edges_gathered = v.nedges * (int64_t)hs->iters;
    rs.phases = K;
}

static int run_nosync(pr_graph* g, double d, double tau, int32_t max_iter, uint32_t mode, double* ranks, Ctx& ctx,
                      int32_t* iters_out, double* delta_out);
static int run_perforated(pr_graph* g, double d, double tau, int32_t max_iter, uint32_t mode, double* ranks,
                          Ctx& ctx, int32_t* iters_out, double* delta_out);
static int residual_check(pr_graph* g, Ctx& ctx, double c, double d, const double* x, const double* y, double* resid,
                          double* out2, int32_t done);

int run(pr_graph* g, double d, double tau, int32_t max_iter, uint32_t mode, double* ranks, Ctx& ctx,
        int32_t* iters_out, double* delta_out) {
    PR_TRY(reset_tickets(g->plain, ctx.stream));
    if (g->pre_done) PR_TRY(reset_tickets(g->reduced, ctx.stream));
    const bool reduced = (mode & PR_USE_REDUCTIONS) != 0;
    const View& v = reduced ? g->reduced : g->plain;
    // Source-blocked views (contrib vector beyond L2) run the asynchronous
    // modes on the Jacobi schedule -- a valid No-Sync schedule in which every
    // read sees the previous sweep's value (reading Q-Y2): measured on config
    // 5, slice passes finalizing rows in place in their last segment needed
    // 88 sweeps against Jacobi's 14 (the in-place updates break the plain
    // iteration's mass conservation on this dangling-free graph).  No-Sync keeps
    // its certificate of the original system.
    const bool blocked_async = (mode & (PR_MODE_ASYNC | PR_MODE_NOSYNC)) && v.nseg > 0;
    const uint32_t mode_in = mode;
    if (blocked_async) mode &= ~(PR_MODE_ASYNC | PR_MODE_NOSYNC);
    if (mode & PR_PERFORATE) return run_perforated(g, d, tau, max_iter, mode, ranks, ctx, iters_out, delta_out);
    if (mode & PR_MODE_NOSYNC) return run_nosync(g, d, tau, max_iter, mode, ranks, ctx, iters_out, delta_out);
    cudaStream_t s = ctx.stream;
    const bool async = (mode & PR_MODE_ASYNC) != 0;
    const bool phased = (mode & PR_MODE_PHASED) != 0;
    const bool timing = (mode & PR_TIMING) != 0;
    // PR_TIMING brackets every tstride-th sweep's launches with events (each
    // event pair also blocks the programmatic launch overlap of its sweep)
    const int tstride = std::max(1, env_int("PRGPU_TIMING_STRIDE", 4));
    const int64_t n = g->n;
    const int64_t nm = reduced ? g->n_members : 0;
    const int64_t launches0 = ctx.launches;
    RunBufs rb;
    PR_TRY(run_buffers(g, ctx, ranks, max_iter, &rb));
    double* x = rb.x;

    int K = 1;  // phases of a sweep (PR_MODE_PHASED: K >= 1)
    if (phased) PR_TRY(phase_plan(g, reduced, ctx, &K));
    GatherCfg gc;
    PR_TRY(gather_config(ctx, v, g, async ? G_INPLACE : G_SYNC, &gc));
    const int64_t cap4 = (int64_t)ctx.num_sms * 4;
    // K-FINALIZE: fixed grid per phase, so each CTA's rows and members (and
    // hence its Delta partial) are a fixed set (deterministic)
    int64_t fgrid_k[SE_MAX_PHASES], foff_k[SE_MAX_PHASES];
    const int64_t fin_cap = (int64_t)ctx.num_sms * env_int("PRGPU_FIN_CTAS_PER_SM", 8);
    int64_t fgrid = 0;
    for (int k = 0; k < K; ++k) {
        const int64_t rows = phased ? v.phase_rb[k + 1] - v.phase_rb[k] : v.nrows;
        const int64_t work = rows + (k == K - 1 ? nm : 0);
        fgrid_k[k] = std::min<int64_t>(std::max<int64_t>((work + GT_NT * FIN_U - 1) / (GT_NT * FIN_U), 1), fin_cap);
        foff_k[k] = fgrid;
        fgrid += fgrid_k[k];
    }
    const int64_t ggrid = async ? gc.grid : fgrid;  // CTAs writing Delta partials first
    const int64_t nz = g->nz;
    const int64_t zgrid = nz > 0 ? std::min<int64_t>((nz + GT_NT * 4 - 1) / (GT_NT * 4), cap4) : 0;
    PR_TRY(ensure_partials(g, ctx, 2 * (ggrid + zgrid)));
    const double c = (1.0 - d) / (double)n;
    if (reduced && nm > 0) PR_TRY(upload_ab(g, ctx, c, d));
    PR_TRY(init_state(g, ctx, tau, max_iter, mode, x, g->cidx, g->y[0], v, nm));

    IterArgs ia_rest{g->st, g->cta_partial, ggrid, 0, 0, g->delta_log};
    IterArgs ia_first = ia_rest;
    ia_first.zero_ctas = zgrid;
    double* zero_partial = g->cta_partial + 2 * ggrid;
    const MemArgs ma{g->mem_srow, g->mem_k, g->mem_info, g->xm, nm, nm > 0 ? (nm + gc.grid - 1) / gc.grid : 0, g->ab};
    FinArgs fa{v.sums, v.nrows, v.rinfo, g->xr, g->mem_srow, g->mem_k, g->mem_info, g->xm, nm, g->ab, nullptr, c, d};
    fa.vec = env_int("PRGPU_FIN_VEC", 1);
    // identical members folded into their source row (sync reduced sweeps; the
    // flag bit needs out-degrees < 2^30, i.e. n <= 2^30)
    const bool fold = reduced && nm > 0 && !async && !phased && n <= ((int64_t)1 << 30) && env_int("PRGPU_FOLD", 1);
    if (fold) {
        PR_TRY(build_fold(g, ctx, v));
        fa.fold = 1;
        fa.rinfo = g->fold_rinfo;
        fa.fold_w = g->fold_w;
        fa.fold_list = g->fold_list;
        fa.nm = g->fold_n;
        fa.fold_rec = g->fold_rec;
        fa.nrec = g->fold_nrec;
        if (g->fold_n > 0) {
            fa.fold_crec = g->fold_crec;
            fa.xc = g->fold_xc;
            PR_LAUNCH(ctx, k_fill_f64, (unsigned)std::min<int64_t>((g->fold_n + 255) / 256, (int64_t)ctx.num_sms * 16),
                      256, 0, g->fold_xc, g->fold_n, 1.0 / (double)n);
        }
    }
    // delayed chain resolution (sync reduced, reading Q-C2): the last
    // max_chain + 1 values of every chain source, slot 0 = x_0 = 1/n
    if (reduced && nm > 0 && !async && !phased && !(mode & PR_CHAIN_EAGER) && g->n_hsrc > 0) {
        const int L = g->max_chain + 1;
        const int64_t need = (int64_t)L * g->n_hsrc;
        if (g->hist_cap < need) {
            dfree(g->hist, s);
            PR_TRY(dalloc(&g->hist, (size_t)need, s));
            g->hist_cap = need;
        }
        PR_LAUNCH(ctx, k_fill_f64, (unsigned)std::min<int64_t>((need + 255) / 256, (int64_t)ctx.num_sms * 16), 256, 0,
                  g->hist, need, 1.0 / (double)n);
        fa.hist = g->hist;
        fa.mh = g->mem_h;
        fa.nh = g->n_hsrc;
        fa.L = L;
    }

    SweepTimer tmr;
    tmr.on = timing;
    tmr.stride = tstride;
    auto sweep = [&](int64_t it) -> int {
        // sync: ping-pong; async / phased: one buffer, in place
        const double* y_in = (async || phased) ? g->y[0] : g->y[it & 1];
        double* y_out = (async || phased) ? g->y[0] : g->y[(it + 1) & 1];
        const IterArgs& ia = it == 0 ? ia_first : ia_rest;
        // in-degree-0 vertices (sweep 1; Q-Z): before the in-place sweep (a
        // valid asynchronous read), after the last gather otherwise
        if (it == 0 && zgrid > 0 && !phased)
            PR_LAUNCH(ctx, k_zero, (unsigned)zgrid, GT_NT, 0, (const int32_t*)g->zlist, nz, c, x, y_out,
                      (const int32_t*)g->outdeg, (const int32_t*)g->cidx, zero_partial);
        PR_TRY(tmr.mark(it, 0, s));
        if (phased) {
            // phase k gathers its rows from the contribs phases 0..k-1 of this
            // sweep wrote (block Gauss-Seidel), then finalizes them in place
            for (int k = 0; k < K; ++k) {
                const int64_t r0 = v.phase_rb[k];
                if (K == 1)
                    PR_TRY(launch_gather(ctx, g, v, y_in, gc));
                else
                    PR_TRY(launch_gather(ctx, g, v.phv[k], y_in, gc, v.sums + r0));
                FinArgs f = fa;
                f.y_out = y_out;
                f.row0 = r0;
                f.nrows = v.phase_rb[k + 1];
                f.nm = k == K - 1 ? nm : 0;
                f.part_off = foff_k[k];
                f.last = k == K - 1;
                // in-degree-0 vertices last (sweep 1), after every gather of the sweep
                if (it == 0 && zgrid > 0 && k == K - 1)
                    PR_LAUNCH(ctx, k_zero, (unsigned)zgrid, GT_NT, 0, (const int32_t*)g->zlist, nz, c, x, y_out,
                              (const int32_t*)g->outdeg, (const int32_t*)g->cidx, zero_partial);
                PR_LAUNCH_PDL(ctx, k_finalize<false>, (unsigned)fgrid_k[k], GT_NT, 0, f, ia);
            }
            PR_TRY(tmr.mark(it, 1, s));
        } else if (async) {
            InPlacePolicy ip{};
            ip.y_in = g->y[0];
            ip.y = g->y[0];
            ip.hot_n = gc.hot_n;
            ip.xr = g->xr;
            ip.rinfo = v.rinfo;
            ip.c = c;
            ip.d = d;
            if (v.nspans > 0 || nm > 0)
                PR_LAUNCH(ctx, k_stream_async, gc.grid, gc.nt, gc.smem, ip, stream_args(v), ma, ia);
            else  // nothing to gather: the zero-in partials still need their reduction
                PR_LAUNCH_PDL(ctx, k_finalize<false>, 1, GT_NT, 0, fa, ia);
            PR_TRY(tmr.mark(it, 1, s));
        } else {
            PR_TRY(launch_gather(ctx, g, v, y_in, gc));
            PR_TRY(tmr.mark(it, 1, s));
            FinArgs f = fa;
            f.y_out = y_out;
            PR_LAUNCH_PDL(ctx, k_finalize<false>, (unsigned)fgrid, GT_NT, 0, f, ia);
            if (it == 0 && nz > 0)
                PR_LAUNCH(ctx, k_zero_y, (unsigned)std::min<int64_t>((nz + 255) / 256, (int64_t)ctx.num_sms * 8),
                          256, 0, (const int32_t*)g->zlist, nz, c, (double*)y_in, (const int32_t*)g->outdeg,
                          (const int32_t*)g->cidx);
        }
        PR_TRY(tmr.mark(it, 2, s));
        return PR_OK;
    };
    LoopStats ls;
    PR_TRY(sweep_loop(g, ctx, max_iter, tau, sweep, [&](int64_t) { return tmr.harvest(g->st_host->iters); }, ls));
    const unsigned ug = (unsigned)std::min<int64_t>((v.nrows + nm + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
    PR_LAUNCH(ctx, k_unpermute, ug, 256, 0, (const double*)g->xr, (const int32_t*)v.vid, v.nrows,
              (const double*)g->xm, (const int32_t*)g->mem_vid, nm, x, fold ? (const int32_t*)g->mem_k : nullptr,
              fold ? (const int32_t*)g->mem_srow : nullptr, fa.fold_crec ? (const int32_t*)g->fold_list : nullptr,
              (const double*)fa.xc, fa.fold_crec ? g->fold_n : 0);
    if (!rb.ranks_dev) {
        PR_CUDA(cudaMemcpyAsync(ranks, x, sizeof(double) * (size_t)n, cudaMemcpyDefault, s));
        PR_CUDA(cudaStreamSynchronize(s));
        ++ls.host_syncs;
    }
    fill_stats(g, ctx, launches0, v, nm, ls.host_syncs, K);
    pr_run_stats& rs = g->last;
    rs.timed_iterations = tmr.timed;
    rs.gather_ms = tmr.gather_ms;
    rs.scatter_ms = tmr.scatter_ms;
    DevState* hs = g->st_host;
    if (blocked_async && (mode_in & PR_MODE_NOSYNC)) {
        // No-Sync's certificate: ||F(x) - x|| of the original system over the
        // final contribs (a converged Jacobi run has it <= d * tau)
        double cert[2] = {0.0, 0.0};
        PR_TRY(ensure_partials(g, ctx, 2 * (ggrid + zgrid) + 2));
        const double* yfin = g->y[hs->iters & 1];
        PR_TRY(residual_check(g, ctx, c, d, x, yfin, g->cta_partial + 2 * (ggrid + zgrid), cert, 1));
        rs.nosync_launches = 1;
        rs.nosync_min_iters = rs.nosync_median_iters = hs->iters;
        rs.residual = (mode_in & PR_NORM_LINF) ? cert[1] : cert[0];
        rs.host_syncs += 1;
        if (rs.residual > tau && hs->status == PR_OK) hs->status = PR_NOT_CONVERGED;
        if (iters_out) *iters_out = hs->iters;
        if (delta_out) *delta_out = rs.residual;
        return hs->status;
    }
    if (iters_out) *iters_out = hs->iters;
    if (delta_out) *delta_out = (mode & PR_NORM_LINF) ? hs->linf : hs->l1;
    return hs->status;
}

// ------------------------------------------------------- certificate --
// ||F(x) - x|| of the original system (F = Eq.(1)) over the contribs y, by one
// synchronous gather of the plain view + k_residual (No-Sync's exit check).
__global__ void k_set_done(DevState* st, int32_t v) { st->done = v; }

static int residual_check(pr_graph* g, Ctx& ctx, double c, double d, const double* x, const double* y, double* resid,
                          double* out2, int32_t done) {
    cudaStream_t s = ctx.stream;
    const View& pv = g->plain;
    GatherCfg gp;
    PR_TRY(gather_config(ctx, pv, g, G_SYNC, &gp));
    PR_CUDA(cudaMemsetAsync(resid, 0, 2 * sizeof(double), s));
    // the certificate gather must run even though the run's state says done
    PR_LAUNCH(ctx, k_set_done, 1, 1, 0, g->st, 0);
    PR_TRY(launch_gather(ctx, g, pv, y, gp));
    if (pv.nrows > 0)
        PR_LAUNCH(ctx, k_residual, (unsigned)std::min<int64_t>((pv.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 8),
                  256, 0, (const double*)pv.sums, pv.nrows, (const int32_t*)pv.vid, x, c, d, resid);
    PR_CUDA(cudaMemcpyAsync(out2, resid, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    PR_LAUNCH(ctx, k_set_done, 1, 1, 0, g->st, done);
    PR_CUDA(cudaStreamSynchronize(s));
    return PR_OK;
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
    const int tstride = std::max(1, env_int("PRGPU_TIMING_STRIDE", 4));
    const int64_t n = g->n;
    const View& v = g->shard;
    const int world = g->shard_world, rank = g->shard_rank;
    const int64_t chunk = g->shard_chunk, H = g->shard_hot;
    const bool peers = g->speer_dev != nullptr && world > 1;
    // NVLS multicast team (multicast.cu): every contrib / delta-pair store is
    // ONE multimem store into all ranks' buffers; the exchange is a barrier only
    const bool mcast = g->mc != nullptr && g->mc->bound;
    const bool barrier_only = peers || mcast;
    const int64_t launches0 = ctx.launches;
    PR_TRY(reset_tickets(v, s));
    if (!g->x) PR_TRY(dalloc(&g->x, (size_t)n, s));
    double* x = g->x;
    const int64_t need_xr = std::max<int64_t>(std::max(g->plain.nrows, v.nrows), 1);
    if (g->xr_cap < need_xr) {
        dfree(g->xr, s);
        PR_TRY(dalloc(&g->xr, (size_t)need_xr, s));
        g->xr_cap = need_xr;
    }
    const int log_cap = max_iter < 4096 ? max_iter : 4096;
    if (g->log_cap < log_cap) {
        dfree(g->delta_log, s);
        PR_TRY(dalloc(&g->delta_log, (size_t)(2 * log_cap), s));
        g->log_cap = log_cap;
    }

    GatherCfg gc;
    PR_TRY(gather_config(ctx, v, g, G_SYNC, &gc));
    if (gc.hot_n > H) {  // the shared-memory tier reads the hot copy only
        gc.hot_n = (int)H;
        gc.smem = (size_t)gc.hot_n * sizeof(double);
    }
    const int64_t cap4 = (int64_t)ctx.num_sms * 4;
    const int64_t fgrid =
        std::min<int64_t>(std::max<int64_t>((v.nrows + GT_NT * FIN_U - 1) / (GT_NT * FIN_U), 1), cap4 * 2);
    const int64_t nz = g->snz;
    const int64_t zgrid = nz > 0 ? std::min<int64_t>((nz + GT_NT * 4 - 1) / (GT_NT * 4), cap4) : 0;
    PR_TRY(ensure_partials(g, ctx, 2 * (fgrid + zgrid)));
    const double c = (1.0 - d) / (double)n;
    // x0 = 1/n and y0 of EVERY contrib slot (the replica starts complete)
    PR_TRY(init_state(g, ctx, tau, max_iter, mode, x, g->scidx, g->sy[0], v, 0));
    IterArgs ia0{g->st, g->cta_partial, 0, 0, 0, g->delta_log};
    const unsigned cgrid = (unsigned)std::max<int64_t>(1, (H + 255) / 256);
    PR_LAUNCH(ctx, k_shard_combine, cgrid, 256, 0, ia0, g->sy[0], (const int32_t*)g->shot_src, H, world, chunk, 0);
    // peer buffers: no rank may store into another's buffers before that rank
    // has initialised them (sweep 1's stores would be overwritten)
    const bool dev_bar = barrier_only && g->sdev_barrier;
    if (dev_bar) {
        PR_TRY(device_barrier(g, ctx));
    } else if (barrier_only && exchange(exchange_ctx, nullptr, chunk, world, (void*)s) != 0) {
        set_error("pr_run_sharded: the exchange callback failed before sweep 1");
        return PR_ECUDA;
    }
    IterArgs ia_rest{g->st, g->cta_partial, fgrid, 0, 0, g->delta_log};
    IterArgs ia_first = ia_rest;
    ia_first.zero_ctas = zgrid;
    double* zero_partial = g->cta_partial + 2 * fgrid;
    const FinArgs fa{v.sums, v.nrows, v.rinfo, g->xr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, nullptr, c, d};
    const int fin_vec = env_int("PRGPU_FIN_VEC", 1);

    SweepTimer tmr;
    tmr.on = timing;
    tmr.stride = tstride;
    auto sweep = [&](int64_t it) -> int {
        double* y_in = g->sy[it & 1];
        double* y_out = g->sy[(it + 1) & 1];
        IterArgs ia = it == 0 ? ia_first : ia_rest;
        ia.shard_out = y_out + H + (int64_t)rank * chunk + chunk - 2;
        double* const* pout = peers ? g->speer_dev + ((it + 1) & 1) * (world - 1) : nullptr;
        ia.peer_y = pout;
        ia.npeer = peers ? world - 1 : 0;
        ia.shard_off = H + (int64_t)rank * chunk + chunk - 2;
        double* mc_out = mcast ? g->mc->y[(it + 1) & 1] : nullptr;  // multicast address of y_out
        if (mcast) ia.mc_out = mc_out + ia.shard_off;
        if (it == 0 && zgrid > 0)
            PR_LAUNCH(ctx, k_zero, (unsigned)zgrid, GT_NT, 0, (const int32_t*)g->szlist, nz, c, x,
                      mcast ? mc_out : y_out, (const int32_t*)g->outdeg, (const int32_t*)g->scidx, zero_partial,
                      mcast ? 1 : 0);
        PR_TRY(tmr.mark(it, 0, s));
        PR_TRY(launch_gather(ctx, g, v, y_in, gc));
        PR_TRY(tmr.mark(it, 1, s));
        FinArgs f = fa;
        f.y_out = y_out;
        f.peer_y = pout;
        f.npeer = peers ? world - 1 : 0;
        f.mc_y = mc_out;
        f.vec = fin_vec;  // as in the unsharded sync sweep: world 1 reproduces its Delta bit for bit
        if (peers || mcast)
            PR_LAUNCH_PDL(ctx, k_finalize<true>, (unsigned)fgrid, GT_NT, 0, f, ia);
        else
            PR_LAUNCH_PDL(ctx, k_finalize<false>, (unsigned)fgrid, GT_NT, 0, f, ia);
        PR_TRY(tmr.mark(it, 2, s));
        // multicast: the in-degree-0 contribs go to every rank's sweep-1 output
        // (k_zero above) and, in sweep 2, to its other buffer (their sweep-2
        // output; in sweep 1 every rank gathers from it)
        if (mcast && it == 1 && nz > 0)
            PR_LAUNCH(ctx, k_zero_y, (unsigned)std::min<int64_t>((nz + 255) / 256, (int64_t)ctx.num_sms * 8), 256, 0,
                      (const int32_t*)g->szlist, nz, c, mc_out, (const int32_t*)g->outdeg, (const int32_t*)g->scidx, 1);
        if (it == 0 && nz > 0 && !mcast) {
            const unsigned zg = (unsigned)std::min<int64_t>((nz + 255) / 256, (int64_t)ctx.num_sms * 8);
            PR_LAUNCH(ctx, k_zero_y, zg, 256, 0, (const int32_t*)g->szlist, nz, c, y_in, (const int32_t*)g->outdeg,
                      (const int32_t*)g->scidx);
            if (peers)  // peers' sweep-1 output buffer (their gathers read the other one)
                PR_LAUNCH(ctx, k_peer_zero, zg, 256, 0, (const int32_t*)g->szlist, nz, c, (const int32_t*)g->outdeg,
                          (const int32_t*)g->scidx, pout, world - 1);
        }
        // ...and their other buffer only in sweep 2 (their sweep-2 output):
        // in sweep 1 it is what they gather from
        if (it == 1 && nz > 0 && peers)
            PR_LAUNCH(ctx, k_peer_zero, (unsigned)std::min<int64_t>((nz + 255) / 256, (int64_t)ctx.num_sms * 8), 256,
                      0, (const int32_t*)g->szlist, nz, c, (const int32_t*)g->outdeg, (const int32_t*)g->scidx, pout,
                      world - 1);
        // all-gather of the chunks (or, with peer buffers, only the
        // cross-rank barrier: every rank's stores landed in every buffer --
        // on the device when the device-side barrier is on: no host sync)
        if (dev_bar) {
            PR_TRY(device_barrier(g, ctx));
        } else if (exchange(exchange_ctx, barrier_only ? nullptr : y_out + H, chunk, world, (void*)s) != 0) {
            set_error("pr_run_sharded: the exchange callback failed at sweep %lld", (long long)it + 1);
            return PR_ECUDA;
        }
        PR_LAUNCH(ctx, k_shard_combine, cgrid, 256, 0, ia, y_out, (const int32_t*)g->shot_src, H, world, chunk, 1);
        return PR_OK;
    };
    LoopStats ls;  // (tau = 0: doubling batches)
    PR_TRY(sweep_loop(g, ctx, max_iter, 0.0, sweep, [&](int64_t) {
        if (g->st_host->peer_err) {
            set_error("pr_run_sharded: the device-side peer barrier timed out (a peer stopped)");
            return (int)PR_ECUDA;
        }
        return tmr.harvest(g->st_host->iters);
    }, ls));
    const unsigned ug = (unsigned)std::min<int64_t>((v.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
    PR_LAUNCH(ctx, k_unpermute, ug, 256, 0, (const double*)g->xr, (const int32_t*)v.vid, v.nrows,
              (const double*)nullptr, (const int32_t*)nullptr, (int64_t)0, x);
    PR_LAUNCH(ctx, k_shard_ranks, (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx.num_sms * 16), 256, 0,
              (const double*)x, (const int32_t*)g->sowner, rank, n, ranks);
    PR_CUDA(cudaStreamSynchronize(s));
    fill_stats(g, ctx, launches0, v, 0, ls.host_syncs, 1);
    pr_run_stats& rs = g->last;
    rs.timed_iterations = tmr.timed;
    rs.gather_ms = tmr.gather_ms;
    rs.scatter_ms = tmr.scatter_ms;
    DevState* hs = g->st_host;
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
    RunBufs rb;
    PR_TRY(run_buffers(g, ctx, ranks, max_iter, &rb));
    double* x = rb.x;
    double* y = g->y[0];
    GatherCfg gc;  // persistent grid (all resident CTAs)
    PR_TRY(gather_config(ctx, v, g, G_INPLACE, &gc));
    const int grid = gc.grid;
    const double c = (1.0 - d) / (double)n;
    if (reduced && nm > 0) PR_TRY(upload_ab(g, ctx, c, d));
    const int64_t cap4 = (int64_t)ctx.num_sms * 4;
    const int64_t nz = g->nz;
    const int64_t zgrid = nz > 0 ? std::min<int64_t>((nz + GT_NT * 4 - 1) / (GT_NT * 4), cap4) : 0;
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
    PR_TRY(init_state(g, ctx, tau, max_iter, mode, x, g->cidx, y, v, nm));
    // in-degree-0 vertices take their fixed value c (Q-Z) before the first sweep
    if (zgrid > 0)
        PR_LAUNCH(ctx, k_zero, (unsigned)zgrid, GT_NT, 0, (const int32_t*)g->zlist, nz, c, x, y,
                  (const int32_t*)g->outdeg, (const int32_t*)g->cidx, resid + 2);
    const int64_t mper = nm > 0 ? (nm + grid - 1) / grid : 0;
    NoSyncArgs na{err, iters, (mode & PR_NORM_LINF) ? 1 : 0, tau, 0};
    int per_sm = 0;
    PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_nosync_stream, gc.nt, gc.smem));
    if ((int64_t)grid > (int64_t)ctx.num_sms * std::max(per_sm, 1)) {
        set_error("pr_run(NOSYNC): grid %d exceeds the resident CTAs", grid);
        return PR_ECUDA;
    }
    std::vector<int32_t> hit(grid);
    std::vector<double> hlog;
    int32_t max_it = 0, min_it = 0, med_it = 0, launches = 0, status = PR_NOT_CONVERGED;
    double cert[2] = {0.0, 0.0};
    const int log_cap = max_iter < 4096 ? max_iter : 4096;
    while (true) {
        PR_LAUNCH(ctx, k_fill_f64, 1, 256, 0, err, (int64_t)(2 * grid), 1e300);
        na.max_local = max_iter - max_it;
        InPlacePolicy ip{};
        ip.y_in = y;
        ip.y = y;
        ip.hot_n = gc.hot_n;
        ip.xr = g->xr;
        ip.rinfo = v.rinfo;
        ip.c = c;
        ip.d = d;
        const MemArgs ma{g->mem_srow, g->mem_k, g->mem_info, g->xm, nm, mper, g->ab};
        if (v.nspans > 0 || nm > 0)
            PR_LAUNCH(ctx, k_nosync_stream, (unsigned)grid, gc.nt, gc.smem, ip, stream_args(v), ma, na);
        const unsigned ug = (unsigned)std::min<int64_t>((v.nrows + nm + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
        PR_LAUNCH(ctx, k_unpermute, ug, 256, 0, (const double*)g->xr, (const int32_t*)v.vid, v.nrows,
                  (const double*)g->xm, (const int32_t*)g->mem_vid, nm, x);
        ++launches;
        // certificate: S over the current contribs, then ||F(x) - x||
        PR_TRY(residual_check(g, ctx, c, d, x, y, resid, cert, 0));
        PR_CUDA(cudaMemcpyAsync(hit.data(), iters, sizeof(int32_t) * (size_t)grid, cudaMemcpyDeviceToHost, s));
        PR_CUDA(cudaStreamSynchronize(s));
        max_it = *std::max_element(hit.begin(), hit.end());
        min_it = *std::min_element(hit.begin(), hit.end());
        {
            std::vector<int32_t> tmp(hit);
            std::nth_element(tmp.begin(), tmp.begin() + tmp.size() / 2, tmp.end());
            med_it = tmp[tmp.size() / 2];
        }
        if (v.nspans == 0 && nm == 0) max_it = min_it = med_it = 1;  // only in-degree-0 vertices: one sweep
        hlog.push_back(cert[0]);
        hlog.push_back(cert[1]);
        const double rn = (mode & PR_NORM_LINF) ? cert[1] : cert[0];
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
    DevState* hs = g->st_host;
    hs->iters = max_it;
    hs->status = status;
    hs->l1 = cert[0];
    hs->linf = cert[1];
    hs->done = 1;
    PR_CUDA(cudaMemcpyAsync(g->st, hs, sizeof(DevState), cudaMemcpyHostToDevice, s));
    if (!rb.ranks_dev) PR_CUDA(cudaMemcpyAsync(ranks, x, sizeof(double) * (size_t)n, cudaMemcpyDefault, s));
    dfree(scratch, s);
    dfree(iters, s);
    PR_CUDA(cudaStreamSynchronize(s));
    fill_stats(g, ctx, launches0, v, nm, launches + 1, 1);
    g->log_len = nlog;
    pr_run_stats& rs = g->last;
    rs.edges_gathered = 0;
    rs.nosync_min_iters = min_it;
    rs.nosync_launches = launches;
    rs.nosync_median_iters = med_it;
    rs.residual = (mode & PR_NORM_LINF) ? cert[1] : cert[0];
    if (iters_out) *iters_out = max_it;
    if (delta_out) *delta_out = rs.residual;
    return status;
}

// ------------------------------------------------------------ perforation --
// PR_PERFORATE (Barriers-Opt, Alg.5; reading Q-P in
// DESIGN.md): synchronous plain sweeps in which K-FINALIZE keeps a sticky
// per-vertex flag (Alg.5's threshold_check): a vertex whose change in a sweep
// is 0 < |delta| < tau * 1e-5 is flagged after that sweep's update and from
// the next sweep on keeps its value (x, and its contrib in both ping-pong
// buffers; |delta| = 0).  The flags alone define the result.  As a pure
// performance step, at the host sync after each batch of 8 sweeps the gathered
// view is COMPACTED to the unflagged rows once >= 5 % of them are flagged, so
// later sweeps stop streaming the frozen rows' edges.  Approximate by design.
// With PR_MODE_ASYNC the sweeps are in place (k_stream_async, the flags in
// InPlacePolicy); with PR_MODE_NOSYNC (No-Sync-Opt, Alg.5 with Alg.3's
// barrier-free loop) each batch is ONE persistent k_nosync_stream launch of at
// most 8 local sweeps per CTA that stops early on the CTA-level convergence
// test, so the compaction still happens between launches.
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

// active-view x back into the full plain-view row order
__global__ void k_pf_writeback(const double* __restrict__ xa, const int32_t* __restrict__ amap, int64_t nr,
                               double* __restrict__ xfull) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += (int64_t)gridDim.x * blockDim.x)
        xfull[amap[r]] = xa[r];
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
    // schedule: synchronous sweeps (Barriers-Opt), in-place launch-level
    // sweeps (ASYNC), or persistent barrier-free launches of at most
    // PF_BATCH local sweeps each (No-Sync-Opt)
    const bool nosync = (mode & PR_MODE_NOSYNC) != 0;
    const bool inplace = nosync || (mode & PR_MODE_ASYNC) != 0;
    const int64_t launches0 = ctx.launches;
    RunBufs rb;
    PR_TRY(run_buffers(g, ctx, ranks, max_iter, &rb));
    double* x = rb.x;
    const double c = (1.0 - d) / (double)n;
    const int64_t cap4 = (int64_t)ctx.num_sms * 4;
    const int64_t fgrid_max =
        std::min<int64_t>(std::max<int64_t>((V.nrows + GT_NT * FIN_U - 1) / (GT_NT * FIN_U), 1), cap4 * 2);
    const int64_t nz = g->nz;
    const int64_t zgrid = nz > 0 ? std::min<int64_t>((nz + GT_NT * 4 - 1) / (GT_NT * 4), cap4) : 0;
    GatherCfg gc_full;
    PR_TRY(gather_config(ctx, V, g, inplace ? G_INPLACE : G_SYNC, &gc_full));
    const int64_t pmax = std::max<int64_t>(fgrid_max, gc_full.grid);
    PR_TRY(ensure_partials(g, ctx, 2 * (pmax + zgrid) + 2));
    uint8_t* fz = nullptr;
    unsigned long long* cnt = nullptr;
    double* err = nullptr;    // No-Sync-Opt: (L1, Linf) each CTA last published
    int32_t* lits = nullptr;  // No-Sync-Opt: local sweeps of each CTA in this launch
    TmpGuard tg_(ctx.stream);
    tg_.track(fz);
    tg_.track(cnt);
    tg_.track(err);
    tg_.track(lits);
    PR_TRY(dalloc(&fz, (size_t)std::max<int64_t>(V.nrows, 1), s));
    PR_TRY(dalloc(&cnt, 1, s));
    PR_CUDA(cudaMemsetAsync(fz, 0, (size_t)std::max<int64_t>(V.nrows, 1), s));
    PR_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
    if (nosync) {
        PR_TRY(dalloc(&err, (size_t)(2 * gc_full.grid), s));
        PR_TRY(dalloc(&lits, (size_t)gc_full.grid, s));
    }
    PR_TRY(init_state(g, ctx, tau, max_iter, mode, x, g->cidx, g->y[0], V, 0));
    const unsigned fg = (unsigned)std::min<int64_t>((V.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
    const double tau_f = tau * 1e-5;  // "threshold*0.00001" (Alg.5; Q-P)

    ActiveView A;
    A.v = V;  // shallow: the plain view's arrays
    A.xr = g->xr;
    A.is_full = true;
    int64_t edges_gathered = 0;
    int32_t compactions = 0;
    int64_t launched = 0;         // sweeps launched (No-Sync-Opt: the largest local count so far)
    int64_t flagged_active = 0;   // flagged rows still in the active view
    GatherCfg gc;
    int64_t fgrid = 0;
    auto setup = [&]() -> int {
        PR_TRY(gather_config(ctx, A.v, g, inplace ? G_INPLACE : G_SYNC, &gc));
        fgrid = std::min<int64_t>(std::max<int64_t>((A.v.nrows + GT_NT * FIN_U - 1) / (GT_NT * FIN_U), 1), cap4 * 2);
        return PR_OK;
    };
    PR_TRY(setup());
    auto inplace_policy = [&]() {
        InPlacePolicy ip{};
        ip.y_in = g->y[0];
        ip.y = g->y[0];
        ip.hot_n = gc.hot_n;
        ip.xr = A.xr;
        ip.rinfo = A.v.rinfo;
        ip.c = c;
        ip.d = d;
        ip.fz = fz;
        ip.tau_f = tau_f;
        ip.nfz = cnt;
        return ip;
    };
    const MemArgs ma0{nullptr, nullptr, nullptr, nullptr, 0, 0, nullptr};
    auto sweep = [&](int64_t it, int) -> int {
        if (inplace) {  // one contrib buffer, updated in place
            const int64_t gg = gc.grid;
            IterArgs ia{g->st, g->cta_partial, gg, 0, it == 0 ? zgrid : 0, g->delta_log};
            if (it == 0 && zgrid > 0)  // in-degree-0 vertices before the first in-place sweep (Q-Z)
                PR_LAUNCH(ctx, k_zero, (unsigned)zgrid, GT_NT, 0, (const int32_t*)g->zlist, nz, c, x, g->y[0],
                          (const int32_t*)g->outdeg, (const int32_t*)g->cidx, g->cta_partial + 2 * gg);
            if (A.v.nspans > 0) {
                PR_LAUNCH(ctx, k_stream_async, gc.grid, gc.nt, gc.smem, inplace_policy(), stream_args(A.v), ma0, ia);
            } else {  // nothing left to gather: the reduction alone (delta 0)
                FinArgs f{A.v.sums, 0, A.v.rinfo, A.xr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, g->y[0], c, d};
                PR_LAUNCH_PDL(ctx, k_finalize<false>, 1, GT_NT, 0, f, ia);
            }
            return PR_OK;
        }
        IterArgs ia{g->st, g->cta_partial, fgrid, 0, it == 0 ? zgrid : 0, g->delta_log};
        const double* y_in = g->y[it & 1];
        double* y_out = g->y[(it + 1) & 1];
        if (it == 0 && zgrid > 0)
            PR_LAUNCH(ctx, k_zero, (unsigned)zgrid, GT_NT, 0, (const int32_t*)g->zlist, nz, c, x, y_out,
                      (const int32_t*)g->outdeg, (const int32_t*)g->cidx, g->cta_partial + 2 * fgrid);
        PR_TRY(launch_gather(ctx, g, A.v, y_in, gc));
        FinArgs f{A.v.sums, A.v.nrows, A.v.rinfo, A.xr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, y_out, c, d};
        f.fz = fz;
        f.tau_f = tau_f;
        f.y_other = (double*)y_in;
        f.nfz = cnt;
        PR_LAUNCH_PDL(ctx, k_finalize<false>, (unsigned)fgrid, GT_NT, 0, f, ia);
        if (it == 0 && nz > 0)
            PR_LAUNCH(ctx, k_zero_y, (unsigned)std::min<int64_t>((nz + 255) / 256, (int64_t)ctx.num_sms * 8), 256, 0,
                      (const int32_t*)g->zlist, nz, c, (double*)y_in, (const int32_t*)g->outdeg,
                      (const int32_t*)g->cidx);
        return PR_OK;
    };
    // No-Sync-Opt: one persistent launch of at most `cap` local sweeps per CTA
    // over the active view, stopping early on the CTA-level convergence test
    // (thread-level convergence) over the deltas the CTAs published
    std::vector<int32_t> hit;
    std::vector<double> herr, hlog;
    double ns_delta[2] = {0.0, 0.0};
    int ns_status = PR_NOT_CONVERGED;
    int32_t ns_launches = 0;
    auto nosync_launch = [&](int cap, int64_t* local_max, double* local_mean) -> int {
        const int grid = gc.grid;
        if (launched == 0 && zgrid > 0)
            PR_LAUNCH(ctx, k_zero, (unsigned)zgrid, GT_NT, 0, (const int32_t*)g->zlist, nz, c, x, g->y[0],
                      (const int32_t*)g->outdeg, (const int32_t*)g->cidx, g->cta_partial);
        PR_LAUNCH(ctx, k_fill_f64, 1, 256, 0, err, (int64_t)(2 * grid), 1e300);
        PR_CUDA(cudaMemsetAsync(lits, 0, sizeof(int32_t) * (size_t)grid, s));
        NoSyncArgs na{err, lits, (mode & PR_NORM_LINF) ? 1 : 0, tau, cap};
        if (A.v.nspans > 0) {
            PR_LAUNCH(ctx, k_nosync_stream, (unsigned)grid, gc.nt, gc.smem, inplace_policy(), stream_args(A.v), ma0,
                      na);
            ++ns_launches;
        }
        hit.resize(grid);
        herr.resize(2 * grid);
        PR_CUDA(cudaMemcpyAsync(hit.data(), lits, sizeof(int32_t) * (size_t)grid, cudaMemcpyDeviceToHost, s));
        PR_CUDA(cudaMemcpyAsync(herr.data(), err, sizeof(double) * 2 * (size_t)grid, cudaMemcpyDeviceToHost, s));
        PR_CUDA(cudaStreamSynchronize(s));
        if (A.v.nspans == 0) {  // nothing left to gather: every delta is 0
            *local_max = 1;
            *local_mean = 1.0;
            ns_delta[0] = ns_delta[1] = 0.0;
        } else {
            *local_max = *std::max_element(hit.begin(), hit.end());
            *local_mean = 0.0;
            for (int32_t h : hit) *local_mean += h;
            *local_mean /= grid;
            ns_delta[0] = ns_delta[1] = 0.0;
            for (int b = 0; b < grid; ++b) {
                ns_delta[0] += herr[2 * b];
                ns_delta[1] = std::max(ns_delta[1], herr[2 * b + 1]);
            }
        }
        hlog.push_back(ns_delta[0]);
        hlog.push_back(ns_delta[1]);
        if (((mode & PR_NORM_LINF) ? ns_delta[1] : ns_delta[0]) <= tau) ns_status = PR_OK;
        return PR_OK;
    };
    DevState* hs = g->st_host;
    int host_syncs = 0;
    int rc = PR_OK;
    while (true) {
        const int nb = (int)std::min<int64_t>(8, max_iter - launched);
        bool finished = false;
        unsigned long long flagged = 0;  // flags set since the last compaction (this view's rows)
        if (nosync) {
            int64_t lmax = 0;
            double lmean = 0.0;
            rc = nosync_launch(nb, &lmax, &lmean);
            if (rc != PR_OK) break;
            PR_CUDA(cudaMemcpyAsync(&flagged, cnt, sizeof(flagged), cudaMemcpyDeviceToHost, s));
            PR_CUDA(cudaStreamSynchronize(s));
            ++host_syncs;
            edges_gathered += (int64_t)((double)A.v.nedges * lmean + 0.5);  // spans are equal-sized: an estimate
            launched += lmax;
            finished = ns_status == PR_OK || launched >= max_iter;
        } else {
            for (int j = 0; j < nb && rc == PR_OK; ++j) rc = sweep(launched + j, j);
            if (rc != PR_OK) break;
            PR_CUDA(cudaMemcpyAsync(hs, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
            PR_CUDA(cudaMemcpyAsync(&flagged, cnt, sizeof(flagged), cudaMemcpyDeviceToHost, s));
            PR_CUDA(cudaStreamSynchronize(s));
            ++host_syncs;
            const int64_t done_sweeps = std::min<int64_t>(hs->iters, launched + nb) - launched;
            edges_gathered += A.v.nedges * std::max<int64_t>(done_sweeps, 0);
            launched += nb;
            finished = hs->done || launched >= max_iter;
        }
        flagged_active = (int64_t)flagged;
        if (finished) break;
        if (flagged_active * 20 < A.v.nrows || flagged_active == 0) continue;  // compact once >= 5 % are flagged
        // ---- compaction (performance only): gather only the unflagged rows ----
        if (!A.is_full)
            PR_LAUNCH(ctx, k_pf_writeback, fg, 256, 0, (const double*)A.xr, (const int32_t*)A.v.vid, A.v.nrows, g->xr);
        ActiveView B;
        B.is_full = false;
        const int64_t nr = A.v.nrows - flagged_active;
        int32_t* src_row = nullptr;
        int64_t* nlen = nullptr;
        int64_t* tot = nullptr;
        TmpGuard tc_(ctx.stream);
        tc_.track(src_row);
        tc_.track(nlen);
        tc_.track(tot);
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
        free_active(A, s);
        A = B;
        // the active rows are all unflagged: fresh flags and count
        PR_CUDA(cudaMemsetAsync(fz, 0, (size_t)std::max<int64_t>(A.v.nrows, 1), s));
        PR_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
        flagged_active = 0;
        ++compactions;
        PR_TRY(setup());
    }
    if (rc == PR_OK) {
        if (!A.is_full)
            PR_LAUNCH(ctx, k_pf_writeback, fg, 256, 0, (const double*)A.xr, (const int32_t*)A.v.vid, A.v.nrows, g->xr);
        const unsigned ug = (unsigned)std::min<int64_t>((V.nrows + 255) / 256 + 1, (int64_t)ctx.num_sms * 16);
        PR_LAUNCH(ctx, k_unpermute, ug, 256, 0, (const double*)g->xr, (const int32_t*)V.vid, V.nrows,
                  (const double*)nullptr, (const int32_t*)nullptr, (int64_t)0, x);
        if (!rb.ranks_dev) PR_CUDA(cudaMemcpyAsync(ranks, x, sizeof(double) * (size_t)n, cudaMemcpyDefault, s));
    }
    const int64_t frozen = V.nrows - A.v.nrows + flagged_active;
    int nlog = 0;
    if (rc == PR_OK && nosync) {  // host-side state and log: the published deltas after each launch
        hs->iters = (int32_t)std::min<int64_t>(launched, max_iter);
        hs->status = ns_status;
        hs->l1 = ns_delta[0];
        hs->linf = ns_delta[1];
        hs->done = 1;
        PR_CUDA(cudaMemcpyAsync(g->st, hs, sizeof(DevState), cudaMemcpyHostToDevice, s));
        nlog = std::min<int>((int)hlog.size() / 2, std::min(max_iter, 4096));
        if (nlog > 0)
            PR_CUDA(cudaMemcpyAsync(g->delta_log, hlog.data(), sizeof(double) * 2 * nlog, cudaMemcpyHostToDevice, s));
    }
    free_active(A, s);
    dfree(fz, s);
    dfree(cnt, s);
    dfree(err, s);
    dfree(lits, s);
    PR_CUDA(cudaStreamSynchronize(s));
    if (rc != PR_OK) return rc;
    fill_stats(g, ctx, launches0, V, 0, host_syncs, 1);
    pr_run_stats& rs = g->last;
    rs.edges_gathered = edges_gathered;
    rs.frozen_rows = frozen;
    rs.compactions = compactions;
    if (nosync) {
        g->log_len = nlog;
        rs.nosync_launches = ns_launches;
    }
    if (iters_out) *iters_out = hs->iters;
    if (delta_out) *delta_out = (mode & PR_NORM_LINF) ? hs->linf : hs->l1;
    return hs->status;
}

}  // namespace prgpu
