// preprocess.cu -- K-PRE-IDENT, K-PRE-CHAIN and the reduced view (STIC-D
// work-saving techniques cited in PAPER.md P:398 §3; readings Q-G, Q-C).
//
// Identical groups: v ~ w iff in(v) == in(w) as sets (after dedup); rep(v) =
// min id of the class; the empty in-set is one class.
//   1. row hash h(v) = mix(indeg) + sum over the row's contrib slots of mix(slot)
//      (edge-stream engine, uint64 sums), for the rows of in-degree > 0 (the
//      in-degree-0 vertices are one class)
//   2. stable radix sort of those ids by the top 32 bits of h -> runs of equal
//      bits, ids ascending
//   3. exact verification of every member against the run's first vertex; on a
//      hash collision the vertex scans its run for the first equal row.
// Chains: chain(v) <=> indeg 1 and outdeg 1; pred(v) = the in-neighbour.
//   Pointer jumping over chain vertices (next = pred while pred is a chain
//   vertex) gives every vertex its head and distance k; vertices that never
//   reach a head lie on pure cycles and are not members.
#include <algorithm>

#include "internal.h"
#include "primitives.cuh"
#include "streamengine.cuh"

namespace prgpu {

// ---------------------------------------------------------------- hashing --
constexpr uint64_t kDegSalt = 0xD6E8FEB86659FD93ULL;

// The empty in-set is one class: its vertices (zlist, ascending) all
// get the smallest of them as representative.
__global__ void k_rep_empty(const int32_t* __restrict__ zl, int64_t nz, int32_t* __restrict__ rep) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nz; i += (int64_t)gridDim.x * blockDim.x)
        rep[zl[i]] = zl[0];
}

__global__ void k_u32_from(const int32_t* __restrict__ a, int64_t n, uint32_t* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a ? (uint32_t)a[i] : (uint32_t)i;
}

// The same row hash on the edge-stream engine (sum type uint64, wrapping):
// S(r) = sum over the row's contrib slots of mix(slot) -- slots are a bijection
// on sources, so equal in-sets <=> equal slot sets; the pad slot adds 0.
struct HashStreamPolicy {
    using T = uint64_t;
    static constexpr bool kHot = false;
    uint64_t* out;     // by view row
    int32_t pad;       // the padding slot (contributes nothing)
    const double* hot;
    int32_t hot_n;
    uint64_t pol_last;
    __device__ __forceinline__ uint64_t load(int32_t u) const {
        return u == pad ? 0ull : mix64((uint64_t)(uint32_t)u * 0x9E3779B97F4A7C15ULL + 0x2545F4914F6CDD1DULL);
    }
    __device__ __forceinline__ void emit(int64_t r, uint64_t s) const { out[r] = s; }
    __device__ __forceinline__ void prep(int64_t, uint32_t) {}
    __device__ __forceinline__ void emit_at(int, int64_t r, uint64_t s) const { out[r] = s; }
    __device__ __forceinline__ void emit_first(int64_t r, uint64_t s) const { out[r] = s; }
};

__global__ void __launch_bounds__(SE_NT, 1) k_rowhash_stream(HashStreamPolicy p, StreamArgs a) { stream_run(p, a); }

// + mix(indeg + salt): rows of different in-degree never share a hash by construction
__global__ void k_hash_deg(uint64_t* __restrict__ h, int64_t nr, const int32_t* __restrict__ vid,
                           const int64_t* __restrict__ rp) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = vid ? vid[r] : r;
        h[r] += mix64((uint64_t)(rp[v + 1] - rp[v]) + kDegSalt);
    }
}



__device__ __forceinline__ bool same_row(const int64_t* rp, const int32_t* col, int32_t u, int32_t v) {
    const int64_t du = rp[u + 1] - rp[u];
    if (du != rp[v + 1] - rp[v]) return false;
    const int32_t* a = col + rp[u];
    const int32_t* b = col + rp[v];
    for (int64_t k = 0; k < du; ++k)
        if (a[k] != b[k]) return false;
    return true;
}

struct RunGet {  // runs of equal top-32 hash bits (the sorted bits)
    const uint64_t* h;
    __device__ int64_t operator()(int64_t i) const { return (i == 0 || (h[i] >> 32) != (h[i - 1] >> 32)) ? 1 : 0; }
};
struct RunEmit {
    int32_t* rid;
    int64_t* rstart;
    __device__ void operator()(int64_t i, int64_t pos, int64_t f) const {
        rid[i] = (int32_t)(pos + f - 1);
        if (f) rstart[pos] = i;
    }
};

__global__ void k_verify(const uint32_t* __restrict__ sv, const int32_t* __restrict__ rid,
                         const int64_t* __restrict__ rstart, int64_t n, const int64_t* __restrict__ rp,
                         const int32_t* __restrict__ col, int32_t* __restrict__ rep) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = (int32_t)sv[i];
        const int64_t s = rstart[rid[i]];
        int32_t r = v;
        if (i != s) {
            const int32_t w = (int32_t)sv[s];
            if (same_row(rp, col, v, w)) {
                r = w;
            } else {  // hash collision: first equal row in the run (smallest id)
                for (int64_t j = s + 1; j < i; ++j) {
                    const int32_t u = (int32_t)sv[j];
                    if (same_row(rp, col, v, u)) {
                        r = u;
                        break;
                    }
                }
            }
        }
        rep[v] = r;
    }
}

// ----------------------------------------------------------------- chains --
__device__ __forceinline__ bool is_chain(const int64_t* rp, const int32_t* od, int32_t v) {
    return rp[v + 1] - rp[v] == 1 && od[v] == 1;
}

struct ChainGet {
    const int64_t* rp;
    const int32_t* od;
    __device__ int64_t operator()(int64_t v) const { return is_chain(rp, od, (int32_t)v) ? 1 : 0; }
};
struct ListEmit {
    int32_t* list;
    __device__ void operator()(int64_t v, int64_t pos, int64_t f) const {
        if (f) list[pos] = (int32_t)v;
    }
};

// Serial walk first: every chain vertex follows its pred links for up to
// CH_WALK steps (R-MAT / config-3 chains are short, so nearly all reach their
// head here); the pointer and distance it stops at are a valid list-ranking
// state, so pointer jumping only runs if some vertex did not resolve (long
// chains, pure cycles) -- flagged in *unresolved.
constexpr int CH_WALK = 64;
__global__ void k_chain_walk(const int32_t* __restrict__ cl, int64_t C, const int64_t* __restrict__ rp,
                             const int32_t* __restrict__ col, const int32_t* __restrict__ od,
                             int32_t* __restrict__ nxt, int32_t* __restrict__ dist, int* __restrict__ unresolved) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < C; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = cl[i];
        int32_t u = v;
        int d = 0;
        bool head = false;
        for (; d < CH_WALK; ++d) {
            const int32_t p = col[rp[u]];
            if (!is_chain(rp, od, p)) {
                head = true;
                break;
            }
            u = p;
        }
        nxt[v] = u;
        dist[v] = d;
        if (!head) atomicOr(unresolved, 1);
    }
}

__global__ void k_chain_jump(const int32_t* __restrict__ cl, int64_t C, const int32_t* __restrict__ nxt,
                             const int32_t* __restrict__ dist, int32_t* __restrict__ nxt2, int32_t* __restrict__ dist2) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < C; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = cl[i];
        const int32_t u = nxt[v];
        nxt2[v] = nxt[u];
        dist2[v] = min(dist[v] + dist[u], 1 << 30);
    }
}

__global__ void k_chain_finish(const int32_t* __restrict__ cl, int64_t C, const int32_t* __restrict__ nxt,
                               const int32_t* __restrict__ dist, const int64_t* __restrict__ rp,
                               const int32_t* __restrict__ col, const int32_t* __restrict__ od,
                               const int32_t* __restrict__ rep, int32_t* __restrict__ csrc, int32_t* __restrict__ ck) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < C; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = cl[i];
        const int32_t h = nxt[v];
        const bool head = !is_chain(rp, od, col[rp[h]]);  // h is a chain vertex whose pred is not
        if (head && dist[v] >= 1) {
            csrc[v] = rep[h];
            ck[v] = dist[v];
        }
    }
}

// ------------------------------------------------------- members / R view --
// In-degree-0 vertices are excluded from both lists: they are written once,
// in the first sweep (g->zlist), and are constant afterwards.
struct MemberGet {
    const int32_t* rep;
    const int32_t* ck;
    const int64_t* rp;
    __device__ int64_t operator()(int64_t v) const {
        return (rp[v + 1] > rp[v] && (rep[v] != (int32_t)v || ck[v] > 0)) ? 1 : 0;
    }
};
struct MemberEmit {
    const int32_t* rep;
    const int32_t* csrc;
    const int32_t* ck;
    int32_t* mvid;
    int32_t* msrc;
    int32_t* mk;
    __device__ void operator()(int64_t v, int64_t pos, int64_t f) const {
        if (!f) return;
        mvid[pos] = (int32_t)v;
        if (ck[v] > 0) {
            msrc[pos] = csrc[v];
            mk[pos] = ck[v];
        } else {
            msrc[pos] = rep[v];
            mk[pos] = 0;
        }
    }
};
struct ComputedGet {
    const int32_t* rep;
    const int32_t* ck;
    const int64_t* rp;
    __device__ int64_t operator()(int64_t v) const {
        return (rp[v + 1] > rp[v] && rep[v] == (int32_t)v && ck[v] == 0) ? 1 : 0;
    }
};
struct DegGet {
    const int64_t* rp;
    const int32_t* vid;
    int64_t nr;
    __device__ int64_t operator()(int64_t i) const {
        if (i >= nr) return 0;
        const int32_t v = vid[i];
        return rp[v + 1] - rp[v];
    }
};
struct PosEmit {
    int64_t* out;
    __device__ void operator()(int64_t i, int64_t pos, int64_t) const { out[i] = pos; }
};

// Reduced view col: rows vid[i] of the plain view's col, packed at rpR[i].
// Edge-parallel: every warp copies a fixed range of the OUTPUT (binary search
// for its first row, then batches of 32 rows), so a mega-hub row is spread
// over many warps instead of serialising one.
__global__ void k_copy_rows(const int32_t* __restrict__ vid, int64_t nr, const int64_t* __restrict__ rp,
                            const int32_t* __restrict__ col, const int64_t* __restrict__ rpR, int32_t* __restrict__ colR) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t ER = rpR[nr];
    // one contiguous output range per warp: a single binary search, then the
    // row walk carries over (a search per 1024-edge chunk was the bottleneck:
    // ~23 dependent loads each)
    const int64_t per = ((ER + nw - 1) / nw + 31) / 32 * 32;
    for (int64_t o0 = w0 * per; o0 < ER; o0 += nw * per) {
        const int64_t o1 = min(ER, o0 + per);
        int64_t lo = 0, hi = nr;  // last row i with rpR[i] <= o0
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (rpR[mid] <= o0)
                lo = mid;
            else
                hi = mid;
        }
        // rows of the chunk, 32 at a time: every lane fetches one row's
        // (output start, source - output offset); then the batch's output
        // range is copied element-parallel (lane k finds its row among the 32
        // by a shuffle binary search), so short rows do not idle the warp and
        // both the loads and the stores stay coalesced
        int64_t i0 = lo, o = o0;
        int64_t ostart = ER, delta = 0;
        if (i0 + lane < nr) {
            ostart = rpR[i0 + lane];
            delta = rp[vid[i0 + lane]] - ostart;
        }
        while (o < o1) {
            // the next batch's row metadata is loaded while this one is copied
            const int64_t rn = i0 + 32 + lane;
            const int64_t nos = rn < nr ? rpR[rn] : ER;
            const int32_t nvid = rn < nr ? vid[rn] : 0;
            const int64_t bend = min(o1, __shfl_sync(0xffffffffu, nos, 0));
            constexpr int CU = 8;  // 8 independent loads in flight per lane
            for (int64_t b0 = o; b0 < bend; b0 += 32 * CU) {
                int32_t val[CU];
#pragma unroll
                for (int u = 0; u < CU; ++u) {
                    const int64_t k = b0 + u * 32 + lane;
                    int q = 0;
#pragma unroll
                    for (int st = 16; st; st >>= 1) {
                        const int64_t v = __shfl_sync(0xffffffffu, ostart, q + st);
                        if (v <= k) q += st;
                    }
                    const int64_t dq = __shfl_sync(0xffffffffu, delta, q);
                    val[u] = k < bend ? __ldg(col + k + dq) : 0;
                }
#pragma unroll
                for (int u = 0; u < CU; ++u) {
                    const int64_t k = b0 + u * 32 + lane;
                    if (k < bend) colR[k] = val[u];
                }
            }
            o = bend;
            i0 += 32;
            ostart = nos;
            delta = rn < nr ? rp[nvid] - nos : 0;
        }
    }
}

// chain sources (the distinct source rows of chain members, k >= 1): compact
// index per row, and per member (-1 for identical members).  The synchronous
// reduced sweep keeps the last max_chain + 1 values of each chain source
// (delayed chain resolution, iterate.cu K-FINALIZE).
__global__ void k_mark_chain_src(const int32_t* __restrict__ mk, const int32_t* __restrict__ msrow, int64_t nm,
                                 int32_t* __restrict__ mark) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nm; i += (int64_t)gridDim.x * blockDim.x)
        if (mk[i] > 0) mark[msrow[i]] = 1;
}
struct MarkGet {
    const int32_t* mark;
    __device__ int64_t operator()(int64_t r) const { return mark[r] ? 1 : 0; }
};
struct MarkEmit {
    int32_t* idx;
    __device__ void operator()(int64_t r, int64_t pos, int64_t f) const { idx[r] = f ? (int32_t)pos : -1; }
};
__global__ void k_member_hist(const int32_t* __restrict__ mk, const int32_t* __restrict__ msrow, int64_t nm,
                              const int32_t* __restrict__ idx, int32_t* __restrict__ mh) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nm; i += (int64_t)gridDim.x * blockDim.x)
        mh[i] = mk[i] > 0 ? idx[msrow[i]] : -1;
}

__global__ void k_rowof(const int32_t* __restrict__ vid, int64_t nrows, int32_t* __restrict__ rowof) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x)
        rowof[vid[r]] = (int32_t)r;
}
__global__ void k_gather_i32(const int32_t* __restrict__ idx, int64_t cnt, const int32_t* __restrict__ tab,
                             int32_t* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = tab[idx[i]];
}

static unsigned grid_of(const Ctx& ctx, int64_t work) {
    int64_t g = (work + 255) / 256;
    int64_t cap = (int64_t)ctx.num_sms * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

static void clear_reductions(pr_graph* g, cudaStream_t s) {
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
    g->n_hsrc = 0;
    dfree(g->xm, s);
    free_view(g->reduced, s);
    g->n_members = 0;
    g->max_chain = 0;
    g->pre_done = false;
    g->pre_flags = 0;
}

static int find_identical(pr_graph* g, Ctx& ctx) {
    cudaStream_t s = ctx.stream;
    uint64_t* h = nullptr;
    uint64_t* h2 = nullptr;
    uint32_t* sv = nullptr;
    uint32_t* sv2 = nullptr;
    uint64_t* hv = nullptr;
    int32_t* rid = nullptr;
    int64_t* rstart = nullptr;
    TmpGuard tg_(ctx.stream);
    tg_.track(h);
    tg_.track(h2);
    tg_.track(sv);
    tg_.track(sv2);
    tg_.track(hv);
    tg_.track(rid);
    tg_.track(rstart);
    // only the rows of in-degree > 0 are hashed and sorted; the in-degree-0
    // vertices form the empty class directly
    const View& v = g->plain;
    const int64_t nr = v.nrows;
    if (g->nz > 0) PR_LAUNCH(ctx, k_rep_empty, grid_of(ctx, g->nz), 256, 0, (const int32_t*)g->zlist, g->nz, g->rep);
    if (nr == 0) return PR_OK;
    PR_TRY(dalloc(&h, (size_t)nr, s));
    PR_TRY(dalloc(&h2, (size_t)nr, s));
    PR_TRY(dalloc(&sv, (size_t)nr, s));
    PR_TRY(dalloc(&sv2, (size_t)nr, s));
    {
        const StreamArgs sa{v.col,  (const uint8_t*)v.sflags, v.step_row, v.nsteps, v.span_steps, v.nspans, v.bin,
                            v.bout, v.b_row, v.b_s0, v.b_s1, v.part_in, v.part_out, v.bticket};
        HashStreamPolicy hp{h, (int32_t)g->n_contrib, nullptr, 0, 0};
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ctx.num_sms, (v.nspans + SE_NT / 32 - 1) / (SE_NT / 32)));
        if (v.nspans > 0) PR_LAUNCH(ctx, k_rowhash_stream, (unsigned)grid, SE_NT, 0, hp, sa);
        PR_LAUNCH(ctx, k_hash_deg, grid_of(ctx, nr), 256, 0, h, nr, (const int32_t*)v.vid, (const int64_t*)g->row_ptr);
    }
    PR_LAUNCH(ctx, k_u32_from, grid_of(ctx, nr), 256, 0, (const int32_t*)v.vid, nr, sv);
    // stable sort of the rows (ids ascending) by the top 32 hash bits (4 radix
    // passes); equal top bits of different rows (~nr^2/2^33 pairs: a few
    // thousand on R-MAT-24, runs of two) are split exactly by k_verify
    bool alt = false;
    PR_TRY((radix_sort<uint64_t, true>(ctx, h, h2, sv, sv2, nr, 32, 64, &alt)));
    const uint64_t* hs = alt ? h2 : h;
    const uint32_t* svs = alt ? sv2 : sv;
    PR_TRY(dalloc(&rid, (size_t)nr, s));
    PR_TRY(dalloc(&rstart, (size_t)nr, s));
    PR_TRY((device_scan<int64_t>(ctx, nr, RunGet{hs}, RunEmit{rid, rstart}, (int64_t*)nullptr)));
    PR_LAUNCH(ctx, k_verify, grid_of(ctx, nr), 256, 0, svs, (const int32_t*)rid, (const int64_t*)rstart, nr,
              (const int64_t*)g->row_ptr, (const int32_t*)g->col, g->rep);
    dfree(h, s);
    dfree(h2, s);
    dfree(sv, s);
    dfree(sv2, s);
    dfree(rid, s);
    dfree(rstart, s);
    return PR_OK;
}

__global__ void k_fill_i32(int32_t* a, int64_t n, int32_t v, int iota) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = iota ? (int32_t)i : v;
}

__global__ void k_max_chain(const int32_t* __restrict__ ck, int64_t n, int* __restrict__ out) {
    int mx = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        mx = max(mx, ck[i]);
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

static int find_chains(pr_graph* g, Ctx& ctx) {
    cudaStream_t s = ctx.stream;
    const int64_t n = g->n;
    int64_t* cnt = nullptr;
    int32_t* cl = nullptr;
    TmpGuard tg_(ctx.stream);
    tg_.track(cnt);
    tg_.track(cl);
    PR_TRY(dalloc(&cnt, 1, s));
    PR_TRY(dalloc(&cl, (size_t)n, s));
    PR_TRY((device_scan<int64_t>(ctx, n, ChainGet{g->row_ptr, g->outdeg}, ListEmit{cl}, cnt)));
    int64_t C = 0;
    PR_TRY(read_count(ctx, cnt, &C));
    if (C > 0) {
        int32_t *nxt = nullptr, *dist = nullptr, *nxt2 = nullptr, *dist2 = nullptr;
        PR_TRY(dalloc(&nxt, (size_t)n, s));
        PR_TRY(dalloc(&dist, (size_t)n, s));
        PR_TRY(dalloc(&nxt2, (size_t)n, s));
        PR_TRY(dalloc(&dist2, (size_t)n, s));
        PR_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t), s));
        PR_LAUNCH(ctx, k_chain_walk, grid_of(ctx, C), 256, 0, (const int32_t*)cl, C, (const int64_t*)g->row_ptr,
                  (const int32_t*)g->col, (const int32_t*)g->outdeg, nxt, dist, (int*)cnt);
        int64_t unresolved = 0;
        PR_TRY(read_count(ctx, cnt, &unresolved));
        // ceil(log2 C) + 1 doublings suffice for any path (the walk only shortens them)
        const int rounds = unresolved ? bits_for((uint64_t)C) + 1 : 0;
        for (int r = 0; r < rounds; ++r) {
            PR_LAUNCH(ctx, k_chain_jump, grid_of(ctx, C), 256, 0, (const int32_t*)cl, C, (const int32_t*)nxt,
                      (const int32_t*)dist, nxt2, dist2);
            int32_t* t = nxt; nxt = nxt2; nxt2 = t;
            t = dist; dist = dist2; dist2 = t;
        }
        PR_LAUNCH(ctx, k_chain_finish, grid_of(ctx, C), 256, 0, (const int32_t*)cl, C, (const int32_t*)nxt,
                  (const int32_t*)dist, (const int64_t*)g->row_ptr, (const int32_t*)g->col,
                  (const int32_t*)g->outdeg, (const int32_t*)g->rep, g->chain_src, g->chain_k);
        dfree(nxt, s);
        dfree(dist, s);
        dfree(nxt2, s);
        dfree(dist2, s);
    }
    dfree(cl, s);
    dfree(cnt, s);
    return PR_OK;
}

int preprocess(pr_graph* g, uint32_t flags, Ctx& ctx) {
    cudaStream_t s = ctx.stream;
    const int64_t n = g->n;
    clear_reductions(g, s);
    if (flags == 0) return PR_OK;
    PR_TRY(dalloc(&g->rep, (size_t)n, s));
    PR_TRY(dalloc(&g->chain_src, (size_t)n, s));
    PR_TRY(dalloc(&g->chain_k, (size_t)n, s));
    PR_LAUNCH(ctx, k_fill_i32, grid_of(ctx, n), 256, 0, g->chain_src, n, -1, 0);
    PR_LAUNCH(ctx, k_fill_i32, grid_of(ctx, n), 256, 0, g->chain_k, n, 0, 0);
    if (flags & PR_PRE_IDENTICAL)
        PR_TRY(find_identical(g, ctx));
    else
        PR_LAUNCH(ctx, k_fill_i32, grid_of(ctx, n), 256, 0, g->rep, n, 0, 1);
    if (flags & PR_PRE_CHAIN) PR_TRY(find_chains(g, ctx));

    // members (scatter list) and the computed set R (reduced gather view)
    int64_t* cnt = nullptr;
    int32_t* mark = nullptr;  // chain sources' history index (below); declared here, where the guard lives
    int32_t* idx = nullptr;
    TmpGuard tg_(ctx.stream);
    tg_.track(cnt);
    tg_.track(mark);
    tg_.track(idx);
    PR_TRY(dalloc(&cnt, 3, s));
    PR_CUDA(cudaMemsetAsync(cnt, 0, 3 * sizeof(int64_t), s));
    PR_LAUNCH(ctx, k_max_chain, grid_of(ctx, n), 256, 0, (const int32_t*)g->chain_k, n, (int*)(cnt + 2));
    PR_TRY(dalloc(&g->mem_vid, (size_t)n, s));
    PR_TRY(dalloc(&g->mem_src, (size_t)n, s));
    PR_TRY(dalloc(&g->mem_k, (size_t)n, s));
    PR_TRY((device_scan<int64_t>(ctx, n, MemberGet{g->rep, g->chain_k, g->row_ptr},
                                 MemberEmit{g->rep, g->chain_src, g->chain_k, g->mem_vid, g->mem_src, g->mem_k}, cnt)));
    View& R = g->reduced;
    PR_TRY(dalloc(&R.vid, (size_t)n, s));
    PR_TRY((device_scan<int64_t>(ctx, n, ComputedGet{g->rep, g->chain_k, g->row_ptr}, ListEmit{R.vid}, cnt + 1)));
    int64_t h[3];
    PR_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
    PR_CUDA(cudaStreamSynchronize(s));
    g->n_members = h[0];
    R.nrows = h[1];
    g->max_chain = (int32_t)(h[2] & 0xffffffff);
    if (g->n_members == 0) {
        // nothing to resolve (config 5): the computed set is every row of
        // in-degree > 0, i.e. the plain view itself -- alias it, no copies
        dfree(R.vid, s);
        dfree(cnt, s);
        R = g->plain;
        R.alias = true;
        g->pre_done = true;
        g->pre_flags = flags;
        return PR_OK;
    }
    PR_TRY(dalloc(&R.row_ptr, (size_t)R.nrows + 1, s));
    R.owns_row_ptr = true;
    PR_TRY((device_scan<int64_t>(ctx, R.nrows + 1, DegGet{g->row_ptr, R.vid, R.nrows}, PosEmit{R.row_ptr}, cnt)));
    PR_TRY(read_count(ctx, cnt, &R.nedges));
    PR_TRY(dalloc(&R.col, (size_t)stream_pad(R.nedges), s));
    if (R.nrows > 0)
        PR_LAUNCH(ctx, k_copy_rows, std::min<unsigned>(grid_of(ctx, R.nrows * 32), (unsigned)ctx.num_sms * 8), 256, 0,
                  (const int32_t*)R.vid, R.nrows,
                  (const int64_t*)g->row_ptr, (const int32_t*)g->plain.col, (const int64_t*)R.row_ptr, R.col);
    PR_TRY(build_view_stream(R, ctx, (int32_t)g->n_contrib, g->outdeg, g->cidx));
    PR_TRY(build_view_blocked(R, ctx, g->n_contrib));
    // source row of every member in the reduced view (K-FINALIZE reads its S)
    if (g->n_members > 0) {
        int32_t* rowof = nullptr;
        PR_TRY(dalloc(&rowof, (size_t)n, s));
        if (R.nrows > 0)
            PR_LAUNCH(ctx, k_rowof, grid_of(ctx, R.nrows), 256, 0, (const int32_t*)R.vid, R.nrows, rowof);
        PR_TRY(dalloc(&g->mem_srow, (size_t)g->n_members, s));
        PR_LAUNCH(ctx, k_gather_i32, grid_of(ctx, g->n_members), 256, 0, (const int32_t*)g->mem_src, g->n_members,
                  (const int32_t*)rowof, g->mem_srow);
        dfree(rowof, s);
        PR_TRY(dalloc(&g->mem_info, (size_t)g->n_members, s));
        PR_LAUNCH(ctx, k_rinfo, grid_of(ctx, g->n_members), 256, 0, (const int32_t*)g->mem_vid, g->n_members,
                  (const int32_t*)g->outdeg, (const int32_t*)g->cidx, g->mem_info);
        if (g->max_chain > 0) {
            PR_TRY(dalloc(&mark, (size_t)std::max<int64_t>(R.nrows, 1), s));
            PR_TRY(dalloc(&idx, (size_t)std::max<int64_t>(R.nrows, 1), s));
            PR_CUDA(cudaMemsetAsync(mark, 0, sizeof(int32_t) * (size_t)std::max<int64_t>(R.nrows, 1), s));
            PR_LAUNCH(ctx, k_mark_chain_src, grid_of(ctx, g->n_members), 256, 0, (const int32_t*)g->mem_k,
                      (const int32_t*)g->mem_srow, g->n_members, mark);
            PR_TRY((device_scan<int64_t>(ctx, R.nrows, MarkGet{mark}, MarkEmit{idx}, cnt)));
            PR_TRY(read_count(ctx, cnt, &g->n_hsrc));
            PR_TRY(dalloc(&g->mem_h, (size_t)g->n_members, s));
            PR_LAUNCH(ctx, k_member_hist, grid_of(ctx, g->n_members), 256, 0, (const int32_t*)g->mem_k,
                      (const int32_t*)g->mem_srow, g->n_members, (const int32_t*)idx, g->mem_h);
            dfree(mark, s);
            dfree(idx, s);
        }
    }
    dfree(cnt, s);
    g->pre_done = true;
    g->pre_flags = flags;
    return PR_OK;
}

}  // namespace prgpu
