// ingest.cu -- K-INGEST: raw edge list -> deduplicated in-CSR + out-degrees
// (§5.2 "converted later to Compressed Sparse Row (CSR)
// format"; SPEC S:69-77 build_csr; readings Q-L, Q-V in DESIGN.md), plus the
// contrib relabelling, the plain view and the edge-stream tables of a view.
//
// Pipeline (all hand-written kernels):
//   pack    validate ids, drop self-loops, key = dst << b | src   (b = bits(n-1))
//   sort    LSD radix sort of the keys on 2b bits (8-bit digits)  -> (dst, src) order
//   unique  adjacent-different flags -> scan -> col_idx and row_ptr in one
//           pass (dedup; row starts from dst changes)
//   outdeg  histogram of src over the deduplicated edges
#include <stdlib.h>

#include <algorithm>

#include "internal.h"
#include "primitives.cuh"

namespace prgpu {

// key = dst << b | src; self-loops (and invalid ids, which abort the build)
// become the sentinel 2^(2b) - 1, which sorts last and is dropped by the
// unique pass (a real key equals it only for the self-loop (2^b-1, 2^b-1)).
// No compaction here: the sort and the unique pass do not care about order.
// Sharded create (world > 1): edges into vertices another rank owns (dst mod
// world != rank) become the sentinel too -- every id is still validated.
__global__ void k_pack(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t m, int64_t n,
                       int b, uint64_t sentinel, uint64_t* __restrict__ keys, int* __restrict__ err, int rank,
                       int world) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool any_bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        const int32_t s = src[i], t = dst[i];
        const bool bad = s < 0 || (int64_t)s >= n || t < 0 || (int64_t)t >= n;
        any_bad |= bad;
        const bool other = world > 1 && (t % world) != rank;
        keys[i] = (bad || s == t || other) ? sentinel : (((uint64_t)(uint32_t)t << b) | (uint32_t)s);
    }
    if (__any_sync(0xffffffffu, any_bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
}

// Sharded create: the rank's own edges (dst mod world == rank, no self-loops)
// appended compactly, every id validated.  One atomic per tile of PO_TILE
// edges (a single counter hit once per warp serialised: 4 ms on R-MAT-24);
// the order of the appended keys is irrelevant -- the sort that follows fixes it.
constexpr int PO_NT = 256, PO_IPT = 8, PO_TILE = PO_NT * PO_IPT;
__global__ void __launch_bounds__(PO_NT) k_pack_own(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                                    int64_t m, int64_t n, int b, uint64_t* __restrict__ keys,
                                                    unsigned long long* __restrict__ cnt, int* __restrict__ err,
                                                    int rank, int world) {
    __shared__ uint32_t wtot[PO_NT / 32];
    __shared__ unsigned long long tbase;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = lanemask_lt();
    bool any_bad = false;
    for (int64_t t0 = (int64_t)blockIdx.x * PO_TILE; t0 < m; t0 += (int64_t)gridDim.x * PO_TILE) {
        uint64_t key[PO_IPT];
        uint32_t rk[PO_IPT];
        uint32_t keepm = 0, wcount = 0;
#pragma unroll
        for (int j = 0; j < PO_IPT; ++j) {  // item j of the tile: warp-contiguous runs of 32
            const int64_t i = t0 + (int64_t)(j * PO_NT) + threadIdx.x;
            bool keep = false;
            key[j] = 0;
            if (i < m) {
                const int32_t s = src[i], t = dst[i];
                const bool bad = s < 0 || (int64_t)s >= n || t < 0 || (int64_t)t >= n;
                any_bad |= bad;
                keep = !bad && s != t && (t % world) == rank;
                key[j] = ((uint64_t)(uint32_t)t << b) | (uint32_t)s;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            rk[j] = wcount + __popc(bal & lt);
            wcount += __popc(bal);
            keepm |= (keep ? 1u : 0u) << j;
        }
        if (lane == 0) wtot[warp] = wcount;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < PO_NT / 32; ++w) {
                const uint32_t c = wtot[w];
                wtot[w] = tot;
                tot += c;
            }
            tbase = tot ? atomicAdd(cnt, (unsigned long long)tot) : 0ull;
        }
        __syncthreads();
        const unsigned long long base = tbase + wtot[warp];
#pragma unroll
        for (int j = 0; j < PO_IPT; ++j)
            if (keepm & (1u << j)) keys[base + rk[j]] = key[j];
        __syncthreads();
    }
    if (__any_sync(0xffffffffu, any_bad) && lane == 0) atomicOr(err, 1);
}

__global__ void k_check_ids(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t m, int64_t n,
                            int* __restrict__ err) {
    bool any_bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        any_bad |= src[i] < 0 || (int64_t)src[i] >= n || dst[i] < 0 || (int64_t)dst[i] >= n;
    if (__any_sync(0xffffffffu, any_bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
}

__global__ void k_outdeg(const int32_t* __restrict__ col, int64_t E, int32_t* __restrict__ outdeg) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&outdeg[col[e]], 1);
}

// outdeg without per-edge atomics: after the LSD passes over the src bits
// alone, the keys are grouped by src; a run [s, e) of source v adds e - s
// (two modular atomics per run: -s at its start, +e at its end).  Self-loop /
// sentinel keys (all 2b bits set) fall in the run of src = 2^b - 1 and are
// subtracted when that is a vertex; duplicates are subtracted by k_uniq_emit.
// Tiles of SR_TILE keys staged through shared memory (coalesced loads, one
// halo key each side), SR_IPT keys per thread.
constexpr int SR_NT = 256, SR_IPT = 8, SR_TILE = SR_NT * SR_IPT;
__global__ void __launch_bounds__(SR_NT) k_src_runs(const uint64_t* __restrict__ k, int64_t m, int b,
                                                    uint64_t sentinel, int64_t n, int32_t* __restrict__ outdeg) {
    __shared__ uint64_t sk[SR_TILE + 2];
    const uint64_t maskb = (1ull << b) - 1;
    for (int64_t tb = (int64_t)blockIdx.x * SR_TILE; tb < m; tb += (int64_t)gridDim.x * SR_TILE) {
        const int tn = (int)min((int64_t)SR_TILE, m - tb);
        for (int i = threadIdx.x; i < tn; i += SR_NT) sk[i + 1] = __ldcs(k + tb + i);
        if (threadIdx.x == 0) sk[0] = tb > 0 ? k[tb - 1] : ~0ull;
        if (threadIdx.x == 1) sk[tn + 1] = tb + tn < m ? k[tb + tn] : ~0ull;
        __syncthreads();
        unsigned nsent = 0;
#pragma unroll
        for (int j = 0; j < SR_IPT; ++j) {
            const int i = j * SR_NT + threadIdx.x;  // striped: conflict-free shared-memory reads
            if (i < tn) {
                const uint64_t key = sk[i + 1];
                const uint64_t v = key & maskb;
                if ((int64_t)v < n) {
                    const int64_t gi = tb + i;
                    unsigned* o = reinterpret_cast<unsigned*>(outdeg + v);
                    // a missing neighbour (~0) never matches: its masked bits
                    // are all ones only for the sentinel's run, handled below
                    if (gi == 0 || (sk[i] & maskb) != v) atomicAdd(o, (unsigned)(-gi));
                    if (gi == m - 1 || (sk[i + 2] & maskb) != v) atomicAdd(o, (unsigned)(gi + 1));
                    nsent += key == sentinel;
                }
            }
        }
        if (nsent) atomicSub(reinterpret_cast<unsigned*>(outdeg + maskb), nsent);
        __syncthreads();
    }
}

// ---- dedup + CSR in one pass over the sorted keys --------------------------
// Key i is kept iff it is not the sentinel and differs from key i-1.
// Kept key i lands at p = its rank among kept keys: col[p] = src; and when it
// starts row d = dst (dst of key i-1 differs, or i == 0), row_ptr[d'+1 .. d]
// = p for the previous dst d' (rows in between have in-degree 0); the rows
// after the last real key are closed by k_close_tail.  Reduce-
// then-scan with UQ_G fixed chunks (deterministic); tiles are staged through
// shared memory so global loads and the col stores are coalesced.
constexpr int UQ_NT = 256;
constexpr int UQ_IPT = 12;
constexpr int UQ_TILE = UQ_NT * UQ_IPT;

__device__ __forceinline__ bool uq_kept(const uint64_t* k, int64_t i, uint64_t sentinel) {
    const uint64_t key = k[i];
    return key != sentinel && (i == 0 || key != k[i - 1]);
}

__global__ void __launch_bounds__(UQ_NT) k_uniq_count(const uint64_t* __restrict__ k, int64_t n, int64_t per_cta,
                                                      uint64_t sentinel, int64_t* __restrict__ partial) {
    __shared__ int64_t sw[33];
    const int64_t b = (int64_t)blockIdx.x * per_cta;
    const int64_t e = min(n, b + per_cta);
    int64_t c = 0;
    for (int64_t i = b + threadIdx.x; i < e; i += UQ_NT) c += uq_kept(k, i, sentinel) ? 1 : 0;
    const int64_t tot = block_sum(c, sw);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(UQ_NT) k_uniq_emit(const uint64_t* __restrict__ k, int64_t n, int64_t per_cta,
                                                     uint64_t sentinel, int b,
                                                     const int64_t* __restrict__ partial, int32_t* __restrict__ col,
                                                     int64_t* __restrict__ row_ptr, int32_t* __restrict__ od_dup) {
    // striped: in stripe j, thread t handles tile item j*UQ_NT + t (conflict-
    // free shared-memory reads, adjacent lanes write adjacent row_ptr
    // entries); the output rank of a kept key = the kept count of the earlier
    // (stripe, warp) groups + its rank in the warp's ballot
    constexpr int NW = UQ_NT / 32;
    __shared__ uint64_t sk[UQ_TILE + 1];
    __shared__ int32_t so[UQ_TILE];
    __shared__ int32_t woff[UQ_IPT * NW + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = lanemask_lt();
    const uint64_t mask = (1ull << b) - 1;
    const int64_t cb = (int64_t)blockIdx.x * per_cta;
    const int64_t ce = min(n, cb + per_cta);
    int64_t base = partial[blockIdx.x];
    for (int64_t tb = cb; tb < ce; tb += UQ_TILE) {
        const int tn = (int)min((int64_t)UQ_TILE, ce - tb);
        for (int i = threadIdx.x; i < tn; i += UQ_NT) sk[i + 1] = k[tb + i];
        if (threadIdx.x == 0) sk[0] = tb > 0 ? k[tb - 1] : ~0ull;
        __syncthreads();
        uint32_t bal[UQ_IPT];
#pragma unroll
        for (int j = 0; j < UQ_IPT; ++j) {
            const int i = j * UQ_NT + threadIdx.x;
            bool kp = false;
            if (i < tn) {
                const uint64_t key = sk[i + 1];
                kp = key != sentinel && (tb + i == 0 || key != sk[i]);
            }
            bal[j] = __ballot_sync(0xffffffffu, kp);
            if (lane == 0) woff[j * NW + warp] = __popc(bal[j]);
            if (od_dup && i < tn && !kp && sk[i + 1] != sentinel)  // a duplicate: outdeg counted it once too often
                atomicSub(od_dup + (sk[i + 1] & mask), 1);
        }
        __syncthreads();
        if (warp == 0) {  // exclusive scan of the UQ_IPT * NW group counts (stripe-major = tile order)
            constexpr int G = UQ_IPT * NW;
            constexpr int PER = (G + 31) / 32;
            int v[PER], run = 0;
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int gi = lane * PER + u;
                v[u] = gi < G ? woff[gi] : 0;
                run += v[u];
            }
            int incl = run;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += t;
            }
            int ex = incl - run;
            __syncwarp();
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int gi = lane * PER + u;
                if (gi < G) woff[gi] = ex;
                ex += v[u];
            }
            if (lane == 31) woff[G] = incl;
        }
        __syncthreads();
        const int tile_tot = woff[UQ_IPT * NW];
#pragma unroll
        for (int j = 0; j < UQ_IPT; ++j) {
            const int i = j * UQ_NT + threadIdx.x;
            if (bal[j] & (1u << lane)) {
                const int q = woff[j * NW + warp] + __popc(bal[j] & lt);
                const uint64_t key = sk[i + 1];
                so[q] = (int32_t)(key & mask);
                const int64_t d = (int64_t)(key >> b);
                const int64_t dp = (tb + i == 0) ? -1 : (int64_t)(sk[i] >> b);
                const int64_t p = base + q;
                for (int64_t r = dp + 1; r <= d; ++r) row_ptr[r] = p;   // first edge of row d
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < tile_tot; i += UQ_NT) col[base + i] = so[i];
        base += tile_tot;
        __syncthreads();
    }
}

// Rows after the last real key's dst (the sentinels sort last) start at E:
// row_ptr[d_last + 1 .. nv] = E.  The last real key is found by a binary
// search for the first sentinel (no rows to close when every key is one).
__global__ void k_close_tail(const uint64_t* __restrict__ k, int64_t n, uint64_t sentinel, int b, int64_t nv,
                             const int64_t* __restrict__ total, int64_t* __restrict__ row_ptr) {
    __shared__ int64_t first_row;
    if (threadIdx.x == 0) {
        int64_t lo = 0, hi = n;  // first index with k[i] == sentinel (keys sorted ascending)
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (k[mid] == sentinel) hi = mid;
            else lo = mid + 1;
        }
        first_row = lo > 0 ? (int64_t)(k[lo - 1] >> b) + 1 : nv + 1;
    }
    __syncthreads();
    const int64_t E = *total;
    for (int64_t r = first_row + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= nv;
         r += (int64_t)gridDim.x * blockDim.x)
        row_ptr[r] = E;
}

int read_count(Ctx& ctx, const int64_t* dev, int64_t* host) {
    PR_CUDA(cudaMemcpyAsync(host, dev, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx.stream));
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    return PR_OK;
}

static unsigned grid_for(const Ctx& ctx, int64_t work, int nt) {
    int64_t g = (work + nt - 1) / nt;
    int64_t cap = (int64_t)ctx.num_sms * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

// Host edge arrays (pinned, single rank): the copy in runs in CH_K chunks on a
// copy stream; each chunk is sorted as soon as it has arrived (pack fused into
// its first pass, the src runs counted per chunk) and merged into the sorted
// prefix of the chunks before it (merge path), so only the last chunk's sort
// and one merge follow the last byte over PCIe.
// chunks: R-MAT-24 e2e step 141.2 / 138.6 / 137.1 / 143.0 ms for 4 / 8 / 16 / 32
// (the ladder's merges grow with the chunk count; the tail shrinks with it)
constexpr int CH_K = 32;  // most chunks (PRGPU_CHUNKS, default 16)
constexpr int64_t CH_MIN = (int64_t)1 << 22;
bool ingest_chunked_applies(int64_t n, int64_t m) {
    const char* e = getenv("PRGPU_CHUNKED");
    return n > 1 && m >= CH_MIN && !(e && e[0] == '0');
}

int ingest(pr_graph* g, const int32_t* src, const int32_t* dst, Ctx& ctx, int rank, int world, bool host_src) {
    const int64_t n = g->n, m = g->m_raw;
    const int b = bits_for((uint64_t)(n - 1));
    cudaStream_t s = ctx.stream;

    uint64_t* keys = nullptr;
    uint64_t* keys_alt = nullptr;
    int64_t* scratch = nullptr;  // [0] = E, [1] = error flag
    uint64_t* keys_m = nullptr;  // host_src: the third buffer of the merge ladder
    int32_t* dsrc = nullptr;     // host_src: device copies of the edge arrays
    int32_t* ddst = nullptr;
    TmpGuard tg_(ctx.stream);
    tg_.track(keys);
    tg_.track(keys_alt);
    tg_.track(scratch);
    tg_.track(keys_m);
    tg_.track(dsrc);
    tg_.track(ddst);

    PR_TRY(dalloc(&scratch, 2, s));
    PR_CUDA(cudaMemsetAsync(scratch, 0, 2 * sizeof(int64_t), s));
    // n == 1 (b == 0): every edge is a self-loop, nothing to sort
    int64_t mk = b > 0 ? m : 0;
    bool od_runs = false;  // outdeg counted from the src runs of the partial sort
    const uint64_t sentinel = b > 0 ? ((2 * b >= 64) ? ~0ull : ((1ull << (2 * b)) - 1)) : 0ull;

    // pack, sort by (dst, src), deduplicate + CSR (row_ptr, col_idx) in one pass.
    // Single rank with 16-byte aligned edge arrays: the pack runs inside the
    // first radix pass (RsPack; R-MAT-24: no 2 GB key write + read-back).
    RsPack pack;
    const bool fuse_pack = world == 1 && mk > 1 && ((((uintptr_t)src) | ((uintptr_t)dst)) & 15) == 0 &&
                           !(getenv("PRGPU_PACK") && getenv("PRGPU_PACK")[0] == '0');
    PR_TRY(dalloc(&g->row_ptr, (size_t)n + 1, s));
    PR_CUDA(cudaMemsetAsync(g->row_ptr, 0, sizeof(int64_t) * (size_t)(n + 1), s));  // E == 0: all rows empty
    if (mk > 0) {
        PR_TRY(dalloc(&keys, (size_t)mk, s));
        if (world > 1) {  // sharded create: only this rank's edges, compacted (the sort sees 1/world of them)
            PR_LAUNCH(ctx, k_pack_own, grid_for(ctx, (mk + PO_IPT - 1) / PO_IPT, PO_NT), PO_NT, 0, src, dst, mk, n, b,
                      keys, (unsigned long long*)scratch, (int*)(scratch + 1), rank, world);
            int64_t h2[2];
            PR_CUDA(cudaMemcpyAsync(h2, scratch, sizeof(h2), cudaMemcpyDeviceToHost, s));
            PR_CUDA(cudaStreamSynchronize(s));
            if (h2[1] != 0) {
                set_error("pr_graph_create: vertex id outside [0, n)");
                return PR_EINVAL;
            }
            mk = h2[0];
            PR_CUDA(cudaMemsetAsync(scratch, 0, sizeof(int64_t), s));
        } else if (host_src) {
            // keys formed chunk by chunk below, from the device copies of the chunks
        } else if (fuse_pack) {
            pack.src = src;  // the first radix pass forms the keys itself
            pack.dst = dst;
            pack.n = n;
            pack.b = b;
            pack.sentinel = sentinel;
            pack.err = (int*)(scratch + 1);
        } else {
            PR_LAUNCH(ctx, k_pack, grid_for(ctx, mk, 256), 256, 0, src, dst, mk, n, b, sentinel, keys,
                      (int*)(scratch + 1), rank, world);
        }
    }
    PR_TRY(dalloc(&g->col, (size_t)(mk > 0 ? mk : 1), s));
    if (mk > 0) {
        PR_TRY(dalloc(&keys_alt, (size_t)mk, s));
        PR_TRY(dalloc(&g->outdeg, (size_t)n, s));
        PR_CUDA(cudaMemsetAsync(g->outdeg, 0, sizeof(int32_t) * (size_t)n, s));
        // sort the src bits, count the src runs (outdeg), then the dst bits --
        // also when the split costs one more pass (b not a multiple of 8): a
        // radix pass is ~5 ms per 1e9 keys, per-edge atomics over the
        // deduplicated sources ~27 ms (config 5, b = 26: create 117 -> 98 ms);
        // b < 8 or PRGPU_OD_RUNS=0: one sort, then per-edge atomics
        od_runs = b >= 8 && !(getenv("PRGPU_OD_RUNS") && getenv("PRGPU_OD_RUNS")[0] == '0');
        const uint64_t* sorted = nullptr;
        if (host_src) {
            PR_TRY(dalloc(&dsrc, (size_t)mk, s));
            PR_TRY(dalloc(&ddst, (size_t)mk, s));
            PR_TRY(dalloc(&keys_m, (size_t)mk, s));
            const int kreq = std::min(CH_K, std::max(1, getenv("PRGPU_CHUNKS") ? atoi(getenv("PRGPU_CHUNKS")) : 16));
            int64_t C = (mk + kreq - 1) / kreq;
            C = (C + RS_TILE - 1) / RS_TILE * RS_TILE;
            const int K = (int)std::max<int64_t>(1, mk / C);  // the last chunk takes the remainder: len in [C, 2C)
            cudaStream_t cs = nullptr;
            cudaEvent_t ev[CH_K + 1] = {};
            struct StreamEvents {  // released on every exit (after the work queued on them)
                cudaStream_t* cs;
                cudaEvent_t* ev;
                bool joined = false;  // the compute stream waits for every chunk copy
                ~StreamEvents() {
                    // early error exit: copies may still be landing in buffers the
                    // guard is about to free on the compute stream
                    if (!joined && *cs) cudaStreamSynchronize(*cs);
                    for (int i = 0; i <= CH_K; ++i)
                        if (ev[i]) cudaEventDestroy(ev[i]);
                    if (*cs) cudaStreamDestroy(*cs);
                }
            } se_{&cs, ev};
            PR_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            for (int i = 0; i <= CH_K; ++i) PR_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
            PR_CUDA(cudaEventRecord(ev[CH_K], s));  // the copy buffers exist on the copy stream
            PR_CUDA(cudaStreamWaitEvent(cs, ev[CH_K], 0));
            auto off_of = [&](int i) { return i < K ? (int64_t)i * C : mk; };
            for (int i = 0; i < K; ++i) {
                const int64_t off = off_of(i), len = off_of(i + 1) - off;
                PR_CUDA(cudaMemcpyAsync(dsrc + off, src + off, sizeof(int32_t) * (size_t)len, cudaMemcpyHostToDevice, cs));
                PR_CUDA(cudaMemcpyAsync(ddst + off, dst + off, sizeof(int32_t) * (size_t)len, cudaMemcpyHostToDevice, cs));
                PR_CUDA(cudaEventRecord(ev[i], cs));
            }
            uint64_t* R = nullptr;        // the buffer the sorted chunks land in (same parity for all)
            uint64_t* P = nullptr;        // the radix ping-pong partner
            const uint64_t* acc = nullptr;
            for (int i = 0; i < K; ++i) {
                const int64_t off = off_of(i), len = off_of(i + 1) - off;
                PR_CUDA(cudaStreamWaitEvent(s, ev[i], 0));
                RsPack pk;
                pk.src = dsrc + off;
                pk.dst = ddst + off;
                pk.n = n;
                pk.b = b;
                pk.sentinel = sentinel;
                pk.err = (int*)(scratch + 1);
                const uint64_t* res = nullptr;
                if (od_runs) {
                    bool a1 = false, a2 = false;
                    PR_TRY((radix_sort<uint64_t, false>(ctx, keys + off, keys_alt + off, nullptr, nullptr, len, 0, b,
                                                        &a1, &pk)));
                    uint64_t* cur = (a1 ? keys_alt : keys) + off;
                    uint64_t* oth = (a1 ? keys : keys_alt) + off;
                    PR_LAUNCH(ctx, k_src_runs, grid_for(ctx, (len + SR_IPT - 1) / SR_IPT, SR_NT), SR_NT, 0,
                              (const uint64_t*)cur, len, b, sentinel, n, g->outdeg);
                    PR_TRY((radix_sort<uint64_t, false>(ctx, cur, oth, nullptr, nullptr, len, b, 2 * b, &a2)));
                    res = a2 ? oth : cur;
                } else {
                    bool alt = false;
                    PR_TRY((radix_sort<uint64_t, false>(ctx, keys + off, keys_alt + off, nullptr, nullptr, len, 0,
                                                        2 * b, &alt, &pk)));
                    res = (alt ? keys_alt : keys) + off;
                }
                if (i == 0) {
                    R = const_cast<uint64_t*>(res);
                    P = R == keys ? keys_alt : keys;
                    acc = R;
                    continue;
                }
                // acc = sorted [0, off); merge with chunk i into P, M, P, ... (never
                // into R, whose next chunks are still to come)
                uint64_t* out = (i & 1) ? P : keys_m;
                PR_TRY(merge_u64(ctx, acc, off, res, len, out));
                acc = out;
            }
            se_.joined = true;
            sorted = acc;
        } else if (od_runs) {
            bool a1 = false, a2 = false;
            PR_TRY((radix_sort<uint64_t, false>(ctx, keys, keys_alt, nullptr, nullptr, mk, 0, b, &a1,
                                                fuse_pack ? &pack : nullptr)));
            uint64_t* cur = a1 ? keys_alt : keys;
            uint64_t* oth = a1 ? keys : keys_alt;
            PR_LAUNCH(ctx, k_src_runs, grid_for(ctx, (mk + SR_IPT - 1) / SR_IPT, SR_NT), SR_NT, 0, (const uint64_t*)cur,
                      mk, b, sentinel, n, g->outdeg);
            PR_TRY((radix_sort<uint64_t, false>(ctx, cur, oth, nullptr, nullptr, mk, b, 2 * b, &a2)));
            sorted = a2 ? oth : cur;
        } else {
            bool alt = false;
            PR_TRY((radix_sort<uint64_t, false>(ctx, keys, keys_alt, nullptr, nullptr, mk, 0, 2 * b, &alt,
                                                fuse_pack ? &pack : nullptr)));
            sorted = alt ? keys_alt : keys;
        }
        int uq_occ = 0;  // every CTA of the emit pass resident (fixed chunks: no second wave)
        PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&uq_occ, k_uniq_emit, UQ_NT, 0));
        int64_t G = std::min<int64_t>((mk + UQ_TILE - 1) / UQ_TILE, (int64_t)ctx.num_sms * std::max(1, uq_occ));
        int64_t per = (mk + G - 1) / G;
        per = (per + UQ_TILE - 1) / UQ_TILE * UQ_TILE;
        G = (mk + per - 1) / per;
        int64_t* part = nullptr;
        PR_TRY(dalloc(&part, (size_t)G, s));
        PR_LAUNCH(ctx, k_uniq_count, (unsigned)G, UQ_NT, 0, sorted, mk, per, sentinel, part);
        PR_LAUNCH(ctx, (k_scan_partials<int64_t>), 1, 1024, 0, part, G, scratch);
        PR_LAUNCH(ctx, k_uniq_emit, (unsigned)G, UQ_NT, 0, sorted, mk, per, sentinel, b, (const int64_t*)part,
                  g->col, g->row_ptr, od_runs ? g->outdeg : nullptr);
        PR_LAUNCH(ctx, k_close_tail, grid_for(ctx, n, 256), 256, 0, sorted, mk, sentinel, b, n,
                  (const int64_t*)scratch, g->row_ptr);
        dfree(part, s);
        dfree(keys, s);
        dfree(keys_alt, s);
    } else if (m > 0) {  // n == 1: still validate the ids
        PR_LAUNCH(ctx, k_check_ids, grid_for(ctx, m, 256), 256, 0, src, dst, m, n, (int*)(scratch + 1));
    }
    int64_t h[2];
    PR_CUDA(cudaMemcpyAsync(h, scratch, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PR_CUDA(cudaStreamSynchronize(s));
    if (h[1] != 0) {
        dfree(scratch, s);
        set_error("pr_graph_create: vertex id outside [0, n)");
        return PR_EINVAL;
    }
    g->E = h[0];

    // outdeg from the sources of the deduplicated edges (unless the src runs gave it)
    if (!g->outdeg) {
        PR_TRY(dalloc(&g->outdeg, (size_t)n, s));
        PR_CUDA(cudaMemsetAsync(g->outdeg, 0, sizeof(int32_t) * (size_t)n, s));
    }
    if (g->E > 0 && !od_runs)
        PR_LAUNCH(ctx, k_outdeg, grid_for(ctx, g->E, 256), 256, 0, (const int32_t*)g->col, g->E, g->outdeg);
    dfree(scratch, s);
    return PR_OK;
}

// ---------------------------------------------------------------- relabel --
// The gather reads contrib values y(u) = x(u)/outdeg(u) only for sources u
// (outdeg > 0).  They are stored compactly (~44 % of n on R-MAT; DESIGN.md
// "Data layout"): the K hottest by (outdeg desc, id asc), so the hottest
// contribs share sectors and fit the gather's on-chip tiers, then the rest in
// row order (ColdGet below).  cidx[v] = position, or -1 for dangling v.
struct NdGet {
    const int32_t* od;
    __device__ int64_t operator()(int64_t v) const { return od[v] > 0 ? 1 : 0; }
};
struct NdEmit {
    const int32_t* od;
    uint64_t* keys;
    int b;
    int32_t maxod;
    __device__ void operator()(int64_t v, int64_t pos, int64_t f) const {
        if (f) keys[pos] = ((uint64_t)(uint32_t)(maxod - od[v]) << b) | (uint64_t)v;
    }
};

__global__ void k_max_i32(const int32_t* __restrict__ a, int64_t n, int* __restrict__ out) {
    int mx = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        mx = max(mx, a[i]);
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

__global__ void k_set_cidx(const uint64_t* __restrict__ sorted, int64_t cnt, uint64_t vmask, int32_t* __restrict__ cidx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        cidx[sorted[i] & vmask] = (int32_t)i;
}

// col (streamed once: evict-first loads and stores) through the cidx table
// (random: kept in L2 with evict_last; 4 bytes x n, beside the 8E-byte stream)
__global__ void k_map_col(const int32_t* __restrict__ col, int64_t E, const int32_t* __restrict__ cidx,
                          int32_t* __restrict__ out) {
    const uint64_t pol = policy_evict_last();
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t E4 = E >> 2;  // col and out are 16-byte aligned (pool allocations)
    const int4* __restrict__ c4 = reinterpret_cast<const int4*>(col);
    int4* __restrict__ o4 = reinterpret_cast<int4*>(out);
    for (int64_t i = t0; i < E4; i += 2 * T) {
        int4 a = __ldcs(c4 + i), b = make_int4(0, 0, 0, 0);
        const bool two = i + T < E4;
        if (two) b = __ldcs(c4 + i + T);
        int4 ra, rb;
        ra.x = ld_hint_s32(cidx + a.x, pol);
        ra.y = ld_hint_s32(cidx + a.y, pol);
        ra.z = ld_hint_s32(cidx + a.z, pol);
        ra.w = ld_hint_s32(cidx + a.w, pol);
        if (two) {
            rb.x = ld_hint_s32(cidx + b.x, pol);
            rb.y = ld_hint_s32(cidx + b.y, pol);
            rb.z = ld_hint_s32(cidx + b.z, pol);
            rb.w = ld_hint_s32(cidx + b.w, pol);
        }
        __stcs(o4 + i, ra);
        if (two) __stcs(o4 + i + T, rb);
    }
    for (int64_t e = (E4 << 2) + t0; e < E; e += T) out[e] = cidx[col[e]];
}

struct ZeroInGet {
    const int64_t* rp;
    __device__ int64_t operator()(int64_t v) const { return rp[v + 1] == rp[v] ? 1 : 0; }
};
struct NonZeroInGet {
    const int64_t* rp;
    __device__ int64_t operator()(int64_t v) const { return rp[v + 1] != rp[v] ? 1 : 0; }
};
struct VListEmit {
    int32_t* list;
    __device__ void operator()(int64_t v, int64_t pos, int64_t f) const {
        if (f) list[pos] = (int32_t)v;
    }
};
// rows of in-degree > 0: vid[i] = v, row_ptr_view[i] = row_ptr[v]; the last
// vertex also closes the view with row_ptr_view[nrows] = row_ptr[n] = E.
struct NonZeroEmit {
    const int64_t* rp;
    int32_t* vid;
    int64_t* rpv;
    int64_t n;
    int64_t nrows;
    __device__ void operator()(int64_t v, int64_t pos, int64_t f) const {
        if (f) {
            vid[pos] = (int32_t)v;
            rpv[pos] = rp[v];
        }
        if (v == n - 1) rpv[nrows] = rp[n];
    }
};

// Slots [K, n_contrib) in row order (PRGPU_DEG_SLOTS): the sources that have
// rows (in-degree > 0) by increasing id, then those of in-degree 0 -- so the
// contrib stores of consecutive rows in K-FINALIZE land in consecutive slots.
struct ColdGet {
    const int32_t* cidx;
    const int64_t* rp;
    int64_t K;
    int rows;  // 1: sources with rows, 0: sources of in-degree 0
    __device__ int64_t operator()(int64_t v) const {
        return (cidx[v] >= K && (int)(rp[v + 1] > rp[v]) == rows) ? 1 : 0;
    }
};
struct ColdEmit {
    int32_t* cidx;
    int64_t K;
    const int64_t* base;  // slots already taken by the first group (device), or null
    __device__ void operator()(int64_t v, int64_t pos, int64_t f) const {
        if (f) cidx[v] = (int32_t)(K + (base ? *base : 0) + pos);
    }
};

int build_relabel(pr_graph* g, Ctx& ctx, bool cold_rows) {
    cudaStream_t s = ctx.stream;
    const int64_t n = g->n;
    int64_t* scratch = nullptr;
    TmpGuard tg_(ctx.stream);
    tg_.track(scratch);

    PR_TRY(dalloc(&scratch, 2, s));
    PR_CUDA(cudaMemsetAsync(scratch, 0, 2 * sizeof(int64_t), s));
    PR_LAUNCH(ctx, k_max_i32, grid_for(ctx, n, 256), 256, 0, (const int32_t*)g->outdeg, n, (int*)(scratch + 1));
    int64_t h[2];
    PR_CUDA(cudaMemcpyAsync(h, scratch, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PR_CUDA(cudaStreamSynchronize(s));
    const int32_t maxod = (int32_t)(h[1] & 0xffffffff);
    const int b = bits_for((uint64_t)(n - 1));
    const char* mode = getenv("PRGPU_RELABEL");
    const bool by_degree = !(mode && mode[0] == 'i');  // "id": keep id order (ablation)

    uint64_t* keys = nullptr;
    uint64_t* keys_alt = nullptr;
    tg_.track(keys);
    tg_.track(keys_alt);
    PR_TRY(dalloc(&keys, (size_t)n, s));
    PR_TRY((device_scan<int64_t>(ctx, n, NdGet{g->outdeg},
                                 NdEmit{g->outdeg, keys, b, by_degree ? maxod : 0}, scratch)));
    PR_TRY(read_count(ctx, scratch, &g->n_contrib));
    const int64_t cnt = g->n_contrib;
    PR_TRY(dalloc(&g->cidx, (size_t)n, s));
    PR_CUDA(cudaMemsetAsync(g->cidx, 0xff, sizeof(int32_t) * (size_t)n, s));
    const uint64_t* sorted = keys;
    if (by_degree && cnt > 1) {
        PR_TRY(dalloc(&keys_alt, (size_t)cnt, s));
        bool alt = false;
        PR_TRY((radix_sort<uint64_t, false>(ctx, keys, keys_alt, nullptr, nullptr, cnt, b,
                                            b + bits_for((uint64_t)maxod), &alt)));
        sorted = alt ? keys_alt : keys;
    }
    if (cnt > 0)
        PR_LAUNCH(ctx, k_set_cidx, grid_for(ctx, cnt, 256), 256, 0, sorted, cnt,
                  b ? ((1ull << b) - 1) : 0ull, g->cidx);
    // only the K = 2^20 hottest keep the degree order (the gather's shared-
    // memory and L1 tiers and the sharded hot copies use slots < SE_L1_TIER; the
    // rest of the first 2^20 keeps the gather's L2 locality): R-MAT-24 reduced
    // K-FINALIZE 0.091 -> 0.076 ms, K-GATHER unchanged (K = 32K / 128K / 512K
    // / 1M / 2M / 4M / all: step 105.65 / 105.86 / 105.37 / 105.34 / 105.54 /
    // 106.04 / 106.63 ms, profiles/r2/ab_degslots.txt).  PRGPU_DEG_SLOTS=k
    // sets K (k <= 0: every slot in degree order).
    const char* ds = getenv("PRGPU_DEG_SLOTS");
    const int64_t kds = ds ? atoll(ds) : (int64_t)1 << 20;
    const int64_t K = kds <= 0 ? cnt : std::max<int64_t>(kds, SE_L1_TIER);
    if (by_degree && cold_rows && K < cnt) {
        PR_TRY((device_scan<int64_t>(ctx, n, ColdGet{g->cidx, g->row_ptr, K, 1}, ColdEmit{g->cidx, K, nullptr},
                                     scratch + 1)));
        PR_TRY((device_scan<int64_t>(ctx, n, ColdGet{g->cidx, g->row_ptr, K, 0},
                                     ColdEmit{g->cidx, K, (const int64_t*)(scratch + 1)}, (int64_t*)nullptr)));
    }
    // zero in-degree vertices (written once, in sweep 1) and the plain view:
    // the rows of in-degree > 0 (identity view when there are no empty rows)
    View& v = g->plain;
    PR_TRY(dalloc(&g->zlist, (size_t)n, s));
    PR_TRY((device_scan<int64_t>(ctx, n, ZeroInGet{g->row_ptr}, VListEmit{g->zlist}, scratch)));
    PR_TRY(read_count(ctx, scratch, &g->nz));
    v.nedges = g->E;
    v.owns_row_ptr = false;
    v.vid = nullptr;
    v.row_ptr = g->row_ptr;
    v.nrows = n;
    if (g->nz > 0) {
        v.nrows = n - g->nz;
        PR_TRY(dalloc(&v.vid, (size_t)(v.nrows > 0 ? v.nrows : 1), s));
        PR_TRY(dalloc(&v.row_ptr, (size_t)v.nrows + 1, s));
        v.owns_row_ptr = true;
        PR_TRY((device_scan<int64_t>(ctx, n, NonZeroInGet{g->row_ptr},
                                     NonZeroEmit{g->row_ptr, v.vid, v.row_ptr, n, v.nrows}, scratch)));
    }
    PR_TRY(dalloc(&v.col, (size_t)stream_pad(g->E), s));
    if (g->E > 0)
        PR_LAUNCH(ctx, k_map_col, grid_for(ctx, g->E, 256), 256, 0, (const int32_t*)g->col, g->E,
                  (const int32_t*)g->cidx, v.col);
    dfree(keys, s);
    dfree(keys_alt, s);
    dfree(scratch, s);
    return PR_OK;
}

void free_view(View& v, cudaStream_t s) {
    if (v.alias) {
        v = View{};
        return;
    }
    free_phase_view(v, s);
    if (v.owns_row_ptr) dfree(v.row_ptr, s);
    v.row_ptr = nullptr;
    dfree(v.col, s);
    dfree(v.vid, s);
    v.nrows = v.nedges = 0;
    dfree(v.sflags, s);
    dfree(v.step_row, s);
    free_spans(v, s);
    dfree(v.sums, s);
    dfree(v.rinfo, s);
    v.nsteps = v.nspans = v.nbound = 0;
    v.span_steps = 1;
    if (v.seg) {
        for (int i = 0; i < v.nseg; ++i) free_view(v.seg[i], s);
        delete[] v.seg;
        v.seg = nullptr;
    }
    v.nseg = 0;
}

// ------------------------------------------------------------ view stream --
// Tables of the edge-stream engine (streamengine.cuh) for a view whose rows
// all have in-degree >= 1: row-start bits, step_row, spans and boundary rows.
__global__ void k_pad_col(int32_t* __restrict__ col, int64_t E, int64_t Epad, int32_t pad) {
    for (int64_t e = E + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < Epad; e += (int64_t)gridDim.x * blockDim.x)
        col[e] = pad;
}
__global__ void k_row_flags(const int64_t* __restrict__ rp, int64_t nrows, uint32_t* __restrict__ fl) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = rp[r];
        atomicOr(fl + (e >> 5), 1u << (e & 31));
    }
}
// step_row[s] = first row r with rp[r] >= s * SE_STEP (rp strictly increasing)
__global__ void k_step_row(const int64_t* __restrict__ rp, int64_t nrows, int64_t nsteps, int32_t* __restrict__ sr) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s <= nsteps; s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t key = s * SE_STEP;
        int64_t lo = 0, hi = nrows;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (rp[mid] < key)
                lo = mid + 1;
            else
                hi = mid;
        }
        sr[s] = (int32_t)lo;
    }
}
struct BoundGet {
    const int64_t* rp;
    int64_t span_e;
    __device__ int64_t operator()(int64_t r) const { return rp[r] / span_e != (rp[r + 1] - 1) / span_e ? 1 : 0; }
};
struct BoundEmit {
    const int64_t* rp;
    int64_t span_e;
    int32_t *b_row, *b_s0, *b_s1, *bin, *bout;
    __device__ void operator()(int64_t r, int64_t b, int64_t f) const {
        if (!f) return;
        const int64_t s0 = rp[r] / span_e, s1 = (rp[r + 1] - 1) / span_e;
        b_row[b] = (int32_t)r;
        b_s0[b] = (int32_t)s0;
        b_s1[b] = (int32_t)s1;
        bout[s0] = (int32_t)b;
        for (int64_t s = s0 + 1; s <= s1; ++s) bin[s] = (int32_t)b;
    }
};

__global__ void k_rinfo(const int32_t* __restrict__ vid, int64_t nrows, const int32_t* __restrict__ od,
                        const int32_t* __restrict__ cidx, int2* __restrict__ info) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = vid ? vid[r] : (int32_t)r;
        info[r] = make_int2(od[v], cidx[v]);
    }
}

int build_view_stream(View& v, Ctx& ctx, int32_t pad_slot, const int32_t* outdeg, const int32_t* cidx) {
    cudaStream_t s = ctx.stream;
    v.nsteps = v.nspans = v.nbound = 0;
    if (v.nrows == 0 || v.nedges == 0) return PR_OK;
    const int64_t Epad = stream_pad(v.nedges);
    v.nsteps = Epad / SE_STEP;
    // one span per resident warp (1 CTA of SE_NT threads per SM): the gather's
    // work per step is uniform, and every span costs two fences and a ticket
    const int64_t warps = (int64_t)ctx.num_sms * (SE_NT / 32);
    int64_t ss = (v.nsteps + warps - 1) / warps;
    if (ss < 1) ss = 1;
    if (const char* e = getenv("PRGPU_SPAN")) {  // tuning override
        const int64_t o = atoll(e);
        if (o >= 1) ss = o;
    }
    if (Epad > v.nedges)
        PR_LAUNCH(ctx, k_pad_col, 1, 256, 0, v.col, v.nedges, Epad, pad_slot);
    PR_TRY(dalloc(&v.sflags, (size_t)v.nsteps * 8, s));
    PR_CUDA(cudaMemsetAsync(v.sflags, 0, sizeof(uint32_t) * (size_t)v.nsteps * 8, s));
    PR_LAUNCH(ctx, k_row_flags, grid_for(ctx, v.nrows, 256), 256, 0, (const int64_t*)v.row_ptr, v.nrows, v.sflags);
    PR_TRY(dalloc(&v.step_row, (size_t)v.nsteps + 1, s));
    PR_LAUNCH(ctx, k_step_row, grid_for(ctx, v.nsteps + 1, 256), 256, 0, (const int64_t*)v.row_ptr, v.nrows,
              v.nsteps, v.step_row);
    PR_TRY(build_spans(v, ctx, ss));
    if (outdeg) {  // a top-level view (sub-views of a blocked view accumulate into their parent's sums)
        PR_TRY(dalloc(&v.sums, (size_t)v.nrows, s));
        PR_TRY(dalloc(&v.rinfo, (size_t)v.nrows, s));
        PR_LAUNCH(ctx, k_rinfo, grid_for(ctx, v.nrows, 256), 256, 0, (const int32_t*)v.vid, v.nrows, outdeg, cidx,
                  v.rinfo);
    }
    return PR_OK;
}

// The span tables of a view for spans of ss steps (needs row_ptr, nsteps).
int build_spans(View& v, Ctx& ctx, int64_t ss) {
    cudaStream_t s = ctx.stream;
    v.span_steps = ss;
    v.nspans = (v.nsteps + ss - 1) / ss;
    PR_TRY(dalloc(&v.bin, (size_t)v.nspans, s));
    PR_TRY(dalloc(&v.bout, (size_t)v.nspans, s));
    PR_CUDA(cudaMemsetAsync(v.bin, 0xff, sizeof(int32_t) * (size_t)v.nspans, s));
    PR_CUDA(cudaMemsetAsync(v.bout, 0xff, sizeof(int32_t) * (size_t)v.nspans, s));
    // boundary rows <= nspans (each crosses at least one of the nspans - 1 span ends)
    const int64_t cap = v.nspans;
    PR_TRY(dalloc(&v.b_row, (size_t)cap, s));
    PR_TRY(dalloc(&v.b_s0, (size_t)cap, s));
    PR_TRY(dalloc(&v.b_s1, (size_t)cap, s));
    int64_t* cnt = nullptr;
    PR_TRY(dalloc(&cnt, 1, s));
    const int64_t span_e = ss * SE_STEP;
    PR_TRY((device_scan<int64_t>(ctx, v.nrows, BoundGet{v.row_ptr, span_e},
                                 BoundEmit{v.row_ptr, span_e, v.b_row, v.b_s0, v.b_s1, v.bin, v.bout}, cnt)));
    PR_TRY(read_count(ctx, cnt, &v.nbound));
    dfree(cnt, s);
    PR_TRY(dalloc(&v.part_in, (size_t)v.nspans, s));
    PR_TRY(dalloc(&v.part_out, (size_t)v.nspans, s));
    const int64_t nb = v.nbound > 0 ? v.nbound : 1;
    PR_TRY(dalloc(&v.bticket, (size_t)nb, s));
    PR_CUDA(cudaMemsetAsync(v.bticket, 0, sizeof(uint32_t) * (size_t)nb, s));
    return PR_OK;
}

void free_spans(View& v, cudaStream_t s) {
    dfree(v.bin, s);
    dfree(v.bout, s);
    dfree(v.b_row, s);
    dfree(v.b_s0, s);
    dfree(v.b_s1, s);
    dfree(v.part_in, s);
    dfree(v.part_out, s);
    dfree(v.bticket, s);
    v.nspans = v.nbound = 0;
}

// PR_MODE_PHASED (reading Q-B): K row-aligned phases.  Phase k owns the rows
// [b_k, b_{k+1}) of the view, b_k = the first row whose first edge e satisfies
// e * K >= k * E (rows in view order, E the view's edges), so no row is split
// between phases.  Each phase is its own edge-stream sub-view (a padded copy of
// its rows' edges with its own row-start bits, steps and spans: one span per
// resident warp); its gather emits into the parent's sums + b_k.
__global__ void k_phase_bounds(const int64_t* __restrict__ rp, int64_t nrows, int K, int64_t* __restrict__ rb) {
    const int k = threadIdx.x;
    if (k > K) return;
    const int64_t E = rp[nrows];
    if (k == 0) {
        rb[0] = 0;
        return;
    }
    if (k == K) {
        rb[K] = nrows;
        return;
    }
    int64_t lo = 0, hi = nrows;  // first row r with rp[r] * K >= k * E
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (rp[mid] * (int64_t)K >= (int64_t)k * E)
            hi = mid;
        else
            lo = mid + 1;
    }
    rb[k] = lo;
}
__global__ void k_rebase_rp(const int64_t* __restrict__ rp, int64_t r0, int64_t cnt, int64_t* __restrict__ out) {
    const int64_t base = rp[r0];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= cnt; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = rp[r0 + i] - base;
}

static void free_stream_subview(View& p, cudaStream_t s) {
    dfree(p.col, s);
    dfree(p.sflags, s);
    dfree(p.step_row, s);
    free_spans(p, s);
    p = View{};
}

int build_phase_view(View& v, Ctx& ctx, int K, int32_t pad_slot) {
    if (v.phv && v.phv_k == K) return PR_OK;
    free_phase_view(v, ctx.stream);
    cudaStream_t s = ctx.stream;
    int64_t* rb = nullptr;
    TmpGuard tg_(ctx.stream);
    tg_.track(rb);
    PR_TRY(dalloc(&rb, (size_t)K + 1, s));
    PR_LAUNCH(ctx, k_phase_bounds, 1, 128, 0, (const int64_t*)v.row_ptr, v.nrows, K, rb);
    PR_CUDA(cudaMemcpyAsync(v.phase_rb, rb, sizeof(int64_t) * (size_t)(K + 1), cudaMemcpyDeviceToHost, s));
    std::vector<int64_t> eb(K + 1);
    PR_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k <= K; ++k)  // first edge of each phase: row_ptr at the bounds
        PR_CUDA(cudaMemcpyAsync(&eb[k], v.row_ptr + v.phase_rb[k], sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PR_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k <= K; ++k) v.phase_eb[k] = eb[k];
    View* ph = new (std::nothrow) View[K];
    if (!ph) {
        set_error("build_phase_view: host allocation failed");
        return PR_ENOMEM;
    }
    v.phv = ph;
    v.phv_k = K;
    for (int k = 0; k < K; ++k) {
        View& p = ph[k];
        p.nrows = v.phase_rb[k + 1] - v.phase_rb[k];
        p.nedges = eb[k + 1] - eb[k];
        if (p.nrows == 0 || p.nedges == 0) continue;
        PR_TRY(dalloc(&p.row_ptr, (size_t)p.nrows + 1, s));
        p.owns_row_ptr = true;
        PR_LAUNCH(ctx, k_rebase_rp, grid_for(ctx, p.nrows + 1, 256), 256, 0, (const int64_t*)v.row_ptr,
                  v.phase_rb[k], p.nrows, p.row_ptr);
        PR_TRY(dalloc(&p.col, (size_t)stream_pad(p.nedges), s));
        PR_CUDA(cudaMemcpyAsync(p.col, v.col + eb[k], sizeof(int32_t) * (size_t)p.nedges, cudaMemcpyDeviceToDevice,
                                s));
        PR_TRY(build_view_stream(p, ctx, pad_slot, nullptr, nullptr));
        dfree(p.row_ptr, s);  // the stream engine does not read row_ptr
        p.owns_row_ptr = false;
    }
    v.phase_k = K;
    return PR_OK;
}

void free_phase_view(View& v, cudaStream_t s) {
    if (!v.phv) return;
    for (int k = 0; k < v.phv_k; ++k) free_stream_subview(v.phv[k], s);
    delete[] v.phv;
    v.phv = nullptr;
    v.phv_k = 0;
    v.phase_k = 0;
}

}  // namespace prgpu
