// csr_count.cu -- K-INGEST, counting form (the default for a single-rank
// create): the deduplicated in-CSR and out-degrees of a raw edge list
// (§5.2 "converted later to Compressed Sparse Row (CSR)
// format"; SPEC S:69-77 build_csr; readings Q-L, Q-V in DESIGN.md) without
// radix-sorting the whole edge list:
//
//   count    validate ids, drop self-loops; raw in- and out-degree of every
//            vertex by atomic adds (duplicates still counted)
//   offsets  exclusive scan of the in-degrees -> start of each row's bucket
//   place    the src of every edge into its dst's bucket (one atomic cursor
//            per row; the order inside a bucket is arbitrary)
//   sort     every bucket ascending; a duplicate becomes SENT and is taken off
//            its row's count and its src's out-degree.  By bucket length L:
//            a thread (L <= 16, sorting network in registers), a warp
//            (L <= 512, bitonic in registers), a CTA (L <= 16384, bitonic in
//            registers + shared memory), or the device-wide radix sort on
//            (bucket, src) keys (longer rows)
//   compact  stream compaction of the non-SENT entries -> col; row_ptr from an
//            exclusive scan of the deduplicated counts
//
// The result equals the sort-based path's (ingest.cu) bit for bit: rows by
// dst, sources ascending and unique within a row.  Every order-dependent step
// (the placement order inside a bucket, the order of the row lists) is undone
// by the per-row sort, so the CSR is deterministic although the atomics are not.
#include <stdlib.h>

#include <algorithm>

#include "internal.h"
#include "primitives.cuh"

namespace prgpu {
namespace {

constexpr int32_t SENT = INT32_MAX;  // never a vertex id (n < INT32_MAX on this path)
constexpr int CN_NT = 256;
constexpr int CN_U = 4;              // edges per thread per iteration (atomics in flight)
constexpr int CN_THREAD_MAX = 16;
constexpr int CN_WARP_MAX = 512;
constexpr int CN_CTA8_MAX = 4096;    // 8 warps x 512
constexpr int CN_CTA32_MAX = 16384;  // 32 warps x 512

// count: raw in-degree (by atomic adds on indeg) and out-degree of every
// vertex over the valid non-self-loop edges; any id outside [0, n) sets *err.
__global__ void __launch_bounds__(CN_NT) k_cn_count(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                                    int64_t m, int64_t n, uint32_t* __restrict__ indeg,
                                                    int32_t* __restrict__ outdeg, int* __restrict__ err) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    bool bad_any = false;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < m; i0 += CN_U * T) {
        int32_t s[CN_U], t[CN_U];
#pragma unroll
        for (int u = 0; u < CN_U; ++u) {
            const int64_t i = i0 + u * T;
            s[u] = i < m ? __ldcs(src + i) : 0;
            t[u] = i < m ? __ldcs(dst + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < CN_U; ++u) {
            if (i0 + u * T < m) {
                const bool bad = s[u] < 0 || (int64_t)s[u] >= n || t[u] < 0 || (int64_t)t[u] >= n;
                bad_any |= bad;
                if (!bad && s[u] != t[u]) {
                    atomicAdd(indeg + t[u], 1u);
                    atomicAdd(outdeg + s[u], 1);
                }
            }
        }
    }
    if (__any_sync(0xffffffffu, bad_any) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
}

// place: tmp[cur[dst]++] = src for every valid non-self-loop edge (invalid
// ids are skipped here; the create fails on *err afterwards).
__global__ void __launch_bounds__(CN_NT) k_cn_place(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                                    int64_t m, int64_t n, uint32_t* __restrict__ cur,
                                                    int32_t* __restrict__ tmp) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < m; i0 += CN_U * T) {
        int32_t s[CN_U], t[CN_U];
        uint32_t p[CN_U];
#pragma unroll
        for (int u = 0; u < CN_U; ++u) {
            const int64_t i = i0 + u * T;
            s[u] = i < m ? __ldcs(src + i) : 0;
            t[u] = i < m ? __ldcs(dst + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < CN_U; ++u) {
            const bool ok = i0 + u * T < m && s[u] >= 0 && (int64_t)s[u] < n && t[u] >= 0 && (int64_t)t[u] < n &&
                            s[u] != t[u];
            p[u] = ok ? atomicAdd(cur + t[u], 1u) : 0xffffffffu;
        }
#pragma unroll
        for (int u = 0; u < CN_U; ++u)
            if (p[u] != 0xffffffffu) tmp[p[u]] = s[u];
    }
}

// ---- sorting networks ------------------------------------------------------
// Bitonic network, ascending overall: in the merge of size k the pair
// (i, i ^ d), i < i ^ d, is put in ascending order iff (i & k) == 0.

// one thread, N registers
template <int N>
__device__ __forceinline__ void thread_bitonic(int32_t (&a)[N]) {
#pragma unroll
    for (int k = 2; k <= N; k *= 2) {
#pragma unroll
        for (int d = k / 2; d > 0; d /= 2) {
#pragma unroll
            for (int i = 0; i < N; ++i) {
                const int p = i ^ d;
                if (p > i) {
                    const int32_t lo = min(a[i], a[p]), hi = max(a[i], a[p]);
                    const bool asc = (i & k) == 0;
                    a[i] = asc ? lo : hi;
                    a[p] = asc ? hi : lo;
                }
            }
        }
    }
}

// A warp holds a chunk of 32*K elements, element j of lane l at index
// i = base + 32*j + l (base: the chunk's first index in the whole sequence,
// which fixes the directions).  One stage of distance D of the merge of size k:
// D < 32 across lanes (shuffles), D >= 32 inside each lane (registers).
template <int K, int D>
__device__ __forceinline__ void bstage(int32_t (&a)[K], int lane, uint32_t base, uint32_t k) {
    if constexpr (D >= 32) {
        constexpr int DJ = D / 32;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            if ((j & DJ) == 0) {
                const int p = j | DJ;
                const bool asc = ((base + (uint32_t)(32 * j + lane)) & k) == 0;
                const int32_t lo = min(a[j], a[p]), hi = max(a[j], a[p]);
                a[j] = asc ? lo : hi;
                a[p] = asc ? hi : lo;
            }
        }
    } else {
        const bool lower = (lane & D) == 0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int32_t b = __shfl_xor_sync(0xffffffffu, a[j], D);
            const bool asc = ((base + (uint32_t)(32 * j + lane)) & k) == 0;
            a[j] = (lower == asc) ? min(a[j], b) : max(a[j], b);
        }
    }
}

// stages D, D/2, ..., 1 of the merge of size k
template <int K, int D>
struct BMerge {
    static __device__ __forceinline__ void run(int32_t (&a)[K], int lane, uint32_t base, uint32_t k) {
        bstage<K, D>(a, lane, base, k);
        BMerge<K, D / 2>::run(a, lane, base, k);
    }
};
template <int K>
struct BMerge<K, 0> {
    static __device__ __forceinline__ void run(int32_t (&)[K], int, uint32_t, uint32_t) {}
};

// merges of size 2, 4, ..., KK
template <int K, int KK>
struct BSort {
    static __device__ __forceinline__ void run(int32_t (&a)[K], int lane, uint32_t base) {
        BSort<K, KK / 2>::run(a, lane, base);
        BMerge<K, KK / 2>::run(a, lane, base, (uint32_t)KK);
    }
};
template <int K>
struct BSort<K, 1> {
    static __device__ __forceinline__ void run(int32_t (&)[K], int, uint32_t) {}
};

// ---- per-row sort + duplicate marking --------------------------------------
// After the sort, entry i of the row is kept iff it differs from entry i - 1;
// a duplicate is written as SENT, and removed from its src's out-degree.

template <int N>
__device__ __forceinline__ int sort_row_thread(int32_t* row, int L, int32_t* outdeg) {
    int32_t a[N];
#pragma unroll
    for (int j = 0; j < N; ++j) a[j] = j < L ? row[j] : SENT;
    thread_bitonic<N>(a);
    int dups = 0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        if (j < L) {
            const bool dup = j > 0 && a[j] == a[j - 1];
            row[j] = dup ? SENT : a[j];
            if (dup) {
                atomicSub(outdeg + a[j], 1);
                ++dups;
            }
        }
    }
    return dups;
}

template <int K>
__device__ __forceinline__ int sort_row_warp(int32_t* row, int L, int lane, int32_t* outdeg) {
    int32_t a[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int i = 32 * j + lane;
        a[j] = i < L ? row[i] : SENT;
    }
    BSort<K, 32 * K>::run(a, lane, 0u);
    int dups = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        int32_t pv = __shfl_up_sync(0xffffffffu, a[j], 1);
        const int32_t q = j > 0 ? __shfl_sync(0xffffffffu, a[j > 0 ? j - 1 : 0], 31) : SENT;
        if (lane == 0) pv = q;
        const int i = 32 * j + lane;
        if (i < L) {
            const bool dup = a[j] == pv;
            row[i] = dup ? SENT : a[j];
            if (dup) {
                atomicSub(outdeg + a[j], 1);
                ++dups;
            }
        }
    }
    return warp_sum(dups);
}

struct CnLists {
    int32_t* w;     // rows with CN_THREAD_MAX < L <= CN_WARP_MAX
    int32_t* c8;    // CN_WARP_MAX < L <= CN_CTA8_MAX
    int32_t* c32;   // CN_CTA8_MAX < L <= CN_CTA32_MAX
    int32_t* h;     // L > CN_CTA32_MAX
    uint32_t* cnt;  // [4] list lengths
};

// Rows of L <= CN_THREAD_MAX sorted by one thread each; every longer row is
// appended to the list of its class (one atomic per warp and class).
__global__ void __launch_bounds__(CN_NT) k_cn_small(const int64_t* __restrict__ off, uint32_t* __restrict__ indeg,
                                                    int64_t n, int32_t* __restrict__ tmp, int32_t* __restrict__ outdeg,
                                                    CnLists ls) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = lanemask_lt();
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t wb = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); wb < n; wb += T) {
        const int64_t v = wb + lane;
        const uint32_t L = v < n ? indeg[v] : 0u;
        int cls = 0;
        if (L > CN_CTA32_MAX) cls = 5;
        else if (L > CN_CTA8_MAX) cls = 4;
        else if (L > CN_WARP_MAX) cls = 3;
        else if (L > CN_THREAD_MAX) cls = 2;
        else if (L > 1) cls = 1;
        if (cls == 1) {
            int32_t* row = tmp + off[v];
            int dups;
            if (L <= 4) dups = sort_row_thread<4>(row, (int)L, outdeg);
            else if (L <= 8) dups = sort_row_thread<8>(row, (int)L, outdeg);
            else dups = sort_row_thread<16>(row, (int)L, outdeg);
            if (dups) indeg[v] = L - (uint32_t)dups;
        }
#pragma unroll
        for (int c = 2; c <= 5; ++c) {
            const uint32_t bal = __ballot_sync(0xffffffffu, cls == c);
            if (bal) {
                const int leader = __ffs(bal) - 1;
                uint32_t b0 = 0;
                if (lane == leader) b0 = atomicAdd(ls.cnt + (c - 2), (uint32_t)__popc(bal));
                b0 = __shfl_sync(0xffffffffu, b0, leader);
                int32_t* lst = c == 2 ? ls.w : c == 3 ? ls.c8 : c == 4 ? ls.c32 : ls.h;
                if (cls == c) lst[b0 + __popc(bal & lt)] = (int32_t)v;
            }
        }
    }
}

// One warp per listed row of CN_THREAD_MAX < L <= CN_WARP_MAX.
__global__ void __launch_bounds__(CN_NT) k_cn_warp(const int32_t* __restrict__ list, const uint32_t* __restrict__ cnt,
                                                   const int64_t* __restrict__ off, uint32_t* __restrict__ indeg,
                                                   int32_t* __restrict__ tmp, int32_t* __restrict__ outdeg) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t N = *cnt;
    for (int64_t x = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); x < N; x += nw) {
        const int32_t v = list[x];
        const int L = (int)indeg[v];
        int32_t* row = tmp + off[v];
        int dups;
        if (L <= 32) dups = sort_row_warp<1>(row, L, lane, outdeg);
        else if (L <= 64) dups = sort_row_warp<2>(row, L, lane, outdeg);
        else if (L <= 128) dups = sort_row_warp<4>(row, L, lane, outdeg);
        else if (L <= 256) dups = sort_row_warp<8>(row, L, lane, outdeg);
        else dups = sort_row_warp<16>(row, L, lane, outdeg);
        if (lane == 0 && dups) indeg[v] = (uint32_t)(L - dups);
    }
}

// One CTA of NW warps per listed row of L <= NW * 512: the row padded with
// SENT to P = 2^p >= L entries; warp w holds entries [512w, 512w + 512) in
// registers (16 per lane) and sorts them; the merges of size k > 512 run
// their stages of distance >= 512 in shared memory and the rest in registers.
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_cn_cta(const int32_t* __restrict__ list, const uint32_t* __restrict__ cnt,
                                                    const int64_t* __restrict__ off, uint32_t* __restrict__ indeg,
                                                    int32_t* __restrict__ tmp, int32_t* __restrict__ outdeg) {
    extern __shared__ int32_t cn_sh[];
    int32_t* s = cn_sh;                 // [NW * 512]
    int32_t* tail = cn_sh + NW * 512;   // [NW] last entry of each warp's chunk
    __shared__ int sdup;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t N = *cnt;
    const uint32_t base = (uint32_t)w * 512u;
    for (int64_t x = blockIdx.x; x < N; x += gridDim.x) {
        const int32_t v = list[x];
        const int L = (int)indeg[v];
        int32_t* row = tmp + off[v];
        uint32_t P = 512;
        while ((int)P < L) P <<= 1;
        const bool act = base < P;
        int32_t a[16];
        if (act) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t i = base + 32u * j + lane;
                a[j] = (int)i < L ? row[i] : SENT;
            }
            BSort<16, 512>::run(a, lane, base);
        }
        for (uint32_t k = 1024; k <= P; k <<= 1) {
            if (act) {
#pragma unroll
                for (int j = 0; j < 16; ++j) s[base + 32u * j + lane] = a[j];
            }
            __syncthreads();
            for (uint32_t d = k >> 1; d >= 512; d >>= 1) {
                for (uint32_t t = threadIdx.x; t < (P >> 1); t += NW * 32) {
                    const uint32_t i = 2 * t - (t & (d - 1));
                    const uint32_t p = i + d;
                    const int32_t x0 = s[i], x1 = s[p];
                    const bool asc = (i & k) == 0;
                    const int32_t lo = min(x0, x1), hi = max(x0, x1);
                    s[i] = asc ? lo : hi;
                    s[p] = asc ? hi : lo;
                }
                __syncthreads();
            }
            if (act) {
#pragma unroll
                for (int j = 0; j < 16; ++j) a[j] = s[base + 32u * j + lane];
                BMerge<16, 256>::run(a, lane, base, k);
            }
        }
        if (act && lane == 31) tail[w] = a[15];
        if (threadIdx.x == 0) sdup = 0;
        __syncthreads();
        int dups = 0;
        if (act) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                int32_t pv = __shfl_up_sync(0xffffffffu, a[j], 1);
                const int32_t q = j > 0 ? __shfl_sync(0xffffffffu, a[j > 0 ? j - 1 : 0], 31) : (w > 0 ? tail[w - 1] : SENT);
                if (lane == 0) pv = q;
                const uint32_t i = base + 32u * j + lane;
                if ((int)i < L) {
                    const bool dup = a[j] == pv;
                    row[i] = dup ? SENT : a[j];
                    if (dup) {
                        atomicSub(outdeg + a[j], 1);
                        ++dups;
                    }
                }
            }
            dups = warp_sum(dups);
            if (lane == 0 && dups) atomicAdd(&sdup, dups);
        }
        __syncthreads();
        if (threadIdx.x == 0 && sdup) indeg[v] = (uint32_t)(L - sdup);
        __syncthreads();  // s, tail and sdup are reused by the next row
    }
}

// Rows longer than CN_CTA32_MAX: keys (h << b | src) of the H listed rows,
// radix-sorted device-wide, then written back with duplicates as SENT.
__global__ void k_cn_hub_keys(const int32_t* __restrict__ list, const int64_t* __restrict__ hb,
                              const int64_t* __restrict__ off, const int32_t* __restrict__ tmp, int b,
                              uint64_t* __restrict__ keys) {
    const int64_t h = blockIdx.x;
    const int32_t v = list[h];
    const int64_t L = hb[h + 1] - hb[h];
    const int32_t* row = tmp + off[v];
    uint64_t* out = keys + hb[h];
    for (int64_t i = threadIdx.x; i < L; i += blockDim.x) out[i] = ((uint64_t)h << b) | (uint32_t)row[i];
}

__global__ void k_cn_hub_back(const uint64_t* __restrict__ sorted, int64_t EH, int b, const int32_t* __restrict__ list,
                              const int64_t* __restrict__ hb, const int64_t* __restrict__ off,
                              uint32_t* __restrict__ indeg, int32_t* __restrict__ tmp, int32_t* __restrict__ outdeg) {
    const uint64_t smask = (1ull << b) - 1ull;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < EH; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = sorted[i];
        const int64_t h = (int64_t)(key >> b);
        const int32_t s = (int32_t)(key & smask);
        const int32_t v = list[h];
        const int64_t j = i - hb[h];
        const bool dup = j > 0 && sorted[i - 1] == key;
        tmp[off[v] + j] = dup ? SENT : s;
        if (dup) {
            atomicSub(outdeg + s, 1);
            atomicSub(indeg + v, 1u);
        }
    }
}

struct CntGet {
    const uint32_t* c;
    __device__ int64_t operator()(int64_t v) const { return (int64_t)c[v]; }
};
// off[v] = exclusive prefix (and off[n] = total); optionally a 32-bit cursor copy
struct OffEmit {
    int64_t* off;
    uint32_t* cur;
    int64_t n;
    __device__ void operator()(int64_t v, int64_t pos, int64_t f) const {
        off[v] = pos;
        if (cur) cur[v] = (uint32_t)pos;
        if (v == n - 1) off[n] = pos + f;
    }
};
struct HubLenGet {
    const int32_t* list;
    const uint32_t* indeg;
    __device__ int64_t operator()(int64_t h) const { return (int64_t)indeg[list[h]]; }
};
struct KeepGet {
    const int32_t* t;
    __device__ int64_t operator()(int64_t i) const { return t[i] != SENT ? 1 : 0; }
};
struct KeepEmit {
    const int32_t* t;
    int32_t* col;
    __device__ void operator()(int64_t i, int64_t pos, int64_t f) const {
        if (f) col[pos] = t[i];
    }
};

unsigned cn_grid(const Ctx& ctx, int64_t work, int nt, int per_sm) {
    int64_t g = (work + nt - 1) / nt;
    const int64_t cap = (int64_t)ctx.num_sms * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

}  // namespace

bool ingest_count_applies(int64_t n, int64_t m) {
    const char* e = getenv("PRGPU_INGEST");
    if (e && e[0] == 'r') return false;  // "radix": the sort-based path (A/B)
    return n > 1 && n < (int64_t)INT32_MAX && m > 0 && m <= (int64_t)UINT32_MAX;
}

int ingest_count(pr_graph* g, const int32_t* src, const int32_t* dst, Ctx& ctx) {
    const int64_t n = g->n, m = g->m_raw;
    cudaStream_t s = ctx.stream;
    uint32_t* indeg = nullptr;
    uint32_t* cur = nullptr;
    int64_t* off = nullptr;
    int32_t* tmp = nullptr;
    int64_t* scratch = nullptr;  // [0] kept raw edges, [1] error flag, [2] E, [3] hub edges
    uint32_t* lcnt = nullptr;
    int32_t* lists = nullptr;
    int64_t* hb = nullptr;
    uint64_t* keys = nullptr;
    uint64_t* keys_alt = nullptr;
    TmpGuard tg_(s);
    tg_.track(indeg);
    tg_.track(cur);
    tg_.track(off);
    tg_.track(tmp);
    tg_.track(scratch);
    tg_.track(lcnt);
    tg_.track(lists);
    tg_.track(hb);
    tg_.track(keys);
    tg_.track(keys_alt);

    PR_TRY(dalloc(&scratch, 4, s));
    PR_CUDA(cudaMemsetAsync(scratch, 0, 4 * sizeof(int64_t), s));
    PR_TRY(dalloc(&indeg, (size_t)n, s));
    PR_CUDA(cudaMemsetAsync(indeg, 0, sizeof(uint32_t) * (size_t)n, s));
    PR_TRY(dalloc(&g->outdeg, (size_t)n, s));
    PR_CUDA(cudaMemsetAsync(g->outdeg, 0, sizeof(int32_t) * (size_t)n, s));
    PR_TRY(dalloc(&g->row_ptr, (size_t)n + 1, s));

    PR_LAUNCH(ctx, k_cn_count, cn_grid(ctx, (m + CN_U - 1) / CN_U, CN_NT, 16), CN_NT, 0, src, dst, m, n, indeg,
              g->outdeg, (int*)(scratch + 1));
    PR_TRY(dalloc(&off, (size_t)n + 1, s));
    PR_TRY(dalloc(&cur, (size_t)n, s));
    PR_TRY((device_scan<int64_t>(ctx, n, CntGet{indeg}, OffEmit{off, cur, n}, scratch)));
    PR_TRY(dalloc(&tmp, (size_t)m, s));
    PR_LAUNCH(ctx, k_cn_place, cn_grid(ctx, (m + CN_U - 1) / CN_U, CN_NT, 16), CN_NT, 0, src, dst, m, n, cur, tmp);
    dfree(cur, s);

    // row classes (list capacities: a row of class c has at least lo_c raw edges)
    const int64_t cap_w = std::min<int64_t>(n, m / (CN_THREAD_MAX + 1) + 1);
    const int64_t cap_c8 = std::min<int64_t>(n, m / (CN_WARP_MAX + 1) + 1);
    const int64_t cap_c32 = std::min<int64_t>(n, m / (CN_CTA8_MAX + 1) + 1);
    const int64_t cap_h = std::min<int64_t>(n, m / (CN_CTA32_MAX + 1) + 1);
    PR_TRY(dalloc(&lists, (size_t)(cap_w + cap_c8 + cap_c32 + cap_h), s));
    PR_TRY(dalloc(&lcnt, 4, s));
    PR_CUDA(cudaMemsetAsync(lcnt, 0, 4 * sizeof(uint32_t), s));
    CnLists ls{lists, lists + cap_w, lists + cap_w + cap_c8, lists + cap_w + cap_c8 + cap_c32, lcnt};
    PR_LAUNCH(ctx, k_cn_small, cn_grid(ctx, n, CN_NT, 16), CN_NT, 0, (const int64_t*)off, indeg, n, tmp, g->outdeg, ls);
    PR_LAUNCH(ctx, k_cn_warp, (unsigned)ctx.num_sms * 8, CN_NT, 0, (const int32_t*)ls.w, (const uint32_t*)lcnt,
              (const int64_t*)off, indeg, tmp, g->outdeg);
    {
        const size_t sm8 = (8 * 512 + 8) * sizeof(int32_t);
        PR_LAUNCH(ctx, k_cn_cta<8>, (unsigned)ctx.num_sms * 8, 256, sm8, (const int32_t*)ls.c8,
                  (const uint32_t*)(lcnt + 1), (const int64_t*)off, indeg, tmp, g->outdeg);
        const size_t sm32 = (32 * 512 + 32) * sizeof(int32_t);
        PR_CUDA(cudaFuncSetAttribute(k_cn_cta<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm32));
        PR_LAUNCH(ctx, k_cn_cta<32>, (unsigned)ctx.num_sms * 2, 1024, sm32, (const int32_t*)ls.c32,
                  (const uint32_t*)(lcnt + 2), (const int64_t*)off, indeg, tmp, g->outdeg);
    }
    uint32_t hc[4];
    int64_t hs[2];
    PR_CUDA(cudaMemcpyAsync(hc, lcnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
    PR_CUDA(cudaMemcpyAsync(hs, scratch, sizeof(hs), cudaMemcpyDeviceToHost, s));
    PR_CUDA(cudaStreamSynchronize(s));
    if (hs[1] != 0) {
        set_error("pr_graph_create: vertex id outside [0, n)");
        return PR_EINVAL;
    }
    const int64_t mk = hs[0];
    const int64_t H = hc[3];
    if (H > 0) {  // the longest rows: device-wide radix sort of (row rank, src) keys
        const int b = bits_for((uint64_t)(n - 1));
        PR_TRY(dalloc(&hb, (size_t)H + 1, s));
        PR_TRY((device_scan<int64_t>(ctx, H, HubLenGet{ls.h, indeg}, OffEmit{hb, nullptr, H}, scratch + 3)));
        PR_TRY(read_count(ctx, scratch + 3, &hs[0]));
        const int64_t EH = hs[0];
        PR_TRY(dalloc(&keys, (size_t)EH, s));
        PR_TRY(dalloc(&keys_alt, (size_t)EH, s));
        PR_LAUNCH(ctx, k_cn_hub_keys, (unsigned)H, 1024, 0, (const int32_t*)ls.h, (const int64_t*)hb,
                  (const int64_t*)off, (const int32_t*)tmp, b, keys);
        bool alt = false;
        PR_TRY((radix_sort<uint64_t, false>(ctx, keys, keys_alt, nullptr, nullptr, EH, 0,
                                            b + bits_for((uint64_t)(H - 1)), &alt)));
        PR_LAUNCH(ctx, k_cn_hub_back, cn_grid(ctx, EH, 256, 16), 256, 0, (const uint64_t*)(alt ? keys_alt : keys), EH,
                  b, (const int32_t*)ls.h, (const int64_t*)hb, (const int64_t*)off, indeg, tmp, g->outdeg);
        dfree(keys, s);
        dfree(keys_alt, s);
        dfree(hb, s);
    }
    // compact: col = the non-SENT entries in order; row_ptr from the deduplicated counts
    PR_TRY(dalloc(&g->col, (size_t)(mk > 0 ? mk : 1), s));
    PR_TRY((device_scan<int64_t>(ctx, mk, KeepGet{tmp}, KeepEmit{tmp, g->col}, scratch + 2)));
    PR_TRY((device_scan<int64_t>(ctx, n, CntGet{indeg}, OffEmit{g->row_ptr, nullptr, n}, (int64_t*)nullptr)));
    PR_TRY(read_count(ctx, scratch + 2, &g->E));
    return PR_OK;
}

}  // namespace prgpu
