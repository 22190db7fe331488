// primitives.cuh -- hand-written device-wide scan, stream compaction and LSD
// radix sort used by graph ingest and preprocessing (no CUB / Thrust).
//
// Design: "reduce-then-scan" with a fixed number G of CTAs, each owning one
// contiguous range of the input, so every result is a deterministic function
// of the input (no decoupled look-back, no atomics on the data path).
#pragma once
#include "common.cuh"

namespace prgpu {

constexpr int SCAN_NT = 256;
constexpr int SCAN_IPT = 8;
constexpr int SCAN_TILE = SCAN_NT * SCAN_IPT;

// Block-wide exclusive sum over one value per thread; returns the exclusive
// prefix and writes the block total to *total (all threads see it).
template <class T>
__device__ __forceinline__ T block_exclusive_sum(T v, T* total, T* smem_warp /*[33]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nwarps ? smem_warp[lane] : T(0);
        T ws = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, ws, o);
            if (lane >= o) ws += y;
        }
        if (lane < nwarps) smem_warp[lane] = ws - w;  // exclusive warp offsets
        if (lane == nwarps - 1) smem_warp[32] = ws;   // block total
    }
    __syncthreads();
    T res = smem_warp[warp] + x - v;
    *total = smem_warp[32];
    __syncthreads();
    return res;
}

template <class T>
__device__ __forceinline__ T block_sum(T v, T* smem_warp) {
    T tot;
    block_exclusive_sum(v, &tot, smem_warp);
    return tot;
}

template <class T, class Get>
__global__ void __launch_bounds__(SCAN_NT) k_scan_reduce(Get get, int64_t n, int64_t per_cta, T* partial) {
    __shared__ T sw[33];
    const int64_t b = (int64_t)blockIdx.x * per_cta;
    const int64_t e = min(n, b + per_cta);
    T s = T(0);
    for (int64_t i = b + threadIdx.x; i < e; i += SCAN_NT) s += get(i);
    T tot = block_sum(s, sw);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// Single CTA: in-place exclusive scan of partial[0..G); *total = sum.
template <class T>
__global__ void __launch_bounds__(1024) k_scan_partials(T* partial, int64_t G, T* total) {
    __shared__ T sw[33];
    T carry = T(0);
    constexpr int IPT = sizeof(T) == 4 ? 32 : 16;  // few block scans: this kernel is latency-bound
    for (int64_t base = 0; base < G; base += 1024 * IPT) {
        T v[IPT];
        T ts = T(0);
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            int64_t i = base + (int64_t)threadIdx.x * IPT + j;
            v[j] = i < G ? partial[i] : T(0);
            ts += v[j];
        }
        T tot;
        T p = carry + block_exclusive_sum(ts, &tot, sw);
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            int64_t i = base + (int64_t)threadIdx.x * IPT + j;
            if (i < G) partial[i] = p;
            p += v[j];
        }
        carry += tot;
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

template <class T, class Get, class Emit>
__global__ void __launch_bounds__(SCAN_NT) k_scan_down(Get get, Emit emit, int64_t n, int64_t per_cta,
                                                       const T* partial) {
    __shared__ T sw[33];
    const int64_t b = (int64_t)blockIdx.x * per_cta;
    const int64_t e = min(n, b + per_cta);
    T running = partial[blockIdx.x];
    for (int64_t tb = b; tb < e; tb += SCAN_TILE) {
        T v[SCAN_IPT];
        T ts = T(0);
#pragma unroll
        for (int j = 0; j < SCAN_IPT; ++j) {
            int64_t i = tb + (int64_t)threadIdx.x * SCAN_IPT + j;
            v[j] = i < e ? get(i) : T(0);
            ts += v[j];
        }
        T tile_total;
        T p = running + block_exclusive_sum(ts, &tile_total, sw);
#pragma unroll
        for (int j = 0; j < SCAN_IPT; ++j) {
            int64_t i = tb + (int64_t)threadIdx.x * SCAN_IPT + j;
            if (i < e) emit(i, p, v[j]);
            p += v[j];
        }
        running += tile_total;
    }
}

inline int64_t scan_grid(const Ctx& ctx, int64_t n, int64_t tile) {
    int64_t g = (n + tile - 1) / tile;
    int64_t cap = (int64_t)ctx.num_sms * 8;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return g;
}

// Exclusive scan: emit(i, exclusive_prefix, get(i)) for every i in [0, n);
// *total_dev (device, nullable) = sum of all get(i).
template <class T, class Get, class Emit>
int device_scan(Ctx& ctx, int64_t n, Get get, Emit emit, T* total_dev) {
    if (n <= 0) {
        if (total_dev) PR_CUDA(cudaMemsetAsync(total_dev, 0, sizeof(T), ctx.stream));
        return PR_OK;
    }
    int64_t G = scan_grid(ctx, n, SCAN_TILE);
    int64_t per = (n + G - 1) / G;
    T* partial = nullptr;
    PR_TRY(dalloc(&partial, (size_t)G, ctx.stream));
    PR_LAUNCH(ctx, (k_scan_reduce<T, Get>), (unsigned)G, SCAN_NT, 0, get, n, per, partial);
    PR_LAUNCH(ctx, (k_scan_partials<T>), 1, 1024, 0, partial, G, total_dev);
    PR_LAUNCH(ctx, (k_scan_down<T, Get, Emit>), (unsigned)G, SCAN_NT, 0, get, emit, n, per,
              (const T*)partial);
    dfree(partial, ctx.stream);
    return PR_OK;
}

// ------------------------------------------------------------ radix sort --
// LSD radix sort, 8-bit digits, "reduce-then-scan" per pass with a fixed
// number G of CTAs, each owning a contiguous chunk of the array (stable and
// deterministic, no look-back).  Tiles of RS_TILE = 3072 keys (256 threads x
// 12) per CTA step at 3 CTAs/SM keep the block barriers per key low and each
// digit's run in a tile ~12 keys long, so the write-out is coalesced
// (R-MAT-24 create: 15.7 ms against 16.1 with 512 x 8 at 2 CTAs/SM, 17.0 with
// 256 x 8 at 4, 16.7 with 384 x 8 at 2).
#ifndef PRGPU_RS_NT
#define PRGPU_RS_NT 256
#endif
#ifndef PRGPU_RS_ROUNDS
#define PRGPU_RS_ROUNDS 12
#endif
#ifndef PRGPU_RS_MINB
#define PRGPU_RS_MINB 3
#endif
constexpr int RS_NT = PRGPU_RS_NT;
constexpr int RS_WARPS = RS_NT / 32;
constexpr int RS_ROUNDS = PRGPU_RS_ROUNDS;         // keys per thread per tile
constexpr int RS_TILE = RS_NT * RS_ROUNDS;
constexpr int RS_BITS = 8;
constexpr int RS_BINS = 1 << RS_BITS;
static_assert(RS_NT >= RS_BINS, "one thread per digit in the tile scan");

// Pack fused into the first radix pass (ingest, single rank): the pass reads
// the raw edge arrays and forms key = dst << b | src itself (self-loops and
// invalid ids -> sentinel, which sorts last; the histogram pass flags invalid
// ids in *err), so the packed key array is never written and read back.
struct RsPack {
    const int32_t* src = nullptr;  // null: the pass reads keys
    const int32_t* dst = nullptr;
    int64_t n = 0;                 // vertices
    int b = 0;
    uint64_t sentinel = 0;
    int* err = nullptr;
};
__device__ __forceinline__ uint64_t rs_pack_key(const RsPack& pk, int32_t s, int32_t t, bool* bad) {
    *bad = s < 0 || (int64_t)s >= pk.n || t < 0 || (int64_t)t >= pk.n;
    return (*bad || s == t) ? pk.sentinel : (((uint64_t)(uint32_t)t << pk.b) | (uint32_t)s);
}

template <class K>
__global__ void __launch_bounds__(RS_NT) k_rs_hist(const K* __restrict__ keys, int64_t n, int64_t per_cta,
                                                   int shift, uint32_t dmask, uint32_t* __restrict__ hist,
                                                   int64_t G, RsPack pk) {
    __shared__ uint32_t cnt[RS_WARPS][RS_BINS];
    for (int i = threadIdx.x; i < RS_WARPS * RS_BINS; i += RS_NT) (&cnt[0][0])[i] = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    const int64_t b = (int64_t)blockIdx.x * per_cta;
    const int64_t e = min(n, b + per_cta);
    if (pk.src) {
        bool any_bad = false;
        for (int64_t i = b + threadIdx.x; i < e; i += RS_NT) {
            bool bad;
            const uint64_t key = rs_pack_key(pk, __ldg(pk.src + i), __ldg(pk.dst + i), &bad);
            any_bad |= bad;
            atomicAdd(&cnt[warp][(uint32_t)(key >> shift) & dmask], 1u);
        }
        if (any_bad) atomicOr(pk.err, 1);
    } else {
        for (int64_t i = b + threadIdx.x; i < e; i += RS_NT) {
            uint32_t d = (uint32_t)(keys[i] >> shift) & dmask;
            atomicAdd(&cnt[warp][d], 1u);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < RS_BINS; d += RS_NT) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) s += cnt[w][d];
        hist[(int64_t)d * G + blockIdx.x] = s;
    }
}

// Offsets of a radix pass without a single-CTA scan of all 256 x G counts:
// CTA d scans digit d's G per-CTA counts in place (exclusive) and writes the
// digit total; k_rs_dbase scans the 256 totals; the scatter adds the digit
// base (75K counts on R-MAT-24: 69 us in one CTA, ~5 us this way).
static __global__ void __launch_bounds__(256) k_rs_digit_scan(uint32_t* __restrict__ hist, int64_t G,
                                                       uint32_t* __restrict__ dtot) {
    __shared__ uint32_t sw[33];
    uint32_t* row = hist + (int64_t)blockIdx.x * G;
    uint32_t carry = 0;
    for (int64_t b0 = 0; b0 < G; b0 += 256) {
        const int64_t i = b0 + threadIdx.x;
        const uint32_t v = i < G ? row[i] : 0u;
        uint32_t tot;
        const uint32_t ex = block_exclusive_sum(v, &tot, sw);
        if (i < G) row[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) dtot[blockIdx.x] = carry;
}
static __global__ void __launch_bounds__(256) k_rs_dbase(const uint32_t* __restrict__ dtot, uint32_t* __restrict__ dbase) {
    __shared__ uint32_t sw[33];
    uint32_t tot;
    const uint32_t v = threadIdx.x < RS_BINS ? dtot[threadIdx.x] : 0u;
    const uint32_t ex = block_exclusive_sum(v, &tot, sw);
    if (threadIdx.x < RS_BINS) dbase[threadIdx.x] = ex;
}

// Lanes of the warp whose digit equals this lane's (bits 0..RS_BITS-1 of d):
// one ballot per bit, each folded in with one LOP3 (peers &= ~(ballot ^ own
// bit broadcast)) -- written in PTX so that ptxas emits 4 instructions per bit
// (the C++ form compiled to a second, negated ballot per bit).
__device__ __forceinline__ uint32_t rs_match_digit(uint32_t d, uint32_t peers) {
#pragma unroll
    for (int bit = 0; bit < RS_BITS; ++bit) {
        uint32_t bb, m;
        asm("{\n\t.reg .pred p;\n\t"
            "and.b32 %1, %2, %3;\n\t"
            "setp.ne.u32 p, %1, 0;\n\t"
            "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
            "selp.b32 %1, -1, 0, p;\n\t}"
            : "=r"(bb), "=&r"(m)
            : "r"(d), "r"(1u << bit));
        peers &= ~(bb ^ m);
    }
    return peers;
}

template <class K, bool HAS_V>
struct RsSmem {
    uint32_t base[RS_BINS];      // global start of each digit for the next tile
    uint32_t adj[RS_BINS];       // global index of tile position i (digit d) = adj[d] + i
    uint32_t wc[RS_WARPS][RS_BINS + 1];
    uint32_t sw[33];
    alignas(16) K sk[RS_TILE];
    alignas(16) uint32_t sv[HAS_V ? RS_TILE : 4];
    // the NEXT tile, staged by one TMA bulk copy while this one is ranked
    alignas(16) K stk[RS_TILE];
    alignas(16) uint32_t stv[HAS_V ? RS_TILE : 4];
    alignas(8) uint64_t bar;
};

// Stable scatter of one 8-bit digit.  Per tile of RS_TILE keys: warp-level
// ranking (match_any), tile-local digit offsets, a local sort into shared
// memory, then a coalesced write-out (consecutive threads write consecutive
// addresses of one digit's run).
template <class K, bool HAS_V, bool PACK = false>
__global__ void __launch_bounds__(RS_NT, HAS_V ? 2 : PRGPU_RS_MINB) k_rs_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                      K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                      int64_t n, int64_t per_cta, int shift, uint32_t dmask,
                                                      const uint32_t* __restrict__ offs, int64_t G,
                                                      const uint32_t* __restrict__ dbase, RsPack pk) {
    extern __shared__ __align__(16) unsigned char rs_raw[];
    RsSmem<K, HAS_V>& sm = *reinterpret_cast<RsSmem<K, HAS_V>*>(rs_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = lanemask_lt();
    if (threadIdx.x < RS_BINS) sm.base[threadIdx.x] = offs[(int64_t)threadIdx.x * G + blockIdx.x] + dbase[threadIdx.x];
    const int64_t b = (int64_t)blockIdx.x * per_cta;
    const int64_t e = min(n, b + per_cta);
    // stage tile [tb, tb + tn) (16-byte rounded; allocations carry >= 64 B of slack)
    // pack form: src tile at stk (as int32), dst tile RS_TILE int32 further; the
    // last, partial tile of the array is read with plain loads instead (user
    // buffers carry no slack for a 16-byte rounded copy)
    int32_t* const ps = reinterpret_cast<int32_t*>(sm.stk);
    int32_t* const pd = ps + RS_TILE;
    static_assert(sizeof(K) != 8 || sizeof(K) * RS_TILE >= 2 * sizeof(int32_t) * RS_TILE, "pack staging fits the key tile");
    auto stage = [&](int64_t tb) {
        const int tn = (int)min((int64_t)RS_TILE, e - tb);
        if (PACK) {
            if (tn < RS_TILE) return;
            const uint32_t pb = (uint32_t)(RS_TILE * sizeof(int32_t));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&sm.bar)), "r"(2 * pb)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(ps)),
                "l"(pk.src + tb), "r"(pb), "r"(smem_addr(&sm.bar))
                : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(pd)),
                "l"(pk.dst + tb), "r"(pb), "r"(smem_addr(&sm.bar))
                : "memory");
            return;
        }
        const uint32_t kb = ((uint32_t)(tn * sizeof(K)) + 15u) & ~15u;
        const uint32_t vb = HAS_V ? (((uint32_t)(tn * 4) + 15u) & ~15u) : 0u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&sm.bar)), "r"(kb + vb)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_addr(sm.stk)),
            "l"(kin + tb), "r"(kb), "r"(smem_addr(&sm.bar))
            : "memory");
        if (HAS_V)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(sm.stv)),
                "l"(vin + tb), "r"(vb), "r"(smem_addr(&sm.bar))
                : "memory");
    };
    if (threadIdx.x == 0) {
        mbar_init(&sm.bar, 1);
        fence_mbar_init();
        if (b < e) stage(b);
    }
    for (int i = threadIdx.x; i < RS_WARPS * (RS_BINS + 1); i += RS_NT) (&sm.wc[0][0])[i] = 0;
    __syncthreads();
    // Barriers per tile: staging consumed / ranked / (scan) / offsets ready /
    // local sort done.  The write-out of tile t overlaps the next tile's
    // staging wait; the wc counters are cleared during the write-out.
    uint32_t phase = 0;
    for (int64_t tb = b; tb < e; tb += RS_TILE) {
        const int tn = (int)min((int64_t)RS_TILE, e - tb);
        K k[RS_ROUNDS];
        uint32_t v[RS_ROUNDS];
        uint32_t dg[RS_ROUNDS];
        uint32_t pos[RS_ROUNDS];
        if (PACK) {
            bool dummy;
            if (tn == RS_TILE) {
                mbar_wait(&sm.bar, phase);
                phase ^= 1u;
#pragma unroll
                for (int r = 0; r < RS_ROUNDS; ++r) {
                    const int li = warp * (32 * RS_ROUNDS) + r * 32 + lane;
                    k[r] = (K)rs_pack_key(pk, ps[li], pd[li], &dummy);
                }
            } else {
#pragma unroll
                for (int r = 0; r < RS_ROUNDS; ++r) {
                    const int li = warp * (32 * RS_ROUNDS) + r * 32 + lane;
                    k[r] = li < tn ? (K)rs_pack_key(pk, __ldg(pk.src + tb + li), __ldg(pk.dst + tb + li), &dummy) : K(0);
                }
            }
        } else {
            mbar_wait(&sm.bar, phase);
            phase ^= 1u;
#pragma unroll
            for (int r = 0; r < RS_ROUNDS; ++r) {
                const int li = warp * (32 * RS_ROUNDS) + r * 32 + lane;
                const bool valid = li < tn;
                k[r] = valid ? sm.stk[li] : K(0);
                if (HAS_V) v[r] = valid ? sm.stv[li] : 0u;
            }
        }
        __syncthreads();  // staging consumed, wc cleared, previous write-out done: prefetch the next tile
        if (threadIdx.x == 0 && tb + RS_TILE < e) {
            fence_proxy_async_smem();
            stage(tb + RS_TILE);
        }
        const int wl = warp * (32 * RS_ROUNDS) + lane;  // tile-local index of round 0
#pragma unroll
        for (int r = 0; r < RS_ROUNDS; ++r) {
            const bool valid = wl + r * 32 < tn;
            const uint32_t d = valid ? ((uint32_t)(k[r] >> shift) & dmask) : RS_BINS;
            dg[r] = d;
            // lanes with the same digit: 8 ballots (MATCH.ANY measured 1.6x slower here)
            uint32_t peers = 0xffffffffu;
            if (tn < RS_TILE) {  // ragged last tile: valid lanes never match invalid ones
                peers = __ballot_sync(0xffffffffu, valid);
                if (!valid) peers = ~peers;
            }
            peers = rs_match_digit(d, peers);
            const uint32_t rank = __popc(peers & lt);
            pos[r] = sm.wc[warp][d] + rank;
            __syncwarp();
            if ((peers & lt) == 0) sm.wc[warp][d] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        {   // digit d = threadIdx.x: tile count, tile-local offset, per-warp offsets
            const int d = threadIdx.x;
            uint32_t cnt = 0;
            if (d < RS_BINS) {
#pragma unroll
                for (int w = 0; w < RS_WARPS; ++w) cnt += sm.wc[w][d];
            }
            uint32_t tot;
            const uint32_t off = block_exclusive_sum(cnt, &tot, sm.sw);
            if (d < RS_BINS) {
                sm.adj[d] = sm.base[d] - off;
                sm.base[d] += cnt;  // advance past this tile (only thread d touches base[d])
                uint32_t run = off;
#pragma unroll
                for (int w = 0; w < RS_WARPS; ++w) {
                    const uint32_t c = sm.wc[w][d];
                    sm.wc[w][d] = run;
                    run += c;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < RS_ROUNDS; ++r) {
            if (dg[r] < RS_BINS) {
                const uint32_t lp = sm.wc[warp][dg[r]] + pos[r];
                sm.sk[lp] = k[r];
                if (HAS_V) sm.sv[lp] = v[r];
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < RS_WARPS * (RS_BINS + 1); i += RS_NT) (&sm.wc[0][0])[i] = 0;
        if (tn == RS_TILE) {
#pragma unroll
            for (int r = 0; r < RS_ROUNDS; ++r) {
                const int i = threadIdx.x + r * RS_NT;
                const K key = sm.sk[i];
                const uint32_t dst = sm.adj[(uint32_t)(key >> shift) & dmask] + (uint32_t)i;
                kout[dst] = key;
                if (HAS_V) vout[dst] = sm.sv[i];
            }
        } else {
            for (int i = threadIdx.x; i < tn; i += RS_NT) {
                const K key = sm.sk[i];
                const uint32_t dst = sm.adj[(uint32_t)(key >> shift) & dmask] + (uint32_t)i;
                kout[dst] = key;
                if (HAS_V) vout[dst] = sm.sv[i];
            }
        }
    }
}

// Stable LSD radix sort of keys[0..n) on bits [begin_bit, end_bit), carrying
// optional uint32 values.  Uses keys_alt / vals_alt as ping-pong buffers.  On
// return *in_alt tells which buffer holds the sorted result.
// pack (optional, 64-bit keys without values): the first pass forms the keys
// from pack.src / pack.dst instead of reading keys (whose contents are ignored)
template <class K, bool HAS_V>
int radix_sort(Ctx& ctx, K* keys, K* keys_alt, uint32_t* vals, uint32_t* vals_alt, int64_t n,
               int begin_bit, int end_bit, bool* in_alt, const RsPack* pack = nullptr) {
    *in_alt = false;
    if (pack && (HAS_V || sizeof(K) != 8)) {
        set_error("radix_sort: the fused pack needs 64-bit keys without values");
        return PR_EINVAL;
    }
    if (n <= 1 || end_bit <= begin_bit) return PR_OK;
    if (n > (int64_t)UINT32_MAX) {
        set_error("radix_sort: %lld keys exceed the 32-bit digit offsets", (long long)n);
        return PR_EINVAL;
    }
    const size_t smem = sizeof(RsSmem<K, HAS_V>);
    PR_CUDA(cudaFuncSetAttribute(k_rs_scatter<K, HAS_V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (pack)
        PR_CUDA(cudaFuncSetAttribute(k_rs_scatter<K, HAS_V, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    int per_sm = 0;
    PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rs_scatter<K, HAS_V>, RS_NT, smem));
    if (per_sm < 1) per_sm = 1;
    int64_t G = (n + RS_TILE - 1) / RS_TILE;
    const int64_t cap = (int64_t)ctx.num_sms * per_sm;
    if (G > cap) G = cap;
    int64_t per = (n + G - 1) / G;
    per = (per + RS_TILE - 1) / RS_TILE * RS_TILE;
    G = (n + per - 1) / per;
    uint32_t* hist = nullptr;
    PR_TRY(dalloc(&hist, (size_t)(RS_BINS * G + 2 * RS_BINS), ctx.stream));
    uint32_t* dtot = hist + RS_BINS * G;
    uint32_t* dbase = dtot + RS_BINS;
    K* kin = keys;
    K* kout = keys_alt;
    uint32_t* vin = vals;
    uint32_t* vout = vals_alt;
    bool alt = false;
    for (int shift = begin_bit; shift < end_bit; shift += RS_BITS) {
        // the last digit covers only the bits left below end_bit: the result is
        // ordered by exactly [begin_bit, end_bit) (stable for everything else)
        const int nb = end_bit - shift < RS_BITS ? end_bit - shift : RS_BITS;
        const uint32_t dmask = (1u << nb) - 1u;
        RsPack pk;
        if (pack && shift == begin_bit) pk = *pack;
        PR_LAUNCH(ctx, (k_rs_hist<K>), (unsigned)G, RS_NT, 0, (const K*)kin, n, per, shift, dmask, hist, G, pk);
        PR_LAUNCH(ctx, k_rs_digit_scan, RS_BINS, 256, 0, hist, G, dtot);
        PR_LAUNCH(ctx, k_rs_dbase, 1, 256, 0, (const uint32_t*)dtot, dbase);
        if (pk.src)
            PR_LAUNCH(ctx, (k_rs_scatter<K, HAS_V, true>), (unsigned)G, RS_NT, smem, (const K*)kin,
                      (const uint32_t*)vin, kout, vout, n, per, shift, dmask, (const uint32_t*)hist, G,
                      (const uint32_t*)dbase, pk);
        else
            PR_LAUNCH(ctx, (k_rs_scatter<K, HAS_V>), (unsigned)G, RS_NT, smem, (const K*)kin,
                      (const uint32_t*)vin, kout, vout, n, per, shift, dmask, (const uint32_t*)hist, G,
                      (const uint32_t*)dbase, pk);
        K* tk = kin; kin = kout; kout = tk;
        uint32_t* tv = vin; vin = vout; vout = tv;
        alt = !alt;
    }
    dfree(hist, ctx.stream);
    *in_alt = alt;
    return PR_OK;
}

// ----------------------------------------------------------------- merge --
// C = the stable merge of sorted A[0, na) and B[0, nb) (merge path: ties take
// A first).  k_merge_part finds, for every tile boundary t*MG_TILE of C, the
// number of A elements before it (one binary search per boundary, all in
// parallel); each CTA then merges its tile's A and B slices from shared memory
// (a binary search per thread for its own diagonal, VT outputs each) and
// writes the tile out coalesced.  Used by the chunked host ingest (ingest.cu).
constexpr int MG_NT = 256, MG_VT = 8, MG_TILE = MG_NT * MG_VT;
static __global__ void k_merge_part(const uint64_t* __restrict__ A, int64_t na, const uint64_t* __restrict__ B, int64_t nb,
                             int64_t ntiles, int64_t* __restrict__ part) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    const int64_t diag = min(t * MG_TILE, na + nb);
    int64_t lo = max((int64_t)0, diag - nb), hi = min(diag, na);
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (A[mid] <= B[diag - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    part[t] = lo;
}
static __global__ void __launch_bounds__(MG_NT) k_merge_tile(const uint64_t* __restrict__ A, int64_t na,
                                                      const uint64_t* __restrict__ B, int64_t nb,
                                                      const int64_t* __restrict__ part, uint64_t* __restrict__ C) {
    __shared__ uint64_t sk[MG_TILE];
    __shared__ uint64_t so[MG_TILE];
    const int64_t t = blockIdx.x;
    const int64_t d0 = t * MG_TILE, d1 = min(d0 + MG_TILE, na + nb);
    const int64_t i0 = part[t], i1 = part[t + 1];
    const int64_t j0 = d0 - i0, j1 = d1 - i1;
    const int la = (int)(i1 - i0), lb = (int)(j1 - j0), ln = la + lb;
    for (int k = threadIdx.x; k < la; k += MG_NT) sk[k] = A[i0 + k];
    for (int k = threadIdx.x; k < lb; k += MG_NT) sk[la + k] = B[j0 + k];
    __syncthreads();
    const int dd = min((int)threadIdx.x * MG_VT, ln);
    int lo = max(0, dd - lb), hi = min(dd, la);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sk[mid] <= sk[la + dd - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    int ia = lo, ib = dd - lo;
#pragma unroll
    for (int v = 0; v < MG_VT; ++v) {
        const int o = dd + v;
        if (o < ln) {
            const bool takeA = ib >= lb || (ia < la && sk[ia] <= sk[la + ib]);
            so[o] = takeA ? sk[ia++] : sk[la + ib++];
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < ln; k += MG_NT) C[d0 + k] = so[k];
}
inline int merge_u64(Ctx& ctx, const uint64_t* A, int64_t na, const uint64_t* B, int64_t nb, uint64_t* C) {
    const int64_t n = na + nb;
    if (n == 0) return PR_OK;
    const int64_t ntiles = (n + MG_TILE - 1) / MG_TILE;
    int64_t* part = nullptr;
    PR_TRY(dalloc(&part, (size_t)ntiles + 1, ctx.stream));
    PR_LAUNCH(ctx, k_merge_part, (unsigned)((ntiles + 1 + 255) / 256), 256, 0, A, na, B, nb, ntiles, part);
    PR_LAUNCH(ctx, k_merge_tile, (unsigned)ntiles, MG_NT, 0, A, na, B, nb, (const int64_t*)part, C);
    dfree(part, ctx.stream);
    return PR_OK;
}

inline int bits_for(uint64_t maxval) {  // number of bits to represent values <= maxval
    int b = 0;
    while (b < 64 && (maxval >> b) != 0) ++b;
    return b;
}

}  // namespace prgpu
