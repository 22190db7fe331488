// streamengine.cuh -- the edge-stream engine behind K-GATHER (sync / reduced /
// async sweeps).  It computes, for every row r of a View,
//     S(r) = sum_{e in row r} y[col[e]]       and calls  emit(r, S(r))
// (emit_at(j, ...) / emit_first(...) for the closures of a step, after
// prep(first row, start bits) let the policy prefetch per-row data),
// i.e. the sum of Eq.(1) over in-neighbours, as ONE flat pass over
// the view's col array with no per-row work units.  It only emits S(r) (one
// store per row, no loads): the rank update, fused contrib and Delta run in the
// row-parallel K-FINALIZE that follows, so the only dependent load chain here
// is col -> gather:
//
//   * the edge array is cut into steps of SE_STEP = 32 lanes x SE_V edges; lane
//     L of a warp owns edges [s*SE_STEP + L*SE_V, +SE_V) of step s, loaded as
//     two 16-byte vectors (coalesced, L1::no_allocate, L2 evict_first), and
//     issues its SE_V gathers back to back;
//   * a bit per edge (flags) marks the first edge of each row.  Segments are
//     summed in registers: within a lane serially, across lanes by a
//     segmented shuffle scan, across the steps of a span by a carried sum;
//     row ids come from step_row[s] (first row starting at or after the step)
//     plus the warp-exclusive count of row starts;
//   * steps are grouped in spans (span_steps consecutive steps), statically
//     assigned to warps (span -> warp span mod #warps).  A row that crosses a
//     span boundary ("boundary row" b, spans s0..s1) is assembled from per-span
//     pieces part_out[s0] + part_in[s0+1] + ... + part_in[s1] (fixed order) by
//     the warp taking its last ticket.
//
// Every sum is taken in an order fixed by the data layout only, so the sweep
// is bit-for-bit deterministic (K-GATHER).  The edge array is padded
// to whole steps with a contrib slot that always holds +0.0 and no row starts,
// so the last row absorbs exact zeros and no lane needs a bounds test.
#pragma once
#include "internal.h"

namespace prgpu {

struct StreamArgs {
    const int32_t* col;        // [nsteps * SE_STEP] contrib slots (padded)
    const uint8_t* flags8;     // [nsteps * 32] bit j of byte i: edge 8i + j starts a row
    const int32_t* step_row;   // [nsteps + 1] first row starting at or after edge s*SE_STEP
    int64_t nsteps;
    int64_t span_steps;
    int64_t nspans;
    const int32_t* bin;        // [nspans] boundary row open at the span's first edge, or -1
    const int32_t* bout;       // [nspans] boundary row started in the span and open at its end, or -1
    const int32_t* b_row;      // [nbound] row id
    const int32_t* b_s0;       // [nbound] first span of the row
    const int32_t* b_s1;       // [nbound] last span of the row
    double* part_in;           // [nspans] (8-byte pieces; reinterpreted for non-fp64 sums)
    double* part_out;          // [nspans]
    uint32_t* bticket;         // [nbound]
};

__device__ __forceinline__ int4 ld_stream_v4(const int32_t* p, uint64_t pol) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t ld_stream_u8(const uint8_t* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// Lane 0 of some warp: hand the piece `val` of boundary row b (from span
// `span`) to the ticket protocol; the last of the b_s1 - b_s0 + 1 pieces sums
// them in span order and finalizes the row.
template <class P>
__device__ __forceinline__ void stream_piece(P& p, const StreamArgs& a, int32_t b, int64_t span,
                                             typename P::T val, bool out_piece) {
    using T = typename P::T;
    static_assert(sizeof(T) == sizeof(double), "8-byte pieces");
    T* pin = reinterpret_cast<T*>(a.part_in);
    T* pout = reinterpret_cast<T*>(a.part_out);
    if (out_piece)
        pout[span] = val;
    else
        pin[span] = val;
    // release: the piece is visible before the ticket moves.  (A __threadfence
    // here compiles to MEMBAR.SC + CCTL.IVALL, which would also invalidate this
    // SM's L1 and with it the L1 tier of hot contribs.)
    // wrapping ticket (atom.inc: count-1 -> 0), so no reset store is needed and
    // pieces of different sweeps may interleave (in-place persistent kernel:
    // the winner then sums each span's latest piece)
    const int32_t s0 = a.b_s0[b], s1 = a.b_s1[b];
    uint32_t t;
    asm volatile("atom.inc.release.gpu.u32 %0, [%1], %2;"
                 : "=r"(t)
                 : "l"(a.bticket + b), "r"((uint32_t)(s1 - s0))
                 : "memory");
    if (t == (uint32_t)(s1 - s0)) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");  // winner only: acquire the other pieces
        T sum = __ldcg(pout + s0);
        for (int32_t s = s0 + 1; s <= s1; ++s) sum += __ldcg(pin + s);
        p.emit((int64_t)a.b_row[b], sum);
    }
}

// One span of steps for the calling warp.
template <class P>
__device__ __forceinline__ void stream_span(P& p, const StreamArgs& a, int64_t span, uint64_t pol_stream) {
    const int lane = threadIdx.x & 31;
    const int64_t sb = span * a.span_steps;
    const int64_t se = min(a.nsteps, sb + a.span_steps);
    const int32_t bin = a.bin[span];
    bool first_closure = true;  // no row has started in this span yet
    using T = typename P::T;
    T carry = T(0);             // sum of the row open at the current step's start
    // software pipeline: the indices, flags and step_row of step s+1 are loaded
    // while the gathers of step s are in flight
    int4 c0 = ld_stream_v4(a.col + sb * SE_STEP + (int64_t)lane * SE_V, pol_stream);
    int4 c1 = ld_stream_v4(a.col + sb * SE_STEP + (int64_t)lane * SE_V + 4, pol_stream);
    uint32_t fn = ld_stream_u8(a.flags8 + sb * 32 + lane);
    int32_t Rn = a.step_row[sb];
    for (int64_t s = sb; s < se; ++s) {
        T v[SE_V];
        v[0] = p.load(c0.x);
        v[1] = p.load(c0.y);
        v[2] = p.load(c0.z);
        v[3] = p.load(c0.w);
        v[4] = p.load(c1.x);
        v[5] = p.load(c1.y);
        v[6] = p.load(c1.z);
        v[7] = p.load(c1.w);
        const uint32_t f = fn;
        const int32_t R0 = Rn;
        if (s + 1 < se) {
            const int64_t e1 = (s + 1) * SE_STEP + (int64_t)lane * SE_V;
            c0 = ld_stream_v4(a.col + e1, pol_stream);
            c1 = ld_stream_v4(a.col + e1 + 4, pol_stream);
            fn = ld_stream_u8(a.flags8 + (s + 1) * 32 + lane);
            Rn = a.step_row[s + 1];
        }
        // row starts: warp-exclusive rank of this lane's first start and the
        // step's total, from ballots of the bit planes of the per-lane count
        // (nf <= 8: 4 planes; no shuffles on the MIO pipe)
        const int nf = __popc(f);
        const uint32_t lt = lanemask_lt();
        int rank0 = 0, nst = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint32_t m = __ballot_sync(0xffffffffu, (nf >> b) & 1);
            rank0 += __popc(m & lt) << b;
            nst += __popc(m) << b;
        }
        const uint32_t smask = __ballot_sync(0xffffffffu, nf > 0);   // lanes holding a row start
        const uint32_t le = lt | (1u << lane);
        p.prep((int64_t)R0 - 1 + rank0, f);  // policy may prefetch per-row data of this lane's closures
        // in-lane segments: the i-th start (i >= 1) of this lane closes slot
        // rank0 + i, i.e. row R0 - 1 + rank0 + i, with the lane-local segment
        T run = T(0), head = T(0);
        int i = 0;
#pragma unroll
        for (int j = 0; j < SE_V; ++j) {
            if (f & (1u << j)) {
                if (i == 0) {
                    head = run;
                } else {
                    p.emit_at(j, (int64_t)R0 - 1 + rank0 + i, run);
                }
                ++i;
                run = T(0);
            }
            run += v[j];
        }
        // open segment of each lane flows right until the next lane with a start
        T o = run;
        if (lane == 0 && nf == 0) o = carry + o;
        // segmented inclusive scan; F = a row starts within the lanes the
        // running sum already covers ([lane - 2d + 1, lane] after the round
        // with distance d), read off the start mask instead of shuffled
        T S = o;
        bool F = nf > 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T tS = __shfl_up_sync(0xffffffffu, S, d);
            if (lane >= d && !F) S = tS + S;
            const int lo = lane - 2 * d + 1;
            F = ((smask & le) >> (lo > 0 ? lo : 0)) != 0;
        }
        T I = __shfl_up_sync(0xffffffffu, S, 1);
        if (lane == 0) I = carry;
        carry = __shfl_sync(0xffffffffu, S, 31);
        if (nf > 0) {  // the first start of this lane closes slot rank0
            const T val = I + head;
            if (rank0 == 0 && first_closure) {
                if (bin >= 0) stream_piece(p, a, bin, span, val, false);
                // else: the span begins with a row start; slot 0 is the previous span's row
            } else {
                p.emit_first((int64_t)R0 - 1 + rank0, val);
            }
        }
        if (nst > 0) first_closure = false;
    }
    if (lane == 0) {
        if (first_closure) {
            stream_piece(p, a, bin, span, carry, false);  // a middle piece of a long row
        } else {
            const int32_t bo = a.bout[span];
            if (bo >= 0) {
                stream_piece(p, a, bo, span, carry, true);
            } else {
                p.emit((int64_t)a.step_row[se] - 1, carry);
            }
        }
    }
}

template <class P>
__device__ __forceinline__ void stream_run(P& p, const StreamArgs& a) {
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint64_t pol = policy_evict_first();
    for (int64_t span = w; span < a.nspans; span += nw) stream_span(p, a, span, pol);
}

}  // namespace prgpu
