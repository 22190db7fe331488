// blocked.cu -- source-blocked views for contrib vectors larger than L2
// ("propagation blocking (binning contributions by ...range)",
// cited in PAPER.md related work P:401).
//
// A synchronous sweep over a view whose contrib vector y (8 B per source) is
// far larger than the 126 MB L2 (config 5: 50M sources = 400 MB) pays a DRAM
// random access per gathered edge.  The blocked form cuts the contrib slots
// into segments of 2^seg_bits slots (64 MB at the default 23 bits) and splits
// the view's edges by the segment of their slot, keeping view-row order inside
// each segment.  A sweep then runs the edge-stream gather once per segment,
// each pass gathering from one L2-resident slice of y and accumulating
// S(r) += S_seg(r) into the view's sums in segment order (deterministic).
// Extra traffic per sweep: the sums read-modify-write of every (row, segment)
// pair, instead of ~32-64 B of DRAM per gathered edge.
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "internal.h"
#include "primitives.cuh"

namespace prgpu {

// rowid[e] = view row of edge e (edge-parallel over 1024-edge chunks).
__global__ void k_edge_rows(const int64_t* __restrict__ rp, int64_t nr, int64_t E, uint32_t* __restrict__ rowid) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t o0 = w0 * 1024; o0 < E; o0 += nw * 1024) {
        const int64_t o1 = min(E, o0 + 1024);
        int64_t lo = 0, hi = nr;  // last row with rp[row] <= o0
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (rp[mid] <= o0)
                lo = mid;
            else
                hi = mid;
        }
        int64_t i = lo, o = o0;
        while (o < o1) {
            const int64_t re = min(o1, rp[i + 1]);
            for (int64_t k = o + lane; k < re; k += 32) rowid[k] = (uint32_t)i;
            o = re;
            ++i;
        }
    }
}

// start[s] = first edge (in the slot-partitioned order) of segment s.
__global__ void k_seg_bounds(const uint32_t* __restrict__ slot, int64_t E, int bits, int nseg,
                             int64_t* __restrict__ start) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        const int sg = (int)(slot[e] >> bits);
        const int sp = e == 0 ? -1 : (int)(slot[e - 1] >> bits);
        for (int q = sp + 1; q <= sg; ++q) start[q] = e;
        if (e == E - 1)
            for (int q = sg + 1; q <= nseg; ++q) start[q] = E;
    }
}

struct SegRunGet {
    const uint32_t* rowid;
    __device__ int64_t operator()(int64_t i) const { return (i == 0 || rowid[i] != rowid[i - 1]) ? 1 : 0; }
};
struct SegRunEmit {
    const uint32_t* rowid;
    int32_t* vid;
    int64_t* rp;
    __device__ void operator()(int64_t i, int64_t pos, int64_t f) const {
        if (f) {
            vid[pos] = (int32_t)rowid[i];
            rp[pos] = i;
        }
    }
};

__global__ void k_set_i64(int64_t* p, int64_t v) { *p = v; }

int build_view_blocked(View& v, Ctx& ctx, int64_t n_contrib) {
    cudaStream_t s = ctx.stream;
    v.nseg = 0;
    v.seg = nullptr;
    if (v.nrows == 0 || v.nedges == 0 || n_contrib <= 0) return PR_OK;
    // policy: blocked when y does not fit comfortably in L2 (PRGPU_SEG_BITS
    // forces a segment size, 0 disables)
    // 64 MB slices measured best on config 5 (16/32/64 MB: 7.8/6.1/5.3 ms per sweep)
    int bits = 23;
    const char* e = getenv("PRGPU_SEG_BITS");
    if (e && *e) {
        bits = atoi(e);
        if (bits <= 0) return PR_OK;
    } else if (n_contrib * 8 <= ((int64_t)96 << 20)) {
        return PR_OK;
    }
    if (bits > 30) bits = 30;
    while (((n_contrib - 1) >> bits) + 1 > 256) ++bits;  // one 8-bit radix pass
    const int nseg = (int)(((n_contrib - 1) >> bits) + 1);
    if (nseg <= 1) return PR_OK;
    const int64_t E = v.nedges;

    uint32_t *keys = nullptr, *keys_alt = nullptr, *rows = nullptr, *rows_alt = nullptr;
    int64_t* start = nullptr;
    TmpGuard tg_(ctx.stream);
    tg_.track(keys);
    tg_.track(keys_alt);
    tg_.track(rows);
    tg_.track(rows_alt);
    tg_.track(start);

    PR_TRY(dalloc(&keys, (size_t)E, s));
    PR_TRY(dalloc(&keys_alt, (size_t)E, s));
    PR_TRY(dalloc(&rows, (size_t)E, s));
    PR_TRY(dalloc(&rows_alt, (size_t)E, s));
    PR_TRY(dalloc(&start, (size_t)nseg + 1, s));
    PR_CUDA(cudaMemcpyAsync(keys, v.col, sizeof(uint32_t) * (size_t)E, cudaMemcpyDeviceToDevice, s));
    const unsigned g = (unsigned)std::min<int64_t>((E + 1023) / 1024 * 32 / 256 + 1, (int64_t)ctx.num_sms * 16);
    PR_LAUNCH(ctx, k_edge_rows, g, 256, 0, (const int64_t*)v.row_ptr, v.nrows, E, rows);
    // stable partition by segment: rows stay in view order inside each segment
    bool alt = false;
    PR_TRY((radix_sort<uint32_t, true>(ctx, keys, keys_alt, rows, rows_alt, E, bits, bits + bits_for((uint64_t)(nseg - 1)),
                                       &alt)));
    const uint32_t* ks = alt ? keys_alt : keys;
    const uint32_t* rs = alt ? rows_alt : rows;
    PR_LAUNCH(ctx, k_seg_bounds, (unsigned)std::min<int64_t>((E + 255) / 256, (int64_t)ctx.num_sms * 16), 256, 0, ks, E,
              bits, nseg, start);
    std::vector<int64_t> hs(nseg + 1);
    PR_CUDA(cudaMemcpyAsync(hs.data(), start, sizeof(int64_t) * (nseg + 1), cudaMemcpyDeviceToHost, s));
    PR_CUDA(cudaStreamSynchronize(s));

    v.seg = new (std::nothrow) View[nseg];
    if (!v.seg) {
        set_error("build_view_blocked: host allocation failed");
        return PR_ENOMEM;
    }
    v.nseg = nseg;
    v.seg_bits = bits;
    int64_t* cnt = nullptr;
    tg_.track(cnt);
    PR_TRY(dalloc(&cnt, 1, s));
    for (int q = 0; q < nseg; ++q) {
        View& sv = v.seg[q];
        const int64_t a = hs[q], len = hs[q + 1] - hs[q];
        sv.nedges = len;
        if (len == 0) continue;
        int32_t* vid_tmp = nullptr;
        PR_TRY(dalloc(&vid_tmp, (size_t)len, s));
        PR_TRY(dalloc(&sv.row_ptr, (size_t)len + 1, s));
        sv.owns_row_ptr = true;
        PR_TRY((device_scan<int64_t>(ctx, len, SegRunGet{rs + a}, SegRunEmit{rs + a, vid_tmp, sv.row_ptr}, cnt)));
        PR_TRY(read_count(ctx, cnt, &sv.nrows));
        PR_LAUNCH(ctx, k_set_i64, 1, 1, 0, sv.row_ptr + sv.nrows, len);
        PR_TRY(dalloc(&sv.vid, (size_t)sv.nrows, s));
        PR_CUDA(cudaMemcpyAsync(sv.vid, vid_tmp, sizeof(int32_t) * (size_t)sv.nrows, cudaMemcpyDeviceToDevice, s));
        dfree(vid_tmp, s);
        PR_TRY(dalloc(&sv.col, (size_t)stream_pad(len), s));
        PR_CUDA(cudaMemcpyAsync(sv.col, ks + a, sizeof(int32_t) * (size_t)len, cudaMemcpyDeviceToDevice, s));
        PR_TRY(build_view_stream(sv, ctx, (int32_t)n_contrib, nullptr, nullptr));
        dfree(sv.row_ptr, s);  // the stream engine does not read row_ptr
        sv.owns_row_ptr = false;
    }
    dfree(cnt, s);
    dfree(keys, s);
    dfree(keys_alt, s);
    dfree(rows, s);
    dfree(rows_alt, s);
    dfree(start, s);
    return PR_OK;
}

}  // namespace prgpu
