// internal.h -- library-private state of libprgpu.
#pragma once
#include <vector>
#include "common.cuh"

namespace prgpu {

// Edge-stream engine (streamengine.cuh): SE_V edges per lane per step.
constexpr int SE_V = 8;
constexpr int SE_STEP = 32 * SE_V;
#ifndef PRGPU_SE_NT
#define PRGPU_SE_NT 1024
#endif
constexpr int SE_NT = PRGPU_SE_NT;          // threads per CTA of the stream gather (1 CTA per SM)
constexpr int SE_NT_IP = 512;               // in-place (async / No-Sync) stream kernels: 128 registers
                                            // for the prefetched finalize operands of a step
// Contribs [0, hot_n) (the highest out-degrees) are copied into shared memory
// by every CTA at the start of a synchronous sweep; [hot_n, SE_L1_TIER) are
// gathered with L1::evict_last, the rest with L1::no_allocate.
// R-MAT-24 K-GATHER by (smem tier, L1 tier) slots: (12K, 32K) 0.777, (16K, 32K)
// 0.770, (18K, 34K) 0.774, (20K, 32K) 0.768, (20K, 36K) 0.767, (20K, 40K) 0.782,
// (22K, 40K) 0.824 ms -- past ~20K the L1 left over is too small for the
// misses in flight (profiles/r2/ab_tiers.txt)
#ifndef PRGPU_SE_HOT_MAX
#define PRGPU_SE_HOT_MAX 20480
#endif
constexpr int SE_HOT_MAX = PRGPU_SE_HOT_MAX;  // 160 KB of fp64
// In-place sweeps read the hot tier as a snapshot taken at the start of the
// (local) sweep, so a larger tier makes sweeps faster but fresher values rarer:
// R-MAT-24 async, hot 0 / 2K / 8K / 16K: 61 / 68 / 73 / 78 sweeps, 109 / 78 / 80 / 82 ms.
constexpr int SE_HOT_IP = 2048;
constexpr int SE_MAX_PHASES = 64;   // PR_MODE_PHASED: most phases per sweep
#ifndef PRGPU_SE_L1_TIER
#define PRGPU_SE_L1_TIER 36864
#endif
constexpr int SE_L1_TIER = PRGPU_SE_L1_TIER;
inline int64_t stream_pad(int64_t E) { return ((E > 0 ? E : 1) + SE_STEP - 1) / SE_STEP * SE_STEP; }
// Threads per CTA of the row-parallel kernels (K-FINALIZE, K-ZERO, ...).
constexpr int GT_NT = 256;

// A set of rows over which the gather runs: all vertices (plain) or the
// computed representatives R (reduced).  Rows are in increasing vertex id.
struct View {
    bool alias = false;             // a shallow copy of another view (owns nothing)
    int64_t nrows = 0;
    int64_t nedges = 0;
    int64_t* row_ptr = nullptr;     // int64[nrows+1] (plain: aliases the canonical row_ptr)
    int32_t* col = nullptr;         // int32[nedges] contrib indices (relabelled sources)
    int32_t* vid = nullptr;         // int32[nrows] vertex id of each row (nullptr: identity)
    bool owns_row_ptr = false;
    // edge-stream engine (build_view_stream; col is padded to nsteps * SE_STEP)
    int64_t nsteps = 0;
    int64_t span_steps = 1;
    int64_t nspans = 0;
    int64_t nbound = 0;
    uint32_t* sflags = nullptr;     // [nsteps * 8] row-start bits
    int32_t* step_row = nullptr;    // [nsteps + 1]
    int32_t* bin = nullptr;         // [nspans]
    int32_t* bout = nullptr;        // [nspans]
    int32_t* b_row = nullptr;       // [nbound]
    int32_t* b_s0 = nullptr;
    int32_t* b_s1 = nullptr;
    double* part_in = nullptr;      // [nspans]
    double* part_out = nullptr;     // [nspans]
    uint32_t* bticket = nullptr;    // [nbound]
    double* sums = nullptr;         // [nrows] S(r) of the current sweep (K-GATHER -> K-FINALIZE)
    // source-blocked form (blocked.cu), for contrib vectors larger than L2:
    // seg[i] holds the edges whose contrib slot lies in [i << seg_bits, (i+1) << seg_bits),
    // rows in view order; its vid maps a sub-view row to the row of THIS view
    int nseg = 0;
    int seg_bits = 0;
    View* seg = nullptr;
    int2* rinfo = nullptr;          // [nrows] (outdeg, contrib slot) of the row's vertex, row order
    // PR_MODE_PHASED (cached per phase count K): phase k gathers and finalizes
    // the rows [phase_rb[k], phase_rb[k+1]) (row-aligned, build_phase_view)
    int phase_k = 0;
    int64_t phase_rb[SE_MAX_PHASES + 1];
    int64_t phase_eb[SE_MAX_PHASES + 1];  // first edge (view edge order) of each phase, [K] = nedges
    View* phv = nullptr;            // [phv_k] edge-stream sub-view of each phase's rows
    int phv_k = 0;
};

// Device-resident iteration state (one per graph).
struct DevState {
    int32_t done;
    int32_t iters;
    int32_t max_iter;
    int32_t norm_linf;
    double tau;
    double l1;
    double linf;
    uint32_t ticket_gather;
    uint32_t ticket_scatter;
    int32_t status;
    int32_t log_cap;
    int32_t peer_err;   // the device-side peer barrier timed out
};

// NVLS multicast team of the sharded contrib buffers (multicast.cu)
struct McState {
    unsigned long long mc = 0;   // CUmemGenericAllocationHandle of the multicast object
    unsigned long long mem = 0;  // this rank's physical allocation bound to it
    bool have_mc = false;
    bool bound = false;
    size_t seg = 0;          // bytes per parity segment (ny doubles + world flags, granularity-rounded)
    size_t size = 0;         // 2 * seg
    void* uva = nullptr;     // unicast mapping of mem (sy[0], sy[1] point into it)
    void* mva = nullptr;     // multicast mapping (multimem.st replicates to every rank)
    double* y[2] = {nullptr, nullptr};  // multicast addresses of the two parities
};

}  // namespace prgpu

struct pr_graph {
    int64_t n = 0;
    int64_t m_raw = 0;
    int64_t E = 0;
    int num_sms = 0;
    int device = 0;
    // canonical in-CSR (bit-exact with the oracle)
    int64_t* row_ptr = nullptr;
    int32_t* col = nullptr;
    int32_t* outdeg = nullptr;
    // contrib relabelling: cidx[v] in [0, n_contrib) for outdeg(v) > 0, else -1
    int32_t* cidx = nullptr;
    int64_t n_contrib = 0;
    // vertices of in-degree 0: x_t = (1-d)/n for every t >= 1 exactly, so they
    // are written once, in the first sweep, and excluded from the gather views
    int32_t* zlist = nullptr;
    int64_t nz = 0;
    prgpu::View plain;
    // reductions
    bool pre_done = false;
    uint32_t pre_flags = 0;
    int32_t* rep = nullptr;
    int32_t* chain_src = nullptr;
    int32_t* chain_k = nullptr;
    int32_t max_chain = 0;
    int64_t n_members = 0;
    int32_t* mem_vid = nullptr;
    int32_t* mem_src = nullptr;
    int32_t* mem_k = nullptr;
    int32_t* mem_srow = nullptr;    // reduced-view row of mem_src (K-FINALIZE reads its S)
    int2* mem_info = nullptr;       // (outdeg, contrib slot) of each member
    int32_t* mem_h = nullptr;       // chain member: index of its source among the chain sources (else -1)
    int64_t n_hsrc = 0;             // distinct chain sources (delayed chain resolution)
    prgpu::View reduced;
    // row sharding over P ranks (pr_graph_shard, shard.cu)
    bool shard_only = false;        // created by pr_graph_create_sharded: only pr_run_sharded applies
    int32_t shard_rank = -1;
    int32_t shard_world = 0;
    int64_t shard_chunk = 0;        // doubles per rank in the exchanged buffer (owned contribs + (L1, Linf))
    int64_t shard_owned = 0;        // vertices this rank computes
    int32_t* sowner = nullptr;      // [n] rank owning each vertex
    int32_t* scidx = nullptr;       // [n] sharded contrib slot (or -1)
    int32_t* szlist = nullptr;      // owned vertices of in-degree 0
    int64_t shard_hot = 0;          // H: contribs [0, H) are copies of the H hottest (gather tiers)
    int32_t* shot_src = nullptr;    // [H] chunk slot of each hot copy
    int64_t snz = 0;
    prgpu::View shard;              // owned rows of in-degree > 0, columns in sharded slots
    double* sy[2] = {nullptr, nullptr};  // [H + world * chunk + 1] ping-pong, last slot = +0.0 (cudaMalloc: IPC-exportable)
    double** speer_dev = nullptr;   // [2][world-1] peers' sy[parity] (pr_shard_set_peers / pr_shard_open_ipc)
    unsigned long long** speer_flags = nullptr;  // [world-1] peers' arrival flags (after their sy[0])
    bool sdev_barrier = false;      // per-sweep synchronisation by the device-side peer barrier
    uint64_t bar_epoch = 0;         // epochs of that barrier so far (the same sequence on every rank)
    prgpu::McState* mc = nullptr;   // NVLS multicast buffers (pr_shard_mc_*), exclusive with the IPC peers
    std::vector<void*> speer_ipc;   // IPC-opened peer bases to close
    // iteration buffers (allocated lazily by pr_run)
    double* x = nullptr;            // fp64[n] (used when the caller's ranks are on the host)
    double* xr = nullptr;           // sync sweeps: x of the view's rows, row order (unpermuted at the end)
    int64_t xr_cap = 0;
    double* xm = nullptr;           // sync sweeps: x of the members, member order
    double* y[2] = {nullptr, nullptr};
    double* cta_partial = nullptr;  // [2 * (gather grid + scatter grid)] (L1, Linf)
    int64_t partial_cap = 0;
    double* ab = nullptr;           // chain alpha/beta [2 * (max_chain+1)]
    double* hist = nullptr;         // [(max_chain+1) * n_hsrc] last values of the chain sources (ring)
    int64_t hist_cap = 0;
    // identical members folded into their source row (sync reduced sweeps,
    // iterate.cu build_fold): rinfo of the reduced view with FOLD_FLAG on the
    // rows that have identical members, their multiplicity 1 + #members, and
    // the members that still need per-sweep work (chain members, and identical
    // members with out-degree > 0: their contrib)
    int2* fold_rinfo = nullptr;
    int32_t* fold_w = nullptr;
    int32_t* fold_list = nullptr;   // chain members
    int64_t fold_n = 0;
    int4* fold_crec = nullptr;      // chain members in fold_list order: (source row, hist index or -1, slot, k)
    double* fold_xc = nullptr;      // x of the chain members in fold_list order (during a run)
    int4* fold_rec = nullptr;       // identical members with a contrib: (source row, outdeg, slot, -)
    int64_t fold_nrec = 0;
    bool fold_ready = false;
    double* delta_log = nullptr;    // [2 * log_cap]
    int32_t log_cap = 0;
    int32_t log_len = 0;            // entries of delta_log written by the last pr_run
    prgpu::DevState* st = nullptr;
    prgpu::DevState* st_host = nullptr;  // pinned
    int64_t launches = 0;
    pr_run_stats last{};
    cudaEvent_t fin_ev = nullptr;   // recorded at the end of every call (pr_destroy waits for it)
};

namespace prgpu {
// host_src: src / dst are pinned host arrays (single rank, m >= 2^22): copied
// in chunks that are sorted and merged while the rest is still in flight
int ingest(pr_graph* g, const int32_t* src, const int32_t* dst, Ctx& ctx, int rank = 0, int world = 1,
           bool host_src = false);
bool ingest_chunked_applies(int64_t n, int64_t m);
// cold_rows: slots past the 2^20 hottest in row order (this rank holds every
// row); false for a per-rank sharded create, whose slots must come out the
// same on every rank from the all-reduced out-degrees alone
int build_relabel(pr_graph* g, Ctx& ctx, bool cold_rows);
int build_view_stream(View& v, Ctx& ctx, int32_t pad_slot, const int32_t* outdeg, const int32_t* cidx);
int build_spans(View& v, Ctx& ctx, int64_t span_steps);
void free_spans(View& v, cudaStream_t s);
int build_phase_view(View& v, Ctx& ctx, int K, int32_t pad_slot);
void free_phase_view(View& v, cudaStream_t s);
int build_view_blocked(View& v, Ctx& ctx, int64_t n_contrib);
void free_view(View& v, cudaStream_t s);
__global__ void k_copy_rows(const int32_t* __restrict__ vid, int64_t nr, const int64_t* __restrict__ rp,
                            const int32_t* __restrict__ col, const int64_t* __restrict__ rpR, int32_t* __restrict__ colR);
__global__ void k_rinfo(const int32_t* __restrict__ vid, int64_t nrows, const int32_t* __restrict__ od,
                        const int32_t* __restrict__ cidx, int2* __restrict__ info);
int preprocess(pr_graph* g, uint32_t flags, Ctx& ctx);
int run(pr_graph* g, double d, double tau, int32_t max_iter, uint32_t mode, double* ranks,
        Ctx& ctx, int32_t* iters_out, double* delta_out);
int read_count(Ctx& ctx, const int64_t* dev, int64_t* host);
int build_shard(pr_graph* g, int rank, int world, Ctx& ctx, bool by_id = false);
void clear_shard(pr_graph* g, cudaStream_t s);
void clear_peers(pr_graph* g);
int set_peers(pr_graph* g, double* const* y0s, double* const* y1s, int world);
int device_barrier(pr_graph* g, Ctx& ctx);
int mc_create(pr_graph* g, void* handle_out);
int mc_attach(pr_graph* g, const void* handle);
int mc_bind(pr_graph* g, Ctx& ctx);
void clear_multicast(pr_graph* g);
int barrier_selftest(int world, int epochs, Ctx& ctx, int* bad_out);
int run_sharded(pr_graph* g, double d, double tau, int32_t max_iter, uint32_t mode, double* ranks, Ctx& ctx,
                pr_exchange_fn exchange, void* exchange_ctx, int32_t* iters_out, double* delta_out);
}  // namespace prgpu
