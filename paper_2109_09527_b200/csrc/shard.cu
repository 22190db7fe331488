// shard.cu -- row sharding of the synchronous pull iteration over P ranks
// ("1-D by destination rows ... balanced by nnz; each GPU
// holds its rows' in-CSR slice and a full replica of y; exchange per
// iteration: all-gather of y_t slices ... plus the two Delta scalars,
// piggy-backed on the all-gather payload").  DESIGN.md §10.
//
// Every rank builds the same canonical graph (ingest is deterministic), then
// pr_graph_shard(rank, world) derives, identically on every rank:
//   * owner[v]: contrib-carrying vertices (outdeg > 0) dealt round-robin in
//     compact slot (degree) order, so every rank
//     owns an equal share of the slots and of each degree class; dangling
//     vertices round-robin by id;
//   * the sharded contrib layout: [0, H) a copy of the H = 32K hottest contribs
//     (the gather's shared-memory and L1 tiers, refreshed after every exchange),
//     then rank r's contribs at H + [r*chunk, r*chunk + cnt_r), chunk = max cnt_r
//     + 2, the last two doubles of a chunk carrying that rank's (L1, Linf) of the
//     sweep; slot H + P*chunk is the +0.0 pad;
//   * this rank's view: its vertices of in-degree > 0 (vertex order), columns
//     remapped to the sharded slots; and its in-degree-0 vertices.
// A sweep (pr_run_sharded) gathers and finalizes the owned rows into the
// rank's chunk; ONE in-place all-gather of the chunks (a caller-supplied
// exchange, e.g. NCCL) then gives every rank the full next contrib vector and
// all P Delta pairs, which k_shard_combine sums in rank order (identical stop
// decision on every rank).
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "internal.h"
#include "primitives.cuh"

namespace prgpu {

static unsigned sh_grid(const Ctx& ctx, int64_t work) {
    const int64_t g = (work + 255) / 256;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)ctx.num_sms * 16));
}

// Ownership: contrib-carrying vertices by blocks of SH_BLOCK consecutive
// compact slots (degree order) dealt round-robin to the ranks, so every rank
// gets an equal share of the slots (the exchanged chunk) and of every degree
// class (the gathered edges); dangling vertices by id blocks, round-robin.
// One-slot blocks: R-MAT's top out-degree vertices are also its top in-degree
// rows, and 256-slot blocks left rank 0 with 1.25x the mean edges at P = 8
// (tools/shard_scaling.py).
constexpr int64_t SH_BLOCK = 1;

__device__ __forceinline__ int64_t sh_local(int64_t c, int P) {  // index of slot c inside its rank's chunk
    return (c / (SH_BLOCK * P)) * SH_BLOCK + c % SH_BLOCK;
}

// owner[v] and the sharded (chunk) slot of every contrib-carrying vertex
__global__ void k_sh_owner(const int32_t* __restrict__ cidx, int64_t n, int P, int64_t H, int64_t chunk,
                           int32_t* __restrict__ owner, int32_t* __restrict__ scidx) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = cidx[v];
        if (c >= 0) {
            const int r = (int)((c / SH_BLOCK) % P);
            owner[v] = r;
            scidx[v] = (int32_t)(H + r * chunk + sh_local(c, P));
        } else {
            owner[v] = (int32_t)((v / SH_BLOCK) % P);
            scidx[v] = -1;
        }
    }
}

// smap[c] = index the gather uses for compact slot c: the hot copy [0, H) for
// the H hottest, else the owner's chunk slot
__global__ void k_sh_smap(int64_t nc, int P, int64_t H, int64_t chunk, int32_t* __restrict__ smap,
                          int32_t* __restrict__ hot_src) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)((c / SH_BLOCK) % P);
        const int64_t cs = H + r * chunk + sh_local(c, P);
        smap[c] = (int32_t)(c < H ? c : cs);
        if (c < H) hot_src[c] = (int32_t)cs;
    }
}

__global__ void k_sh_map_col(int32_t* __restrict__ col, int64_t E, const int32_t* __restrict__ smap) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
        col[e] = smap[col[e]];
}

struct ShOwnGet {  // owned vertices with (rows) / without (zero list) in-edges
    const int32_t* owner;
    const int64_t* rp;
    int rank;
    bool rows;
    __device__ int64_t operator()(int64_t v) const {
        const bool has = rp[v + 1] > rp[v];
        return (owner[v] == rank && has == rows) ? 1 : 0;
    }
};
struct ShListEmit {
    int32_t* list;
    __device__ void operator()(int64_t v, int64_t pos, int64_t f) const {
        if (f) list[pos] = (int32_t)v;
    }
};
struct ShDegGet {
    const int64_t* rp;
    const int32_t* vid;
    int64_t nr;
    __device__ int64_t operator()(int64_t i) const {
        if (i >= nr) return 0;
        const int32_t v = vid[i];
        return rp[v + 1] - rp[v];
    }
};
struct ShPosEmit {
    int64_t* out;
    __device__ void operator()(int64_t i, int64_t pos, int64_t) const { out[i] = pos; }
};

// ---- id ownership (pr_graph_create_sharded): owner(v) = v mod P, for rows
// and contribs alike, so a rank can ingest only the edges into its vertices.
// A rank's contribs sit in its chunk in contrib (degree) order.
__global__ void k_sh_inv(const int32_t* __restrict__ cidx, int64_t n, int32_t* __restrict__ inv) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if (cidx[v] >= 0) inv[cidx[v]] = (int32_t)v;
}
__global__ void k_sh_idkeys(const int32_t* __restrict__ inv, int64_t nc, int P, uint64_t* __restrict__ keys) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x)
        keys[c] = ((uint64_t)(uint32_t)(inv[c] % P) << 32) | (uint64_t)c;
}
// first sorted position of every owner (start[P] = nc); keys sorted by owner
__global__ void k_sh_starts(const uint64_t* __restrict__ keys, int64_t nc, int P, int64_t* __restrict__ start) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(keys[i] >> 32);
        const int rp = i == 0 ? -1 : (int)(keys[i - 1] >> 32);
        for (int q = rp + 1; q <= r; ++q) start[q] = i;
        if (i == nc - 1)
            for (int q = r + 1; q <= P; ++q) start[q] = nc;
    }
}
__global__ void k_sh_owner_mod(int64_t n, int P, int32_t* __restrict__ owner, int32_t* __restrict__ scidx) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        owner[v] = (int32_t)(v % P);
        scidx[v] = -1;
    }
}
__global__ void k_sh_idslots(const uint64_t* __restrict__ keys, int64_t nc, const int64_t* __restrict__ start,
                             const int32_t* __restrict__ inv, int64_t H, int64_t chunk, int32_t* __restrict__ scidx,
                             int32_t* __restrict__ smap, int32_t* __restrict__ hot_src) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(keys[i] >> 32);
        const int64_t c = (int64_t)(keys[i] & 0xffffffffu);
        const int64_t cs = H + r * chunk + (i - start[r]);
        scidx[inv[c]] = (int32_t)cs;
        smap[c] = (int32_t)(c < H ? c : cs);
        if (c < H) hot_src[c] = (int32_t)cs;
    }
}

void clear_peers(pr_graph* g) {
    if (g->speer_dev) {
        cudaFree(g->speer_dev);
        g->speer_dev = nullptr;
    }
    for (void* p : g->speer_ipc)
        if (p) cudaIpcCloseMemHandle(p);
    g->speer_ipc.clear();
}

void clear_shard(pr_graph* g, cudaStream_t s) {
    free_view(g->shard, s);
    dfree(g->sowner, s);
    dfree(g->scidx, s);
    dfree(g->szlist, s);
    dfree(g->shot_src, s);
    g->shard_hot = 0;
    clear_peers(g);
    for (int b = 0; b < 2; ++b)
        if (g->sy[b]) {
            cudaStreamSynchronize(s);
            cudaFree(g->sy[b]);
            g->sy[b] = nullptr;
        }
    g->shard_rank = -1;
    g->shard_world = 0;
    g->shard_chunk = 0;
    g->snz = 0;
    g->shard_owned = 0;
}

int build_shard(pr_graph* g, int rank, int world, Ctx& ctx, bool by_id) {
    cudaStream_t s = ctx.stream;
    clear_shard(g, s);
    const int64_t n = g->n, nc = g->n_contrib;
    TmpGuard tg_(s);
    int32_t* smap = nullptr;
    int64_t* cnt = nullptr;
    int32_t* inv = nullptr;
    uint64_t* keys = nullptr;
    uint64_t* keys_alt = nullptr;
    int64_t* start = nullptr;
    tg_.track(smap);
    tg_.track(cnt);
    tg_.track(inv);
    tg_.track(keys);
    tg_.track(keys_alt);
    tg_.track(start);
    PR_TRY(dalloc(&cnt, 2, s));
    const int64_t H = std::min<int64_t>(SE_L1_TIER, nc);  // hot copy: the smem and L1 tiers of the gather
    PR_TRY(dalloc(&g->sowner, (size_t)n, s));
    PR_TRY(dalloc(&g->scidx, (size_t)n, s));
    if (nc > 0) {
        PR_TRY(dalloc(&smap, (size_t)nc, s));
        PR_TRY(dalloc(&g->shot_src, (size_t)std::max<int64_t>(H, 1), s));
    }
    int64_t chunk = 2;
    if (!by_id) {
        // chunk = most slots any rank owns, + (L1, Linf)
        const int64_t nb = (nc + SH_BLOCK - 1) / SH_BLOCK;
        int64_t cmax = 0;
        for (int r = 0; r < world && r < nb; ++r) {
            const int64_t blocks = (nb - r + world - 1) / world;  // blocks r, r + world, ...
            int64_t cr = blocks * SH_BLOCK;
            if ((nb - 1) % world == r) cr -= nb * SH_BLOCK - nc;  // the last block is partial
            cmax = std::max(cmax, cr);
        }
        chunk = cmax + 2;
        if (H + (int64_t)world * chunk + 1 > INT32_MAX) {
            set_error("pr_graph_shard: sharded contrib layout exceeds int32 slots");
            return PR_EINVAL;
        }
        PR_LAUNCH(ctx, k_sh_owner, sh_grid(ctx, n), 256, 0, (const int32_t*)g->cidx, n, world, H, chunk, g->sowner,
                  g->scidx);
        if (nc > 0) PR_LAUNCH(ctx, k_sh_smap, sh_grid(ctx, nc), 256, 0, nc, world, H, chunk, smap, g->shot_src);
    } else {
        // owner(v) = v mod P; a rank's contribs in contrib order inside its chunk:
        // sort the contrib slots by owner (stable: slots stay ascending)
        PR_LAUNCH(ctx, k_sh_owner_mod, sh_grid(ctx, n), 256, 0, n, world, g->sowner, g->scidx);
        std::vector<int64_t> hs(world + 1, 0);
        if (nc > 0) {
            PR_TRY(dalloc(&inv, (size_t)nc, s));
            PR_TRY(dalloc(&keys, (size_t)nc, s));
            PR_TRY(dalloc(&keys_alt, (size_t)nc, s));
            PR_TRY(dalloc(&start, (size_t)world + 1, s));
            PR_LAUNCH(ctx, k_sh_inv, sh_grid(ctx, n), 256, 0, (const int32_t*)g->cidx, n, inv);
            PR_LAUNCH(ctx, k_sh_idkeys, sh_grid(ctx, nc), 256, 0, (const int32_t*)inv, nc, world, keys);
            bool alt = false;
            if (world > 1)
                PR_TRY((radix_sort<uint64_t, false>(ctx, keys, keys_alt, nullptr, nullptr, nc, 32,
                                                    32 + bits_for((uint64_t)(world - 1)), &alt)));
            const uint64_t* sk = alt ? keys_alt : keys;
            PR_LAUNCH(ctx, k_sh_starts, sh_grid(ctx, nc), 256, 0, sk, nc, world, start);
            PR_CUDA(cudaMemcpyAsync(hs.data(), start, sizeof(int64_t) * (size_t)(world + 1), cudaMemcpyDeviceToHost, s));
            PR_CUDA(cudaStreamSynchronize(s));
            int64_t cmax = 0;
            for (int r = 0; r < world; ++r) cmax = std::max(cmax, hs[r + 1] - hs[r]);
            chunk = cmax + 2;
            if (H + (int64_t)world * chunk + 1 > INT32_MAX) {
                set_error("pr_graph_create_sharded: sharded contrib layout exceeds int32 slots");
                return PR_EINVAL;
            }
            PR_LAUNCH(ctx, k_sh_idslots, sh_grid(ctx, nc), 256, 0, sk, nc, (const int64_t*)start,
                      (const int32_t*)inv, H, chunk, g->scidx, smap, g->shot_src);
        }
    }

    // owned rows (vertex order) and owned in-degree-0 vertices
    View& S = g->shard;
    S = View{};
    PR_TRY(dalloc(&S.vid, (size_t)std::max<int64_t>(n, 1), s));
    PR_TRY((device_scan<int64_t>(ctx, n, ShOwnGet{g->sowner, g->row_ptr, rank, true}, ShListEmit{S.vid}, cnt)));
    PR_TRY(read_count(ctx, cnt, &S.nrows));
    PR_TRY(dalloc(&g->szlist, (size_t)std::max<int64_t>(n, 1), s));
    PR_TRY((device_scan<int64_t>(ctx, n, ShOwnGet{g->sowner, g->row_ptr, rank, false}, ShListEmit{g->szlist}, cnt)));
    PR_TRY(read_count(ctx, cnt, &g->snz));
    g->shard_owned = S.nrows + g->snz;

    PR_TRY(dalloc(&S.row_ptr, (size_t)S.nrows + 1, s));
    S.owns_row_ptr = true;
    PR_TRY((device_scan<int64_t>(ctx, S.nrows + 1, ShDegGet{g->row_ptr, S.vid, S.nrows}, ShPosEmit{S.row_ptr}, cnt)));
    PR_TRY(read_count(ctx, cnt, &S.nedges));
    PR_TRY(dalloc(&S.col, (size_t)stream_pad(S.nedges), s));
    if (S.nrows > 0) {
        const unsigned gc = (unsigned)std::max<int64_t>(
            1, std::min<int64_t>((S.nedges + 1023) / 1024 * 32 / 256 + 1, (int64_t)ctx.num_sms * 8));
        PR_LAUNCH(ctx, k_copy_rows, gc, 256, 0, (const int32_t*)S.vid, S.nrows, (const int64_t*)g->row_ptr,
                  (const int32_t*)g->plain.col, (const int64_t*)S.row_ptr, S.col);
        PR_LAUNCH(ctx, k_sh_map_col, sh_grid(ctx, S.nedges), 256, 0, S.col, S.nedges, (const int32_t*)smap);
    }
    PR_TRY(build_view_stream(S, ctx, (int32_t)(H + (int64_t)world * chunk), g->outdeg, g->scidx));
    const int64_t ny = H + (int64_t)world * chunk + 1;
    for (int b = 0; b < 2; ++b) {  // plain cudaMalloc: exportable by cudaIpcGetMemHandle (pr_shard_export_ipc)
        PR_CUDA(cudaMalloc(&g->sy[b], sizeof(double) * (size_t)ny));
        PR_CUDA(cudaMemsetAsync(g->sy[b], 0, sizeof(double) * (size_t)ny, s));
    }
    g->shard_rank = rank;
    g->shard_world = world;
    g->shard_chunk = chunk;
    g->shard_hot = H;
    return PR_OK;
}

// Peer buffers: y0s[r] / y1s[r] = rank r's sy[0] / sy[1] as addressable from
// this device (same device, peer access or IPC-opened); entry [rank] unused.
int set_peers(pr_graph* g, double* const* y0s, double* const* y1s, int world) {
    if (g->speer_dev) {
        cudaFree(g->speer_dev);
        g->speer_dev = nullptr;
    }
    if (world <= 1) return PR_OK;
    std::vector<double*> h(2 * (size_t)(world - 1));
    int q = 0;
    for (int r = 0; r < world; ++r) {
        if (r == g->shard_rank) continue;
        h[q] = y0s[r];
        h[(world - 1) + q] = y1s[r];
        ++q;
    }
    PR_CUDA(cudaMalloc(&g->speer_dev, sizeof(double*) * h.size()));
    PR_CUDA(cudaMemcpy(g->speer_dev, h.data(), sizeof(double*) * h.size(), cudaMemcpyHostToDevice));
    return PR_OK;
}

}  // namespace prgpu
