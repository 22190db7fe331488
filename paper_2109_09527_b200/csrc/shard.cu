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
    if (g->speer_flags) {
        cudaFree(g->speer_flags);
        g->speer_flags = nullptr;
    }
    g->sdev_barrier = false;
    for (void* p : g->speer_ipc)
        if (p) cudaIpcCloseMemHandle(p);
    g->speer_ipc.clear();
}

void clear_shard(pr_graph* g, cudaStream_t s) {
    clear_multicast(g);  // (its buffers are sy[0], sy[1])
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
    // plain cudaMalloc: exportable by cudaIpcGetMemHandle (pr_shard_export_ipc);
    // sy[0] carries `world` uint64 arrival flags of the device-side peer
    // barrier after its ny doubles (slot r written by rank r)
    for (int b = 0; b < 2; ++b) {
        const int64_t cnt = ny + (b == 0 ? world : 0);
        PR_CUDA(cudaMalloc(&g->sy[b], sizeof(double) * (size_t)cnt));
        PR_CUDA(cudaMemsetAsync(g->sy[b], 0, sizeof(double) * (size_t)cnt, s));
    }
    g->bar_epoch = 0;
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
    if (g->speer_flags) {
        cudaFree(g->speer_flags);
        g->speer_flags = nullptr;
    }
    if (world <= 1) return PR_OK;
    const int64_t ny = g->shard_hot + (int64_t)g->shard_world * g->shard_chunk + 1;
    std::vector<double*> h(2 * (size_t)(world - 1));
    std::vector<unsigned long long*> f(world - 1);
    int q = 0;
    for (int r = 0; r < world; ++r) {
        if (r == g->shard_rank) continue;
        h[q] = y0s[r];
        h[(world - 1) + q] = y1s[r];
        f[q] = reinterpret_cast<unsigned long long*>(y0s[r] + ny);  // rank r's arrival flags
        ++q;
    }
    PR_CUDA(cudaMalloc(&g->speer_dev, sizeof(double*) * h.size()));
    PR_CUDA(cudaMemcpy(g->speer_dev, h.data(), sizeof(double*) * h.size(), cudaMemcpyHostToDevice));
    PR_CUDA(cudaMalloc(&g->speer_flags, sizeof(unsigned long long*) * f.size()));
    PR_CUDA(cudaMemcpy(g->speer_flags, f.data(), sizeof(unsigned long long*) * f.size(), cudaMemcpyHostToDevice));
    return PR_OK;
}

// ---- device-side peer barrier (the exchange's per-sweep synchronisation
// without the host): rank r stores `epoch` into slot r of every peer's
// arrival flags (release, system scope), then waits until every peer has
// stored it into its own flags (acquire).  Every write the rank's earlier
// kernels made (stream order: they happen before this kernel) -- the peer
// stores of K-FINALIZE in particular -- is visible to a peer that has seen the
// flag.  Epochs only grow (every rank runs the same sequence of barriers), so
// the flags never need resetting.  A wait longer than ~20 s sets *err and
// returns (no hang on a dead peer).
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ bool peer_barrier(unsigned long long* mine, unsigned long long* const* peers, const int* peer_rank, int npeer,
                             int rank, unsigned long long epoch) {
    __threadfence_system();
    for (int q = 0; q < npeer; ++q) st_release_sys_u64(peers[q] + rank, epoch);
    const long long t0 = clock64();
    for (int q = 0; q < npeer; ++q) {
        const int r = peer_rank[q];
        while (ld_acquire_sys_u64(mine + r) < epoch) {
            if (clock64() - t0 > 40000000000ll) return false;  // ~20 s at 2 GHz
            __nanosleep(64);
        }
    }
    __threadfence_system();
    return true;
}
__global__ void k_peer_barrier(unsigned long long* mine, unsigned long long* const* peers, int npeer, int rank,
                               int world, unsigned long long epoch, int* err) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int prank[64];
    int q = 0;
    for (int r = 0; r < world && q < 64; ++r)
        if (r != rank) prank[q++] = r;
    if (!peer_barrier(mine, peers, prank, npeer, rank, epoch)) atomicExch(err, 1);
}
// NVLS form: ONE multimem store of the epoch into slot `rank` of every team
// member's flags (the multicast address of the flags), then the same wait.
__global__ void k_mc_barrier(unsigned long long* mine, unsigned long long* mc_flags, int rank, int world,
                             unsigned long long epoch, int* err) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    __threadfence_system();
    asm volatile("multimem.st.release.sys.global.u64 [%0], %1;" ::"l"(mc_flags + rank), "l"(epoch) : "memory");
    const long long t0 = clock64();
    for (int r = 0; r < world; ++r) {
        if (r == rank) continue;
        while (ld_acquire_sys_u64(mine + r) < epoch) {
            if (clock64() - t0 > 40000000000ll) {
                atomicExch(err, 1);
                return;
            }
            __nanosleep(64);
        }
    }
    __threadfence_system();
}

int device_barrier(pr_graph* g, Ctx& ctx) {
    const int world = g->shard_world;
    if (world > 1 && g->mc && g->mc->bound) {
        const int64_t ny = g->shard_hot + (int64_t)world * g->shard_chunk + 1;
        g->bar_epoch += 1;
        PR_LAUNCH(ctx, k_mc_barrier, 1, 32, 0, reinterpret_cast<unsigned long long*>(g->sy[0] + ny),
                  reinterpret_cast<unsigned long long*>(g->mc->y[0] + ny), g->shard_rank, world,
                  (unsigned long long)g->bar_epoch, &g->st->peer_err);
        return PR_OK;
    }
    if (world <= 1 || !g->speer_flags) return PR_OK;
    if (world > 65) {
        set_error("device peer barrier: world %d > 65", world);
        return PR_EINVAL;
    }
    const int64_t ny = g->shard_hot + (int64_t)world * g->shard_chunk + 1;
    g->bar_epoch += 1;
    PR_LAUNCH(ctx, k_peer_barrier, 1, 32, 0, reinterpret_cast<unsigned long long*>(g->sy[0] + ny),
              (unsigned long long* const*)g->speer_flags, world - 1, g->shard_rank, world,
              (unsigned long long)g->bar_epoch, &g->st->peer_err);
    return PR_OK;
}

// Self-test of the barrier protocol on one GPU: the guide forbids separate
// launches that wait on one another, so `world` emulated ranks are the blocks
// of ONE cooperative launch (co-resident by construction), each running the
// same peer_barrier over its own flag array; per epoch every block writes its
// value, passes the barrier and checks every other block's value of that
// epoch (two parities: a block can only overwrite parity p after the next
// barrier, which every reader of p has passed).  *bad counts mismatches and
// timeouts.
__global__ void k_barrier_selftest(unsigned long long* flags, double* data, int world, int epochs, int* bad) {
    const int r = blockIdx.x;
    if (threadIdx.x != 0) return;
    unsigned long long* peers[64];
    int prank[64];
    int q = 0;
    for (int o = 0; o < world; ++o)
        if (o != r) {
            peers[q] = flags + (int64_t)o * world;
            prank[q] = o;
            ++q;
        }
    for (int e = 1; e <= epochs; ++e) {
        double* d = data + (int64_t)(e & 1) * world;
        d[r] = (double)e * 1000.0 + r;
        if (!peer_barrier(flags + (int64_t)r * world, peers, prank, world - 1, r, (unsigned long long)e)) {
            atomicAdd(bad, 1000000);
            return;
        }
        for (int o = 0; o < world; ++o) {
            const double v = *(volatile double*)(d + o);
            if (v != (double)e * 1000.0 + o) atomicAdd(bad, 1);
        }
    }
}

int barrier_selftest(int world, int epochs, Ctx& ctx, int* bad_out) {
    if (world < 1 || world > 64 || epochs < 1) {
        set_error("pr_selftest_peer_barrier: world in [1, 64], epochs >= 1");
        return PR_EINVAL;
    }
    int dev = 0, coop = 0, sms = 0;
    PR_CUDA(cudaGetDevice(&dev));
    PR_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    PR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (!coop || world > sms) {
        set_error("pr_selftest_peer_barrier: no cooperative launch of %d blocks on this device", world);
        return PR_ECUDA;
    }
    unsigned long long* flags = nullptr;
    double* data = nullptr;
    int* bad = nullptr;
    TmpGuard tg_(ctx.stream);
    tg_.track(flags);
    tg_.track(data);
    tg_.track(bad);
    PR_TRY(dalloc(&flags, (size_t)world * world, ctx.stream));
    PR_TRY(dalloc(&data, 2 * (size_t)world, ctx.stream));
    PR_TRY(dalloc(&bad, 1, ctx.stream));
    PR_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned long long) * (size_t)world * world, ctx.stream));
    PR_CUDA(cudaMemsetAsync(data, 0, sizeof(double) * 2 * (size_t)world, ctx.stream));
    PR_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx.stream));
    void* args[] = {&flags, &data, &world, &epochs, &bad};
    PR_CUDA(cudaLaunchCooperativeKernel((const void*)k_barrier_selftest, dim3(world), dim3(32), args, 0, ctx.stream));
    ctx.launches += 1;
    PR_CUDA(cudaMemcpyAsync(bad_out, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    return PR_OK;
}

}  // namespace prgpu
