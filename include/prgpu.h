/*
 * prgpu.h -- C ABI of libprgpu: the synchronous (and optional No-Sync-style
 * asynchronous) fp64 PageRank pull iteration of arXiv 2109.09527 on one B200.
 *
 * Citations: "P:N" = PAPER.md line N (section / equation / algorithm named),
 * "S:N" = SPEC.md line N, "Q-x" = a reading of the paper listed in DESIGN.md.
 *
 * What is computed (Eq.(1)):
 *     pr(v) = (1-d)/n + d * sum_{(u,v) in E} pr(u)/outdeg(u)
 * iterated from pr = 1/n (Alg.1) "while err > threshold" with
 * err = the L1 (default; BASELINE configs) or L-inf norm of
 * the change over one sweep, reset every sweep (Q-E).  Dangling vertices
 * (outdeg 0) contribute nothing and nothing is redistributed (Alg.2 P:489-491;
 * Q-D).  Self-loops and duplicate edges are removed when the graph is built
 * (Q-L).
 *
 * Conventions for every call:
 *  - Pointers may be device pointers or host pointers (pageable or pinned);
 *    the library detects which with CUDA unified addressing and copies host
 *    data inside the call.  Pointer arguments are never retained after return.
 *  - `stream` is a cudaStream_t passed as void* (NULL = the legacy default
 *    stream).  All device work of a call is ordered on that stream.
 *  - Return values are PR_* status codes; on any status other than PR_OK and
 *    PR_NOT_CONVERGED, pr_last_error() returns a message (thread-local, valid
 *    until the next call from the same thread).  The library never aborts and
 *    never throws across the ABI.
 *  - One pr_graph is used by one stream at a time; distinct graphs are
 *    independent.
 */
#ifndef PRGPU_H
#define PRGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pr_graph pr_graph;     /* opaque; owned by the library */

/* Status codes (mirror the CLI exit-code convention of SPEC S:483). */
#define PR_OK             0   /* converged / success */
#define PR_EINVAL         1   /* invalid argument (ids out of range, d not in (0,1), ...) */
#define PR_NOT_CONVERGED  2   /* max_iter reached; ranks and iterations still written */
#define PR_ESTATE         3   /* call not valid in the graph's state (e.g. reductions not built) */
#define PR_ENOMEM        (-1) /* device or host allocation failed */
#define PR_ECUDA         (-2) /* a CUDA runtime error; see pr_last_error() */

/* pr_preprocess flags */
#define PR_PRE_IDENTICAL  1u  /* identical in-neighbour groups (STIC-D, §3) */
#define PR_PRE_CHAIN      2u  /* chains of in=1/out=1 vertices (STIC-D, §3; Q-C) */

/* pr_run mode bits */
#define PR_MODE_SYNC      0u  /* synchronous pull, double-buffered contribs (Alg.1) */
#define PR_MODE_ASYNC     1u  /* in-place No-Sync-style sweeps (Alg.3; Q-Y); on a
                                 source-blocked view (contrib vector beyond L2) the Jacobi
                                 schedule, a valid No-Sync schedule (Q-Y2) */
#define PR_NORM_L1        0u  /* stop when sum_v |x_t(v)-x_{t-1}(v)| <= threshold (configs) */
#define PR_NORM_LINF      2u  /* stop when max_v |x_t(v)-x_{t-1}(v)| <= threshold */
#define PR_USE_REDUCTIONS 4u  /* compute one vertex per identical group, resolve chain
                                 members from their head; needs pr_preprocess */
#define PR_TIMING         8u  /* record CUDA events around the gather / finalize launches of
                                 every 4th sweep (PRGPU_TIMING_STRIDE; bench roofline) */
#define PR_MODE_NOSYNC   16u  /* persistent barrier-free No-Sync kernel with thread-level
                                 (here: CTA-level) convergence (Alg.3 P:535-565, P:416-418;
                                 SURVEY f1): one launch, every CTA sweeps its own static work
                                 in place until the sum (L1) / max (L-inf) of the deltas the
                                 CTAs last published is <= threshold; then the residual
                                 ||F(x) - x|| of the ORIGINAL system is certified by one
                                 synchronous gather and the kernel is relaunched if it is
                                 above threshold.  iterations = the largest number of local
                                 sweeps of any CTA.  On a source-blocked view: launch-level
                                 sweeps on the Jacobi schedule, then the same certificate
                                 (Q-Y2). */
#define PR_PERFORATE     32u  /* loop perforation (Alg.5), plain view
                                 only: a vertex whose change in a sweep is
                                 0 < |delta| < threshold * 1e-5 gets Alg.5's sticky
                                 threshold_check flag and keeps its value from the next sweep
                                 on; flagged rows are compacted out of the gather at batch
                                 ends (performance only) (APPROXIMATE: the result is not the
                                 fixed point; the stop test counts frozen vertices as 0).
                                 Alone: synchronous sweeps (Barriers-Opt).  With
                                 PR_MODE_ASYNC: in-place sweeps.  With PR_MODE_NOSYNC
                                 (No-Sync-Opt): persistent barrier-free launches of <= 8
                                 local sweeps per CTA with the CTA-level stop test, no
                                 certificate (iterations = the sum over launches of the
                                 largest local count; final delta = the published sum). */
#define PR_CHAIN_EAGER  128u  /* with PR_USE_REDUCTIONS in the synchronous mode: resolve chain
                                 members in the SAME sweep from their head's new value (reading
                                 Q-C as first written; information crosses a chain in one sweep,
                                 but the sweep no longer conserves the plain iteration's
                                 invariants, e.g. sum(x) = 1 without dangling vertices).  Default
                                 (delayed, reading Q-C2): x_t(v_k) = alpha_j + beta_j *
                                 x_{t-j}(source), j = min(k, t) -- Eq.(1) unrolled along the chain,
                                 so the reduced sweep reproduces the plain (Jacobi) trajectory
                                 while still gathering no chain member.  The phased, async and
                                 No-Sync modes always resolve members eagerly (in place). */
#define PR_MODE_PHASED   64u  /* block Gauss-Seidel in K ordered, ROW-ALIGNED phases (Q-B):
                                 one contrib buffer; the rows of the view (vertex order) are
                                 cut at b_k = the first row whose first edge e has
                                 e * K >= k * E; phase k gathers its rows from the values
                                 phases 0..k-1 of the same sweep wrote and updates them in
                                 place (the in-place reads of Alg.3 P:545-565 in a fixed
                                 order); members (eager, Q-C) and, in sweep 1, the in-degree-0
                                 vertices after the last phase.  Deterministic; equals the
                                 oracle's block Gauss-Seidel with the same K.  K = PRGPU_PHASES
                                 (default: 8 when each phase still has >= 24 edge steps of
                                 256 per resident warp, fewer on small graphs; one phase on a
                                 source-blocked view).  Exclusive with ASYNC / NOSYNC /
                                 PERFORATE. */

/*
 * pr_graph_create -- build the in-edge CSR and out-degrees on the device
 * (§5.2 "converted later to Compressed Sparse Row (CSR) format";
 * Alg.1 P:433 "CSR representation").
 *   n      number of vertices, 1 <= n <= 2^31-1 (dense 0-based ids, Q-V)
 *   m      number of raw edges, 0 <= m <= 2^31-1
 *   src,dst  int32[m] raw edge list (src -> dst); duplicates and self-loops
 *          allowed (removed here).  Host or device memory; read only.  Pinned
 *          host arrays with m >= 2^22 are copied in chunks on a stream of the
 *          library's own, each chunk sorted while the next ones are in
 *          flight; the call returns after the last copy (the caller may then
 *          reuse the arrays).
 *   out    receives the new graph (NULL on failure)
 * Result: row_ptr int64[n+1], col_idx int32[E] (sources of each row sorted
 * ascending), outdeg int32[n], all bit-exact functions of the edge set.
 * Synchronises `stream` once (to learn E).
 * Errors: PR_EINVAL for n/m out of range, NULL pointers with m > 0, or any id
 * outside [0,n) (detected on the device; no graph is created).
 */
int pr_graph_create(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                    void *stream, pr_graph **out);

/*
 * pr_preprocess -- find the STIC-D work-saving structure (§3):
 *   PR_PRE_IDENTICAL: rep[v] = min id of the class of vertices with the same
 *       in-neighbour set; the empty in-set is one class (Q-G).
 *   PR_PRE_CHAIN: chain vertex <=> in-degree 1 and out-degree 1; members are
 *       the chain vertices at distance k >= 1 from a head h (chain(h) and not
 *       chain(pred(h))); their source is rep(h); pure cycles are excluded (Q-C).
 * Calling again replaces the previous result.  flags == 0 clears it.
 * Synchronises `stream` a few times (counts).  Errors: PR_EINVAL (NULL g or
 * unknown flag bits).
 */
int pr_preprocess(pr_graph *g, uint32_t flags, void *stream);

/*
 * pr_run -- iterate to convergence.
 *   d          damping, 0 < d < 1 ("initialized to 0.85")
 *   threshold  >= 0 (P:438 uses 1e-16 with L-inf; configs use 1e-10 / 1e-12 L1)
 *   max_iter   >= 1; reaching it returns PR_NOT_CONVERGED with valid ranks
 *   mode       one of PR_MODE_SYNC (0) / PR_MODE_ASYNC / PR_MODE_NOSYNC /
 *              PR_MODE_PHASED, or'ed
 *              with PR_NORM_LINF, PR_USE_REDUCTIONS, PR_TIMING; PR_PERFORATE with
 *              SYNC / ASYNC / NOSYNC on the plain view
 *   ranks      fp64[n] output in vertex-id order (host or device, caller-owned)
 *   iters_out  (host, nullable) number of update sweeps including the final
 *              one that met the stop test (Q-I); PR_MODE_NOSYNC: the
 *              largest number of local sweeps of any CTA
 *   final_delta_out (host, nullable) the stop-test norm of the last sweep;
 *              PR_MODE_NOSYNC: the certified ||F(x) - x||
 * Sync and phased modes are deterministic (fixed-order reductions): identical
 * inputs give bit-identical ranks and iteration counts.  The async and No-Sync modes are
 * not deterministic; they reach the same fixed point (Lemma 2).
 * PR_PERFORATE is approximate (Alg.5): frozen vertices keep their value.
 * Errors: PR_EINVAL (bad d / threshold / max_iter / NULL ranks / unknown or
 * incompatible mode bits), PR_ESTATE (PR_USE_REDUCTIONS before pr_preprocess).
 */
int pr_run(pr_graph *g, double d, double threshold, int32_t max_iter, void *stream,
           uint32_t mode, double *ranks, int32_t *iters_out, double *final_delta_out);

/* pr_destroy -- release every device buffer of g.  NULL-safe.  Waits for the
 * work the last call on g enqueued (on whatever stream it used) to finish, then
 * returns the buffers to the library's memory pool. */
void pr_destroy(pr_graph *g);

/* pr_release_memory -- return the device memory the library's private pool
 * keeps for reuse (all library allocations come from that pool, never from the
 * process's default pool; freed blocks stay reserved in it so a later
 * pr_graph_create does not map memory mid-call) to the device.  Synchronises
 * the device.  Safe with live graphs (only unused blocks are released).
 * Returns PR_OK or PR_ECUDA. */
int pr_release_memory(void);

/* pr_last_error -- message for the last failing call on this thread ("" if none). */
const char *pr_last_error(void);

/* ---- introspection (tests, bench) ------------------------------------- */

/* Sizes: n, E (deduplicated edges), number of member vertices resolved by
 * scatter in reduced mode (identical non-representatives + chain members),
 * longest chain distance k.  Any output pointer may be NULL. */
int pr_graph_info(const pr_graph *g, int64_t *n, int64_t *E, int64_t *n_members,
                  int32_t *max_chain);

/* Copy the canonical in-CSR into caller buffers (host or device):
 * row_ptr int64[n+1], col_idx int32[E], outdeg int32[n].  Any may be NULL. */
int pr_get_csr(const pr_graph *g, int64_t *row_ptr, int32_t *col_idx, int32_t *outdeg,
               void *stream);

/* Copy the reductions: rep int32[n] (identity if identical groups were not
 * requested), chain_src int32[n] (rep(head) or -1), chain_k int32[n] (k or 0).
 * PR_ESTATE before pr_preprocess.  Any may be NULL. */
int pr_get_reductions(const pr_graph *g, int32_t *rep, int32_t *chain_src, int32_t *chain_k,
                      void *stream);

/* Per-sweep (L1, L-inf) deltas of the last pr_run: writes min(cap, iters)
 * pairs into host buffer log[2*cap]; returns the number of pairs written
 * (>= 0), or on error a negative value (-PR_EINVAL, PR_ECUDA) with the
 * message in pr_last_error(). */
int pr_get_delta_log(const pr_graph *g, double *log, int32_t cap);

/* Statistics of the last pr_run (and of the graph's lifetime). */
typedef struct {
    int32_t iterations;         /* sweeps performed (== *iters_out) */
    int32_t status;             /* PR_OK or PR_NOT_CONVERGED */
    double  delta_l1;           /* last sweep's L1 delta */
    double  delta_linf;         /* last sweep's L-inf delta */
    int64_t run_launches;       /* kernels launched by the last pr_run (incl. early-exit ones) */
    int64_t total_launches;     /* kernels launched for this graph since pr_graph_create */
    int32_t host_syncs;         /* stream synchronisations inside the last pr_run */
    int32_t timed_iterations;   /* PR_TIMING: sweeps timed */
    double  gather_ms;          /* PR_TIMING: summed CUDA-event time of the gather launches
                                   (K-GATHER; in-place modes: the whole fused sweep) */
    double  scatter_ms;         /* PR_TIMING: summed time of the launches after the gather:
                                   K-FINALIZE in sync mode (rows + members), 0 in place */
    int64_t gather_rows;        /* rows one gather launch processes (in-degree > 0: all, or |R| reduced) */
    int64_t gather_edges;       /* edges one gather launch processes */
    int64_t scatter_members;    /* members one scatter launch processes (0 plain) */
    int64_t n_contrib;          /* vertices with outdeg > 0 (size of the contrib vector) */
    int64_t n_tasks;            /* reserved: always 0 (the round-1 row-task engine was removed) */
    int32_t nosync_min_iters;   /* PR_MODE_NOSYNC: fewest local sweeps of any CTA */
    int32_t nosync_launches;    /* PR_MODE_NOSYNC: persistent launches (1 + relaunches) */
    int32_t nosync_median_iters;/* PR_MODE_NOSYNC: median local sweeps over the CTAs (the max
                                   usually belongs to the least-loaded CTA, which sweeps its
                                   short share more often) */
    double  residual;           /* PR_MODE_NOSYNC: certified ||F(x) - x|| (run norm) at exit */
    int64_t edges_gathered;     /* edges gathered over the whole run (all sweeps) */
    int64_t frozen_rows;        /* PR_PERFORATE: rows no longer gathered at exit */
    int32_t compactions;        /* PR_PERFORATE: times the gathered rows were compacted */
    int32_t phases;             /* phases per sweep (PR_MODE_PHASED: K; else 1) */
} pr_run_stats;

int pr_get_run_stats(const pr_graph *g, pr_run_stats *out);

/*
 * pr_get_phase_plan -- the phase plan of the last PR_MODE_PHASED run on the
 * plain (reduced = 0) or reduced view (Q-B): phase k gathers and updates the
 * view rows [row_bounds[k], row_bounds[k+1]) (the view's rows in vertex order),
 * whose in-edges are the view's edges [edge_bounds[k], edge_bounds[k+1]) (each
 * row's in-edges in CSR order).  Host arrays of cap >= K+1 entries.
 * Returns K >= 1, or on error a negative value (-PR_EINVAL: bad arguments or
 * cap; -PR_ESTATE: no phased run on that view yet) with the message in
 * pr_last_error().
 */
int pr_get_phase_plan(const pr_graph *g, int32_t reduced, int64_t *edge_bounds, int64_t *row_bounds,
                      int32_t cap);

/*
 * ---- Row sharding over P ranks ----
 * The sync pull iteration split by destination rows: every rank holds the
 * in-edges of the vertices it owns and a full replica of the contrib vector;
 * after each sweep ONE in-place all-gather of fixed-size per-rank chunks
 * (owned contribs + that rank's (L1, L-inf) delta) gives every rank the next
 * contrib vector and all deltas, summed in rank order for an identical stop
 * decision.  The paper has no multi-device form; the sweep is Eq.(1)
 * over the owned rows, exactly as in pr_run.
 *
 * pr_exchange_fn -- caller-supplied exchange: on `stream`, all-gather IN PLACE
 * the `world` chunks of `chunk` doubles of the device buffer `buf`
 * (world * chunk doubles; this rank's chunk, at rank * chunk, is filled when
 * the call is made, ordered on `stream`).  Called once per sweep from the
 * host thread running pr_run_sharded, before the rank-order delta reduction
 * is enqueued.  Returns 0, or nonzero to abort the run with PR_ECUDA.
 */
typedef int (*pr_exchange_fn)(void *ctx, double *buf, int64_t chunk, int32_t world, void *stream);

/*
 * pr_allreduce_fn -- caller-supplied sum all-reduce, in place, of `count` int32
 * values of the device buffer `buf` over the `world` ranks, ordered on
 * `stream` (e.g. torch.distributed / NCCL all_reduce).  Returns 0, or nonzero
 * to abort with PR_ECUDA.
 */
typedef int (*pr_allreduce_fn)(void *ctx, int32_t *buf, int64_t count, int32_t world, void *stream);

/*
 * pr_graph_create_sharded -- build ONLY this rank's share of a world-rank row
 * partition straight from the raw edge list (the same list on every rank,
 * host or device, as pr_graph_create): vertex v is owned by rank v mod world,
 * rows and contribs alike; the rank sorts and deduplicates only the edges into
 * its vertices (1/world of them), sums the partial out-degrees with one
 * `allreduce` over n int32 (every deduplicated edge lives on exactly one rank:
 * the owner of its dst), then derives the contrib order and the sharded layout
 * identically on every rank (a rank's contribs sit in its chunk in contrib
 * order).  Must be called on every rank (the all-reduce is collective).  The
 * graph is for pr_run_sharded / pr_get_shard_info / the peer calls only:
 * pr_run, pr_preprocess and pr_graph_shard return PR_ESTATE; pr_graph_info's
 * E and pr_get_csr describe the rank's edges (rows of other ranks' vertices
 * are empty).  world = 1 equals pr_graph_create + pr_graph_shard(0, 1).
 * Errors as pr_graph_create, plus PR_EINVAL for a bad rank / world or a NULL
 * allreduce and PR_ECUDA when the all-reduce fails.
 */
int pr_graph_create_sharded(int64_t n, int64_t m, const int32_t *src, const int32_t *dst, int32_t rank,
                            int32_t world, pr_allreduce_fn allreduce, void *allreduce_ctx, void *stream,
                            pr_graph **out);

/*
 * pr_graph_shard -- make g (created from the SAME edge list on every rank) the
 * rank's share of a world-rank row partition: contrib-carrying vertices are
 * dealt round-robin in the internal contrib (out-degree) order, so every rank
 * owns an equal share of the contribs and of each degree class; dangling
 * vertices round-robin by id.  Deterministic: every rank derives the same
 * partition.  1 <= world <= 4096, 0 <= rank < world
 * (else PR_EINVAL).  pr_run / pr_preprocess keep working on the whole graph.
 */
int pr_graph_shard(pr_graph *g, int32_t rank, int32_t world, void *stream);

/*
 * pr_run_sharded -- the synchronous plain iteration (PR_MODE_SYNC, optionally
 * PR_NORM_LINF / PR_TIMING; other bits PR_EINVAL) over this rank's rows.
 *   ranks  fp64[n] DEVICE buffer: owned vertices get their rank, every other
 *          entry 0.0 (so a sum all-reduce over the ranks assembles the vector
 *          exactly); a host pointer is PR_EINVAL
 *   exchange, exchange_ctx  the all-gather above (non-NULL)
 *   iters_out / final_delta_out as pr_run (identical on every rank)
 * PR_ESTATE without a prior pr_graph_shard.  world = 1 is bit-identical to
 * pr_run(PR_MODE_SYNC).
 */
int pr_run_sharded(pr_graph *g, double d, double threshold, int32_t max_iter, void *stream, uint32_t mode,
                   double *ranks, pr_exchange_fn exchange, void *exchange_ctx, int32_t *iters_out,
                   double *final_delta_out);

/*
 * Peer buffers -- the exchange fused into K-FINALIZE: with every rank's two
 * contrib buffers addressable from this device (same device, peer access, or
 * CUDA IPC below), each new contrib, zero-in-degree contrib and the rank's
 * (L1, L-inf) pair are stored straight into every peer's buffer by the
 * kernels that produce them, and pr_run_sharded calls the exchange with
 * buf = NULL, meaning only: return when every rank has finished its work
 * enqueued so far (e.g. stream synchronize + a host barrier) -- once after
 * the initialisation and once per sweep.
 *   pr_shard_buffers     this rank's buffers (device pointers, len doubles each)
 *   pr_shard_set_peers   y0s[r], y1s[r] = rank r's buffers as addressable here
 *                        (host arrays of world device pointers; [rank] unused);
 *                        world = 0 or NULL arrays: back to the all-gather
 *   pr_shard_export_ipc  2 cudaIpcMemHandle_t (64 B each) of this rank's buffers
 *   pr_shard_open_ipc    handles = world x 2 such handles (rank-major); opens
 *                        the peers' and sets them (closed by pr_destroy)
 * All return PR_OK, PR_EINVAL, PR_ESTATE (no pr_graph_shard) or PR_ECUDA.
 */
int pr_shard_buffers(const pr_graph *g, void **y0, void **y1, int64_t *len);

/*
 * NVLS multicast team -- the B200 form of the
 * fused exchange: the rank's two contrib buffers (+ the barrier flags) become
 * one physical allocation bound to a multicast object whose team is the
 * world's GPUs; K-FINALIZE stores every new contrib (and the delta pair, and
 * the in-degree-0 contribs) with ONE multimem.st into the multicast address,
 * which the switch replicates into every rank's buffer; pr_run_sharded then
 * calls the exchange with buf = NULL (a barrier only, as with peer buffers;
 * pr_shard_device_barrier makes it a device-side one).  Collective setup, in
 * this order across the ranks:
 *   pr_shard_mc_create  rank 0: creates the object (team size = world) and
 *                       writes its 64-byte fabric handle to handle_out
 *                       (NULL allowed when world = 1)
 *   pr_shard_mc_attach  every rank (rank 0 with NULL): imports the handle and
 *                       adds its device to the team
 *   pr_shard_mc_bind    every rank, after EVERY rank attached: binds its
 *                       memory and maps the unicast and multicast addresses
 *                       (the buffers are zeroed; exclusive with the IPC peer
 *                       buffers; released by pr_graph_shard / pr_destroy)
 * PR_ESTATE on an unsharded graph, PR_ECUDA when the device or driver lacks
 * multicast (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED) or fabric handles.
 */
int pr_shard_mc_create(pr_graph *g, void *handle_out);
int pr_shard_mc_attach(pr_graph *g, const void *handle);
int pr_shard_mc_bind(pr_graph *g, void *stream);

/*
 * pr_shard_device_barrier -- with peer buffers set, on != 0 replaces the
 * per-sweep host barrier (the exchange callback with buf = NULL) by a
 * device-side one: after the rank's finalize and peer stores, one thread
 * stores the barrier epoch into every peer's arrival flags (st.release.sys,
 * slot = this rank) and spins until every peer's epoch has arrived in its own
 * flags (ld.acquire.sys) -- no host synchronisation inside the sweep loop.
 * Every rank must make the same calls in the same order (the epochs count
 * barriers).  A wait over ~20 s aborts the run with PR_ECUDA.  world <= 65.
 * PR_ESTATE without peer buffers (world > 1).  Not measured across GPUs here.
 */
int pr_shard_device_barrier(pr_graph *g, int32_t on);

/*
 * pr_selftest_peer_barrier -- diagnostic: the barrier protocol above run by
 * `world` emulated ranks = the blocks of ONE cooperative launch on this
 * device (launches that wait on one another must not share a GPU), `epochs`
 * barriers, each checking that every rank sees every other rank's write of
 * that epoch.  PR_OK, or PR_ECUDA with the count in pr_last_error().
 */
int pr_selftest_peer_barrier(int32_t world, int32_t epochs, void *stream);
int pr_shard_set_peers(pr_graph *g, void *const *y0s, void *const *y1s, int32_t world);
int pr_shard_export_ipc(const pr_graph *g, void *handles);
int pr_shard_open_ipc(pr_graph *g, const void *handles, int32_t world);

typedef struct {
    int32_t rank;
    int32_t world;
    int64_t owned_vertices;  /* vertices this rank computes */
    int64_t rows;            /* owned vertices of in-degree > 0 (gathered) */
    int64_t edges;           /* in-edges of those rows */
    int64_t chunk;           /* doubles per rank in the exchanged buffer */
} pr_shard_info;

int pr_get_shard_info(const pr_graph *g, pr_shard_info *out);

#ifdef __cplusplus
}
#endif
#endif /* PRGPU_H */
