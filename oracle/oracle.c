/*
 * oracle/oracle.c -- plain, slow, single-threaded fp64 CPU oracle for the
 * PageRank pull iteration of arXiv 2109.09527.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  The
 * product path (paper_2109_09527_b200, libprgpu) never calls it and shares no
 * code, header, table or constant generator with it.
 *
 * Citations: "P:N" = PAPER.md line N, "S:N" = SPEC.md line N (the reference
 * text), "Q-x" = a reading listed in DESIGN.md §Readings.
 *
 * Every function below is pinned by tests/test_oracle_pins.py against
 * closed forms, a dense linear solve (numpy), brute force on tiny inputs and
 * the mass / contraction identities.  No function is "parity unpinned".
 *
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction; Q-F), no threads.
 */
#define _GNU_SOURCE
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------ sums -- */
/* Neumaier-compensated summation (used for the convergence deltas and the
 * residual certificate so that the oracle's Delta is not order-sensitive at
 * the 1e-16 level). */
typedef struct { double s, c; } nsum_t;
static inline void nsum_add(nsum_t *a, double v) {
    double t = a->s + v;
    if (fabs(a->s) >= fabs(v)) a->c += (a->s - t) + v; else a->c += (v - t) + a->s;
    a->s = t;
}
static inline double nsum_get(const nsum_t *a) { return a->s + a->c; }

/* ------------------------------------------------------------------- CSR -- */
static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/*
 * In-edge CSR of the simple graph G = (V, E): "converted later to Compressed
 * Sparse Row (CSR) format" (§5.2), "Graph G <- (V,E)  CSR representation"
 * (Alg.1).  Self-loops dropped and duplicates collapsed; within a row
 * sources ascending (Q-L).  outdeg counts DISTINCT non-loop
 * out-edges (P:452 outDeg, P:493 outdeg).
 *
 * Plain definition: sort the (dst, src) pairs, drop loops and repeats.
 * Written as: bucket by dst (counting), sort each bucket by src, unique.
 *
 * Returns E (>= 0), -1 if some id is outside [0, n), -2 out of memory.
 * col_idx must hold m entries; row_ptr n+1; outdeg n.
 */
int64_t or_build_csr(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                     int64_t *row_ptr, int32_t *col_idx, int32_t *outdeg) {
    for (int64_t i = 0; i < m; ++i)
        if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) return -1;
    int64_t *start = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    if (!start || !tmp) { free(start); free(tmp); return -2; }
    for (int64_t i = 0; i < m; ++i)
        if (src[i] != dst[i]) start[dst[i] + 1] += 1;
    for (int64_t v = 0; v < n; ++v) start[v + 1] += start[v];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    if (!fill) { free(start); free(tmp); return -2; }
    memcpy(fill, start, sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < m; ++i)
        if (src[i] != dst[i]) tmp[fill[dst[i]]++] = src[i];
    free(fill);
    int64_t E = 0;
    for (int64_t v = 0; v < n; ++v) {
        row_ptr[v] = E;
        int64_t b = start[v], e = start[v + 1];
        qsort(tmp + b, (size_t)(e - b), sizeof(int32_t), cmp_i32);
        for (int64_t k = b; k < e; ++k)
            if (k == b || tmp[k] != tmp[k - 1]) col_idx[E++] = tmp[k];
    }
    row_ptr[n] = E;
    free(start); free(tmp);
    for (int64_t v = 0; v < n; ++v) outdeg[v] = 0;
    for (int64_t e = 0; e < E; ++e) outdeg[col_idx[e]] += 1;
    return E;
}

/* ------------------------------------------------------ identical groups -- */
/*
 * STIC-D identical nodes (§3): "If two nodes have incoming edges from
 * the same set, then the two nodes would have the same PageRank ... PageRank
 * is calculated on one vertex from each class."  Classes = equal in-sets
 * (after dedup); the empty in-set is one class; representative = the
 * minimum vertex id of the class.  Q-G.
 *
 * Plain definition: sort the vertices by their sorted in-list (then by id) and
 * cut runs of equal lists.  (The GPU path hashes; this does not.)
 */
typedef struct { const int64_t *rp; const int32_t *col; } rows_ctx;

static int cmp_rows(const void *a, const void *b, void *ctx_) {
    const rows_ctx *ctx = (const rows_ctx *)ctx_;
    int32_t u = *(const int32_t *)a, v = *(const int32_t *)b;
    int64_t du = ctx->rp[u + 1] - ctx->rp[u], dv = ctx->rp[v + 1] - ctx->rp[v];
    if (du != dv) return du < dv ? -1 : 1;
    const int32_t *ru = ctx->col + ctx->rp[u], *rv = ctx->col + ctx->rp[v];
    for (int64_t k = 0; k < du; ++k)
        if (ru[k] != rv[k]) return ru[k] < rv[k] ? -1 : 1;
    return (u > v) - (u < v);
}

static int same_row(const int64_t *rp, const int32_t *col, int32_t u, int32_t v) {
    int64_t du = rp[u + 1] - rp[u];
    if (du != rp[v + 1] - rp[v]) return 0;
    return memcmp(col + rp[u], col + rp[v], sizeof(int32_t) * (size_t)du) == 0;
}

int or_identical(int64_t n, const int64_t *rp, const int32_t *col, int32_t *rep) {
    int32_t *ord = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (!ord) return -2;
    for (int64_t v = 0; v < n; ++v) ord[v] = (int32_t)v;
    rows_ctx ctx = { rp, col };
    qsort_r(ord, (size_t)n, sizeof(int32_t), cmp_rows, &ctx);
    int64_t i = 0;
    while (i < n) {
        int64_t j = i + 1;
        while (j < n && same_row(rp, col, ord[i], ord[j])) ++j;
        for (int64_t k = i; k < j; ++k) rep[ord[k]] = ord[i];   /* ord[i] is the min id */
        i = j;
    }
    free(ord);
    return 0;
}

/* ----------------------------------------------------------------- chains -- */
/*
 * STIC-D chains (§3, garbled: "If a set of nodes form a chain, each node
 * has only one incoming edge, and one outgoing edge, the PageRank of a vertex
 * with such a node is easy to compute").  Reading Q-C:
 *   chain vertex  <=>  in-degree 1 and out-degree 1 (deduplicated);
 *   head h        <=>  chain(h) and not chain(pred(h));
 *   members       =   the chain vertices reached from a head by following the
 *                     unique out-edge, at distance k = 1, 2, ... from h;
 *   source        =   rep(h) (the head may be an identical non-representative).
 * Vertices on pure cycles of chain vertices are never reached from a head and
 * are not members.  Output: chain_src[v] = rep(head) or -1; chain_k[v] = k or 0.
 * Plain definition: a sequential walk from every head along succ().
 * Returns the maximum k (0 if there are no members), -2 out of memory.
 */
int or_chains(int64_t n, const int64_t *rp, const int32_t *col, const int32_t *od,
              const int32_t *rep, int32_t *chain_src, int32_t *chain_k) {
    int32_t *succ = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (!succ) return -2;
    for (int64_t v = 0; v < n; ++v) { succ[v] = -1; chain_src[v] = -1; chain_k[v] = 0; }
    for (int64_t v = 0; v < n; ++v)
        for (int64_t e = rp[v]; e < rp[v + 1]; ++e)
            if (od[col[e]] == 1) succ[col[e]] = (int32_t)v;
#define IS_CHAIN(v) ((rp[(v) + 1] - rp[(v)]) == 1 && od[(v)] == 1)
    int maxk = 0;
    for (int64_t h = 0; h < n; ++h) {
        if (!IS_CHAIN(h)) continue;
        int32_t p = col[rp[h]];
        if (IS_CHAIN(p)) continue;                 /* not a head */
        int32_t w = succ[h];
        int k = 1;
        while (w >= 0 && IS_CHAIN(w) && k <= n) {
            chain_src[w] = rep[h];
            chain_k[w] = k;
            if (k > maxk) maxk = k;
            ++k;
            w = succ[w];
        }
    }
#undef IS_CHAIN
    free(succ);
    return maxk;
}

/* --------------------------------------------------------------- PageRank -- */
enum { OR_NORM_LINF = 1, OR_REDUCED = 2, OR_GAUSS_SEIDEL = 4, OR_BLOCK_GS = 8, OR_PERFORATE = 16 };

/*
 * One synchronous (Jacobi) sweep over all vertices, Eq.(1) in the
 * "sum, then times d" form of Alg.2 (Q-F):
 *     x_out(v) = (1-d)/n + d * sum_{u in in(v), ascending} x_in(u)/outdeg(u).
 * Dangling vertices (outdeg 0) never appear in any in(v), so they contribute
 * nothing (Q-D).
 */
void or_jacobi_step(int64_t n, const int64_t *rp, const int32_t *col, const int32_t *od,
                    double d, const double *x_in, double *x_out) {
    const double c = (1.0 - d) / (double)n;
    for (int64_t v = 0; v < n; ++v) {
        double s = 0.0;
        for (int64_t e = rp[v]; e < rp[v + 1]; ++e) s += x_in[col[e]] / (double)od[col[e]];
        x_out[v] = c + d * s;
    }
}

/*
 * Blocks of the block Gauss-Seidel sweep (reading Q-B: No-Sync's
 * in-place update, Alg.3, in a FIXED order).  The rows are the
 * vertices the sweep gathers, in ascending id: every vertex of in-degree > 0
 * (plain), or (OR_REDUCED) those that are their class representative and not a
 * chain member.  With E_R the rows' in-edges and off(i) the in-edges of the
 * rows before row i, block k of K is the rows [b_k, b_{k+1}):
 *     b_0 = 0,  b_K = R,  b_k = the first i with off(i) * K >= k * E_R,
 * i.e. a block starts at the first row starting at or after the k-th K-th of
 * the edges, so no row is split between blocks.
 * rows_out (nullable, n entries) receives the rows; bounds_out K+1 entries.
 * Returns R, or -1 on bad arguments.
 */
int64_t or_block_bounds(int64_t n, const int64_t *rp, const int32_t *rep, const int32_t *chain_k,
                        int32_t mode, int32_t K, int32_t *rows_out, int64_t *bounds_out) {
    if (K < 1 || ((mode & OR_REDUCED) && (!rep || !chain_k))) return -1;
    int64_t R = 0, ER = 0;
    for (int64_t v = 0; v < n; ++v) {
        if (rp[v + 1] == rp[v]) continue;
        if ((mode & OR_REDUCED) && (rep[v] != v || chain_k[v] > 0)) continue;
        if (rows_out) rows_out[R] = (int32_t)v;
        ++R;
        ER += rp[v + 1] - rp[v];
    }
    bounds_out[0] = 0;
    for (int32_t k = 1; k < K; ++k) bounds_out[k] = R;
    bounds_out[K] = R;
    int64_t off = 0, i = 0;
    for (int64_t v = 0; v < n; ++v) {
        if (rp[v + 1] == rp[v]) continue;
        if ((mode & OR_REDUCED) && (rep[v] != v || chain_k[v] > 0)) continue;
        for (int32_t k = 1; k < K; ++k)
            if (bounds_out[k] == R && off * (int64_t)K >= (int64_t)k * ER) bounds_out[k] = i;
        off += rp[v + 1] - rp[v];
        ++i;
    }
    return R;
}

/*
 * Power iteration to convergence.
 *   x_0 = 1/n ("prPrev(u_i) <- 1/n"), or x_init when given (a resumed
 *   run: the sweeps are memoryless, so running to tau1 and then resuming to
 *   tau2 < tau1 gives exactly the iterates of one run to tau2).
 *   iterate "while err > threshold" (Q-S): stop at the first t with
 *   Delta_t <= tau, or at t = max_iter (status 2).
 *   Delta_t = sum_v |x_t(v) - x_{t-1}(v)| (L1, BASELINE configs; Q-N) or
 *   max_v |...| (L-inf, P:454 / P:463), reset every iteration (Q-E), over ALL
 *   n vertices (Q-R).
 *   iters = number of update sweeps including the final one (Q-I).
 * mode:
 *   0               plain synchronous (Alg.1 semantics)
 *   OR_REDUCED      reduced synchronous: representatives of R gathered as
 *                   above; identical members copy their representative
 *                   (P:398); chain members resolved in the same iteration by
 *                   the single-in-neighbour instance of Eq.(1), in order of
 *                   increasing distance from the head (Q-C)
 *   OR_GAUSS_SEIDEL in-place ascending sweep (No-Sync with one thread,
 *                   Alg.3)
 *   OR_BLOCK_GS     block Gauss-Seidel in `nblocks` blocks (or_block_bounds;
 *                   reading Q-B): block by block, every row of the block gathers
 *                   x(u)/outdeg(u) as x stands when the block starts (the
 *                   updates of the earlier blocks of the same sweep visible,
 *                   Alg.3's in-place pr(u) <- tmp), then the block's
 *                   rows are updated; after the last block, (with OR_REDUCED)
 *                   the members as in the reduced mode, then the vertices of
 *                   in-degree 0 take (1-d)/n (Eq.(1) with an empty sum).
 *                   nblocks = 1 is the synchronous sweep.
 *   OR_PERFORATE    loop perforation (Alg.5; reading Q-P), plain
 *                   synchronous only: a vertex whose change in a sweep is
 *                   0 != |delta| < tau * 0.00001 (or perf_thr, if >= 0) gets its
 *                   threshold_check flag set after that sweep, and from the
 *                   next sweep on is not computed: it keeps its value
 *                   (|delta| = 0)
 *   | OR_NORM_LINF  use the max norm for the stop test
 * delta_log (nullable) receives (L1, Linf) per iteration: 2*max_iter doubles.
 * frozen_out (nullable, OR_PERFORATE) receives the flags (0/1 per vertex).
 * Returns 0 converged, 2 max_iter reached, -2 out of memory, 1 bad args.
 */
int or_pagerank(int64_t n, const int64_t *rp, const int32_t *col, const int32_t *od,
                double d, double tau, int32_t max_iter, int32_t mode,
                const int32_t *rep, const int32_t *chain_k, int32_t nblocks, double perf_thr,
                const double *x_init,
                double *x_out, double *delta_log, int32_t *iters_out, double *final_delta,
                uint8_t *frozen_out) {
    if (n < 1 || !(d > 0.0 && d < 1.0) || !(tau >= 0.0) || max_iter < 1) return 1;
    if ((mode & OR_REDUCED) && (!rep || !chain_k)) return 1;
    if ((mode & OR_BLOCK_GS) && nblocks < 1) return 1;
    if ((mode & OR_PERFORATE) && (mode & (OR_REDUCED | OR_GAUSS_SEIDEL | OR_BLOCK_GS))) return 1;
    const double c = (1.0 - d) / (double)n;
    const double tau_f = perf_thr >= 0.0 ? perf_thr : tau * 1e-5;   /* "threshold*0.00001" */
    double *xp = (double *)malloc(sizeof(double) * (size_t)n);
    double *xn = (double *)malloc(sizeof(double) * (size_t)n);
    double *sb = NULL;                 /* block GS: the sums of one block */
    int32_t *rows = NULL; int64_t *bb = NULL;
    uint8_t *frozen = NULL;
    int32_t *by_k = NULL; int64_t *k_start = NULL; int maxk = 0;
    if (!xp || !xn) { free(xp); free(xn); return -2; }
    if (mode & OR_BLOCK_GS) {
        rows = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
        bb = (int64_t *)malloc(sizeof(int64_t) * ((size_t)nblocks + 1));
        sb = (double *)malloc(sizeof(double) * (size_t)n);
        if (!rows || !bb || !sb) { free(xp); free(xn); free(rows); free(bb); free(sb); return -2; }
        or_block_bounds(n, rp, rep, chain_k, mode, nblocks, rows, bb);
    }
    if (mode & OR_PERFORATE) {
        frozen = (uint8_t *)calloc((size_t)n, 1);
        if (!frozen) { free(xp); free(xn); return -2; }
    }
    if (mode & OR_REDUCED) {
        /* chain members bucketed by distance k from their head */
        for (int64_t v = 0; v < n; ++v) if (chain_k[v] > maxk) maxk = chain_k[v];
        k_start = (int64_t *)calloc((size_t)maxk + 2, sizeof(int64_t));
        by_k = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
        for (int64_t v = 0; v < n; ++v) if (chain_k[v] > 0) k_start[chain_k[v] + 1] += 1;
        for (int k = 0; k <= maxk; ++k) k_start[k + 1] += k_start[k];
        int64_t *f = (int64_t *)malloc(sizeof(int64_t) * ((size_t)maxk + 1));
        memcpy(f, k_start, sizeof(int64_t) * ((size_t)maxk + 1));
        for (int64_t v = 0; v < n; ++v) if (chain_k[v] > 0) by_k[f[chain_k[v]]++] = (int32_t)v;
        free(f);
    }
    for (int64_t v = 0; v < n; ++v) xp[v] = x_init ? x_init[v] : 1.0 / (double)n;
    int status = 2; int32_t t = 0; double delta = 0.0;
    for (t = 1; t <= max_iter; ++t) {
        nsum_t l1 = { 0.0, 0.0 }; double linf = 0.0;
        if (mode & OR_GAUSS_SEIDEL) {
            for (int64_t v = 0; v < n; ++v) {
                double prev = xp[v], s = 0.0;
                for (int64_t e = rp[v]; e < rp[v + 1]; ++e) s += xp[col[e]] / (double)od[col[e]];
                xp[v] = c + d * s;
                double a = fabs(xp[v] - prev);
                nsum_add(&l1, a); if (a > linf) linf = a;
            }
            memcpy(xn, xp, sizeof(double) * (size_t)n);
        } else {
            if (mode & OR_BLOCK_GS) {
                /* xn is updated in place, block by block; xp keeps x_{t-1} for Delta */
                memcpy(xn, xp, sizeof(double) * (size_t)n);
                for (int32_t k = 0; k < nblocks; ++k) {
                    for (int64_t i = bb[k]; i < bb[k + 1]; ++i) {
                        int32_t v = rows[i];
                        double s = 0.0;
                        for (int64_t e = rp[v]; e < rp[v + 1]; ++e) s += xn[col[e]] / (double)od[col[e]];
                        sb[i] = s;
                    }
                    for (int64_t i = bb[k]; i < bb[k + 1]; ++i) xn[rows[i]] = c + d * sb[i];
                }
            } else {
                for (int64_t v = 0; v < n; ++v) {
                    if ((mode & OR_REDUCED) && (rep[v] != v || chain_k[v] > 0)) continue;
                    if (frozen && frozen[v]) { xn[v] = xp[v]; continue; }   /* skipped (Alg.5) */
                    double s = 0.0;
                    for (int64_t e = rp[v]; e < rp[v + 1]; ++e) s += xp[col[e]] / (double)od[col[e]];
                    xn[v] = c + d * s;
                }
            }
            if (mode & OR_REDUCED) {
                for (int64_t v = 0; v < n; ++v)          /* identical members */
                    if (rep[v] != v) xn[v] = xn[rep[v]];
                for (int k = 1; k <= maxk; ++k)          /* chains, head outwards */
                    for (int64_t i = k_start[k]; i < k_start[k + 1]; ++i) {
                        int32_t v = by_k[i], p = col[rp[v]];
                        xn[v] = c + d * (xn[p] / (double)od[p]);
                    }
            }
            if (mode & OR_BLOCK_GS)                      /* in-degree 0: Eq.(1), empty sum */
                for (int64_t v = 0; v < n; ++v)
                    if (rp[v + 1] == rp[v]) xn[v] = c;
            for (int64_t v = 0; v < n; ++v) {
                double a = fabs(xn[v] - xp[v]);
                nsum_add(&l1, a); if (a > linf) linf = a;
                if (frozen && !frozen[v] && a != 0.0 && a < tau_f) frozen[v] = 1;
            }
            double *sw = xp; xp = xn; xn = sw;           /* prPrev = pr */
        }
        double l1v = nsum_get(&l1);
        if (delta_log) { delta_log[2 * (t - 1)] = l1v; delta_log[2 * (t - 1) + 1] = linf; }
        delta = (mode & OR_NORM_LINF) ? linf : l1v;
        if (delta <= tau) { status = 0; break; }
    }
    if (t > max_iter) t = max_iter;
    memcpy(x_out, xp, sizeof(double) * (size_t)n);
    if (iters_out) *iters_out = t;
    if (final_delta) *final_delta = delta;
    if (frozen_out && frozen) memcpy(frozen_out, frozen, (size_t)n);
    free(xp); free(xn); free(by_k); free(k_start); free(rows); free(bb); free(sb); free(frozen);
    return status;
}

/*
 * Residual certificate: r(x) = x - (c*1 + d*M*x), M_{vu} = 1/outdeg(u) for
 * u -> v (Eq.(1) as a linear system; dangling columns zero, Q-D).  Returns
 * ||r||_1 (Neumaier sum).  Since ||(I - dM)^{-1}||_1 <= 1/(1-d),
 * ||x - x*||_1 <= ||r||_1 / (1-d) for ANY candidate x (parity of
 * the async mode, Lemma 2).  r_out (nullable) gets r per vertex.
 */
double or_residual_l1(int64_t n, const int64_t *rp, const int32_t *col, const int32_t *od,
                      double d, const double *x, double *r_out) {
    const double c = (1.0 - d) / (double)n;
    nsum_t acc = { 0.0, 0.0 };
    for (int64_t v = 0; v < n; ++v) {
        nsum_t s = { 0.0, 0.0 };
        for (int64_t e = rp[v]; e < rp[v + 1]; ++e) nsum_add(&s, x[col[e]] / (double)od[col[e]]);
        double r = x[v] - (c + d * nsum_get(&s));
        if (r_out) r_out[v] = r;
        nsum_add(&acc, fabs(r));
    }
    return nsum_get(&acc);
}
