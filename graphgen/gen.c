/*
 * graphgen/gen.c -- seeded synthetic RAW edge-list generators (test and bench
 * input infrastructure).
 *
 * This module holds NONE of the PageRank method's arithmetic.  It only draws
 * raw (src, dst) pairs.  Both sides -- the CPU oracle (oracle/) and the CUDA
 * library (libprgpu) -- consume the same raw arrays and each removes
 * self-loops and duplicate edges itself.
 *
 * Workload recipes:
 *   cfg 1  G(n,m): m ordered pairs, src uniform, dst uniform over [0,n)\{src}
 *   cfg 2/4 R-MAT ("using the RMAT graph library")
 *          quadrant probabilities (a,b,c,d), no noise, ids permuted.
 *   cfg 3  structured power law: Zipf(1.1) in-degree, planted identical
 *          groups ("identical nodes") and chains ("chain").
 *   cfg 5  uniform random, out-degree Poisson(lambda).
 *
 * Random numbers: counter-based splitmix64, draw(seed, stream, index), so the
 * output is independent of the OpenMP thread count.
 *
 * Bounded-bias note: uniform integers in [0,k) use the multiply-high mapping
 * floor(x*k/2^64) of a 64-bit draw x; its bias is < k/2^64 (< 3e-12 for
 * k <= 5e7), which is documented in DESIGN.md instead of rejection sampling.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* splitmix64 output number `idx` of the sequence keyed by (seed, stream). */
static inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t idx) {
    uint64_t key = mix64(seed * GOLDEN + mix64(stream + 0x632BE59BD9B4E019ULL));
    return mix64(key + (idx + 1) * GOLDEN);
}

static inline double u01(uint64_t x) { return (double)(x >> 11) * (1.0 / 9007199254740992.0); }

static inline uint64_t below(uint64_t x, uint64_t k) {
    return (uint64_t)(((unsigned __int128)x * (unsigned __int128)k) >> 64);
}

uint64_t gg_draw(uint64_t seed, uint64_t stream, uint64_t idx) { return draw(seed, stream, idx); }

/* Fisher-Yates shuffle of perm[0..k) (caller fills it), stream-dedicated. */
static void shuffle_i32(int32_t *perm, int64_t k, uint64_t seed, uint64_t stream) {
    for (int64_t i = k - 1; i > 0; --i) {
        int64_t j = (int64_t)below(draw(seed, stream, (uint64_t)i), (uint64_t)(i + 1));
        int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
}

/* ---------------------------------------------------------------- cfg 1 -- */
int64_t gg_gnm(int64_t n, int64_t m, uint64_t seed, int32_t *src, int32_t *dst) {
    if (n < 2 || m < 0) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        int64_t s = (int64_t)below(draw(seed, 1, (uint64_t)i), (uint64_t)n);
        int64_t t = (int64_t)below(draw(seed, 2, (uint64_t)i), (uint64_t)(n - 1));
        if (t >= s) t += 1;               /* uniform over [0,n) \ {s} */
        src[i] = (int32_t)s; dst[i] = (int32_t)t;
    }
    return m;
}

/* ------------------------------------------------------------- cfg 2, 4 -- */
/* One uniform per (edge, level): quadrant (0,0) w.p. a, (0,1) b, (1,0) c,
 * (1,1) d = 1-a-b-c.  Row bit -> src, column bit -> dst, MSB first.  Then a
 * random permutation pi (Fisher-Yates, stream 3) is applied to both ends. */
int64_t gg_rmat(int scale, int64_t m, double a, double b, double c, uint64_t seed,
                int permute, int32_t *src, int32_t *dst) {
    if (scale < 1 || scale > 30 || m < 0) return -1;
    const int64_t n = (int64_t)1 << scale;
    const double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        uint32_t s = 0, t = 0;
        for (int l = 0; l < scale; ++l) {
            double r = u01(draw(seed, 1, (uint64_t)i * (uint64_t)scale + (uint64_t)l));
            uint32_t rb, cb;
            if (r < a)        { rb = 0; cb = 0; }
            else if (r < ab)  { rb = 0; cb = 1; }
            else if (r < abc) { rb = 1; cb = 0; }
            else              { rb = 1; cb = 1; }
            s = (s << 1) | rb; t = (t << 1) | cb;
        }
        src[i] = (int32_t)s; dst[i] = (int32_t)t;
    }
    if (permute) {
        int32_t *pi = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
        if (!pi) return -2;
        for (int64_t v = 0; v < n; ++v) pi[v] = (int32_t)v;
        shuffle_i32(pi, n, seed, 3);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < m; ++i) { src[i] = pi[src[i]]; dst[i] = pi[dst[i]]; }
        free(pi);
    }
    return m;
}

/* ---------------------------------------------------------------- cfg 5 -- */
/* Out-degree k_u ~ Poisson(lambda) by inversion (sequential CDF search, one
 * uniform per vertex, stream 1); each out-edge's dst uniform over [0,n)\{u}
 * (stream 2, index = global edge slot).  src == NULL: return the count only. */
static int poisson_inv(double u, double lambda) {
    double p = exp(-lambda), cdf = p;
    int k = 0;
    while (u > cdf && k < 100000) { ++k; p *= lambda / k; cdf += p; if (p == 0.0 && cdf < u) break; }
    return k;
}

int64_t gg_poisson(int64_t n, double lambda, uint64_t seed, int64_t *offsets /*n+1, scratch*/,
                   int32_t *src, int32_t *dst) {
    if (n < 2 || lambda <= 0) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < n; ++u) offsets[u + 1] = poisson_inv(u01(draw(seed, 1, (uint64_t)u)), lambda);
    offsets[0] = 0;
    for (int64_t u = 0; u < n; ++u) offsets[u + 1] += offsets[u];
    if (!src) return offsets[n];
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t u = 0; u < n; ++u) {
        for (int64_t e = offsets[u]; e < offsets[u + 1]; ++e) {
            int64_t t = (int64_t)below(draw(seed, 2, (uint64_t)e), (uint64_t)(n - 1));
            if (t >= u) t += 1;
            src[e] = (int32_t)u; dst[e] = (int32_t)t;
        }
    }
    return offsets[n];
}

/* ---------------------------------------------------------------- cfg 3 -- */
/* Structured power-law graph (reading of config 3):
 *  (i)   roles from a random permutation (stream 10): first chain_frac*n are
 *        chain vertices, next group_frac*n group members, the rest base.
 *  (ii)  n_base_draws edges: src uniform over non-chain vertices (stream 11),
 *        dst = Zipf(alpha) rank-frequency over base vertices in a random
 *        popularity order (order: stream 12; draws: stream 13).
 *  (iii) group members are cut into groups of size U{2..64} (stream 14); each
 *        group gets a source set of U{1..16} base vertices (stream 15) and
 *        every member receives an edge from every source in the set.
 *  (iv)  chain vertices are cut into chains of length U{2..16} (stream 16);
 *        each chain is p -> v1 -> ... -> vL -> s with p, s uniform base
 *        vertices (stream 17).
 * Outputs (optional, may be NULL): planted_group[n] (group id or -1),
 * planted_chain[n] (chain id or -1), planted_pos[n] (1..L on chains, else 0).
 * src == NULL: return the raw edge count only. */
typedef struct { int64_t n, nchain, ngroup, nbase; int32_t *perm; } roles_t;

static int make_roles(int64_t n, double chain_frac, double group_frac, uint64_t seed, roles_t *r) {
    r->n = n;
    r->nchain = (int64_t)llround(chain_frac * (double)n);
    r->ngroup = (int64_t)llround(group_frac * (double)n);
    r->nbase = n - r->nchain - r->ngroup;
    if (r->nbase < 2) return -1;
    r->perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!r->perm) return -2;
    for (int64_t v = 0; v < n; ++v) r->perm[v] = (int32_t)v;
    shuffle_i32(r->perm, n, seed, 10);
    return 0;
}
/* perm[0..nchain) chain, perm[nchain..nchain+ngroup) group, rest base. */

static int64_t cut_sizes(int64_t total, int lo, int hi, uint64_t seed, uint64_t stream, int32_t *sizes) {
    /* sizes U{lo..hi}; a remainder < lo is merged into the last piece. */
    int64_t k = 0, used = 0;
    while (used < total) {
        int64_t s = lo + (int64_t)below(draw(seed, stream, (uint64_t)k), (uint64_t)(hi - lo + 1));
        if (total - used - s < lo && total - used - s > 0) s = total - used;  /* absorb remainder */
        if (s > total - used) s = total - used;
        if (sizes) sizes[k] = (int32_t)s;
        used += s; ++k;
    }
    return k;
}

int64_t gg_structured(int64_t n, int64_t n_base_draws, double zipf_alpha, double chain_frac,
                      double group_frac, uint64_t seed, int32_t *src, int32_t *dst,
                      int32_t *planted_group, int32_t *planted_chain, int32_t *planted_pos) {
    roles_t R;
    if (make_roles(n, chain_frac, group_frac, seed, &R) != 0) return -1;
    const int32_t *chainv = R.perm, *groupv = R.perm + R.nchain, *basev = R.perm + R.nchain + R.ngroup;
    const int64_t nonchain = R.ngroup + R.nbase;
    const int32_t *nonchainv = R.perm + R.nchain;

    int64_t ngroups = R.ngroup >= 2 ? cut_sizes(R.ngroup, 2, 64, seed, 14, NULL) : 0;
    int64_t nchains = R.nchain >= 2 ? cut_sizes(R.nchain, 2, 16, seed, 16, NULL) : 0;
    int32_t *gsz = (int32_t *)malloc(sizeof(int32_t) * (size_t)(ngroups + 1));
    int32_t *csz = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nchains + 1));
    if (ngroups) cut_sizes(R.ngroup, 2, 64, seed, 14, gsz);
    if (nchains) cut_sizes(R.nchain, 2, 16, seed, 16, csz);

    /* count */
    int64_t total = n_base_draws;
    for (int64_t g = 0; g < ngroups; ++g) {
        int64_t ks = 1 + (int64_t)below(draw(seed, 15, (uint64_t)g * 17u), 16);
        total += ks * gsz[g];
    }
    for (int64_t ch = 0; ch < nchains; ++ch) total += csz[ch] + 1;
    if (!src) { free(gsz); free(csz); free(R.perm); return total; }

    /* (ii) Zipf base draws */
    int32_t *pop = (int32_t *)malloc(sizeof(int32_t) * (size_t)R.nbase);
    double *cdf = (double *)malloc(sizeof(double) * (size_t)R.nbase);
    memcpy(pop, basev, sizeof(int32_t) * (size_t)R.nbase);
    shuffle_i32(pop, R.nbase, seed, 12);
    double acc = 0.0;
    for (int64_t k = 0; k < R.nbase; ++k) { acc += pow((double)(k + 1), -zipf_alpha); cdf[k] = acc; }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_base_draws; ++i) {
        int64_t si = (int64_t)below(draw(seed, 11, (uint64_t)i), (uint64_t)nonchain);
        double u = u01(draw(seed, 13, (uint64_t)i)) * acc;
        int64_t lo = 0, hi = R.nbase - 1;           /* first k with cdf[k] > u */
        while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (cdf[mid] > u) hi = mid; else lo = mid + 1; }
        int32_t s = nonchainv[si], t = pop[lo];
        if (s == t) t = pop[lo == 0 ? 1 : lo - 1];   /* keep draws loop-free */
        src[i] = s; dst[i] = t;
    }
    free(cdf); free(pop);

    int64_t e = n_base_draws;
    if (planted_group) for (int64_t v = 0; v < n; ++v) planted_group[v] = -1;
    if (planted_chain) for (int64_t v = 0; v < n; ++v) planted_chain[v] = -1;
    if (planted_pos) for (int64_t v = 0; v < n; ++v) planted_pos[v] = 0;

    /* (iii) identical groups */
    int64_t off = 0;
    for (int64_t g = 0; g < ngroups; ++g) {
        int64_t ks = 1 + (int64_t)below(draw(seed, 15, (uint64_t)g * 17u), 16);
        for (int64_t j = 0; j < gsz[g]; ++j) {
            int32_t w = groupv[off + j];
            if (planted_group) planted_group[w] = (int32_t)g;
            for (int64_t q = 0; q < ks; ++q) {
                int64_t bi = (int64_t)below(draw(seed, 15, (uint64_t)g * 17u + 1u + (uint64_t)q), (uint64_t)R.nbase);
                src[e] = basev[bi]; dst[e] = w; ++e;
            }
        }
        off += gsz[g];
    }
    /* (iv) chains p -> v1 -> ... -> vL -> s */
    off = 0;
    for (int64_t ch = 0; ch < nchains; ++ch) {
        int32_t p = basev[below(draw(seed, 17, (uint64_t)ch * 2u), (uint64_t)R.nbase)];
        int32_t s = basev[below(draw(seed, 17, (uint64_t)ch * 2u + 1u), (uint64_t)R.nbase)];
        int32_t prev = p;
        for (int64_t j = 0; j < csz[ch]; ++j) {
            int32_t v = chainv[off + j];
            if (planted_chain) planted_chain[v] = (int32_t)ch;
            if (planted_pos) planted_pos[v] = (int32_t)(j + 1);
            src[e] = prev; dst[e] = v; ++e; prev = v;
        }
        src[e] = prev; dst[e] = s; ++e;
        off += csz[ch];
    }
    free(gsz); free(csz); free(R.perm);
    return e;
}

/* Order-dependent 64-bit checksum of a raw edge list (drift detection). */
uint64_t gg_checksum_edges(int64_t m, const int32_t *src, const int32_t *dst) {
    uint64_t h = 0x12345678ULL;
    for (int64_t i = 0; i < m; ++i)
        h = mix64(h ^ (((uint64_t)(uint32_t)src[i] << 32) | (uint32_t)dst[i])) + (uint64_t)i;
    return h;
}
