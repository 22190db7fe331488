"""Pins of the CPU oracle against things other than itself (no GPU).

Each test states what fixes the expected value: a SPEC worked example
(tests/golden/spec_examples.json), a closed form of Eq.(1), a
dense linear solve with numpy, brute force on tiny inputs, or an identity of
the iteration (mass, L1 contraction).  A plausible oracle bug -- a dropped
(1-d)/n, d applied twice, a transposed M, a wrong dangling rule, a stop test
off by one, a wrong representative -- fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from tests import graphs as G

HERE = os.path.dirname(os.path.abspath(__file__))
SPEC = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))
D = 0.85


def csr_of(n, edges):
    s, t = G.edges_to_arrays(edges)
    return oracle.build_csr(n, s, t)


# ------------------------------------------------------------------- CSR --
@pytest.mark.parametrize("ex", SPEC["csr"], ids=lambda e: e["cite"])
def test_csr_spec_examples(ex):
    g = csr_of(ex["n"], ex["edges"])
    if "row_ptr" in ex:
        assert g.row_ptr.tolist() == ex["row_ptr"]
        assert g.col_idx.tolist() == ex["col_idx"]
    if "E" in ex:
        assert g.E == ex["E"]
    assert g.outdeg.tolist() == ex["outdeg"]


@pytest.mark.parametrize("seed", range(12))
def test_csr_brute_force(seed):
    n = [1, 2, 3, 7, 30, 200][seed % 6]
    edges = G.random_edges(n, 5 * n + seed, seed)
    g = csr_of(n, edges)
    rp, col, od = G.bf_csr(n, edges)
    assert g.row_ptr.tolist() == rp
    assert g.col_idx.tolist() == col
    assert g.outdeg.tolist() == od
    # round trip: re-emitted pairs == deduplicated, loop-free pair set
    back = sorted((int(g.col_idx[e]), v) for v in range(n) for e in range(g.row_ptr[v], g.row_ptr[v + 1]))
    assert back == G.bf_pairs(n, edges)


def test_csr_rejects_bad_ids():
    with pytest.raises(ValueError):
        csr_of(3, [(0, 3)])
    with pytest.raises(ValueError):
        csr_of(3, [(-1, 0)])


def test_csr_empty_and_loops_only():
    g = csr_of(4, [])
    assert g.E == 0 and g.row_ptr.tolist() == [0] * 5
    g = csr_of(3, [(0, 0), (1, 1), (1, 1)])
    assert g.E == 0 and g.outdeg.tolist() == [0, 0, 0]


# ------------------------------------------------------- identical groups --
@pytest.mark.parametrize("ex", SPEC["identical"], ids=lambda e: e["cite"])
def test_identical_spec_examples(ex):
    g = csr_of(ex["n"], ex["edges"])
    assert oracle.identical(g).tolist() == ex["rep"]


@pytest.mark.parametrize("seed", range(8))
def test_identical_brute_force(seed):
    if seed % 2:
        n, edges = G.planted_graph(seed)
    else:
        n = 40 + 20 * seed
        edges = G.random_edges(n, 2 * n, seed)   # sparse: many equal in-sets
    g = csr_of(n, edges)
    assert oracle.identical(g).tolist() == G.bf_identical(n, edges)


# ----------------------------------------------------------------- chains --
def test_chain_path_closed_structure():
    L = 8
    g = csr_of(L, G.path(L))
    rep = oracle.identical(g)
    cs, ck, mk = oracle.chains(g, rep)
    # vertex 0: in-degree 0; vertices 1..L-2 are chain vertices; head = 1
    assert ck.tolist() == [0, 0] + list(range(1, L - 2)) + [0]
    assert cs.tolist() == [-1, -1] + [1] * (L - 3) + [-1]
    assert mk == L - 3


def test_chain_pure_cycle_excluded():
    g = csr_of(6, G.cycle(6))
    cs, ck, mk = oracle.chains(g, oracle.identical(g))
    assert (cs == -1).all() and (ck == 0).all() and mk == 0


def test_chain_head_is_identical_member():
    # p -> a, p -> h, h -> x1 -> x2 -> s ; a and h identical (in-set {p}); rep(h) = a
    p, a, h, x1, x2, s = range(6)
    edges = [(p, a), (p, h), (h, x1), (x1, x2), (x2, s), (a, s), (s, p)]
    g = csr_of(6, edges)
    rep = oracle.identical(g)
    assert rep[h] == a
    cs, ck, _ = oracle.chains(g, rep)
    assert cs[x1] == a and ck[x1] == 1 and cs[x2] == a and ck[x2] == 2
    assert G.bf_chains(6, edges, rep.tolist()) == (cs.tolist(), ck.tolist())


@pytest.mark.parametrize("seed", range(8))
def test_chains_brute_force(seed):
    n, edges = G.planted_graph(seed, chains=(2, 5, 16, 1))
    g = csr_of(n, edges)
    rep = oracle.identical(g)
    cs, ck, _ = oracle.chains(g, rep)
    bs, bk = G.bf_chains(n, edges, rep.tolist())
    assert cs.tolist() == bs and ck.tolist() == bk
    assert (ck > 0).sum() >= (2 - 1) + (5 - 1) + (16 - 1)


# ------------------------------------------------------------ closed forms --
@pytest.mark.parametrize("ex", SPEC["pagerank"], ids=lambda e: e["cite"])
def test_pagerank_spec_examples(ex):
    g = csr_of(ex["n"], ex["edges"])
    r = oracle.pagerank(g, ex["d"], ex["tau"], 1000, norm_linf=ex["norm"] == "linf")
    np.testing.assert_allclose(r.x, ex["x"], rtol=0, atol=1e-15)
    if "iters" in ex:
        assert r.iters == ex["iters"]


def test_single_vertex_l1_two_iterations():
    g = csr_of(1, [])
    r = oracle.pagerank(g, D, 1e-12, 1000)
    assert r.x.tolist() == [1 - D] and r.iters == 2 and r.delta == 0.0


@pytest.mark.parametrize("n", [3, 17, 1000])
def test_cycle_uniform_stops_at_one(n):
    g = csr_of(n, G.cycle(n))
    r = oracle.pagerank(g, D, 1e-12, 1000)
    np.testing.assert_allclose(r.x, 1.0 / n, rtol=1e-14)
    assert r.iters == 1


@pytest.mark.parametrize("n", [2, 5, 101])
def test_in_star(n):
    g = csr_of(n, G.in_star(n))
    r = oracle.pagerank(g, D, 0.0, 1000)
    c = (1 - D) / n
    assert r.iters == 3 and r.delta == 0.0
    np.testing.assert_allclose(r.x[1:], c, rtol=1e-15)
    np.testing.assert_allclose(r.x[0], c * (1 + D * (n - 1)), rtol=1e-14)


@pytest.mark.parametrize("n", [3, 9])
def test_out_star(n):
    g = csr_of(n, G.out_star(n))
    r = oracle.pagerank(g, D, 0.0, 1000)
    c = (1 - D) / n
    np.testing.assert_allclose(r.x[0], c, rtol=1e-15)
    np.testing.assert_allclose(r.x[1:], c + D * c / (n - 1), rtol=1e-14)


def test_path_closed_form():
    L = 12
    g = csr_of(L, G.path(L))
    r = oracle.pagerank(g, D, 0.0, 1000)
    c = (1 - D) / L
    j = np.arange(L)
    np.testing.assert_allclose(r.x, c * (1 - D ** (j + 1)) / (1 - D), rtol=1e-14)


def test_complete_graph_uniform():
    n = 9
    g = csr_of(n, G.complete(n))
    r = oracle.pagerank(g, D, 1e-14, 1000)
    np.testing.assert_allclose(r.x, 1.0 / n, rtol=1e-14)
    assert len(set(oracle.identical(g).tolist())) == n


# ------------------------------------------------------------ dense solve --
def _dense_cases():
    out = []
    for seed in range(4):
        n = 50 + 40 * seed
        out.append((f"gnm{seed}", n, G.random_edges(n, 4 * n, 100 + seed)))
    for seed in range(3):
        n, e = G.planted_graph(200 + seed, n_base=100, chains=(10, 3, 7))
        out.append((f"planted{seed}", n, e))
    import graphgen
    s, t = graphgen.rmat(7, 16 * 128, seed=7)
    out.append(("rmat7", 128, list(zip(s.tolist(), t.tolist()))))
    return out


@pytest.mark.parametrize("case", _dense_cases(), ids=lambda c: c[0])
def test_dense_solve_all_modes(case):
    _, n, edges = case
    xs, _ = G.dense_pagerank(n, edges, D)
    g = csr_of(n, edges)
    rep = oracle.identical(g)
    cs, ck, _ = oracle.chains(g, rep)
    plain = oracle.pagerank(g, D, 1e-14, 5000)
    red = oracle.pagerank(g, D, 1e-14, 5000, reduced=True, rep=rep, chain_k=ck)
    gs = oracle.pagerank(g, D, 1e-14, 5000, gauss_seidel=True)
    for r in (plain, red, gs):
        assert r.status == 0
        assert np.abs(r.x - xs).sum() <= 1e-12
    # reductions "change nothing" at the fixed point (north_star (c))
    assert np.abs(red.x - plain.x).sum() <= 1e-12


def test_identical_only_reduction_is_bit_identical():
    """Q-G: equal in-lists give the same fp sum, so identical-only reduced mode
    reproduces plain mode bit for bit, with the same iteration count."""
    n, edges = G.planted_graph(5, n_base=150, chains=())
    g = csr_of(n, edges)
    rep = oracle.identical(g)
    assert (rep != np.arange(n)).sum() > 5
    plain = oracle.pagerank(g, D, 1e-12, 1000)
    red = oracle.pagerank(g, D, 1e-12, 1000, reduced=True, rep=rep, chain_k=np.zeros(n, np.int32))
    assert red.iters == plain.iters
    assert np.array_equal(red.x, plain.x)


def test_chain_relation_exact_in_reduced_mode():
    n, edges = G.planted_graph(9, chains=(16, 4))
    g = csr_of(n, edges)
    rep = oracle.identical(g)
    cs, ck, mk = oracle.chains(g, rep)
    r = oracle.pagerank(g, D, 1e-12, 1000, reduced=True, rep=rep, chain_k=ck)
    c = (1 - D) / n
    for v in np.nonzero(ck > 0)[0]:
        p = g.col_idx[g.row_ptr[v]]
        assert r.x[v] == c + D * (r.x[p] / g.outdeg[p])
    members = np.nonzero(rep != np.arange(n))[0]
    assert np.array_equal(r.x[members], r.x[rep[members]])


# --------------------------------------------------------------- identities --
def test_mass_identity_every_iteration():
    n = 300
    edges = G.random_edges(n, 2 * n, 42)
    g = csr_of(n, edges)
    assert (g.outdeg == 0).any()
    x = np.full(n, 1.0 / n)
    for _ in range(30):
        y = oracle.jacobi_step(g, D, x)
        lhs = math.fsum(y)
        rhs = (1 - D) + D * math.fsum(x[g.outdeg > 0])
        assert abs(lhs - rhs) <= 1e-14
        x = y


def test_mass_is_one_without_dangling():
    n = 200
    edges = G.cycle(n) + G.random_edges(n, 3 * n, 3, loops=False)
    g = csr_of(n, edges)
    assert (g.outdeg > 0).all()
    r = oracle.pagerank(g, D, 1e-13, 1000)
    assert abs(math.fsum(r.x) - 1.0) <= 1e-12


def test_l1_contraction_and_iteration_bound():
    n = 400
    g = csr_of(n, G.random_edges(n, 3 * n, 11))
    tau = 1e-12
    r = oracle.pagerank(g, D, tau, 1000)
    l1 = r.delta_log[:, 0]
    assert (l1[1:] <= D * l1[:-1] * (1 + 1e-9) + 1e-18).all()
    assert r.iters <= 1 + math.ceil(math.log(tau / 2) / math.log(D))


def test_linf_not_monotone_lemma1_counterexample():
    """Q-M: Lemma 1's premise fails; L1 still contracts."""
    a, b, u, a2, b2, u2, v = range(7)
    edges = [(a, u), (b, u), (a2, u2), (b2, u2), (u, v), (u2, v)]
    g = csr_of(7, edges)
    r = oracle.pagerank(g, D, 0.0, 10)
    linf = r.delta_log[:, 1]
    l1 = r.delta_log[:, 0]
    assert (np.diff(linf[:3]) > 0).any()
    assert (l1[1:] <= D * l1[:-1] + 1e-18).all()


def test_stop_rule_delta_equal_tau_stops():
    """Q-S: 'while err > threshold' -- Delta == tau stops."""
    n = 100
    g = csr_of(n, G.random_edges(n, 3 * n, 5))
    full = oracle.pagerank(g, D, 1e-12, 1000)
    k = 20
    tau = full.delta_log[k - 1, 0]
    r = oracle.pagerank(g, D, tau, 1000)
    assert r.iters == k and r.status == 0
    r2 = oracle.pagerank(g, D, np.nextafter(tau, 0), 1000)
    assert r2.iters == k + 1


def test_max_iter_status():
    n = 100
    g = csr_of(n, G.random_edges(n, 3 * n, 5))
    r = oracle.pagerank(g, D, 0.0, 7)
    assert r.status == 2 and r.iters == 7 and r.delta_log.shape[0] == 7


def test_linf_norm_uses_max():
    n = 100
    g = csr_of(n, G.random_edges(n, 3 * n, 5))
    r = oracle.pagerank(g, D, 1e-13, 1000, norm_linf=True)
    assert r.delta_log[-1, 1] <= 1e-13 < r.delta_log[-2, 1]


# ------------------------------------------------------------- certificate --
def test_residual_certificate_bounds_true_error():
    n = 150
    edges = G.random_edges(n, 3 * n, 8)
    xs, M = G.dense_pagerank(n, edges, D)
    g = csr_of(n, edges)
    rng = np.random.default_rng(0)
    for scale in (1e-3, 1e-8, 1e-12):
        x = xs + scale * rng.standard_normal(n) / n
        res, r = oracle.residual_l1(g, D, x, want_r=True)
        np.testing.assert_allclose(r, x - ((1 - D) / n + D * M @ x), rtol=0, atol=1e-16)
        assert np.abs(x - xs).sum() <= res / (1 - D) * (1 + 1e-9) + 1e-16


def test_gauss_seidel_is_in_place_sweep():
    """No-Sync with one thread is Gauss-Seidel; the first sweep
    differs from Jacobi exactly where a smaller id feeds a larger one."""
    g = csr_of(3, [(0, 1), (1, 2), (2, 0)])
    r = oracle.pagerank(g, D, 0.0, 1, gauss_seidel=True)
    c = (1 - D) / 3
    x0 = 1 / 3
    x_0 = c + D * x0
    x_1 = c + D * x_0
    x_2 = c + D * x_1
    np.testing.assert_allclose(r.x, [x_0, x_1, x_2], rtol=1e-15)


# ---- block Gauss-Seidel (reading Q-B) and loop perforation (Alg.5, Q-P) --
BGS = json.load(open(os.path.join(HERE, "golden", "block_gs_examples.json")))


def _frac(s):
    from fractions import Fraction
    return float(Fraction(s))


@pytest.mark.parametrize("ex", BGS["block_gs"], ids=lambda e: e["name"])
def test_block_gs_hand_examples(ex):
    """Hand-derived sweeps (tests/golden/block_gs_examples.json): block bounds
    (no row split at a boundary), in-place reads of the earlier blocks, Jacobi
    reads inside a block, in-degree-0 vertices after the blocks, and Delta."""
    g = csr_of(ex["n"], ex["edges"])
    _, b = oracle.block_bounds(g, ex["K"])
    assert b.tolist() == ex["bounds"]
    r = oracle.pagerank(g, ex["d"], 0.0, ex["sweeps"], blocks=ex["K"])
    assert r.iters == ex["sweeps"]
    np.testing.assert_allclose(r.x, [_frac(s) for s in ex["x"]], rtol=1e-15)
    np.testing.assert_allclose(r.delta_log[:, 0], [_frac(s) for s in ex["l1"]], rtol=1e-14)
    np.testing.assert_allclose(r.delta_log[:, 1], [_frac(s) for s in ex["linf"]], rtol=1e-14)


@pytest.mark.parametrize("seed", range(8))
def test_block_bounds_rule_brute_force(seed):
    """b_k = the first row whose first edge e has e*K >= k*E, over the rows a
    sweep gathers (in-degree > 0; reduced: representatives, not chain
    members), checked against a direct scan of every row start."""
    n, edges = G.planted_graph(300 + seed, n_base=60, chains=(4, 7))
    g = csr_of(n, edges)
    rep = oracle.identical(g)
    _, ck, _ = oracle.chains(g, rep)
    deg = np.diff(g.row_ptr)
    for reduced in (False, True):
        keep = deg > 0
        if reduced:
            keep &= (rep == np.arange(n)) & (ck == 0)
        rows_bf = np.nonzero(keep)[0]
        starts = np.concatenate([[0], np.cumsum(deg[rows_bf])])
        E = int(starts[-1])
        for K in (1, 2, 3, 5, 17, E + 3):
            rows, b = oracle.block_bounds(g, K, reduced, rep, ck)
            assert rows.tolist() == rows_bf.tolist()
            want = [0] + [next((i for i in range(len(rows_bf)) if starts[i] * K >= k * E), len(rows_bf))
                          for k in range(1, K)] + [len(rows_bf)]
            assert b.tolist() == want


def test_block_gs_one_block_is_jacobi():
    """K = 1 is the synchronous sweep, bit for bit (plain and reduced)."""
    n, edges = G.planted_graph(5, n_base=120, chains=(9, 3))
    g = csr_of(n, edges)
    rep = oracle.identical(g)
    _, ck, _ = oracle.chains(g, rep)
    for kw in ({}, {"reduced": True, "rep": rep, "chain_k": ck}):
        a = oracle.pagerank(g, D, 1e-13, 500, **kw)
        b = oracle.pagerank(g, D, 1e-13, 500, blocks=1, **kw)
        assert a.iters == b.iters and np.array_equal(a.x, b.x)
        np.testing.assert_allclose(a.delta_log, b.delta_log, rtol=1e-12, atol=1e-18)


def test_block_gs_one_row_per_block_is_gauss_seidel():
    """A block per row (K = E puts a boundary at every row start) on a graph
    where every vertex has in-edges = the ascending in-place sweep (Alg.3 with
    one thread), bit for bit."""
    n = 90
    g = csr_of(n, G.cycle(n) + G.random_edges(n, 300, 8))
    assert (np.diff(g.row_ptr) > 0).all()
    r = oracle.pagerank(g, D, 0.0, 6, blocks=g.E)
    gs = oracle.pagerank(g, D, 0.0, 6, gauss_seidel=True)
    assert np.array_equal(r.x, gs.x)


@pytest.mark.parametrize("case", _dense_cases()[:5], ids=lambda c: c[0])
@pytest.mark.parametrize("K", [2, 3, 8])
def test_block_gs_reaches_dense_solve(case, K):
    """Any block order reaches the fixed point of (I - dM)x = c1 (Lemma 2,
    P:607-628), plain and reduced."""
    _, n, edges = case
    xs, _ = G.dense_pagerank(n, edges, D)
    g = csr_of(n, edges)
    rep = oracle.identical(g)
    _, ck, _ = oracle.chains(g, rep)
    for kw in ({}, {"reduced": True, "rep": rep, "chain_k": ck}):
        r = oracle.pagerank(g, D, 1e-14, 5000, blocks=K, **kw)
        assert r.status == 0 and np.abs(r.x - xs).sum() <= 1e-12


@pytest.mark.parametrize("ex", BGS["perforate"], ids=lambda e: e["name"])
def test_perforate_hand_example(ex):
    g = csr_of(ex["n"], ex["edges"])
    r = oracle.pagerank(g, ex["d"], ex["tau"], ex["max_iter"], perforate=True, perf_thr=ex["perf_thr"])
    assert r.iters == ex["iters"] and r.status == 0
    np.testing.assert_allclose(r.x, [_frac(s) for s in ex["x"]], rtol=1e-15)
    assert r.frozen.tolist() == ex["frozen"]
    np.testing.assert_allclose(r.delta_log[:, 0], [_frac(s) for s in ex["l1"]], rtol=1e-14, atol=1e-17)


def test_perforate_default_threshold_and_no_freeze_is_jacobi():
    """The threshold is tau * 1e-5: with tau = 0 nothing can freeze
    and the run is the synchronous one bit for bit; with perf_thr = 0 too."""
    n, edges = G.planted_graph(9, n_base=150, chains=(5,))
    g = csr_of(n, edges)
    a = oracle.pagerank(g, D, 0.0, 60)
    for kw in ({}, {"perf_thr": 0.0}):
        b = oracle.pagerank(g, D, 0.0, 60, perforate=True, **kw)
        assert np.array_equal(a.x, b.x) and not b.frozen.any()
    # tau > 0: the default threshold is tau * 1e-5 exactly
    t = 1e-9
    c1 = oracle.pagerank(g, D, t, 500, perforate=True)
    c2 = oracle.pagerank(g, D, t, 500, perforate=True, perf_thr=t * 1e-5)
    assert c1.iters == c2.iters and np.array_equal(c1.x, c2.x) and np.array_equal(c1.frozen, c2.frozen)


def test_perforate_frozen_values_are_constant():
    """A flagged vertex keeps the value of the sweep that flagged it: the
    flags of a run cut at sweep t are a subset of those at t + k, and the
    vertices flagged at t have the same value at t + k."""
    import graphgen
    s, t = graphgen.rmat(14, 16 << 14, seed=3)
    g = oracle.build_csr(1 << 14, s, t)
    tau = 1e-10
    runs = [oracle.pagerank(g, D, tau, m, perforate=True) for m in (80, 90, 100, 500)]
    for a, b in zip(runs, runs[1:]):
        fa = a.frozen.astype(bool)
        assert (b.frozen.astype(bool) | ~fa).all()
        assert np.array_equal(a.x[fa], b.x[fa])
    assert runs[-1].frozen.sum() > 0
    # approximate: near, not at, the fixed point
    exact = oracle.pagerank(g, D, 1e-14, 2000)
    err = np.abs(runs[-1].x - exact.x).sum()
    assert err <= 1e-6
