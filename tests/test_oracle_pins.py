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


# ---- the phased-sweep model (reading Q-B), pinned to Jacobi and Gauss-Seidel
def _phased_inputs(n, edges):
    from tests import graphs as G
    s, t = G.edges_to_arrays(edges)
    g = oracle.build_csr(n, s, t)
    rows = np.nonzero(np.diff(g.row_ptr) > 0)[0]
    return g, rows


def test_phased_model_one_phase_is_jacobi():
    """One phase over the whole stream = the synchronous sweep (Eq.(1))."""
    from tests import graphs as G
    n = 120
    g, rows = _phased_inputs(n, G.random_edges(n, 500, 5) + [(0, 1)])
    E = int(g.row_ptr[-1])
    x, log = oracle.phased_sweeps(g, 0.85, 4, rows, [0, E], [0, len(rows)])
    ref = oracle.pagerank(g, 0.85, 0.0, 4)
    assert np.array_equal(x, ref.x)
    np.testing.assert_allclose(log, ref.delta_log, rtol=1e-12, atol=1e-18)


def test_phased_model_one_row_per_phase_is_gauss_seidel():
    """One row per phase, rows ascending, every vertex with in-edges = the
    in-place ascending sweep (Alg.3 with one thread), bit for bit."""
    from tests import graphs as G
    n = 90
    edges = G.cycle(n) + G.random_edges(n, 300, 8)     # every vertex has in-degree >= 1
    g, rows = _phased_inputs(n, edges)
    assert len(rows) == n
    eb = list(g.row_ptr)                              # a phase boundary at every row start
    rb = list(range(n + 1))
    x, log = oracle.phased_sweeps(g, 0.85, 5, rows, eb, rb)
    ref = oracle.pagerank(g, 0.85, 0.0, 5, gauss_seidel=True)
    np.testing.assert_allclose(x, ref.x, rtol=1e-15, atol=0)
    np.testing.assert_allclose(log[:, 1], ref.delta_log[:, 1], rtol=1e-12, atol=1e-18)


def test_phased_model_reaches_the_fixed_point():
    """Any block order converges to the same fixed point (Lemma 2)."""
    from tests import graphs as G
    n = 150
    g, rows = _phased_inputs(n, G.random_edges(n, 600, 13))
    E = int(g.row_ptr[-1])
    eb = [0, E // 3, (2 * E) // 3, E]
    # rows ending in each edge range
    ends = g.row_ptr[rows + 1]
    rb = [0] + [int(np.searchsorted(ends, b, side="right")) for b in eb[1:-1]] + [len(rows)]
    x, _ = oracle.phased_sweeps(g, 0.85, 200, rows, eb, rb)
    tight = oracle.pagerank(g, 0.85, 1e-15, 2000)
    assert np.abs(x - tight.x).max() <= 1e-12
