"""GPU tests of PR_MODE_PHASED: in-place sweeps in K ordered, row-aligned
phases (block Gauss-Seidel, DESIGN.md Q-B; the in-place reads of Alg.3
P:545-565 in a fixed order).

Pins, none of which uses the CUDA path as its own reference:
  * element-wise parity with the oracle's block Gauss-Seidel sweep
    (oracle.pagerank(blocks=K), which derives its blocks itself from the rule
    of reading Q-B), sweep by sweep and converged, plain and reduced;
  * one phase is an in-place Jacobi sweep: bit-identical to PR_MODE_SYNC
    (ranks and sweep count), whose parity with the oracle is pinned elsewhere;
  * K phases reach the oracle's fixed point (residual certificate of the
    original system, and an oracle run at tau/100);
  * the mode is deterministic (fixed phases, fixed-order sums);
  * on R-MAT (many dangling vertices) it needs fewer sweeps than Jacobi.  (Not
    on every graph: on a graph without dangling vertices Jacobi conserves
    sum(x) exactly and its L1 delta falls faster than the in-place one's,
    DESIGN.md Q-Y.)
"""
import numpy as np
import pytest

import graphgen
import oracle
from tests import graphs as G
from tests.test_gpu_parity import D, TOL_V, dev

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_09527_b200 as m
    return m


def run(pr, g, n, tau, mode, max_iter=2000):
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    st, it, fd = g.run(x, D, tau, max_iter, mode=mode)
    return st, it, fd, x.cpu().numpy()


def check_fixed_point(pr, g, ref_g, n, tau, extra=0):
    st, it, fd, x = run(pr, g, n, tau, pr.PR_MODE_PHASED | extra)
    assert st == pr.PR_OK and fd <= tau
    res = oracle.residual_l1(ref_g, D, x)
    tight = oracle.pagerank(ref_g, D, tau / 100, 5000)
    err = np.abs(x - tight.x).sum()
    assert err <= res / (1 - D) + 5.67 * tau / 100 + 1e-15
    assert np.abs(x - tight.x).max() <= max(TOL_V, 10 * tau)
    return it, x


GRAPHS = {
    "planted0": lambda: G.planted_graph(0, n_base=150, chains=(2, 9, 16, 1)),
    "planted3": lambda: G.planted_graph(3, n_base=150, chains=(2, 9, 16, 1)),
    "random": lambda: (400, G.random_edges(400, 1600, 17)),
    "in_star": lambda: (300, G.in_star(300)),
    "path": lambda: (64, G.path(64)),
    "single": lambda: (1, []),
    "no_edges": lambda: (9, []),
}


@pytest.mark.parametrize("name", sorted(GRAPHS))
@pytest.mark.parametrize("span", ["1", ""])
def test_one_phase_is_sync(pr, monkeypatch, name, span):
    monkeypatch.setenv("PRGPU_PHASES", "1")
    if span:
        monkeypatch.setenv("PRGPU_SPAN", span)
    n, edges = GRAPHS[name]()
    s, t = G.edges_to_arrays(edges)
    with pr.Graph(n, dev(s), dev(t)) as g:
        g.preprocess()
        for extra in (0, pr.PR_USE_REDUCTIONS, pr.PR_NORM_LINF):
            # (the phased mode resolves chains eagerly, Q-C: compare with the eager sync form)
            a = run(pr, g, n, 1e-12, extra | (pr.PR_CHAIN_EAGER if extra & pr.PR_USE_REDUCTIONS else 0))
            b = run(pr, g, n, 1e-12, pr.PR_MODE_PHASED | extra)
            assert a[:3] == b[:3] and np.array_equal(a[3], b[3]), (extra, a[:3], b[:3])
            assert g.stats()["phases"] == 1


@pytest.mark.parametrize("name", sorted(GRAPHS))
@pytest.mark.parametrize("phases", ["2", "8", "64"])
def test_phased_fixed_point(pr, monkeypatch, name, phases):
    monkeypatch.setenv("PRGPU_PHASES", phases)
    monkeypatch.setenv("PRGPU_SPAN", "1")  # many spans, so the phases really split the rows
    n, edges = GRAPHS[name]()
    s, t = G.edges_to_arrays(edges)
    ref_g = oracle.build_csr(n, s, t)
    with pr.Graph(n, dev(s), dev(t)) as g:
        check_fixed_point(pr, g, ref_g, n, 1e-12)
        g.preprocess()
        check_fixed_point(pr, g, ref_g, n, 1e-12, pr.PR_USE_REDUCTIONS)


@pytest.mark.parametrize("cfg", [2, 3])
def test_phased_configs(pr, monkeypatch, cfg):
    monkeypatch.setenv("PRGPU_PHASES", "8")
    gen = graphgen.make_config(cfg)
    ref_g = oracle.build_csr(gen.n, gen.src, gen.dst)
    with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g:
        it, x = check_fixed_point(pr, g, ref_g, gen.n, gen.tau)
        assert g.stats()["phases"] > 1
        again = run(pr, g, gen.n, gen.tau, pr.PR_MODE_PHASED)
        assert again[1] == it and np.array_equal(again[3], x)  # deterministic
        g.preprocess()
        it_r, _ = check_fixed_point(pr, g, ref_g, gen.n, gen.tau, pr.PR_USE_REDUCTIONS)


def test_phased_default_phase_count(pr):
    """Small graphs default to one phase (the launches would cost more than
    the sweeps saved); PRGPU_PHASES overrides."""
    gen = graphgen.make_config(2)
    with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g:
        run(pr, g, gen.n, gen.tau, pr.PR_MODE_PHASED)
        assert g.stats()["phases"] == 1


def test_phased_rmat_fewer_sweeps(pr, monkeypatch):
    """R-MAT (config 4's generator at scale 16): the phased sweep count drops
    well below Jacobi's, and stays deterministic across runs."""
    monkeypatch.setenv("PRGPU_PHASES", "8")
    gen = graphgen.make_config(4, scale_override=16)
    ref_g = oracle.build_csr(gen.n, gen.src, gen.dst)
    with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g:
        it_sync = run(pr, g, gen.n, gen.tau, 0)[1]
        it, x = check_fixed_point(pr, g, ref_g, gen.n, gen.tau)
        assert it < it_sync, (it, it_sync)
        again = run(pr, g, gen.n, gen.tau, pr.PR_MODE_PHASED)
        assert again[1] == it and np.array_equal(again[3], x)


def test_phased_blocked_view_runs_one_phase(pr, monkeypatch):
    monkeypatch.setenv("PRGPU_SEG_BITS", "6")
    n, edges = G.planted_graph(1, n_base=150, chains=(2, 9, 16, 1))
    s, t = G.edges_to_arrays(edges)
    with pr.Graph(n, dev(s), dev(t)) as g:
        a = run(pr, g, n, 1e-12, 0)
        b = run(pr, g, n, 1e-12, pr.PR_MODE_PHASED)
        assert g.stats()["phases"] == 1
        assert a[:3] == b[:3] and np.array_equal(a[3], b[3])


def test_phased_mode_validation(pr):
    n = 50
    s, t = G.edges_to_arrays(G.random_edges(n, 200, 3))
    with pr.Graph(n, dev(s), dev(t)) as g:
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        for bad in (pr.PR_MODE_ASYNC, pr.PR_MODE_NOSYNC, pr.PR_PERFORATE):
            with pytest.raises(pr.PRError) as e:
                pr.pr_run(g.handle, D, 1e-10, 10, x, mode=pr.PR_MODE_PHASED | bad)
            assert e.value.code == pr.PR_EINVAL


def _oracle_reductions(ref_g):
    rep = oracle.identical(ref_g)
    _, ck, _ = oracle.chains(ref_g, rep)
    return rep, ck


@pytest.mark.parametrize("name", ["planted0", "planted3", "random", "in_star", "path"])
@pytest.mark.parametrize("phases", ["2", "3", "8", "64"])
def test_phased_matches_oracle_block_gs(pr, monkeypatch, name, phases):
    """Sweep by sweep (tau = 0, 1 and 3 sweeps) and converged, plain and
    reduced: the GPU's phased run equals the oracle's block Gauss-Seidel run
    with the same K element by element; the GPU's phase plan equals the blocks
    the oracle derives from the rule (row bounds)."""
    monkeypatch.setenv("PRGPU_PHASES", phases)
    monkeypatch.setenv("PRGPU_SPAN", "1")  # many spans: boundary rows inside the phases
    K = int(phases)
    n, edges = GRAPHS[name]()
    s, t = G.edges_to_arrays(edges)
    ref_g = oracle.build_csr(n, s, t)
    rep, ck = _oracle_reductions(ref_g)
    with pr.Graph(n, dev(s), dev(t)) as g:
        g.preprocess()
        for reduced in (False, True):
            extra = pr.PR_USE_REDUCTIONS if reduced else 0
            kw = {"reduced": True, "rep": rep, "chain_k": ck} if reduced else {}
            for sweeps in (1, 3):
                st, it, fd, x = run(pr, g, n, 0.0, pr.PR_MODE_PHASED | extra, max_iter=sweeps)
                assert it == sweeps and g.stats()["phases"] == K
                ref = oracle.pagerank(ref_g, D, 0.0, sweeps, blocks=K, **kw)
                np.testing.assert_allclose(x, ref.x, rtol=1e-13, atol=1e-18)
                np.testing.assert_allclose(g.delta_log()[:, 0], ref.delta_log[:, 0], rtol=1e-9, atol=1e-18)
            eb, rb = pr.pr_get_phase_plan(g.handle, reduced)
            _, ob = oracle.block_bounds(ref_g, K, reduced, rep, ck)
            assert rb.tolist() == ob.tolist()
            st, it, fd, x = run(pr, g, n, 1e-12, pr.PR_MODE_PHASED | extra)
            ref = oracle.pagerank(ref_g, D, 1e-12, 2000, blocks=K, **kw)
            assert st == pr.PR_OK and abs(it - ref.iters) <= 1
            if it != ref.iters:
                assert abs(ref.delta - 1e-12) <= 1e-3 * 1e-12
            assert np.abs(x - ref.x).max() <= TOL_V and np.abs(x - ref.x).sum() <= 1e-9


@pytest.mark.parametrize("cfg", [2, 3])
def test_phased_configs_match_oracle_block_gs(pr, monkeypatch, cfg):
    """Configs 2 and 3 at their tau, 8 phases: iteration count within +/-1
    and ranks within 1e-10 of the oracle's block Gauss-Seidel run (plain)."""
    monkeypatch.setenv("PRGPU_PHASES", "8")
    gen = graphgen.make_config(cfg)
    ref_g = oracle.build_csr(gen.n, gen.src, gen.dst)
    ref = oracle.pagerank(ref_g, D, gen.tau, gen.max_iter, blocks=8)
    with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g:
        st, it, fd, x = run(pr, g, gen.n, gen.tau, pr.PR_MODE_PHASED)
        assert st == pr.PR_OK and g.stats()["phases"] == 8
        assert abs(it - ref.iters) <= 1
        assert np.abs(x - ref.x).max() <= TOL_V and np.abs(x - ref.x).sum() <= 1e-9


def test_phase_plan_errors(pr):
    n = 30
    s, t = G.edges_to_arrays(G.random_edges(n, 90, 4))
    with pr.Graph(n, dev(s), dev(t)) as g:
        with pytest.raises(pr.PRError) as e:
            pr.pr_get_phase_plan(g.handle)
        assert e.value.code == pr.PR_ESTATE
