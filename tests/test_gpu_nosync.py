"""GPU tests of PR_MODE_NOSYNC: the persistent barrier-free No-Sync kernel
(Alg.3; thread-level convergence P:416-418).

The result is not deterministic (CTAs race), so parity is pinned through the
fixed point (Lemma 2): the library certifies ||F(x) - x|| <= tau of
the ORIGINAL system, and the oracle checks the same certificate plus the
distance to an oracle run at tau/100 (||x - x*||_1 <= ||F(x)-x||_1 / (1-d)).
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


def run_nosync(pr, g, n, tau, extra=0, max_iter=5000):
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    st, it, fd = g.run(x, D, tau, max_iter, mode=pr.PR_MODE_NOSYNC | extra)
    return st, it, fd, x.cpu().numpy()


def check_nosync(pr, g, ref_g, n, tau, extra=0):
    st, it, fd, x = run_nosync(pr, g, n, tau, extra)
    assert st == pr.PR_OK, st
    stats = g.stats()
    assert fd <= tau and stats["residual"] == fd
    assert 1 <= stats["nosync_min_iters"] <= stats["nosync_median_iters"] <= stats["iterations"] == it
    res = oracle.residual_l1(ref_g, D, x)              # independent certificate
    assert res <= tau * (1 + 1e-6) + 1e-15 or extra & pr.PR_NORM_LINF
    tight = oracle.pagerank(ref_g, D, tau / 100, 5000)
    err = np.abs(x - tight.x).sum()
    assert err <= res / (1 - D) + 5.67 * tau / 100 + 1e-15
    assert np.abs(x - tight.x).max() <= max(TOL_V, 10 * tau)
    log = g.delta_log()
    assert log.shape == (stats["nosync_launches"], 2) and log[-1, 0] == stats["delta_l1"]
    return it, stats


HAND = {
    "single": (1, []),
    "two_cycle": (2, G.cycle(2)),
    "cycle17": (17, G.cycle(17)),
    "in_star": (50, G.in_star(50)),
    "out_star": (50, G.out_star(50)),
    "path": (40, G.path(40)),
    "complete": (12, G.complete(12)),
    "no_edges": (7, []),
}


@pytest.mark.parametrize("name", sorted(HAND))
def test_nosync_hand_graphs(pr, name):
    n, edges = HAND[name]
    s, t = G.edges_to_arrays(edges)
    ref_g = oracle.build_csr(n, s, t)
    with pr.Graph(n, dev(s), dev(t)) as g:
        check_nosync(pr, g, ref_g, n, 1e-13)


@pytest.mark.parametrize("seed", range(4))
def test_nosync_planted_plain_and_reduced(pr, seed):
    n, edges = G.planted_graph(seed, n_base=150, chains=(2, 9, 16, 1))
    s, t = G.edges_to_arrays(edges)
    ref_g = oracle.build_csr(n, s, t)
    with pr.Graph(n, dev(s), dev(t)) as g:
        check_nosync(pr, g, ref_g, n, 1e-12)
        g.preprocess()
        check_nosync(pr, g, ref_g, n, 1e-12, pr.PR_USE_REDUCTIONS)


def test_nosync_linf(pr):
    n = 400
    s, t = G.edges_to_arrays(G.random_edges(n, 4 * n, 91))
    ref_g = oracle.build_csr(n, s, t)
    with pr.Graph(n, dev(s), dev(t)) as g:
        st, it, fd, x = run_nosync(pr, g, n, 1e-14, pr.PR_NORM_LINF)
        assert st == pr.PR_OK and fd <= 1e-14
        tight = oracle.pagerank(ref_g, D, 1e-16, 5000)
        assert np.abs(x - tight.x).max() <= 1e-12


@pytest.mark.parametrize("cfg", [2, 3])
def test_nosync_configs(pr, cfg):
    gen = graphgen.make_config(cfg)
    ref_g = oracle.build_csr(gen.n, gen.src, gen.dst)
    with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g:
        check_nosync(pr, g, ref_g, gen.n, gen.tau)
        g.preprocess()
        check_nosync(pr, g, ref_g, gen.n, gen.tau, pr.PR_USE_REDUCTIONS)


def test_nosync_max_iter_and_modes(pr):
    n = 300
    s, t = G.edges_to_arrays(G.random_edges(n, 3 * n, 5))
    with pr.Graph(n, dev(s), dev(t)) as g:
        st, it, fd, x = run_nosync(pr, g, n, 0.0, max_iter=3)
        assert st == pr.PR_NOT_CONVERGED and it == 3
        x0 = torch.empty(n, dtype=torch.float64, device="cuda")
        with pytest.raises(pr.PRError) as e:
            pr.pr_run(g.handle, D, 1e-10, 10, x0, mode=pr.PR_MODE_NOSYNC | pr.PR_MODE_ASYNC)
        assert e.value.code == pr.PR_EINVAL


def test_sync_after_nosync_is_unaffected(pr, monkeypatch):
    """A persistent No-Sync launch stops with its CTAs at different sweeps, so
    the boundary-row tickets it shares with the synchronous engine can be left
    mid-count; the following synchronous runs must still be bit-identical to a
    fresh graph's (one-step spans: every row crossing a step is a boundary row)."""
    monkeypatch.setenv("PRGPU_SPAN", "1")
    gen = graphgen.make_config(4, scale_override=14)
    with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g0:
        x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
        g0.run(x, D, 1e-10, 1000)
        fresh = x.cpu().numpy()
        g0.run(x, D, 1e-10, 1000, mode=pr.PR_PERFORATE)
        fresh_pf = x.cpu().numpy()
    with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g:
        x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
        for _ in range(3):
            g.run(x, D, 1e-10, 1000, mode=pr.PR_MODE_NOSYNC)
            g.run(x, D, 1e-10, 1000)
            assert np.array_equal(x.cpu().numpy(), fresh)
            g.run(x, D, 1e-10, 1000, mode=pr.PR_MODE_NOSYNC)
            g.run(x, D, 1e-10, 1000, mode=pr.PR_PERFORATE)
            assert np.array_equal(x.cpu().numpy(), fresh_pf)
