"""GPU tests of the edge-stream gather's decomposition (streamengine.cuh).

The sync sweep is K-GATHER (flat edge stream: steps of 256 edges, spans of
steps per warp, boundary rows assembled from per-span pieces by a ticket) +
K-FINALIZE.  Its result must not depend on how the edge array is cut:
  * span size (PRGPU_SPAN, read at graph build) changes only the summation
    association -> oracle tolerance, iteration count +/-1 rule;
  * the shared-memory hot tier (PRGPU_HOT) changes only WHERE a contrib is
    read from -> bit-identical ranks and Delta logs;
  * source-blocked views (PRGPU_SEG_BITS) -> oracle tolerance, in every mode.
"""
import numpy as np
import pytest

import graphgen
import oracle
from tests import graphs as G
from tests.test_gpu_parity import D, assert_close, assert_iters, dev, gpu_run

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_09527_b200 as m
    return m


def hub_graph(n=6000, seed=5):
    """Random graph plus two long rows (a 5000-edge hub and a 700-edge row) and
    a block of in-degree-1 rows, so rows start and end at every position of a
    step and cross many span boundaries."""
    rng = np.random.default_rng(seed)
    edges = list(zip(rng.integers(0, n, 6 * n).tolist(), rng.integers(0, n, 6 * n).tolist()))
    edges += [(int(u), 3) for u in rng.permutation(n)[:5000]]
    edges += [(int(u), 4000) for u in rng.permutation(n)[:700]]
    edges += [(int(v) - 1, int(v)) for v in range(100, 400)]
    s, t = G.edges_to_arrays(edges)
    return n, s, t


@pytest.mark.parametrize("span", [1, 2, 3, 5, 17, 1000])
def test_span_sizes_match_oracle(pr, monkeypatch, span):
    monkeypatch.setenv("PRGPU_SPAN", str(span))
    n, s, t = hub_graph()
    ref_g = oracle.build_csr(n, s, t)
    ref = oracle.pagerank(ref_g, D, 1e-12, 1000)
    rep_o = oracle.identical(ref_g)
    cs_o, ck_o, _ = oracle.chains(ref_g, rep_o)
    ref_r = oracle.pagerank(ref_g, D, 1e-12, 1000, reduced=True, rep=rep_o, chain_k=ck_o)
    with pr.Graph(n, dev(s), dev(t)) as g:
        st, it, fd, x = gpu_run(pr, g, n, 1e-12)
        assert_iters(it, ref, 1e-12)
        assert_close(x, ref.x)
        g.preprocess()
        st, it, fd, xr = gpu_run(pr, g, n, 1e-12, mode=pr.PR_USE_REDUCTIONS | pr.PR_CHAIN_EAGER)
        assert_iters(it, ref_r, 1e-12)
        assert_close(xr, ref_r.x)


@pytest.mark.parametrize("span", [1, 4])
def test_single_long_row_spans(pr, monkeypatch, span):
    """One row holding every edge (in-star): its pieces cross all spans."""
    monkeypatch.setenv("PRGPU_SPAN", str(span))
    n = 20000
    s, t = G.edges_to_arrays(G.in_star(n))
    ref_g = oracle.build_csr(n, s, t)
    ref = oracle.pagerank(ref_g, D, 1e-13, 1000)
    with pr.Graph(n, dev(s), dev(t)) as g:
        st, it, fd, x = gpu_run(pr, g, n, 1e-13)
        assert it == ref.iters
        assert_close(x, ref.x)


def test_hot_tier_is_bit_identical(pr, monkeypatch):
    gen = graphgen.make_config(4, scale_override=14)
    runs = []
    with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g:
        g.preprocess()
        for hot in ("0", "1", "7", "4096", "16384"):
            monkeypatch.setenv("PRGPU_HOT", hot)
            for mode in (0, pr.PR_USE_REDUCTIONS):
                st, it, fd, x = gpu_run(pr, g, gen.n, 1e-10, mode=mode)
                runs.append((hot, mode, it, x, g.delta_log()))
    for mode in (0, pr.PR_USE_REDUCTIONS):
        rs = [r for r in runs if r[1] == mode]
        for r in rs[1:]:
            assert r[2] == rs[0][2]
            assert np.array_equal(r[3], rs[0][3]), (r[0], mode)
            assert np.array_equal(r[4], rs[0][4])


def test_stream_deterministic_across_graph_builds(pr):
    gen = graphgen.make_config(2, scale_override=16)
    xs = []
    for _ in range(2):
        with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g:
            g.preprocess()
            xs.append(gpu_run(pr, g, gen.n, 1e-10, mode=pr.PR_USE_REDUCTIONS)[3])
    assert np.array_equal(xs[0], xs[1])


@pytest.mark.parametrize("bits", [3, 6, 10])
def test_blocked_segments_match_oracle(pr, monkeypatch, bits):
    """Source-blocked sweeps (PRGPU_SEG_BITS forces 2^bits contrib slots per
    segment): the per-segment partial sums add up to the oracle's result."""
    monkeypatch.setenv("PRGPU_SEG_BITS", str(bits))
    n, s, t = hub_graph()
    ref_g = oracle.build_csr(n, s, t)
    ref = oracle.pagerank(ref_g, D, 1e-12, 1000)
    rep_o = oracle.identical(ref_g)
    cs_o, ck_o, _ = oracle.chains(ref_g, rep_o)
    ref_r = oracle.pagerank(ref_g, D, 1e-12, 1000, reduced=True, rep=rep_o, chain_k=ck_o)
    with pr.Graph(n, dev(s), dev(t)) as g:
        st, it, fd, x = gpu_run(pr, g, n, 1e-12)
        assert_iters(it, ref, 1e-12)
        assert_close(x, ref.x)
        a = gpu_run(pr, g, n, 1e-12)[3]
        assert np.array_equal(a, x)                      # deterministic
        g.preprocess()
        st, it, fd, xr = gpu_run(pr, g, n, 1e-12, mode=pr.PR_USE_REDUCTIONS | pr.PR_CHAIN_EAGER)
        assert_iters(it, ref_r, 1e-12)
        assert_close(xr, ref_r.x)
        st, it, fd, xd = gpu_run(pr, g, n, 1e-12, mode=pr.PR_USE_REDUCTIONS)   # delayed: the plain run
        assert_iters(it, ref, 1e-12)
        assert_close(xd, ref.x)


def test_blocked_rmat(pr, monkeypatch):
    monkeypatch.setenv("PRGPU_SEG_BITS", "8")
    gen = graphgen.make_config(4, scale_override=14)
    ref_g = oracle.build_csr(gen.n, gen.src, gen.dst)
    ref = oracle.pagerank(ref_g, D, 1e-10, 1000)
    with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g:
        st, it, fd, x = gpu_run(pr, g, gen.n, 1e-10)
        assert_iters(it, ref, 1e-10)
        assert_close(x, ref.x)


@pytest.mark.parametrize("bits", [4, 8])
def test_blocked_views_with_every_mode(pr, monkeypatch, bits):
    """Source-blocked views: the in-place modes run on the Jacobi schedule
    (reading Q-Y2), No-Sync adds its certificate (a blocked sync gather),
    perforation runs blocked first, unblocked after compaction -- all must
    reach the oracle's fixed point (perforation: the oracle's perforated run;
    with ASYNC / NOSYNC it is the same synchronous perforated run, Q-Y2)."""
    monkeypatch.setenv("PRGPU_SEG_BITS", str(bits))
    n, s, t = hub_graph(seed=11)
    ref_g = oracle.build_csr(n, s, t)
    tight = oracle.pagerank(ref_g, D, 1e-14, 5000)
    with pr.Graph(n, dev(s), dev(t)) as g:
        g.preprocess()
        for mode in (pr.PR_MODE_ASYNC, pr.PR_MODE_NOSYNC, pr.PR_MODE_NOSYNC | pr.PR_USE_REDUCTIONS,
                     pr.PR_MODE_ASYNC | pr.PR_USE_REDUCTIONS):
            st, it, fd, x = gpu_run(pr, g, n, 1e-12, max_iter=5000, mode=mode)
            assert st == pr.PR_OK
            assert np.abs(x - tight.x).max() <= 1e-10, mode
        # perforation (Alg.5): a vertex can freeze where its change crosses zero,
        # so the result is compared with the oracle's perforated run, not x*
        st, it, fd, x = gpu_run(pr, g, n, 1e-12, mode=pr.PR_PERFORATE)
        ref_p = oracle.pagerank(ref_g, D, 1e-12, 1000, perforate=True)
        assert st == pr.PR_OK and abs(it - ref_p.iters) <= 1
        assert np.abs(x - ref_p.x).max() <= 1e-10 and np.abs(x - ref_p.x).sum() <= 1e-9
        for extra in (pr.PR_MODE_ASYNC, pr.PR_MODE_NOSYNC):
            st2, it2, _, x2 = gpu_run(pr, g, n, 1e-12, mode=pr.PR_PERFORATE | extra)
            assert st2 == st and it2 == it and np.array_equal(x2, x)


def test_perforation_can_freeze_everything(pr):
    """A graph that converges row by row (a long path) lets perforation freeze
    rows until the active view is empty; the run still ends correctly."""
    n = 3000
    s, t = G.edges_to_arrays(G.path(n))
    ref_g = oracle.build_csr(n, s, t)
    ref = oracle.pagerank(ref_g, D, 1e-13, 5000)
    with pr.Graph(n, dev(s), dev(t)) as g:
        for mode in (pr.PR_PERFORATE, pr.PR_PERFORATE | pr.PR_MODE_ASYNC, pr.PR_PERFORATE | pr.PR_MODE_NOSYNC):
            st, it, fd, x = gpu_run(pr, g, n, 1e-13, max_iter=5000, mode=mode)
            assert st == pr.PR_OK, mode
            assert np.abs(x - ref.x).max() <= 1e-12, mode
