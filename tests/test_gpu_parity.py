"""GPU parity: libprgpu (through the C ABI) vs the CPU fp64 oracle.

Bars (BASELINE.json north_star):
  * integer outputs (in-CSR, outdeg, identical reps, chains) bit-exact;
  * sync mode: per-vertex |diff| <= 1e-10, L1 <= 1e-9, iterations within +/-1
    of the oracle in the same mode (a +/-1 is accepted only where the
    oracle's Delta at the boundary is within 1e-9*tau of tau);
  * async mode: same fixed point, pinned by the oracle's residual
    certificate ||x - x*||_1 <= ||r(x)||_1 / (1-d) and by an oracle run at tau/100.
"""
import numpy as np
import pytest

import graphgen
import oracle
from tests import graphs as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

D = 0.85
TOL_V = 1e-10
TOL_L1 = 1e-9


@pytest.fixture(scope="module")
def pr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_09527_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_graph(pr, n, src, dst):
    return pr.Graph(n, dev(src), dev(dst))


def gpu_csr(pr, g, n, E):
    rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    col = torch.empty(max(E, 1), dtype=torch.int32, device="cuda")
    od = torch.empty(n, dtype=torch.int32, device="cuda")
    pr.pr_get_csr(g.handle, rp, col, od)
    return rp.cpu().numpy(), col[:E].cpu().numpy(), od.cpu().numpy()


def gpu_reductions(pr, g, n):
    rep = torch.empty(n, dtype=torch.int32, device="cuda")
    cs = torch.empty(n, dtype=torch.int32, device="cuda")
    ck = torch.empty(n, dtype=torch.int32, device="cuda")
    pr.pr_get_reductions(g.handle, rep, cs, ck)
    return rep.cpu().numpy(), cs.cpu().numpy(), ck.cpu().numpy()


def gpu_run(pr, g, n, tau, max_iter=1000, mode=0):
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    st, it, fd = g.run(x, D, tau, max_iter, mode=mode)
    return st, it, fd, x.cpu().numpy()


def assert_iters(it_gpu, ref, tau, linf=False):
    if it_gpu == ref.iters:
        return
    assert abs(it_gpu - ref.iters) == 1, (it_gpu, ref.iters)
    k = min(it_gpu, ref.iters)
    dk = ref.delta_log[k - 1, 1 if linf else 0]
    assert abs(dk - tau) <= 1e-9 * tau, f"+/-1 iteration mismatch away from the threshold: {dk} vs {tau}"


def assert_close(xg, xo):
    diff = np.abs(xg - xo)
    assert diff.max() <= TOL_V, diff.max()
    assert diff.sum() <= TOL_L1, diff.sum()


def check_all(pr, n, src, dst, tau=1e-12, reductions=True, async_mode=True):
    ref_g = oracle.build_csr(n, src, dst)
    with gpu_graph(pr, n, src, dst) as g:
        info = g.info()
        assert info["E"] == ref_g.E
        rp, col, od = gpu_csr(pr, g, n, ref_g.E)
        assert np.array_equal(rp, ref_g.row_ptr)
        assert np.array_equal(col, ref_g.col_idx)
        assert np.array_equal(od, ref_g.outdeg)
        ref = oracle.pagerank(ref_g, D, tau, 1000)
        st, it, fd, xg = gpu_run(pr, g, n, tau)
        assert st == ref.status
        assert_iters(it, ref, tau)
        assert_close(xg, ref.x)
        if reductions:
            g.preprocess(pr.PR_PRE_IDENTICAL | pr.PR_PRE_CHAIN)
            rep_o = oracle.identical(ref_g)
            cs_o, ck_o, mk = oracle.chains(ref_g, rep_o)
            rep, cs, ck = gpu_reductions(pr, g, n)
            assert np.array_equal(rep, rep_o)
            assert np.array_equal(cs, cs_o)
            assert np.array_equal(ck, ck_o)
            assert g.info()["max_chain"] == mk
            # delayed chain resolution (default, Q-C2): the plain trajectory
            st, it, fd, xr = gpu_run(pr, g, n, tau, mode=pr.PR_USE_REDUCTIONS)
            assert_iters(it, ref, tau)
            assert_close(xr, ref.x)
            members = np.nonzero(rep_o != np.arange(n))[0]
            assert np.array_equal(xr[members], xr[rep_o[members]])  # exact copies
            # eager (same-sweep) chain resolution: the oracle's reduced mode (Q-C)
            ref_r = oracle.pagerank(ref_g, D, tau, 1000, reduced=True, rep=rep_o, chain_k=ck_o)
            st, it, fd, xe = gpu_run(pr, g, n, tau, mode=pr.PR_USE_REDUCTIONS | pr.PR_CHAIN_EAGER)
            assert_iters(it, ref_r, tau)
            assert_close(xe, ref_r.x)
            assert np.array_equal(xe[members], xe[rep_o[members]])
        if async_mode:
            check_async(pr, g, ref_g, n, tau)
    return ref_g


def check_async(pr, g, ref_g, n, tau, mode_extra=0):
    st, it, fd, xa = gpu_run(pr, g, n, tau, mode=pr.PR_MODE_ASYNC | mode_extra)
    assert st == 0 and fd <= tau
    res = oracle.residual_l1(ref_g, D, xa)
    tight = oracle.pagerank(ref_g, D, tau / 100, 5000)
    err = np.abs(xa - tight.x).sum()
    # certificate: ||xa - x*||_1 <= res/(1-d); oracle at tau/100 is within 5.67*tau/100 of x*
    assert err <= res / (1 - D) + 5.67 * tau / 100 + 1e-15
    assert np.abs(xa - tight.x).max() <= max(TOL_V, 10 * tau)
    return it


# ------------------------------------------------------------- hand graphs --
HAND = {
    "single": (1, []),
    "two_cycle": (2, G.cycle(2)),
    "cycle17": (17, G.cycle(17)),
    "in_star": (50, G.in_star(50)),
    "out_star": (50, G.out_star(50)),
    "path": (40, G.path(40)),
    "long_path": (300, G.path(300)),      # chain longer than the 64-link serial walk: pointer jumping resumes
    "cycle_tail": (90, G.cycle(20) + [(i, i + 1) for i in range(19, 89)]),   # 68-long chain off a cycle
    "complete": (12, G.complete(12)),
    "no_edges": (7, []),
    "loops_only": (5, [(i, i) for i in range(5)] * 3),
    "dups_only": (4, [(0, 1)] * 50),
    "spec_csr2": (2, [(0, 1), (0, 1), (0, 0)]),
}


@pytest.mark.parametrize("name", sorted(HAND))
def test_hand_graphs(pr, name):
    n, edges = HAND[name]
    s, t = G.edges_to_arrays(edges)
    check_all(pr, n, s, t, tau=1e-13)


def test_single_vertex_closed_form(pr):
    with gpu_graph(pr, 1, np.zeros(0, np.int32), np.zeros(0, np.int32)) as g:
        st, it, fd, x = gpu_run(pr, g, 1, 1e-12)
        assert x.tolist() == [1 - D] and it == 2 and st == 0


def test_cycle_uniform_closed_form(pr):
    n = 1000
    s, t = G.edges_to_arrays(G.cycle(n))
    with gpu_graph(pr, n, s, t) as g:
        st, it, fd, x = gpu_run(pr, g, n, 1e-12)
        np.testing.assert_allclose(x, 1.0 / n, rtol=1e-14)
        assert it == 1


@pytest.mark.parametrize("seed", range(6))
def test_random_small(pr, seed):
    n = [3, 10, 64, 100, 150, 200][seed]
    edges = G.random_edges(n, 4 * n, 1000 + seed)
    s, t = G.edges_to_arrays(edges)
    ref_g = check_all(pr, n, s, t)
    rp, col, od = G.bf_csr(n, edges)                 # brute force too
    assert ref_g.row_ptr.tolist() == rp and ref_g.col_idx.tolist() == col


@pytest.mark.parametrize("seed", range(4))
def test_planted(pr, seed):
    n, edges = G.planted_graph(seed, n_base=150, chains=(2, 9, 16, 1))
    s, t = G.edges_to_arrays(edges)
    check_all(pr, n, s, t)


# ------------------------------------------------------------- edge cases --
def test_invalid_ids_rejected(pr):
    s = np.array([0, 1, 5], np.int32)
    t = np.array([1, 2, 0], np.int32)
    with pytest.raises(pr.PRError) as e:
        pr.Graph(5, dev(s), dev(t))
    assert e.value.code == pr.PR_EINVAL
    with pytest.raises(pr.PRError):
        pr.Graph(5, dev(np.array([-1], np.int32)), dev(np.array([0], np.int32)))


def test_run_argument_errors(pr):
    s, t = G.edges_to_arrays(G.cycle(5))
    with gpu_graph(pr, 5, s, t) as g:
        x = torch.empty(5, dtype=torch.float64, device="cuda")
        for d, tau, mi in [(0.0, 1e-10, 10), (1.0, 1e-10, 10), (0.85, -1.0, 10), (0.85, float("nan"), 10),
                           (0.85, 1e-10, 0)]:
            with pytest.raises(pr.PRError) as e:
                pr.pr_run(g.handle, d, tau, mi, x)
            assert e.value.code == pr.PR_EINVAL
        with pytest.raises(pr.PRError) as e:
            pr.pr_run(g.handle, 0.85, 1e-10, 10, x, mode=pr.PR_USE_REDUCTIONS)
        assert e.value.code == pr.PR_ESTATE


def test_max_iter_and_tau_zero(pr):
    n = 300
    s, t = G.edges_to_arrays(G.random_edges(n, 3 * n, 77))
    ref_g = oracle.build_csr(n, s, t)
    ref = oracle.pagerank(ref_g, D, 0.0, 7)
    with gpu_graph(pr, n, s, t) as g:
        st, it, fd, x = gpu_run(pr, g, n, 0.0, max_iter=7)
        assert st == pr.PR_NOT_CONVERGED and it == 7
        assert_close(x, ref.x)
        log = g.delta_log()
        assert log.shape == (7, 2)
        np.testing.assert_allclose(log, ref.delta_log, rtol=1e-9, atol=1e-18)


def test_linf_norm_mode(pr):
    n = 300
    s, t = G.edges_to_arrays(G.random_edges(n, 3 * n, 78))
    ref_g = oracle.build_csr(n, s, t)
    ref = oracle.pagerank(ref_g, D, 1e-15, 1000, norm_linf=True)
    with gpu_graph(pr, n, s, t) as g:
        st, it, fd, x = gpu_run(pr, g, n, 1e-15, mode=pr.PR_NORM_LINF)
        assert_iters(it, ref, 1e-15, linf=True)
        assert_close(x, ref.x)


def test_determinism_sync(pr):
    g0 = graphgen.make_config(4, scale_override=14)
    with gpu_graph(pr, g0.n, g0.src, g0.dst) as g:
        a = gpu_run(pr, g, g0.n, 1e-10)
        b = gpu_run(pr, g, g0.n, 1e-10)
        assert a[1] == b[1] and np.array_equal(a[3], b[3])
        assert np.array_equal(g.delta_log(), g.delta_log())
    with gpu_graph(pr, g0.n, g0.src, g0.dst) as g:
        c = gpu_run(pr, g, g0.n, 1e-10)
        assert c[1] == a[1] and np.array_equal(c[3], a[3])


@pytest.mark.parametrize("deg", [0, 1, 31, 32, 33, 1023, 1024, 1025, 8192, 8193, 20000, 70001])
def test_row_length_boundaries(pr, deg):
    """Rows at the engine's bin boundaries (SHORT=32, LONG=1024, HUB_CHUNK=8192)."""
    n = max(deg + 50, 100)
    rng = np.random.default_rng(deg)
    edges = [(int(u), 0) for u in rng.permutation(np.arange(1, n))[:deg]]
    edges += [(int(u), int(v)) for u, v in zip(rng.integers(0, n, 5 * n), rng.integers(0, n, 5 * n))]
    edges += [(0, int(v)) for v in rng.integers(1, n, 3)]
    s, t = G.edges_to_arrays(edges)
    check_all(pr, n, s, t, reductions=(deg % 2 == 0), async_mode=(deg % 3 == 0))


def test_host_buffers_e2e(pr):
    """Host (numpy) edge arrays and host ranks through the same ABI calls."""
    n, edges = G.planted_graph(3)
    s, t = G.edges_to_arrays(edges)
    ref_g = oracle.build_csr(n, s, t)
    ref = oracle.pagerank(ref_g, D, 1e-12, 1000)
    g = pr.Graph(n, s, t)          # numpy => host pointers
    x = np.zeros(n, np.float64)
    st, it, fd = g.run(x, D, 1e-12, 1000)
    assert_iters(it, ref, 1e-12)
    assert_close(x, ref.x)
    xp = torch.zeros(n, dtype=torch.float64).pin_memory()
    g.run(xp, D, 1e-12, 1000)
    assert_close(xp.numpy(), ref.x)
    g.close()


# --------------------------------------------------------------- configs --
def _config_case(pr, k, full_oracle=True):
    gen = graphgen.make_config(k)
    return check_all(pr, gen.n, gen.src, gen.dst, tau=gen.tau, async_mode=(k != 3)), gen


def test_config1_gnm(pr):
    _config_case(pr, 1)


def test_config2_rmat20(pr):
    _config_case(pr, 2)


def test_config3_structured(pr):
    ref_g, gen = _config_case(pr, 3)
    # planted structure is found: planted groups inside one class, planted chain members detected
    with gpu_graph(pr, gen.n, gen.src, gen.dst) as g:
        g.preprocess()
        rep, cs, ck = gpu_reductions(pr, g, gen.n)
        pos = gen.planted["pos"]
        assert (ck[pos >= 2] >= 1).all()
        grp = gen.planted["group"]
        order = np.argsort(grp, kind="stable")
        gs, rs = grp[order], rep[order]
        starts = np.r_[0, np.nonzero(np.diff(gs))[0] + 1]
        for a, b in zip(starts, np.r_[starts[1:], len(gs)]):
            if gs[a] >= 0:
                assert (rs[a:b] == rs[a]).all()


def test_config3_delayed_chains_keep_the_plain_sweep_count(pr):
    """Config 3 (dangling-free, 5 % of the vertices on chains): eager chain
    resolution breaks the plain iteration's mass conservation and needs about
    twice the sweeps (finding about Q-C); the delayed resolution
    reproduces the plain trajectory, so the reduced run takes the plain sweep
    count while gathering fewer edges per sweep."""
    gen = graphgen.make_config(3)
    ref_g = oracle.build_csr(gen.n, gen.src, gen.dst)
    ref = oracle.pagerank(ref_g, D, gen.tau, gen.max_iter)
    with gpu_graph(pr, gen.n, gen.src, gen.dst) as g:
        st, it_p, fd, xp = gpu_run(pr, g, gen.n, gen.tau)
        g.preprocess()
        st, it_r, fd, xr = gpu_run(pr, g, gen.n, gen.tau, mode=pr.PR_USE_REDUCTIONS)
        s = g.stats()
        st, it_e, fd, xe = gpu_run(pr, g, gen.n, gen.tau, mode=pr.PR_USE_REDUCTIONS | pr.PR_CHAIN_EAGER)
    assert_iters(it_r, ref, gen.tau)
    assert_close(xr, ref.x)
    assert it_r <= it_p + 1 and it_e > it_r
    assert s["gather_edges"] < ref_g.E


def test_config3_async(pr):
    gen = graphgen.make_config(3)
    ref_g = oracle.build_csr(gen.n, gen.src, gen.dst)
    with gpu_graph(pr, gen.n, gen.src, gen.dst) as g:
        check_async(pr, g, ref_g, gen.n, gen.tau)


@pytest.mark.parametrize("n", [256, 300, 1 << 16])
def test_outdeg_split_sort_edge_cases(pr, n):
    """Ingest counts outdeg from the src runs of a partial sort when that costs
    no extra radix pass (b = 8, 16, 24, ...; n = 300 has b = 9 and takes the
    atomic path): self-loops and duplicates on the LAST vertex (whose src bits
    equal the sentinel's when n = 2^b) must not be counted."""
    rng = np.random.default_rng(n)
    m = 20 * n
    s = rng.integers(0, n, m, dtype=np.int64)
    t = rng.integers(0, n, m, dtype=np.int64)
    last = n - 1
    extra_s = np.array([last] * 40 + [last] * 30 + [0] * 5, np.int64)
    extra_t = np.array([last] * 40 + [3] * 30 + [0] * 5, np.int64)        # self-loops, duplicates
    s = np.concatenate([s, extra_s]).astype(np.int32)
    t = np.concatenate([t, extra_t]).astype(np.int32)
    ref_g = oracle.build_csr(n, s, t)
    with gpu_graph(pr, n, s, t) as g:
        rp, col, od = gpu_csr(pr, g, n, ref_g.E)
        assert np.array_equal(od, ref_g.outdeg)
        assert np.array_equal(rp, ref_g.row_ptr) and np.array_equal(col, ref_g.col_idx)


def test_run_loop_batches_with_and_without_timing(pr):
    """The sweep loop launches batches sized by a geometric fit of the
    batch-end deltas: with or without PR_TIMING
    (events every 4th sweep) the run is bit-identical, stops at the oracle's
    sweep count, and synchronises the host only a handful of times."""
    gen = graphgen.make_config(2)
    ref = oracle.pagerank(oracle.build_csr(gen.n, gen.src, gen.dst), D, gen.tau, gen.max_iter)
    with gpu_graph(pr, gen.n, gen.src, gen.dst) as g:
        a = gpu_run(pr, g, gen.n, gen.tau)
        sa = g.stats()
        b = gpu_run(pr, g, gen.n, gen.tau, mode=pr.PR_TIMING)
        sb = g.stats()
    assert a[1] == b[1] and np.array_equal(a[3], b[3])
    assert_iters(a[1], ref, gen.tau)
    assert sb["timed_iterations"] >= a[1] // 4 - 1 and sb["gather_ms"] > 0
    assert sa["timed_iterations"] == 0
    assert sa["host_syncs"] <= 8 and sb["host_syncs"] <= 8


@pytest.mark.parametrize("k", ["32768", "0"])
def test_cold_slots_in_row_order(pr, k, monkeypatch):
    """Contrib slots past the K hottest in row order (PRGPU_DEG_SLOTS;
    k = 0: every slot by out-degree; K is raised to the L1 tier, 36864): a
    graph of 64K sources, so that most rows' slots follow the row order; every mode's
    result must match the oracle as with any other slot order."""
    monkeypatch.setenv("PRGPU_DEG_SLOTS", k)
    src, dst = graphgen.rmat(17, 8 << 17, seed=31)
    check_all(pr, 1 << 17, src, dst, tau=1e-11)


@pytest.mark.parametrize("seed", range(3))
def test_chain_relation_at_exit(pr, seed):
    """at exit every chain member v with predecessor p (its only
    in-neighbour, out-degree 1) satisfies x(v) = c + d * x(p) to 1e-14
    relative in the eager reduced mode (x_t(v) = alpha_k + beta_k * x_t(src),
    the same-sweep chain, Q-C), and to the convergence error in the delayed
    mode (x_t(v) = c + d * x_{t-1}(p): the plain trajectory, Q-C2);
    identical members equal their representative exactly."""
    n, edges = G.planted_graph(seed, n_base=200, chains=(2, 9, 16, 5))
    s, t = G.edges_to_arrays(edges)
    ref_g = oracle.build_csr(n, s, t)
    c = (1 - D) / n
    with gpu_graph(pr, n, s, t) as g:
        g.preprocess(pr.PR_PRE_IDENTICAL | pr.PR_PRE_CHAIN)
        rep, cs, ck = gpu_reductions(pr, g, n)
        members = np.nonzero(ck > 0)[0]
        assert len(members) > 0
        pred = ref_g.col_idx[ref_g.row_ptr[members]]
        assert np.all(np.diff(ref_g.row_ptr)[members] == 1) and np.all(ref_g.outdeg[pred] == 1)
        tau = 1e-13
        _, _, _, xe = gpu_run(pr, g, n, tau, mode=pr.PR_USE_REDUCTIONS | pr.PR_CHAIN_EAGER)
        rel = np.abs(xe[members] - (c + D * xe[pred])) / xe[members]
        assert rel.max() <= 1e-14, rel.max()
        _, _, _, xd = gpu_run(pr, g, n, tau, mode=pr.PR_USE_REDUCTIONS)
        assert np.abs(xd[members] - (c + D * xd[pred])).max() <= 10 * tau
        ident = np.nonzero(rep != np.arange(n))[0]
        assert np.array_equal(xe[ident], xe[rep[ident]]) and np.array_equal(xd[ident], xd[rep[ident]])
