"""GPU parity at BASELINE.json's full sizes (configs 4 and 5), in the launch
configuration bench.py times (persistent gather grid, reduced and plain modes),
plus the in-place async and the persistent No-Sync modes on both.

A converged oracle run at these sizes takes ~10 min single-threaded (config 4:
644 s measured, tests/golden/config_iters.json), so this suite checks (and
tests/test_gpu_fullsize_converged.py, slow, compares with CONVERGED oracle
runs; its log is profiles/r2/fullsize_converged_parity.log):
  * integer outputs bit-exact against the oracle (full arrays, compared by hash);
  * the first 3 sweeps element by element against the oracle's first 3 sweeps
    (same arithmetic path, tau = 0);
  * the converged result against the oracle's own CONVERGED run, sampled
    (tests/golden/config_samples_<k>.json, written by tests/golden/make_samples.py
    from graphgen + oracle only): 1024 seeded vertices, the 64 largest ranks and
    identical / chain members one by one (<= 1e-10), every vertex through 512
    bucket sums (their summed |diff| <= the L1 bar 1e-9) and 8 signed projections;
  * and through properties that hold at any size: the
    oracle's residual certificate ||x - x*||_1 <= ||r(x)||_1/(1-d) (for a sync
    run ||r(x_k)||_1 = Delta_{k+1} <= d*tau), the mass identity, and the
    iteration count against the oracle's own count stored by
    tests/golden/make_iters.py.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import graphgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ITERS = json.load(open(os.path.join(HERE, "golden", "config_iters.json")))
GOLD = json.load(open(os.path.join(HERE, "golden", "config_checksums.json")))
TOL_V, TOL_L1 = 1e-10, 1e-9   # north_star: per-vertex |diff| <= 1e-10, L1 <= 1e-9


def _samples(k):
    """The oracle's CONVERGED plain run at config k, sampled (written by
    tests/golden/make_samples.py from graphgen + oracle only)."""
    p = os.path.join(HERE, "golden", f"config_samples_{k}.json")
    return json.load(open(p)) if os.path.exists(p) else None


def _unhex(a):
    return np.array([float.fromhex(v) for v in a], np.float64)


def check_against_samples(k, x, iters, tol_v=TOL_V, tol_l1=TOL_L1, iters_pm=1, tol_b=10 * TOL_V):
    """x (a converged full-size result) against the oracle's stored samples:
    sampled / top / member vertices one by one, every vertex through its bucket
    sum (sum_b |B_b - B'_b| <= ||x - x'||_1), signed projections."""
    from tests.golden import make_samples as ms
    S = _samples(k)
    assert S is not None, f"tests/golden/config_samples_{k}.json missing (run tests/golden/make_samples.py {k})"
    assert S["n"] == x.shape[0]
    if iters_pm is not None:
        assert abs(iters - S["iters"]) <= iters_pm, (iters, S["iters"])
        if iters != S["iters"]:   # only where the oracle's last delta sits at the threshold
            assert abs(float.fromhex(S["final_delta"]) - S["tau"]) <= 1e-3 * S["tau"]
    worst = 0.0
    for key in ("sample", "top", "identical", "chain"):
        ids = np.asarray(S[key + "_ids"], np.int64)
        if ids.size == 0:
            continue
        dv = np.abs(x[ids] - _unhex(S[key + "_x"]))
        worst = max(worst, float(dv.max()))
        assert dv.max() <= tol_v, (key, int(ids[dv.argmax()]), float(dv.max()))
    assert S["nb"] == ms.NB
    db = np.abs(ms.bucket_sums(x) - _unhex(S["bucket_sums"]))
    assert db.sum() <= tol_l1, float(db.sum())
    assert db.max() <= tol_b, float(db.max())   # one vertex off by > 10x the bar shows in its bucket
    dp = np.abs(np.array(ms.projections(x, k)) - _unhex(S["projections"]))
    assert dp.max() <= tol_l1, float(dp.max())
    return worst, float(db.sum())


@pytest.fixture(scope="module")
def pr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_09527_b200 as m
    return m


def sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def run(pr, g, n, d, tau, max_iter, mode=0):
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    st, it, fd = g.run(x, d, tau, max_iter, mode=mode)
    return st, it, fd, x.cpu().numpy()


def _fullsize(pr, k, async_too):
    gen = graphgen.make_config(k)
    n, d = gen.n, gen.d
    ref_g = oracle.build_csr(n, gen.src, gen.dst)
    s = torch.from_numpy(gen.src).cuda()
    t = torch.from_numpy(gen.dst).cuda()
    g = pr.Graph(n, s, t)
    del s, t
    try:
        assert g.info()["E"] == ref_g.E
        rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        col = torch.empty(ref_g.E, dtype=torch.int32, device="cuda")
        od = torch.empty(n, dtype=torch.int32, device="cuda")
        pr.pr_get_csr(g.handle, rp, col, od)
        assert sha(rp.cpu().numpy()) == sha(ref_g.row_ptr)
        assert sha(col.cpu().numpy()) == sha(ref_g.col_idx)
        assert sha(od.cpu().numpy()) == sha(ref_g.outdeg)
        del rp, col, od
        if str(k) in GOLD:
            assert sha(ref_g.row_ptr, ref_g.col_idx, ref_g.outdeg) == GOLD[str(k)]["csr_sha256"]

        # first three sweeps, element by element
        ref3 = oracle.pagerank(ref_g, d, 0.0, 3)
        st, it, fd, x3 = run(pr, g, n, d, 0.0, 3)
        assert it == 3 and st == pr.PR_NOT_CONVERGED
        assert np.abs(x3 - ref3.x).max() <= 1e-14
        np.testing.assert_allclose(g.delta_log(), ref3.delta_log, rtol=1e-9)

        # converged plain sync run: certificate, mass identity, iteration count
        st, it, fd, x = run(pr, g, n, d, gen.tau, gen.max_iter)
        assert st == pr.PR_OK and fd <= gen.tau
        res = oracle.residual_l1(ref_g, d, x)
        assert res <= d * gen.tau * (1 + 1e-6) + 1e-15
        assert res / (1 - d) <= 6e-10
        if str(k) in ITERS:
            ref_it = ITERS[str(k)]["plain_iters"]
            assert abs(it - ref_it) <= 1
            if it != ref_it:   # only where the oracle's last delta sits at the threshold
                assert abs(ITERS[str(k)]["plain_final_delta"] - gen.tau) <= 1e-3 * gen.tau
        # ... and against the oracle's converged run itself, sampled (sync = the same trajectory)
        w, bs = check_against_samples(k, x, it)
        print(f"config {k} sync plain vs oracle samples: max |diff| {w:.3g}, bucket L1 {bs:.3g}")
        log = g.delta_log()
        assert (log[1:, 0] <= d * log[:-1, 0] * (1 + 1e-9) + 1e-18).all()   # L1 contraction
        dangling_mass = math.fsum(x[ref_g.outdeg == 0])
        total = math.fsum(x)
        # fixed point: S* = (1-d) + d (S* - D*)  =>  S* = 1 - d D*/(1-d), within the certificate
        assert abs(total - (1 - d * dangling_mass / (1 - d))) <= 10 * res / (1 - d) + 1e-12

        # reduced mode: integer reductions vs oracle, converged certificate
        g.preprocess()
        if k == 4:
            rep_o = oracle.identical(ref_g)
            cs_o, ck_o, _ = oracle.chains(ref_g, rep_o)
            rep = torch.empty(n, dtype=torch.int32, device="cuda")
            cs = torch.empty(n, dtype=torch.int32, device="cuda")
            ck = torch.empty(n, dtype=torch.int32, device="cuda")
            pr.pr_get_reductions(g.handle, rep, cs, ck)
            assert sha(rep.cpu().numpy()) == sha(rep_o) == GOLD["4"]["rep_sha256"]
            assert sha(cs.cpu().numpy(), ck.cpu().numpy()) == sha(cs_o, ck_o) == GOLD["4"]["chain_sha256"]
        st, it, fd, xr = run(pr, g, n, d, gen.tau, gen.max_iter, mode=pr.PR_USE_REDUCTIONS)
        assert st == pr.PR_OK
        res_r = oracle.residual_l1(ref_g, d, xr)
        assert res_r / (1 - d) <= 6e-10
        assert np.abs(xr - x).max() <= 1e-10 and np.abs(xr - x).sum() <= 2e-9
        check_against_samples(k, xr, it)   # delayed chains: the oracle's plain trajectory (Q-C2)

        if async_too:
            # phased in-place sweeps (default phase count: 8 on R-MAT-24, 1 on the blocked config 5)
            for extra in (0, pr.PR_USE_REDUCTIONS):
                st, it_p, fd, xp = run(pr, g, n, d, gen.tau, gen.max_iter, mode=pr.PR_MODE_PHASED | extra)
                assert st == pr.PR_OK and fd <= gen.tau
                assert g.stats()["phases"] == (8 if k == 4 else 1)
                assert oracle.residual_l1(ref_g, d, xp) / (1 - d) <= 1e-8
                assert np.abs(xp - x).max() <= 1e-10
                check_against_samples(k, xp, it_p, tol_l1=2e-9, iters_pm=None, tol_b=2e-9)
                if k == 4:
                    assert it_p < it   # block Gauss-Seidel: fewer sweeps on R-MAT
            st, it_a, fd, xa = run(pr, g, n, d, gen.tau, gen.max_iter, mode=pr.PR_MODE_ASYNC)
            assert st == pr.PR_OK and fd <= gen.tau
            res_a = oracle.residual_l1(ref_g, d, xa)
            assert res_a / (1 - d) <= 1e-8
            assert np.abs(xa - x).max() <= 1e-10
            # in-place results and the oracle's run are each within 5.67 tau (L1) of x*: up to ~1.2e-9 apart
            check_against_samples(k, xa, it_a, tol_l1=2e-9, iters_pm=None, tol_b=2e-9)
            # persistent barrier-free No-Sync (f1): certified residual of the original system
            st, it_n, fd, xn = run(pr, g, n, d, gen.tau, gen.max_iter, mode=pr.PR_MODE_NOSYNC)
            assert st == pr.PR_OK and fd <= gen.tau
            res_n = oracle.residual_l1(ref_g, d, xn)
            assert res_n <= gen.tau * (1 + 1e-6) + 1e-15
            assert np.abs(xn - x).max() <= 1e-10
            check_against_samples(k, xn, it_n, tol_l1=2e-9, iters_pm=None, tol_b=2e-9)
            st, it_n, fd, xn = run(pr, g, n, d, gen.tau, gen.max_iter,
                                   mode=pr.PR_MODE_NOSYNC | pr.PR_USE_REDUCTIONS)
            assert st == pr.PR_OK and fd <= gen.tau
            assert oracle.residual_l1(ref_g, d, xn) / (1 - d) <= 1e-9
    finally:
        g.close()


def test_config4_rmat24_fullsize(pr):
    _fullsize(pr, 4, async_too=True)


def test_config5_poisson_fullsize(pr):
    _fullsize(pr, 5, async_too=True)
