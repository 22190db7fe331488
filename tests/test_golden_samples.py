"""The sampled-golden checker of the full-size GPU tests, exercised on CPU.

tests/golden/config_samples_<k>.json holds samples of the ORACLE's converged
run (tests/golden/make_samples.py); tests/test_gpu_fullsize.py compares the
GPU's converged full-size ranks with them.  Here (no GPU): the stored config-2
file equals a fresh oracle run, and the checker rejects the mistakes it is
there to catch (one vertex off by more than the bar outside the sampled set, a
global scale error, a wrong iteration count)."""
import json
import os

import numpy as np
import pytest

import graphgen
import oracle
from tests.test_gpu_fullsize import TOL_L1, TOL_V, _samples, check_against_samples

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def run2():
    g = graphgen.make_config(2)
    c = oracle.build_csr(g.n, g.src, g.dst)
    return oracle.pagerank(c, g.d, g.tau, g.max_iter)


def test_stored_samples_equal_a_fresh_oracle_run(run2):
    w, bs = check_against_samples(2, run2.x, run2.iters, tol_v=0.0, tol_l1=0.0, iters_pm=0, tol_b=0.0)
    assert w == 0.0 and bs == 0.0
    assert _samples(2)["iters"] == json.load(open(os.path.join(HERE, "golden", "config_iters.json")))["2"]["plain_iters"]


def test_checker_rejects_a_single_vertex_outside_the_samples(run2):
    S = _samples(2)
    listed = set(S["sample_ids"]) | set(S["top_ids"]) | set(S["identical_ids"]) | set(S["chain_ids"])
    v = next(u for u in range(1000, 2000) if u not in listed)
    x = run2.x.copy()
    x[v] += 20 * TOL_V
    with pytest.raises(AssertionError):
        check_against_samples(2, x, run2.iters)
    x[v] = run2.x[v] + 0.5 * TOL_V          # inside the bar: accepted
    check_against_samples(2, x, run2.iters)


def test_checker_rejects_scale_and_iteration_errors(run2):
    with pytest.raises(AssertionError):
        check_against_samples(2, run2.x * (1 + 20 * TOL_L1), run2.iters)
    with pytest.raises(AssertionError):
        check_against_samples(2, run2.x, run2.iters + 2)
    x = run2.x.copy()
    x[_samples(2)["top_ids"][0]] += 2 * TOL_V
    with pytest.raises(AssertionError):
        check_against_samples(2, x, run2.iters)


@pytest.mark.parametrize("k", [4, 5])
def test_fullsize_sample_files_present_and_consistent(k):
    S = _samples(k)
    assert S is not None, f"run tests/golden/make_samples.py {k}"
    it = json.load(open(os.path.join(HERE, "golden", "config_iters.json")))[str(k)]
    assert S["iters"] == it["plain_iters"] and S["E"] == it["E"]
    assert abs(float.fromhex(S["final_delta"]) - it["plain_final_delta"]) <= 1e-12 * it["plain_final_delta"]
    xs = np.array([float.fromhex(v) for v in S["bucket_sums"]])
    assert abs(xs.sum() - it["rank_sum"]) <= 1e-12      # the bucket sums cover every vertex once
