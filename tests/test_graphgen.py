"""Input generator checks (no GPU): determinism, exact counts, distributions,
planted structure, and frozen checksums (drift detection)."""
import json
import os

import numpy as np
import pytest

import graphgen
import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "config_checksums.json")))


def test_rmat_deterministic_and_exact_count():
    a = graphgen.rmat(10, 10_000, seed=9)
    b = graphgen.rmat(10, 10_000, seed=9)
    c = graphgen.rmat(10, 10_000, seed=10)
    assert a[0].shape == (10_000,)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert not np.array_equal(a[0], c[0])
    assert a[0].min() >= 0 and a[0].max() < 1024


def test_rmat_uniform_quadrants():
    m = 200_000
    s, t = graphgen.rmat(8, m, seed=1, a=0.25, b=0.25, c=0.25, permute=False)
    top = (s >> 7) * 2 + (t >> 7)        # first-level quadrant
    freq = np.bincount(top, minlength=4) / m
    assert np.abs(freq - 0.25).max() < 0.01


def test_rmat_skewed_quadrants():
    m = 200_000
    s, t = graphgen.rmat(8, m, seed=1, permute=False)
    top = (s >> 7) * 2 + (t >> 7)
    freq = np.bincount(top, minlength=4) / m
    np.testing.assert_allclose(freq, [0.57, 0.19, 0.19, 0.05], atol=0.01)


def test_gnm_no_loops():
    s, t = graphgen.gnm(50, 5000, seed=3)
    assert (s != t).all() and s.max() < 50 and t.max() < 50


def test_poisson_mean_and_no_loops():
    s, t = graphgen.poisson(20_000, 20.0, seed=5)
    od = np.bincount(s, minlength=20_000)
    assert abs(od.mean() - 20.0) < 0.15
    assert abs(od.var() - 20.0) < 1.0
    assert (s != t).all()


def test_structured_planted_structure_small():
    n = 20_000
    s, t, pl = graphgen.structured(n, 150_000, seed=3)
    g = oracle.build_csr(n, s, t)
    rep = oracle.identical(g)
    grp = pl["group"]
    for gid in np.unique(grp[grp >= 0])[:200]:
        mem = np.nonzero(grp == gid)[0]
        assert len(set(rep[mem].tolist())) == 1            # planted group within one class
    ch = pl["chain"]
    chain_v = np.nonzero(ch >= 0)[0]
    indeg = np.diff(g.row_ptr)
    assert (indeg[chain_v] == 1).all() and (g.outdeg[chain_v] == 1).all()
    cs, ck, mk = oracle.chains(g, rep)
    pos = pl["pos"]
    assert (ck[pos >= 2] >= 1).all()                       # planted members are detected
    assert mk >= 15


@pytest.mark.parametrize("k", ["1", "2"])
def test_frozen_checksums(k):
    rec = GOLD[k]
    g = graphgen.make_config(int(k))
    assert g.n == rec["n"] and g.m == rec["m_raw"]
    assert str(g.checksum()) == rec["raw_checksum"]


@pytest.mark.parametrize("k", ["1", "2"])
def test_frozen_oracle_csr(k):
    """Oracle drift detection: CSR / reductions of the generated configs match
    the values tests/golden/make_golden.py froze."""
    import hashlib
    rec = GOLD[k]
    g = graphgen.make_config(int(k))
    c = oracle.build_csr(g.n, g.src, g.dst)
    h = hashlib.sha256()
    for a in (c.row_ptr, c.col_idx, c.outdeg):
        h.update(np.ascontiguousarray(a).tobytes())
    assert c.E == rec["E"] and h.hexdigest() == rec["csr_sha256"]
    rep = oracle.identical(c)
    assert hashlib.sha256(rep.tobytes()).hexdigest() == rec["rep_sha256"]
