"""GPU parity of the ingest (K-INGEST, csrc/ingest.cu) against the oracle's
CSR (SPEC S:69-77 build_csr; §5.2), bit for bit, on rows of
in-degree at and around every power of two up to 40000 (the radix tiles,
warps and dedup chunks see short, long and tile-straddling rows), with
duplicates and self-loops in every length class, sources in ascending,
descending and random input order, and rows whose sources are all one value.
(Written for the counting-form ingest experiment, commit e65f465, which was
measured slower and removed; the cases stay as CSR edge cases.)
"""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

BOUNDARY_LENGTHS = [0, 1, 2, 3, 4, 5, 8, 9, 15, 16, 17, 31, 32, 33, 63, 64, 65, 128, 129, 255, 256, 257,
                    511, 512, 513, 1000, 1024, 1025, 2048, 4095, 4096, 4097, 8192, 16383, 16384, 16385,
                    20000, 40000]


@pytest.fixture(scope="module")
def pr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_09527_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def csr_of(pr, n, src, dst):
    with pr.Graph(n, dev(src), dev(dst)) as g:
        E = g.info()["E"]
        rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        col = torch.empty(max(E, 1), dtype=torch.int32, device="cuda")
        od = torch.empty(n, dtype=torch.int32, device="cuda")
        pr.pr_get_csr(g.handle, rp, col, od)
        return E, rp.cpu().numpy(), col[:E].cpu().numpy(), od.cpu().numpy()


def check(pr, n, src, dst):
    ref = oracle.build_csr(n, src, dst)
    E, rp, col, od = csr_of(pr, n, src, dst)
    assert E == ref.E
    assert np.array_equal(rp, ref.row_ptr)
    assert np.array_equal(col, ref.col_idx)
    assert np.array_equal(od, ref.outdeg)


def class_graph(seed, n, lengths, order, dup_frac):
    """Row v = 10 * i + 7 gets lengths[i] raw in-edges: sources in the given
    order, a fraction dup_frac of them repeats of earlier ones, one self-loop
    per row of length >= 3."""
    rng = np.random.default_rng(seed)
    src, dst = [], []
    for i, L in enumerate(lengths):
        v = 10 * i + 7
        if L == 0:
            continue
        s = rng.integers(0, n, L)
        k = int(L * dup_frac)
        if k:
            s[L - k:] = s[rng.integers(0, max(L - k, 1), k)]
        if order == "asc":
            s = np.sort(s)
        elif order == "desc":
            s = np.sort(s)[::-1]
        if L >= 3:
            s[L // 2] = v
        src.append(s)
        dst.append(np.full(L, v))
    src = np.concatenate(src).astype(np.int32)
    dst = np.concatenate(dst).astype(np.int32)
    p = rng.permutation(len(src))  # edge order in the input is irrelevant
    return src[p], dst[p]


@pytest.mark.parametrize("order", ["random", "asc", "desc"])
@pytest.mark.parametrize("dup_frac", [0.0, 0.3])
def test_row_classes(pr, order, dup_frac):
    n = 100_000
    src, dst = class_graph(11, n, BOUNDARY_LENGTHS, order, dup_frac)
    check(pr, n, src, dst)


def test_single_source_rows(pr):
    """Rows whose sources are one value (all but one entry duplicates), in
    every class; and sources drawn from a handful of values."""
    n = 50_000
    src, dst = [], []
    for i, L in enumerate(BOUNDARY_LENGTHS):
        v = 10 * i + 3
        src.append(np.full(L, (v * 7 + 1) % n))
        dst.append(np.full(L, v))
        src.append(np.arange(L) % 5 + 11)
        dst.append(np.full(L, v + 1))
    src = np.concatenate(src).astype(np.int32)
    dst = np.concatenate(dst).astype(np.int32)
    check(pr, n, src, dst)


def test_many_hub_rows(pr):
    """300 rows of in-degree 16400 over 4000 sources (dense rows, many
    duplicates)."""
    n = 4_000
    rng = np.random.default_rng(5)
    rows = 300
    L = 16_400
    dst = np.repeat(np.arange(rows, dtype=np.int32) * 13 % n, L)
    src = rng.integers(0, n, rows * L).astype(np.int32)
    check(pr, n, src, dst)


def test_self_loops_only_and_tiny(pr):
    n = 10
    s = np.arange(10, dtype=np.int32)
    check(pr, n, s, s.copy())
    check(pr, 2, np.array([0, 1, 0], np.int32), np.array([1, 0, 1], np.int32))


def test_invalid_ids(pr):
    for s, t in (([0, 1, 7], [1, 2, 0]), ([0, 1, 2], [1, -3, 0]), ([0, 1, 2], [1, 2, 1 << 30])):
        with pytest.raises(pr.PRError) as e:
            pr.Graph(5, dev(np.array(s)), dev(np.array(t)))
        assert e.value.code == pr.PR_EINVAL


@pytest.mark.parametrize("m", [2, 3072 * 4, 3072 * 5 + 17, 100_003])
def test_pack_fused_first_pass(pr, m, monkeypatch):
    """The pack fused into the first radix pass (aligned edge arrays) against
    the separate pack kernel (PRGPU_PACK=0) and the oracle: whole tiles, a
    ragged last tile (plain loads instead of the bulk copy), two edges."""
    n = 5000
    rng = np.random.default_rng(m)
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    src[::7] = dst[::7]  # self-loops
    check(pr, n, src, dst)
    monkeypatch.setenv("PRGPU_PACK", "0")
    check(pr, n, src, dst)


def test_unaligned_edge_arrays(pr):
    """Edge arrays that are not 16-byte aligned take the separate pack kernel."""
    n, m = 3000, 20_001
    rng = np.random.default_rng(9)
    s_all = torch.from_numpy(rng.integers(0, n, m + 1).astype(np.int32)).cuda()
    t_all = torch.from_numpy(rng.integers(0, n, m + 1).astype(np.int32)).cuda()
    s, t = s_all[1:], t_all[1:]
    assert s.data_ptr() % 16 != 0
    ref = oracle.build_csr(n, s.cpu().numpy(), t.cpu().numpy())
    with pr.Graph(n, s, t) as g:
        assert g.info()["E"] == ref.E
        rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        col = torch.empty(max(ref.E, 1), dtype=torch.int32, device="cuda")
        od = torch.empty(n, dtype=torch.int32, device="cuda")
        pr.pr_get_csr(g.handle, rp, col, od)
        assert np.array_equal(rp.cpu().numpy(), ref.row_ptr)
        assert np.array_equal(col[:ref.E].cpu().numpy(), ref.col_idx)
        assert np.array_equal(od.cpu().numpy(), ref.outdeg)


@pytest.mark.parametrize("where", [5, 3072 * 2 + 100])
def test_invalid_id_in_full_and_ragged_tiles(pr, where):
    n, m = 1000, 3072 * 2 + 200
    rng = np.random.default_rng(where)
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    dst[where] = n
    with pytest.raises(pr.PRError) as e:
        pr.Graph(n, dev(src), dev(dst))
    assert e.value.code == pr.PR_EINVAL


def csr_from(pr, n, s, t):
    with pr.Graph(n, s, t) as g:
        E = g.info()["E"]
        rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        col = torch.empty(max(E, 1), dtype=torch.int32, device="cuda")
        od = torch.empty(n, dtype=torch.int32, device="cuda")
        pr.pr_get_csr(g.handle, rp, col, od)
        return E, rp.cpu().numpy(), col[:E].cpu().numpy(), od.cpu().numpy()


@pytest.mark.parametrize("m,n", [((1 << 22) + 12345, 1 << 20), (3 * (1 << 22) + 7, 50_000)])
def test_host_pinned_chunked_ingest(pr, m, n, monkeypatch):
    """Pinned host edge arrays take the chunked ingest (copy in CH_K chunks,
    each sorted on arrival and merged into the sorted prefix): the CSR equals
    the oracle's and the one-shot host copy's (PRGPU_CHUNKED=0)."""
    rng = np.random.default_rng(m)
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    idx = np.arange(0, m - 1, 5)                     # duplicates (some straddle chunk boundaries)
    src[idx] = src[idx + 1]
    dst[idx] = dst[idx + 1]
    dst[::11] = src[::11]                            # self-loops
    ref = oracle.build_csr(n, src, dst)
    s_h = torch.from_numpy(src).pin_memory()
    t_h = torch.from_numpy(dst).pin_memory()
    E, rp, col, od = csr_from(pr, n, s_h, t_h)
    assert E == ref.E
    assert np.array_equal(rp, ref.row_ptr)
    assert np.array_equal(col, ref.col_idx)
    assert np.array_equal(od, ref.outdeg)
    monkeypatch.setenv("PRGPU_CHUNKED", "0")
    E2, rp2, col2, od2 = csr_from(pr, n, s_h, t_h)
    assert E2 == E and np.array_equal(rp2, rp) and np.array_equal(col2, col) and np.array_equal(od2, od)


def test_host_pinned_chunked_rmat_run(pr):
    """R-MAT scale 20 from pinned host buffers: CSR and the reduced run match
    the device-buffer create."""
    import graphgen
    gen = graphgen.make_config(2)
    x1 = torch.empty(gen.n, dtype=torch.float64, device="cuda")
    x2 = torch.empty(gen.n, dtype=torch.float64, device="cuda")
    with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g1, \
            pr.Graph(gen.n, torch.from_numpy(gen.src).pin_memory(), torch.from_numpy(gen.dst).pin_memory()) as g2:
        for g in (g1, g2):
            g.preprocess()
        r1 = g1.run(x1, gen.d, gen.tau, gen.max_iter, mode=pr.PR_USE_REDUCTIONS)
        r2 = g2.run(x2, gen.d, gen.tau, gen.max_iter, mode=pr.PR_USE_REDUCTIONS)
        assert r1 == r2 and torch.equal(x1, x2)


def test_host_pinned_invalid_id_last_chunk(pr):
    n, m = 1000, (1 << 22) + 100
    rng = np.random.default_rng(3)
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    dst[m - 3] = n + 5
    with pytest.raises(pr.PRError) as e:
        pr.Graph(n, torch.from_numpy(src).pin_memory(), torch.from_numpy(dst).pin_memory())
    assert e.value.code == pr.PR_EINVAL
