"""GPU tests of the row-sharded sync iteration (pr_graph_shard / pr_run_sharded;
SURVEY §8(e) / f3).

There is one GPU here, so P ranks run in ONE process on it: each rank is a
host thread driving its own pr_graph; the per-sweep exchange is a loopback
all-gather (device copies between the ranks' buffers after a host barrier).
No kernel ever waits on another rank's kernel: every wait is on the host.
The library code under test is exactly what runs across GPUs; only the
exchange callback differs (torch.distributed / NCCL there).

Pins (none uses the CUDA path as its own reference):
  * world = 1 is bit-identical to pr_run(PR_MODE_SYNC), whose oracle parity is
    pinned in test_gpu_parity;
  * P > 1: the assembled ranks match the oracle (1e-10 per vertex, 1e-9 L1,
    iteration count within the +/-1 rule), every vertex is owned exactly once,
    the rows and edges of the shards partition the plain view's.
"""
import threading

import numpy as np
import pytest

import graphgen
import oracle
from tests import graphs as G
from tests.test_gpu_parity import D, assert_close, assert_iters, dev

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_09527_b200 as m
    return m


class Loopback:
    """In-process all-gather of the ranks' chunks (one GPU, host barriers)."""

    def __init__(self, pr, world):
        self.pr = pr
        self.world = world
        self.bufs = [None] * world
        self.bar = threading.Barrier(world)

    def exchange_for(self, rank):
        def ex(buf, chunk, world, stream):
            assert world == self.world
            torch.cuda.synchronize()
            self.bufs[rank] = self.pr.device_f64(buf, chunk * world)
            self.bar.wait()
            mine = self.bufs[rank]
            for r in range(world):
                if r != rank:
                    mine[r * chunk:(r + 1) * chunk].copy_(self.bufs[r][r * chunk:(r + 1) * chunk])
            torch.cuda.synchronize()
            self.bar.wait()
        return ex


class PeerBarrier:
    """The exchange of the peer-store form: the kernels already wrote every
    rank's buffers; only wait until all ranks' stores of the sweep are done."""

    def __init__(self, world):
        self.bar = threading.Barrier(world)

    def exchange_for(self, rank):
        def ex(buf, chunk, world, stream):
            assert buf is None
            torch.cuda.synchronize()
            self.bar.wait()
        return ex


class LoopAllreduce:
    """In-process sum all-reduce of int32 device buffers (host copies after a
    host barrier; no kernel waits on another rank)."""

    def __init__(self, pr, world):
        self.pr = pr
        self.world = world
        self.host = [None] * world
        self.bar = threading.Barrier(world)

    def for_rank(self, rank):
        def ar(buf, count, world, stream):
            assert world == self.world
            torch.cuda.synchronize()
            t = self.pr.device_i32(buf, count)
            self.host[rank] = t.cpu()
            self.bar.wait()
            tot = torch.stack(self.host).sum(0, dtype=torch.int64).to(torch.int32)
            self.bar.wait()
            t.copy_(tot)
            torch.cuda.synchronize()
        return ar


def create_local(pr, n, s, t, world):
    """pr_graph_create_sharded on `world` in-process ranks (threads: the
    out-degree all-reduce is collective)."""
    ar = LoopAllreduce(pr, world)
    graphs = [None] * world
    errs = []

    def work(r):
        try:
            graphs[r] = pr.Graph.sharded(n, dev(s), dev(t), r, world, ar.for_rank(r))
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            ar.bar.abort()
    ths = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    if errs:
        for g in graphs:
            if g is not None:
                g.close()
        raise errs[0]
    return graphs


def run_world(pr, n, s, t, world, tau, max_iter=1000, mode=0, peers=False, local=False):
    """Shard one graph over `world` in-process ranks; returns the assembled
    ranks, per-rank (status, iters, delta) and shard infos.  peers=True: the
    exchange fused into the kernels (every rank stores into every rank's
    buffers; pr_shard_set_peers with the other graphs' device pointers)."""
    graphs = create_local(pr, n, s, t, world) if local else [pr.Graph(n, dev(s), dev(t)) for _ in range(world)]
    try:
        if not local:
            for r, g in enumerate(graphs):
                g.shard(r, world)
        infos = [g.shard_info() for g in graphs]
        xs = [torch.full((n,), float("nan"), dtype=torch.float64, device="cuda") for _ in range(world)]
        lb = Loopback(pr, world)
        if peers:
            bufs = [g.shard_buffers() for g in graphs]
            for g in graphs:
                g.set_peers([b[0] for b in bufs], [b[1] for b in bufs])
            lb = PeerBarrier(world)
        out = [None] * world
        errs = []

        def work(r):
            try:
                out[r] = graphs[r].run_sharded(xs[r], lb.exchange_for(r), D, tau, max_iter, mode)
            except BaseException as e:  # noqa: BLE001
                errs.append(e)
                lb.bar.abort()
        ths = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        if errs:
            raise errs[0]
        torch.cuda.synchronize()
        x = torch.stack(xs).sum(0).cpu().numpy()     # the sum all-reduce of the owned parts
        logs = [g.delta_log() for g in graphs]
        return x, out, infos, logs
    finally:
        for g in graphs:
            g.close()


GRAPHS = {
    "planted": lambda: G.planted_graph(2, n_base=150, chains=(2, 9, 16, 1)),
    "random": lambda: (400, G.random_edges(400, 1600, 23)),
    "in_star": lambda: (300, G.in_star(300)),
    "out_star": lambda: (64, G.out_star(64)),
    "path": lambda: (50, G.path(50)),
    "cycle": lambda: (31, G.cycle(31)),
    "single": lambda: (1, []),
    "no_edges": lambda: (9, []),
}


@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_world1_is_sync(pr, name):
    n, edges = GRAPHS[name]()
    s, t = G.edges_to_arrays(edges)
    with pr.Graph(n, dev(s), dev(t)) as g:
        x0 = torch.empty(n, dtype=torch.float64, device="cuda")
        ref = g.run(x0, D, 1e-12, 1000)
        ref_log = g.delta_log()
    x, out, infos, logs = run_world(pr, n, s, t, 1, 1e-12)
    assert out[0] == ref
    assert np.array_equal(x, x0.cpu().numpy())
    assert np.array_equal(logs[0], ref_log)
    assert infos[0]["owned_vertices"] == n


@pytest.mark.parametrize("name", sorted(GRAPHS))
@pytest.mark.parametrize("world", [2, 3, 5])
def test_sharded_matches_oracle(pr, name, world):
    n, edges = GRAPHS[name]()
    s, t = G.edges_to_arrays(edges)
    ref_g = oracle.build_csr(n, s, t)
    tau = 1e-12
    ref = oracle.pagerank(ref_g, D, tau, 1000)
    x, out, infos, logs = run_world(pr, n, s, t, world, tau)
    assert len({o for o in out}) == 1                    # identical status / iterations / delta on every rank
    st, it, fd = out[0]
    assert st == ref.status
    assert_iters(it, ref, tau)
    assert_close(x, ref.x)
    assert sum(i["owned_vertices"] for i in infos) == n
    assert sum(i["edges"] for i in infos) == ref_g.E
    assert sum(i["rows"] for i in infos) == int((np.diff(ref_g.row_ptr) > 0).sum())
    assert all(np.array_equal(lg, logs[0]) for lg in logs)


@pytest.mark.parametrize("cfg,world", [(2, 2), (2, 4), (3, 3)])
def test_sharded_configs(pr, cfg, world):
    gen = graphgen.make_config(cfg)
    ref_g = oracle.build_csr(gen.n, gen.src, gen.dst)
    ref = oracle.pagerank(ref_g, gen.d, gen.tau, gen.max_iter)
    x, out, infos, logs = run_world(pr, gen.n, gen.src, gen.dst, world, gen.tau, gen.max_iter)
    st, it, fd = out[0]
    assert st == ref.status
    assert_iters(it, ref, gen.tau)
    assert_close(x, ref.x)
    # nnz balance: no shard gathers more than 1.5x its share of the edges (no mega-hub dominates here)
    share = ref_g.E / world
    assert max(i["edges"] for i in infos) <= 1.5 * share + 1


def test_sharded_linf_and_max_iter(pr):
    n = 300
    s, t = G.edges_to_arrays(G.random_edges(n, 1200, 77))
    ref_g = oracle.build_csr(n, s, t)
    x, out, _, _ = run_world(pr, n, s, t, 2, 0.0, max_iter=4)
    assert out[0][:2] == (pr.PR_NOT_CONVERGED, 4)
    ref = oracle.pagerank(ref_g, D, 0.0, 4)
    assert np.abs(x - ref.x).max() <= 1e-14
    x, out, _, _ = run_world(pr, n, s, t, 2, 1e-14, mode=pr.PR_NORM_LINF)
    ref = oracle.pagerank(ref_g, D, 1e-14, 1000, norm_linf=True)
    assert out[0][0] == pr.PR_OK
    assert_iters(out[0][1], ref, 1e-14, linf=True)
    assert_close(x, ref.x)


def test_shard_validation(pr):
    n = 50
    s, t = G.edges_to_arrays(G.random_edges(n, 200, 3))
    with pr.Graph(n, dev(s), dev(t)) as g:
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        with pytest.raises(pr.PRError) as e:
            g.run_sharded(x, lambda *a: None)
        assert e.value.code == pr.PR_ESTATE
        for rank, world in ((0, 0), (2, 2), (-1, 3), (0, 5000)):
            with pytest.raises(pr.PRError) as e:
                g.shard(rank, world)
            assert e.value.code == pr.PR_EINVAL
        g.shard(0, 1)
        with pytest.raises(pr.PRError) as e:
            g.run_sharded(torch.empty(n, dtype=torch.float64), lambda *a: None)     # host ranks
        assert e.value.code == pr.PR_EINVAL
        with pytest.raises(pr.PRError) as e:
            g.run_sharded(x, lambda *a: None, mode=pr.PR_MODE_ASYNC)
        assert e.value.code == pr.PR_EINVAL

        def boom(*a):
            raise RuntimeError("exchange failed")
        with pytest.raises(RuntimeError, match="exchange failed"):
            g.run_sharded(x, boom)
        g.run(x, D, 1e-10, 100)     # the whole-graph path still works after sharding


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_multiprocess(pr, tmp_path, world):
    """The real multi-process path: torchrun, one process per rank, the
    torch.distributed exchange (gloo here; every rank on cuda:0 -- the waits
    are host-side collectives, no kernel waits on another rank)."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    out = tmp_path / "shard.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(root, "tests", "shard_worker.py"),
           "2", str(out)]
    subprocess.run(cmd, check=True, timeout=600, cwd=root)
    r = json.load(open(out))
    ranks = r["ranks"]
    assert len({(x["st"], x["it"], x["fd"]) for x in ranks}) == 1
    assert ranks[0]["st"] == r["oracle_status"]
    it, ref_it = ranks[0]["it"], r["oracle_iters"]
    if it != ref_it:
        assert abs(it - ref_it) == 1
        assert abs(r["oracle_log"][min(it, ref_it) - 1] - 1e-10) <= 1e-9 * 1e-10
    assert r["max_diff"] <= 1e-10 and r["l1_diff"] <= 1e-9
    assert sum(x["info"]["owned_vertices"] for x in ranks) == graphgen.make_config(2).n


def test_nccl_exchange_world1(pr, tmp_path):
    """The NCCL branch of torch_dist_exchange (in-place all_gather_into_tensor on
    the library's stream), in a one-rank NCCL process group: bit-identical to
    the sync run."""
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    store = dist.FileStore(str(tmp_path / "store"), 1)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1)
    try:
        gen = graphgen.make_config(2)
        with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g:
            x0 = torch.empty(gen.n, dtype=torch.float64, device="cuda")
            ref = g.run(x0, gen.d, gen.tau, gen.max_iter)
            g.shard(0, 1)
            x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
            out = g.run_sharded(x, pr.torch_dist_exchange(), gen.d, gen.tau, gen.max_iter)
            assert out == ref and torch.equal(x, x0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["planted", "random", "in_star", "no_edges"])
@pytest.mark.parametrize("world", [2, 3])
def test_peer_store_exchange_matches_allgather(pr, name, world):
    """The exchange fused into K-FINALIZE (peer stores) gives bit-identically
    the ranks, sweeps and deltas of the all-gather exchange, and the oracle's."""
    n, edges = GRAPHS[name]()
    s, t = G.edges_to_arrays(edges)
    a = run_world(pr, n, s, t, world, 1e-12)
    b = run_world(pr, n, s, t, world, 1e-12, peers=True)
    assert a[1] == b[1] and np.array_equal(a[0], b[0])
    assert all(np.array_equal(x, y) for x, y in zip(a[3], b[3]))
    ref = oracle.pagerank(oracle.build_csr(n, s, t), D, 1e-12, 1000)
    assert_close(b[0], ref.x)


def test_peer_store_config(pr):
    gen = graphgen.make_config(2)
    ref = oracle.pagerank(oracle.build_csr(gen.n, gen.src, gen.dst), gen.d, gen.tau, gen.max_iter)
    x, out, _, _ = run_world(pr, gen.n, gen.src, gen.dst, 4, gen.tau, gen.max_iter, peers=True)
    assert_iters(out[0][1], ref, gen.tau)
    assert_close(x, ref.x)


@pytest.mark.parametrize("world", [2])
def test_peer_store_multiprocess_ipc(pr, tmp_path, world):
    """One process per rank, buffers shared by CUDA IPC handles exchanged over
    torch.distributed (every rank on cuda:0 here), the exchange reduced to a
    barrier."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    out = tmp_path / "shard_ipc.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(root, "tests", "shard_worker.py"),
           "2", str(out), "peers"]
    subprocess.run(cmd, check=True, timeout=600, cwd=root)
    r = json.load(open(out))
    assert len({(x["st"], x["it"], x["fd"]) for x in r["ranks"]}) == 1
    assert r["max_diff"] <= 1e-10 and r["l1_diff"] <= 1e-9


# ------------------------------------------- per-rank ingest (create_sharded) --
@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_local_ingest_world1_is_sync(pr, name):
    """pr_graph_create_sharded with world = 1 equals pr_graph_create +
    pr_graph_shard(0, 1), hence pr_run(PR_MODE_SYNC), bit for bit."""
    n, edges = GRAPHS[name]()
    s, t = G.edges_to_arrays(edges)
    with pr.Graph(n, dev(s), dev(t)) as g:
        x0 = torch.empty(n, dtype=torch.float64, device="cuda")
        ref = g.run(x0, D, 1e-12, 1000)
    x, out, infos, logs = run_world(pr, n, s, t, 1, 1e-12, local=True)
    assert out[0] == ref
    assert np.array_equal(x, x0.cpu().numpy())
    assert infos[0]["owned_vertices"] == n


@pytest.mark.parametrize("name", sorted(GRAPHS))
@pytest.mark.parametrize("world", [2, 3, 5])
def test_local_ingest_matches_oracle(pr, name, world):
    """Every rank ingests only the edges into its vertices (v mod world):
    the shards partition the edges, rows and vertices, and the assembled
    ranks match the oracle (1e-10 / 1e-9, the +/-1 rule)."""
    n, edges = GRAPHS[name]()
    s, t = G.edges_to_arrays(edges)
    ref_g = oracle.build_csr(n, s, t)
    tau = 1e-12
    ref = oracle.pagerank(ref_g, D, tau, 1000)
    x, out, infos, logs = run_world(pr, n, s, t, world, tau, local=True)
    assert len({o for o in out}) == 1
    st, it, fd = out[0]
    assert st == ref.status
    assert_iters(it, ref, tau)
    assert_close(x, ref.x)
    assert sum(i["owned_vertices"] for i in infos) == n
    assert [i["owned_vertices"] for i in infos] == [len(range(r, n, world)) for r in range(world)]
    assert sum(i["edges"] for i in infos) == ref_g.E
    assert sum(i["rows"] for i in infos) == int((np.diff(ref_g.row_ptr) > 0).sum())


def test_local_ingest_rank_csr_and_outdeg(pr):
    """A rank's CSR holds exactly the rows of its vertices (bit-exact with the
    oracle's rows), and the all-reduced out-degrees are the graph's."""
    n, edges = G.planted_graph(4, n_base=150, chains=(3, 7))
    s, t = G.edges_to_arrays(edges)
    ref_g = oracle.build_csr(n, s, t)
    world = 3
    graphs = create_local(pr, n, s, t, world)
    try:
        for r, g in enumerate(graphs):
            E = g.info()["E"]
            rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
            col = torch.empty(max(E, 1), dtype=torch.int32, device="cuda")
            od = torch.empty(n, dtype=torch.int32, device="cuda")
            pr.pr_get_csr(g.handle, rp, col, od)
            rp, col, od = rp.cpu().numpy(), col[:E].cpu().numpy(), od.cpu().numpy()
            assert np.array_equal(od, ref_g.outdeg)
            mine = [v for v in range(n) if v % world == r]
            assert E == sum(int(ref_g.row_ptr[v + 1] - ref_g.row_ptr[v]) for v in mine)
            for v in range(n):
                got = col[rp[v]:rp[v + 1]]
                want = ref_g.col_idx[ref_g.row_ptr[v]:ref_g.row_ptr[v + 1]] if v % world == r else []
                assert np.array_equal(got, want)
    finally:
        for g in graphs:
            g.close()


def test_local_ingest_validation(pr):
    n = 40
    s, t = G.edges_to_arrays(G.random_edges(n, 160, 5))
    for rank, world in ((0, 0), (2, 2), (-1, 3), (0, 5000)):
        with pytest.raises(pr.PRError) as e:
            pr.Graph.sharded(n, dev(s), dev(t), rank, world, lambda *a: None)
        assert e.value.code == pr.PR_EINVAL
    with pytest.raises(RuntimeError, match="allreduce failed"):
        def boom(*a):
            raise RuntimeError("allreduce failed")
        pr.Graph.sharded(n, dev(s), dev(t), 0, 1, boom)
    bad = t.copy()
    bad[3] = n                                           # ids are validated on every rank
    with pytest.raises(pr.PRError) as e:
        pr.Graph.sharded(n, dev(s), dev(bad), 0, 1, lambda *a: None)
    assert e.value.code == pr.PR_EINVAL
    g = pr.Graph.sharded(n, dev(s), dev(t), 0, 1, lambda *a: None)
    try:
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        for call in (lambda: g.run(x, D, 1e-10, 10), lambda: g.preprocess(), lambda: g.shard(0, 1)):
            with pytest.raises(pr.PRError) as e:
                call()
            assert e.value.code == pr.PR_ESTATE
    finally:
        g.close()


@pytest.mark.parametrize("cfg,world", [(2, 4), (3, 3)])
def test_local_ingest_configs(pr, cfg, world):
    gen = graphgen.make_config(cfg)
    ref_g = oracle.build_csr(gen.n, gen.src, gen.dst)
    ref = oracle.pagerank(ref_g, gen.d, gen.tau, gen.max_iter)
    x, out, infos, logs = run_world(pr, gen.n, gen.src, gen.dst, world, gen.tau, gen.max_iter, local=True)
    st, it, fd = out[0]
    assert st == ref.status
    assert_iters(it, ref, gen.tau)
    assert_close(x, ref.x)
    share = ref_g.E / world
    assert max(i["edges"] for i in infos) <= 1.5 * share + 1


@pytest.mark.parametrize("name", ["planted", "random"])
def test_local_ingest_peer_stores(pr, name):
    """The fused peer-store exchange on locally ingested shards: bit-identical
    to their all-gather exchange."""
    n, edges = GRAPHS[name]()
    s, t = G.edges_to_arrays(edges)
    a = run_world(pr, n, s, t, 3, 1e-12, local=True)
    b = run_world(pr, n, s, t, 3, 1e-12, local=True, peers=True)
    assert a[1] == b[1] and np.array_equal(a[0], b[0])


def test_local_ingest_multiprocess(pr, tmp_path):
    """torchrun, one process per rank, the torch.distributed all-reduce and
    exchange (gloo; every rank on cuda:0, host-side collectives only)."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    out = tmp_path / "shard_local.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(root, "tests", "shard_worker.py"),
           "2", str(out), "local"]
    subprocess.run(cmd, check=True, timeout=600, cwd=root)
    r = json.load(open(out))
    assert len({(x["st"], x["it"], x["fd"]) for x in r["ranks"]}) == 1
    assert r["max_diff"] <= 1e-10 and r["l1_diff"] <= 1e-9


# ------------------------------------------------------ device-side barrier --
@pytest.mark.parametrize("world", [2, 3, 8, 32])
def test_peer_barrier_protocol_selftest(pr, world):
    """The device-side peer barrier (release store of the epoch into every
    peer's flags, acquire spin on one's own) run by `world` emulated ranks =
    the blocks of one cooperative launch (separate launches that wait on one
    another must not share a GPU): every rank sees every other rank's write
    of each epoch after passing that epoch's barrier."""
    pr.pr_selftest_peer_barrier(world, 300)


def test_device_barrier_world1_and_validation(pr):
    n, edges = GRAPHS["planted"]()
    s, t = G.edges_to_arrays(edges)
    with pr.Graph(n, dev(s), dev(t)) as g:
        with pytest.raises(pr.PRError) as e:
            pr.pr_shard_device_barrier(g.handle, True)          # not sharded yet
        assert e.value.code == pr.PR_ESTATE
        x0 = torch.empty(n, dtype=torch.float64, device="cuda")
        ref = g.run(x0, D, 1e-12, 1000)
        g.shard(0, 1)
        pr.pr_shard_device_barrier(g.handle, True)               # world 1: nothing to wait for
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        assert g.run_sharded(x, lambda *a: None, D, 1e-12, 1000) == ref
        assert torch.equal(x, x0)
    graphs = [pr.Graph(n, dev(s), dev(t)) for _ in range(2)]
    try:
        graphs[0].shard(0, 2)
        with pytest.raises(pr.PRError) as e:
            pr.pr_shard_device_barrier(graphs[0].handle, True)   # world 2 without peer buffers
        assert e.value.code == pr.PR_ESTATE
    finally:
        for g in graphs:
            g.close()


# ------------------------------------------------------------ NVLS multicast --
def _multicast_usable(pr):
    """NVLS needs the device attribute AND a multicast object the driver lets
    this process create (on the one-GPU slice of this pool cuMulticastCreate
    returns CUDA_ERROR_INVALID_VALUE for every handle type and team size,
    tools/probe_multicast.py, although the attribute reads 1)."""
    n, edges = GRAPHS["random"]()
    s_, t_ = G.edges_to_arrays(edges)
    with pr.Graph(n, dev(s_), dev(t_)) as g:
        g.shard(0, 1)
        try:
            pr.shard_multicast_local(g.handle)
            return True
        except pr.PRError as e:
            if "cuMulticast" in str(e) or "driver entry point" in str(e):
                return False
            raise


@pytest.mark.parametrize("name", ["planted", "random", "in_star", "no_edges", "single"])
@pytest.mark.parametrize("devbar", [False, True])
def test_multicast_world1_is_sync(pr, name, devbar):
    """The NVLS form of the fused exchange on a one-GPU team: every contrib,
    delta pair and in-degree-0 contrib is stored with multimem.st through the
    multicast address (the switch's replication to a team of one); the run is
    bit-identical to the plain world-1 run (hence to pr_run)."""
    if not _multicast_usable(pr):
        pytest.skip("NVLS multicast objects cannot be created on this device / slice")
    n, edges = GRAPHS[name]()
    s, t = G.edges_to_arrays(edges)
    with pr.Graph(n, dev(s), dev(t)) as g:
        x0 = torch.empty(n, dtype=torch.float64, device="cuda")
        ref = g.run(x0, D, 1e-12, 1000)
        ref_log = g.delta_log()
        g.shard(0, 1)
        pr.shard_multicast_local(g.handle)
        if devbar:
            pr.pr_shard_device_barrier(g.handle, True)
        calls = []
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        out = g.run_sharded(x, lambda buf, *a: calls.append(buf), D, 1e-12, 1000)
        assert out == ref
        assert torch.equal(x, x0)
        assert np.array_equal(g.delta_log(), ref_log)
        assert all(b is None for b in calls)              # barrier-only exchange
        if devbar:
            assert not calls                             # no host call inside the sweep loop
        again = g.run_sharded(x, lambda *a: None, D, 1e-12, 1000)   # a second run on the same team
        assert again == ref and torch.equal(x, x0)
        with pytest.raises(pr.PRError) as e:             # exclusive with the IPC peer buffers
            g.set_peers([0], [0])
        assert e.value.code == pr.PR_ESTATE


def test_multicast_local_ingest_world1(pr):
    if not _multicast_usable(pr):
        pytest.skip("NVLS multicast objects cannot be created on this device / slice")
    gen = graphgen.make_config(2)
    with pr.Graph(gen.n, dev(gen.src), dev(gen.dst)) as g:
        x0 = torch.empty(gen.n, dtype=torch.float64, device="cuda")
        ref = g.run(x0, gen.d, gen.tau, gen.max_iter)
    g = pr.Graph.sharded(gen.n, dev(gen.src), dev(gen.dst), 0, 1, lambda *a: None)
    try:
        pr.shard_multicast_local(g.handle)
        x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
        assert g.run_sharded(x, lambda *a: None, gen.d, gen.tau, gen.max_iter) == ref
        assert torch.equal(x, x0)
    finally:
        g.close()
