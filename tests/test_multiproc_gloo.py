"""N>1 host logic of bench.py on CPU with the gloo backend (world_size 2).

bench.py runs one replica per rank ("replicas only"): the
timed region is reduced as the MAX over ranks, the work as the SUM, and the
reference arm runs on rank 0 only.  These helpers are exercised here without
a GPU."""
import os
import socket
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        t = bench.max_over_ranks(10.0 + rank, ws)        # per-rank elapsed ms
        u = bench.sum_over_ranks(100.0 * (rank + 1), ws)  # per-rank units
        bench.barrier(ws)
        q.put((rank, t, u))
    finally:
        dist.destroy_process_group()


def test_max_and_sum_over_ranks_gloo():
    ws = 2
    q = mp.get_context("spawn").Queue()
    port = _free_port()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    out = sorted(q.get(timeout=5) for _ in range(ws))
    for rank, t, u in out:
        assert t == 11.0          # max over ranks
        assert u == 300.0         # sum over ranks


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "tests", "golden", "config_iters.json")),
                    reason="needs the oracle's iteration counts")
def test_reference_arm_two_ranks_rank0_only():
    """`torchrun --nproc-per-node 2 bench.py --impl reference`: rank 0 prints one
    JSON line, rank 1 exits 0 without work (gloo, CPU, config 1)."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--config", "1", "--steps", "2", "--warmup", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    import json
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["cpu_baseline"]["kind"] == "oracle"
