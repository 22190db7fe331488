"""Per-rank cost of the row-sharded sweep (pr_run_sharded) on ONE GPU: for each
world size P, every rank's shard is built and swept alone for a fixed number
of sweeps with a no-op exchange (its gather + finalize + combine kernels are
exactly those of a P-GPU run; only the all-gather is missing).  Reports the
slowest rank's sweep time and the exchanged bytes per sweep, from which the
P-GPU sweep is projected as compute + all-gather at an assumed NVLink rate.
With "local" among the arguments every rank's shard is made by
pr_graph_create_sharded (the rank's edges only); the out-degree all-reduce is
stood in for by writing the graph's out-degrees (what the all-reduce returns),
and each rank's create time is reported too (full ingest: every rank creates
the whole graph, reported as create_full_ms).
Usage: python tools/shard_scaling.py [config] [P ...] [local] > out.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

args = [a for a in sys.argv[1:] if a != "local"]
local = "local" in sys.argv[1:]
cfg = int(args[0]) if args else 4
Ps = [int(a) for a in args[1:]] or [1, 2, 4, 8]
SWEEPS = 20
NVLINK_GBS = 700.0   # assumed effective all-gather receive rate per GPU (NVLink 5: 900 GB/s per direction)
gen = graphgen.make_config(cfg)
s = torch.from_numpy(gen.src).cuda()
t = torch.from_numpy(gen.dst).cuda()
x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
out = {"config": cfg, "workload": gen.name, "sweeps": SWEEPS, "assumed_allgather_GBs": NVLINK_GBS,
       "ingest": "local" if local else "full", "P": {}}
base = None


def timed(fn):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    r = fn()
    b.record(st)
    torch.cuda.synchronize()
    return r, a.elapsed_time(b)


with pr.Graph(gen.n, s, t) as g0:   # the graph's out-degrees (what the all-reduce returns)
    E = g0.info()["E"]
    rp0 = torch.empty(gen.n + 1, dtype=torch.int64, device="cuda")
    col0 = torch.empty(E, dtype=torch.int32, device="cuda")
    od0 = torch.empty(gen.n, dtype=torch.int32, device="cuda")
    pr.pr_get_csr(g0.handle, rp0, col0, od0)
    del rp0, col0
timed(lambda: pr.Graph(gen.n, s, t).close())
_, create_full_ms = timed(lambda: pr.Graph(gen.n, s, t).close())
out["create_full_ms"] = round(create_full_ms, 3)


def allreduce_standin(buf, count, world, stream):
    torch.cuda.synchronize()
    pr.device_i32(buf, count).copy_(od0)


def make(r, P):
    if local:
        return pr.Graph.sharded(gen.n, s, t, r, P, allreduce_standin)
    g = pr.Graph(gen.n, s, t)
    g.shard(r, P)
    return g
for P in Ps:
    per = []
    for r in range(P):
        make(r, P).close()   # warm (pool)
        g, create_ms = timed(lambda: make(r, P))
        with g:
            info = g.shard_info()
            g.run_sharded(x, lambda *a: None, gen.d, 0.0, 3)   # warm
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            g.run_sharded(x, lambda *a: None, gen.d, 0.0, SWEEPS)
            b.record(st)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / SWEEPS
            per.append({"rank": r, "sweep_ms": round(ms, 4), "edges": info["edges"], "rows": info["rows"],
                        "chunk": info["chunk"], "create_ms": round(create_ms, 3)})
    # the fused exchange's kernel-side cost: rank 0 storing every contrib into
    # P - 1 peer buffers (scratch buffers on this GPU stand in for the peers;
    # over NVLink the stores are remote, which this cannot measure)
    if P > 1:
        with make(0, P) as g:
            y0, y1, ln = g.shard_buffers()
            scratch = [(torch.zeros(ln, dtype=torch.float64, device="cuda"),
                        torch.zeros(ln, dtype=torch.float64, device="cuda")) for _ in range(P - 1)]
            p0 = [y0] + [a.data_ptr() for a, _ in scratch]
            p1 = [y1] + [b_.data_ptr() for _, b_ in scratch]
            g.set_peers(p0, p1)
            g.run_sharded(x, lambda *a: None, gen.d, 0.0, 3)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            g.run_sharded(x, lambda *a: None, gen.d, 0.0, SWEEPS)
            b.record(st)
            torch.cuda.synchronize()
            peer_ms = round(a.elapsed_time(b) / SWEEPS, 4)
            del scratch
    else:
        peer_ms = None
    worst = max(p["sweep_ms"] for p in per)
    chunk = per[0]["chunk"]
    recv = (P - 1) * chunk * 8
    comm_ms = recv / (NVLINK_GBS * 1e9) * 1e3
    if base is None:
        base = worst
    rec = {"ranks": per, "slowest_rank_sweep_ms": worst, "rank0_sweep_ms_with_peer_stores_local": peer_ms,
           "allgather_recv_bytes_per_rank": recv,
           "projected_sweep_ms_no_overlap": round(worst + comm_ms, 4),
           "projected_speedup_vs_1gpu": round(base / (worst + comm_ms), 2),
           "edge_imbalance": round(max(p["edges"] for p in per) / (sum(p["edges"] for p in per) / P), 4),
           "slowest_rank_create_ms": max(p["create_ms"] for p in per)}
    out["P"][P] = rec
    print(P, json.dumps(rec)[:300], file=sys.stderr, flush=True)
print(json.dumps(out))
