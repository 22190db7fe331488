"""Worker of tests/test_gpu_shard.py::test_sharded_multiprocess: one rank of a
torchrun job (gloo process group, every rank on cuda:0) running the sharded
iteration through the real torch.distributed exchange, then checking the
assembled ranks against the oracle on rank 0.  Usage (torchrun):
  shard_worker.py <config> <out.json> [peers|local]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import graphgen  # noqa: E402
import oracle  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

cfg, out = int(sys.argv[1]), sys.argv[2]
peers = len(sys.argv) > 3 and sys.argv[3] == "peers"
local = len(sys.argv) > 3 and sys.argv[3] == "local"   # pr_graph_create_sharded: per-rank ingest
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
gen = graphgen.make_config(cfg)
src_d, dst_d = torch.from_numpy(gen.src).cuda(), torch.from_numpy(gen.dst).cuda()
if local:
    graph = pr.Graph.sharded(gen.n, src_d, dst_d, rank, world, pr.torch_dist_allreduce())
else:
    graph = pr.Graph(gen.n, src_d, dst_d)
with graph as g:
    if not local:
        g.shard(rank, world)
    if peers:  # the exchange fused into the kernels: CUDA IPC buffers, barrier-only exchange
        pr.torch_dist_peer_setup(g.handle)
    x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
    st, it, fd = g.run_sharded(x, pr.torch_dist_exchange(), gen.d, gen.tau, gen.max_iter)
    info = g.shard_info()
xs = x.cpu()
dist.all_reduce(xs)                       # disjoint owned parts: the sum is exact
res = [None] * world
dist.all_gather_object(res, {"st": st, "it": it, "fd": fd, "info": info})
if rank == 0:
    ref_g = oracle.build_csr(gen.n, gen.src, gen.dst)
    ref = oracle.pagerank(ref_g, gen.d, gen.tau, gen.max_iter)
    diff = np.abs(xs.numpy() - ref.x)
    json.dump({"ranks": res, "max_diff": float(diff.max()), "l1_diff": float(diff.sum()),
               "oracle_iters": ref.iters, "oracle_status": ref.status,
               "oracle_log": ref.delta_log[:, 0].tolist()}, open(out, "w"))
dist.barrier()
dist.destroy_process_group()
