"""PRGPU_PROFILE=2 breakdown of pr_graph_create_sharded for one rank (tool).
Usage: PRGPU_PROFILE=2 python tools/profile_create_sharded.py [config=4] [P=8] [rank=0]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rank = int(sys.argv[3]) if len(sys.argv) > 3 else 0
gen = graphgen.make_config(cfg)
s = torch.from_numpy(gen.src).cuda()
t = torch.from_numpy(gen.dst).cuda()
with pr.Graph(gen.n, s, t) as g0:
    E = g0.info()["E"]
    rp0 = torch.empty(gen.n + 1, dtype=torch.int64, device="cuda")
    col0 = torch.empty(E, dtype=torch.int32, device="cuda")
    od0 = torch.empty(gen.n, dtype=torch.int32, device="cuda")
    pr.pr_get_csr(g0.handle, rp0, col0, od0)


def standin(buf, count, world, stream):
    torch.cuda.synchronize()
    pr.device_i32(buf, count).copy_(od0)


for rep in range(3):
    print(f"--- rep {rep}", file=sys.stderr, flush=True)
    pr.Graph.sharded(gen.n, s, t, rank, P, standin).close()
    torch.cuda.synchronize()
