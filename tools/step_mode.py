"""One pr_run of config k in a given mode (for ncu captures of the in-place,
No-Sync and blocked kernels).  Usage: python tools/step_mode.py <config> <mode>
mode: async | nosync | plain | perforate"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

cfg, mode = int(sys.argv[1]), sys.argv[2]
gen = graphgen.make_config(cfg)
s = torch.from_numpy(gen.src).cuda()
t = torch.from_numpy(gen.dst).cuda()
x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
g = pr.Graph(gen.n, s, t)
m = {"async": pr.PR_MODE_ASYNC, "nosync": pr.PR_MODE_NOSYNC, "plain": 0, "perforate": pr.PR_PERFORATE}[mode]
st, it, fd = g.run(x, gen.d, gen.tau, gen.max_iter, mode=m)
print(gen.name, mode, "status", st, "iters", it, "delta", fd)
g.close()
