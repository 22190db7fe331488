"""One bench step (create + preprocess + reduced run + destroy) on config k, for launch lists."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mode = sys.argv[2] if len(sys.argv) > 2 else "reduced"
gen = graphgen.make_config(cfg)
s = torch.from_numpy(gen.src).cuda()
t = torch.from_numpy(gen.dst).cuda()
x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
g = pr.Graph(gen.n, s, t)
m = 0
if mode == "reduced":
    g.preprocess()
    m = pr.PR_USE_REDUCTIONS
st, it, fd = g.run(x, gen.d, gen.tau, gen.max_iter, mode=m)
print(gen.name, mode, "iters", it, g.stats()["total_launches"], "launches")
g.close()
torch.cuda.synchronize()
