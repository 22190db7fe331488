"""Exercise every kernel path on small graphs, for compute-sanitizer
(memcheck / racecheck / initcheck / synccheck).
Usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402
from tests import graphs as G  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def graphs():
    yield "planted", G.planted_graph(1, n_base=150, chains=(2, 9, 16, 1))
    n = 300
    yield "random", (n, G.random_edges(n, 4 * n, 7))
    yield "in_star", (2000, G.in_star(2000))
    yield "path", (500, G.path(500))
    yield "dups", (4, [(0, 1)] * 50)
    yield "single", (1, [])
    gen = graphgen.make_config(4, scale_override=12)
    yield "rmat12", (gen.n, list(zip(gen.src.tolist(), gen.dst.tolist())))


MODES = [0, pr.PR_USE_REDUCTIONS, pr.PR_MODE_ASYNC, pr.PR_MODE_ASYNC | pr.PR_USE_REDUCTIONS, pr.PR_MODE_NOSYNC,
         pr.PR_MODE_NOSYNC | pr.PR_USE_REDUCTIONS, pr.PR_PERFORATE, pr.PR_PERFORATE | pr.PR_MODE_ASYNC,
         pr.PR_PERFORATE | pr.PR_MODE_NOSYNC, pr.PR_NORM_LINF, pr.PR_MODE_PHASED,
         pr.PR_MODE_PHASED | pr.PR_USE_REDUCTIONS]

env_sets = [{}, {"PRGPU_SEG_BITS": "5"}, {"PRGPU_SPAN": "1", "PRGPU_PHASES": "16"}, {"PRGPU_PHASES": "3"}]
runs = 0
for envs in env_sets:
    for k, v in envs.items():
        os.environ[k] = v
    for name, (n, edges) in graphs():
        s, t = G.edges_to_arrays(edges)
        with pr.Graph(n, dev(s), dev(t)) as g:
            g.preprocess()
            x = torch.empty(n, dtype=torch.float64, device="cuda")
            for m in MODES:
                g.run(x, 0.85, 1e-12, 300, mode=m)
                runs += 1
            rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
            col = torch.empty(max(1, g.info()["E"]), dtype=torch.int32, device="cuda")
            od = torch.empty(n, dtype=torch.int32, device="cuda")
            pr.pr_get_csr(g.handle, rp, col, od)
    for k in envs:
        del os.environ[k]
torch.cuda.synchronize()
print(f"sanitize_run: {runs} runs ok")
