"""Profiling driver: build config k on the GPU and run a fixed number of sweeps.
Usage: python tools/prof_run.py <config> <mode: plain|reduced|async|nosync|phased|..._reduced> <sweeps> [scale_override]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

cfg = int(sys.argv[1])
mode = sys.argv[2]
sweeps = int(sys.argv[3])
scale = int(sys.argv[4]) if len(sys.argv) > 4 else None
gen = graphgen.make_config(cfg, scale_override=scale)
s = torch.from_numpy(gen.src).cuda()
t = torch.from_numpy(gen.dst).cuda()
x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
g = pr.Graph(gen.n, s, t)
m = {"plain": 0, "reduced": pr.PR_USE_REDUCTIONS, "async": pr.PR_MODE_ASYNC, "nosync": pr.PR_MODE_NOSYNC,
     "nosync_reduced": pr.PR_MODE_NOSYNC | pr.PR_USE_REDUCTIONS, "phased": pr.PR_MODE_PHASED,
     "phased_reduced": pr.PR_MODE_PHASED | pr.PR_USE_REDUCTIONS}[mode]
if "reduced" in mode:
    g.preprocess()
st, it, fd = g.run(x, gen.d, 0.0, sweeps, mode=m | pr.PR_TIMING)
stt = g.stats()
ti = max(1, stt["timed_iterations"])
print(gen.name, mode, "iters", it, "gather ms/launch", round(stt["gather_ms"] / ti, 4),
      "finalize/scatter ms/launch", round(stt["scatter_ms"] / ti, 4),
      "rows", stt["gather_rows"], "edges", stt["gather_edges"], "ncontrib", stt["n_contrib"])
g.close()
