"""Time to converge and sweeps of PR_MODE_PHASED for several phase counts
(PRGPU_PHASES is read per run), against sync and async, on one config.
Usage: python tools/phase_sweep.py [config] [K ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
Ks = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8, 16, 32, 64]
gen = graphgen.make_config(cfg)
s = torch.from_numpy(gen.src).cuda()
t = torch.from_numpy(gen.dst).cuda()
g = pr.Graph(gen.n, s, t)
g.preprocess()
x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()


def timed(mode, reps=3):
    best = None
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        rc, it, fd = g.run(x, gen.d, gen.tau, gen.max_iter, mode=mode)
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        if best is None or ms < best[0]:
            best = (round(ms, 3), it, rc)
    return best


out = {"config": cfg, "workload": gen.name}
for red in (0, pr.PR_USE_REDUCTIONS):
    tag = "reduced" if red else "plain"
    out[f"{tag}_sync"] = timed(red)
    out[f"{tag}_async"] = timed(red | pr.PR_MODE_ASYNC)
    for K in Ks:
        os.environ["PRGPU_PHASES"] = str(K)
        r = timed(red | pr.PR_MODE_PHASED)
        out[f"{tag}_phased{K}"] = r + (g.stats()["phases"],)
        print(tag, K, r, file=sys.stderr, flush=True)
print(json.dumps(out))
