"""Time to converge of several modes on one BASELINE config, measured
interleaved (mode A, B, C, A, B, C, ...) so clock / power drift hits every mode
alike; median of the reps, plus the PR_TIMING gather / finalize split (tool).
Usage: python tools/mode_times.py <config> [reps=7] [modes=plain,reduced,async]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

MODES = {"plain": 0, "reduced": pr.PR_USE_REDUCTIONS, "eager": pr.PR_USE_REDUCTIONS | pr.PR_CHAIN_EAGER,
         "phased": pr.PR_MODE_PHASED, "async": pr.PR_MODE_ASYNC, "nosync": pr.PR_MODE_NOSYNC,
         "perforated": pr.PR_PERFORATE}
k = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
names = (sys.argv[3] if len(sys.argv) > 3 else "plain,reduced,async").split(",")
gen = graphgen.make_config(k)
s = torch.from_numpy(gen.src).cuda()
t = torch.from_numpy(gen.dst).cuda()
x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
g = pr.Graph(gen.n, s, t)
g.preprocess()
times = {m: [] for m in names}
iters = {}
for m in names:  # warm-up (fold tables, phase views, pools)
    g.run(x, gen.d, gen.tau, gen.max_iter, mode=MODES[m])
for _ in range(reps):
    for m in names:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        rc, it, _ = g.run(x, gen.d, gen.tau, gen.max_iter, mode=MODES[m])
        b.record(st)
        torch.cuda.synchronize()
        times[m].append(a.elapsed_time(b))
        iters[m] = (it, rc)
out = {"config": k, "workload": gen.name, "reps": reps, "lib": os.environ.get("PRGPU_LIB", "default")}
for m in names:
    g.run(x, gen.d, gen.tau, gen.max_iter, mode=MODES[m] | pr.PR_TIMING)
    ss = g.stats()
    ti = max(1, ss["timed_iterations"])
    v = sorted(times[m])
    out[m] = {"median_ms": round(v[len(v) // 2], 3), "min_ms": round(v[0], 3), "iterations": iters[m][0],
              "status": iters[m][1], "gather_ms": round(ss["gather_ms"] / ti, 4),
              "finalize_ms": round(ss["scatter_ms"] / ti, 4)}
print(json.dumps(out))
