"""A/B of dynamic span assignment (PRGPU_DYN_SPAN=F) against static spans on
one config: gather ms per sweep, time to converge, and the max |x| difference
to the static run (different span layouts sum in a different order).
Usage: python tools/dyn_span_ab.py [config] [F ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
Fs = [int(a) for a in sys.argv[2:]] or [0, 4, 8, 16, 32]
gen = graphgen.make_config(cfg)
g = pr.Graph(gen.n, torch.from_numpy(gen.src).cuda(), torch.from_numpy(gen.dst).cuda())
g.preprocess()
x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
ref = None
for F in Fs:
    os.environ["PRGPU_DYN_SPAN"] = str(F)
    os.environ["PRGPU_TIMING_STRIDE"] = "1"
    g.run(x, gen.d, 0.0, 30, mode=pr.PR_USE_REDUCTIONS | pr.PR_TIMING)
    s = g.stats()
    gms = s["gather_ms"] / max(1, s["timed_iterations"])
    os.environ["PRGPU_TIMING_STRIDE"] = "4"
    best = None
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        rc, it, fd = g.run(x, gen.d, gen.tau, gen.max_iter, mode=pr.PR_USE_REDUCTIONS)
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    xs = x.clone()
    if ref is None:
        ref = xs
    print(f"F={F:3d} gather {gms:.4f} ms/sweep  converge {best:.3f} ms  iters {it}  "
          f"max|dx| vs first {float((xs - ref).abs().max()):.3e}", flush=True)
