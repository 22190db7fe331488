"""Repeat full steps (create, preprocess, reduced run, destroy) on config k and
print per-phase CUDA-event times.  Usage: python tools/loop_step.py [config=4] [steps=4]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
gen = graphgen.make_config(cfg)
s = torch.from_numpy(gen.src).cuda()
t = torch.from_numpy(gen.dst).cuda()
x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
best = None
for i in range(steps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(st)
    g = pr.Graph(gen.n, s, t)
    e[1].record(st)
    g.preprocess()
    e[2].record(st)
    g.run(x, gen.d, gen.tau, gen.max_iter, mode=pr.PR_USE_REDUCTIONS)
    e[3].record(st)
    g.close()
    torch.cuda.synchronize()
    r = [e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])]
    if i and (best is None or sum(r) < sum(best)):
        best = r
print(f"{os.environ.get('PRGPU_LIB', 'libprgpu.so').split('/')[-1]} {gen.name}: create {best[0]:.2f} "
      f"preprocess {best[1]:.2f} run {best[2]:.2f} total {sum(best):.2f} ms")
