"""Time pr_graph_create / pr_preprocess on config k (CUDA events, after warm-up).
Usage: python tools/time_create.py [config=4] [reps=3]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
gen = graphgen.make_config(cfg)
s = torch.from_numpy(gen.src).cuda()
t = torch.from_numpy(gen.dst).cuda()
stream = torch.cuda.current_stream()
cr, pp = [], []
for i in range(reps + 1):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(stream)
    g = pr.Graph(gen.n, s, t)
    e[1].record(stream)
    g.preprocess()
    e[2].record(stream)
    torch.cuda.synchronize()
    if i:
        cr.append(e[0].elapsed_time(e[1]))
        pp.append(e[1].elapsed_time(e[2]))
    info = g.info()
    g.close()
print(f"{gen.name}: E={info['E']} members={info['n_members']} create ms {min(cr):.2f} (all {[round(x, 2) for x in cr]}) "
      f"preprocess ms {min(pp):.2f}")
