import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2109_09527_b200 as pr
from tests import graphs as G
import oracle
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
for name, (n, edges) in [("complete", (12, G.complete(12))), ("dups", (4, [(0, 1)] * 50)), ("dups2", (4, [(0, 1)] * 50))]:
    s, t = G.edges_to_arrays(edges)
    g = pr.Graph(n, dev(s), dev(t))
    E = g.info()["E"]
    rp = torch.empty(n + 1, dtype=torch.int64, device="cuda"); col = torch.empty(max(E,1), dtype=torch.int32, device="cuda")
    od = torch.empty(n, dtype=torch.int32, device="cuda")
    pr.pr_get_csr(g.handle, rp, col, od)
    print(name, "E", E, rp.cpu().numpy()[:6], od.cpu().numpy()[:6], flush=True)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    print(g.run(x, 0.85, 1e-13, 1000), flush=True)
    g.preprocess()
    print(g.run(x, 0.85, 1e-13, 1000, mode=pr.PR_USE_REDUCTIONS), flush=True)
    print(g.run(x, 0.85, 1e-13, 1000, mode=pr.PR_MODE_ASYNC), flush=True)
    g.close()
