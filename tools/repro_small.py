import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2109_09527_b200 as pr
n = 4
s = torch.zeros(50, dtype=torch.int32, device="cuda")
t = torch.ones(50, dtype=torch.int32, device="cuda")
g = pr.Graph(n, s, t)
rp = torch.empty(n + 1, dtype=torch.int64, device="cuda"); col = torch.empty(1, dtype=torch.int32, device="cuda")
od = torch.empty(n, dtype=torch.int32, device="cuda")
pr.pr_get_csr(g.handle, rp, col, od)
print(rp.cpu().numpy(), col.cpu().numpy(), od.cpu().numpy())
