"""Correlate per-warp gather time (PRGPU_TRACE) with the rows of each warp's
span, plain view of config k (one span per warp).  Usage:
  python tools/trace_rows.py <config> <trace-out>   (runs the plain sweep itself)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

cfg, tr = int(sys.argv[1]), sys.argv[2]
os.environ["PRGPU_TRACE"] = tr
gen = graphgen.make_config(cfg)
g = pr.Graph(gen.n, torch.from_numpy(gen.src).cuda(), torch.from_numpy(gen.dst).cuda())
x = torch.empty(gen.n, dtype=torch.float64, device="cuda")
g.run(x, gen.d, 0.0, 3)
rp = torch.empty(gen.n + 1, dtype=torch.int64, device="cuda")
col = torch.empty(g.info()["E"], dtype=torch.int32, device="cuda")
od = torch.empty(gen.n, dtype=torch.int32, device="cuda")
pr.pr_get_csr(g.handle, rp, col, od)
rp, col, od = rp.cpu().numpy(), col.cpu().numpy(), od.cpu().numpy()
deg = np.diff(rp)
starts = np.cumsum(np.r_[0, deg[deg > 0]])[:-1]          # plain view: rows of in-degree > 0, vertex order
E = int(rp[-1])
nsteps = (E + 255) // 256
a = np.loadtxt(tr).reshape(-1, 2)
W = len(a)
ss = -(-nsteps // W)
nspans = -(-nsteps // ss)
span_rows = np.bincount(np.minimum(starts // (ss * 256), nspans - 1), minlength=nspans)
busy = (a[:nspans, 1] - a[:nspans, 0]) / 1e3
ok = busy > 0
full = np.arange(nspans) < nspans - 1
sel = ok & full
c = np.corrcoef(busy[sel], span_rows[sel])[0, 1]
print(f"spans {nspans} steps/span {ss}; busy us mean {busy[sel].mean():.1f} std {busy[sel].std():.1f}; "
      f"rows/span mean {span_rows[sel].mean():.0f} std {span_rows[sel].std():.0f}; corr(busy, rows) = {c:.3f}")
A = np.vstack([span_rows[sel], np.ones(sel.sum())]).T
coef = np.linalg.lstsq(A, busy[sel], rcond=None)[0]
print(f"busy ~ {coef[1]:.1f} us + {coef[0] * 1e3:.3f} ns/row  (rows explain {c * c * 100:.0f} % of the variance)")
# cold gathers: sources outside the 32K highest out-degree vertices (the shared-memory + L1 tiers)
order = np.argsort(-od, kind="stable")
tier = np.full(gen.n, 2, np.int8)
tier[order[:16384]] = 0
tier[order[16384:32768]] = 1
t = tier[col]
span_of_edge = np.minimum(np.arange(E) // (ss * 256), nspans - 1)
cold = np.bincount(span_of_edge, weights=(t == 2), minlength=nspans)
l1 = np.bincount(span_of_edge, weights=(t == 1), minlength=nspans)
A = np.vstack([span_rows[sel], cold[sel], l1[sel], np.ones(sel.sum())]).T
coef, res, *_ = np.linalg.lstsq(A, busy[sel], rcond=None)
pred = A @ coef
r2 = 1 - ((busy[sel] - pred) ** 2).sum() / ((busy[sel] - busy[sel].mean()) ** 2).sum()
print(f"cold/span mean {cold[sel].mean():.0f} std {cold[sel].std():.0f}; corr(busy, cold) = "
      f"{np.corrcoef(busy[sel], cold[sel])[0, 1]:.3f}")
print(f"busy ~ {coef[3]:.1f} us + {coef[0] * 1e3:.2f} ns/row + {coef[1] * 1e3:.3f} ns/cold + {coef[2] * 1e3:.3f} ns/L1-tier"
      f"  (R^2 = {r2:.2f}); residual std {np.std(busy[sel] - pred):.1f} us")
