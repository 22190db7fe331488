"""LDG vs cp.async.cg (L1-bypassing LDGSTS) for the random contrib gather (tool;
tools/cpasync_ceiling.cu).  Flat gather over (a) uniform random slots and (b) the
relabelled col array of a config, with several shared-memory tier sizes.
Usage: python tools/cpasync_ceiling.py [config=4]"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

so = os.path.join(ROOT, "tools", "libcpasync_ceiling.so")
cu = os.path.join(ROOT, "tools", "cpasync_ceiling.cu")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(cu):
    subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                           "-o", so, cu])
lib = ctypes.CDLL(so)
lib.cpasync_run.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                            ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dev = torch.device("cuda:0")
gen = graphgen.make_config(cfg)
s = torch.from_numpy(gen.src).to(dev)
t = torch.from_numpy(gen.dst).to(dev)
g = pr.Graph(gen.n, s, t)
info = g.info()
n, E = info["n"], info["E"]
rp = torch.empty(n + 1, dtype=torch.int64, device=dev)
ci = torch.empty(E, dtype=torch.int32, device=dev)
od = torch.empty(n, dtype=torch.int32, device=dev)
pr.pr_get_csr(g.handle, rp, ci, od)
g.close()
del s, t, rp
order = torch.sort(-od.to(torch.int64) * (1 << 32) + torch.arange(n, device=dev)).indices
rank = torch.empty(n, dtype=torch.int64, device=dev)
rank[order] = torch.arange(n, device=dev)
real = rank[ci.to(torch.int64)].to(torch.int32).contiguous()
nslots = int((od > 0).sum())
del rank, order, ci
uni = torch.randint(0, nslots, (E,), dtype=torch.int32, device=dev)
y = torch.rand(nslots + 2, dtype=torch.float64, device=dev)
out = torch.empty(148 * 1024 * 2, dtype=torch.float64, device=dev)


def run(col, hot, a):
    ms = ctypes.c_float()
    best = 1e9
    for _ in range(3):
        rc = lib.cpasync_run(col.data_ptr(), col.numel(), y.data_ptr(), hot, a, 5, out.data_ptr(), ctypes.byref(ms))
        assert rc == 0, rc
        best = min(best, ms.value)
    return best


print(f"{gen.name}: E={E} slots={nslots}")
for name, col in (("uniform", uni), ("relabelled col", real)):
    for hot in (0, 4096, 8192, 12288):
        l, a = run(col, hot, 0), run(col, hot, 1)
        print(f"{name:15s} hot={hot:6d}: LDG {l:.4f} ms, cp.async.cg {a:.4f} ms", flush=True)
    l = run(col, 16384, 0), run(col, 20480, 0)
    print(f"{name:15s} LDG only, hot=16384 / 20480: {l[0]:.4f} / {l[1]:.4f} ms", flush=True)
