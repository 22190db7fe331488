"""Slice-blocked hub gather ceiling (tool).  Splits the relabelled edges of a
config into the rows with in-degree >= T (hub part: grouped by the 16K-slot
slice of their contrib slot, gathered from a shared-memory copy of the slice,
tools/hub_ceiling.cu) and the rest (the flat tiered gather of
tools/gather_ceiling.cu), and times both against the flat gather of all edges.
Usage: python tools/hub_ceiling.py [config=4] [T=256,1024] [tiers=k1,k2,...]
With `tiers=`: instead of hub rows, the edges of ALL rows whose slot lies in tiers 2..k+1
(slots [16K, 16K*(k+1)): the sources just past the shared-memory tier) form the slice part.
A T of 0 skips the hub-row variants."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402


def lib_of(name):
    so = os.path.join(ROOT, "tools", f"lib{name}.so")
    cu = os.path.join(ROOT, "tools", f"{name}.cu")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(cu):
        subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
                               "-fPIC", "-o", so, cu])
    return ctypes.CDLL(so)


so_c = os.path.join(ROOT, "tools", "libceiling.so")
cu_c = os.path.join(ROOT, "tools", "gather_ceiling.cu")
if not os.path.exists(so_c) or os.path.getmtime(so_c) < os.path.getmtime(cu_c):
    subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so_c, cu_c])
ceil = ctypes.CDLL(so_c)
ceil.ceiling_run.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                             ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                             ctypes.POINTER(ctypes.c_float)]
hub = lib_of("hub_ceiling")
hub.hub_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                        ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
Ts = [int(t) for t in (sys.argv[2] if len(sys.argv) > 2 else "256,1024").split(",")]
gen = graphgen.make_config(cfg)
dev = torch.device("cuda:0")
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
del s, t
order = torch.sort(-od.to(torch.int64) * (1 << 32) + torch.arange(n, device=dev)).indices
rank = torch.empty(n, dtype=torch.int64, device=dev)
rank[order] = torch.arange(n, device=dev)
slot = rank[ci.to(torch.int64)]
nslots = int((od > 0).sum())
indeg = rp[1:] - rp[:-1]
rows = torch.repeat_interleave(torch.arange(n, device=dev), indeg)
y = torch.rand(nslots + 1, dtype=torch.float64, device=dev)
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.empty(sms * 8 * 1024, dtype=torch.float64, device=dev)


def flat(col, hot=16384):
    ms = ctypes.c_float()
    best = 1e9
    for _ in range(3):
        ceil.ceiling_run(col.data_ptr(), col.numel(), y.data_ptr(), hot, 2, 1, 5, 1024, -32768, out.data_ptr(),
                         ctypes.byref(ms))
        best = min(best, ms.value)
    return best


allcol = slot.to(torch.int32).contiguous()
t_all = flat(allcol)
print(f"{gen.name}: E={E} flat tiered gather of all edges {t_all:.4f} ms", flush=True)
SL, U = 16384, 32
tiers = []
for a in sys.argv[3:]:
    if a.startswith("tiers="):
        tiers = [int(k) for k in a[6:].split(",")]
variants = [("T", T) for T in Ts if T > 0] + [("tiers", k) for k in tiers]
for kind, T in variants:
    if kind == "T":
        hubm = indeg[rows] >= T
    else:
        hubm = (slot >= SL) & (slot < SL * (1 + T))
    rest = allcol[~hubm].contiguous()
    hs = slot[hubm]
    q = hs // SL
    key = torch.sort(q * (1 << 32) + torch.arange(hs.numel(), device=dev)).values  # stable by slice
    idx = key & 0xffffffff
    hs = hs[idx]
    q = hs // SL
    cnt = torch.bincount(q, minlength=(nslots + SL - 1) // SL)
    unit_e = U * 256
    padded = (cnt + unit_e - 1) // unit_e * unit_e
    offs = torch.cumsum(padded, 0) - padded
    tot = int(padded.sum())
    lsl = torch.full((tot,), SL, dtype=torch.int32, device=dev)
    start = torch.cumsum(cnt, 0) - cnt
    pos = offs[q] + (torch.arange(hs.numel(), device=dev) - start[q])
    lsl[pos] = (hs - q * SL).to(torch.int32)
    lsl16 = lsl.to(torch.int16).contiguous()
    nunits = tot // unit_e
    us = torch.repeat_interleave(torch.arange(cnt.numel(), device=dev, dtype=torch.int32), padded // unit_e).contiguous()
    ms = ctypes.c_float()
    best = 1e9
    for _ in range(3):
        rc = hub.hub_run(lsl16.data_ptr(), us.data_ptr(), nunits, U, y.data_ptr(), nslots, out.data_ptr(), 5,
                         ctypes.byref(ms))
        best = min(best, ms.value)
    t_rest = flat(rest)
    print(f"{kind}={T}: hub edges {hs.numel() / E:.3f} of E (padded {tot / max(1, hs.numel()):.3f}x, {nunits} units), "
          f"hub part {best:.4f} ms (rc {rc}), rest {rest.numel() / E:.3f} of E {t_rest:.4f} ms, "
          f"sum {best + t_rest:.4f} ms vs flat {t_all:.4f} ms", flush=True)
