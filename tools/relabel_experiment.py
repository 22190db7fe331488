"""Contrib-slot relabelling experiment (tool): does ordering the COLD sources
(beyond the shared-memory + L1 hot tiers) by their first appearance in the
edge stream cut the L2 requests of the flat gather?

The gather-ceiling kernel (tools/gather_ceiling.cu, acc += y[col[e]], lane L
owning 8 consecutive edges of each 256-edge step like K-GATHER) runs over the
SAME edges with the contrib slots assigned as
  degree : (outdeg desc, id asc)                                   (K-GATHER's)
  first  : the top H by degree as before, the rest by the first edge that
           gathers them (consecutive first-gathers share 32-byte sectors)
and the cold gathers loaded with L1::no_allocate, L1::evict_first or default.
Usage: python tools/relabel_experiment.py [config=4] [H=32768]
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2109_09527_b200 as pr  # noqa: E402

so = os.path.join(ROOT, "tools", "libceiling.so")
src_cu = os.path.join(ROOT, "tools", "gather_ceiling.cu")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src_cu):
    subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so, src_cu])
lib = ctypes.CDLL(so)
lib.ceiling_run.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                            ctypes.POINTER(ctypes.c_float)]
lib.ceiling_set_cold.argtypes = [ctypes.c_int]

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
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
ci64 = ci.to(torch.int64)
order = torch.sort(-od.to(torch.int64) * (1 << 32) + torch.arange(n, device=dev)).indices
deg_rank = torch.empty(n, dtype=torch.int64, device=dev)
deg_rank[order] = torch.arange(n, device=dev)
nsrc = int((od > 0).sum())

# first edge that gathers each source
first = torch.full((n,), E, dtype=torch.int64, device=dev)
first.scatter_reduce_(0, ci64, torch.arange(E, device=dev), reduce="amin")
cold = deg_rank >= H
key = torch.where(cold, H + first, deg_rank)          # hot keep their degree rank (< H), cold by first edge
key = torch.where(od > 0, key, torch.full_like(key, 1 << 62))
ord2 = torch.sort(key).indices
first_rank = torch.empty(n, dtype=torch.int64, device=dev)
first_rank[ord2] = torch.arange(n, device=dev)

# cold sources in vertex-id order (rows and slots both ascending: K-FINALIZE's
# contrib stores of the cold rows would be coalesced)
key3 = torch.where(cold, H + torch.arange(n, device=dev), deg_rank)
key3 = torch.where(od > 0, key3, torch.full_like(key3, 1 << 62))
ord3 = torch.sort(key3).indices
id_rank = torch.empty(n, dtype=torch.int64, device=dev)
id_rank[ord3] = torch.arange(n, device=dev)

y = torch.rand(nsrc, dtype=torch.float64, device=dev)
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.empty(sms * 8 * 1024, dtype=torch.float64, device=dev)
rows = torch.repeat_interleave(torch.arange(n, device=dev), (rp[1:] - rp[:-1]))
variants = (("degree", deg_rank, False), ("rowsorted", deg_rank, True))
if len(sys.argv) > 3:
    variants = variants + (("first", first_rank, False), ("idorder", id_rank, False))
for name, rank, rowsort in variants:
    col = rank[ci64].to(torch.int32).contiguous()
    if rowsort:   # each row's edges ascending by contrib slot (sum order only)
        key = rows * (1 << 32) + col.to(torch.int64)
        col = (torch.sort(key).values & 0xffffffff).to(torch.int32).contiguous()
        del key
    # sectors per warp instruction (32 lanes x 1 gather, lane L = edges 8L..8L+7
    # of a step) for the cold gathers: distinct 32-byte sectors of one lane's 8
    # gathers (what L1 allocation can merge)
    c = col[: (E // 256) * 256].view(-1, 32, 8).to(torch.int64)
    sect = c // 4
    coldm = c >= H
    lane_sect = torch.where(coldm, sect, torch.full_like(sect, -1))
    srt = torch.sort(lane_sect, dim=2).values
    distinct = ((srt[:, :, 1:] != srt[:, :, :-1]) & (srt[:, :, 1:] >= 0)).sum() + (srt[:, :, 0] >= 0).sum()
    ncold = int(coldm.sum())
    for cm, cname in ((0, "no_allocate"), (1, "evict_first"), (2, "default")):
        lib.ceiling_set_cold(cm)
        ms = ctypes.c_float()
        best = 1e9
        for _ in range(3):
            lib.ceiling_run(col.data_ptr(), E, y.data_ptr(), 16384, 2, 1, 5, 1024, -H, out.data_ptr(),
                            ctypes.byref(ms))
            best = min(best, ms.value)
        print(f"{gen.name} slots={name:7s} cold={cname:12s} {best:.4f} ms/pass  {E / best / 1e6:.1f} G gathers/s  "
              f"cold gathers {ncold / E:.3f} of E, distinct cold sectors per lane-step {int(distinct) / max(1, ncold):.3f}",
              flush=True)
