"""Gather-ceiling microbenchmark (tool): how fast can ANY kernel stream the
relabelled col array of a config and gather y[col] on this B200?

Usage: python tools/gather_ceiling.py [config=4]
Prints one line per variant (ms per pass, G gathers/s, wavefront estimate).
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
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so, os.path.join(ROOT, "tools", "gather_ceiling.cu")])
lib = ctypes.CDLL(so)
lib.ceiling_tma.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                            ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]
lib.ceiling_run.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]

lib.ceiling_cluster.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int)]

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
which = sys.argv[2] if len(sys.argv) > 2 else "all"
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
# relabel sources by (outdeg desc, id asc), as K-GATHER's contrib slots
order = torch.sort(-od.to(torch.int64) * (1 << 32) + torch.arange(n, device=dev)).indices
cidx = torch.empty(n, dtype=torch.int64, device=dev)
cidx[order] = torch.arange(n, device=dev)
col = cidx[ci.to(torch.int64)].to(torch.int32).contiguous()
nsrc = int((od > 0).sum())
y = torch.rand(nsrc, dtype=torch.float64, device=dev)
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.empty(sms * 8 * 1024, dtype=torch.float64, device=dev)
clk = 1.965e9


REF = {}


def check(colv, label):
    # every variant sums y[col[e]] over the same whole chunks; compare the totals
    tot = float(out.sum())
    key = colv.data_ptr()
    if key not in REF:
        REF[key] = tot
    rel = abs(tot - REF[key]) / abs(REF[key])
    assert rel < 1e-9, (label, tot, REF[key])


def run_tma(colv, stages, threads, label="skewed TMA gather4"):
    ms = ctypes.c_float()
    out.zero_()
    rc = lib.ceiling_tma(colv.data_ptr(), colv.numel() // 128 * 128, y.data_ptr(), nsrc, stages, threads, 10,
                         out.data_ptr(), ctypes.byref(ms))
    assert rc == 0, rc
    check(colv, label)
    gps = colv.numel() / (ms.value * 1e-3) / 1e9
    print(f"{label:38s} stages={stages} thr={threads}: {ms.value:.4f} ms  {gps:7.1f} G gathers/s  "
          f"{gps * 1e9 / (sms * clk):.3f} gathers/SM/cycle@1965MHz", flush=True)


def run(colv, hot, unroll, cps, label, threads=256, tier=0):
    ms = ctypes.c_float()
    out.zero_()
    rc = lib.ceiling_run(colv.data_ptr(), colv.numel(), y.data_ptr(), hot, unroll, cps, 10, threads, tier, out.data_ptr(),
                         ctypes.byref(ms))
    assert rc == 0, rc
    if unroll == 1:
        check(colv, label)
    gps = colv.numel() / (ms.value * 1e-3) / 1e9
    print(f"{label:38s} hot={hot:6d} U={unroll} ctas/sm={cps} thr={threads} tier={tier}: {ms.value:.4f} ms  {gps:7.1f} G gathers/s  "
          f"{gps * 1e9 / (sms * clk):.3f} gathers/SM/cycle@1965MHz", flush=True)


def run_cluster(colv, HL, HD, cl, tier=0, label="skewed + cluster DSMEM tier"):
    ms = ctypes.c_float()
    grid = ctypes.c_int()
    out.zero_()
    E4 = colv.numel() // 512 * 512
    rc = lib.ceiling_cluster(colv.data_ptr(), E4, y.data_ptr(), HL, HD, cl, tier, 10, out.data_ptr(),
                             ctypes.byref(ms), ctypes.byref(grid))
    assert rc == 0, rc
    gps = E4 / (ms.value * 1e-3) / 1e9
    print(f"{label:38s} CL={cl} HL={HL:6d} HD={HD:6d} (on-chip {HL + cl * HD:7d}) tier={tier} grid={grid.value}: "
          f"{ms.value:.4f} ms  {gps:7.1f} G gathers/s  {gps * 1e9 / (sms * clk):.3f} gathers/SM/cycle@1965MHz", flush=True)


lib.ceiling_hybrid.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                               ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_void_p,
                               ctypes.POINTER(ctypes.c_float)]


def run_hybrid(colv, nT, stages, frac, label):
    ms = ctypes.c_float()
    out.zero_()
    E128 = colv.numel() // 128 * 128
    rc = lib.ceiling_hybrid(colv.data_ptr(), E128, y.data_ptr(), nsrc, nT, stages, frac, 10, out.data_ptr(),
                            ctypes.byref(ms))
    assert rc == 0, rc
    gps = E128 / (ms.value * 1e-3) / 1e9
    print(f"{label:38s} tma_warps={nT:2d} stages={stages} tma_frac={frac:.2f}: {ms.value:.4f} ms  {gps:7.1f} G gathers/s  "
          f"{gps * 1e9 / (sms * clk):.3f} gathers/SM/cycle@1965MHz", flush=True)


print(f"{gen.name}: n={n} E={E} sources={nsrc}")
if which == "hybrid":
    u = torch.randint(0, nsrc, (E,), dtype=torch.int32, device=dev)
    run_hybrid(u, 0, 2, 0.0, "uniform, LDG warps only (32)")
    run_hybrid(u, 32, 1, 1.0, "uniform, TMA warps only (32)")
    for nT in (4, 8, 12, 16):
        for frac in (0.15, 0.25, 0.35, 0.45):
            run_hybrid(u, nT, 2, frac, "uniform, hybrid")
    run_hybrid(u, 8, 3, 0.3, "uniform, hybrid")
    run_hybrid(u, 8, 4, 0.3, "uniform, hybrid")
    sys.exit(0)
if which == "cluster":
    run(col, 16384, 4, 1, "skewed + hot smem + L1 tier (current)", threads=1024, tier=32768)
    for cl, HL, HD, tier in ((1, 16384, 0, 32768), (2, 16384, 12288, 0), (2, 16384, 12288, 65536),
                             (2, 8192, 20480, 0), (2, 0, 28672, 0), (4, 16384, 12288, 0), (4, 8192, 20480, 0),
                             (4, 0, 28672, 0), (8, 8192, 20480, 0), (8, 0, 28672, 0)):
        try:
            run_cluster(col, HL, HD, cl, tier)
        except AssertionError as e:
            print("cluster variant failed", cl, HL, HD, e, flush=True)
    sys.exit(0)
for mb in (4, 8, 16, 24, 32, 48, 64, 96):
    slots = mb * (1 << 20) // 8
    u = torch.randint(0, min(slots, nsrc), (E,), dtype=torch.int32, device=dev)
    run(u, 0, 4, 2, f"uniform over {mb} MB", threads=1024)
    del u
import sys as _s
_s.exit(0)
for tier in (0, 8192, 32768, 65536):
    run(col, 0, 4, 2, "skewed, L1 tier", threads=1024, tier=tier)
for hot in (12288, 16384, 20480):
    for tier in (0, 32768, 65536):
        run(col, hot, 4, 1, "skewed + hot smem + L1 tier", threads=1024, tier=tier)
