"""paper_2109_09527_b200 -- Python binding of libprgpu (include/prgpu.h).

Argument marshalling only: every step of the PageRank path (ingest,
preprocessing, the iteration) runs in libprgpu's CUDA kernels for sm_100a.
There is no CPU fallback: importing this package on a machine without the
built ``libprgpu.so`` raises immediately, and calls without a CUDA device fail
with the library's own error.

The names mirror the C ABI: :func:`pr_graph_create`, :func:`pr_preprocess`,
:func:`pr_run`, :func:`pr_destroy` (+ introspection).  Buffers may be torch
tensors (CUDA or CPU) or numpy arrays; the library accepts host or device
pointers and copies host data inside the call.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PRGPU_LIB") or os.path.join(_HERE, "libprgpu.so")

PR_OK = 0
PR_EINVAL = 1
PR_NOT_CONVERGED = 2
PR_ESTATE = 3
PR_ENOMEM = -1
PR_ECUDA = -2

PR_PRE_IDENTICAL = 1
PR_PRE_CHAIN = 2

PR_MODE_SYNC = 0
PR_MODE_ASYNC = 1
PR_NORM_L1 = 0
PR_NORM_LINF = 2
PR_USE_REDUCTIONS = 4
PR_TIMING = 8
PR_MODE_NOSYNC = 16
PR_PERFORATE = 32
PR_MODE_PHASED = 64
PR_CHAIN_EAGER = 128

# every symbol include/prgpu.h declares (tests check the .so exports them)
ABI_SYMBOLS = (
    "pr_graph_create", "pr_preprocess", "pr_run", "pr_destroy", "pr_release_memory", "pr_last_error",
    "pr_graph_info", "pr_get_csr", "pr_get_reductions", "pr_get_delta_log", "pr_get_run_stats",
    "pr_graph_shard", "pr_graph_create_sharded", "pr_run_sharded", "pr_get_shard_info", "pr_get_phase_plan",
    "pr_shard_buffers", "pr_shard_set_peers", "pr_shard_device_barrier", "pr_selftest_peer_barrier",
    "pr_shard_mc_create", "pr_shard_mc_attach", "pr_shard_mc_bind", "pr_shard_export_ipc", "pr_shard_open_ipc",
)


class PRError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libprgpu error {code}: {msg}")
        self.code = code


class pr_run_stats(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("status", ctypes.c_int32),
        ("delta_l1", ctypes.c_double),
        ("delta_linf", ctypes.c_double),
        ("run_launches", ctypes.c_int64),
        ("total_launches", ctypes.c_int64),
        ("host_syncs", ctypes.c_int32),
        ("timed_iterations", ctypes.c_int32),
        ("gather_ms", ctypes.c_double),
        ("scatter_ms", ctypes.c_double),
        ("gather_rows", ctypes.c_int64),
        ("gather_edges", ctypes.c_int64),
        ("scatter_members", ctypes.c_int64),
        ("n_contrib", ctypes.c_int64),
        ("n_tasks", ctypes.c_int64),
        ("nosync_min_iters", ctypes.c_int32),
        ("nosync_launches", ctypes.c_int32),
        ("nosync_median_iters", ctypes.c_int32),
        ("residual", ctypes.c_double),
        ("edges_gathered", ctypes.c_int64),
        ("frozen_rows", ctypes.c_int64),
        ("compactions", ctypes.c_int32),
        ("phases", ctypes.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class pr_shard_info(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("owned_vertices", ctypes.c_int64),
        ("rows", ctypes.c_int64),
        ("edges", ctypes.c_int64),
        ("chunk", ctypes.c_int64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# int (*pr_exchange_fn)(void *ctx, double *buf, int64_t chunk, int32_t world, void *stream)
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                               ctypes.c_void_p)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                ctypes.c_void_p)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libprgpu.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    i64, i32, u32, dbl, p = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_double, ctypes.c_void_p
    pp = ctypes.POINTER(ctypes.c_void_p)
    lib.pr_graph_create.argtypes = [i64, i64, p, p, p, pp]
    lib.pr_graph_create.restype = ctypes.c_int
    lib.pr_preprocess.argtypes = [p, u32, p]
    lib.pr_preprocess.restype = ctypes.c_int
    lib.pr_run.argtypes = [p, dbl, dbl, i32, p, u32, p, ctypes.POINTER(i32), ctypes.POINTER(dbl)]
    lib.pr_run.restype = ctypes.c_int
    lib.pr_destroy.argtypes = [p]
    lib.pr_destroy.restype = None
    lib.pr_release_memory.argtypes = []
    lib.pr_release_memory.restype = ctypes.c_int
    lib.pr_last_error.argtypes = []
    lib.pr_last_error.restype = ctypes.c_char_p
    lib.pr_graph_info.argtypes = [p, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i32)]
    lib.pr_graph_info.restype = ctypes.c_int
    lib.pr_get_csr.argtypes = [p, p, p, p, p]
    lib.pr_get_csr.restype = ctypes.c_int
    lib.pr_get_reductions.argtypes = [p, p, p, p, p]
    lib.pr_get_reductions.restype = ctypes.c_int
    lib.pr_get_delta_log.argtypes = [p, p, i32]
    lib.pr_get_delta_log.restype = ctypes.c_int
    lib.pr_get_run_stats.argtypes = [p, ctypes.POINTER(pr_run_stats)]
    lib.pr_get_run_stats.restype = ctypes.c_int
    lib.pr_graph_shard.argtypes = [p, i32, i32, p]
    lib.pr_graph_shard.restype = ctypes.c_int
    lib.pr_shard_mc_create.argtypes = [p, p]
    lib.pr_shard_mc_create.restype = ctypes.c_int
    lib.pr_shard_mc_attach.argtypes = [p, p]
    lib.pr_shard_mc_attach.restype = ctypes.c_int
    lib.pr_shard_mc_bind.argtypes = [p, p]
    lib.pr_shard_mc_bind.restype = ctypes.c_int
    lib.pr_shard_device_barrier.argtypes = [p, i32]
    lib.pr_shard_device_barrier.restype = ctypes.c_int
    lib.pr_selftest_peer_barrier.argtypes = [i32, i32, p]
    lib.pr_selftest_peer_barrier.restype = ctypes.c_int
    lib.pr_graph_create_sharded.argtypes = [i64, i64, p, p, i32, i32, ALLREDUCE_FN, p, p, pp]
    lib.pr_graph_create_sharded.restype = ctypes.c_int
    lib.pr_run_sharded.argtypes = [p, dbl, dbl, i32, p, u32, p, EXCHANGE_FN, p, ctypes.POINTER(i32),
                                   ctypes.POINTER(dbl)]
    lib.pr_run_sharded.restype = ctypes.c_int
    lib.pr_get_shard_info.argtypes = [p, ctypes.POINTER(pr_shard_info)]
    lib.pr_get_shard_info.restype = ctypes.c_int
    lib.pr_get_phase_plan.argtypes = [p, i32, p, p, i32]
    lib.pr_get_phase_plan.restype = ctypes.c_int
    lib.pr_shard_buffers.argtypes = [p, pp, pp, ctypes.POINTER(i64)]
    lib.pr_shard_buffers.restype = ctypes.c_int
    lib.pr_shard_set_peers.argtypes = [p, pp, pp, i32]
    lib.pr_shard_set_peers.restype = ctypes.c_int
    lib.pr_shard_export_ipc.argtypes = [p, p]
    lib.pr_shard_export_ipc.restype = ctypes.c_int
    lib.pr_shard_open_ipc.argtypes = [p, p, i32]
    lib.pr_shard_open_ipc.restype = ctypes.c_int
    return lib


lib = _load()


def _ptr(a) -> int | None:
    """Address of a torch tensor / numpy array (contiguous), or None."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    if hasattr(a, "ctypes"):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    raise TypeError(type(a))


def _numel(a) -> int:
    if hasattr(a, "numel"):
        return int(a.numel())
    return int(a.size)


def _out(a, dtype: str, need: int, what: str):
    """Address of a caller-owned output buffer the library writes `need`
    elements of `dtype` into: checked for dtype, contiguity and length (a
    float32 or short buffer would be a silent out-of-bounds write)."""
    if a is None:
        return None
    dt = str(getattr(a, "dtype", ""))
    if not dt.endswith(dtype):
        raise TypeError(f"{what} must be {dtype}, got {dt}")
    if _numel(a) < need:
        raise ValueError(f"{what} holds {_numel(a)} elements, needs {need}")
    return _ptr(a)


def _stream(stream) -> int | None:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def last_error() -> str:
    return (lib.pr_last_error() or b"").decode()


def _check(rc: int, ok=(PR_OK,)):
    if rc not in ok:
        raise PRError(rc, last_error())
    return rc


def pr_graph_create(n: int, src, dst, stream=None) -> ctypes.c_void_p:
    """In-CSR + out-degrees on the device.  src/dst int32[m]."""
    m = int(src.shape[0])
    if int(dst.shape[0]) != m:
        raise ValueError("src and dst lengths differ")
    for a in (src, dst):
        dt = str(getattr(a, "dtype", ""))
        if "int32" not in dt:
            raise TypeError(f"edge arrays must be int32, got {dt}")
    out = ctypes.c_void_p()
    _check(lib.pr_graph_create(n, m, _ptr(src) if m else None, _ptr(dst) if m else None,
                               _stream(stream), ctypes.byref(out)))
    return out


def pr_preprocess(g, flags: int = PR_PRE_IDENTICAL | PR_PRE_CHAIN, stream=None) -> None:
    _check(lib.pr_preprocess(g, flags, _stream(stream)))


def pr_run(g, d: float, threshold: float, max_iter: int, ranks, stream=None, mode: int = 0):
    """Iterate to convergence; returns (status, iterations, final_delta)."""
    it = ctypes.c_int32(0)
    fd = ctypes.c_double(0.0)
    rptr = _out(ranks, "float64", pr_graph_info(g)["n"], "ranks")
    rc = _check(lib.pr_run(g, d, threshold, max_iter, _stream(stream), mode, rptr,
                           ctypes.byref(it), ctypes.byref(fd)), ok=(PR_OK, PR_NOT_CONVERGED))
    return rc, it.value, fd.value


def pr_destroy(g) -> None:
    lib.pr_destroy(g)


def pr_graph_info(g):
    n, E, nm = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    mc = ctypes.c_int32()
    _check(lib.pr_graph_info(g, ctypes.byref(n), ctypes.byref(E), ctypes.byref(nm), ctypes.byref(mc)))
    return {"n": n.value, "E": E.value, "n_members": nm.value, "max_chain": mc.value}


def pr_get_csr(g, row_ptr, col_idx, outdeg, stream=None) -> None:
    inf = pr_graph_info(g)
    _check(lib.pr_get_csr(g, _out(row_ptr, "int64", inf["n"] + 1, "row_ptr"), _out(col_idx, "int32", inf["E"], "col_idx"),
                          _out(outdeg, "int32", inf["n"], "outdeg"), _stream(stream)))


def pr_get_reductions(g, rep, chain_src, chain_k, stream=None) -> None:
    n = pr_graph_info(g)["n"]
    _check(lib.pr_get_reductions(g, _out(rep, "int32", n, "rep"), _out(chain_src, "int32", n, "chain_src"),
                                 _out(chain_k, "int32", n, "chain_k"), _stream(stream)))


def pr_release_memory() -> None:
    """Return the library pool's unused device memory to the device."""
    _check(lib.pr_release_memory())


def pr_get_delta_log(g, cap: int):
    import numpy as np
    buf = np.zeros((max(cap, 1), 2), np.float64)
    k = lib.pr_get_delta_log(g, buf.ctypes.data, cap)
    if k < 0:
        raise PRError(-k if k == -PR_EINVAL else k, last_error())
    return buf[:k]


def pr_get_run_stats(g) -> dict:
    st = pr_run_stats()
    _check(lib.pr_get_run_stats(g, ctypes.byref(st)))
    return st.as_dict()


def pr_get_phase_plan(g, reduced: bool = False):
    """(edge_bounds, row_bounds) of the last PR_MODE_PHASED run on that view."""
    import numpy as np
    eb = np.zeros(65, np.int64)
    rb = np.zeros(65, np.int64)
    k = lib.pr_get_phase_plan(g, 1 if reduced else 0, eb.ctypes.data, rb.ctypes.data, 65)
    if k < 0:
        raise PRError(-k if k in (-PR_EINVAL, -PR_ESTATE) else k, last_error())
    return eb[:k + 1].copy(), rb[:k + 1].copy()


def pr_graph_shard(g, rank: int, world: int, stream=None) -> None:
    """Make g this rank's share of a world-rank row partition."""
    _check(lib.pr_graph_shard(g, rank, world, _stream(stream)))


def pr_get_shard_info(g) -> dict:
    info = pr_shard_info()
    _check(lib.pr_get_shard_info(g, ctypes.byref(info)))
    return info.as_dict()


def device_f64(ptr: int, count: int):
    """A torch view (no copy) of `count` doubles of device memory at `ptr`."""
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                    "version": 2, "strides": None}
    return torch.as_tensor(_CAI(), device="cuda")


def pr_shard_buffers(g):
    """(y0_ptr, y1_ptr, length in doubles) of this rank's contrib buffers."""
    a, b, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    _check(lib.pr_shard_buffers(g, ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)))
    return a.value, b.value, n.value


def pr_shard_set_peers(g, y0s, y1s) -> None:
    """Peer buffers (lists of world device pointers; this rank's entry unused);
    None: back to the all-gather exchange."""
    if y0s is None:
        _check(lib.pr_shard_set_peers(g, None, None, 0))
        return
    w = len(y0s)
    A = (ctypes.c_void_p * w)(*[v or 0 for v in y0s])
    B = (ctypes.c_void_p * w)(*[v or 0 for v in y1s])
    _check(lib.pr_shard_set_peers(g, A, B, w))


def pr_shard_mc_create(g) -> bytes:
    buf = ctypes.create_string_buffer(64)
    _check(lib.pr_shard_mc_create(g, buf))
    return buf.raw


def pr_shard_mc_attach(g, handle) -> None:
    _check(lib.pr_shard_mc_attach(g, handle))


def pr_shard_mc_bind(g, stream=None) -> None:
    _check(lib.pr_shard_mc_bind(g, _stream(stream)))


def shard_multicast_local(g) -> None:
    """The NVLS team of a world-1 shard (create + attach + bind in one process)."""
    _check(lib.pr_shard_mc_create(g, None))
    _check(lib.pr_shard_mc_attach(g, None))
    pr_shard_mc_bind(g)


def torch_dist_multicast_setup(g, group=None) -> None:
    """The NVLS team over torch.distributed: rank 0 creates and shares the
    fabric handle, every rank attaches, then (after all attached) binds."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    h = pr_shard_mc_create(g) if rank == 0 else None
    allh = [None]
    if rank == 0:
        allh = [h]
    dist.broadcast_object_list(allh, src=0, group=group)
    pr_shard_mc_attach(g, None if rank == 0 else allh[0])
    dist.barrier(group=group)
    pr_shard_mc_bind(g)
    dist.barrier(group=group)


def pr_shard_device_barrier(g, on: bool = True) -> None:
    """Per-sweep synchronisation of the peer-store exchange on the device."""
    _check(lib.pr_shard_device_barrier(g, 1 if on else 0))


def pr_selftest_peer_barrier(world: int, epochs: int = 64, stream=None) -> None:
    """The device barrier's protocol on emulated ranks (one cooperative launch)."""
    _check(lib.pr_selftest_peer_barrier(world, epochs, _stream(stream)))


def pr_shard_export_ipc(g) -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.pr_shard_export_ipc(g, buf))
    return buf.raw


def pr_shard_open_ipc(g, handles) -> None:
    """handles: the world ranks' pr_shard_export_ipc bytes, in rank order."""
    blob = b"".join(handles)
    _check(lib.pr_shard_open_ipc(g, blob, len(handles)))


def torch_dist_peer_setup(g, group=None) -> None:
    """Exchange this rank's buffer IPC handles over torch.distributed and open
    the peers' (the fused peer-store exchange, one process per GPU)."""
    import torch.distributed as dist
    mine = pr_shard_export_ipc(g)
    allh = [None] * dist.get_world_size(group)
    dist.all_gather_object(allh, mine, group=group)
    pr_shard_open_ipc(g, allh)


def device_i32(ptr: int, count: int):
    """A torch view (no copy) of `count` int32 of device memory at `ptr`."""
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (int(count),), "typestr": "<i4", "data": (int(ptr), False),
                                    "version": 2, "strides": None}
    return torch.as_tensor(_CAI(), device="cuda")


def pr_graph_create_sharded(n: int, src, dst, rank: int, world: int, allreduce, stream=None) -> ctypes.c_void_p:
    """This rank's share of a world-rank row partition, ingesting only the
    edges into its vertices (v mod world == rank); `allreduce(buf_ptr, count,
    world, stream_ptr)` sums `count` int32 in place over the ranks."""
    m = int(src.shape[0])
    if int(dst.shape[0]) != m:
        raise ValueError("src and dst lengths differ")
    for a in (src, dst):
        dt = str(getattr(a, "dtype", ""))
        if "int32" not in dt:
            raise TypeError(f"edge arrays must be int32, got {dt}")
    err = []

    def _cb(ctx, buf, count, world_, strm):
        try:
            allreduce(buf, count, world_, strm)
            return 0
        except BaseException as e:  # reported after the call returns
            err.append(e)
            return 1
    cb = ALLREDUCE_FN(_cb)
    out = ctypes.c_void_p()
    rc = lib.pr_graph_create_sharded(n, m, _ptr(src) if m else None, _ptr(dst) if m else None, rank, world, cb,
                                     None, _stream(stream), ctypes.byref(out))
    if err:
        raise err[0]
    _check(rc)
    return out


def torch_dist_allreduce(group=None):
    """The out-degree all-reduce of pr_graph_create_sharded through
    torch.distributed (NCCL, or gloo through a host copy)."""
    import torch
    import torch.distributed as dist

    nccl = dist.get_backend(group) == "nccl"

    def allreduce(buf: int, count: int, world: int, stream: int):
        t = device_i32(buf, count)
        s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()
        with torch.cuda.stream(s):
            if nccl:
                dist.all_reduce(t, group=group)
            else:
                s.synchronize()
                h = t.cpu()
                dist.all_reduce(h, group=group)
                t.copy_(h)
                torch.cuda.synchronize()
    return allreduce


def torch_dist_exchange(group=None):
    """The per-sweep exchange of pr_run_sharded through torch.distributed
    (NCCL over NVLink on a GPU node): an in-place all_gather_into_tensor of the
    world chunks, ordered on the library's stream."""
    import torch
    import torch.distributed as dist

    nccl = dist.get_backend(group) == "nccl"

    def exchange(buf: int, chunk: int, world: int, stream: int):
        if buf is None:  # peer buffers: the kernels already stored everything; only synchronise
            (torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()).synchronize()
            dist.barrier(group=group)
            return
        full = device_f64(buf, chunk * world)
        rank = dist.get_rank(group)
        # stream 0 (ctypes passes it as None) is the legacy default stream
        s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()
        with torch.cuda.stream(s):
            if nccl:
                dist.all_gather_into_tensor(full, full[rank * chunk:(rank + 1) * chunk], group=group)
            else:  # gloo (multi-process tests on one GPU): list all-gather, host-synchronous
                s.synchronize()
                parts = list(full.view(world, chunk).unbind(0))
                dist.all_gather(parts, parts[rank].clone(), group=group)
                torch.cuda.synchronize()
    return exchange


def pr_run_sharded(g, d: float, threshold: float, max_iter: int, ranks, exchange, stream=None, mode: int = 0):
    """The sharded sync iteration; `exchange(buf_ptr, chunk, world, stream_ptr)`
    all-gathers the chunks in place.  Returns (status, iterations, final_delta);
    ranks (device fp64[n]) holds the owned vertices' ranks, 0.0 elsewhere."""
    err = []

    def _cb(ctx, buf, chunk, world, strm):
        try:
            exchange(buf, chunk, world, strm)
            return 0
        except BaseException as e:  # reported after the call returns
            err.append(e)
            return 1
    cb = EXCHANGE_FN(_cb)
    it = ctypes.c_int32(0)
    fd = ctypes.c_double(0.0)
    rptr = _out(ranks, "float64", pr_graph_info(g)["n"], "ranks")
    rc = lib.pr_run_sharded(g, d, threshold, max_iter, _stream(stream), mode, rptr, cb, None,
                            ctypes.byref(it), ctypes.byref(fd))
    if err:
        raise err[0]
    _check(rc, ok=(PR_OK, PR_NOT_CONVERGED))
    return rc, it.value, fd.value


class Graph:
    """RAII convenience wrapper around one pr_graph (still only marshalling)."""

    def __init__(self, n: int, src, dst, stream=None, handle=None):
        self.n = n
        self.handle = handle if handle is not None else pr_graph_create(n, src, dst, stream)

    @classmethod
    def sharded(cls, n: int, src, dst, rank: int, world: int, allreduce, stream=None):
        """pr_graph_create_sharded: only this rank's rows are ingested."""
        return cls(n, None, None, handle=pr_graph_create_sharded(n, src, dst, rank, world, allreduce, stream))

    def preprocess(self, flags: int = PR_PRE_IDENTICAL | PR_PRE_CHAIN, stream=None):
        pr_preprocess(self.handle, flags, stream)
        return self

    def run(self, ranks, d=0.85, threshold=1e-10, max_iter=1000, mode=0, stream=None):
        return pr_run(self.handle, d, threshold, max_iter, ranks, stream, mode)

    def shard(self, rank: int, world: int, stream=None):
        pr_graph_shard(self.handle, rank, world, stream)
        return self

    def shard_info(self):
        return pr_get_shard_info(self.handle)

    def shard_buffers(self):
        return pr_shard_buffers(self.handle)

    def set_peers(self, y0s, y1s=None):
        pr_shard_set_peers(self.handle, y0s, y1s)

    def run_sharded(self, ranks, exchange, d=0.85, threshold=1e-10, max_iter=1000, mode=0, stream=None):
        return pr_run_sharded(self.handle, d, threshold, max_iter, ranks, exchange, stream, mode)

    def info(self):
        return pr_graph_info(self.handle)

    def stats(self):
        return pr_get_run_stats(self.handle)

    def delta_log(self, cap=4096):
        return pr_get_delta_log(self.handle, cap)

    def close(self):
        if self.handle is not None:
            pr_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
