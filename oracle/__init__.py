"""CPU fp64 oracle for the PageRank pull iteration (arXiv 2109.09527).

TEST INFRASTRUCTURE ONLY -- imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` leg, never by the
product package.  It shares no code with ``paper_2109_09527_b200``.

Thin ctypes wrapper over ``oracle/oracle.c`` (plain single-threaded C, built
with ``-O2 -ffp-contract=off``).  Each function cites the passage it follows
in ``oracle.c``; the pins live in ``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

NORM_LINF = 1
REDUCED = 2
GAUSS_SEIDEL = 4


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                               "-std=gnu11", "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, i32, dbl, p = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p
        lib.or_build_csr.argtypes = [i64, i64, p, p, p, p, p]
        lib.or_build_csr.restype = i64
        lib.or_identical.argtypes = [i64, p, p, p]
        lib.or_identical.restype = ctypes.c_int
        lib.or_chains.argtypes = [i64, p, p, p, p, p, p]
        lib.or_chains.restype = ctypes.c_int
        lib.or_jacobi_step.argtypes = [i64, p, p, p, dbl, p, p]
        lib.or_jacobi_step.restype = None
        lib.or_pagerank.argtypes = [i64, p, p, p, dbl, dbl, i32, i32, p, p, p, p, p, p]
        lib.or_pagerank.restype = ctypes.c_int
        lib.or_residual_l1.argtypes = [i64, p, p, p, dbl, p, p]
        lib.or_residual_l1.restype = dbl
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


@dataclass
class CSR:
    n: int
    row_ptr: np.ndarray   # int64[n+1]
    col_idx: np.ndarray   # int32[E]
    outdeg: np.ndarray    # int32[n]

    @property
    def E(self) -> int:
        return int(self.row_ptr[-1])


def build_csr(n: int, src: np.ndarray, dst: np.ndarray) -> CSR:
    """In-CSR after removing loops and duplicates."""
    src = np.ascontiguousarray(src, np.int32)
    dst = np.ascontiguousarray(dst, np.int32)
    m = int(src.shape[0])
    rp = np.empty(n + 1, np.int64)
    col = np.empty(max(m, 1), np.int32)
    od = np.empty(n, np.int32)
    E = _load().or_build_csr(n, m, _p(src), _p(dst), _p(rp), _p(col), _p(od))
    if E == -1:
        raise ValueError("vertex id out of range")
    if E < 0:
        raise MemoryError("or_build_csr")
    return CSR(n, rp, col[:E], od)


def identical(g: CSR) -> np.ndarray:
    """rep[v] = min id of v's equal-in-set class."""
    rep = np.empty(g.n, np.int32)
    if _load().or_identical(g.n, _p(g.row_ptr), _p(g.col_idx), _p(rep)) != 0:
        raise MemoryError
    return rep


def chains(g: CSR, rep: np.ndarray):
    """(chain_src, chain_k, max_k) under reading Q-C of P:398."""
    cs = np.empty(g.n, np.int32)
    ck = np.empty(g.n, np.int32)
    mk = _load().or_chains(g.n, _p(g.row_ptr), _p(g.col_idx), _p(g.outdeg), _p(rep), _p(cs), _p(ck))
    if mk < 0:
        raise MemoryError
    return cs, ck, int(mk)


def jacobi_step(g: CSR, d: float, x: np.ndarray) -> np.ndarray:
    out = np.empty(g.n, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    _load().or_jacobi_step(g.n, _p(g.row_ptr), _p(g.col_idx), _p(g.outdeg), d, _p(x), _p(out))
    return out


@dataclass
class Result:
    x: np.ndarray
    iters: int
    status: int
    delta: float
    delta_log: np.ndarray   # (iters, 2): L1, Linf
    seconds: float


def pagerank(g: CSR, d: float = 0.85, tau: float = 1e-10, max_iter: int = 1000, *,
             norm_linf: bool = False, reduced: bool = False, gauss_seidel: bool = False,
             rep: np.ndarray | None = None, chain_k: np.ndarray | None = None) -> Result:
    """Eq.(1) power iteration (Alg.1); see oracle.c."""
    mode = (NORM_LINF if norm_linf else 0) | (REDUCED if reduced else 0) | \
        (GAUSS_SEIDEL if gauss_seidel else 0)
    x = np.empty(g.n, np.float64)
    log = np.zeros((max_iter, 2), np.float64)
    it = ctypes.c_int32(0)
    dl = ctypes.c_double(0.0)
    t0 = time.perf_counter()
    st = _load().or_pagerank(g.n, _p(g.row_ptr), _p(g.col_idx), _p(g.outdeg), d, tau, max_iter,
                             mode, _p(rep), _p(chain_k), _p(x), _p(log),
                             ctypes.byref(it), ctypes.byref(dl))
    sec = time.perf_counter() - t0
    if st not in (0, 2):
        raise ValueError(f"or_pagerank status {st}")
    return Result(x, it.value, st, dl.value, log[: it.value].copy(), sec)


def residual_l1(g: CSR, d: float, x: np.ndarray, want_r: bool = False):
    """||x - (c1 + dMx)||_1; ||x - x*||_1 <= this / (1-d)."""
    x = np.ascontiguousarray(x, np.float64)
    r = np.empty(g.n, np.float64) if want_r else None
    v = _load().or_residual_l1(g.n, _p(g.row_ptr), _p(g.col_idx), _p(g.outdeg), d, _p(x), _p(r))
    return (v, r) if want_r else v


def phased_sweeps(g: CSR, d: float, sweeps: int, rows: np.ndarray, edge_bounds, row_bounds):
    """In-place sweeps in a fixed block order -- reading Q-B of
    No-Sync's in-place update (Alg.3: "pr(u) <- tmp" is visible to
    every later read), with Eq.(1) per vertex.  Test model of
    PR_MODE_PHASED, written from that reading, not from the kernels:
      * `rows` are the vertices of the view in order; the view's edge stream
        is each row's in-edges in CSR order, one row after the other;
      * a sweep runs phases k = 0..K-1 in order: phase k adds y(u) =
        x(u)/outdeg(u), AS IT STANDS WHEN THE PHASE STARTS, for the stream
        edges [edge_bounds[k], edge_bounds[k+1]) to their rows' sums, then
        sets x(v) = (1-d)/n + d * S(v) for the rows [row_bounds[k],
        row_bounds[k+1]) (a row crossing a phase boundary keeps the sums of
        both phases);
      * vertices of in-degree 0 take x = (1-d)/n at the end of sweep 1
        (after every gather of that sweep; constant afterwards, Q-Z).
    Returns (x, delta_log[(sweeps, 2)] of (L1, Linf) per sweep)."""
    n = g.n
    c = (1.0 - d) / n
    rows = np.asarray(rows, np.int64)
    od = g.outdeg.astype(np.float64)
    x = np.full(n, 1.0 / n)
    y = np.where(g.outdeg > 0, x / np.where(g.outdeg > 0, od, 1.0), 0.0)
    deg = (g.row_ptr[rows + 1] - g.row_ptr[rows]).astype(np.int64)
    src = (np.concatenate([g.col_idx[g.row_ptr[v]:g.row_ptr[v + 1]] for v in rows]) if len(rows)
           else np.zeros(0, np.int32)).astype(np.int64)
    row_of_edge = np.repeat(np.arange(len(rows)), deg)
    zero = np.nonzero(np.diff(g.row_ptr) == 0)[0]
    K = len(edge_bounds) - 1
    log = np.zeros((sweeps, 2))
    for t in range(sweeps):
        xold = x.copy()
        S = np.zeros(len(rows))
        for k in range(K):
            e0, e1 = int(edge_bounds[k]), int(edge_bounds[k + 1])
            for e in range(e0, e1):                 # sequential: CSR order within each row
                S[row_of_edge[e]] += y[src[e]]
            r0, r1 = int(row_bounds[k]), int(row_bounds[k + 1])
            for i in range(r0, r1):
                v = rows[i]
                x[v] = c + d * S[i]
                if g.outdeg[v] > 0:
                    y[v] = x[v] / od[v]
        if t == 0:
            for v in zero:
                x[v] = c
                if g.outdeg[v] > 0:
                    y[v] = c / od[v]
        diff = np.abs(x - xold)
        log[t] = (diff.sum(), diff.max())
    return x, log
